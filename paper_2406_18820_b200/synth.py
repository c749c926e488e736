"""Synthetic inputs: the deterministic generator's host half.

Element i of a stream is splitmix64(base + i) reduced to 24 bits
(ucp/tensor.py:116-184); ``stream_base`` (FNV-1a of ``name\\x1ftag`` mixed
with the seed) is computed here on the host, the elements by
``ucp_gen_state`` on the GPU.
"""

from __future__ import annotations

_M = (1 << 64) - 1


def _fnv1a(data: bytes) -> int:
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & _M
    return h


def _finalise(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M
    return z ^ (z >> 31)


def stream_base(seed: int, name: str, tag: str) -> int:
    return _finalise((seed & _M) ^ _fnv1a(f"{name}\x1f{tag}".encode("utf-8")))
