"""A numpy model of the partial-noise kernel's fast path (noise1 in
csrc/ucp_b200.cu: `steps` nextafter steps done as +-steps on the bit pattern
when they cross neither zero nor +-inf, the reference's nextafter loop
otherwise) against the oracle restatement of ucp/parallel.py:340-370, on every
exponent's edge mantissas, the neighbourhoods of zero and of the largest
finite value, and random bit patterns, for every rank of tp up to 16. The GPU
kernel itself is checked against the reference's own tables and the same
edges in tests/test_gpu_parity.py."""

import numpy as np
import pytest

from oracle import ucp_oracle as O


def _step_up(u):
    mag = u & 0x7FFFFFFF
    out = np.where(u >> 31, u - 1, u + 1).astype(np.uint32)
    out = np.where(mag == 0, np.uint32(1), out)
    return np.where((mag > 0x7F800000) | (u == 0x7F800000), u, out).astype(np.uint32)


def _step_down(u):
    mag = u & 0x7FFFFFFF
    out = np.where(u >> 31, u + 1, u - 1).astype(np.uint32)
    out = np.where(mag == 0, np.uint32(0x80000001), out)
    return np.where((mag > 0x7F800000) | (u == 0xFF800000), u, out).astype(np.uint32)


def _kernel_model(u: np.ndarray, t: int, tp: int) -> np.ndarray:
    if tp <= 1 or (tp % 2 == 1 and t == tp - 1):
        return u
    steps = np.uint32(t // 2 + 1)
    mag = u & np.uint32(0x7FFFFFFF)
    neg = (u >> 31) != 0
    fast = (mag > steps) & (mag.astype(np.uint64) + int(steps) <= 0x7F800000)
    hi = np.where(neg, u - steps, u + steps).astype(np.uint32)
    lo = np.where(neg, u + steps, u - steps).astype(np.uint32)
    h2, l2 = u.copy(), u.copy()
    for _ in range(int(steps)):
        h2, l2 = _step_up(h2), _step_down(l2)
    hi, lo = np.where(fast, hi, h2), np.where(fast, lo, l2)
    f = lambda b: b.view(np.float32).astype(np.float64)  # noqa: E731
    with np.errstate(all="ignore"):
        ok = (f(hi) + f(lo)) == 2.0 * f(u)
    ok &= (mag != 0) & (mag < 0x7F800000)
    return np.where(ok, lo if t & 1 else hi, u).astype(np.uint32)


def _patterns() -> np.ndarray:
    m = np.array([0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 0x7FFFF7, 0x7FFFF8, 0x7FFFF9, 0x7FFFFA, 0x7FFFFB,
                  0x7FFFFC, 0x7FFFFD, 0x7FFFFE, 0x7FFFFF], dtype=np.uint32)
    edges = ((np.arange(256, dtype=np.uint32)[:, None] << 23) | m[None, :]).reshape(-1)
    rand = np.random.default_rng(5).integers(0, 2 ** 32, size=1 << 18, dtype=np.uint64)
    u = np.concatenate([edges, np.arange(0, 64, dtype=np.uint32),
                        np.arange(0x7F7FFFC0, 0x7F800010, dtype=np.uint32), rand.astype(np.uint32)])
    return np.concatenate([u, u | np.uint32(0x80000000)])


@pytest.mark.parametrize("tp", [2, 3, 4, 5, 8, 16])
def test_noise_fast_path_model_matches_oracle(tp):
    u = _patterns()
    x = u.view(np.float32)
    for t in range(tp):
        with np.errstate(all="ignore"):
            want = O.partial_noise(x, t, tp).view(np.uint32)
        assert np.array_equal(_kernel_model(u, t, tp), want), (tp, t)
