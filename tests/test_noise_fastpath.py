"""Partial noise (ucp/parallel.py:340-370) as the kernels compute it.

* The branch-free integer form the OPS kernels run (ucp_noise_bits in
  csrc/ucp_noise.h, compiled here by g++ from the same header) against a C
  restatement of the reference (nextafterf stepping + the f64 pair test):
  dense over the zero / subnormal / first-normal range and the top binade of
  both signs, strided over the rest, for every step count up to 8 (every rank
  of tp <= 16). tools/noise_exhaustive.cpp run without a stride covers all
  2^32 patterns (profiles/noise_exhaustive_r02.log: 68.7 G cases, 0
  mismatches).
* A numpy model of the previous fast path (UCP_NOISE_INT=0: `steps` nextafter
  steps as +-steps on the bit pattern when they cross neither zero nor +-inf,
  the nextafter loop otherwise) against the oracle restatement, on every
  exponent's edge mantissas, the neighbourhoods of zero and of the largest
  finite value, and random bit patterns, for every rank of tp up to 16.

The GPU kernel itself is checked against the reference's own tables and the
same edges in tests/test_gpu_parity.py."""

import json
import os
import shutil
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

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


@pytest.fixture(scope="module")
def noise_ex(tmp_path_factory):
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    exe = str(tmp_path_factory.mktemp("noise") / "noise_ex")
    subprocess.run(["g++", "-O2", "-fopenmp", "-std=c++17",
                    os.path.join(ROOT, "tools", "noise_exhaustive.cpp"), "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("rng", [
    (1, 0, 1 << 25),                        # +0, subnormals, first two normal binades
    (1, 0x7E800000, 0x80000000 + (1 << 25)),  # top binades, inf, NaN, -0, negative subnormals
    (1, 0xFE800000, 1 << 32),               # negative top binades, -inf, negative NaN
    (65521, 0, 1 << 32),                    # every region, strided
])
def test_integer_noise_matches_reference_restatement(noise_ex, rng):
    stride, lo, hi = rng
    out = subprocess.run([noise_ex, "8", str(stride), str(lo), str(hi)], capture_output=True,
                         text=True, timeout=300)
    res = json.loads(out.stdout)
    assert out.returncode == 0 and res["mismatches"] == 0, res
    assert res["checked"] > 0
