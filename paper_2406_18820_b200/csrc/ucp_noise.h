// partial_noise on f32 bit patterns, branch-free (ucp/parallel.py:340-370).
//
// Shared by the OPS kernels in ucp_b200.cu and the host-side exhaustive check
// (tools/noise_exhaustive.cpp, tests/test_noise_fastpath.py), so the function
// the GPU runs is the one proven against the reference over all 2^32 inputs.
//
// The reference steps x `s = t/2 + 1` times with nextafter towards +inf (hi)
// and -inf (lo) and keeps hi (even t) or lo (odd t) only where
// f64(hi) + f64(lo) == 2 * f64(x) and x is finite and non-zero. On bit
// patterns, with a = |x|'s magnitude bits:
//   * the step away from zero is the pattern u + s (sign kept), the step
//     towards zero u - s, or -- for a < s, crossing +-0 -- the opposite sign
//     with magnitude s - a (one step per ulp, +-0 counted once);
//   * the f64 sum is exact (both values are f32 within a factor 2, or
//     subnormal), so the test is real equality hi - x == x - lo, i.e. the
//     s ulps above and below x all have one spacing. Spacing is
//     monotone in the magnitude and equal for exponent fields 0 and 1, so
//     the test is: the patterns a - s (0 when crossing) and a + s - 1 have
//     one exponent field, or a + s - 1 < 2^24;
//   * a + s >= 0x7f800000 makes the away step +-inf (or x is inf / NaN): the
//     sum is not 2x and x is kept; a == 0 keeps x (the reference's x != 0).
// Uniform per run: tp <= 1 and the odd trailing rank return x unchanged.

#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define UCP_NOISE_HD __host__ __device__ __forceinline__
#else
#define UCP_NOISE_HD static inline
#endif

#ifndef UCP_NOISE_V2
#define UCP_NOISE_V2 1  // 0: the first integer form (r02za), kept for A/B
#endif

#if UCP_NOISE_V2
// Fewer operations, same function: a - 1 < 0x7f7fffff - s (unsigned) is
// a != 0 && a + s < 0x7f800000 in one compare; a - s may wrap when the steps
// cross zero (a < s), which the m2 < 2^24 clause covers; the kept pattern is
// u -+ s, except towards zero across it: opposite sign, magnitude s - a.
UCP_NOISE_HD uint32_t ucp_noise_bits(uint32_t u, uint32_t s, uint32_t odd) {
  const uint32_t a = u & 0x7fffffffu;
  const uint32_t am1 = a - 1u;
  const uint32_t m2 = am1 + s;
  const bool same = (((a - s) ^ m2) < 0x00800000u) || (m2 < 0x01000000u);
  const bool ok = (am1 < 0x7f7fffffu - s) && same;
  const bool tw = ((u >> 31) ^ odd) != 0u;  // towards zero
  const uint32_t step = tw ? u - s : u + s;
  const uint32_t cross = ((u & 0x80000000u) ^ 0x80000000u) + (s - a);
  const uint32_t chosen = (tw && a < s) ? cross : step;
  return ok ? chosen : u;
}
#else
UCP_NOISE_HD uint32_t ucp_noise_bits(uint32_t u, uint32_t s, uint32_t odd) {
  const uint32_t a = u & 0x7fffffffu;
  const uint32_t sgn = u & 0x80000000u;
  const uint32_t m2 = a + s - 1u;                   // top pattern a step starts from
  const uint32_t m1 = a > s ? a - s : 0u;           // bottom pattern (0 when crossing)
  const bool same = ((m1 ^ m2) < 0x00800000u) || (m2 < 0x01000000u);
  const bool ok = (a != 0u) && (m2 < 0x7f7fffffu) && same;
  const uint32_t away = u + s;
  const uint32_t toward = a >= s ? u - s : ((sgn ^ 0x80000000u) | (s - a));
  // even t keeps hi (towards +inf), odd t keeps lo: for x < 0 hi is the step towards zero
  const bool tw = ((sgn >> 31) ^ odd) != 0u;
  const uint32_t chosen = tw ? toward : away;
  return ok ? chosen : u;
}
#endif

// The per-run constants of ucp_noise_bits: s (steps) and odd, or s = 0 when
// the run leaves every element unchanged.
UCP_NOISE_HD uint32_t ucp_noise_steps(int t, int tp) {
  if (tp <= 1 || ((tp & 1) && t == tp - 1)) return 0u;
  return (uint32_t)(t / 2 + 1);
}
