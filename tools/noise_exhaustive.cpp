// Exhaustive check of ucp_noise_bits (paper_2406_18820_b200/csrc/ucp_noise.h,
// the function the OPS kernels run) against a restatement of the reference's
// partial_noise (ucp/parallel.py:340-370): nextafterf stepping and the f64
// pair test, for every f32 bit pattern in [lo, hi) by `stride` and every
// step count 1..S (both parities, i.e. every rank of tp <= 2S).
//
//   g++ -O2 -fopenmp -std=c++17 tools/noise_exhaustive.cpp -o /tmp/noise_ex
//   /tmp/noise_ex [S=8] [stride=1] [lo=0] [hi=2^32]
//
// Test infrastructure only; prints one JSON line, exit status 1 on any
// mismatch. No -ffast-math: the check relies on IEEE f32/f64.
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2406_18820_b200/csrc/ucp_noise.h"

static inline float f_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static inline uint32_t b_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

int main(int argc, char** argv) {
  const int S = argc > 1 ? atoi(argv[1]) : 8;
  const uint64_t stride = argc > 2 ? strtoull(argv[2], 0, 0) : 1;
  const uint64_t lo = argc > 3 ? strtoull(argv[3], 0, 0) : 0;
  const uint64_t hi = argc > 4 ? strtoull(argv[4], 0, 0) : (1ull << 32);
  uint64_t checked = 0, bad = 0, changed = 0;
  uint32_t first_bad = 0;
  int first_s = 0, first_odd = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : checked, bad, changed)
  for (int64_t blk = 0; blk < 4096; ++blk) {
    const uint64_t b0 = lo + (hi - lo) * (uint64_t)blk / 4096, b1 = lo + (hi - lo) * (uint64_t)(blk + 1) / 4096;
    uint64_t start = b0 + (stride - (b0 - lo) % stride) % stride;
    for (uint64_t v = start; v < b1; v += stride) {
      const uint32_t u = (uint32_t)v;
      const float x = f_of(u);
      float h = x, l = x;
      const bool base_ok = isfinite(x) && x != 0.0f;
      for (int s = 1; s <= S; ++s) {
        h = nextafterf(h, INFINITY);
        l = nextafterf(l, -INFINITY);
        const bool ok = base_ok && ((double)h + (double)l == 2.0 * (double)x);
        for (uint32_t odd = 0; odd < 2; ++odd) {
          const uint32_t want = ok ? b_of(odd ? l : h) : u;
          const uint32_t got = ucp_noise_bits(u, (uint32_t)s, odd);
          ++checked;
          changed += want != u;
          if (got != want) {
            if (!bad) {
#pragma omp critical
              { first_bad = u; first_s = s; first_odd = (int)odd; }
            }
            ++bad;
          }
        }
      }
    }
  }
  printf("{\"steps_max\": %d, \"stride\": %llu, \"lo\": %llu, \"hi\": %llu, \"checked\": %llu, "
         "\"changed\": %llu, \"mismatches\": %llu",
         S, (unsigned long long)stride, (unsigned long long)lo, (unsigned long long)hi,
         (unsigned long long)checked, (unsigned long long)changed, (unsigned long long)bad);
  if (bad) printf(", \"first\": [\"0x%08x\", %d, %d]", first_bad, first_s, first_odd);
  printf("}\n");
  return bad ? 1 : 0;
}
