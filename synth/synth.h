/* synth.h — seeded, counter-based synthetic column generators.
 *
 * This module is INPUT GENERATION ONLY. It holds none of the method's
 * arithmetic (no packing, no formats, no operators). It is the one piece of
 * code that both sides of the parity contract use: the CPU oracle (oracle/)
 * reads columns from synth_fill_host(), the GPU path's tests and bench.py
 * fill device buffers with synth_fill_device(). Both produce bit-identical
 * values because the generator is counter-based: value i depends only on
 * (recipe, i), never on how the rows are split across threads or ranks.
 *
 * Definitions (the PRNG family follows SPEC.md S:518,
 * "splitmix-style"):
 *   gamma    = 0x9E3779B97F4A7C15
 *   mix64(z) : z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
 *              z *= 0x94D049BB133111EB; z ^= z>>31
 *   R(s, i)  = mix64(s + (i+1)*gamma)      (i-th output of splitmix64(s))
 *   seed(0)  = 42, seed(c) = mix64(42 + c) for c >= 1
 *   U(x, m)  = floor(x * m / 2^64)          (exact 128-bit product)
 *
 * Recipes (one struct describes every column of the five BASELINE.json
 * configs and of the paper's Table `tab:datach` columns C1..C4,
 * PAPER.md P:537-561):
 *   SYN_MASK    v = (R(seed,i) & mask) + add
 *   SYN_RANGE   v = U(R(seed,i), m) + add
 *   SYN_OUTLIER o = U(R(seed,i), m) == 0; r = R(seed2,i);
 *               v = o ? (outlier_const ? mask2 : (r & mask2)) : (r & mask)
 *   SYN_RUNS    r = R(seed,i); inc_0 = 0; for i >= 1:
 *               inc_i = ((r & 63) == 0) ? 1 + ((r >> 6) & 15) : 0;
 *               v_i = add + sum_{k<=i} inc_k   (non-decreasing; runs of
 *               geometric length, mean 64, steps uniform in [1,16])
 *   skew != 0   v = (U(R(skew_seed,i), skew_m) != 0) ? skew_low : base value
 *               (the select micro-benchmark's 90% "lowest value" skew,
 *               PAPER.md P:569-570)
 */
#ifndef SYNTH_H
#define SYNTH_H
#include <stdint.h>

#ifdef __CUDACC__
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum { SYN_MASK = 0, SYN_RANGE = 1, SYN_OUTLIER = 2, SYN_RUNS = 3 };

typedef struct {
  uint32_t kind;
  uint32_t skew;
  uint64_t seed, seed2;
  uint64_t mask, mask2;
  uint64_t m;
  uint64_t add;
  uint64_t outlier_const;
  uint64_t skew_seed, skew_low, skew_m;
} synth_recipe;

#define SYNTH_GAMMA 0x9E3779B97F4A7C15ull

SYNTH_HD uint64_t synth_mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
SYNTH_HD uint64_t synth_R(uint64_t s, uint64_t i) { return synth_mix64(s + (i + 1) * SYNTH_GAMMA); }
SYNTH_HD uint64_t synth_seed(uint64_t c) { return c == 0 ? 42ull : synth_mix64(42ull + c); }
SYNTH_HD uint64_t synth_U(uint64_t x, uint64_t m) {
#ifdef __CUDA_ARCH__
  return __umul64hi(x, m);
#else
  return (uint64_t)(((unsigned __int128)x * m) >> 64);
#endif
}
/* increment of SYN_RUNS at row i (row 0 has none) */
SYNTH_HD uint64_t synth_run_inc(uint64_t seed, uint64_t i) {
  if (i == 0) return 0;
  uint64_t r = synth_R(seed, i);
  return ((r & 63) == 0) ? 1 + ((r >> 6) & 15) : 0;
}
/* value of a non-RUNS recipe at row i */
SYNTH_HD uint64_t synth_value(const synth_recipe *p, uint64_t i) {
  uint64_t v;
  if (p->kind == SYN_MASK) {
    v = (synth_R(p->seed, i) & p->mask) + p->add;
  } else if (p->kind == SYN_RANGE) {
    v = synth_U(synth_R(p->seed, i), p->m) + p->add;
  } else { /* SYN_OUTLIER */
    int o = synth_U(synth_R(p->seed, i), p->m) == 0;
    uint64_t r = synth_R(p->seed2, i);
    v = o ? (p->outlier_const ? p->mask2 : (r & p->mask2)) : (r & p->mask);
  }
  if (p->skew && synth_U(synth_R(p->skew_seed, i), p->skew_m) != 0) v = p->skew_low;
  return v;
}

/* Host: fill out[0..n) with rows [start, start+n) of the recipe. */
void synth_fill_host(const synth_recipe *p, uint64_t start, uint64_t n, uint64_t *out);
/* Device (libsynth_dev.so): same rows into device buffer out, on stream.
 * Returns 0 on success, a cudaError_t value otherwise. */
int synth_fill_device(const synth_recipe *p, uint64_t start, uint64_t n, uint64_t *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif
