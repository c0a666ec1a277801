// morph.cu — direct morphs ("changing the data representation from
// one compressed format to another" without materialising the rows).
//
// RLE -> DELTA_BP{B}: inside a run every delta is 0; at a run start that is not
// the first row of an output block the delta is v_k - v_{k-1} (mod 2^64); the
// block's base is the value of the run covering its first row (D-6, D-9). So the
// output follows from the runs alone:
//   1. per run: the block width w_b = max ebw(step) over the run starts inside
//      block b (atomicMax), the bases of the blocks whose first row the run
//      covers, and the remainder rows it covers (raw values);
//   2. the generic scan of w_b -> cw (D-4);
//   3. per run: its step, ORed into the zeroed payload at bit cw[b]*B + j*w_b
//      (one 64-bit atomicOr per word touched, at most two).
// Work and traffic are proportional to the runs (c3: 8.4 M runs for 2^29 rows),
// not to the rows.
#include "common.cuh"
#include "grid.cuh"
#include "launch.h"

namespace ms {

static uint32_t lg2(uint32_t x) {
  uint32_t l = 0;
  while ((1u << l) < x) ++l;
  return l;
}

__global__ void __launch_bounds__(256) rle2delta_width_kernel(ColView c, uint32_t B, uint32_t log2B, uint64_t nb,
                                                              uint32_t* __restrict__ wk, uint64_t* __restrict__ ref,
                                                              uint64_t* __restrict__ rem) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t main_rows = nb << log2B;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < c.nruns; k += stride) {
    const uint64_t v = __ldg(c.payload + 2 * k);
    // rows [s, e), clamped to the column (a corrupt body is reported by StartsEpi)
    const uint64_t s = __ldg(c.run_starts + k), e = min(__ldg(c.run_starts + k + 1), c.n);
    if (s >= e) continue;
    if (k > 0 && s < main_rows && (s & (B - 1))) {
      const uint64_t d = v - __ldg(c.payload + 2 * (k - 1));
      const uint32_t w = ebw64(d);
      if (w) atomicMax(wk + (s >> log2B), w);
    }
    // bases of the blocks whose first row lies in [s, e)
    for (uint64_t b = (s + B - 1) >> log2B; (b << log2B) < e && b < nb; ++b) ref[b] = v;
    // remainder rows
    for (uint64_t r = s > main_rows ? s : main_rows; r < e; ++r) rem[r - main_rows] = v;
  }
}

__global__ void __launch_bounds__(256) rle2delta_pack_kernel(ColView c, uint32_t B, uint32_t log2B, uint64_t nb,
                                                             const uint64_t* __restrict__ cwx, uint32_t* __restrict__ cw,
                                                             unsigned long long* __restrict__ payload, uint32_t* err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t main_rows = nb << log2B;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < c.nruns; k += stride) {
    const uint64_t s = __ldg(c.run_starts + k);
    if (k == 0 || s >= main_rows || !(s & (B - 1)) || s >= min(__ldg(c.run_starts + k + 1), c.n)) continue;
    const uint64_t b = s >> log2B;
    const uint64_t d = __ldg(c.payload + 2 * k) - __ldg(c.payload + 2 * (k - 1));
    const uint64_t c0 = cwx[b];
    const uint32_t w = (uint32_t)(cwx[b + 1] - c0);
    if (!w) continue;
    const uint64_t bit = c0 * B + (s & (B - 1)) * (uint64_t)w;
    const uint64_t q = bit >> 6;
    const uint32_t sh = (uint32_t)(bit & 63);
    atomicOr(payload + q, (unsigned long long)(d << sh));
    if (sh && sh + w > 64) atomicOr(payload + q + 1, (unsigned long long)(d >> (64 - sh)));
  }
  // cw[b + 1] for every block (grid-stride over blocks)
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride) {
    if (cwx[b + 1] > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
    cw[b + 1] = (uint32_t)cwx[b + 1];
  }
}

cudaError_t launch_rle2delta_widths(const ColView& c, uint32_t B, uint64_t nb, uint32_t* wk, uint64_t* ref,
                                    uint64_t* rem, cudaStream_t s) {
  cudaError_t e = nb ? cudaMemsetAsync(wk, 0, 4 * nb, s) : cudaSuccess;
  if (e != cudaSuccess || !c.nruns) return e;
  uint64_t g = (c.nruns + 255) / 256;
  if (g > (uint64_t)num_sms() * 16) g = num_sms() * 16;
  ProfScope prof_("rle2delta_width", s);
  rle2delta_width_kernel<<<(int)g, 256, 0, s>>>(c, B, lg2(B), nb, wk, ref, rem);
  return cudaGetLastError();
}

cudaError_t launch_rle2delta_pack(const ColView& c, uint32_t B, uint64_t nb, const uint64_t* cwx, uint32_t* cw,
                                  uint64_t* payload, uint32_t* err, cudaStream_t s) {
  const uint64_t work = c.nruns > nb ? c.nruns : nb;
  if (!work) return cudaSuccess;
  uint64_t g = (work + 255) / 256;
  if (g > (uint64_t)num_sms() * 16) g = num_sms() * 16;
  ProfScope prof_("rle2delta_pack", s);
  rle2delta_pack_kernel<<<(int)g, 256, 0, s>>>(c, B, lg2(B), nb, cwx, cw,
                                                reinterpret_cast<unsigned long long*>(payload), err);
  return cudaGetLastError();
}

}  // namespace ms
