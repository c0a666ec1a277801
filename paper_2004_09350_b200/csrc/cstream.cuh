// cstream.cuh — compress of uncompressed u64 values into a block format (DYN_BP,
// FOR_BP, DELTA_BP, D-4..D-7) in slot mode: the values are streamed
// through shared memory and each 2048-row tile is encoded by two warps (the
// staged engine's 256-thread CTA per tile spends a quarter of its time in
// __syncthreads and ~6,700 warp instructions per tile).
//
// compress_stream_kernel: persistent, one CTA per SM, each CTA a contiguous run of
// tiles; warp 0 issues one TMA bulk copy per tile (16 KiB) into stage li % 10
// (mbarrier complete_tx); consumer pair li % 10 (two warps, no CTA barrier):
//   pass 1  per block, warp h takes the 32-row groups h, h + 2, ... (row 32g +
//           lane): the extremes (DELTA: of d = v - v_prev, d_0 = 0, D-6) reduced
//           across the warp and combined in shared memory;
//   widths  lane b: w_b (DYN: ebw(max), FOR: ebw(max - min), DELTA: ebw(max d)),
//           exclusive prefix over the tile's blocks -> bw, ref, slot offsets;
//   pack    thread t of the pair builds u32 words t, t + 64, ... of each block
//           from the <= 3 codes that overlap it and stores them to the tile's
//           slot (coalesced); rows past the last full block go to the remainder.
// The scan of bw and tile_copy_kernel then place the tiles as for the engine.
#pragma once
#include "common.cuh"
#include "engine.cuh"
#include "tma.cuh"

namespace ms {

constexpr int kCsStages = 10;
constexpr int kCsPair = 2;  // consumer warps per stage
constexpr int kCsThreads = (1 + kCsPair * kCsStages) * 32;

struct CsPair {  // per stage: the tile's block statistics
  unsigned long long lo[kChunk / 128], hi[kChunk / 128];
  uint32_t w[kChunk / 128], ex[kChunk / 128];
};

__host__ __device__ constexpr size_t cs_smem_bytes() {
  return (size_t)kCsStages * kChunk * 8 + kCsStages * sizeof(CsPair) + 2 * kCsStages * 8;
}

__device__ __forceinline__ void cs_bar(uint32_t id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id + 1) : "memory"); }

__global__ void __launch_bounds__(kCsThreads, 1)
    compress_stream_kernel(const uint64_t* __restrict__ in, uint64_t n, OutView o, uint32_t* err) {
  extern __shared__ __align__(128) uint64_t cs_sm[];
  CsPair* cps = reinterpret_cast<CsPair*>(cs_sm + (size_t)kCsStages * kChunk);
  uint64_t* full = reinterpret_cast<uint64_t*>(cps + kCsStages);
  uint64_t* empty = full + kCsStages;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t n_tiles = (n + kChunk - 1) / kChunk;
  const uint64_t per_cta = (n_tiles + gridDim.x - 1) / gridDim.x;
  const uint64_t i_lo = (uint64_t)blockIdx.x * per_cta;
  const uint64_t i_hi = min(n_tiles, i_lo + per_cta);
  if (threadIdx.x == 0) {
    for (int k = 0; k < kCsStages; ++k) {
      mbar_init(full + k, 1);
      mbar_init(empty + k, kCsPair);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (i_lo >= i_hi) return;
  if (wid == 0) {  // ---------------- producer
    if (lane) return;
    for (uint64_t li = 0; i_lo + li < i_hi; ++li) {
      const uint32_t sg = (uint32_t)(li % kCsStages);
      const uint64_t round = li / kCsStages;
      if (round) mbar_wait(empty + sg, (uint32_t)((round - 1) & 1));
      const uint64_t r0 = (i_lo + li) * kChunk;
      const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, n - r0);
      const uint32_t bytes = (cnt & ~1u) * 8;  // 16-byte multiple; an odd last row is read by the consumer
      mbar_arrive_tx(full + sg, bytes);
      if (bytes) bulk_g2s(cs_sm + (size_t)sg * kChunk, in + r0, bytes, full + sg);
    }
    return;
  }
  // ------------------------------------ consumer pairs: pair p takes tiles p, p + S, ... (stage p)
  const uint32_t p = (wid - 1) / kCsPair, h = (wid - 1) % kCsPair, tt = h * 32 + lane;
  CsPair& W = cps[p];
  uint64_t* V = cs_sm + (size_t)p * kChunk;
  const uint32_t B = o.B, lg = o.log2B;
  const int32_t fmt = o.format;
  const bool is_for = fmt == MS_FOR_BP, is_delta = fmt == MS_DELTA_BP;
  const uint64_t nbm = (n >> lg) << lg;  // rows in full blocks
  uint32_t round = 0;
  for (uint64_t li = p; i_lo + li < i_hi; li += kCsStages, ++round) {
    mbar_wait(full + p, round & 1);
    const uint64_t t = i_lo + li, r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, n - r0);
    const uint32_t nmain = r0 < nbm ? (uint32_t)min((uint64_t)cnt, nbm - r0) : 0u;  // a multiple of B
    const uint32_t nbc = nmain >> lg;
    const uint64_t kb0 = r0 >> lg;
    if (tt < nbc) {
      W.lo[tt] = ~0ull;
      W.hi[tt] = 0ull;
    }
    if ((cnt & 1) && tt == 0) V[cnt - 1] = __ldg(in + r0 + cnt - 1);
    cs_bar(p);
    // pass 1: warp h takes the 32-row groups h, h + 2, ...; per block: the extremes (DELTA:
    // of the differences v - v_prev, d_0 = 0), reduced across the warp, combined in shared memory
    for (uint32_t b = 0; b < nbc; ++b) {
      uint64_t lo = ~0ull, hi = 0;
      const uint32_t i1 = (b + 1) << lg;
#pragma unroll 4
      for (uint32_t i = (b << lg) + h * 32 + lane; i < i1; i += 32 * kCsPair) {
        const uint64_t v = V[i];
        if (is_delta) {
          const uint64_t d = (i & (B - 1)) ? v - V[i - 1] : 0ull;
          hi = d > hi ? d : hi;
        } else {
          lo = v < lo ? v : lo;
          hi = v > hi ? v : hi;
        }
      }
#pragma unroll
      for (int q = 16; q > 0; q >>= 1) {
        const uint64_t a2 = __shfl_xor_sync(kFull, lo, q), b2 = __shfl_xor_sync(kFull, hi, q);
        lo = a2 < lo ? a2 : lo;
        hi = b2 > hi ? b2 : hi;
      }
      if (lane == 0) {
        if (!is_delta) atomicMin(&W.lo[b], (unsigned long long)lo);
        atomicMax(&W.hi[b], (unsigned long long)hi);
      }
    }
    cs_bar(p);
    // widths, references, offsets of the blocks in the tile's slot (units of B/32 u32 words)
    if (h == 0) {
      uint32_t w = 0;
      if (lane < nbc) {
        const uint64_t blo = W.lo[lane], bhi = W.hi[lane];
        w = ebw64(is_for ? bhi - blo : bhi);
        o.bw[kb0 + lane] = w;
        if (is_for) o.ref[kb0 + lane] = blo;
        if (is_delta) o.ref[kb0 + lane] = V[lane << lg];
      }
      uint32_t incl = w;
#pragma unroll
      for (int q = 1; q < 32; q <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, q);
        if (lane >= (uint32_t)q) incl += y;
      }
      if (lane < nbc) {
        W.w[lane] = w;
        W.ex[lane] = incl - w;
      }
    }
    cs_bar(p);
    // pack: thread tt builds u32 words tt, tt + 64, ... of each block from the codes overlapping them
    uint32_t* slot32 = reinterpret_cast<uint32_t*>(o.slots + t * kChunk);
    for (uint32_t b = 0; b < nbc; ++b) {
      const uint32_t wb = W.w[b];
      if (!wb) continue;
      const uint64_t* cb = V + (b << lg);
      const uint64_t sub = is_for ? W.lo[b] : 0ull;
      const uint32_t nw = wb << (lg - 5);  // B * w / 32 words
      const uint32_t magic = 0xffffffffu / wb + 1u;
      uint32_t* dst = slot32 + (W.ex[b] << (lg - 5));
      for (uint32_t m = tt; m < nw; m += 32 * kCsPair) {
        const uint32_t bit0 = m * 32;
        uint32_t j = div_small(bit0, wb, magic);
        // codes j, j+1, ... (DELTA: differences, the previous value carried along)
        uint64_t v = cb[j];
        uint64_t prev = is_delta ? (j ? cb[j - 1] : v) : sub;
        uint64_t acc = (v - prev) >> (bit0 - j * wb);
        for (++j; j < B; ++j) {
          const uint32_t jb = j * wb;
          if (jb >= bit0 + 32) break;
          if (is_delta) prev = v;
          v = cb[j];
          acc |= (v - prev) << (jb - bit0);
        }
        dst[m] = (uint32_t)acc;
      }
    }
    // rows past the last full block: the uncompressed remainder
    for (uint32_t i = nmain + tt; i < cnt; i += 32 * kCsPair) o.rem[r0 + i - nbm] = V[i];
    cs_bar(p);
    if (lane == 0) mbar_arrive(empty + p);
  }
}

}  // namespace ms
