// cstream.cuh — compress of uncompressed u64 values into a block format (DYN_BP,
// FOR_BP, DELTA_BP, D-4..D-7) in slot mode: the values are streamed
// through shared memory and each 2048-row tile is encoded by two warps (the
// staged engine's 256-thread CTA per tile spends a quarter of its time in
// __syncthreads and ~6,700 warp instructions per tile).
//
// compress_stream_kernel: persistent, one CTA per SM, each CTA a contiguous run of
// tiles; warp 0 issues one TMA bulk copy per tile (16 KiB) into stage li % 13
// (mbarrier complete_tx); consumer pair li % 13 (two warps, no CTA barrier):
//   pass 1  per block, warp h takes the 32-row groups h, h + 2, ... (row 32g +
//           lane): FOR: the extremes; DYN / DELTA: the OR of the values (DELTA: of
//           d = v - v_prev, d_0 = 0, D-6) — ebw(max) = ebw(OR) — reduced across
//           the warp (redux) and combined in shared memory;
//   widths  lane b: w_b (DYN: ebw(max), FOR: ebw(max - min), DELTA: ebw(max d)),
//           exclusive prefix over the tile's blocks -> bw, ref, slot offsets;
//   pack    thread t of the pair builds u32 words t, t + 64, ... of each block
//           from the codes that overlap it, at the block's width as a
//           compile-time constant (switch over 1..64), and stores them to the
//           tile's slot (coalesced); rows past the last full block go to the
//           remainder.
// The scan of bw and tile_copy_kernel then place the tiles as for the engine.
#pragma once
#include "common.cuh"
#include "engine.cuh"
#include "tma.cuh"

namespace ms {

constexpr int kCsStages = 13;
constexpr int kCsPair = 2;  // consumer warps per stage
constexpr int kCsThreads = (1 + kCsPair * kCsStages) * 32;

struct CsPair {  // per stage: the tile's block statistics
  unsigned long long lo[kChunk / 128], hi[kChunk / 128];
  uint32_t w[kChunk / 128], ex[kChunk / 128];
  uint32_t wmax, pad_[3];  // the tile's largest block width
};

__host__ __device__ constexpr size_t cs_smem_bytes() {
  return (size_t)kCsStages * kChunk * 8 + kCsStages * sizeof(CsPair) + 2 * kCsStages * 8;
}

__device__ __forceinline__ void cs_bar(uint32_t id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id + 1) : "memory"); }

// u32 words m = tt, tt + 64, ... of a block of B codes at the compile-time width W
// (B * W / 32 words): word m starts inside code j = 32m / W (a division by a
// constant) at bit sh = 32m - jW; the codes j + 1, ... that fill it follow, at
// most 32 / W + 1 of them (DELTA: code = v_j - v_{j-1}, code 0 = 0; else v - sub).
template <int W, bool DELTA, bool SUB>
__device__ __forceinline__ void cs_pack_block(const uint64_t* __restrict__ cb, uint64_t sub, uint32_t B,
                                              uint32_t* __restrict__ dst, uint32_t tt) {
  constexpr int K = 32 / W + 1;  // codes after the first that may overlap one word
  const uint32_t nw = (uint32_t)W * (B >> 5);
  for (uint32_t m = tt; m < nw; m += 32 * kCsPair) {
    const uint32_t bit0 = m * 32, j = bit0 / (uint32_t)W, sh = bit0 - j * (uint32_t)W;
    uint64_t v = cb[j];
    uint64_t prev = DELTA ? (j ? cb[j - 1] : v) : (SUB ? sub : 0ull);  // DELTA: the previous value carried along
    uint64_t acc = (v - prev) >> sh;
    uint32_t filled = (uint32_t)W - sh;
#pragma unroll
    for (int k = 1; k <= K; ++k) {
      if (filled < 32) {
        if (DELTA) prev = v;
        v = cb[j + k];
        acc |= (v - prev) << filled;
        filled += W;
      }
    }
    dst[m] = (uint32_t)acc;
  }
}

template <bool DELTA, bool SUB>
__device__ __forceinline__ void cs_pack_dispatch(uint32_t w, const uint64_t* cb, uint64_t sub, uint32_t B,
                                                 uint32_t* dst, uint32_t tt) {
  switch (w) {
#define MS_CS_CASE(W) \
  case W:             \
    cs_pack_block<W, DELTA, SUB>(cb, sub, B, dst, tt); \
    break;
    MS_CS_CASE(1) MS_CS_CASE(2) MS_CS_CASE(3) MS_CS_CASE(4) MS_CS_CASE(5) MS_CS_CASE(6) MS_CS_CASE(7)
    MS_CS_CASE(8) MS_CS_CASE(9) MS_CS_CASE(10) MS_CS_CASE(11) MS_CS_CASE(12) MS_CS_CASE(13) MS_CS_CASE(14)
    MS_CS_CASE(15) MS_CS_CASE(16) MS_CS_CASE(17) MS_CS_CASE(18) MS_CS_CASE(19) MS_CS_CASE(20) MS_CS_CASE(21)
    MS_CS_CASE(22) MS_CS_CASE(23) MS_CS_CASE(24) MS_CS_CASE(25) MS_CS_CASE(26) MS_CS_CASE(27) MS_CS_CASE(28)
    MS_CS_CASE(29) MS_CS_CASE(30) MS_CS_CASE(31) MS_CS_CASE(32) MS_CS_CASE(33) MS_CS_CASE(34) MS_CS_CASE(35)
    MS_CS_CASE(36) MS_CS_CASE(37) MS_CS_CASE(38) MS_CS_CASE(39) MS_CS_CASE(40) MS_CS_CASE(41) MS_CS_CASE(42)
    MS_CS_CASE(43) MS_CS_CASE(44) MS_CS_CASE(45) MS_CS_CASE(46) MS_CS_CASE(47) MS_CS_CASE(48) MS_CS_CASE(49)
    MS_CS_CASE(50) MS_CS_CASE(51) MS_CS_CASE(52) MS_CS_CASE(53) MS_CS_CASE(54) MS_CS_CASE(55) MS_CS_CASE(56)
    MS_CS_CASE(57) MS_CS_CASE(58) MS_CS_CASE(59) MS_CS_CASE(60) MS_CS_CASE(61) MS_CS_CASE(62) MS_CS_CASE(63)
    MS_CS_CASE(64)
#undef MS_CS_CASE
    default:
      break;
  }
}


// ---- narrow blocks (w <= 16): the word-per-thread builder reads the code at the
// start of each word, 32 / W elements apart, so the lanes of a half-warp fall on
// W (odd W) or fewer bank pairs (ncu at c3, DELTA, W ~ 5: 4.4-way conflicts, 62 % of
// the shared-load wavefronts, the L1 pipe at 88 %). Instead the tile's codes are
// staged once as u32 at 33 words per 32 rows (cs_stage_codes: conflict-free row
// reads, conflict-free writes, in place over the tile's first 8.25 KiB), and thread
// u packs rows [32u, 32u + 32) = exactly W output words from 32 conflict-free
// loads (bank (33u + i) mod 32), every shift a compile-time constant.
constexpr uint32_t kCsNarrow = 16;  // widest block of the staged path
constexpr uint32_t kCsUnitStride = 33;

template <int W>
__device__ __forceinline__ void cs_pack_unit(const uint32_t* __restrict__ c, uint32_t* __restrict__ dst) {
  constexpr int V = (W % 4 == 0) ? 4 : ((W % 2 == 0) ? 2 : 1);
  uint32_t o[V];
  uint64_t acc = 0;
  int filled = 0, k = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    acc |= (uint64_t)c[i] << filled;
    filled += W;
    if (filled >= 32) {
      o[k % V] = (uint32_t)acc;
      acc >>= 32;
      filled -= 32;
      ++k;
      if (k % V == 0) {
        if constexpr (V == 4) *reinterpret_cast<uint4*>(dst + k - 4) = make_uint4(o[0], o[1], o[2], o[3]);
        else if constexpr (V == 2) *reinterpret_cast<uint2*>(dst + k - 2) = make_uint2(o[0], o[1]);
        else dst[k - 1] = o[0];
      }
    }
  }
}

__device__ __forceinline__ void cs_pack_unit_dispatch(uint32_t w, const uint32_t* c, uint32_t* dst) {
  switch (w) {
#define MS_CU_CASE(W) \
  case W:             \
    cs_pack_unit<W>(c, dst); \
    break;
    MS_CU_CASE(1) MS_CU_CASE(2) MS_CU_CASE(3) MS_CU_CASE(4) MS_CU_CASE(5) MS_CU_CASE(6) MS_CU_CASE(7)
    MS_CU_CASE(8) MS_CU_CASE(9) MS_CU_CASE(10) MS_CU_CASE(11) MS_CU_CASE(12) MS_CU_CASE(13) MS_CU_CASE(14)
    MS_CU_CASE(15) MS_CU_CASE(16)
#undef MS_CU_CASE
    default:
      break;
  }
}

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
      const uint32_t i0 = (b << lg) + h * 32 + lane, i1 = (b + 1) << lg;
      if (is_for) {  // FOR: the extremes themselves (ref = min, w = ebw(max - min))
        uint64_t lo = ~0ull, hi = 0;
#pragma unroll 4
        for (uint32_t i = i0; i < i1; i += 32 * kCsPair) {
          const uint64_t v = V[i];
          lo = v < lo ? v : lo;
          hi = v > hi ? v : hi;
        }
#pragma unroll
        for (int q = 16; q > 0; q >>= 1) {
          const uint64_t a2 = __shfl_xor_sync(kFull, lo, q), b2 = __shfl_xor_sync(kFull, hi, q);
          lo = a2 < lo ? a2 : lo;
          hi = b2 > hi ? b2 : hi;
        }
        if (lane == 0) {
          atomicMin(&W.lo[b], (unsigned long long)lo);
          atomicMax(&W.hi[b], (unsigned long long)hi);
        }
      } else {  // DYN / DELTA: only ebw(max) is needed, and ebw(max) = ebw(OR): one OR per row
        uint32_t ol = 0, oh = 0;
        if (is_delta) {
#pragma unroll 4
          for (uint32_t i = i0; i < i1; i += 32 * kCsPair) {
            const uint64_t d = (i & (B - 1)) ? V[i] - V[i - 1] : 0ull;
            ol |= (uint32_t)d;
            oh |= (uint32_t)(d >> 32);
          }
        } else {
#pragma unroll 4
          for (uint32_t i = i0; i < i1; i += 32 * kCsPair) {
            const uint2 v = *reinterpret_cast<const uint2*>(V + i);
            ol |= v.x;
            oh |= v.y;
          }
        }
        ol = __reduce_or_sync(kFull, ol);
        oh = __reduce_or_sync(kFull, oh);
        if (lane == 0) atomicOr(&W.hi[b], ((unsigned long long)oh << 32) | ol);
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
      const uint32_t wm = __reduce_max_sync(kFull, w);
      if (lane == 0) W.wmax = wm;
    }
    cs_bar(p);
    // pack: thread tt builds u32 words tt, tt + 64, ... of each block from the codes overlapping them,
    // at the block's width as a compile-time constant (cs_pack_block<W>)
    uint32_t* slot32 = reinterpret_cast<uint32_t*>(o.slots + t * kChunk);
    if (nmain == (uint32_t)kChunk && W.wmax <= kCsNarrow) {
      // narrow tile: stage the codes as u32 (their low words are exact: w <= 16), 33 words per
      // 32 rows, over the tile itself. Batch tb = rows [512 tb, 512 tb + 512): read into
      // registers, barrier, write words [528 tb, 528 tb + 528) = rows [264 tb, 264 tb + 264) of
      // the tile, all read in this or an earlier batch; later batches read rows >= 512 tb + 511.
      uint32_t* C = reinterpret_cast<uint32_t*>(V);
#pragma unroll 1
      for (uint32_t tb = 0; tb < kChunk / 512; ++tb) {
        uint32_t c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t i = (16 * tb + 2 * k + h) * 32 + lane;
          const uint32_t v = (uint32_t)V[i];
          if (is_delta) c[k] = (i & (B - 1)) ? v - (uint32_t)V[i - 1] : 0u;
          else if (is_for) c[k] = v - (uint32_t)W.lo[i >> lg];
          else c[k] = v;
        }
        cs_bar(p);
#pragma unroll
        for (int k = 0; k < 8; ++k) C[(16 * tb + 2 * k + h) * kCsUnitStride + lane] = c[k];
      }
      cs_bar(p);
      const uint32_t b = (tt * 32) >> lg, wb = W.w[b];
      if (wb)
        cs_pack_unit_dispatch(wb, C + tt * kCsUnitStride,
                              slot32 + (W.ex[b] << (lg - 5)) + (tt - (b << (lg - 5))) * wb);
    } else {
    for (uint32_t b = 0; b < nbc; ++b) {
      const uint32_t wb = W.w[b];
      if (!wb) continue;
      const uint64_t* cb = V + (b << lg);
      const uint64_t sub = is_for ? W.lo[b] : 0ull;
      uint32_t* dst = slot32 + (W.ex[b] << (lg - 5));
      if (is_delta) cs_pack_dispatch<true, false>(wb, cb, sub, B, dst, tt);
      else if (is_for) cs_pack_dispatch<false, true>(wb, cb, sub, B, dst, tt);
      else cs_pack_dispatch<false, false>(wb, cb, sub, B, dst, tt);  // DYN: the values themselves
    }
    }
    // rows past the last full block: the uncompressed remainder
    for (uint32_t i = nmain + tt; i < cnt; i += 32 * kCsPair) o.rem[r0 + i - nbm] = V[i];
    cs_bar(p);
    if (lane == 0) mbar_arrive(empty + p);
  }
}

}  // namespace ms
