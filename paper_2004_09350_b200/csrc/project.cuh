// project.cuh — an alternative project path (opt-in, MS_PROJECT_PIPE=1), kept
// for measurement: sorted positions as DELTA_BP{G} (G = 32*PER <= 512, the
// select output format P:584), data in a block format with per-block headers
// (DYN_BP / FOR_BP, random access extended per D-12), output in a
// block format of size G or uncompressed. Per item: positions decoded with a
// streaming bit reader; the data window's block headers (<= 32 blocks) loaded
// once and broadcast by shuffles; one bulk L2 prefetch of the window; 8
// independent 32-bit gathers per lane in flight; codes packed lane-contiguously
// (pack_lane_codes) with a deferred look-back for cw (D-4). The items are
// software-pipelined (see project_pipe_kernel). Measured on B200 at BJ.c5 it
// is slower than ProjectSource + warp_encode_deferred_kernel (4.4 vs 3.25 ms:
// three tiles per warp cost occupancy and the gather stays L2-latency bound),
// so the default path is the latter; DESIGN.md §7 records the numbers.
#pragma once
#include "common.cuh"
#include "launch.h"
#include "positions.cuh"

namespace ms {

// Streaming LSB-first bit reader over u32 words (D-1).
struct BitReader {
  const uint32_t* p;
  uint64_t acc;
  uint32_t avail;
  __device__ __forceinline__ void init(const uint64_t* payload, uint64_t bit) {
    p = reinterpret_cast<const uint32_t*>(payload) + (bit >> 5);
    const uint32_t s = (uint32_t)(bit & 31);
    acc = __ldg(p++) >> s;
    avail = 32 - s;
  }
  __device__ __forceinline__ uint64_t get(uint32_t w) {  // 0 <= w <= 32
    if (avail < w) {
      acc |= (uint64_t)__ldg(p++) << avail;
      avail += 32;
    }
    const uint64_t v = acc & ((1ull << w) - 1);
    acc >>= w;
    avail -= w;
    return v;
  }
};

// out-of-line random access for the rare positions (keeps the unrolled fast path small)
__device__ __noinline__ uint64_t read_row_checked(const ColView& data, uint64_t p, uint64_t row_offset,
                                                   uint32_t* err) {
  const bool ok = p >= row_offset && p - row_offset < data.n;
  if (!ok) {
    atomicOr(err, err_bit(MS_E_RANGE));
    return 0ull;
  }
  return read_row(data, p - row_offset);
}

}  // namespace ms

namespace ms {

// ----------------------------------------------------------------------------
// project_pipe_kernel (opt-in, MS_PROJECT_PIPE=1): the same operation as
// ProjectSource + the deferred encoder, software-pipelined across items so that no memory round trip of an
// item is waited for on its own. Items (full positions blocks) are assigned
// statically, warp gw taking gw, gw + NW, gw + 2NW, ...; per iteration, with
// cur = the item being gathered and nxt = cur + NW:
//   1. load nxt's positions header (cw, base)        -- in flight during 2
//   2. gather cur, first half (lane-strided, from L2: its window was prefetched
//      one iteration ago)
//   3. load nxt's positions payload words            -- in flight during 4
//   4. gather cur, second half
//   5. decode nxt's positions into its tile, load nxt's data-window headers
//                                                    -- in flight during 6-7
//   6. cur: codes, width, pack in place, publish the width (look-back)
//   7. resolve the exclusive width prefix of the previous item and store it
//   8. bulk-prefetch nxt's data window into L2
// Three tiles per warp rotate through the roles prev (packed, awaiting its
// prefix) / cur / nxt. Look-back deadlock freedom: item i is published before
// its warp waits on anything newer than i - 2NW, and every warp is resident.
struct PipeWin {
  uint64_t p_first, p_last, row0;
  uint64_t h_ref;
  uint32_t hdr, c0, nblk;
  bool ok;
};

template <int PER>
__device__ __forceinline__ void pipe_window(const ColView& data, const uint64_t* T, uint64_t row_offset,
                                            uint32_t lane, PipeWin& W) {
  constexpr uint32_t G = 32 * PER;
  const uint64_t main_rows = data.nb << data.log2B;
  W.p_first = T[pidx(0)];
  W.p_last = T[pidx(G - 1)];
  const uint64_t plo = W.p_first - row_offset, phi = W.p_last - row_offset;
  const uint64_t b_lo = plo >> data.log2B;
  W.ok = W.p_first >= row_offset && W.p_last >= W.p_first && phi < main_rows && ((phi >> data.log2B) - b_lo) < 32;
  W.hdr = 0;
  W.h_ref = 0;
  W.c0 = 0;
  W.nblk = 0;
  W.row0 = row_offset + (b_lo << data.log2B);
  if (W.ok) {
    const uint64_t bj = b_lo + lane;
    W.c0 = __ldg(data.cw + b_lo);
    if (bj < data.nb) {
      const uint32_t a = __ldg(data.cw + bj);
      const uint32_t a1 = __ldg(data.cw + bj + 1);
      W.hdr = ((a - W.c0) << 7) | (a1 - a);
      if (data.format == MS_FOR_BP) W.h_ref = __ldg(data.ref + bj);
    }
    W.nblk = (uint32_t)((phi >> data.log2B) - b_lo) + 1;
  }
}

__device__ __forceinline__ void pipe_prefetch(const ColView& data, const PipeWin& W, uint32_t lane) {
  if (!W.ok) return;
  const uint32_t h = __shfl_sync(kFull, W.hdr, (W.nblk - 1) & 31);
  const uint64_t bytes = (uint64_t)((h >> 7) + (h & 127)) * (data.B / 8);
  if (lane == 0 && bytes >= 16) {
    const uint64_t* a = data.payload + (uint64_t)W.c0 * (data.B / 64);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"((uint32_t)(bytes & ~15ull)) : "memory");
  }
}

// gather ranks q*32 + lane for q in [Q0, Q0 + QN) of the tile: positions in, values out
template <int Q0, int QN>
__device__ __forceinline__ void pipe_gather(const ColView& data, uint64_t* T, const PipeWin& W, uint64_t row_offset,
                                            uint32_t lane, uint32_t* err) {
  if (!W.ok) {
#pragma unroll 2
    for (int q = Q0; q < Q0 + QN; ++q) {
      const uint32_t i = q * 32 + lane;
      T[pidx(i)] = read_row_checked(data, T[pidx(i)], row_offset, err);
    }
    return;
  }
  const uint32_t* base32 = reinterpret_cast<const uint32_t*>(data.payload) + (((uint64_t)W.c0 * data.B) >> 5);
  const uint32_t dmask = data.B - 1;
  uint32_t lo[QN], hi[QN], meta[QN];
  uint32_t rare = 0;
#pragma unroll
  for (int u = 0; u < QN; ++u) {
    const uint64_t pq = T[pidx((Q0 + u) * 32 + lane)];
    const bool inw = pq - W.p_first <= W.p_last - W.p_first;
    const uint32_t rel = inw ? (uint32_t)(pq - W.row0) : 0u;
    const uint32_t bsel = (rel >> data.log2B) & 31;
    const uint32_t h = __shfl_sync(kFull, W.hdr, bsel);
    const uint32_t w = h & 127;
    const uint32_t bit = (h >> 7) * data.B + (rel & dmask) * w;
    const bool ok = inw && w <= 32;
    rare |= (uint32_t)!ok << u;
    const uint32_t i = bit >> 5, sft = bit & 31;
    lo[u] = ok && w ? __ldg(base32 + i) : 0u;
    hi[u] = ok && sft + w > 32 ? __ldg(base32 + i + 1) : 0u;
    meta[u] = sft | (min(w, 32u) << 5) | (bsel << 11);
  }
#pragma unroll
  for (int u = 0; u < QN; ++u) {
    const uint32_t sft = meta[u] & 31, w = (meta[u] >> 5) & 63, bsel = meta[u] >> 11;
    const uint64_t rf = data.format == MS_FOR_BP ? __shfl_sync(kFull, W.h_ref, bsel) : 0ull;
    const uint32_t i = (Q0 + u) * 32 + lane;
    if ((rare >> u) & 1) T[pidx(i)] = read_row_checked(data, T[pidx(i)], row_offset, err);
    else T[pidx(i)] = rf + (uint64_t)(__funnelshift_r(lo[u], hi[u], sft) & (uint32_t)((1ull << w) - 1));
  }
}

template <int PER>
__global__ void __launch_bounds__(128) project_pipe_kernel(ColView pos, ColView data, uint64_t row_offset, PosEnc e,
                                                           uint64_t n_full, uint64_t* status, uint32_t* err,
                                                           uint32_t prefetch) {
  constexpr uint32_t G = 32 * PER;
  constexpr uint32_t TS = tile_slots(G);
  extern __shared__ __align__(16) uint64_t pp_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t* tiles = pp_sm + (uint64_t)wid * 3 * TS;
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  const uint64_t NW = (uint64_t)gridDim.x * (blockDim.x >> 5);
  uint64_t item = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  if (item >= n_full) return;

  // positions decode of one block into tile T (lane-consecutive ranks), from its header
  // and (for narrow deltas) five preloaded payload words
  auto decode = [&](uint64_t it, uint32_t cw0, uint32_t wp, uint64_t bref, const uint32_t (&x)[5], uint64_t* T) {
    const uint64_t bit0 = (uint64_t)cw0 * G + (uint64_t)PER * lane * wp;
    uint64_t p[PER];
    uint64_t acc = 0;
    if (wp == 0) {
#pragma unroll
      for (int q = 0; q < PER; ++q) p[q] = 0;
    } else if (wp <= 8) {
      const uint32_t sft = (uint32_t)(bit0 & 31);
      uint64_t win = ((uint64_t)x[1] << 32 | x[0]) >> sft;
      uint32_t avail = 64 - sft, k = 2;
      const uint64_t m = (1ull << wp) - 1;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        if (avail < wp) {
          const uint32_t nx = k == 2 ? x[2] : (k == 3 ? x[3] : x[4]);
          win |= (uint64_t)nx << avail;
          avail += 32;
          ++k;
        }
        acc += win & m;
        p[q] = acc;
        win >>= wp;
        avail -= wp;
      }
    } else if (wp <= 32) {
      BitReader br;
      br.init(pos.payload, bit0);
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        acc += br.get(wp);
        p[q] = acc;
      }
    } else {
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        acc += unpack_at(pos.payload, bit0 + (uint64_t)q * wp, wp);
        p[q] = acc;
      }
    }
    const uint64_t incl = warp_incl_scan(acc);
    const uint64_t base = bref + incl - acc;
#pragma unroll
    for (int q = 0; q < PER; ++q) T[pidx(PER * lane + q)] = p[q] + base;
    __syncwarp();
  };
  auto preload = [&](uint32_t cw0, uint32_t wp, uint32_t (&x)[5]) {
    const uint64_t bit0 = (uint64_t)cw0 * G + (uint64_t)PER * lane * wp;
    const uint32_t* w32 = reinterpret_cast<const uint32_t*>(pos.payload) + (bit0 >> 5);
    const uint32_t nwd = wp && wp <= 8 ? (((uint32_t)(bit0 & 31) + PER * wp + 31) >> 5) : 0u;
#pragma unroll
    for (int k = 0; k < 5; ++k) x[k] = (uint32_t)k < nwd ? __ldg(w32 + k) : 0u;
  };
  auto store = [&](uint64_t it, uint32_t w, uint64_t ref, const uint64_t* T) {
    const uint64_t E = lookback_resolve(status, it, w);
    if (lane == 0) {
      if (E + w > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
      e.cw[it + 1] = (uint32_t)(E + w);
      if (e.format != MS_DYN_BP) e.ref[it] = ref;
    }
    uint64_t* dst = e.payload + E * (G / 64);
    const uint32_t nw64 = G / 64 * w;
    for (uint32_t m = lane; m < nw64; m += 32) dst[m] = T[m];
    __syncwarp();
  };

  // prologue: items i0 and i1 = i0 + NW decoded, their windows' headers loaded, i0 prefetched
  int t_cur = 0, t_n1 = 1, t_free = 2;
  PipeWin W, W1;
  auto front = [&](uint64_t it, uint64_t* T, PipeWin& Wo) {
    const uint32_t cw0 = __ldg(pos.cw + it), wp = __ldg(pos.cw + it + 1) - cw0;
    const uint64_t bref = __ldg(pos.ref + it);
    uint32_t x[5];
    preload(cw0, wp, x);
    decode(it, cw0, wp, bref, x, T);
    pipe_window<PER>(data, T, row_offset, lane, Wo);
  };
  front(item, tiles + t_cur * TS, W);
  if (prefetch) pipe_prefetch(data, W, lane);
  if (item + NW < n_full) front(item + NW, tiles + t_n1 * TS, W1);
  uint64_t prev = ~0ull, prev_ref = 0;
  uint32_t prev_w = 0;
  while (true) {
    uint64_t* T = tiles + t_cur * TS;
    const uint64_t n1 = item + NW, n2 = item + 2 * NW;
    const bool has_n1 = n1 < n_full, has_n2 = n2 < n_full;
    // 1. the next item's window into L2, a whole iteration ahead of its gather
    if (prefetch && has_n1) pipe_prefetch(data, W1, lane);
    // 2. the item after next: positions header
    uint32_t ncw0 = 0, nwp = 0;
    uint64_t nref = 0;
    if (has_n2) {
      ncw0 = __ldg(pos.cw + n2);
      nwp = __ldg(pos.cw + n2 + 1) - ncw0;
      nref = __ldg(pos.ref + n2);
    }
    // 3. gather, first half
    pipe_gather<0, PER / 2>(data, T, W, row_offset, lane, err);
    // 4. the item after next: payload words
    uint32_t x[5];
    preload(ncw0, has_n2 ? nwp : 0u, x);
    // 5. gather, second half
    pipe_gather<PER / 2, PER / 2>(data, T, W, row_offset, lane, err);
    __syncwarp();
    // 6. the previous item: resolve its prefix, store it (frees its tile)
    if (prev != ~0ull) {
      store(prev, prev_w, prev_ref, tiles + t_free * TS);
      prev = ~0ull;
    }
    // 7. the item after next: positions into the free tile, window headers
    PipeWin W2;
    if (has_n2) {
      decode(n2, ncw0, nwp, nref, x, tiles + t_free * TS);
      pipe_window<PER>(data, tiles + t_free * TS, row_offset, lane, W2);
    }
    // 8. this item: encode, publish (block formats) or store (UNCOMPR)
    if (!is_block) {
      uint64_t* dst = e.payload + item * G;
#pragma unroll 4
      for (int q = 0; q < PER; ++q) dst[q * 32 + lane] = T[pidx(q * 32 + lane)];
      __syncwarp();
    } else {
      uint64_t c[PER];
#pragma unroll
      for (int q = 0; q < PER; ++q) c[q] = T[pidx(lane * PER + q)];
      uint64_t ref = 0, mx = 0;
      if (e.format == MS_DELTA_BP) {
        const uint64_t last = __shfl_up_sync(kFull, c[PER - 1], 1);
        ref = __shfl_sync(kFull, c[0], 0);
#pragma unroll
        for (int q = PER - 1; q > 0; --q) c[q] -= c[q - 1];
        c[0] = lane ? c[0] - last : 0ull;
      } else if (e.format == MS_FOR_BP) {
        uint64_t lo = c[0];
#pragma unroll
        for (int q = 1; q < PER; ++q) lo = c[q] < lo ? c[q] : lo;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t t = __shfl_xor_sync(kFull, lo, o);
          lo = t < lo ? t : lo;
        }
        ref = lo;
#pragma unroll
        for (int q = 0; q < PER; ++q) c[q] -= lo;
      }
#pragma unroll
      for (int q = 0; q < PER; ++q) mx = c[q] > mx ? c[q] : mx;
      const uint32_t w = ebw64(warp_max(mx));
      __syncwarp();
      pack_lane_codes<PER>(reinterpret_cast<uint32_t*>(T), c, w, lane);
      lookback_publish(status, item, w);
      prev = item;
      prev_w = w;
      prev_ref = ref;
    }
    if (!has_n1) break;
    // rotate: cur -> (prev's tile), n1 -> cur, n2 -> n1
    const int t_old = t_cur;
    t_cur = t_n1;
    t_n1 = t_free;
    t_free = t_old;
    W = W1;
    W1 = W2;
    item = n1;
  }
  if (prev != ~0ull) store(prev, prev_w, prev_ref, tiles + t_cur * TS);
}

}  // namespace ms

namespace ms {
// the final partial positions block of project_pipe_kernel: one value per lane step
__global__ void project_tail_kernel(ColView pos, ColView data, uint64_t row_offset, PosEnc e, uint64_t r0,
                                    uint32_t* err) {
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  for (uint64_t i = threadIdx.x; r0 + i < e.n_out; i += blockDim.x) {
    const uint64_t v = read_row_checked(data, read_row(pos, r0 + i), row_offset, err);
    if (is_block) e.rem[i] = v;
    else e.payload[r0 + i] = v;
  }
}
}  // namespace ms
