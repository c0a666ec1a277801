// project.cuh — project for the configuration the paper's simple
// query runs: sorted positions as DELTA_BP{G} (G = 32*PER <= 512,
// the select output format P:584), data in a block format with per-block
// headers (DYN_BP / FOR_BP, random access extended per D-12), output in a block
// format with the same block size (output block k <-> positions block k) or
// uncompressed. Everything stays in registers between the two layers:
//   positions  lane j decodes codes [PER*j, PER*j + PER) of positions block k
//              with a streaming bit reader (one 32-bit load per 32 bits),
//              warp prefix sum of the lane sums + the block base (D-6);
//   gather     the block headers of the data window (<= 32 data blocks, lane
//              i -> block b_lo + i: window-relative cw, width, reference) are
//              loaded once and broadcast by shuffles; one bulk L2 prefetch of
//              the window's payload; each value is then one or two 32-bit
//              loads + a funnel shift (w <= 32; wider blocks, positions in the
//              data remainder and windows wider than 32 blocks take read_row);
//   output     FOR: codes v - min, DELTA: differences, DYN: values; width by a
//              warp max; packed lane-contiguously into a shared-memory block
//              (pack_lane_codes); the exclusive width prefix (cw, D-4) by a
//              deferred decoupled look-back (two blocks per warp), then one
//              coalesced store. UNCOMPR output is stored directly.
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

// Source for warp_encode_deferred_kernel (positions.cuh): the same decode and
// gather as project_fast_kernel, with the positions transposed through the
// warp's shared-memory tile so that the gather runs lane-strided (rank q*32 +
// lane: neighbouring lanes read neighbouring rows, i.e. the same sectors) and
// the values land in the tile for the lane-consecutive encoder.
template <int PER>
struct ProjectFastSource {
  ColView pos;
  ColView data;
  uint64_t row_offset;
  uint32_t prefetch;
  __device__ __forceinline__ void load(uint32_t item, uint64_t r0, uint32_t cnt, uint64_t* P, uint32_t lane,
                                       uint32_t* err) const {
    constexpr uint32_t G = 32 * PER;
    if (cnt < G || r0 + G > (pos.nb << pos.log2B)) {  // partial block: one value at a time
      for (uint32_t i = lane; i < cnt; i += 32) P[pidx(i)] = read_row_checked(data, read_row(pos, r0 + i), row_offset, err);
      __syncwarp();
      return;
    }
    // ---- positions (lane-consecutive decode, into the tile)
    {
      const uint32_t cw0 = __ldg(pos.cw + item);
      const uint32_t wp = __ldg(pos.cw + item + 1) - cw0;
      const uint64_t bit0 = (uint64_t)cw0 * G + (uint64_t)PER * lane * wp;
      uint64_t p[PER];
      uint64_t acc = 0;
      if (wp == 0) {
#pragma unroll
        for (int q = 0; q < PER; ++q) p[q] = 0;
      } else if (wp <= 8 && PER == 16) {  // the lane's <= 128 + 31 bits: five loads issued together
        const uint32_t* w32 = reinterpret_cast<const uint32_t*>(pos.payload) + (bit0 >> 5);
        const uint32_t sft = (uint32_t)(bit0 & 31), nwd = (sft + PER * wp + 31) >> 5;
        const uint32_t x0 = __ldg(w32), x1 = nwd > 1 ? __ldg(w32 + 1) : 0u, x2 = nwd > 2 ? __ldg(w32 + 2) : 0u,
                       x3 = nwd > 3 ? __ldg(w32 + 3) : 0u, x4 = nwd > 4 ? __ldg(w32 + 4) : 0u;
        uint64_t win = ((uint64_t)x1 << 32 | x0) >> sft;
        uint32_t avail = 64 - sft, k = 2;
        const uint64_t m = (1ull << wp) - 1;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          if (avail < wp) {
            const uint32_t nx = k == 2 ? x2 : (k == 3 ? x3 : x4);
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
      const uint64_t base = __ldg(pos.ref + item) + incl - acc;
#pragma unroll
      for (int q = 0; q < PER; ++q) P[pidx(PER * lane + q)] = p[q] + base;
    }
    __syncwarp();
    // ---- data window headers
    const uint64_t main_rows = data.nb << data.log2B;
    const uint64_t p_first = P[pidx(0)], p_last = P[pidx(G - 1)];
    const uint64_t plo = p_first - row_offset, phi = p_last - row_offset;
    const uint64_t b_lo = plo >> data.log2B;
    const bool window = p_first >= row_offset && p_last >= p_first && phi < main_rows &&
                        ((phi >> data.log2B) - b_lo) < 32;
    if (!window) {
#pragma unroll 4
      for (int q = 0; q < PER; ++q) {
        const uint32_t i = q * 32 + lane;
        P[pidx(i)] = read_row_checked(data, P[pidx(i)], row_offset, err);
      }
      __syncwarp();
      return;
    }
    uint32_t h_cw = 0, h_w = 0;
    uint64_t h_ref = 0;
    const uint32_t c0 = __ldg(data.cw + b_lo);
    {
      const uint64_t bj = b_lo + lane;
      if (bj < data.nb) {
        const uint32_t a = __ldg(data.cw + bj);
        h_cw = a - c0;
        h_w = __ldg(data.cw + bj + 1) - a;
        if (data.format == MS_FOR_BP) h_ref = __ldg(data.ref + bj);
      }
      const uint32_t nblk = (uint32_t)((phi >> data.log2B) - b_lo) + 1;
      const uint32_t c_hi = __shfl_sync(kFull, h_cw + h_w, (nblk - 1) & 31);
      const uint64_t bytes = (uint64_t)c_hi * (data.B / 8);
      if (prefetch && lane == 0 && bytes >= 16) {  // one bulk L2 prefetch of the window's payload
        const uint64_t* a = data.payload + (uint64_t)c0 * (data.B / 64);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"((uint32_t)(bytes & ~15ull))
                     : "memory");
      }
    }
    // ---- gather, lane-strided, 8 loads (pairs) in flight per lane
    const uint64_t win_bit0 = (uint64_t)c0 * data.B;
    const uint32_t* base32 = reinterpret_cast<const uint32_t*>(data.payload) + (win_bit0 >> 5);
    const uint32_t hdr = (h_cw << 7) | h_w;  // window-relative cw <= 32 * 64, width <= 64
    const uint32_t dmask = data.B - 1;
    const uint64_t row0 = row_offset + (b_lo << data.log2B);
    uint32_t rare = 0;  // bit q: unsorted position or a block wider than 32 bits
    constexpr int kB = PER < 8 ? PER : 8;
#pragma unroll
    for (int q0 = 0; q0 < PER; q0 += kB) {
      uint32_t lo[kB], hi[kB], meta[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const uint64_t pq = P[pidx((q0 + u) * 32 + lane)];
        const bool inw = pq - p_first <= p_last - p_first;
        const uint32_t rel = inw ? (uint32_t)(pq - row0) : 0u;
        const uint32_t bsel = (rel >> data.log2B) & 31;
        const uint32_t h = __shfl_sync(kFull, hdr, bsel);
        const uint32_t w = h & 127;
        const uint32_t bit = (h >> 7) * data.B + (rel & dmask) * w;
        const bool ok = inw && w <= 32;
        rare |= (uint32_t)!ok << (q0 + u);
        const uint32_t i = bit >> 5, sft = bit & 31;
        lo[u] = ok && w ? __ldg(base32 + i) : 0u;
        hi[u] = ok && sft + w > 32 ? __ldg(base32 + i + 1) : 0u;
        meta[u] = sft | (min(w, 32u) << 5) | (bsel << 11);
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const uint32_t sft = meta[u] & 31, w = (meta[u] >> 5) & 63, bsel = meta[u] >> 11;
        const uint64_t rf = data.format == MS_FOR_BP ? __shfl_sync(kFull, h_ref, bsel) : 0ull;
        const uint32_t i = (q0 + u) * 32 + lane;
        const uint64_t val = rf + (uint64_t)(__funnelshift_r(lo[u], hi[u], sft) & (uint32_t)((1ull << w) - 1));
        if ((rare >> (q0 + u)) & 1) P[pidx(i)] = read_row_checked(data, P[pidx(i)], row_offset, err);
        else P[pidx(i)] = val;
      }
    }
    __syncwarp();
  }
};

template <int PER>
__global__ void __launch_bounds__(128) project_fast_kernel(ColView pos, ColView data, uint64_t row_offset, PosEnc e,
                                                           uint64_t n_items, uint64_t* status, uint32_t* ticket,
                                                           uint32_t* err, uint32_t prefetch) {
  constexpr uint32_t G = 32 * PER;
  constexpr uint32_t kBufU32 = 2 * G;  // one block at w <= 64
  extern __shared__ __align__(16) uint32_t pj_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* bufs = pj_sm + (size_t)wid * 2 * kBufU32;
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  const uint64_t main_rows = data.nb << data.log2B;
  const uint32_t dmask = data.B - 1;
  uint64_t prev = ~0ull, prev_ref = 0;
  uint32_t prev_w = 0, cur = 0;
  auto store = [&](uint64_t item, uint32_t w, uint64_t ref, const uint32_t* T) {
    const uint64_t E = lookback_resolve(status, item, w);
    if (lane == 0) {
      if (E + w > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
      e.cw[item + 1] = (uint32_t)(E + w);
      if (e.format != MS_DYN_BP) e.ref[item] = ref;
    }
    uint64_t* dst = e.payload + E * (G / 64);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(T);
    const uint32_t nw64 = G / 64 * w;
    for (uint32_t m = lane; m < nw64; m += 32) dst[m] = src[m];
    __syncwarp();
  };
  while (true) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(ticket, 1u);
    item = __shfl_sync(kFull, item, 0);
    if (item >= n_items) break;
    const uint64_t r0 = (uint64_t)item * G;
    if (r0 + G > e.n_out) {  // final partial block: raw positions -> raw values (remainder / payload)
      for (uint32_t i = lane; r0 + i < e.n_out; i += 32) {
        const uint64_t pp = read_row(pos, r0 + i);
        const bool ok = pp >= row_offset && pp - row_offset < data.n;
        if (!ok) atomicOr(err, err_bit(MS_E_RANGE));
        const uint64_t val = ok ? read_row(data, pp - row_offset) : 0ull;
        if (is_block) e.rem[i] = val;
        else e.payload[r0 + i] = val;
      }
      continue;
    }
    // ---- positions block `item`
    uint64_t p[PER];
    {
      const uint32_t cw0 = __ldg(pos.cw + item);
      const uint32_t wp = __ldg(pos.cw + item + 1) - cw0;
      const uint64_t bit0 = (uint64_t)cw0 * G + (uint64_t)PER * lane * wp;
      uint64_t acc = 0;
      if (wp == 0) {
#pragma unroll
        for (int q = 0; q < PER; ++q) p[q] = 0;
      } else if (wp <= 8 && PER == 16) {  // the lane's <= 128 + 31 bits: five loads issued together
        const uint32_t* w32 = reinterpret_cast<const uint32_t*>(pos.payload) + (bit0 >> 5);
        const uint32_t sft = (uint32_t)(bit0 & 31), nwd = (sft + PER * wp + 31) >> 5;
        const uint32_t x0 = __ldg(w32), x1 = nwd > 1 ? __ldg(w32 + 1) : 0u, x2 = nwd > 2 ? __ldg(w32 + 2) : 0u,
                       x3 = nwd > 3 ? __ldg(w32 + 3) : 0u, x4 = nwd > 4 ? __ldg(w32 + 4) : 0u;
        uint64_t win = ((uint64_t)x1 << 32 | x0) >> sft;
        uint32_t avail = 64 - sft, k = 2;
        const uint64_t m = (1ull << wp) - 1;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
          if (avail < wp) {
            const uint32_t nx = k == 2 ? x2 : (k == 3 ? x3 : x4);
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
      const uint64_t base = __ldg(pos.ref + item) + incl - acc;
#pragma unroll
      for (int q = 0; q < PER; ++q) p[q] += base;
    }
    // ---- data window headers
    const uint64_t p_first = __shfl_sync(kFull, p[0], 0), p_last = __shfl_sync(kFull, p[PER - 1], 31);
    const uint64_t plo = p_first - row_offset, phi = p_last - row_offset;
    const uint64_t b_lo = plo >> data.log2B;
    const bool window = p_first >= row_offset && p_last >= p_first && phi < main_rows &&
                        ((phi >> data.log2B) - b_lo) < 32;
    uint32_t h_cw = 0, h_w = 0;
    uint64_t h_ref = 0, win_bit0 = 0;
    if (window) {
      const uint64_t bj = b_lo + lane;
      const uint32_t c0 = __ldg(data.cw + b_lo);
      if (bj < data.nb) {
        const uint32_t a = __ldg(data.cw + bj);
        h_cw = a - c0;
        h_w = __ldg(data.cw + bj + 1) - a;
        if (data.format == MS_FOR_BP) h_ref = __ldg(data.ref + bj);
      }
      win_bit0 = (uint64_t)c0 * data.B;
      const uint32_t nblk = (uint32_t)((phi >> data.log2B) - b_lo) + 1;
      const uint32_t c_hi = __shfl_sync(kFull, h_cw + h_w, (nblk - 1) & 31);
      const uint64_t bytes = (uint64_t)c_hi * (data.B / 8);
      if (prefetch && lane == 0 && bytes >= 16) {  // one bulk L2 prefetch of the window's payload
        const uint64_t* a = data.payload + (uint64_t)c0 * (data.B / 64);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"((uint32_t)(bytes & ~15ull))
                     : "memory");
      }
    }
    // ---- gather: per batch of 8 positions all loads are issued before any is used
    uint64_t v[PER];
    if (window) {
      const uint32_t* base32 = reinterpret_cast<const uint32_t*>(data.payload) + (win_bit0 >> 5);
      const uint32_t hdr = (h_cw << 7) | h_w;  // window-relative cw <= 32 * 64, width <= 64
      uint32_t rare = 0;                        // bit q: unsorted position or a block wider than 32 bits
      constexpr int kB = PER < 8 ? PER : 8;
#pragma unroll
      for (int q0 = 0; q0 < PER; q0 += kB) {
        uint32_t lo[kB], hi[kB], meta[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int q = q0 + u;
          const bool inw = p[q] - p_first <= p_last - p_first;
          const uint32_t rel = inw ? (uint32_t)(p[q] - row_offset - (b_lo << data.log2B)) : 0u;
          const uint32_t bsel = (rel >> data.log2B) & 31;
          const uint32_t h = __shfl_sync(kFull, hdr, bsel);
          const uint32_t w = h & 127;
          const uint32_t bit = (h >> 7) * data.B + (rel & dmask) * w;
          const bool ok = inw && w <= 32;
          rare |= (uint32_t)!ok << q;
          const uint32_t i = bit >> 5, sft = bit & 31;
          lo[u] = ok && w ? __ldg(base32 + i) : 0u;
          hi[u] = ok && sft + w > 32 ? __ldg(base32 + i + 1) : 0u;
          meta[u] = sft | (min(w, 32u) << 5) | (bsel << 11);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const uint32_t sft = meta[u] & 31, w = (meta[u] >> 5) & 63, bsel = meta[u] >> 11;
          const uint64_t rf = data.format == MS_FOR_BP ? __shfl_sync(kFull, h_ref, bsel) : 0ull;
          v[q0 + u] = rf + (uint64_t)(__funnelshift_r(lo[u], hi[u], sft) & (uint32_t)((1ull << w) - 1));
        }
      }
      if (rare) {
#pragma unroll
        for (int q = 0; q < PER; ++q)
          if ((rare >> q) & 1) v[q] = read_row_checked(data, p[q], row_offset, err);
      }
    } else {
#pragma unroll
      for (int q = 0; q < PER; ++q) v[q] = read_row_checked(data, p[q], row_offset, err);
    }
    // ---- output
    if (!is_block) {  // UNCOMPR (the host routes other formats elsewhere)
      uint64_t* dst = e.payload + (uint64_t)item * G + PER * lane;
#pragma unroll
      for (int q = 0; q < PER; ++q) dst[q] = v[q];
      continue;
    }
    uint64_t ref = 0, mx = 0;
    if (e.format == MS_DELTA_BP) {
      const uint64_t last = __shfl_up_sync(kFull, v[PER - 1], 1);
      ref = __shfl_sync(kFull, v[0], 0);
#pragma unroll
      for (int q = PER - 1; q > 0; --q) v[q] -= v[q - 1];
      v[0] = lane ? v[0] - last : 0ull;
    } else if (e.format == MS_FOR_BP) {
      uint64_t lo = v[0];
#pragma unroll
      for (int q = 1; q < PER; ++q) lo = v[q] < lo ? v[q] : lo;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t t = __shfl_xor_sync(kFull, lo, o);
        lo = t < lo ? t : lo;
      }
      ref = lo;
#pragma unroll
      for (int q = 0; q < PER; ++q) v[q] -= lo;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) mx = v[q] > mx ? v[q] : mx;
    const uint32_t w = ebw64(warp_max(mx));
    uint32_t* T = bufs + cur * kBufU32;
    pack_lane_codes<PER>(T, v, w, lane);
    lookback_publish(status, item, w);
    if (prev != ~0ull) store(prev, prev_w, prev_ref, bufs + (cur ^ 1) * kBufU32);
    prev = item;
    prev_w = w;
    prev_ref = ref;
    cur ^= 1;
  }
  if (prev != ~0ull) store(prev, prev_w, prev_ref, bufs + (cur ^ 1) * kBufU32);
}

}  // namespace ms
