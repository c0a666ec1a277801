// projwin.cuh — project with the data window streamed into shared
// memory by TMA, for sorted DELTA_BP{G} positions (G = 32*PER <= 512, the
// select output format P:584) over DYN_BP / FOR_BP data (random access through
// the cw / ref headers, D-12), into a block format of size G or UNCOMPR.
//
// At BJ.c5 density (6.25%) the positions of one output block touch ~80% of the
// 64-byte DRAM bursts of their data window, so reading the window whole, in
// order, costs no more DRAM traffic than a gather — and it turns ~512 dependent
// random reads into one bulk copy whose latency can be hidden. Each warp (one
// warp per CTA) owns items k, k + NW, ... and runs a software pipeline over
// half-blocks (ranks [0, G/2) and [G/2, G) of an item):
//   - the item's positions are decoded into a shared-memory tile (streaming
//     bit reader, warp prefix sum; lane-consecutive ranks), and the headers of
//     its data window (<= 32 data blocks: window-relative cw, width, reference)
//     are loaded once, lane i <-> block b_lo + i;
//   - each half's window (the data blocks its positions span) is fetched by
//     one cp.async.bulk into a 2-slot ring, completion on an mbarrier; the copy
//     of the next half is in flight while the current half is gathered, and
//     the next item's positions and headers are loaded while the second half's
//     copy is in flight;
//   - the gather reads 1-2 32-bit words per value from shared memory (lanes
//     take ranks q*32 + lane), so values land in the tile lane-strided;
//   - codes (FOR: v - min, DELTA: differences, DYN: v), width, lane-contiguous
//     packing in place, and a deferred decoupled look-back for cw (D-4): item k
//     is stored when the warp reaches item k + NW.
// Halves whose window does not fit a slot, unsorted positions, data blocks
// wider than 32 bits and the data remainder fall back to reads from global
// memory (read_row / funnel over two 32-bit loads).
#pragma once
#include "common.cuh"
#include "launch.h"
#include "positions.cuh"
#include "project.cuh"
#include "tma.cuh"

namespace ms {

constexpr uint32_t kWinSlotBytes = 14336;  // one half-block window (BJ.c5: 8-9 blocks x 1280 B)

struct WinHdr {
  uint64_t p_first, p_last, row0;  // positions range of the item, first row of block b_lo (global)
  uint64_t h_ref;                  // lane i: reference of block b_lo + i (FOR)
  uint64_t c0;                     // cw[b_lo]
  uint32_t hdr;                    // lane i: (cw[b_lo+i] - c0) << 7 | width
  bool ok;
};

template <int PER>
__device__ __forceinline__ void win_headers(const ColView& data, const uint64_t* T, uint64_t row_offset,
                                            uint32_t lane, WinHdr& W) {
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
  W.row0 = row_offset + (b_lo << data.log2B);
  if (W.ok) {
    const uint64_t bj = b_lo + lane;
    W.c0 = __ldg(data.cw + b_lo);
    if (bj < data.nb) {
      const uint32_t a = __ldg(data.cw + bj);
      const uint32_t a1 = __ldg(data.cw + bj + 1);
      W.hdr = ((uint32_t)(a - W.c0) << 7) | (a1 - a);
      if (data.format == MS_FOR_BP) W.h_ref = __ldg(data.ref + bj);
    }
  }
}

// the slot window of ranks [r0, r0 + n) of the tile: blocks [ba, bb] (window-relative)
struct HalfWin {
  uint64_t pa, pb;  // first and last position of the half (sorted: every position lies in between)
  uint32_t ba, cwa, bytes;
  bool ok;
};

__device__ __forceinline__ HalfWin half_window(const ColView& data, const WinHdr& W, const uint64_t* T,
                                               uint32_t r0, uint32_t n) {
  HalfWin H{0, 0, 0, 0, 0, false};
  const uint64_t pa = T[pidx(r0)], pb = T[pidx(r0 + n - 1)];
  const bool sorted = W.ok && pa >= W.p_first && pb >= pa && pb <= W.p_last;
  const uint32_t ba = sorted ? (uint32_t)((pa - W.row0) >> data.log2B) & 31 : 0u;
  const uint32_t bb = sorted ? (uint32_t)((pb - W.row0) >> data.log2B) & 31 : 0u;
  const uint32_t ha = __shfl_sync(kFull, W.hdr, ba), hb = __shfl_sync(kFull, W.hdr, bb);
  if (!sorted) return H;
  H.pa = pa;
  H.pb = pb;
  H.ba = ba;
  H.cwa = ha >> 7;
  const uint64_t bytes = (uint64_t)((hb >> 7) + (hb & 127) - (ha >> 7)) * (data.B / 8);
  H.bytes = (uint32_t)bytes;
  H.ok = bytes <= kWinSlotBytes;
  return H;
}

// gather ranks r0 + q*32 + lane, q < n/32, from the slot (or global memory)
__device__ __forceinline__ void win_gather(const ColView& data, uint64_t* T, const WinHdr& W, const HalfWin& H,
                                           const uint32_t* slot, uint32_t r0, uint32_t n, uint64_t row_offset,
                                           uint32_t lane, uint32_t* err) {
  const uint32_t dmask = data.B - 1;
  const uint32_t* g32 = reinterpret_cast<const uint32_t*>(data.payload) + ((W.c0 * data.B) >> 5);
  for (uint32_t q = 0; q < n / 32; ++q) {
    const uint32_t i = r0 + q * 32 + lane;
    const uint64_t p = T[pidx(i)];
    const bool inw = H.ok ? (p - H.pa <= H.pb - H.pa) : W.ok && (p - W.p_first <= W.p_last - W.p_first);
    const uint32_t rel = inw ? (uint32_t)(p - W.row0) : 0u;
    const uint32_t bsel = (rel >> data.log2B) & 31;
    const uint32_t h = __shfl_sync(kFull, W.hdr, bsel);
    const uint64_t rf = data.format == MS_FOR_BP ? __shfl_sync(kFull, W.h_ref, bsel) : 0ull;
    const uint32_t w = h & 127;
    uint64_t v;
    if (!inw || w > 32) {
      v = read_row_checked(data, p, row_offset, err);
    } else {
      const uint32_t bit = (h >> 7) * data.B + (rel & dmask) * w;  // window-relative
      uint32_t lo, hi;
      if (H.ok) {
        const uint32_t sb = bit - H.cwa * data.B;  // slot-relative
        const uint32_t k = sb >> 5, s = sb & 31;
        lo = w ? slot[k] : 0u;
        hi = (s + w > 32) ? slot[k + 1] : 0u;
        v = rf + (uint64_t)(__funnelshift_r(lo, hi, s) & (uint32_t)((1ull << w) - 1));
      } else {
        const uint32_t k = bit >> 5, s = bit & 31;
        lo = w ? __ldg(g32 + k) : 0u;
        hi = (s + w > 32) ? __ldg(g32 + k + 1) : 0u;
        v = rf + (uint64_t)(__funnelshift_r(lo, hi, s) & (uint32_t)((1ull << w) - 1));
      }
    }
    T[pidx(i)] = v;
  }
}

template <int PER>
__global__ void __launch_bounds__(32) project_win_kernel(ColView pos, ColView data, uint64_t row_offset, PosEnc e,
                                                         uint64_t n_full, uint64_t* status, uint32_t* err) {
  constexpr uint32_t G = 32 * PER;
  constexpr uint32_t H2 = G / 2;
  constexpr uint32_t TS = tile_slots(G);
  extern __shared__ __align__(128) uint64_t pw_sm[];
  __shared__ __align__(8) uint64_t bars[2];
  const uint32_t lane = threadIdx.x;
  uint32_t* slots = reinterpret_cast<uint32_t*>(pw_sm);  // 2 x kWinSlotBytes
  uint64_t* tiles = pw_sm + 2 * kWinSlotBytes / 8;       // 3 x TS
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  const uint64_t NW = gridDim.x;
  uint64_t item = blockIdx.x;
  if (item >= n_full) return;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncwarp();
  uint32_t phase[2] = {0u, 0u};

  auto decode = [&](uint64_t it, uint64_t* T) {
    const uint32_t cw0 = __ldg(pos.cw + it), wp = __ldg(pos.cw + it + 1) - cw0;
    const uint64_t bref = __ldg(pos.ref + it);
    const uint64_t bit0 = (uint64_t)cw0 * G + (uint64_t)PER * lane * wp;
    uint64_t acc = 0;
    uint64_t p[PER];
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
    const uint64_t base = bref + incl - acc;
#pragma unroll
    for (int q = 0; q < PER; ++q) T[pidx(PER * lane + q)] = p[q] + base;
    __syncwarp();
  };
  auto issue = [&](const WinHdr& W, const HalfWin& H, int s) {
    if (!H.ok || !H.bytes) return;
    if (lane == 0) {
      const char* src = reinterpret_cast<const char*>(data.payload) + (W.c0 + H.cwa) * (uint64_t)(data.B / 8);
      mbar_arrive_tx(&bars[s], H.bytes);
      bulk_g2s(slots + s * (kWinSlotBytes / 4), src, H.bytes, &bars[s]);
    }
  };
  auto wait = [&](const HalfWin& H, int s) {
    if (!H.ok || !H.bytes) return;
    mbar_wait(&bars[s], phase[s]);
    phase[s] ^= 1u;
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

  // prologue
  int t_cur = 0, t_nxt = 1, t_prev = 2;
  WinHdr W;
  decode(item, tiles + t_cur * TS);
  win_headers<PER>(data, tiles + t_cur * TS, row_offset, lane, W);
  HalfWin H0 = half_window(data, W, tiles + t_cur * TS, 0, H2);
  issue(W, H0, 0);
  uint64_t prev = ~0ull, prev_ref = 0;
  uint32_t prev_w = 0;
  while (true) {
    uint64_t* T = tiles + t_cur * TS;
    const uint64_t nxt = item + NW;
    const bool has_nxt = nxt < n_full;
    // second half's window in flight while the first half is gathered
    const HalfWin H1 = half_window(data, W, T, H2, H2);
    issue(W, H1, 1);
    wait(H0, 0);
    win_gather(data, T, W, H0, slots, 0, H2, row_offset, lane, err);
    __syncwarp();
    // the next item's positions and headers while the second half's copy is in flight
    WinHdr Wn;
    HalfWin Hn0{0, 0, 0, 0, 0, false};
    if (has_nxt) {
      decode(nxt, tiles + t_nxt * TS);
      win_headers<PER>(data, tiles + t_nxt * TS, row_offset, lane, Wn);
      Hn0 = half_window(data, Wn, tiles + t_nxt * TS, 0, H2);
      issue(Wn, Hn0, 0);  // slot 0 is free: the first half is gathered
    }
    wait(H1, 1);
    win_gather(data, T, W, H1, slots + kWinSlotBytes / 4, H2, H2, row_offset, lane, err);
    __syncwarp();
    // encode, publish; store the previous item
    if (!is_block) {
      uint64_t* dst = e.payload + item * G;
      for (uint32_t i = lane; i < G; i += 32) dst[i] = T[pidx(i)];
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
      if (prev != ~0ull) store(prev, prev_w, prev_ref, tiles + t_prev * TS);
      prev = item;
      prev_w = w;
      prev_ref = ref;
      const int t = t_prev;
      t_prev = t_cur;
      t_cur = t;  // the stored tile becomes free
    }
    if (!has_nxt) break;
    const int t = t_cur;
    t_cur = t_nxt;
    t_nxt = t;
    W = Wn;
    H0 = Hn0;
    item = nxt;
  }
  if (prev != ~0ull) store(prev, prev_w, prev_ref, tiles + t_prev * TS);
}

}  // namespace ms
