// positions.cuh — output-side buffer layer of select: turn the
// select bit mask into the positions column in any output format.
//
// Output ranks are cut into items of G ranks: G = B for block formats (one
// item = one output block), G = 512 otherwise. The segment scan that computes
// each segment's output rank also finds, for every item starting inside the
// segment, the item's first position (gstart). The encoder then runs one warp
// per item, items taken in order from a ticket: expand the item's positions
// from the mask starting at gstart into a shared-memory tile (the paper's
// L1-resident output buffer), compute the block's width (DELTA: widest
// difference, FOR: ebw(max - min), DYN: ebw(max)), get the exclusive
// prefix of the widths by decoupled look-back (cw, D-4), pack and store whole
// words. The final partial block goes to the uncompressed remainder.
#pragma once
#include "common.cuh"
#include "launch.h"

namespace ms {

// Shared-memory tile index with one pad slot every 16 entries: keeps both the
// lane-consecutive (16 entries per lane) and the lane-strided access patterns
// of the 8-byte tile free of bank conflicts.
__device__ __forceinline__ uint32_t pidx(uint32_t i) { return i + (i >> 4); }
__host__ __device__ constexpr uint32_t tile_slots(uint32_t G) { return G + G / 16 + 2; }

// ------------------------------------------------------------------ sources
// select: expand the item's positions from the mask, starting at gstart[item]
struct MaskSource {
  const uint32_t* bits;
  uint64_t NS;
  const uint64_t* gstart;
  uint64_t row_offset;
  __device__ __forceinline__ void load(uint32_t item, uint64_t r0, uint32_t cnt, uint64_t* P, uint32_t lane,
                                       uint32_t* err) const {
    const uint64_t n_words = NS * kSegWords;
    const uint64_t row = __ldg(gstart + item) - row_offset;
    uint64_t wi = row >> 5;
    uint32_t first_mask = ~0u << (row & 31);
    uint32_t got = 0;
    while (got < cnt && wi < n_words) {
      uint32_t wv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint64_t m = wi + q * 32 + lane;
        wv[q] = m < n_words ? __ldg(bits + m) : 0u;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t word = wv[q];
        if (q == 0 && lane == 0) word &= first_mask;
        const uint32_t pc = __popc(word);
        uint32_t incl = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(kFull, incl, o);
          if (lane >= (uint32_t)o) incl += t;
        }
        uint32_t k = got + incl - pc;
        const uint64_t base = row_offset + (wi + q * 32 + lane) * 32;
        while (word && k < cnt) {
          const int b = __ffs(word) - 1;
          word &= word - 1;
          P[pidx(k++)] = base + b;
        }
        got += __shfl_sync(kFull, incl, 31);
      }
      first_mask = ~0u;
      wi += 128;
    }
    __syncwarp();
  }
};

// project: decode the item's positions (ranks r0 .. r0+cnt of the
// positions column), then gather data[p - row_offset] for each. Positions:
// DELTA_BP with B == item size (block-aligned: warp prefix sum of the
// deltas), or any O(1)-addressable format. Data: O(1) formats; the block
// headers (cw, ref) of the data window are loaded once per warp (lane j ->
// block b_lo + j) and broadcast by shuffles; each lane then has its 16
// payload loads in flight at once.
template <int BATCH>
struct ProjectSource {
  ColView pos;
  ColView data;
  uint64_t row_offset;
  uint32_t prefetch;  // bulk-prefetch the data window into L2 before gathering
  // the gathered value of rank i (position p) goes to f(i, p, v); load() stores it in P
  struct Store {
    uint64_t* P;
    __device__ __forceinline__ void operator()(uint32_t i, uint64_t, uint64_t v) const { P[pidx(i)] = v; }
  };
  __device__ __forceinline__ void load(uint32_t item, uint64_t r0, uint32_t cnt, uint64_t* P, uint32_t lane,
                                       uint32_t* err) const {
    load_with(item, r0, cnt, P, lane, err, Store{P});
  }
  // positions of ranks [r0, r0 + cnt) into P, then each one's data value to f
  template <class F>
  __device__ __forceinline__ void load_with(uint32_t item, uint64_t r0, uint32_t cnt, uint64_t* P, uint32_t lane,
                                            uint32_t* err, const F& f) const {
    // ---- positions
    if (pos.format == MS_DELTA_BP && r0 + cnt <= (pos.nb << pos.log2B)) {  // block-aligned: B == G (host checks)
      const uint64_t b = r0 >> pos.log2B;
      const uint32_t cw0 = __ldg(pos.cw + b);
      const uint32_t w = __ldg(pos.cw + b + 1) - cw0;
      const uint64_t bit0 = (uint64_t)cw0 * pos.B;
      const uint32_t per = pos.B / 32;  // consecutive codes per lane
      uint64_t acc = 0;
      if (per == 16 && w >= 1 && w <= 8) {  // the lane's <= 128 + 31 bits: five loads issued together
        const uint64_t lb = bit0 + (uint64_t)lane * 16 * w;
        const uint32_t* w32 = reinterpret_cast<const uint32_t*>(pos.payload) + (lb >> 5);
        const uint32_t sft = (uint32_t)(lb & 31), nwd = (sft + 16 * w + 31) >> 5;
        const uint32_t x0 = __ldg(w32), x1 = nwd > 1 ? __ldg(w32 + 1) : 0u, x2 = nwd > 2 ? __ldg(w32 + 2) : 0u,
                       x3 = nwd > 3 ? __ldg(w32 + 3) : 0u, x4 = nwd > 4 ? __ldg(w32 + 4) : 0u;
        uint64_t win = ((uint64_t)x1 << 32 | x0) >> sft;
        uint32_t avail = 64 - sft, k = 2;
        const uint64_t m = (1ull << w) - 1;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (avail < w) {
            const uint32_t nx = k == 2 ? x2 : (k == 3 ? x3 : x4);
            win |= (uint64_t)nx << avail;
            avail += 32;
            ++k;
          }
          acc += win & m;
          P[pidx(lane * 16 + q)] = acc;
          win >>= w;
          avail -= w;
        }
      } else {
        for (uint32_t q = 0; q < per; ++q) {
          acc += unpack_at(pos.payload, bit0 + (uint64_t)(lane * per + q) * w, w);
          P[pidx(lane * per + q)] = acc;
        }
      }
      uint64_t incl = warp_incl_scan(acc);
      const uint64_t base = __ldg(pos.ref + b) + incl - acc;
      __syncwarp();
      for (uint32_t q = 0; q < per; ++q) P[pidx(lane * per + q)] += base;
    } else {
      for (uint32_t i = lane; i < cnt; i += 32) P[pidx(i)] = read_row(pos, r0 + i);
    }
    __syncwarp();
    // ---- gather
    if (data.format == MS_DYN_BP || data.format == MS_FOR_BP) {
      const uint64_t main_rows = data.nb << data.log2B;
      const uint64_t p_first = P[pidx(0)], p_last = P[pidx(cnt - 1)];
      const uint64_t plo = p_first - row_offset, phi = p_last - row_offset;  // sorted positions
      const uint64_t b_lo = plo >> data.log2B;
      const bool window = p_first >= row_offset && phi < main_rows && ((phi >> data.log2B) - b_lo) < 32 &&
                          p_last >= p_first;
      uint32_t h_cw = 0;
      uint64_t h_ref = 0;
      if (window) {
        const uint64_t bj = b_lo + lane;
        if (bj <= data.nb) h_cw = __ldg(data.cw + bj);
        if (bj < data.nb && data.format == MS_FOR_BP) h_ref = __ldg(data.ref + bj);
      }
      const uint32_t h_cw_next = __shfl_down_sync(kFull, h_cw, 1);
      uint32_t h_last = 0;
      if (window) {
        const uint64_t bj = b_lo + 32;
        h_last = (lane == 31 && bj <= data.nb) ? __ldg(data.cw + bj) : 0u;
      }
      const uint32_t h_cw1 = lane == 31 ? h_last : h_cw_next;
      if (window && prefetch) {  // one bulk L2 prefetch of the whole payload window
        const uint32_t c_lo = __shfl_sync(kFull, h_cw, 0);
        const uint32_t nblk = (uint32_t)((phi >> data.log2B) - b_lo) + 1;
        const uint32_t c_hi = __shfl_sync(kFull, h_cw1, (nblk - 1) & 31);
        const uint64_t bytes = (uint64_t)(c_hi - c_lo) * (data.B / 8);
        if (lane == 0 && bytes >= 16) {
          const uint64_t* a = data.payload + (uint64_t)c_lo * (data.B / 64);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"((uint32_t)(bytes & ~15ull))
                       : "memory");
        }
      }
      for (uint32_t i0 = 0; i0 < cnt; i0 += 32 * BATCH) {
        uint64_t v[BATCH], pp[BATCH];
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const uint32_t i = i0 + q * 32 + lane;
          const uint64_t p = i < cnt ? P[pidx(i)] : row_offset;
          pp[q] = p;
          const bool ok = p >= row_offset && p - row_offset < data.n;
          if (i < cnt && !ok) atomicOr(err, err_bit(MS_E_RANGE));
          const uint64_t r = ok ? p - row_offset : 0;
          const uint64_t b = r >> data.log2B;
          uint32_t cw0 = 0, w = 0;
          uint64_t rf = 0;
          const bool in_win = window && b >= b_lo && b - b_lo < 32 && r < main_rows;  // (unsorted positions)
          if (window) {
            const int src = (int)(b - b_lo) & 31;
            cw0 = __shfl_sync(kFull, h_cw, src);
            w = __shfl_sync(kFull, h_cw1, src) - cw0;
            rf = __shfl_sync(kFull, h_ref, src);
          }
          if (in_win) {
          } else if (r < main_rows) {
            cw0 = __ldg(data.cw + b);
            w = __ldg(data.cw + b + 1) - cw0;
            rf = data.format == MS_FOR_BP ? __ldg(data.ref + b) : 0ull;
          } else {
            cw0 = 0; w = 0;
            rf = __ldg(data.rem + (r - main_rows));
          }
          if (data.format == MS_DYN_BP) rf = (r < main_rows) ? 0ull : rf;
          v[q] = rf + unpack_at(data.payload, (uint64_t)cw0 * data.B + (r & (data.B - 1)) * (uint64_t)w, w);
        }
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const uint32_t i = i0 + q * 32 + lane;
          if (i < cnt) f(i, pp[q], v[q]);
        }
      }
    } else if (data.format == MS_STATIC_BP || data.format == MS_UNCOMPR) {
      // O(1) addresses (bit r * w): a bulk L2 prefetch of the window between the
      // first and last position (sorted positions; at most kStaticWindow bytes),
      // then BATCH independent loads in flight per lane
      constexpr uint64_t kStaticWindow = 32768;
      const uint32_t w = data.format == MS_STATIC_BP ? data.w : 64u;
      const uint64_t p_first = P[pidx(0)], p_last = P[pidx(cnt - 1)];
      if (prefetch && lane == 0 && p_first >= row_offset && p_last >= p_first && p_last - row_offset < data.n) {
        const uint64_t a_lo = (((p_first - row_offset) * w) >> 6) & ~1ull;  // 16-byte aligned word
        const uint64_t a_hi = (((p_last - row_offset + 1) * w + 63) >> 6);
        const uint64_t bytes = ((a_hi - a_lo) * 8) & ~15ull;
        if (bytes >= 16 && bytes <= kStaticWindow)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(data.payload + a_lo), "r"((uint32_t)bytes)
                       : "memory");
      }
      for (uint32_t i0 = 0; i0 < cnt; i0 += 32 * BATCH) {
        uint64_t v[BATCH], pp[BATCH];
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const uint32_t i = i0 + q * 32 + lane;
          const uint64_t p = i < cnt ? P[pidx(i)] : row_offset;
          pp[q] = p;
          const bool ok = p >= row_offset && p - row_offset < data.n;
          if (i < cnt && !ok) atomicOr(err, err_bit(MS_E_RANGE));
          const uint64_t r = ok ? p - row_offset : 0;
          v[q] = !ok ? 0ull : (w == 64 ? __ldg(data.payload + r) : unpack_at(data.payload, r * w, w));
        }
#pragma unroll
        for (int q = 0; q < BATCH; ++q) {
          const uint32_t i = i0 + q * 32 + lane;
          if (i < cnt) f(i, pp[q], v[q]);
        }
      }
    } else {
      for (uint32_t i = lane; i < cnt; i += 32) {
        const uint64_t p = P[pidx(i)];
        uint64_t v = 0;
        if (p < row_offset || p - row_offset >= data.n) atomicOr(err, err_bit(MS_E_RANGE));
        else v = read_row(data, p - row_offset);
        f(i, p, v);
      }
    }
    __syncwarp();
  }
};

// Output-side buffer layer, one warp per item (G output rows): the Source fills
// the item's values into the warp's shared-memory tile (the paper's L1-resident
// output buffer), the block width is published as a look-back aggregate, the
// exclusive prefix resolved, and the block packed into whole words. (A
// two-tile software pipeline that defers the look-back was measured slower:
// it halves occupancy, and these kernels are latency-bound.)
// Dynamic shared memory: warps x G uint64.
template <class Src>
__device__ __forceinline__ void encode_finish(const PosEnc& e, uint32_t item, uint64_t* P, uint32_t cnt,
                                              uint32_t w, uint64_t rmin, uint64_t* status, uint32_t* err,
                                              uint32_t lane) {
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  const uint64_t r0 = (uint64_t)item * e.G;
  if (!is_block) {
    if (e.format == MS_UNCOMPR) {
      for (uint32_t i = lane; i < cnt; i += 32) e.payload[r0 + i] = P[pidx(i)];
    } else if (e.format == MS_RLE) {
      for (uint32_t i = lane; i < cnt; i += 32) {
        e.payload[2 * (r0 + i)] = P[pidx(i)];
        e.payload[2 * (r0 + i) + 1] = 1;
      }
    } else {  // STATIC_BP: item = ranks [512k, 512k+cnt) at bit 512k*w (word aligned)
      const uint32_t ws = e.w;
      const uint64_t mask = low_mask(ws);
      const uint64_t wbase = (uint64_t)item * 8 * ws;
      const uint32_t nwords = (uint32_t)(((uint64_t)cnt * ws + 63) / 64);
      const uint32_t magic = 0xffffffffu / ws + 1u;
      for (uint32_t m = lane; m < nwords; m += 32) {
        const uint32_t bit0 = m * 64;
        uint32_t j = div_small(bit0, ws, magic);
        const uint32_t sft = bit0 - j * ws;
        uint64_t acc = (P[pidx(j)] & mask) >> sft;
        for (++j; j < cnt; ++j) {
          const uint32_t jb = j * ws;
          if (jb >= bit0 + 64) break;
          acc |= (P[pidx(j)] & mask) << (jb - bit0);
        }
        e.payload[wbase + m] = acc;
      }
    }
    return;
  }
  if (cnt < e.G) {  // final partial block -> uncompressed remainder
    for (uint32_t i = lane; i < cnt; i += 32) e.rem[i] = P[pidx(i)];
    return;
  }
  const uint64_t E = lookback_resolve(status, item, w);
  if (lane == 0) {
    if (E + w > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
    e.cw[item + 1] = (uint32_t)(E + w);
    if (e.format == MS_DELTA_BP) e.ref[item] = P[pidx(0)];
    if (e.format == MS_FOR_BP) e.ref[item] = rmin;
  }
  if (!w) return;
  const uint64_t wbase = E * (e.G >> 6);
  const uint32_t nwords = (e.G >> 6) * w;
  const uint32_t magic = 0xffffffffu / w + 1u;
  for (uint32_t m = lane; m < nwords; m += 32) {
    const uint32_t bit0 = m * 64;
    uint32_t j = div_small(bit0, w, magic);
    const uint32_t sft = bit0 - j * w;
    auto code = [&](uint32_t i) -> uint64_t {
      if (e.format == MS_DELTA_BP) return i ? P[pidx(i)] - P[pidx(i - 1)] : 0ull;
      if (e.format == MS_FOR_BP) return P[pidx(i)] - rmin;
      return P[pidx(i)];
    };
    uint64_t acc = code(j) >> sft;
    for (++j; j < cnt; ++j) {
      const uint32_t jb = j * w;
      if (jb >= bit0 + 64) break;
      acc |= code(j) << (jb - bit0);
    }
    e.payload[wbase + m] = acc;
  }
}

template <class Src>
__global__ void __launch_bounds__(128) warp_encode_kernel(Src src, PosEnc e, uint64_t n_items, uint64_t* status,
                                                          uint32_t* ticket, uint32_t* err) {
  extern __shared__ __align__(16) uint64_t enc_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t* P = enc_sm + (uint64_t)wid * tile_slots(e.G);
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  while (true) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(ticket, 1u);
    item = __shfl_sync(kFull, item, 0);
    if (item >= n_items) break;
    const uint64_t r0 = (uint64_t)item * e.G;
    const uint32_t cnt = (uint32_t)min((uint64_t)e.G, e.n_out - r0);
    src.load(item, r0, cnt, P, lane, err);
    uint32_t w = 0;
    uint64_t rmin = 0;
    if (is_block && cnt == e.G) {
      uint64_t mx = 0;
      if (e.format == MS_DELTA_BP) {
        for (uint32_t i = lane; i < cnt; i += 32) {
          const uint64_t d = i ? P[pidx(i)] - P[pidx(i - 1)] : 0ull;
          mx = d > mx ? d : mx;
        }
        mx = warp_max(mx);
      } else {  // FOR: ebw(max - min); DYN: ebw(max) (values need not be sorted: project)
        uint64_t lo = ~0ull, hi = 0;
        for (uint32_t i = lane; i < cnt; i += 32) {
          const uint64_t x = P[pidx(i)];
          lo = x < lo ? x : lo;
          hi = x > hi ? x : hi;
        }
        hi = warp_max(hi);
        if (e.format == MS_FOR_BP) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const uint64_t t = __shfl_xor_sync(kFull, lo, o);
            lo = t < lo ? t : lo;
          }
          mx = hi - lo;
          rmin = lo;
        } else {
          mx = hi;
        }
      }
      w = ebw64(mx);
      lookback_publish(status, item, w);
    }
    encode_finish<Src>(e, item, P, cnt, w, rmin, status, err, lane);
    __syncwarp();
  }
}

// Stream lane j's PER codes c[q] (< 2^w, w <= 64) into the u32 words of a
// block at bits [PER*j*w, PER*(j+1)*w): zero the block's B*w/32 words, then
// plain stores inside the lane's range and atomicOr on the (at most two) words
// shared with its neighbours. All 32 lanes call.
template <int PER>
__device__ __forceinline__ void pack_lane_codes(uint32_t* buf, const uint64_t (&c)[PER], uint32_t w, uint32_t lane) {
  const uint32_t nw32 = PER * w;
  for (uint32_t i = lane; i < nw32; i += 32) buf[i] = 0;
  __syncwarp();
  stream_codes<PER>(buf, c, w, PER * lane * w);
  __syncwarp();
}

// Output-side buffer layer with a deferred look-back, one warp per item of
// G = 32*PER ranks (G <= 512), two tiles per warp: the Source fills the item's
// values into tile A; lane j takes ranks [PER*j, PER*j + PER) into registers,
// forms the codes (DELTA: differences, FOR: minus the block minimum, DYN: the
// values) and the block width, packs the block in place (pack_lane_codes) and
// publishes the width as its look-back aggregate. Only then does the warp
// resolve the exclusive width prefix of its PREVIOUS item — whose predecessors
// have had a whole item's gather to publish — and store that block from tile B
// with coalesced 64-bit stores at word cw[k] * G / 64. Non-block formats and
// the final partial block need no prefix and are written directly.
template <class Src, int PER>
__global__ void __launch_bounds__(128) warp_encode_deferred_kernel(Src src, PosEnc e, uint64_t n_items,
                                                                   uint64_t* status, uint32_t* ticket,
                                                                   uint32_t* err) {
  constexpr uint32_t G = 32 * PER;
  extern __shared__ __align__(16) uint64_t enc_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t* tiles = enc_sm + (uint64_t)wid * 2 * tile_slots(G);
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  uint64_t prev = ~0ull, prev_ref = 0;
  uint32_t prev_w = 0, cur = 0;
  auto store = [&](uint64_t item, uint32_t w, uint64_t ref, const uint64_t* T) {
    const uint64_t E = lookback_resolve(status, item, w);
    if (lane == 0) {
      if (E + w > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
      e.cw[item + 1] = (uint32_t)(E + w);
      if (e.format != MS_DYN_BP) e.ref[item] = ref;
    }
    uint64_t* dst = e.payload + E * (G / 64);
    const uint32_t nw64 = G / 64 * w;
    for (uint32_t m = lane; m < nw64; m += 32) dst[m] = T[m];
    __syncwarp();
  };
  while (true) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(ticket, 1u);
    item = __shfl_sync(kFull, item, 0);
    if (item >= n_items) break;
    uint64_t* P = tiles + cur * tile_slots(G);
    const uint64_t r0 = (uint64_t)item * G;
    const uint32_t cnt = (uint32_t)min((uint64_t)G, e.n_out - r0);
    src.load(item, r0, cnt, P, lane, err);
    if (!is_block || cnt < G) {  // no prefix needed
      encode_finish<Src>(e, item, P, cnt, 0, 0, status, err, lane);
      __syncwarp();
      continue;
    }
    uint64_t c[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) c[q] = P[pidx(lane * PER + q)];
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
    pack_lane_codes<PER>(reinterpret_cast<uint32_t*>(P), c, w, lane);
    lookback_publish(status, item, w);
    if (prev != ~0ull) store(prev, prev_w, prev_ref, tiles + (cur ^ 1) * tile_slots(G));
    prev = item;
    prev_w = w;
    prev_ref = ref;
    cur ^= 1;
  }
  if (prev != ~0ull) store(prev, prev_w, prev_ref, tiles + (cur ^ 1) * tile_slots(G));
}

// Slot variant of the output-side buffer layer (no look-back at all): one tile
// per warp, items in grid-stride order; a full block is packed at its own width
// and written to its fixed-size slot (slot_words u64), its width to wk[k] and its
// reference to ref[k]; the scan of wk gives cw, and pos_copy_kernel moves each
// block to word cw[k] * G / 64. Non-block formats and the final partial block
// are written directly.
// One full block of G = 32*PER values in the tile P (project's gathered values or
// select's positions) re-encoded at its own width into its fixed-size slot
// (slot_words u64): lane j takes ranks [PER*j, PER*j + PER) into registers,
// forms the codes (DELTA: differences, FOR: minus the block minimum, DYN: the
// values), packs them in place (pack_lane_codes) and stores the block; the width
// goes to wk[item], the reference to ref[item].
template <int PER>
__device__ __forceinline__ void slot_encode_block(const PosEnc& e, uint64_t item, uint64_t* P,
                                                  uint64_t* __restrict__ slots, uint32_t slot_words,
                                                  uint32_t* __restrict__ wk, uint32_t* err, uint32_t lane) {
  constexpr uint32_t G = 32 * PER;
  uint64_t c[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) c[q] = P[pidx(lane * PER + q)];
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
  pack_lane_codes<PER>(reinterpret_cast<uint32_t*>(P), c, w, lane);
  const uint32_t nw64 = G / 64 * w;
  if (nw64 > slot_words) {  // a width above the host's bound (an understated hint)
    if (lane == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
  } else {
    uint64_t* dst = slots + item * slot_words;
    for (uint32_t m = lane; m < nw64; m += 32) dst[m] = P[m];
  }
  if (lane == 0) {
    wk[item] = w;
    if (e.format != MS_DYN_BP) e.ref[item] = ref;
  }
  __syncwarp();
}

// Slot variant of the output-side buffer layer (no look-back at all): one tile
// per warp, items in grid-stride order; a full block is packed at its own width
// and written to its fixed-size slot (slot_encode_block); the scan of wk gives
// cw, and pos_copy_kernel moves each block to word cw[k] * G / 64. Non-block
// formats and the final partial block are written directly.
template <class Src, int PER>
__global__ void __launch_bounds__(128) warp_encode_slot_kernel(Src src, PosEnc e, uint64_t n_items,
                                                               uint64_t* __restrict__ slots, uint32_t slot_words,
                                                               uint32_t* __restrict__ wk, uint32_t* err) {
  constexpr uint32_t G = 32 * PER;
  extern __shared__ __align__(16) uint64_t enc_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t* P = enc_sm + (uint64_t)wid * tile_slots(G);
  const bool is_block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  const uint64_t NW = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t item = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wid; item < n_items; item += NW) {
    const uint64_t r0 = item * G;
    const uint32_t cnt = (uint32_t)min((uint64_t)G, e.n_out - r0);
    src.load((uint32_t)item, r0, cnt, P, lane, err);
    if (!is_block || cnt < G) {
      encode_finish<Src>(e, (uint32_t)item, P, cnt, 0, 0, nullptr, err, lane);
      __syncwarp();
      continue;
    }
    slot_encode_block<PER>(e, item, P, slots, slot_words, wk, err, lane);
  }
}

}  // namespace ms
