// posdelta.cuh — select's output-side buffer layer for the positions format the
// paper recommends for select outputs, DELTA_BP ("the output is always
// sorted"), straight from the select bit mask to the packed column
// (P:486-490), for block sizes B <= 512.
//
// Output block k holds output ranks [kB, kB + B); its first position gstart[k]
// comes from the segment scan. Three launches, none of which waits on another
// CTA (a look-back per block or per tile of blocks stalls whole CTAs on their
// predecessors, measured 3x slower on B200):
//   pos_width  one warp per block: w_k = ebw(max_j d_j), d_j = p_j - p_{j-1},
//              d_0 = 0 (D-6);
//   scan       exclusive prefix of w_k -> cw (D-4), the generic scan kernel;
//   pos_pack   one warp per block: the same walk, codes streamed into a
//              shared-memory copy of the block, stored with coalesced 64-bit
//              stores at word cw[k] * B / 64; cw[k+1], base = p_0 = gstart[k].
//              The final partial block goes raw to the remainder.
// Per block the walk is pd_item512 (B = 512, span < 512 words, i.e. selectivity
// above ~3.1 %: words in registers, set bits scattered by rank into shared
// memory, then 16 ranks per lane packed at a compile-time width),
// pd_fast_item (span <= kPdStageU32 words: words staged in shared memory, B/32
// ranks per lane located by a search) or, for sparse masks, the round-based
// walker pd_walk. No position is materialised outside the SM.
#pragma once
#include "common.cuh"
#include "launch.h"

namespace ms {

constexpr int kPdWarps = 8;  // warps per CTA (independent)
constexpr int kPdLaneWords = 8;
constexpr int kPdRoundWords = 32 * kPdLaneWords;
constexpr uint32_t kPdStageU32 = 1024;      // mask words staged per warp (also a slow block's pack buffer: 2B u32)
constexpr uint32_t kPdPackU32 = 16 * 16;    // a fast block: B/32 * w <= 16 * 15 u32
constexpr uint32_t kPdWarpU32 = kPdStageU32 + kPdPackU32;

// One walk over the mask for output block `item`: ranks [0, cnt) starting at
// relative row row0. PACK = false: returns the lane's max delta. PACK = true:
// writes the codes (width w) into buf (zeroed, u32 words), or, when raw !=
// nullptr, the global positions into raw[rank].
template <bool PACK>
__device__ __forceinline__ uint64_t pd_walk(const uint32_t* __restrict__ bits, uint64_t n_words, uint64_t row0,
                                            uint32_t cnt, uint32_t w, uint32_t* buf, uint64_t* raw,
                                            uint64_t row_offset, uint32_t lane, uint32_t* err) {
  const uint64_t wi = row0 >> 5;
  const uint32_t fmask = ~0u << (row0 & 31);
  uint64_t wb = wi & ~3ull;  // 16-byte aligned
  uint32_t got = 0;
  uint64_t carry = 0;  // 1 + last position of the previous rounds (0: none)
  uint64_t maxd = 0;
  while (got < cnt) {
    if (wb >= n_words) {  // fewer set bits than the scan counted
      if (lane == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
      break;
    }
    const uint64_t wl = wb + (uint64_t)kPdLaneWords * lane;
    uint32_t x[kPdLaneWords];
    if (wl + kPdLaneWords <= n_words) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(bits + wl));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(bits + wl) + 1);
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
      x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < kPdLaneWords; ++q) x[q] = wl + q < n_words ? __ldg(bits + wl + q) : 0u;
    }
    uint32_t c = 0;
    uint64_t lastp = 0;
#pragma unroll
    for (int q = 0; q < kPdLaneWords; ++q) {
      const uint64_t m = wl + q;
      if (m < wi) x[q] = 0;
      else if (m == wi) x[q] &= fmask;
      c += __popc(x[q]);
      if (x[q]) lastp = m * 32 + 32 - __clz(x[q]);
    }
    uint32_t inc = c;
    uint64_t mx = lastp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, inc, o);
      const uint64_t tm = __shfl_up_sync(kFull, mx, o);
      if (lane >= (uint32_t)o) {
        inc += t;
        mx = tm > mx ? tm : mx;
      }
    }
    const uint32_t total = __shfl_sync(kFull, inc, 31);
    const uint64_t round_last = __shfl_sync(kFull, mx, 31);
    uint64_t prev = __shfl_up_sync(kFull, mx, 1);
    if (lane == 0) prev = 0;
    prev = prev > carry ? prev : carry;
    uint32_t k = got + inc - c;
    if (c && k < cnt) {
      uint64_t acc = 0;
      uint32_t nb = 0, widx = 0;
      bool first = true;
      if (PACK && !raw) {
        const uint64_t o = (uint64_t)k * w;
        widx = (uint32_t)(o >> 5);
        nb = (uint32_t)(o & 31);
      }
      auto flush = [&](uint32_t v) {
        if (first) {
          atomicOr(buf + widx, v);
          first = false;
        } else {
          buf[widx] = v;
        }
        ++widx;
      };
      auto put = [&](uint32_t code, uint32_t cw_) {
        acc |= (uint64_t)code << nb;
        nb += cw_;
        if (nb >= 32) {
          flush((uint32_t)acc);
          acc >>= 32;
          nb -= 32;
        }
      };
#pragma unroll
      for (int q = 0; q < kPdLaneWords; ++q) {
        uint32_t word = x[q];
        const uint64_t rb = (wl + q) * 32;
        while (word && k < cnt) {
          const uint32_t bt = __ffs(word) - 1;
          word &= word - 1;
          const uint64_t p1 = rb + bt + 1;  // 1 + position
          const uint64_t d = k ? p1 - prev : 0ull;
          prev = p1;
          if (!PACK) {
            maxd = d > maxd ? d : maxd;
          } else if (raw) {
            raw[k] = p1 - 1 + row_offset;
          } else if (w <= 32) {
            put((uint32_t)d, w);
          } else {
            put((uint32_t)d, 32);
            put((uint32_t)(d >> 32), w - 32);
          }
          ++k;
        }
      }
      if (PACK && !raw && nb) atomicOr(buf + widx, (uint32_t)acc);
    }
    got += total;
    carry = round_last > carry ? round_last : carry;
    wb += kPdRoundWords;
  }
  return maxd;
}

// Fast block walk, for blocks whose mask span (first word of this block to the
// word of the next block's first position) fits the stage: lane j owns the
// PER = B/32 consecutive ranks [PER*j, PER*j + PER).
//   1. lane j loads C consecutive words [wa + C*j, +C) (16-byte loads), masks
//      the rows before the block's first position, stages them in shared
//      memory and counts their set bits; warp exclusive scan -> rank of each
//      lane's chunk;
//   2. lane j finds the chunk holding rank PER*j (binary search over the chunk
//      prefixes by shuffles), walks to its word and bit, then extracts PER
//      positions in order (32-bit, relative to word wa);
//   3. d_q = p_q - p_{q-1} (d_0 of lane j from lane j-1's last position, 0
//      for rank 0). The span bounds every delta by 32 * kPdStageU32 < 2^15.
// PACK = false: returns w = ebw(max d). PACK = true: streams lane j's codes —
// (AUTO_W: at the width it computes; else at the given w) —
// the contiguous bit range [PER*j*w, PER*(j+1)*w) — into buf (B*w/32 u32,
// zeroed here): plain stores inside the range, atomicOr on the two words it
// may share with its neighbours; returns w.
template <int PER, bool PACK, bool AUTO_W>
__device__ __forceinline__ uint32_t pd_after_stage(uint32_t cnt, uint32_t C, uint64_t wa, uint32_t w,
                                                   const uint32_t* stage, uint32_t* buf, uint32_t lane) {
  uint32_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, inc, o);
    if (lane >= (uint32_t)o) inc += t;
  }
  const uint32_t ex = inc - cnt;
  // 2. locate rank PER*j: the last lane L with ex_L <= r
  const uint32_t r = PER * lane;
  uint32_t L = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const uint32_t cand = L + step;
    const uint32_t exc = __shfl_sync(kFull, ex, cand & 31);
    if (cand < 32 && exc <= r) L = cand;
  }
  uint32_t skip = r - __shfl_sync(kFull, ex, L);
  uint32_t m = C * L;  // staged word index
  uint32_t cur = stage[m];
  while (true) {
    const uint32_t pc = __popc(cur);
    if (skip < pc) break;
    skip -= pc;
    cur = stage[++m];
  }
  for (; skip; --skip) cur &= cur - 1;
  uint32_t pos[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    while (!cur) cur = stage[++m];
    pos[q] = m * 32 + (__ffs(cur) - 1);
    cur &= cur - 1;
  }
  // 3. deltas
  const uint32_t prev_last = __shfl_up_sync(kFull, pos[PER - 1], 1);
  uint32_t d[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) d[q] = q ? pos[q] - pos[q - 1] : (lane ? pos[0] - prev_last : 0u);
  if (!PACK || AUTO_W) {
    uint32_t mx = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) mx = d[q] > mx ? d[q] : mx;
    mx = __reduce_max_sync(kFull, mx);
    w = 32 - __clz(mx);
    if (!PACK) return w;
  }
  // 4. pack (w <= 15)
  const uint32_t nw32 = PER * w;  // == B * w / 32
  for (uint32_t i = lane; i < nw32; i += 32) buf[i] = 0;
  __syncwarp();
  if (w) {
    const uint32_t o = PER * lane * w;
    uint32_t widx = o >> 5, nb = o & 31;
    uint32_t acc = 0;
    bool first = true;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      acc |= d[q] << nb;
      nb += w;
      if (nb >= 32) {
        if (first) {
          atomicOr(buf + widx, acc);
          first = false;
        } else {
          buf[widx] = acc;
        }
        ++widx;
        nb -= 32;
        acc = nb ? d[q] >> (w - nb) : 0u;
      }
    }
    if (nb) atomicOr(buf + widx, acc);
  }
  __syncwarp();
  return w;
}

template <int PER, bool PACK, bool AUTO_W = false>
__device__ __forceinline__ uint32_t pd_fast_item(const uint32_t* __restrict__ bits, uint64_t n_words, uint64_t row0,
                                                 uint64_t span_words, uint32_t w, uint32_t* stage, uint32_t* buf,
                                                 uint32_t lane) {
  const uint64_t wi = row0 >> 5;
  const uint32_t fmask = ~0u << (row0 & 31);
  const uint64_t wa = wi & ~3ull;
  const uint32_t need = (uint32_t)((wi - wa) + span_words);
  const uint32_t C = ((need + 127) / 128) * 4;  // words per lane, multiple of 4, 32*C >= need
  const uint32_t wi_rel = (uint32_t)(wi - wa);
  // 1. stage + count
  const uint64_t c0 = wa + (uint64_t)C * lane;
  uint4* st4 = reinterpret_cast<uint4*>(stage) + (C / 4) * lane;
  uint32_t cnt = 0;
  for (uint32_t q = 0; q < C; q += 4) {
    const uint64_t m = c0 + q;
    uint32_t x0, x1, x2, x3;
    if (m + 4 <= n_words) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(bits + m));
      x0 = a.x; x1 = a.y; x2 = a.z; x3 = a.w;
    } else {
      x0 = m < n_words ? __ldg(bits + m) : 0u;
      x1 = m + 1 < n_words ? __ldg(bits + m + 1) : 0u;
      x2 = m + 2 < n_words ? __ldg(bits + m + 2) : 0u;
      x3 = 0u;
    }
    if (m == wa) {  // the first four words hold the block start (wi - wa < 4)
      x0 = wi_rel > 0 ? 0u : x0 & fmask;
      x1 = wi_rel > 1 ? 0u : (wi_rel == 1 ? x1 & fmask : x1);
      x2 = wi_rel > 2 ? 0u : (wi_rel == 2 ? x2 & fmask : x2);
      x3 = wi_rel == 3 ? x3 & fmask : x3;
    }
    st4[q / 4] = make_uint4(x0, x1, x2, x3);
    cnt += __popc(x0) + __popc(x1) + __popc(x2) + __popc(x3);
  }
  __syncwarp();
  return pd_after_stage<PER, PACK, AUTO_W>(cnt, C, wa, w, stage, buf, lane);
}

// ---------------------------------------------------------------------------
// B = 512 blocks whose mask span fits 16 words per lane (first word of the
// block .. word of the next block's first position < 512 words, i.e. a
// selectivity above ~3.1 %). Count-distributed instead of rank-distributed:
//   1. lane j holds the 4G consecutive words [wa + 4Gj, +4G) in registers
//      (G = span / 128 rounded up; words outside [row0, rowE) masked), counts
//      their set bits; a warp scan gives the rank of the lane's first bit;
//   2. each lane scatters its positions (u16, relative to word wa) into
//      p16[rank] — one find-lowest / clear / store per set bit, no search;
//   3. lane j reads ranks [16j, 16j + 16), d_q = p_q - p_{q-1} (d_0 = 0,
//      D-6), w = ebw(max d) by a warp max, and packs its 16 codes at a
//      compile-time width: its bits are exactly the halfwords [jw, jw + w)
//      of the block (16w bits), so lanes never share a store.
// The span bounds every relative row by 512 * 32, so d < 2^14 and w <= 14.
template <int W>
__device__ __forceinline__ void pd_pack16(const uint32_t (&d)[16], uint16_t* out, uint32_t lane) {
  constexpr int NS = (16 * W + 31) / 32;
  uint32_t s[NS + 1];
#pragma unroll
  for (int i = 0; i <= NS; ++i) s[i] = 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int bit = q * W, wd = bit >> 5, sh = bit & 31;
    s[wd] |= d[q] << sh;
    if (sh + W > 32) s[wd + 1] |= d[q] >> (32 - sh);
  }
  if (W % 2 == 0) {
    uint32_t* o32 = reinterpret_cast<uint32_t*>(out) + lane * (W / 2);
#pragma unroll
    for (int i = 0; i < W / 2; ++i) o32[i] = s[i];
  } else {
    uint16_t* o = out + lane * W;
#pragma unroll
    for (int h = 0; h < W; ++h) o[h] = (uint16_t)(s[h >> 1] >> ((h & 1) * 16));
  }
}

// Ranks [16j, 16j + 16) -> d, w = ebw(max d), the block packed into p16 (in place).
__device__ __forceinline__ uint32_t pd_pack512(uint16_t* p16, uint32_t lane) {
  const uint4 a = reinterpret_cast<const uint4*>(p16)[2 * lane];
  const uint4 b = reinterpret_cast<const uint4*>(p16)[2 * lane + 1];
  const uint32_t pw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint32_t p[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    p[2 * i] = pw[i] & 0xffffu;
    p[2 * i + 1] = pw[i] >> 16;
  }
  const uint32_t prev = __shfl_up_sync(kFull, p[15], 1);
  uint32_t d[16];
  d[0] = lane ? p[0] - prev : 0u;
  uint32_t mx = d[0];
#pragma unroll
  for (int q = 1; q < 16; ++q) {
    d[q] = p[q] - p[q - 1];
    mx = d[q] > mx ? d[q] : mx;
  }
  mx = __reduce_max_sync(kFull, mx);
  const uint32_t w = 32u - __clz(mx);
  __syncwarp();
  switch (w) {
    case 1: pd_pack16<1>(d, p16, lane); break;
    case 2: pd_pack16<2>(d, p16, lane); break;
    case 3: pd_pack16<3>(d, p16, lane); break;
    case 4: pd_pack16<4>(d, p16, lane); break;
    case 5: pd_pack16<5>(d, p16, lane); break;
    case 6: pd_pack16<6>(d, p16, lane); break;
    case 7: pd_pack16<7>(d, p16, lane); break;
    case 8: pd_pack16<8>(d, p16, lane); break;
    case 9: pd_pack16<9>(d, p16, lane); break;
    case 10: pd_pack16<10>(d, p16, lane); break;
    case 11: pd_pack16<11>(d, p16, lane); break;
    case 12: pd_pack16<12>(d, p16, lane); break;
    case 13: pd_pack16<13>(d, p16, lane); break;
    case 14: pd_pack16<14>(d, p16, lane); break;
    default: break;  // w == 0 cannot happen past rank 0: positions are distinct
  }
  __syncwarp();
  return w;
}

// Steps 1-2 with C words per lane (compile time, so the words stay in
// registers): lane j holds words [wi + Cj, wi + Cj + C) of the S-word span.
template <int C>
__device__ __forceinline__ bool pd_scatter512(const uint32_t* __restrict__ bits, uint64_t row0, uint64_t rowE,
                                              uint16_t* p16, uint32_t lane) {
  const uint64_t wi = row0 >> 5;
  const uint32_t S = (uint32_t)((rowE >> 5) - wi) + 1u;
  const uint32_t lmask = (1u << (rowE & 31)) - 1u;  // rows before the next block's first position
  const uint32_t base = C * lane;
  const uint32_t* src = bits + wi + base;
  uint32_t x[C];
  uint32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) {
    uint32_t v = 0u;
    if (base + i < S) v = __ldg(src + i);
    if (base + i == S - 1) v &= lmask;
    x[i] = v;
  }
  if (lane == 0) x[0] &= ~0u << (row0 & 31);
#pragma unroll
  for (int i = 0; i < C; ++i) cnt += __popc(x[i]);
  uint32_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, inc, o);
    if (lane >= (uint32_t)o) inc += t;
  }
  if (__shfl_sync(kFull, inc, 31) != 512u) return false;  // the scan's block start disagrees with the mask
  // highest set bit first (one FLO per position, no bit reversal), from the
  // lane's last rank down
  uint32_t dst = (uint32_t)__cvta_generic_to_shared(p16 + inc - 1);  // the lane's last rank
#pragma unroll
  for (int i = C - 1; i >= 0; --i) {
    uint32_t word = x[i];
    const uint32_t rb = (base + i) * 32u;
    while (word) {
      uint32_t b, m;
      asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(word));         // highest set bit
      asm("bmsk.clamp.b32 %0, 0, %1;" : "=r"(m) : "r"(b));    // the bits below it
      word &= m;
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst), "h"((unsigned short)(rb + b)) : "memory");
      dst -= 2;
    }
  }
  __syncwarp();
  return true;
}

__device__ __forceinline__ uint32_t pd_item512(const uint32_t* __restrict__ bits, uint64_t row0, uint64_t rowE,
                                               uint16_t* p16, uint32_t lane, uint32_t* err) {
  const uint32_t S = (uint32_t)((rowE >> 5) - (row0 >> 5)) + 1u;  // <= 512 (caller)
  bool ok;
  switch ((S + 31) / 32) {
#define PD_C(c) case c: ok = pd_scatter512<c>(bits, row0, rowE, p16, lane); break;
    PD_C(1) PD_C(2) PD_C(3) PD_C(4) PD_C(5) PD_C(6) PD_C(7) PD_C(8)
    PD_C(9) PD_C(10) PD_C(11) PD_C(12) PD_C(13) PD_C(14) PD_C(15) PD_C(16)
#undef PD_C
    default: ok = false;
  }
  if (!ok) {
    if (lane == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
    return 0u;
  }
  return pd_pack512(p16, lane);
}

__device__ __forceinline__ bool pd_span(const uint64_t* gstart, uint64_t item, uint64_t n_items, uint64_t row0,
                                        uint64_t row_offset, uint64_t* span) {
  if (item + 1 >= n_items) return false;  // the last block's span is unknown: walker
  *span = ((__ldg(gstart + item + 1) - row_offset) >> 5) - (row0 >> 5) + 1;
  return *span + 4 <= kPdStageU32;
}

// A walk that packs every block at cw[k] = cwx[k] (exclusive prefix of the widths);
// launched for outputs without a full block, where it writes the raw remainder.
__global__ void __launch_bounds__(kPdWarps * 32) pos_pack_kernel(const uint32_t* __restrict__ bits,
                                                                 uint64_t n_words,
                                                                 const uint64_t* __restrict__ gstart,
                                                                 uint64_t row_offset, PosEnc e, uint64_t n_items,
                                                                 const uint64_t* __restrict__ cwx, uint32_t* err) {
  extern __shared__ __align__(16) uint32_t pd_sm[];  // per warp: stage | fast pack buffer
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* stage = pd_sm + (size_t)wid * kPdWarpU32;
  const uint32_t B = e.G;
  const uint64_t n_full = e.n_out / B;
  const uint64_t nwarps = (uint64_t)gridDim.x * kPdWarps;
  for (uint64_t item = (uint64_t)blockIdx.x * kPdWarps + wid; item < n_items; item += nwarps) {
    const uint64_t row0 = __ldg(gstart + item) - row_offset;
    if (item >= n_full) {  // final partial block -> raw remainder
      pd_walk<true>(bits, n_words, row0, (uint32_t)(e.n_out - item * B), 0, nullptr, e.rem, row_offset, lane, err);
      continue;
    }
    const uint64_t E = __ldg(cwx + item);
    const uint32_t w = (uint32_t)(__ldg(cwx + item + 1) - E);
    uint64_t span;
    const uint32_t* packed;
    if (pd_span(gstart, item, n_items, row0, row_offset, &span)) {
      uint32_t* buf = stage + kPdStageU32;
      if (B == 512) pd_fast_item<16, true>(bits, n_words, row0, span, w, stage, buf, lane);
      else if (B == 256) pd_fast_item<8, true>(bits, n_words, row0, span, w, stage, buf, lane);
      else pd_fast_item<4, true>(bits, n_words, row0, span, w, stage, buf, lane);
      packed = buf;
    } else {
      const uint32_t nw32 = B / 32 * w;
      for (uint32_t m = lane; m < nw32; m += 32) stage[m] = 0;
      __syncwarp();
      if (w) pd_walk<true>(bits, n_words, row0, B, w, stage, nullptr, row_offset, lane, err);
      __syncwarp();
      packed = stage;
    }
    if (lane == 0) {
      if (E + w > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
      e.cw[item + 1] = (uint32_t)(E + w);
      e.ref[item] = row0 + row_offset;
    }
    const uint64_t* src = reinterpret_cast<const uint64_t*>(packed);
    uint64_t* dst = e.payload + E * (B / 64);
    const uint32_t nw64 = B / 64 * w;
    for (uint32_t m = lane; m < nw64; m += 32) dst[m] = src[m];
    __syncwarp();
  }
}


// ---------------------------------------------------------------------------
// Single-walk variant (the default): pos_slot packs every full block at its own
// width into a fixed-size slot (B * wcap bits, wcap = ebw(rows - 1) bounds
// every delta) and records w_k and the base; the generic scan turns the widths
// into cw; pos_copy moves each block from its slot to word cw[k] * B / 64. The
// extra traffic (slots written and read back, ~2 x the positions image) costs
// less than a second walk of the mask.
__global__ void __launch_bounds__(kPdWarps * 32, 5) pos_slot_kernel(const uint32_t* __restrict__ bits,
                                                                 uint64_t n_words,
                                                                 const uint64_t* __restrict__ gstart,
                                                                 uint64_t row_offset, PosEnc e, uint64_t n_items,
                                                                 uint64_t* __restrict__ slots, uint32_t slot_words,
                                                                 uint32_t* __restrict__ wk, uint32_t* err) {
  extern __shared__ __align__(16) uint32_t pd_sm[];  // per warp: stage | fast pack buffer
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* stage = pd_sm + (size_t)wid * kPdWarpU32;
  const uint32_t B = e.G;
  const uint64_t n_full = e.n_out / B;
  const uint64_t nwarps = (uint64_t)gridDim.x * kPdWarps;
  uint64_t item = (uint64_t)blockIdx.x * kPdWarps + wid;
  // the block's first position and the next block's, one item ahead (two dependent
  // DRAM round trips per block otherwise: gstart, then the mask)
  uint64_t g0 = 0, g1 = 0;
  if (item < n_items) g0 = __ldg(gstart + item);
  if (item + 1 < n_items) g1 = __ldg(gstart + item + 1);
  for (; item < n_items; item += nwarps) {
    const uint64_t row0 = g0 - row_offset, rowE = g1 - row_offset;
    const uint64_t nx = item + nwarps;
    if (nx < n_items) g0 = __ldg(gstart + nx);
    if (nx + 1 < n_items) g1 = __ldg(gstart + nx + 1);
    if (item >= n_full) {  // final partial block -> raw remainder
      pd_walk<true>(bits, n_words, row0, (uint32_t)(e.n_out - item * B), 0, nullptr, e.rem, row_offset, lane, err);
      continue;
    }
    uint64_t span;
    uint32_t w;
    const uint32_t* packed;
    if (B == 512 && item + 1 < n_items && (rowE >> 5) - (row0 >> 5) < 512) {
      w = pd_item512(bits, row0, rowE, reinterpret_cast<uint16_t*>(stage), lane, err);
      packed = stage;
    } else if (pd_span(gstart, item, n_items, row0, row_offset, &span)) {
      uint32_t* buf = stage + kPdStageU32;
      w = B == 512   ? pd_fast_item<16, true, true>(bits, n_words, row0, span, 0, stage, buf, lane)
          : B == 256 ? pd_fast_item<8, true, true>(bits, n_words, row0, span, 0, stage, buf, lane)
                     : pd_fast_item<4, true, true>(bits, n_words, row0, span, 0, stage, buf, lane);
      packed = buf;
    } else {
      w = ebw64(warp_max(pd_walk<false>(bits, n_words, row0, B, 0, nullptr, nullptr, row_offset, lane, err)));
      const uint32_t nw32 = B / 32 * w;
      for (uint32_t m = lane; m < nw32; m += 32) stage[m] = 0;
      __syncwarp();
      if (w) pd_walk<true>(bits, n_words, row0, B, w, stage, nullptr, row_offset, lane, err);
      __syncwarp();
      packed = stage;
    }
    const uint32_t n16 = B / 128 * w;  // 16-byte units (B >= 128)
    if (n16 * 2 > slot_words) {  // cannot happen: wcap bounds every delta
      if (lane == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
    } else {
      const uint4* src = reinterpret_cast<const uint4*>(packed);
      uint4* dst = reinterpret_cast<uint4*>(slots + item * slot_words);
      for (uint32_t m = lane; m < n16; m += 32) dst[m] = src[m];
    }
    if (lane == 0) {
      wk[item] = w;
      e.ref[item] = row0 + row_offset;
    }
    __syncwarp();
  }
}

// LPB lanes per block (32 / LPB blocks per warp): slot -> payload at cw[k] * B / 64
// (16-byte copies), cw[k+1]. Narrow blocks (positions, w ~ 5: 4w 16-byte units at
// B = 512) take 8 lanes each, so a warp's header loads cover four blocks at once.
template <int LPB>
__global__ void __launch_bounds__(256) pos_copy_kernel(PosEnc e, uint64_t n_full, const uint64_t* __restrict__ slots,
                                                       uint32_t slot_words, const uint64_t* __restrict__ cwx,
                                                       uint32_t* err) {
  constexpr int kPerWarp = 32 / LPB;
  const uint32_t lane = threadIdx.x & 31, sub = lane % LPB;
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t w0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kPerWarp; w0 < n_full;
       w0 += nwarps * kPerWarp) {
    const uint64_t item = w0 + lane / LPB;
    if (item >= n_full) continue;
    const uint64_t E = __ldg(cwx + item);
    const uint32_t w = (uint32_t)(__ldg(cwx + item + 1) - E);
    if (sub == 0) {
      if (E + w > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
      e.cw[item + 1] = (uint32_t)(E + w);
    }
    const uint32_t n2 = e.G / 128 * w;  // 16-byte units (B*w/64 words, B >= 128)
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(slots + item * slot_words);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(e.payload + E * (e.G / 64));
    for (uint32_t m = sub; m < n2; m += LPB) dst[m] = __ldg(src + m);
  }
}

}  // namespace ms
