// posdelta.cuh — select's output-side buffer layer for the positions format the
// paper recommends for select outputs, DELTA_BP ("the output is always
// sorted"), straight from the select bit mask to the packed column
// (P:486-490), for block sizes B <= 512.
//
// Output block k holds output ranks [kB, kB + B); its first position gstart[k]
// comes from the segment scan. Three launches, none of which waits on another
// CTA (a look-back per block or per tile of blocks stalls whole CTAs on their
// predecessors, measured 3x slower on B200):
//   pos_slot   one warp per block: one walk of the block's mask span, d_j =
//              p_j - p_{j-1}, d_0 = 0 (D-6), w_k = ebw(max_j d_j), the
//              block packed in shared memory and stored to a fixed-size slot;
//   scan       exclusive prefix of w_k -> cw (D-4), the generic scan kernel;
//   pos_copy   every block from its slot to word cw[k] * B / 64.
// The final partial block goes raw to the remainder. Per block the walk
// is pd_item512 (B = 512, span < 512 words, i.e. selectivity above ~3.1 %: words
// in registers, set bits scattered by rank into shared memory, 16 ranks per lane
// packed at a compile-time width) or pd_item_walk (everything else: rounds of
// 512 words, the same scatter with u32 rows, a runtime-width pack). No position
// is materialised outside the SM.
#pragma once
#include "common.cuh"
#include "launch.h"

namespace ms {

constexpr int kPdWarps = 8;  // warps per CTA (independent)
constexpr int kPdLaneWords = 8;
constexpr int kPdRoundWords = 32 * kPdLaneWords;
constexpr uint32_t kPdWarpU32 = 1024;  // shared memory per warp: a block of B <= 512 codes at w <= 64 bits

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


// Single-pass walk for the other full blocks (sparser masks, B < 512, the block
// before the last): rounds of 512 words (16 per lane, 16-byte loads), set bits
// scattered by rank into p32 (u32 rows relative to word wa) until B are found;
// then lane j reads ranks [PER*j, PER*j + PER), d_q = p_q - p_{q-1}, w = ebw(max d)
// (<= 32), and streams its codes — the bit range [PER*j*w, PER*(j+1)*w) — into
// the block buffer (zeroed; atomicOr on the two words a lane may share).
// Returns false when the block spans 2^32 rows or more (relative rows would
// wrap): the caller falls back to the two-walk pd_walk.
template <int PER>
__device__ __forceinline__ bool pd_item_walk(const uint32_t* __restrict__ bits, uint64_t n_words, uint64_t row0,
                                             uint32_t* p32, uint32_t lane, uint32_t* err, uint32_t* w_out) {
  constexpr uint32_t B = PER * 32;
  constexpr uint32_t kRoundWords = 512;
  const uint64_t wi = row0 >> 5, wa = wi & ~3ull;
  const uint32_t fmask = ~0u << (row0 & 31);
  uint32_t got = 0;
  for (uint64_t wb = wa; got < B; wb += kRoundWords) {
    if (wb >= n_words) {  // fewer set bits than the scan counted
      if (lane == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
      *w_out = 0;
      return true;
    }
    if ((wb - wa + kRoundWords) * 32 > 0xffffffffull) return false;
    const uint64_t wl = wb + 16ull * lane;
    uint32_t x[16];
    if (wl + 16 <= n_words) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(bits + wl) + g);
        x[4 * g] = v.x; x[4 * g + 1] = v.y; x[4 * g + 2] = v.z; x[4 * g + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = wl + i < n_words ? __ldg(bits + wl + i) : 0u;
    }
    if (wl == wa) {  // lane 0 of the first round holds the block's first word (wi - wa < 4)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (wa + i < wi) x[i] = 0u;
        else if (wa + i == wi) x[i] &= fmask;
      }
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) cnt += __popc(x[i]);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, inc, o);
      if (lane >= (uint32_t)o) inc += t;
    }
    uint32_t r = got + inc - cnt;
    if (r < B) {
      const uint32_t rb = (uint32_t)(wl - wa) * 32u;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        uint32_t word = x[i];
        while (word && r < B) {
          p32[r++] = rb + 32u * i + (__ffs(word) - 1);
          word &= word - 1u;
        }
      }
    }
    got += __shfl_sync(kFull, inc, 31);
  }
  __syncwarp();
  uint32_t d[PER];  // the positions, then (in place, last first) their deltas
#pragma unroll
  for (int q = 0; q < PER; ++q) d[q] = p32[PER * lane + q];
  const uint32_t prev = __shfl_up_sync(kFull, d[PER - 1], 1);
  uint32_t mx = 0;
#pragma unroll
  for (int q = PER - 1; q >= 0; --q) {
    d[q] = q ? d[q] - d[q - 1] : (lane ? d[0] - prev : 0u);
    mx = d[q] > mx ? d[q] : mx;
  }
  mx = __reduce_max_sync(kFull, mx);
  const uint32_t w = 32u - __clz(mx);
  __syncwarp();
  const uint32_t nw32 = PER * w;  // == B * w / 32
  for (uint32_t i = lane; i < nw32; i += 32) p32[i] = 0u;
  __syncwarp();
  if (w) {
    const uint32_t o = PER * lane * w;
    uint32_t widx = o >> 5, nb = o & 31;
    uint64_t acc = 0;
    bool first = true;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      acc |= (uint64_t)d[q] << nb;
      nb += w;
      if (nb >= 32) {
        if (first) {
          atomicOr(p32 + widx, (uint32_t)acc);
          first = false;
        } else {
          p32[widx] = (uint32_t)acc;
        }
        ++widx;
        nb -= 32;
        acc >>= 32;
      }
    }
    if (nb) atomicOr(p32 + widx, (uint32_t)acc);
  }
  __syncwarp();
  *w_out = w;
  return true;
}

// Outputs without a full block: the remainder alone, raw positions.
__global__ void __launch_bounds__(kPdWarps * 32) pos_rem_kernel(const uint32_t* __restrict__ bits, uint64_t n_words,
                                                                const uint64_t* __restrict__ gstart,
                                                                uint64_t row_offset, PosEnc e, uint32_t* err) {
  if (threadIdx.x >= 32) return;
  const uint64_t row0 = __ldg(gstart) - row_offset;
  pd_walk<true>(bits, n_words, row0, (uint32_t)e.n_out, 0, nullptr, e.rem, row_offset, threadIdx.x, err);
}

// ---------------------------------------------------------------------------
// pos_slot packs every full block at its own width into a fixed-size slot
// (B * wcap bits, wcap = ebw(rows - 1) bounds every delta) and records w_k and
// the base; the generic scan turns the widths into cw; pos_copy moves each
// block from its slot to word cw[k] * B / 64. The extra traffic (slots written
// and read back, ~2 x the positions image) costs less than a second walk of the
// mask. One warp per block, kPdWarpU32 words of shared memory per warp.
// A packed block (stage, B*w bits) to its slot, its width and base.
__device__ __forceinline__ void pd_store_slot(uint64_t item, uint32_t w, uint64_t base, const PosEnc& e,
                                              uint64_t* slots, uint32_t slot_words, uint32_t* wk,
                                              const uint32_t* stage, uint32_t lane, uint32_t* err) {
  const uint32_t n16 = e.G / 128 * w;  // 16-byte units (B >= 128)
  if (n16 * 2 > slot_words) {  // cannot happen: wcap bounds every delta
    if (lane == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(stage);
    uint4* dst = reinterpret_cast<uint4*>(slots + item * slot_words);
    for (uint32_t m = lane; m < n16; m += 32) dst[m] = src[m];
  }
  if (lane == 0) {
    wk[item] = w;
    e.ref[item] = base;
  }
  __syncwarp();
}

// MODE kPdDense (B = 512): pd_item512 only; a block whose span does not fit (and
// the block before the last) is appended to dlist (*dcount: count) and left to a
// kPdDeferredOnly launch, whose warps take the listed blocks one each. The walk's
// registers stay out of the fast path. kPdAll: the walk for every block.
constexpr int kPdAll = 0, kPdDense = 1, kPdDeferredOnly = 2;

// One full block by the walk (pd_item_walk; two walks past 2^32 rows) into its slot.
__device__ __forceinline__ void pd_walk_block(const uint32_t* __restrict__ bits, uint64_t n_words, uint64_t row0,
                                              uint64_t item, uint64_t row_offset, const PosEnc& e, uint64_t* slots,
                                              uint32_t slot_words, uint32_t* wk, uint32_t* stage, uint32_t lane,
                                              uint32_t* err) {
  const uint32_t B = e.G;
  uint32_t w = 0;
  const bool done = B == 512   ? pd_item_walk<16>(bits, n_words, row0, stage, lane, err, &w)
                    : B == 256 ? pd_item_walk<8>(bits, n_words, row0, stage, lane, err, &w)
                               : pd_item_walk<4>(bits, n_words, row0, stage, lane, err, &w);
  if (!done) {  // a block spanning >= 2^32 rows: two walks, codes up to 64 bits
    w = ebw64(warp_max(pd_walk<false>(bits, n_words, row0, B, 0, nullptr, nullptr, row_offset, lane, err)));
    const uint32_t nw32 = B / 32 * w;
    for (uint32_t m = lane; m < nw32; m += 32) stage[m] = 0;
    __syncwarp();
    if (w) pd_walk<true>(bits, n_words, row0, B, w, stage, nullptr, row_offset, lane, err);
    __syncwarp();
  }
  pd_store_slot(item, w, row0 + row_offset, e, slots, slot_words, wk, stage, lane, err);
}

template <int MODE>
__global__ void __launch_bounds__(kPdWarps * 32, 5) pos_slot_kernel(const uint32_t* __restrict__ bits,
                                                                 uint64_t n_words,
                                                                 const uint64_t* __restrict__ gstart,
                                                                 uint64_t row_offset, PosEnc e, uint64_t n_items,
                                                                 uint64_t* __restrict__ slots, uint32_t slot_words,
                                                                 uint32_t* __restrict__ wk, uint32_t* dcount,
                                                                 uint32_t* dlist, uint32_t* err) {
  extern __shared__ __align__(16) uint32_t pd_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* stage = pd_sm + (size_t)wid * kPdWarpU32;
  const uint32_t B = e.G;
  const uint64_t n_full = e.n_out / B;
  const uint64_t nwarps = (uint64_t)gridDim.x * kPdWarps;
  const uint64_t gw = (uint64_t)blockIdx.x * kPdWarps + wid;
  if (MODE == kPdDeferredOnly) {  // the listed blocks, one per warp
    const uint32_t nd = *reinterpret_cast<volatile uint32_t*>(dcount);
    for (uint64_t i = gw; i < nd; i += nwarps) {
      const uint64_t item = __ldg(dlist + i);
      pd_walk_block(bits, n_words, __ldg(gstart + item) - row_offset, item, row_offset, e, slots, slot_words, wk,
                    stage, lane, err);
    }
    return;
  }
  uint64_t item = gw;
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
    if (MODE == kPdDense) {
      if (item + 1 < n_items && (rowE >> 5) - (row0 >> 5) < 512) {
        const uint32_t w = pd_item512(bits, row0, rowE, reinterpret_cast<uint16_t*>(stage), lane, err);
        pd_store_slot(item, w, row0 + row_offset, e, slots, slot_words, wk, stage, lane, err);
      } else if (lane == 0) {
        dlist[atomicAdd(dcount, 1u)] = (uint32_t)item;
      }
    } else {
      pd_walk_block(bits, n_words, row0, item, row_offset, e, slots, slot_words, wk, stage, lane, err);
    }
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
