// select_fast.cuh — the vector-register core of select for bit-packed inputs
// (STATIC_BP, DYN_BP / FOR_BP with B >= 512, UNCOMPR): per warp, 512-row
// segments staged into shared memory with cp.async (3-stage ring, no register
// round trip), unpacked with a compile-time bit width (one instantiation per
// width 0..64, switch-dispatched per segment), the predicate evaluated in the
// code domain (the specialized-operator shortcut of P:352: the constant is
// translated once per block instead of decoding FOR values), and compacted
// with warp ballot + popc into one 32-bit mask word per 32 rows.
#pragma once
#include "common.cuh"
#include "tma.cuh"

namespace ms {

constexpr int kBufU32 = 1024 + 8;        // 4 KiB (512 rows x 64 bit) + padding for look-ahead reads

enum : int { FAST_UNCOMPR = 0, FAST_STATIC = 1, FAST_BLOCK = 2 };

// predicate passed to the fast kernel: keep = ((v - lo) <= span) != neg, or bitmap.
// iv[W] = the code-domain interval (a, s) of code_interval for codes of width W
// and reference 0 (STATIC_BP, DYN_BP: the common case), neg in bit W of iv_neg;
// filled on the host by fast_pred_table() so a lane reads it from the parameter
// bank at a compile-time index instead of translating the constant per 32 rows.
struct FastPred {
  uint64_t lo, span;
  uint32_t neg;
  uint32_t is_bitmap;
  const uint64_t* bitmap;
  uint64_t bits;
  uint32_t iv[33][2];
  uint64_t iv_neg;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Code-domain translation of the range predicate for codes c in [0, 2^W), W <= 32,
// with values v = ref + c: returns (a, s, neg) such that
// keep(c) = ((c - a) mod 2^32 <= s) != neg.
__host__ __device__ __forceinline__ void code_interval(uint64_t lo, uint64_t span, uint32_t neg0, uint64_t ref, uint32_t W,
                                              uint32_t& a, uint32_t& s, uint32_t& neg) {
  const uint64_t M1 = W >= 64 ? ~0ull : ((1ull << W) - 1);  // largest code
  const uint64_t d = lo - ref;                              // matching codes: (c - d) mod 2^64 <= span
  const uint64_t e = d + span;
  if (e >= d) {  // no wrap: c in [d, e]
    if (d > M1) {  // empty
      a = 0; s = 0xffffffffu; neg = neg0 ^ 1u;
      return;
    }
    const uint64_t hi = e < M1 ? e : M1;
    a = (uint32_t)d; s = (uint32_t)(hi - d); neg = neg0;
  } else {  // wrap: c in [0, e] U [d, 2^64) -> complement within [0, M1] is [e+1, d-1]
    if (e + 1 > M1) {  // complement empty: everything matches
      a = 0; s = 0xffffffffu; neg = neg0;
      return;
    }
    const uint64_t chi = (d - 1) < M1 ? (d - 1) : M1;
    a = (uint32_t)(e + 1); s = (uint32_t)(chi - (e + 1)); neg = neg0 ^ 1u;
  }
}

// the per-width table of FastPred (reference 0)
inline void fast_pred_table(FastPred& fp) {
  fp.iv_neg = 0;
  for (uint32_t W = 1; W <= 32; ++W) {
    uint32_t a, sp, ng;
    code_interval(fp.lo, fp.span, fp.neg, 0, W, a, sp, ng);
    fp.iv[W][0] = a;
    fp.iv[W][1] = sp;
    fp.iv_neg |= (uint64_t)(ng & 1u) << W;
  }
  fp.iv[0][0] = fp.iv[0][1] = 0;
}

// ---- lane-consecutive core: lane l of a half-warp owns rows 32l .. 32l+31 of
// a segment = exactly W consecutive 32-bit words at word offset l*W (aligned:
// 32 rows x W bits = W words), loaded with the widest aligned shared-memory
// vector loads, unpacked with compile-time shifts, the predicate applied and
// the lane's mask word built directly (no ballot, no cross-lane routing).
template <int W>
__device__ __forceinline__ void load_words(const uint32_t* __restrict__ p, uint32_t (&r)[W + 1]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int i = 0; i < W; i += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + i);
      r[i] = v.x; r[i + 1] = v.y; r[i + 2] = v.z; r[i + 3] = v.w;
    }
  } else if constexpr (W % 2 == 0) {
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      const uint2 v = *reinterpret_cast<const uint2*>(p + i);
      r[i] = v.x; r[i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) r[i] = p[i];
  }
  r[W] = 0;
}

template <int W>
__device__ __forceinline__ uint64_t code_at(const uint32_t (&r)[W + 1], int i) {
  constexpr uint64_t mask = W >= 64 ? ~0ull : ((1ull << (W & 63)) - 1);
  const int bit = i * W, q = bit >> 5, sh = bit & 31;
  if (W <= 32) {
    uint32_t c = (sh + W <= 32) ? (r[q] >> sh) : __funnelshift_r(r[q], r[q + 1], sh);
    return (uint64_t)(c & (uint32_t)mask);
  }
  const uint32_t lo = __funnelshift_r(r[q], r[q + 1], sh);
  const uint32_t hi = (q + 2 <= W) ? __funnelshift_r(r[q + 1], r[(q + 2) <= W ? q + 2 : W], sh) : (r[q + 1] >> sh);
  return (((uint64_t)hi << 32) | lo) & mask;
}

// one lane's 32 rows: returns the mask word (bit i <=> row 32l + i matched)
template <int W>
__device__ __forceinline__ uint32_t lane_rows(const uint32_t* __restrict__ p, const FastPred& pr, uint64_t ref) {
  if constexpr (W == 0) {
    bool keep;
    if (pr.is_bitmap) keep = ref < pr.bits && ((__ldg(pr.bitmap + (ref >> 6)) >> (ref & 63)) & 1ull);
    else keep = ((ref - pr.lo) <= pr.span) != (pr.neg != 0);
    return keep ? 0xffffffffu : 0u;
  } else {
    uint32_t r[W + 1];
    load_words<W>(p, r);
    uint32_t m = 0;
    if (pr.is_bitmap) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const uint64_t v = ref + code_at<W>(r, i);
        const bool keep = v < pr.bits && ((__ldg(pr.bitmap + (v >> 6)) >> (v & 63)) & 1ull);
        m |= (keep ? 1u : 0u) << i;
      }
    } else if constexpr (W <= 32) {
      uint32_t a, sp, ng;
      if (ref == 0) {
        a = pr.iv[W][0];
        sp = pr.iv[W][1];
        ng = (uint32_t)(pr.iv_neg >> W) & 1u;
      } else {
        code_interval(pr.lo, pr.span, pr.neg, ref, W, a, sp, ng);
      }
      constexpr uint32_t cmask = W >= 32 ? 0xffffffffu : ((1u << (W & 31)) - 1u);
      if (a == 0 && (sp & (sp + 1)) == 0 && sp < cmask) {
        // prefix interval [0, 2^k): a code matches iff its bits k..W-1 are zero — one
        // AND with a shifted mask per row, no extraction of the code (the specialized-
        // operator shortcut of P:352 applied to the bit layout)
        const uint32_t hi = cmask & ~sp;  // the code's high bits
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int bit = i * W, q = bit >> 5, sh = bit & 31;
          bool z;
          if (sh + W <= 32) z = (r[q] & (hi << sh)) == 0u;
          else z = (__funnelshift_r(r[q], r[q + 1], sh) & hi) == 0u;
          if (z) m |= 1u << i;  // (a predicated OR with a constant)
        }
      } else if (sp >= cmask) {
        m = ~0u;  // every code of the block matches
      } else {
        // general interval [a, a + sp] (inside [0, 2^W)): each code is read top-aligned,
        // ct = c * 2^K + g with K = 32 - W and g < 2^K the bits of the code below it,
        // so c - a <= sp  <=>  ct - a * 2^K <= T = sp * 2^K + 2^K - 1 (a code below a
        // wraps past T). The test is the carry of (ct - a * 2^K) + ~T (set iff the row
        // does NOT match), shifted into the inverted mask by addc: three instructions
        // per row (shift-subtract, add with carry-out, add with carry-in), no mask
        // extraction, no compare-and-select.
        constexpr int K = 32 - W;
        const uint32_t at = a << K;
        const uint32_t nT = ~((sp << K) | ((1u << K) - 1u));
        uint32_t mi = 0;
#pragma unroll
        for (int i = 31; i >= 0; --i) {  // row 31 first: addc doubles the mask each row
          const int bit = i * W, q = bit >> 5, sh = bit & 31;
          uint32_t ct;
          if (sh + W <= 32) ct = r[q] << (32 - sh - W);
          else ct = __funnelshift_l(r[q], r[q + 1], 64 - sh - W);
          const uint32_t d = ct - at;
          asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, %3, %3;\n\t}"
              : "=r"(mi)
              : "r"(d), "r"(nT), "r"(mi));
        }
        m = ~mi;
      }
      if (ng) m = ~m;  // the negated predicates, once per 32 rows
    } else {
      const uint64_t d = pr.lo - ref;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const bool keep = ((code_at<W>(r, i) - d) <= pr.span) != (pr.neg != 0);
        m |= (keep ? 1u : 0u) << i;
      }
    }
    return m;
  }
}

// Words [Q0, Q0 + NW) of a lane's W words (zero past W) with the widest vector
// shared-memory loads their alignment allows: lanes are W words apart, so scalar
// loads at an even W hit the same bank gcd(W, 32) ways (8 at W = 40); 16-byte
// loads leave at most two lanes of a quarter-warp on one bank group.
template <int W, int Q0, int NW, bool VEC>
__device__ __forceinline__ void load_lane_range(const uint32_t* __restrict__ p, uint32_t (&r)[NW]) {
  constexpr int V = !VEC ? 1 : (W % 4 == 0 && Q0 % 4 == 0) ? 4 : ((W % 2 == 0 && Q0 % 2 == 0) ? 2 : 1);
#pragma unroll
  for (int i = 0; i < NW; i += V) {
    if (V == 4 && i + 3 < NW && Q0 + i + 3 < W) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + Q0 + i);
      r[i] = v.x; r[i + 1] = v.y; r[i + 2] = v.z; r[i + 3] = v.w;
    } else if (V >= 2 && i + 1 < NW && Q0 + i + 1 < W) {
      const uint2 v = *reinterpret_cast<const uint2*>(p + Q0 + i);
      r[i] = v.x; r[i + 1] = v.y;
      if (V == 4) {
#pragma unroll
        for (int k = 2; k < V; ++k)
          if (i + k < NW) r[i + k] = (Q0 + i + k < W) ? p[Q0 + i + k] : 0u;
      }
    } else {
#pragma unroll
      for (int k = 0; k < V; ++k)
        if (i + k < NW) r[i + k] = (Q0 + i + k < W) ? p[Q0 + i + k] : 0u;
    }
  }
}

// W > 32: the same 32 rows in two halves of 16 rows (16*W bits each) so that at
// most W/2 + 2 words are live in registers; the second half starts at the
// compile-time bit offset 16*W.
template <int W, int H, bool VEC>
__device__ __forceinline__ uint32_t half_rows(const uint32_t* __restrict__ p, const FastPred& pr, uint64_t ref,
                                              uint64_t d) {
  constexpr int B0 = H * 16 * W;       // first bit of this half
  constexpr int Q0 = B0 >> 5;          // first word
  constexpr int NW = ((B0 & 31) + 16 * W + 31) / 32 + 1;
  constexpr uint64_t mask = W >= 64 ? ~0ull : ((1ull << (W & 63)) - 1);
  uint32_t r[NW];
  load_lane_range<W, Q0, NW, VEC>(p, r);
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int bit = (B0 & 31) + i * W, q = bit >> 5, sh = bit & 31;
    const uint32_t lo = __funnelshift_r(r[q], r[q + 1], sh);
    const uint32_t hi = __funnelshift_r(r[q + 1], r[q + 2 < NW ? q + 2 : NW - 1], sh);
    const uint64_t code = (((uint64_t)hi << 32) | lo) & mask;
    bool keep;
    if (pr.is_bitmap) {
      const uint64_t v = ref + code;
      keep = v < pr.bits && ((__ldg(pr.bitmap + (v >> 6)) >> (v & 63)) & 1ull);
    } else {
      keep = ((code - d) <= pr.span) != (pr.neg != 0);
    }
    m |= (keep ? 1u : 0u) << (i + 16 * H);
  }
  return m;
}

// W > 32, a code-domain interval [a, a + s] inside [0, 2^32): a code matches iff
// its low 32 bits are in the interval AND its high W - 32 bits are zero. The
// low-word test runs for every row (one funnel shift, one add, one compare); the
// high bits are checked only for the candidates it leaves (at most as many as the
// matches plus the rare rows whose low word alone falls in the interval).
template <int W, int H, bool VEC>
__device__ __forceinline__ uint32_t half_low32(const uint32_t* __restrict__ p, uint32_t a, uint32_t s) {
  constexpr int B0 = H * 16 * W;
  constexpr int Q0 = B0 >> 5;
  constexpr int NW = ((B0 & 31) + 16 * W + 31) / 32 + 1;
  uint32_t r[NW];
  load_lane_range<W, Q0, NW, VEC>(p, r);
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int bit = (B0 & 31) + i * W, q = bit >> 5, sh = bit & 31;
    const uint32_t lo = sh ? __funnelshift_r(r[q], r[q + 1], sh) : r[q];
    m |= ((lo - a) <= s ? 1u : 0u) << (i + 16 * H);
  }
  return m;
}

template <int W, bool VEC>
__device__ __forceinline__ uint32_t lane_rows_wide(const uint32_t* __restrict__ p, const FastPred& pr,
                                                   uint64_t ref) {
  const uint64_t d = pr.lo - ref;
  if (!pr.is_bitmap && d + pr.span >= d && d + pr.span <= 0xffffffffull) {
    uint32_t cand = half_low32<W, 0, VEC>(p, (uint32_t)d, (uint32_t)pr.span) | half_low32<W, 1, VEC>(p, (uint32_t)d,
                                                                                           (uint32_t)pr.span);
    uint32_t m = cand;
    while (cand) {  // confirm: the high W - 32 bits of the candidate's code are zero
      const uint32_t i = __ffs(cand) - 1;
      cand &= cand - 1;
      const uint32_t bit = i * W + 32, q = bit >> 5, sh = bit & 31;
      uint64_t hi = (uint64_t)p[q] >> sh;
      if (sh + (W - 32) > 32) hi |= (uint64_t)p[q + 1] << (32 - sh);
      if (hi & ((1ull << (W - 32)) - 1)) m &= ~(1u << i);
    }
    return pr.neg ? ~m : m;
  }
  return half_rows<W, 0, VEC>(p, pr, ref, d) | half_rows<W, 1, VEC>(p, pr, ref, d);
}

// VEC: the wide cores stage their words with vector loads (the per-warp-ring core,
// launched for widths > 32); the streamed core (widths <= 32, a wider block only
// under an understated max_width hint) keeps scalar loads, which keep it free of
// spills.
template <bool VEC>
__device__ __forceinline__ uint32_t lane_dispatch(uint32_t w, const uint32_t* p, const FastPred& pr, uint64_t ref) {
  switch (w) {
#define MS_LANE_CASE(W) \
  case W:               \
    return W <= 32 ? lane_rows<(W <= 32 ? W : 1)>(p, pr, ref) : lane_rows_wide<(W > 32 ? W : 33), VEC>(p, pr, ref);
    MS_LANE_CASE(0) MS_LANE_CASE(1) MS_LANE_CASE(2) MS_LANE_CASE(3) MS_LANE_CASE(4) MS_LANE_CASE(5)
    MS_LANE_CASE(6) MS_LANE_CASE(7) MS_LANE_CASE(8) MS_LANE_CASE(9) MS_LANE_CASE(10) MS_LANE_CASE(11)
    MS_LANE_CASE(12) MS_LANE_CASE(13) MS_LANE_CASE(14) MS_LANE_CASE(15) MS_LANE_CASE(16) MS_LANE_CASE(17)
    MS_LANE_CASE(18) MS_LANE_CASE(19) MS_LANE_CASE(20) MS_LANE_CASE(21) MS_LANE_CASE(22) MS_LANE_CASE(23)
    MS_LANE_CASE(24) MS_LANE_CASE(25) MS_LANE_CASE(26) MS_LANE_CASE(27) MS_LANE_CASE(28) MS_LANE_CASE(29)
    MS_LANE_CASE(30) MS_LANE_CASE(31) MS_LANE_CASE(32) MS_LANE_CASE(33) MS_LANE_CASE(34) MS_LANE_CASE(35)
    MS_LANE_CASE(36) MS_LANE_CASE(37) MS_LANE_CASE(38) MS_LANE_CASE(39) MS_LANE_CASE(40) MS_LANE_CASE(41)
    MS_LANE_CASE(42) MS_LANE_CASE(43) MS_LANE_CASE(44) MS_LANE_CASE(45) MS_LANE_CASE(46) MS_LANE_CASE(47)
    MS_LANE_CASE(48) MS_LANE_CASE(49) MS_LANE_CASE(50) MS_LANE_CASE(51) MS_LANE_CASE(52) MS_LANE_CASE(53)
    MS_LANE_CASE(54) MS_LANE_CASE(55) MS_LANE_CASE(56) MS_LANE_CASE(57) MS_LANE_CASE(58) MS_LANE_CASE(59)
    MS_LANE_CASE(60) MS_LANE_CASE(61) MS_LANE_CASE(62) MS_LANE_CASE(63) MS_LANE_CASE(64)
#undef MS_LANE_CASE
    default:
      return 0;
  }
}

// ---- sum core: the same lane-consecutive unpack, accumulating the codes
// W > 32: rows [16H, 16H + 16) of the lane, words staged in registers by vector loads
template <int W, int H, bool VEC>
__device__ __forceinline__ uint64_t lane_sum_half(const uint32_t* __restrict__ p) {
  constexpr int B0 = H * 16 * W;
  constexpr int Q0 = B0 >> 5;
  constexpr int NW = ((B0 & 31) + 16 * W + 31) / 32 + 1;
  constexpr uint64_t mask = W >= 64 ? ~0ull : ((1ull << (W & 63)) - 1);
  uint32_t r[NW];
  load_lane_range<W, Q0, NW, VEC>(p, r);
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int bit = (B0 & 31) + i * W, q = bit >> 5, sh = bit & 31;
    const uint32_t lo = __funnelshift_r(r[q], r[q + 1], sh);
    const uint32_t hi = __funnelshift_r(r[q + 1], r[q + 2 < NW ? q + 2 : NW - 1], sh);
    acc += (((uint64_t)hi << 32) | lo) & mask;
  }
  return acc;
}

template <int W, bool VEC>
__device__ __forceinline__ uint64_t lane_sum(const uint32_t* __restrict__ p) {
  if constexpr (W == 0) {
    return 0;
  } else if constexpr (W <= 32) {
    uint32_t r[W + 1];
    load_words<W>(p, r);
    uint64_t acc = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += code_at<W>(r, i);
    return acc;
  } else {
    return lane_sum_half<W, 0, VEC>(p) + lane_sum_half<W, 1, VEC>(p);
  }
}

template <bool VEC>
__device__ __forceinline__ uint64_t lane_sum_dispatch(uint32_t w, const uint32_t* p) {
  switch (w) {
#define MS_SUM_CASE(W) \
  case W:              \
    return lane_sum<W, VEC>(p);
    MS_SUM_CASE(0) MS_SUM_CASE(1) MS_SUM_CASE(2) MS_SUM_CASE(3) MS_SUM_CASE(4) MS_SUM_CASE(5) MS_SUM_CASE(6)
    MS_SUM_CASE(7) MS_SUM_CASE(8) MS_SUM_CASE(9) MS_SUM_CASE(10) MS_SUM_CASE(11) MS_SUM_CASE(12)
    MS_SUM_CASE(13) MS_SUM_CASE(14) MS_SUM_CASE(15) MS_SUM_CASE(16) MS_SUM_CASE(17) MS_SUM_CASE(18)
    MS_SUM_CASE(19) MS_SUM_CASE(20) MS_SUM_CASE(21) MS_SUM_CASE(22) MS_SUM_CASE(23) MS_SUM_CASE(24)
    MS_SUM_CASE(25) MS_SUM_CASE(26) MS_SUM_CASE(27) MS_SUM_CASE(28) MS_SUM_CASE(29) MS_SUM_CASE(30)
    MS_SUM_CASE(31) MS_SUM_CASE(32) MS_SUM_CASE(33) MS_SUM_CASE(34) MS_SUM_CASE(35) MS_SUM_CASE(36)
    MS_SUM_CASE(37) MS_SUM_CASE(38) MS_SUM_CASE(39) MS_SUM_CASE(40) MS_SUM_CASE(41) MS_SUM_CASE(42)
    MS_SUM_CASE(43) MS_SUM_CASE(44) MS_SUM_CASE(45) MS_SUM_CASE(46) MS_SUM_CASE(47) MS_SUM_CASE(48)
    MS_SUM_CASE(49) MS_SUM_CASE(50) MS_SUM_CASE(51) MS_SUM_CASE(52) MS_SUM_CASE(53) MS_SUM_CASE(54)
    MS_SUM_CASE(55) MS_SUM_CASE(56) MS_SUM_CASE(57) MS_SUM_CASE(58) MS_SUM_CASE(59) MS_SUM_CASE(60)
    MS_SUM_CASE(61) MS_SUM_CASE(62) MS_SUM_CASE(63) MS_SUM_CASE(64)
#undef MS_SUM_CASE
    default:
      return 0;
  }
}


enum : int { CORE_SELECT = 0, CORE_SUM = 1 };

// Per-warp contiguous range of full 512-row segments, taken two at a time
// (half-warp h handles segment 2p+h). Lane 0 streams the pair's packed payload
// (64*(wA+wB) bytes, contiguous, 64-byte aligned) into a per-warp ring of
// kStages shared-memory slots with ONE TMA bulk copy tracked by one mbarrier;
// widths / references travel with the slot.
constexpr int kPairBufWide = 2048 + 16;   // two segments at up to 64 bits + padding
constexpr int kPairBufNarrow = 1024 + 16; // two segments at up to 32 bits + padding
constexpr int kPairBufMedium = 1536 + 16; // two segments at up to 48 bits + padding
template <int KIND, int kStages = 2, int kFastWarps = 4, int kMinBlocks = 3, int kPairBufU32 = kPairBufWide,
          int CORE = CORE_SELECT>
__global__ void __launch_bounds__(kFastWarps * 32, kMinBlocks) select_fast_kernel(ColView c, FastPred pred,
                                                                                 uint32_t* __restrict__ bits,
                                                                                 uint32_t* __restrict__ seg_info,
                                                                                 uint64_t NS, uint64_t spw,
                                                                                 uint32_t* err,
                                                                                 unsigned long long* sum_out) {
  extern __shared__ __align__(128) uint32_t fsm[];
  __shared__ __align__(8) uint64_t bars[kFastWarps][kStages];
  __shared__ uint64_t sref[kFastWarps][kStages][2];
  __shared__ uint32_t sw[kFastWarps][kStages][2];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t half = lane >> 4, hl = lane & 15;
  const uint64_t gw = (uint64_t)blockIdx.x * kFastWarps + wid;
  const uint64_t s_begin = gw * spw;  // spw is even
  if (s_begin >= NS) return;
  const uint64_t s_end = min(NS, s_begin + spw);
  uint32_t* buf = fsm + wid * (kStages * kPairBufU32);
  if (KIND != FAST_UNCOMPR && lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&bars[wid][k], 1);
    mbar_fence_init();
  }
  __syncwarp();

  auto meta = [&](uint64_t s, uint32_t& w, uint64_t& off, uint64_t& ref) {
    ref = 0;
    if constexpr (KIND == FAST_STATIC) {
      w = c.w;
      off = s * 8 * (uint64_t)w;
    } else {
      const uint64_t b = (s << 9) >> c.log2B;
      const uint32_t cw0 = __ldg(c.cw + b);
      w = __ldg(c.cw + b + 1) - cw0;
      off = (uint64_t)cw0 * (c.B >> 6) + (s & ((c.B >> 9) - 1)) * 8 * (uint64_t)w;
      if (c.ref) ref = __ldg(c.ref + b);
    }
    if (w > 64) {  // corrupt width table
      w = 65;
      atomicOr(err, err_bit(MS_E_CORRUPT));
    }
  };
  auto issue = [&](uint64_t s, int stage) {  // segments s, s+1
    if (KIND == FAST_UNCOMPR || s >= s_end || lane != 0) return;
    uint32_t wa, wb = 0;
    uint64_t off, ra, rb = 0, offb;
    meta(s, wa, off, ra);
    if (s + 1 < s_end) meta(s + 1, wb, offb, rb);
    sw[wid][stage][0] = wa;
    sw[wid][stage][1] = wb;
    sref[wid][stage][0] = ra;
    sref[wid][stage][1] = rb;
    uint32_t bytes = (wa <= 64 ? 64 * wa : 0) + (wb <= 64 ? 64 * wb : 0);
    if (bytes > (kPairBufU32 - 16) * 4) {  // a width larger than the max_width hint: never overrun the slot
      sw[wid][stage][0] = sw[wid][stage][1] = 65;
      bytes = 0;
      atomicOr(err, err_bit(MS_E_CORRUPT));
    }
    mbar_arrive_tx(&bars[wid][stage], bytes);
    if (bytes) bulk_g2s(buf + stage * kPairBufU32, c.payload + off, bytes, &bars[wid][stage]);
  };

  for (int k = 0; k < kStages - 1; ++k) issue(s_begin + 2 * k, k);
  int stage = 0;
  uint32_t phase = 0;
  uint64_t sum_acc = 0;
  for (uint64_t s = s_begin; s < s_end; s += 2) {
    issue(s + 2 * (kStages - 1), (stage + kStages - 1) % kStages);
    const uint64_t my_seg = s + half;
    const bool valid = my_seg < s_end;
    uint32_t m = 0;
    if constexpr (KIND == FAST_UNCOMPR) {
      if (valid) {
        const uint64_t* v = c.payload + my_seg * kSegRows + hl * 32;
        uint64_t x[32];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(v + i));
          x[i] = t.x; x[i + 1] = t.y;
        }
        if constexpr (CORE == CORE_SUM) {
#pragma unroll
          for (int i = 0; i < 32; ++i) sum_acc += x[i];
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            bool keep;
            if (pred.is_bitmap) keep = x[i] < pred.bits && ((__ldg(pred.bitmap + (x[i] >> 6)) >> (x[i] & 63)) & 1ull);
            else keep = ((x[i] - pred.lo) <= pred.span) != (pred.neg != 0);
            m |= (keep ? 1u : 0u) << i;
          }
        }
      }
    } else {
      mbar_wait(&bars[wid][stage], phase);
      const uint32_t wa = sw[wid][stage][0];
      const uint32_t w = sw[wid][stage][half];
      const uint64_t ref = sref[wid][stage][half];
      const uint32_t* p = buf + stage * kPairBufU32 + (half ? 16 * wa : 0) + hl * w;
      if (valid) {
        if constexpr (CORE == CORE_SUM) {
          sum_acc += lane_sum_dispatch<true>(w, p) + (hl == 0 ? (uint64_t)kSegRows * ref : 0ull);
        } else {
          m = lane_dispatch<true>(w, p, pred, ref);
        }
      }
    }
    __syncwarp();
    if constexpr (CORE == CORE_SELECT) {
      if (valid) bits[my_seg * kSegWords + hl] = m;
      uint32_t cnt = __popc(m);
      uint32_t last = m ? hl * 32 + 32 - __clz(m) : 0u;
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(kFull, cnt, o);
        last = max(last, __shfl_xor_sync(kFull, last, o));
      }
      if (valid && hl == 0) seg_info[my_seg] = cnt | (last << 16);
    }
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
  if constexpr (CORE == CORE_SUM) {
    sum_acc = warp_sum(sum_acc);
    if (lane == 0 && sum_acc) atomicAdd(sum_out, (unsigned long long)sum_acc);
  }
}

}  // namespace ms
