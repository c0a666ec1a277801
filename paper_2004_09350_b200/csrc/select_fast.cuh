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

namespace ms {

constexpr int kStages = 3;
constexpr int kBufU32 = 1024 + 8;        // 4 KiB (512 rows x 64 bit) + padding for look-ahead reads
constexpr int kFastWarps = 8;            // warps per CTA

enum : int { FAST_UNCOMPR = 0, FAST_STATIC = 1, FAST_BLOCK = 2 };

// predicate passed to the fast kernel: keep = ((v - lo) <= span) != neg, or bitmap
struct FastPred {
  uint64_t lo, span;
  uint32_t neg;
  uint32_t is_bitmap;
  const uint64_t* bitmap;
  uint64_t bits;
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
__device__ __forceinline__ void code_interval(uint64_t lo, uint64_t span, uint32_t neg0, uint64_t ref, uint32_t W,
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

// Decode + predicate one 512-row segment of width W from shared memory (u32
// words, LSB-first). Lane l handles rows l + 32k; word index l*W/32 + k*W and
// shift l*W mod 32 are per-lane constants. Lane k (< 16) receives mask word k.
template <int W>
__device__ __forceinline__ uint32_t seg_range32(const uint32_t* __restrict__ s, uint32_t a, uint32_t sp,
                                                uint32_t neg, uint32_t lane) {
  uint32_t my = 0;
  if constexpr (W == 0) {
    const bool keep = ((0u - a) <= sp) != (neg != 0);
    return lane < kSegWords ? (keep ? 0xffffffffu : 0u) : 0u;
  } else {
    constexpr uint32_t mask = W >= 32 ? 0xffffffffu : ((1u << (W & 31)) - 1);
    const uint32_t bitl = lane * W;
    const uint32_t* p = s + (bitl >> 5);
    const uint32_t sh = bitl & 31;
#pragma unroll
    for (int k = 0; k < kSegWords; ++k) {
      const uint32_t code = __funnelshift_r(p[k * W], p[k * W + 1], sh) & mask;
      const bool keep = ((code - a) <= sp) != (neg != 0);
      const uint32_t word = __ballot_sync(kFull, keep);
      if (lane == (uint32_t)k) my = word;
    }
  }
  return my;
}

template <int W>
__device__ __forceinline__ uint32_t seg_range64(const uint32_t* __restrict__ s, uint64_t d, uint64_t sp,
                                                uint32_t neg, uint32_t lane) {
  uint32_t my = 0;
  constexpr uint64_t mask = W >= 64 ? ~0ull : ((1ull << (W & 63)) - 1);
  const uint32_t bitl = lane * W;
  const uint32_t* p = s + (bitl >> 5);
  const uint32_t sh = bitl & 31;
#pragma unroll
  for (int k = 0; k < kSegWords; ++k) {
    const uint32_t w0 = p[k * W], w1 = p[k * W + 1], w2 = p[k * W + 2];
    const uint64_t code =
        (((uint64_t)__funnelshift_r(w1, w2, sh) << 32) | __funnelshift_r(w0, w1, sh)) & mask;
    const bool keep = ((code - d) <= sp) != (neg != 0);
    const uint32_t word = __ballot_sync(kFull, keep);
    if (lane == (uint32_t)k) my = word;
  }
  return my;
}

template <int W>
__device__ __forceinline__ uint32_t seg_bitmap(const uint32_t* __restrict__ s, uint64_t ref, const uint64_t* bm,
                                               uint64_t bits, uint32_t lane) {
  uint32_t my = 0;
  constexpr uint64_t mask = W >= 64 ? ~0ull : ((1ull << (W & 63)) - 1);
  const uint32_t bitl = lane * W;
  const uint32_t* p = s + (bitl >> 5);
  const uint32_t sh = bitl & 31;
#pragma unroll 4
  for (int k = 0; k < kSegWords; ++k) {
    uint64_t code = 0;
    if (W > 0) {
      const uint32_t w0 = p[k * W], w1 = p[k * W + 1], w2 = W > 32 ? p[k * W + 2] : 0u;
      code = (((uint64_t)__funnelshift_r(w1, w2, sh) << 32) | __funnelshift_r(w0, w1, sh)) & mask;
    }
    const uint64_t v = ref + code;
    const bool keep = v < bits && ((__ldg(bm + (v >> 6)) >> (v & 63)) & 1ull);
    const uint32_t word = __ballot_sync(kFull, keep);
    if (lane == (uint32_t)k) my = word;
  }
  return my;
}

// runtime width -> compile-time width (one instantiation per width)
template <int W>
__device__ __forceinline__ uint32_t seg_one(const uint32_t* s, const FastPred& p, uint64_t ref, uint32_t lane) {
  if (p.is_bitmap) return seg_bitmap<W>(s, ref, p.bitmap, p.bits, lane);
  if constexpr (W <= 32) {
    uint32_t a, sp, ng;
    code_interval(p.lo, p.span, p.neg, ref, W, a, sp, ng);
    return seg_range32<W>(s, a, sp, ng, lane);
  } else {
    return seg_range64<W>(s, p.lo - ref, p.span, p.neg, lane);
  }
}

__device__ __forceinline__ uint32_t seg_dispatch(uint32_t w, const uint32_t* s, const FastPred& p, uint64_t ref,
                                              uint32_t lane) {
  switch (w) {
#define MS_SEG_CASE(W) \
  case W:              \
    return seg_one<W>(s, p, ref, lane);
    MS_SEG_CASE(0) MS_SEG_CASE(1) MS_SEG_CASE(2) MS_SEG_CASE(3) MS_SEG_CASE(4) MS_SEG_CASE(5) MS_SEG_CASE(6)
    MS_SEG_CASE(7) MS_SEG_CASE(8) MS_SEG_CASE(9) MS_SEG_CASE(10) MS_SEG_CASE(11) MS_SEG_CASE(12)
    MS_SEG_CASE(13) MS_SEG_CASE(14) MS_SEG_CASE(15) MS_SEG_CASE(16) MS_SEG_CASE(17) MS_SEG_CASE(18)
    MS_SEG_CASE(19) MS_SEG_CASE(20) MS_SEG_CASE(21) MS_SEG_CASE(22) MS_SEG_CASE(23) MS_SEG_CASE(24)
    MS_SEG_CASE(25) MS_SEG_CASE(26) MS_SEG_CASE(27) MS_SEG_CASE(28) MS_SEG_CASE(29) MS_SEG_CASE(30)
    MS_SEG_CASE(31) MS_SEG_CASE(32) MS_SEG_CASE(33) MS_SEG_CASE(34) MS_SEG_CASE(35) MS_SEG_CASE(36)
    MS_SEG_CASE(37) MS_SEG_CASE(38) MS_SEG_CASE(39) MS_SEG_CASE(40) MS_SEG_CASE(41) MS_SEG_CASE(42)
    MS_SEG_CASE(43) MS_SEG_CASE(44) MS_SEG_CASE(45) MS_SEG_CASE(46) MS_SEG_CASE(47) MS_SEG_CASE(48)
    MS_SEG_CASE(49) MS_SEG_CASE(50) MS_SEG_CASE(51) MS_SEG_CASE(52) MS_SEG_CASE(53) MS_SEG_CASE(54)
    MS_SEG_CASE(55) MS_SEG_CASE(56) MS_SEG_CASE(57) MS_SEG_CASE(58) MS_SEG_CASE(59) MS_SEG_CASE(60)
    MS_SEG_CASE(61) MS_SEG_CASE(62) MS_SEG_CASE(63) MS_SEG_CASE(64)
#undef MS_SEG_CASE
    default:
      return 0;
  }
}

// UNCOMPR segment: 16 coalesced 64-bit loads per lane, predicate on the values
__device__ __forceinline__ uint32_t seg_uncompr(const uint64_t* __restrict__ v, const FastPred& p, uint32_t lane) {
  uint64_t x[kSegWords];
#pragma unroll
  for (int k = 0; k < kSegWords; ++k) x[k] = __ldg(v + lane + 32 * k);
  uint32_t my = 0;
#pragma unroll
  for (int k = 0; k < kSegWords; ++k) {
    bool keep;
    if (p.is_bitmap) keep = x[k] < p.bits && ((__ldg(p.bitmap + (x[k] >> 6)) >> (x[k] & 63)) & 1ull);
    else keep = ((x[k] - p.lo) <= p.span) != (p.neg != 0);
    const uint32_t word = __ballot_sync(kFull, keep);
    if (lane == (uint32_t)k) my = word;
  }
  return my;
}

// ---- TMA bulk copy + mbarrier helpers (sm_90+; SASS UBLKCP / SYNCS)
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

// Per-warp contiguous range of full 512-row segments [s_begin, s_end). Lane 0
// streams each segment's packed payload (64*w bytes, 64-byte aligned) into a
// per-warp ring of kStages shared-memory slots with one TMA bulk copy, tracked
// by one mbarrier per slot; the width / reference of the segment travel with
// the slot, so decoding needs no further global reads.
template <int KIND>
__global__ void __launch_bounds__(kFastWarps * 32, 2) select_fast_kernel(ColView c, FastPred pred,
                                                                        uint32_t* __restrict__ bits,
                                                                        uint32_t* __restrict__ seg_info, uint64_t NS,
                                                                        uint64_t spw) {
  extern __shared__ __align__(128) uint32_t fsm[];
  __shared__ __align__(8) uint64_t bars[kFastWarps][kStages];
  __shared__ uint64_t sref[kFastWarps][kStages];
  __shared__ uint32_t sw[kFastWarps][kStages];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)blockIdx.x * kFastWarps + wid;
  const uint64_t s_begin = gw * spw;
  if (s_begin >= NS) return;
  const uint64_t s_end = min(NS, s_begin + spw);
  uint32_t* buf = fsm + wid * (kStages * kBufU32);
  if (KIND != FAST_UNCOMPR && lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(&bars[wid][k], 1);
    mbar_fence_init();
  }
  __syncwarp();

  auto issue = [&](uint64_t s, int stage) {
    if (KIND == FAST_UNCOMPR || s >= s_end || lane != 0) return;
    uint32_t w;
    uint64_t off, ref = 0;
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
    if (w > 64) w = 65;  // corrupt width: decoded as no match (dispatch default)
    sw[wid][stage] = w;
    sref[wid][stage] = ref;
    const uint32_t bytes = w <= 64 ? 64 * w : 0;
    mbar_arrive_tx(&bars[wid][stage], bytes);
    if (bytes) bulk_g2s(buf + stage * kBufU32, c.payload + off, bytes, &bars[wid][stage]);
  };

  for (int k = 0; k < kStages - 1; ++k) issue(s_begin + k, k);
  int stage = 0;
  uint32_t phase = 0;
  for (uint64_t s = s_begin; s < s_end; ++s) {
    issue(s + kStages - 1, (stage + kStages - 1) % kStages);
    uint32_t my;
    if constexpr (KIND == FAST_UNCOMPR) {
      my = seg_uncompr(c.payload + s * kSegRows, pred, lane);
    } else {
      mbar_wait(&bars[wid][stage], phase);
      my = seg_dispatch(sw[wid][stage], buf + stage * kBufU32, pred, sref[wid][stage], lane);
    }
    __syncwarp();
    if (lane < kSegWords) bits[s * kSegWords + lane] = my;
    const uint32_t cnt = __reduce_add_sync(kFull, __popc(my));
    const uint32_t last = __reduce_max_sync(kFull, my ? lane * 32 + 32 - __clz(my) : 0u);
    if (lane == 0) seg_info[s] = cnt | (last << 16);
    if (++stage == kStages) {
      stage = 0;
      phase ^= 1u;
    }
  }
}

}  // namespace ms
