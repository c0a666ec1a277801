// selstream.cuh — the select (and sum) core of select_fast.cuh in a
// producer / consumer CTA, for bit-packed inputs of width <= 32 (STATIC_BP,
// DYN_BP / FOR_BP with B >= 512): the column is streamed through shared memory
// in chunks of 16 segments (8192 rows).
//
//   select_stream_kernel  persistent, one CTA per SM, each CTA a contiguous run
//                         of chunks; S stages of 1024*maxw bytes (S <= 10 from
//                         the max_width hint) and 2S consumer warps. Warp 0
//                         computes the chunk descriptors 32 at a time (payload
//                         byte range, header ranges; ss_chunk) and issues one
//                         TMA bulk copy of the chunk's payload plus
//                         its headers into stage li % S (mbarrier complete_tx);
//                         consumer pair li % S evaluates the chunk (warp h:
//                         segments [8h, 8h+8), two at a time, half-warp: one
//                         segment, lane_dispatch:
//                         lane-consecutive compile-time-width unpack, code-domain
//                         predicate) and writes the mask words and seg_info,
//                         then releases the stage (or, CORE_SUM, accumulates).
//                         A chunk wider than the hint is read from global memory.
// The per-warp ring of select_fast_kernel keeps one segment pair in flight per
// warp; here a whole CTA's stages are in flight while its warps compute.
#pragma once
#include "common.cuh"
#include "select_fast.cuh"
#include "tma.cuh"

namespace ms {

constexpr uint32_t kSsSegs = 16;      // segments per chunk
constexpr int kSsMaxStages = 10;     // stages; two consumer warps per stage
constexpr uint32_t kSsCwU32 = 24;     // cw of <= 16 blocks + 1, 16-byte aligned (+ 6)
constexpr uint32_t kSsRefU64 = 20;    // ref of <= 16 blocks, 16-byte aligned (+ 2)

struct SsChunk {
  uint64_t byte0;   // payload byte of the chunk's first segment
  uint32_t bytes;   // payload bytes (0xffffffff: wider than the max_width hint -> not staged)
  uint32_t ia, ja;  // first cw / ref index copied
  uint32_t ncw, nref;
  uint32_t nseg;
};

struct alignas(16) SsHead {  // per stage: headers + chunk descriptor (16-byte aligned)
  uint32_t cw[kSsCwU32];
  uint64_t ref[kSsRefU64];
  SsChunk m;
  uint32_t pad[1];
};

__host__ __device__ inline size_t ss_stage_bytes(uint32_t maxw) {  // payload + slack for look-ahead reads
  return (size_t)kSsSegs * 64 * maxw + 64;
}
__host__ __device__ inline size_t ss_smem_bytes(uint32_t maxw, int S) {
  return (ss_stage_bytes(maxw) + sizeof(SsHead)) * S + 2 * kSsMaxStages * 8 + 32 * sizeof(SsChunk);
}
// stages (= consumer warps) for a max width: as many as fit 220 KiB, at most kSsMaxStages
__host__ __device__ inline int ss_stages(uint32_t maxw) {
  const size_t fixed = 2 * kSsMaxStages * 8 + 32 * sizeof(SsChunk);
  const size_t per = ss_stage_bytes(maxw) + sizeof(SsHead);
  const size_t s = (220 * 1024 - fixed) / per;
  return (int)(s > (size_t)kSsMaxStages ? kSsMaxStages : s);
}

// chunk k's descriptor (segments [16k, 16k+16) of NS): its payload byte range
// (64-byte aligned: segments start at multiples of 8 words) and the 16-byte
// aligned header ranges (cw, ref) that lie inside the arrays (the consumer
// reads any entry past them from global memory). Split in two so the producer
// can issue the loads of the next batch before it issues the current one.
struct SsRaw {
  uint32_t a0, a1, e0, e1;
};
template <int KIND>
__device__ __forceinline__ SsRaw ss_raw(const ColView& c, uint64_t NS, uint64_t k) {
  SsRaw r{0, 0, 0, 0};
  if constexpr (KIND == FAST_BLOCK) {
    const uint64_t s0 = k * kSsSegs, s1 = min(NS, s0 + kSsSegs);
    const uint64_t m = (c.B >> 9) - 1;
    const uint64_t b0 = (s0 * kSegRows) >> c.log2B, b1 = (s1 * kSegRows) >> c.log2B;
    r.a0 = __ldg(c.cw + b0);
    if (s0 & m) r.a1 = __ldg(c.cw + b0 + 1);
    r.e0 = __ldg(c.cw + b1);
    if (s1 & m) r.e1 = __ldg(c.cw + b1 + 1);
  }
  return r;
}
template <int KIND>
__device__ __forceinline__ SsChunk ss_chunk(const ColView& c, uint64_t NS, uint32_t maxw, uint64_t k,
                                            const SsRaw& r) {
  SsChunk m{};
  const uint64_t s0 = k * kSsSegs, s1 = min(NS, s0 + kSsSegs);
  m.nseg = (uint32_t)(s1 - s0);
  uint64_t w0, w1;
  if constexpr (KIND == FAST_STATIC) {
    w0 = s0 * 8 * (uint64_t)c.w;
    w1 = s1 * 8 * (uint64_t)c.w;
  } else {
    const uint64_t msk = (c.B >> 9) - 1;
    w0 = (uint64_t)r.a0 * (c.B >> 6) + (s0 & msk) * 8 * (uint64_t)(r.a1 - r.a0);
    w1 = (uint64_t)r.e0 * (c.B >> 6) + (s1 & msk) * 8 * (uint64_t)(r.e1 - r.e0);
  }
  m.byte0 = w0 * 8;
  const uint64_t bytes = (w1 - w0) * 8;
  m.bytes = w1 >= w0 && bytes <= (uint64_t)kSsSegs * 64 * maxw ? (uint32_t)bytes : 0xffffffffu;
  if constexpr (KIND == FAST_BLOCK) {
    const uint64_t b0 = (s0 * kSegRows) >> c.log2B, b1 = (s1 * kSegRows - 1) >> c.log2B;
    const uint64_t ia = b0 & ~3ull, ib = min((b1 + 2 + 3) & ~3ull, (c.nb + 1) & ~3ull);
    m.ia = (uint32_t)ia;
    m.ncw = ib > ia ? (uint32_t)(ib - ia) : 0u;
    if (c.ref) {
      const uint64_t ja = b0 & ~1ull, jb = min((b1 + 1 + 1) & ~1ull, c.nb & ~1ull);
      m.ja = (uint32_t)ja;
      m.nref = jb > ja ? (uint32_t)(jb - ja) : 0u;
    }
  }
  return m;
}

template <int KIND, int CORE>
__global__ void __launch_bounds__((1 + 2 * kSsMaxStages) * 32, 1)
    select_stream_kernel(ColView c, FastPred pred, uint32_t* __restrict__ bits, uint32_t* __restrict__ seg_info,
                         uint64_t NS, uint32_t maxw, uint32_t* err,
                         unsigned long long* sum_out) {
  extern __shared__ __align__(128) uint8_t ss_sm[];
  const int S = (int)(blockDim.x >> 6);  // stages (blockDim = (1 + 2S) warps)
  const size_t sb = ss_stage_bytes(maxw);
  uint8_t* stage_base = ss_sm;
  SsHead* heads = reinterpret_cast<SsHead*>(ss_sm + sb * S);
  uint64_t* full = reinterpret_cast<uint64_t*>(heads + S);
  uint64_t* empty = full + kSsMaxStages;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t nchunks = (NS + kSsSegs - 1) / kSsSegs;
  const uint64_t per_cta = (nchunks + gridDim.x - 1) / gridDim.x;
  const uint64_t i_lo = (uint64_t)blockIdx.x * per_cta;
  const uint64_t i_hi = min(nchunks, i_lo + per_cta);
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) {
      mbar_init(full + k, 1);
      mbar_init(empty + k, 2);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (i_lo >= i_hi) return;
  if (wid == 0) {  // ---------------- producer: descriptors for 32 chunks at a time (lane j: chunk base + j)
    const char* pay = reinterpret_cast<const char*>(c.payload);
    SsChunk* pm = reinterpret_cast<SsChunk*>(empty + kSsMaxStages);  // [32]
    SsRaw raw = ss_raw<KIND>(c, NS, min(i_lo + lane, i_hi - 1));
    for (uint64_t base = i_lo; base < i_hi; base += 32) {
      const uint64_t k = base + lane;
      const SsChunk mine = ss_chunk<KIND>(c, NS, maxw, min(k, i_hi - 1), raw);
      if (base + 32 < i_hi) raw = ss_raw<KIND>(c, NS, min(k + 32, i_hi - 1));  // next batch in flight
      __syncwarp();
      pm[lane] = mine;
      __syncwarp();
      if (lane == 0) {
        const uint32_t nj = (uint32_t)min((uint64_t)32, i_hi - base);
        for (uint32_t j = 0; j < nj; ++j) {
          const uint64_t li = base + j - i_lo;
          const uint32_t sg = (uint32_t)(li % S);
          const uint64_t round = li / S;
          if (round) mbar_wait(empty + sg, (uint32_t)((round - 1) & 1));
          const SsChunk m = pm[j];
          SsHead& H = heads[sg];
          H.m = m;
          if (m.bytes == 0xffffffffu) {  // wider than the hint: the consumers read global memory
            H.m.ncw = H.m.nref = 0;
            mbar_arrive(full + sg);
            continue;
          }
          const uint32_t cb = m.ncw * 4, rb = m.nref * 8;
          mbar_arrive_tx(full + sg, m.bytes + cb + rb);
          if (m.bytes) bulk_g2s(stage_base + sb * sg, pay + m.byte0, m.bytes, full + sg);
          if (cb) bulk_g2s(H.cw, c.cw + m.ia, cb, full + sg);
          if (rb) bulk_g2s(H.ref, c.ref + m.ja, rb, full + sg);
        }
      }
      __syncwarp();
    }
    return;
  }
  // ------------------------------------ consumers: warps 2p+1, 2p+2 take chunks p, p + S, ... (stage li % S),
  // warp h of the two the segments [8h, 8h+8) of each
  const uint32_t cwarp = wid - 1, pr = cwarp >> 1, sub = cwarp & 1;
  const uint32_t half = lane >> 4, hl = lane & 15;
  const uint32_t* gpay = reinterpret_cast<const uint32_t*>(c.payload);
  uint64_t sum_acc = 0;
  for (uint64_t li = pr; i_lo + li < i_hi; li += S) {
    const uint32_t sg = (uint32_t)(li % S);
    mbar_wait(full + sg, (uint32_t)((li / S) & 1));
    const SsHead& H = heads[sg];
    const SsChunk m = H.m;
    // a chunk wider than the max_width hint was not staged: read from global memory
    const bool staged = m.bytes != 0xffffffffu;
    const uint32_t* base = staged ? reinterpret_cast<const uint32_t*>(stage_base + sb * sg) : gpay + m.byte0 / 4;
    const uint64_t s0 = (i_lo + li) * kSsSegs;
    const uint32_t q_end = min(m.nseg, 8 * sub + 8);
    for (uint32_t p = 8 * sub; p < q_end; p += 2) {
      const uint32_t q = p + half;
      const bool valid = q < q_end;
      const uint64_t seg = s0 + q;
      uint32_t mword = 0;
      if (valid) {
        uint32_t w;
        uint64_t ref = 0, word;
        if constexpr (KIND == FAST_STATIC) {
          w = c.w;
          word = (uint64_t)q * 8 * w;
        } else {
          const uint64_t b = (seg * kSegRows) >> c.log2B;
          const uint32_t hb = (uint32_t)(b - m.ia);
          const uint32_t cw0 = hb < m.ncw ? H.cw[hb] : __ldg(c.cw + b);
          w = (hb + 1 < m.ncw ? H.cw[hb + 1] : __ldg(c.cw + b + 1)) - cw0;
          word = (uint64_t)cw0 * (c.B >> 6) + (seg & ((c.B >> 9) - 1)) * 8 * (uint64_t)w - m.byte0 / 8;
          if (c.ref) ref = b - m.ja < m.nref ? H.ref[b - m.ja] : __ldg(c.ref + b);
        }
        if (w > 64) {  // corrupt width table
          if (hl == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
        } else {
          const uint32_t* pp = base + 2 * word + hl * w;
          if constexpr (CORE == CORE_SUM) {
            sum_acc += lane_sum_dispatch<false>(w, pp) + (hl == 0 ? (uint64_t)kSegRows * ref : 0ull);
          } else {
            mword = lane_dispatch<false>(w, pp, pred, ref);
          }
        }
      }
      if constexpr (CORE == CORE_SELECT) {
        if (valid) bits[seg * kSegWords + hl] = mword;
        uint32_t cnt = __popc(mword);
        uint32_t last = mword ? hl * 32 + 32 - __clz(mword) : 0u;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          cnt += __shfl_xor_sync(kFull, cnt, o);
          last = max(last, __shfl_xor_sync(kFull, last, o));
        }
        if (valid && hl == 0) seg_info[seg] = cnt | (last << 16);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + sg);
  }
  if constexpr (CORE == CORE_SUM) {
    sum_acc = warp_sum(sum_acc);
    if (lane == 0 && sum_acc) atomicAdd(sum_out, (unsigned long long)sum_acc);
  }
}

}  // namespace ms
