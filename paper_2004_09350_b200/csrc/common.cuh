// common.cuh — device building blocks of libms (sm_100a).
//
// The paper's operator is three layers: a column layer (host
// launcher: main part / remainder split, sizes, allocation), a buffer layer
// (format-specific decompression on the input side, compression on the output
// side) and a vector-register layer (the operator core). On the GPU:
//   buffer layer  -> CTA-cooperative tile decoders/encoders over a shared-memory
//                    tile of 2048 rows (the paper's 2048-element, 16 KiB
//                    output buffer, is the same size by design);
//   register core -> per-thread predicate / gather / accumulate, warp ballot +
//                    popc compaction (the "bit mask" of P:484-486).
// Device-wide prefixes (output offsets, cumulative widths) use a decoupled
// look-back over work items taken in order from an atomic ticket.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ms.h"

namespace ms {

constexpr int kChunk = 2048;               // rows per work item / tile
constexpr int kThreads = 256;              // CTA size of the generic engine
constexpr int kVPT = kChunk / kThreads;    // 8 values per thread
constexpr int kMaxBlocksPerChunk = kChunk / 128;
constexpr int kSegRows = 512;             // rows per select segment (16 mask words)
constexpr int kSegWords = kSegRows / 32;
constexpr unsigned kFull = 0xffffffffu;

// device error bits: bit s <=> ms_status s
__host__ __device__ constexpr uint32_t err_bit(int s) { return 1u << s; }

// ---------------------------------------------------------------- views
// A column as kernels see it (by value in kernel parameters).
struct ColView {
  int32_t format;
  uint32_t w;          // STATIC_BP width
  uint32_t maxw;       // block formats: largest block width hint (0 = unknown)
  uint32_t B;          // block size (block formats)
  uint32_t log2B;
  uint64_t n, nb, nrem, nruns;
  const uint64_t* payload;
  const uint32_t* cw;
  const uint64_t* ref;
  const uint64_t* rem;
  const uint64_t* run_starts;  // RLE: exclusive prefix of run lengths, nruns+1 entries (scratch)
  const uint32_t* chunk_run;   // RLE: index of the run covering row 2048*c (scratch)
};

// ------------------------------------------------------------ bit helpers
// effective bit width: 0 for 0, else index of highest set bit + 1
__device__ __forceinline__ uint32_t ebw64(uint64_t x) { return 64u - (uint32_t)__clzll((long long)x); }

__device__ __forceinline__ uint64_t low_mask(uint32_t w) { return w >= 64 ? ~0ull : ((1ull << w) - 1); }

// value at stream bit `bit`, width w (0..64), LSB-first uint64 words (D-1)
__device__ __forceinline__ uint64_t unpack_at(const uint64_t* __restrict__ p, uint64_t bit, uint32_t w) {
  if (w == 0) return 0;
  const uint64_t word = bit >> 6;
  const uint32_t s = (uint32_t)(bit & 63);
  uint64_t v = __ldg(p + word) >> s;
  if (s + w > 64) v |= __ldg(p + word + 1) << (64 - s);
  return v & low_mask(w);
}

// 64-bit look-back status words: GPU-scope relaxed accesses (single-copy
// atomic; the flag and the value travel in the same word, so no ordering with
// other data is needed). `volatile` would compile to system-scope loads.
__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------------------------ scans
__device__ __forceinline__ uint64_t warp_incl_scan(uint64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t t = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_sum(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ uint64_t warp_max(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t t = __shfl_xor_sync(kFull, v, o);
    v = t > v ? t : v;
  }
  return v;
}

// CTA-wide exclusive scan (kThreads threads). sm must hold >= 10 uint64.
// Returns the exclusive prefix; *total gets the CTA total. Ends with a barrier.
__device__ __forceinline__ uint64_t cta_excl_scan(uint64_t v, uint64_t* sm, uint64_t* total) {
  constexpr int kWarps = kThreads / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t inc = warp_incl_scan(v);
  if (lane == 31) sm[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    uint64_t x = lane < kWarps ? sm[lane] : 0;
    uint64_t xi = warp_incl_scan(x);
    if (lane < kWarps) sm[lane] = xi - x;
    if (lane == kWarps - 1) sm[kWarps] = xi;
  }
  __syncthreads();
  const uint64_t ex = sm[wid] + inc - v;
  if (total) *total = sm[kWarps];
  __syncthreads();
  return ex;
}

// ------------------------------------------------------- decoupled look-back
// status word: [63:62] flag (0 invalid, 1 aggregate, 2 inclusive prefix),
// [61:0] value. Items are taken in increasing order from an atomic ticket, so
// every item only waits on items that are already being processed by resident
// CTAs (no deadlock).
constexpr uint64_t kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

// Exclusive prefix of item t (t >= 1) from the status words of its
// predecessors; call with ALL 32 lanes of ONE warp. Each round reads a window of
// 128 predecessors (lane j: items base-4j .. base-4j-3, four independent loads
// in flight), spins only on the ones not yet published, and stops at the first
// inclusive prefix (flag P) in descending item order. The window width sets how
// fast the P frontier can advance (128 items per L2 round trip).
__device__ __forceinline__ uint64_t lookback_walk(uint64_t* status, uint64_t t) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = (int64_t)t - 1;
  while (true) {
    uint64_t s[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t idx = base - 4 * lane - i;
      s[i] = idx >= 0 ? ld_volatile(&status[idx]) : kFlagP;  // before item 0: prefix 0
    }
    int spins = 0;
    while (((s[0] >> 62) == 0) | ((s[1] >> 62) == 0) | ((s[2] >> 62) == 0) | ((s[3] >> 62) == 0)) {
      if (++spins > 4) __nanosleep(32);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if ((s[i] >> 62) == 0) s[i] = ld_volatile(&status[base - 4 * lane - i]);
    }
    int first_i = 4;
#pragma unroll
    for (int i = 3; i >= 0; --i)
      if ((s[i] >> 62) == 2) first_i = i;
    const unsigned pmask = __ballot_sync(kFull, first_i < 4);
    const int first_lane = pmask ? __ffs(pmask) - 1 : 32;
    uint64_t v = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (lane < first_lane || (lane == first_lane && i <= first_i)) v += s[i] & kValMask;
    excl += warp_sum(v);
    if (pmask) break;
    base -= 128;
  }
  excl &= kValMask;
  return excl;
}

// Call with ALL 32 lanes of ONE warp. Returns the exclusive prefix of item t.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, uint64_t t, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    if (lane == 0) st_volatile(&status[0], kFlagP | agg);
    return 0;
  }
  if (lane == 0) st_volatile(&status[t], kFlagA | agg);
  const uint64_t excl = lookback_walk(status, t);
  if (lane == 0) st_volatile(&status[t], kFlagP | ((excl + agg) & kValMask));
  return excl;
}

// Split look-back: publish the aggregate early, resolve the exclusive prefix
// later (by then the predecessors have had time to publish theirs).
__device__ __forceinline__ void lookback_publish(uint64_t* status, uint64_t t, uint64_t agg) {
  if ((threadIdx.x & 31) == 0) st_volatile(&status[t], (t == 0 ? kFlagP : kFlagA) | agg);
}
__device__ __forceinline__ uint64_t lookback_resolve(uint64_t* status, uint64_t t, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (t == 0) return 0;
  const uint64_t excl = lookback_walk(status, t);
  if (lane == 0) st_volatile(&status[t], kFlagP | ((excl + agg) & kValMask));
  return excl;
}

// Stream N codes c[q] (< 2^w, w <= 64) into u32 words `buf` at bits
// [bit0, bit0 + N*w) — the caller's contiguous range: plain stores for the words
// inside it, atomicOr for the (at most two) words it may share with the
// neighbouring ranges. `buf` must be zeroed; the caller synchronises.
template <int N>
__device__ __forceinline__ void stream_codes(uint32_t* buf, const uint64_t (&c)[N], uint32_t w, uint32_t bit0) {
  if (!w) return;
  uint32_t widx = bit0 >> 5, nb = bit0 & 31;
  uint64_t acc = 0;
  bool first = true;
  auto flush = [&]() {
    if (first) {
      atomicOr(buf + widx, (uint32_t)acc);
      first = false;
    } else {
      buf[widx] = (uint32_t)acc;
    }
    ++widx;
    acc >>= 32;
    nb -= 32;
  };
#pragma unroll
  for (int q = 0; q < N; ++q) {
    if (w <= 32) {
      acc |= c[q] << nb;
      nb += w;
      if (nb >= 32) flush();
    } else {
      acc |= (c[q] & 0xffffffffull) << nb;
      nb += 32;
      flush();
      acc |= (c[q] >> 32) << nb;
      nb += w - 32;
      if (nb >= 32) flush();
    }
  }
  if (nb) atomicOr(buf + widx, (uint32_t)acc);
}

// floor(x / w) for x < 2^20, 1 <= w <= 64, given magic = 0xffffffff / w + 1
// (computed once per block): a multiply-high plus one correction step
__device__ __forceinline__ uint32_t div_small(uint32_t x, uint32_t w, uint32_t magic) {
  if (w == 1) return x;
  uint32_t q = __umulhi(x, magic);
  if (q * w > x) --q;
  if ((q + 1) * w <= x) ++q;
  return q;
}

// select-in-word: position of the (k+1)-th set bit of x (k < popc(x))
__device__ __forceinline__ uint32_t select_bit(uint32_t x, uint32_t k) {  // by halving: five popcounts
  uint32_t pos = 0;
#pragma unroll
  for (int h = 16; h > 0; h >>= 1) {
    const uint32_t c = __popc(x & ((1u << h) - 1u));
    if (k >= c) {
      k -= c;
      x >>= h;
      pos += h;
    }
  }
  return pos;
}

// ---------------------------------------------------------- random access
// value at row r of a column (r < c.n). O(1) for UNCOMPR, STATIC_BP, DYN_BP,
// FOR_BP (cw / ref headers, D-12); O(B) for DELTA_BP (prefix inside the
// block); O(log R) for RLE (search of the run starts).
__device__ __forceinline__ uint64_t read_row(const ColView& c, uint64_t r) {
  switch (c.format) {
    case MS_UNCOMPR:
      return __ldg(c.payload + r);
    case MS_STATIC_BP:
      return unpack_at(c.payload, r * c.w, c.w);
    case MS_DYN_BP:
    case MS_FOR_BP:
    case MS_DELTA_BP: {
      if (r >= (c.nb << c.log2B)) return __ldg(c.rem + (r - (c.nb << c.log2B)));
      const uint64_t b = r >> c.log2B;
      const uint32_t j = (uint32_t)(r & (c.B - 1));
      const uint32_t cw0 = __ldg(c.cw + b);
      const uint32_t w = __ldg(c.cw + b + 1) - cw0;
      const uint64_t bit0 = (uint64_t)cw0 * c.B;
      if (c.format == MS_DYN_BP) return unpack_at(c.payload, bit0 + (uint64_t)j * w, w);
      if (c.format == MS_FOR_BP) return __ldg(c.ref + b) + unpack_at(c.payload, bit0 + (uint64_t)j * w, w);
      uint64_t v = __ldg(c.ref + b);
      for (uint32_t q = 0; q <= j; ++q) v += unpack_at(c.payload, bit0 + (uint64_t)q * w, w);
      return v;
    }
    case MS_RLE: {
      uint64_t lo = 0, hi = c.nruns;  // find last k with starts[k] <= r
      while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(c.run_starts + mid) <= r) lo = mid; else hi = mid;
      }
      return __ldg(c.payload + 2 * lo);
    }
  }
  return 0;
}

// -------------------------------------------------------- tile decoder
// Shared memory of the generic engine.
struct EngineSmem {
  alignas(16) uint64_t vals[kChunk];
  uint64_t ex[kThreads];
  uint64_t scan[16];
  uint64_t bmin[kMaxBlocksPerChunk], bmax[kMaxBlocksPerChunk], bex[kMaxBlocksPerChunk + 1];
  uint32_t bw[kMaxBlocksPerChunk];
  uint32_t item;
  uint32_t flag;
  uint64_t aux;
};

// sm[0..8) = v[0..8) for thread-consecutive rows (thread t owns 8 rows at 64 t bytes):
// four 128-bit stores, thread t starting at pair (t >> 1) & 3 so that the 8 threads
// of a wavefront hit 8 distinct 16-byte bank groups (plain stores: 16-way conflicts)
__device__ __forceinline__ void store8_rotated(uint64_t* sm, const uint64_t (&v)[kVPT]) {
  static_assert(kVPT == 8, "store8_rotated assumes 8 rows per thread");
  const uint32_t rot = (threadIdx.x >> 1) & 3;
#pragma unroll
  for (uint32_t k = 0; k < 4; ++k) {
    const uint32_t p = (k + rot) & 3;
    const uint64_t a0 = (p & 1) ? v[2] : v[0], a1 = (p & 1) ? v[3] : v[1];
    const uint64_t b0 = (p & 1) ? v[6] : v[4], b1 = (p & 1) ? v[7] : v[5];
    reinterpret_cast<ulonglong2*>(sm)[p] = make_ulonglong2((p & 2) ? b0 : a0, (p & 2) ? b1 : a1);
  }
}

// Decode rows [r0, r0+cnt) of column c into sm.vals (buffer layer, input side,
// P:479-481). r0 is a multiple of kChunk (hence of every block size), cnt <= kChunk.
// Ends with a barrier.
__device__ __forceinline__ void load_rows(const ColView& c, uint64_t r0, uint32_t cnt, EngineSmem& sm) {
  const int tid = threadIdx.x;
  switch (c.format) {
    // the O(1) formats: all kVPT loads of a thread issued before any is stored
    // (a runtime-bounded loop would serialise one memory latency per row)
    case MS_UNCOMPR: {
      uint64_t v[kVPT];
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        const uint32_t i = tid + q * kThreads;
        v[q] = i < cnt ? __ldg(c.payload + r0 + i) : 0ull;
      }
#pragma unroll
      for (int q = 0; q < kVPT; ++q) sm.vals[tid + q * kThreads] = v[q];
      break;
    }
    case MS_STATIC_BP: {
      uint64_t v[kVPT];
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        const uint32_t i = tid + q * kThreads;
        v[q] = i < cnt ? unpack_at(c.payload, (r0 + i) * c.w, c.w) : 0ull;
      }
#pragma unroll
      for (int q = 0; q < kVPT; ++q) sm.vals[tid + q * kThreads] = v[q];
      break;
    }
    case MS_DYN_BP:
    case MS_FOR_BP: {
      uint64_t v[kVPT];
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        const uint32_t i = tid + q * kThreads;
        v[q] = i < cnt ? read_row(c, r0 + i) : 0ull;
      }
#pragma unroll
      for (int q = 0; q < kVPT; ++q) sm.vals[tid + q * kThreads] = v[q];
      break;
    }
    case MS_DELTA_BP: {
      // thread t owns rows [8t, 8t+8): local prefix of the deltas, CTA scan,
      // then subtract the prefix at the block head (segmented scan).
      const uint32_t i0 = tid * kVPT;
      const uint64_t r = r0 + i0;
      const uint64_t main_rows = c.nb << c.log2B;
      uint64_t loc[kVPT];
      uint64_t tsum = 0;
      const bool in_main = i0 < cnt && r < main_rows;
      uint64_t b = 0, ref_b = 0;
      if (in_main) {
        b = r >> c.log2B;
        const uint32_t j0 = (uint32_t)(r & (c.B - 1));
        const uint32_t cw0 = __ldg(c.cw + b);
        const uint32_t w = __ldg(c.cw + b + 1) - cw0;
        ref_b = __ldg(c.ref + b);  // issued with the header, used after the scan
        // in-block bit positions in 32 bits (j * w < 2^17); the block starts word-aligned (B % 64 == 0)
        const uint64_t* __restrict__ blk = c.payload + (uint64_t)cw0 * (c.B / 64);
        const uint64_t mask = low_mask(w);
        uint32_t pos = j0 * w;
#pragma unroll
        for (int q = 0; q < kVPT; ++q) {
          uint64_t x = 0;
          if (w) {
            const uint32_t wi = pos >> 6, sh = pos & 63;
            x = __ldg(blk + wi) >> sh;
            if (sh + w > 64) x |= __ldg(blk + wi + 1) << (64 - sh);
          }
          tsum += x & mask;
          loc[q] = tsum;
          pos += w;
        }
      }
      const uint64_t ex = cta_excl_scan(in_main ? tsum : 0, sm.scan, nullptr);
      sm.ex[tid] = ex;
      __syncthreads();
      if (in_main) {
        const uint32_t head = (uint32_t)(((b << c.log2B) - r0) / kVPT);
        const uint64_t base = ref_b + (ex - sm.ex[head]);
#pragma unroll
        for (int q = 0; q < kVPT; ++q) loc[q] += base;
        store8_rotated(sm.vals + i0, loc);
      } else {
        for (int q = 0; q < kVPT; ++q)
          if (i0 + q < cnt) sm.vals[i0 + q] = __ldg(c.rem + (r + q - main_rows));
      }
      break;
    }
    case MS_RLE: {
      // mark run starts inside the chunk, scan the marks -> run index per row
      const uint64_t k0 = __ldg(c.chunk_run + (r0 / kChunk));
      const uint32_t i0 = tid * kVPT;
      // reuse sm.vals as the mark array (1 = a run starts at this row, row > r0)
#pragma unroll
      for (int q = 0; q < kVPT; ++q) sm.vals[tid + q * kThreads] = 0;
      __syncthreads();
      for (uint64_t k = k0 + 1 + tid;; k += kThreads) {
        if (k >= c.nruns) break;
        const uint64_t s = __ldg(c.run_starts + k);
        if (s >= r0 + cnt) break;
        if (s > r0) sm.vals[s - r0] = 1;  // s <= r0: corrupt (non-monotone) starts, reported by StartsEpi
      }
      __syncthreads();
      uint64_t loc[kVPT];
      uint64_t tsum = 0;
#pragma unroll
      for (int q = 0; q < kVPT; q += 2) {
        const ulonglong2 m2 = reinterpret_cast<const ulonglong2*>(sm.vals + i0)[q / 2];
        tsum += m2.x;
        loc[q] = tsum;
        tsum += m2.y;
        loc[q + 1] = tsum;
      }
      const uint64_t ex = cta_excl_scan(tsum, sm.scan, nullptr);
      if (i0 + kVPT <= cnt) {
#pragma unroll
        for (int q = 0; q < kVPT; ++q) loc[q] = __ldg(c.payload + 2 * (k0 + ex + loc[q]));
        store8_rotated(sm.vals + i0, loc);
      } else {
        for (int q = 0; q < kVPT; ++q)
          if (i0 + q < cnt) sm.vals[i0 + q] = __ldg(c.payload + 2 * (k0 + ex + loc[q]));
      }
      break;
    }
  }
  __syncthreads();
}

}  // namespace ms
