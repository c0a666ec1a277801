// stage.cuh — the engine's column source with its input staged through shared
// memory (compress / decompress / morph).
//
// A tile's compressed input is one contiguous word range of the payload (plus, for
// the block formats, its blocks' cw / ref header entries, D-4 / D-6 / D-7). The
// staged engine copies the NEXT tile's range into shared memory with cp.async
// while it decodes and encodes the current one, and the header entries one more
// tile ahead (the payload range follows from them), so a CTA never waits on a
// dependent global round trip per tile: the plain engine (load_rows) was
// latency-bound at ~2 ms for 2^29 rows of c3 whatever the bytes.
//
//   iteration k (tile t = blockIdx.x + k * gridDim.x):
//     wait for group k-1 {payload(t), headers(t + G)}; barrier
//     issue group k {payload(t + G) -> buffer (k+1)&1, headers(t + 2G) -> slot (k+2)%3}
//     decode tile t from buffer k&1 / slot k%3 into sm.vals; encode_tile
#pragma once
#include "engine.cuh"

namespace ms {

struct StageSmem {
  alignas(16) uint64_t words[2][kChunk + 2];  // <= 2048 words per tile (64 bits per row) + alignment
  uint32_t cw[3][kMaxBlocksPerChunk + 1];
  uint64_t ref[3][kMaxBlocksPerChunk];
  uint32_t off[2];  // word offset of the tile's first word in words[buf] (16-byte copies)
};

__device__ __forceinline__ void st_cp8(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void st_cp16(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void st_cp4(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void st_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void st_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__host__ __device__ inline bool stageable_format(int32_t f) {
  return f == MS_UNCOMPR || f == MS_STATIC_BP || f == MS_DYN_BP || f == MS_FOR_BP || f == MS_DELTA_BP;
}

// F: the source format (compile-time: no dead decode paths, fewer registers)
template <int F>
struct StagedCol {
  ColView c;
  uint64_t main_rows;  // block formats: nb * B

  __device__ __forceinline__ bool is_block() const {
    return F == MS_DYN_BP || F == MS_FOR_BP || F == MS_DELTA_BP;
  }
  // full blocks of tile t: [kb0, kb0 + nbk)
  __device__ __forceinline__ uint32_t tile_blocks(uint64_t t, uint64_t& kb0) const {
    kb0 = (t * kChunk) >> c.log2B;
    if (kb0 >= c.nb) return 0;
    const uint64_t kb1 = min(kb0 + (kChunk >> c.log2B), c.nb);
    return (uint32_t)(kb1 - kb0);
  }
  __device__ __forceinline__ void issue_headers(uint64_t t, StageSmem& st, int slot) const {
    if (!is_block()) return;
    uint64_t kb0;
    const uint32_t nbk = tile_blocks(t, kb0);
    if (!nbk) return;
    const int tid = threadIdx.x;
    if (tid <= (int)nbk) st_cp4(&st.cw[slot][tid], c.cw + kb0 + tid);
    if (F != MS_DYN_BP && tid < (int)nbk) st_cp8(&st.ref[slot][tid], c.ref + kb0 + tid);
  }
  // word range [lo, hi) of tile t's payload; block formats read it from the staged headers
  __device__ __forceinline__ void range(uint64_t t, uint32_t cnt, const StageSmem& st, int slot, uint64_t& lo,
                                        uint64_t& hi) const {
    const uint64_t r0 = t * kChunk;
    if (F == MS_UNCOMPR) {
      lo = r0;
      hi = r0 + cnt;
    } else if (F == MS_STATIC_BP) {
      lo = (r0 * c.w) >> 6;
      hi = ((r0 + cnt) * c.w + 63) >> 6;
    } else {
      uint64_t kb0;
      const uint32_t nbk = tile_blocks(t, kb0);
      lo = hi = 0;
      if (nbk) {
        lo = (uint64_t)st.cw[slot][0] * (c.B / 64);
        hi = (uint64_t)st.cw[slot][nbk] * (c.B / 64);
      }
    }
  }
  // payload(t) -> words[buf][off ..], off = lo & 1 when the payload is 16-byte aligned
  // (16-byte copies from the even word below lo; the odd last word by an 8-byte copy)
  __device__ __forceinline__ void issue_payload(uint64_t t, uint64_t n, StageSmem& st, int buf, int slot) const {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, n - r0);
    uint64_t lo, hi;
    range(t, cnt, st, slot, lo, hi);
    const bool al16 = (reinterpret_cast<uintptr_t>(c.payload) & 15) == 0;
    if (threadIdx.x == 0) st.off[buf] = al16 ? (uint32_t)(lo & 1) : 0u;  // read after the next barrier
    if (hi <= lo) return;
    if (al16) {
      const uint64_t base = lo & ~1ull;
      const uint32_t nw = (uint32_t)(hi - base), npair = nw >> 1;
      const ulonglong2* src = reinterpret_cast<const ulonglong2*>(c.payload + base);
      for (uint32_t i = threadIdx.x; i < npair; i += kThreads) st_cp16(&st.words[buf][2 * i], src + i);
      if ((nw & 1) && threadIdx.x == 0) st_cp8(&st.words[buf][nw - 1], c.payload + base + nw - 1);
    } else {
      for (uint32_t i = threadIdx.x; i < (uint32_t)(hi - lo); i += kThreads) st_cp8(&st.words[buf][i], c.payload + lo + i);
    }
  }
  // rows [r0, r0 + cnt) of tile t from the staged words into sm.vals (ends with a
  // barrier), or, kMaxOnly, only their running maximum in mx (no stores, no barrier)
  template <bool kMaxOnly>
  __device__ __forceinline__ void decode(uint64_t t, uint32_t cnt, const StageSmem& st, int buf, int slot,
                                         EngineSmem& sm, uint64_t& mx) const {
    const int tid = threadIdx.x;
    const uint64_t r0 = t * kChunk;
    const uint64_t* __restrict__ wd = st.words[buf] + st.off[buf];
    auto put = [&](uint32_t i, uint64_t v) {
      if (kMaxOnly) mx = v > mx ? v : mx;
      else sm.vals[i] = v;
    };
    switch (F) {
      case MS_UNCOMPR:
#pragma unroll
        for (int q = 0; q < kVPT; ++q) {
          const uint32_t i = tid + q * kThreads;
          if (i < cnt) put(i, wd[i]);
        }
        break;
      case MS_STATIC_BP: {
        const uint32_t w = c.w;
        const uint64_t mask = low_mask(w);
#pragma unroll
        for (int q = 0; q < kVPT; ++q) {
          const uint32_t i = tid + q * kThreads;
          if (i < cnt) {
            const uint32_t pos = i * w, wi = pos >> 6, sh = pos & 63;
            uint64_t x = wd[wi] >> sh;
            if (sh + w > 64) x |= wd[wi + 1] << (64 - sh);
            put(i, x & mask);
          }
        }
        break;
      }
      case MS_DYN_BP:
      case MS_FOR_BP: {
        const uint32_t nmain = r0 < main_rows ? (uint32_t)min((uint64_t)cnt, main_rows - r0) : 0u;
        const uint32_t cwb = nmain ? st.cw[slot][0] : 0u;
#pragma unroll
        for (int q = 0; q < kVPT; ++q) {
          const uint32_t i = tid + q * kThreads;
          if (i < nmain) {
            const uint32_t b = i >> c.log2B;
            const uint32_t cw0 = st.cw[slot][b], w = st.cw[slot][b + 1] - cw0;
            const uint32_t pos = (cw0 - cwb) * c.B + (i & (c.B - 1)) * w, wi = pos >> 6, sh = pos & 63;
            uint64_t x = 0;
            if (w) {
              x = wd[wi] >> sh;
              if (sh + w > 64) x |= wd[wi + 1] << (64 - sh);
              x &= low_mask(w);
            }
            put(i, F == MS_FOR_BP ? st.ref[slot][b] + x : x);
          } else if (i < cnt) {
            put(i, __ldg(c.rem + (r0 + i - main_rows)));
          }
        }
        break;
      }
      case MS_DELTA_BP: {
        // thread t owns rows [8t, 8t+8): local prefix of the codes, CTA scan, minus the
        // prefix at the block head, plus the block base (D-6)
        const uint32_t i0 = tid * kVPT;
        const uint32_t nmain = r0 < main_rows ? (uint32_t)min((uint64_t)cnt, main_rows - r0) : 0u;
        const bool in_main = i0 < nmain;
        uint64_t loc[kVPT];
        uint64_t tsum = 0;
        uint32_t b = 0;
        if (in_main) {
          b = i0 >> c.log2B;
          const uint32_t cw0 = st.cw[slot][b], w = st.cw[slot][b + 1] - cw0;
          uint32_t pos = (cw0 - st.cw[slot][0]) * c.B + (i0 & (c.B - 1)) * w;
          if (w <= 28) {  // 8 codes sum below 2^31: 32-bit words, funnel shifts, 32-bit prefix
            const uint32_t* __restrict__ w32 = reinterpret_cast<const uint32_t*>(wd);
            const uint32_t mask = w ? 0xffffffffu >> (32 - w) : 0u;
            uint32_t s32 = 0;
#pragma unroll
            for (int q = 0; q < kVPT; ++q) {
              const uint32_t k = pos >> 5;
              s32 += __funnelshift_r(w32[k], w32[k + 1], pos & 31) & mask;
              loc[q] = s32;
              pos += w;
            }
            tsum = s32;
          } else {
            const uint64_t mask = low_mask(w);
#pragma unroll
            for (int q = 0; q < kVPT; ++q) {
              const uint32_t wi = pos >> 6, sh = pos & 63;
              uint64_t x = wd[wi] >> sh;
              if (sh + w > 64) x |= wd[wi + 1] << (64 - sh);
              tsum += x & mask;
              loc[q] = tsum;
              pos += w;
            }
          }
        }
        const uint64_t ex = cta_excl_scan(in_main ? tsum : 0, sm.scan, nullptr);
        sm.ex[tid] = ex;
        __syncthreads();
        if (in_main) {
          const uint32_t head = (b << c.log2B) / kVPT;
          const uint64_t base = st.ref[slot][b] + (ex - sm.ex[head]);
#pragma unroll
          for (int q = 0; q < kVPT; ++q) loc[q] += base;
          if (kMaxOnly) {
#pragma unroll
            for (int q = 0; q < kVPT; ++q) mx = loc[q] > mx ? loc[q] : mx;
          } else {
            store8_rotated(sm.vals + i0, loc);
          }
        } else {
          for (int q = 0; q < kVPT; ++q)
            if (i0 + q < cnt) put(i0 + q, __ldg(c.rem + (r0 + i0 + q - main_rows)));
        }
        break;
      }
    }
    if (!kMaxOnly) __syncthreads();
  }
};

// kMaxOnly: the auto-static-width pre-pass (OUT_MAX_ONLY), its own instantiation
template <bool kMaxOnly, int F>
__global__ void __launch_bounds__(kThreads, 3) engine_staged_kernel(StagedCol<F> src, OutView out, uint32_t* err) {
  __shared__ EngineSmem sm;
  extern __shared__ __align__(16) unsigned char st_raw[];
  StageSmem& st = *reinterpret_cast<StageSmem*>(st_raw);
  const uint64_t n = out.n;
  const uint64_t n_items = (n + kChunk - 1) / kChunk;
  const uint64_t G = gridDim.x;
  uint64_t t = blockIdx.x;
  if (t >= n_items) return;
  // prologue: headers(t) (needed for the range of payload(t)), then group -1
  src.issue_headers(t, st, 0);
  st_commit();
  st_wait_all();
  __syncthreads();
  src.issue_payload(t, n, st, 0, 0);
  if (t + G < n_items) src.issue_headers(t + G, st, 1);
  st_commit();
  uint64_t mx = 0;
  for (uint32_t k = 0; t < n_items; t += G, ++k) {
    st_wait_all();
    __syncthreads();
    const int buf = k & 1, slot = k % 3;
    if (t + G < n_items) {
      src.issue_payload(t + G, n, st, buf ^ 1, (k + 1) % 3);
      if (t + 2 * G < n_items) src.issue_headers(t + 2 * G, st, (k + 2) % 3);
    }
    st_commit();
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, n - r0);
    // an uncompressed source is encoded straight from its staging buffer (r0 is even:
    // no word offset)
    if (kMaxOnly) {  // auto static width: decode straight into a running max
      src.template decode<true>(t, cnt, st, buf, slot, sm, mx);
    } else {
      uint64_t* vals = sm.vals;
      if (F == MS_UNCOMPR) vals = st.words[buf];
      else src.template decode<false>(t, cnt, st, buf, slot, sm, mx);
      encode_tile(out, (uint32_t)t, r0, cnt, n, sm, err, vals);
    }
    __syncthreads();
  }
  if (kMaxOnly) {
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(out.max_out, (unsigned long long)mx);
  }
}

}  // namespace ms
