// Microbenchmark: cycles per 512-rank block extraction variants (one warp per block,
// 8 warps per SM, 148 CTAs), mask in dynamic shared memory as in select_pos.cu.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o extract extract.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sidx16(uint32_t q) { return q + (q >> 4); }
struct Sm { uint32_t M[8192]; uint64_t st[8][544]; uint32_t st32[32][544]; uint16_t pre[1][8192 + 64]; };
__device__ __forceinline__ uint32_t nth_bit(uint32_t x, uint32_t n) {  // branch-free position of set bit n
  uint32_t pos = 0, c;
  c = __popc(x & 0xffffu); if (n >= c) { n -= c; pos += 16; x >>= 16; }
  c = __popc(x & 0xffu); if (n >= c) { n -= c; pos += 8; x >>= 8; }
  c = __popc(x & 0xfu); if (n >= c) { n -= c; pos += 4; x >>= 4; }
  c = __popc(x & 0x3u); if (n >= c) { n -= c; pos += 2; x >>= 2; }
  c = x & 1u; if (n >= c) pos += 1;
  return pos;
}

template <int V>
__global__ void kern(uint32_t ds, int reps, unsigned long long* out, uint32_t* sink) {
  extern __shared__ __align__(128) unsigned char dyn[];
  Sm& S = *reinterpret_cast<Sm*>(dyn);
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < 8192; i += blockDim.x) {
    uint32_t x = 0;
    for (int b = 0; b < 32; ++b) {
      uint32_t h = (i * 32 + b) * 2654435761u;
      h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
      if ((h & ((1u << ds) - 1)) == 0) x |= 1u << b;
    }
    S.M[i] = x;
  }
  __syncthreads();
  const uint32_t* M = S.M;
  unsigned long long tot = 0;
  uint32_t chk = 0;
  for (int rep = 0; rep < reps; ++rep) {
    const uint32_t span = 512u << ds >> 5;  // words holding ~512 matches
    const uint32_t wa = ((rep * 97 + wid * 512) * 8) & (8191 & ~(span - 1));
    const uint32_t r0 = 0, r1 = 512;
    const uint32_t K = (span + 31) >> 5;
    const uint32_t w0 = wa + lane * K, w1 = w0 + K;
    __syncwarp();
    const uint64_t c0 = clock64();
    uint32_t c = 0;
    for (uint32_t w = w0; w < w1; ++w) c += __popc(M[w]);
    uint32_t inc = c;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (uint32_t)o) inc += y;
    }
    uint32_t r = inc - c;
    if constexpr (V == 0) {  // current: u64 stores, while loop
      uint64_t* st = S.st[wid & 7];
      for (uint32_t w = w0; w < w1 && r < r1; ++w) {
        uint32_t x = M[w];
        while (x && r < r1) {
          const uint32_t b = __ffs(x) - 1;
          x &= x - 1;
          st[sidx16(r - r0)] = 1000ull + w * 32 + b;
          ++r;
        }
      }
    } else if constexpr (V == 1) {  // counted loop, u32 stores
      uint32_t* st = S.st32[wid];
      for (uint32_t w = w0; w < w1; ++w) {
        uint32_t x = M[w];
        const uint32_t pc = __popc(x);
        const uint32_t n = r < r1 ? min(pc, r1 - r) : 0u;
        const uint32_t base = w * 32;
        uint32_t q = r - r0;
        for (uint32_t k = 0; k < n; ++k) {
          st[sidx16(q + k)] = base + __ffs(x) - 1;
          x &= x - 1;
        }
        r += pc;
      }
    } else if constexpr (V == 2) {  // all words preloaded (K <= 8 unrolled), counted loops
      uint32_t* st = S.st32[wid];
      uint32_t xs[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) xs[i] = (uint32_t)i < K ? M[w0 + i] : 0u;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        uint32_t x = xs[i];
        const uint32_t pc = __popc(x);
        const uint32_t n = r < r1 ? min(pc, r1 - r) : 0u;
        const uint32_t base = (w0 + i) * 32;
        const uint32_t q = r - r0;
        for (uint32_t k = 0; k < n; ++k) {
          st[sidx16(q + k)] = base + __ffs(x) - 1;
          x &= x - 1;
        }
        r += pc;
      }
    } else if constexpr (V >= 8) {
      // per-word block-local prefix (u16) into pre[wid][w - wa], then rank-parallel
      // branch-free binary search: lane j takes ranks 16j..16j+15 (V8) or j+32i (V9)
      uint16_t* P = S.pre[0];
      {
        uint32_t run = r;  // rank of the lane's first match (block-local: wa has rank 0)
        for (uint32_t w = w0; w < w1; ++w) { P[w - wa] = (uint16_t)run; run += __popc(M[w]); }
      }
      const uint32_t nw = span;
      __syncwarp();
      uint32_t* st = S.st32[wid];
      uint32_t lg = 31 - __clz(nw);  // nw is a power of two here
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t rk = V == 8 ? 16 * lane + i : lane + 32 * i;
        uint32_t m = 0;
        for (uint32_t step = nw >> 1; step; step >>= 1)
          if (P[m + step] <= rk) m += step;
        const uint32_t x = M[wa + m];
        const uint32_t b = V == 10 ? __fns(x, 0, (int)(rk - P[m]) + 1) : nth_bit(x, rk - P[m]);
        st[sidx16(rk)] = (wa + m) * 32 + b;
      }
      (void)lg;
    } else if constexpr (V >= 4) {  // counted loop, u32 stores, bit index variants
      uint32_t* st = S.st32[wid];
      for (uint32_t w = w0; w < w1; ++w) {
        uint32_t x = M[w];
        const uint32_t pc = __popc(x);
        const uint32_t n = r < r1 ? min(pc, r1 - r) : 0u;
        const uint32_t base = w * 32;
        uint32_t q = r - r0;
        for (uint32_t k = 0; k < n; ++k) {
          uint32_t b;
          if constexpr (V == 4) b = 31 - __clz(x & (0u - x));
          else if constexpr (V == 5) b = __popc((x & (0u - x)) - 1);
          else if constexpr (V == 6) b = k;  // no index computation (loop cost only)
          else b = S.M[((x & (0u - x)) * 0x077CB531u) >> 27] & 31;  // table lookup stand-in
          st[sidx16(q + k)] = base + b;
          x &= x - 1;
        }
        r += pc;
      }
    } else {  // V3: 64-bit pairs of words
      uint32_t* st = S.st32[wid];
      for (uint32_t w = w0; w < w1; w += 2) {
        uint64_t x = (uint64_t)M[w] | ((w + 1 < w1) ? (uint64_t)M[w + 1] << 32 : 0ull);
        const uint32_t pc = __popcll(x);
        const uint32_t n = r < r1 ? min(pc, r1 - r) : 0u;
        const uint32_t base = w * 32;
        const uint32_t q = r - r0;
        for (uint32_t k = 0; k < n; ++k) {
          st[sidx16(q + k)] = base + __ffsll(x) - 1;
          x &= x - 1;
        }
        r += pc;
      }
    }
    __syncwarp();
    tot += clock64() - c0;
    chk += V == 0 ? (uint32_t)S.st[wid & 7][lane] : S.st32[wid][lane];
    if (V >= 8 && rep == 0 && blockIdx.x == 0 && wid == 0 && lane < 3) printf("V%d ds%u lane%u: %u %u %u\n", V, ds, lane, S.st32[0][sidx16(lane)], S.st32[0][sidx16(lane+100)], S.st32[0][sidx16(511)]);
  }
  if (lane == 0 && wid < 8) out[blockIdx.x * 8 + wid] = tot / reps;
  if (chk == 0xdeadbeef) sink[0] = chk;
}

template <int V>
void run(uint32_t ds, unsigned long long* out, uint32_t* sink, int warps = 8) {
  cudaFuncSetAttribute(kern<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Sm));
  kern<V><<<148, 32 * warps, sizeof(Sm)>>>(ds, 200, out, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148 * 8];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148 * 8; ++i) m += h[i];
  printf("V%d density 1/%u warps %d: %.0f cycles per 512-rank block per warp -> %.0f cycles per block per SM (%s)\n", V, 1u << ds, warps, m / (148 * 8), m / (148 * 8) / warps, cudaGetErrorString(e));
}

int main() {
  unsigned long long* out; uint32_t* sink;
  cudaMalloc(&out, 148 * 8 * 8); cudaMalloc(&sink, 4);
  cudaMalloc(&out, 148 * 32 * 8);
  for (uint32_t ds : {1u, 4u}) for (int w : {8, 16, 32}) run<1>(ds, out, sink, w);
  return 0;
}
