// INT32 issue-rate microbenchmark for the ALU roofline ("the INT32
// issue rate of sm_100 and the clock during memory-bound kernels are not measured
// yet. Microbenchmark them first"). Each thread runs 8 independent chains of the
// instructions the unpack / predicate / pack cores are made of (SHF funnel shift,
// LOP3, IADD3, ISETP+SEL), fully unrolled; lanes-ops per clock per SM = executed
// ops / (SM cycles * SMs). The SM clock is read in-kernel (clock64 vs %globaltimer).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int32_rate int32_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) kern(uint32_t seed, int iters, uint32_t* sink, unsigned long long* clk) {
  uint32_t a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed * (threadIdx.x + 17 * k + 1);
  const uint32_t b = seed ^ 0x9e3779b9u;
  uint64_t c0 = clock64(), t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if constexpr (OP == 0) a[k] = __funnelshift_r(a[k], b, r + 1);          // SHF.R.W
        else if constexpr (OP == 1) a[k] = (a[k] & b) ^ (a[k] >> 3);            // LOP3 (+SHF)
        else if constexpr (OP == 2) a[k] = a[k] + a[(k + 1) & 7] + (uint32_t)r;  // IADD3
        else a[k] = (a[k] - b) <= (uint32_t)(r * 977) ? a[k] + 1 : a[k] ^ b;    // ISETP + SEL-ish
      }
    }
  }
  uint64_t c1 = clock64(), t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) x ^= a[k];
  if (x == 0x12345678) sink[0] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t* sink; unsigned long long* clk;
  cudaMalloc(&sink, 4); cudaMalloc(&clk, 16);
  const char* names[4] = {"SHF.R.W funnel shift", "LOP3 (+SHF)", "IADD3", "compare + select"};
  const int iters = 4000, blocks = sms * 8;
  printf("{\"sms\": %d, \"results\": [", sms);
  for (int op = 0; op < 4; ++op) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto launch = [&]() {
      if (op == 0) kern<0><<<blocks, 256>>>(7, iters, sink, clk);
      else if (op == 1) kern<1><<<blocks, 256>>>(7, iters, sink, clk);
      else if (op == 2) kern<2><<<blocks, 256>>>(7, iters, sink, clk);
      else kern<3><<<blocks, 256>>>(7, iters, sink, clk);
    };
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2]; cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
    const double mhz = (double)h[0] / ((double)h[1] * 1e-3);
    const double lane_ops = (double)blocks * 256 * iters * 16 * 8;  // one source op per chain step
    const double per_clk_sm = lane_ops / (ms * 1e-3 * mhz * 1e6) / sms;
    printf("%s{\"op\": \"%s\", \"ms\": %.3f, \"sm_mhz\": %.0f, \"lane_ops_per_clk_per_sm\": %.1f, "
           "\"tera_lane_ops_per_s\": %.2f}", op ? ", " : "", names[op], ms, mhz, per_clk_sm, lane_ops / (ms * 1e-3) / 1e12);
  }
  printf("]}\n");
  return 0;
}
