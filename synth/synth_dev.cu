// synth_dev.cu — device side of the synthetic generators (see synth.h).
// Input generation only: this file is compiled into its own library
// (synth/libsynth_dev.so) and shares nothing with the product library.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>
#include "synth.h"

namespace {

__global__ void fill_kernel(synth_recipe p, uint64_t start, uint64_t n, uint64_t *out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = synth_value(&p, start + i);
}

__global__ void runs_inc_kernel(uint64_t seed, uint64_t start, uint64_t n, uint64_t *out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = synth_run_inc(seed, start + i);
}

// sum of increments over rows [0, start): added to out[0] before the scan
__global__ void runs_prefix_kernel(uint64_t seed, uint64_t start, uint64_t *out0) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t acc = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < start; i += stride)
    acc += synth_run_inc(seed, i);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd((unsigned long long *)out0, (unsigned long long)acc);
}

__global__ void add_scalar_kernel(uint64_t *x, uint64_t v) { *x += v; }

}  // namespace

extern "C" int synth_fill_device(const synth_recipe *p, uint64_t start, uint64_t n, uint64_t *out,
                                 void *stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n == 0) return 0;
  int grid = 148 * 16, block = 256;
  if (p->kind != SYN_RUNS) {
    fill_kernel<<<grid, block, 0, stream>>>(*p, start, n, out);
    return (int)cudaGetLastError();
  }
  runs_inc_kernel<<<grid, block, 0, stream>>>(p->seed, start, n, out);
  add_scalar_kernel<<<1, 1, 0, stream>>>(out, p->add);
  if (start) runs_prefix_kernel<<<grid, block, 0, stream>>>(p->seed, start, out);
  // inclusive scan in chunks of 2^30 rows, carrying the running total
  const uint64_t chunk = 1ull << 30;
  size_t tmp_bytes = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, out, out, (int)(n < chunk ? n : chunk), stream);
  void *tmp = nullptr;
  cudaError_t e = cudaMallocAsync(&tmp, tmp_bytes, stream);
  if (e != cudaSuccess) return (int)e;
  for (uint64_t off = 0; off < n; off += chunk) {
    uint64_t len = n - off < chunk ? n - off : chunk;
    if (off) {
      // carry: out[off] += out[off-1]
      cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, out + off - 1, out + off - 1, 2, stream);
    }
    cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, out + off, out + off, (int)len, stream);
  }
  cudaFreeAsync(tmp, stream);
  return (int)cudaGetLastError();
}
