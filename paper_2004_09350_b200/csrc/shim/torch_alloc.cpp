// torch_alloc.cpp — native allocation callbacks for ms_ctx that route libms'
// device allocations (outputs and scratch) into PyTorch's CUDA caching
// allocator without a Python round trip. Plumbing only: libms itself never sees
// a torch type (include/ms.h takes plain function pointers); the Python binding
// loads this shim and passes ms_torch_alloc / ms_torch_free as ms_ctx.alloc/free.
#include <c10/cuda/CUDACachingAllocator.h>
#include <cuda_runtime.h>

extern "C" {
__attribute__((visibility("default"))) void* ms_torch_alloc(void* /*ctx*/, size_t bytes, void* stream) {
  try {
    return c10::cuda::CUDACachingAllocator::raw_alloc_with_stream(bytes, reinterpret_cast<cudaStream_t>(stream));
  } catch (...) {
    return nullptr;  // out of memory -> MS_E_NOMEM
  }
}
__attribute__((visibility("default"))) void ms_torch_free(void* /*ctx*/, void* ptr, void* /*stream*/) {
  if (ptr) c10::cuda::CUDACachingAllocator::raw_delete(ptr);
}
}
