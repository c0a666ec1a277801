// kernels.cu — instrumentation, engine launches, scans, RLE, sums at positions / grouped.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "engine.cuh"
#include "stage.cuh"
#include "cstream.cuh"
#include "grid.cuh"
#include "launch.h"

namespace ms {

// ----------------------------------------------------------------- size read-backs
// The few words an op reads back (sizes, error bits) are written by one small kernel
// straight into pinned host memory, then the stream is synchronised: one launch
// instead of several pageable device-to-host copies in the gap after each op.
__global__ void readback_kernel(uint64_t* __restrict__ host, const uint64_t* __restrict__ dev, uint32_t count,
                                const uint32_t* __restrict__ w0, const uint32_t* __restrict__ w1,
                                const uint64_t* __restrict__ d2) {
  const uint32_t t = threadIdx.x;
  if (t < count) host[t] = dev[t];
  if (t == 32) host[32] = w0 ? *w0 : 0u;
  if (t == 33) host[33] = w1 ? *w1 : 0u;
  if (t == 34) host[34] = d2 ? *d2 : 0ull;
}

uint64_t* pinned_words() {
  thread_local uint64_t* p[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!p[dev] && cudaHostAlloc((void**)&p[dev], 64 * sizeof(uint64_t), cudaHostAllocPortable) != cudaSuccess)
    p[dev] = nullptr;
  return p[dev];
}

cudaError_t launch_readback(uint64_t* host, const uint64_t* dev, uint32_t count, const uint32_t* w0,
                            const uint32_t* w1, const uint64_t* d2, cudaStream_t s) {
  readback_kernel<<<1, 64, 0, s>>>(host, dev, count, w0, w1, d2);
  count_launch();
  return cudaGetLastError();
}
// ----------------------------------------------------------------- launch-config cache
namespace {
struct CfgKey {
  int dev;
  const void* k;
  int threads;
  size_t smem;
  bool operator==(const CfgKey& o) const { return dev == o.dev && k == o.k && threads == o.threads && smem == o.smem; }
};
std::mutex g_cfg_mu;
std::vector<std::pair<CfgKey, int>> g_occ;
std::vector<std::pair<CfgKey, int>> g_smem;  // threads unused: the largest opt-in set so far
}  // namespace

void set_smem_once(const void* kernel, size_t smem) {
  if (smem <= 48 * 1024) return;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(g_cfg_mu);
  for (auto& e : g_smem)
    if (e.first.dev == dev && e.first.k == kernel) {
      if (e.first.smem >= smem) return;
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      e.first.smem = smem;
      return;
    }
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  g_smem.push_back({CfgKey{dev, kernel, 0, smem}, 0});
}

int occupancy_cached(const void* kernel, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const CfgKey key{dev, kernel, threads, smem};
  {
    std::lock_guard<std::mutex> g(g_cfg_mu);
    for (auto& e : g_occ)
      if (e.first == key) return e.second;
  }
  set_smem_once(kernel, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  std::lock_guard<std::mutex> g(g_cfg_mu);
  g_occ.push_back({key, per_sm});
  return per_sm;
}


static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

// ---------------------------------------------------------- profiling
// Optional CUDA-event timing of every kernel launch, on the launching stream
// (bench.py reads the dominant kernel's average duration from here).
namespace {
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<int> g_prof_on{0};
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;
cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfScope::ProfScope(const char* name, cudaStream_t s) : name_(name), s_(s), on_(g_prof_on.load() != 0) {
  count_launch();
  if (!on_) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  a_ = (void*)prof_event();
  b_ = (void*)prof_event();
  cudaEventRecord((cudaEvent_t)a_, s_);
}
ProfScope::~ProfScope() {
  if (!on_) return;
  cudaEventRecord((cudaEvent_t)b_, s_);
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_recs.push_back({name_, (cudaEvent_t)a_, (cudaEvent_t)b_});
}

void profile_enable(int on) { g_prof_on.store(on); }

int profile_read(ms_kernel_time* out, int max) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  std::vector<ms_kernel_time> acc;
  for (auto& r : g_prof_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& k : acc)
      if (std::strcmp(k.name, r.name) == 0) {
        k.launches += 1;
        k.total_ms += ms;
        found = true;
      }
    if (!found) {
      ms_kernel_time k{};
      std::strncpy(k.name, r.name, sizeof(k.name) - 1);
      k.launches = 1;
      k.total_ms = ms;
      acc.push_back(k);
    }
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  int n = 0;
  for (auto& k : acc)
    if (n < max && out) out[n++] = k;
  return (int)acc.size();
}

int num_sms() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

static uint64_t n_items_hint(const OutView& o) {
  // an upper bound of the item count for grid sizing (n_dev may be device-resident)
  return (o.n + kChunk - 1) / kChunk;
}

// ----------------------------------------------------------------- engine
template <int F>
static cudaError_t launch_staged(const ColView& src, const OutView& out, uint32_t* err, bool max_only,
                                 cudaStream_t s) {
  static bool attr[64][2] = {};  // per device and instantiation
  int dev = 0;
  cudaGetDevice(&dev);
  auto k = max_only ? engine_staged_kernel<true, F> : engine_staged_kernel<false, F>;
  const int dyn = (int)sizeof(StageSmem);
  if (dev < 0 || dev >= 64 || !attr[dev][max_only]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr[dev][max_only] = true;
  }
  int per_sm = 0;
  per_sm = occupancy_cached((const void*)k, kThreads, dyn);
  if (per_sm < 1) per_sm = 1;
  const uint64_t items = n_items_hint(out);
  uint64_t g = (uint64_t)per_sm * num_sms();
  if (items < g) g = items;
  StagedCol<F> sc{src, src.nb << src.log2B};
  ProfScope prof_("engine_col", s);
  k<<<(int)(g ? g : 1), kThreads, dyn, s>>>(sc, out, err);
  return cudaGetLastError();
}

cudaError_t launch_engine_col(const ColView& src, const OutView& out, uint32_t* err, cudaStream_t s) {
  // compress of u64 values into a block format, slot mode: warp-per-tile streamed encoder (cstream.cuh)
  if (src.format == MS_UNCOMPR && out.slots && !out.n_dev && out.B >= 128 &&
      (out.format == MS_DYN_BP || out.format == MS_FOR_BP || out.format == MS_DELTA_BP) &&
      (reinterpret_cast<uintptr_t>(src.payload) & 15) == 0 && src.n == out.n) {
    auto k = compress_stream_kernel;
    const size_t smem = cs_smem_bytes();
    set_smem_once((const void*)k, smem);
    const uint64_t tiles = (src.n + kChunk - 1) / kChunk;
    const int grid = (int)(tiles < (uint64_t)num_sms() ? tiles : (uint64_t)num_sms());
    ProfScope prof_("compress_stream", s);
    k<<<grid, kCsThreads, smem, s>>>(src.payload, src.n, out, err);
    return cudaGetLastError();
  }
  // staged input (stage.cuh) whenever tiles go in a static order: every output but
  // a block format written with the look-back
  const bool ordered = !out.slots && (out.format == MS_DYN_BP || out.format == MS_FOR_BP || out.format == MS_DELTA_BP);
  if (stageable_format(src.format) && !out.n_dev && !ordered) {
    const bool max_only = out.format == OUT_MAX_ONLY;
    switch (src.format) {
      case MS_UNCOMPR: return launch_staged<MS_UNCOMPR>(src, out, err, max_only, s);
      case MS_STATIC_BP: return launch_staged<MS_STATIC_BP>(src, out, err, max_only, s);
      case MS_DYN_BP: return launch_staged<MS_DYN_BP>(src, out, err, max_only, s);
      case MS_FOR_BP: return launch_staged<MS_FOR_BP>(src, out, err, max_only, s);
      default: return launch_staged<MS_DELTA_BP>(src, out, err, max_only, s);
    }
  }
  auto k = engine_kernel<ColSource>;
  int grid = persistent_grid(k, kThreads, n_items_hint(out));
  ProfScope prof_("engine_col", s);
  k<<<grid, kThreads, 0, s>>>(ColSource{src}, out, err);
  return cudaGetLastError();
}

cudaError_t launch_engine_bitmask(const uint32_t* bits, const uint64_t* tile_off, const uint32_t* start_tile,
                                  uint64_t n_words, uint64_t row_offset, const OutView& out, uint32_t* err,
                                  cudaStream_t s) {
  auto k = engine_kernel<BitmaskSource>;
  int grid = persistent_grid(k, kThreads, n_items_hint(out));
  ProfScope prof_("engine_bitmask", s);
  k<<<grid, kThreads, 0, s>>>(BitmaskSource{bits, tile_off, start_tile, n_words, row_offset}, out, err);
  return cudaGetLastError();
}

cudaError_t launch_engine_gather(const ColView& pos, const ColView& data, uint64_t row_offset, const OutView& out,
                                 uint32_t* err, cudaStream_t s) {
  auto k = engine_kernel<GatherSource>;
  int grid = persistent_grid(k, kThreads, n_items_hint(out));
  ProfScope prof_("engine_gather", s);
  k<<<grid, kThreads, 0, s>>>(GatherSource{pos, data, row_offset}, out, err);
  return cudaGetLastError();
}

cudaError_t launch_tile_copy(const OutView& o, uint64_t n_tiles, uint64_t nb, const uint64_t* cwx, uint32_t* err,
                             cudaStream_t s) {
  if (!n_tiles || !nb) return cudaSuccess;
  uint64_t g = (n_tiles + 7) / 8;  // a warp per tile, 8 warps per CTA
  if (g > (uint64_t)num_sms() * 8) g = num_sms() * 8;
  ProfScope prof_("tile_copy", s);
  tile_copy_kernel<<<(int)g, 256, 0, s>>>(o, n_tiles, nb, cwx, err);
  return cudaGetLastError();
}

// ----------------------------------------------------------- generic scan
// Exclusive prefix over N values in one pass (decoupled look-back); epi(idx,
// exclusive, value) consumes each entry, epi_total(total) is called once.
// The epilogue's max key (select: 1 + largest position; widths: the largest) over
// the CTA, then one atomicMax per CTA: a per-warp atomic on one address serialises
// ~30K updates at L2 on a 2^32-row select.
template <class Epi>
__device__ __forceinline__ void cta_max_key(const Epi& epi, uint64_t key) {
  __shared__ uint64_t red[kThreads / 32];
  key = warp_max(key);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t m = 0;
    for (int k = 0; k < kThreads / 32; ++k) m = red[k] > m ? red[k] : m;
    if (m) epi.max_key(m);
  }
}

template <class In, class Epi>
__global__ void __launch_bounds__(kThreads) scan_kernel(In in, Epi epi, uint64_t N, uint64_t* status,
                                                        uint32_t* ticket) {
  __shared__ uint64_t scan_sm[16];
  __shared__ uint32_t s_item;
  __shared__ uint64_t s_E;
  const uint64_t n_items = (N + kChunk - 1) / kChunk;
  const int tid = threadIdx.x;
  uint64_t key = 0;  // the largest key this thread saw: one atomic per CTA at the end
  while (true) {
    if (tid == 0) s_item = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= n_items) break;
    const uint64_t base = (uint64_t)item * kChunk + tid * kVPT;
    uint64_t v[kVPT];
    uint64_t tsum = 0;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      v[q] = base + q < N ? in(base + q) : 0;
      tsum += v[q];
    }
    uint64_t tot;
    const uint64_t ex = cta_excl_scan(tsum, scan_sm, &tot);
    if (tid < 32) {
      const uint64_t E = lookback_warp(status, item, tot);
      if (tid == 0) s_E = E;
    }
    __syncthreads();
    uint64_t off = s_E + ex;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      if (base + q < N) {
        epi(base + q, off, v[q]);
        const uint64_t kq = epi.key(base + q);
        key = kq > key ? kq : key;
        if (base + q == N - 1) epi.total(off + v[q]);
      }
      off += v[q];
    }
    __syncthreads();
  }
  cta_max_key(epi, key);
}

// Reduce-then-scan (no look-back): tile sums, one CTA scans them in place, then
// every tile rescans its values from its tile offset. Three short launches instead
// of a single pass whose per-tile look-back stalls behind the ~1,000 tiles in flight.
template <class In>
__global__ void __launch_bounds__(kThreads) scan_reduce_kernel(In in, uint64_t N, uint64_t* tile_sum) {
  __shared__ uint64_t red[kThreads / 32];
  const uint64_t n_items = (N + kChunk - 1) / kChunk;
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    // the sum is order-free: lane-strided (coalesced) reads
    const uint64_t base = item * kChunk + threadIdx.x;
    uint64_t t = 0;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) t += base + q * kThreads < N ? in(base + q * kThreads) : 0;
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t a = 0;
      for (int k = 0; k < kThreads / 32; ++k) a += red[k];
      tile_sum[item] = a;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) scan_tiles_kernel(uint64_t* v, uint64_t T) {  // in place, exclusive
  __shared__ uint64_t wsum[32];
  __shared__ uint64_t carry;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (uint64_t b = 0; b < T; b += 1024) {
    const uint64_t i = b + tid;
    const uint64_t x = i < T ? v[i] : 0;
    const uint64_t inc = warp_incl_scan(x);
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const uint64_t ws = wsum[lane];
      wsum[lane] = warp_incl_scan(ws) - ws;
    }
    __syncthreads();
    const uint64_t c0 = carry;
    if (i < T) v[i] = c0 + wsum[wid] + inc - x;
    __syncthreads();
    if (tid == 1023) carry = c0 + wsum[wid] + inc;
    __syncthreads();
  }
}

// Warp-striped apply: warp w of the CTA owns the tile's elements [256w, 256w + 256),
// lane l the elements 256w + 32q + l (q < 8): every load and every epilogue store
// of the warp is one contiguous run (the thread-consecutive mapping touched 32
// lines per instruction). Offsets: a warp scan per row q with the rows' carry,
// then the warps' totals across the CTA.
template <class In, class Epi>
__global__ void __launch_bounds__(kThreads) scan_apply_kernel(In in, Epi epi, uint64_t N, const uint64_t* tile_off) {
  __shared__ uint64_t wsum[kThreads / 32 + 1];
  const uint64_t n_items = (N + kChunk - 1) / kChunk;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t key = 0;  // the largest key this thread saw: one atomic per CTA at the end
  // the thread's values one tile ahead: the tile's load round trip overlaps the
  // previous tile's scan and epilogue
  uint64_t nxt[kVPT];
  {
    const uint64_t b0 = (uint64_t)blockIdx.x * kChunk + wid * (32 * kVPT) + lane;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) nxt[q] = b0 + 32 * q < N ? in(b0 + 32 * q) : 0;
  }
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint64_t base = item * kChunk + wid * (32 * kVPT) + lane;
    uint64_t v[kVPT];
#pragma unroll
    for (int q = 0; q < kVPT; ++q) v[q] = nxt[q];
    const uint64_t toff = tile_off[item];
    {
      const uint64_t b1 = base + (uint64_t)gridDim.x * kChunk;
#pragma unroll
      for (int q = 0; q < kVPT; ++q) nxt[q] = b1 + 32 * q < N ? in(b1 + 32 * q) : 0;
    }
    uint64_t ex[kVPT];
    uint64_t carry = 0;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint64_t inc = warp_incl_scan(v[q]);
      ex[q] = carry + inc - v[q];
      carry += __shfl_sync(kFull, inc, 31);
    }
    if (lane == 0) wsum[wid] = carry;
    __syncthreads();
    if (wid == 0) {
      const uint64_t x = lane < kThreads / 32 ? wsum[lane] : 0;
      const uint64_t xi = warp_incl_scan(x);
      if (lane < kThreads / 32) wsum[lane] = xi - x;
    }
    __syncthreads();
    const uint64_t wb = toff + wsum[wid];
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint64_t idx = base + 32 * q;
      if (idx < N) {
        epi(idx, wb + ex[q], v[q]);
        const uint64_t kq = epi.key(idx);
        key = kq > key ? kq : key;
        if (idx == N - 1) epi.total(wb + ex[q] + v[q]);
      }
    }
    __syncthreads();  // wsum is rewritten by the next tile
  }
  cta_max_key(epi, key);
}

template <class In, class Epi>
static cudaError_t run_scan(In in, Epi epi, uint64_t N, uint64_t* status, uint32_t* ticket, cudaStream_t s) {
  if (N == 0) return cudaSuccess;
  const uint64_t T = (N + kChunk - 1) / kChunk;
  ProfScope prof_("scan", s);
  if (T > 1) {  // reduce-then-scan (status holds >= T + 1 entries); one tile: a single kernel
    auto kr = scan_reduce_kernel<In>;
    auto ka = scan_apply_kernel<In, Epi>;
    kr<<<persistent_grid(kr, kThreads, T), kThreads, 0, s>>>(in, N, status);
    scan_tiles_kernel<<<1, 1024, 0, s>>>(status, T);
    ka<<<persistent_grid(ka, kThreads, T), kThreads, 0, s>>>(in, epi, N, status);
    count_launch();  // three launches under one profiling scope
    count_launch();
    return cudaGetLastError();
  }
  auto k = scan_kernel<In, Epi>;
  k<<<persistent_grid(k, kThreads, T), kThreads, 0, s>>>(in, epi, N, status, ticket);
  return cudaGetLastError();
}

struct U32In {
  const uint32_t* p;
  __device__ uint64_t operator()(uint64_t i) const { return p[i]; }
};
struct SegIn {  // seg_info: count in the low 16 bits
  const uint32_t* p;
  __device__ uint64_t operator()(uint64_t i) const { return p[i] & 0xffffu; }
};
struct NoKey {
  __device__ uint64_t key(uint64_t) const { return 0; }
  __device__ void max_key(uint64_t) const {}
};

// row (within its 512-row segment) of the set bit of rank q (q < the segment's
// count): the segment's 16 mask words in four independent 16-byte loads, the word
// by a popcount walk in registers, the bit by halving. Out of line: rare (one call
// per output block) and register-heavy next to the scan's unrolled epilogue.
__device__ __forceinline__ uint32_t seg_row_of_rank(const uint32_t* __restrict__ seg, uint32_t q) {
  static_assert(kSegWords == 16, "segment = 16 mask words");
  uint32_t w[16];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(seg) + i);
    w[4 * i] = t.x; w[4 * i + 1] = t.y; w[4 * i + 2] = t.z; w[4 * i + 3] = t.w;
  }
  uint32_t word = 0, wdi = 0;
  bool found = false;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t pc = __popc(w[i]);
    if (!found) {
      if (q < pc) {
        found = true;
        word = w[i];
        wdi = i;
      } else {
        q -= pc;
      }
    }
  }
  return wdi * 32 + select_bit(word, q);
}

// select: segment offsets, 1 + max position, and the first position of every
// output item (G ranks) that starts inside a segment (select-in-segment on the mask)
struct SegEpi {
  uint64_t* seg_off;  // only seg_off[NS] (the total) is written: the encoders start from gstart
  uint64_t* gstart;
  const uint32_t* seg_info;
  const uint32_t* bits;
  unsigned long long* max_pos1;  // 1 + largest selected position (0 if none)
  uint64_t row_offset;
  uint64_t NS;
  uint32_t lgG;  // output item size G = 2^lgG
  __device__ void operator()(uint64_t idx, uint64_t off, uint64_t c) const {
    if (!c) return;
    const uint64_t G = 1ull << lgG;
    uint64_t k = (off + G - 1) >> lgG;
    if ((k << lgG) >= off + c) return;  // no output item starts in this segment
    for (; (k << lgG) < off + c; ++k)
      gstart[k] = row_offset + idx * kSegRows + seg_row_of_rank(bits + idx * kSegWords, (uint32_t)((k << lgG) - off));
  }
  __device__ uint64_t key(uint64_t idx) const {
    const uint32_t last = seg_info[idx] >> 16;
    return last ? row_offset + idx * kSegRows + last : 0;
  }
  __device__ void max_key(uint64_t k) const { atomicMax(max_pos1, (unsigned long long)k); }
  __device__ void total(uint64_t t) const { seg_off[NS] = t; }
};

// The segment scan's apply pass with the block starts deferred: a thread that
// finds output blocks starting in its segments queues (k, segment, rank) in
// shared memory; after the tile's offsets are known the whole CTA resolves the
// queue, one block start per thread. Inline (SegEpi::operator()) every thread of
// a warp would walk a segment's words whenever one lane has a start (~6 % of
// the segments at BJ.c5, i.e. almost every warp, eight times per tile).
constexpr int kSegQ = 2048;
__global__ void __launch_bounds__(kThreads, 5) seg_apply_kernel(SegIn in, SegEpi epi, uint64_t N,
                                                             const uint64_t* tile_off) {
  __shared__ uint64_t scan_sm[16];
  __shared__ uint64_t qk[kSegQ];
  __shared__ uint32_t qr[kSegQ];  // segment within the tile (11 bits) << 16 | rank in the segment
  __shared__ uint32_t q_n;
  const uint64_t n_items = (N + kChunk - 1) / kChunk;
  const int tid = threadIdx.x;
  const uint64_t G = 1ull << epi.lgG;
  if (tid == 0) q_n = 0;
  uint64_t key = 0;
  // the thread's 8 seg_info words (count | 1-based last row << 16), one tile ahead
  auto load8 = [&](uint64_t item, uint32_t (&r)[kVPT]) {
    const uint64_t base = item * kChunk + tid * kVPT;
    if (item < n_items && base + kVPT <= N) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(in.p + base));
      const uint4 b = __ldg(reinterpret_cast<const uint4*>(in.p + base) + 1);
      r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < kVPT; ++q) r[q] = item < n_items && base + q < N ? __ldg(in.p + base + q) : 0u;
    }
  };
  uint32_t nxt[kVPT];
  load8(blockIdx.x, nxt);
  for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const uint64_t t0 = item * kChunk, base = t0 + tid * kVPT;
    uint32_t info[kVPT];
    uint64_t tsum = 0;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      info[q] = nxt[q];
      tsum += info[q] & 0xffffu;
    }
    const uint64_t toff = tile_off[item];
    load8(item + gridDim.x, nxt);
    const uint64_t ex = cta_excl_scan(tsum, scan_sm, nullptr);  // ends with a barrier
    uint64_t off = toff + ex;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint64_t idx = base + q, c = info[q] & 0xffffu;
      if (idx < N && c) {
        for (uint64_t k = (off + G - 1) >> epi.lgG; (k << epi.lgG) < off + c; ++k) {
          const uint32_t rank = (uint32_t)((k << epi.lgG) - off);
          const uint32_t slot = atomicAdd(&q_n, 1u);
          if (slot < (uint32_t)kSegQ) {
            qk[slot] = k;
            qr[slot] = (uint32_t)(idx - t0) << 16 | rank;
          } else {  // queue full (block sizes < 512 at high selectivity): resolve here
            epi.gstart[k] = epi.row_offset + idx * kSegRows + seg_row_of_rank(epi.bits + idx * kSegWords, rank);
          }
        }
        key = epi.row_offset + idx * kSegRows + (info[q] >> 16);  // increasing in idx
      }
      if (idx == N - 1) epi.total(off + c);
      off += c;
    }
    __syncthreads();
    const uint32_t nq = q_n < (uint32_t)kSegQ ? q_n : (uint32_t)kSegQ;
    for (uint32_t t = tid; t < nq; t += kThreads) {
      const uint64_t idx = t0 + (qr[t] >> 16);
      epi.gstart[qk[t]] =
          epi.row_offset + idx * kSegRows + seg_row_of_rank(epi.bits + idx * kSegWords, qr[t] & 0xffffu);
    }
    __syncthreads();
    if (tid == 0) q_n = 0;
  }
  cta_max_key(epi, key);
}

cudaError_t launch_seg_scan(const uint32_t* seg_info, const uint32_t* bits, uint64_t NS, uint64_t row_offset,
                            uint32_t G, uint64_t* seg_off, uint64_t* gstart, unsigned long long* max_pos1,
                            uint64_t* status, uint32_t* ticket, cudaStream_t s) {
  uint32_t lg = 0;
  while ((1u << lg) < G) ++lg;  // G is a power of two (block sizes 128..2048, or 512)
  const SegIn in{seg_info};
  const SegEpi epi{seg_off, gstart, seg_info, bits, max_pos1, row_offset, NS, lg};
  const uint64_t T = (NS + kChunk - 1) / kChunk;
  if (T <= 1) return run_scan(in, epi, NS, status, ticket, s);  // one tile: the single-pass kernel
  ProfScope prof_("scan", s);
  auto kr = scan_reduce_kernel<SegIn>;
  kr<<<persistent_grid(kr, kThreads, T), kThreads, 0, s>>>(in, NS, status);
  scan_tiles_kernel<<<1, 1024, 0, s>>>(status, T);
  seg_apply_kernel<<<persistent_grid(seg_apply_kernel, kThreads, T), kThreads, 0, s>>>(in, epi, NS, status);
  count_launch();
  count_launch();
  return cudaGetLastError();
}

// exclusive prefix into off[0..T), total into off[T], the largest count into off[T + 1]
// (block widths: the output's max_width hint without a separate pass)
struct CountEpi {
  uint64_t* off;
  uint64_t T;
  const uint32_t* cnt;
  __device__ void operator()(uint64_t idx, uint64_t o, uint64_t c) const { off[idx] = o; }
  __device__ void total(uint64_t t) const { off[T] = t; }
  __device__ uint64_t key(uint64_t idx) const { return cnt[idx]; }
  __device__ void max_key(uint64_t k) const { atomicMax(reinterpret_cast<unsigned long long*>(off + T + 1), k); }
};

cudaError_t launch_count_scan(const uint32_t* counts, uint64_t T, uint64_t* off, uint64_t* status,
                              uint32_t* ticket, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(off + T + 1, 0, 8, s);
  if (e != cudaSuccess) return e;
  return run_scan(U32In{counts}, CountEpi{off, T, counts}, T, status, ticket, s);
}

// RLE: run starts = exclusive prefix of the lengths; lengths must be >= 1 and
// sum to n (a corrupt body otherwise)
struct LenIn {
  const uint64_t* payload;
  __device__ uint64_t operator()(uint64_t i) const { return payload[2 * i + 1]; }
};
struct StartsEpi : NoKey {
  uint64_t* starts;
  uint64_t R, n;
  uint32_t* err;
  __device__ void operator()(uint64_t idx, uint64_t off, uint64_t len) const {
    starts[idx] = off;
    // every length is >= 1 and every run ends inside the column: this also catches
    // totals that wrap mod 2^64 (non-monotone starts)
    if (len == 0 || len > n || off > n - len) atomicOr(err, err_bit(MS_E_CORRUPT));
  }
  __device__ void total(uint64_t t) const {
    starts[R] = t;
    if (t != n) atomicOr(err, err_bit(MS_E_CORRUPT));
  }
};

cudaError_t launch_rle_starts(const uint64_t* payload, uint64_t R, uint64_t n, uint64_t* starts, uint64_t* status,
                              uint32_t* ticket, uint32_t* err, cudaStream_t s) {
  return run_scan(LenIn{payload}, StartsEpi{{}, starts, R, n, err}, R, status, ticket, s);
}

__global__ void chunk_run_kernel(const uint64_t* starts, uint64_t R, uint64_t n, uint32_t* chunk_run) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < R; k += stride) {
    const uint64_t s = starts[k];
    const uint64_t e = min(starts[k + 1], n);
    for (uint64_t c = (s + kChunk - 1) / kChunk; c * kChunk < e; ++c) chunk_run[c] = (uint32_t)k;
  }
}

cudaError_t launch_chunk_run(const uint64_t* starts, uint64_t R, uint64_t n, uint32_t* chunk_run, cudaStream_t s) {
  if (R == 0) return cudaSuccess;
  ProfScope prof_("chunk_run", s);
  chunk_run_kernel<<<num_sms() * 8, 256, 0, s>>>(starts, R, n, chunk_run);
  return cudaGetLastError();
}

// RLE decompression (P:163 runs; S:115-131 decode): a warp takes 32 consecutive
// runs, broadcasts each run's (value, start, end) by shuffle and writes its rows
// with coalesced stores (lanes on consecutive rows): ~ceil(len/32) store
// instructions per run, no per-row search or scan.
__global__ void __launch_bounds__(256) rle_expand_kernel(const uint64_t* __restrict__ payload,
                                                         const uint64_t* __restrict__ starts, uint64_t R, uint64_t n,
                                                         uint64_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t k0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; k0 < R;
       k0 += nwarps * 32) {
    const uint64_t k = k0 + lane;
    uint64_t v = 0, s = 0, e = 0;
    if (k < R) {
      v = __ldg(payload + 2 * k);
      s = __ldg(starts + k);
      e = min(__ldg(starts + k + 1), n);
    }
    const uint32_t nr = (uint32_t)min((uint64_t)32, R - k0);
    for (uint32_t r = 0; r < nr; ++r) {
      const uint64_t vr = __shfl_sync(kFull, v, r), sr = __shfl_sync(kFull, s, r), er = __shfl_sync(kFull, e, r);
      for (uint64_t i = sr + lane; i < er; i += 32) out[i] = vr;
    }
  }
}

cudaError_t launch_rle_expand(const uint64_t* payload, const uint64_t* starts, uint64_t R, uint64_t n, uint64_t* out,
                              cudaStream_t s) {
  if (R == 0) return cudaSuccess;
  uint64_t g = (R + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms() * 8;
  if (g > cap) g = cap;
  ProfScope prof_("rle_expand", s);
  rle_expand_kernel<<<(int)g, 256, 0, s>>>(payload, starts, R, n, out);
  return cudaGetLastError();
}

// ------------------------------------------------------ RLE compression
__global__ void __launch_bounds__(kThreads) rle_count_kernel(const uint64_t* __restrict__ v, uint64_t n,
                                                             uint32_t* counts) {
  __shared__ uint32_t wsum[kThreads / 32];
  const uint64_t T = (n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < T; t += gridDim.x) {
    // rows t*kChunk + tid + q*kThreads (coalesced), all 16 loads in flight together
    uint64_t a[kVPT], b[kVPT];
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint64_t r = t * kChunk + threadIdx.x + q * kThreads;
      a[q] = r < n ? __ldg(v + r) : 0ull;
      b[q] = (r >= 1 && r < n) ? __ldg(v + r - 1) : ~a[q];
    }
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint64_t r = t * kChunk + threadIdx.x + q * kThreads;
      if (r < n && a[q] != b[q]) ++c;
    }
    c = (uint32_t)warp_sum(c);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int k = 0; k < kThreads / 32; ++k) s += wsum[k];
      counts[t] = s;
    }
    __syncthreads();
  }
}

cudaError_t launch_rle_count(const uint64_t* v, uint64_t n, uint32_t* counts, cudaStream_t s) {
  const uint64_t T = (n + kChunk - 1) / kChunk;
  if (!T) return cudaSuccess;
  ProfScope prof_("rle_count", s);
  rle_count_kernel<<<persistent_grid(rle_count_kernel, kThreads, T), kThreads, 0, s>>>(v, n, counts);
  return cudaGetLastError();
}

// rows lane-strided (t*kChunk + tid + q*kThreads: coalesced, as rle_count); a run
// start's rank inside the tile = the starts of earlier (step, warp) groups (a scan
// over the 8 x 8 ballot counts) + the earlier lanes of its own ballot
__global__ void __launch_bounds__(kThreads) rle_write_kernel(const uint64_t* __restrict__ v, uint64_t n,
                                                             const uint64_t* chunk_off, uint64_t* payload,
                                                             uint64_t* starts) {
  constexpr int kWarps = kThreads / 32;
  static_assert(kVPT * kWarps == 64, "two ballot counts per lane of one warp");
  __shared__ uint32_t grp[kVPT * kWarps];  // counts, then exclusive offsets, of (step q, warp w) at q*kWarps+w
  const uint64_t T = (n + kChunk - 1) / kChunk;
  const int tid = threadIdx.x;
  const uint32_t lane = tid & 31, wid = tid >> 5;
  for (uint64_t t = blockIdx.x; t < T; t += gridDim.x) {
    uint64_t a[kVPT], b[kVPT];
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint64_t r = t * kChunk + tid + q * kThreads;
      a[q] = r < n ? __ldg(v + r) : 0ull;
      b[q] = (r >= 1 && r < n) ? __ldg(v + r - 1) : ~a[q];
    }
    const uint64_t off = __ldg(chunk_off + t);  // with the rows: not a second dependent load after the scan
    uint32_t bal[kVPT];
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint64_t r = t * kChunk + tid + q * kThreads;
      bal[q] = __ballot_sync(kFull, r < n && a[q] != b[q]);
      if (lane == 0) grp[q * kWarps + wid] = __popc(bal[q]);
    }
    __syncthreads();
    if (tid < 32) {
      const uint32_t c0 = grp[2 * tid], c1 = grp[2 * tid + 1];
      uint32_t x = c0 + c1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, o);
        if ((int)lane >= o) x += y;
      }
      const uint32_t ex = x - c0 - c1;
      grp[2 * tid] = ex;
      grp[2 * tid + 1] = ex + c0;
    }
    __syncthreads();
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll
    for (int q = 0; q < kVPT; ++q)
      if ((bal[q] >> lane) & 1u) {
        const uint64_t idx = off + grp[q * kWarps + wid] + __popc(bal[q] & below);
        payload[2 * idx] = a[q];
        starts[idx] = t * kChunk + tid + q * kThreads;
      }
    __syncthreads();  // grp is rewritten by the next tile
  }
}

cudaError_t launch_rle_write(const uint64_t* v, uint64_t n, const uint64_t* chunk_off, uint64_t* payload,
                             uint64_t* starts, cudaStream_t s) {
  const uint64_t T = (n + kChunk - 1) / kChunk;
  if (!T) return cudaSuccess;
  ProfScope prof_("rle_write", s);
  rle_write_kernel<<<persistent_grid(rle_write_kernel, kThreads, T), kThreads, 0, s>>>(v, n, chunk_off, payload,
                                                                                        starts);
  return cudaGetLastError();
}

__global__ void rle_len_kernel(const uint64_t* starts, uint64_t R, uint64_t n, uint64_t* payload) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < R; k += stride)
    payload[2 * k + 1] = (k + 1 < R ? starts[k + 1] : n) - starts[k];
}

cudaError_t launch_rle_len(const uint64_t* starts, uint64_t R, uint64_t n, uint64_t* payload, cudaStream_t s) {
  if (!R) return cudaSuccess;
  ProfScope prof_("rle_len", s);
  rle_len_kernel<<<num_sms() * 8, 256, 0, s>>>(starts, R, n, payload);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads) sum_at_kernel(ColView data, ColView pos, uint64_t row_offset,
                                                          unsigned long long* out, uint32_t* err) {
  __shared__ EngineSmem sm;
  __shared__ EngineSmem dsm;  // decoded data tile (sequential formats)
  __shared__ uint64_t wsum[kThreads / 32];
  __shared__ unsigned long long s_lo, s_hi;
  const uint64_t T = (pos.n + kChunk - 1) / kChunk;
  // DELTA_BP / RLE data have no O(1) random access (D-12): when a chunk's positions
  // span few data tiles, decode those tiles once (load_rows) and pick the values
  // from shared memory instead of one O(B) / O(log R) read_row per position
  const bool seq = data.format == MS_DELTA_BP || data.format == MS_RLE;
  uint64_t acc = 0;
  for (uint64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, pos.n - r0);
    load_rows(pos, r0, cnt, sm);
    bool tiled = false;
    if (seq) {
      if (threadIdx.x == 0) {
        s_lo = ~0ull;
        s_hi = 0;
      }
      __syncthreads();
      unsigned long long lo = ~0ull, hi = 0;
      for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
        const uint64_t p = sm.vals[i];
        lo = p < lo ? p : lo;
        hi = p > hi ? p : hi;
      }
      atomicMin(&s_lo, lo);
      atomicMax(&s_hi, hi);
      __syncthreads();
      const uint64_t plo = s_lo, phi = s_hi;
      tiled = plo >= row_offset && phi - row_offset < data.n && (phi - plo) < 4ull * kChunk;
      if (tiled) {
        const uint64_t t_lo = (plo - row_offset) / kChunk, t_hi = (phi - row_offset) / kChunk;
        for (uint64_t dt = t_lo; dt <= t_hi; ++dt) {
          const uint64_t d0 = dt * kChunk;
          const uint32_t dcnt = (uint32_t)min((uint64_t)kChunk, data.n - d0);
          load_rows(data, d0, dcnt, dsm);  // ends with a barrier
          for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
            const uint64_t r = sm.vals[i] - row_offset;
            if (r >= d0 && r < d0 + dcnt) acc += dsm.vals[r - d0];
          }
          __syncthreads();
        }
      }
    }
    if (!tiled) {
      for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
        const uint64_t p = sm.vals[i];
        if (p < row_offset || p - row_offset >= data.n) atomicOr(err, err_bit(MS_E_RANGE));
        else acc += read_row(data, p - row_offset);
      }
    }
    __syncthreads();
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int k = 0; k < kThreads / 32; ++k) t += wsum[k];
    if (t) atomicAdd(out, (unsigned long long)t);
  }
}

cudaError_t launch_sum_at(const ColView& data, const ColView& pos, uint64_t row_offset, unsigned long long* out,
                          uint32_t* err, cudaStream_t s) {
  const uint64_t T = (pos.n + kChunk - 1) / kChunk;
  if (!T) return cudaSuccess;
  ProfScope prof_("sum_at", s);
  sum_at_kernel<<<persistent_grid(sum_at_kernel, kThreads, T), kThreads, 0, s>>>(data, pos, row_offset, out, err);
  return cudaGetLastError();
}

// grouped sum with an uncompressed result: per-CTA shared-memory
// histogram when the groups fit, else global atomics
constexpr uint32_t kSmemGroups = 1024;
__global__ void __launch_bounds__(kThreads) sum_grouped_kernel(ColView gid, ColView vals, uint64_t n_groups,
                                                               unsigned long long* sums, uint32_t* err) {
  __shared__ EngineSmem sm;
  __shared__ uint64_t g[kChunk];
  __shared__ unsigned long long hist[kSmemGroups];
  const bool use_smem = n_groups <= kSmemGroups;
  if (use_smem)
    for (uint32_t k = threadIdx.x; k < n_groups; k += kThreads) hist[k] = 0;
  const uint64_t T = (gid.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, gid.n - r0);
    load_rows(gid, r0, cnt, sm);
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) g[i] = sm.vals[i];
    __syncthreads();
    load_rows(vals, r0, cnt, sm);
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      const uint64_t k = g[i];
      if (k >= n_groups) {
        atomicOr(err, err_bit(MS_E_RANGE));
        continue;
      }
      if (use_smem) atomicAdd(&hist[k], (unsigned long long)sm.vals[i]);
      else atomicAdd(&sums[k], (unsigned long long)sm.vals[i]);
    }
    __syncthreads();
  }
  if (use_smem) {
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < n_groups; k += kThreads)
      if (hist[k]) atomicAdd(&sums[k], hist[k]);
  }
}

cudaError_t launch_sum_grouped(const ColView& gid, const ColView& vals, uint64_t n_groups,
                               unsigned long long* sums, uint32_t* err, cudaStream_t s) {
  const uint64_t T = (gid.n + kChunk - 1) / kChunk;
  if (!T) return cudaSuccess;
  ProfScope prof_("sum_grouped", s);
  sum_grouped_kernel<<<persistent_grid(sum_grouped_kernel, kThreads, T), kThreads, 0, s>>>(gid, vals, n_groups,
                                                                                          sums, err);
  return cudaGetLastError();
}

}  // namespace ms
