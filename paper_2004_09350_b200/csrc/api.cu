// api.cu — the C ABI of libms (include/ms.h): the paper's "column layer"
// (P:469, 477-479): validates descriptors, splits columns into main part and
// remainder (by descriptor), sizes and allocates outputs, launches the
// kernels and performs the op's single read-back synchronisation.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "engine.cuh"
#include "launch.h"

using namespace ms;

__device__ uint32_t g_ms_sticky_err;  // errors of the non-synchronising ops

namespace {

constexpr uint64_t kAlign = 256;
constexpr uint64_t kStreamAvgWindow = 22 * 1024;  // project: stream when the mean window (bytes) is below
inline uint64_t align_up(uint64_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }
inline bool is_block(int32_t f) { return f == MS_DYN_BP || f == MS_FOR_BP || f == MS_DELTA_BP; }
inline bool valid_B(uint32_t B) { return B == 128 || B == 256 || B == 512 || B == 1024 || B == 2048; }
inline uint32_t log2u(uint32_t x) { return 31u - (uint32_t)__builtin_clz(x); }
inline uint32_t ebw_host(uint64_t x) { return x ? 64u - (uint32_t)__builtin_clzll(x) : 0u; }
inline uint64_t words_for(uint64_t n, uint32_t w) { return (n * (uint64_t)w + 63) / 64; }

struct Ctx {
  const ms_ctx* c;
  cudaStream_t s;
  explicit Ctx(const ms_ctx* cc) : c(cc), s(cc ? (cudaStream_t)cc->stream : nullptr) {}
  void* alloc(uint64_t bytes) const {
    if (bytes == 0) bytes = kAlign;
    if (c && c->alloc) return c->alloc(c->alloc_ctx, (size_t)bytes, c->stream);
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  }
  void free(void* p) const {
    if (!p) return;
    if (c && c->free) c->free(c->alloc_ctx, p, c->stream);
    else cudaFreeAsync(p, s);
  }
};

// One scratch allocation per op, carved into 256-byte aligned regions.
// Per-op scratch from the stream's caching allocator. Regions asked zeroed are laid
// out together after the others, so commit() clears all of them with ONE memset
// (one launch per op instead of one per region); their offsets carry kZeroTag
// until at() maps them (offset arithmetic on a returned offset stays valid).
struct Scratch {
  static constexpr uint64_t kZeroTag = 1ull << 62;
  const Ctx& ctx;
  uint64_t size = 0, zsize = 0, zstart = 0;
  char* base = nullptr;
  explicit Scratch(const Ctx& c) : ctx(c) {}
  ~Scratch() { ctx.free(base); }
  uint64_t add(uint64_t bytes, bool zero) {
    const uint64_t b = bytes ? bytes : 8;
    if (zero) {
      const uint64_t off = zsize;
      zsize = align_up(zsize + b);
      return kZeroTag | off;
    }
    const uint64_t off = size;
    size = align_up(size + b);
    return off;
  }
  bool commit() {
    zstart = align_up(size);
    const uint64_t total = zstart + zsize;
    base = (char*)ctx.alloc(total ? total : kAlign);
    if (!base) return false;
    return !zsize || cudaMemsetAsync(base + zstart, 0, zsize, ctx.s) == cudaSuccess;
  }
  template <class T>
  T* at(uint64_t off) const {
    return reinterpret_cast<T*>(base + ((off & kZeroTag) ? zstart + (off & ~kZeroTag) : off));
  }
};

ms_status status_from_bits(uint32_t bits) {
  const ms_status order[] = {MS_E_CORRUPT, MS_E_RANGE, MS_E_WIDTH_OVERFLOW, MS_E_INVALID, MS_E_UNSUPPORTED,
                             MS_E_NOMEM};
  for (ms_status s : order)
    if (bits & err_bit(s)) return s;
  return MS_OK;
}

ms_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return MS_OK;
  if (e == cudaErrorMemoryAllocation) return MS_E_NOMEM;
  return MS_E_CUDA;
}

#define MS_TRY_CUDA(expr)                    \
  do {                                       \
    cudaError_t e_ = (expr);                 \
    if (e_ != cudaSuccess) return cuda_status(e_); \
  } while (0)
#define MS_TRY(expr)                         \
  do {                                       \
    ms_status s_ = (expr);                   \
    if (s_ != MS_OK) return s_;              \
  } while (0)

ms_status check_fmt(const ms_fmt& f) {
  switch (f.format) {
    case MS_UNCOMPR:
    case MS_RLE:
      return MS_OK;
    case MS_STATIC_BP:
      return f.bit_width <= 64 ? MS_OK : MS_E_INVALID;
    case MS_DYN_BP:
    case MS_FOR_BP:
    case MS_DELTA_BP:
      return valid_B(f.block_size) ? MS_OK : MS_E_INVALID;
    default:
      return MS_E_UNSUPPORTED;
  }
}

// descriptor consistency of an input column (host side)
ms_status check_col(const ms_column* c) {
  if (!c) return MS_E_INVALID;
  const uint64_t n = c->n;
  switch (c->fmt.format) {
    case MS_UNCOMPR:
      if (c->payload_words != n || (n && !c->payload)) return MS_E_INVALID;
      return MS_OK;
    case MS_STATIC_BP:
      if (c->fmt.bit_width < 1 || c->fmt.bit_width > 64) return MS_E_INVALID;
      if (c->payload_words != words_for(n, c->fmt.bit_width) || (n && !c->payload)) return MS_E_INVALID;
      return MS_OK;
    case MS_RLE:
      if (c->payload_words != 2 * c->n_runs || (c->n_runs && !c->payload)) return MS_E_INVALID;
      if ((c->n_runs == 0) != (n == 0) || c->n_runs > n) return MS_E_INVALID;
      return MS_OK;
    case MS_DYN_BP:
    case MS_FOR_BP:
    case MS_DELTA_BP: {
      const uint32_t B = c->fmt.block_size;
      if (!valid_B(B)) return MS_E_INVALID;
      if (c->n_blocks != n / B || c->n_rem != n % B || !c->cw) return MS_E_INVALID;
      if (c->fmt.format != MS_DYN_BP && c->n_blocks && !c->ref) return MS_E_INVALID;
      if (c->n_rem && !c->rem) return MS_E_INVALID;
      if (c->payload_words && !c->payload) return MS_E_INVALID;
      if (c->payload_words % (B / 64)) return MS_E_CORRUPT;
      return MS_OK;
    }
    default:
      return MS_E_UNSUPPORTED;
  }
}

ColView view_of(const ms_column* c) {
  ColView v{};
  v.format = c->fmt.format;
  v.w = c->fmt.bit_width;
  v.maxw = c->fmt.format == MS_STATIC_BP ? c->fmt.bit_width : (c->fmt.max_width <= 64 ? c->fmt.max_width : 0);
  v.B = is_block(c->fmt.format) ? c->fmt.block_size : 1;
  v.log2B = log2u(v.B);
  v.n = c->n;
  v.nb = c->n_blocks;
  v.nrem = c->n_rem;
  v.nruns = c->n_runs;
  v.payload = c->payload;
  v.cw = c->cw;
  v.ref = c->ref;
  v.rem = c->rem;
  return v;
}

// RLE inputs need run starts (and the run covering each 2048-row chunk) to be
// decoded tile by tile; both are transient scratch.
struct RlePrep {
  uint64_t starts = 0, chunk_run = 0, status = 0, ticket = 0;
  bool used = false;
};
void plan_rle(Scratch& sc, const ms_column* c, RlePrep& p) {
  if (!c || c->fmt.format != MS_RLE) return;
  p.used = true;
  p.starts = sc.add(8 * (c->n_runs + 1), false);
  p.chunk_run = sc.add(4 * ((c->n + kChunk - 1) / kChunk + 1), false);
  p.status = sc.add(8 * ((c->n_runs + kChunk - 1) / kChunk + 1), true);
  p.ticket = sc.add(8, true);
}
cudaError_t run_rle(const Scratch& sc, const ms_column* c, const RlePrep& p, ColView& v, uint32_t* err) {
  if (!p.used) return cudaSuccess;
  uint64_t* starts = sc.at<uint64_t>(p.starts);
  uint32_t* cr = sc.at<uint32_t>(p.chunk_run);
  cudaError_t e = launch_rle_starts(c->payload, c->n_runs, c->n, starts, sc.at<uint64_t>(p.status),
                                    sc.at<uint32_t>(p.ticket), err, sc.ctx.s);
  if (e != cudaSuccess) return e;
  e = launch_chunk_run(starts, c->n_runs, c->n, cr, sc.ctx.s);
  v.run_starts = starts;
  v.chunk_run = cr;
  return e;
}

// Allocate an output column: one allocation, 256-byte aligned sections.
ms_status alloc_column(const Ctx& ctx, ms_column* out, const ms_fmt& fmt, uint64_t n, uint64_t payload_cap_words,
                       uint64_t n_runs) {
  std::memset(out, 0, sizeof(*out));
  out->fmt = fmt;
  out->fmt.max_width = 0;
  out->n = n;
  uint64_t nb = 0, nrem = 0;
  if (is_block(fmt.format)) {
    nb = n / fmt.block_size;
    nrem = n % fmt.block_size;
  } else {
    out->fmt.block_size = fmt.format == MS_STATIC_BP ? 0 : fmt.block_size;
  }
  out->n_blocks = nb;
  out->n_rem = nrem;
  out->n_runs = n_runs;
  const uint64_t o_pay = 0;
  uint64_t sz = align_up(8 * payload_cap_words);
  uint64_t o_cw = sz, o_ref = sz, o_rem = sz;
  if (is_block(fmt.format)) {
    o_cw = sz;
    sz = align_up(sz + 4 * (nb + 1));
    o_ref = sz;
    if (fmt.format != MS_DYN_BP) sz = align_up(sz + 8 * nb);
    o_rem = sz;
    sz = align_up(sz + 8 * nrem);
  }
  char* base = (char*)ctx.alloc(sz);
  if (!base) return MS_E_NOMEM;
  out->alloc = base;
  out->alloc_bytes = sz;
  out->payload = (uint64_t*)(base + o_pay);
  if (is_block(fmt.format)) {
    out->cw = (uint32_t*)(base + o_cw);
    out->ref = fmt.format != MS_DYN_BP ? (uint64_t*)(base + o_ref) : nullptr;
    out->rem = (uint64_t*)(base + o_rem);
  }
  return MS_OK;
}

void release(const Ctx& ctx, ms_column* c) {
  if (c && c->alloc) ctx.free(c->alloc);
  if (c) std::memset(c, 0, sizeof(*c));
}

OutView out_view(ms_column* o, uint64_t* status, uint32_t* ticket) {
  OutView v{};
  v.format = o->fmt.format;
  v.w = o->fmt.bit_width;
  v.B = is_block(o->fmt.format) ? o->fmt.block_size : 1;
  v.log2B = log2u(v.B);
  v.n = o->n;
  v.n_dev = nullptr;
  v.payload = o->payload;
  v.cw = o->cw;
  v.ref = o->ref;
  v.rem = o->rem;
  v.status = status;
  v.ticket = ticket;
  return v;
}

// device-to-device copy of the four image sections of `in` into `out` (same shape)
cudaError_t copy_sections(const Ctx& ctx, const ms_column* in, ms_column* out) {
  cudaError_t e = cudaSuccess;
  if (in->payload_words)
    e = cudaMemcpyAsync(out->payload, in->payload, 8 * in->payload_words, cudaMemcpyDeviceToDevice, ctx.s);
  if (e == cudaSuccess && is_block(in->fmt.format)) {
    e = cudaMemcpyAsync(out->cw, in->cw, 4 * (in->n_blocks + 1), cudaMemcpyDeviceToDevice, ctx.s);
    if (e == cudaSuccess && out->ref && in->n_blocks)
      e = cudaMemcpyAsync(out->ref, in->ref, 8 * in->n_blocks, cudaMemcpyDeviceToDevice, ctx.s);
    if (e == cudaSuccess && in->n_rem)
      e = cudaMemcpyAsync(out->rem, in->rem, 8 * in->n_rem, cudaMemcpyDeviceToDevice, ctx.s);
  }
  return e;
}

// Copy a column whose payload was over-allocated into an exact-size allocation
// when asked to (MS_FLAG_SHRINK); otherwise the slack stays with the column (no copy).
ms_status maybe_shrink(const Ctx& ctx, ms_column* out) {
  const uint64_t need = align_up(8 * out->payload_words);
  const uint64_t have = (uint64_t)((char*)(out->cw ? (void*)out->cw : (void*)nullptr) - (char*)out->payload);
  const bool force = ctx.c && (ctx.c->flags & MS_FLAG_SHRINK);
  if (!out->cw || have <= need || !force) return MS_OK;
  ms_column t;
  MS_TRY(alloc_column(ctx, &t, out->fmt, out->n, out->payload_words, out->n_runs));
  t.payload_words = out->payload_words;
  t.fmt.max_width = out->fmt.max_width;
  const cudaError_t e = copy_sections(ctx, out, &t);
  if (e != cudaSuccess) {
    release(ctx, &t);  // the caller releases *out on error
    return cuda_status(e);
  }
  release(ctx, out);
  *out = t;
  return MS_OK;
}

// Read back `count` u64 slots from device into host, synchronise, decode errors.
ms_status readback(const Ctx& ctx, const uint64_t* dev, uint64_t* host, size_t count) {
  uint64_t* pin = count && count <= 32 ? pinned_words() : nullptr;
  if (pin) {
    MS_TRY_CUDA(launch_readback(pin, dev, (uint32_t)count, nullptr, nullptr, nullptr, ctx.s));
  } else if (count) {
    MS_TRY_CUDA(cudaMemcpyAsync(host, dev, 8 * count, cudaMemcpyDeviceToHost, ctx.s));
  }
  MS_TRY_CUDA(cudaStreamSynchronize(ctx.s));
  MS_TRY_CUDA(cudaGetLastError());
  if (pin) std::memcpy(host, pin, 8 * count);
  return MS_OK;
}

// finish an output: read the error word and, for block formats, cw[nb] and
// the largest block width (the max_width hint of the descriptor)
ms_status finish_output(const Ctx& ctx, ms_column* out, const uint32_t* err_dev,
                        const uint64_t* maxw_pre = nullptr) {
  uint64_t h[2] = {0, 0};
  uint32_t maxw = 0;
  uint64_t maxw64 = 0;
  uint32_t* maxw_dev = nullptr;
  if (is_block(out->fmt.format) && out->n_blocks && !maxw_pre) {
    maxw_dev = (uint32_t*)ctx.alloc(4);
    if (!maxw_dev) return MS_E_NOMEM;
    cudaError_t e = cudaMemsetAsync(maxw_dev, 0, 4, ctx.s);
    if (e == cudaSuccess) e = launch_max_width(out->cw, out->n_blocks, maxw_dev, ctx.s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&maxw, maxw_dev, 4, cudaMemcpyDeviceToHost, ctx.s);
    if (e != cudaSuccess) {
      ctx.free(maxw_dev);
      return cuda_status(e);
    }
  }
  uint64_t* pin = pinned_words();
  if (pin && !maxw_dev) {  // one read-back kernel into pinned memory: err, cw[nb], the width scan's maximum
    const bool mp = is_block(out->fmt.format) && out->n_blocks && maxw_pre;
    MS_TRY_CUDA(launch_readback(pin, nullptr, 0, err_dev, is_block(out->fmt.format) ? out->cw + out->n_blocks : nullptr,
                                mp ? maxw_pre : nullptr, ctx.s));
    MS_TRY_CUDA(cudaStreamSynchronize(ctx.s));
    MS_TRY_CUDA(cudaGetLastError());
    h[0] = pin[32];
    h[1] = pin[33];
    maxw64 = pin[34];
  } else {
    if (is_block(out->fmt.format) && out->n_blocks && maxw_pre)
      MS_TRY_CUDA(cudaMemcpyAsync(&maxw64, maxw_pre, 8, cudaMemcpyDeviceToHost, ctx.s));
    MS_TRY_CUDA(cudaMemcpyAsync(&h[0], err_dev, 4, cudaMemcpyDeviceToHost, ctx.s));
    if (is_block(out->fmt.format))
      MS_TRY_CUDA(cudaMemcpyAsync(&h[1], out->cw + out->n_blocks, 4, cudaMemcpyDeviceToHost, ctx.s));
    MS_TRY_CUDA(cudaStreamSynchronize(ctx.s));
  }
  ctx.free(maxw_dev);
  MS_TRY_CUDA(cudaGetLastError());
  if (maxw_pre) maxw = (uint32_t)maxw64;
  const ms_status st = status_from_bits((uint32_t)h[0]);
  if (st != MS_OK) return st;
  if (is_block(out->fmt.format)) {
    if (out->n_blocks == 0) h[1] = 0;
    out->payload_words = (uint32_t)h[1] * (uint64_t)(out->fmt.block_size / 64);
    out->fmt.max_width = maxw;
  } else {
    out->fmt.max_width = 0;
  }
  return MS_OK;
}

uint32_t* sticky_err() {
  static uint32_t* p[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!p[dev]) cudaGetSymbolAddress((void**)&p[dev], g_ms_sticky_err);
  return p[dev];
}

// predicate in range form: keep = ((v - lo) <= span) != neg (D-11)
ms_status make_pred(const ms_pred* p, PredSpec& ps) {
  std::memset(&ps, 0, sizeof(ps));
  const uint64_t MAX = ~0ull;
  auto range = [&](uint64_t lo, uint64_t hi) { ps.lo = lo; ps.span = hi - lo; ps.neg = 0; };
  auto none = [&]() { ps.lo = 0; ps.span = MAX; ps.neg = 1; };
  switch (p->op) {
    case MS_EQ: range(p->a, p->a); break;
    case MS_NE: range(p->a, p->a); ps.neg = 1; break;
    case MS_LT: if (p->a == 0) none(); else range(0, p->a - 1); break;
    case MS_LE: range(0, p->a); break;
    case MS_GT: if (p->a == MAX) none(); else range(p->a + 1, MAX); break;
    case MS_GE: range(p->a, MAX); break;
    case MS_BETWEEN: if (p->b <= p->a) none(); else range(p->a, p->b - 1); break;
    case MS_IN_BITMAP:
      if (!p->bitmap && p->bitmap_bits) return MS_E_INVALID;
      ps.is_bitmap = 1;
      ps.bitmap = p->bitmap;
      ps.bitmap_bits = p->bitmap_bits;
      break;
    default:
      return MS_E_INVALID;
  }
  return MS_OK;
}

bool same_fmt(const ms_fmt& a, const ms_fmt& b) {
  if (a.format != b.format) return false;
  if (a.format == MS_STATIC_BP) return a.bit_width == b.bit_width;
  if (is_block(a.format)) return a.block_size == b.block_size;
  return true;
}

// ------------------------------------------------------------ op bodies
// Encode a source (described by launch functor) into fmt; shared by compress,
// morph and project. n_out is host-known. `launch(out_view)` enqueues the engine.
template <class Launch>
ms_status encode_into(const Ctx& ctx, Scratch& sc, uint64_t meta_off, uint64_t st_off, uint64_t tk_off,
                      uint64_t tk2_off, ms_fmt fmt, uint64_t n, uint64_t payload_cap_words, Launch launch,
                      ms_column* out) {
  uint32_t* err = sc.at<uint32_t>(meta_off);
  const bool auto_width = fmt.format == MS_STATIC_BP && fmt.bit_width == 0;
  if (auto_width) {  // auto width: max pass first
    OutView mv{};
    mv.format = OUT_MAX_ONLY;
    mv.n = n;
    mv.ticket = sc.at<uint32_t>(tk2_off);
    mv.max_out = sc.at<unsigned long long>(meta_off + 8);
    MS_TRY_CUDA(launch(mv));
    uint64_t h[2];
    MS_TRY(readback(ctx, sc.at<uint64_t>(meta_off), h, 2));
    MS_TRY(status_from_bits((uint32_t)h[0]));
    fmt.bit_width = ebw_host(h[1]) ? ebw_host(h[1]) : 1;
  }
  uint64_t cap = payload_cap_words;
  if (fmt.format == MS_STATIC_BP) cap = words_for(n, fmt.bit_width);
  if (fmt.format == MS_UNCOMPR) cap = n;
  MS_TRY(alloc_column(ctx, out, fmt, n, cap, 0));
  if (fmt.format == MS_UNCOMPR) out->payload_words = n;
  if (fmt.format == MS_STATIC_BP) out->payload_words = cap;
  if (is_block(fmt.format)) MS_TRY_CUDA(cudaMemsetAsync(out->cw, 0, 4, ctx.s));  // cw[0] = 0 even when n = 0
  OutView ov = out_view(out, sc.at<uint64_t>(st_off), sc.at<uint32_t>(tk_off));
  ov.fits = auto_width;  // the width bounds every value by construction
  // block formats: slot mode (no look-back)
  const uint64_t n_tiles = (n + kChunk - 1) / kChunk, nb = is_block(fmt.format) ? n / fmt.block_size : 0;
  // (8 bytes per row of slots; when they cannot be allocated the engine falls back
  // to the in-order look-back, which needs no slots)
  bool slot_mode = nb != 0;
  void* slot_mem = nullptr;
  uint64_t *cwx = nullptr, *scan_st = nullptr;
  uint32_t* scan_tk = nullptr;
  const uint64_t chunks = (nb + kChunk - 1) / kChunk + 1;
  if (slot_mode) {
    const uint64_t bytes = align_up(n_tiles * kChunk * 8ull) + align_up(4 * nb) + align_up(8 * (nb + 2)) +
                           align_up(8 * chunks) + kAlign;
    slot_mem = ctx.alloc(bytes);
    slot_mode = slot_mem != nullptr;
  }
  if (slot_mode) {
    char* b = (char*)slot_mem;
    ov.slots = (uint64_t*)b;
    b += align_up(n_tiles * kChunk * 8ull);
    ov.bw = (uint32_t*)b;
    b += align_up(4 * nb);
    cwx = (uint64_t*)b;
    b += align_up(8 * (nb + 2));
    scan_st = (uint64_t*)b;
    b += align_up(8 * chunks);
    scan_tk = (uint32_t*)b;
    cudaError_t z = cudaMemsetAsync(scan_st, 0, align_up(8 * chunks) + kAlign, ctx.s);
    if (z != cudaSuccess) {
      ctx.free(slot_mem);
      release(ctx, out);
      return cuda_status(z);
    }
  }
  cudaError_t e = launch(ov);
  if (e == cudaSuccess && slot_mode) e = launch_count_scan(ov.bw, nb, cwx, scan_st, scan_tk, ctx.s);
  if (e == cudaSuccess && slot_mode) e = launch_tile_copy(ov, n_tiles, nb, cwx, err, ctx.s);
  if (e != cudaSuccess) {
    ctx.free(slot_mem);
    release(ctx, out);
    return cuda_status(e);
  }
  ms_status st = finish_output(ctx, out, err, slot_mode ? cwx + nb + 1 : nullptr);
  ctx.free(slot_mem);
  if (st == MS_OK) st = maybe_shrink(ctx, out);
  if (st != MS_OK) release(ctx, out);
  return st;
}

// RLE compression of raw device values: count run starts per tile,
// scan, write (value, start), then lengths from consecutive starts.
ms_status compress_rle(const Ctx& ctx, const uint64_t* values, uint64_t n, ms_column* out) {
  const uint64_t T = (n + kChunk - 1) / kChunk;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_cnt = sc.add(4 * (T + 1), false);
  const uint64_t o_off = sc.add(8 * (T + 2), true);
  const uint64_t o_st = sc.add(8 * ((T + kChunk - 1) / kChunk + 1), true);
  const uint64_t o_tk = sc.add(8, true);
  if (!sc.commit()) return MS_E_NOMEM;
  MS_TRY_CUDA(launch_rle_count(values, n, sc.at<uint32_t>(o_cnt), ctx.s));
  MS_TRY_CUDA(launch_count_scan(sc.at<uint32_t>(o_cnt), T, sc.at<uint64_t>(o_off), sc.at<uint64_t>(o_st),
                                sc.at<uint32_t>(o_tk), ctx.s));
  uint64_t R = 0;
  MS_TRY(readback(ctx, sc.at<uint64_t>(o_off) + T, &R, 1));
  ms_fmt f{MS_RLE, 0, 0, 0};
  MS_TRY(alloc_column(ctx, out, f, n, 2 * R, R));
  out->payload_words = 2 * R;
  uint64_t* starts = (uint64_t*)ctx.alloc(8 * (R + 1));
  if (!starts) {
    release(ctx, out);
    return MS_E_NOMEM;
  }
  cudaError_t e = launch_rle_write(values, n, sc.at<uint64_t>(o_off), out->payload, starts, ctx.s);
  if (e == cudaSuccess) e = launch_rle_len(starts, R, n, out->payload, ctx.s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.s);
  ctx.free(starts);
  if (e != cudaSuccess) {
    release(ctx, out);
    return cuda_status(e);
  }
  return MS_OK;
}

// worst-case payload words of a block-format column of n values when every
// block may need 64 bits
uint64_t full_cap(uint64_t n, uint32_t B) { return (n / B) * B; }

// The output-side buffer layer of every position-producing operator (select,
// intersect / merge, group extents): a mask of NS * 16 u32 words (1 bit per row,
// rows >= n zero) plus per-segment info (count | 1-based last row << 16) ->
// positions row_offset + row in out_fmt. Runs the segment scan, the
// op's sizing read-back (with the producer's device error word err_in), the
// encoders, and the final read-back of the widths.
ms_status positions_from_mask(const Ctx& ctx, uint32_t* bits, uint32_t* seg_info, uint64_t NS, uint64_t n,
                              uint64_t row_offset, ms_fmt out_fmt, const uint32_t* err_in, ms_column* out) {
  const uint32_t G = is_block(out_fmt.format) ? out_fmt.block_size : (uint32_t)kSegRows;  // output item size
  const uint64_t items_max = (n + G - 1) / G + 1;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);  // [0] err, [1] 1 + max position
  const uint64_t o_off = sc.add(8 * (NS + 1), false);  // the scan writes every entry
  const uint64_t o_gs = sc.add(8 * (items_max + 1), false);
  const uint64_t o_st1 = sc.add(8 * ((NS + kChunk - 1) / kChunk + 1), true);
  const uint64_t o_tk1 = sc.add(8, true);
  const bool pos_delta = out_fmt.format == MS_DELTA_BP && G <= 512;  // posdelta.cuh
  // other formats with items <= 512: the slot encoder (MaskSource), no look-back
  const bool pos_slots = !pos_delta && G <= 512 && out_fmt.format != MS_RLE;
  const uint64_t o_st2 = sc.add(pos_delta || pos_slots ? 8 : 8 * (items_max + 1), true);  // look-back status
  const uint64_t o_tk2 = sc.add(8, true);
  const bool wscan = pos_delta || pos_slots;
  const uint64_t o_wk = wscan ? sc.add(4 * (items_max + 1), false) : 0;
  const uint64_t o_cwx = wscan ? sc.add(8 * (items_max + 2), false) : 0;
  const uint64_t o_dlz = pos_delta ? sc.add(8, true) : 0;                      // deferred blocks: count
  const uint64_t o_dlc = pos_delta ? sc.add(4 * (items_max + 1), false) : 0;    // deferred blocks: entries
  const uint64_t o_st3 = wscan ? sc.add(8 * ((items_max + kChunk - 1) / kChunk + 1), true) : 0;
  const uint64_t o_tk3 = wscan ? sc.add(8, true) : 0;
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  uint64_t* seg_off = sc.at<uint64_t>(o_off);
  MS_TRY_CUDA(launch_seg_scan(seg_info, bits, NS, row_offset, G, seg_off, sc.at<uint64_t>(o_gs),
                              sc.at<unsigned long long>(o_meta + 8), sc.at<uint64_t>(o_st1), sc.at<uint32_t>(o_tk1),
                              ctx.s));
  uint64_t h[4] = {0, 0, 0, 0};
  if (uint64_t* pin = pinned_words()) {  // the op's sizing read-back: one kernel into pinned memory
    MS_TRY_CUDA(launch_readback(pin, sc.at<uint64_t>(o_meta), 2, err_in, nullptr, NS ? seg_off + NS : nullptr, ctx.s));
    MS_TRY_CUDA(cudaStreamSynchronize(ctx.s));
    MS_TRY_CUDA(cudaGetLastError());
    h[0] = pin[0];
    h[1] = pin[1];
    h[2] = pin[34];
    h[3] = pin[32];
  } else {
    if (NS) MS_TRY_CUDA(cudaMemcpyAsync(&h[2], seg_off + NS, 8, cudaMemcpyDeviceToHost, ctx.s));
    if (err_in) MS_TRY_CUDA(cudaMemcpyAsync(&h[3], err_in, 4, cudaMemcpyDeviceToHost, ctx.s));
    MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), h, 2));
  }
  MS_TRY(status_from_bits((uint32_t)h[0] | (uint32_t)h[3]));
  const uint64_t n_out = NS ? h[2] : 0;
  const uint64_t max_pos = h[1] ? h[1] - 1 : 0;
  // size the output (n_out and the largest position are known now)
  uint64_t cap = 0;
  ms_fmt f = out_fmt;
  switch (f.format) {
    case MS_UNCOMPR: cap = n_out; break;
    case MS_RLE: cap = 2 * n_out; break;
    case MS_STATIC_BP: {
      const uint32_t need = n_out ? (ebw_host(max_pos) ? ebw_host(max_pos) : 1) : 1;
      if (f.bit_width == 0) f.bit_width = need;
      else if (n_out && ebw_host(max_pos) > f.bit_width) return MS_E_WIDTH_OVERFLOW;
      cap = words_for(n_out, f.bit_width);
      break;
    }
    default: {
      const uint32_t B = f.block_size;
      const uint64_t nb = n_out / B;
      uint64_t wsum = 64 * nb;
      if (f.format == MS_DYN_BP) {
        wsum = nb * ebw_host(max_pos);
      } else if (nb) {  // sum_k ebw(span_k) <= nb (1 + log2(n / nb)) (Jensen)
        const uint64_t q = (n + nb - 1) / nb;
        const uint64_t lg = q > 1 ? 64 - __builtin_clzll(q - 1) : 0;
        wsum = nb * (1 + lg);
        if (wsum > 64 * nb) wsum = 64 * nb;
      }
      cap = wsum * (B / 64);
    }
  }
  if (is_block(f.format) && 64 * (n_out / f.block_size) > 0xffffffffull) return MS_E_INVALID;
  MS_TRY(alloc_column(ctx, out, f, n_out, cap, f.format == MS_RLE ? n_out : 0));
  if (f.format == MS_UNCOMPR || f.format == MS_RLE || f.format == MS_STATIC_BP) out->payload_words = cap;
  if (is_block(f.format)) {
    cudaError_t e = cudaMemsetAsync(out->cw, 0, 4, ctx.s);
    if (e != cudaSuccess) { release(ctx, out); return cuda_status(e); }
  }
  if (n_out) {
    PosEnc pe{};
    pe.format = f.format;
    pe.w = f.bit_width;
    pe.G = G;
    pe.log2G = log2u(G);
    pe.n_out = n_out;
    pe.payload = out->payload;
    pe.cw = out->cw;
    pe.ref = out->ref;
    pe.rem = out->rem;
    // single-walk slots for DELTA_BP positions: every delta is < NS * 512 rows, so
    // wcap = ebw(NS * 512 - 1) bits per code bound every block (B * wcap / 64 words per slot)
    uint64_t* slots = nullptr;
    uint32_t slot_words = 0;
    if (pos_delta && f.format == MS_DELTA_BP) {
      const uint32_t wcap = ebw_host(NS * kSegRows - 1);
      slot_words = G / 64 * (wcap ? wcap : 1);
      slots = (uint64_t*)ctx.alloc(8 * (n_out / G) * (uint64_t)slot_words);
      if (!slots) { release(ctx, out); return MS_E_NOMEM; }
    }
    if (pos_slots && is_block(f.format) && n_out / G) {  // DYN_BP / FOR_BP positions: 64-bit slots
      slot_words = G;  // G / 64 * 64
      slots = (uint64_t*)ctx.alloc(8 * (n_out / G) * (uint64_t)slot_words);
      if (!slots) { release(ctx, out); return MS_E_NOMEM; }
    }
    cudaError_t e =
        pos_delta && f.format == MS_DELTA_BP
            ? launch_positions_delta(pe, bits, NS, sc.at<uint64_t>(o_gs), row_offset,
                                     sc.at<uint32_t>(o_wk), sc.at<uint64_t>(o_cwx), sc.at<uint64_t>(o_st3),
                                     sc.at<uint32_t>(o_tk3), slots, slot_words, sc.at<uint32_t>(o_dlz), sc.at<uint32_t>(o_dlc), err, ctx.s)
        : pos_slots
            ? launch_positions_slots(pe, bits, NS, sc.at<uint64_t>(o_gs), row_offset, slots,
                                     slot_words, sc.at<uint32_t>(o_wk), sc.at<uint64_t>(o_cwx),
                                     sc.at<uint64_t>(o_st3), sc.at<uint32_t>(o_tk3), err, ctx.s)
            : launch_positions(pe, bits, NS, sc.at<uint64_t>(o_gs), row_offset,
                               sc.at<uint64_t>(o_st2), sc.at<uint32_t>(o_tk2), err, ctx.s);
    ctx.free(slots);  // stream-ordered free: the copy kernel is queued before it
    if (e != cudaSuccess) {
      release(ctx, out);
      return cuda_status(e);
    }
  }
  const bool wmax_known = (pos_delta || pos_slots) && is_block(f.format) && n_out / G;
  ms_status st = finish_output(ctx, out, err, wmax_known ? sc.at<uint64_t>(o_cwx) + n_out / G + 1 : nullptr);
  if (st == MS_OK) st = maybe_shrink(ctx, out);
  if (st != MS_OK) release(ctx, out);
  return st;
}


}  // namespace

// ===================================================================== ABI
extern "C" {

int ms_abi_version(void) { return MS_ABI_VERSION; }
uint64_t ms_launch_count(void) { return launch_count(); }
void ms_profile_enable(int on) { profile_enable(on); }
int ms_profile_read(ms_kernel_time* out, int max) { return profile_read(out, max); }

const char* ms_status_str(ms_status s) {
  switch (s) {
    case MS_OK: return "MS_OK";
    case MS_E_INVALID: return "MS_E_INVALID";
    case MS_E_WIDTH_OVERFLOW: return "MS_E_WIDTH_OVERFLOW";
    case MS_E_UNSUPPORTED: return "MS_E_UNSUPPORTED";
    case MS_E_RANGE: return "MS_E_RANGE";
    case MS_E_CORRUPT: return "MS_E_CORRUPT";
    case MS_E_NOMEM: return "MS_E_NOMEM";
    case MS_E_CUDA: return "MS_E_CUDA";
  }
  return "MS_E_UNKNOWN";
}

uint64_t ms_column_bytes(const ms_column* c) {
  if (!c) return 0;
  uint64_t b = 8 * c->payload_words;
  if (is_block(c->fmt.format)) {
    b += 4 * (c->n_blocks + 1) + 8 * c->n_rem;
    if (c->fmt.format != MS_DYN_BP) b += 8 * c->n_blocks;
  }
  return b;
}

void ms_column_release(const ms_ctx* ctx, ms_column* col) { release(Ctx(ctx), col); }

ms_status ms_compress(const ms_ctx* ctx_, const uint64_t* values, uint64_t n, ms_fmt fmt, ms_column* out) {
  if (!out) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_fmt(fmt));
  if (n && !values) return MS_E_INVALID;
  Ctx ctx(ctx_);
  if (is_block(fmt.format) && 64 * (n / fmt.block_size) > 0xffffffffull) return MS_E_INVALID;  // D-4
  if (fmt.format == MS_RLE) return compress_rle(ctx, values, n, out);
  ms_column in{};
  in.fmt = ms_fmt{MS_UNCOMPR, 0, 0, 0};
  in.n = n;
  in.payload_words = n;
  in.payload = const_cast<uint64_t*>(values);
  const ColView src = view_of(&in);
  const uint64_t items = (n + kChunk - 1) / kChunk;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_st = sc.add(8 * (items + 1), true);
  const uint64_t o_tk = sc.add(8, true);
  const uint64_t o_tk2 = sc.add(8, true);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  auto launch = [&](const OutView& ov) { return launch_engine_col(src, ov, err, ctx.s); };
  return encode_into(ctx, sc, o_meta, o_st, o_tk, o_tk2, fmt, n,
                     is_block(fmt.format) ? full_cap(n, fmt.block_size) : 0, launch, out);
}

ms_status ms_decompress(const ms_ctx* ctx_, const ms_column* in, uint64_t* values) {
  MS_TRY(check_col(in));
  if (in->n && !values) return MS_E_INVALID;
  if (in->n == 0) return MS_OK;
  Ctx ctx(ctx_);
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_tk = sc.add(8, true);
  RlePrep rp;
  plan_rle(sc, in, rp);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView src = view_of(in);
  MS_TRY_CUDA(run_rle(sc, in, rp, src, err));
  if (in->fmt.format == MS_RLE) {  // runs expanded directly, no tile decode
    MS_TRY_CUDA(launch_rle_expand(in->payload, src.run_starts, in->n_runs, in->n, values, ctx.s));
    uint64_t h = 0;
    MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), &h, 1));
    return status_from_bits((uint32_t)h);
  }
  ms_column o{};
  o.fmt = ms_fmt{MS_UNCOMPR, 0, 0, 0};
  o.n = in->n;
  o.payload = values;
  OutView ov = out_view(&o, nullptr, sc.at<uint32_t>(o_tk));
  MS_TRY_CUDA(launch_engine_col(src, ov, err, ctx.s));
  uint64_t h = 0;
  MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), &h, 1));
  return status_from_bits((uint32_t)h);
}

ms_status ms_morph(const ms_ctx* ctx_, const ms_column* in, ms_fmt fmt, ms_column* out) {
  if (!out) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_col(in));
  MS_TRY(check_fmt(fmt));
  Ctx ctx(ctx_);
  const uint64_t n = in->n;
  if (is_block(fmt.format) && 64 * (n / fmt.block_size) > 0xffffffffull) return MS_E_INVALID;
  if (same_fmt(in->fmt, fmt)) {  // identity morph: byte-identical
    MS_TRY(alloc_column(ctx, out, in->fmt, n, in->payload_words, in->n_runs));
    out->payload_words = in->payload_words;
    out->fmt.max_width = in->fmt.max_width;
    const cudaError_t e = copy_sections(ctx, in, out);
    if (e != cudaSuccess) {
      release(ctx, out);  // *out zeroed, nothing leaks
      return cuda_status(e);
    }
    return MS_OK;
  }
  if (delta_direct_supported(view_of(in)) && fmt.format == MS_STATIC_BP) {
    // DELTA_BP -> STATIC_BP directly (delta.cu): [max pass for the auto width,] then every
    // output word written once (into u64 values the staged engine is faster: 1.5 vs 2.7 ms
    // for c3's 2^29 rows)
    Scratch sc(ctx);
    const uint64_t o_meta = sc.add(64, true);  // [0] err, [1] max
    if (!sc.commit()) return MS_E_NOMEM;
    uint32_t* err = sc.at<uint32_t>(o_meta);
    const ColView v = view_of(in);
    ms_fmt f = fmt;
    if (f.format == MS_STATIC_BP && f.bit_width == 0) {
      // the width from the block headers when their bounds agree, else from a max pass
      MS_TRY_CUDA(launch_delta_bounds(v, sc.at<unsigned long long>(o_meta + 16), ctx.s));
      uint64_t h[4];
      MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), h, 4));
      uint32_t wb = ebw_host(h[3]);
      if (ebw_host(h[2]) != wb) {
        MS_TRY_CUDA(launch_delta_max(v, sc.at<unsigned long long>(o_meta + 8), err, ctx.s));
        MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), h, 2));
        MS_TRY(status_from_bits((uint32_t)h[0]));
        wb = ebw_host(h[1]);
      }
      f.bit_width = wb ? wb : 1;
    }
    const uint64_t words = f.format == MS_UNCOMPR ? n : words_for(n, f.bit_width);
    MS_TRY(alloc_column(ctx, out, f, n, words, 0));
    out->payload_words = words;
    cudaError_t e = f.format == MS_UNCOMPR ? launch_delta_decode(v, out->payload, err, ctx.s)
                                           : launch_delta_to_static(v, f.bit_width, out->payload, err, ctx.s);
    uint64_t h = 0;
    ms_status st = e == cudaSuccess ? readback(ctx, sc.at<uint64_t>(o_meta), &h, 1) : cuda_status(e);
    if (st == MS_OK) st = status_from_bits((uint32_t)h);
    if (st != MS_OK) release(ctx, out);
    return st;
  }
  if (in->fmt.format == MS_RLE && fmt.format == MS_DELTA_BP) {
    // direct morph: from the runs alone (morph.cu)
    const uint32_t B = fmt.block_size;
    const uint64_t nb = n / B, nrem = n % B;
    Scratch sc(ctx);
    const uint64_t o_meta = sc.add(64, true);
    const uint64_t o_wk = sc.add(4 * (nb + 1), false);
    const uint64_t o_cwx = sc.add(8 * (nb + 2), false);
    const uint64_t o_ref = sc.add(8 * (nb + 1), false);
    const uint64_t o_rem = sc.add(8 * (nrem + 1), false);
    const uint64_t o_st = sc.add(8 * ((nb + kChunk - 1) / kChunk + 1), true);
    const uint64_t o_tk = sc.add(8, true);
    RlePrep rp;
    plan_rle(sc, in, rp);
    if (!sc.commit()) return MS_E_NOMEM;
    uint32_t* err = sc.at<uint32_t>(o_meta);
    ColView src = view_of(in);
    MS_TRY_CUDA(run_rle(sc, in, rp, src, err));
    MS_TRY_CUDA(launch_rle2delta_widths(src, B, nb, sc.at<uint32_t>(o_wk), sc.at<uint64_t>(o_ref),
                                        sc.at<uint64_t>(o_rem), ctx.s));
    uint64_t h[2] = {0, 0};
    if (nb) {
      MS_TRY_CUDA(launch_count_scan(sc.at<uint32_t>(o_wk), nb, sc.at<uint64_t>(o_cwx), sc.at<uint64_t>(o_st),
                                    sc.at<uint32_t>(o_tk), ctx.s));
      MS_TRY_CUDA(cudaMemcpyAsync(&h[1], sc.at<uint64_t>(o_cwx) + nb, 8, cudaMemcpyDeviceToHost, ctx.s));
    }
    MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), h, 1));
    MS_TRY(status_from_bits((uint32_t)h[0]));
    if (h[1] > 0xffffffffull) return MS_E_INVALID;  // D-4 limit
    const uint64_t words = h[1] * (B / 64);
    MS_TRY(alloc_column(ctx, out, fmt, n, words, 0));
    out->payload_words = words;
    cudaError_t e = cudaMemsetAsync(out->cw, 0, 4, ctx.s);
    if (e == cudaSuccess && words) e = cudaMemsetAsync(out->payload, 0, 8 * words, ctx.s);
    if (e == cudaSuccess && nb)
      e = cudaMemcpyAsync(out->ref, sc.at<uint64_t>(o_ref), 8 * nb, cudaMemcpyDeviceToDevice, ctx.s);
    if (e == cudaSuccess && nrem)
      e = cudaMemcpyAsync(out->rem, sc.at<uint64_t>(o_rem), 8 * nrem, cudaMemcpyDeviceToDevice, ctx.s);
    if (e == cudaSuccess && nb)
      e = launch_rle2delta_pack(src, B, nb, sc.at<uint64_t>(o_cwx), out->cw, out->payload, err, ctx.s);
    if (e != cudaSuccess) {
      release(ctx, out);
      return cuda_status(e);
    }
    ms_status st = finish_output(ctx, out, err, nb ? sc.at<uint64_t>(o_cwx) + nb + 1 : nullptr);
    if (st != MS_OK) release(ctx, out);
    return st;
  }
  if (fmt.format == MS_RLE) {  // tile by tile from the decoded input (plan.cu), no staging column
    const uint64_t T = (n + kChunk - 1) / kChunk;
    Scratch sc(ctx);
    const uint64_t o_meta = sc.add(64, true);
    const uint64_t o_cnt = sc.add(4 * (T + 1), false);
    const uint64_t o_fl = sc.add(16 * (T + 1), false);
    const uint64_t o_off = sc.add(8 * (T + 2), true);
    const uint64_t o_st = sc.add(8 * ((T + kChunk - 1) / kChunk + 1), true);
    const uint64_t o_tk = sc.add(8, true);
    RlePrep rp;
    plan_rle(sc, in, rp);
    if (!sc.commit()) return MS_E_NOMEM;
    uint32_t* err = sc.at<uint32_t>(o_meta);
    ColView src = view_of(in);
    MS_TRY_CUDA(run_rle(sc, in, rp, src, err));
    MS_TRY_CUDA(launch_rle_count_col(src, sc.at<uint32_t>(o_cnt), sc.at<uint64_t>(o_fl), ctx.s));
    MS_TRY_CUDA(launch_count_scan(sc.at<uint32_t>(o_cnt), T, sc.at<uint64_t>(o_off), sc.at<uint64_t>(o_st),
                                  sc.at<uint32_t>(o_tk), ctx.s));
    uint64_t h[2] = {0, 0};
    if (T) MS_TRY_CUDA(cudaMemcpyAsync(&h[1], sc.at<uint64_t>(o_off) + T, 8, cudaMemcpyDeviceToHost, ctx.s));
    MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), h, 1));
    MS_TRY(status_from_bits((uint32_t)h[0]));
    const uint64_t R = h[1];
    ms_fmt f{MS_RLE, 0, 0, 0};
    MS_TRY(alloc_column(ctx, out, f, n, 2 * R, R));
    out->payload_words = 2 * R;
    uint64_t* starts = (uint64_t*)ctx.alloc(8 * (R + 1));
    if (!starts) {
      release(ctx, out);
      return MS_E_NOMEM;
    }
    cudaError_t e = launch_rle_write_col(src, sc.at<uint64_t>(o_fl), sc.at<uint64_t>(o_off), out->payload, starts,
                                         ctx.s);
    if (e == cudaSuccess) e = launch_rle_len(starts, R, n, out->payload, ctx.s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx.s);
    ctx.free(starts);
    if (e != cudaSuccess) {
      release(ctx, out);
      return cuda_status(e);
    }
    return MS_OK;
  }
  const uint64_t items = (n + kChunk - 1) / kChunk;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_st = sc.add(8 * (items + 1), true);
  const uint64_t o_tk = sc.add(8, true);
  const uint64_t o_tk2 = sc.add(8, true);
  RlePrep rp;
  plan_rle(sc, in, rp);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView src = view_of(in);
  MS_TRY_CUDA(run_rle(sc, in, rp, src, err));
  auto launch = [&](const OutView& ov) { return launch_engine_col(src, ov, err, ctx.s); };
  return encode_into(ctx, sc, o_meta, o_st, o_tk, o_tk2, fmt, n,
                     is_block(fmt.format) ? full_cap(n, fmt.block_size) : 0, launch, out);
}

ms_status ms_select(const ms_ctx* ctx_, const ms_column* in, const ms_pred* pred, uint64_t row_offset,
                    ms_fmt out_fmt, ms_column* out) {
  if (!out || !pred) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_col(in));
  MS_TRY(check_fmt(out_fmt));
  PredSpec ps;
  MS_TRY(make_pred(pred, ps));
  Ctx ctx(ctx_);
  const uint64_t n = in->n;
  const uint64_t NS = (n + kSegRows - 1) / kSegRows;  // 512-row segments
  const uint64_t n_words = NS * kSegWords;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);  // [0] err
  const uint64_t o_bits = sc.add(4 * n_words, false);
  const uint64_t o_seg = sc.add(4 * (NS + 1), false);
  const uint64_t o_list = sc.add(4 * ((NS * kSegRows + kChunk - 1) / kChunk + 2), false);  // pruning work list
  RlePrep rp;
  plan_rle(sc, in, rp);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView src = view_of(in);
  MS_TRY_CUDA(run_rle(sc, in, rp, src, err));
  MS_TRY_CUDA(launch_select(src, ps, sc.at<uint32_t>(o_bits), sc.at<uint32_t>(o_seg), NS, sc.at<uint32_t>(o_list),
                            err, ctx.s));
  return positions_from_mask(ctx, sc.at<uint32_t>(o_bits), sc.at<uint32_t>(o_seg), NS, n, row_offset, out_fmt, err,
                             out);
}

ms_status ms_project(const ms_ctx* ctx_, const ms_column* data, const ms_column* positions, uint64_t row_offset,
                     ms_fmt out_fmt, ms_column* out) {
  if (!out) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_col(data));
  MS_TRY(check_col(positions));
  MS_TRY(check_fmt(out_fmt));
  if (out_fmt.format == MS_RLE) return MS_E_UNSUPPORTED;
  Ctx ctx(ctx_);
  const uint64_t n = positions->n;
  // DELTA_BP / RLE data have no O(1) row access (D-12): the gather engine decodes
  // only the data tiles a positions tile spans (no whole-column materialisation, DP3)
  if (is_block(out_fmt.format) && 64 * (n / out_fmt.block_size) > 0xffffffffull) return MS_E_INVALID;
  const uint64_t items = (n + 127) / 128;  // enough for any item size (>= 128 rows)
  // the slot path (no look-back status) serves item sizes <= 512 into block formats or UNCOMPR
  const uint32_t G0 = is_block(out_fmt.format) ? out_fmt.block_size : (uint32_t)kSegRows;
  const int32_t pf0 = positions->fmt.format, df0 = data->fmt.format;
  const bool warp_path = (pf0 == MS_UNCOMPR || pf0 == MS_STATIC_BP || pf0 == MS_DYN_BP || pf0 == MS_FOR_BP ||
                          (pf0 == MS_DELTA_BP && positions->fmt.block_size == G0)) &&
                         (df0 == MS_UNCOMPR || df0 == MS_STATIC_BP || df0 == MS_DYN_BP || df0 == MS_FOR_BP) &&
                         !(out_fmt.format == MS_STATIC_BP && out_fmt.bit_width == 0);
  const bool slot_path = warp_path && G0 <= 512 &&
                         (is_block(out_fmt.format) || out_fmt.format == MS_UNCOMPR || out_fmt.format == MS_STATIC_BP);
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_st = sc.add(slot_path ? 8 : 8 * (items + 1), true);
  const uint64_t o_tk = sc.add(8, true);
  const uint64_t o_tk2 = sc.add(8, true);
  const uint64_t o_wk = sc.add(4 * (items + 1), false);
  const uint64_t o_cwx = sc.add(8 * (items + 2), false);
  const uint64_t o_st3 = sc.add(8 * ((items + kChunk - 1) / kChunk + 1), true);
  const uint64_t o_tk3 = sc.add(8, true);
  RlePrep rp_pos, rp_data;
  plan_rle(sc, positions, rp_pos);
  plan_rle(sc, data, rp_data);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView pv = view_of(positions), dv = view_of(data);
  MS_TRY_CUDA(run_rle(sc, positions, rp_pos, pv, err));
  MS_TRY_CUDA(run_rle(sc, data, rp_data, dv, err));
  uint64_t cap = 0;
  if (is_block(out_fmt.format)) {
    uint32_t wmax = 64;  // projected codes cannot be wider than a static data width
    if (data->fmt.format == MS_STATIC_BP && out_fmt.format != MS_DELTA_BP) wmax = data->fmt.bit_width;
    cap = (n / out_fmt.block_size) * (out_fmt.block_size / 64) * wmax;
  }
  // warp pipeline (positions decoded block-aligned, data gathered with header broadcast)
  const uint32_t G = is_block(out_fmt.format) ? out_fmt.block_size : (uint32_t)kSegRows;
  const int32_t pf = positions->fmt.format, df = data->fmt.format;
  const bool pos_ok = pf == MS_UNCOMPR || pf == MS_STATIC_BP || pf == MS_DYN_BP || pf == MS_FOR_BP ||
                      (pf == MS_DELTA_BP && positions->fmt.block_size == G);
  const bool data_ok = df == MS_UNCOMPR || df == MS_STATIC_BP || df == MS_DYN_BP || df == MS_FOR_BP;
  const bool out_ok = !(out_fmt.format == MS_STATIC_BP && out_fmt.bit_width == 0);
  if (pos_ok && data_ok && out_ok) {
    ms_fmt f = out_fmt;
    if (f.format == MS_STATIC_BP) cap = words_for(n, f.bit_width);
    if (f.format == MS_UNCOMPR) cap = n;
    MS_TRY(alloc_column(ctx, out, f, n, cap, 0));
    if (f.format == MS_UNCOMPR || f.format == MS_STATIC_BP) out->payload_words = cap;
    cudaError_t e = cudaSuccess;
    if (is_block(f.format)) e = cudaMemsetAsync(out->cw, 0, 4, ctx.s);
    PosEnc pe{};
    pe.format = f.format;
    pe.w = f.bit_width;
    pe.G = G;
    pe.log2G = log2u(G);
    pe.n_out = n;
    pe.payload = out->payload;
    pe.cw = out->cw;
    pe.ref = out->ref;
    pe.rem = out->rem;
    // per-block slots (no look-back) for block outputs of size <= 512 and UNCOMPR; the
    // slot holds a block at the largest width its codes can have
    const bool slotted = slot_path;
    uint64_t* slots = nullptr;
    uint32_t slot_words = 0;
    if (slotted && is_block(f.format) && n / G) {
      uint32_t wcap = 64;
      if (df == MS_STATIC_BP && f.format != MS_DELTA_BP) wcap = data->fmt.bit_width ? data->fmt.bit_width : 64;
      slot_words = G / 64 * wcap;
      slots = (uint64_t*)ctx.alloc(8 * (n / G) * (uint64_t)slot_words);
      if (!slots) e = cudaErrorMemoryAllocation;
    }
    // dense positions stream the data windows through shared memory (projstream.cuh): when the
    // average window of an output block (the data payload over the blocks, if the positions span
    // the column) fits a stage with room for its spread
    void* wins = nullptr;
    const uint64_t n_items_out = (n + G - 1) / G;
    if (e == cudaSuccess && slots && !(ctx.c && (ctx.c->flags & MS_FLAG_GATHER)) &&
        project_stream_supported(pv, dv, pe) && 8 * data->payload_words <= (n / G) * (uint64_t)kStreamAvgWindow) {
      wins = ctx.alloc(project_stream_win_bytes(n_items_out));
      if (!wins) e = cudaErrorMemoryAllocation;
    }
    if (e == cudaSuccess)
      e = slotted ? launch_project_slots(pv, dv, row_offset, pe, slots, slot_words, sc.at<uint32_t>(o_wk),
                                         sc.at<uint64_t>(o_cwx), sc.at<uint64_t>(o_st3), sc.at<uint32_t>(o_tk3), wins,
                                         8 * data->payload_words, err, ctx.s)
                  : launch_project_warp(pv, dv, row_offset, pe, sc.at<uint64_t>(o_st), sc.at<uint32_t>(o_tk), err,
                                        ctx.s);
    ctx.free(wins);
    ctx.free(slots);
    if (e != cudaSuccess) {
      release(ctx, out);
      return cuda_status(e);
    }
    ms_status st = finish_output(ctx, out, err,
                                 slotted && is_block(f.format) && n / G ? sc.at<uint64_t>(o_cwx) + n / G + 1 : nullptr);
    if (st == MS_OK) st = maybe_shrink(ctx, out);
    if (st != MS_OK) release(ctx, out);
    return st;
  }
  auto launch = [&](const OutView& ov) { return launch_engine_gather(pv, dv, row_offset, ov, err, ctx.s); };
  return encode_into(ctx, sc, o_meta, o_st, o_tk, o_tk2, out_fmt, n, cap, launch, out);
}

ms_status ms_agg_sum(const ms_ctx* ctx_, const ms_column* in, const ms_column* positions, uint64_t row_offset,
                     uint64_t* sum) {
  MS_TRY(check_col(in));
  if (positions) MS_TRY(check_col(positions));
  if (!sum) return MS_E_INVALID;
  Ctx ctx(ctx_);
  MS_TRY_CUDA(cudaMemsetAsync(sum, 0, 8, ctx.s));
  uint32_t* err = sticky_err();
  const bool need_rle = in->fmt.format == MS_RLE || (positions && positions->fmt.format == MS_RLE);
  if (!need_rle) {
    if (positions)
      MS_TRY_CUDA(launch_sum_at(view_of(in), view_of(positions), row_offset, (unsigned long long*)sum, err, ctx.s));
    else if (in->n)
      MS_TRY_CUDA(launch_sum(view_of(in), (unsigned long long*)sum, err, ctx.s));
    return MS_OK;
  }
  Scratch sc(ctx);
  RlePrep rp_in, rp_pos;
  plan_rle(sc, in, rp_in);
  plan_rle(sc, positions, rp_pos);
  if (!sc.commit()) return MS_E_NOMEM;
  ColView iv = view_of(in);
  MS_TRY_CUDA(run_rle(sc, in, rp_in, iv, err));
  if (positions) {
    ColView pv = view_of(positions);
    MS_TRY_CUDA(run_rle(sc, positions, rp_pos, pv, err));
    MS_TRY_CUDA(launch_sum_at(iv, pv, row_offset, (unsigned long long*)sum, err, ctx.s));
  } else if (in->n) {
    MS_TRY_CUDA(launch_sum(iv, (unsigned long long*)sum, err, ctx.s));
  }
  return MS_OK;  // scratch is freed stream-ordered after the kernels
}

ms_status ms_agg_sum_grouped(const ms_ctx* ctx_, const ms_column* gid, const ms_column* vals, uint64_t n_groups,
                             uint64_t* sums) {
  MS_TRY(check_col(gid));
  MS_TRY(check_col(vals));
  if (gid->n != vals->n) return MS_E_INVALID;  // LengthMismatch
  if (n_groups && !sums) return MS_E_INVALID;
  Ctx ctx(ctx_);
  if (n_groups) MS_TRY_CUDA(cudaMemsetAsync(sums, 0, 8 * n_groups, ctx.s));
  if (gid->n == 0) return MS_OK;
  uint32_t* err = sticky_err();
  Scratch sc(ctx);
  RlePrep rp_g, rp_v;
  plan_rle(sc, gid, rp_g);
  plan_rle(sc, vals, rp_v);
  if (!sc.commit()) return MS_E_NOMEM;
  ColView gv = view_of(gid), vv = view_of(vals);
  MS_TRY_CUDA(run_rle(sc, gid, rp_g, gv, err));
  MS_TRY_CUDA(run_rle(sc, vals, rp_v, vv, err));
  MS_TRY_CUDA(launch_sum_grouped(gv, vv, n_groups, (unsigned long long*)sums, err, ctx.s));
  return MS_OK;
}

ms_status ms_column_to_device(const ms_ctx* ctx_, const ms_column* h, ms_column* out) {
  if (!out) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_col(h));
  Ctx ctx(ctx_);
  uint32_t mw = 0;
  if (is_block(h->fmt.format)) {  // validate the host width table; the max_width hint
    if (h->cw[0] != 0) return MS_E_CORRUPT;
    for (uint64_t b = 0; b < h->n_blocks; ++b) {
      if (h->cw[b + 1] < h->cw[b]) return MS_E_CORRUPT;
      const uint32_t w = h->cw[b + 1] - h->cw[b];
      if (w > 64) return MS_E_CORRUPT;
      mw = w > mw ? w : mw;
    }
    if ((uint64_t)h->cw[h->n_blocks] * (h->fmt.block_size / 64) != h->payload_words) return MS_E_CORRUPT;
  }
  MS_TRY(alloc_column(ctx, out, h->fmt, h->n, h->payload_words, h->n_runs));
  out->payload_words = h->payload_words;
  if (is_block(h->fmt.format)) out->fmt.max_width = mw;
  auto cp = [&](void* d, const void* s, uint64_t bytes) {
    return bytes ? cudaMemcpyAsync(d, s, bytes, cudaMemcpyHostToDevice, ctx.s) : cudaSuccess;
  };
  cudaError_t e = cp(out->payload, h->payload, 8 * h->payload_words);
  if (e == cudaSuccess && is_block(h->fmt.format)) {
    e = cp(out->cw, h->cw, 4 * (h->n_blocks + 1));
    if (e == cudaSuccess && out->ref) e = cp(out->ref, h->ref, 8 * h->n_blocks);
    if (e == cudaSuccess) e = cp(out->rem, h->rem, 8 * h->n_rem);
  }
  if (e != cudaSuccess) {
    release(ctx, out);
    return cuda_status(e);
  }
  return MS_OK;
}

ms_status ms_column_to_host(const ms_ctx* ctx_, const ms_column* d, ms_column* h) {
  MS_TRY(check_col(d));
  if (!h) return MS_E_INVALID;
  Ctx ctx(ctx_);
  auto cp = [&](void* dst, const void* s, uint64_t bytes) {
    if (!bytes) return cudaSuccess;
    if (!dst) return cudaErrorInvalidValue;
    return cudaMemcpyAsync(dst, s, bytes, cudaMemcpyDeviceToHost, ctx.s);
  };
  MS_TRY_CUDA(cp(h->payload, d->payload, 8 * d->payload_words));
  if (is_block(d->fmt.format)) {
    MS_TRY_CUDA(cp(h->cw, d->cw, 4 * (d->n_blocks + 1)));
    if (d->ref) MS_TRY_CUDA(cp(h->ref, d->ref, 8 * d->n_blocks));
    MS_TRY_CUDA(cp(h->rem, d->rem, 8 * d->n_rem));
  }
  MS_TRY_CUDA(cudaStreamSynchronize(ctx.s));
  h->fmt = d->fmt;
  h->n = d->n;
  h->n_blocks = d->n_blocks;
  h->n_rem = d->n_rem;
  h->n_runs = d->n_runs;
  h->payload_words = d->payload_words;
  h->alloc = nullptr;
  h->alloc_bytes = 0;
  return MS_OK;
}

// ------------------------------------------------------------ plan-level operators (plan.cu)
ms_status ms_format_sizes(const ms_ctx* ctx_, const ms_column* in, uint32_t block_size, uint64_t* sizes,
                          ms_fmt* best) {
  MS_TRY(check_col(in));
  if (!sizes || !valid_B(block_size)) return MS_E_INVALID;
  Ctx ctx(ctx_);
  const uint64_t n = in->n, B = block_size, nb = n / B, nrem = n % B;
  const uint64_t T = (n + kChunk - 1) / kChunk;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);   // [0] err
  const uint64_t o_acc = sc.add(64, true);    // max, sum w DYN, sum w DELTA, sum w FOR, runs
  const uint64_t o_fl = sc.add(16 * (T + 1), false);
  RlePrep rp;
  plan_rle(sc, in, rp);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView v = view_of(in);
  MS_TRY_CUDA(run_rle(sc, in, rp, v, err));
  MS_TRY_CUDA(launch_profile(v, block_size, sc.at<unsigned long long>(o_acc), sc.at<uint64_t>(o_fl), ctx.s));
  uint64_t h[8] = {0};
  MS_TRY_CUDA(cudaMemcpyAsync(h + 1, sc.at<uint64_t>(o_acc), 40, cudaMemcpyDeviceToHost, ctx.s));
  MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), h, 1));  // the op's one sync
  MS_TRY(status_from_bits((uint32_t)h[0]));
  const uint64_t mx = h[1], hdr = 4 * (nb + 1) + 8 * nrem;
  const uint32_t w = ebw_host(mx) ? ebw_host(mx) : 1;
  sizes[0] = 8 * n;                                   // UNCOMPR
  sizes[1] = 8 * words_for(n, w);                     // STATIC_BP at its auto width
  sizes[2] = 8 * (h[2] * (B / 64)) + hdr;             // DYN_BP{B}
  sizes[3] = 8 * (h[3] * (B / 64)) + hdr + 8 * nb;    // DELTA_BP{B}
  sizes[4] = 8 * (h[4] * (B / 64)) + hdr + 8 * nb;    // FOR_BP{B}
  sizes[5] = n ? 16 * h[5] : 0;                       // RLE
  if (best) {
    int k = 0;
    for (int i = 1; i < MS_N_CANDIDATES; ++i)
      if (sizes[i] < sizes[k]) k = i;  // ties: the earlier (simpler) format
    const int32_t order[MS_N_CANDIDATES] = {MS_UNCOMPR, MS_STATIC_BP, MS_DYN_BP, MS_DELTA_BP, MS_FOR_BP, MS_RLE};
    *best = ms_fmt{order[k], order[k] == MS_STATIC_BP ? w : 0u, is_block(order[k]) ? block_size : 0u, 0u};
  }
  return MS_OK;
}

// intersect (op 0) / merge (op 1) of two strictly increasing position columns via a
// bit mask over the positions' common range, then the select output encoders
static ms_status set_op(const ms_ctx* ctx_, const ms_column* a, const ms_column* b, int op, ms_fmt out_fmt,
                        ms_column* out) {
  if (!out) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_col(a));
  MS_TRY(check_col(b));
  MS_TRY(check_fmt(out_fmt));
  Ctx ctx(ctx_);
  Scratch s1(ctx);
  const uint64_t o_meta = s1.add(64, true);
  const uint64_t o_ends = s1.add(32, false);
  RlePrep ra, rb;
  plan_rle(s1, a, ra);
  plan_rle(s1, b, rb);
  if (!s1.commit()) return MS_E_NOMEM;
  uint32_t* err = s1.at<uint32_t>(o_meta);
  ColView va = view_of(a), vb = view_of(b);
  MS_TRY_CUDA(run_rle(s1, a, ra, va, err));
  MS_TRY_CUDA(run_rle(s1, b, rb, vb, err));
  MS_TRY_CUDA(launch_ends(va, vb, s1.at<uint64_t>(o_ends), ctx.s));
  uint64_t e[4];
  MS_TRY(readback(ctx, s1.at<uint64_t>(o_ends), e, 4));  // sizing sync: the ranges
  uint64_t lo = 0, hi = 0;
  bool empty = false;
  if (op == 0) {
    empty = !a->n || !b->n || std::max(e[0], e[2]) > std::min(e[1], e[3]);
    lo = std::max(e[0], e[2]);
    hi = std::min(e[1], e[3]);
  } else if (!a->n && !b->n) {
    empty = true;
  } else {
    lo = !a->n ? e[2] : (!b->n ? e[0] : std::min(e[0], e[2]));
    hi = !a->n ? e[3] : (!b->n ? e[1] : std::max(e[1], e[3]));
  }
  const uint64_t nbits = empty ? 0 : hi - lo + 1;
  if (!empty && nbits == 0) return MS_E_INVALID;  // the whole 2^64 range
  const uint64_t NS = (nbits + kSegRows - 1) / kSegRows, n_words = NS * kSegWords;
  Scratch s2(ctx);
  const uint64_t o_ba = s2.add(4 * n_words, true);
  const uint64_t o_bb = s2.add(4 * n_words, true);
  const uint64_t o_fa = s2.add(16 * ((a->n + kChunk - 1) / kChunk + 1), false);
  const uint64_t o_fb = s2.add(16 * ((b->n + kChunk - 1) / kChunk + 1), false);
  const uint64_t o_seg = s2.add(4 * (NS + 1), false);
  if (!s2.commit()) return MS_E_NOMEM;
  uint32_t* ba = s2.at<uint32_t>(o_ba);
  if (!empty) {
    MS_TRY_CUDA(launch_pos_bitmap(va, lo, nbits, ba, s2.at<uint64_t>(o_fa), err, ctx.s));
    MS_TRY_CUDA(launch_pos_bitmap(vb, lo, nbits, s2.at<uint32_t>(o_bb), s2.at<uint64_t>(o_fb), err, ctx.s));
    MS_TRY_CUDA(launch_bits_combine(ba, s2.at<uint32_t>(o_bb), n_words, op, ctx.s));
    MS_TRY_CUDA(launch_seg_info(ba, NS, s2.at<uint32_t>(o_seg), ctx.s));
  }
  return positions_from_mask(ctx, ba, s2.at<uint32_t>(o_seg), NS, nbits, lo, out_fmt, err, out);
}

ms_status ms_intersect(const ms_ctx* ctx, const ms_column* a, const ms_column* b, ms_fmt out_fmt, ms_column* out) {
  return set_op(ctx, a, b, 0, out_fmt, out);
}
ms_status ms_merge(const ms_ctx* ctx, const ms_column* a, const ms_column* b, ms_fmt out_fmt, ms_column* out) {
  return set_op(ctx, a, b, 1, out_fmt, out);
}

static uint64_t pow2_at_least(uint64_t x) {
  uint64_t c = 1024;
  while (c < x) c <<= 1;
  return c;
}

ms_status ms_group(const ms_ctx* ctx_, const ms_column* keys, const ms_column* prev_ids, uint64_t max_groups,
                   ms_fmt ids_fmt, ms_fmt extents_fmt, ms_column* out_ids, ms_column* out_extents) {
  if (!out_ids || !out_extents) return MS_E_INVALID;
  std::memset(out_ids, 0, sizeof(*out_ids));
  std::memset(out_extents, 0, sizeof(*out_extents));
  MS_TRY(check_col(keys));
  if (prev_ids) MS_TRY(check_col(prev_ids));
  MS_TRY(check_fmt(ids_fmt));
  MS_TRY(check_fmt(extents_fmt));
  if (prev_ids && prev_ids->n != keys->n) return MS_E_INVALID;  // LengthMismatch
  Ctx ctx(ctx_);
  const uint64_t n = keys->n;
  const uint64_t groups = max_groups && max_groups < n ? max_groups : n;
  const uint64_t cap = pow2_at_least(2 * (groups ? groups : 1));
  const uint64_t NS = (n + kSegRows - 1) / kSegRows, n_words = NS * kSegWords;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_state = sc.add(4 * cap, true);
  const uint64_t o_key = sc.add(8 * cap, false);
  const uint64_t o_key2 = sc.add(prev_ids ? 8 * cap : 8, false);
  const uint64_t o_first = sc.add(8 * cap, false);
  const uint64_t o_bits = sc.add(4 * n_words, true);
  const uint64_t o_cnt = sc.add(4 * (NS + 1), false);
  const uint64_t o_off = sc.add(8 * (NS + 2), false);
  const uint64_t o_st = sc.add(8 * ((NS + kChunk - 1) / kChunk + 1), true);
  const uint64_t o_tk = sc.add(8, true);
  const uint64_t o_seg = sc.add(4 * (NS + 1), false);
  const uint64_t o_ids = sc.add(8 * n, false);
  RlePrep rk, rpv;
  plan_rle(sc, keys, rk);
  plan_rle(sc, prev_ids, rpv);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView vk = view_of(keys), vp{};
  MS_TRY_CUDA(run_rle(sc, keys, rk, vk, err));
  if (prev_ids) {
    vp = view_of(prev_ids);
    MS_TRY_CUDA(run_rle(sc, prev_ids, rpv, vp, err));
  }
  uint32_t* state = sc.at<uint32_t>(o_state);
  uint64_t* key = sc.at<uint64_t>(o_key);
  uint64_t* key2 = prev_ids ? sc.at<uint64_t>(o_key2) : nullptr;
  auto* first = sc.at<unsigned long long>(o_first);
  uint32_t* bits = sc.at<uint32_t>(o_bits);
  MS_TRY_CUDA(cudaMemsetAsync(first, 0xff, 8 * cap, ctx.s));
  if (n) {
    MS_TRY_CUDA(launch_group(vk, vp, state, key, key2, cap, first, bits, err, ctx.s));
    MS_TRY_CUDA(launch_seg_count(bits, NS, sc.at<uint32_t>(o_cnt), ctx.s));
    MS_TRY_CUDA(launch_count_scan(sc.at<uint32_t>(o_cnt), NS, sc.at<uint64_t>(o_off), sc.at<uint64_t>(o_st),
                                  sc.at<uint32_t>(o_tk), ctx.s));
    MS_TRY_CUDA(launch_group_ids(vk, vp, state, key, key2, cap, first, bits, sc.at<uint64_t>(o_off),
                                 sc.at<uint64_t>(o_ids), err, ctx.s));
    MS_TRY_CUDA(launch_seg_info(bits, NS, sc.at<uint32_t>(o_seg), ctx.s));
  }
  // extents: the first row of every group = the set bits of the mask (sync, errors read here)
  MS_TRY(positions_from_mask(ctx, bits, sc.at<uint32_t>(o_seg), NS, n, 0, extents_fmt, err, out_extents));
  const ms_status st = ms_compress(ctx_, sc.at<uint64_t>(o_ids), n, ids_fmt, out_ids);
  if (st != MS_OK) release(ctx, out_extents);
  return st;
}

ms_status ms_join(const ms_ctx* ctx_, const ms_column* left, const ms_column* right, ms_fmt left_fmt,
                  ms_fmt right_fmt, ms_column* out_left, ms_column* out_right) {
  if (!out_left || !out_right) return MS_E_INVALID;
  std::memset(out_left, 0, sizeof(*out_left));
  std::memset(out_right, 0, sizeof(*out_right));
  MS_TRY(check_col(left));
  MS_TRY(check_col(right));
  MS_TRY(check_fmt(left_fmt));
  MS_TRY(check_fmt(right_fmt));
  Ctx ctx(ctx_);
  const bool build_right = right->n <= left->n;  // build side = the smaller column
  const ms_column* build = build_right ? right : left;
  const ms_column* probe = build_right ? left : right;
  const uint64_t cap = pow2_at_least(2 * (build->n ? build->n : 1));
  const uint64_t T = (probe->n + kChunk - 1) / kChunk;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_state = sc.add(4 * cap, true);
  const uint64_t o_key = sc.add(8 * cap, false);
  const uint64_t o_cnt = sc.add(4 * cap, true);
  const uint64_t o_off = sc.add(8 * (cap + 2), false);
  const uint64_t o_fill = sc.add(4 * cap, true);
  const uint64_t o_rows = sc.add(8 * build->n, false);
  const uint64_t o_st1 = sc.add(8 * ((cap + kChunk - 1) / kChunk + 1), true);
  const uint64_t o_tk1 = sc.add(8, true);
  const uint64_t o_tc = sc.add(4 * (T + 1), false);
  const uint64_t o_toff = sc.add(8 * (T + 2), false);
  const uint64_t o_st2 = sc.add(8 * ((T + kChunk - 1) / kChunk + 1), true);
  const uint64_t o_tk2 = sc.add(8, true);
  RlePrep rb, rp;
  plan_rle(sc, build, rb);
  plan_rle(sc, probe, rp);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView vb = view_of(build), vpr = view_of(probe);
  MS_TRY_CUDA(run_rle(sc, build, rb, vb, err));
  MS_TRY_CUDA(run_rle(sc, probe, rp, vpr, err));
  uint32_t* state = sc.at<uint32_t>(o_state);
  uint64_t* key = sc.at<uint64_t>(o_key);
  uint32_t* cnt = sc.at<uint32_t>(o_cnt);
  uint64_t* off = sc.at<uint64_t>(o_off);
  uint64_t* toff = sc.at<uint64_t>(o_toff);
  uint64_t total = 0;
  if (build->n && probe->n) {
    MS_TRY_CUDA(launch_join_build(vb, state, key, cap, cnt, err, ctx.s));
    MS_TRY_CUDA(launch_count_scan(cnt, cap, off, sc.at<uint64_t>(o_st1), sc.at<uint32_t>(o_tk1), ctx.s));
    MS_TRY_CUDA(launch_join_place(vb, state, key, cap, cnt, off, sc.at<uint32_t>(o_fill), sc.at<uint64_t>(o_rows),
                                  err, ctx.s));
    MS_TRY_CUDA(launch_join_probe(vpr, state, key, cap, cnt, off, sc.at<uint64_t>(o_rows), sc.at<uint32_t>(o_tc),
                                  toff, nullptr, nullptr, false, err, ctx.s));
    MS_TRY_CUDA(launch_count_scan(sc.at<uint32_t>(o_tc), T, toff, sc.at<uint64_t>(o_st2), sc.at<uint32_t>(o_tk2),
                                  ctx.s));
    uint64_t h[2] = {0, 0};
    MS_TRY_CUDA(cudaMemcpyAsync(&h[1], toff + T, 8, cudaMemcpyDeviceToHost, ctx.s));
    MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), h, 1));  // sizing sync: the number of pairs
    MS_TRY(status_from_bits((uint32_t)h[0]));
    total = h[1];
  }
  uint64_t* pairs = (uint64_t*)ctx.alloc(16 * (total ? total : 1));
  if (!pairs) return MS_E_NOMEM;
  uint64_t *pp = pairs, *pb = pairs + total;
  ms_status st = MS_OK;
  if (total) st = cuda_status(launch_join_probe(vpr, state, key, cap, cnt, off, sc.at<uint64_t>(o_rows),
                                                sc.at<uint32_t>(o_tc), toff, pp, pb, true, err, ctx.s));
  if (st == MS_OK) st = ms_compress(ctx_, build_right ? pp : pb, total, left_fmt, out_left);
  if (st == MS_OK) {
    st = ms_compress(ctx_, build_right ? pb : pp, total, right_fmt, out_right);
    if (st != MS_OK) release(ctx, out_left);
  }
  ctx.free(pairs);
  return st;
}

ms_status ms_calc(const ms_ctx* ctx_, int32_t op, const ms_column* a, const ms_column* b, ms_fmt out_fmt,
                  ms_column* out) {
  if (!out) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_col(a));
  MS_TRY(check_col(b));
  MS_TRY(check_fmt(out_fmt));
  if (a->n != b->n) return MS_E_INVALID;  // LengthMismatch
  if (op != MS_ADD && op != MS_SUB && op != MS_MUL) return MS_E_INVALID;
  Ctx ctx(ctx_);
  const uint64_t n = a->n;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_out = sc.add(8 * n, false);
  RlePrep ra, rb;
  plan_rle(sc, a, ra);
  plan_rle(sc, b, rb);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  ColView va = view_of(a), vb = view_of(b);
  MS_TRY_CUDA(run_rle(sc, a, ra, va, err));
  MS_TRY_CUDA(run_rle(sc, b, rb, vb, err));
  MS_TRY_CUDA(launch_calc(va, vb, op, sc.at<uint64_t>(o_out), ctx.s));
  uint64_t h = 0;
  MS_TRY(readback(ctx, sc.at<uint64_t>(o_meta), &h, 1));
  MS_TRY(status_from_bits((uint32_t)h));
  return ms_compress(ctx_, sc.at<uint64_t>(o_out), n, out_fmt, out);
}

ms_status ms_semijoin(const ms_ctx* ctx_, const ms_column* keys, const ms_column* positions, uint64_t row_offset,
                      const uint64_t* bitmap, uint64_t bitmap_bits, ms_fmt out_fmt, ms_column* out) {
  if (!out) return MS_E_INVALID;
  std::memset(out, 0, sizeof(*out));
  MS_TRY(check_col(keys));
  MS_TRY(check_col(positions));
  MS_TRY(check_fmt(out_fmt));
  if (bitmap_bits && !bitmap) return MS_E_INVALID;
  const int32_t pf = positions->fmt.format, kf = keys->fmt.format;
  const bool fused = (pf == MS_UNCOMPR || pf == MS_STATIC_BP || pf == MS_DYN_BP || pf == MS_FOR_BP ||
                      (pf == MS_DELTA_BP && positions->fmt.block_size == (uint32_t)kSegRows)) &&
                     (kf == MS_UNCOMPR || kf == MS_STATIC_BP || kf == MS_DYN_BP || kf == MS_FOR_BP);
  Ctx ctx(ctx_);
  const uint64_t n1 = positions->n;
  if (!fused) {  // the operator-at-a-time chain (D-16): project, select IN_BITMAP, project
    ms_column kp, idx;
    MS_TRY(ms_project(ctx_, keys, positions, row_offset, ms_fmt{MS_UNCOMPR, 0, 0, 0}, &kp));
    ms_pred p{MS_IN_BITMAP, 0, 0, 0, bitmap, bitmap_bits};
    ms_status st = ms_select(ctx_, &kp, &p, 0, ms_fmt{MS_DELTA_BP, 0, 512, 0}, &idx);
    release(ctx, &kp);
    if (st != MS_OK) return st;
    st = ms_project(ctx_, positions, &idx, 0, out_fmt, out);
    release(ctx, &idx);
    return st;
  }
  // fused (K7, row space): the surviving positions as a mask over the keys' rows,
  // turned into pos2 by the select output layer
  (void)n1;
  const uint64_t nk = keys->n;
  const uint64_t NS = (nk + kSegRows - 1) / kSegRows;
  Scratch sc(ctx);
  const uint64_t o_meta = sc.add(64, true);
  const uint64_t o_bits = sc.add(4 * NS * kSegWords, true);
  const uint64_t o_seg = sc.add(4 * (NS + 1), false);
  if (!sc.commit()) return MS_E_NOMEM;
  uint32_t* err = sc.at<uint32_t>(o_meta);
  MS_TRY_CUDA(launch_semi_rows(view_of(positions), view_of(keys), row_offset, bitmap, bitmap_bits,
                               sc.at<uint32_t>(o_bits), err, ctx.s));
  if (NS) MS_TRY_CUDA(launch_seg_info(sc.at<uint32_t>(o_bits), NS, sc.at<uint32_t>(o_seg), ctx.s));
  return positions_from_mask(ctx, sc.at<uint32_t>(o_bits), sc.at<uint32_t>(o_seg), NS, nk, row_offset, out_fmt, err,
                             out);
}

ms_status ms_check_errors(const ms_ctx* ctx_) {
  Ctx ctx(ctx_);
  uint32_t h = 0;
  uint32_t* p = sticky_err();
  MS_TRY_CUDA(cudaMemcpyAsync(&h, p, 4, cudaMemcpyDeviceToHost, ctx.s));
  MS_TRY_CUDA(cudaMemsetAsync(p, 0, 4, ctx.s));
  MS_TRY_CUDA(cudaStreamSynchronize(ctx.s));
  MS_TRY_CUDA(cudaGetLastError());
  return status_from_bits(h);
}

}  // extern "C"
