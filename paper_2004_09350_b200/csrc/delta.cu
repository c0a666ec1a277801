// delta.cu — DELTA_BP decoding into uncompressed values or a static-BP stream in
// one pass per block of codes (decompress / morph DELTA_BP -> STATIC_BP, P:362-389;
// the paper's "direct morphing" without an intermediate column). DELTA decoding
// needs the in-block inclusive prefix of the deltas (D-6); the generic engine does
// it with a CTA-wide scan per 2048-row tile and ~75 instructions per row. Here a
// warp owns a 2048-row tile and lane j the 64 consecutive rows [64j, 64j + 64)
// (inside one block, since 64 | B): the lane sums its 64 codes (read from a
// contiguous, 8-byte aligned 64w-bit range of the payload), a segmented warp scan
// over the lanes of each block gives every lane its prefix, and a second pass over
// the same codes emits the values — as a running maximum (the auto static width),
// as u64 values, or packed at the static width — through a shared-memory tile that
// is stored with coalesced writes.
#include "common.cuh"
#include "grid.cuh"
#include "launch.h"

namespace ms {

namespace {

constexpr int kDWarps = 4;               // warps per CTA
constexpr int kDRows = 2048;             // rows per warp tile
constexpr int kDLane = kDRows / 32;      // rows per lane

enum : int { DM_MAX = 0, DM_U64 = 1, DM_STATIC = 2 };

// Streaming reader of w-bit codes from an 8-byte aligned LSB-first range (D-1) of
// the shared-memory copy of a tile's payload.
struct CodeReader {
  const uint64_t* p;
  uint64_t win;   // unread bits of the current word, low-aligned
  uint32_t have;  // bits in win
  uint32_t w;
  uint64_t mask;
  __device__ __forceinline__ void init(const uint64_t* q, uint32_t width) {
    p = q;
    w = width;
    mask = low_mask(width);
    win = 0;
    have = 0;
  }
  __device__ __forceinline__ uint64_t next() {
    if (w == 0) return 0;
    if (have >= w) {
      const uint64_t c = win & mask;
      win = w == 64 ? 0 : win >> w;
      have -= w;
      return c;
    }
    const uint64_t x = *p++;  // (shared memory: the staged tile)
    const uint64_t c = (win | (have ? x << have : x)) & mask;  // the low `have` bits from win
    const uint32_t used = w - have;                             // bits taken from x
    win = used == 64 ? 0 : x >> used;
    have = 64 - used;
    return c;
  }
};

// The lane's 64 codes at a compile-time width W <= 32 (two halves of 32 codes = W
// u32 words each; shifts and word indices are constants): f(code) in order.
template <int W, class F>
__device__ __forceinline__ void lane_codes(const uint32_t* __restrict__ p, F&& f) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    uint32_t r[W + 1];
#pragma unroll
    for (int k = 0; k < W; ++k) r[k] = p[h * W + k];
    r[W] = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int bit = i * W, q = bit >> 5, sh = bit & 31;
      uint32_t c = W == 0 ? 0u : ((sh + W <= 32) ? (r[q] >> sh) : __funnelshift_r(r[q], r[q + 1], sh));
      if (W < 32) c &= (W == 0 ? 0u : (0xffffffffu >> (32 - (W == 0 ? 1 : W))));
      f((uint64_t)c);
    }
  }
}

template <class F>
__device__ __forceinline__ bool lane_codes_dispatch(uint32_t w, const uint32_t* p, F&& f) {
  switch (w) {
#define MS_LC(W) \
  case W:        \
    lane_codes<W>(p, f); \
    return true;
    MS_LC(0) MS_LC(1) MS_LC(2) MS_LC(3) MS_LC(4) MS_LC(5) MS_LC(6) MS_LC(7) MS_LC(8) MS_LC(9) MS_LC(10)
    MS_LC(11) MS_LC(12) MS_LC(13) MS_LC(14) MS_LC(15) MS_LC(16) MS_LC(17) MS_LC(18) MS_LC(19) MS_LC(20)
    MS_LC(21) MS_LC(22) MS_LC(23) MS_LC(24) MS_LC(25) MS_LC(26) MS_LC(27) MS_LC(28) MS_LC(29) MS_LC(30)
    MS_LC(31) MS_LC(32)
#undef MS_LC
    default:
      return false;  // wider: the runtime-width reader
  }
}

template <int MODE>
__global__ void __launch_bounds__(kDWarps * 32) delta_decode_kernel(ColView c, uint64_t main_rows, uint32_t ws,
                                                                    uint32_t stage_words, uint32_t out_words,
                                                                    uint64_t* __restrict__ out,
                                                                    unsigned long long* max_out, uint32_t* err) {
  extern __shared__ __align__(16) uint64_t dd_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t* stg = dd_sm + (size_t)wid * (stage_words + out_words);  // the tile's payload words
  uint64_t* tile = stg + stage_words;                               // the tile's output
  const uint32_t gl = c.B / kDLane;  // lanes per block (B >= 128: 2..32)
  const uint64_t n_tiles = (main_rows + kDRows - 1) / kDRows;
  const uint64_t wpc = c.B / 64;     // payload words per unit of cw
  uint64_t mx = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * kDWarps + wid; t < n_tiles; t += (uint64_t)gridDim.x * kDWarps) {
    const uint64_t row0 = t * kDRows;
    const uint64_t r0 = row0 + (uint64_t)lane * kDLane;  // the lane's first row
    const bool active = r0 < main_rows;
    uint32_t w = 0, cw0 = 0, cw1 = 0;
    uint64_t base = 0;
    if (active) {
      const uint64_t b = r0 >> c.log2B;
      cw0 = __ldg(c.cw + b);
      cw1 = __ldg(c.cw + b + 1);
      w = cw1 - cw0;
      if (w > 64) {
        atomicOr(err, err_bit(MS_E_CORRUPT));
        w = 0;
      }
      base = __ldg(c.ref + b);
    }
    // stage the tile's payload (contiguous over its blocks) with independent loads
    const uint64_t t_lo = (uint64_t)__shfl_sync(kFull, cw0, 0) * wpc;
    const uint64_t t_hi = (uint64_t)__reduce_max_sync(kFull, active ? cw1 : 0u) * wpc;
    const uint32_t n_tw = (uint32_t)(t_hi - t_lo);
    if (n_tw > stage_words) {  // a block wider than the max_width hint: never overrun the stage
      if (lane == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
      continue;
    }
    for (uint32_t i = lane; i < n_tw; i += 32) stg[i] = __ldg(c.payload + t_lo + i);
    __syncwarp();
    CodeReader rd{};
    if (active) {
      const uint64_t bit = (uint64_t)cw0 * c.B + (r0 & (c.B - 1)) * w;  // a multiple of 64
      rd.init(stg + ((bit >> 6) - t_lo), w);
    }
    // pass 1: the lane's sum of codes; segmented exclusive scan over the lanes of its block
    const uint32_t* p32 = active ? reinterpret_cast<const uint32_t*>(rd.p) : nullptr;
    uint64_t sum = 0;
    if (active && !lane_codes_dispatch(w, p32, [&](uint64_t c) { sum += c; })) {
      CodeReader r1 = rd;
      for (int q = 0; q < kDLane; ++q) sum += r1.next();
    }
    uint64_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, inc, o, gl);
      if ((lane & (gl - 1)) >= (uint32_t)o) inc += y;
    }
    uint64_t v = base + (inc - sum);
    const uint32_t rows = (uint32_t)min((uint64_t)kDRows, main_rows - row0);
    // pass 2: the values
    if (MODE == DM_MAX) {
      auto f = [&](uint64_t c) {
        v += c;
        mx = v > mx ? v : mx;
      };
      if (active && !lane_codes_dispatch(w, p32, f))
        for (int q = 0; q < kDLane; ++q) f(rd.next());
    } else if (MODE == DM_U64) {
      uint32_t q = 0;
      auto f = [&](uint64_t c) {
        v += c;
        tile[lane * kDLane + q++] = v;
      };
      if (active && !lane_codes_dispatch(w, p32, f))
        for (int k = 0; k < kDLane; ++k) f(rd.next());
      __syncwarp();
      uint64_t* dst = out + row0;  // (caller memory: 8-byte stores, coalesced across the warp)
      for (uint32_t i = lane; i < rows; i += 32) dst[i] = tile[i];
    } else {  // DM_STATIC: the lane's 64 values at ws bits = ws u64 words at word (r0 * ws) / 64
      if (active) {
        uint64_t acc = 0;
        uint32_t nb = 0, wi = 0;
        uint64_t* my = tile + (size_t)lane * ws;
        const uint64_t lim = ws >= 64 ? ~0ull : (1ull << ws) - 1;
        bool over = false;
        auto f = [&](uint64_t c) {
          v += c;
          over |= v > lim;
          acc |= v << nb;
          nb += ws;
          if (nb >= 64) {
            my[wi++] = acc;
            nb -= 64;
            acc = nb ? v >> (ws - nb) : 0ull;
          }
        };
        if (!lane_codes_dispatch(w, p32, f))
          for (int q = 0; q < kDLane; ++q) f(rd.next());
        if (over) atomicOr(err, err_bit(MS_E_WIDTH_OVERFLOW));
      }
      __syncwarp();
      const uint32_t nwords = rows / kDLane * ws;  // whole lanes only (64 | rows)
      uint64_t* dst = out + (row0 * ws >> 6);
      for (uint32_t i = lane; i < nwords; i += 32) dst[i] = tile[i];
    }
    __syncwarp();
  }
  if (MODE == DM_MAX) {
    mx = warp_max(mx);
    if (lane == 0 && mx) atomicMax(max_out, (unsigned long long)mx);
  }
}

// the remainder rows (raw, D-7): max / copy / pack starting at the word of row main_rows
template <int MODE>
__global__ void delta_rem_kernel(ColView c, uint64_t main_rows, uint32_t ws, uint64_t* out,
                                 unsigned long long* max_out, uint32_t* err) {
  const uint64_t nrem = c.n - main_rows;
  if (MODE == DM_STATIC) {  // one thread: < B values into whole words (main_rows * ws is a multiple of 64)
    if (threadIdx.x != 0) return;
    uint64_t acc = 0, *dst = out + (main_rows * ws >> 6);
    uint32_t nb = 0;
    const uint64_t lim = ws >= 64 ? ~0ull : (1ull << ws) - 1;
    for (uint64_t i = 0; i < nrem; ++i) {
      const uint64_t v = __ldg(c.rem + i);
      if (v > lim) atomicOr(err, err_bit(MS_E_WIDTH_OVERFLOW));
      acc |= v << nb;
      nb += ws;
      if (nb >= 64) {
        *dst++ = acc;
        nb -= 64;
        acc = nb ? v >> (ws - nb) : 0ull;
      }
    }
    if (nb) *dst = acc;
    return;
  }
  uint64_t mx = 0;
  for (uint64_t i = threadIdx.x; i < nrem; i += blockDim.x) {
    const uint64_t v = __ldg(c.rem + i);
    if (MODE == DM_U64) out[main_rows + i] = v;
    mx = v > mx ? v : mx;
  }
  if (MODE == DM_MAX) {
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_out, (unsigned long long)mx);
  }
}

template <int MODE>
cudaError_t run(const ColView& c, uint32_t ws, uint64_t* out, unsigned long long* max_out, uint32_t* err,
                cudaStream_t s) {
  const uint64_t main_rows = c.nb << c.log2B;
  if (main_rows) {
    auto k = delta_decode_kernel<MODE>;
    // per warp: the tile's payload at the widest block (max_width hint; 64 if unknown) + its output
    const uint32_t mw = c.maxw >= 1 && c.maxw <= 64 ? c.maxw : 64u;
    const uint32_t stage_words = kDRows * mw / 64 + 2;
    const uint32_t out_words = MODE == DM_MAX ? 0u : (MODE == DM_U64 ? (uint32_t)kDRows : 32u * ws);
    const size_t smem = (size_t)kDWarps * (stage_words + out_words) * 8;
    set_smem_once((const void*)k, smem);
    int per_sm = 0;
    per_sm = occupancy_cached((const void*)k, kDWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    const uint64_t need = ((main_rows + kDRows - 1) / kDRows + kDWarps - 1) / kDWarps;
    if (need < grid) grid = need;
    ProfScope prof_(MODE == DM_MAX ? "delta_max" : (MODE == DM_U64 ? "delta_decode" : "delta_to_static"), s);
    k<<<(int)grid, kDWarps * 32, smem, s>>>(c, main_rows, ws, stage_words, out_words, out, max_out, err);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (c.n > main_rows) {
    ProfScope prof_("delta_rem", s);
    delta_rem_kernel<MODE><<<1, 256, 0, s>>>(c, main_rows, ws, out, max_out, err);
  }
  return cudaGetLastError();
}

}  // namespace

// Header bounds of a DELTA_BP column's maximum (for the auto width of a morph into
// STATIC_BP): every block's first value ref[b] is a value (lower bound); its
// values are at most ref[b] + (B - 1)(2^w_b - 1) unless that sum passes 2^64
// (the differences wrap: no bound, 2^64 - 1); the remainder is exact. When
// ebw(lower) == ebw(upper) the width is known without decoding a block.
__global__ void delta_bounds_kernel(ColView c, unsigned long long* lohi) {
  uint64_t lo = 0, hi = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < c.nb; b += stride) {
    const uint64_t r = __ldg(c.ref + b);
    const uint32_t w = __ldg(c.cw + b + 1) - __ldg(c.cw + b);
    uint64_t u = ~0ull;
    if (w < 64) {
      const uint64_t step = (1ull << w) - 1;
      const uint64_t m = (uint64_t)(c.B - 1);
      if (step == 0 || m <= ~0ull / step) {
        const uint64_t span = m * step;
        if (r <= ~0ull - span) u = r + span;
      }
    }
    lo = r > lo ? r : lo;
    hi = u > hi ? u : hi;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.nrem; i += stride) {
    const uint64_t v = __ldg(c.rem + i);
    lo = v > lo ? v : lo;
    hi = v > hi ? v : hi;
  }
  lo = warp_max(lo);
  hi = warp_max(hi);
  if ((threadIdx.x & 31) == 0) {
    if (lo) atomicMax(lohi, (unsigned long long)lo);
    if (hi) atomicMax(lohi + 1, (unsigned long long)hi);
  }
}

cudaError_t launch_delta_bounds(const ColView& c, unsigned long long* lohi, cudaStream_t s) {
  uint64_t grid = (c.nb + c.nrem + 255) / 256;
  if (grid > (uint64_t)num_sms() * 8) grid = num_sms() * 8;
  if (!grid) grid = 1;
  ProfScope prof_("delta_bounds", s);
  delta_bounds_kernel<<<(int)grid, 256, 0, s>>>(c, lohi);
  return cudaGetLastError();
}

bool delta_direct_supported(const ColView& c) { return c.format == MS_DELTA_BP && c.B >= 128; }

cudaError_t launch_delta_decode(const ColView& c, uint64_t* out, uint32_t* err, cudaStream_t s) {
  return run<DM_U64>(c, 64, out, nullptr, err, s);
}
cudaError_t launch_delta_max(const ColView& c, unsigned long long* max_out, uint32_t* err, cudaStream_t s) {
  return run<DM_MAX>(c, 0, nullptr, max_out, err, s);
}
cudaError_t launch_delta_to_static(const ColView& c, uint32_t ws, uint64_t* payload, uint32_t* err, cudaStream_t s) {
  return run<DM_STATIC>(c, ws, payload, nullptr, err, s);
}

}  // namespace ms
