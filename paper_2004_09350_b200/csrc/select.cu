// select.cu — select cores (fast compile-time-width core, generic core) and the
// whole-column sum that reuses the fast core (select_fast.cuh).
#include "common.cuh"
#include "engine.cuh"
#include "grid.cuh"
#include "select_fast.cuh"
#include "selstream.cuh"
#include "launch.h"

namespace ms {

// ------------------------------------------------------- select: predicate
// Header-only block decisions (the specialized-operator shortcut of P:352,
// SURVEY.md §8(f) #1): a block whose values are known from its header alone to
// lie in [L, H] needs no decoding when the predicate is constant on [L, H].
enum : uint32_t { kDecode = 0, kNone = 1, kAll = 2 };
__device__ __forceinline__ uint32_t range_decision(uint64_t lo, uint64_t span, uint32_t neg, uint64_t L, uint64_t H) {
  const uint64_t xl = L - lo, xh = H - lo;  // keep(v) <=> (v - lo) <= span, != neg
  uint32_t d = kDecode;
  if (xl <= xh) {  // [L, H] maps to [xl, xh] without wrapping
    if (xh <= span) d = kAll;
    else if (xl > span) d = kNone;
  } else if (span == ~0ull) {
    d = kAll;
  }
  if (d != kDecode && neg) d = kAll + kNone - d;
  return d;
}

struct RangePred {
  uint64_t lo, span;
  uint32_t neg;
  __device__ __forceinline__ bool operator()(uint64_t v) const { return ((v - lo) <= span) != (neg != 0); }
  __device__ __forceinline__ uint32_t decide(uint64_t L, uint64_t H) const { return range_decision(lo, span, neg, L, H); }
};
struct BitmapPred {
  const uint64_t* bm;
  uint64_t bits;
  __device__ __forceinline__ bool operator()(uint64_t v) const {
    return v < bits && ((__ldg(bm + (v >> 6)) >> (v & 63)) & 1ull);
  }
  __device__ __forceinline__ uint32_t decide(uint64_t, uint64_t) const { return kDecode; }
};

// Header-only decision for a whole 2048-row tile of a block format (all blocks of
// the tile in the main part): the tile is decided when every block's value range,
// known from its header alone, gets the same constant verdict. DYN_BP: [0, 2^w);
// FOR_BP: [ref, ref + 2^w); DELTA_BP: [base, base + (B - 1)(2^w - 1)] (deltas are
// unsigned; valid when that bound does not overflow).
template <class Pred>
__device__ __forceinline__ uint32_t tile_decision(const ColView& c, const Pred& pred, uint64_t r0, uint32_t cnt) {
  if (c.format != MS_DYN_BP && c.format != MS_FOR_BP && c.format != MS_DELTA_BP) return kDecode;
  if (cnt != (uint32_t)kChunk || r0 + kChunk > (c.nb << c.log2B)) return kDecode;
  uint32_t verdict = kDecode;
  for (uint64_t b = r0 >> c.log2B; b < (r0 + kChunk) >> c.log2B; ++b) {
    const uint32_t w = __ldg(c.cw + b + 1) - __ldg(c.cw + b);
    if (w > 64) return kDecode;
    const uint64_t M1 = w >= 64 ? ~0ull : ((1ull << w) - 1);
    uint64_t L = 0, H = M1;
    if (c.format == MS_FOR_BP) {
      L = __ldg(c.ref + b);
      H = L + M1;
      if (H < L) return kDecode;
    } else if (c.format == MS_DELTA_BP) {
      L = __ldg(c.ref + b);
      const uint64_t steps = (uint64_t)(c.B - 1);
      if (M1 && __umul64hi(M1, steps)) return kDecode;
      H = L + M1 * steps;
      if (H < L) return kDecode;
    }
    const uint32_t d = pred.decide(L, H);
    if (d == kDecode || (verdict != kDecode && d != verdict)) return kDecode;
    verdict = d;
  }
  return verdict;
}

// Generic select core for formats without a fast path (DELTA_BP, RLE, block
// sizes < 512): per tile of 2048 rows, decode into shared memory, evaluate the
// predicate, ballot -> one 32-bit mask word per 32 rows; per 512-row segment
// write count | (1-based last matching row << 16). Only segments in [s0, s1)
// are written (the fast kernel covers the others).
template <class Pred>
__global__ void __launch_bounds__(kThreads) select_generic_kernel(ColView c, Pred pred, uint32_t* bits,
                                                                  uint32_t* seg_info, uint64_t s0, uint64_t s1,
                                                                  const uint32_t* list, const uint32_t* n_list) {
  __shared__ EngineSmem sm;
  __shared__ uint32_t words[kChunk / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t t0 = (s0 * kSegRows) / kChunk;
  const uint64_t t1 = (s1 * kSegRows + kChunk - 1) / kChunk;
  __shared__ uint32_t s_dec;
  const uint64_t n_iter = list ? *n_list : t1 - t0;  // the undecided tiles of tile_prune_kernel, or all
  for (uint64_t it = blockIdx.x; it < n_iter; it += gridDim.x) {
    const uint64_t t = list ? list[it] : t0 + it;
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, c.n - r0);
    if (threadIdx.x == 0) s_dec = tile_decision(c, pred, r0, cnt);
    __syncthreads();
    const uint32_t dec = s_dec;
    constexpr int kWordsPerWarp = kChunk / 32 / (kThreads / 32);
    if (dec != kDecode) {  // decided from the headers: no decoding
      if (lane < kWordsPerWarp) words[wid * kWordsPerWarp + lane] = dec == kAll ? 0xffffffffu : 0u;
    } else {
      load_rows(c, r0, cnt, sm);
#pragma unroll
      for (int q = 0; q < kWordsPerWarp; ++q) {
        const uint32_t m = wid * kWordsPerWarp + q;
        const uint32_t i = m * 32 + lane;
        const bool p = i < cnt && pred(sm.vals[i]);
        const uint32_t word = __ballot_sync(kFull, p);
        if (lane == 0) words[m] = word;
      }
    }
    __syncthreads();
    constexpr int kSegsPerTile = kChunk / kSegRows;
    if (wid < kSegsPerTile) {
      const uint64_t sg = t * kSegsPerTile + wid;
      if (sg >= s0 && sg < s1) {
        const uint32_t my = lane < kSegWords ? words[wid * kSegWords + lane] : 0u;
        if (lane < kSegWords) bits[sg * kSegWords + lane] = my;
        const uint32_t cnt_ = (uint32_t)warp_sum(__popc(my));
        const uint32_t last = (uint32_t)warp_max(my ? lane * 32 + 32 - __clz(my) : 0u);
        if (lane == 0) seg_info[sg] = cnt_ | (last << 16);
      }
    }
    __syncthreads();
  }
}

__global__ void max_width_kernel(const uint32_t* cw, uint64_t nb, uint32_t* out) {
  uint32_t m = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += stride)
    m = max(m, cw[b + 1] - cw[b]);
  m = __reduce_max_sync(kFull, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

cudaError_t launch_max_width(const uint32_t* cw, uint64_t nb, uint32_t* out, cudaStream_t s) {
  if (!nb) return cudaSuccess;
  uint64_t grid = (nb + 255) / 256;
  if (grid > (uint64_t)num_sms() * 8) grid = num_sms() * 8;
  ProfScope prof_("max_width", s);
  max_width_kernel<<<(int)grid, 256, 0, s>>>(cw, nb, out);
  return cudaGetLastError();
}

// Header-only pass over the tiles of a block-format column (one thread per tile):
// a decided tile gets its 64 mask words and 4 segment counts written directly; the
// others are listed for select_generic_kernel. At BJ.c3 (sorted values, a value
// range covering ~2% of the column) all but a handful of tiles are decided here.
__global__ void __launch_bounds__(256) tile_prune_kernel(ColView c, RangePred pred, uint32_t* bits,
                                                         uint32_t* seg_info, uint64_t s0, uint64_t s1,
                                                         uint32_t* list, uint32_t* n_list) {
  const uint64_t t0 = (s0 * kSegRows) / kChunk;
  const uint64_t t1 = (s1 * kSegRows + kChunk - 1) / kChunk;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = t0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += stride) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, c.n - r0);
    const uint32_t dec = tile_decision(c, pred, r0, cnt);
    if (dec == kDecode) {
      list[atomicAdd(n_list, 1u)] = (uint32_t)t;
      continue;
    }
    const uint32_t word = dec == kAll ? 0xffffffffu : 0u;
    const uint32_t info = dec == kAll ? (uint32_t)kSegRows | ((uint32_t)kSegRows << 16) : 0u;
    for (uint64_t sg = t * (kChunk / kSegRows); sg < (t + 1) * (kChunk / kSegRows); ++sg) {
      if (sg < s0 || sg >= s1) continue;
      uint4* wq = reinterpret_cast<uint4*>(bits + sg * kSegWords);
#pragma unroll
      for (int q = 0; q < kSegWords / 4; ++q) wq[q] = make_uint4(word, word, word, word);
      seg_info[sg] = info;
    }
  }
}

// RLE: the predicate is evaluated once per run (P:163's per-run view of
// the column); a matching run sets its row range in the mask — whole 32-bit words
// by plain stores, the (at most two) partial words by atomicOr — and the
// per-segment counts follow from the mask.
template <class Pred>
__global__ void __launch_bounds__(256) rle_mask_kernel(ColView c, Pred pred, uint32_t* bits) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < c.nruns; k += stride) {
    if (!pred(__ldg(c.payload + 2 * k))) continue;
    // rows [a, e), clamped to the column: a corrupt body (reported by StartsEpi)
    // never writes outside the mask
    const uint64_t a = __ldg(c.run_starts + k), e = min(__ldg(c.run_starts + k + 1), c.n);
    if (a >= e) continue;
    const uint64_t wa = a >> 5, we = (e - 1) >> 5;
    const uint32_t ma = ~0u << (a & 31), me = ~0u >> (31 - ((e - 1) & 31));
    if (wa == we) {
      atomicOr(bits + wa, ma & me);
    } else {
      atomicOr(bits + wa, ma);
      for (uint64_t q = wa + 1; q < we; ++q) bits[q] = ~0u;
      atomicOr(bits + we, me);
    }
  }
}

// per 512-row segment: count | (1-based last matching row << 16), from the mask;
// a warp takes eight segments per step (lane l: 16 bytes, words 4l .. 4l + 3)
__global__ void __launch_bounds__(256) seg_info_kernel(const uint32_t* bits, uint64_t NS, uint32_t* seg_info) {
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31, q = lane & 3;
  for (uint64_t s8 = gw; s8 * 8 < NS; s8 += nw) {
    const uint64_t sg = s8 * 8 + (lane >> 2);
    uint4 m = make_uint4(0u, 0u, 0u, 0u);
    if (sg < NS) m = __ldg(reinterpret_cast<const uint4*>(bits + sg * kSegWords) + q);
    uint32_t cnt = __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
    const uint32_t wb = q * 128;  // the lane's first row in the segment
    uint32_t last = m.w ? wb + 128 - __clz(m.w)
                        : m.z ? wb + 96 - __clz(m.z) : m.y ? wb + 64 - __clz(m.y) : m.x ? wb + 32 - __clz(m.x) : 0u;
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
      cnt += __shfl_xor_sync(kFull, cnt, o);
      last = max(last, __shfl_xor_sync(kFull, last, o));
    }
    if (sg < NS && q == 0) seg_info[sg] = cnt | (last << 16);
  }
}

cudaError_t launch_seg_info(const uint32_t* bits, uint64_t NS, uint32_t* seg_info, cudaStream_t s) {
  if (!NS) return cudaSuccess;
  uint64_t g2 = (NS + 63) / 64;  // 8 warps x 8 segments per CTA step
  if (g2 > (uint64_t)num_sms() * 8) g2 = num_sms() * 8;
  ProfScope prof_("seg_info", s);
  seg_info_kernel<<<(int)g2, 256, 0, s>>>(bits, NS, seg_info);
  return cudaGetLastError();
}

cudaError_t launch_select(const ColView& c, const PredSpec& p, uint32_t* bits, uint32_t* seg_info, uint64_t NS,
                          uint32_t* tile_list, uint32_t* err, cudaStream_t s) {
  if (NS == 0) return cudaSuccess;
  if (c.format == MS_RLE && c.run_starts) {
    cudaError_t e = cudaMemsetAsync(bits, 0, 4 * NS * kSegWords, s);
    if (e != cudaSuccess) return e;
    uint64_t g = (c.nruns + 255) / 256;
    if (g > (uint64_t)num_sms() * 16) g = num_sms() * 16;
    if (g) {
      ProfScope prof_("select_rle", s);
      if (p.is_bitmap) rle_mask_kernel<<<(int)g, 256, 0, s>>>(c, BitmapPred{p.bitmap, p.bitmap_bits}, bits);
      else rle_mask_kernel<<<(int)g, 256, 0, s>>>(c, RangePred{p.lo, p.span, p.neg}, bits);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_seg_info(bits, NS, seg_info, s);
  }
  // fast path: UNCOMPR, STATIC_BP, DYN_BP / FOR_BP with B >= 512, on full 512-row segments
  int kind = -1;
  uint64_t ns_fast = 0;
  if (c.format == MS_UNCOMPR) { kind = FAST_UNCOMPR; ns_fast = c.n / kSegRows; }
  if (c.format == MS_STATIC_BP) { kind = FAST_STATIC; ns_fast = c.n / kSegRows; }
  if ((c.format == MS_DYN_BP || c.format == MS_FOR_BP) && c.B >= (uint32_t)kSegRows) {
    kind = FAST_BLOCK;
    ns_fast = (c.nb << c.log2B) / kSegRows;
  }
  if (kind >= 0 && ns_fast) {
    FastPred fp{p.lo, p.span, p.neg, (uint32_t)p.is_bitmap, p.bitmap, p.bitmap_bits, {}, 0};
    fast_pred_table(fp);
    auto pick = [&](auto k, int stages, int warps_per_cta, int bufu32 = kPairBufWide) {
      const size_t smem = (size_t)warps_per_cta * stages * bufu32 * 4;
      set_smem_once((const void*)k, smem);
      int per_sm = 0;
      per_sm = occupancy_cached((const void*)k, warps_per_cta * 32, smem);
      if (per_sm < 1) per_sm = 1;
      const uint64_t warps = (uint64_t)per_sm * num_sms() * warps_per_cta;
      uint64_t spw = (ns_fast + warps - 1) / warps;
      spw += spw & 1;  // whole segment pairs per warp
      const uint64_t used = (ns_fast + spw - 1) / spw;
      const int grid = (int)((used + warps_per_cta - 1) / warps_per_cta);
      ProfScope prof_("select_fast", s);
      k<<<grid, warps_per_cta * 32, smem, s>>>(c, fp, bits, seg_info, ns_fast, spw, err, nullptr);
    };
    // staging slots sized from the descriptor's max_width hint: narrow (<= 32 bits, 2 x 2 KiB
    // per pair, 6 CTAs/SM), medium (<= 48 bits, 4 CTAs/SM) or wide (3 CTAs/SM). Measured on B200
    // (BJ.c5): 3-stage and 8-warp variants of the narrow kernel were 8-50% slower.
    const bool narrow = kind == FAST_UNCOMPR || (c.maxw >= 1 && c.maxw <= 32);
    const bool medium = !narrow && c.maxw >= 33 && c.maxw <= 48;
    // narrow bit-packed columns: the CTA-streamed core (selstream.cuh)
    const uint32_t mw = kind == FAST_STATIC ? c.w : c.maxw;
    const bool stream = kind != FAST_UNCOMPR && mw >= 1 && mw <= 32;
    auto pick_stream = [&](auto k) {
      const int S = ss_stages(mw);
      const size_t smem = ss_smem_bytes(mw, S);
      set_smem_once((const void*)k, smem);
      const uint64_t nchunks = (ns_fast + kSsSegs - 1) / kSsSegs;
      const int grid = (int)(nchunks < (uint64_t)num_sms() ? nchunks : (uint64_t)num_sms());
      ProfScope prof_("select_stream", s);
      k<<<grid, (1 + 2 * S) * 32, smem, s>>>(c, fp, bits, seg_info, ns_fast, mw, err, nullptr);
    };
#define MS_PICK(K)                                                                                   \
  do {                                                                                               \
    if (stream) pick_stream(select_stream_kernel<K == FAST_UNCOMPR ? FAST_STATIC : K, CORE_SELECT>);  \
    else if (narrow) pick(select_fast_kernel<K, 2, 4, 6, kPairBufNarrow>, 2, 4, kPairBufNarrow);     \
    else if (medium) pick(select_fast_kernel<K, 2, 4, 4, kPairBufMedium>, 2, 4, kPairBufMedium);     \
    else pick(select_fast_kernel<K, 2, 4, 3>, 2, 4);                                                 \
  } while (0)
    if (kind == FAST_UNCOMPR) MS_PICK(FAST_UNCOMPR);
    else if (kind == FAST_STATIC) MS_PICK(FAST_STATIC);
    else MS_PICK(FAST_BLOCK);
#undef MS_PICK
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (ns_fast < NS) {  // the rest (other formats, partial segments, block remainders)
    const uint64_t tiles = ((NS * kSegRows + kChunk - 1) / kChunk) - (ns_fast * kSegRows) / kChunk;
    const bool prune = !p.is_bitmap && tile_list &&
                       (c.format == MS_DELTA_BP || c.format == MS_FOR_BP || c.format == MS_DYN_BP);
    uint32_t* n_list = prune ? tile_list + tiles + 1 : nullptr;
    if (prune) {  // header-only decisions first; only undecided tiles are decoded
      cudaError_t e = cudaMemsetAsync(n_list, 0, 4, s);
      if (e != cudaSuccess) return e;
      uint64_t g = (tiles + 255) / 256;
      if (g > (uint64_t)num_sms() * 8) g = num_sms() * 8;
      ProfScope prof_("select_prune", s);
      tile_prune_kernel<<<(int)g, 256, 0, s>>>(c, RangePred{p.lo, p.span, p.neg}, bits, seg_info, ns_fast, NS,
                                                tile_list, n_list);
    }
    ProfScope prof_("select_generic", s);
    if (p.is_bitmap) {
      auto k = select_generic_kernel<BitmapPred>;
      k<<<persistent_grid(k, kThreads, tiles), kThreads, 0, s>>>(c, BitmapPred{p.bitmap, p.bitmap_bits}, bits,
                                                                 seg_info, ns_fast, NS, nullptr, nullptr);
    } else {
      auto k = select_generic_kernel<RangePred>;
      k<<<persistent_grid(k, kThreads, tiles), kThreads, 0, s>>>(c, RangePred{p.lo, p.span, p.neg}, bits,
                                                                 seg_info, ns_fast, NS,
                                                                 prune ? tile_list : nullptr, n_list);
    }
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ sums
// sum of a whole column mod 2^64, using the format identities:
// RLE sum v*len; FOR B*ref + sum codes; DELTA B*base + sum (B-j) d_j.
__global__ void __launch_bounds__(kThreads) sum_kernel(ColView c, unsigned long long* out) {
  __shared__ uint64_t wsum[kThreads / 32];
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t gthreads = (uint64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  uint64_t acc = 0;
  switch (c.format) {
    case MS_UNCOMPR:
      for (uint64_t i = gtid; i < c.n; i += gthreads) acc += __ldg(c.payload + i);
      break;
    case MS_STATIC_BP:
      for (uint64_t i = gtid; i < c.n; i += gthreads) acc += unpack_at(c.payload, i * c.w, c.w);
      break;
    case MS_RLE:
      for (uint64_t k = gtid; k < c.nruns; k += gthreads) acc += __ldg(c.payload + 2 * k) * __ldg(c.payload + 2 * k + 1);
      break;
    default: {
      const uint64_t gwarp = gtid >> 5, gwarps = gthreads >> 5;
      for (uint64_t b = gwarp; b < c.nb; b += gwarps) {
        const uint32_t cw0 = __ldg(c.cw + b);
        const uint32_t w = __ldg(c.cw + b + 1) - cw0;
        const uint64_t bit0 = (uint64_t)cw0 * c.B;
        uint64_t s = 0;
        if (w) {
          for (uint32_t j = lane; j < c.B; j += 32) {
            const uint64_t code = unpack_at(c.payload, bit0 + (uint64_t)j * w, w);
            s += c.format == MS_DELTA_BP ? (uint64_t)(c.B - j) * code : code;
          }
        }
        if (lane == 0 && c.format != MS_DYN_BP) s += (uint64_t)c.B * __ldg(c.ref + b);
        acc += s;
      }
      for (uint64_t i = gtid; i < c.nrem; i += gthreads) acc += __ldg(c.rem + i);
      break;
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) wsum[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int k = 0; k < kThreads / 32; ++k) t += wsum[k];
    if (t) atomicAdd(out, (unsigned long long)t);
  }
}

// rows [r0, n) of a column, one value at a time (the tail the fast scan leaves)
__global__ void sum_rows_kernel(ColView c, uint64_t r0, unsigned long long* out) {
  uint64_t acc = 0;
  for (uint64_t r = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < c.n; r += (uint64_t)gridDim.x * blockDim.x)
    acc += read_row(c, r);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

cudaError_t launch_sum(const ColView& c, unsigned long long* out, uint32_t* err, cudaStream_t s) {
  // fast path: the select scan machinery with a sum core, over full 512-row segments
  int kind = -1;
  uint64_t ns_fast = 0;
  if (c.format == MS_UNCOMPR) { kind = FAST_UNCOMPR; ns_fast = c.n / kSegRows; }
  if (c.format == MS_STATIC_BP) { kind = FAST_STATIC; ns_fast = c.n / kSegRows; }
  if ((c.format == MS_DYN_BP || c.format == MS_FOR_BP) && c.B >= (uint32_t)kSegRows) {
    kind = FAST_BLOCK;
    ns_fast = (c.nb << c.log2B) / kSegRows;
  }
  if (kind < 0 || !ns_fast) {
    ProfScope prof_("sum", s);
    sum_kernel<<<persistent_grid(sum_kernel, kThreads, ~0ull), kThreads, 0, s>>>(c, out);
    return cudaGetLastError();
  }
  const bool narrow = kind == FAST_UNCOMPR || (c.maxw >= 1 && c.maxw <= 32);
  FastPred fp{};
  auto pick = [&](auto k, int bufu32) {
    const size_t smem = (size_t)4 * 2 * bufu32 * 4;
    set_smem_once((const void*)k, smem);
    int per_sm = 0;
    per_sm = occupancy_cached((const void*)k, 4 * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const uint64_t warps = (uint64_t)per_sm * num_sms() * 4;
    uint64_t spw = (ns_fast + warps - 1) / warps;
    spw += spw & 1;
    const uint64_t used = (ns_fast + spw - 1) / spw;
    const int grid = (int)((used + 3) / 4);
    ProfScope prof_("sum_fast", s);
    k<<<grid, 4 * 32, smem, s>>>(c, fp, nullptr, nullptr, ns_fast, spw, err, out);
  };
  const uint32_t mw = kind == FAST_STATIC ? c.w : c.maxw;
  const bool stream = kind != FAST_UNCOMPR && mw >= 1 && mw <= 32;
  auto pick_stream = [&](auto k) {
    const int S = ss_stages(mw);
    const size_t smem = ss_smem_bytes(mw, S);
    set_smem_once((const void*)k, smem);
    const uint64_t nchunks = (ns_fast + kSsSegs - 1) / kSsSegs;
    const int grid = (int)(nchunks < (uint64_t)num_sms() ? nchunks : (uint64_t)num_sms());
    ProfScope prof_("sum_stream", s);
    k<<<grid, (1 + 2 * S) * 32, smem, s>>>(c, fp, nullptr, nullptr, ns_fast, mw, err, out);
  };
#define MS_PICK_SUM(K)                                                                               \
  do {                                                                                               \
    if (stream) pick_stream(select_stream_kernel<K == FAST_UNCOMPR ? FAST_STATIC : K, CORE_SUM>);     \
    else if (narrow) pick(select_fast_kernel<K, 2, 4, 6, kPairBufNarrow, CORE_SUM>, kPairBufNarrow); \
    else pick(select_fast_kernel<K, 2, 4, 3, kPairBufWide, CORE_SUM>, kPairBufWide);                 \
  } while (0)
  if (kind == FAST_UNCOMPR) MS_PICK_SUM(FAST_UNCOMPR);
  else if (kind == FAST_STATIC) MS_PICK_SUM(FAST_STATIC);
  else MS_PICK_SUM(FAST_BLOCK);
#undef MS_PICK_SUM
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const uint64_t r0 = ns_fast * kSegRows;
  if (r0 < c.n) {
    ProfScope prof_("sum_tail", s);
    sum_rows_kernel<<<8, 256, 0, s>>>(c, r0, out);
  }
  return cudaGetLastError();
}

// sum of data at positions (select -> project -> sum fused)
}  // namespace ms
