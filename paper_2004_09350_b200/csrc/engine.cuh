// engine.cuh — the generic on-the-fly de/re-compression engine (P:297-337,
// 468-505): a persistent kernel takes work items (2048 output rows) in order
// from a ticket, fills a shared-memory tile from a Source (decode of a column,
// expansion of a select bit mask, or a gather through positions), and encodes
// the tile into the output format with the output-side buffer layer below.
// Block formats need the exclusive prefix of the block widths (cw, D-4): it
// comes from a decoupled look-back over the per-item width sums, so the whole
// output is produced in one pass with one store per word.
#pragma once
#include "common.cuh"

namespace ms {

enum : int32_t { OUT_MAX_ONLY = 100 };  // pseudo-format: only reduce the max (auto static width)

struct OutView {
  int32_t format;
  uint32_t w;
  uint32_t B;
  uint32_t log2B;
  uint64_t n;                // logical length if n_dev == nullptr
  const uint64_t* n_dev;     // device-resident logical length (select outputs)
  uint64_t* payload;
  uint32_t* cw;
  uint64_t* ref;
  uint64_t* rem;
  uint64_t* status;          // look-back status, one per item
  uint32_t* ticket;
  unsigned long long* max_out;  // OUT_MAX_ONLY target
  uint32_t fits;                // STATIC_BP: w came from the max pass, no value can overflow it
  // slot mode (block formats): tile k's blocks are packed into slots[k * kChunk ...]
  // (64 bits per row bounds every width), their widths go to bw[block]; the host
  // scans bw into cw and tile_copy_kernel moves every tile to its place — no look-back
  uint64_t* slots;
  uint32_t* bw;
};

// Output word m (bits [64m, 64m+64)) of a packed stream of `cnt` codes of width
// w (1..64), m < 2^14 (a tile: <= 2048 codes); code(j) yields the j-th code,
// already < 2^w. 32-bit index math with a multiply-high division (div_small).
template <class CodeFn>
__device__ __forceinline__ uint64_t pack_word(CodeFn code, uint32_t cnt, uint32_t w, uint32_t m, uint32_t magic) {
  const uint32_t bit0 = m * 64;
  uint32_t j = div_small(bit0, w, magic);
  const uint32_t s = bit0 - j * w;
  uint64_t acc = j < cnt ? code(j) >> s : 0;
  for (++j; j < cnt; ++j) {
    const uint32_t jb = j * w;
    if (jb >= bit0 + 64) break;
    acc |= code(j) << (jb - bit0);
  }
  return acc;
}

// The same for 32-bit output words (bits [32m, 32m+32)) when w <= 32: the codes'
// low halves are enough and every step is one 32-bit instruction. Little-endian:
// u32 word 2k (2k+1) is the low (high) half of u64 word k, so the stream is the same.
__device__ __forceinline__ uint32_t pack_word32(const uint64_t* v, uint32_t cnt, uint32_t w, uint32_t mask, uint32_t m,
                                                uint32_t magic, uint32_t sub = 0) {
  const uint32_t* __restrict__ v32 = reinterpret_cast<const uint32_t*>(v);
  const uint32_t bit0 = m * 32;
  uint32_t j = div_small(bit0, w, magic);
  uint32_t jb = j * w;
  uint32_t acc = j < cnt ? ((v32[2 * j] - sub) & mask) >> (bit0 - jb) : 0u;
  for (++j, jb += w; j < cnt && jb < bit0 + 32; ++j, jb += w) acc |= ((v32[2 * j] - sub) & mask) << (jb - bit0);
  return acc;
}

// Output-side buffer layer: encode sm.vals[0..cnt) = rows
// [r0, r0+cnt) of the output column. Item index = r0 / kChunk.
// vals: the tile's rows (sm.vals, or a staged input buffer encoded in place)
__device__ __forceinline__ void encode_tile(const OutView& o, uint32_t item, uint64_t r0, uint32_t cnt,
                                            uint64_t n, EngineSmem& sm, uint32_t* err, uint64_t* vals) {
  const int tid = threadIdx.x;
  switch (o.format) {
    case MS_UNCOMPR:
      if (cnt == kChunk && (reinterpret_cast<uintptr_t>(o.payload) & 15) == 0) {  // full tile: 128-bit stores
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(o.payload + r0);
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(vals);
#pragma unroll
        for (int q = 0; q < kVPT / 2; ++q) dst[tid + q * kThreads] = src[tid + q * kThreads];
      } else {
        for (uint32_t i = tid; i < cnt; i += kThreads) o.payload[r0 + i] = vals[i];
      }
      return;
    case MS_RLE:  // only for inputs without equal neighbours (select positions): runs of length 1
      for (uint32_t i = tid; i < cnt; i += kThreads) {
        o.payload[2 * (r0 + i)] = vals[i];
        o.payload[2 * (r0 + i) + 1] = 1;
      }
      return;
    case OUT_MAX_ONLY: {
      uint64_t mx = 0;
      for (uint32_t i = tid; i < cnt; i += kThreads) mx = vals[i] > mx ? vals[i] : mx;
      mx = warp_max(mx);
      if ((tid & 31) == 0 && mx) atomicMax(o.max_out, (unsigned long long)mx);
      return;
    }
    case MS_STATIC_BP: {
      const uint32_t w = o.w;
      if (w < 64 && !o.fits)
        for (uint32_t i = tid; i < cnt; i += kThreads)
          if (vals[i] >> w) atomicOr(err, err_bit(MS_E_WIDTH_OVERFLOW));
      const uint64_t mask = low_mask(w);
      const uint64_t wbase = (uint64_t)item * (kChunk / 64) * w;
      const uint32_t magic = 0xffffffffu / w + 1u;
      if (w <= 32) {
        // u32 words; an odd count ends in the low half of the last u64 word, whose high
        // half (no codes) is written 0 as the u64 path would
        const uint32_t n32 = (cnt * w + 31) / 32, n32e = (n32 + 1) & ~1u;
        uint32_t* dst = reinterpret_cast<uint32_t*>(o.payload + wbase);
        const uint32_t m32 = 0xffffffffu >> (32 - w);
        const uint32_t* __restrict__ v32 = reinterpret_cast<const uint32_t*>(vals);
        // word m's first code j = floor(32 m / w) at bit offset s = 32 m - j w; the
        // thread's next word is kThreads words on = q codes + r bits (no division per word)
        uint32_t j = div_small(32 * tid, w, magic), sb = 32 * tid - j * w;
        const uint32_t q = (32 * kThreads) / w, r = 32 * kThreads - q * w;
        for (uint32_t m = tid; m < n32e; m += kThreads) {
          uint32_t acc = 0;
          if (m < n32) {
            acc = (v32[2 * j] & m32) >> sb;
            uint32_t jj = j + 1, sh = w - sb;  // the next code starts at bit w - s of the word
            for (; sh < 32 && jj < cnt; ++jj, sh += w) acc |= (v32[2 * jj] & m32) << sh;
          }
          dst[m] = acc;
          j += q;
          sb += r;
          if (sb >= w) {
            sb -= w;
            ++j;
          }
        }
        return;
      }
      const uint64_t nwords = ((uint64_t)cnt * w + 63) / 64;
      auto code = [&](uint32_t j) { return vals[j] & mask; };
      for (uint32_t m = tid; m < nwords; m += kThreads) o.payload[wbase + m] = pack_word(code, cnt, w, m, magic);
      return;
    }
    default:
      break;
  }
  // ---- block formats: DYN_BP / FOR_BP / DELTA_BP
  const uint32_t B = o.B, lg = o.log2B;
  const uint32_t nbc = cnt >> lg;  // full blocks in this tile (all but the last tile: kChunk/B)
  const uint64_t kb0 = r0 >> lg;   // global index of the tile's first block
  const bool is_for = o.format == MS_FOR_BP;
  if (tid < kMaxBlocksPerChunk) {
    sm.bmin[tid] = ~0ull;
    sm.bmax[tid] = 0;
    sm.bw[tid] = 0;
  }
  __syncthreads();
  // codes (DELTA: in-block differences) and per-block widths, rows lane-strided
  // (tid + q * kThreads: conflict-free shared-memory access; a warp's 32 rows lie in
  // one block, B >= 128). DYN / DELTA: w_b = max ebw(code) by one 32-bit warp
  // reduction (redux.sync) per block run; FOR: 64-bit min and max, each as two
  // 32-bit reductions (high halves, then low halves of the lanes at the high max).
  // DELTA codes replace the values in place afterwards; the block bases are kept in
  // bmin (unused by DELTA).
  {
    const uint32_t nmain = nbc << lg;
    const uint32_t lane = tid & 31;
    uint64_t cq[kVPT];
    uint64_t lmin = ~0ull, lmax = 0;
    uint32_t lw = 0;
    uint32_t cur = ~0u;
    auto flush = [&]() {
      if (is_for) {
        const uint32_t hmax = __reduce_max_sync(kFull, (uint32_t)(lmax >> 32));
        const uint32_t lmx = __reduce_max_sync(kFull, (uint32_t)(lmax >> 32) == hmax ? (uint32_t)lmax : 0u);
        const uint32_t hmin = __reduce_min_sync(kFull, (uint32_t)(lmin >> 32));
        const uint32_t lmn = __reduce_min_sync(kFull, (uint32_t)(lmin >> 32) == hmin ? (uint32_t)lmin : ~0u);
        if (lane == 0) {
          atomicMin((unsigned long long*)&sm.bmin[cur], ((unsigned long long)hmin << 32) | lmn);
          atomicMax((unsigned long long*)&sm.bmax[cur], ((unsigned long long)hmax << 32) | lmx);
        }
      } else {
        const uint32_t wm = __reduce_max_sync(kFull, lw);
        if (lane == 0 && wm) atomicMax(&sm.bw[cur], wm);
      }
      lmin = ~0ull;
      lmax = 0;
      lw = 0;
    };
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      const uint32_t j = tid + q * kThreads;
      const uint32_t wrow = (tid & ~31u) + q * kThreads;  // the warp's first row at this step
      uint64_t c = 0;
      if (j < nmain) {
        const uint64_t v = vals[j];
        if (o.format == MS_DELTA_BP) {
          if (j & (B - 1)) c = v - vals[j - 1];
          else sm.bmin[j >> lg] = v;  // the block's base (D-6)
        } else {
          c = v;
        }
      }
      cq[q] = c;
      if (wrow < nmain) {
        const uint32_t blk = wrow >> lg;
        if (blk != cur && cur != ~0u) flush();
        cur = blk;
        if (is_for) {
          lmin = c < lmin ? c : lmin;
          lmax = c > lmax ? c : lmax;
        } else {
          const uint32_t e = ebw64(c);
          lw = e > lw ? e : lw;
        }
      }
    }
    if (cur != ~0u) flush();
    if (o.format == MS_DELTA_BP) {
      __syncthreads();  // every value read before the codes overwrite them
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        const uint32_t j = tid + q * kThreads;
        if (j < nmain) vals[j] = cq[q];
      }
    }
  }
  __syncthreads();
  if (tid < 32) {
    const int lane = tid;
    uint32_t w = 0;
    if (lane < (int)nbc) {
      w = is_for ? ebw64(sm.bmax[lane] - sm.bmin[lane]) : sm.bw[lane];
      sm.bw[lane] = w;
    }
    const uint64_t incl = warp_incl_scan(w);
    const uint64_t tile_sum = __shfl_sync(kFull, incl, 31);
    const uint64_t E = o.slots ? 0ull : lookback_warp(o.status, item, tile_sum);
    if (lane < (int)nbc) {
      const uint64_t c_incl = E + incl;
      if (o.slots) {
        o.bw[kb0 + lane] = w;
      } else {
        if (c_incl > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
        o.cw[kb0 + lane + 1] = (uint32_t)c_incl;
      }
      sm.bex[lane] = E + incl - w;
      if (is_for || o.format == MS_DELTA_BP) o.ref[kb0 + lane] = sm.bmin[lane];
    }
    if (lane == (int)nbc) sm.bex[lane] = E + tile_sum;  // end of the tile's last block
    if (item == 0 && lane == 0) o.cw[0] = 0;
  }
  __syncthreads();
  // pack: the tile's blocks are consecutive in the output, so its u64 words are one
  // flat range [0, (bex[nbc] - bex[0]) * B / 64) over all threads; word m belongs to
  // the block whose range holds it (a cursor that only moves forward)
  if (nbc) {
    const uint64_t e0 = sm.bex[0];
    const uint32_t wpb = B / 64;  // u64 words per unit of width
    const uint32_t total = (uint32_t)(sm.bex[nbc] - e0) * wpb;
    uint64_t* const dst = (o.slots ? o.slots + (uint64_t)item * kChunk : o.payload) + e0 * wpb;
    uint32_t bi = 0, bstart = 0, bend = (uint32_t)(sm.bex[1] - e0) * wpb;
    uint32_t w = sm.bw[0], magic = w ? 0xffffffffu / w + 1u : 0u;
    for (uint32_t m = tid; m < total; m += kThreads) {
      if (m >= bend) {
        while (m >= bend) {
          ++bi;
          bstart = bend;
          bend = (uint32_t)(sm.bex[bi + 1] - e0) * wpb;
        }
        w = sm.bw[bi];
        magic = 0xffffffffu / w + 1u;  // w > 0: the block has words
      }
      const uint64_t* v = vals + (bi << lg);
      const uint32_t mb = m - bstart;  // word within the block
      uint64_t word;
      if (w <= 32) {  // two 32-bit words; FOR codes v - ref fit the low halves
        const uint32_t m32 = 0xffffffffu >> (32 - w);
        const uint32_t sub = is_for ? (uint32_t)sm.bmin[bi] : 0u;
        word = (uint64_t)pack_word32(v, B, w, m32, 2 * mb, magic, sub) |
               ((uint64_t)pack_word32(v, B, w, m32, 2 * mb + 1, magic, sub) << 32);
      } else if (is_for) {
        const uint64_t rf = sm.bmin[bi];
        auto code = [&](uint32_t j) { return v[j] - rf; };
        word = pack_word(code, B, w, mb, magic);
      } else {
        auto code = [&](uint32_t j) { return v[j]; };  // DELTA: the codes were written in place
        word = pack_word(code, B, w, mb, magic);
      }
      dst[m] = word;
    }
  }
  const uint32_t rem_cnt = cnt - (nbc << lg);
  if (rem_cnt) {  // the final partial block -> uncompressed remainder
    for (uint32_t i = tid; i < rem_cnt; i += kThreads) o.rem[i] = vals[(nbc << lg) + i];
  }
}

// slot mode, second half: tile k's packed blocks (slot words [0, (cwx[kb1] - cwx[kb0]) * B / 64))
// -> payload word cwx[kb0] * B / 64, and cw[b + 1] = cwx[b + 1] for its blocks. One warp per tile
// (a CTA per tile left most threads idle on narrow tiles — 1.3 KB at 5 bits — and every tile
// waits on its offsets before its copy: 8x the tiles in flight per SM).
static __global__ void __launch_bounds__(256) tile_copy_kernel(OutView o, uint64_t n_tiles, uint64_t nb, const uint64_t* cwx,
                                                        uint32_t* err) {
  const uint32_t per = kChunk >> o.log2B;  // blocks per full tile
  const uint32_t lane = threadIdx.x & 31, wpc = blockDim.x >> 5;
  const uint64_t n_warps = (uint64_t)gridDim.x * wpc;
  for (uint64_t t = (uint64_t)blockIdx.x * wpc + (threadIdx.x >> 5); t < n_tiles; t += n_warps) {
    const uint64_t kb0 = t * per;
    if (kb0 >= nb) break;
    const uint64_t kb1 = min(kb0 + per, nb);
    const uint64_t E = __ldg(cwx + kb0);
    const uint64_t words = (__ldg(cwx + kb1) - E) * (o.B / 64);
    for (uint64_t b = kb0 + lane; b < kb1; b += 32) {
      const uint64_t c1 = __ldg(cwx + b + 1);
      if (c1 > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // D-4 limit
      o.cw[b + 1] = (uint32_t)c1;
    }
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(o.slots + t * kChunk);
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(o.payload + E * (o.B / 64));
    // B >= 128: the tile's words start 16-byte aligned on both sides (B/64 * w words, B/64 even)
    const uint64_t n2 = words / 2;
#pragma unroll 4
    for (uint64_t m = lane; m < n2; m += 32) dst[m] = src[m];
  }
}

// ------------------------------------------------------------------ sources
// Decode of rows [r0, r0+cnt) of a column (compress / decompress / morph).
struct ColSource {
  static constexpr int kMinBlocks = 4;  // 64 registers: 4 CTAs per SM (latency-bound decode)
  ColView c;
  __device__ __forceinline__ void load(uint32_t item, uint64_t r0, uint32_t cnt, EngineSmem& sm, uint32_t* err) const {
    load_rows(c, r0, cnt, sm);
  }
};

// Expansion of the select bit mask into positions (ranks r0 .. r0+cnt of the
// output). Bit j of mask word m <=> row 32m + j matched.
struct BitmaskSource {
  static constexpr int kMinBlocks = 1;
  const uint32_t* bits;
  const uint64_t* seg_off;      // exclusive prefix of per-segment counts (segments of kSegRows rows)
  const uint32_t* start_seg;    // per output item: segment holding rank kChunk*item
  uint64_t n_words;
  uint64_t row_offset;
  __device__ __forceinline__ void load(uint32_t item, uint64_t r0, uint32_t cnt, EngineSmem& sm, uint32_t* err) const {
    const int tid = threadIdx.x;
    const uint64_t t = start_seg[item];
    uint64_t rank = seg_off[t];  // rank of the first set bit at or after word t*kSegWords
    uint64_t w0 = t * kSegWords;
    const uint64_t end = r0 + cnt;
    while (true) {
      const uint64_t m = w0 + tid;
      uint32_t word = m < n_words ? __ldg(bits + m) : 0u;
      uint64_t tot;
      const uint64_t ex = cta_excl_scan(__popc(word), sm.scan, &tot);
      uint64_t q = rank + ex;
      while (word) {
        const int j = __ffs(word) - 1;
        word &= word - 1;
        if (q >= r0 && q < end) sm.vals[q - r0] = row_offset + m * 32 + j;
        ++q;
      }
      rank += tot;
      w0 += kThreads;
      if (rank >= end || w0 >= n_words) break;
    }
    __syncthreads();
  }
};

// Gather through positions (project): rows of the positions column
// give global positions p; the value is data[p - row_offset]. For the O(1)
// random-access formats each thread issues the header loads (cw, ref) of all
// its positions, then all payload loads, so every thread has 8-16 independent
// loads in flight instead of a dependent chain per position.
struct GatherSource {
  static constexpr int kMinBlocks = 2;  // <= 128 registers (unbounded: 190, one CTA per SM)
  ColView pos;
  ColView data;
  uint64_t row_offset;
  __device__ __forceinline__ void load(uint32_t item, uint64_t r0, uint32_t cnt, EngineSmem& sm, uint32_t* err) const {
    load_rows(pos, r0, cnt, sm);
    const int tid = threadIdx.x;
    if (data.format == MS_FOR_BP || data.format == MS_DYN_BP) {
      const uint64_t main_rows = data.nb << data.log2B;
      uint64_t r[kVPT], b[kVPT];
      uint32_t cw0[kVPT], w[kVPT];
      uint64_t rf[kVPT];
      bool ok[kVPT];
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        const uint32_t i = tid + q * kThreads;
        const uint64_t p = i < cnt ? sm.vals[i] : row_offset;
        ok[q] = i < cnt && p >= row_offset && p - row_offset < data.n;
        if (i < cnt && !ok[q]) atomicOr(err, err_bit(MS_E_RANGE));
        r[q] = ok[q] ? p - row_offset : 0;
        b[q] = r[q] >> data.log2B;
      }
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        const bool inm = ok[q] && r[q] < main_rows;
        cw0[q] = inm ? __ldg(data.cw + b[q]) : 0u;
        w[q] = inm ? __ldg(data.cw + b[q] + 1) : 0u;
        rf[q] = inm && data.format == MS_FOR_BP ? __ldg(data.ref + b[q]) : 0ull;
        if (ok[q] && !inm) rf[q] = __ldg(data.rem + (r[q] - main_rows));
      }
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        const bool inm = ok[q] && r[q] < main_rows;
        w[q] -= cw0[q];
        const uint64_t bit = (uint64_t)cw0[q] * data.B + (uint64_t)(r[q] & (data.B - 1)) * w[q];
        const uint64_t v = inm ? unpack_at(data.payload, bit, w[q]) : 0ull;
        const uint32_t i = tid + q * kThreads;
        if (i < cnt) sm.vals[i] = rf[q] + v;
      }
    } else {
      // DELTA_BP / RLE data (no O(1) access, D-12): when the tile's positions span few
      // data tiles, decode those once into a second buffer and pick the values there
      __shared__ EngineSmem dsm;
      __shared__ unsigned long long g_lo, g_hi;
      const bool seq = data.format == MS_DELTA_BP || data.format == MS_RLE;
      bool tiled = false;
      if (seq) {
        if (tid == 0) {
          g_lo = ~0ull;
          g_hi = 0;
        }
        __syncthreads();
        unsigned long long lo = ~0ull, hi = 0;
        for (uint32_t i = tid; i < cnt; i += kThreads) {
          const uint64_t p = sm.vals[i];
          lo = p < lo ? p : lo;
          hi = p > hi ? p : hi;
        }
        atomicMin(&g_lo, lo);
        atomicMax(&g_hi, hi);
        __syncthreads();
        const uint64_t plo = g_lo, phi = g_hi;
        tiled = cnt && plo >= row_offset && phi - row_offset < data.n && (phi - plo) < 32ull * kChunk;
        if (tiled) {
          uint64_t v[kVPT];
#pragma unroll
          for (int q = 0; q < kVPT; ++q) v[q] = 0;
          for (uint64_t dt = (plo - row_offset) / kChunk; dt <= (phi - row_offset) / kChunk; ++dt) {
            const uint64_t d0 = dt * kChunk;
            const uint32_t dcnt = (uint32_t)min((uint64_t)kChunk, data.n - d0);
            load_rows(data, d0, dcnt, dsm);  // ends with a barrier
#pragma unroll
            for (int q = 0; q < kVPT; ++q) {
              const uint32_t i = tid + q * kThreads;
              if (i < cnt) {
                const uint64_t r = sm.vals[i] - row_offset;
                if (r >= d0 && r < d0 + dcnt) v[q] = dsm.vals[r - d0];
              }
            }
            __syncthreads();
          }
#pragma unroll
          for (int q = 0; q < kVPT; ++q) {
            const uint32_t i = tid + q * kThreads;
            if (i < cnt) sm.vals[i] = v[q];
          }
        }
      }
      if (!tiled) {
        for (uint32_t i = tid; i < cnt; i += kThreads) {
          const uint64_t p = sm.vals[i];
          uint64_t v = 0;
          if (p < row_offset || p - row_offset >= data.n) atomicOr(err, err_bit(MS_E_RANGE));
          else v = read_row(data, p - row_offset);
          sm.vals[i] = v;
        }
      }
    }
    __syncthreads();
  }
};

template <class Src>
__global__ void __launch_bounds__(kThreads, Src::kMinBlocks) engine_kernel(Src src, OutView out, uint32_t* err) {
  __shared__ EngineSmem sm;
  const uint64_t n = out.n_dev ? *out.n_dev : out.n;
  const uint64_t n_items = (n + kChunk - 1) / kChunk;
  // tiles in ticket order only when the output needs the look-back (block formats
  // without slots); otherwise a static grid-stride order saves an atomic per tile
  const bool ordered = !out.slots && (out.format == MS_DYN_BP || out.format == MS_FOR_BP ||
                                      out.format == MS_DELTA_BP);
  uint64_t next = blockIdx.x;
  if (out.format == OUT_MAX_ONLY) {  // auto static width: a running max per thread, one atomic per warp at the end
    uint64_t mx = 0;
    for (uint64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const uint64_t r0 = item * kChunk;
      const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, n - r0);
      src.load((uint32_t)item, r0, cnt, sm, err);
      for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) mx = sm.vals[i] > mx ? sm.vals[i] : mx;
      __syncthreads();
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(out.max_out, (unsigned long long)mx);
    return;
  }
  while (true) {
    if (ordered) {
      if (threadIdx.x == 0) sm.item = atomicAdd(out.ticket, 1u);
      __syncthreads();
    }
    const uint32_t item = ordered ? sm.item : (uint32_t)next;
    next += gridDim.x;
    if (item >= n_items) break;
    const uint64_t r0 = (uint64_t)item * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, n - r0);
    src.load(item, r0, cnt, sm, err);
    encode_tile(out, item, r0, cnt, n, sm, err, sm.vals);
    __syncthreads();
  }
}

}  // namespace ms
