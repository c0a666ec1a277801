// plan.cu — the plan-level operators beyond select / project / sum / morph
// (SURVEY.md §8(f) #2 and #3): the exact-size format profile that drives the
// per-intermediate format choice (PAPER.md P:66-68 DP2, P:722-735 cost-based
// selection on the compression-rate objective), and the
// star-schema operators SPEC.md S:295-321 lists (intersect / merge of sorted
// positions, equi-join, group ids, elementwise arithmetic; "operators ...
// sufficient to execute the SSB").
//
// Every input is read through the tile decoder of the generic engine
// (load_rows: 2048 rows into shared memory per CTA iteration, any format), so no
// operator decompresses a whole input column into HBM (DP3).
#include "common.cuh"
#include "grid.cuh"
#include "launch.h"

namespace ms {

namespace {

// splitmix64 finalizer (hash of a key / group combination)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t ld_acq_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ------------------------------------------------------------ format profile
// One pass over the column, tile by tile: for every full block of B rows its max,
// min and largest in-block delta (v_j - v_{j-1} mod 2^64, d_0 = 0, D-6); the
// column maximum; the number of runs. acc: [0] max, [1] sum_b ebw(max_b) (DYN_BP),
// [2] sum_b ebw(max delta_b) (DELTA_BP), [3] sum_b ebw(max_b - min_b) (FOR_BP),
// [4] runs (value changes + 1). B divides the 2048-row tile.
__global__ void __launch_bounds__(kThreads) profile_kernel(ColView c, uint32_t B, unsigned long long* acc,
                                                           uint64_t* first_last) {
  __shared__ EngineSmem sm;
  __shared__ uint64_t wmax[kThreads / 32], wmin[kThreads / 32], wdel[kThreads / 32];
  __shared__ unsigned long long cta[5];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < 5) cta[tid] = 0;
  const uint64_t n_tiles = (c.n + kChunk - 1) / kChunk;
  const uint64_t main_rows = c.n / B * B;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, c.n - r0);
    load_rows(c, r0, cnt, sm);
    // thread tid: rows [8 tid, 8 tid + 8) of the tile
    const uint32_t i0 = tid * kVPT;
    uint64_t mx = 0, mn = ~0ull, md = 0, chg = 0;
    uint64_t prev = i0 > 0 ? sm.vals[i0 - 1] : 0ull;
    for (uint32_t q = 0; q < kVPT; ++q) {
      const uint32_t i = i0 + q;
      if (i >= cnt) break;
      const uint64_t v = sm.vals[i];
      const uint64_t r = r0 + i;
      mx = v > mx ? v : mx;
      mn = v < mn ? v : mn;
      if ((r & (B - 1)) != 0) {  // not a block start: a delta inside the block
        const uint64_t d = v - prev;
        md = d > md ? d : md;
      }
      if (i > 0 && v != prev) ++chg;  // a run boundary inside the tile
      prev = v;
    }
    // run boundaries between tiles: from the tiles' first / last values (runs_kernel)
    if (tid == 0) {
      first_last[2 * t] = sm.vals[0];
      first_last[2 * t + 1] = sm.vals[cnt - 1];
    }
    // global max (every row, remainder included)
    uint64_t m32 = warp_max(mx);
    if (lane == 0 && m32) atomicMax(&cta[0], (unsigned long long)m32);
    const uint64_t ch = warp_sum(chg);
    if (lane == 0 && ch) atomicAdd(&cta[4], (unsigned long long)ch);
    // per block: threads of a block are B / 8 consecutive threads; reduce within
    // groups of G = min(32, B / 8) lanes, then across the block's warps
    const uint32_t G = B / kVPT < 32 ? B / kVPT : 32u;
    uint64_t bmx = (i0 < cnt) ? mx : 0ull, bmn = (i0 < cnt) ? mn : ~0ull, bmd = (i0 < cnt) ? md : 0ull;
    for (uint32_t o = G / 2; o; o >>= 1) {
      const uint64_t a = __shfl_xor_sync(kFull, bmx, o), b = __shfl_xor_sync(kFull, bmn, o),
                     d = __shfl_xor_sync(kFull, bmd, o);
      bmx = a > bmx ? a : bmx;
      bmn = b < bmn ? b : bmn;
      bmd = d > bmd ? d : bmd;
    }
    const uint32_t wpb = B / kVPT / 32;  // warps per block (0 when a warp holds several blocks)
    if (wpb <= 1) {
      if ((lane & (G - 1)) == 0) {
        const uint64_t blk_row = r0 + i0;  // first row of this group's block
        if (blk_row + B <= main_rows && blk_row < main_rows) {
          atomicAdd(&cta[1], (unsigned long long)ebw64(bmx));
          atomicAdd(&cta[2], (unsigned long long)ebw64(bmd));
          atomicAdd(&cta[3], (unsigned long long)ebw64(bmx - bmn));
        }
      }
    } else {
      if (lane == 0) {
        wmax[wid] = bmx;
        wmin[wid] = bmn;
        wdel[wid] = bmd;
      }
      __syncthreads();
      if (tid < kThreads / 32 && tid % wpb == 0) {
        uint64_t a = 0, b = ~0ull, d = 0;
        for (uint32_t k = 0; k < wpb; ++k) {
          a = wmax[tid + k] > a ? wmax[tid + k] : a;
          b = wmin[tid + k] < b ? wmin[tid + k] : b;
          d = wdel[tid + k] > d ? wdel[tid + k] : d;
        }
        const uint64_t blk_row = r0 + (uint64_t)tid * 32 * kVPT;
        if (blk_row + B <= main_rows) {
          atomicAdd(&cta[1], (unsigned long long)ebw64(a));
          atomicAdd(&cta[2], (unsigned long long)ebw64(d));
          atomicAdd(&cta[3], (unsigned long long)ebw64(a - b));
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) {
    atomicMax(acc + 0, cta[0]);
    for (int k = 1; k < 5; ++k) atomicAdd(acc + k, cta[k]);
  }
}

__global__ void runs_kernel(const uint64_t* first_last, uint64_t n_tiles, unsigned long long* acc) {
  uint64_t k = 0;
  for (uint64_t t = 1 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles;
       t += (uint64_t)gridDim.x * blockDim.x)
    k += first_last[2 * t] != first_last[2 * t - 1];
  k = warp_sum(k);
  if ((threadIdx.x & 31) == 0 && k) atomicAdd(acc + 4, (unsigned long long)k);
  if (blockIdx.x == 0 && threadIdx.x == 0 && n_tiles) atomicAdd(acc + 4, 1ull);  // the first run
}

// per 512-row segment: set bits of its 16 mask words
__global__ void seg_count_kernel(const uint32_t* bits, uint64_t NS, uint32_t* cnt) {
  for (uint64_t sg = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; sg < NS; sg += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int k = 0; k < kSegWords; ++k) c += __popc(bits[sg * kSegWords + k]);
    cnt[sg] = c;
  }
}

// ------------------------------------------------------------ positions -> bitmap
// Sets bit (p - base) of `bits` for every position p of column c inside
// [base, base + nbits); checks that the positions are strictly increasing (inside
// the tile here; across tiles through first / last, checked by sorted_check).
__global__ void __launch_bounds__(kThreads) pos_bitmap_kernel(ColView c, uint64_t base, uint64_t nbits,
                                                              uint32_t* bits, uint64_t* first_last, uint32_t* err) {
  __shared__ EngineSmem sm;
  const uint64_t n_tiles = (c.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, c.n - r0);
    load_rows(c, r0, cnt, sm);
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      const uint64_t p = sm.vals[i];
      if (i > 0 && p <= sm.vals[i - 1]) atomicOr(err, err_bit(MS_E_INVALID));  // NotSorted
      if (p >= base && p - base < nbits) atomicOr(bits + ((p - base) >> 5), 1u << ((p - base) & 31));
    }
    if (threadIdx.x == 0) {
      first_last[2 * t] = sm.vals[0];
      first_last[2 * t + 1] = sm.vals[cnt - 1];
    }
    __syncthreads();
  }
}

__global__ void sorted_check_kernel(const uint64_t* first_last, uint64_t n_tiles, uint32_t* err) {
  for (uint64_t t = 1 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles;
       t += (uint64_t)gridDim.x * blockDim.x)
    if (first_last[2 * t] <= first_last[2 * t - 1]) atomicOr(err, err_bit(MS_E_INVALID));
}

// value of row r by one warp: DELTA_BP blocks are summed lane-parallel (the codes up
// to row r, B / 32 per lane, plus the base), every other format by read_row
__device__ uint64_t row_by_warp(const ColView& c, uint64_t r) {
  const uint32_t lane = threadIdx.x & 31;
  if (c.format != MS_DELTA_BP || r >= (c.nb << c.log2B)) return read_row(c, r);
  const uint64_t b = r >> c.log2B;
  const uint32_t j = (uint32_t)(r & (c.B - 1));
  const uint32_t cw0 = __ldg(c.cw + b);
  const uint32_t w = __ldg(c.cw + b + 1) - cw0;
  uint64_t s = 0;
  for (uint32_t q = lane; q <= j; q += 32) s += unpack_at(c.payload, (uint64_t)cw0 * c.B + (uint64_t)q * w, w);
  return __ldg(c.ref + b) + warp_sum(s);
}

// the first and last value of two columns (positions: their ranges); one warp
__global__ void ends_kernel(ColView a, ColView b, uint64_t* out) {
  const uint64_t a0 = a.n ? row_by_warp(a, 0) : 0, a1 = a.n ? row_by_warp(a, a.n - 1) : 0;
  const uint64_t b0 = b.n ? row_by_warp(b, 0) : 0, b1 = b.n ? row_by_warp(b, b.n - 1) : 0;
  if (threadIdx.x == 0) {
    out[0] = a0;
    out[1] = a1;
    out[2] = b0;
    out[3] = b1;
  }
}

__global__ void bits_combine_kernel(uint32_t* a, const uint32_t* b, uint64_t n_words, int op) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_words; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = op ? (a[i] | b[i]) : (a[i] & b[i]);
}

// ------------------------------------------------------------ hash table
// Open addressing, linear probing; slot state 0 empty, 1 being claimed, 2 ready.
struct HT {
  uint32_t* state;
  uint64_t* key;
  uint64_t* key2;  // second key component (group: the previous group id), or nullptr
  uint64_t mask;   // capacity - 1 (power of two)
};

// slot of (k, k2); inserted when absent and `insert`; ~0 when absent and !insert or full
__device__ uint64_t ht_slot(const HT& h, uint64_t k, uint64_t k2, bool insert, uint32_t* err) {
  uint64_t s = mix64(k ^ mix64(k2 + 0x9E3779B97F4A7C15ull)) & h.mask;
  for (uint64_t probe = 0; probe <= h.mask; ++probe) {
    uint32_t st = ld_acq_u32(h.state + s);
    if (st == 0) {
      if (!insert) return ~0ull;
      if (atomicCAS(h.state + s, 0u, 1u) == 0u) {
        h.key[s] = k;
        if (h.key2) h.key2[s] = k2;
        st_rel_u32(h.state + s, 2u);
        return s;
      }
      st = ld_acq_u32(h.state + s);
    }
    while (st != 2u) st = ld_acq_u32(h.state + s);
    if (__ldcg(h.key + s) == k && (!h.key2 || __ldcg(h.key2 + s) == k2)) return s;
    s = (s + 1) & h.mask;
  }
  atomicOr(err, err_bit(MS_E_NOMEM));  // table full
  return ~0ull;
}

// group: insert (prev id, key) of every row, keep the smallest row per group
__global__ void __launch_bounds__(kThreads) group_insert_kernel(ColView keys, ColView prev, HT h,
                                                                unsigned long long* first, uint32_t* err) {
  __shared__ EngineSmem sk, sp;
  const uint64_t n_tiles = (keys.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, keys.n - r0);
    load_rows(keys, r0, cnt, sk);
    if (prev.n) load_rows(prev, r0, cnt, sp);
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      const uint64_t s = ht_slot(h, sk.vals[i], prev.n ? sp.vals[i] : 0ull, true, err);
      if (s != ~0ull) atomicMin(first + s, (unsigned long long)(r0 + i));
    }
    __syncthreads();
  }
}

// every group's first row -> one bit in the n-row mask
__global__ void group_mark_kernel(HT h, const unsigned long long* first, uint32_t* bits) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= h.mask; s += (uint64_t)gridDim.x * blockDim.x)
    if (h.state[s] == 2u) {
      const uint64_t r = first[s];
      atomicOr(bits + (r >> 5), 1u << (r & 31));
    }
}

// id of every row = rank of its group's first row among all first rows (dense ids in
// first-occurrence order): segment offset + popcount inside the segment
__global__ void __launch_bounds__(kThreads) group_ids_kernel(ColView keys, ColView prev, HT h,
                                                             const unsigned long long* first, const uint32_t* bits,
                                                             const uint64_t* seg_off, uint64_t* ids, uint32_t* err) {
  __shared__ EngineSmem sk, sp;
  const uint64_t n_tiles = (keys.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, keys.n - r0);
    load_rows(keys, r0, cnt, sk);
    if (prev.n) load_rows(prev, r0, cnt, sp);
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) {
      const uint64_t s = ht_slot(h, sk.vals[i], prev.n ? sp.vals[i] : 0ull, false, err);
      if (s == ~0ull) {
        atomicOr(err, err_bit(MS_E_CORRUPT));
        continue;
      }
      const uint64_t f = first[s];
      const uint64_t seg = f / kSegRows;
      uint64_t rank = seg_off[seg];
      const uint64_t w_end = f >> 5;
      for (uint64_t w = seg * kSegWords; w < w_end; ++w) rank += __popc(__ldg(bits + w));
      rank += __popc(__ldg(bits + w_end) & ((1u << (f & 31)) - 1u));
      ids[r0 + i] = rank;
    }
    __syncthreads();
  }
}

// join, build side: count the rows of every key
__global__ void __launch_bounds__(kThreads) join_count_kernel(ColView build, HT h, uint32_t* cnt, uint32_t* err) {
  __shared__ EngineSmem sm;
  const uint64_t n_tiles = (build.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t c = (uint32_t)min((uint64_t)kChunk, build.n - r0);
    load_rows(build, r0, c, sm);
    for (uint32_t i = threadIdx.x; i < c; i += kThreads) {
      const uint64_t s = ht_slot(h, sm.vals[i], 0, true, err);
      if (s != ~0ull) atomicAdd(cnt + s, 1u);
    }
    __syncthreads();
  }
}

// join, build side: every row into its key's range [off, off + cnt) (arbitrary order)
__global__ void __launch_bounds__(kThreads) join_place_kernel(ColView build, HT h, const uint64_t* off,
                                                              uint32_t* fill, uint64_t* rows, uint32_t* err) {
  __shared__ EngineSmem sm;
  const uint64_t n_tiles = (build.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t c = (uint32_t)min((uint64_t)kChunk, build.n - r0);
    load_rows(build, r0, c, sm);
    for (uint32_t i = threadIdx.x; i < c; i += kThreads) {
      const uint64_t s = ht_slot(h, sm.vals[i], 0, false, err);
      if (s == ~0ull) {
        atomicOr(err, err_bit(MS_E_CORRUPT));
        continue;
      }
      rows[off[s] + atomicAdd(fill + s, 1u)] = r0 + i;
    }
    __syncthreads();
  }
}

// join: each key's build rows in ascending order (the build-match order);
// insertion sort per key (keys of a star-schema dimension are unique: lists of 1)
__global__ void join_sort_kernel(uint64_t cap, const uint32_t* cnt, const uint64_t* off, uint64_t* rows) {
  for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < cap; s += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cnt[s];
    if (c < 2) continue;
    uint64_t* r = rows + off[s];
    for (uint32_t i = 1; i < c; ++i) {
      const uint64_t x = r[i];
      uint32_t j = i;
      for (; j > 0 && r[j - 1] > x; --j) r[j] = r[j - 1];
      r[j] = x;
    }
  }
}

// join, probe side: matches per 2048-row tile (pass 1), then the pairs in probe order
// (pass 2) at the tile's offset (exclusive scan of pass 1)
template <bool WRITE>
__global__ void __launch_bounds__(kThreads) join_probe_kernel(ColView probe, HT h, const uint32_t* cnt,
                                                              const uint64_t* off, const uint64_t* rows,
                                                              uint32_t* tile_cnt, const uint64_t* tile_off,
                                                              uint64_t* out_probe, uint64_t* out_build,
                                                              uint32_t* err) {
  __shared__ EngineSmem sm;
  __shared__ uint64_t scan_sm[16];
  const uint64_t n_tiles = (probe.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t c = (uint32_t)min((uint64_t)kChunk, probe.n - r0);
    load_rows(probe, r0, c, sm);
    // thread tid: rows [8 tid, 8 tid + 8) (probe order inside the tile)
    const uint32_t i0 = threadIdx.x * kVPT;
    uint64_t slot[kVPT];
    uint64_t m = 0;
#pragma unroll
    for (int q = 0; q < kVPT; ++q) {
      slot[q] = i0 + q < c ? ht_slot(h, sm.vals[i0 + q], 0, false, err) : ~0ull;
      m += slot[q] != ~0ull ? cnt[slot[q]] : 0u;
    }
    uint64_t tot = 0;
    const uint64_t ex = cta_excl_scan(m, scan_sm, &tot);
    if (!WRITE) {
      if (threadIdx.x == 0) {
        if (tot > 0xffffffffull) atomicOr(err, err_bit(MS_E_INVALID));  // > 2^32 - 1 pairs from one tile
        tile_cnt[t] = (uint32_t)tot;
      }
    } else {
      uint64_t o = tile_off[t] + ex;
#pragma unroll
      for (int q = 0; q < kVPT; ++q) {
        if (slot[q] == ~0ull) continue;
        const uint64_t b = off[slot[q]];
        const uint32_t k = cnt[slot[q]];
        for (uint32_t j = 0; j < k; ++j, ++o) {
          out_probe[o] = r0 + i0 + q;
          out_build[o] = rows[b + j];
        }
      }
    }
    __syncthreads();
  }
}

// calc: out[i] = a[i] op b[i] mod 2^64 (ADD 0, SUB 1, MUL 2)
__global__ void __launch_bounds__(kThreads) calc_kernel(ColView a, ColView b, int op, uint64_t* out) {
  __shared__ EngineSmem sa, sb;
  const uint64_t n_tiles = (a.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t c = (uint32_t)min((uint64_t)kChunk, a.n - r0);
    load_rows(a, r0, c, sa);
    load_rows(b, r0, c, sb);
    for (uint32_t i = threadIdx.x; i < c; i += kThreads) {
      const uint64_t x = sa.vals[i], y = sb.vals[i];
      out[r0 + i] = op == 0 ? x + y : (op == 1 ? x - y : x * y);
    }
    __syncthreads();
  }
}

inline uint64_t grid_min(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ------------------------------------------------------------ RLE encoding of a column source
// morph into RLE tile by tile (no uncompressed staging of the input, DP3): pass 1
// counts the run starts inside each 2048-row tile and records the tile's first /
// last value; rle_fix adds the starts at tile boundaries; after the scan, pass 2
// decodes the tile again and writes (value, start) of every run at its index.
__global__ void __launch_bounds__(kThreads) rle_count_col_kernel(ColView c, uint32_t* counts, uint64_t* first_last) {
  __shared__ EngineSmem sm;
  __shared__ uint32_t wsum[kThreads / 32];
  const uint64_t T = (c.n + kChunk - 1) / kChunk;
  for (uint64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, c.n - r0);
    load_rows(c, r0, cnt, sm);
    uint32_t k = 0;
    for (uint32_t i = threadIdx.x; i < cnt; i += kThreads) k += i == 0 ? (t == 0) : (sm.vals[i] != sm.vals[i - 1]);
    k = (uint32_t)warp_sum(k);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (int q = 0; q < kThreads / 32; ++q) s += wsum[q];
      counts[t] = s;
      first_last[2 * t] = sm.vals[0];
      first_last[2 * t + 1] = sm.vals[cnt - 1];
    }
    __syncthreads();
  }
}

__global__ void rle_fix_kernel(uint32_t* counts, const uint64_t* first_last, uint64_t T) {
  for (uint64_t t = 1 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (uint64_t)gridDim.x * blockDim.x)
    counts[t] += first_last[2 * t] != first_last[2 * t - 1];
}

__global__ void __launch_bounds__(kThreads) rle_write_col_kernel(ColView c, const uint64_t* first_last,
                                                                 const uint64_t* tile_off, uint64_t* payload,
                                                                 uint64_t* starts) {
  __shared__ EngineSmem sm;
  __shared__ uint32_t wcnt[kThreads / 32 + 1];
  const uint64_t T = (c.n + kChunk - 1) / kChunk;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint64_t r0 = t * kChunk;
    const uint32_t cnt = (uint32_t)min((uint64_t)kChunk, c.n - r0);
    load_rows(c, r0, cnt, sm);
    uint64_t base = tile_off[t];
    // rows in order, 256 at a time: ballot per warp, warp offsets by a small scan
    for (uint32_t i0 = 0; i0 < cnt; i0 += kThreads) {
      const uint32_t i = i0 + threadIdx.x;
      bool st = false;
      if (i < cnt) {
        const uint64_t prev = i > 0 ? sm.vals[i - 1] : (t > 0 ? first_last[2 * t - 1] : ~sm.vals[0]);
        st = sm.vals[i] != prev;
      }
      const uint32_t bal = __ballot_sync(kFull, st);
      if (lane == 0) wcnt[wid] = __popc(bal);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int q = 0; q < kThreads / 32; ++q) {
          const uint32_t x = wcnt[q];
          wcnt[q] = s;
          s += x;
        }
        wcnt[kThreads / 32] = s;
      }
      __syncthreads();
      if (st) {
        const uint64_t idx = base + wcnt[wid] + __popc(bal & ((1u << lane) - 1u));
        payload[2 * idx] = sm.vals[i];
        starts[idx] = r0 + i;
      }
      base += wcnt[kThreads / 32];
      __syncthreads();
    }
  }
}

template <class K>
int tiles_grid(K k, uint64_t n) {
  return persistent_grid(k, kThreads, (n + kChunk - 1) / kChunk);
}

}  // namespace

// ---------------------------------------------------------------- launchers
cudaError_t launch_profile(const ColView& c, uint32_t B, unsigned long long* acc, uint64_t* first_last,
                           cudaStream_t s) {
  if (!c.n) return cudaSuccess;
  {
    ProfScope prof_("profile", s);
    profile_kernel<<<tiles_grid(profile_kernel, c.n), kThreads, 0, s>>>(c, B, acc, first_last);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const uint64_t T = (c.n + kChunk - 1) / kChunk;
  ProfScope prof_("profile_runs", s);
  runs_kernel<<<(int)grid_min((T + 255) / 256, 1024), 256, 0, s>>>(first_last, T, acc);
  return cudaGetLastError();
}

cudaError_t launch_seg_count(const uint32_t* bits, uint64_t NS, uint32_t* cnt, cudaStream_t s) {
  if (!NS) return cudaSuccess;
  ProfScope prof_("seg_count", s);
  seg_count_kernel<<<(int)grid_min((NS + 255) / 256, (uint64_t)num_sms() * 16), 256, 0, s>>>(bits, NS, cnt);
  return cudaGetLastError();
}

cudaError_t launch_ends(const ColView& a, const ColView& b, uint64_t* out, cudaStream_t s) {
  ProfScope prof_("ends", s);
  ends_kernel<<<1, 32, 0, s>>>(a, b, out);
  return cudaGetLastError();
}

cudaError_t launch_pos_bitmap(const ColView& c, uint64_t base, uint64_t nbits, uint32_t* bits, uint64_t* first_last,
                              uint32_t* err, cudaStream_t s) {
  if (!c.n) return cudaSuccess;
  const uint64_t T = (c.n + kChunk - 1) / kChunk;
  {
    ProfScope prof_("pos_bitmap", s);
    pos_bitmap_kernel<<<tiles_grid(pos_bitmap_kernel, c.n), kThreads, 0, s>>>(c, base, nbits, bits, first_last, err);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || T < 2) return e;
  ProfScope prof_("sorted_check", s);
  sorted_check_kernel<<<(int)grid_min((T + 255) / 256, 1024), 256, 0, s>>>(first_last, T, err);
  return cudaGetLastError();
}

cudaError_t launch_bits_combine(uint32_t* a, const uint32_t* b, uint64_t n_words, int op, cudaStream_t s) {
  if (!n_words) return cudaSuccess;
  ProfScope prof_("bits_combine", s);
  bits_combine_kernel<<<(int)grid_min((n_words + 255) / 256, (uint64_t)num_sms() * 16), 256, 0, s>>>(a, b,
                                                                                                        n_words, op);
  return cudaGetLastError();
}

static HT make_ht(uint32_t* state, uint64_t* key, uint64_t* key2, uint64_t cap) { return HT{state, key, key2, cap - 1}; }

cudaError_t launch_group(const ColView& keys, const ColView& prev, uint32_t* state, uint64_t* key, uint64_t* key2,
                         uint64_t cap, unsigned long long* first, uint32_t* bits, uint32_t* err, cudaStream_t s) {
  const HT h = make_ht(state, key, key2, cap);
  {
    ProfScope prof_("group_insert", s);
    group_insert_kernel<<<tiles_grid(group_insert_kernel, keys.n), kThreads, 0, s>>>(keys, prev, h, first, err);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ProfScope prof_("group_mark", s);
  group_mark_kernel<<<(int)grid_min((cap + 255) / 256, (uint64_t)num_sms() * 16), 256, 0, s>>>(h, first, bits);
  return cudaGetLastError();
}

cudaError_t launch_group_ids(const ColView& keys, const ColView& prev, uint32_t* state, uint64_t* key, uint64_t* key2,
                             uint64_t cap, const unsigned long long* first, const uint32_t* bits,
                             const uint64_t* seg_off, uint64_t* ids, uint32_t* err, cudaStream_t s) {
  const HT h = make_ht(state, key, key2, cap);
  ProfScope prof_("group_ids", s);
  group_ids_kernel<<<tiles_grid(group_ids_kernel, keys.n), kThreads, 0, s>>>(keys, prev, h, first, bits, seg_off, ids,
                                                                              err);
  return cudaGetLastError();
}

cudaError_t launch_join_build(const ColView& build, uint32_t* state, uint64_t* key, uint64_t cap, uint32_t* cnt,
                              uint32_t* err, cudaStream_t s) {
  const HT h = make_ht(state, key, nullptr, cap);
  ProfScope prof_("join_count", s);
  join_count_kernel<<<tiles_grid(join_count_kernel, build.n), kThreads, 0, s>>>(build, h, cnt, err);
  return cudaGetLastError();
}

cudaError_t launch_join_place(const ColView& build, uint32_t* state, uint64_t* key, uint64_t cap, const uint32_t* cnt,
                              const uint64_t* off, uint32_t* fill, uint64_t* rows, uint32_t* err, cudaStream_t s) {
  const HT h = make_ht(state, key, nullptr, cap);
  {
    ProfScope prof_("join_place", s);
    join_place_kernel<<<tiles_grid(join_place_kernel, build.n), kThreads, 0, s>>>(build, h, off, fill, rows, err);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  ProfScope prof_("join_sort", s);
  join_sort_kernel<<<(int)grid_min((cap + 255) / 256, (uint64_t)num_sms() * 16), 256, 0, s>>>(cap, cnt, off,
                                                                                                  rows);
  return cudaGetLastError();
}

cudaError_t launch_join_probe(const ColView& probe, uint32_t* state, uint64_t* key, uint64_t cap, const uint32_t* cnt,
                              const uint64_t* off, const uint64_t* rows, uint32_t* tile_cnt, const uint64_t* tile_off,
                              uint64_t* out_probe, uint64_t* out_build, bool write, uint32_t* err, cudaStream_t s) {
  const HT h = make_ht(state, key, nullptr, cap);
  if (!probe.n) return cudaSuccess;
  if (write) {
    ProfScope prof_("join_probe_write", s);
    join_probe_kernel<true><<<tiles_grid(join_probe_kernel<true>, probe.n), kThreads, 0, s>>>(
        probe, h, cnt, off, rows, tile_cnt, tile_off, out_probe, out_build, err);
  } else {
    ProfScope prof_("join_probe_count", s);
    join_probe_kernel<false><<<tiles_grid(join_probe_kernel<false>, probe.n), kThreads, 0, s>>>(
        probe, h, cnt, off, rows, tile_cnt, tile_off, out_probe, out_build, err);
  }
  return cudaGetLastError();
}

cudaError_t launch_rle_count_col(const ColView& c, uint32_t* counts, uint64_t* first_last, cudaStream_t s) {
  const uint64_t T = (c.n + kChunk - 1) / kChunk;
  if (!T) return cudaSuccess;
  {
    ProfScope prof_("rle_count_col", s);
    rle_count_col_kernel<<<tiles_grid(rle_count_col_kernel, c.n), kThreads, 0, s>>>(c, counts, first_last);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || T < 2) return e;
  ProfScope prof_("rle_fix", s);
  rle_fix_kernel<<<(int)grid_min((T + 255) / 256, 1024), 256, 0, s>>>(counts, first_last, T);
  return cudaGetLastError();
}

cudaError_t launch_rle_write_col(const ColView& c, const uint64_t* first_last, const uint64_t* tile_off,
                                 uint64_t* payload, uint64_t* starts, cudaStream_t s) {
  if (!c.n) return cudaSuccess;
  ProfScope prof_("rle_write_col", s);
  rle_write_col_kernel<<<tiles_grid(rle_write_col_kernel, c.n), kThreads, 0, s>>>(c, first_last, tile_off, payload,
                                                                                  starts);
  return cudaGetLastError();
}

cudaError_t launch_calc(const ColView& a, const ColView& b, int op, uint64_t* out, cudaStream_t s) {
  if (!a.n) return cudaSuccess;
  ProfScope prof_("calc", s);
  calc_kernel<<<tiles_grid(calc_kernel, a.n), kThreads, 0, s>>>(a, b, op, out);
  return cudaGetLastError();
}

}  // namespace ms
