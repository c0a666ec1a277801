// select_pos.cu — select -> DELTA_BP{512} positions in ONE pass over the input
// (SURVEY.md §7 H1). The paper's operator with on-the-fly de/re-compression
// (P:297-337, 468-505): the input-side buffer layer decompresses a block into
// a cache-resident buffer, the core evaluates the predicate and
// compacts the matches with a bit mask, and the output-side buffer
// layer recompresses the positions once a block is full and writes the final
// partial block uncompressed. DELTA_BP is the paper's recommended
// positions format ("the output is always sorted").
//
// One persistent CTA per SM, three warp roles, tiles of TS 512-row segments
// (32K..256K rows, sized so every SM gets several) taken in order from an
// atomic ticket:
//   producer  (1 warp)  streams each tile's compressed payload into a shared-
//                       memory ring, one TMA bulk copy per stage of 16
//                       segments (the segments of a stage are contiguous in
//                       every supported layout); block headers (widths, FOR
//                       references) are loaded one stage ahead;
//   scanners  (8 warps)  unpack with a compile-time bit width (select_fast.cuh),
//                       evaluate the predicate in the code domain and write one
//                       32-bit mask word per 32 rows and one count per segment
//                       into the tile's shared-memory mask (double-buffered;
//                       the mask never reaches HBM). The last scanner warp to
//                       finish a tile turns the segment counts into prefixes
//                       and publishes the tile count (decoupled look-back #1
//                       aggregate) at once — independent of the encoders;
//   encoders  (8 warps)  per tile: its last B-1 positions to a small scratch
//                       ("tail", flagged), look-back #1 -> output rank O_t, the
//                       head of the first owned block from the predecessors'
//                       tails, the widths w_k = ebw(max delta) of the owned
//                       blocks (D-6, blocks spread over the warps), look-back #2
//                       on the width sum -> the tile's cw offset (D-4), then
//                       every owned block packed in shared memory and stored
//                       once at its final place. Block k (ranks [kB, kB+B)) is
//                       owned by the tile holding rank kB+B-1; the last tile
//                       writes the final partial block raw.
// HBM traffic: the compressed input once and the positions image once, plus per
// tile < B u32 of tail and a few status words. No bit mask, no per-block slots,
// no copy pass.
#include "common.cuh"
#include "grid.cuh"
#include "launch.h"
#include "select_fast.cuh"
#include "tma.cuh"

namespace ms {

// instrumentation (ms_debug_trace): when non-null, 16 u64 per tile (8 %globaltimer stamps, 8 counters)
__device__ uint64_t* g_sp_trace = nullptr;

namespace {

__device__ __forceinline__ void trace(uint64_t t, int k) {
  if (g_sp_trace && (threadIdx.x & 31) == 0) {
    uint64_t ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    g_sp_trace[t * 16 + k] = ns;
  }
}
__device__ __forceinline__ void trace_val(uint64_t t, int k, uint64_t v) {
  if (g_sp_trace && (threadIdx.x & 31) == 0) g_sp_trace[t * 16 + k] = v;
}

constexpr int kB = 512;                        // output block (positions per DELTA block)
constexpr int kPer = kB / 32;                  // ranks per lane in a block
constexpr int kNSW = 8;                        // scanner warps
constexpr int kNE = 8;                         // encoder warps
constexpr int kSP = 2 * kNSW;                  // segments per stage
constexpr int kThreadsSP = (kNSW + kNE + 1) * 32;
constexpr int kMaxTS = 512;                    // segments per tile (max)
constexpr int kMaxWords = kMaxTS * kSegWords;  // mask words per tile (max)
constexpr int kMaxStages = 8;
constexpr int kEncBar = 1;                     // named barrier of the encoder warps
constexpr uint64_t kNone = ~0ull;

struct SpArgs {
  ColView c;
  FastPred pred;
  uint64_t n, NS, ns_fast, T, row_offset;
  uint32_t TS;          // segments per tile (power of two, 64..512)
  uint32_t stage_u32, nst;
  uint32_t* ticket;
  uint64_t* st1;        // look-back on the tile counts (T words, zeroed)
  uint64_t* st2;        // look-back on the tile width sums (T words, zeroed)
  uint32_t* cnt;        // tile counts (T)
  uint32_t* tflag;      // tail written (T, zeroed)
  uint32_t* tail;       // per tile: its last min(count, B-1) rows (relative to the tile)
  uint64_t* meta;       // [0] err word, [1] n_out, [2] cw[nb], [3] max block width (zeroed)
  uint32_t* err;
  uint64_t* payload;
  uint32_t* cw;
  uint64_t* ref;
  uint64_t* rem;
  uint64_t cap_words;   // payload capacity
};

struct SpSmem {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t mfull[2], mempty[2];
  uint64_t stile[kMaxStages];  // tile of the stage (kNone: no more tiles)
  uint32_t sidx[kMaxStages];   // stage index inside its tile
  uint32_t sw[kMaxStages][kSP];
  uint32_t soff[kMaxStages][kSP];
  uint64_t sref[kMaxStages][kSP];
  uint64_t mtile[2];           // tile of the mask buffer (kNone: stop)
  uint32_t tc[2];              // tile count
  uint32_t sdone[2];           // scanner warps done with the buffer's tile
  uint16_t segcnt[2][kMaxTS];
  uint32_t spre[2][kMaxTS + 1];  // exclusive prefix of the segment counts
  alignas(16) uint32_t mask[2][kMaxWords];
  // encoders
  uint64_t hbuf[kB];                   // head: ranks [k_a B, O_t) as local rows
  alignas(16) uint64_t stg[kNE][kB + kB / 16];  // per encoder warp: a block's positions, then its codes
  uint32_t wl[kMaxTS * kSegRows / kB + 2];  // widths of the owned blocks -> exclusive prefix
  uint64_t eO, eC;                     // the tile's output rank and cw offset
  uint32_t eW;
};

constexpr size_t sp_static_bytes() { return (sizeof(SpSmem) + 127) & ~(size_t)127; }

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ bool fast_keep(const FastPred& pr, uint64_t v) {
  if (pr.is_bitmap) return v < pr.bits && ((__ldg(pr.bitmap + (v >> 6)) >> (v & 63)) & 1ull);
  return ((v - pr.lo) <= pr.span) != (pr.neg != 0);
}

// widths 0..32 only (the narrow variant: every block width <= 32 by the max_width hint)
__device__ __forceinline__ uint32_t lane_dispatch_narrow(uint32_t w, const uint32_t* p, const FastPred& pr,
                                                         uint64_t ref) {
  switch (w) {
#define MS_NARROW_CASE(W) \
  case W:                 \
    return lane_rows<W>(p, pr, ref);
    MS_NARROW_CASE(0) MS_NARROW_CASE(1) MS_NARROW_CASE(2) MS_NARROW_CASE(3) MS_NARROW_CASE(4)
    MS_NARROW_CASE(5) MS_NARROW_CASE(6) MS_NARROW_CASE(7) MS_NARROW_CASE(8) MS_NARROW_CASE(9)
    MS_NARROW_CASE(10) MS_NARROW_CASE(11) MS_NARROW_CASE(12) MS_NARROW_CASE(13) MS_NARROW_CASE(14)
    MS_NARROW_CASE(15) MS_NARROW_CASE(16) MS_NARROW_CASE(17) MS_NARROW_CASE(18) MS_NARROW_CASE(19)
    MS_NARROW_CASE(20) MS_NARROW_CASE(21) MS_NARROW_CASE(22) MS_NARROW_CASE(23) MS_NARROW_CASE(24)
    MS_NARROW_CASE(25) MS_NARROW_CASE(26) MS_NARROW_CASE(27) MS_NARROW_CASE(28) MS_NARROW_CASE(29)
    MS_NARROW_CASE(30) MS_NARROW_CASE(31) MS_NARROW_CASE(32)
#undef MS_NARROW_CASE
    default:
      return 0;
  }
}

__device__ __forceinline__ void enc_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(kEncBar), "n"(kNE * 32) : "memory");
}

// Exclusive prefix of item t from the status words of its predecessors (flag in
// [63:62]: 1 aggregate, 2 inclusive prefix). Lane j reads item base - j; the
// walk stops at the nearest inclusive prefix as soon as every item between it
// and t is published (it never waits on items behind that prefix). All 32 lanes.
__device__ __forceinline__ uint64_t sp_walk(const uint64_t* status, uint64_t t) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = (int64_t)t - 1;
  while (true) {
    const int64_t idx = base - (int64_t)lane;
    uint64_t s = idx >= 0 ? ld_volatile(status + idx) : kFlagP;
    int spins = 0;
    while (true) {
      const uint32_t pm = __ballot_sync(kFull, (s >> 62) == 2);
      const uint32_t vm = __ballot_sync(kFull, (s >> 62) != 0);
      const uint32_t stop = pm & (0u - pm);                        // nearest inclusive prefix (0: none)
      const uint32_t need = stop ? (stop | (stop - 1)) : kFull;    // lanes up to it
      if ((vm & need) == need) {
        const uint64_t v = ((need >> lane) & 1u) ? (s & kValMask) : 0ull;
        excl += warp_sum(v);
        if (stop) return excl & kValMask;
        break;
      }
      if (++spins > 8) __nanosleep(20);
      if ((s >> 62) == 0 && idx >= 0) s = ld_volatile(status + idx);
    }
    base -= 32;
  }
}

// item 0 publishes its inclusive prefix directly; every other item publishes its
// aggregate (sp_publish, after a fence over the caller's data), then resolves
// (sp_resolve: walk, fence, inclusive prefix)
__device__ __forceinline__ void sp_publish(uint64_t* status, uint64_t t, uint64_t agg) {
  __threadfence();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) st_volatile(status + t, (t == 0 ? kFlagP : kFlagA) | agg);
}
__device__ __forceinline__ uint64_t sp_resolve(uint64_t* status, uint64_t t, uint64_t agg) {
  if (t == 0) return 0;
  const uint64_t excl = sp_walk(status, t);
  __threadfence();
  if ((threadIdx.x & 31) == 0) st_volatile(status + t, kFlagP | ((excl + agg) & kValMask));
  return excl;
}

// ------------------------------------------------------------ mask walking
// A tile's mask: spre[s] = matches before segment s; segment s's words at [16 s, 16 s + 16).
// The word holding tile rank r (< the tile's count), and the matches before that word.
__device__ __forceinline__ void locate_word(const uint32_t* M, const uint32_t* spre, uint32_t nseg, uint32_t r,
                                            uint32_t& m, uint32_t& pre) {
  uint32_t s = 0;
#pragma unroll
  for (uint32_t step = kMaxTS / 2; step; step >>= 1)
    if (s + step < nseg && spre[s + step] <= r) s += step;
  pre = spre[s];
  m = s * kSegWords;
  const uint4* g4 = reinterpret_cast<const uint4*>(M + m);
#pragma unroll 1
  for (int q = 0; q < kSegWords / 4 - 1; ++q) {  // whole groups of four words
    const uint4 v = g4[q];
    const uint32_t pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    if (r - pre < pc) break;
    pre += pc;
    m += 4;
  }
  while (true) {
    const uint32_t pc = __popc(M[m]);
    if (r - pre < pc) break;
    pre += pc;
    ++m;
  }
}

// staging slot of rank q of a block: one u64 of padding per 16, so that lane j's 16
// consecutive ranks start 17 u64 apart (at most 2-way bank conflicts)
__device__ __forceinline__ uint32_t sidx16(uint32_t q) { return q + (q >> 4); }

// Tile ranks [r0, r0 + cnt) (cnt >= 1) -> st[sidx16(off + i)] = row0 + local row of rank
// r0 + i. Word-parallel: the mask words spanning the ranks are cut into 32 contiguous
// chunks; chunk popcounts and a warp scan give every lane the rank of its first
// match, then each lane scatters its own matches. All 32 lanes; ends with __syncwarp.
__device__ __forceinline__ void extract_ranks(const uint32_t* __restrict__ M, const uint32_t* __restrict__ spre,
                                              uint32_t nseg, uint32_t r0, uint32_t cnt, uint64_t row0,
                                              uint64_t* st, uint32_t off, uint32_t lane, int64_t dbg_t = -1) {
  const uint64_t c0 = clock64();
  uint32_t m = 0, pre = 0;
  if (lane < 2) locate_word(M, spre, nseg, lane ? r0 + cnt - 1 : r0, m, pre);
  const uint32_t wa = __shfl_sync(kFull, m, 0), preA = __shfl_sync(kFull, pre, 0);
  const uint32_t wb = __shfl_sync(kFull, m, 1);
  const uint32_t K = (wb - wa + 32) >> 5;  // words per lane
  const uint32_t w0 = wa + lane * K;
  const uint32_t w1 = min(w0 + K, wb + 1);
  uint32_t c = 0;
  for (uint32_t w = w0; w < w1; ++w) c += __popc(M[w]);
  uint32_t inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, inc, o);
    if (lane >= (uint32_t)o) inc += y;
  }
  uint32_t r = preA + inc - c;  // rank of the lane's first match
  const uint32_t r1 = r0 + cnt;
  const uint64_t c1 = clock64();
  for (uint32_t w = w0; w < w1 && r < r1; ++w) {
    uint32_t x = M[w];
    if (r < r0) {  // matches below the range (first word only)
      const uint32_t pc = __popc(x);
      if (r + pc <= r0) {
        r += pc;
        continue;
      }
      for (; r < r0; ++r) x &= x - 1;
    }
    while (x && r < r1) {
      const uint32_t b = __ffs(x) - 1;
      x &= x - 1;
      st[sidx16(off + r - r0)] = row0 + w * 32 + b;
      ++r;
    }
  }
  __syncwarp();
  if (dbg_t >= 0) {
    trace_val(dbg_t, 8, c1 - c0);
    trace_val(dbg_t, 9, clock64() - c1);
    trace_val(dbg_t, 13, wb - wa + 1);
  }
}

// ------------------------------------------------------------------ encoders
__device__ __forceinline__ void sp_encode_tile(const SpArgs& a, SpSmem& S, uint32_t bq, uint64_t t, uint32_t e,
                                               uint32_t lane) {
  const uint64_t TR = (uint64_t)a.TS * kSegRows;
  const uint64_t row0 = t * TR;
  const uint32_t c = S.tc[bq];
  const bool last = t == a.T - 1;
  const uint32_t* M = S.mask[bq];
  const uint32_t* spre = S.spre[bq];
  const uint32_t nseg = a.TS;
  uint64_t* st = S.stg[e];

  // 1. warp 0: tail (then its flag), look-back #1, head
  if (e == 0) {
    trace(t, 1);
    const uint32_t L = c < (uint32_t)(kB - 1) ? c : (uint32_t)(kB - 1);
    if (L) {
      extract_ranks(M, spre, nseg, c - L, L, 0, st, 0, lane);
      uint32_t* tb = a.tail + t * (uint64_t)(kB - 1);
      for (uint32_t i = lane; i < L; i += 32) tb[i] = (uint32_t)st[sidx16(i)];
      __syncwarp();
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_relaxed_u32(a.tflag + t, 1u);
    trace(t, 2);
    const uint64_t O = sp_resolve(a.st1, t, c);
    trace(t, 3);
    const uint64_t ka = O / kB, kb = (O + c) / kB;
    const uint32_t h = (uint32_t)(O - ka * kB);
    if (h && (kb > ka || last)) {  // the head: ranks [ka B, O) from the predecessors' tails, newest first
      uint32_t need = h;
      int64_t j = (int64_t)t - 1;
      while (need && j >= 0) {
        const int64_t jl = j - (int64_t)lane;
        const uint32_t cj = jl >= 0 ? __ldcg(a.cnt + jl) : 0u;
        for (int l = 0; l < 32 && need && j - l >= 0; ++l) {
          const uint32_t cl = __shfl_sync(kFull, cj, l);
          if (!cl) continue;
          const uint64_t tj = (uint64_t)(j - l);
          if (lane == 0) {
            int spins = 0;
            while (ld_relaxed_u32(a.tflag + tj) == 0)
              if (++spins > 8) __nanosleep(20);
          }
          __syncwarp();
          __threadfence();
          const uint32_t take = cl < need ? cl : need;
          const uint32_t Lj = cl < (uint32_t)(kB - 1) ? cl : (uint32_t)(kB - 1);
          const uint32_t* tb = a.tail + tj * (uint64_t)(kB - 1) + (Lj - take);
          for (uint32_t i = lane; i < take; i += 32) S.hbuf[need - take + i] = tj * TR + __ldcg(tb + i);
          need -= take;
        }
        j -= 32;
      }
      if (need && lane == 0) atomicOr(a.err, err_bit(MS_E_CORRUPT));  // fewer earlier matches than ranks
    }
    if (lane == 0) {
      S.eO = O;
      if (last) a.meta[1] = O + c;
    }
    trace(t, 4);
  }
  enc_sync();
  const uint64_t O = S.eO;
  const uint64_t ka = O / kB, kb = (O + c) / kB;
  const uint32_t nbk = (uint32_t)(kb - ka);

  // global ranks [g0, g0 + n) into the staging buffer (slot i = rank g0 + i):
  // ranks below O from the head, the others from this tile's mask
  auto fill = [&](uint64_t g0, uint32_t n, int64_t dbg_t = -1) {
    const uint64_t own0 = g0 > O ? g0 : O;
    const uint32_t nh = (uint32_t)(own0 - g0);
    for (uint32_t i = lane; i < nh; i += 32) st[sidx16(i)] = S.hbuf[g0 + i - ka * kB];
    if (n > nh) extract_ranks(M, spre, nseg, (uint32_t)(own0 - O), n - nh, row0, st, nh, lane, dbg_t);
    __syncwarp();
  };
  // lane j: positions of ranks [16j, 16j+16) -> deltas in place (d_0 = 0 at the block
  // start, D-6); returns the block width
  auto deltas = [&](uint64_t (&p)[kPer]) -> uint32_t {
#pragma unroll
    for (int i = 0; i < kPer; ++i) p[i] = st[sidx16(kPer * lane + i)];
    const uint64_t prev = __shfl_up_sync(kFull, p[kPer - 1], 1);
    uint64_t mx = 0;
#pragma unroll
    for (int i = kPer - 1; i >= 1; --i) {
      p[i] -= p[i - 1];
      mx = p[i] > mx ? p[i] : mx;
    }
    p[0] = lane ? p[0] - prev : 0ull;
    mx = p[0] > mx ? p[0] : mx;
    return __reduce_max_sync(kFull, ebw64(mx));
  };

  // 2. pass 1: widths of the owned blocks (spread over the encoder warps)
  const uint64_t p1c0 = clock64();
  for (uint32_t i = e; i < nbk; i += kNE) {
    const uint64_t b0 = clock64();
    const bool dbg = e == 1 && i == 1 + kNE;
    fill((ka + i) * kB, kB, dbg ? (int64_t)t : -1);
    const uint64_t b1 = clock64();
    uint64_t p[kPer];
    const uint32_t w = deltas(p);
    if (lane == 0) S.wl[i] = w;
    __syncwarp();
    if (dbg) {
      trace_val(t, 10, b1 - b0);
      trace_val(t, 11, clock64() - b1);
    }
  }
  if (e == 1) {
    trace_val(t, 12, clock64() - p1c0);
    trace_val(t, 14, nbk);
  }
  enc_sync();
  if (e == 0) trace(t, 5);

  // 3. warp 0: prefix of the widths, look-back #2
  if (e == 0) {
    uint32_t W = 0, wmax = 0;
    for (uint32_t i0 = 0; i0 < nbk; i0 += 32) {
      const uint32_t w = i0 + lane < nbk ? S.wl[i0 + lane] : 0u;
      uint32_t inc = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= (uint32_t)o) inc += y;
      }
      if (i0 + lane < nbk) S.wl[i0 + lane] = W + inc - w;
      W += __shfl_sync(kFull, inc, 31);
      wmax = max(wmax, __reduce_max_sync(kFull, w));
    }
    sp_publish(a.st2, t, W);
    const uint64_t C = sp_resolve(a.st2, t, W);
    trace(t, 6);
    if (lane == 0) {
      S.eC = C;
      S.eW = W;
      if (C + W > 0xffffffffull || (C + W) * (kB / 64) > a.cap_words) atomicOr(a.err, err_bit(MS_E_INVALID));
      if (wmax) atomicMax(reinterpret_cast<unsigned long long*>(a.meta + 3), (unsigned long long)wmax);
      if (last) a.meta[2] = C + W;
    }
  }
  enc_sync();
  const uint64_t C = S.eC;
  const uint32_t W = S.eW;
  const bool fits = (C + W) * (kB / 64) <= a.cap_words && C + W <= 0xffffffffull;

  // 4. pass 2: every owned block packed in place (staging -> codes), one coalesced store
  //    at cw[k] * B / 64
  for (uint32_t i = e; fits && i < nbk; i += kNE) {
    const uint64_t k = ka + i;
    fill(k * kB, kB);
    const uint64_t base = st[0];
    uint64_t p[kPer];
    const uint32_t w = deltas(p);
    const uint64_t cwk = C + S.wl[i];
    __syncwarp();
    uint32_t* buf = reinterpret_cast<uint32_t*>(st);
    const uint32_t n32 = (uint32_t)(kB / 32) * w;
    for (uint32_t q = lane; q < n32; q += 32) buf[q] = 0;
    __syncwarp();
    stream_codes<kPer>(buf, p, w, kPer * lane * w);
    __syncwarp();
    const uint32_t n16 = (uint32_t)(kB / 128) * w;  // 16-byte units
    uint4* dst = reinterpret_cast<uint4*>(a.payload + cwk * (kB / 64));
    const uint4* src = reinterpret_cast<const uint4*>(buf);
    for (uint32_t q = lane; q < n16; q += 32) dst[q] = src[q];
    if (lane == 0) {
      a.cw[k + 1] = (uint32_t)(cwk + w);
      a.ref[k] = base + a.row_offset;
    }
    __syncwarp();
  }

  // 5. the last tile: the final partial block, raw
  if (e == 0 && last) {
    const uint32_t R = (uint32_t)(O + c - kb * kB);
    if (R) {
      fill(kb * kB, R);
      for (uint32_t i = lane; i < R; i += 32) a.rem[i] = a.row_offset + st[sidx16(i)];
    }
  }
  enc_sync();
  if (e == 0) trace(t, 7);
}

// -------------------------------------------------------------------- kernel
template <int KIND, bool NARROW>
__global__ void __launch_bounds__(kThreadsSP, 1) select_pos_kernel(SpArgs a) {
  extern __shared__ __align__(128) unsigned char sp_dyn[];
  SpSmem& S = *reinterpret_cast<SpSmem*>(sp_dyn);
  uint32_t* ring = reinterpret_cast<uint32_t*>(sp_dyn + sp_static_bytes());
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t nst = a.nst, SPT = a.TS / kSP;  // stages per tile
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < nst; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], kNSW);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&S.mfull[i], 1);
      mbar_init(&S.mempty[i], 1);
      S.sdone[i] = 0;
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (wid == kNSW + kNE) {
    // ------------------------------------------------------------ producer
    // segment meta: width, payload word offset, FOR reference (0 if not staged)
    auto meta = [&](uint64_t s, uint32_t& w, uint64_t& off, uint64_t& ref) {
      w = 0;
      off = 0;
      ref = 0;
      if (lane >= (uint32_t)kSP || s >= a.ns_fast) return;
      if constexpr (KIND == FAST_UNCOMPR) {
        w = 64;
        off = s * (uint64_t)kSegRows;
      } else if constexpr (KIND == FAST_STATIC) {
        w = a.c.w;
        off = s * 8 * (uint64_t)w;
      } else {
        const uint64_t b = (s << 9) >> a.c.log2B;
        const uint32_t cw0 = __ldg(a.c.cw + b);
        w = __ldg(a.c.cw + b + 1) - cw0;
        off = (uint64_t)cw0 * (a.c.B >> 6) + (s & ((a.c.B >> 9) - 1)) * 8 * (uint64_t)w;
        if (a.c.ref) ref = __ldg(a.c.ref + b);
      }
    };
    auto take = [&]() {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(a.ticket, 1u);
      return (uint64_t)__shfl_sync(kFull, t, 0);
    };
    uint64_t g = 0;
    uint64_t t = take();
    uint32_t si = 0;
    uint32_t nw = 0;
    uint64_t noff = 0, nref = 0;
    if (t < a.T) meta(t * a.TS + lane, nw, noff, nref);
    while (true) {
      const uint32_t st = (uint32_t)(g % nst);
      if (g >= nst) mbar_wait(&S.empty[st], (uint32_t)((g / nst) - 1) & 1u);
      if (t >= a.T) {  // no more tiles
        if (lane == 0) {
          S.stile[st] = kNone;
          mbar_arrive(&S.full[st]);
        }
        break;
      }
      uint32_t w = nw;
      const uint64_t off = noff, ref = nref;
      const uint64_t s = t * a.TS + si * kSP + lane;
      const bool in = lane < (uint32_t)kSP && s < a.ns_fast;
      const uint64_t t_cur = t;
      const uint32_t si_cur = si;
      if (++si == SPT) {  // the next stage's headers are loaded while this stage is issued
        si = 0;
        t = take();
      }
      if (t < a.T) meta(t * a.TS + si * kSP + lane, nw, noff, nref);
      const uint32_t cap_w = NARROW ? 32u : 64u;
      if (w > cap_w && in) {  // corrupt width table, or a width above the max_width hint
        atomicOr(a.err, err_bit(MS_E_CORRUPT));
        w = 65;
      }
      const uint32_t bytes = (in && w <= cap_w) ? 64 * w : 0u;
      uint32_t inc = bytes;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= (uint32_t)o) inc += y;
      }
      uint32_t total = __shfl_sync(kFull, inc, 31);
      const uint64_t off0 = __shfl_sync(kFull, off, 0);
      if (total > 4 * a.stage_u32) {  // cannot happen with a correct hint; never overrun the stage
        if (lane == 0) atomicOr(a.err, err_bit(MS_E_CORRUPT));
        w = 65;
        total = 0;
      }
      if (lane < (uint32_t)kSP) {
        S.sw[st][lane] = w;
        S.soff[st][lane] = (inc - bytes) >> 2;
        S.sref[st][lane] = ref;
      }
      __syncwarp();
      if (lane == 0) {
        S.stile[st] = t_cur;
        S.sidx[st] = si_cur;
        mbar_arrive_tx(&S.full[st], total);
        if (total) bulk_g2s(ring + (size_t)st * a.stage_u32, a.c.payload + off0, total, &S.full[st]);
      }
      __syncwarp();
      ++g;
    }
  } else if (wid < kNSW) {
    // ------------------------------------------------------------ scanners
    const uint32_t half = lane >> 4, hl = lane & 15;
    uint64_t g = 0;
    uint32_t q = 0;
    while (true) {
      const uint32_t st = (uint32_t)(g % nst);
      mbar_wait(&S.full[st], (uint32_t)(g / nst) & 1u);
      const uint64_t t = S.stile[st];
      const uint32_t bq = q & 1;
      if (t == kNone) {  // no more tiles: a stop mark for the encoders
        if (q >= 2) mbar_wait(&S.mempty[bq], ((q >> 1) - 1) & 1u);
        if (lane == 0) {
          const uint32_t old = atomicAdd(&S.sdone[bq], 1u);
          if (old == kNSW - 1) {
            S.mtile[bq] = kNone;
            mbar_arrive(&S.mfull[bq]);
          }
        }
        break;
      }
      const uint32_t si = S.sidx[st];
      if (si == 0 && q >= 2) mbar_wait(&S.mempty[bq], ((q >> 1) - 1) & 1u);
      const uint32_t sl = wid * 2 + half;  // segment in the stage
      const uint32_t seg = si * kSP + sl;  // segment in the tile
      const uint64_t s = t * a.TS + seg;
      uint32_t m = 0;
      if (s < a.ns_fast) {
        const uint32_t w = S.sw[st][sl];
        const uint32_t* p = ring + (size_t)st * a.stage_u32 + S.soff[st][sl] + hl * (w <= 64 ? w : 0);
        const uint64_t ref = S.sref[st][sl];
        if constexpr (KIND == FAST_UNCOMPR) m = w == 64 ? lane_rows_wide<64>(p, a.pred, 0) : 0u;
        else if constexpr (NARROW) m = lane_dispatch_narrow(w, p, a.pred, ref);
        else m = lane_dispatch(w, p, a.pred, ref);
      } else if (s < a.NS) {  // rows beyond the staged segments (partial segment, block remainder)
        const uint64_t r0 = s * kSegRows + hl * 32;
        for (int i = 0; i < 32; ++i)
          if (r0 + i < a.n && fast_keep(a.pred, read_row(a.c, r0 + i))) m |= 1u << i;
      }
      S.mask[bq][seg * kSegWords + hl] = m;
      uint32_t cnt = __popc(m);
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
      if (hl == 0) S.segcnt[bq][seg] = (uint16_t)cnt;
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[st]);
      if (si == SPT - 1) {  // this warp is done with the tile; the last one publishes its count
        uint32_t old = 0;
        if (lane == 0) {
          __threadfence_block();
          old = atomicAdd(&S.sdone[bq], 1u);
        }
        old = __shfl_sync(kFull, old, 0);
        if (old == kNSW - 1) {
          __threadfence_block();
          const uint32_t per = a.TS / 32;  // segments per lane
          uint32_t loc = 0;
          for (uint32_t k = 0; k < per; ++k) loc += S.segcnt[bq][lane * per + k];
          uint32_t inc = loc;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, inc, o);
            if (lane >= (uint32_t)o) inc += y;
          }
          uint32_t run = inc - loc;
          for (uint32_t k = 0; k < per; ++k) {
            S.spre[bq][lane * per + k] = run;
            run += S.segcnt[bq][lane * per + k];
          }
          const uint32_t c = __shfl_sync(kFull, inc, 31);
          if (lane == 0) {
            S.spre[bq][a.TS] = c;
            S.tc[bq] = c;
            S.mtile[bq] = t;
            S.sdone[bq] = 0;
            a.cnt[t] = c;
          }
          sp_publish(a.st1, t, c);  // look-back #1 aggregate, as soon as the mask is complete
          trace(t, 0);
          __syncwarp();
          if (lane == 0) mbar_arrive(&S.mfull[bq]);
        }
        ++q;
      }
      ++g;
    }
  } else {
    // ------------------------------------------------------------ encoders
    const uint32_t e = wid - kNSW;
    for (uint32_t q = 0;; ++q) {
      const uint32_t bq = q & 1;
      mbar_wait(&S.mfull[bq], (q >> 1) & 1u);
      const uint64_t t = S.mtile[bq];
      if (t == kNone) break;
      sp_encode_tile(a, S, bq, t, e, lane);
      if (e == 0 && lane == 0) mbar_arrive(&S.mempty[bq]);
    }
  }
}

template <int KIND, bool NARROW>
cudaError_t sp_launch(const SpArgs& a0, uint32_t maxw_cap, cudaStream_t s) {
  SpArgs a = a0;
  auto k = select_pos_kernel<KIND, NARROW>;
  a.stage_u32 = kSP * (kSegRows / 32) * maxw_cap + 16;  // + padding (keeps 16-byte alignment)
  const size_t fixed = sp_static_bytes();
  int dev = 0, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const size_t avail = (size_t)smem_max > fixed ? (size_t)smem_max - fixed : 0;
  uint32_t nst = (uint32_t)(avail / (4ull * a.stage_u32));
  if (nst > 6) nst = 6;
  if (nst < 2) return cudaErrorInvalidConfiguration;
  a.nst = nst;
  const size_t smem = fixed + (size_t)nst * 4 * a.stage_u32;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  uint64_t grid = (uint64_t)num_sms();
  if (grid > a.T) grid = a.T;
  ProfScope prof_("select_pos", s);
  k<<<(int)grid, kThreadsSP, smem, s>>>(a);
  return cudaGetLastError();
}

// input kinds of the one-pass path: the select_fast layouts (STATIC_BP, UNCOMPR,
// DYN_BP / FOR_BP with B >= 512); ns_fast = the full 512-row segments they stage
int sp_kind(const ColView& c, uint64_t* ns_fast) {
  if (c.format == MS_UNCOMPR) { *ns_fast = c.n / kSegRows; return FAST_UNCOMPR; }
  if (c.format == MS_STATIC_BP) { *ns_fast = c.n / kSegRows; return FAST_STATIC; }
  if ((c.format == MS_DYN_BP || c.format == MS_FOR_BP) && c.B >= (uint32_t)kSegRows) {
    *ns_fast = (c.nb << c.log2B) / kSegRows;
    return FAST_BLOCK;
  }
  return -1;
}

}  // namespace

// segments per tile: the largest power of two in [64, 512] that still gives every
// SM at least four tiles (fewer, larger tiles amortise the two look-backs)
uint32_t select_pos_tile_segs(uint64_t n) {
  const uint64_t NS = (n + kSegRows - 1) / kSegRows;
  uint32_t ts = kMaxTS;
  while (ts > 64 && NS < (uint64_t)ts * 4 * num_sms()) ts >>= 1;
  return ts;
}

uint64_t select_pos_tiles(uint64_t n) {
  const uint64_t TR = (uint64_t)select_pos_tile_segs(n) * kSegRows;
  return (n + TR - 1) / TR;
}

bool select_pos_supported(const ColView& c, uint32_t B) {
  uint64_t ns = 0;
  return B == (uint32_t)kB && c.n > 0 && sp_kind(c, &ns) >= 0;
}

// Upper bound of sum_k w_k over the full blocks of any DELTA_BP{B} positions
// column drawn from n rows: m blocks, block k's B-1 deltas are >= 1 and its
// max delta x_k <= span_k - (B-2), sum_k span_k <= n - m, so sum_k x_k <=
// n - m(B-1) and sum_k ebw(x_k) <= m + m log2((n - m(B-1)) / m) (Jensen),
// bounded over m in 4096 intervals (the bound is monotone in each factor).
uint64_t select_pos_width_bound(uint64_t n, uint32_t B) {
  const uint64_t M = n / B;
  if (M == 0) return 0;
  const uint64_t steps = M < 4096 ? M : 4096;
  double best = 0;
  for (uint64_t i = 0; i < steps; ++i) {
    const uint64_t m_lo = 1 + (M - 1) * i / steps, m_hi = 1 + (M - 1) * (i + 1) / steps;
    const double S = (double)n - (double)m_lo * (double)(B - 1);
    double f = (double)m_hi * (1.0 + (S > m_lo ? log2(S / (double)m_lo) : 0.0));
    const double cap = 64.0 * (double)m_hi;
    if (f > cap) f = cap;
    if (f > best) best = f;
  }
  return (uint64_t)best + 64;
}

cudaError_t set_select_pos_trace(uint64_t* p) { return cudaMemcpyToSymbol(g_sp_trace, &p, sizeof(p)); }

cudaError_t launch_select_pos(const ColView& c, const PredSpec& p, uint32_t B, uint64_t row_offset,
                              uint32_t* ticket, uint64_t* st1, uint64_t* st2, uint32_t* cnt, uint32_t* tflag,
                              uint32_t* tail, uint64_t* meta, uint32_t* err, uint64_t* payload, uint32_t* cw,
                              uint64_t* ref, uint64_t* rem, uint64_t cap_words, cudaStream_t s) {
  uint64_t ns_fast = 0;
  const int kind = sp_kind(c, &ns_fast);
  if (kind < 0 || B != (uint32_t)kB) return cudaErrorNotSupported;
  SpArgs a{};
  a.c = c;
  a.pred = FastPred{p.lo, p.span, p.neg, (uint32_t)p.is_bitmap, p.bitmap, p.bitmap_bits};
  a.n = c.n;
  a.NS = (c.n + kSegRows - 1) / kSegRows;
  a.ns_fast = ns_fast;
  a.TS = select_pos_tile_segs(c.n);
  a.T = select_pos_tiles(c.n);
  a.row_offset = row_offset;
  a.ticket = ticket;
  a.st1 = st1;
  a.st2 = st2;
  a.cnt = cnt;
  a.tflag = tflag;
  a.tail = tail;
  a.meta = meta;
  a.err = err;
  a.payload = payload;
  a.cw = cw;
  a.ref = ref;
  a.rem = rem;
  a.cap_words = cap_words;
  if (a.T == 0) return cudaSuccess;
  const uint32_t maxw = kind == FAST_STATIC ? c.w : c.maxw;
  const bool narrow = kind != FAST_UNCOMPR && maxw >= 1 && maxw <= 32;
  if (kind == FAST_UNCOMPR) return sp_launch<FAST_UNCOMPR, false>(a, 64, s);
  if (kind == FAST_STATIC)
    return narrow ? sp_launch<FAST_STATIC, true>(a, maxw, s) : sp_launch<FAST_STATIC, false>(a, 64, s);
  return narrow ? sp_launch<FAST_BLOCK, true>(a, maxw, s) : sp_launch<FAST_BLOCK, false>(a, 64, s);
}

}  // namespace ms
