// select_pos.cu — select -> DELTA_BP{B} positions in ONE pass over the input
// (SURVEY.md §7 H1). The paper's operator with on-the-fly de/re-compression
// (P:297-337, 468-505): the input-side buffer layer decompresses a block into
// a cache-resident buffer, the core evaluates the predicate and
// compacts the matches with a bit mask, and the output-side buffer
// layer recompresses the positions once a block is full and writes the final
// partial block uncompressed. DELTA_BP is the paper's recommended
// positions format ("the output is always sorted").
//
// On B200 one persistent CTA per SM runs three warp roles:
//   producer  (1 warp)  takes 32K-row tiles in order from an atomic ticket and
//                       streams each tile's compressed payload into a shared-
//                       memory ring with one TMA bulk copy per stage (16 or 32
//                       segments of 512 rows; the segments of a stage are
//                       contiguous in every supported format), headers (block
//                       widths, FOR references) computed by its lanes;
//   scanners  (NSW warps) unpack with a compile-time bit width (lane-consecutive
//                       layout, select_fast.cuh), evaluate the predicate in the
//                       code domain and write one 32-bit mask word per 32 rows
//                       into the tile's shared-memory mask (4 KiB, never HBM);
//   encoders  (4 warps)  each own every 4th tile of the CTA: popcount prefix of
//                       the mask, the tile's last B-1 positions to a small
//                       scratch ("tail"), decoupled look-back #1 on the counts
//                       (output rank O_t), the head of the first owned block
//                       from the predecessors' tails, block widths
//                       w_k = ebw(max delta) (D-6), decoupled look-back #2 on
//                       the width sums (cw offset, D-4), then every owned block
//                       packed in shared memory and stored once at its final
//                       place. Block k (ranks [kB, kB+B)) is owned by the tile
//                       holding rank kB+B-1; the last tile writes the remainder.
// HBM traffic: the compressed input once, the positions image once, plus the
// tails (< B u16 per 32K rows) and two status words per tile. No bit mask, no
// per-block slots, no copy pass.
#include "common.cuh"
#include "grid.cuh"
#include "launch.h"
#include "select_fast.cuh"
#include "tma.cuh"

namespace ms {

namespace {

constexpr int kTileSegs = 64;                       // 512-row segments per tile
constexpr int kTileRows = kTileSegs * kSegRows;     // 32768
constexpr int kTileWords = kTileRows / 32;          // mask words per tile
constexpr int kTileGroups = kTileWords / 4;         // 16-byte groups of mask words
constexpr int kEnc = 4;                             // encoder warps
constexpr int kBufs = kEnc + 2;                     // tile masks in flight
constexpr int kMaxStages = 6;                       // ring stages (runtime count <= this)

struct SpArgs {
  ColView c;
  FastPred pred;
  uint64_t n, NS, ns_fast, T, row_offset;
  uint32_t stage_u32, nst;
  uint32_t* ticket;
  uint64_t* st1;       // look-back on the tile counts (T words, zeroed)
  uint64_t* st2;       // look-back on the tile width sums (T words, zeroed)
  uint32_t* cnt;       // tile counts (T)
  uint16_t* tail;      // per tile: its last min(count, B-1) rows (relative to the tile)
  uint64_t* meta;      // [1] n_out, [2] cw[nb], [3] max block width (zeroed)
  uint32_t* err;
  uint64_t* payload;
  uint32_t* cw;
  uint64_t* ref;
  uint64_t* rem;
  uint64_t cap_words;  // payload capacity
};

template <int B>
struct EncSmem {
  uint16_t pre4[kTileGroups];          // set bits in groups [0, g) of the tile mask
  uint64_t hbuf[B];                    // the head: ranks [k_a B, O_t) as local rows
  alignas(16) uint32_t pack[2 * B];    // one block at up to 64 bits per code
  uint32_t wl[kTileRows / B + 2];      // widths of the owned blocks, then their exclusive prefix
};

template <int NSW, int B>
struct SpSmem {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t mfull[kBufs], mempty[kBufs];
  uint64_t stile[kMaxStages];  // tile of the stage (~0: no more tiles)
  uint64_t mtile[kBufs];       // tile of the mask buffer (~0: stop)
  uint32_t sidx[kMaxStages];   // stage index inside its tile
  uint32_t sw[kMaxStages][2 * NSW];
  uint32_t soff[kMaxStages][2 * NSW];
  uint64_t sref[kMaxStages][2 * NSW];
  alignas(16) uint32_t mask[kBufs][kTileWords];
  EncSmem<B> enc[kEnc];
};

template <int NSW, int B>
constexpr size_t sp_static_bytes() {
  return (sizeof(SpSmem<NSW, B>) + 127) & ~(size_t)127;
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

// Decoupled look-back with release/acquire around it: the caller's data writes
// (tails, counts) are fenced before the aggregate is published, the inclusive
// prefix is published after a fence (so data seen by this tile is visible to
// whoever sees its prefix), and the walk is followed by a fence before the
// caller reads predecessors' data. Call with all 32 lanes of one warp.
__device__ __forceinline__ uint64_t sp_lookback(uint64_t* status, uint64_t t, uint64_t agg) {
  const uint32_t lane = threadIdx.x & 31;
  __threadfence();
  __syncwarp();
  if (t == 0) {
    if (lane == 0) st_volatile(&status[0], kFlagP | agg);
    return 0;
  }
  if (lane == 0) st_volatile(&status[t], kFlagA | agg);
  const uint64_t excl = lookback_walk(status, t);
  __threadfence();
  if (lane == 0) st_volatile(&status[t], kFlagP | ((excl + agg) & kValMask));
  return excl;
}

// ------------------------------------------------------------------ encoder
template <int B>
__device__ __forceinline__ void sp_encode_tile(const SpArgs& a, uint64_t t, const uint32_t* __restrict__ M,
                                               EncSmem<B>& E, uint32_t lane) {
  constexpr int PER = B / 32;  // ranks per lane in a block
  const uint64_t row0 = t * (uint64_t)kTileRows;

  // 1. popcount prefix over 16-byte groups (conflict-free: lane l reads group 32i + l)
  uint32_t run = 0;
#pragma unroll
  for (int i = 0; i < kTileGroups / 32; ++i) {
    const uint32_t g = i * 32 + lane;
    const uint4 v = reinterpret_cast<const uint4*>(M)[g];
    const uint32_t x = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= (uint32_t)o) inc += y;
    }
    E.pre4[g] = (uint16_t)(run + inc - x);
    run += __shfl_sync(kFull, inc, 31);
  }
  const uint32_t c = run;  // matches in the tile
  __syncwarp();

  // rank r (< c) of the tile -> word m, remaining bits cur (rank r is cur's lowest set bit)
  auto locate = [&](uint32_t r, uint32_t& m, uint32_t& cur) {
    uint32_t g = 0;
#pragma unroll
    for (uint32_t step = kTileGroups / 2; step; step >>= 1)
      if (E.pre4[g + step] <= r) g += step;
    uint32_t skip = r - E.pre4[g];
    m = 4 * g;
    cur = M[m];
    while (true) {
      const uint32_t pc = __popc(cur);
      if (skip < pc || m == kTileWords - 1) break;
      skip -= pc;
      cur = M[++m];
    }
    for (; skip; --skip) cur &= cur - 1;
  };
  auto next = [&](uint32_t& m, uint32_t& cur) -> uint32_t {
    while (!cur && m < kTileWords - 1) cur = M[++m];
    const uint32_t b = __ffs(cur) - 1;
    cur &= cur - 1;
    return m * 32 + b;
  };

  // 2. the tail: the tile's last min(c, B-1) positions (relative rows)
  const uint32_t L = c < (uint32_t)(B - 1) ? c : (uint32_t)(B - 1);
  if (PER * lane < L) {
    uint32_t m, cur;
    locate(c - L + PER * lane, m, cur);
    uint16_t* tb = a.tail + t * (uint64_t)(B - 1) + PER * lane;
    const uint32_t k = L - PER * lane < (uint32_t)PER ? L - PER * lane : (uint32_t)PER;
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if ((uint32_t)i < k) tb[i] = (uint16_t)next(m, cur);
  }
  if (lane == 0) a.cnt[t] = c;

  // 3. look-back #1: output rank of the tile's first match
  const uint64_t O = sp_lookback(a.st1, t, c);
  const uint64_t Eo = O + c;
  const uint64_t ka = O / B, kb = Eo / B;
  const uint32_t h = (uint32_t)(O - ka * B);
  const bool last = t == a.T - 1;
  if (last && lane == 0) a.meta[1] = Eo;

  // 4. the head (ranks [ka B, O)) from the predecessors' tails, newest first
  if (h && (kb > ka || last)) {
    uint32_t need = h;
    int64_t j = (int64_t)t - 1;
    while (need && j >= 0) {
      const int64_t jl = j - (int64_t)lane;
      const uint32_t cj = jl >= 0 ? __ldcg(a.cnt + jl) : 0u;
      for (int l = 0; l < 32 && need && j - l >= 0; ++l) {
        const uint32_t cl = __shfl_sync(kFull, cj, l);
        if (!cl) continue;
        const uint32_t take = cl < need ? cl : need;
        const uint32_t Lj = cl < (uint32_t)(B - 1) ? cl : (uint32_t)(B - 1);
        const uint64_t tj = (uint64_t)(j - l);
        const uint16_t* tb = a.tail + tj * (uint64_t)(B - 1) + (Lj - take);
        for (uint32_t i = lane; i < take; i += 32)
          E.hbuf[need - take + i] = tj * (uint64_t)kTileRows + __ldcg(tb + i);
        need -= take;
      }
      j -= 32;
    }
    if (need && lane == 0) atomicOr(a.err, err_bit(MS_E_CORRUPT));  // fewer predecessors' matches than ranks
  }
  __syncwarp();

  // positions (local rows) of ranks [kB + PER*lane, +PER) of block k
  auto block_pos = [&](uint64_t k, uint64_t (&p)[PER]) {
    const uint64_t g0 = k * B + (uint64_t)PER * lane;
    uint32_t m = 0, cur = 0;
    if (g0 + PER > O) locate((uint32_t)(g0 >= O ? g0 - O : 0), m, cur);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const uint64_t g = g0 + i;
      p[i] = g < O ? E.hbuf[g - ka * B] : row0 + next(m, cur);
    }
  };
  // in place: positions -> deltas (d_0 = 0 at the block start, D-6); returns the block width
  auto deltas = [&](uint64_t (&p)[PER]) -> uint32_t {
    const uint64_t prev = __shfl_up_sync(kFull, p[PER - 1], 1);
    uint64_t mx = 0;
#pragma unroll
    for (int i = PER - 1; i >= 1; --i) {
      p[i] -= p[i - 1];
      mx = p[i] > mx ? p[i] : mx;
    }
    p[0] = lane ? p[0] - prev : 0ull;
    mx = p[0] > mx ? p[0] : mx;
    return __reduce_max_sync(kFull, ebw64(mx));
  };

  // 5. pass 1: widths of the owned blocks
  const uint32_t nbk = (uint32_t)(kb - ka);
  for (uint32_t i = 0; i < nbk; ++i) {
    uint64_t p[PER];
    block_pos(ka + i, p);
    const uint32_t w = deltas(p);
    if (lane == 0) E.wl[i] = w;
  }
  __syncwarp();
  uint32_t W = 0, wmax = 0;
  for (uint32_t i0 = 0; i0 < nbk; i0 += 32) {
    const uint32_t w = i0 + lane < nbk ? E.wl[i0 + lane] : 0u;
    uint32_t inc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= (uint32_t)o) inc += y;
    }
    __syncwarp();
    if (i0 + lane < nbk) E.wl[i0 + lane] = W + inc - w;  // exclusive prefix inside the tile
    W += __shfl_sync(kFull, inc, 31);
    wmax = max(wmax, __reduce_max_sync(kFull, w));
  }
  __syncwarp();

  // 6. look-back #2: cw offset of the tile's first owned block
  const uint64_t C = sp_lookback(a.st2, t, W);
  if (lane == 0) {
    if (C + W > 0xffffffffull || (C + W) * (B / 64) > a.cap_words) atomicOr(a.err, err_bit(MS_E_INVALID));
    if (wmax) atomicMax(reinterpret_cast<unsigned long long*>(a.meta + 3), (unsigned long long)wmax);
    if (last) a.meta[2] = C + W;
  }
  const bool fits = (C + W) * (B / 64) <= a.cap_words && C + W <= 0xffffffffull;

  // 7. pass 2: pack every owned block in shared memory, one coalesced store at cw[k] * B / 64
  for (uint32_t i = 0; fits && i < nbk; ++i) {
    const uint64_t k = ka + i;
    uint64_t p[PER];
    block_pos(k, p);
    const uint64_t base = __shfl_sync(kFull, p[0], 0);
    const uint32_t w = deltas(p);
    const uint64_t cwk = C + __shfl_sync(kFull, E.wl[i], 0);  // (same value in every lane)
    const uint32_t n32 = (uint32_t)(B / 32) * w;
    for (uint32_t m = lane; m < n32; m += 32) E.pack[m] = 0;
    __syncwarp();
    stream_codes<PER>(E.pack, p, w, PER * lane * w);
    __syncwarp();
    const uint32_t n16 = (uint32_t)(B / 128) * w;  // 16-byte units
    uint4* dst = reinterpret_cast<uint4*>(a.payload + cwk * (B / 64));
    const uint4* src = reinterpret_cast<const uint4*>(E.pack);
    for (uint32_t m = lane; m < n16; m += 32) dst[m] = src[m];
    if (lane == 0) {
      a.cw[k + 1] = (uint32_t)(cwk + w);
      a.ref[k] = base + a.row_offset;
    }
    __syncwarp();
  }

  // 8. the last tile: the final partial block, raw
  if (last) {
    const uint32_t R = (uint32_t)(Eo - kb * B);
    if (PER * lane < R) {
      const uint64_t g0 = kb * B + (uint64_t)PER * lane;
      uint32_t m = 0, cur = 0;
      if (g0 + PER > O) locate((uint32_t)(g0 >= O ? g0 - O : 0), m, cur);
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const uint64_t g = g0 + i;
        if (g < Eo) a.rem[g - kb * B] = a.row_offset + (g < O ? E.hbuf[g - ka * B] : row0 + next(m, cur));
      }
    }
  }
}

// -------------------------------------------------------------------- kernel
template <int NSW, int B, int KIND, bool NARROW>
__global__ void __launch_bounds__((NSW + kEnc + 1) * 32, 1) select_pos_kernel(SpArgs a) {
  extern __shared__ __align__(128) unsigned char sp_dyn[];
  auto& S = *reinterpret_cast<SpSmem<NSW, B>*>(sp_dyn);
  uint32_t* ring = reinterpret_cast<uint32_t*>(sp_dyn + sp_static_bytes<NSW, B>());
  constexpr uint32_t SP = 2 * NSW;             // segments per stage
  constexpr uint32_t SPT = kTileSegs / SP;     // stages per tile
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t nst = a.nst;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < nst; ++i) {
      mbar_init(&S.full[i], 1);
      mbar_init(&S.empty[i], NSW);
    }
    for (int i = 0; i < kBufs; ++i) {
      mbar_init(&S.mfull[i], NSW);
      mbar_init(&S.mempty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (wid == NSW + kEnc) {
    // ------------------------------------------------------------ producer
    uint64_t g = 0;
    while (true) {
      uint32_t t = 0;
      if (lane == 0) t = atomicAdd(a.ticket, 1u);
      t = __shfl_sync(kFull, t, 0);
      const bool end = t >= a.T;
      for (uint32_t si = 0; si < SPT; ++si, ++g) {
        const uint32_t st = (uint32_t)(g % nst);
        if (g >= nst) mbar_wait(&S.empty[st], (uint32_t)((g / nst) - 1) & 1u);
        if (end) {
          if (lane == 0) {
            S.stile[st] = ~0ull;
            mbar_arrive(&S.full[st]);
          }
          ++g;
          break;
        }
        const uint64_t s = (uint64_t)t * kTileSegs + si * SP + lane;
        const bool in = lane < SP && s < a.ns_fast;
        uint32_t w = 0;
        uint64_t off = 0, ref = 0;
        if (in) {
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
        }
        const uint32_t cap_w = NARROW ? 32u : 64u;
        if (w > cap_w) {  // corrupt width table, or a width above the max_width hint
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
        if (lane < SP) {
          S.sw[st][lane] = w;
          S.soff[st][lane] = (inc - bytes) >> 2;
          S.sref[st][lane] = ref;
        }
        __syncwarp();
        if (lane == 0) {
          S.stile[st] = t;
          S.sidx[st] = si;
          mbar_arrive_tx(&S.full[st], total);
          if (total) bulk_g2s(ring + (size_t)st * a.stage_u32, a.c.payload + off0, total, &S.full[st]);
        }
        __syncwarp();
      }
      if (end) break;
    }
  } else if (wid < NSW) {
    // ------------------------------------------------------------ scanners
    const uint32_t half = lane >> 4, hl = lane & 15;
    uint64_t g = 0;
    uint32_t q = 0;
    while (true) {
      const uint32_t st = (uint32_t)(g % nst);
      mbar_wait(&S.full[st], (uint32_t)(g / nst) & 1u);
      const uint64_t t = S.stile[st];
      if (t == ~0ull) {  // no more tiles: one stop mark per encoder warp
        for (int i = 0; i < kEnc; ++i, ++q) {
          const uint32_t bq = q % kBufs;
          if (q >= (uint32_t)kBufs) mbar_wait(&S.mempty[bq], ((q / kBufs) - 1) & 1u);
          if (lane == 0) {
            S.mtile[bq] = ~0ull;
            mbar_arrive(&S.mfull[bq]);
          }
        }
        break;
      }
      const uint32_t si = S.sidx[st];
      const uint32_t bq = q % kBufs;
      if (si == 0 && q >= (uint32_t)kBufs) mbar_wait(&S.mempty[bq], ((q / kBufs) - 1) & 1u);
      const uint32_t sl = wid * 2 + half;  // segment in the stage
      const uint32_t seg = si * SP + sl;   // segment in the tile
      const uint64_t s = t * kTileSegs + seg;
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
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&S.empty[st]);
        if (si == SPT - 1) {
          S.mtile[bq] = t;
          mbar_arrive(&S.mfull[bq]);
        }
      }
      if (si == SPT - 1) ++q;
      ++g;
    }
  } else {
    // ------------------------------------------------------------ encoders
    const uint32_t e = wid - NSW;
    for (uint32_t q = e;; q += kEnc) {
      const uint32_t bq = q % kBufs;
      mbar_wait(&S.mfull[bq], (q / kBufs) & 1u);
      const uint64_t t = S.mtile[bq];
      if (t == ~0ull) break;
      sp_encode_tile<B>(a, t, S.mask[bq], S.enc[e], lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.mempty[bq]);
    }
  }
}

template <int NSW, int B, int KIND, bool NARROW>
cudaError_t sp_launch(const SpArgs& a0, uint32_t maxw_cap, cudaStream_t s) {
  SpArgs a = a0;
  auto k = select_pos_kernel<NSW, B, KIND, NARROW>;
  constexpr uint32_t SP = 2 * NSW;
  a.stage_u32 = SP * (kSegRows / 32) * maxw_cap + 16;  // + padding (16-byte multiple)
  const size_t fixed = sp_static_bytes<NSW, B>();
  int dev = 0, smem_max = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  size_t avail = (size_t)smem_max > fixed ? (size_t)smem_max - fixed : 0;
  uint32_t nst = (uint32_t)(avail / (4ull * a.stage_u32));
  if (nst > 4) nst = 4;
  if (nst < 2) return cudaErrorInvalidConfiguration;
  a.nst = nst;
  const size_t smem = fixed + (size_t)nst * 4 * a.stage_u32;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  uint64_t grid = (uint64_t)num_sms();
  if (grid > a.T) grid = a.T;
  ProfScope prof_("select_pos", s);
  k<<<(int)grid, (NSW + kEnc + 1) * 32, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

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

// input kinds of the one-pass path: the select_fast layouts (STATIC_BP, UNCOMPR,
// DYN_BP / FOR_BP with B >= 512); ns_fast = the full 512-row segments they stage
static int sp_kind(const ColView& c, uint64_t* ns_fast) {
  if (c.format == MS_UNCOMPR) { *ns_fast = c.n / kSegRows; return FAST_UNCOMPR; }
  if (c.format == MS_STATIC_BP) { *ns_fast = c.n / kSegRows; return FAST_STATIC; }
  if ((c.format == MS_DYN_BP || c.format == MS_FOR_BP) && c.B >= (uint32_t)kSegRows) {
    *ns_fast = (c.nb << c.log2B) / kSegRows;
    return FAST_BLOCK;
  }
  return -1;
}

bool select_pos_supported(const ColView& c, uint32_t B) {
  uint64_t ns = 0;
  return B == 512 && c.n > 0 && sp_kind(c, &ns) >= 0;
}

cudaError_t launch_select_pos(const ColView& c, const PredSpec& p, uint32_t B, uint64_t row_offset,
                              uint32_t* ticket, uint64_t* st1, uint64_t* st2, uint32_t* cnt, uint16_t* tail,
                              uint64_t* meta, uint32_t* err, uint64_t* payload, uint32_t* cw, uint64_t* ref,
                              uint64_t* rem, uint64_t cap_words, cudaStream_t s) {
  uint64_t ns_fast = 0;
  const int kind = sp_kind(c, &ns_fast);
  if (kind < 0) return cudaErrorNotSupported;
  const uint64_t NS = (c.n + kSegRows - 1) / kSegRows;
  const uint32_t maxw = kind == FAST_STATIC ? c.w : c.maxw;
  SpArgs a{};
  a.c = c;
  a.pred = FastPred{p.lo, p.span, p.neg, (uint32_t)p.is_bitmap, p.bitmap, p.bitmap_bits};
  a.n = c.n;
  a.NS = NS;
  a.ns_fast = ns_fast;
  a.T = (c.n + kTileRows - 1) / kTileRows;
  a.row_offset = row_offset;
  a.ticket = ticket;
  a.st1 = st1;
  a.st2 = st2;
  a.cnt = cnt;
  a.tail = tail;
  a.meta = meta;
  a.err = err;
  a.payload = payload;
  a.cw = cw;
  a.ref = ref;
  a.rem = rem;
  a.cap_words = cap_words;
  if (a.T == 0) return cudaSuccess;
  const bool narrow = kind != FAST_UNCOMPR && maxw >= 1 && maxw <= 32;
  const uint32_t cap = narrow ? maxw : 64u;
  // narrow: 16 scanner warps (32 segments per stage); wide: 8 (16 segments per stage)
#define MS_SP_B(K_)                                                                  \
  do {                                                                               \
    if (narrow) {                                                                    \
      if (B == 512) return sp_launch<16, 512, K_, true>(a, cap, s);                  \
    } else {                                                                         \
      if (B == 512) return sp_launch<8, 512, K_, false>(a, cap, s);                  \
    }                                                                                \
  } while (0)
  if (kind == FAST_STATIC) MS_SP_B(FAST_STATIC);
  else if (kind == FAST_BLOCK) MS_SP_B(FAST_BLOCK);
  else if (kind == FAST_UNCOMPR) {
    if (B == 512) return sp_launch<8, 512, FAST_UNCOMPR, false>(a, 64, s);
  }
#undef MS_SP_B
  return cudaErrorNotSupported;
}

uint64_t select_pos_tiles(uint64_t n) { return (n + kTileRows - 1) / kTileRows; }

}  // namespace ms
