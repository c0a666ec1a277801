// projstream.cuh — project for dense positions: the data column is
// streamed through shared memory in row order instead of gathered sector by
// sector.
//
// Output block k (512 positions, ranks [512k, 512k+512)) reads the data rows
// [ref_k, ref_{k+1}] of the DELTA_BP{512} positions column (ref = the block's
// first position, D-6): consecutive windows tile the data column with one row
// of overlap, so every payload byte is read about once (a gather reads whole
// 32-byte sectors; at c5 density, one position per 16 rows of 20-bit codes,
// most sectors are touched anyway, and the bulk L2 prefetch of the gather
// path lets overlapping windows re-read ~1 GB).
//
//   project_window_kernel  one thread per block: the window's byte range in the
//                          data payload, the positions block, the header ranges
//                          (the copies must be 16-byte aligned) -> PsWin;
//   project_stream_kernel  persistent, one CTA per SM, each CTA a contiguous
//                          run of blocks; 7 stages, 7 consumer pairs. Warp 0
//                          (producer) issues, per block, TMA bulk copies of the
//                          payload window, the positions block and the data
//                          headers into stage li % 7 (mbarrier complete_tx);
//                          consumer pair li % 7 (two warps): warp h decodes the
//                          positions of ranks [256h, 256h+256) from shared
//                          memory into window-relative rows (lane j: 8
//                          consecutive codes, warp prefix sum), thread t builds
//                          the table entry of the window's block t (bit base,
//                          width, mask); warp h unpacks its ranks' codes from
//                          the window (lane-strided: neighbouring lanes read
//                          neighbouring codes) tracking the extremes, releases
//                          the stage, and the pair builds the block's slot
//                          words straight from the values (pair_encode).
//                          Blocks whose window does not fit a stage, the final
//                          partial block and blocks with positions outside
//                          their window take the gather path (ProjectSource).
// Measured at BJ.c5 (2^32 rows): 1.88 ms against 2.37 for the gather kernel; it
// reads 1.0x the Y image (ncu) at ~6.3 TB/s. Fewer consumer warps left it
// consumer-bound (4 pairs: 2.78 ms, 6 pairs: 2.13 ms).
#pragma once
#include "common.cuh"
#include "positions.cuh"
#include "tma.cuh"

namespace ms {

constexpr int kPsStages = 7;                 // stages per CTA (windows in flight or in use)
constexpr int kPsPairs = 7;                  // consumer pairs per CTA (<= kPsStages: a pair waits on one
                                             // phase of its stage at a time)
constexpr int kPsThreads = (1 + 2 * kPsPairs) * 32;
constexpr uint32_t kPsWinBytes = 24 * 1024;  // payload window cap per block
constexpr uint32_t kPsPosBytes = 1024;       // positions block cap (w <= 16 at B = 512)
constexpr uint32_t kPsMaxBlk = 60;           // data blocks per window
constexpr uint32_t kPsCwU32 = 68;            // >= kPsMaxBlk + 1 + 2 * 3 (16-byte alignment)
constexpr uint32_t kPsRefU64 = 64;           // >= kPsMaxBlk + 2
constexpr uint32_t kPsNotStreamed = 0xffffffffu;

struct PsWin {      // one output block's window (global, written by project_window_kernel)
  uint64_t r0, r1;  // data rows [r0, r1) relative to row_offset
  uint64_t byte_a;  // payload byte of the window's first (16-byte aligned) byte
  uint64_t pbyte;   // positions payload byte of the block
  uint64_t b0;      // first data block of the window
  uint32_t wbytes;  // window bytes (kPsNotStreamed: gather path)
  uint32_t wp;      // positions width
  uint32_t ia, ja;  // first cw / ref index copied (16-byte aligned)
  uint32_t ncw, nref;
};

struct PsStage {  // one stage in shared memory (16-byte aligned members)
  uint32_t win[kPsWinBytes / 4 + 4];  // + slack: unpacks read up to two words past the last code
  uint32_t pos[kPsPosBytes / 4 + 8];
  uint32_t cw[kPsCwU32];
  uint64_t ref[kPsRefU64];
  PsWin m;
};

struct PsPair {  // the consumer pair's working set
  uint64_t P[tile_slots(512)];  // window-relative rows -> gathered values -> packed block
  uint4 tab[64];                // per data block of the window: {bit base, w, mask, 0}
  uint64_t xch[8];              // min / max exchange between the two warps
  uint32_t tot[4];              // each warp's sum of position codes
};

__host__ __device__ constexpr size_t ps_smem_bytes(int S = kPsStages, int NP = kPsPairs) {
  return sizeof(PsStage) * S + sizeof(PsPair) * NP + 2 * 32 * sizeof(PsWin) + 2 * S * 8;
}

// Window of block k (thread per block). Streamed only if the block is full, its
// first position is a row of this column, the window lies in the main blocks
// and every copy fits its stage buffer and stays inside its array.
__global__ void project_window_kernel(ColView pos, ColView data, uint64_t row_offset, uint64_t n_out,
                                      uint64_t data_pay_bytes, PsWin* __restrict__ win) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t n_items = (n_out + 511) / 512;
  if (k >= n_items) return;
  PsWin m{};
  m.wbytes = kPsNotStreamed;
  const uint64_t main_rows = data.nb << data.log2B;
  if (k < pos.nb && (k + 1) * 512 <= n_out) {
    const uint64_t p0 = __ldg(pos.ref + k);
    uint64_t pn;  // first position of the next block (or the remainder / column end)
    bool have_next = true;
    if (k + 1 < pos.nb) pn = __ldg(pos.ref + k + 1);
    else if (pos.nrem) pn = __ldg(pos.rem);
    else have_next = false;
    const uint64_t r0 = p0 - row_offset;
    uint64_t r1 = main_rows;
    if (have_next && pn >= row_offset && pn - row_offset < main_rows) r1 = pn - row_offset + 1;
    const uint32_t cwp = __ldg(pos.cw + k), wp = __ldg(pos.cw + k + 1) - cwp;
    if (p0 >= row_offset && r0 < r1 && r1 <= main_rows && wp <= 16) {
      const uint64_t b0 = r0 >> data.log2B, b1 = (r1 - 1) >> data.log2B;
      const uint64_t ia = b0 & ~3ull, ib = (b1 + 2 + 3) & ~3ull;  // cw[b0 .. b1+1]
      const uint64_t ja = b0 & ~1ull, jb = (b1 + 1 + 1) & ~1ull;  // ref[b0 .. b1]
      const bool is_for = data.format == MS_FOR_BP;
      if (b1 - b0 < kPsMaxBlk && ib <= ((data.nb + 1) & ~3ull) && (!is_for || jb <= (data.nb & ~1ull))) {
        const uint32_t c0 = __ldg(data.cw + b0), c0n = __ldg(data.cw + b0 + 1);
        const uint32_t c1 = __ldg(data.cw + b1), c1n = __ldg(data.cw + b1 + 1);
        const uint64_t bit_a = (uint64_t)c0 * data.B + (r0 & (data.B - 1)) * (uint64_t)(c0n - c0);
        const uint64_t bit_b = (uint64_t)c1 * data.B + (((r1 - 1) & (data.B - 1)) + 1) * (uint64_t)(c1n - c1);
        const uint64_t byte_a = (bit_a >> 3) & ~15ull;
        const uint64_t byte_b = (((bit_b + 7) >> 3) + 15) & ~15ull;
        if (byte_b <= data_pay_bytes && byte_b - byte_a <= kPsWinBytes) {
          m.r0 = r0;
          m.r1 = r1;
          m.byte_a = byte_a;
          m.pbyte = (uint64_t)cwp * 64;
          m.b0 = b0;
          m.wbytes = (uint32_t)(byte_b - byte_a);
          m.wp = wp;
          m.ia = (uint32_t)ia;
          m.ja = (uint32_t)ja;
          m.ncw = (uint32_t)(ib - ia);
          m.nref = is_for ? (uint32_t)(jb - ja) : 0u;
        }
      }
    }
  }
  win[k] = m;
}

__device__ __forceinline__ void pair_bar(uint32_t pair) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(pair + 1) : "memory");
}
// the pair's barrier with an OR over its 64 threads' predicates
__device__ __forceinline__ bool pair_bar_or(uint32_t pair, bool v) {
  uint32_t r;
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.u32 q, %1, 0;\nbar.red.or.pred p, %2, 64, q;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(pair + 1)
      : "memory");
  return r != 0;
}

// The block's 512 values in X.P re-encoded by the pair into its slot (the
// output-side buffer layer of P:486-490, slot form): the codes (DELTA:
// differences, FOR: minus the block minimum, DYN: the values) and the width
// from the pair's extremes (lo, hi: from the gather, else from P here), then
// thread t builds the slot's u32 words t, t + 64, ... directly from P (each word
// ORs the <= 3 codes that overlap it) and stores them; wk / ref by thread 0.
__device__ __forceinline__ void pair_encode(const PosEnc& e, uint64_t item, PsPair& X, uint32_t t, uint32_t pair,
                                            uint64_t lo, uint64_t hi, bool have_ext,
                                            uint64_t* __restrict__ slots, uint32_t slot_words,
                                            uint32_t* __restrict__ wk, uint32_t* err) {
  const uint32_t lane = t & 31, half = t >> 5;
  const bool delta = e.format == MS_DELTA_BP;
  if (!have_ext || delta) {
    lo = ~0ull;
    hi = 0;
#pragma unroll
    for (uint32_t u = 0; u < 8; ++u) {
      const uint32_t i = half * 256 + u * 32 + lane;
      uint64_t v = X.P[pidx(i)];
      if (delta) v = i ? v - X.P[pidx(i - 1)] : 0ull;
      lo = v < lo ? v : lo;
      hi = v > hi ? v : hi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t a = __shfl_xor_sync(kFull, lo, o), b = __shfl_xor_sync(kFull, hi, o);
      lo = a < lo ? a : lo;
      hi = b > hi ? b : hi;
    }
    if (lane == 0) {
      X.xch[4 + 2 * half] = lo;
      X.xch[5 + 2 * half] = hi;
    }
    pair_bar(pair);
    lo = min(X.xch[4], X.xch[6]);
    hi = max(X.xch[5], X.xch[7]);
  }
  const bool is_for = e.format == MS_FOR_BP;
  const uint64_t base = is_for ? lo : 0ull;
  const uint32_t w = ebw64(is_for ? hi - lo : hi);
  const uint32_t nw32 = 16 * w;
  if (8 * w > slot_words) {
    if (t == 0) atomicOr(err, err_bit(MS_E_CORRUPT));
  } else if (w) {
    uint32_t* dst = reinterpret_cast<uint32_t*>(slots + item * slot_words);
    const uint32_t magic = 0xffffffffu / w + 1u;
    auto code = [&](uint32_t j) -> uint64_t {
      const uint64_t v = X.P[pidx(j)];
      return delta ? (j ? v - X.P[pidx(j - 1)] : 0ull) : v - base;
    };
    for (uint32_t m = t; m < nw32; m += 64) {
      const uint32_t bit0 = m * 32;
      uint32_t j = div_small(bit0, w, magic);
      uint64_t acc = code(j) >> (bit0 - j * w);
      for (++j; j < 512; ++j) {
        const uint32_t jb = j * w;
        if (jb >= bit0 + 32) break;
        acc |= code(j) << (jb - bit0);
      }
      dst[m] = (uint32_t)acc;
    }
  }
  if (t == 0) {
    wk[item] = w;
    if (is_for) e.ref[item] = lo;
    else if (delta) e.ref[item] = X.P[pidx(0)];
  }
  pair_bar(pair);
}

// code of width w (<= 64) at bit `bit` of the shared-memory window
__device__ __forceinline__ uint64_t ps_code(const uint32_t* wv, uint64_t bit, uint32_t w) {
  const uint32_t i = (uint32_t)(bit >> 5), s = (uint32_t)(bit & 31);
  if (w <= 32) {
    const uint32_t x = __funnelshift_r(wv[i], wv[i + 1], s);
    return w == 32 ? x : (x & ((1u << w) - 1));
  }
  const uint64_t lo = __funnelshift_r(wv[i], wv[i + 1], s);
  const uint64_t hi = __funnelshift_r(wv[i + 1], wv[i + 2], s);
  return (lo | hi << 32) & low_mask(w);
}

template <int kPsStages, int kPsPairs>
__global__ void __launch_bounds__((1 + 2 * kPsPairs) * 32, 1)
    project_stream_kernel(ProjectSource<4> src, PosEnc e, uint64_t n_items, const PsWin* __restrict__ wins,
                          uint64_t* __restrict__ slots, uint32_t slot_words, uint32_t* __restrict__ wk,
                          uint32_t* err) {
  constexpr uint32_t G = 512;
  extern __shared__ __align__(128) uint8_t ps_sm[];
  PsStage* st = reinterpret_cast<PsStage*>(ps_sm);
  PsPair* pairs = reinterpret_cast<PsPair*>(ps_sm + sizeof(PsStage) * kPsStages);
  PsWin* pm = reinterpret_cast<PsWin*>(pairs + kPsPairs);  // [2][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(pm + 64);
  uint64_t* empty = full + kPsStages;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t per_cta = (n_items + gridDim.x - 1) / gridDim.x;
  const uint64_t i_lo = (uint64_t)blockIdx.x * per_cta;
  const uint64_t i_hi = min(n_items, i_lo + per_cta);
  if (threadIdx.x == 0) {
    for (int c = 0; c < kPsStages; ++c) {
      mbar_init(full + c, 1);
      mbar_init(empty + c, 2);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (i_lo >= i_hi) return;
  const ColView& dv = src.data;
  if (wid == 0) {  // ---------------- producer
    const char* pay = reinterpret_cast<const char*>(dv.payload);
    const char* ppay = reinterpret_cast<const char*>(src.pos.payload);
    if (i_lo + lane < i_hi) pm[lane] = wins[i_lo + lane];
    __syncwarp();
    for (uint64_t base = i_lo, b = 0; base < i_hi; base += 32, ++b) {
      const bool hn = base + 32 + lane < i_hi;
      PsWin nx;
      if (hn) nx = wins[base + 32 + lane];
      if (lane == 0) {
        const PsWin* cur = pm + (b & 1) * 32;
        const uint32_t nj = (uint32_t)min((uint64_t)32, i_hi - base);
        for (uint32_t j = 0; j < nj; ++j) {
          const uint64_t li = base + j - i_lo;
          const uint32_t c = (uint32_t)(li % kPsStages);
          const uint64_t round = li / kPsStages;
          if (round) mbar_wait(empty + c, (uint32_t)((round - 1) & 1));
          const PsWin m = cur[j];
          st[c].m = m;
          if (m.wbytes == kPsNotStreamed) {
            mbar_arrive(full + c);
            continue;
          }
          const uint32_t pb = m.wp * 64, cb = m.ncw * 4, rb = m.nref * 8;
          mbar_arrive_tx(full + c, m.wbytes + pb + cb + rb);
          if (m.wbytes) bulk_g2s(st[c].win, pay + m.byte_a, m.wbytes, full + c);
          if (pb) bulk_g2s(st[c].pos, ppay + m.pbyte, pb, full + c);
          bulk_g2s(st[c].cw, dv.cw + m.ia, cb, full + c);
          if (rb) bulk_g2s(st[c].ref, dv.ref + m.ja, rb, full + c);
        }
      }
      __syncwarp();
      if (hn) pm[((b + 1) & 1) * 32 + lane] = nx;
      __syncwarp();
    }
    return;
  }
  // ------------------------------------ consumer pairs: pair p takes the CTA's blocks p, p + kPsPairs, ...;
  // block li sits in stage li % kPsStages (kPsStages > kPsPairs: windows load while every pair works)
  const uint32_t pair = (wid - 1) >> 1, half = (wid - 1) & 1, t = half * 32 + lane;
  PsPair& X = pairs[pair];
  const uint32_t B = dv.B, lgB = dv.log2B;
  const bool is_for = dv.format == MS_FOR_BP;
  for (uint64_t li = pair; i_lo + li < i_hi; li += kPsPairs) {
    const uint64_t item = i_lo + li;
    const uint32_t sg = (uint32_t)(li % kPsStages);
    PsStage& S = st[sg];
    mbar_wait(full + sg, (uint32_t)((li / kPsStages) & 1));
    const PsWin m = S.m;
    const uint32_t cnt = (uint32_t)min((uint64_t)G, e.n_out - item * G);
    bool ok = m.wbytes != kPsNotStreamed;
    uint64_t lo = ~0ull, hi = 0;
    if (ok) {
      // positions: warp h decodes ranks [256h, 256h+256), lane j the 8 ranks 256h + 8j + [0, 8),
      // into rows relative to the warp's first rank (the other warp's total comes after the barrier)
      const uint32_t wp = m.wp, nrows = (uint32_t)(m.r1 - m.r0);
      const uint32_t pmask = (1u << wp) - 1;  // wp <= 16
      const uint32_t lb = (256 * half + 8 * lane) * wp;
      const uint32_t* w32 = S.pos + (lb >> 5);
      const uint32_t sft = lb & 31;
      uint32_t d[8];
      if (wp <= 8) {  // the lane's <= 64 + 31 bits: three words
        const uint32_t x0 = w32[0], x1 = w32[1], x2 = w32[2];
        uint64_t win = ((uint64_t)x1 << 32 | x0) >> sft;
        uint32_t avail = 64 - sft;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (avail < wp) {
            win |= (uint64_t)x2 << avail;
            avail += 32;
          }
          d[q] = (uint32_t)win & pmask;
          win >>= wp;
          avail -= wp;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t bit = lb + q * wp;
          d[q] = __funnelshift_r(S.pos[bit >> 5], S.pos[(bit >> 5) + 1], bit & 31) & pmask;
        }
      }
      uint32_t acc = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += d[q];  // < 2^19
      uint32_t incl = acc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (lane == 31) X.tot[half] = incl;
      uint32_t r = incl - acc;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        r += d[q];
        X.P[pidx(256 * half + 8 * lane + q)] = r;
      }
      // per data block of the window: bit base relative to the staged window, width, mask
      const uint32_t nblk = (uint32_t)(((m.r1 - 1) >> lgB) - m.b0) + 1;
      const uint32_t hsh = (uint32_t)(m.b0 - m.ia);
      bool wide = false;
      if (t < nblk) {
        const uint32_t c0 = S.cw[hsh + t], w = S.cw[hsh + t + 1] - c0;
        const uint32_t base = (uint32_t)((uint64_t)c0 * B - m.byte_a * 8);
        X.tab[t] = make_uint4(base, w, w >= 32 ? ~0u : ((1u << w) - 1), 0u);
        wide = w > 32;
      }
      wide = pair_bar_or(pair, wide);
      const uint32_t tot0 = X.tot[0];
      ok = tot0 + X.tot[1] < nrows;  // the block's last row inside the window (sorted block: the largest)
      if (ok) {
        const uint32_t r0m = (uint32_t)(m.r0 & (B - 1)) + (half ? tot0 : 0u);
        const uint64_t* sref = S.ref + (uint32_t)(m.b0 - m.ja);
        if (!wide) {
#pragma unroll 4
          for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t i = half * 256 + u * 32 + lane;
            const uint32_t x = (uint32_t)X.P[pidx(i)] + r0m, blk = x >> lgB;
            const uint4 tb = X.tab[blk];
            const uint32_t bit = tb.x + (x & (B - 1)) * tb.y;
            const uint32_t code = __funnelshift_r(S.win[bit >> 5], S.win[(bit >> 5) + 1], bit & 31) & tb.z;
            const uint64_t v = is_for ? sref[blk] + code : (uint64_t)code;
            X.P[pidx(i)] = v;
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
          }
        } else {
          for (uint32_t u = 0; u < 8; ++u) {
            const uint32_t i = half * 256 + u * 32 + lane;
            const uint32_t x = (uint32_t)X.P[pidx(i)] + r0m, blk = x >> lgB;
            const uint4 tb = X.tab[blk];
            const uint32_t bit = tb.x + (x & (B - 1)) * tb.y;
            const uint64_t code = ps_code(S.win, bit, tb.y);
            const uint64_t v = is_for ? sref[blk] + code : code;
            X.P[pidx(i)] = v;
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t a = __shfl_xor_sync(kFull, lo, o), b = __shfl_xor_sync(kFull, hi, o);
          lo = a < lo ? a : lo;
          hi = b > hi ? b : hi;
        }
        if (lane == 0) {
          X.xch[2 * half] = lo;
          X.xch[2 * half + 1] = hi;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + sg);  // the stage is free once both warps are past it
    if (!ok) {  // gather path (window too large, final partial block, positions outside the window)
      if (half == 0) src.load((uint32_t)item, item * G, cnt, X.P, lane, err);
    }
    pair_bar(pair);
    if (cnt < G) {
      if (half == 0) encode_finish<ProjectSource<4>>(e, (uint32_t)item, X.P, cnt, 0, 0, nullptr, err, lane);
      pair_bar(pair);
      continue;
    }
    if (ok) {
      lo = min(X.xch[0], X.xch[2]);
      hi = max(X.xch[1], X.xch[3]);
    }
    pair_encode(e, item, X, t, pair, lo, hi, ok, slots, slot_words, wk, err);
  }
}

}  // namespace ms
