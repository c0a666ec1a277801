// encode.cu — output-side buffer layers: select positions (posdelta.cuh for
// DELTA_BP, positions.cuh otherwise) and project's gather + re-encode.
#include "common.cuh"
#include "grid.cuh"
#include "positions.cuh"
#include "posdelta.cuh"
#include "projstream.cuh"
#include "launch.h"

namespace ms {

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// ------------------------------------------------- select output encoder
template <class Src>
static cudaError_t run_warp_encode(const Src& src, const PosEnc& e0, uint64_t* status, uint32_t* ticket,
                                   uint32_t* err, const char* name, cudaStream_t s) {
  const PosEnc& e = e0;
  const uint64_t n_items = (e.n_out + e.G - 1) / e.G;
  if (!n_items) return cudaSuccess;
  if (e.G <= 512) {  // deferred look-back, two tiles per warp
    auto launch = [&](auto k) {
      const int warps = 4;
      const size_t smem = (size_t)warps * 2 * tile_slots(e.G) * 8;
      set_smem_once((const void*)k, smem);
      int per_sm = 0;
      per_sm = occupancy_cached((const void*)k, warps * 32, smem);
      if (per_sm < 1) per_sm = 1;
      uint64_t grid = (uint64_t)per_sm * num_sms();
      const uint64_t need = (n_items + warps - 1) / warps;
      if (need < grid) grid = need;
      ProfScope prof_(name, s);
      k<<<(int)grid, warps * 32, smem, s>>>(src, e, n_items, status, ticket, err);
      return cudaGetLastError();
    };
    if (e.G == 512) return launch(warp_encode_deferred_kernel<Src, 16>);
    if (e.G == 256) return launch(warp_encode_deferred_kernel<Src, 8>);
    return launch(warp_encode_deferred_kernel<Src, 4>);
  }
  auto k = warp_encode_kernel<Src>;
  const int warps = e.G >= 2048 ? 2 : 4;
  const size_t smem = (size_t)warps * tile_slots(e.G) * 8;
  set_smem_once((const void*)k, smem);
  int per_sm = 0;
  per_sm = occupancy_cached((const void*)k, warps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)per_sm * num_sms();
  const uint64_t need = (n_items + warps - 1) / warps;
  if (need < grid) grid = need;
  ProfScope prof_(name, s);
  k<<<(int)grid, warps * 32, smem, s>>>(src, e, n_items, status, ticket, err);
  return cudaGetLastError();
}

cudaError_t launch_positions(const PosEnc& e, const uint32_t* bits, uint64_t NS, const uint64_t* gstart,
                             uint64_t row_offset, uint64_t* status, uint32_t* ticket, uint32_t* err, cudaStream_t s) {
  return run_warp_encode(MaskSource{bits, NS, gstart, row_offset}, e, status, ticket, err, "pos_encode", s);
}


cudaError_t launch_positions_delta(const PosEnc& e, const uint32_t* bits, uint64_t NS, const uint64_t* gstart,
                                   uint64_t row_offset, uint32_t* wk, uint64_t* cwx, uint64_t* scan_status,
                                   uint32_t* scan_ticket, uint64_t* slots, uint32_t slot_words, uint32_t* dcount, uint32_t* dlist,
                                   uint32_t* err, cudaStream_t s) {
  const uint64_t n_items = (e.n_out + e.G - 1) / e.G;
  const uint64_t n_full = e.n_out / e.G;
  if (!n_items) return cudaSuccess;
  const uint64_t n_words = NS * kSegWords;
  auto grid_for = [&](auto k, size_t smem, uint64_t items) {
    set_smem_once((const void*)k, smem);
    int per_sm = 0;
    per_sm = occupancy_cached((const void*)k, kPdWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t g = (uint64_t)per_sm * num_sms();
    const uint64_t need = (items + kPdWarps - 1) / kPdWarps;
    return (int)(need < g ? (need ? need : 1) : g);
  };
  if (slots && n_full) {  // single walk: slots, scan, copy
    const size_t smem = (size_t)kPdWarps * kPdWarpU32 * 4;
    // B = 512: blocks whose span fits take pd_item512, the others (sparse regions, the
    // block before the last) are deferred to a second launch that walks them
    const bool dense = e.G == 512;
    {
      ProfScope prof_("pos_slot", s);
      if (dense) {
        const int grid = grid_for(pos_slot_kernel<kPdDense>, smem, n_items);
        pos_slot_kernel<kPdDense><<<grid, kPdWarps * 32, smem, s>>>(bits, n_words, gstart, row_offset, e, n_items,
                                                                   slots, slot_words, wk, dcount, dlist, err);
        pos_slot_kernel<kPdDeferredOnly><<<grid, kPdWarps * 32, smem, s>>>(bits, n_words, gstart, row_offset, e,
                                                                          n_items, slots, slot_words, wk, dcount, dlist, err);
        count_launch();
      } else {
        const int grid = grid_for(pos_slot_kernel<kPdAll>, smem, n_items);
        pos_slot_kernel<kPdAll><<<grid, kPdWarps * 32, smem, s>>>(bits, n_words, gstart, row_offset, e, n_items,
                                                                 slots, slot_words, wk, dcount, dlist, err);
      }
    }
    cudaError_t r = cudaGetLastError();
    if (r != cudaSuccess) return r;
    r = launch_count_scan(wk, n_full, cwx, scan_status, scan_ticket, s);
    if (r != cudaSuccess) return r;
    uint64_t cgrid = (n_full + 31) / 32;  // 8 lanes per block
    ProfScope prof_("pos_copy", s);
    pos_copy_kernel<8><<<(int)cgrid, 256, 0, s>>>(e, n_full, slots, slot_words, cwx, err);
    return cudaGetLastError();
  }
  // no full block: the remainder alone (raw positions)
  ProfScope prof_("pos_rem", s);
  pos_rem_kernel<<<1, 32, 0, s>>>(bits, n_words, gstart, row_offset, e, err);
  return cudaGetLastError();
}

cudaError_t launch_project_warp(const ColView& pos, const ColView& data, uint64_t row_offset, const PosEnc& e,
                                uint64_t* status, uint32_t* ticket, uint32_t* err, cudaStream_t s) {
  // gather + encode with a look-back on the output widths (items > 512, or outputs the slot path
  // does not serve); 4 independent gathers in flight per lane, one bulk L2 prefetch per window
  return run_warp_encode(ProjectSource<4>{pos, data, row_offset, 1u}, e, status, ticket, err, "project_warp", s);
}

// ------------------------------------------------------------ K7: fused semi-join
// pos2 = {p in pos1 : bitmap[keys[p - row_offset]]} (the star-schema semi-join of
// BJ.c4, D-16). One warp per 512-position block of pos1: decode the block,
// gather the keys at its positions (ProjectSource: header broadcast, bulk L2
// prefetch, 4 gathers in flight per lane), test the bitmap. The gathered keys
// never reach HBM (no k1' column, no select pass over it).
// The row-space form (used by ms_semijoin): the same per-block gather and bitmap
// test, but a surviving position p sets bit p - row_offset of a mask over the
// keys' rows (seg_info_kernel then counts its segments), so the select output
// layer turns the mask straight into pos2 — no positions-through-
// positions project (which decoded every pos1 block again). Requires pos1
// strictly increasing (every positions column the library produces); a block
// that is not, or whose successor does not start after it, flags MS_E_INVALID.
// A surviving position p (its key v in the bitmap) sets bit p - row_offset of the
// zeroed row mask.
struct SemiRowSet {
  const uint64_t* bitmap;
  uint64_t bits_n, row_offset, n_rows;
  uint32_t* mask;
  __device__ __forceinline__ void operator()(uint32_t, uint64_t p, uint64_t v) const {
    const uint64_t r = p - row_offset;
    if (p < row_offset || r >= n_rows) return;  // MS_E_RANGE raised by the loader
    if (v < bits_n && ((__ldg(bitmap + (v >> 6)) >> (v & 63)) & 1ull)) atomicOr(mask + (r >> 5), 1u << (r & 31));
  }
};

__global__ void __launch_bounds__(128) semi_rows_kernel(ProjectSource<4> src, uint64_t n1, SemiRowSet set,
                                                        uint32_t* err) {
  constexpr uint32_t G = kSegRows;
  extern __shared__ __align__(16) uint64_t sj_sm[];
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t* P = sj_sm + (uint64_t)wid * tile_slots(G);
  const uint64_t n_items = (n1 + G - 1) / G;
  const uint64_t NW = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t item = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wid; item < n_items; item += NW) {
    const uint64_t r0 = item * G;
    const uint32_t cnt = (uint32_t)min((uint64_t)G, n1 - r0);
    src.load_with((uint32_t)item, r0, cnt, P, lane, err, set);
    // strictly increasing inside the block and into the next block
    bool bad = false;
    for (uint32_t i = lane + 1; i < cnt; i += 32) bad |= P[pidx(i)] <= P[pidx(i - 1)];
    if (lane == 0 && r0 + cnt < n1) {  // the next block's first position (DELTA_BP: its base, O(1))
      const ColView& pc = src.pos;
      const uint64_t nxt = pc.format == MS_DELTA_BP && ((r0 + cnt) >> pc.log2B) < pc.nb &&
                                   !((r0 + cnt) & (pc.B - 1))
                               ? __ldg(pc.ref + ((r0 + cnt) >> pc.log2B))
                               : read_row(pc, r0 + cnt);
      bad |= nxt <= P[pidx(cnt - 1)];
    }
    if (__any_sync(kFull, bad) && lane == 0) atomicOr(err, err_bit(MS_E_INVALID));
    __syncwarp();
  }
}

cudaError_t launch_semi_rows(const ColView& pos1, const ColView& keys, uint64_t row_offset, const uint64_t* bitmap,
                             uint64_t bitmap_bits, uint32_t* mask, uint32_t* err, cudaStream_t s) {
  const uint64_t n_items = (pos1.n + kSegRows - 1) / kSegRows;
  if (!n_items) return cudaSuccess;
  const ProjectSource<4> src{pos1, keys, row_offset, 1u};
  const SemiRowSet set{bitmap, bitmap_bits, row_offset, keys.n, mask};
  const int warps = 4;
  const size_t smem = (size_t)warps * tile_slots(kSegRows) * 8;
  set_smem_once((const void*)semi_rows_kernel, smem);
  int per_sm = occupancy_cached((const void*)semi_rows_kernel, warps * 32, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)per_sm * num_sms();
  const uint64_t need = (n_items + warps - 1) / warps;
  if (need < grid) grid = need;
  ProfScope prof_("semi_rows", s);
  semi_rows_kernel<<<(int)grid, warps * 32, smem, s>>>(src, pos1.n, set, err);
  return cudaGetLastError();
}


// select positions in a format other than DELTA_BP (items <= 512): MaskSource into
// the slot encoder; block formats then scan the widths and copy (no look-back)
cudaError_t launch_positions_slots(const PosEnc& e, const uint32_t* bits, uint64_t NS, const uint64_t* gstart,
                                   uint64_t row_offset, uint64_t* slots, uint32_t slot_words, uint32_t* wk,
                                   uint64_t* cwx, uint64_t* scan_status, uint32_t* scan_ticket, uint32_t* err,
                                   cudaStream_t s) {
  const uint64_t n_items = (e.n_out + e.G - 1) / e.G;
  const uint64_t n_full = e.n_out / e.G;
  if (!n_items) return cudaSuccess;
  const MaskSource src{bits, NS, gstart, row_offset};
  auto launch = [&](auto k) {
    const int warps = 4;
    const size_t smem = (size_t)warps * tile_slots(e.G) * 8;
    set_smem_once((const void*)k, smem);
    int per_sm = 0;
    per_sm = occupancy_cached((const void*)k, warps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    const uint64_t need = (n_items + warps - 1) / warps;
    if (need < grid) grid = need;
    ProfScope prof_("pos_encode", s);
    k<<<(int)grid, warps * 32, smem, s>>>(src, e, n_items, slots, slot_words, wk, err);
    return cudaGetLastError();
  };
  cudaError_t r = e.G == 512   ? launch(warp_encode_slot_kernel<MaskSource, 16>)
                  : e.G == 256 ? launch(warp_encode_slot_kernel<MaskSource, 8>)
                               : launch(warp_encode_slot_kernel<MaskSource, 4>);
  if (r != cudaSuccess) return r;
  const bool block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  if (!block || !n_full) return cudaSuccess;
  r = launch_count_scan(wk, n_full, cwx, scan_status, scan_ticket, s);
  if (r != cudaSuccess) return r;
  uint64_t cgrid = (n_full + 31) / 32;  // 8 lanes per block
  ProfScope prof_("pos_copy", s);
  pos_copy_kernel<8><<<(int)cgrid, 256, 0, s>>>(e, n_full, slots, slot_words, cwx, err);
  return cudaGetLastError();
}

// project with per-block slots (no look-back): gather + encode into slots, scan the
// widths, copy the blocks to their places (pos_copy_kernel is format-agnostic).
cudaError_t launch_project_slots(const ColView& pos, const ColView& data, uint64_t row_offset, const PosEnc& e0,
                                 uint64_t* slots, uint32_t slot_words, uint32_t* wk, uint64_t* cwx,
                                 uint64_t* scan_status, uint32_t* scan_ticket, void* stream_wins,
                                 uint64_t data_pay_bytes, uint32_t* err, cudaStream_t s) {
  const PosEnc& e = e0;
  const uint64_t n_items = (e.n_out + e.G - 1) / e.G;
  const uint64_t n_full = e.n_out / e.G;
  if (!n_items) return cudaSuccess;
  const uint32_t pf = 1;  // one bulk L2 prefetch of each data window
  auto launch = [&](auto k, auto src) {
    const int warps = 4;
    const size_t smem = (size_t)warps * tile_slots(e.G) * 8;
    set_smem_once((const void*)k, smem);
    int per_sm = 0;
    per_sm = occupancy_cached((const void*)k, warps * 32, smem);
      if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    const uint64_t need = (n_items + warps - 1) / warps;
    if (need < grid) grid = need;
    ProfScope prof_("project_slot", s);
    k<<<(int)grid, warps * 32, smem, s>>>(src, e, n_items, slots, slot_words, wk, err);
    return cudaGetLastError();
  };
  const ProjectSource<4> src{pos, data, row_offset, pf};
  cudaError_t r;
  if (stream_wins && e.G == 512) {
    PsWin* wins = static_cast<PsWin*>(stream_wins);
    {
      ProfScope prof_("project_window", s);
      project_window_kernel<<<(int)((n_items + 255) / 256), 256, 0, s>>>(pos, data, row_offset, e.n_out,
                                                                         data_pay_bytes, wins);
      r = cudaGetLastError();
    }
    if (r != cudaSuccess) return r;
    auto k = project_stream_kernel<kPsStages, kPsPairs>;
    const size_t smem = ps_smem_bytes();
    set_smem_once((const void*)k, smem);
    const uint64_t grid = n_items < (uint64_t)num_sms() ? n_items : (uint64_t)num_sms();
    ProfScope prof_("project_stream", s);
    k<<<(int)grid, kPsThreads, smem, s>>>(src, e, n_items, wins, slots, slot_words, wk, err);
    r = cudaGetLastError();
  } else {
    r = e.G == 512   ? launch(warp_encode_slot_kernel<ProjectSource<4>, 16>, src)
                  : e.G == 256 ? launch(warp_encode_slot_kernel<ProjectSource<4>, 8>, src)
                               : launch(warp_encode_slot_kernel<ProjectSource<4>, 4>, src);
  }
  if (r != cudaSuccess) return r;
  const bool block = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  if (!block || !n_full) return cudaSuccess;
  r = launch_count_scan(wk, n_full, cwx, scan_status, scan_ticket, s);
  if (r != cudaSuccess) return r;
  uint64_t cgrid = (n_full + 7) / 8;
  ProfScope prof_("project_copy", s);
  pos_copy_kernel<32><<<(int)cgrid, 256, 0, s>>>(e, n_full, slots, slot_words, cwx, err);
  return cudaGetLastError();
}


bool project_stream_supported(const ColView& pos, const ColView& data, const PosEnc& e) {
  const bool block_out = e.format == MS_DYN_BP || e.format == MS_FOR_BP || e.format == MS_DELTA_BP;
  return block_out && e.G == 512 && e.n_out >= 512 && pos.format == MS_DELTA_BP && pos.B == 512 &&
         (data.format == MS_DYN_BP || data.format == MS_FOR_BP) && data.B >= 64 && data.nb > 0 &&
         aligned16(pos.payload) && aligned16(data.payload) && aligned16(data.cw) &&
         (data.format != MS_FOR_BP || aligned16(data.ref));
}

size_t project_stream_win_bytes(uint64_t n_items) { return sizeof(PsWin) * n_items; }

}  // namespace ms
