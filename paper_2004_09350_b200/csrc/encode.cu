// encode.cu — output-side buffer layers: select positions (posdelta.cuh for
// DELTA_BP, positions.cuh otherwise) and project's gather + re-encode.
#include "common.cuh"
#include "grid.cuh"
#include "positions.cuh"
#include "posdelta.cuh"
#include "launch.h"

namespace ms {

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
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, warps * 32, smem);
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
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, warps * 32, smem);
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
                                   uint32_t* scan_ticket, uint64_t* slots, uint32_t slot_words, uint32_t* err,
                                   cudaStream_t s) {
  const uint64_t n_items = (e.n_out + e.G - 1) / e.G;
  const uint64_t n_full = e.n_out / e.G;
  if (!n_items) return cudaSuccess;
  const uint64_t n_words = NS * kSegWords;
  auto grid_for = [&](auto k, size_t smem, uint64_t items) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kPdWarps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t g = (uint64_t)per_sm * num_sms();
    const uint64_t need = (items + kPdWarps - 1) / kPdWarps;
    return (int)(need < g ? (need ? need : 1) : g);
  };
  if (slots && n_full) {  // single walk: slots, scan, copy
    const size_t smem = (size_t)kPdWarps * kPdWarpU32 * 4;
    const int grid = grid_for(pos_slot_kernel, smem, n_items);
    {
      ProfScope prof_("pos_slot", s);
      pos_slot_kernel<<<grid, kPdWarps * 32, smem, s>>>(bits, n_words, gstart, row_offset, e, n_items, slots,
                                                         slot_words, wk, err);
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
  const size_t smem = (size_t)kPdWarps * kPdWarpU32 * 4;
  const int grid = grid_for(pos_pack_kernel, smem, n_items);
  ProfScope prof_("pos_pack", s);
  pos_pack_kernel<<<grid, kPdWarps * 32, smem, s>>>(bits, n_words, gstart, row_offset, e, n_items, cwx, err);
  return cudaGetLastError();
}

cudaError_t launch_project_warp(const ColView& pos, const ColView& data, uint64_t row_offset, const PosEnc& e,
                                uint64_t* status, uint32_t* ticket, uint32_t* err, cudaStream_t s) {
  // gather + encode with a look-back on the output widths (items > 512, or outputs the slot path
  // does not serve); 4 independent gathers in flight per lane, one bulk L2 prefetch per window
  return run_warp_encode(ProjectSource<4>{pos, data, row_offset, 1u}, e, status, ticket, err, "project_warp", s);
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
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, warps * 32, smem);
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
                                 uint64_t* scan_status, uint32_t* scan_ticket, uint32_t* err, cudaStream_t s) {
  const PosEnc& e = e0;
  const uint64_t n_items = (e.n_out + e.G - 1) / e.G;
  const uint64_t n_full = e.n_out / e.G;
  if (!n_items) return cudaSuccess;
  const uint32_t pf = 1;  // one bulk L2 prefetch of each data window
  auto launch = [&](auto k, auto src) {
    const int warps = 4;
    const size_t smem = (size_t)warps * tile_slots(e.G) * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, warps * 32, smem);
      if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)per_sm * num_sms();
    const uint64_t need = (n_items + warps - 1) / warps;
    if (need < grid) grid = need;
    ProfScope prof_("project_slot", s);
    k<<<(int)grid, warps * 32, smem, s>>>(src, e, n_items, slots, slot_words, wk, err);
    return cudaGetLastError();
  };
  const ProjectSource<4> src{pos, data, row_offset, pf};
  cudaError_t r = e.G == 512   ? launch(warp_encode_slot_kernel<ProjectSource<4>, 16>, src)
                  : e.G == 256 ? launch(warp_encode_slot_kernel<ProjectSource<4>, 8>, src)
                               : launch(warp_encode_slot_kernel<ProjectSource<4>, 4>, src);
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

}  // namespace ms
