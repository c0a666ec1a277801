// launch.h — host-side launch wrappers of libms' kernels (internal, C++).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ms.h"

namespace ms {

struct ColView;
struct OutView;

// instrumentation: kernel launches issued by this library, optional event timing
void count_launch();
uint64_t launch_count();
class ProfScope {  // counts one launch; brackets it with events when profiling is on
 public:
  ProfScope(const char* name, cudaStream_t s);
  ~ProfScope();

 private:
  const char* name_;
  cudaStream_t s_;
  bool on_;
  void* a_ = nullptr;
  void* b_ = nullptr;
};
void profile_enable(int on);
int profile_read(ms_kernel_time* out, int max);

// predicate in the range form keep = ((v - lo) <= span) != neg, or a bitmap
struct PredSpec {
  int is_bitmap;
  uint64_t lo, span;
  uint32_t neg;
  const uint64_t* bitmap;
  uint64_t bitmap_bits;
};

// launch-configuration queries cached per (device, kernel): the dynamic shared-memory
// opt-in is set once per size, the occupancy computed once per (threads, smem) — both
// are host round trips that otherwise sit in the gap after every size read-back
void set_smem_once(const void* kernel, size_t smem);
// pinned host words of this thread and device (64 u64; nullptr if cudaHostAlloc fails)
uint64_t* pinned_words();
// host[0..count) = dev[0..count) (count <= 32), host[32] = *w0, host[33] = *w1, host[34] = *d2 (null: 0)
cudaError_t launch_readback(uint64_t* host, const uint64_t* dev, uint32_t count, const uint32_t* w0,
                            const uint32_t* w1, const uint64_t* d2, cudaStream_t s);
int occupancy_cached(const void* kernel, int threads, size_t smem);
cudaError_t launch_engine_col(const ColView& src, const OutView& out, uint32_t* err, cudaStream_t s);
cudaError_t launch_engine_bitmask(const uint32_t* bits, const uint64_t* tile_off, const uint32_t* start_tile,
                                  uint64_t n_words, uint64_t row_offset, const OutView& out, uint32_t* err,
                                  cudaStream_t s);
cudaError_t launch_engine_gather(const ColView& pos, const ColView& data, uint64_t row_offset, const OutView& out,
                                 uint32_t* err, cudaStream_t s);

// engine slot mode: tiles' packed blocks (OutView.slots) -> payload at the scanned cw (cwx, nb + 1 entries)
cudaError_t launch_tile_copy(const OutView& o, uint64_t n_tiles, uint64_t nb, const uint64_t* cwx, uint32_t* err,
                             cudaStream_t s);
// select core: bit mask (16 words per 512-row segment) + seg_info (count | last << 16)
// tile_list: scratch of (NS * 512 / 2048 + 2) u32 for the header-only pruning of block formats (or nullptr)
cudaError_t launch_select(const ColView& c, const PredSpec& p, uint32_t* bits, uint32_t* seg_info, uint64_t NS,
                          uint32_t* tile_list, uint32_t* err, cudaStream_t s);
// exclusive scan of per-segment counts -> seg_off[0..NS], start_seg[] per output item, 1 + max position
// ... and, for every output item of G ranks starting in a segment, the item's first position
cudaError_t launch_seg_scan(const uint32_t* seg_info, const uint32_t* bits, uint64_t NS, uint64_t row_offset,
                            uint32_t G, uint64_t* seg_off, uint64_t* gstart, unsigned long long* max_pos1,
                            uint64_t* status, uint32_t* ticket, cudaStream_t s);
// select output encoder (positions.cuh): E1, cw scan, E2
struct PosEnc {  // output of the warp encoder
  int32_t format;      // output format
  uint32_t w;          // STATIC_BP width
  uint32_t G, log2G;   // item size: B for block formats, 512 otherwise
  uint64_t n_out;      // output length
  uint64_t* payload;
  uint32_t* cw;
  uint64_t* ref;
  uint64_t* rem;
};
cudaError_t launch_positions(const PosEnc& e, const uint32_t* bits, uint64_t NS, const uint64_t* gstart,
                             uint64_t row_offset, uint64_t* status, uint32_t* ticket, uint32_t* err, cudaStream_t s);
// positions as DELTA_BP{B <= 512} straight from the mask (posdelta.cuh): widths, scan, pack.
// Scratch: wk (n_full u32), cwx (n_full + 1 u64), scan status ((n_full + 2047) / 2048 + 1 u64, zeroed), ticket (zeroed).
// slots != nullptr: single walk into per-block slots of slot_words u64 (n_full slots), then scan + copy;
// else two walks (widths, scan, pack).
cudaError_t launch_positions_delta(const PosEnc& e, const uint32_t* bits, uint64_t NS, const uint64_t* gstart,
                                   uint64_t row_offset, uint32_t* wk, uint64_t* cwx, uint64_t* scan_status,
                                   uint32_t* scan_ticket, uint64_t* slots, uint32_t slot_words,
                                   uint32_t* dcount,  // zeroed: the number of deferred blocks
                                   uint32_t* dlist,   // the deferred blocks
                                   uint32_t* err, cudaStream_t s);
// select positions in other formats (items <= 512) through the slot encoder (+ scan, copy for block formats)
cudaError_t launch_positions_slots(const PosEnc& e, const uint32_t* bits, uint64_t NS, const uint64_t* gstart,
                                   uint64_t row_offset, uint64_t* slots, uint32_t slot_words, uint32_t* wk,
                                   uint64_t* cwx, uint64_t* scan_status, uint32_t* scan_ticket, uint32_t* err,
                                   cudaStream_t s);
// project through the warp encoder (positions DELTA_BP with B == G, or O(1) formats; data O(1) formats)
cudaError_t launch_project_warp(const ColView& pos, const ColView& data, uint64_t row_offset, const PosEnc& e,
                                uint64_t* status, uint32_t* ticket, uint32_t* err, cudaStream_t s);

// project into per-block slots (G <= 512, block formats or UNCOMPR), scan of the widths, copy.
// Scratch: slots (n/G * slot_words u64), wk (n/G u32), cwx (n/G + 1 u64), scan status (zeroed), ticket (zeroed).
// stream_wins (64 B per item, or nullptr): the streamed variant (projstream.cuh) for dense DELTA_BP{512}
// positions over DYN_BP / FOR_BP data; data_pay_bytes bounds its payload reads.
cudaError_t launch_project_slots(const ColView& pos, const ColView& data, uint64_t row_offset, const PosEnc& e,
                                 uint64_t* slots, uint32_t slot_words, uint32_t* wk, uint64_t* cwx,
                                 uint64_t* scan_status, uint32_t* scan_ticket, void* stream_wins,
                                 uint64_t data_pay_bytes, uint32_t* err, cudaStream_t s);
// whether the streamed project applies (host-side shape checks; the caller adds the density rule)
bool project_stream_supported(const ColView& pos, const ColView& data, const PosEnc& e);
size_t project_stream_win_bytes(uint64_t n_items);

// direct morph RLE -> DELTA_BP{B} (morph.cu): per-run widths / bases / remainder, then (after the
// width scan and the exact allocation) the steps ORed into the zeroed payload and cw
cudaError_t launch_rle2delta_widths(const ColView& c, uint32_t B, uint64_t nb, uint32_t* wk, uint64_t* ref,
                                    uint64_t* rem, cudaStream_t s);
cudaError_t launch_rle2delta_pack(const ColView& c, uint32_t B, uint64_t nb, const uint64_t* cwx, uint32_t* cw,
                                  uint64_t* payload, uint32_t* err, cudaStream_t s);

// RLE run starts (exclusive prefix of lengths), validation against n
cudaError_t launch_rle_starts(const uint64_t* payload, uint64_t R, uint64_t n, uint64_t* starts, uint64_t* status,
                              uint32_t* ticket, uint32_t* err, cudaStream_t s);
cudaError_t launch_rle_expand(const uint64_t* payload, const uint64_t* starts, uint64_t R, uint64_t n, uint64_t* out,
                              cudaStream_t s);
cudaError_t launch_chunk_run(const uint64_t* starts, uint64_t R, uint64_t n, uint32_t* chunk_run, cudaStream_t s);
// RLE compression of raw device values
cudaError_t launch_rle_count(const uint64_t* v, uint64_t n, uint32_t* counts, cudaStream_t s);
// off: T + 2 entries (exclusive prefix, total, max count)
cudaError_t launch_count_scan(const uint32_t* counts, uint64_t T, uint64_t* off, uint64_t* status,
                              uint32_t* ticket, cudaStream_t s);
cudaError_t launch_rle_write(const uint64_t* v, uint64_t n, const uint64_t* chunk_off, uint64_t* payload,
                             uint64_t* starts, cudaStream_t s);
cudaError_t launch_rle_len(const uint64_t* starts, uint64_t R, uint64_t n, uint64_t* payload, cudaStream_t s);

cudaError_t launch_sum(const ColView& c, unsigned long long* out, uint32_t* err, cudaStream_t s);
cudaError_t launch_sum_at(const ColView& data, const ColView& pos, uint64_t row_offset, unsigned long long* out,
                          uint32_t* err, cudaStream_t s);
cudaError_t launch_sum_grouped(const ColView& gid, const ColView& vals, uint64_t n_groups,
                               unsigned long long* sums, uint32_t* err, cudaStream_t s);

// per 512-row segment of a mask: count | (1-based last set row << 16) (select.cu)
cudaError_t launch_seg_info(const uint32_t* bits, uint64_t NS, uint32_t* seg_info, cudaStream_t s);

// plan-level operators (plan.cu)
// format profile: acc (5 u64, zeroed) = [max, sum ebw(max_b), sum ebw(maxdelta_b), sum ebw(max_b - min_b),
// runs]; first_last: 2 u64 per 2048-row tile (scratch)
cudaError_t launch_profile(const ColView& c, uint32_t B, unsigned long long* acc, uint64_t* first_last,
                           cudaStream_t s);
cudaError_t launch_seg_count(const uint32_t* bits, uint64_t NS, uint32_t* cnt, cudaStream_t s);
cudaError_t launch_ends(const ColView& a, const ColView& b, uint64_t* out, cudaStream_t s);  // out: a0 a1 b0 b1
cudaError_t launch_pos_bitmap(const ColView& c, uint64_t base, uint64_t nbits, uint32_t* bits, uint64_t* first_last,
                              uint32_t* err, cudaStream_t s);
cudaError_t launch_bits_combine(uint32_t* a, const uint32_t* b, uint64_t n_words, int op, cudaStream_t s);
cudaError_t launch_group(const ColView& keys, const ColView& prev, uint32_t* state, uint64_t* key, uint64_t* key2,
                         uint64_t cap, unsigned long long* first, uint32_t* bits, uint32_t* err, cudaStream_t s);
cudaError_t launch_group_ids(const ColView& keys, const ColView& prev, uint32_t* state, uint64_t* key, uint64_t* key2,
                             uint64_t cap, const unsigned long long* first, const uint32_t* bits,
                             const uint64_t* seg_off, uint64_t* ids, uint32_t* err, cudaStream_t s);
cudaError_t launch_join_build(const ColView& build, uint32_t* state, uint64_t* key, uint64_t cap, uint32_t* cnt,
                              uint32_t* err, cudaStream_t s);
cudaError_t launch_join_place(const ColView& build, uint32_t* state, uint64_t* key, uint64_t cap, const uint32_t* cnt,
                              const uint64_t* off, uint32_t* fill, uint64_t* rows, uint32_t* err, cudaStream_t s);
cudaError_t launch_join_probe(const ColView& probe, uint32_t* state, uint64_t* key, uint64_t cap, const uint32_t* cnt,
                              const uint64_t* off, const uint64_t* rows, uint32_t* tile_cnt, const uint64_t* tile_off,
                              uint64_t* out_probe, uint64_t* out_build, bool write, uint32_t* err, cudaStream_t s);
cudaError_t launch_calc(const ColView& a, const ColView& b, int op, uint64_t* out, cudaStream_t s);
// K7 (encode.cu): mask over pos1's ranks of the positions whose key is in the bitmap (select mask
// layout: 16 words + one seg_info per 512 ranks); pos1 DELTA_BP{512} or O(1) formats, keys O(1) formats
// K7, row space: surviving positions as bits of a zeroed mask over the keys' rows
cudaError_t launch_semi_rows(const ColView& pos1, const ColView& keys, uint64_t row_offset, const uint64_t* bitmap,
                             uint64_t bitmap_bits, uint32_t* mask, uint32_t* err, cudaStream_t s);

// RLE encoding from a column source (morph into RLE): counts per 2048-row tile (first_last: 2 u64 per
// tile), then, after the scan of the counts, (value, start) of every run
cudaError_t launch_rle_count_col(const ColView& c, uint32_t* counts, uint64_t* first_last, cudaStream_t s);
cudaError_t launch_rle_write_col(const ColView& c, const uint64_t* first_last, const uint64_t* tile_off,
                                 uint64_t* payload, uint64_t* starts, cudaStream_t s);

// DELTA_BP (B >= 128) decoded by lanes of 64 rows (delta.cu): into u64 values, its maximum, or a
// static-BP stream at width ws (every payload word written; MS_E_WIDTH_OVERFLOW if a value needs more)
// header bounds of a DELTA_BP column's maximum: lohi[0] = lower, lohi[1] = upper (zeroed by the caller)
cudaError_t launch_delta_bounds(const ColView& c, unsigned long long* lohi, cudaStream_t s);
bool delta_direct_supported(const ColView& c);
cudaError_t launch_delta_decode(const ColView& c, uint64_t* out, uint32_t* err, cudaStream_t s);
cudaError_t launch_delta_max(const ColView& c, unsigned long long* max_out, uint32_t* err, cudaStream_t s);
cudaError_t launch_delta_to_static(const ColView& c, uint32_t ws, uint64_t* payload, uint32_t* err, cudaStream_t s);

int num_sms();
// largest block width max(cw[b+1] - cw[b]) into *out (zero-initialised)
cudaError_t launch_max_width(const uint32_t* cw, uint64_t nb, uint32_t* out, cudaStream_t s);

}  // namespace ms
