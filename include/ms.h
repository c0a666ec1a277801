/* ms.h — C ABI of libms, the B200-native (sm_100a) compression-enabled
 * operator-at-a-time hot path of MorphStore (arXiv 2004.09350).
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, D-n = a reading of
 * the paper listed in DESIGN.md §3.
 *
 * The paper's model: every base column and every intermediate is a column of
 * unsigned 64-bit integers kept in exactly one lightweight
 * integer format; operators run "on-the-fly
 * de/re-compression": decompress the input block by block inside
 * the operator, operate, and recompress the output into a format chosen
 * independently of the input's, never materialising the whole column
 * uncompressed (DP3). Here every operator is one or a few CUDA kernels
 * that do unpack -> operate -> repack per tile on the GPU.
 *
 * CONVENTIONS (all entry points):
 *  - Host functions. Every pointer inside ms_column and ms_pred is a DEVICE
 *    pointer unless the function says "host". Work is enqueued on ctx->stream
 *    (a cudaStream_t; NULL = legacy default stream) of the current device.
 *  - Ownership: input columns and buffers are borrowed; the caller keeps them
 *    alive until the stream work completes. Output columns are allocated with
 *    ctx->alloc (one allocation per column, 256-byte aligned sections, recorded
 *    in column->alloc/alloc_bytes; NULL alloc => cudaMallocAsync) and belong to
 *    the caller, who frees them with ms_column_release().
 *  - Synchronisation: producers whose output size depends on the data
 *    (ms_select, block-format ms_compress / ms_morph / ms_project) synchronise
 *    the stream to read the size back into the descriptor; ms_agg_sum* never
 *    synchronise (results stay in device memory).
 *  - Errors: every function returns an ms_status. Host-side validation covers
 *    descriptor consistency; device-side checks (a code wider than a static
 *    width, a position out of range, a corrupt width table) are OR-ed into a
 *    device error word read back at the op's synchronisation point. On error
 *    *out is zeroed and nothing leaks. Error names follow SPEC.md:
 *    WidthOverflow S:41/119/154, UnsupportedFormat S:145/290, IndexOutOfRange
 *    S:59/290, CorruptBody S:127, LengthMismatch S:316.
 *  - No CPU fallback: every step runs in this library's sm_100a kernels.
 */
#ifndef MS_H
#define MS_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MS_ABI_VERSION 1

#if defined(__GNUC__)
#define MS_API __attribute__((visibility("default")))
#else
#define MS_API
#endif

/* Formats (P:420-421 lists static BP, SIMD-BP, DELTA and FOR cascades; RLE is
 * P:113-115, required by the north star). Normative byte layouts: DESIGN.md §3.
 *  MS_UNCOMPR    payload = n uint64 values.
 *  MS_STATIC_BP  "BP with one block and fixed bit width": value i at
 *                stream bits [i*w, i*w+w), LSB-first over little-endian uint64
 *                words (D-1), zero padding (D-2); no remainder (D-7).
 *  MS_DYN_BP     BP per block of B values at the block's effective bit width
 *                (SIMD-BP512 analog P:436): nb = floor(n/B) blocks,
 *                w_b = ebw(max code of block b), cw[0] = 0,
 *                cw[b+1] = cw[b] + w_b, block b packed like STATIC_BP{w_b} at
 *                payload word cw[b]*B/64 (D-4); the n mod B last values raw in
 *                rem, the "uncompressed remainder".
 *  MS_FOR_BP     DYN_BP over codes v - ref[b], ref[b] = block minimum (D-5).
 *  MS_DELTA_BP   DYN_BP over codes d_0 = 0, d_j = v_j - v_{j-1} mod 2^64 within
 *                the block, ref[b] = first value of the block (D-6).
 *  MS_RLE        maximal runs as (value, length) uint64 pairs (D-9). */
typedef enum {
  MS_UNCOMPR = 0, MS_STATIC_BP = 1, MS_DYN_BP = 2, MS_DELTA_BP = 3, MS_FOR_BP = 4, MS_RLE = 5
} ms_format;

/* Column descriptor {format, bit width, block size} (BASELINE.json north_star).
 * bit_width: STATIC_BP 1..64; 0 on an output spec = auto = max(1, ebw(max)).
 * block_size: DYN/FOR/DELTA 128, 256, 512, 1024 or 2048; ignored otherwise.
 * max_width: block formats: the largest block width of the column if known
 *   (1..64), 0 = unknown. Not part of the image; a sizing hint that libms
 *   producers fill in and scans use to pick narrower staging buffers. An
 *   understated hint costs speed, never correctness: a chunk that does not fit
 *   the staging buffer it sized is read from global memory instead. Ignored on
 *   output specs. */
typedef struct {
  int32_t format;
  uint32_t bit_width;
  uint32_t block_size;
  uint32_t max_width;
} ms_fmt;

/* A column: compressed main part + uncompressed remainder + metadata.
 * All pointers are device pointers. Footprint = the bytes of payload, cw, ref
 * and rem (ms_column_bytes). */
typedef struct {
  ms_fmt fmt;
  uint64_t n;             /* logical values (RLE: sum of run lengths) */
  uint64_t n_blocks;      /* block formats: floor(n/B); else 0 */
  uint64_t n_rem;         /* block formats: n mod B; else 0 */
  uint64_t n_runs;        /* RLE only */
  uint64_t payload_words; /* UNCOMPR n; STATIC_BP ceil(n*w/64); block formats cw[nb]*B/64; RLE 2*n_runs */
  uint64_t *payload;      /* uint64 words */
  uint32_t *cw;           /* block formats: n_blocks+1 cumulative widths; else NULL */
  uint64_t *ref;          /* FOR: block minima; DELTA: block bases; else NULL */
  uint64_t *rem;          /* block formats: n_rem raw values; else NULL */
  void *alloc;            /* owning allocation (library-produced columns), else NULL */
  uint64_t alloc_bytes;
} ms_column;

/* Select predicates (P:567-569 point predicate; S:271 comparison set; D-11):
 * unsigned comparisons against a; MS_BETWEEN is a <= v < b; MS_IN_BITMAP keeps
 * v iff v < bitmap_bits and bit v of the device bitmap (LSB-first uint64 words)
 * is set — a semi-join against a dense dimension bitmap (BASELINE configs[3]). */
typedef enum { MS_EQ = 0, MS_NE, MS_LT, MS_LE, MS_GT, MS_GE, MS_BETWEEN, MS_IN_BITMAP } ms_cmp;
typedef struct {
  int32_t op;
  uint32_t _reserved;
  uint64_t a, b;
  const uint64_t *bitmap; /* device */
  uint64_t bitmap_bits;
} ms_pred;

/* Allocation callbacks: PyTorch's caching allocator from the Python binding. */
typedef void *(*ms_alloc_fn)(void *alloc_ctx, size_t bytes, void *stream);
typedef void (*ms_free_fn)(void *alloc_ctx, void *ptr, void *stream);

#define MS_FLAG_SHRINK 1u /* copy variable-size outputs into an exact-size allocation (default: a producer
                           that sizes its output before the kernel keeps the slack of its provable capacity
                           in alloc_bytes; nothing is copied) */
#define MS_FLAG_GATHER 2u /* ms_project: always gather the data rows sector by sector, never stream the data
                           windows through shared memory (a measurement switch; the output is identical) */

typedef struct {
  void *stream;           /* cudaStream_t */
  ms_alloc_fn alloc;      /* NULL => cudaMallocAsync on stream */
  ms_free_fn free;
  void *alloc_ctx;
  uint32_t flags;
  uint32_t _reserved;
} ms_ctx;

typedef enum {
  MS_OK = 0, MS_E_INVALID, MS_E_WIDTH_OVERFLOW, MS_E_UNSUPPORTED, MS_E_RANGE, MS_E_CORRUPT, MS_E_NOMEM,
  MS_E_CUDA
} ms_status;

/* compress: encode n device values (uint64) into fmt.
 * values: device, n uint64, borrowed. MS_E_WIDTH_OVERFLOW if a STATIC_BP value
 * needs more than bit_width bits. MS_E_INVALID for a bad block size or
 * if a block format's cw[nb] would exceed 2^32-1 (D-4: shard such columns). */
MS_API ms_status ms_compress(const ms_ctx *ctx, const uint64_t *values, uint64_t n, ms_fmt fmt, ms_column *out);

/* decompress: decode column `in` into caller-owned device buffer values (n uint64)
 * (S:124-131). MS_E_CORRUPT if a block width exceeds 64 or cw decreases. */
MS_API ms_status ms_decompress(const ms_ctx *ctx, const ms_column *in, uint64_t *values);

/* morph: change the representation to fmt without a device round trip through
 * an uncompressed column (direct morphing): per tile decode(A) ->
 * encode(B). The result is byte-identical to compress(decompress(in), fmt)
 * (S:158); morph(x, x.fmt) is byte-identical to x. Every path decodes
 * the input tile by tile (no uncompressed copy of the column; DP3). */
MS_API ms_status ms_morph(const ms_ctx *ctx, const ms_column *in, ms_fmt fmt, ms_column *out);

/* select: positions row_offset + i of the rows i whose value satisfies pred,
 * strictly increasing, re-encoded in out_fmt (D-10).
 * row_offset makes positions global when a column is sharded by row range. */
MS_API ms_status ms_select(const ms_ctx *ctx, const ms_column *in, const ms_pred *pred, uint64_t row_offset,
                    ms_fmt out_fmt, ms_column *out_positions);

/* project: out_i = data[pos_i - row_offset], re-encoded in out_fmt (
 * S:286-290). Random access into any format (D-12: O(1) for UNCOMPR, STATIC_BP,
 * DYN_BP and FOR_BP; block-local for DELTA_BP; by run search for RLE).
 * MS_E_RANGE if a position lies outside [row_offset, row_offset + data->n).
 * out_fmt MS_RLE is MS_E_UNSUPPORTED. */
MS_API ms_status ms_project(const ms_ctx *ctx, const ms_column *data, const ms_column *positions, uint64_t row_offset,
                     ms_fmt out_fmt, ms_column *out);

/* agg_sum: *sum (device uint64) = sum of the column's values mod 2^64 (
 * D-13), or, with positions != NULL, of data[pos - row_offset] over positions
 * (select -> project -> sum fused). Uses the format identities where
 * they apply: RLE sum v*len, FOR B*ref + sum codes, DELTA
 * B*base + sum (B-j)*d_j. Never synchronises; *sum is overwritten.
 * Host-side validation errors are returned; device-side errors (MS_E_RANGE for
 * a position outside [row_offset, row_offset + in->n), MS_E_CORRUPT for a
 * corrupt RLE body or width table) are ORed into the library's sticky device
 * error word and reported ONLY by ms_check_errors (no other call reads it). */
MS_API ms_status ms_agg_sum(const ms_ctx *ctx, const ms_column *in, const ms_column *positions, uint64_t row_offset,
                     uint64_t *sum);

/* agg_sum_grouped: sums[g] = sum of vals_i with gid_i = g, g < n_groups, mod 2^64;
 * output uncompressed. sums: device, n_groups uint64,
 * overwritten. MS_E_INVALID if gid->n != vals->n (LengthMismatch S:316);
 * MS_E_RANGE if a gid >= n_groups (a device-side error: reported only by
 * ms_check_errors, like ms_agg_sum's). Never synchronises. */
MS_API ms_status ms_agg_sum_grouped(const ms_ctx *ctx, const ms_column *gid, const ms_column *vals, uint64_t n_groups,
                             uint64_t *sums);

/* Host <-> device transfer of a whole column image (the e2e path).
 * ms_column_to_device: host_col's section pointers are HOST pointers (pinned
 * memory makes the copies asynchronous); the result is a library-allocated
 * device column. ms_column_to_host: copies the device column's sections into
 * caller-owned HOST buffers given in host_col (pointers must be sized for the
 * device column's sections; descriptor fields are filled in). Both enqueue on
 * ctx->stream; ms_column_to_host synchronises. ms_column_to_device validates a
 * block-format image on the host before any allocation or copy: cw[0] = 0, cw
 * non-decreasing, every block width <= 64 and payload_words = cw[nb] * B / 64,
 * else MS_E_CORRUPT. */
MS_API ms_status ms_column_to_device(const ms_ctx *ctx, const ms_column *host_col, ms_column *out);
MS_API ms_status ms_column_to_host(const ms_ctx *ctx, const ms_column *dev_col, ms_column *host_col);

/* ---- plan-level operators (paper_2004_09350_b200/csrc/plan.cu) ---- */

/* Exact footprints (ms_column_bytes) of `in` re-encoded in each candidate format,
 * from ONE pass over the column (per block of block_size rows: max, min, largest
 * in-block delta; the column max; the run count) — the compression-rate objective
 * of the paper's cost-based format selection (DP2, P:66-68;
 * S:384-394). sizes (HOST, MS_N_CANDIDATES uint64) in the order UNCOMPR,
 * STATIC_BP (at its auto width), DYN_BP{block_size}, DELTA_BP{block_size},
 * FOR_BP{block_size}, RLE. *best (may be NULL) = the smallest, ties broken by that
 * order (simplest first). One synchronisation. */
#define MS_N_CANDIDATES 6
MS_API ms_status ms_format_sizes(const ms_ctx *ctx, const ms_column *in, uint32_t block_size, uint64_t *sizes,
                                 ms_fmt *best);

/* Sorted intersection / duplicate-free union of two strictly increasing position
 * columns (conjunctive / disjunctive predicates of star-schema plans),
 * out in out_fmt. Via a 1-bit mask over the inputs' common range and the select
 * output encoders. MS_E_INVALID if an input is not strictly increasing (NotSorted).
 * Two synchronisations (the inputs' ranges; the output size). */
MS_API ms_status ms_intersect(const ms_ctx *ctx, const ms_column *a, const ms_column *b, ms_fmt out_fmt,
                              ms_column *out);
MS_API ms_status ms_merge(const ms_ctx *ctx, const ms_column *a, const ms_column *b, ms_fmt out_fmt,
                          ms_column *out);

/* Group ids: out_ids[i] = dense id of the (prev_ids[i], keys[i])
 * combination in order of first occurrence (prev_ids may be NULL: keys alone);
 * out_extents[g] = row of the first occurrence of group g (strictly increasing
 * positions, in extents_fmt; UNCOMPR per S:309). max_groups: capacity hint of the
 * hash table (0 = keys->n); more distinct groups than the table holds is
 * MS_E_NOMEM. MS_E_INVALID if prev_ids->n != keys->n (LengthMismatch). */
MS_API ms_status ms_group(const ms_ctx *ctx, const ms_column *keys, const ms_column *prev_ids, uint64_t max_groups,
                          ms_fmt ids_fmt, ms_fmt extents_fmt, ms_column *out_ids, ms_column *out_extents);

/* Equi-join: all pairs (i, j) with left[i] == right[j] as two
 * position columns (positions into left, positions into right) in left_fmt /
 * right_fmt. The build side is the smaller column (right on a tie); pairs are in
 * probe-row order, then ascending build row. Hash table in device memory; the pair
 * lists are materialised uncompressed once before their compression. */
MS_API ms_status ms_join(const ms_ctx *ctx, const ms_column *left, const ms_column *right, ms_fmt left_fmt,
                         ms_fmt right_fmt, ms_column *out_left, ms_column *out_right);

/* Semi-join against a key bitmap (BJ.c4's star-schema join, D-16):
 * out = the positions p of `positions` (sorted row ids, global: row_offset + row
 * of `keys`) whose key keys[p - row_offset] is in the bitmap (bit k of bitmap[k/64]
 * for k < bitmap_bits), in out_fmt. Equal to project(positions, select(project(
 * keys, positions), IN_BITMAP)) — the fused form (K7) gathers the keys of each
 * 512-position block into shared memory and tests them there, so the projected
 * keys are never written; the surviving positions are set in a mask over the keys'
 * rows and encoded by the select output layer. MS_E_RANGE if a position lies
 * outside the keys; MS_E_INVALID if the positions are not strictly increasing (as
 * every positions column this library produces is). */
MS_API ms_status ms_semijoin(const ms_ctx *ctx, const ms_column *keys, const ms_column *positions,
                             uint64_t row_offset, const uint64_t *bitmap, uint64_t bitmap_bits, ms_fmt out_fmt,
                             ms_column *out);

/* Elementwise arithmetic mod 2^64 (star-schema measures such as
 * price x discount): out[i] = a[i] op b[i], op = MS_ADD / MS_SUB / MS_MUL.
 * MS_E_INVALID if a->n != b->n (LengthMismatch) or op is unknown. */
enum { MS_ADD = 0, MS_SUB = 1, MS_MUL = 2 };
MS_API ms_status ms_calc(const ms_ctx *ctx, int32_t op, const ms_column *a, const ms_column *b, ms_fmt out_fmt,
                         ms_column *out);

/* Reads and clears the library's sticky device error word for ctx->stream's
 * device (errors raised by the non-synchronising ops). Synchronises. */
MS_API ms_status ms_check_errors(const ms_ctx *ctx);

MS_API void ms_column_release(const ms_ctx *ctx, ms_column *col);
/* footprint in bytes: payload + cw + ref + rem (no padding, no descriptor) */
MS_API uint64_t ms_column_bytes(const ms_column *col);
MS_API const char *ms_status_str(ms_status s);
MS_API int ms_abi_version(void);
/* number of kernel launches this library issued in this process (instrumentation
 * for bench.py's gpu_launches) */
MS_API uint64_t ms_launch_count(void);

/* Kernel timing instrumentation: when enabled, every kernel launch is
 * bracketed by CUDA events recorded on its launching stream. ms_profile_read
 * waits for the recorded events, writes up to max per-kernel aggregates
 * (name, launches, summed milliseconds) into out (host), clears the records
 * and returns the number of distinct kernels. */
typedef struct {
  char name[48];
  uint64_t launches;
  double total_ms;
} ms_kernel_time;
MS_API void ms_profile_enable(int on);
MS_API int ms_profile_read(ms_kernel_time *out, int max);

#ifdef __cplusplus
}
#endif
#endif /* MS_H */
