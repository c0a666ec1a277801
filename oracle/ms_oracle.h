/* ms_oracle.h — the CPU ORACLE for the compression-enabled hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product (paper_2004_09350_b200/libms.so) never links, loads or calls it,
 * and the two share no source, header, table or helper. The only common text
 * is the format definition (DESIGN.md §3 "Normative formats", SURVEY.md §8(c)
 * c.2), which each side implements on its own.
 *
 * Style: plain, slow, obviously correct. Every format is encoded and decoded
 * value by value and bit by bit ("for k < w: set bit k"); every operator runs
 * on the fully decoded uint64 sequence, i.e. the paper's "purely
 * uncompressed" degree of integration wrapped by
 * decode/encode — the definitions of SURVEY.md §8(c) c.1.
 *
 * Pins: tests/test_oracle_*.py (not gpu) check every function here against
 * SPEC.md's worked examples, closed forms, brute force on tiny inputs and the
 * paper's printed numbers (Table tab:datach widths, simple-query footprints).
 * Nothing here is "parity unpinned".
 */
#ifndef MS_ORACLE_H
#define MS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* format tags (numeric values fixed by DESIGN.md §3; restated, not shared) */
enum { ORC_UNCOMPR = 0, ORC_STATIC_BP = 1, ORC_DYN_BP = 2, ORC_DELTA_BP = 3, ORC_FOR_BP = 4, ORC_RLE = 5 };
enum { ORC_EQ = 0, ORC_NE, ORC_LT, ORC_LE, ORC_GT, ORC_GE, ORC_BETWEEN, ORC_IN_BITMAP };
enum { ORC_OK = 0, ORC_E_INVALID, ORC_E_WIDTH_OVERFLOW, ORC_E_UNSUPPORTED, ORC_E_RANGE, ORC_E_CORRUPT,
       ORC_E_NOMEM };

typedef struct {
  int32_t format;
  uint32_t bit_width;   /* STATIC_BP: 1..64 (0 on input = auto) */
  uint32_t block_size;  /* DYN/DELTA/FOR: 128..2048 power of two; else 1 */
  uint32_t _pad;
  uint64_t n, n_blocks, n_rem, n_runs, payload_words;
  uint64_t *payload;    /* malloc'ed by the oracle */
  uint32_t *cw;         /* block formats: n_blocks+1 entries */
  uint64_t *ref;        /* FOR: block minimum; DELTA: block base */
  uint64_t *rem;        /* block formats: n_rem raw values */
} orc_column;

/* §2.1 NS: effective bit width */
uint32_t orc_ebw(uint64_t v);
/* static bit packing into an LSB-first stream */
int orc_pack(const uint64_t *v, uint64_t n, uint32_t w, uint64_t *words /* ceil(n*w/64) */);
void orc_unpack(const uint64_t *words, uint64_t n, uint32_t w, uint64_t *v);
uint64_t orc_get_at(const uint64_t *words, uint32_t w, uint64_t i);

int orc_encode(const uint64_t *v, uint64_t n, int32_t format, uint32_t bit_width, uint32_t block_size,
               orc_column *out);
int orc_decode(const orc_column *c, uint64_t *v /* c->n values */);
void orc_free(orc_column *c);
uint64_t orc_footprint(const orc_column *c);

int orc_select(const orc_column *c, int32_t op, uint64_t a, uint64_t b, const uint64_t *bitmap,
               uint64_t bitmap_bits, uint64_t row_offset, int32_t out_format, uint32_t out_width,
               uint32_t out_block, orc_column *out);
int orc_project(const orc_column *data, const orc_column *pos, uint64_t row_offset, int32_t out_format,
                uint32_t out_width, uint32_t out_block, orc_column *out);
int orc_agg_sum(const orc_column *c, const orc_column *pos /* NULL = all */, uint64_t row_offset,
                uint64_t *sum);
int orc_agg_sum_grouped(const orc_column *gid, const orc_column *vals, uint64_t n_groups, uint64_t *sums);
int orc_morph(const orc_column *c, int32_t format, uint32_t bit_width, uint32_t block_size, orc_column *out);

/* streaming helpers for the large configs: the same definitions applied to a
 * raw value array (no format), used to count/sum shard by shard */
uint64_t orc_count_raw(const uint64_t *v, uint64_t n, int32_t op, uint64_t a, uint64_t b,
                       const uint64_t *bitmap, uint64_t bitmap_bits);

#ifdef __cplusplus
}
#endif
#endif
