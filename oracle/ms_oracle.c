/* ms_oracle.c — CPU ORACLE (test infrastructure only; see ms_oracle.h).
 *
 * Each function cites the passage it follows. PAPER.md = P:n,
 * SPEC.md = S:n, SURVEY.md §8(c) readings = D-n (all restated in DESIGN.md).
 */
#include "ms_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- NS / BP */

/* "the effective bit width of the largest value"; ebw(0) = 0 */
uint32_t orc_ebw(uint64_t v) {
  uint32_t w = 0;
  while (v) { ++w; v >>= 1; }
  return w;
}

/* stream bit b is bit (b mod 64) of word floor(b/64) — D-1 (LSB-first) */
static void set_bit(uint64_t *words, uint64_t b) { words[b / 64] |= (uint64_t)1 << (b % 64); }
static uint64_t get_bit(const uint64_t *words, uint64_t b) { return (words[b / 64] >> (b % 64)) & 1; }

/* write value v at stream bits [off, off+w), bit by bit */
static void put_code(uint64_t *words, uint64_t off, uint64_t v, uint32_t w) {
  for (uint32_t k = 0; k < w; ++k)
    if ((v >> k) & 1) set_bit(words, off + k);
}
static uint64_t get_code(const uint64_t *words, uint64_t off, uint32_t w) {
  uint64_t v = 0;
  for (uint32_t k = 0; k < w; ++k) v |= get_bit(words, off + k) << k;
  return v;
}

static uint64_t words_for(uint64_t n, uint32_t w) { return (n * (uint64_t)w + 63) / 64; }

/* static BP "with one block and fixed bit width"; value i at bits [i*w, i*w+w);
 * padding bits zero (D-2). Returns ORC_E_WIDTH_OVERFLOW if a value needs more than w bits. */
int orc_pack(const uint64_t *v, uint64_t n, uint32_t w, uint64_t *words) {
  if (w < 1 || w > 64) return ORC_E_INVALID;
  memset(words, 0, words_for(n, w) * 8);
  for (uint64_t i = 0; i < n; ++i) {
    if (orc_ebw(v[i]) > w) return ORC_E_WIDTH_OVERFLOW;
    put_code(words, i * w, v[i], w);
  }
  return ORC_OK;
}
void orc_unpack(const uint64_t *words, uint64_t n, uint32_t w, uint64_t *v) {
  for (uint64_t i = 0; i < n; ++i) v[i] = get_code(words, i * w, w);
}
/* random access by bit offset i*w */
uint64_t orc_get_at(const uint64_t *words, uint32_t w, uint64_t i) { return get_code(words, i * w, w); }

/* ----------------------------------------------------------------- column */

static int is_block_fmt(int32_t f) { return f == ORC_DYN_BP || f == ORC_DELTA_BP || f == ORC_FOR_BP; }
static int valid_block(uint32_t B) { return B == 128 || B == 256 || B == 512 || B == 1024 || B == 2048; }

void orc_free(orc_column *c) {
  if (!c) return;
  free(c->payload); free(c->cw); free(c->ref); free(c->rem);
  memset(c, 0, sizeof(*c));
}

/* footprint = bytes of (payload, cw, ref, rem) — SURVEY §8(c) c.2 "Footprint" */
uint64_t orc_footprint(const orc_column *c) {
  uint64_t bytes = 8 * c->payload_words;
  if (is_block_fmt(c->format)) {
    bytes += 4 * (c->n_blocks + 1) + 8 * c->n_rem;
    if (c->format != ORC_DYN_BP) bytes += 8 * c->n_blocks;
  }
  return bytes;
}

static void *zalloc(uint64_t bytes) { return calloc(bytes ? bytes : 1, 1); }

/* encode_F(v): the canonical image of each format (P:433-440 column layout; D-3..D-9) */
int orc_encode(const uint64_t *v, uint64_t n, int32_t format, uint32_t bit_width, uint32_t block_size,
               orc_column *out) {
  memset(out, 0, sizeof(*out));
  out->format = format;
  out->n = n;
  out->block_size = 1;
  if (format == ORC_UNCOMPR) {
    /* 64-bit values are the uncompressed base type */
    out->payload_words = n;
    out->payload = (uint64_t *)zalloc(8 * n);
    if (!out->payload) return ORC_E_NOMEM;
    for (uint64_t i = 0; i < n; ++i) out->payload[i] = v[i];
    return ORC_OK;
  }
  if (format == ORC_STATIC_BP) {
    uint32_t w = bit_width;
    if (w > 64) return ORC_E_INVALID;
    if (w == 0) { /* auto: max(1, ebw(max v)) (c.2) */
      uint64_t mx = 0;
      for (uint64_t i = 0; i < n; ++i) if (v[i] > mx) mx = v[i];
      w = orc_ebw(mx);
      if (w == 0) w = 1;
    }
    out->bit_width = w;
    out->payload_words = words_for(n, w);
    out->payload = (uint64_t *)zalloc(8 * out->payload_words);
    if (!out->payload) return ORC_E_NOMEM;
    int rc = orc_pack(v, n, w, out->payload);
    if (rc) { orc_free(out); return rc; }
    return ORC_OK;
  }
  if (format == ORC_RLE) {
    /* (value, length) pairs of maximal runs (D-9) */
    uint64_t runs = 0;
    for (uint64_t i = 0; i < n; ++i) if (i == 0 || v[i] != v[i - 1]) ++runs;
    out->n_runs = runs;
    out->payload_words = 2 * runs;
    out->payload = (uint64_t *)zalloc(16 * runs);
    if (!out->payload) return ORC_E_NOMEM;
    uint64_t r = 0;
    for (uint64_t i = 0; i < n; ++i) {
      if (i == 0 || v[i] != v[i - 1]) {
        out->payload[2 * r] = v[i];
        out->payload[2 * r + 1] = 0;
        ++r;
      }
      out->payload[2 * (r - 1) + 1] += 1;
    }
    return ORC_OK;
  }
  if (!is_block_fmt(format)) return ORC_E_UNSUPPORTED;
  if (!valid_block(block_size)) return ORC_E_INVALID;
  uint64_t B = block_size;
  uint64_t nb = n / B, nrem = n % B; /* compressed main part + remainder */
  out->block_size = block_size;
  out->n_blocks = nb;
  out->n_rem = nrem;
  out->cw = (uint32_t *)zalloc(4 * (nb + 1));
  out->rem = (uint64_t *)zalloc(8 * nrem);
  if (format != ORC_DYN_BP) out->ref = (uint64_t *)zalloc(8 * nb);
  uint64_t *codes = (uint64_t *)zalloc(8 * B);
  if (!out->cw || !out->rem || (format != ORC_DYN_BP && !out->ref) || !codes) {
    free(codes); orc_free(out); return ORC_E_NOMEM;
  }
  /* pass 1: per-block codes and widths (BP: per block, width of the largest value) */
  uint64_t total_w = 0;
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t *x = v + b * B;
    uint64_t refv = 0;
    if (format == ORC_FOR_BP) { /* FOR: difference to a reference value; ref = block min (D-5) */
      refv = x[0];
      for (uint64_t j = 1; j < B; ++j) if (x[j] < refv) refv = x[j];
      for (uint64_t j = 0; j < B; ++j) codes[j] = x[j] - refv;
    } else if (format == ORC_DELTA_BP) { /* DELTA: difference to the predecessor; base per block (D-6) */
      refv = x[0];
      codes[0] = 0;
      for (uint64_t j = 1; j < B; ++j) codes[j] = x[j] - x[j - 1]; /* mod 2^64 */
    } else {
      for (uint64_t j = 0; j < B; ++j) codes[j] = x[j];
    }
    uint64_t mx = 0;
    for (uint64_t j = 0; j < B; ++j) if (codes[j] > mx) mx = codes[j];
    uint32_t w = orc_ebw(mx);
    if (out->ref) out->ref[b] = refv;
    total_w += w;
    if (total_w > 0xFFFFFFFFull) { free(codes); orc_free(out); return ORC_E_INVALID; } /* D-4 limit */
    out->cw[b + 1] = (uint32_t)total_w;
  }
  out->payload_words = total_w * B / 64;
  out->payload = (uint64_t *)zalloc(8 * out->payload_words);
  if (!out->payload) { free(codes); orc_free(out); return ORC_E_NOMEM; }
  /* pass 2: pack block b at stream bit cw[b]*B (word cw[b]*B/64) */
  for (uint64_t b = 0; b < nb; ++b) {
    const uint64_t *x = v + b * B;
    uint32_t w = out->cw[b + 1] - out->cw[b];
    uint64_t base_bit = (uint64_t)out->cw[b] * B;
    for (uint64_t j = 0; j < B; ++j) {
      uint64_t code;
      if (format == ORC_FOR_BP) code = x[j] - out->ref[b];
      else if (format == ORC_DELTA_BP) code = j ? x[j] - x[j - 1] : 0;
      else code = x[j];
      put_code(out->payload, base_bit + j * w, code, w);
    }
  }
  for (uint64_t j = 0; j < nrem; ++j) out->rem[j] = v[nb * B + j]; /* uncompressed remainder */
  free(codes);
  return ORC_OK;
}

/* decode(c): the logical sequence (remainder taken into account) */
int orc_decode(const orc_column *c, uint64_t *v) {
  uint64_t n = c->n;
  if (c->format == ORC_UNCOMPR) {
    for (uint64_t i = 0; i < n; ++i) v[i] = c->payload[i];
    return ORC_OK;
  }
  if (c->format == ORC_STATIC_BP) {
    if (c->bit_width < 1 || c->bit_width > 64) return ORC_E_CORRUPT;
    orc_unpack(c->payload, n, c->bit_width, v);
    return ORC_OK;
  }
  if (c->format == ORC_RLE) {
    uint64_t i = 0;
    for (uint64_t r = 0; r < c->n_runs; ++r) {
      uint64_t len = c->payload[2 * r + 1];
      if (len == 0 || i + len > n) return ORC_E_CORRUPT;
      for (uint64_t k = 0; k < len; ++k) v[i++] = c->payload[2 * r];
    }
    return i == n ? ORC_OK : ORC_E_CORRUPT;
  }
  if (!is_block_fmt(c->format)) return ORC_E_UNSUPPORTED;
  uint64_t B = c->block_size;
  if (!valid_block((uint32_t)B) || c->n_blocks * B + c->n_rem != n || c->cw[0] != 0) return ORC_E_CORRUPT;
  for (uint64_t b = 0; b < c->n_blocks; ++b) {
    if (c->cw[b + 1] < c->cw[b] || c->cw[b + 1] - c->cw[b] > 64) return ORC_E_CORRUPT;
    uint32_t w = c->cw[b + 1] - c->cw[b];
    uint64_t base_bit = (uint64_t)c->cw[b] * B;
    uint64_t *x = v + b * B;
    for (uint64_t j = 0; j < B; ++j) {
      uint64_t code = get_code(c->payload, base_bit + j * w, w);
      if (c->format == ORC_FOR_BP) x[j] = c->ref[b] + code;
      else if (c->format == ORC_DELTA_BP) x[j] = j ? x[j - 1] + code : c->ref[b] + code; /* mod 2^64 */
      else x[j] = code;
    }
  }
  for (uint64_t j = 0; j < c->n_rem; ++j) v[c->n_blocks * B + j] = c->rem[j];
  return ORC_OK;
}

/* -------------------------------------------------------------- operators */

/* predicates of the select operator (D-11) */
static int pred(uint64_t x, int32_t op, uint64_t a, uint64_t b, const uint64_t *bm, uint64_t bits) {
  switch (op) {
    case ORC_EQ: return x == a;
    case ORC_NE: return x != a;
    case ORC_LT: return x < a;
    case ORC_LE: return x <= a;
    case ORC_GT: return x > a;
    case ORC_GE: return x >= a;
    case ORC_BETWEEN: return a <= x && x < b;
    case ORC_IN_BITMAP: return x < bits && ((bm[x / 64] >> (x % 64)) & 1);
  }
  return 0;
}

static int valid_op(int32_t op) { return op >= ORC_EQ && op <= ORC_IN_BITMAP; }

uint64_t orc_count_raw(const uint64_t *v, uint64_t n, int32_t op, uint64_t a, uint64_t b,
                       const uint64_t *bitmap, uint64_t bitmap_bits) {
  uint64_t cnt = 0;
  for (uint64_t i = 0; i < n; ++i) cnt += pred(v[i], op, a, b, bitmap, bitmap_bits) ? 1 : 0;
  return cnt;
}

static uint64_t *decode_alloc(const orc_column *c, int *rc) {
  uint64_t *v = (uint64_t *)zalloc(8 * c->n);
  if (!v) { *rc = ORC_E_NOMEM; return NULL; }
  *rc = orc_decode(c, v);
  if (*rc) { free(v); return NULL; }
  return v;
}

/* select: "outputs a sorted column containing the positions in the input column that store
 * matching data elements"; positions are row_offset + i (D-10), re-encoded in the
 * requested output format (on-the-fly de/re-compression). */
int orc_select(const orc_column *c, int32_t op, uint64_t a, uint64_t b, const uint64_t *bitmap,
               uint64_t bitmap_bits, uint64_t row_offset, int32_t out_format, uint32_t out_width,
               uint32_t out_block, orc_column *out) {
  memset(out, 0, sizeof(*out));
  if (!valid_op(op)) return ORC_E_INVALID;
  int rc;
  uint64_t *v = decode_alloc(c, &rc);
  if (!v) return rc;
  uint64_t *pos = (uint64_t *)zalloc(8 * c->n);
  if (!pos) { free(v); return ORC_E_NOMEM; }
  uint64_t m = 0;
  for (uint64_t i = 0; i < c->n; ++i)
    if (pred(v[i], op, a, b, bitmap, bitmap_bits)) pos[m++] = row_offset + i;
  rc = orc_encode(pos, m, out_format, out_width, out_block, out);
  free(v); free(pos);
  return rc;
}

/* project: out_i = data[pos_i - row_offset]; positions outside
 * [row_offset, row_offset + n) are an error. */
int orc_project(const orc_column *data, const orc_column *pos, uint64_t row_offset, int32_t out_format,
                uint32_t out_width, uint32_t out_block, orc_column *out) {
  memset(out, 0, sizeof(*out));
  int rc;
  uint64_t *v = decode_alloc(data, &rc);
  if (!v) return rc;
  uint64_t *p = decode_alloc(pos, &rc);
  if (!p) { free(v); return rc; }
  uint64_t *o = (uint64_t *)zalloc(8 * pos->n);
  if (!o) { free(v); free(p); return ORC_E_NOMEM; }
  for (uint64_t i = 0; i < pos->n; ++i) {
    if (p[i] < row_offset || p[i] - row_offset >= data->n) { free(v); free(p); free(o); return ORC_E_RANGE; }
    o[i] = v[p[i] - row_offset];
  }
  rc = orc_encode(o, pos->n, out_format, out_width, out_block, out);
  free(v); free(p); free(o);
  return rc;
}

/* sum: "aggregates all data elements" mod 2^64 (D-13); with positions, the sum of the
 * data at those positions (fused project+sum, same result as P:600-601's chain). */
int orc_agg_sum(const orc_column *c, const orc_column *pos, uint64_t row_offset, uint64_t *sum) {
  int rc;
  uint64_t *v = decode_alloc(c, &rc);
  if (!v) return rc;
  uint64_t s = 0;
  if (!pos) {
    for (uint64_t i = 0; i < c->n; ++i) s += v[i];
  } else {
    uint64_t *p = decode_alloc(pos, &rc);
    if (!p) { free(v); return rc; }
    for (uint64_t i = 0; i < pos->n; ++i) {
      if (p[i] < row_offset || p[i] - row_offset >= c->n) { free(v); free(p); return ORC_E_RANGE; }
      s += v[p[i] - row_offset];
    }
    free(p);
  }
  free(v);
  *sum = s;
  return ORC_OK;
}

/* grouped sum: out[k] = sum of vals_i with gid_i = k, uncompressed result */
int orc_agg_sum_grouped(const orc_column *gid, const orc_column *vals, uint64_t n_groups, uint64_t *sums) {
  if (gid->n != vals->n) return ORC_E_INVALID; /* LengthMismatch */
  int rc;
  uint64_t *g = decode_alloc(gid, &rc);
  if (!g) return rc;
  uint64_t *v = decode_alloc(vals, &rc);
  if (!v) { free(g); return rc; }
  for (uint64_t k = 0; k < n_groups; ++k) sums[k] = 0;
  for (uint64_t i = 0; i < gid->n; ++i) {
    if (g[i] >= n_groups) { free(g); free(v); return ORC_E_RANGE; }
    sums[g[i]] += v[i];
  }
  free(g); free(v);
  return ORC_OK;
}

/* morph: change the representation from one format to another; defined as
 * encode_F(decode(c)). */
int orc_morph(const orc_column *c, int32_t format, uint32_t bit_width, uint32_t block_size, orc_column *out) {
  memset(out, 0, sizeof(*out));
  int rc;
  uint64_t *v = decode_alloc(c, &rc);
  if (!v) return rc;
  rc = orc_encode(v, c->n, format, bit_width, block_size, out);
  free(v);
  return rc;
}
