/*
 * essl_oracle.c -- CPU oracle for the ESSL loader hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain-C restatement of the
 * reference algorithm (cropload, /root/reference/pkg/src/cropload) used
 * as the parity checker for the CUDA path and as the CPU baseline in
 * bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2404_00509_b200) never links or calls it.
 *
 * Parity is pinned against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py, run with the reference importable)
 * -- see tests/test_oracle_golden.py.
 *
 * Every function cites the reference file:line it restates.  Paths are
 * relative to /root/reference/pkg/src/cropload/.
 *
 * Build: see oracle/Makefile (-O2 -ffp-contract=off: the reference's
 * float64 resize and float32 normalize are evaluated without FMA
 * contraction, imgops.py:24-60, :231-240).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ */
/* Status codes shared with the CUDA path (include/essl.h).            */
/* ------------------------------------------------------------------ */
enum {
  ST_OK = 0,
  ST_CORRUPT_HUFFMAN = 1,   /* decode_kernels.py:14-15 status 1 */
  ST_MISSING_RST = 3,       /* status 3 */
  ST_TRUNCATED = 4,         /* codec.py:329-330 */
  ST_CRC = 5,               /* container.py:263-264 */
  ST_UNSUPPORTED = 6,       /* progressive / multi-scan (ref falls back) */
  ST_RECT = 7,              /* codec.py:52-56 ValueError */
  ST_MALFORMED = 8,         /* parse_stream DecodeError family */
  ST_HUFFTABLE = 9,         /* _huff_lut errors, codec.py:274-287 */
  ST_QUANT = 10,            /* _quant_for, codec.py:405-409 */
};

/* Reason codes for ST_MALFORMED / ST_UNSUPPORTED / ST_HUFFTABLE (message
 * text lives on the host side, paper_2404_00509_b200/errors.py). */
enum {
  R_NONE = 0,
  R_NO_SOI = 1,          /* codec.py:126-127 */
  R_EXPECTED_MARKER = 2, /* :138-139 */
  R_UNEXPECTED_END = 3,  /* :104-105 */
  R_TRUNC_SEGMENT = 4,   /* :151-152 */
  R_TRUNC_DQT = 5,       /* :162-163 */
  R_TRUNC_DHT = 6,       /* :179-180, :184-185 */
  R_MULTI_SOF = 7,       /* :189-190 */
  R_PRECISION = 8,       /* :193-194 */
  R_ZERO_DIM = 9,        /* :198-199 */
  R_NCOMP = 10,          /* :200-201 */
  R_SAMPLING = 11,       /* :210-211 */
  R_SOF_TYPE = 12,       /* :213-217 */
  R_SOS_BEFORE_SOF = 13, /* :221-222 */
  R_UNKNOWN_COMP = 14,   /* :232-233 */
  R_NO_IMAGE = 15,       /* :248-249 */
  R_RST_NO_DRI = 16,     /* :316-317 */
  R_TOO_MANY_RST = 17,   /* :318-319 */
  R_PROGRESSIVE = 18,    /* :461-469 fallback (unsupported here) */
  R_MULTI_SCAN = 19,
  R_HUFF_UNDEFINED = 20, /* :274-275 */
  R_HUFF_OVERFLOW = 21,  /* :286-287 */
  R_HUFF_TOO_MANY = 22,  /* > 256 symbols (builder limit, not in ref) */
  R_SEGMENT = 23,        /* segment body shorter than its fields */
};

/* ------------------------------------------------------------------ */
/* rng.py: splitmix64 counter streams                                   */
/* ------------------------------------------------------------------ */
#define GAMMA 0x9E3779B97F4A7C15ULL
#define MIX1 0xBF58476D1CE4E5B9ULL
#define MIX2 0x94D049BB133111EBULL

static inline uint64_t mix64(uint64_t z) { /* rng.py:27-31 */
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}

ORC_API uint64_t orc_rng_init(uint64_t seed, uint64_t epoch, uint64_t index,
                              uint64_t domain) { /* rng.py:39-44 */
  uint64_t h = mix64(seed);
  h = mix64(h ^ (epoch * GAMMA));
  h = mix64(h ^ (index * GAMMA));
  h = mix64(h ^ (domain * GAMMA));
  return h;
}

ORC_API uint64_t orc_rng_next(uint64_t *st) { /* rng.py:46-48 */
  *st += GAMMA;
  return mix64(*st);
}

ORC_API double orc_rng_random(uint64_t *st) { /* rng.py:50-52 */
  return (double)(orc_rng_next(st) >> 11) * 0x1p-53;
}

static inline double rng_uniform(uint64_t *st, double lo, double hi) {
  return lo + (hi - lo) * orc_rng_random(st); /* rng.py:54-55 */
}

ORC_API int64_t orc_rng_randint(uint64_t *st, int64_t n) { /* rng.py:57-60 */
  double r = orc_rng_random(st) * (double)n;
  int64_t v = (int64_t)r;
  return v >= n ? n - 1 : v;
}

ORC_API void orc_epoch_permutation(uint64_t seed, uint64_t epoch, int64_t n,
                                   int64_t *out) { /* rng.py:80-87 */
  uint64_t st = orc_rng_init(seed, epoch, 0, 3);
  for (int64_t i = 0; i < n; i++) out[i] = i;
  for (int64_t i = n - 1; i > 0; i--) {
    int64_t j = orc_rng_randint(&st, i + 1);
    int64_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
}

/* pipeline.py:51-75 sample_rrc. out = {x, y, w, h}. */
ORC_API void orc_sample_rrc(uint64_t *st, int64_t src_w, int64_t src_h,
                            double scale_lo, double scale_hi, double ratio_lo,
                            double ratio_hi, int max_attempts, int32_t *out) {
  double area = (double)(src_w * src_h);
  double log_lo = log(ratio_lo), log_hi = log(ratio_hi);
  for (int a = 0; a < max_attempts; a++) {
    double target = area * rng_uniform(st, scale_lo, scale_hi);
    double aspect = exp(rng_uniform(st, log_lo, log_hi));
    int64_t w = (int64_t)(sqrt(target * aspect) + 0.5);
    int64_t h = (int64_t)(sqrt(target / aspect) + 0.5);
    if (0 < w && w <= src_w && 0 < h && h <= src_h) {
      int64_t x = orc_rng_randint(st, src_w - w + 1);
      int64_t y = orc_rng_randint(st, src_h - h + 1);
      out[0] = (int32_t)x; out[1] = (int32_t)y;
      out[2] = (int32_t)w; out[3] = (int32_t)h;
      return;
    }
  }
  double in_ratio = (double)src_w / (double)src_h;
  int64_t w, h;
  if (in_ratio < ratio_lo) {
    w = src_w;
    int64_t t = (int64_t)((double)w / ratio_lo + 0.5);
    if (t < 1) t = 1;
    h = t < src_h ? t : src_h;
  } else if (in_ratio > ratio_hi) {
    h = src_h;
    int64_t t = (int64_t)((double)h * ratio_hi + 0.5);
    if (t < 1) t = 1;
    w = t < src_w ? t : src_w;
  } else {
    w = src_w;
    h = src_h;
  }
  out[0] = (int32_t)((src_w - w) / 2); out[1] = (int32_t)((src_h - h) / 2);
  out[2] = (int32_t)w; out[3] = (int32_t)h;
}

/* masking.py:44-45 masked_count = floor(ratio*tokens + 0.5) */
ORC_API int orc_mask_count(int tokens, double ratio) {
  return (int)floor(ratio * (double)tokens + 0.5);
}

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* masking.py:48-56 sample_mask + rng.py:73-77 shuffle. */
ORC_API void orc_sample_mask(uint64_t *st, int n, int k, int32_t *out) {
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
  for (int i = 0; i < n; i++) perm[i] = i;
  for (int i = n - 1; i > 0; i--) {
    int64_t j = orc_rng_randint(st, i + 1);
    int32_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  memcpy(out, perm, sizeof(int32_t) * k);
  qsort(out, k, sizeof(int32_t), cmp_i32);
  free(perm);
}

/* ------------------------------------------------------------------ */
/* CRC32 (zlib polynomial), container.py:263                           */
/* ------------------------------------------------------------------ */
static uint32_t crc_table[256];
static pthread_once_t crc_once = PTHREAD_ONCE_INIT;
static void crc_init(void) {
  for (uint32_t i = 0; i < 256; i++) {
    uint32_t c = i;
    for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    crc_table[i] = c;
  }
}
ORC_API uint32_t orc_crc32(const uint8_t *p, size_t n) {
  pthread_once(&crc_once, crc_init);
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; i++) c = crc_table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

/* ------------------------------------------------------------------ */
/* JPEG: tables.py:14-23 zigzag                                         */
/* ------------------------------------------------------------------ */
static const int ZZ[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

typedef struct {
  int defined;
  uint8_t bits[16];
  int nvals;
  uint8_t vals[256];
} HuffSpec;

typedef struct {
  int cid, h, v, tq;
  int w, ph, bw, bh, BW, BH; /* codec.py:254-265 */
} Comp;

typedef struct {
  int ns;
  int comp[4];            /* frame component index per slot */
  HuffSpec dc[4], ac[4];  /* snapshot at SOS time, codec.py:234-236 */
  int ss, se, ah, al, ri;
  int start, end;
} Scan;

typedef struct {
  int width, height, progressive, ncomp;
  Comp comps[4];
  int has_quant[16];
  int32_t quant[16][64]; /* natural order */
  int nscans;
  Scan scan; /* first scan only (fast path needs exactly one) */
  int hmax, vmax, mcus_x, mcus_y;
} Frame;

typedef struct {
  int status, reason, offset;
} Err;

#define FAIL(st, rs, off)                                                   \
  do {                                                                      \
    e->status = (st); e->reason = (rs); e->offset = (off);                  \
    return -1;                                                              \
  } while (0)

static int rd_u16(const uint8_t *d, int n, int pos, int *v, Err *e) {
  if (pos + 2 > n) FAIL(ST_MALFORMED, R_UNEXPECTED_END, pos); /* codec.py:103-106 */
  *v = (d[pos] << 8) | d[pos + 1];
  return 0;
}

/* codec.py:109-121 */
static int entropy_end(const uint8_t *d, int n, int pos) {
  for (;;) {
    while (pos < n && d[pos] != 0xFF) pos++;
    if (pos >= n || pos + 1 >= n) return n;
    int m = d[pos + 1];
    if (m == 0x00 || (m >= 0xD0 && m <= 0xD7) || m == 0xFF) {
      pos += (m != 0xFF) ? 2 : 1;
      continue;
    }
    return pos;
  }
}

/* codec.py:124-251 parse_stream (+ _finish_geometry 254-265). */
static int parse_stream(const uint8_t *d, int n, Frame *f, Err *e) {
  HuffSpec huff[2][16];
  memset(huff, 0, sizeof(huff));
  memset(f, 0, sizeof(*f));
  int have_sof = 0, ri = 0;
  if (n < 4 || d[0] != 0xFF || d[1] != 0xD8) FAIL(ST_MALFORMED, R_NO_SOI, 0);
  int pos = 2;
  while (pos < n) {
    if (d[pos] != 0xFF) FAIL(ST_MALFORMED, R_EXPECTED_MARKER, pos);
    while (pos < n && d[pos] == 0xFF) pos++;
    if (pos >= n) break;
    int marker = d[pos++];
    if (marker == 0xD9) break;
    if (marker == 0x01 || (marker >= 0xD0 && marker <= 0xD7)) continue;
    int seglen;
    if (rd_u16(d, n, pos, &seglen, e)) return -1;
    if (seglen < 2 || pos + seglen > n) FAIL(ST_MALFORMED, R_TRUNC_SEGMENT, pos);
    int body = pos + 2, end = pos + seglen;
    if (marker == 0xDB) { /* DQT */
      int p = body;
      while (p < end) {
        int pq = d[p] >> 4, tq = d[p] & 15;
        p++;
        int count = 64 * (pq == 1 ? 2 : 1);
        if (p + count > end) FAIL(ST_MALFORMED, R_TRUNC_DQT, p);
        for (int k = 0; k < 64; k++) {
          int val = pq == 1 ? ((d[p + 2 * k] << 8) | d[p + 2 * k + 1]) : d[p + k];
          f->quant[tq][ZZ[k]] = val;
        }
        f->has_quant[tq] = 1;
        p += count;
      }
    } else if (marker == 0xC4) { /* DHT */
      int p = body;
      while (p < end) {
        int tc = d[p] >> 4, th = d[p] & 15;
        p++;
        if (p + 16 > end) FAIL(ST_MALFORMED, R_TRUNC_DHT, p);
        int total = 0;
        uint8_t bits[16];
        for (int i = 0; i < 16; i++) { bits[i] = d[p + i]; total += bits[i]; }
        p += 16;
        if (p + total > end) FAIL(ST_MALFORMED, R_TRUNC_DHT, p);
        if (tc < 2) {
          HuffSpec *h = &huff[tc][th];
          h->defined = total <= 256 ? 1 : 2;
          memcpy(h->bits, bits, 16);
          h->nvals = total <= 256 ? total : 256;
          memcpy(h->vals, d + p, h->nvals);
        }
        p += total;
      }
    } else if (marker == 0xC0 || marker == 0xC1 || marker == 0xC2) { /* SOF */
      if (have_sof) FAIL(ST_MALFORMED, R_MULTI_SOF, pos);
      if (body + 6 > n) FAIL(ST_MALFORMED, R_SEGMENT, body);
      f->progressive = marker == 0xC2;
      if (d[body] != 8) FAIL(ST_MALFORMED, R_PRECISION, body);
      if (rd_u16(d, n, body + 1, &f->height, e)) return -1;
      if (rd_u16(d, n, body + 3, &f->width, e)) return -1;
      int nc = d[body + 5];
      if (f->height == 0 || f->width == 0) FAIL(ST_MALFORMED, R_ZERO_DIM, body + 1);
      if (nc != 1 && nc != 3) FAIL(ST_MALFORMED, R_NCOMP, body + 5);
      int p = body + 6;
      if (p + 3 * nc > n) FAIL(ST_MALFORMED, R_SEGMENT, p);
      for (int i = 0; i < nc; i++) {
        f->comps[i].cid = d[p];
        f->comps[i].h = d[p + 1] >> 4;
        f->comps[i].v = d[p + 1] & 15;
        f->comps[i].tq = d[p + 2];
        p += 3;
      }
      for (int i = 0; i < nc; i++) {
        int h = f->comps[i].h, v = f->comps[i].v;
        if (!(h == 1 || h == 2 || h == 4) || !(v == 1 || v == 2 || v == 4))
          FAIL(ST_MALFORMED, R_SAMPLING, pos);
      }
      f->ncomp = nc;
      have_sof = 1;
    } else if (marker == 0xC3 || marker == 0xC5 || marker == 0xC6 ||
               marker == 0xC7 || marker == 0xC9 || marker == 0xCA ||
               marker == 0xCB || marker == 0xCD || marker == 0xCE ||
               marker == 0xCF) {
      FAIL(ST_MALFORMED, R_SOF_TYPE, pos);
    } else if (marker == 0xDD) { /* DRI */
      if (rd_u16(d, n, body, &ri, e)) return -1;
    } else if (marker == 0xDA) { /* SOS */
      if (!have_sof) FAIL(ST_MALFORMED, R_SOS_BEFORE_SOF, pos);
      if (body >= n) FAIL(ST_MALFORMED, R_SEGMENT, body);
      int ns = d[body], p = body + 1;
      if (p + 2 * ns + 3 > n) FAIL(ST_MALFORMED, R_SEGMENT, p);
      Scan sc;
      memset(&sc, 0, sizeof(sc));
      sc.ns = ns;
      for (int s = 0; s < ns; s++) {
        int cs = d[p], td = d[p + 1] >> 4, ta = d[p + 1] & 15;
        int idx = -1;
        for (int i = 0; i < f->ncomp; i++)
          if (f->comps[i].cid == cs) { idx = i; break; }
        if (idx < 0) FAIL(ST_MALFORMED, R_UNKNOWN_COMP, p);
        if (s < 4) {
          sc.comp[s] = idx;
          sc.dc[s] = huff[0][td];
          sc.ac[s] = huff[1][ta];
        }
        p += 2;
      }
      sc.ss = d[p]; sc.se = d[p + 1]; sc.ah = d[p + 2] >> 4; sc.al = d[p + 2] & 15;
      sc.ri = ri;
      sc.start = end;
      sc.end = entropy_end(d, n, end);
      if (f->nscans == 0) f->scan = sc;
      f->nscans++;
      pos = sc.end;
      continue;
    }
    pos = end;
  }
  if (!have_sof || f->nscans == 0) FAIL(ST_MALFORMED, R_NO_IMAGE, pos);
  /* _finish_geometry */
  f->hmax = f->vmax = 1;
  for (int i = 0; i < f->ncomp; i++) {
    if (f->comps[i].h > f->hmax) f->hmax = f->comps[i].h;
    if (f->comps[i].v > f->vmax) f->vmax = f->comps[i].v;
  }
  f->mcus_x = (f->width + 8 * f->hmax - 1) / (8 * f->hmax);
  f->mcus_y = (f->height + 8 * f->vmax - 1) / (8 * f->vmax);
  for (int i = 0; i < f->ncomp; i++) {
    Comp *c = &f->comps[i];
    c->w = (f->width * c->h + f->hmax - 1) / f->hmax;
    c->ph = (f->height * c->v + f->vmax - 1) / f->vmax;
    c->bw = (c->w + 7) / 8;
    c->bh = (c->ph + 7) / 8;
    c->BW = f->mcus_x * c->h;
    c->BH = f->mcus_y * c->v;
  }
  return 0;
}

/* codec.py:272-295 _huff_lut: 16-bit lookahead, (sym<<8)|len, -1 bad. */
static int huff_lut(const HuffSpec *h, int32_t *lut, Err *e) {
  if (!h->defined) FAIL(ST_HUFFTABLE, R_HUFF_UNDEFINED, -1);
  if (h->defined == 2) FAIL(ST_HUFFTABLE, R_HUFF_TOO_MANY, -1);
  for (int i = 0; i < 65536; i++) lut[i] = -1;
  int code = 0, vi = 0;
  for (int len = 1; len <= 16; len++) {
    for (int c = 0; c < h->bits[len - 1]; c++) {
      if (code >= (1 << len)) FAIL(ST_HUFFTABLE, R_HUFF_OVERFLOW, -1);
      int start = code << (16 - len);
      int32_t ent = ((int32_t)h->vals[vi] << 8) | len;
      for (int k = 0; k < (1 << (16 - len)); k++) lut[start + k] = ent;
      code++;
      vi++;
    }
    code <<= 1;
  }
  return 0;
}

/* decode_kernels.py:27-61 destuff_scan. Returns clean length. */
ORC_API int orc_destuff(const uint8_t *raw, int start, int n, uint8_t *out,
                        int64_t *restarts, int max_r, int *n_restarts,
                        int *end_out) {
  int i = start, o = 0, r = 0;
  while (i < n) {
    uint8_t b = raw[i];
    if (b == 0xFF) {
      if (i + 1 >= n) break;
      uint8_t m = raw[i + 1];
      if (m == 0x00) { out[o++] = 0xFF; i += 2; continue; }
      if (m >= 0xD0 && m <= 0xD7) {
        if (r < max_r) restarts[r] = o;
        r++;
        i += 2;
        continue;
      }
      break;
    }
    out[o++] = b;
    i++;
  }
  *n_restarts = r;
  if (end_out) *end_out = i;
  return o;
}

/* Bit reader, decode_kernels.py:64-108.  vpos counts bytes loaded into a
 * 40-bit window (0xFF past the end), cnt = valid bits. */
typedef struct {
  const uint8_t *data;
  int64_t n;
  int64_t vpos;
  uint64_t buf;
  int cnt;
} BR;

static inline void br_fill(BR *b) {
  while (b->cnt < 25) {
    uint64_t byte = b->vpos < b->n ? b->data[b->vpos] : 0xFF;
    b->buf = ((b->buf << 8) | byte) & 0xFFFFFFFFFFULL;
    b->cnt += 8;
    b->vpos++;
  }
}
static inline int br_hd(BR *b, const int32_t *lut) {
  br_fill(b);
  int32_t ent = lut[(b->buf >> (b->cnt - 16)) & 0xFFFF];
  if (ent < 0) return -1;
  b->cnt -= ent & 0xFF;
  return ent >> 8;
}
static inline int br_gb(BR *b, int nbits) {
  if (nbits == 0) return 0;
  br_fill(b);
  int v = (int)((b->buf >> (b->cnt - nbits)) & ((1u << nbits) - 1));
  b->cnt -= nbits;
  return v;
}
static inline int extend(int v, int size) {
  if (size == 0) return 0;
  if (v < (1 << (size - 1))) return v - (1 << size) + 1;
  return v;
}

/* decode_kernels.py:111-179 decode_scan_baseline.  Coefficient arrays
 * are int32 [BH][BW][64] per component (natural order). */
static int decode_scan_baseline(const uint8_t *data, int64_t clean_len,
                                const int64_t *restarts, int n_restarts,
                                int ri, int32_t *const *luts_dc,
                                int32_t *const *luts_ac, const int *comp_sel,
                                const int *comp_h, const int *comp_v, int ns,
                                int mx_count, int row_stop, int32_t **coefs,
                                const int *coef_bw, int64_t *vpos_out,
                                int *cnt_out) {
  BR b = {data, clean_len, 0, 0, 0};
  int64_t preds[4] = {0, 0, 0, 0};
  int64_t mcu = 0;
  int rseg = 0;
  for (int my = 0; my < row_stop; my++) {
    for (int mx = 0; mx < mx_count; mx++) {
      if (ri > 0 && mcu > 0 && mcu % ri == 0) {
        if (rseg >= n_restarts) { *vpos_out = b.vpos; *cnt_out = b.cnt; return 3; }
        b.vpos = restarts[rseg];
        b.buf = 0;
        b.cnt = 0;
        rseg++;
        for (int s = 0; s < ns; s++) preds[s] = 0;
      }
      for (int s = 0; s < ns; s++) {
        int ci = comp_sel[s];
        int32_t *tgt = coefs[ci];
        int bwid = coef_bw[ci];
        int vv = comp_v[s], hh = comp_h[s];
        for (int by = 0; by < vv; by++) {
          int brow = my * vv + by;
          for (int bx = 0; bx < hh; bx++) {
            int bcol = mx * hh + bx;
            int32_t *blk = tgt + ((int64_t)brow * bwid + bcol) * 64;
            int sym = br_hd(&b, luts_dc[s]);
            if (sym < 0 || sym > 15) { *vpos_out = b.vpos; *cnt_out = b.cnt; return 1; }
            int dv = br_gb(&b, sym);
            preds[s] += extend(dv, sym);
            blk[0] = (int32_t)preds[s];
            int k = 1;
            while (k < 64) {
              int rs = br_hd(&b, luts_ac[s]);
              if (rs < 0) { *vpos_out = b.vpos; *cnt_out = b.cnt; return 1; }
              int r = rs >> 4, sz = rs & 15;
              if (sz == 0) {
                if (r == 15) { k += 16; continue; }
                break;
              }
              k += r;
              if (k > 63) { *vpos_out = b.vpos; *cnt_out = b.cnt; return 1; }
              int av = br_gb(&b, sz);
              blk[ZZ[k]] = extend(av, sz);
              k++;
            }
          }
        }
      }
      mcu++;
    }
  }
  *vpos_out = b.vpos;
  *cnt_out = b.cnt;
  return 0;
}

/* decode_kernels.py:388-534 reconstruct_blocks (int64 islow IDCT). */
#define F_0_298631336 2446
#define F_0_390180644 3196
#define F_0_541196100 4433
#define F_0_765366865 6270
#define F_0_899976223 7373
#define F_1_175875602 9633
#define F_1_501321110 12299
#define F_1_847759065 15137
#define F_1_961570560 16069
#define F_2_053119869 16819
#define F_2_562915447 20995
#define F_3_072711026 25172

ORC_API void orc_idct_block(const int32_t *coef, const int32_t *quant,
                            uint8_t *dst, int stride) {
  int64_t ws[64];
  for (int col = 0; col < 8; col++) {
    int64_t d0 = (int64_t)coef[col] * quant[col];
    int64_t d1 = (int64_t)coef[col + 8] * quant[col + 8];
    int64_t d2 = (int64_t)coef[col + 16] * quant[col + 16];
    int64_t d3 = (int64_t)coef[col + 24] * quant[col + 24];
    int64_t d4 = (int64_t)coef[col + 32] * quant[col + 32];
    int64_t d5 = (int64_t)coef[col + 40] * quant[col + 40];
    int64_t d6 = (int64_t)coef[col + 48] * quant[col + 48];
    int64_t d7 = (int64_t)coef[col + 56] * quant[col + 56];
    if (!d1 && !d2 && !d3 && !d4 && !d5 && !d6 && !d7) {
      int64_t dc = d0 * 4; /* d0 << 2 */
      for (int i = 0; i < 8; i++) ws[col + 8 * i] = dc;
      continue;
    }
    int64_t z1 = (d2 + d6) * F_0_541196100;
    int64_t t2 = z1 - d6 * F_1_847759065;
    int64_t t3 = z1 + d2 * F_0_765366865;
    int64_t t0 = (d0 + d4) * 8192;
    int64_t t1 = (d0 - d4) * 8192;
    int64_t t10 = t0 + t3, t13 = t0 - t3, t11 = t1 + t2, t12 = t1 - t2;
    int64_t o0 = d7, o1 = d5, o2 = d3, o3 = d1;
    z1 = o0 + o3;
    int64_t z2 = o1 + o2, z3 = o0 + o2, z4 = o1 + o3;
    int64_t z5 = (z3 + z4) * F_1_175875602;
    o0 *= F_0_298631336; o1 *= F_2_053119869;
    o2 *= F_3_072711026; o3 *= F_1_501321110;
    z1 = -z1 * F_0_899976223; z2 = -z2 * F_2_562915447;
    z3 = -z3 * F_1_961570560 + z5; z4 = -z4 * F_0_390180644 + z5;
    o0 += z1 + z3; o1 += z2 + z4; o2 += z2 + z3; o3 += z1 + z4;
    ws[col] = (t10 + o3 + 1024) >> 11;
    ws[col + 56] = (t10 - o3 + 1024) >> 11;
    ws[col + 8] = (t11 + o2 + 1024) >> 11;
    ws[col + 48] = (t11 - o2 + 1024) >> 11;
    ws[col + 16] = (t12 + o1 + 1024) >> 11;
    ws[col + 40] = (t12 - o1 + 1024) >> 11;
    ws[col + 24] = (t13 + o0 + 1024) >> 11;
    ws[col + 32] = (t13 - o0 + 1024) >> 11;
  }
  for (int row = 0; row < 8; row++) {
    int64_t *w = ws + row * 8;
    uint8_t *o = dst + (int64_t)row * stride;
    if (!w[1] && !w[2] && !w[3] && !w[4] && !w[5] && !w[6] && !w[7]) {
      int64_t v = ((w[0] + 16) >> 5) + 128;
      v = v < 0 ? 0 : v > 255 ? 255 : v;
      for (int i = 0; i < 8; i++) o[i] = (uint8_t)v;
      continue;
    }
    int64_t z1 = (w[2] + w[6]) * F_0_541196100;
    int64_t t2 = z1 - w[6] * F_1_847759065;
    int64_t t3 = z1 + w[2] * F_0_765366865;
    int64_t t0 = (w[0] + w[4]) * 8192;
    int64_t t1 = (w[0] - w[4]) * 8192;
    int64_t t10 = t0 + t3, t13 = t0 - t3, t11 = t1 + t2, t12 = t1 - t2;
    int64_t o0 = w[7], o1 = w[5], o2 = w[3], o3 = w[1];
    z1 = o0 + o3;
    int64_t z2 = o1 + o2, z3 = o0 + o2, z4 = o1 + o3;
    int64_t z5 = (z3 + z4) * F_1_175875602;
    o0 *= F_0_298631336; o1 *= F_2_053119869;
    o2 *= F_3_072711026; o3 *= F_1_501321110;
    z1 = -z1 * F_0_899976223; z2 = -z2 * F_2_562915447;
    z3 = -z3 * F_1_961570560 + z5; z4 = -z4 * F_0_390180644 + z5;
    o0 += z1 + z3; o1 += z2 + z4; o2 += z2 + z3; o3 += z1 + z4;
    int64_t r[8];
    r[0] = ((t10 + o3 + 131072) >> 18) + 128;
    r[7] = ((t10 - o3 + 131072) >> 18) + 128;
    r[1] = ((t11 + o2 + 131072) >> 18) + 128;
    r[6] = ((t11 - o2 + 131072) >> 18) + 128;
    r[2] = ((t12 + o1 + 131072) >> 18) + 128;
    r[5] = ((t12 - o1 + 131072) >> 18) + 128;
    r[3] = ((t13 + o0 + 131072) >> 18) + 128;
    r[4] = ((t13 - o0 + 131072) >> 18) + 128;
    for (int i = 0; i < 8; i++) {
      int64_t v = r[i];
      o[i] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
    }
  }
}

static inline uint8_t clamp255(int v) { return (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v); }

/* ------------------------------------------------------------------ */
/* decode_crop, codec.py:448-511                                        */
/* ------------------------------------------------------------------ */
typedef struct {
  Frame f;
  int row_stop, mx0, mx1, my0, my1, gx, gy;
  int32_t *coefs[4];
  int coef_bw[4];
  uint8_t *planes[4];
  int plane_stride[4];
  int64_t clean_len;
  uint8_t *clean;
} DecodeState;

static void ds_free(DecodeState *s) {
  for (int i = 0; i < 4; i++) { free(s->coefs[i]); free(s->planes[i]); }
  free(s->clean);
  memset(s, 0, sizeof(*s));
}

/* Runs parse + validate + entropy decode up to row_stop.  On success the
 * coefficient arrays are allocated and filled. */
static int decode_entropy(const uint8_t *data, int n, int x, int y, int w,
                          int h, int full, DecodeState *s, Err *e) {
  memset(s, 0, sizeof(*s));
  Frame *f = &s->f;
  if (parse_stream(data, n, f, e)) return -1;
  if (full) { x = 0; y = 0; w = f->width; h = f->height; }
  if (w < 1 || h < 1 || x < 0 || y < 0 || x + w > f->width || y + h > f->height)
    FAIL(ST_RECT, R_NONE, -1); /* codec.py:52-56 */
  /* fast-path predicate codec.py:461-462; the reference falls back to a
   * full CPU decode otherwise -- the GPU path reports unsupported. */
  if (f->progressive) FAIL(ST_UNSUPPORTED, R_PROGRESSIVE, -1);
  if (f->nscans != 1 || f->scan.ns != f->ncomp) FAIL(ST_UNSUPPORTED, R_MULTI_SCAN, -1);
  Scan *sc = &f->scan;
  int comp_sel[4], comp_h[4], comp_v[4];
  int mcu_w, mcu_h;
  if (sc->ns == 1) { /* _scan_units codec.py:340-343 */
    Comp *c = &f->comps[sc->comp[0]];
    s->gx = c->bw; s->gy = c->bh;
    comp_sel[0] = sc->comp[0]; comp_h[0] = 1; comp_v[0] = 1;
  } else {
    s->gx = f->mcus_x; s->gy = f->mcus_y;
    for (int i = 0; i < sc->ns; i++) {
      comp_sel[i] = sc->comp[i];
      comp_h[i] = f->comps[sc->comp[i]].h;
      comp_v[i] = f->comps[sc->comp[i]].v;
    }
  }
  if (f->ncomp > 1) { mcu_w = 8 * f->hmax; mcu_h = 8 * f->vmax; }
  else { mcu_w = mcu_h = 8; }
  s->mx0 = x / mcu_w; s->mx1 = (x + w - 1) / mcu_w;
  s->my0 = y / mcu_h; s->my1 = (y + h - 1) / mcu_h;
  s->row_stop = s->my1 + 1;
  for (int i = 0; i < f->ncomp; i++) { /* _alloc_coefs codec.py:401-402 */
    Comp *c = &f->comps[i];
    s->coefs[i] = (int32_t *)calloc((size_t)c->BH * c->BW * 64, sizeof(int32_t));
    s->coef_bw[i] = c->BW;
  }
  int max_restarts = sc->ri ? (s->gx * s->gy) / sc->ri : 0;
  int seglen = sc->end - sc->start;
  s->clean = (uint8_t *)malloc(seglen > 0 ? seglen : 1);
  int max_r = sc->ri > 0 ? max_restarts + 2 : 0;
  int64_t *restarts = (int64_t *)malloc(sizeof(int64_t) * (max_r > 0 ? max_r : 1));
  int nr = 0;
  s->clean_len = orc_destuff(data + sc->start, 0, seglen, s->clean, restarts,
                             max_r, &nr, NULL);
  if (sc->ri == 0 && nr > 0) { free(restarts); FAIL(ST_MALFORMED, R_RST_NO_DRI, sc->start); }
  if (nr > max_restarts + 2) { free(restarts); FAIL(ST_MALFORMED, R_TOO_MANY_RST, sc->start); }
  /* _lut_stack: DC specs of all slots, then AC specs (codec.py:490). */
  int32_t *lut_dc[4] = {0}, *lut_ac[4] = {0};
  int rc = 0;
  for (int i = 0; i < sc->ns && !rc; i++) {
    lut_dc[i] = (int32_t *)malloc(65536 * 4);
    rc = huff_lut(&sc->dc[i], lut_dc[i], e);
  }
  for (int i = 0; i < sc->ns && !rc; i++) {
    lut_ac[i] = (int32_t *)malloc(65536 * 4);
    rc = huff_lut(&sc->ac[i], lut_ac[i], e);
  }
  int st = 0;
  int64_t vpos = 0;
  int cnt = 0;
  if (!rc) {
    st = decode_scan_baseline(s->clean, s->clean_len, restarts, nr, sc->ri,
                              lut_dc, lut_ac, comp_sel, comp_h, comp_v, sc->ns,
                              s->gx, s->row_stop, s->coefs, s->coef_bw, &vpos,
                              &cnt);
  }
  for (int i = 0; i < 4; i++) { free(lut_dc[i]); free(lut_ac[i]); }
  free(restarts);
  if (rc) return -1;
  /* _check_consumed codec.py:323-330 */
  if (st == 1) {
    int64_t off = vpos < seglen ? vpos : seglen;
    FAIL(ST_CORRUPT_HUFFMAN, R_NONE, sc->start + (int)off);
  }
  if (st == 3) FAIL(ST_MISSING_RST, R_NONE, sc->start);
  if (8 * vpos - cnt > 8 * s->clean_len) FAIL(ST_TRUNCATED, R_NONE, sc->end);
  return 0;
}

/* _reconstruct_region + _emit_rgb, codec.py:412-431, 502-509. */
static int reconstruct_emit(DecodeState *s, int x, int y, int w, int h,
                            uint8_t *out, Err *e) {
  Frame *f = &s->f;
  for (int i = 0; i < f->ncomp; i++) {
    Comp *c = &f->comps[i];
    int fh = f->ncomp > 1 ? c->h : 1, fv = f->ncomp > 1 ? c->v : 1;
    int by0 = s->my0 * fv, by1 = (s->my1 + 1) * fv;
    int bx0 = s->mx0 * fh, bx1 = (s->mx1 + 1) * fh;
    if (by1 > c->bh) by1 = c->bh;
    if (bx1 > c->bw) bx1 = c->bw;
    if (!f->has_quant[c->tq & 15] || c->tq > 15) FAIL(ST_QUANT, R_NONE, c->tq);
    s->plane_stride[i] = c->BW * 8;
    s->planes[i] = (uint8_t *)calloc((size_t)c->BH * 8 * c->BW * 8, 1);
    for (int by = by0; by < by1; by++)
      for (int bx = bx0; bx < bx1; bx++)
        orc_idct_block(s->coefs[i] + ((int64_t)by * c->BW + bx) * 64,
                       f->quant[c->tq], s->planes[i] + (int64_t)by * 8 * s->plane_stride[i] + bx * 8,
                       s->plane_stride[i]);
  }
  if (f->ncomp == 1) { /* gray_region_to_rgb decode_kernels.py:579-589 */
    for (int yy = 0; yy < h; yy++)
      for (int xx = 0; xx < w; xx++) {
        uint8_t v = s->planes[0][(int64_t)(y + yy) * s->plane_stride[0] + x + xx];
        uint8_t *o = out + ((int64_t)yy * w + xx) * 3;
        o[0] = o[1] = o[2] = v;
      }
    return 0;
  }
  /* ycc_region_to_rgb decode_kernels.py:537-576 */
  Comp *c0 = &f->comps[0], *c1 = &f->comps[1], *c2 = &f->comps[2];
  for (int yy = 0; yy < h; yy++) {
    int sy = y + yy;
    int ry = sy * c0->v / f->vmax, by_ = sy * c1->v / f->vmax, cy_ = sy * c2->v / f->vmax;
    for (int xx = 0; xx < w; xx++) {
      int sx = x + xx;
      int yv = s->planes[0][(int64_t)ry * s->plane_stride[0] + sx * c0->h / f->hmax];
      int cb = s->planes[1][(int64_t)by_ * s->plane_stride[1] + sx * c1->h / f->hmax] - 128;
      int cr = s->planes[2][(int64_t)cy_ * s->plane_stride[2] + sx * c2->h / f->hmax] - 128;
      int r = yv + ((91881 * cr + 32768) >> 16);
      int g = yv + ((-22554 * cb - 46802 * cr + 32768) >> 16);
      int b = yv + ((116130 * cb + 32768) >> 16);
      uint8_t *o = out + ((int64_t)yy * w + xx) * 3;
      o[0] = clamp255(r); o[1] = clamp255(g); o[2] = clamp255(b);
    }
  }
  return 0;
}

/* Public: decode_crop.  full!=0 decodes the whole image (decode_full,
 * codec.py:434-445; identical to a full-rect crop for baseline streams).
 * stats = {mcus_entropy_decoded, mcus_reconstructed}.  err = {status,
 * reason, offset}.  Returns status. */
ORC_API int orc_decode_crop(const uint8_t *data, int n, int x, int y, int w,
                            int h, int full, uint8_t *out, int32_t *stats,
                            int32_t *err) {
  DecodeState s;
  Err e = {0, 0, -1};
  if (decode_entropy(data, n, x, y, w, h, full, &s, &e)) goto fail;
  if (full) { x = 0; y = 0; w = s.f.width; h = s.f.height; }
  if (reconstruct_emit(&s, x, y, w, h, out, &e)) goto fail;
  if (stats) {
    if (full) {
      int total = s.f.ncomp > 1 ? s.f.mcus_x * s.f.mcus_y
                                : s.f.comps[0].bw * s.f.comps[0].bh;
      stats[0] = total;
      stats[1] = total;
    } else {
      stats[0] = s.row_stop * s.gx;
      stats[1] = (s.my1 - s.my0 + 1) * (s.mx1 - s.mx0 + 1);
    }
  }
  ds_free(&s);
  if (err) { err[0] = 0; err[1] = 0; err[2] = -1; }
  return 0;
fail:
  ds_free(&s);
  if (err) { err[0] = e.status; err[1] = e.reason; err[2] = e.offset; }
  return e.status;
}

/* Frame info: out = {width, height, ncomp, progressive, nscans, ri,
 * hmax, vmax, mcus_x, mcus_y, scan_start, scan_end}. */
ORC_API int orc_jpeg_info(const uint8_t *data, int n, int32_t *out, int32_t *err) {
  Frame f;
  Err e = {0, 0, -1};
  if (parse_stream(data, n, &f, &e)) {
    if (err) { err[0] = e.status; err[1] = e.reason; err[2] = e.offset; }
    return e.status;
  }
  out[0] = f.width; out[1] = f.height; out[2] = f.ncomp; out[3] = f.progressive;
  out[4] = f.nscans; out[5] = f.scan.ri; out[6] = f.hmax; out[7] = f.vmax;
  out[8] = f.mcus_x; out[9] = f.mcus_y; out[10] = f.scan.start; out[11] = f.scan.end;
  return 0;
}

/* Coefficient dump: int32 [BH][BW][64] natural order per component for
 * rows < row_stop of the crop (zeros elsewhere), exactly the arrays
 * decode_crop holds before reconstruction (codec.py:483-500).  `out` must
 * hold sum_c BH_c*BW_c*64 int32; dims = {BH0,BW0,BH1,BW1,BH2,BW2}. */
ORC_API int orc_dump_coefs(const uint8_t *data, int n, int x, int y, int w,
                           int h, int32_t *out, int64_t out_cap, int32_t *dims,
                           int32_t *err) {
  DecodeState s;
  Err e = {0, 0, -1};
  if (decode_entropy(data, n, x, y, w, h, 0, &s, &e)) {
    ds_free(&s);
    if (err) { err[0] = e.status; err[1] = e.reason; err[2] = e.offset; }
    return e.status;
  }
  int64_t off = 0;
  for (int i = 0; i < 3; i++) { dims[2 * i] = 0; dims[2 * i + 1] = 0; }
  for (int i = 0; i < s.f.ncomp; i++) {
    Comp *c = &s.f.comps[i];
    int64_t cnt = (int64_t)c->BH * c->BW * 64;
    if (off + cnt <= out_cap) memcpy(out + off, s.coefs[i], cnt * 4);
    off += cnt;
    dims[2 * i] = c->BH;
    dims[2 * i + 1] = c->BW;
  }
  ds_free(&s);
  if (err) { err[0] = 0; err[1] = 0; err[2] = -1; }
  return off <= out_cap ? 0 : -1;
}

/* ------------------------------------------------------------------ */
/* imgops.py:24-60 _resize_bilinear_kernel (float64, no FMA)           */
/* ------------------------------------------------------------------ */
ORC_API void orc_resize_bilinear(const uint8_t *src, int ih, int iw,
                                 uint8_t *out, int oh, int ow) {
  double sy = (double)ih / (double)oh, sx = (double)iw / (double)ow;
  for (int oy = 0; oy < oh; oy++) {
    double fy = ((double)oy + 0.5) * sy - 0.5;
    if (fy < 0.0) fy = 0.0;
    int y0 = (int)fy;
    if (y0 > ih - 1) y0 = ih - 1;
    int y1 = y0 + 1;
    if (y1 > ih - 1) y1 = ih - 1;
    double wy = fy - (double)y0;
    for (int ox = 0; ox < ow; ox++) {
      double fx = ((double)ox + 0.5) * sx - 0.5;
      if (fx < 0.0) fx = 0.0;
      int x0 = (int)fx;
      if (x0 > iw - 1) x0 = iw - 1;
      int x1 = x0 + 1;
      if (x1 > iw - 1) x1 = iw - 1;
      double wx = fx - (double)x0;
      for (int c = 0; c < 3; c++) {
        double s00 = src[((int64_t)y0 * iw + x0) * 3 + c];
        double s01 = src[((int64_t)y0 * iw + x1) * 3 + c];
        double s10 = src[((int64_t)y1 * iw + x0) * 3 + c];
        double s11 = src[((int64_t)y1 * iw + x1) * 3 + c];
        double top = (1.0 - wx) * s00 + wx * s01;
        double bot = (1.0 - wx) * s10 + wx * s11;
        int v = (int)((1.0 - wy) * top + wy * bot + 0.5);
        if (v > 255) v = 255;
        out[((int64_t)oy * ow + ox) * 3 + c] = (uint8_t)v;
      }
    }
  }
}

static const float IMAGENET_MEAN[3] = {0.485f, 0.456f, 0.406f}; /* imgops.py:16-17 */
static const float IMAGENET_STD[3] = {0.229f, 0.224f, 0.225f};

/* imgops.py:231-248 normalize: uint8 HWC -> float32 CHW. */
ORC_API void orc_normalize(const uint8_t *img, int h, int w, float *out) {
  volatile float one = 1.0f, d255 = 255.0f;
  float inv255 = one / d255;
  for (int c = 0; c < 3; c++) {
    float m = IMAGENET_MEAN[c], s = IMAGENET_STD[c];
    for (int y = 0; y < h; y++)
      for (int x = 0; x < w; x++) {
        float v = (float)img[((int64_t)y * w + x) * 3 + c];
        out[((int64_t)c * h + y) * w + x] = (v * inv255 - m) / s;
      }
  }
}

/* ------------------------------------------------------------------ */
/* 3-Aug / 3-Aug+ pixel ops (imgops.py:75-227) on uint8 HWC images      */
/* ------------------------------------------------------------------ */
static inline int luma601(int r, int g, int b) { /* imgops.py:78-81 */
  return (19595 * r + 38470 * g + 7471 * b + 32768) >> 16;
}

/* imgops.py:75-91 grayscale. */
ORC_API void orc_grayscale(const uint8_t *img, int h, int w, uint8_t *out) {
  for (int64_t p = 0; p < (int64_t)h * w; p++) {
    int v = luma601(img[3 * p], img[3 * p + 1], img[3 * p + 2]);
    out[3 * p] = out[3 * p + 1] = out[3 * p + 2] = (uint8_t)v;
  }
}

/* imgops.py:94-108 solarize (>= threshold inverts). */
ORC_API void orc_solarize(const uint8_t *img, int h, int w, int threshold, uint8_t *out) {
  for (int64_t i = 0; i < (int64_t)h * w * 3; i++)
    out[i] = img[i] >= threshold ? (uint8_t)(255 - img[i]) : img[i];
}

/* imgops.py:111-119 _reflect (Python modulo). */
static int reflect_idx(int i, int n) {
  if (n == 1) return 0;
  int period = 2 * n - 2;
  i = ((i % period) + period) % period;
  if (i >= n) i = period - i;
  return i;
}

/* imgops.py:122-163 gaussian_blur given its normalised weights (ntaps =
 * 2*radius+1; the weights are numpy's, computed by the caller exactly as
 * imgops.py:157-160 does).  Horizontal float64 pass into tmp, vertical pass
 * with int(acc + 0.5) capped at 255; sequential accumulation, no FMA. */
ORC_API void orc_gaussian_blur(const uint8_t *img, int h, int w, const double *wts, int ntaps,
                               uint8_t *out) {
  int r = (ntaps - 1) / 2;
  double *tmp = (double *)malloc(sizeof(double) * (size_t)h * w * 3);
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++)
      for (int c = 0; c < 3; c++) {
        double acc = 0.0;
        for (int k = 0; k < ntaps; k++)
          acc += wts[k] * (double)img[((int64_t)y * w + reflect_idx(x + k - r, w)) * 3 + c];
        tmp[((int64_t)y * w + x) * 3 + c] = acc;
      }
  for (int y = 0; y < h; y++)
    for (int x = 0; x < w; x++)
      for (int c = 0; c < 3; c++) {
        double acc = 0.0;
        for (int k = 0; k < ntaps; k++)
          acc += wts[k] * tmp[((int64_t)reflect_idx(y + k - r, h) * w + x) * 3 + c];
        int v = (int)(acc + 0.5);
        if (v > 255) v = 255;
        out[((int64_t)y * w + x) * 3 + c] = (uint8_t)v;
      }
  free(tmp);
}

static inline uint8_t blend1(double factor, double v, double target) { /* imgops.py:170-178 */
  int q = (int)floor(factor * v + (1.0 - factor) * target + 0.5);
  return (uint8_t)(q < 0 ? 0 : q > 255 ? 255 : q);
}

/* imgops.py:199-210 _luma_mean. */
ORC_API double orc_luma_mean(const uint8_t *img, int h, int w) {
  double acc = 0.0;
  for (int64_t p = 0; p < (int64_t)h * w; p++)
    acc += luma601(img[3 * p], img[3 * p + 1], img[3 * p + 2]);
  return acc / (double)((int64_t)h * w);
}

/* imgops.py:213-227 adjust_brightness (kind 0), adjust_contrast (1),
 * adjust_saturation (2). */
ORC_API void orc_adjust(const uint8_t *img, int h, int w, int kind, double factor, uint8_t *out) {
  int64_t np_ = (int64_t)h * w;
  double target = kind == 1 ? orc_luma_mean(img, h, w) : 0.0;
  for (int64_t p = 0; p < np_; p++) {
    double g = kind == 2 ? (double)luma601(img[3 * p], img[3 * p + 1], img[3 * p + 2]) : target;
    for (int c = 0; c < 3; c++) out[3 * p + c] = blend1(factor, (double)img[3 * p + c], g);
  }
}

/* Per-sample 3-Aug draw results (pipeline.py:88-101); weights come from
 * numpy (see oracle.py blur_weights). */
typedef struct {
  int32_t op;     /* -1 none, 0 grayscale, 1 solarize, 2 blur */
  int32_t ntaps;  /* blur: 2*radius+1 */
  int32_t jitter; /* 1: brightness, contrast, saturation */
  int32_t pad;
  double factors[3];
  double wts[32];
} OrcAug;

/* apply_aug after the flip (pipeline.py:88-101), in place on img. */
ORC_API void orc_apply_aug_ops(uint8_t *img, int h, int w, const OrcAug *a) {
  size_t nb = (size_t)h * w * 3;
  uint8_t *t = (uint8_t *)malloc(nb);
  if (a->op == 0) orc_grayscale(img, h, w, t);
  else if (a->op == 1) orc_solarize(img, h, w, 128, t); /* SOLARIZE_THRESHOLD imgops.py:19 */
  else if (a->op == 2) orc_gaussian_blur(img, h, w, a->wts, a->ntaps, t);
  if (a->op >= 0) memcpy(img, t, nb);
  if (a->jitter) {
    for (int kind = 0; kind < 3; kind++) {
      orc_adjust(img, h, w, kind, a->factors[kind], t);
      memcpy(img, t, nb);
    }
  }
  free(t);
}

/* ------------------------------------------------------------------ */
/* Loader sample (pipeline.py:219-235) and a threaded batch driver      */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t seed, epoch;
  int res;
  double scale_lo, scale_hi, ratio_lo, ratio_hi;
  int mask_grid;     /* 0 = no mask */
  int mask_k;
} OrcLoaderCfg;

/* Fill one sample.  rect_out = {x,y,w,h,flip}.  pixels [3,res,res] f32,
 * u8 [res,res,3] (may be NULL), mask [k] (may be NULL). Returns status;
 * err = {status, reason, offset}. */
ORC_API int orc_fill_sample(const uint8_t *payload, int len, uint32_t crc,
                            int img_w, int img_h, int64_t index,
                            const OrcLoaderCfg *cfg, float *pixels,
                            uint8_t *u8, int32_t *mask, int32_t *rect_out,
                            const OrcAug *aug, int32_t *err) {
  if (orc_crc32(payload, len) != crc) {
    if (err) { err[0] = ST_CRC; err[1] = 0; err[2] = -1; }
    return ST_CRC;
  }
  uint64_t st = orc_rng_init(cfg->seed, cfg->epoch, (uint64_t)index, 0);
  int32_t r[4];
  orc_sample_rrc(&st, img_w, img_h, cfg->scale_lo, cfg->scale_hi,
                 cfg->ratio_lo, cfg->ratio_hi, 10, r);
  uint8_t *region = (uint8_t *)malloc((size_t)r[2] * r[3] * 3);
  int32_t e3[3];
  int rc = orc_decode_crop(payload, len, r[0], r[1], r[2], r[3], 0, region, NULL, e3);
  if (rc) {
    free(region);
    if (err) memcpy(err, e3, sizeof(e3));
    return rc;
  }
  int res = cfg->res;
  uint8_t *img = (uint8_t *)malloc((size_t)res * res * 3);
  orc_resize_bilinear(region, r[3], r[2], img, res, res);
  free(region);
  int flip = orc_rng_random(&st) < 0.5; /* pipeline.py:86-87 */
  if (flip) {
    for (int yy = 0; yy < res; yy++) {
      uint8_t *row = img + (int64_t)yy * res * 3;
      for (int a = 0, b = res - 1; a < b; a++, b--)
        for (int c = 0; c < 3; c++) {
          uint8_t t = row[a * 3 + c];
          row[a * 3 + c] = row[b * 3 + c];
          row[b * 3 + c] = t;
        }
    }
  }
  if (aug) orc_apply_aug_ops(img, res, res, aug); /* pipeline.py:88-101 */
  orc_normalize(img, res, res, pixels);
  if (u8) memcpy(u8, img, (size_t)res * res * 3);
  free(img);
  if (mask && cfg->mask_grid > 0) {
    uint64_t ms = orc_rng_init(cfg->seed, cfg->epoch, (uint64_t)index, 1);
    orc_sample_mask(&ms, cfg->mask_grid * cfg->mask_grid, cfg->mask_k, mask);
  }
  if (rect_out) { memcpy(rect_out, r, sizeof(r)); rect_out[4] = flip; }
  if (err) { err[0] = 0; err[1] = 0; err[2] = -1; }
  return 0;
}

typedef struct {
  const uint8_t *base;
  const uint64_t *offsets;
  const uint32_t *lengths, *crcs;
  const uint16_t *widths, *heights;
  const int64_t *indices;
  int n;
  const OrcLoaderCfg *cfg;
  float *pixels;
  uint8_t *u8;
  int32_t *mask;
  const OrcAug *aug; /* per batch position, or NULL (simple) */
  int32_t *status;
  volatile int next;
} BatchJob;

static void *batch_worker(void *arg) {
  BatchJob *j = (BatchJob *)arg;
  int res = j->cfg->res, k = j->cfg->mask_k;
  for (;;) {
    int i = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (i >= j->n) break;
    int64_t idx = j->indices[i];
    int32_t e3[3];
    j->status[i] = orc_fill_sample(
        j->base + j->offsets[idx], (int)j->lengths[idx], j->crcs[idx],
        j->widths[idx], j->heights[idx], idx, j->cfg,
        j->pixels + (int64_t)i * 3 * res * res,
        j->u8 ? j->u8 + (int64_t)i * res * res * 3 : NULL,
        j->mask ? j->mask + (int64_t)i * k : NULL, NULL, j->aug ? j->aug + i : NULL, e3);
  }
  return NULL;
}

/* One loader batch over `n` dataset indices with `nthreads` threads
 * (Loader._fill_sample over a pool, pipeline.py:256-266).  Record arrays
 * are indexed by dataset index (container.py:46-51). */
ORC_API int orc_loader_batch(const uint8_t *base, const uint64_t *offsets,
                             const uint32_t *lengths, const uint32_t *crcs,
                             const uint16_t *widths, const uint16_t *heights,
                             const int64_t *indices, int n,
                             const OrcLoaderCfg *cfg, float *pixels,
                             uint8_t *u8, int32_t *mask, const OrcAug *aug,
                             int32_t *status, int nthreads) {
  BatchJob j = {base, offsets, lengths, crcs, widths, heights, indices, n,
                cfg, pixels, u8, mask, aug, status, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) {
    batch_worker(&j);
  } else {
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, batch_worker, &j);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    free(th);
  }
  int bad = 0;
  for (int i = 0; i < n; i++) bad |= status[i] != 0;
  return bad;
}
