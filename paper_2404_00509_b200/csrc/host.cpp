// Host-side C++ of libessl: sampling (rng.py, pipeline.py:51-87), epoch
// permutation, and the dataset builder pieces (codec.py:574-632 encoder,
// synthetic images) used to make fixtures and benchmark inputs.
//
// Compiled with -ffp-contract=off: the reference evaluates every float64
// expression with one rounding per operation (CPython semantics), and the
// RRC uses glibc log/exp/sqrt exactly as CPython's math module does.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "essl.h"

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

inline double rnd(uint64_t *st) {
  *st += kGamma;
  return (double)(mix64(*st) >> 11) * 0x1p-53;
}

inline int64_t randint(uint64_t *st, int64_t n) {
  const int64_t v = (int64_t)(rnd(st) * (double)n);
  return v >= n ? n - 1 : v;
}

}  // namespace

extern "C" {

uint64_t essl_rng_init(uint64_t seed, uint64_t epoch, uint64_t index, uint64_t domain) {
  uint64_t h = mix64(seed);
  h = mix64(h ^ (epoch * kGamma));
  h = mix64(h ^ (index * kGamma));
  h = mix64(h ^ (domain * kGamma));
  return h;
}

uint64_t essl_rng_next(uint64_t *state) {
  *state += kGamma;
  return mix64(*state);
}

double essl_rng_random(uint64_t *state) { return rnd(state); }

int64_t essl_rng_randint(uint64_t *state, int64_t n) { return randint(state, n); }

// rng.py:80-87
int essl_epoch_permutation(uint64_t seed, uint64_t epoch, int64_t n, int64_t *out) {
  if (n < 0 || (n > 0 && !out)) return ESSL_E_ARG;
  uint64_t st = essl_rng_init(seed, epoch, 0, 3);
  for (int64_t i = 0; i < n; i++) out[i] = i;
  for (int64_t i = n - 1; i > 0; i--) {
    const int64_t j = randint(&st, i + 1);
    const int64_t t = out[i];
    out[i] = out[j];
    out[j] = t;
  }
  return ESSL_OK;
}

namespace {
// pipeline.py:51-75 with log(ratio) precomputed (the batch path computes the
// two logs once per batch; same values)
int sample_rrc_logs(uint64_t *st, int64_t src_w, int64_t src_h, double scale_lo, double scale_hi,
                    double ratio_lo, double ratio_hi, double log_lo, double log_hi, int max_attempts,
                    int32_t *xywh) {
  const double area = (double)(src_w * src_h);
  for (int a = 0; a < max_attempts; a++) {
    const double target = area * (scale_lo + (scale_hi - scale_lo) * rnd(st));
    const double aspect = std::exp(log_lo + (log_hi - log_lo) * rnd(st));
    const int64_t w = (int64_t)(std::sqrt(target * aspect) + 0.5);
    const int64_t h = (int64_t)(std::sqrt(target / aspect) + 0.5);
    if (0 < w && w <= src_w && 0 < h && h <= src_h) {
      const int64_t x = randint(st, src_w - w + 1);
      const int64_t y = randint(st, src_h - h + 1);
      xywh[0] = (int32_t)x; xywh[1] = (int32_t)y;
      xywh[2] = (int32_t)w; xywh[3] = (int32_t)h;
      return ESSL_OK;
    }
  }
  const double in_ratio = (double)src_w / (double)src_h;
  int64_t w = src_w, h = src_h;
  if (in_ratio < ratio_lo) {
    w = src_w;
    int64_t t = (int64_t)((double)w / ratio_lo + 0.5);
    h = std::min<int64_t>(src_h, std::max<int64_t>(1, t));
  } else if (in_ratio > ratio_hi) {
    h = src_h;
    int64_t t = (int64_t)((double)h * ratio_hi + 0.5);
    w = std::min<int64_t>(src_w, std::max<int64_t>(1, t));
  }
  xywh[0] = (int32_t)((src_w - w) / 2); xywh[1] = (int32_t)((src_h - h) / 2);
  xywh[2] = (int32_t)w; xywh[3] = (int32_t)h;
  return ESSL_OK;
}
}  // namespace

// pipeline.py:51-75
int essl_sample_rrc(uint64_t *st, int64_t src_w, int64_t src_h, double scale_lo, double scale_hi,
                    double ratio_lo, double ratio_hi, int max_attempts, int32_t *xywh) {
  if (!st || !xywh || src_w < 1 || src_h < 1) return ESSL_E_ARG;
  return sample_rrc_logs(st, src_w, src_h, scale_lo, scale_hi, ratio_lo, ratio_hi, std::log(ratio_lo),
                         std::log(ratio_hi), max_attempts, xywh);
}

// Loader._fill_sample draws (pipeline.py:221-222, 86-87) for a batch.
int essl_rrc_batch(uint64_t seed, uint64_t epoch, const int64_t *indices, int n,
                   const uint16_t *widths, const uint16_t *heights, double scale_lo,
                   double scale_hi, double ratio_lo, double ratio_hi, essl_sample *samples) {
  if (n < 0 || (n > 0 && (!indices || !widths || !heights || !samples))) return ESSL_E_ARG;
  const double log_lo = std::log(ratio_lo), log_hi = std::log(ratio_hi);
  for (int i = 0; i < n; i++) {
    const int64_t idx = indices[i];
    uint64_t st = essl_rng_init(seed, epoch, (uint64_t)idx, 0);
    int32_t r[4];
    if (widths[idx] < 1 || heights[idx] < 1) return ESSL_E_ARG;
    sample_rrc_logs(&st, widths[idx], heights[idx], scale_lo, scale_hi, ratio_lo, ratio_hi, log_lo, log_hi,
                    10, r);
    samples[i].x = r[0]; samples[i].y = r[1]; samples[i].w = r[2]; samples[i].h = r[3];
    samples[i].flip = rnd(&st) < 0.5 ? 1 : 0;
  }
  return ESSL_OK;
}

// apply_aug's draws (pipeline.py:85-101), after the RRC draws on the same
// pipeline stream.  BLUR_SIGMA_RANGE / JITTER_STRENGTH: imgops.py:20-21.
int essl_aug_draw(uint64_t *st, int level, int32_t *flip, essl_aug *aug) {
  if (!st || level < ESSL_AUG_SIMPLE || level > ESSL_AUG_3AUG_PLUS) return ESSL_E_ARG;
  const int32_t f = rnd(st) < 0.5 ? 1 : 0;
  if (flip) *flip = f;
  if (!aug) return level == ESSL_AUG_SIMPLE ? ESSL_OK : ESSL_E_ARG;
  std::memset(aug, 0, sizeof(*aug));
  aug->op = ESSL_AUG_OP_NONE;
  aug->threshold = 128;  // SOLARIZE_THRESHOLD, imgops.py:19
  if (level != ESSL_AUG_SIMPLE) {
    aug->op = (int32_t)randint(st, 3);
    if (aug->op == ESSL_AUG_OP_BLUR) {
      aug->sigma = 0.1 + (2.0 - 0.1) * rnd(st);                 // rng.uniform(0.1, 2.0)
      aug->radius = std::max(1, (int)std::ceil(3.0 * aug->sigma));  // imgops.py:156
    }
  }
  if (level == ESSL_AUG_3AUG_PLUS) {
    const double s = 0.3, lo = 1.0 - s, hi = 1.0 + s;
    aug->jitter = 1;
    for (int k = 0; k < 3; k++) aug->factors[k] = lo + (hi - lo) * rnd(st);
  }
  return ESSL_OK;
}

int essl_aug_batch(uint64_t seed, uint64_t epoch, const int64_t *indices, int n,
                   const uint16_t *widths, const uint16_t *heights, double scale_lo,
                   double scale_hi, double ratio_lo, double ratio_hi, int level,
                   essl_sample *samples, essl_aug *aug) {
  if (n < 0 || (n > 0 && (!indices || !widths || !heights || !samples)) ||
      (level != ESSL_AUG_SIMPLE && n > 0 && !aug))
    return ESSL_E_ARG;
  for (int i = 0; i < n; i++) {
    const int64_t idx = indices[i];
    uint64_t st = essl_rng_init(seed, epoch, (uint64_t)idx, 0);
    int32_t r[4];
    int rc = essl_sample_rrc(&st, widths[idx], heights[idx], scale_lo, scale_hi, ratio_lo,
                             ratio_hi, 10, r);
    if (rc) return rc;
    samples[i].x = r[0]; samples[i].y = r[1]; samples[i].w = r[2]; samples[i].h = r[3];
    rc = essl_aug_draw(&st, level, &samples[i].flip, aug ? aug + i : nullptr);
    if (rc) return rc;
  }
  return ESSL_OK;
}

int essl_mask_count(int tokens, double ratio) {  // masking.py:43-45
  return (int)std::floor(ratio * (double)tokens + 0.5);
}

// ---------------------------------------------------------------------------
// Encoder: restatement of encode_jpeg (codec.py:574-632) and its kernels
// (jpeg/encode_kernels.py:16-202) -- baseline, 4:2:0, Annex-K tables,
// float64 FDCT with the pinned basis (tables.py:116-143).

namespace {

const int kZZ[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                     12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                     35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                     58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

const int kQLuma[64] = {16, 11, 10, 16, 24,  40,  51,  61,  12, 12, 14, 19, 26,  58,  60,  55,
                        14, 13, 16, 24, 40,  57,  69,  56,  14, 17, 22, 29, 51,  87,  80,  62,
                        18, 22, 37, 56, 68,  109, 103, 77,  24, 35, 55, 64, 81,  104, 113, 92,
                        49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99};
const int kQChroma[64] = {17, 18, 24, 47, 99, 99, 99, 99, 18, 21, 26, 66, 99, 99, 99, 99,
                          24, 26, 56, 99, 99, 99, 99, 99, 47, 66, 99, 99, 99, 99, 99, 99,
                          99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99,
                          99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99, 99};

// Annex K.3 tables: code counts per length and symbols.
const uint8_t kDcLumaBits[16] = {0, 1, 5, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0, 0, 0};
const uint8_t kDcLumaVals[12] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};
const uint8_t kDcChromaBits[16] = {0, 3, 1, 1, 1, 1, 1, 1, 1, 1, 1, 0, 0, 0, 0, 0};
const uint8_t kDcChromaVals[12] = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11};
const uint8_t kAcLumaBits[16] = {0, 2, 1, 3, 3, 2, 4, 3, 5, 5, 4, 4, 0, 0, 1, 0x7d};
const uint8_t kAcLumaVals[162] = {
    0x01, 0x02, 0x03, 0x00, 0x04, 0x11, 0x05, 0x12, 0x21, 0x31, 0x41, 0x06, 0x13, 0x51, 0x61,
    0x07, 0x22, 0x71, 0x14, 0x32, 0x81, 0x91, 0xa1, 0x08, 0x23, 0x42, 0xb1, 0xc1, 0x15, 0x52,
    0xd1, 0xf0, 0x24, 0x33, 0x62, 0x72, 0x82, 0x09, 0x0a, 0x16, 0x17, 0x18, 0x19, 0x1a, 0x25,
    0x26, 0x27, 0x28, 0x29, 0x2a, 0x34, 0x35, 0x36, 0x37, 0x38, 0x39, 0x3a, 0x43, 0x44, 0x45,
    0x46, 0x47, 0x48, 0x49, 0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58, 0x59, 0x5a, 0x63, 0x64,
    0x65, 0x66, 0x67, 0x68, 0x69, 0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a, 0x83,
    0x84, 0x85, 0x86, 0x87, 0x88, 0x89, 0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97, 0x98, 0x99,
    0x9a, 0xa2, 0xa3, 0xa4, 0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4, 0xb5, 0xb6,
    0xb7, 0xb8, 0xb9, 0xba, 0xc2, 0xc3, 0xc4, 0xc5, 0xc6, 0xc7, 0xc8, 0xc9, 0xca, 0xd2, 0xd3,
    0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda, 0xe1, 0xe2, 0xe3, 0xe4, 0xe5, 0xe6, 0xe7, 0xe8,
    0xe9, 0xea, 0xf1, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8, 0xf9, 0xfa};
const uint8_t kAcChromaBits[16] = {0, 2, 1, 2, 4, 4, 3, 4, 7, 5, 4, 4, 0, 1, 2, 0x77};
const uint8_t kAcChromaVals[162] = {
    0x00, 0x01, 0x02, 0x03, 0x11, 0x04, 0x05, 0x21, 0x31, 0x06, 0x12, 0x41, 0x51, 0x07, 0x61,
    0x71, 0x13, 0x22, 0x32, 0x81, 0x08, 0x14, 0x42, 0x91, 0xa1, 0xb1, 0xc1, 0x09, 0x23, 0x33,
    0x52, 0xf0, 0x15, 0x62, 0x72, 0xd1, 0x0a, 0x16, 0x24, 0x34, 0xe1, 0x25, 0xf1, 0x17, 0x18,
    0x19, 0x1a, 0x26, 0x27, 0x28, 0x29, 0x2a, 0x35, 0x36, 0x37, 0x38, 0x39, 0x3a, 0x43, 0x44,
    0x45, 0x46, 0x47, 0x48, 0x49, 0x4a, 0x53, 0x54, 0x55, 0x56, 0x57, 0x58, 0x59, 0x5a, 0x63,
    0x64, 0x65, 0x66, 0x67, 0x68, 0x69, 0x6a, 0x73, 0x74, 0x75, 0x76, 0x77, 0x78, 0x79, 0x7a,
    0x82, 0x83, 0x84, 0x85, 0x86, 0x87, 0x88, 0x89, 0x8a, 0x92, 0x93, 0x94, 0x95, 0x96, 0x97,
    0x98, 0x99, 0x9a, 0xa2, 0xa3, 0xa4, 0xa5, 0xa6, 0xa7, 0xa8, 0xa9, 0xaa, 0xb2, 0xb3, 0xb4,
    0xb5, 0xb6, 0xb7, 0xb8, 0xb9, 0xba, 0xc2, 0xc3, 0xc4, 0xc5, 0xc6, 0xc7, 0xc8, 0xc9, 0xca,
    0xd2, 0xd3, 0xd4, 0xd5, 0xd6, 0xd7, 0xd8, 0xd9, 0xda, 0xe2, 0xe3, 0xe4, 0xe5, 0xe6, 0xe7,
    0xe8, 0xe9, 0xea, 0xf2, 0xf3, 0xf4, 0xf5, 0xf6, 0xf7, 0xf8, 0xf9, 0xfa};

struct EncTable {
  uint32_t code[256];
  uint8_t size[256];
  void build(const uint8_t *bits, const uint8_t *vals) {  // codec.py:526-539
    std::memset(code, 0, sizeof(code));
    std::memset(size, 0, sizeof(size));
    uint32_t c = 0;
    int vi = 0;
    for (int len = 1; len <= 16; len++) {
      for (int i = 0; i < bits[len - 1]; i++) {
        code[vals[vi]] = c;
        size[vals[vi]] = (uint8_t)len;
        c++;
        vi++;
      }
      c <<= 1;
    }
  }
};

struct EncTables {
  EncTable dcl, acl, dcc, acc;
  double basis[8][8];
  EncTables() {
    dcl.build(kDcLumaBits, kDcLumaVals);
    acl.build(kAcLumaBits, kAcLumaVals);
    dcc.build(kDcChromaBits, kDcChromaVals);
    acc.build(kAcChromaBits, kAcChromaVals);
    // tables.py:116-143: cos(k*pi/16) pinned as hex literals
    const double cos16[8] = {1.0, 0x1.f6297cff75cb0p-1, 0x1.d906bcf328d46p-1, 0x1.a9b66290ea1a3p-1,
                             0x1.6a09e667f3bcdp-1, 0x1.1c73b39ae68c9p-1, 0x1.87de2a6aea964p-2,
                             0x1.8f8b83c69a60dp-3};
    const double isqrt2 = 0x1.6a09e667f3bccp-1;
    for (int u = 0; u < 8; u++) {
      const double cu = u == 0 ? isqrt2 : 1.0;
      for (int x = 0; x < 8; x++) {
        int k = ((2 * x + 1) * u) % 32;
        double sign = 1.0;
        if (k > 16) k = 32 - k;
        if (k > 8) { k = 16 - k; sign = -1.0; }
        const double base = k == 8 ? 0.0 : cos16[k];
        basis[u][x] = 0.5 * cu * sign * base;
      }
    }
  }
};

const EncTables &enc_tables() {
  static const EncTables t;
  return t;
}

struct BitWriter {  // encode_kernels.py:93-107 _put_bits (with 0xFF stuffing)
  uint8_t *out;
  int64_t cap, pos = 0;
  uint64_t buf = 0;
  int cnt = 0;
  bool overflow = false;
  void put(uint32_t code, int size) {
    buf = (buf << size) | code;
    cnt += size;
    while (cnt >= 8) {
      const uint8_t b = (uint8_t)((buf >> (cnt - 8)) & 0xFF);
      emit(b);
      if (b == 0xFF) emit(0);
      cnt -= 8;
    }
    buf &= (cnt ? ((1ull << cnt) - 1) : 0);
  }
  void emit(uint8_t b) {
    if (pos < cap) out[pos] = b; else overflow = true;
    pos++;
  }
};

inline int nbits(int v) {  // encode_kernels.py:110-116
  int n = 0;
  while (v) { v >>= 1; n++; }
  return n;
}

// encode_kernels.py:119-151
int encode_block(const int32_t *blk, int pred, const EncTable &dc, const EncTable &ac, BitWriter &bw) {
  const int d = blk[0];
  const int diff = d - pred;
  const int mag = diff >= 0 ? diff : -diff;
  const int s = nbits(mag);
  bw.put(dc.code[s], dc.size[s]);
  if (s > 0) bw.put((uint32_t)(diff >= 0 ? diff : diff + (1 << s) - 1) & ((1u << s) - 1), s);
  int run = 0;
  for (int k = 1; k < 64; k++) {
    const int v = blk[kZZ[k]];
    if (v == 0) { run++; continue; }
    while (run > 15) { bw.put(ac.code[0xF0], ac.size[0xF0]); run -= 16; }
    const int m = v >= 0 ? v : -v;
    const int sz = nbits(m);
    const int rs = (run << 4) | sz;
    bw.put(ac.code[rs & 0xFF], ac.size[rs & 0xFF]);
    bw.put((uint32_t)(v >= 0 ? v : v + (1 << sz) - 1) & ((1u << sz) - 1), sz);
    run = 0;
  }
  if (run > 0) bw.put(ac.code[0], ac.size[0]);
  return d;
}

// encode_kernels.py:62-90: float64 FDCT + round-half-away quantisation.
void fdct_quant(const uint8_t *plane, int pitch, int bx, int by, const int *q, const double (*B)[8],
                int32_t *out) {
  double blk[8][8], tmp[8][8];
  for (int i = 0; i < 8; i++)
    for (int j = 0; j < 8; j++) blk[i][j] = (double)plane[(by * 8 + i) * pitch + bx * 8 + j] - 128.0;
  for (int u = 0; u < 8; u++)
    for (int j = 0; j < 8; j++) {
      double acc = 0.0;
      for (int x = 0; x < 8; x++) acc += B[u][x] * blk[x][j];
      tmp[u][j] = acc;
    }
  for (int u = 0; u < 8; u++)
    for (int v = 0; v < 8; v++) {
      double acc = 0.0;
      for (int j = 0; j < 8; j++) acc += tmp[u][j] * B[v][j];
      const double qq = (double)q[u * 8 + v];
      out[u * 8 + v] = acc >= 0.0 ? (int32_t)(acc / qq + 0.5) : -(int32_t)(-acc / qq + 0.5);
    }
}

void put_u16(std::vector<uint8_t> &v, int x) {
  v.push_back((uint8_t)(x >> 8));
  v.push_back((uint8_t)(x & 0xFF));
}

}  // namespace

int64_t essl_encode_jpeg(const uint8_t *rgb, int h, int w, int quality, int restart_interval,
                         uint8_t *out, int64_t out_cap) {
  if (!rgb || h < 1 || w < 1 || quality < 1 || quality > 100 || h > 65535 || w > 65535)
    return ESSL_E_ARG;
  const EncTables &T = enc_tables();
  // tables.py:95-111 quality scaling
  const int scale = quality < 50 ? 5000 / quality : 200 - quality * 2;
  int ql[64], qc[64];
  for (int i = 0; i < 64; i++) {
    ql[i] = std::min(255, std::max(1, (kQLuma[i] * scale + 50) / 100));
    qc[i] = std::min(255, std::max(1, (kQChroma[i] * scale + 50) / 100));
  }
  const int mx = (w + 15) / 16, my = (h + 15) / 16;
  const int yp = mx * 16, cp = mx * 8;
  std::vector<uint8_t> Y((size_t)my * 16 * yp), cbf((size_t)h * w), crf((size_t)h * w);
  std::vector<uint8_t> Cb((size_t)my * 8 * cp), Cr((size_t)my * 8 * cp);
  // encode_kernels.py:16-33
  for (int py = 0; py < my * 16; py++) {
    const int sy = py < h ? py : h - 1;
    for (int px = 0; px < yp; px++) {
      const int sx = px < w ? px : w - 1;
      const uint8_t *p = rgb + ((size_t)sy * w + sx) * 3;
      const int r = p[0], g = p[1], b = p[2];
      Y[(size_t)py * yp + px] = (uint8_t)((19595 * r + 38470 * g + 7471 * b + 32768) >> 16);
      if (py < h && px < w) {
        cbf[(size_t)py * w + px] = (uint8_t)((-11059 * r - 21709 * g + 32768 * b + 8421375) >> 16);
        crf[(size_t)py * w + px] = (uint8_t)((32768 * r - 27439 * g - 5329 * b + 8421375) >> 16);
      }
    }
  }
  // encode_kernels.py:36-59
  for (int cy = 0; cy < my * 8; cy++) {
    const int y0 = std::min(2 * cy, h - 1), y1 = std::min(2 * cy + 1, h - 1);
    for (int cx = 0; cx < cp; cx++) {
      const int x0 = std::min(2 * cx, w - 1), x1 = std::min(2 * cx + 1, w - 1);
      const int s1 = cbf[(size_t)y0 * w + x0] + cbf[(size_t)y0 * w + x1] + cbf[(size_t)y1 * w + x0] +
                     cbf[(size_t)y1 * w + x1];
      const int s2 = crf[(size_t)y0 * w + x0] + crf[(size_t)y0 * w + x1] + crf[(size_t)y1 * w + x0] +
                     crf[(size_t)y1 * w + x1];
      Cb[(size_t)cy * cp + cx] = (uint8_t)((s1 + 2) >> 2);
      Cr[(size_t)cy * cp + cx] = (uint8_t)((s2 + 2) >> 2);
    }
  }
  // header (codec.py:619-631)
  std::vector<uint8_t> hd = {0xFF, 0xD8, 0xFF, 0xE0, 0, 16, 'J', 'F', 'I', 'F', 0, 1, 1, 0, 0, 1, 0, 1, 0, 0};
  hd.push_back(0xFF); hd.push_back(0xDB); put_u16(hd, 2 + 2 * 65);
  hd.push_back(0);
  for (int k = 0; k < 64; k++) hd.push_back((uint8_t)ql[kZZ[k]]);
  hd.push_back(1);
  for (int k = 0; k < 64; k++) hd.push_back((uint8_t)qc[kZZ[k]]);
  hd.push_back(0xFF); hd.push_back(0xC0); put_u16(hd, 17); hd.push_back(8);
  put_u16(hd, h); put_u16(hd, w); hd.push_back(3);
  hd.push_back(1); hd.push_back(0x22); hd.push_back(0);
  hd.push_back(2); hd.push_back(0x11); hd.push_back(1);
  hd.push_back(3); hd.push_back(0x11); hd.push_back(1);
  {
    std::vector<uint8_t> body;
    const struct { int tc; const uint8_t *bits; const uint8_t *vals; } specs[4] = {
        {0x00, kDcLumaBits, kDcLumaVals}, {0x10, kAcLumaBits, kAcLumaVals},
        {0x01, kDcChromaBits, kDcChromaVals}, {0x11, kAcChromaBits, kAcChromaVals}};
    for (auto &s : specs) {
      body.push_back((uint8_t)s.tc);
      int tot = 0;
      for (int i = 0; i < 16; i++) { body.push_back(s.bits[i]); tot += s.bits[i]; }
      for (int i = 0; i < tot; i++) body.push_back(s.vals[i]);
    }
    hd.push_back(0xFF); hd.push_back(0xC4); put_u16(hd, (int)body.size() + 2);
    hd.insert(hd.end(), body.begin(), body.end());
  }
  if (restart_interval > 0) {
    hd.push_back(0xFF); hd.push_back(0xDD); put_u16(hd, 4); put_u16(hd, restart_interval);
  }
  const uint8_t sos[14] = {0xFF, 0xDA, 0, 12, 3, 1, 0x00, 2, 0x11, 3, 0x11, 0, 63, 0};
  hd.insert(hd.end(), sos, sos + 14);
  if ((int64_t)hd.size() > out_cap) return ESSL_E_CAPACITY;
  std::memcpy(out, hd.data(), hd.size());
  BitWriter bw;
  bw.out = out + hd.size();
  bw.cap = out_cap - (int64_t)hd.size();
  // encode_kernels.py:154-202 interleaved 4:2:0 scan
  int pY = 0, pCb = 0, pCr = 0, rst = 0;
  int32_t blk[64];
  int64_t mcu = 0;
  for (int m_y = 0; m_y < my; m_y++) {
    for (int m_x = 0; m_x < mx; m_x++) {
      if (restart_interval > 0 && mcu > 0 && mcu % restart_interval == 0) {
        if (bw.cnt > 0) bw.put((1u << (8 - bw.cnt)) - 1, 8 - bw.cnt);
        bw.emit(0xFF);
        bw.emit((uint8_t)(0xD0 + (rst & 7)));
        rst++;
        pY = pCb = pCr = 0;
      }
      for (int by = 0; by < 2; by++)
        for (int bx = 0; bx < 2; bx++) {
          fdct_quant(Y.data(), yp, m_x * 2 + bx, m_y * 2 + by, ql, T.basis, blk);
          pY = encode_block(blk, pY, T.dcl, T.acl, bw);
        }
      fdct_quant(Cb.data(), cp, m_x, m_y, qc, T.basis, blk);
      pCb = encode_block(blk, pCb, T.dcc, T.acc, bw);
      fdct_quant(Cr.data(), cp, m_x, m_y, qc, T.basis, blk);
      pCr = encode_block(blk, pCr, T.dcc, T.acc, bw);
      mcu++;
    }
  }
  if (bw.cnt > 0) bw.put((1u << (8 - bw.cnt)) - 1, 8 - bw.cnt);
  bw.emit(0xFF);
  bw.emit(0xD9);
  if (bw.overflow) return ESSL_E_CAPACITY;
  return (int64_t)hd.size() + bw.pos;
}

// Own deterministic synthetic image generator for benchmark datasets:
// multi-scale smooth colour fields, hard-edged rectangles/ellipses and
// Gaussian sensor noise (sigma 6), all from splitmix64(seed).
int essl_synth_image(uint64_t seed, int h, int w, uint8_t *rgb) {
  if (!rgb || h < 1 || w < 1) return ESSL_E_ARG;
  uint64_t st = essl_rng_init(seed, 0x5EED, 0, 7);
  std::vector<double> img((size_t)h * w * 3, 0.0);
  const int cells_list[3] = {3, 7, 17};
  for (int cells : cells_list) {
    std::vector<double> f((size_t)cells * cells * 3);
    for (auto &v : f) v = 255.0 * rnd(&st);
    for (int y = 0; y < h; y++) {
      const double fy = h > 1 ? (double)y * (cells - 1) / (h - 1) : 0.0;
      int y0 = std::min((int)fy, cells - 2);
      const double wy = fy - y0;
      for (int x = 0; x < w; x++) {
        const double fx = w > 1 ? (double)x * (cells - 1) / (w - 1) : 0.0;
        int x0 = std::min((int)fx, cells - 2);
        const double wx = fx - x0;
        for (int c = 0; c < 3; c++) {
          auto F = [&](int yy, int xx) { return f[((size_t)yy * cells + xx) * 3 + c]; };
          const double top = F(y0, x0) * (1 - wx) + F(y0, x0 + 1) * wx;
          const double bot = F(y0 + 1, x0) * (1 - wx) + F(y0 + 1, x0 + 1) * wx;
          img[((size_t)y * w + x) * 3 + c] += (top * (1 - wy) + bot * wy) / 3.0;
        }
      }
    }
  }
  for (int sidx = 0; sidx < 6; sidx++) {
    double col[3] = {255.0 * rnd(&st), 255.0 * rnd(&st), 255.0 * rnd(&st)};
    const bool rect = rnd(&st) < 0.5;
    const int cy = (int)(rnd(&st) * h), cx = (int)(rnd(&st) * w);
    const int hh = h / 8 + 1 + (int)(rnd(&st) * (h / 2 - h / 8 + 1));
    const int ww = w / 8 + 1 + (int)(rnd(&st) * (w / 2 - w / 8 + 1));
    const double alpha = 0.5 + 0.45 * rnd(&st);
    for (int y = 0; y < h; y++)
      for (int x = 0; x < w; x++) {
        bool in;
        if (rect) {
          in = y >= cy && y < cy + hh && x >= cx && x < cx + ww;
        } else {
          const double dy = (double)(y - cy) / std::max(2, hh / 2), dx = (double)(x - cx) / std::max(2, ww / 2);
          in = dy * dy + dx * dx <= 1.0;
        }
        if (!in) continue;
        for (int c = 0; c < 3; c++) {
          double &v = img[((size_t)y * w + x) * 3 + c];
          v = v * (1 - alpha) + col[c] * alpha;
        }
      }
  }
  for (size_t i = 0; i < img.size(); i += 2) {  // Box-Muller, sigma 6
    double u1 = rnd(&st), u2 = rnd(&st);
    if (u1 < 1e-300) u1 = 1e-300;
    const double r = std::sqrt(-2.0 * std::log(u1)) * 6.0;
    img[i] += r * std::cos(6.283185307179586 * u2);
    if (i + 1 < img.size()) img[i + 1] += r * std::sin(6.283185307179586 * u2);
  }
  for (size_t i = 0; i < img.size(); i++) {
    const double v = img[i];
    rgb[i] = (uint8_t)(v < 0 ? 0 : v > 255 ? 255 : v);
  }
  return ESSL_OK;
}

}  // extern "C"
