// Shared device-side definitions for libessl (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "essl.h"

namespace essl {

// Bounds-checked builds (ESSL_CHECKED, `ESSL_CHECKED=1 python -m
// paper_2404_00509_b200.build`): every scratch / output access named by a
// check id is verified on the device and violations are counted (no trap:
// the run continues and the count is read back with essl_check_read).  This
// stands in for compute-sanitizer, which is closed on the GPU pool.
enum CheckId : int {
  CK_LIST = 0,     // k_entropy unit-list / block-record / sentinel stores
  CK_COEF = 1,     // coefficient window / table stores (k_entropy)
  CK_MS_COEF = 2,  // multi-scan full coefficient arrays
  CK_PLANE = 3,    // k_idct plane stores
  CK_CLEAN = 4,    // k_prep clean-stream bytes / restart table
  CK_SRC = 5,      // k_resize shared source-row staging
  CK_OUT = 6,      // k_resize output stores
  CK_CKPT = 7,     // k_entropy checkpoint (block record) reads of later lanes
  CK_COUNT = 16,
};
#ifdef ESSL_CHECKED
#define ESSL_CHECK(table, cond, id) \
  do {                                \
    if (!(cond)) atomicAdd(&(table)[(id)], 1u); \
  } while (0)
#else
#define ESSL_CHECK(table, cond, id) \
  do {                                \
  } while (0)
#endif
void check_read_decode(unsigned int *out, bool reset);
void check_read_pixels(unsigned int *out, bool reset);

constexpr int kDecodeThreads = 256;  // k_prep: one CTA per image
constexpr int kEntropyLanes = 64;     // k_entropy: subsequences (threads) per image
constexpr int kContinuationBits = 8192;  // k_entropy: list room per lane for its continuation
constexpr int kMaxWarmBits = 4096;
constexpr int kFastBits = 10;        // first-level Huffman lookahead
constexpr int kMaxTables = 6;        // distinct (class,id) tables a 3-slot scan can use
constexpr int kMaxBpm = 48;          // blocks per MCU (h,v <= 4, 3 components)
constexpr int kHdrCache = 2048;      // payload prefix staged in shared memory

// Reason sub-codes (must match oracle/essl_oracle.c and errors.py).
enum Reason : int32_t {
  R_NONE = 0, R_NO_SOI = 1, R_EXPECTED_MARKER = 2, R_UNEXPECTED_END = 3,
  R_TRUNC_SEGMENT = 4, R_TRUNC_DQT = 5, R_TRUNC_DHT = 6, R_MULTI_SOF = 7,
  R_PRECISION = 8, R_ZERO_DIM = 9, R_NCOMP = 10, R_SAMPLING = 11,
  R_SOF_TYPE = 12, R_SOS_BEFORE_SOF = 13, R_UNKNOWN_COMP = 14,
  R_NO_IMAGE = 15, R_RST_NO_DRI = 16, R_TOO_MANY_RST = 17,
  R_PROGRESSIVE = 18, R_MULTI_SCAN = 19, R_HUFF_UNDEFINED = 20,
  R_HUFF_OVERFLOW = 21, R_HUFF_TOO_MANY = 22, R_SEGMENT = 23,
  R_COEF_RANGE = 24, R_SCRATCH = 25, R_PROG_DC_SE = 26, R_PROG_AC_NCOMP = 27,
  R_PARTIAL_INTERLEAVE = 28, R_TOO_MANY_SCANS = 29,
};

// Per-image decode products consumed by the pixel kernels.  Written by
// k_decode (one CTA per image), read by k_resize / k_crop_u8.
struct ImgInfo {
  int32_t status, reason, offset;
  int32_t width, height, ncomp;
  int32_t hmax, vmax;
  int32_t comp_h[3], comp_v[3];
  // crop window per component in blocks (full MCU extents, codec.py:502-508)
  int32_t wby0[3], wbx0[3], wbh[3], wbw[3];
  int32_t plane_pitch[3];
  uint64_t plane_off[3];  // bytes into Scratch::plane
  uint64_t coef_off[3];   // int16 elements into Scratch::coef (the window's first block)
  int32_t coef_pitch[3];  // blocks per coefficient-array row
  int32_t mcus_entropy, mcus_recon;
  int32_t rx, ry, rw, rh, flip;
  int32_t fmt;  // 0: coefficient window (int16); 1: per-block tables into the unit lists
  int64_t dbg[16];  // phase clocks / counters (essl_debug_stats)
};

// Device scratch owned by the context; per-image regions are carved with
// atomics on `counters` (reset per batch), so placement is order-free and
// results never depend on it.
struct Scratch {
  uint8_t *clean;
  uint64_t clean_cap;
  int16_t *coef;
  uint64_t coef_cap;  // elements
  uint8_t *plane;
  uint64_t plane_cap;
  unsigned long long *counters;  // [0] clean bytes, [1] coef elems, [2] plane bytes, [3] list entries
  ImgInfo *info;
  uint8_t *hdr;  // per-image DecodeHdr handed from k_prep to k_entropy
  uint32_t *list;   // unit lists (k_entropy), carved per image with counters[3]
  uint64_t list_cap;  // entries
  uint8_t *tabcache;  // built Huffman tables reused across images (k_prep; tabcache_bytes())
};

// Optional per-CTA execution trace (ESSL_OPT_TRACE): {start ns, end ns,
// kernel id, SM id} per CTA, appended at an atomic cursor.
struct CtaTrace {
  unsigned long long *buf;
  unsigned int *count;
  unsigned int cap;
};

struct TraceScope {
  const CtaTrace &t;
  unsigned long long t0;
  int kid;
  __device__ __forceinline__ static unsigned long long now() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    return v;
  }
  __device__ __forceinline__ TraceScope(const CtaTrace &t_, int kid_) : t(t_), t0(0), kid(kid_) {
    if (t.buf && threadIdx.x == 0) t0 = now();
  }
  __device__ __forceinline__ ~TraceScope() {
    if (t.buf && threadIdx.x == 0) {
      const unsigned int i = atomicAdd(t.count, 1u);
      if (i < t.cap) {
        unsigned int sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        t.buf[4 * i] = t0;
        t.buf[4 * i + 1] = now();
        t.buf[4 * i + 2] = (unsigned long long)kid;
        t.buf[4 * i + 3] = sm;
      }
    }
  }
};

struct DecodeParams {
  const uint8_t *blob;
  const essl_sample *samples;  // device copy of the batch descriptors
  int n;
  Scratch s;
  int mode;          // ESSL_DECODE_*
  int seq_bits;      // minimum subsequence length per lane (bits)
  int warm_bits;     // each lane (but lane 0) starts this far before its subsequence
  int stage_bytes;   // k_entropy read rings (0: plain global reads)
  int early_exit;    // k_entropy: phase 1 stops near the crop's last needed block (N2)
  int prep_part_off; // k_prep: byte offset of the CRC partials in dynamic smem
  essl_result *results;  // optional
  int32_t *dbg_lanes;    // optional per-lane decode records [n][kEntropyLanes][8]
  CtaTrace trace;
};

struct PixelParams {
  const ImgInfo *info;
  const uint8_t *plane;
  int n, res;
  int out_kind;
  void *out;
  int64_t out_stride;  // elements per sample
  uint8_t *out_u8;
  int src_words;       // k_resize shared source rows: band source rows x widest crop
  int band;            // k_resize output rows per CTA (<= kMaxBandRows)
  // 3-Aug: per-image draws (device) or nullptr.  Images whose op is a point
  // op (none / grayscale / solarize) without jitter are finished here (point
  // op fused before normalize); blur or jitter images go to aug_u8 for
  // k_aug_blur / k_aug_out.
  const essl_aug *aug;
  uint8_t *aug_u8;
  // MAE visible tokens (optional): bf16 [n, n_keep, patch*patch*3], rows
  // placed by ids_restore (device int64 [n, (res/patch)^2])
  void *vis;
  const int64_t *vis_restore;
  int patch, n_keep;
  int cols;  // k_resize output columns per thread (8: 128-bit bf16 stores, 4: 64-bit)
  CtaTrace trace;
};

// 3-Aug stage (k_aug_blur / k_aug_out): a = resized (flipped) uint8 HWC
// images, b = blurred copies (written for blur images only).
struct AugOutParams {
  const uint8_t *a;
  uint8_t *b;
  const essl_aug *aug;  // device, n entries
  int n, h, w;
  int out_kind;
  void *out;
  int64_t out_stride;
  uint8_t *out_u8;
  int fused_points;  // 1: point-op-only images were finished by k_resize (skip them)
};

// splitmix64 (rng.py:27-31)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t rng_init(uint64_t seed, uint64_t epoch,
                                                      uint64_t index, uint64_t domain) {
  uint64_t h = mix64(seed);
  h = mix64(h ^ (epoch * kGamma));
  h = mix64(h ^ (index * kGamma));
  h = mix64(h ^ (domain * kGamma));
  return h;
}

// One payload of a pinned-container gather (essl_stage_pinned).
struct GatherDesc {
  uint64_t src, dst;
  uint32_t len, pad;
};

// launch wrappers (defined in the .cu files)
void launch_prep(const DecodeParams &p, cudaStream_t st, int max_len);
void launch_entropy(const DecodeParams &p, cudaStream_t st, int max_len);
void launch_idct(const DecodeParams &p, cudaStream_t st);
size_t decode_hdr_bytes();
size_t tabcache_bytes();
void launch_resize(const PixelParams &p, cudaStream_t st);
void launch_aug(const AugOutParams &p, int max_radius, cudaStream_t st);
void launch_host_gather(const uint8_t *src, const GatherDesc *d, int n, uint8_t *dst, int ctas,
                        bool tma, cudaStream_t st);
constexpr int kMaxBandRows = 64;      // k_resize: output rows per CTA, at most
int band_source_rows(int h, int res, int band);
size_t resize_smem(const PixelParams &p);
void launch_crop_u8(const ImgInfo *info, const uint8_t *plane, int n, uint8_t *out,
                    const uint64_t *offsets, cudaStream_t st);
void launch_mask(uint64_t seed, uint64_t epoch, const int64_t *index, int n, int tokens,
                 int k, int32_t *mask, int64_t *keep, int64_t *restore, cudaStream_t st);
void launch_mask_states(const uint64_t *states, int n, int tokens, int k, int32_t *mask,
                        int64_t *keep, int64_t *restore, cudaStream_t st);
void launch_gather(const void *pix, int n, int res, int patch, const int64_t *keep,
                   int n_keep, void *tokens, cudaStream_t st);
void launch_gather_restore(const void *pix, int n, int res, int patch, const int64_t *restore,
                           int n_keep, void *tokens, cudaStream_t st);
void launch_resize_u8(const uint8_t *src, int ih, int iw, uint8_t *dst, int oh, int ow,
                      int flip, cudaStream_t st);
void launch_normalize_u8(const uint8_t *src, int h, int w, float *dst, cudaStream_t st);
void launch_results(const ImgInfo *info, int n, essl_result *res, cudaStream_t st);
void launch_dump_coefs(const Scratch &sc, int n, int16_t *out, const uint64_t *offsets,
                       cudaStream_t st);

}  // namespace essl
