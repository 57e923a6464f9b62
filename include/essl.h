/*
 * essl.h -- C ABI of libessl, the B200-native (sm_100a) implementation of
 * the ESSL / DailyMAE data-loading hot path:
 *
 *   read_sample -> sample_rrc -> decode_crop -> resize_bilinear -> hflip
 *               -> normalize -> sample_mask            (+ ids_keep/restore)
 *
 * The reference (cropload, Python+numba) has no native ABI; its operator
 * boundary is the Python API.  Each entry point below names the reference
 * interface it replaces (paths relative to /root/reference/pkg/src/cropload).
 * Plain pointers and sizes only; no torch types.  Every device call is
 * stream-ordered on the caller's cudaStream_t (passed as void*), never
 * synchronises implicitly, and returns 0 on success or a negative
 * ESSL_E_* code (message via essl_last_error()).
 *
 * Threading: an essl_ctx is single-consumer (reference SPEC.md:555, "a
 * session is single-consumer"); use one context per rank / consumer thread.
 */
#ifndef ESSL_H_
#define ESSL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ---- API return codes ------------------------------------------------- */
#define ESSL_OK 0
#define ESSL_E_ARG -1      /* invalid argument */
#define ESSL_E_CUDA -2     /* CUDA runtime error */
#define ESSL_E_CAPACITY -3 /* batch / scratch capacity exceeded */
#define ESSL_E_NOMEM -4

/* ---- per-image status (int32 status[] arrays) ---------------------------
 * Mirrors the reference scan status codes (jpeg/decode_kernels.py:14-15)
 * plus the exception family of jpeg/codec.py and container.py. */
#define ESSL_ST_OK 0
#define ESSL_ST_CORRUPT_HUFFMAN 1 /* DecodeError "corrupt entropy-coded data" */
#define ESSL_ST_MISSING_RST 3     /* DecodeError "missing restart marker" */
#define ESSL_ST_TRUNCATED 4       /* DecodeError "truncated entropy-coded data" */
#define ESSL_ST_CRC 5             /* CorruptionError "checksum mismatch" */
#define ESSL_ST_UNSUPPORTED 6     /* progressive / multi-scan (no CPU fallback) */
#define ESSL_ST_RECT 7            /* ValueError: crop rect out of bounds */
#define ESSL_ST_MALFORMED 8       /* DecodeError from parse_stream */
#define ESSL_ST_HUFFTABLE 9       /* DecodeError from _huff_lut */
#define ESSL_ST_QUANT 10          /* DecodeError "missing quantization table" */
#define ESSL_ST_CAPACITY 11       /* image exceeds the context's scratch */

/* ---- output layouts (essl_decode_rrc out_kind) ------------------------- */
#define ESSL_OUT_BF16_NCHW 0 /* bf16 [n,3,res,res], RNE of the f32 value */
#define ESSL_OUT_F32_NCHW 1  /* float32 [n,3,res,res] == ImageBatch.pixels */
#define ESSL_OUT_NONE 2      /* only the optional uint8 view */

/* ---- decoder modes (essl_ctx_set_option ESSL_OPT_DECODE_MODE) ---------- */
#define ESSL_DECODE_SPECULATIVE 0 /* self-synchronising parallel decode */
#define ESSL_DECODE_SERIAL 1      /* one thread per image (validation) */

#define ESSL_OPT_DECODE_MODE 1
#define ESSL_OPT_SEQ_BITS 2        /* minimum subsequence length per lane (bits, >= 32) */
#define ESSL_OPT_CHECKPOINT_BITS 3 /* accepted and validated, no effect: every block start is a checkpoint */
#define ESSL_OPT_PROFILE 4      /* 1: bracket every launch with CUDA events */
#define ESSL_OPT_WARMUP_BITS 5  /* lanes start this far before their subsequence (0..4096) */
#define ESSL_OPT_STAGE_BYTES 6  /* largest clean stream staged in shared memory (0: never) */
#define ESSL_OPT_GATHER_CTAS 7  /* k_host_gather CTAs (bus-read gather; 0: one per payload) */
#define ESSL_OPT_GATHER_TMA 8   /* 1 (default): bus-read gather with bulk (TMA) copies; 0: LSU loads */
#define ESSL_OPT_DEBUG_LANES 9  /* 1: record per-lane speculative-decode state (essl_debug_lanes) */
#define ESSL_OPT_TRACE 10       /* n > 0: record up to n CTA executions (essl_trace_read); 0 off */
#define ESSL_OPT_RESIZE_COLS 11 /* k_resize output columns per thread: 2 (default), 4 or 8 */
#define ESSL_OPT_RESIZE_BAND 12 /* k_resize output rows per CTA, at most (1..64, default 64) */
#define ESSL_OPT_EARLY_EXIT 13  /* 1 (default): entropy decode stops near the crop's last needed row */
#define ESSL_OPT_PROFILE_KERNELS 14 /* bitmask of ESSL_K_* launches ESSL_OPT_PROFILE brackets (default all) */

/* kernel ids for essl_ctx_profile_read */
#define ESSL_K_DECODE 0
#define ESSL_K_RESIZE 1
#define ESSL_K_CROP 2
#define ESSL_K_MASK 3
#define ESSL_K_GATHER 4
#define ESSL_K_DUMP 5
#define ESSL_K_PREP 6    /* k_prep: CRC, parse, destuff, tables */
#define ESSL_K_ENTROPY 7 /* k_entropy: Huffman decode */
#define ESSL_K_IDCT 8    /* k_idct: dequant + IDCT */
#define ESSL_K_STAGE 9   /* k_host_gather: pinned-container payload gather */
#define ESSL_K_AUG 10    /* k_aug_blur + k_aug_out: 3-Aug / 3-Aug+ */
#define ESSL_K_COUNT 11

typedef struct essl_ctx essl_ctx;

/* One sample of a batch.  `offset` indexes the byte blob passed to
 * essl_decode_rrc (a device-resident container or the staging buffer).
 * (x, y, w, h) is the RandomResizedCrop window (pipeline.py:51-75,
 * codec.py:43-56); flip is the apply_aug draw (pipeline.py:86-87). */
typedef struct {
  uint64_t offset;
  uint32_t length;
  uint32_t crc32; /* expected zlib CRC32 (container.py:46-51 "checksum") */
  int32_t x, y, w, h;
  int32_t flip;
  int32_t check_crc; /* 0 skips the CRC check (decode_crop has none) */
} essl_sample;

/* Per-image results: stats mirror DecodeStats (codec.py:59-71). */
typedef struct {
  int32_t status;
  int32_t reason; /* sub-code for MALFORMED / UNSUPPORTED / HUFFTABLE */
  int32_t offset; /* byte offset for DecodeError(offset) or -1 */
  int32_t mcus_entropy_decoded;
  int32_t mcus_reconstructed;
  int32_t width, height, ncomp;
} essl_result;

/* ---- 3-Aug / 3-Aug+ (apply_aug, pipeline.py:78-101; imgops.py:75-227) ----
 * Per-sample parameters of the augmentation applied after the flip.  Filled
 * by essl_aug_draw / essl_aug_batch from the sample's pipeline stream,
 * except `weights`: gaussian_blur's taps (imgops.py:157-160) are numpy exp
 * values in the reference, so the caller evaluates them the same way
 * (exp(-(x*x)/(2*sigma*sigma)) over x = -radius..radius, divided by their
 * sum) and writes 2*radius+1 of them. */
#define ESSL_AUG_SIMPLE 0     /* AugLevel.SIMPLE: flip only */
#define ESSL_AUG_3AUG 1       /* + one of grayscale / solarize / blur */
#define ESSL_AUG_3AUG_PLUS 2  /* + brightness, contrast, saturation jitter */
#define ESSL_AUG_OP_NONE (-1)
#define ESSL_AUG_OP_GRAY 0     /* imgops.py:75-91, BT.601 fixed point */
#define ESSL_AUG_OP_SOLARIZE 1 /* imgops.py:94-108, v >= threshold -> 255 - v */
#define ESSL_AUG_OP_BLUR 2     /* imgops.py:122-163, separable, reflect padding */
#define ESSL_AUG_MAX_RADIUS 12
typedef struct {
  int32_t op;        /* ESSL_AUG_OP_* */
  int32_t radius;    /* blur radius max(1, ceil(3 sigma)), <= ESSL_AUG_MAX_RADIUS */
  int32_t jitter;    /* 1: adjust_brightness, _contrast, _saturation in order */
  int32_t threshold; /* solarize threshold (SOLARIZE_THRESHOLD = 128) */
  double sigma;      /* blur sigma ~ U[0.1, 2.0) (BLUR_SIGMA_RANGE) */
  double factors[3]; /* brightness, contrast, saturation ~ U[0.7, 1.3) */
  double weights[2 * ESSL_AUG_MAX_RADIUS + 1];
  double reserved;
} essl_aug;

/* ---- context ------------------------------------------------------------
 * Replaces: Loader.__init__ (pipeline.py:181-195) resource setup.  The
 * context owns device scratch sized for `max_batch` images of at most
 * `max_side` pixels per side and `max_payload` bytes each, plus pinned
 * staging for `max_batch * max_payload` bytes (double-buffered).
 * max_payload <= 4 MiB. */
int essl_ctx_create(int device, int max_batch, int max_side, int max_payload,
                    int flags, essl_ctx **out);
int essl_ctx_destroy(essl_ctx *ctx);
int essl_ctx_set_option(essl_ctx *ctx, int option, int64_t value);
/* The value a new context starts with for `option` (no device needed). */
int essl_option_default(int option, int64_t *value);
/* Number of kernels this context launched since creation (bench evidence). */
int64_t essl_ctx_launch_count(const essl_ctx *ctx);
/* With ESSL_OPT_PROFILE on: synchronise the recorded events, add each
 * kernel's device time (ms) and launch count into ms[ESSL_K_COUNT] /
 * count[ESSL_K_COUNT], and clear the record. */
int essl_ctx_profile_read(essl_ctx *ctx, double *ms, int64_t *count);
/* Profiling timeline: record a process-wide reference point on `stream`;
 * essl_ctx_profile_timeline then returns (without clearing) up to `max`
 * recorded launches as kernel id + start/end in ms after that reference.
 * Returns the number written (>= 0) or a negative error. */
int essl_profile_mark(void *stream);
int essl_ctx_profile_timeline(essl_ctx *ctx, int32_t *kid, double *t0_ms, double *t1_ms, int max);
/* Debug: per-image decode phase clocks / counters of the last batch
 * (int64[16*n]: k_prep/k_entropy phase clocks, fixpoint iterations,
 * subsequence count | redo count << 32).  Synchronous. */
int essl_debug_stats(essl_ctx *ctx, int64_t *out, int n);
/* Debug: per-lane records of the last speculative decode (ESSL_OPT_DEBUG_LANES
 * on), int32[n][64][8]: {nseq, phase-1 stop bit, stop block slot, checkpoints,
 * phase-1 error, continuation stop bit, continuation status (0 merged,
 * 1 error, 2 end of data), merge lane} (-1 where not run).  Synchronous. */
int essl_debug_lanes(essl_ctx *ctx, int32_t *out, int n);
/* Debug: CTA execution records since the last read (ESSL_OPT_TRACE on),
 * uint64[max][4] = {start ns, end ns (globaltimer), kernel id (ESSL_K_*),
 * SM id} for k_prep / k_entropy / k_idct / k_resize.  Synchronises the
 * device; returns the number of records written. */
int essl_trace_read(essl_ctx *ctx, uint64_t *out, int max);
/* Bounds-check counters of a checked build (ESSL_CHECKED): out[i] = the
 * number of out-of-bounds accesses caught by check i (scratch lists,
 * coefficient windows, multi-scan arrays, planes, clean streams, resize
 * staging, outputs, checkpoints) on the current device since the last reset.
 * Returns 1 for a checked build, 0 otherwise (the counters stay 0), <0 on
 * error.  Synchronous. */
int essl_check_read(uint32_t *out, int n, int reset);
const char *essl_last_error(void);
const char *essl_version(void);
/* Stream-ordered copy of `bytes` between host (pinned) and device memory
 * (cudaMemcpyDefault), for the loader's per-batch index / label / status
 * transfers without switching the caller's current stream. */
int essl_memcpy_async(void *dst, const void *src, uint64_t bytes, void *stream);

/* ---- staging (host bytes -> device) -------------------------------------
 * Replaces: ContainerHandle.read_sample (container.py:249-265) bytes path.
 * Gathers n payloads (host pointers, e.g. an mmap) into the context's
 * pinned ring slot `slot` (0/1) with `nthreads` host threads, then issues
 * one async H2D copy on `stream`.  Writes each sample's offset inside the
 * staged blob into samples[i].offset and returns the device blob pointer
 * in *dev_blob.  Payloads are 64-byte aligned in the blob. */
int essl_stage(essl_ctx *ctx, int slot, const uint8_t *const *src,
               const uint32_t *len, int n, essl_sample *samples,
               int nthreads, void *stream, const uint8_t **dev_blob);
/* Pinned-container staging (the e2e host->device path): the container's host
 * bytes are page-locked once (essl_host_register: read-only, mapped
 * registration of the file mapping; essl_host_device_ptr gives its device
 * address).  Each batch's payloads are then gathered host->device by one
 * light kernel reading the pinned container over the bus (k_host_gather)
 * into the context's staging slot, with the same 64-byte packing and
 * `samples` rewrite as essl_stage.  Replaces: ContainerHandle.read_sample's
 * payload slice (container.py:249-265) for a whole batch. */
int essl_host_register(void *ptr, uint64_t bytes, int readonly);
int essl_host_unregister(void *ptr);
int essl_host_device_ptr(void *ptr, void **dev_ptr);
int essl_stage_pinned(essl_ctx *ctx, int slot, const uint8_t *dev_base, const uint64_t *src_off,
                      const uint32_t *len, int n, essl_sample *samples, void *stream,
                      const uint8_t **dev_blob);

/* ---- the hot path --------------------------------------------------------
 * Replaces: Loader._fill_sample (pipeline.py:219-235) for a whole batch:
 * CRC check (container.py:263) -> decode_crop (codec.py:448-511) ->
 * resize_bilinear (imgops.py:63-72) -> hflip (imgops.py:256) ->
 * normalize (imgops.py:243-248).
 * `blob` is a DEVICE pointer; samples[] is HOST memory (copied async).
 * out: [n,3,res,res] in out_kind layout with sample stride out_stride
 * elements (0 = dense); out_u8: optional uint8 [n,res,res,3] view
 * (ImageBatch.uint8, pipeline.py:114).  results: optional DEVICE array of
 * n essl_result. */
int essl_decode_rrc(essl_ctx *ctx, const uint8_t *blob,
                    const essl_sample *samples, int n, int res, int out_kind,
                    void *out, int64_t out_stride, uint8_t *out_u8,
                    essl_result *results, void *stream);

/* Same with the 3-Aug / 3-Aug+ stage (pipeline.py:88-101) between the flip
 * and normalize: aug is a HOST array of n essl_aug (NULL: simple).  The
 * uint8 view (out_u8) holds the augmented image (ImageBatch.uint8 is the
 * image normalize sees, pipeline.py:228-232). */
int essl_decode_rrc_aug(essl_ctx *ctx, const uint8_t *blob,
                        const essl_sample *samples, const essl_aug *aug, int n,
                        int res, int out_kind, void *out, int64_t out_stride,
                        uint8_t *out_u8, essl_result *results, void *stream);

/* Same, plus the MAE visible tokens of every image (N1/a20: patchify
 * 'nchpwq->nhwpqc' of the bf16 normalized pixels) written by
 * the resize kernel itself: tokens_bf16 is DEVICE bf16 [n, n_keep,
 * patch*patch*3] and row r of image i is the patch t with ids_restore[i][t]
 * == r < n_keep (ids_restore: DEVICE int64 [n, (res/patch)^2], e.g. from
 * essl_mask earlier on the same stream).  tokens_bf16 == NULL: no tokens
 * (== essl_decode_rrc_aug). */
int essl_decode_rrc_visible(essl_ctx *ctx, const uint8_t *blob,
                            const essl_sample *samples, const essl_aug *aug,
                            int n, int res, int out_kind, void *out,
                            int64_t out_stride, uint8_t *out_u8, int patch,
                            const int64_t *ids_restore, int n_keep,
                            void *tokens_bf16, essl_result *results,
                            void *stream);

/* Replaces: decode_crop(bytes, CropRect) (codec.py:448-511) for a batch of
 * crops: writes each uint8 [h,w,3] region at out + out_offsets[i]
 * (device pointer + host offsets). */
int essl_decode_crop_u8(essl_ctx *ctx, const uint8_t *blob,
                        const essl_sample *samples, int n, uint8_t *out,
                        const uint64_t *out_offsets, essl_result *results,
                        void *stream);

/* Debug/parity: the int16 coefficients of every block in the crop window
 * (natural order, dequantisation not applied), per component c as
 * [wbh_c][wbw_c][64], components back to back, at out + out_offsets[i]
 * (element offsets, capacity out_cap elements).  geometry (HOST int32
 * [12*n]) receives {wby0, wbx0, wbh, wbw} per component.  Synchronises.
 * (decode_scan_baseline output, decode_kernels.py:111-179, rows <
 * row_stop; the crop window of codec.py:502-508.) */
int essl_dump_coefs(essl_ctx *ctx, const uint8_t *blob,
                    const essl_sample *samples, int n, int16_t *out,
                    const uint64_t *out_offsets, int64_t out_cap,
                    int32_t *geometry, essl_result *results, void *stream);

/* ---- MAE masking ----------------------------------------------------------
 * Replaces: sample_mask (masking.py:48-56) with SampleRng(seed, epoch,
 * index, DOMAIN_MASK) (pipeline.py:233-235), plus the MAE conventions
 * ids_keep = sorted(complement(mask)), ids_restore = argsort(concat(
 * ids_keep, mask)).  index: DEVICE int64[n].  Any of the outputs may be
 * NULL.  tokens = grid*grid <= 4096. */
int essl_mask(essl_ctx *ctx, uint64_t seed, uint64_t epoch,
              const int64_t *index, int n, int tokens, int k,
              int32_t *mask_sorted, int64_t *ids_keep, int64_t *ids_restore,
              void *stream);

/* Same, from explicit per-sample stream states (DEVICE uint64[n]): the
 * state of SampleRng(seed, epoch, index, DOMAIN_MASK) before the shuffle
 * (rng.py:39-44), for callers holding an arbitrary SampleRng. */
int essl_mask_from_states(essl_ctx *ctx, const uint64_t *states, int n,
                          int tokens, int k, int32_t *mask_sorted,
                          int64_t *ids_keep, int64_t *ids_restore,
                          void *stream);

/* Visible-token gather of MAE patchify (nchpwq->nhwpqc): pixels bf16
 * [n,3,res,res] -> tokens bf16 [n, n_keep, patch*patch*3]. */
int essl_gather_visible(essl_ctx *ctx, const void *pixels_bf16, int n,
                        int res, int patch, const int64_t *ids_keep,
                        int n_keep, void *tokens_bf16, void *stream);

/* ---- standalone pixel ops (device pointers) ------------------------------
 * Replace imgops.resize_bilinear (imgops.py:63-72), hflip (:256) and
 * normalize (:243-248) on caller-provided uint8 HWC images. */
int essl_resize_u8(const uint8_t *src, int ih, int iw, uint8_t *dst, int oh,
                   int ow, int flip, void *stream);
int essl_normalize_u8(const uint8_t *src, int h, int w, float *dst,
                      void *stream);
/* apply_aug's pixel stage after the flip (pipeline.py:88-101) on n uint8
 * HWC images [n,h,w,3] (DEVICE src/dst, may not alias); aug is a HOST
 * array of n essl_aug.  Replaces grayscale / solarize / gaussian_blur /
 * adjust_brightness / adjust_contrast / adjust_saturation (imgops.py:75-227)
 * as a batch.  h, w <= the context's max_side. */
int essl_augment_u8(essl_ctx *ctx, const uint8_t *src, int n, int h, int w,
                    const essl_aug *aug, uint8_t *dst, void *stream);

/* ---- native batch enqueue ---------------------------------------------------
 * Replaces: Loader._fill_sample for a whole batch plus the batch assembly of
 * Loader.epoch (pipeline.py:219-267) in ONE stream-ordered call, so the host
 * side of a batch costs microseconds: descriptors from the record table +
 * RandomResizedCrop / flip draws (host C++), index/label upload, optional
 * pinned-container gather, MAE mask (before the pixels: the fused visible
 * tokens read ids_restore), decode + resize + normalize, result download.
 * The record table (container.py:46-51 RECORD_DTYPE columns) is copied once
 * into an essl_dataset. */
typedef struct essl_dataset essl_dataset;
int essl_dataset_create(int64_t n, const uint64_t *offsets, const uint32_t *lengths,
                        const uint32_t *crc32, const uint16_t *widths,
                        const uint16_t *heights, const int64_t *labels,
                        essl_dataset **out);
int essl_dataset_destroy(essl_dataset *ds);

typedef struct {
  uint64_t seed, epoch;       /* SampleRng keys (rng.py:39-44) */
  double scale[2], ratio[2];  /* RrcConfig (pipeline.py:31-48) */
  int32_t res, out_kind;      /* output resolution, ESSL_OUT_* */
  int32_t check_crc;          /* 1: verify each payload's CRC32 (container.py:263) */
  int32_t tokens, masked;     /* MAE mask: N tokens, k masked (0 tokens: no mask) */
  int32_t patch;              /* patch size (visible tokens) */
} essl_batch_cfg;

typedef struct {
  const uint8_t *blob;         /* DEVICE resident container bytes, or NULL: */
  const uint8_t *pinned_base;  /* DEVICE address of the page-locked container */
  int32_t stage_slot;          /* staging slot (0/1) of the pinned gather */
  int32_t stage_chain;         /* > 0: the gather runs after the device's previous chained
                                  gather, on this many CTAs (a pipeline fill: the oldest
                                  batch's payloads arrive first); 0: concurrent */
  const essl_aug *aug;         /* HOST n 3-Aug entries (essl_aug_batch), or NULL */
  void *pixels;                /* DEVICE [n,3,res,res] out_kind, caller-owned */
  int64_t pixel_stride;        /* elements between samples (0: dense) */
  uint8_t *u8;                 /* DEVICE uint8 [n,res,res,3] view, or NULL */
  int64_t *index_label;        /* DEVICE int64 [2n]: indices, then labels */
  int32_t *mask;               /* DEVICE outputs of the mask (any may be NULL) */
  int64_t *ids_keep, *ids_restore;
  void *tokens;                /* DEVICE bf16 visible tokens [n, N-k, patch^2*3], or NULL */
  essl_result *results;        /* DEVICE [n] */
  essl_result *results_host;   /* HOST pinned [n] copy of results, or NULL */
  void *wait_stream;           /* cudaStream_t whose work so far precedes this batch's
                                  work on `stream` (the consumer's stream), or NULL */
} essl_batch_io;

int essl_batch_enqueue(essl_ctx *ctx, const essl_dataset *ds, const essl_batch_cfg *cfg,
                       const int64_t *indices, int n, const essl_batch_io *io,
                       void *stream);

/* ABI check for bindings: sizeof of the public structs, in the order
 * essl_sample, essl_result, essl_aug, essl_batch_cfg, essl_batch_io.
 * Writes min(n, 5) sizes; returns 5. */
int essl_abi_sizes(int64_t *out, int n);

/* ---- host-side sampling (C++, glibc libm: bit-exact with CPython) ---------
 * Replace rng.py:27-87 and pipeline.py:51-87. */
uint64_t essl_rng_init(uint64_t seed, uint64_t epoch, uint64_t index,
                       uint64_t domain);
uint64_t essl_rng_next(uint64_t *state);
double essl_rng_random(uint64_t *state);
int64_t essl_rng_randint(uint64_t *state, int64_t n);
int essl_epoch_permutation(uint64_t seed, uint64_t epoch, int64_t n,
                           int64_t *out);
/* One RRC rect (+ flip draw when flip_out != NULL) for (seed, epoch, index). */
int essl_sample_rrc(uint64_t *state, int64_t src_w, int64_t src_h,
                    double scale_lo, double scale_hi, double ratio_lo,
                    double ratio_hi, int max_attempts, int32_t *xywh);
/* Batch: rects + flips for dataset indices (record dims w/h indexed by
 * dataset index), filling samples[i].{x,y,w,h,flip}. */
int essl_rrc_batch(uint64_t seed, uint64_t epoch, const int64_t *indices,
                   int n, const uint16_t *widths, const uint16_t *heights,
                   double scale_lo, double scale_hi, double ratio_lo,
                   double ratio_hi, essl_sample *samples);
int essl_mask_count(int tokens, double ratio); /* masking.py:43-45 */
/* apply_aug's draws (pipeline.py:85-101) from a pipeline stream positioned
 * after sample_rrc: flip, then for 3-Aug op = randint(3) and, for the blur,
 * sigma = uniform(0.1, 2.0); for 3-Aug+ three uniform(0.7, 1.3) factors.
 * Leaves aug->weights zero (see essl_aug). */
int essl_aug_draw(uint64_t *state, int level, int32_t *flip, essl_aug *aug);
/* essl_rrc_batch + essl_aug_draw per sample (aug may be NULL for SIMPLE). */
int essl_aug_batch(uint64_t seed, uint64_t epoch, const int64_t *indices,
                   int n, const uint16_t *widths, const uint16_t *heights,
                   double scale_lo, double scale_hi, double ratio_lo,
                   double ratio_hi, int level, essl_sample *samples,
                   essl_aug *aug);

/* ---- dataset builder (row f2; fixtures and benchmark inputs) --------------
 * encode_jpeg (codec.py:574-632): baseline 4:2:0, Annex-K tables, float64
 * FDCT with the pinned basis.  Returns the byte count written to out, or a
 * negative code when out_cap is too small. */
int64_t essl_encode_jpeg(const uint8_t *rgb, int h, int w, int quality,
                         int restart_interval, uint8_t *out, int64_t out_cap);
/* Deterministic synthetic natural-style image (own generator). */
int essl_synth_image(uint64_t seed, int h, int w, uint8_t *rgb);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif
#endif /* ESSL_H_ */
