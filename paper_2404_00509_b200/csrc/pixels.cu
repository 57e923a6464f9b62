// Pixel-side kernels:
//   k_resize   : YCbCr planes -> colour convert (decode_kernels.py:537-589) ->
//                bilinear (imgops.py:24-60) -> hflip (imgops.py:256) ->
//                normalize (imgops.py:231-240) -> bf16/f32 NCHW (+ u8 NHWC)
//   k_crop_u8  : YCbCr planes -> RGB uint8 crop region (codec.py:422-431)
//   k_mask     : sample_mask (masking.py:48-56) + ids_keep / ids_restore
//   k_gather   : MAE patchify + visible-token gather
//   k_resize_u8 / k_normalize_u8 : standalone imgops
//
// Exactness: the resize is float64 without contraction (__dmul_rn/__dadd_rn),
// normalize is float32 IEEE (__fmul_rn/__fsub_rn/__fdiv_rn), so uint8 and
// float32 outputs are bit-identical to the reference; bf16 is the RNE of the
// exact float32.
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>

#include "essl_common.cuh"

namespace essl {

__device__ unsigned int g_check_pix[CK_COUNT];  // ESSL_CHECK counters (checked builds)

void check_read_pixels(unsigned int *out, bool reset) {
  cudaMemcpyFromSymbol(out, g_check_pix, sizeof(unsigned int) * CK_COUNT);
  if (reset) {
    static const unsigned int zero[CK_COUNT] = {};
    cudaMemcpyToSymbol(g_check_pix, zero, sizeof(zero));
  }
}

constexpr int kPixThreads = 256;

__device__ __forceinline__ int clamp255(int v) { return v < 0 ? 0 : (v > 255 ? 255 : v); }

// Per-image source accessor over the decoded crop-window planes.
struct PlaneSrc {
  const uint8_t *p[3];
  int pitch[3];
  int oy[3], ox[3];  // window origin in component samples
  int h[3], v[3];
  int lh, lv, ncomp;  // log2(hmax), log2(vmax): sampling factors are 1, 2 or 4
  __device__ __forceinline__ void load(const ImgInfo &I, const uint8_t *plane) {
    ncomp = I.ncomp;
    lh = I.hmax == 4 ? 2 : I.hmax - 1;
    lv = I.vmax == 4 ? 2 : I.vmax - 1;
#pragma unroll
    for (int c = 0; c < 3; c++) {
      p[c] = plane + I.plane_off[c];
      pitch[c] = I.plane_pitch[c];
      oy[c] = I.wby0[c] * 8;
      ox[c] = I.wbx0[c] * 8;
      h[c] = I.comp_h[c];
      v[c] = I.comp_v[c];
    }
  }
  // RGB of image pixel (sy, sx): replication upsampling + fixed-point
  // YCbCr->RGB (decode_kernels.py:551-576), gray replicated (579-589).
  __device__ __forceinline__ void rgb(int sy, int sx, int &r, int &g, int &b) const {
    int ro[3], co[3];
    row_off(sy, ro);
    col_off(sx, co);
    rgb_at(ro, co, r, g, b);
  }
  // sy * v / vmax and sx * h / hmax with vmax, hmax powers of two
  // (decode_kernels.py:551-558), split into a row part and a column part
  __device__ __forceinline__ void row_off(int sy, int ro[3]) const {
#pragma unroll
    for (int c = 0; c < 3; c++) ro[c] = (((sy * v[c]) >> lv) - oy[c]) * pitch[c];
  }
  __device__ __forceinline__ void col_off(int sx, int co[3]) const {
#pragma unroll
    for (int c = 0; c < 3; c++) co[c] = ((sx * h[c]) >> lh) - ox[c];
  }
  __device__ __forceinline__ void rgb_at(const int ro[3], const int co[3], int &r, int &g,
                                         int &b) const {
    const int yv = p[0][ro[0] + co[0]];
    if (ncomp == 1) {
      r = g = b = yv;
      return;
    }
    const int cb = (int)p[1][ro[1] + co[1]] - 128;
    const int cr = (int)p[2][ro[2] + co[2]] - 128;
    r = clamp255(yv + ((91881 * cr + 32768) >> 16));
    g = clamp255(yv + ((-22554 * cb - 46802 * cr + 32768) >> 16));
    b = clamp255(yv + ((116130 * cb + 32768) >> 16));
  }
};

// Bilinear tap geometry for one output coordinate (imgops.py:33-53).
__device__ __forceinline__ void tap(int o, double scale, int in, int &i0, int &i1, double &w) {
  double f = __dsub_rn(__dmul_rn((double)o + 0.5, scale), 0.5);
  if (f < 0.0) f = 0.0;
  i0 = __double2int_rz(f);
  if (i0 > in - 1) i0 = in - 1;
  i1 = i0 + 1;
  if (i1 > in - 1) i1 = in - 1;
  w = __dsub_rn(f, (double)i0);
}

__device__ __forceinline__ int bilerp2(double wx, double wy, double ax, double ay, int s00, int s01,
                                       int s10, int s11) {
  const double top = __dadd_rn(__dmul_rn(ax, (double)s00), __dmul_rn(wx, (double)s01));
  const double bot = __dadd_rn(__dmul_rn(ax, (double)s10), __dmul_rn(wx, (double)s11));
  const double v = __dadd_rn(__dadd_rn(__dmul_rn(ay, top), __dmul_rn(wy, bot)), 0.5);
  const int iv = __double2int_rz(v);
  return iv > 255 ? 255 : iv;
}

// imgops.py:49-57 for one channel: weights' complements 1 - w as in the reference.
__device__ __forceinline__ int bilerp(double wx, double wy, int s00, int s01, int s10, int s11) {
  return bilerp2(wx, wy, __dsub_rn(1.0, wx), __dsub_rn(1.0, wy), s00, s01, s10, s11);
}

__device__ __forceinline__ int luma601(int r, int g, int b) {  // imgops.py:78-81
  return (19595 * r + 38470 * g + 7471 * b + 32768) >> 16;
}

// imgops.py:231-240: (f32(v) * f32(1/255) - mean) / std, IEEE float32.
__device__ __forceinline__ float norm_value(int c, int v) {
  const float inv255 = __fdiv_rn(1.0f, 255.0f);
  const float mean = c == 0 ? 0.485f : (c == 1 ? 0.456f : 0.406f);
  const float sd = c == 0 ? 0.229f : (c == 1 ? 0.224f : 0.225f);
  return __fdiv_rn(__fsub_rn(__fmul_rn((float)v, inv255), mean), sd);
}

// k_resize: one CTA per band of P.band (<= kMaxBandRows) output rows of one
// image, 256 threads.
//  1. the source rows the band's bilinear taps touch are colour-converted
//     once into shared memory (RGBX words, coalesced plane reads; crops too
//     wide for the shared budget read the planes directly instead);
//  2. the column taps (x0, x1, 4096*wx; flip folded in) are tabulated once per
//     CTA in shared memory, the band's row taps likewise;
//  3. a thread owns kCols = 8 consecutive output columns of a contiguous
//     chunk of the band's rows: per source row the 8x3 horizontal
//     interpolations stay in registers while consecutive output rows share
//     the row; per output row it produces 8 pixels, normalizes them through a
//     256-entry LUT of the exact fp32 value and writes one 128-bit store per
//     channel (8 bf16; two for f32), plus optionally the uint8 NHWC view and
//     the MAE visible tokens of the pixel's patch.
// grid: (ceil(res / P.band), n); dynamic smem: P.src_words source words +
// res column taps.
constexpr int kResizeMaxDyn = 200 * 1024;

// The exact fp32 normalize value of every (channel, uint8) and its bf16 RNE,
// computed once per device (init_device_pixels) with the same IEEE ops.
__device__ float g_norm_lut[768];
__device__ __nv_bfloat16 g_norm_lutb[768];

__global__ void k_init_norm_luts() {
  const int i = threadIdx.x;
  const float f = norm_value(i >> 8, i & 255);
  g_norm_lut[i] = f;
  g_norm_lutb[i] = __float2bfloat16_rn(f);
}

struct __align__(8) ColTap {
  uint16_t x0, x1;  // source columns of the tap (crop-relative)
  float wxk;        // float32(wx) * 4096
};

// Source rows [ys0, ys0 + nrows) of the crop -> RGBX words src[r * iw + x].
__device__ __forceinline__ void stage_rows(const ImgInfo &I, const PlaneSrc &S, int ys0, int nrows,
                                           uint32_t *src, int src_words) {
  (void)src_words;
  const int iw = I.rw;
  // Fast path (luma at full horizontal resolution, chroma at full or half:
  // 4:2:0, 4:2:2, 4:4:4, gray): work items are (row, group of 4 image
  // columns aligned to 4), so the luma plane is read 4 bytes at a time and
  // half-resolution chroma 2 bytes at a time (planes are MCU-aligned windows:
  // a group never leaves them), and each chroma sample's colour terms are
  // computed once for the two pixels that replicate it (decode_kernels.py:
  // 551-576: R = Y + (91881 Cr + 32768) >> 16, G = Y + (-22554 Cb - 46802 Cr
  // + 32768) >> 16, B = Y + (116130 Cb + 32768) >> 16, clamped).
  const bool fast = I.comp_h[0] == I.hmax &&
                    (I.ncomp == 1 || ((2 * I.comp_h[1] == I.hmax || I.comp_h[1] == I.hmax) &&
                                      (2 * I.comp_h[2] == I.hmax || I.comp_h[2] == I.hmax)));
  if (fast) {
    const int g0 = I.rx >> 2, ng = ((I.rx + iw + 3) >> 2) - g0;
    const bool half1 = I.ncomp == 3 && 2 * I.comp_h[1] == I.hmax;
    const bool half2 = I.ncomp == 3 && 2 * I.comp_h[2] == I.hmax;
    // a thread keeps one group of 4 columns (its column offsets fixed) and
    // walks rows rpp apart: no per-item division or column arithmetic
    const int cpr = ng < kPixThreads ? ng : kPixThreads;  // groups per pass
    const int rpp = kPixThreads / cpr;                    // rows per pass
    const int rt = threadIdx.x / cpr, gt = threadIdx.x - rt * cpr;
    for (int Gi = gt; rt < rpp && Gi < ng; Gi += cpr)
    for (int r = rt; r < nrows; r += rpp) {
      const int G = g0 + Gi;
      int ro[3];
      S.row_off(I.ry + ys0 + r, ro);
      const uint32_t y4 = *reinterpret_cast<const uint32_t *>(S.p[0] + ro[0] + 4 * G - S.ox[0]);
      uint32_t w[4];
      if (I.ncomp == 1) {
#pragma unroll
        for (int i = 0; i < 4; i++) w[i] = ((y4 >> (8 * i)) & 255u) * 0x010101u;
      } else {
        // chroma bytes of the group's 4 pixels (replicated when half resolution)
        uint32_t cb4, cr4;
        if (half1) {
          const uint32_t t = *reinterpret_cast<const uint16_t *>(S.p[1] + ro[1] + 2 * G - S.ox[1]);
          cb4 = __byte_perm(t, 0, 0x1100);
        } else {
          cb4 = *reinterpret_cast<const uint32_t *>(S.p[1] + ro[1] + 4 * G - S.ox[1]);
        }
        if (half2) {
          const uint32_t t = *reinterpret_cast<const uint16_t *>(S.p[2] + ro[2] + 2 * G - S.ox[2]);
          cr4 = __byte_perm(t, 0, 0x1100);
        } else {
          cr4 = *reinterpret_cast<const uint32_t *>(S.p[2] + ro[2] + 4 * G - S.ox[2]);
        }
        // colour terms per distinct chroma pair (pixels 2k, 2k+1 share one
        // when both chroma planes are half resolution)
        int dr[4], dg[4], db[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          if (i & 1 && half1 && half2) {
            dr[i] = dr[i - 1]; dg[i] = dg[i - 1]; db[i] = db[i - 1];
            continue;
          }
          const int cb = (int)((cb4 >> (8 * i)) & 255u) - 128;
          const int cr = (int)((cr4 >> (8 * i)) & 255u) - 128;
          dr[i] = (91881 * cr + 32768) >> 16;
          dg[i] = (-22554 * cb - 46802 * cr + 32768) >> 16;
          db[i] = (116130 * cb + 32768) >> 16;
        }
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int yv = (int)((y4 >> (8 * i)) & 255u);
          w[i] = (uint32_t)clamp255(yv + dr[i]) | ((uint32_t)clamp255(yv + dg[i]) << 8) |
                 ((uint32_t)clamp255(yv + db[i]) << 16);
        }
      }
      const int x = 4 * G - I.rx;
      uint32_t *row = src + r * iw;
      ESSL_CHECK(g_check_pix, (r + 1) * iw <= src_words, CK_SRC);
#pragma unroll
      for (int i = 0; i < 4; i++)
        if ((unsigned)(x + i) < (unsigned)iw) row[x + i] = w[i];
    }
  } else {
    // generic sampling factors: each thread keeps one column (its plane
    // column offsets fixed) and walks rows, four in flight; no per-pixel
    // division.
    const int cpr = iw < kPixThreads ? iw : kPixThreads;      // columns per pass
    const int rpp = iw < kPixThreads ? kPixThreads / iw : 1;  // rows per pass
    const int r0 = threadIdx.x / cpr, x0 = threadIdx.x - r0 * cpr;
    if (r0 < rpp) {
      for (int x = x0; x < iw; x += cpr) {
        int co[3];
        S.col_off(I.rx + x, co);
        for (int r = r0; r < nrows; r += 4 * rpp) {
          int rr[4], gg[4], bb[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            int ro[3];
            S.row_off(I.ry + ys0 + min(r + u * rpp, nrows - 1), ro);
            S.rgb_at(ro, co, rr[u], gg[u], bb[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; u++)
            if (r + u * rpp < nrows)
              src[(r + u * rpp) * iw + x] = (uint32_t)rr[u] | ((uint32_t)gg[u] << 8) | ((uint32_t)bb[u] << 16);
        }
      }
    }
  }
}

// RGBX word of crop pixel (y, x) straight from the planes (crops whose
// source rows do not fit the shared budget).
__device__ __forceinline__ uint32_t plane_rgbx(const ImgInfo &I, const PlaneSrc &S, int y, int x) {
  int r, g, b;
  S.rgb(I.ry + y, I.rx + x, r, g, b);
  return (uint32_t)r | ((uint32_t)g << 8) | ((uint32_t)b << 16);
}

// PLAIN: no 3-Aug, no uint8 view, no visible tokens -- each channel's 8
// values are finished (and stored) on their own, which keeps the register
// footprint at the two rows of interpolated values.
// W consecutive 32-bit words to global memory as one vector store
// (W = 4: 128-bit, 2: 64-bit, 1: 32-bit); CS: streaming (evict-first).
template <int W, bool CS = true>
__device__ __forceinline__ void st_words(void *p, const uint32_t *w) {
  if constexpr (W == 4) {
    const uint4 v = make_uint4(w[0], w[1], w[2], w[3]);
    if (CS) __stcs(reinterpret_cast<uint4 *>(p), v); else *reinterpret_cast<uint4 *>(p) = v;
  } else if constexpr (W == 2) {
    const uint2 v = make_uint2(w[0], w[1]);
    if (CS) __stcs(reinterpret_cast<uint2 *>(p), v); else *reinterpret_cast<uint2 *>(p) = v;
  } else {
    if (CS) __stcs(reinterpret_cast<unsigned int *>(p), w[0]); else *reinterpret_cast<uint32_t *>(p) = w[0];
  }
}

// The exact float64 value of channel c of output pixel (row pair yy, column
// ox) -- the ambiguous case of the float32 evaluation (imgops.py:49-56).
template <bool STAGED>
__device__ __noinline__ int exact_value(const ImgInfo &I, const PlaneSrc &S, const uint32_t *src,
                                        int iw, int ys0, int2 yy, int ox, int res, double sx,
                                        double wy, int c) {
  int tx0, tx1;
  double wx;
  tap(I.flip ? res - 1 - ox : ox, sx, iw, tx0, tx1, wx);
  uint32_t a00, a01, a10, a11;
  if (STAGED) {
    a00 = src[yy.x * iw + tx0]; a01 = src[yy.x * iw + tx1];
    a10 = src[yy.y * iw + tx0]; a11 = src[yy.y * iw + tx1];
  } else {
    a00 = plane_rgbx(I, S, ys0 + yy.x, tx0); a01 = plane_rgbx(I, S, ys0 + yy.x, tx1);
    a10 = plane_rgbx(I, S, ys0 + yy.y, tx0); a11 = plane_rgbx(I, S, ys0 + yy.y, tx1);
  }
  return bilerp2(wx, wy, __dsub_rn(1.0, wx), __dsub_rn(1.0, wy), (a00 >> (8 * c)) & 255,
                 (a01 >> (8 * c)) & 255, (a10 >> (8 * c)) & 255, (a11 >> (8 * c)) & 255);
}

template <bool AUG, bool STAGED, bool PLAIN, int COLS>
__global__ void __launch_bounds__(kPixThreads, COLS == 8 ? 2 : (COLS == 4 ? 3 : 4)) k_resize(PixelParams P) {
  TraceScope trace_(P.trace, ESSL_K_RESIZE);
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ float lut[3][256];
  __shared__ __nv_bfloat16 lutb[3][256];
  __shared__ double s_scale[2];
  __shared__ int2 ry[kMaxBandRows];
  __shared__ double rw[kMaxBandRows];
  __shared__ float rwf[kMaxBandRows];
  const int img = blockIdx.y;
  const ImgInfo &I = P.info[img];
  if (I.status != 0) return;
  const int res = P.res;
  // 3-Aug (pipeline.py:88-101): point ops are finished here, blur / jitter
  // images leave their uint8 resize to k_aug_blur / k_aug_out
  int out_kind = P.out_kind, aop = ESSL_AUG_OP_NONE, athr = 0;
  uint8_t *out_u8 = P.out_u8;
  bool vis = P.vis != nullptr;
  if (AUG) {
    const essl_aug &A = P.aug[img];
    if (A.op == ESSL_AUG_OP_BLUR || A.jitter) {
      out_kind = ESSL_OUT_NONE;
      out_u8 = P.aug_u8;
      vis = false;
    } else {
      aop = A.op;
      athr = A.threshold;
    }
  }
  const int ih = I.rh, iw = I.rw;
  if (out_kind == ESSL_OUT_F32_NCHW)
    for (int i = threadIdx.x; i < 768; i += kPixThreads) lut[i >> 8][i & 255] = g_norm_lut[i];
  if (out_kind == ESSL_OUT_BF16_NCHW || vis)
    for (int i = threadIdx.x; i < 768; i += kPixThreads) lutb[i >> 8][i & 255] = g_norm_lutb[i];
  if (threadIdx.x == 0) {  // imgops.py:35-36 scale factors, once per CTA
    s_scale[0] = __ddiv_rn((double)ih, (double)res);
    s_scale[1] = __ddiv_rn((double)iw, (double)res);
  }
  __syncthreads();
  const int ob0 = blockIdx.x * P.band;
  const int ob1 = min(ob0 + P.band, res);
  const double sy = s_scale[0], sx = s_scale[1];
  // source rows of the band (taps are monotone in the output row)
  int ys0, ys1, dummy;
  double wdum;
  tap(ob0, sy, ih, ys0, dummy, wdum);
  tap(ob1 - 1, sy, ih, dummy, ys1, wdum);
  const int nrows = ys1 - ys0 + 1;
  uint32_t *src = reinterpret_cast<uint32_t *>(dyn);  // [nrows][iw] (STAGED)
  ColTap *ctab = reinterpret_cast<ColTap *>(dyn + (size_t)P.src_words * 4);
  PlaneSrc S;
  S.load(I, P.plane);
  if (STAGED) stage_rows(I, S, ys0, nrows, src, P.src_words);
  // column taps (imgops.py:42-47; hflip after resize: output column ox reads
  // the resize's column res-1-ox) and the band's row taps (imgops.py:37-41)
  for (int ox = threadIdx.x; ox < res; ox += kPixThreads) {
    int x0, x1;
    double wx;
    tap(I.flip ? res - 1 - ox : ox, sx, iw, x0, x1, wx);
    ColTap t;
    t.x0 = (uint16_t)x0;
    t.x1 = (uint16_t)x1;
    t.wxk = __fmul_rn(__double2float_rn(wx), 4096.0f);
    ctab[ox] = t;
  }
  if (threadIdx.x < ob1 - ob0) {
    int y0, y1;
    double wy;
    tap(ob0 + threadIdx.x, sy, ih, y0, y1, wy);
    ry[threadIdx.x] = make_int2(y0 - ys0, y1 - ys0);
    rw[threadIdx.x] = wy;
    rwf[threadIdx.x] = __double2float_rn(wy);
  }
  __syncthreads();
  // Separable evaluation.  The reference value is float64 (imgops.py:49-56):
  //   v = (1-wy)*((1-wx)*s00 + wx*s01) + wy*((1-wx)*s10 + wx*s11) + 0.5,
  //   px = int(v) (v <= 255.5, so the min(., 255) never binds).
  // It is evaluated here in float32, scaled by 4096 (exact for integer
  // samples): T = 4096*s0 + 2048 + (4096*wx)*(s1 - s0) per source row (one
  // fma, kept in registers while consecutive output rows share the row),
  // V = T0 + wy*(T1 - T0).  Float32 error, in those units: wx, wy rounded to
  // float32 (<= 2^-24 * 255 * 4096 = 0.0625 each), four roundings at
  // magnitude < 2^20 (<= 0.03125 each): |V - 4096*v| < 0.25.  With
  // x = round(V), |x - 4096*v| < 0.75, so x mod 4096 in [1, 4094] proves
  // int(v) == x >> 12.  Otherwise (x within one unit of a multiple of 4096:
  // ~0.05% of channels, more with dyadic weights giving integral values) the
  // pixel is recomputed with the reference's float64 expression (exact_px).
  //   x + 1 = bits(V + 1.5*2^23 + 1) - 0x4B400000  (round to nearest through
  //   the magic constant; V + 1.5*2^23 + 1 < 2^24 keeps unit spacing).
  const int ngrp = (res + COLS - 1) / COLS;
  const int band_rows = ob1 - ob0;
  // slices of rows: thread (group g, slice s) owns rows [r0, r1) of the band
  const int nsl = ngrp >= kPixThreads ? 1 : min(kPixThreads / ngrp, band_rows);
  const int sl = ngrp >= kPixThreads ? 0 : threadIdx.x / ngrp;
  if (sl >= nsl) return;
  const int r0 = sl * band_rows / nsl, r1 = (sl + 1) * band_rows / nsl;
  const int64_t plane_sz = (int64_t)res * res;
  const int64_t stride = P.out_stride ? P.out_stride : 3 * plane_sz;
  // 128-bit stores need every (image, plane, row, group) start 16-byte aligned
  const int esz = out_kind == ESSL_OUT_F32_NCHW ? 4 : 2;
  constexpr int va = COLS * 2 > 16 ? 16 : COLS * 2;  // bf16 store width
  const int al = out_kind == ESSL_OUT_F32_NCHW ? (COLS == 2 ? 8 : 16) : va;
  const bool vec = (res % COLS) == 0 && ((stride * esz) % al) == 0 &&
                   ((reinterpret_cast<uintptr_t>(P.out) % al) == 0);
  const bool vec_u8 = COLS >= 4 && (res % COLS) == 0 &&
                      ((reinterpret_cast<uintptr_t>(out_u8) % (COLS >= 4 ? COLS / 2 : 1)) == 0);
  const int patch = P.patch, gp = patch > 0 ? res / patch : 0;
  const int tok_dim = patch * patch * 3;
  const bool vec_vis = patch % COLS == 0 && (reinterpret_cast<uintptr_t>(P.vis) % va) == 0;
  constexpr float kMagic1 = 12582913.0f;   // 1.5 * 2^23 + 1
  constexpr int kMagicBits = 0x4B400000;   // bits of 1.5 * 2^23
  constexpr float kByteBias = 8388608.0f;  // bits 0x4B000000 | byte == 2^23 + byte
  for (int grp = ngrp >= kPixThreads ? threadIdx.x : threadIdx.x - sl * ngrp; grp < ngrp;
       grp += ngrp >= kPixThreads ? kPixThreads : ngrp) {
    const int oxa = grp * COLS;
    const int ncol = min(COLS, res - oxa);
    // narrow groups keep their column taps in registers; 8-column groups
    // re-read them from shared memory per source row (registers go to the
    // 2 x 24 interpolated values)
    const ColTap *ct = ctab + oxa;
    ColTap treg[COLS <= 4 ? COLS : 1];
    if constexpr (COLS <= 4) {
#pragma unroll
      for (int j = 0; j < COLS; j++) treg[j] = ct[min(j, ncol - 1)];
    }
    int cy0 = -1, cy1 = -1;
    float h0[COLS][3], h1[COLS][3];
    auto hrow = [&](int y, float h[COLS][3]) {
#pragma unroll
      for (int j = 0; j < COLS; j++) {
        const ColTap t = COLS <= 4 ? treg[COLS <= 4 ? j : 0] : ct[min(j, ncol - 1)];
        const float wxkj = t.wxk;
        uint32_t a0, a1;
        if (STAGED) {
          a0 = src[y * iw + t.x0];
          a1 = src[y * iw + t.x1];
        } else {
          a0 = plane_rgbx(I, S, ys0 + y, t.x0);
          a1 = plane_rgbx(I, S, ys0 + y, t.x1);
        }
#pragma unroll
        for (int c = 0; c < 3; c++) {
          // 2^23 + byte, exactly (byte c of the RGBX word under exponent 0x4B)
          const float f0 = __uint_as_float(__byte_perm(a0, 0x4B000000u, c | 0x7540));
          const float f1 = __uint_as_float(__byte_perm(a1, 0x4B000000u, c | 0x7540));
          // 4096*s0 + 2048 (exact) + (4096*wx) * (s1 - s0), one rounding
          const float base = __fmaf_rn(f0, 4096.0f, 2048.0f - 4096.0f * kByteBias);
          h[j][c] = __fmaf_rn(wxkj, __fsub_rn(f1, f0), base);
        }
      }
    };
    for (int r = r0; r < r1; r++) {
      const int2 yy = ry[r];
      const float wy = rwf[r];
      if (yy.x != cy0) {
        if (yy.x == cy1) {
#pragma unroll
          for (int j = 0; j < COLS; j++)
#pragma unroll
            for (int c = 0; c < 3; c++) h0[j][c] = h1[j][c];
        } else {
          hrow(yy.x, h0);
        }
        cy0 = yy.x;
      }
      if (yy.y != cy1) {
        if (yy.y == cy0) {
#pragma unroll
          for (int j = 0; j < COLS; j++)
#pragma unroll
            for (int c = 0; c < 3; c++) h1[j][c] = h0[j][c];
        } else {
          hrow(yy.y, h1);
        }
        cy1 = yy.y;
      }
      const int oy = ob0 + r;
      const int64_t o = img * stride + (int64_t)oy * res + oxa;
      const bool full = ncol == COLS;
      if (PLAIN) {
#pragma unroll
        for (int c = 0; c < 3; c++) {
          int pc[COLS];
          int amb = 4095;
#pragma unroll
          for (int j = 0; j < COLS; j++) {
            const float v = __fmaf_rn(wy, __fsub_rn(h1[j][c], h0[j][c]), h0[j][c]);
            const int y1 = __float_as_int(__fadd_rn(v, kMagic1)) - kMagicBits;  // round(v) + 1
            amb = min(amb, y1 & 4094);  // 0: round(v) mod 4096 in {4095, 0}
            pc[j] = y1 >> 12;           // == round(v) >> 12 when not ambiguous
          }
          if (amb == 0) {  // rare: the exact float64 expression for the ambiguous values
#pragma unroll
            for (int j = 0; j < COLS; j++) {
              const float v = __fmaf_rn(wy, __fsub_rn(h1[j][c], h0[j][c]), h0[j][c]);
              if (((__float_as_int(__fadd_rn(v, kMagic1)) - kMagicBits) & 4094) == 0)
                pc[j] = exact_value<STAGED>(I, S, src, iw, ys0, yy, oxa + min(j, ncol - 1), res, sx, rw[r], c);
            }
          }
          if (out_kind == ESSL_OUT_BF16_NCHW) {
            __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(P.out) + o + c * plane_sz;
            if (vec) {
              uint32_t w[COLS / 2];
#pragma unroll
              for (int q = 0; q < COLS / 2; q++)
                w[q] = (uint32_t)__bfloat16_as_ushort(lutb[c][pc[2 * q]]) |
                       ((uint32_t)__bfloat16_as_ushort(lutb[c][pc[2 * q + 1]]) << 16);
              // streaming store: the model's input is not re-read here; keep L2
              // for the unit lists / planes of the batches in flight
              st_words<COLS / 2>(out, w);
            } else {
#pragma unroll
              for (int j = 0; j < COLS; j++)
                if (j < ncol) out[j] = lutb[c][pc[j]];
            }
          } else if (out_kind == ESSL_OUT_F32_NCHW) {
            float *out = reinterpret_cast<float *>(P.out) + o + c * plane_sz;
            if (vec) {
              if constexpr (COLS == 2) {
                __stcs(reinterpret_cast<float2 *>(out), make_float2(lut[c][pc[0]], lut[c][pc[1]]));
              } else {
#pragma unroll
                for (int q = 0; q < COLS / 4; q++)
                  __stcs(reinterpret_cast<float4 *>(out) + q,
                         make_float4(lut[c][pc[4 * q]], lut[c][pc[4 * q + 1]], lut[c][pc[4 * q + 2]],
                                     lut[c][pc[4 * q + 3]]));
              }
            } else {
#pragma unroll
              for (int j = 0; j < COLS; j++)
                if (j < ncol) out[j] = lut[c][pc[j]];
            }
          }
        }
        continue;
      }
      int px[COLS][3];
      int amb = 4095;
#pragma unroll
      for (int j = 0; j < COLS; j++)
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const float v = __fmaf_rn(wy, __fsub_rn(h1[j][c], h0[j][c]), h0[j][c]);
          const int y1 = __float_as_int(__fadd_rn(v, kMagic1)) - kMagicBits;  // round(v) + 1
          amb = min(amb, y1 & 4094);  // 0: round(v) mod 4096 in {4095, 0}
          px[j][c] = y1 >> 12;        // == round(v) >> 12 when not ambiguous
        }
      if (amb == 0) {  // rare: the exact float64 expression for the ambiguous pixels
#pragma unroll
        for (int j = 0; j < COLS; j++) {
          bool a = false;
#pragma unroll
          for (int c = 0; c < 3; c++) {
            const float v = __fmaf_rn(wy, __fsub_rn(h1[j][c], h0[j][c]), h0[j][c]);
            a |= ((__float_as_int(__fadd_rn(v, kMagic1)) - kMagicBits) & 4094) == 0;
          }
          if (a) {
#pragma unroll
            for (int c = 0; c < 3; c++)
              px[j][c] = exact_value<STAGED>(I, S, src, iw, ys0, yy, oxa + min(j, ncol - 1), res, sx,
                                             rw[r], c);
          }
        }
      }
      if (AUG && aop == ESSL_AUG_OP_GRAY) {  // imgops.py:75-91
#pragma unroll
        for (int j = 0; j < COLS; j++) px[j][0] = px[j][1] = px[j][2] = luma601(px[j][0], px[j][1], px[j][2]);
      } else if (AUG && aop == ESSL_AUG_OP_SOLARIZE) {  // imgops.py:94-108
#pragma unroll
        for (int j = 0; j < COLS; j++)
#pragma unroll
          for (int c = 0; c < 3; c++) px[j][c] = px[j][c] >= athr ? 255 - px[j][c] : px[j][c];
      }
      if (out_kind == ESSL_OUT_BF16_NCHW) {
        __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(P.out) + o;
        if (vec) {
#pragma unroll
          for (int c = 0; c < 3; c++) {
            uint32_t w[COLS / 2];
#pragma unroll
            for (int q = 0; q < COLS / 2; q++)
              w[q] = (uint32_t)__bfloat16_as_ushort(lutb[c][px[2 * q][c]]) |
                     ((uint32_t)__bfloat16_as_ushort(lutb[c][px[2 * q + 1][c]]) << 16);
            st_words<COLS / 2>(out + c * plane_sz, w);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 3; c++)
#pragma unroll
            for (int j = 0; j < COLS; j++)
              if (j < ncol) out[c * plane_sz + j] = lutb[c][px[j][c]];
        }
      } else if (out_kind == ESSL_OUT_F32_NCHW) {
        float *out = reinterpret_cast<float *>(P.out) + o;
        if (vec) {
#pragma unroll
          for (int c = 0; c < 3; c++) {
            if constexpr (COLS == 2) {
              __stcs(reinterpret_cast<float2 *>(out + c * plane_sz),
                     make_float2(lut[c][px[0][c]], lut[c][px[1][c]]));
            } else {
#pragma unroll
              for (int q = 0; q < COLS / 4; q++)
                __stcs(reinterpret_cast<float4 *>(out + c * plane_sz) + q,
                       make_float4(lut[c][px[4 * q][c]], lut[c][px[4 * q + 1][c]],
                                   lut[c][px[4 * q + 2][c]], lut[c][px[4 * q + 3][c]]));
            }
          }
        } else {
#pragma unroll
          for (int c = 0; c < 3; c++)
#pragma unroll
            for (int j = 0; j < COLS; j++)
              if (j < ncol) out[c * plane_sz + j] = lut[c][px[j][c]];
        }
      }
      if (out_u8) {
        uint8_t *out = out_u8 + (int64_t)img * plane_sz * 3 + ((int64_t)oy * res + oxa) * 3;
        if (vec_u8 && full) {
          constexpr int nw = COLS >= 4 ? 3 * COLS / 4 : 1;
          uint32_t w[nw];
#pragma unroll
          for (int q = 0; q < (COLS >= 4 ? nw : 0); q++) {
            uint32_t v = 0;
#pragma unroll
            for (int b = 0; b < 4; b++) v |= (uint32_t)px[(4 * q + b) / 3][(4 * q + b) % 3] << (8 * b);
            w[q] = v;
          }
#pragma unroll
          for (int q = 0; q < (COLS >= 4 ? 3 : 0); q++)
            st_words<COLS >= 4 ? COLS / 4 : 1, false>(out + COLS * q, w + (COLS / 4) * q);
        } else {
#pragma unroll
          for (int j = 0; j < COLS; j++)
            if (j < ncol)
#pragma unroll
              for (int c = 0; c < 3; c++) out[3 * j + c] = (uint8_t)px[j][c];
        }
      }
      if (vis && patch > 0) {
        // MAE visible tokens (patchify 'nchpwq->nhwpqc'): the
        // pixel's patch is visible when ids_restore maps it below n_keep;
        // its token row holds (q, c) pairs of patch row oy % patch
        __nv_bfloat16 *tok = reinterpret_cast<__nv_bfloat16 *>(P.vis);
        const int64_t *rest = P.vis_restore + (int64_t)img * gp * gp;
        if (vec_vis && full) {
          const int id = (oy / patch) * gp + oxa / patch;
          const int64_t rk = rest[id];
          if (rk < P.n_keep) {
            __nv_bfloat16 *t = tok + ((int64_t)img * P.n_keep + rk) * tok_dim +
                               ((oy % patch) * patch + oxa % patch) * 3;
            uint32_t w[3 * COLS / 2];
#pragma unroll
            for (int q = 0; q < 3 * COLS / 2; q++) {
              const int e0 = 2 * q, e1 = 2 * q + 1;
              w[q] = (uint32_t)__bfloat16_as_ushort(lutb[e0 % 3][px[e0 / 3][e0 % 3]]) |
                     ((uint32_t)__bfloat16_as_ushort(lutb[e1 % 3][px[e1 / 3][e1 % 3]]) << 16);
            }
#pragma unroll
            for (int q = 0; q < 3; q++) st_words<COLS / 2>(t + COLS * q, w + (COLS / 2) * q);
          }
        } else {
#pragma unroll
          for (int j = 0; j < COLS; j++) {
            if (j >= ncol) continue;
            const int ox = oxa + j;
            const int64_t rk = rest[(oy / patch) * gp + ox / patch];
            if (rk >= P.n_keep) continue;
            __nv_bfloat16 *t = tok + ((int64_t)img * P.n_keep + rk) * tok_dim +
                               ((oy % patch) * patch + ox % patch) * 3;
#pragma unroll
            for (int c = 0; c < 3; c++) t[c] = lutb[c][px[j][c]];
          }
        }
      }
    }
  }
}

constexpr int kPairBandRows = 32;

// k_resize_pairs: the round-1 shape, and the fastest measured in the
// multi-stream pipeline (A/B on B200, cfg2: 975k img/s vs 937k for the
// template kernel at 2 columns and 925k at 4 / 852k at 8 columns with
// 128-bit stores): a thread owns a PAIR of output columns (paired 32-bit bf16
// / 64-bit f32 stores) of half a 32-row band, its two column taps in
// registers.  Used for staged batches without visible tokens; everything
// else takes k_resize.
// RES > 0: the output resolution fixed at compile time (224, the pretraining
// resolution and the bench's, and the progressive stages 112 / 160 / 192):
// plane / row offsets and the thread layout fold into constants (fewer live
// registers, fewer rematerialised values; +2.1% cfg2).
template <bool AUG, int RES = 0>
__global__ void __launch_bounds__(kPixThreads, 4) k_resize_pairs(PixelParams P) {
  TraceScope trace_(P.trace, ESSL_K_RESIZE);
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ float lut[3][256];
  __shared__ __nv_bfloat16 lutb[3][256];
  __shared__ double s_scale[2];
  const int img = blockIdx.y;
  const ImgInfo &I = P.info[img];
  if (I.status != 0) return;
  const int res = RES > 0 ? RES : P.res;
  // 3-Aug (pipeline.py:88-101): point ops are finished here, blur / jitter
  // images leave their uint8 resize to k_aug_blur / k_aug_out
  int out_kind = P.out_kind, aop = ESSL_AUG_OP_NONE, athr = 0;
  uint8_t *out_u8 = P.out_u8;
  if (AUG) {
    const essl_aug &A = P.aug[img];
    if (A.op == ESSL_AUG_OP_BLUR || A.jitter) {
      out_kind = ESSL_OUT_NONE;
      out_u8 = P.aug_u8;
    } else {
      aop = A.op;
      athr = A.threshold;
    }
  }
  const int ih = I.rh, iw = I.rw;
  if (P.out_kind == ESSL_OUT_F32_NCHW)
    for (int i = threadIdx.x; i < 768; i += kPixThreads) lut[i >> 8][i & 255] = g_norm_lut[i];
  else
    for (int i = threadIdx.x; i < 768; i += kPixThreads) lutb[i >> 8][i & 255] = g_norm_lutb[i];
  if (threadIdx.x == 0) {  // imgops.py:35-36 scale factors, once per CTA
    s_scale[0] = __ddiv_rn((double)ih, (double)res);
    s_scale[1] = __ddiv_rn((double)iw, (double)res);
  }
  __syncthreads();
  const int ob0 = blockIdx.x * P.band;
  const int ob1 = min(ob0 + P.band, res);
  const double sy = s_scale[0], sx = s_scale[1];
  // source rows of the band (taps are monotone in the output row)
  int ys0, ys1, dummy;
  double wdum;
  tap(ob0, sy, ih, ys0, dummy, wdum);
  tap(ob1 - 1, sy, ih, dummy, ys1, wdum);
  const int nrows = ys1 - ys0 + 1;
  uint32_t *src = reinterpret_cast<uint32_t *>(dyn);                         // [nrows][iw]
  PlaneSrc S;
  S.load(I, P.plane);
  // source rows -> RGBX words in shared memory (stage_rows)
  stage_rows(I, S, ys0, nrows, src, P.src_words);
  // row taps of the band (imgops.py:37-41), shared by every column
  __shared__ int2 ry[kPairBandRows];
  __shared__ double rw[kPairBandRows];
  __shared__ float rwf[kPairBandRows];
  if (threadIdx.x < ob1 - ob0) {
    int y0, y1;
    double wy;
    tap(ob0 + threadIdx.x, sy, ih, y0, y1, wy);
    ry[threadIdx.x] = make_int2(y0 - ys0, y1 - ys0);
    rw[threadIdx.x] = wy;
    rwf[threadIdx.x] = __double2float_rn(wy);
  }
  __syncthreads();
  // Separable evaluation.  The reference value is float64 (imgops.py:49-56):
  //   v = (1-wy)*((1-wx)*s00 + wx*s01) + wy*((1-wx)*s10 + wx*s11) + 0.5,
  //   px = int(v) (v <= 255.5, so the min(., 255) never binds).
  // It is evaluated here in float32, scaled by 4096 (exact for integer
  // samples): T = 4096*s0 + 2048 + (4096*wx)*(s1 - s0) per source row (one
  // fma, kept in registers while consecutive output rows share the row),
  // V = T0 + wy*(T1 - T0).  Float32 error, in those units: wx, wy rounded to
  // float32 (<= 2^-24 * 255 * 4096 = 0.0625 each), four roundings at
  // magnitude < 2^20 (<= 0.03125 each): |V - 4096*v| < 0.25.  With
  // x = round(V), |x - 4096*v| < 0.75, so x mod 4096 in [1, 4094] proves
  // int(v) == x >> 12.  Otherwise (x within one unit of a multiple of 4096:
  // ~0.05% of channels, more with dyadic weights giving integral values) the
  // pixel is recomputed with the reference's float64 expression (bilerp2).
  //   x + 1 = bits(V + 1.5*2^23 + 1) - 0x4B400000  (round to nearest through
  //   the magic constant; V + 1.5*2^23 + 1 < 2^24 keeps unit spacing).
  // A thread owns a pair of adjacent output columns (paired bf16 / f32
  // stores); small outputs split the band's rows over groups of threads.
  const int npair = (res + 1) >> 1;
  const int ng = npair >= kPixThreads ? 1 : kPixThreads / npair;
  const int g = ng > 1 ? threadIdx.x / npair : 0;
  const int cstart = ng > 1 ? threadIdx.x % npair : threadIdx.x;
  const int cstep = ng > 1 ? npair : kPixThreads;
  const int rpg = (ob1 - ob0 + ng - 1) / ng;
  const int rb = g * rpg, re = min(ob1 - ob0, rb + rpg);
  const int64_t plane_sz = (int64_t)res * res;
  const int64_t stride = P.out_stride ? P.out_stride : 3 * plane_sz;
  // paired stores need an even element offset for every (image, plane, row)
  const bool pair_ok = (res & 1) == 0 && (stride & 1) == 0 &&
                       ((reinterpret_cast<uintptr_t>(P.out) & 7) == 0);
  if (g >= ng) return;
  constexpr float kMagic1 = 12582913.0f;   // 1.5 * 2^23 + 1
  constexpr int kMagicBits = 0x4B400000;   // bits of 1.5 * 2^23
  constexpr float kByteBias = 8388608.0f;  // bits 0x4B000000 | byte == 2^23 + byte
  for (int q = cstart; q < npair; q += cstep) {
    const int oxa = 2 * q;
    const bool two = oxa + 1 < res;
    int x0[2], x1[2];
    double wx[2];
    float wxk[2];
#pragma unroll
    for (int j = 0; j < 2; j++) {
      const int ox = min(oxa + j, res - 1);
      tap(I.flip ? res - 1 - ox : ox, sx, iw, x0[j], x1[j], wx[j]);  // hflip after resize
      wxk[j] = __fmul_rn(__double2float_rn(wx[j]), 4096.0f);
    }
    int cy0 = -1, cy1 = -1;
    float h0[2][3], h1[2][3];
    auto hrow = [&](int y, float h[2][3]) {
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const uint32_t a0 = src[y * iw + x0[j]], a1 = src[y * iw + x1[j]];
#pragma unroll
        for (int c = 0; c < 3; c++) {
          // 2^23 + byte, exactly (byte c of the RGBX word under exponent 0x4B)
          const float f0 = __uint_as_float(__byte_perm(a0, 0x4B000000u, c | 0x7540));
          const float f1 = __uint_as_float(__byte_perm(a1, 0x4B000000u, c | 0x7540));
          // 4096*s0 + 2048 (exact) + (4096*wx) * (s1 - s0), one rounding
          const float base = __fmaf_rn(f0, 4096.0f, 2048.0f - 4096.0f * kByteBias);
          h[j][c] = __fmaf_rn(wxk[j], __fsub_rn(f1, f0), base);
        }
      }
    };
    for (int r = rb; r < re; r++) {
      const int2 yy = ry[r];
      const float wy = rwf[r];
      if (yy.x != cy0) {  // (uniform across the CTA's columns: no divergence)
        if (yy.x == cy1) {
#pragma unroll
          for (int j = 0; j < 2; j++)
#pragma unroll
            for (int c = 0; c < 3; c++) h0[j][c] = h1[j][c];
        } else {
          hrow(yy.x, h0);
        }
        cy0 = yy.x;
      }
      if (yy.y != cy1) {
        if (yy.y == cy0) {
#pragma unroll
          for (int j = 0; j < 2; j++)
#pragma unroll
            for (int c = 0; c < 3; c++) h1[j][c] = h0[j][c];
        } else {
          hrow(yy.y, h1);
        }
        cy1 = yy.y;
      }
      int px[2][3];
      int amb[2] = {4095, 4095};
#pragma unroll
      for (int j = 0; j < 2; j++)
#pragma unroll
        for (int c = 0; c < 3; c++) {
          const float v = __fmaf_rn(wy, __fsub_rn(h1[j][c], h0[j][c]), h0[j][c]);
          const int y1 = __float_as_int(__fadd_rn(v, kMagic1)) - kMagicBits;  // round(v) + 1
          amb[j] = min(amb[j], y1 & 4094);  // 0: round(v) mod 4096 in {4095, 0}
          px[j][c] = y1 >> 12;              // == round(v) >> 12 when not ambiguous
        }
#pragma unroll
      for (int j = 0; j < 2; j++)
        if (amb[j] == 0) {  // rare: the exact float64 expression (imgops.py:49-56)
          const double wyd = rw[r];
          const uint32_t a00 = src[yy.x * iw + x0[j]], a01 = src[yy.x * iw + x1[j]];
          const uint32_t a10 = src[yy.y * iw + x0[j]], a11 = src[yy.y * iw + x1[j]];
#pragma unroll
          for (int c = 0; c < 3; c++)
            px[j][c] = bilerp2(wx[j], wyd, __dsub_rn(1.0, wx[j]), __dsub_rn(1.0, wyd),
                               (a00 >> (8 * c)) & 255, (a01 >> (8 * c)) & 255,
                               (a10 >> (8 * c)) & 255, (a11 >> (8 * c)) & 255);
        }
      if (AUG && aop == ESSL_AUG_OP_GRAY) {  // imgops.py:75-91
#pragma unroll
        for (int j = 0; j < 2; j++) px[j][0] = px[j][1] = px[j][2] = luma601(px[j][0], px[j][1], px[j][2]);
      } else if (AUG && aop == ESSL_AUG_OP_SOLARIZE) {  // imgops.py:94-108
#pragma unroll
        for (int j = 0; j < 2; j++)
#pragma unroll
          for (int c = 0; c < 3; c++) px[j][c] = px[j][c] >= athr ? 255 - px[j][c] : px[j][c];
      }
      const int oy = ob0 + r;
      const int64_t o = img * stride + (int64_t)oy * res + oxa;
      ESSL_CHECK(g_check_pix, out_kind == ESSL_OUT_NONE || (o >= 0 && o + 2 * plane_sz + (two ? 2 : 1) <= (int64_t)P.n * stride), CK_OUT);
      if (out_kind == ESSL_OUT_BF16_NCHW) {
        __nv_bfloat16 *out = reinterpret_cast<__nv_bfloat16 *>(P.out) + o;
        if (pair_ok) {
#pragma unroll
          for (int c = 0; c < 3; c++) {
            const uint32_t lo = __bfloat16_as_ushort(lutb[c][px[0][c]]);
            const uint32_t hi = __bfloat16_as_ushort(lutb[c][px[1][c]]);
            // streaming store: the model's input is not re-read here; keep L2
            // for the unit lists / planes of the batches in flight
            __stcs(reinterpret_cast<unsigned int *>(out + c * plane_sz), lo | (hi << 16));
          }
        } else {
#pragma unroll
          for (int c = 0; c < 3; c++) {
            out[c * plane_sz] = lutb[c][px[0][c]];
            if (two) out[c * plane_sz + 1] = lutb[c][px[1][c]];
          }
        }
      } else if (out_kind == ESSL_OUT_F32_NCHW) {
        float *out = reinterpret_cast<float *>(P.out) + o;
        if (pair_ok) {
#pragma unroll
          for (int c = 0; c < 3; c++)
            __stcs(reinterpret_cast<float2 *>(out + c * plane_sz), make_float2(lut[c][px[0][c]], lut[c][px[1][c]]));
        } else {
#pragma unroll
          for (int c = 0; c < 3; c++) {
            out[c * plane_sz] = lut[c][px[0][c]];
            if (two) out[c * plane_sz + 1] = lut[c][px[1][c]];
          }
        }
      }
      if (out_u8) {
        uint8_t *out = out_u8 + (int64_t)img * plane_sz * 3 + ((int64_t)oy * res + oxa) * 3;
#pragma unroll
        for (int c = 0; c < 3; c++) out[c] = (uint8_t)px[0][c];
        if (two)
#pragma unroll
          for (int c = 0; c < 3; c++) out[3 + c] = (uint8_t)px[1][c];
      }
    }
  }
}

// Source rows a band of `band` output rows can touch for a crop of height
// h resized to res (taps y0..y1 of rows ob0..ob0+band-1, imgops.py:33-41).
int band_source_rows(int h, int res, int band) {
  return (int)(((int64_t)band * h + res - 1) / res) + 3;
}

size_t resize_smem(const PixelParams &p) {
  return (size_t)p.src_words * 4 + (size_t)p.res * sizeof(ColTap);
}

template <int COLS>
void launch_resize_cols(const PixelParams &p, dim3 grid, size_t dyn, bool staged, bool plain,
                        cudaStream_t st) {
  if (p.aug) {
    if (staged) k_resize<true, true, false, COLS><<<grid, kPixThreads, dyn, st>>>(p);
    else k_resize<true, false, false, COLS><<<grid, kPixThreads, dyn, st>>>(p);
  } else if (plain) {
    if (staged) k_resize<false, true, true, COLS><<<grid, kPixThreads, dyn, st>>>(p);
    else k_resize<false, false, true, COLS><<<grid, kPixThreads, dyn, st>>>(p);
  } else {
    if (staged) k_resize<false, true, false, COLS><<<grid, kPixThreads, dyn, st>>>(p);
    else k_resize<false, false, false, COLS><<<grid, kPixThreads, dyn, st>>>(p);
  }
}

template <int COLS>
void resize_attrs() {
  for (auto f : {k_resize<false, true, true, COLS>, k_resize<false, false, true, COLS>,
                 k_resize<false, true, false, COLS>, k_resize<false, false, false, COLS>,
                 k_resize<true, true, false, COLS>, k_resize<true, false, false, COLS>})
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kResizeMaxDyn);
}

void launch_resize(const PixelParams &p, cudaStream_t st) {
  if (p.n <= 0) return;
  const size_t dyn = resize_smem(p);
  dim3 grid((p.res + p.band - 1) / p.band, p.n);
  const bool staged = p.src_words > 0;
  const bool plain = !p.aug && !p.out_u8 && !p.vis;
  if (p.cols == 2 && staged && !p.vis && p.band <= kPairBandRows) {
    if (p.aug) k_resize_pairs<true><<<grid, kPixThreads, (size_t)p.src_words * 4, st>>>(p);
    else if (p.res == 224) k_resize_pairs<false, 224><<<grid, kPixThreads, (size_t)p.src_words * 4, st>>>(p);
    else if (p.res == 192) k_resize_pairs<false, 192><<<grid, kPixThreads, (size_t)p.src_words * 4, st>>>(p);
    else if (p.res == 160) k_resize_pairs<false, 160><<<grid, kPixThreads, (size_t)p.src_words * 4, st>>>(p);
    else if (p.res == 112) k_resize_pairs<false, 112><<<grid, kPixThreads, (size_t)p.src_words * 4, st>>>(p);
    else k_resize_pairs<false><<<grid, kPixThreads, (size_t)p.src_words * 4, st>>>(p);
    return;
  }
  if (p.cols == 2) launch_resize_cols<2>(p, grid, dyn, staged, plain, st);
  else if (p.cols == 4) launch_resize_cols<4>(p, grid, dyn, staged, plain, st);
  else launch_resize_cols<8>(p, grid, dyn, staged, plain, st);
}

// decode_crop output: uint8 [h, w, 3] at out + offsets[img].
__global__ void k_crop_u8(const ImgInfo *info, const uint8_t *plane, uint8_t *out,
                          const uint64_t *offsets) {
  const int img = blockIdx.y;
  const ImgInfo &I = info[img];
  if (I.status != 0) return;
  PlaneSrc S;
  S.load(I, plane);
  uint8_t *o = out + offsets[img];
  const int64_t npx = (int64_t)I.rw * I.rh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int yy = (int)(i / I.rw), xx = (int)(i % I.rw);
    int r, g, b;
    S.rgb(I.ry + yy, I.rx + xx, r, g, b);
    o[i * 3 + 0] = (uint8_t)r;
    o[i * 3 + 1] = (uint8_t)g;
    o[i * 3 + 2] = (uint8_t)b;
  }
}

void launch_crop_u8(const ImgInfo *info, const uint8_t *plane, int n, uint8_t *out,
                    const uint64_t *offsets, cudaStream_t st) {
  if (n <= 0) return;
  k_crop_u8<<<dim3(64, n), 256, 0, st>>>(info, plane, out, offsets);
}

// ---------------------------------------------------------------------------
// MAE masking: one warp per sample.  Fisher-Yates draws are independent of
// the permutation state (counter-based stream), so lanes compute them in
// parallel; lane 0 applies the swaps; ballot/popc ranks give the sorted mask,
// ids_keep and ids_restore.

__global__ void k_mask(uint64_t seed, uint64_t epoch, const int64_t *index, const uint64_t *states,
                       int tokens, int k, int32_t *mask, int64_t *keep, int64_t *restore) {
  extern __shared__ int16_t sm[];
  int16_t *perm = sm;             // [tokens]
  int16_t *jd = sm + tokens;      // [tokens] draw for step d
  const int s = blockIdx.x;
  const int lane = threadIdx.x;
  const uint64_t st0 = states ? states[s] : rng_init(seed, epoch, (uint64_t)index[s], 1);  // DOMAIN_MASK
  for (int t = lane; t < tokens; t += 32) perm[t] = (int16_t)t;
  for (int d = lane; d < tokens - 1; d += 32) {
    const int i = tokens - 1 - d;
    const uint64_t u = mix64(st0 + (uint64_t)(d + 1) * kGamma);
    const double r = __dmul_rn((double)(u >> 11), 0x1p-53);  // rng.py:50-52
    int j = (int)__double2ll_rz(__dmul_rn(r, (double)(i + 1)));  // rng.py:57-60
    if (j >= i + 1) j = i;
    jd[d] = (int16_t)j;
  }
  __syncwarp();
  if (lane == 0) {
    for (int d = 0; d < tokens - 1; d++) {
      const int i = tokens - 1 - d, j = jd[d];
      const int16_t a = perm[i];
      perm[i] = perm[j];
      perm[j] = a;
    }
  }
  __syncwarp();
  // membership: jd reused as flags
  for (int t = lane; t < tokens; t += 32) jd[t] = 0;
  __syncwarp();
  for (int q = lane; q < k; q += 32) jd[perm[q]] = 1;
  __syncwarp();
  int base_m = 0, base_k = 0;
  const int nkeep = tokens - k;
  for (int t0 = 0; t0 < tokens; t0 += 32) {
    const int t = t0 + lane;
    const bool in = t < tokens;
    const bool m = in && jd[t];
    const unsigned bm = __ballot_sync(0xFFFFFFFFu, m);
    const unsigned bk = __ballot_sync(0xFFFFFFFFu, in && !m);
    const unsigned lower = (1u << lane) - 1;
    if (in) {
      if (m) {
        const int rm = base_m + __popc(bm & lower);
        if (mask) mask[(int64_t)s * k + rm] = t;
        if (restore) restore[(int64_t)s * tokens + t] = nkeep + rm;
      } else {
        const int rk = base_k + __popc(bk & lower);
        if (keep) keep[(int64_t)s * nkeep + rk] = t;
        if (restore) restore[(int64_t)s * tokens + t] = rk;
      }
    }
    base_m += __popc(bm);
    base_k += __popc(bk);
  }
}

void launch_mask(uint64_t seed, uint64_t epoch, const int64_t *index, int n, int tokens, int k,
                 int32_t *mask, int64_t *keep, int64_t *restore, cudaStream_t st) {
  if (n <= 0 || tokens <= 0) return;
  k_mask<<<n, 32, 2 * tokens * sizeof(int16_t), st>>>(seed, epoch, index, nullptr, tokens, k, mask,
                                                       keep, restore);
}

void launch_mask_states(const uint64_t *states, int n, int tokens, int k, int32_t *mask,
                        int64_t *keep, int64_t *restore, cudaStream_t st) {
  if (n <= 0 || tokens <= 0) return;
  k_mask<<<n, 32, 2 * tokens * sizeof(int16_t), st>>>(0, 0, nullptr, states, tokens, k, mask, keep,
                                                       restore);
}

// MAE patchify ('nchpwq->nhwpqc') of the visible tokens: thread = 8 bf16 of
// one token row (patch row pr, 8 consecutive (q, c) elements).
__global__ void k_gather(const __nv_bfloat16 *pix, int res, int patch, const int64_t *keep,
                         int n_keep, __nv_bfloat16 *tok) {
  const int s = blockIdx.y;
  const int dim = patch * patch * 3;
  const int g = res / patch;
  const int64_t total = (int64_t)n_keep * dim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int ti = (int)(e / dim), w = (int)(e % dim);
    const int id = (int)keep[(int64_t)s * n_keep + ti];
    const int ph = id / g, pw = id % g;
    const int pr = w / (patch * 3), rem = w % (patch * 3);
    const int pc = rem / 3, c = rem % 3;
    tok[(int64_t)s * total + e] =
        pix[(((int64_t)s * 3 + c) * res + ph * patch + pr) * res + pw * patch + pc];
  }
}

// Same tokens placed by ids_restore (token id -> row rank when < n_keep):
// the 3-Aug path's gather from finished pixels.
__global__ void k_gather_restore(const __nv_bfloat16 *pix, int res, int patch, const int64_t *restore,
                                 int n_keep, __nv_bfloat16 *tok) {
  const int s = blockIdx.x;
  const int g = res / patch, T = g * g, dim = patch * patch * 3;
  for (int64_t e = threadIdx.x; e < (int64_t)T * dim; e += blockDim.x) {
    const int id = (int)(e / dim), w = (int)(e % dim);
    const int64_t rk = restore[(int64_t)s * T + id];
    if (rk >= n_keep) continue;
    const int ph = id / g, pw = id % g;
    const int pr = w / (patch * 3), rem = w % (patch * 3);
    const int pc = rem / 3, c = rem % 3;
    tok[((int64_t)s * n_keep + rk) * dim + w] =
        pix[(((int64_t)s * 3 + c) * res + ph * patch + pr) * res + pw * patch + pc];
  }
}

void launch_gather_restore(const void *pix, int n, int res, int patch, const int64_t *restore,
                           int n_keep, void *tokens, cudaStream_t st) {
  if (n <= 0 || n_keep <= 0) return;
  k_gather_restore<<<n, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16 *>(pix), res, patch,
                                      restore, n_keep, reinterpret_cast<__nv_bfloat16 *>(tokens));
}

void launch_gather(const void *pix, int n, int res, int patch, const int64_t *keep, int n_keep,
                   void *tokens, cudaStream_t st) {
  if (n <= 0 || n_keep <= 0) return;
  k_gather<<<dim3(48, n), 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16 *>(pix), res, patch,
                                         keep, n_keep, reinterpret_cast<__nv_bfloat16 *>(tokens));
}

// ---------------------------------------------------------------------------
// standalone imgops on a single HWC uint8 image

__global__ void k_resize_u8(const uint8_t *src, int ih, int iw, uint8_t *dst, int oh, int ow,
                            int flip) {
  const int64_t npx = (int64_t)oh * ow;
  const double sy = __ddiv_rn((double)ih, (double)oh), sx = __ddiv_rn((double)iw, (double)ow);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int oy = (int)(i / ow), ox = (int)(i % ow);
    const int xs = flip ? ow - 1 - ox : ox;
    int y0, y1, x0, x1;
    double wy, wx;
    tap(oy, sy, ih, y0, y1, wy);
    tap(xs, sx, iw, x0, x1, wx);
#pragma unroll
    for (int c = 0; c < 3; c++) {
      dst[i * 3 + c] = (uint8_t)bilerp(wx, wy, src[((int64_t)y0 * iw + x0) * 3 + c],
                                       src[((int64_t)y0 * iw + x1) * 3 + c],
                                       src[((int64_t)y1 * iw + x0) * 3 + c],
                                       src[((int64_t)y1 * iw + x1) * 3 + c]);
    }
  }
}

void launch_resize_u8(const uint8_t *src, int ih, int iw, uint8_t *dst, int oh, int ow, int flip,
                      cudaStream_t st) {
  k_resize_u8<<<148, 256, 0, st>>>(src, ih, iw, dst, oh, ow, flip);
}

__global__ void k_normalize_u8(const uint8_t *src, int h, int w, float *dst) {
  const int64_t npx = (int64_t)h * w;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int c = 0; c < 3; c++) dst[c * npx + i] = norm_value(c, src[i * 3 + c]);
  }
}

void launch_normalize_u8(const uint8_t *src, int h, int w, float *dst, cudaStream_t st) {
  k_normalize_u8<<<148, 256, 0, st>>>(src, h, w, dst);
}

// ---------------------------------------------------------------------------
// 3-Aug / 3-Aug+ stage (apply_aug after the flip, pipeline.py:88-101) on
// uint8 HWC images: k_aug_blur (gaussian_blur, tiled) then k_aug_out (point
// op, jitter, normalize / uint8 out).  All float64 arithmetic is one
// rounding per operation in the reference's order (numba without
// fastmath), so results are bit-identical.

constexpr int kAugTile = 32;
constexpr int kAugBlurThreads = 256;
constexpr int kAugOutThreads = 512;

__device__ __forceinline__ int reflect_idx(int i, int n) {  // imgops.py:111-119
  if (n == 1) return 0;
  const int period = 2 * n - 2;
  i %= period;
  if (i < 0) i += period;
  return i >= n ? period - i : i;
}


// floor(factor * v + (1 - factor) * target + 0.5) clamped (imgops.py:166-196)
__device__ __forceinline__ int blend1(double f, int v, double target) {
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(f, (double)v), __dmul_rn(__dsub_rn(1.0, f), target)),
                             0.5);
  return clamp255(__double2int_rd(s));
}

size_t aug_blur_smem(int radius) {
  const int sh = kAugTile + 2 * radius;
  return 32 * sizeof(double) + (size_t)sh * kAugTile * 3 * sizeof(double) + (size_t)sh * sh * 3;
}

// gaussian_blur (imgops.py:122-163) for one kAugTile^2 output tile: the
// reflect-indexed source tile with its radius halo is staged in shared
// memory, the float64 horizontal pass (imgops.py:122-134) fills a tile of
// (th + 2r) rows, the vertical pass (:137-151) rounds int(acc + 0.5) capped
// at 255.  grid: (tiles_x * tiles_y, n); images without the blur exit.
__global__ void __launch_bounds__(kAugBlurThreads) k_aug_blur(const uint8_t *src, int h, int w,
                                                              const essl_aug *aug, uint8_t *dst) {
  const essl_aug &A = aug[blockIdx.y];
  if (A.op != ESSL_AUG_OP_BLUR) return;
  extern __shared__ __align__(16) unsigned char aug_sm[];
  const int r = A.radius, nt = 2 * r + 1;
  const int tiles_x = (w + kAugTile - 1) / kAugTile;
  const int ty0 = (blockIdx.x / tiles_x) * kAugTile, tx0 = (blockIdx.x % tiles_x) * kAugTile;
  const int th = min(kAugTile, h - ty0), tw = min(kAugTile, w - tx0);
  const int sh = th + 2 * r, spitch = (tw + 2 * r) * 3, tpitch = tw * 3;
  double *wt = reinterpret_cast<double *>(aug_sm);
  double *tmp = wt + 32;
  uint8_t *s = reinterpret_cast<uint8_t *>(tmp + (size_t)(kAugTile + 2 * r) * kAugTile * 3);
  const size_t img_off = (size_t)blockIdx.y * h * w * 3;
  const uint8_t *in = src + img_off;
  if (threadIdx.x < nt) wt[threadIdx.x] = A.weights[threadIdx.x];
  // rows by warp, bytes by lane (no per-element division); tiles whose halo
  // lies inside the image copy rows straight, border tiles reflect-index
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kAugBlurThreads / 32;
  const bool inner = ty0 - r >= 0 && ty0 + th + r <= h && tx0 - r >= 0 && tx0 + tw + r <= w;
  for (int yy = warp; yy < sh; yy += nw) {
    const int sy = inner ? ty0 - r + yy : reflect_idx(ty0 - r + yy, h);
    const uint8_t *srow = in + (size_t)sy * w * 3;
    uint8_t *drow = s + yy * spitch;
    if (inner) {
      const uint8_t *p = srow + (size_t)(tx0 - r) * 3;
      for (int rem = lane; rem < spitch; rem += 32) drow[rem] = p[rem];
    } else {
      for (int rem = lane; rem < spitch; rem += 32) {
        const int xx = rem / 3, c = rem - xx * 3;
        drow[rem] = srow[reflect_idx(tx0 - r + xx, w) * 3 + c];
      }
    }
  }
  __syncthreads();
  for (int yy = warp; yy < sh; yy += nw) {
    const uint8_t *srow = s + yy * spitch;
    double *trow = tmp + yy * tpitch;
    for (int rem = lane; rem < tpitch; rem += 32) {
      const uint8_t *row = srow + rem;  // tap k at row[3 k]
      double acc = 0.0;
      for (int k = 0; k < nt; k++) acc = __dadd_rn(acc, __dmul_rn(wt[k], (double)row[3 * k]));
      trow[rem] = acc;
    }
  }
  __syncthreads();
  uint8_t *out = dst + img_off;
  for (int yy = warp; yy < th; yy += nw) {
    uint8_t *orow = out + ((size_t)(ty0 + yy) * w + tx0) * 3;
    for (int rem = lane; rem < tpitch; rem += 32) {
      const double *col = tmp + yy * tpitch + rem;
      double acc = 0.0;
      for (int k = 0; k < nt; k++) acc = __dadd_rn(acc, __dmul_rn(wt[k], col[k * tpitch]));
      const int v = __double2int_rz(__dadd_rn(acc, 0.5));
      orow[rem] = (uint8_t)(v > 255 ? 255 : v);
    }
  }
}

// Point op (grayscale / solarize; the blur was applied by k_aug_blur).
__device__ __forceinline__ void aug_point(int op, int thr, const uint8_t *p, int px[3]) {
  px[0] = p[0]; px[1] = p[1]; px[2] = p[2];
  if (op == ESSL_AUG_OP_GRAY) {
    px[0] = px[1] = px[2] = luma601(px[0], px[1], px[2]);
  } else if (op == ESSL_AUG_OP_SOLARIZE) {
#pragma unroll
    for (int c = 0; c < 3; c++) px[c] = px[c] >= thr ? 255 - px[c] : px[c];
  }
}

// One CTA per image: (3-Aug+) luma mean of the brightness-adjusted image
// (imgops.py:199-216; integer sum, exact), then per pixel the point op,
// brightness, contrast, saturation (imgops.py:213-227), normalize through the
// exact LUT (imgops.py:231-240) into bf16/f32 NCHW and/or the uint8 view.
// Brightness (target 0) and contrast (target the image mean) are functions
// of one uint8 value, so each is tabulated once per image (256 float64
// blends, the same operations as per pixel); only saturation, whose target
// is the pixel's own luma, stays per pixel.
__global__ void __launch_bounds__(kAugOutThreads) k_aug_out(AugOutParams P) {
  const int img = blockIdx.x;
  const essl_aug &A = P.aug[img];
  if (P.fused_points && A.op != ESSL_AUG_OP_BLUR && !A.jitter) return;  // finished in k_resize
  const int op = A.op, thr = A.threshold, jitter = A.jitter;
  const double fb = A.factors[0], fc = A.factors[1], fs = A.factors[2];
  const int64_t npx = (int64_t)P.h * P.w;
  const uint8_t *src = (op == ESSL_AUG_OP_BLUR ? P.b : P.a) + (size_t)img * npx * 3;
  __shared__ float lut[3][256];
  __shared__ __nv_bfloat16 lutb[3][256];
  __shared__ unsigned long long part[kAugOutThreads / 32];
  __shared__ uint8_t bri[256], con[256];
  static_assert(kAugOutThreads >= 256, "one thread per table entry");
  if (P.out_kind == ESSL_OUT_F32_NCHW)
    for (int i = threadIdx.x; i < 768; i += kAugOutThreads) lut[i >> 8][i & 255] = g_norm_lut[i];
  else if (P.out_kind == ESSL_OUT_BF16_NCHW)
    for (int i = threadIdx.x; i < 768; i += kAugOutThreads) lutb[i >> 8][i & 255] = g_norm_lutb[i];
  if (jitter && threadIdx.x < 256) bri[threadIdx.x] = (uint8_t)blend1(fb, threadIdx.x, 0.0);
  __syncthreads();
  // groups of 4 pixels (12 source bytes = 3 words; 4 outputs per channel =
  // one 8-byte bf16 / 16-byte f32 store) when every address is aligned for
  // it; the scalar loop takes the rest (odd sizes, the tail)
  const int64_t stride = P.out_stride ? P.out_stride : 3 * npx;
  const size_t osz = P.out_kind == ESSL_OUT_F32_NCHW ? 4 : 2;
  const bool vec = (npx & 3) == 0 && ((uintptr_t)src & 3) == 0 && (stride & 3) == 0 &&
                   ((uintptr_t)P.out & (4 * osz - 1)) == 0 && ((uintptr_t)P.out_u8 & 3) == 0;
  const int64_t ngrp = vec ? npx >> 2 : 0;
  const uint32_t *src4 = reinterpret_cast<const uint32_t *>(src);
  if (jitter) {
    unsigned long long sum = 0;
    for (int64_t g = threadIdx.x; g < ngrp; g += kAugOutThreads) {
      alignas(16) uint8_t b[12];
      *reinterpret_cast<uint3 *>(b) = make_uint3(src4[3 * g], src4[3 * g + 1], src4[3 * g + 2]);
#pragma unroll
      for (int j = 0; j < 4; j++) {
        int px[3];
        aug_point(op, thr, b + 3 * j, px);
        sum += (unsigned)luma601(bri[px[0]], bri[px[1]], bri[px[2]]);
      }
    }
    for (int64_t i = 4 * ngrp + threadIdx.x; i < npx; i += kAugOutThreads) {
      int px[3];
      aug_point(op, thr, src + 3 * i, px);
      sum += (unsigned)luma601(bri[px[0]], bri[px[1]], bri[px[2]]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x < 256) {
      unsigned long long tot = 0;
#pragma unroll
      for (int k = 0; k < kAugOutThreads / 32; k++) tot += part[k];
      const double mean = __ddiv_rn((double)tot, (double)npx);  // acc / (h * w), acc an exact integer
      con[threadIdx.x] = (uint8_t)blend1(fc, threadIdx.x, mean);
    }
    __syncthreads();
  }
  auto finish = [&](int px[3]) {
    if (jitter) {
#pragma unroll
      for (int c = 0; c < 3; c++) px[c] = con[bri[px[c]]];                  // brightness, contrast
      const double g = (double)luma601(px[0], px[1], px[2]);
#pragma unroll
      for (int c = 0; c < 3; c++) px[c] = blend1(fs, px[c], g);             // saturation
    }
  };
  for (int64_t g = threadIdx.x; g < ngrp; g += kAugOutThreads) {
    alignas(16) uint8_t b[12];
    *reinterpret_cast<uint3 *>(b) = make_uint3(src4[3 * g], src4[3 * g + 1], src4[3 * g + 2]);
    int q[4][3];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      aug_point(op, thr, b + 3 * j, q[j]);
      finish(q[j]);
    }
    const int64_t i = 4 * g;
    if (P.out_kind == ESSL_OUT_BF16_NCHW) {
      __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(P.out) + img * stride + i;
#pragma unroll
      for (int c = 0; c < 3; c++) {
        __nv_bfloat162 lo = __halves2bfloat162(lutb[c][q[0][c]], lutb[c][q[1][c]]);
        __nv_bfloat162 hi = __halves2bfloat162(lutb[c][q[2][c]], lutb[c][q[3][c]]);
        *reinterpret_cast<uint2 *>(o + c * npx) =
            make_uint2(*reinterpret_cast<uint32_t *>(&lo), *reinterpret_cast<uint32_t *>(&hi));
      }
    } else if (P.out_kind == ESSL_OUT_F32_NCHW) {
      float *o = reinterpret_cast<float *>(P.out) + img * stride + i;
#pragma unroll
      for (int c = 0; c < 3; c++)
        *reinterpret_cast<float4 *>(o + c * npx) =
            make_float4(lut[c][q[0][c]], lut[c][q[1][c]], lut[c][q[2][c]], lut[c][q[3][c]]);
    }
    if (P.out_u8) {
      alignas(16) uint8_t ob[12];
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int c = 0; c < 3; c++) ob[3 * j + c] = (uint8_t)q[j][c];
      *reinterpret_cast<uint3 *>(P.out_u8 + ((size_t)img * npx + i) * 3) = *reinterpret_cast<uint3 *>(ob);
    }
  }
  for (int64_t i = 4 * ngrp + threadIdx.x; i < npx; i += kAugOutThreads) {
    int px[3];
    aug_point(op, thr, src + 3 * i, px);
    finish(px);
    if (P.out_kind == ESSL_OUT_BF16_NCHW) {
      __nv_bfloat16 *o = reinterpret_cast<__nv_bfloat16 *>(P.out) + img * stride + i;
#pragma unroll
      for (int c = 0; c < 3; c++) o[c * npx] = lutb[c][px[c]];
    } else if (P.out_kind == ESSL_OUT_F32_NCHW) {
      float *o = reinterpret_cast<float *>(P.out) + img * stride + i;
#pragma unroll
      for (int c = 0; c < 3; c++) o[c * npx] = lut[c][px[c]];
    }
    if (P.out_u8) {
      uint8_t *o = P.out_u8 + ((size_t)img * npx + i) * 3;
#pragma unroll
      for (int c = 0; c < 3; c++) o[c] = (uint8_t)px[c];
    }
  }
}

void launch_aug(const AugOutParams &p, int max_radius, cudaStream_t st) {
  if (p.n <= 0) return;
  if (max_radius > 0) {
    const int tiles = ((p.h + kAugTile - 1) / kAugTile) * ((p.w + kAugTile - 1) / kAugTile);
    k_aug_blur<<<dim3(tiles, p.n), kAugBlurThreads, aug_blur_smem(max_radius), st>>>(
        p.a, p.h, p.w, p.aug, p.b);
  }
  k_aug_out<<<p.n, kAugOutThreads, 0, st>>>(p);
}

// ---------------------------------------------------------------------------
// Pinned-container gather: payload bytes read host->device over the bus by
// a light kernel.  Bus reads have microsecond latency and hold the SM's
// outstanding-miss resources for that long, so the gather runs on a few
// CTAs only (`ctas`, ESSL_OPT_GATHER_CTAS) that loop over the batch's
// payloads with 8 x 16 B loads in flight per thread -- the other SMs' memory
// pipelines (the decode kernels of other batches) stay unaffected.  Sources
// are 64-byte aligned in the container (container.py:26); an unaligned
// source takes the byte path.
constexpr int kGatherThreads = 256;
constexpr int kGatherLoads = 8;

__global__ void __launch_bounds__(kGatherThreads) k_host_gather(const uint8_t *src,
                                                                const GatherDesc *desc, int n,
                                                                uint8_t *dst) {
  for (int j = blockIdx.x; j < n; j += gridDim.x) {
    const GatherDesc d = desc[j];
    const uint8_t *s = src + d.src;
    uint8_t *o = dst + d.dst;
    if (((d.src | d.dst) & 15) == 0) {
      const int4 *s4 = reinterpret_cast<const int4 *>(s);
      int4 *o4 = reinterpret_cast<int4 *>(o);
      const uint32_t n16 = d.len / 16;
      for (uint32_t i = threadIdx.x; i < n16; i += kGatherLoads * kGatherThreads) {
        int4 v[kGatherLoads];
#pragma unroll
        for (int u = 0; u < kGatherLoads; u++)
          if (i + u * kGatherThreads < n16) v[u] = s4[i + u * kGatherThreads];
#pragma unroll
        for (int u = 0; u < kGatherLoads; u++)
          if (i + u * kGatherThreads < n16) o4[i + u * kGatherThreads] = v[u];
      }
      for (uint32_t i = n16 * 16 + threadIdx.x; i < d.len; i += kGatherThreads) o[i] = s[i];
    } else {
      for (uint32_t i = threadIdx.x; i < d.len; i += kGatherThreads) o[i] = s[i];
    }
  }
}

// TMA variant: one thread per CTA drives a ring of bulk copies (cp.async.bulk
// global->shared completing on an mbarrier, then shared->global): the bus
// reads are tracked by the CTA's bulk-copy engine instead of the LSU miss
// queues the co-resident decode kernels use.  16-byte-aligned body via TMA,
// the (< 16 B) tail and unaligned payloads by the other lanes.
constexpr int kTmaChunk = 4096;  // (32 KB of stages: the gather's CTAs fit next to the decode kernels; 16 KB chunks: e2e -1.7%)
constexpr int kTmaStages = 8;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(32) k_host_gather_tma(const uint8_t *src, const GatherDesc *desc,
                                                        int n, uint8_t *dst) {
  extern __shared__ __align__(128) uint8_t gbuf[];
  __shared__ __align__(8) uint64_t bar[kTmaStages];
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int i = 0; i < kTmaStages; i++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  for (int j = blockIdx.x; j < n; j += gridDim.x) {  // tails / unaligned payloads: lanes 1..31
    const GatherDesc d = desc[j];
    const bool al = ((d.src | d.dst) & 15) == 0;
    for (uint32_t i = (al ? d.len & ~15u : 0u) + lane; i < d.len; i += 32) dst[d.dst + i] = src[d.src + i];
  }
  if (lane != 0) return;
  // issue cursor (ji, oi) runs up to kTmaStages chunks ahead of the store cursor (js, os)
  int ji = blockIdx.x, js = blockIdx.x;
  uint32_t oi = 0, os = 0, issued = 0, stored = 0;
  auto body = [&](int j) -> uint32_t {
    const GatherDesc d = desc[j];
    return ((d.src | d.dst) & 15) == 0 ? (d.len & ~15u) : 0u;
  };
  auto advance = [&](int &jj, uint32_t &oo) {  // next chunk start (skips empty bodies)
    while (jj < n && oo >= body(jj)) {
      jj += gridDim.x;
      oo = 0;
    }
  };
  advance(ji, oi);
  advance(js, os);
  while (js < n) {
    while (ji < n && issued - stored < (uint32_t)kTmaStages) {
      const GatherDesc d = desc[ji];
      const uint32_t bytes = min((uint32_t)kTmaChunk, body(ji) - oi);
      const int st = issued % kTmaStages;
      if (issued >= (uint32_t)kTmaStages)  // the store that last read this buffer is done
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const uint32_t b = smem_u32(&bar[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(gbuf + st * kTmaChunk)),
          "l"(src + d.src + oi), "r"(bytes), "r"(b)
          : "memory");
      issued++;
      oi += bytes;
      advance(ji, oi);
    }
    const GatherDesc d = desc[js];
    const uint32_t bytes = min((uint32_t)kTmaChunk, body(js) - os);
    const int st = stored % kTmaStages;
    const uint32_t b = smem_u32(&bar[st]);
    const uint32_t phase = (stored / kTmaStages) & 1;
    asm volatile(
        "{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W_%=;\n}" ::"r"(b),
        "r"(phase)
        : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + d.dst + os),
                 "r"(smem_u32(gbuf + st * kTmaChunk)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    stored++;
    os += bytes;
    advance(js, os);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

void launch_host_gather(const uint8_t *src, const GatherDesc *d, int n, uint8_t *dst, int ctas,
                        bool tma, cudaStream_t st) {
  if (n <= 0) return;
  const int grid = ctas > 0 && ctas < n ? ctas : n;
  if (tma) {
    k_host_gather_tma<<<grid, 32, kTmaChunk * kTmaStages, st>>>(src, d, n, dst);
  } else {
    k_host_gather<<<grid, kGatherThreads, 0, st>>>(src, d, n, dst);
  }
}

// Per-device one-time setup (api.cu, once per device): the normalize LUTs
// (__device__ arrays exist per device) and the dynamic shared-memory opt-ins.
void init_device_pixels() {
  k_init_norm_luts<<<1, 768>>>();
  resize_attrs<2>();
  resize_attrs<4>();
  cudaFuncSetAttribute(k_resize_pairs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kResizeMaxDyn);
  for (auto f : {k_resize_pairs<false, 224>, k_resize_pairs<false, 192>, k_resize_pairs<false, 160>,
                 k_resize_pairs<false, 112>})
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kResizeMaxDyn);
  cudaFuncSetAttribute(k_resize_pairs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kResizeMaxDyn);
  resize_attrs<8>();
  cudaFuncSetAttribute(k_aug_blur, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)aug_blur_smem(ESSL_AUG_MAX_RADIUS));
  cudaFuncSetAttribute(k_host_gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kTmaChunk * kTmaStages);
}

}  // namespace essl
