// k_prep + k_entropy + k_idct.  Replace, for a whole batch,
//   container.py:249-265   read_sample CRC check
//   jpeg/codec.py:124-265  parse_stream + _finish_geometry
//   jpeg/codec.py:272-320  _huff_lut / _destuff
//   jpeg/decode_kernels.py:27-179  destuff_scan / bit reader / decode_scan_baseline
//   jpeg/codec.py:323-330  _check_consumed
//   jpeg/decode_kernels.py:388-534 reconstruct_blocks (crop window only)
//
// k_prep (one 256-thread CTA per image) stages the compressed payload in
// shared memory (16-byte loads) and does the byte-level work there: CRC32,
// marker parse, destuff (into a global clean stream of big-endian words),
// Huffman table build, window zeroing.  It hands a per-image DecodeHdr to
// k_entropy.  Payloads too large for shared memory run on global (SMEM=false).
//
// k_entropy decodes one image per 64-thread CTA.  A restart-free baseline
// scan is a serial chain: the decoder state (bit position, zig-zag index k,
// block in MCU b) at any point depends on everything before it.  The clean
// stream (up to an estimate of where the crop's last needed block ends,
// codec.py:494-498 row_stop) is cut into <= 64 subsequences; lane t decodes
// its subsequence from a guessed state (k=0, b=0) after a warm-up, storing
// every unit in its list and recording checkpoints (bit position, b, blocks
// so far) at block starts, then continues past its end until its path
// reaches a checkpoint of a later lane with the same state.  Two decoders in
// the same state produce the same future, so the exact path (lane 0 starts
// exactly) is lane 0's path, then the path of the lane it merged into from
// the merge checkpoint, and so on; each unit is decoded once.
// Per-segment DC sums give every crop-window block its predictor and list
// position (k_idct gathers from the lists).  Streams with restart intervals
// (DRI) decode one interval per lane; multi-scan streams (progressive,
// sequential non-interleaved) decode every scan in dependency waves into
// full coefficient arrays.
//
// k_idct dequantises + inverse-transforms the crop-window blocks with all
// threads of the GPU (8 lanes per block).
#include <cstdint>
#include <type_traits>

#include "essl_common.cuh"

namespace essl {

__device__ unsigned int g_check_dec[CK_COUNT];  // ESSL_CHECK counters (checked builds)

void check_read_decode(unsigned int *out, bool reset) {
  cudaMemcpyFromSymbol(out, g_check_dec, sizeof(unsigned int) * CK_COUNT);
  if (reset) {
    static const unsigned int zero[CK_COUNT] = {};
    cudaMemcpyToSymbol(g_check_dec, zero, sizeof(zero));
  }
}

__constant__ uint8_t c_zz[64] = {
    0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

// x^(2^k) mod P (reflected CRC-32), k = 0..31; filled by init_crc_tables().
__constant__ uint32_t c_x2n[32];
// Multiply-by-x^(8*kCrcChunk*2^j) mod P as 4 byte tables per level j
// (GF(2)-linear map), global memory, filled by init_crc_tables().
constexpr int kCrcChunk = 132;  // 33 words: lanes hit distinct smem banks
constexpr int kCrcLevels = 16;
__constant__ const uint32_t *c_crc_mul;  // [kCrcLevels][4][256]
constexpr int kCrcMaxChunks = 2048;      // payloads <= 256 KB use the table tree

constexpr uint32_t kNoEnd = 0xFFFFFFF0u;
constexpr int kNT = kDecodeThreads;
constexpr int kLanes = kEntropyLanes;
constexpr uint32_t kContBits = kContinuationBits;

// Huffman decode tables.  One 16-bit entry per kFastBits-bit lookahead:
//   bits 0-4   tot  = code length + magnitude bits (0: see below)
//   bits 5-11  kinc = zig-zag advance: DC 1; AC run+1, ZRL 16, EOB 64;
//                     127 marks a DC category > 15 (decode error)
//   bits 12-15 size = magnitude bits
// tot == 0: entry 0 is an invalid code; otherwise bits 5-15 hold 1 + the
// index of a second-level table for codes longer than kFastBits (indexed by
// the next kSubBits bits), or kSubCanon (canonical maxcode walk, only for
// hostile tables with more than kSubTabs long-code prefixes).  Symbol
// semantics are those of the 16-bit LUT of codec.py:272-295 and the scan
// loop of decode_kernels.py:139-177.
constexpr int kSubBits = 16 - kFastBits;
constexpr int kSubTabs = 8;
constexpr uint32_t kSubCanon = 0x7FF;

struct __align__(16) HuffTab {
  uint16_t fast[1 << kFastBits];
  uint16_t sub[kSubTabs << kSubBits];
  int32_t lim[17];  // first[L] + count[L]
  int32_t first[17];
  int16_t vptr[17];
  uint8_t vals[256];
  int dht_pos, nvals, is_dc, nsub;
};

// The part of a HuffTab the entropy decoder keeps in shared memory (the
// canonical arrays stay in global memory: only hostile tables reach them).
struct __align__(16) HuffFast {
  uint16_t fast[1 << kFastBits];
  uint16_t sub[kSubTabs << kSubBits];
};

__host__ __device__ __forceinline__ uint32_t huff_entry(bool dc, int sym, int len) {
  int size, kinc;
  if (dc) {
    size = sym > 15 ? 1 : sym;
    kinc = sym > 15 ? 127 : 1;
  } else {
    const int run = sym >> 4;
    size = sym & 15;
    kinc = size ? run + 1 : (run == 15 ? 16 : 64);
  }
  return (uint32_t)(len + size) | ((uint32_t)kinc << 5) | ((uint32_t)size << 12);
}

// Geometry, stream location and tables handed from k_prep to k_entropy
// (global, one per image; k_entropy keeps a copy in shared memory).
struct __align__(16) DecodeHead {
  int32_t status, reason, offset;
  int32_t ns, bpm, gx, gy, row_stop, mx0, mx1, my0, my1, ncomp, ntab;
  uint32_t limit_blocks, clean_bits, clean_words, tab_index_word;
  uint32_t wmax;  // last readable word of the clean stream (0xFF padding)
  uint32_t cpad;  // first 16-byte chunk of the clean stream that is all 0xFF padding
  int32_t scan_ri, scan_start, scan_end, n_restarts, max_restarts;
  int32_t slot_comp[4], slot_h[4], slot_v[4], slot_nb[4];
  int32_t wby0[3], wbx0[3], wbh[3], wbw[3], bw[3], bh[3];
  int32_t quant_missing;  // -1: all dequantisation tables present
  // multi-scan streams (progressive / several scans): full decode of every
  // scan into full coefficient arrays (k_entropy multiscan path)
  int32_t multiscan, progressive;
  int32_t comp_id[3];     // component identifiers (SOF)
  int32_t comp_hv[3];     // h << 4 | v per component
  int32_t coef_pitch[3];  // blocks per coefficient-array row (window width; BW when multiscan)
  uint32_t rst_off;       // restart table, words from the clean region start
  uint64_t coef_off[3], coef_base, clean_off;
  // device address of each used Huffman table: the context's table cache
  // slot when the image's DHT matched it (no per-image copy), else the
  // image's own DecodeHdr::tab entry
  uint64_t tab_ptr[kMaxTables];
  uint8_t blk_slot[kMaxBpm], blk_dy[kMaxBpm], blk_dx[kMaxBpm];
  uint8_t zz[64];
};
// + the dequantisation and Huffman tables (k_prep writes them to global
// memory directly; k_entropy's shared copy of the head leaves them out)
struct __align__(16) DecodeHdr : DecodeHead {
  int32_t q[3][64];  // dequantisation tables, natural order
  HuffTab tab[kMaxTables];
};

// Built Huffman tables reused across images (per context, persistent):
// slot t caches the t-th distinct table of the first image that claimed it
// (state 0 empty, 1 being written, 2 ready).  An image whose t-th table has
// the same class and the same DHT counts + symbols copies the built table
// instead of building it (a batch of images from one encoder shares them).
struct __align__(16) TabCacheSlot {
  unsigned int state;
  int len, is_dc, pad;
  uint8_t key[16 + 256];  // DHT counts + symbols
  HuffTab tab;
};

struct ParseState {
  int pos, n, ri, have_sof, progressive, width, height, ncomp, nscans;
  int comp_id[3], comp_h[3], comp_v[3], comp_tq[3];
  int quant_pos[16], quant_pq[16];
  int huff_pos[2][16], huff_tot[2][16];
  int ns, slot_comp[4], slot_dpos[4], slot_dtot[4], slot_apos[4], slot_atot[4];
  int scan_ri, scan_start, scan_end;
  int status, reason, offset;
  int cmd, dstart;
};

struct __align__(16) PrepSmem {
  DecodeHead h;
  struct {
    uint32_t T[4][256];  // slice-by-4 CRC tables (chunk partials: dynamic smem)
  } crc;
  long long ph[8];
  ParseState ps;
  uint32_t K[8];
  uint32_t warp_tot[kNT / 32][4];
  uint16_t sub_pf[kMaxTables][kSubTabs];
  int stop, carry, dstop;
  long long t0;
  // the (< 16) bytes before the scan that the in-place destuff overwrites
  // (its output starts 16-byte aligned): the tail of the segment before SOS
  // can be the last DHT, whose bytes the table code reads afterwards
  int save_lo, save_hi;
  uint8_t save[16];
};

// A marker-segment byte of the payload after the in-place destuff: the bytes
// it overwrote come from the save area.
__device__ __forceinline__ uint8_t seg_byte(const PrepSmem &S, const uint8_t *raw, int i) {
  return (i >= S.save_lo && i < S.save_hi) ? S.save[i - S.save_lo] : raw[i];
}

// ---------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ int extend_bits(uint32_t v, int size) {  // decode_kernels.py:101-108
  return (size && v < (1u << (size - 1))) ? (int)v - (1 << size) + 1 : (int)v;
}

__device__ __forceinline__ uint32_t multmodp(uint32_t a, uint32_t b) {
  // a(x) * b(x) modulo the reflected CRC-32 polynomial (zlib multmodp).
  uint32_t p = 0;
#pragma unroll 4
  for (int i = 0; i < 32; i++) {
    if (a & (0x80000000u >> i)) p ^= b;
    b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
  }
  return p;
}

__device__ uint32_t x2nmodp(uint64_t n, int k) {  // x^(n * 2^k) mod P
  uint32_t p = 0x80000000u;
  while (n) {
    if (n & 1) p = multmodp(c_x2n[k & 31], p);
    n >>= 1;
    k++;
  }
  return p;
}

__device__ __forceinline__ bool is_rst(uint32_t m) { return m >= 0xD0 && m <= 0xD7; }
__device__ __forceinline__ bool has_ff(uint32_t w) { return __vcmpeq4(w, 0xFFFFFFFFu) != 0; }

// 0x80 in each byte of t that is zero, 0 elsewhere (exact: no cross-byte carries)
__device__ __forceinline__ uint32_t zero_bytes(uint32_t t) {
  const uint32_t y = (t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
  return ~(y | t | 0x7F7F7F7Fu);
}
// the four 0x80 byte flags of zero_bytes() -> a 4-bit mask (bit q = byte q)
__device__ __forceinline__ uint32_t byte_flags(uint32_t f80) { return ((f80 >> 7) * 0x01020408u) >> 24; }
// 16-byte group masks: bytes == 0xFF, bytes in RST0..RST7 (0xD0-0xD7)
__device__ __forceinline__ void group_masks(const uint32_t w[4], uint32_t &ff, uint32_t &rst) {
  ff = 0;
  rst = 0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    ff |= byte_flags(zero_bytes(~w[k])) << (4 * k);
    rst |= byte_flags(zero_bytes((w[k] & 0xF8F8F8F8u) ^ 0xD0D0D0D0u)) << (4 * k);
  }
}
// any byte of the four words == 0xFF (a filter: false positives are fine)
__device__ __forceinline__ bool any_ff4(const uint4 v) {
  const uint32_t t = (~v.x - 0x01010101u) & v.x;  // high bit of a byte of ~x zero ...
  const uint32_t u = (~v.y - 0x01010101u) & v.y;
  const uint32_t q = (~v.z - 0x01010101u) & v.z;
  const uint32_t r = (~v.w - 0x01010101u) & v.w;
  return ((t | u | q | r) & 0x80808080u) != 0;
}

// Block-wide exclusive scan of four u32 values (kNT threads, warp shuffles).
// Returns the block totals in tot[].
__device__ void block_scan4(uint32_t (*warp_tot)[4], uint32_t v[4], uint32_t tot[4]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t x = v[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
      if (lane >= o) x += y;
    }
    inc[q] = x;
  }
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < 4; q++) warp_tot[warp][q] = inc[q];
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t before = 0, all = 0;
    for (int w = 0; w < kNT / 32; w++) {
      const uint32_t t = warp_tot[w][q];
      if (w < warp) before += t;
      all += t;
    }
    v[q] = inc[q] - v[q] + before;
    tot[q] = all;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// header parse (thread 0), codec.py:124-251

struct PayloadView {  // the payload bytes (shared or global memory)
  const uint8_t *d;
  int n;
  __device__ __forceinline__ int operator[](int i) const { return d[i]; }
};

__device__ void parse_fail(ParseState &P, int reason, int off) {
  P.status = ESSL_ST_MALFORMED;
  P.reason = reason;
  P.offset = off;
  P.cmd = 2;
}

// Runs until the next SOS (cmd=1, dstart set), EOI/end (cmd=0) or error (cmd=2).
__device__ void parse_until_sos(ParseState &P, const PayloadView &d) {
  const int n = d.n;
  while (P.pos < n) {
    int pos = P.pos;
    if (d[pos] != 0xFF) return parse_fail(P, R_EXPECTED_MARKER, pos);
    while (pos < n && d[pos] == 0xFF) pos++;
    if (pos >= n) break;
    const int marker = d[pos++];
    if (marker == 0xD9) { P.pos = n; break; }
    if (marker == 0x01 || is_rst(marker)) { P.pos = pos; continue; }
    if (pos + 2 > n) return parse_fail(P, R_UNEXPECTED_END, pos);
    const int seglen = (d[pos] << 8) | d[pos + 1];
    if (seglen < 2 || pos + seglen > n) return parse_fail(P, R_TRUNC_SEGMENT, pos);
    const int body = pos + 2, end = pos + seglen;
    if (marker == 0xDB) {  // DQT
      int p = body;
      while (p < end) {
        int pq = d[p] >> 4, tq = d[p] & 15;
        p++;
        int count = 64 * (pq == 1 ? 2 : 1);
        if (p + count > end) return parse_fail(P, R_TRUNC_DQT, p);
        P.quant_pos[tq] = p;
        P.quant_pq[tq] = pq;
        p += count;
      }
    } else if (marker == 0xC4) {  // DHT
      int p = body;
      while (p < end) {
        int tc = d[p] >> 4, th = d[p] & 15;
        p++;
        if (p + 16 > end) return parse_fail(P, R_TRUNC_DHT, p);
        int total = 0;
        for (int i = 0; i < 16; i++) total += d[p + i];
        int bits_pos = p;
        p += 16;
        if (p + total > end) return parse_fail(P, R_TRUNC_DHT, p);
        if (tc < 2) {
          P.huff_pos[tc][th] = bits_pos;
          P.huff_tot[tc][th] = total;
        }
        p += total;
      }
    } else if (marker == 0xC0 || marker == 0xC1 || marker == 0xC2) {  // SOF0/1/2
      if (P.have_sof) return parse_fail(P, R_MULTI_SOF, pos);
      if (body + 6 > n) return parse_fail(P, R_SEGMENT, body);
      P.progressive = marker == 0xC2;
      if (d[body] != 8) return parse_fail(P, R_PRECISION, body);
      P.height = (d[body + 1] << 8) | d[body + 2];
      P.width = (d[body + 3] << 8) | d[body + 4];
      int nc = d[body + 5];
      if (P.height == 0 || P.width == 0) return parse_fail(P, R_ZERO_DIM, body + 1);
      if (nc != 1 && nc != 3) return parse_fail(P, R_NCOMP, body + 5);
      int p = body + 6;
      if (p + 3 * nc > n) return parse_fail(P, R_SEGMENT, p);
      for (int i = 0; i < nc; i++) {
        P.comp_id[i] = d[p];
        P.comp_h[i] = d[p + 1] >> 4;
        P.comp_v[i] = d[p + 1] & 15;
        P.comp_tq[i] = d[p + 2];
        p += 3;
      }
      for (int i = 0; i < nc; i++) {
        int h = P.comp_h[i], v = P.comp_v[i];
        if (!(h == 1 || h == 2 || h == 4) || !(v == 1 || v == 2 || v == 4))
          return parse_fail(P, R_SAMPLING, pos);
      }
      P.ncomp = nc;
      P.have_sof = 1;
    } else if (marker == 0xC3 || marker == 0xC5 || marker == 0xC6 || marker == 0xC7 ||
               marker == 0xC9 || marker == 0xCA || marker == 0xCB || marker == 0xCD ||
               marker == 0xCE || marker == 0xCF) {
      return parse_fail(P, R_SOF_TYPE, pos);
    } else if (marker == 0xDD) {  // DRI
      if (body + 2 > n) return parse_fail(P, R_UNEXPECTED_END, body);
      P.ri = (d[body] << 8) | d[body + 1];
    } else if (marker == 0xDA) {  // SOS
      if (!P.have_sof) return parse_fail(P, R_SOS_BEFORE_SOF, pos);
      if (body >= n) return parse_fail(P, R_SEGMENT, body);
      int ns = d[body], p = body + 1;
      if (p + 2 * ns + 3 > n) return parse_fail(P, R_SEGMENT, p);
      for (int s = 0; s < ns; s++) {
        int cs = d[p], td = d[p + 1] >> 4, ta = d[p + 1] & 15;
        int idx = -1;
        for (int i = 0; i < P.ncomp; i++)
          if (P.comp_id[i] == cs) { idx = i; break; }
        if (idx < 0) return parse_fail(P, R_UNKNOWN_COMP, p);
        if (P.nscans == 0 && s < 4) {
          P.slot_comp[s] = idx;
          P.slot_dpos[s] = P.huff_pos[0][td];
          P.slot_dtot[s] = P.huff_tot[0][td];
          P.slot_apos[s] = P.huff_pos[1][ta];
          P.slot_atot[s] = P.huff_tot[1][ta];
        }
        p += 2;
      }
      if (P.nscans == 0) {
        P.ns = ns;
        P.scan_ri = P.ri;
        P.scan_start = end;
      }
      P.dstart = end;
      P.cmd = 1;
      return;
    }
    P.pos = end;
  }
  if (!P.have_sof || P.nscans == 0) return parse_fail(P, R_NO_IMAGE, P.pos < n ? P.pos : n);
  P.cmd = 0;
}

// ---------------------------------------------------------------------------
// entropy decoding primitives (decode_kernels.py:64-179)

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// Bit reader over the clean stream (big-endian words; k_prep byte-swaps).
// SH: each lane reads through its own 64-byte ring in shared memory, filled
// by cp.async one pair of 16-byte chunks ahead of consumption -- refills are short
// LDS reads with no global latency on the decode chain, and the footprint is
// 64 bytes per lane whatever the payload size.  !SH: plain global loads
// (validation path).  Words past the data read as 0xFF padding
// (_br_fill, decode_kernels.py:64-74): global reads clamp to the last word,
// ring chunks past the data clamp to chunk `cpad` (all 0xFF, k_prep).
template <bool SH>
struct Reader {
  const uint32_t *w;  // global words
  uint32_t wmax;      // last word index (global path)
  uint32_t cpad;      // first all-0xFF 16-byte chunk (ring path)
  uint32_t rs;        // this lane's ring (shared-window address, 16 words)
  uint64_t buf;       // left-aligned bit buffer
  int n;              // valid bits in buf
  uint32_t wi;        // index of the next word to load
  uint32_t p;         // absolute bit position of buf's MSB
  uint32_t nx0, nx1;  // global path: words wi, wi + 1, loaded ahead
  __device__ __forceinline__ uint32_t ld(uint32_t i) const {
    if (SH) return lds_u32(rs + ((i & 15) << 2));
    return __ldg(w + min(i, wmax));
  }
  // ring: 4 chunks of 16 bytes, fetched in pairs (c, c+1), c even, one
  // commit group per pair.  Entering an even chunk c frees the pair (c-2,
  // c-1): fetch (c+2, c+3) into it, then wait until at most that newest pair
  // is pending -- the pair (c, c+1), fetched one pair (~46 units) ago, is done.
  __device__ __forceinline__ void issue_pair(uint32_t c, bool pred) const {
    const uint32_t dst = rs + ((c & 3) << 4);
    const uint32_t *s0 = w + 4 * (size_t)min(c, cpad);
    const uint32_t *s1 = w + 4 * (size_t)min(c + 1, cpad);
    asm volatile(
        "{ .reg .pred q; setp.ne.u32 q, %0, 0;\n"
        "  @q cp.async.cg.shared.global [%1], [%2], 16;\n"
        "  @q cp.async.cg.shared.global [%3], [%4], 16;\n"
        "  cp.async.commit_group;\n"
        "  cp.async.wait_group 1; }" ::"r"((uint32_t)pred),
        "r"(dst), "l"(s0), "r"(dst + 16), "l"(s1)
        : "memory");
  }
  __device__ __forceinline__ void init(uint32_t pos) {
    const uint32_t i = pos >> 5;
    const int off = pos & 31;
    if (SH) {
      // drain this lane's copies still in flight: they target the same slots
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      const uint32_t c = (i >> 2) & ~1u;  // the pair holding word i
#pragma unroll
      for (uint32_t q = 0; q < 4; q++) {
        const uint32_t dst = rs + (((c + q) & 3) << 4);
        const uint32_t *src = w + 4 * (size_t)min(c + q, cpad);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group;\n cp.async.wait_group 0;" ::: "memory");
    }
    buf = (((uint64_t)ld(i) << 32) | ld(i + 1)) << off;
    n = 64 - off;
    wi = i + 2;
    p = pos;
    if (!SH) {
      nx0 = ld(wi);
      nx1 = ld(wi + 1);
    }
    // the ring holds chunks c..c+3 with c = 2*(i/8); if wi already entered
    // the next pair, its crossing fetch (c+4, c+5) is due now
    if (SH && (wi & ~7u) != (i & ~7u)) issue_pair((wi >> 2) + 2, true);
  }
  // keeps >= 33 bits buffered: one unit (code + magnitude) is <= 31 bits
  __device__ __forceinline__ void refill() {
    if (SH) {
      // the next word is read every step, unconditionally (a short LDS, no
      // branch -- in a warp some lane refills almost every step)
      const uint32_t wv = ld(wi);
      const bool rf = n <= 32;
      buf |= rf ? (uint64_t)wv << (32 - n) : 0ull;
      n += rf ? 32 : 0;
      wi += rf ? 1u : 0u;
      const bool cross = rf && (wi & 7) == 0;  // entered an even chunk
      if (cross) issue_pair((wi >> 2) + 2, true);
    } else {
      // two words loaded ahead in registers: a load has ~8 units to land
      const bool rf = n <= 32;
      buf |= rf ? (uint64_t)nx0 << (32 - n) : 0ull;
      n += rf ? 32 : 0;
      if (rf) {
        wi++;
        nx0 = nx1;
        nx1 = ld(wi + 1);
      }
    }
  }
  __device__ __forceinline__ uint32_t hi() const { return (uint32_t)(buf >> 32); }
  __device__ __forceinline__ void skip(int bits) {
    buf <<= bits;
    n -= bits;
    p += bits;
  }
};

// Phase-1 / continuation reader (run_path, the hot loops): a 32-word window
// [lo, lo + 32) of the clean stream per lane in a shared-memory ring, filled
// by cp.async a quarter (8 words) at a time, and three words of it in
// registers: w0 (the word holding bit p), w1, w2.  Per unit: one funnel shift
// for the 32-bit lookahead, and on crossing a word boundary a shift of the
// register words and one LDS of the next (the LDS feeds w2, read two words
// later, off the decode chain).  Ring maintenance runs once per group of
// kGroup units (top_up, the same step for every lane of the warp): quarters
// whose words are all in registers are refetched kRingWords ahead, and the
// lane waits only for the quarters the next group can reach (a group moves p
// by < 8 words; units are at most 31 bits).
constexpr int kRingWords = 32;
constexpr int kGroup = 16;

struct RingReader {
  const uint32_t *w;  // global words
  uint32_t cpad;      // first all-0xFF 16-byte chunk
  uint32_t rs;        // this lane's ring (shared-window address, 128-byte aligned)
  uint32_t w0, w1, w2;
  uint32_t o, qa, p;  // bit offset in w0, 4 x the word index of w2, bit position
  uint32_t lo, pend;  // ring window start (words, multiple of 8); quarters in flight
  __device__ __forceinline__ uint32_t q() const { return (qa >> 2) - 2u; }  // word index of w0
  __device__ __forceinline__ uint32_t ld(uint32_t i) const { return lds_u32(rs + ((i & (kRingWords - 1)) << 2)); }
  // quarter j = words [8j, 8j + 8) = 16-byte chunks 2j, 2j + 1 (clamped to the
  // all-0xFF padding chunk past the data), one commit group
  __device__ __forceinline__ void fetch(uint32_t j, bool pred) const {
    const uint32_t dst = rs + (((8u * j) & (kRingWords - 1)) << 2);
    const uint32_t *s0 = w + 4 * (size_t)min(2u * j, cpad);
    const uint32_t *s1 = w + 4 * (size_t)min(2u * j + 1u, cpad);
    asm volatile(
        "{ .reg .pred q; setp.ne.u32 q, %0, 0;\n"
        "  @q cp.async.cg.shared.global [%1], [%2], 16;\n"
        "  @q cp.async.cg.shared.global [%3], [%4], 16;\n"
        "  @q cp.async.commit_group; }" ::"r"((uint32_t)pred),
        "r"(dst), "l"(s0), "r"(dst + 16), "l"(s1)
        : "memory");
  }
  __device__ __forceinline__ void init(uint32_t pos) {
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // this lane's copies in flight target the ring
    const uint32_t q = pos >> 5;
    qa = 4u * (q + 2u);
    o = pos & 31;
    p = pos;
    lo = q & ~7u;
#pragma unroll
    for (uint32_t j = 0; j < kRingWords / 8; j++) fetch(lo / 8 + j, true);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    pend = 0;
    w0 = ld(q);
    w1 = ld(q + 1);
    w2 = ld(q + 2);
  }
  __device__ __forceinline__ void top_up() {
    // quarters below q + 3 are in registers or consumed: refetch them ahead
    // (a group advances q by at most kGroup words)
    const uint32_t q = this->q();
    const bool f0 = lo + 8 <= q + 3;
    fetch(lo / 8 + kRingWords / 8, f0);
    lo += f0 ? 8u : 0u;
    pend += f0 ? 1u : 0u;
#pragma unroll 1
    while (lo + 8 <= q + 3) {
      fetch(lo / 8 + kRingWords / 8, true);
      lo += 8;
      pend++;
    }
    // the next group loads words up to q + 2 + kGroup: the newest pending
    // quarters starting beyond that may stay in flight, the others must be
    // complete
    const uint32_t top = lo + kRingWords;  // quarter starts: top - 8, top - 16, ...
    const uint32_t reach = q + 2 + kGroup;
    uint32_t allow = 0;
    if (pend >= 1 && top - 8 > reach) allow = 1;
    if (pend >= 2 && top - 16 > reach) allow = 2;
    if (allow < pend) {
      if (allow == 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
      else if (allow == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 2;" ::: "memory");
      pend = allow;
    }
    static_assert(kGroup <= 24, "the ring must hold a group's reach");
  }
  __device__ __forceinline__ uint32_t hi() const { return __funnelshift_l(w1, w0, o); }
  __device__ __forceinline__ void skip(int bits) {
    o += bits;
    p += bits;
    if (o >= 32) {
      o -= 32;
      qa += 4;
      w0 = w1;
      w1 = w2;
      w2 = lds_u32((qa & 4u * (kRingWords - 1)) | rs);
    }
  }
};

// Long codes of a table whose long-code prefixes overflow the sub-tables
// (hostile DHT only): canonical maxcode walk, same symbols as codec.py:272-295.
// Long codes (rare: a divergent branch): second-level table, or the canonical
// maxcode walk for hostile tables with more long-code prefixes than
// sub-tables (same symbols as codec.py:272-295).
__device__ __forceinline__ uint32_t lookup_long(const HuffFast &F, const HuffTab &T, uint32_t e,
                                                uint32_t hi) {
  const uint32_t si = e >> 5, code16 = hi >> 16;
  if (si <= (uint32_t)kSubTabs) return F.sub[((si - 1) << kSubBits) | (code16 & ((1u << kSubBits) - 1))];
#pragma unroll 1
  for (int L = kFastBits + 1; L <= 16; L++) {
    const int c = (int)(code16 >> (16 - L));
    if (c < T.lim[L] && c >= T.first[L]) return huff_entry(T.is_dc, T.vals[T.vptr[L] + c - T.first[L]], L);
  }
  return 0;
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  unsigned short v;
  asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  unsigned short v;
  asm("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}

// Per-image decode context held in registers by every lane.  The table
// offsets d0..a2 are byte offsets into the shared first-level tables
// (kTabStride per table); TS (tables in shared memory) reads those, !TS reads
// the same entries from the global HuffTab array (images using more than
// kSmemTabs tables, and the validation path).  Second-level sub-tables and the
// canonical arrays (long codes, rare) are always read from global memory.
constexpr uint32_t kTabStride = (1u << kFastBits) * 2u;
constexpr int kSmemTabs = 4;
struct EntCtx {
  const uint64_t *gtab;  // the full tables' device addresses (DecodeHead::tab_ptr, shared copy)
  uint32_t tabs_s;      // shared first-level tables, as a shared-window address
  uint32_t zz_s;        // zig-zag -> natural table (shared-window address)
  uint32_t d0, d1, d2, a0, a1, a2;  // byte offsets of the DC / AC table per scan slot
  int c1, c2, bpm, gx;
  uint32_t cbits, limit;
  uint32_t cend;  // end of the range phase 1 covers (N2 estimate; cbits without it)
  const uint32_t *list_lo, *list_hi;  // the unit-list pool incl. overflow sinks (ESSL_CHECK)
  const int16_t *coef_lo, *coef_hi;   // the coefficient scratch (ESSL_CHECK)
  const uint32_t *words;  // clean stream (global)
  uint32_t ring_s;        // this lane's read ring (shared-window address)
  uint32_t stage_s;       // this lane's list staging row (kGroup words, shared-window address)
  uint32_t wmax, cpad;
  __device__ __forceinline__ uint32_t tab_off(int k, int b) const {
    const bool s1 = b >= c1, s2 = b >= c2;
    const uint32_t d = s2 ? d2 : (s1 ? d1 : d0);
    const uint32_t a = s2 ? a2 : (s1 ? a1 : a0);
    return k == 0 ? d : a;
  }
  // first-level entry (tot == 0: long code pointer or invalid)
  template <bool TS>
  __device__ __forceinline__ uint32_t lookup_fast(int k, int b, uint32_t hi) const {
    const uint32_t off = tab_off(k, b);
    if (TS) return lds_u16(tabs_s + off + ((hi >> (32 - kFastBits)) << 1));
    return __ldg(&reinterpret_cast<const HuffTab *>(gtab[off / kTabStride])->fast[hi >> (32 - kFastBits)]);
  }
  __device__ __forceinline__ uint32_t zz(int i) const { return lds_u8(zz_s + (uint32_t)i); }
  __device__ __forceinline__ uint32_t lookup_long(int k, int b, uint32_t e, uint32_t hi) const {
    const HuffTab &T = *reinterpret_cast<const HuffTab *>(gtab[tab_off(k, b) / kTabStride]);
    return essl::lookup_long(*reinterpret_cast<const HuffFast *>(&T), T, e, hi);
  }
  template <bool TS>
  __device__ __forceinline__ uint32_t lookup(int k, int b, uint32_t hi) const {
    uint32_t e = lookup_fast<TS>(k, b, hi);
    if ((e & 31) == 0 && e != 0) e = lookup_long(k, b, e, hi);
    return e;
  }
  template <bool SH>
  __device__ __forceinline__ void reader(Reader<SH> &r, uint32_t pos) const {
    r.w = words;
    r.rs = ring_s;
    r.wmax = wmax;
    r.cpad = cpad;
    r.init(pos);
  }
  __device__ __forceinline__ void reader(RingReader &r, uint32_t pos) const {
    r.w = words;
    r.rs = ring_s;
    r.cpad = cpad;
    r.init(pos);
  }
};

// One decoded unit's fields; bad <=> decode_kernels.py would return status 1
// (invalid code, DC category > 15, or k + run > 63).
#define UNIT_FIELDS(e, k)                                     \
  const int tot = (int)((e) & 31);                            \
  const int kinc = (int)(((e) >> 5) & 127);                   \
  const int size = (int)((e) >> 12);                          \
  const int knew = (k) + kinc;                                \
  const bool bad = tot == 0 || (size != 0 && knew > 64)


// Magnitude bits of a unit, not yet sign-extended (size 0 -> 0): the
// `size` bits after the code, (hi << code_len) >> (32 - size) as one funnel
// shift of (0 : hi << code_len).
__device__ __forceinline__ uint32_t unit_raw(uint32_t hi, int tot, int size) {
  return __funnelshift_l(hi << (tot - size), 0u, size);
}

// JPEG sign extension of `size` magnitude bits (decode_kernels.py:101-108).
__device__ __forceinline__ int extend_raw(uint32_t raw, int size) {
  const uint32_t half = (1u << size) >> 1;
  return raw < half ? (int)raw - (int)((1u << size) - 1u) : (int)raw;
}

// Unit list entry: raw magnitude bits | size << 16 | knew << 20, knew = the
// zig-zag index after the unit (1..127: a DC unit has knew == 1, an AC
// coefficient sits at zig-zag index knew - 1, EOB / ZRL are zeros stored at
// min(knew, 64) - 1, a position the block leaves zero).  Every unit is
// stored; sign extension and the zig-zag -> natural mapping happen in the
// consumers (k_idct), off the decode chain.
__device__ __forceinline__ uint32_t unit_entry(uint32_t raw, int size, int knew) {
  return raw | ((uint32_t)size << 16) | ((uint32_t)knew << 20);
}
__device__ __forceinline__ int entry_value(uint32_t e) { return extend_raw(e & 0xFFFFu, (e >> 16) & 15); }
__device__ __forceinline__ int entry_zz(uint32_t e) { return (int)min(e >> 20, 64u) - 1; }
constexpr uint32_t kEntrySentinel = 1u << 20;  // a DC entry: ends the last block

// Block record: {index of the block's DC entry in the lane's unit list,
// pb = bit position of the block start << 6 | block-in-MCU}.  Every block
// start of a lane's path gets one, so the records double as the path's
// checkpoints: record m of a list is the decoder state after m complete
// blocks (a list always begins at a block start).

// Per-lane record (shared memory).
struct LaneRec {
  // phase 1 (decode from a guess): stop state, blocks, usable block records
  // (checkpoints), list length, lane-0 error
  uint32_t xp, nblk, nck, errp, nlist, nbs;
  int8_t xk, xb, err, ovf, xbe;
};

// Per-lane continuation result and exact-path segment, written after the
// lane's staging row (EntSmem::stage) has served its last group: they live in
// that row.
struct LaneTail {
  // phase 2 (continuation): 0 merged into checkpoint (cj, cm), 1 decode error
  // at cp, 2 end of data at cp (state ek, eb)
  int8_t cst, cbe, ek, eb;
  uint32_t cj, cm, cn, cp, cpb;  // (cpb: the merge record's pb)
  // resolution: the lane's segment of the exact path
  uint32_t w_ord, w_p, w_b, w_A, w_nb;
};

// Phase 1 (CONT=false): decode [p0, send) from the guess (k=0, b=0), storing
// every unit in the lane's list and a record (= checkpoint) at every block
// start.  Lane 0 starts at the exact state, so an error
// there is the reference's error; other lanes re-guess one bit later and drop
// their list and checkpoints (the path before an error is not a decode path),
// except at the end of the data (the fill bits after the final block), where
// the lane simply stops.
// Phase 2 (CONT=true): from the phase-1 stop state, decode on (appending to
// the list) until the path reaches a checkpoint of a later lane with the same
// (bit position, block-in-MCU) at a block start -- two decoders in the same
// state produce the same future -- or errors, or runs off the data.
// Per-group maintenance (ring reader) and per-unit refill (the global-memory
// validation reader keeps its 64-bit buffer topped up before every unit).
__device__ __forceinline__ void top_up_of(Reader<false> &) {}
__device__ __forceinline__ void top_up_of(RingReader &r) { r.top_up(); }
__device__ __forceinline__ void refill_of(Reader<false> &r) { r.refill(); }
__device__ __forceinline__ void refill_of(RingReader &) {}

// A group's list entries go to the lane's shared staging row (one STS per
// unit) and leave in one burst per group: 16-byte stores when the group is
// full and the destination aligned.  Per-unit 4-byte global stores from 32
// lanes to 32 different lists cost 32 L2 writes each and held their address
// registers until the LSU read them (k_entropy alone: +39% without them).
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void flush_stage(const EntCtx &C, uint32_t *lp, uint32_t cnt) {
  ESSL_CHECK(g_check_dec, cnt == 0 || (lp >= C.list_lo && lp + cnt <= C.list_hi), CK_LIST);
  if (cnt == (uint32_t)kGroup && (reinterpret_cast<uintptr_t>(lp) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < kGroup / 4; q++) {
      uint4 v;
      v.x = lds_u32(C.stage_s + 16 * q);
      v.y = lds_u32(C.stage_s + 16 * q + 4);
      v.z = lds_u32(C.stage_s + 16 * q + 8);
      v.w = lds_u32(C.stage_s + 16 * q + 12);
      reinterpret_cast<uint4 *>(lp)[q] = v;
    }
  } else {
#pragma unroll 1
    for (uint32_t i = 0; i < cnt; i++) lp[i] = lds_u32(C.stage_s + 4 * i);
  }
}

template <bool CONT, bool SH>
__device__ void run_path(const EntCtx &C, int lane, int nseq, uint32_t p0, uint32_t sbeg, uint32_t send,
                         uint32_t *list, uint32_t cap, uint2 *bsl, uint32_t bcap, const uint2 *bsl0,
                         uint32_t bstride, LaneRec *Ls, LaneRec &R, LaneTail *T, unsigned int *dbg) {
  // SH: the ring reader (shared-memory window, grouped maintenance); !SH:
  // plain global reads (validation)
  using Rd = typename std::conditional<SH, RingReader, Reader<false>>::type;
  Rd r;
  int k, b;
  uint32_t nblk, nl, nbs;
  int be = 0;
  // continuation cursor over later lanes' block records
  int j = lane + 1;
  uint32_t m = 0, jn = 0, cand = 0xFFFFFFFFu;
  if (CONT) {
    C.reader(r, R.xp);
    k = R.xk;
    b = R.xb;
    nblk = 0;
    nl = R.nlist;
    nbs = R.nbs;
    jn = Ls[j].nck;
    send = C.cend;  // no checkpoint lies beyond the covered range
  } else {
    C.reader(r, p0);
    k = 0;
    b = 0;
    nblk = 0;
    nl = 0;
    nbs = 0;
  }
  auto seek = [&](uint32_t q) {
#pragma unroll 1
    while (true) {
      if (m >= jn) {
        if (++j >= nseq) { cand = 0xFFFFFFFFu; return; }
        m = 0;
        jn = Ls[j].nck;
        continue;
      }
      ESSL_CHECK(g_check_dec, (const uint32_t *)(bsl0 + j * bstride + m) >= C.list_lo &&
                                  (const uint32_t *)(bsl0 + j * bstride + m + 1) <= C.list_hi, CK_CKPT);
      cand = bsl0[j * bstride + m].y;
      if ((cand >> 6) >= q) return;
      m++;
    }
  };
  if (CONT) seek(r.p);
  int st = 2;
  uint32_t dbg_guess = 0;
  if (!CONT && p0 < sbeg) {
    // Warm-up [p0, sbeg): decode only, nothing stored.  The path through it
    // is never part of the exact path through this lane's list: the
    // previous lane's continuation starts at sbeg, so it can only merge at
    // a checkpoint at or after sbeg.  Stop at the first block start at or
    // after sbeg, where the list (and its first record) begins.
    bool stop = false, done = false;
#pragma unroll 1
    while (!done) {
      top_up_of(r);
#pragma unroll 1
      for (int u = 0; u < kGroup; u++) {
        refill_of(r);
        const uint32_t hi = r.hi();
        uint32_t e = C.lookup_fast<SH>(k, b, hi);
        int tot = (int)(e & 31), kinc = (int)((e >> 5) & 127), size = (int)(e >> 12);
        int knew = k + kinc;
        if (tot == 0 || (size != 0 && knew > 64)) {
          if (tot == 0 && e != 0) {
            e = C.lookup_long(k, b, e, hi);
            tot = (int)(e & 31); kinc = (int)((e >> 5) & 127); size = (int)(e >> 12);
            knew = k + kinc;
          }
          if (tot == 0 || (size != 0 && knew > 64)) {  // off the path: re-guess one bit on
            if (r.p + 8 > C.cbits) { stop = true; done = true; break; }
            C.reader(r, r.p + 1);
            dbg_guess++;
            k = 0;
            b = 0;
            nblk = 0;
            break;  // (a fresh ring: maintenance restarts)
          }
        }
        r.skip(tot);
        const bool bend = knew >= 64;
        const int bn = b + 1 == C.bpm ? 0 : b + 1;
        k = bend ? 0 : knew;
        b = bend ? bn : b;
        nblk += bend;
        if (bend && r.p >= sbeg) { done = true; break; }
      }
    }
    if (stop) send = 0;  // the main loop does not run; the lane's path ends here
    nblk = 0;              // (blocks count from the list start)
  }
  // Capacity and the stop position are checked once per group of kGroup
  // units: a group that might not fit stores into the kGroup-slot sinks past
  // the list / record capacities (the lists are then incomplete: ovf), and a
  // lane stops at the end of the group that reaches `send` (decoding a few
  // units further is harmless: the path is the same).
  uint32_t *lp = list + nl;
  uint2 *bp = bsl + nbs;
  bool sink = false;
  uint32_t nrec_ok = 0xFFFFFFFFu;  // records stored before the sinks took over
  bool run = r.p < send;
#pragma unroll 1
  while (run) {
    top_up_of(r);
    if (nl + kGroup > cap || nbs + kGroup > bcap) {
      if (!sink) nrec_ok = nbs;
      lp = list + cap;
      bp = bsl + bcap;
      sink = true;
    }
    uint32_t used = kGroup;  // entries staged this group
#pragma unroll 2
    for (int u = 0; u < kGroup; u++) {
      refill_of(r);
      const uint32_t hi = r.hi();
      uint32_t e = C.lookup_fast<SH>(k, b, hi);
      int tot = (int)(e & 31), kinc = (int)((e >> 5) & 127), size = (int)(e >> 12);
      int knew = k + kinc;
      if (tot == 0 || (size != 0 && knew > 64)) {  // long code or decode error (rare)
        if (tot == 0 && e != 0) {
          e = C.lookup_long(k, b, e, hi);
          tot = (int)(e & 31); kinc = (int)((e >> 5) & 127); size = (int)(e >> 12);
          knew = k + kinc;
        }
        if (tot == 0 || (size != 0 && knew > 64)) {
          if (CONT || lane == 0) {
            st = 1;
            R.errp = r.p;
            run = false;
            used = u;
            break;
          }
          // the last lane reading past the final block into the fill bits /
          // 0xFF padding: its path ends here (keep its list and checkpoints --
          // dropping them would leave nothing for the previous lane to merge
          // into and run that lane's continuation over this whole subsequence)
          if (r.p + 8 > C.cbits) { run = false; used = u; break; }
          C.reader(r, r.p + 1);
          dbg_guess++;
          k = 0;
          b = 0;
          nblk = 0;
          nl = 0;
          nbs = 0;
          lp = list;
          bp = bsl;
          used = 0;
          sink = false;
          nrec_ok = 0xFFFFFFFFu;
          run = r.p < send;
          break;  // (a fresh ring: maintenance restarts)
        }
      }
      const uint32_t raw = unit_raw(hi, tot, size);
      sts_u32(C.stage_s + 4u * (uint32_t)u, unit_entry(raw, size, knew));
      if (k == 0) {  // block record: where the block's units start, the block start state
        ESSL_CHECK(g_check_dec, (const uint32_t *)bp >= C.list_lo && (const uint32_t *)(bp + 1) <= C.list_hi, CK_LIST);
        *bp = make_uint2(nl + (uint32_t)u, (r.p << 6) | (uint32_t)b);
        bp++;
        nbs++;
      }
      r.skip(tot);
      be = knew >= 64;
      const int bn = b + 1 == C.bpm ? 0 : b + 1;
      k = be ? 0 : knew;
      b = be ? bn : b;
      nblk += be;
      if (CONT && be) {
        if ((cand >> 6) < r.p) seek(r.p);
        if (cand == ((r.p << 6) | (uint32_t)b)) { st = 0; run = false; used = u + 1; break; }
      }
    }
    flush_stage(C, lp, used);
    lp += used;
    nl += used;
    if (r.p >= send) run = false;
  }
  const bool ovf = sink;
  asm volatile("cp.async.wait_all;" ::: "memory");  // the ring is reused after phase 2 (DC sums)
  if (CONT) {
    // (the staging row is done: the tail lives there now)
    T->cst = (int8_t)st;
    T->cj = (uint32_t)j;
    T->cm = m;
    T->cpb = cand;
    T->cn = nblk;
    T->cp = st == 1 ? R.errp : r.p;
    T->ek = (int8_t)k;
    T->eb = (int8_t)b;
    T->cbe = (int8_t)be;
    R.nlist = nl;
    R.nbs = nbs;
    if (ovf) R.ovf = 1;
  } else {
    atomicAdd(dbg + 0, nl);  // (units stored in phase 1)
    atomicAdd(dbg + 1, dbg_guess);
    atomicMax(dbg + 2, nl);
    R.err = st == 1;
    R.xp = r.p;
    R.xk = (int8_t)k;
    R.xb = (int8_t)b;
    R.xbe = (int8_t)be;
    R.nblk = nblk;
    R.nck = min(nbs, nrec_ok);  // records a continuation may merge into
    R.nlist = nl;
    R.nbs = nbs;
    R.ovf = ovf;
  }
  ESSL_CHECK(g_check_dec, ovf || (list + nl >= C.list_lo && list + nl < C.list_hi), CK_LIST);
  if (!ovf) list[nl] = kEntrySentinel;  // sentinel: a DC entry ends the last block
}

// Extension of an owner's path past the estimated end of the crop's rows
// (N2: phase 1 and the continuations cover only the bits up to an estimate of
// the position of the crop's last needed block, codec.py:494-498 row_stop).
// Serial decode on the exact path from the path's stop state X, appending
// units and block records to the owner's lists exactly like phase 1, until
// `need` more blocks complete (stops at that block end), a decode error, or
// the end of the data.  Updates X, the list lengths and the block count
// `added`; returns 0 (reached), 1 (error at X.p) or 2 (data ended first).
struct PathEnd {
  uint32_t p;
  int k, b, be;
};

template <bool SH>
__device__ int extend_path(const EntCtx &C, uint32_t *list, uint32_t cap, uint2 *bsl, uint32_t bcap,
                           uint32_t &nlist, uint32_t &nblist, PathEnd &X, uint32_t need,
                           uint32_t &added, int &ovf) {
  Reader<SH> r;
  C.reader(r, X.p);
  int k = X.k, b = X.b, be = X.be;
  uint32_t nl = nlist, nbs = nblist, nblk = 0;
  uint32_t *lp = list + min(nl, cap);
  uint2 *bp = bsl + min(nbs, bcap);
  int st = 2;
#pragma unroll 1
  while (r.p < C.cbits) {
    r.refill();
    const uint32_t hi = r.hi();
    const uint32_t e = C.lookup<SH>(k, b, hi);
    UNIT_FIELDS(e, k);
    if (bad) {
      st = 1;
      break;
    }
    const uint32_t raw = unit_raw(hi, tot, size);
    const bool isdc = k == 0;
    ESSL_CHECK(g_check_dec, lp >= C.list_lo && lp < C.list_hi, CK_LIST);
    *lp = unit_entry(raw, size, knew);
    if (isdc) {
      ESSL_CHECK(g_check_dec, (const uint32_t *)bp >= C.list_lo && (const uint32_t *)(bp + 1) <= C.list_hi, CK_LIST);
      *bp = make_uint2(nl, (r.p << 6) | (uint32_t)b);
      bp += nbs < bcap;
      nbs++;
    }
    lp += nl < cap;
    nl++;
    r.skip(tot);
    be = knew >= 64;
    k = be ? 0 : knew;
    b = be ? (b + 1 == C.bpm ? 0 : b + 1) : b;
    nblk += be;
    if (be && nblk == need) {
      st = 0;
      break;
    }
  }
  X.p = r.p;
  X.k = k;
  X.b = b;
  X.be = be;
  added = nblk;
  nlist = nl;
  nblist = nbs;
  if (nl >= cap || nbs > bcap) ovf = 1;
  else list[nl] = kEntrySentinel;  // sentinel
  return st;
}

// Serial decode from (p, k, b) until `need` more blocks complete or a decode
// error: returns the error's unit position or kNoEnd.  Used to classify a
// stream whose data ends before the crop's last row (corrupt vs truncated).
template <bool SH>
__device__ uint32_t tail_run(const EntCtx &C, uint32_t p, int k, int b, uint32_t need) {
  Reader<SH> r;
  C.reader(r, p);
#pragma unroll 1
  while (need > 0) {
    r.refill();
    const uint32_t e = C.lookup<SH>(k, b, r.hi());
    UNIT_FIELDS(e, k);
    if (bad) return r.p;
    r.skip(tot);
    if (knew >= 64) {
      k = 0;
      b = b + 1 == C.bpm ? 0 : b + 1;
      need--;
    } else {
      k = knew;
    }
  }
  return kNoEnd;
}

struct WriteOut {
  int err, range;
  uint32_t errp;
};

// Crop-window coefficient pointer of block (mx, my, b), or null outside.
__device__ __forceinline__ int16_t *window_block(const DecodeHead &H, int16_t *coef, int mx, int my, int b) {
  if (my < H.my0 || my > H.my1 || mx < H.mx0 || mx > H.mx1) return nullptr;
  const int s = H.blk_slot[b];
  const int c = H.slot_comp[s];
  const int byr = (my - H.my0) * H.slot_v[s] + H.blk_dy[b];
  const int bxr = (mx - H.mx0) * H.slot_h[s] + H.blk_dx[b];
  return coef + H.coef_off[c] + ((uint64_t)byr * H.wbw[c] + bxr) * 64;
}

// Re-decoding write pass (restart intervals, serial mode, list overflow):
// decode `nb` blocks from (p0, k=0, b0) whose absolute block index is A,
// storing crop-window coefficients (natural order, int16); DC predictors
// start from pred[] (decode_kernels.py:150-177).  The block reaching `limit`
// records the bit position after it (p_final).
template <bool SH>
__device__ void write_run(const EntCtx &C, const DecodeHead &H, int16_t *coef, uint32_t p0, int b0,
                          uint32_t A, uint32_t nb, int32_t pred[3], WriteOut &o, uint32_t *p_final) {
  Reader<SH> r;
  C.reader(r, p0);
  int k = 0, b = b0;
  uint32_t blk = A;
  const uint32_t end = A + nb;
  const uint32_t mcu = A / (uint32_t)C.bpm;
  int my = (int)(mcu / (uint32_t)C.gx), mx = (int)(mcu % (uint32_t)C.gx);
  int16_t *cur = window_block(H, coef, mx, my, b);
  int32_t pr0 = pred[0], pr1 = pred[1], pr2 = pred[2];
  o.err = 0;
  o.range = 0;
#pragma unroll 1
  while (blk < end) {
    r.refill();
    const uint32_t hi = r.hi();
    const uint32_t e = C.lookup<SH>(k, b, hi);
    UNIT_FIELDS(e, k);
    if (bad) {
      o.err = 1;
      o.errp = r.p;
      break;
    }
    const int v = extend_raw(unit_raw(hi, tot, size), size);
    if (k == 0) {
      const int s = (b >= C.c1) + (b >= C.c2);
      const int32_t pv = (s == 0 ? pr0 : (s == 1 ? pr1 : pr2)) + v;
      pr0 = s == 0 ? pv : pr0;
      pr1 = s == 1 ? pv : pr1;
      pr2 = s == 2 ? pv : pr2;
      if (cur) {
        if (pv < -32768 || pv > 32767) o.range = 1;
        ESSL_CHECK(g_check_dec, cur >= C.coef_lo && cur + 64 <= C.coef_hi, CK_COEF);
        cur[0] = (int16_t)pv;
      }
    } else if (size != 0 && cur) {
      ESSL_CHECK(g_check_dec, cur >= C.coef_lo && cur + 64 <= C.coef_hi, CK_COEF);
      cur[H.zz[knew - 1]] = (int16_t)v;
    }
    r.skip(tot);
    if (knew >= 64) {
      k = 0;
      blk++;
      b = b + 1 == C.bpm ? 0 : b + 1;
      if (b == 0 && ++mx == C.gx) { mx = 0; my++; }
      if (blk == C.limit && p_final) *p_final = r.p;
      cur = window_block(H, coef, mx, my, b);
    } else {
      k = knew;
    }
  }
  pred[0] = pr0;
  pred[1] = pr1;
  pred[2] = pr2;
}

constexpr int kSegChunk = 8;

// DC pass A over a segment's block records (nb blocks from record `ord`,
// block-in-MCU b0): the segment's DC-difference sums per scan slot.
__device__ void seg_dc_sums(const EntCtx &C, const uint32_t *list, const uint2 *bsl, uint32_t ord, int b0,
                            uint32_t nb, int32_t sum[3]) {
  int b = b0;
  int32_t s0 = 0, s1 = 0, s2 = 0;
  // chunks of kSegChunk blocks: the record loads, then the (dependent) DC
  // entry loads, each batch in flight together
#pragma unroll 1
  for (uint32_t i0 = 0; i0 < nb; i0 += kSegChunk) {
    uint32_t x[kSegChunk], e[kSegChunk];
#pragma unroll
    for (int u = 0; u < kSegChunk; u++) x[u] = i0 + u < nb ? bsl[ord + i0 + u].x : 0u;
#pragma unroll
    for (int u = 0; u < kSegChunk; u++) e[u] = i0 + u < nb ? list[x[u]] : 0u;
#pragma unroll
    for (int u = 0; u < kSegChunk; u++) {
      if (i0 + u < nb) {
        const int32_t v = entry_value(e[u]);
        const int s = (b >= C.c1) + (b >= C.c2);
        s0 += s == 0 ? v : 0;
        s1 += s == 1 ? v : 0;
        s2 += s == 2 ? v : 0;
        b = b + 1 == C.bpm ? 0 : b + 1;
      }
    }
  }
  sum[0] = s0;
  sum[1] = s1;
  sum[2] = s2;
}

// DC pass B: the reference's DC predictor of every block of the segment
// (decode_kernels.py:150-153) continuing from base[]; each crop-window block
// gets its table entry {global unit-list index of its DC entry, DC value} in
// the first 8 bytes of its coefficient slot (k_idct gathers the block from
// the list).
__device__ void seg_table(const EntCtx &C, const DecodeHead &H, int16_t *coef, const uint32_t *list,
                          const uint2 *bsl, uint32_t ord, uint32_t lgbase, int b0, uint32_t A, uint32_t nb,
                          uint32_t nrec, uint32_t nlist, const int32_t base[3], int &range) {
  const uint32_t mcu = A / (uint32_t)C.bpm;
  int my = (int)(mcu / (uint32_t)C.gx), mx = (int)(mcu % (uint32_t)C.gx);
  int b = b0;
  int32_t p0 = base[0], p1 = base[1], p2 = base[2];
#pragma unroll 1
  for (uint32_t i0 = 0; i0 < nb; i0 += kSegChunk) {
    // the chunk's records (+ the next record: where the last block's units
    // end), then their DC entries
    uint32_t x[kSegChunk + 1], e[kSegChunk];
#pragma unroll
    for (int u = 0; u <= kSegChunk; u++) {
      const uint32_t i = i0 + u;
      x[u] = (u < kSegChunk ? i < nb : true) && ord + i < nrec ? bsl[ord + i].x : nlist;
    }
#pragma unroll
    for (int u = 0; u < kSegChunk; u++) e[u] = i0 + u < nb ? list[x[u]] : 0u;
#pragma unroll
    for (int u = 0; u < kSegChunk; u++) {
      if (i0 + u < nb) {
        const int s = (b >= C.c1) + (b >= C.c2);
        const int32_t pv = (s == 0 ? p0 : (s == 1 ? p1 : p2)) + entry_value(e[u]);
        p0 = s == 0 ? pv : p0;
        p1 = s == 1 ? pv : p1;
        p2 = s == 2 ? pv : p2;
        int16_t *cur = window_block(H, coef, mx, my, b);
        if (cur) {
          if (pv < -32768 || pv > 32767) range = 1;
          // the block's AC entries run up to the next block's DC entry (or the
          // list's sentinel): their count rides in the entry's high half
          const uint32_t next = u + 1 < kSegChunk ? (i0 + u + 1 < nb ? x[u + 1] : (ord + i0 + u + 1 < nrec ? bsl[ord + i0 + u + 1].x : nlist)) : x[kSegChunk];
          const uint32_t cnt = min(next - x[u] - 1u, 63u);
          ESSL_CHECK(g_check_dec, cur >= C.coef_lo && cur + 4 <= C.coef_hi, CK_COEF);
          *reinterpret_cast<uint2 *>(cur) = make_uint2(lgbase + x[u], ((uint32_t)pv & 0xFFFFu) | (cnt << 16));
        }
        if (++b == C.bpm) {
          b = 0;
          if (++mx == C.gx) { mx = 0; my++; }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// IDCT, decode_kernels.py:388-534 (islow, exact)

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

template <typename T>
__device__ __forceinline__ void idct_1d(T d0, T d1, T d2, T d3, T d4, T d5, T d6, T d7,
                                        T out[8], T bias, int shift) {
  T z1 = (d2 + d6) * (T)F_0_541196100;
  T t2 = z1 - d6 * (T)F_1_847759065;
  T t3 = z1 + d2 * (T)F_0_765366865;
  T t0 = (d0 + d4) * (T)8192;
  T t1 = (d0 - d4) * (T)8192;
  T t10 = t0 + t3, t13 = t0 - t3, t11 = t1 + t2, t12 = t1 - t2;
  T o0 = d7, o1 = d5, o2 = d3, o3 = d1;
  z1 = o0 + o3;
  T z2 = o1 + o2, z3 = o0 + o2, z4 = o1 + o3;
  T z5 = (z3 + z4) * (T)F_1_175875602;
  o0 *= (T)F_0_298631336; o1 *= (T)F_2_053119869;
  o2 *= (T)F_3_072711026; o3 *= (T)F_1_501321110;
  z1 = -z1 * (T)F_0_899976223; z2 = -z2 * (T)F_2_562915447;
  z3 = -z3 * (T)F_1_961570560 + z5; z4 = -z4 * (T)F_0_390180644 + z5;
  o0 += z1 + z3; o1 += z2 + z4; o2 += z2 + z3; o3 += z1 + z4;
  out[0] = (t10 + o3 + bias) >> shift;
  out[7] = (t10 - o3 + bias) >> shift;
  out[1] = (t11 + o2 + bias) >> shift;
  out[6] = (t11 - o2 + bias) >> shift;
  out[2] = (t12 + o1 + bias) >> shift;
  out[5] = (t12 - o1 + bias) >> shift;
  out[3] = (t13 + o0 + bias) >> shift;
  out[4] = (t13 - o0 + bias) >> shift;
}

// Eight lanes per 8x8 block: lane j owns column j in pass 1 and row j in pass
// 2 (transpose through shared memory).  int32 arithmetic is used when it is
// provably exact: every intermediate of one 1-D pass is a linear form with
// sum|c| <= 61214 (tools/idct_bound.py), so |input| <= 35079 keeps pass 1 and
// |ws| <= 35078 keeps pass 2 below 2^31; otherwise the lane group falls back
// to int64, matching the reference's unbounded ints.
constexpr int kIdctMax1 = 35079;
constexpr int kIdctMax2 = 35078;

__device__ __forceinline__ int grp_max8(int v) {
  v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, 1));
  v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, 2));
  v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, 4));
  return v;
}

// Must be called by all 32 lanes of a warp (lanes with valid=false idle).
// blk: the block's 64 coefficients (natural order, int32, shared memory).
__device__ __forceinline__ void idct_pass2_64(const int64_t w64[8], int32_t *tr, uint32_t &lo,
                                              uint32_t &hi) {
  // int64 transpose through two 32-bit halves, then the int64 row pass
  const int j = threadIdx.x & 7;
  int64_t x[8];
#pragma unroll
  for (int r = 0; r < 8; r++) tr[r * 8 + j] = (int32_t)(uint32_t)(w64[r] & 0xFFFFFFFF);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = (uint32_t)tr[j * 8 + i];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; r++) tr[r * 8 + j] = (int32_t)(w64[r] >> 32);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] |= (int64_t)tr[j * 8 + i] << 32;
  __syncwarp();
  lo = hi = 0;
  if (!(x[1] | x[2] | x[3] | x[4] | x[5] | x[6] | x[7])) {
    int64_t v = ((x[0] + 16) >> 5) + 128;
    uint32_t u = (uint32_t)(v < 0 ? 0 : v > 255 ? 255 : v);
    lo = hi = u * 0x01010101u;
  } else {
    int64_t o[8];
    idct_1d<int64_t>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], o, 131072, 18);
#pragma unroll
    for (int i = 0; i < 8; i++) {
      int64_t v = o[i] + 128;
      uint32_t u = (uint32_t)(v < 0 ? 0 : v > 255 ? 255 : v);
      if (i < 4) lo |= u << (8 * i); else hi |= u << (8 * (i - 4));
    }
  }
}

// Must be called by all 32 lanes of a warp (lanes with valid=false idle).
// blk: the block's 64 dequantised coefficients (natural order, int32,
// shared memory).
__device__ void idct_block_8lanes(bool valid, const int32_t *blk, uint8_t *dst, int pitch,
                                  int32_t *tr /* 64 ints per 8-lane group */) {
  const int j = threadIdx.x & 7;
  int32_t d[8];
  int mabs = 0;
#pragma unroll
  for (int r = 0; r < 8; r++) {
    d[r] = valid ? blk[8 * r + j] : 0;
    mabs = max(mabs, abs(d[r]));
  }
  const bool wide1 = grp_max8(mabs) > kIdctMax1;
  uint32_t lo = 0, hi = 0;
  if (!wide1) {
    // int32 column pass (exact: |input| <= kIdctMax1)
    int32_t w[8];
    if (!(d[1] | d[2] | d[3] | d[4] | d[5] | d[6] | d[7])) {  // DC-only column (exact shortcut)
#pragma unroll
      for (int r = 0; r < 8; r++) w[r] = d[0] * 4;
    } else {
      idct_1d<int32_t>(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], w, 1024, 11);
    }
    int m2 = 0;
#pragma unroll
    for (int r = 0; r < 8; r++) m2 = max(m2, abs(w[r]));
    if (grp_max8(m2) <= kIdctMax2) {
      // transpose: column j -> tr[r*8 + j]; int32 row pass
#pragma unroll
      for (int r = 0; r < 8; r++) tr[r * 8 + j] = w[r];
      __syncwarp();
      int32_t x[8];
#pragma unroll
      for (int i = 0; i < 8; i++) x[i] = tr[j * 8 + i];
      __syncwarp();
      if (!(x[1] | x[2] | x[3] | x[4] | x[5] | x[6] | x[7])) {
        int v = ((x[0] + 16) >> 5) + 128;
        uint32_t u = (uint32_t)(v < 0 ? 0 : v > 255 ? 255 : v);
        lo = hi = u * 0x01010101u;
      } else {
        int32_t o[8];
        idct_1d<int32_t>(x[0], x[1], x[2], x[3], x[4], x[5], x[6], x[7], o, 131072, 18);
#pragma unroll
        for (int i = 0; i < 8; i++) {
          int v = o[i] + 128;
          uint32_t u = (uint32_t)(v < 0 ? 0 : v > 255 ? 255 : v);
          if (i < 4) lo |= u << (8 * i); else hi |= u << (8 * (i - 4));
        }
      }
    } else {
      int64_t w64[8];
#pragma unroll
      for (int r = 0; r < 8; r++) w64[r] = w[r];
      idct_pass2_64(w64, tr, lo, hi);
    }
  } else {
    // the reference's unbounded ints: int64 column pass, int64 row pass
    int64_t w64[8];
    idct_1d<int64_t>(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], w64, 1024, 11);
    idct_pass2_64(w64, tr, lo, hi);
  }
  if (valid) *reinterpret_cast<uint2 *>(dst + (int64_t)j * pitch) = make_uint2(lo, hi);
}

// ---------------------------------------------------------------------------

__device__ __forceinline__ void hdr_status(DecodeHead &H, int st, int reason, int off) {
  if (H.status == 0) {
    H.status = st;
    H.reason = reason;
    H.offset = off;
  }
}

__device__ __forceinline__ int corrupt_offset(const DecodeHead &H, uint32_t errp) {
  // _check_consumed: scan.start + min(vpos, seglen); the reference's reader
  // keeps >= 25 bits buffered, so vpos = ceil((p + 25) / 8) at the failing unit.
  const uint32_t seglen = (uint32_t)(H.scan_end - H.scan_start);
  const uint32_t vpos = (errp + 25 + 7) / 8;
  return H.scan_start + (int)min(vpos, seglen);
}

static_assert(sizeof(DecodeHead) % 16 == 0 && sizeof(HuffTab) % 16 == 0, "hdr copy");

__device__ __forceinline__ DecodeHdr *hdr_of(const Scratch &s, int img) {
  return reinterpret_cast<DecodeHdr *>(s.hdr) + img;
}

// ===========================================================================
// k_prep: CRC, parse, destuff, tables, window zeroing (one CTA per image)
// ===========================================================================
template <bool SMEM>
__global__ void __launch_bounds__(kNT, 4) k_prep(DecodeParams P) {
  TraceScope trace_(P.trace, ESSL_K_PREP);
  extern __shared__ __align__(16) uint8_t dyn[];  // [payload (SMEM)][CRC chunk partials]
  __shared__ PrepSmem S;
  DecodeHead &H = S.h;
  const int img = blockIdx.x;
  const int tid = threadIdx.x;
  DecodeHdr *G = hdr_of(P.s, img);  // tables are built here directly
  uint32_t *crc_part = reinterpret_cast<uint32_t *>(dyn + P.prep_part_off);
  const essl_sample smp = P.samples[img];
  const uint8_t *g = P.blob + smp.offset;
  const int n = (int)smp.length;
  const int n_pad = (n + 15) / 16 * 16 + 16;
  ImgInfo *info = P.s.info + img;
  const uint8_t *raw = SMEM ? dyn : g;
  PayloadView pv{raw, n};

  if (tid < 64) H.zz[tid] = c_zz[tid];
  if (tid == 0) {
    S.t0 = clock64();
    H.status = 0; H.reason = 0; H.offset = -1;
    H.ntab = 0; H.ns = 0; H.ncomp = 0; H.quant_missing = -1;
    H.limit_blocks = 0; H.clean_bits = 0; H.clean_words = 0; H.scan_ri = 0; H.wmax = 0; H.cpad = 0;
    H.multiscan = 0; H.progressive = 0;
  }
  // ---- stage the payload into shared memory (16-byte loads) ----------------
  if (SMEM) {
    if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
      const int n16 = n / 16;
      const int4 *src = reinterpret_cast<const int4 *>(g);
      int4 *dst = reinterpret_cast<int4 *>(dyn);
      for (int i = tid; i < n16; i += kNT) dst[i] = __ldg(src + i);
      for (int i = n16 * 16 + tid; i < n; i += kNT) dyn[i] = g[i];
    } else {
      for (int i = tid; i < n; i += kNT) dyn[i] = g[i];
    }
    for (int i = n + tid; i < n_pad; i += kNT) dyn[i] = 0;
  }
  for (int e = tid; e < 256; e += kNT) {  // CRC tables (slice-by-4)
    uint32_t c = e;
#pragma unroll
    for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    S.crc.T[0][e] = c;
  }
  __syncthreads();
  for (int e = tid; e < 256; e += kNT) {
    uint32_t c = S.crc.T[0][e];
#pragma unroll
    for (int t = 1; t < 4; t++) {
      c = (c >> 8) ^ S.crc.T[0][c & 0xFF];
      S.crc.T[t][e] = c;
    }
  }
  __syncthreads();

  // ---- CRC32 (container.py:263) -------------------------------------------
  // The message is zero-prepended to C2 (a power of two) chunks of 132 bytes
  // (leading zeros do not change a zero-init CRC); the 0xFFFFFFFF init is
  // applied by complementing the first 4 message bytes.  Chunk CRCs
  // (slice-by-4) combine in a binary tree; the left operand is multiplied by
  // x^(8 * 132 * 2^j) mod P through precomputed byte tables (GF(2)-linear).
  if (tid == 0) S.ph[0] = clock64();
  if (smp.check_crc) {
    const int C = (n + kCrcChunk - 1) / kCrcChunk;
    int C2 = 1, lv = 0;
    while (C2 < C) { C2 <<= 1; lv++; }
    uint32_t crc = 0;
    if (n < 4 || C2 > kCrcMaxChunks) {
      if (tid == 0) {  // tiny or huge payloads: serial bytewise CRC
        uint32_t c = 0xFFFFFFFFu;
        for (int i = 0; i < n; i++) c = S.crc.T[0][(c ^ raw[i]) & 0xFF] ^ (c >> 8);
        crc = c ^ 0xFFFFFFFFu;
      }
    } else {
      const int Z = C2 * kCrcChunk - n;
      for (int ch = tid; ch < C2; ch += kNT) {
        uint32_t c = 0;
        const int base = ch * kCrcChunk - Z;
        if (SMEM && base >= 4 && base + kCrcChunk <= n) {
          // a chunk inside the message past its first 4 bytes: its words
          // come from aligned shared-memory words by one funnel shift each
          // (kCrcChunk is a multiple of 4, so every chunk has the same shift)
          const uint32_t *w32 = reinterpret_cast<const uint32_t *>(raw) + (base >> 2);
          const uint32_t sh = 8u * (uint32_t)(base & 3);
          uint32_t lo = w32[0];
#pragma unroll 3
          for (int j = 0; j < kCrcChunk / 4; j++) {
            const uint32_t hi = w32[j + 1];
            c ^= __funnelshift_r(lo, hi, sh);
            lo = hi;
            c = S.crc.T[3][c & 0xFF] ^ S.crc.T[2][(c >> 8) & 0xFF] ^ S.crc.T[1][(c >> 16) & 0xFF] ^
                S.crc.T[0][c >> 24];
          }
        } else if (base + kCrcChunk > 0) {
#pragma unroll 3
          for (int j = 0; j < kCrcChunk; j += 4) {
            uint32_t w = 0;
#pragma unroll
            for (int b = 0; b < 4; b++) {
              const int r = base + j + b;
              uint32_t byte = r >= 0 ? raw[r] : 0u;
              if (r >= 0 && r < 4) byte ^= 0xFF;
              w |= byte << (8 * b);
            }
            c ^= w;
            c = S.crc.T[3][c & 0xFF] ^ S.crc.T[2][(c >> 8) & 0xFF] ^ S.crc.T[1][(c >> 16) & 0xFF] ^
                S.crc.T[0][c >> 24];
          }
        }
        crc_part[ch] = c;
      }
      __syncthreads();
      const uint32_t *M = c_crc_mul;
#pragma unroll 1
      for (int j = 0; j < lv; j++) {
        const int stride = 1 << j;
        const uint32_t *T = M + j * 1024;
        for (int i = tid * 2 * stride; i < C2; i += kNT * 2 * stride) {
          const uint32_t a = crc_part[i];
          const uint32_t m = __ldg(T + (a & 0xFF)) ^ __ldg(T + 256 + ((a >> 8) & 0xFF)) ^
                             __ldg(T + 512 + ((a >> 16) & 0xFF)) ^ __ldg(T + 768 + (a >> 24));
          crc_part[i] = m ^ crc_part[i + stride];
        }
        __syncthreads();
      }
      crc = crc_part[0] ^ 0xFFFFFFFFu;
    }
    if (tid == 0 && crc != smp.crc32) hdr_status(H, ESSL_ST_CRC, 0, -1);
  }
  __syncthreads();
  if (tid == 0) S.ph[1] = clock64();

  // ---- parse (thread 0) + parallel entropy-segment end search --------------
  ParseState &PS = S.ps;
  if (tid == 0) {
    PS.pos = 2; PS.n = n; PS.ri = 0; PS.have_sof = 0; PS.progressive = 0;
    PS.ncomp = 0; PS.nscans = 0; PS.status = 0; PS.cmd = 0; PS.ns = 0;
    PS.scan_start = 0; PS.scan_end = 0; PS.scan_ri = 0; PS.width = 0; PS.height = 0;
    for (int i = 0; i < 16; i++) { PS.quant_pos[i] = -1; PS.huff_pos[0][i] = -1; PS.huff_pos[1][i] = -1; }
    if (n < 4 || raw[0] != 0xFF || raw[1] != 0xD8) parse_fail(PS, R_NO_SOI, 0);
    else PS.cmd = 3;  // continue
  }
  __syncthreads();
  if (H.status == 0) {
#pragma unroll 1
    while (true) {
      if (tid == 0 && PS.cmd != 2) parse_until_sos(PS, pv);
      __syncthreads();
      if (PS.cmd != 1) break;
      // entropy_end (codec.py:109-121): the first FF followed by a byte that
      // is not 00, RSTn or FF.  For the first scan the same pass finds where
      // destuff_scan stops (decode_kernels.py:27-61): the first FF followed by
      // a byte that is not 00 or RSTn (FF FF fill bytes end the clean data).
      const bool first = PS.nscans == 0;
      if (tid == 0) { S.stop = n; if (first) S.dstop = n; }
      __syncthreads();
      const int d0 = PS.dstart;
      for (int r0 = d0 & ~15; r0 < n - 1; r0 += kNT * 16) {
        const int g0 = r0 + tid * 16;
        const int a = max(g0, d0), e = min(g0 + 16, n - 1);
        if (a >= e) continue;
        // 16 bytes per thread per round: one 16-byte shared load filters out
        // the (common) groups without an FF byte
        bool d_found = !first;
        if (SMEM) {
          const uint4 v = *reinterpret_cast<const uint4 *>(raw + g0);
          if (!any_ff4(v)) continue;
          // exact FF positions of the group inside [a, e), then only those
          const uint32_t w[4] = {v.x, v.y, v.z, v.w};
          uint32_t ffm = 0;
#pragma unroll
          for (int k = 0; k < 4; k++) ffm |= byte_flags(zero_bytes(~w[k])) << (4 * k);
          ffm &= ((1u << (e - g0)) - 1u) & ~((1u << (a - g0)) - 1u);
#pragma unroll 1
          for (; ffm; ffm &= ffm - 1) {
            const int i = g0 + __ffs(ffm) - 1;
            const int m = raw[i + 1];
            if (m == 0x00 || is_rst(m)) continue;
            if (!d_found) { atomicMin(&S.dstop, i); d_found = true; }
            if (m != 0xFF) { atomicMin(&S.stop, i); break; }
          }
          continue;
        }
        for (int i = a; i < e; i++) {
          if (raw[i] != 0xFF) continue;
          const int m = raw[i + 1];
          if (m == 0x00 || is_rst(m)) continue;
          if (!d_found) { atomicMin(&S.dstop, i); d_found = true; }
          if (m != 0xFF) { atomicMin(&S.stop, i); break; }
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (PS.nscans == 0) PS.scan_end = S.stop;
        PS.nscans++;
        PS.pos = S.stop;
        PS.cmd = 3;
      }
      __syncthreads();
    }
    if (tid == 0 && PS.cmd == 2) hdr_status(H, PS.status, PS.reason, PS.offset);
  }
  __syncthreads();

  // ---- geometry, validation (codec.py:254-265, 448-482) --------------------
  if (tid == 0) {
    int hmax = 1, vmax = 1;
    for (int i = 0; i < PS.ncomp; i++) {
      hmax = max(hmax, PS.comp_h[i]);
      vmax = max(vmax, PS.comp_v[i]);
    }
    const int W = PS.width, Hh = PS.height;
    info->width = W; info->height = Hh; info->ncomp = PS.ncomp;
    info->hmax = hmax; info->vmax = vmax;
    for (int i = 0; i < 3; i++) {
      info->comp_h[i] = i < PS.ncomp ? PS.comp_h[i] : 1;
      info->comp_v[i] = i < PS.ncomp ? PS.comp_v[i] : 1;
    }
    info->rx = smp.x; info->ry = smp.y; info->rw = smp.w; info->rh = smp.h;
    info->flip = smp.flip;
    H.ncomp = PS.ncomp;
    H.scan_ri = PS.scan_ri;
    H.scan_start = PS.scan_start;
    H.scan_end = PS.scan_end;
    if (H.status == 0) {
      const int mcus_x = (W + 8 * hmax - 1) / (8 * hmax), mcus_y = (Hh + 8 * vmax - 1) / (8 * vmax);
      for (int i = 0; i < PS.ncomp; i++) {
        const int cw = (W * PS.comp_h[i] + hmax - 1) / hmax, ch = (Hh * PS.comp_v[i] + vmax - 1) / vmax;
        H.bw[i] = (cw + 7) / 8;
        H.bh[i] = (ch + 7) / 8;
      }
      const int x = smp.x, y = smp.y, w = smp.w, h = smp.h;
      if (w < 1 || h < 1 || x < 0 || y < 0 || x + w > W || y + h > Hh) {
        hdr_status(H, ESSL_ST_RECT, 0, -1);
      } else if (PS.progressive || PS.nscans != 1 || PS.ns != PS.ncomp) {
        // the reference's full-decode fallback (codec.py:461-469): every scan
        // decoded in full into full coefficient arrays [BH][BW][64] per
        // component (int16, carved here), the crop window reconstructed from
        // them; stats count every MCU (codec.py:466-469)
        H.multiscan = 1;
        H.progressive = PS.progressive;
        H.gx = mcus_x;
        H.gy = mcus_y;
        const int mcu_w = 8 * hmax, mcu_h = 8 * vmax;
        H.mx0 = x / mcu_w; H.mx1 = (x + w - 1) / mcu_w;
        H.my0 = y / mcu_h; H.my1 = (y + h - 1) / mcu_h;
        H.row_stop = mcus_y;
        const int total_mcus = PS.ncomp > 1 ? mcus_x * mcus_y : H.bw[0] * H.bh[0];
        info->mcus_entropy = total_mcus;
        info->mcus_recon = total_mcus;
        uint64_t total = 0;
        for (int c = 0; c < 3; c++) {
          H.wbh[c] = 0; H.wbw[c] = 0; H.wby0[c] = 0; H.wbx0[c] = 0; H.coef_off[c] = 0;
          H.coef_pitch[c] = 0; H.comp_hv[c] = 0; H.comp_id[c] = -1;
        }
        for (int c = 0; c < PS.ncomp; c++) {
          const int BW = mcus_x * PS.comp_h[c], BH = mcus_y * PS.comp_v[c];
          H.comp_hv[c] = (PS.comp_h[c] << 4) | PS.comp_v[c];
          H.comp_id[c] = PS.comp_id[c];
          H.wby0[c] = H.my0 * PS.comp_v[c];
          H.wbx0[c] = H.mx0 * PS.comp_h[c];
          H.wbh[c] = (H.my1 - H.my0 + 1) * PS.comp_v[c];
          H.wbw[c] = (H.mx1 - H.mx0 + 1) * PS.comp_h[c];
          H.coef_pitch[c] = BW;
          H.coef_off[c] = total;
          total += (uint64_t)BH * BW * 64;
        }
        const unsigned long long cbase = atomicAdd(&P.s.counters[1], (unsigned long long)total);
        if (cbase + total > P.s.coef_cap) {
          hdr_status(H, ESSL_ST_CAPACITY, R_SCRATCH, -1);
        } else {
          for (int c = 0; c < 3; c++) H.coef_off[c] += cbase;
          H.coef_base = cbase;
        }
        for (int i = 0; i < PS.ncomp; i++) {
          const int tq = PS.comp_tq[i];
          if (tq > 15 || PS.quant_pos[tq] < 0) { H.quant_missing = tq; break; }
        }
      } else {
        const int ns = PS.ns;
        H.ns = ns;
        int mcu_w, mcu_h;
        if (ns == 1) {
          H.gx = H.bw[PS.slot_comp[0]];
          H.gy = H.bh[PS.slot_comp[0]];
          mcu_w = mcu_h = 8;
        } else {
          H.gx = mcus_x;
          H.gy = mcus_y;
          mcu_w = 8 * hmax;
          mcu_h = 8 * vmax;
        }
        int bpm = 0;
        for (int s = 0; s < ns; s++) {
          const int c = PS.slot_comp[s];
          const int hh = ns > 1 ? PS.comp_h[c] : 1, vv = ns > 1 ? PS.comp_v[c] : 1;
          H.slot_comp[s] = c; H.slot_h[s] = hh; H.slot_v[s] = vv; H.slot_nb[s] = hh * vv;
          for (int dy = 0; dy < vv; dy++)
            for (int dx = 0; dx < hh; dx++) {
              H.blk_slot[bpm] = s; H.blk_dy[bpm] = dy; H.blk_dx[bpm] = dx;
              bpm++;
            }
        }
        for (int s = ns; s < 4; s++) { H.slot_nb[s] = 64; H.slot_comp[s] = 0; H.slot_h[s] = 1; H.slot_v[s] = 1; }
        H.bpm = bpm;
        H.mx0 = x / mcu_w; H.mx1 = (x + w - 1) / mcu_w;
        H.my0 = y / mcu_h; H.my1 = (y + h - 1) / mcu_h;
        H.row_stop = H.my1 + 1;
        H.limit_blocks = (uint32_t)H.row_stop * H.gx * bpm;
        info->mcus_entropy = H.row_stop * H.gx;
        info->mcus_recon = (H.my1 - H.my0 + 1) * (H.mx1 - H.mx0 + 1);
        uint64_t total = 0;
        for (int c = 0; c < 3; c++) { H.wbh[c] = 0; H.wbw[c] = 0; H.wby0[c] = 0; H.wbx0[c] = 0; H.coef_off[c] = 0; }
        for (int s = 0; s < ns; s++) {
          const int c = H.slot_comp[s];
          H.wby0[c] = H.my0 * H.slot_v[s];
          H.wbx0[c] = H.mx0 * H.slot_h[s];
          H.wbh[c] = (H.my1 - H.my0 + 1) * H.slot_v[s];
          H.wbw[c] = (H.mx1 - H.mx0 + 1) * H.slot_h[s];
          H.coef_off[c] = total;
          H.coef_pitch[c] = H.wbw[c];
          total += (uint64_t)H.wbh[c] * H.wbw[c] * 64;
        }
        const unsigned long long cbase = atomicAdd(&P.s.counters[1], (unsigned long long)total);
        if (cbase + total > P.s.coef_cap) {
          hdr_status(H, ESSL_ST_CAPACITY, R_SCRATCH, -1);
        } else {
          for (int c = 0; c < 3; c++) H.coef_off[c] += cbase;
          H.coef_base = cbase;
        }
        // global region: clean bytes + restart table
        const int seglen = PS.scan_end - PS.scan_start;
        H.max_restarts = PS.scan_ri ? (H.gx * H.gy) / PS.scan_ri : 0;
        const int max_r = PS.scan_ri ? H.max_restarts + 2 : 0;
        const uint64_t clean_bytes = ((uint64_t)seglen + 64 + 15) / 16 * 16;
        const uint64_t alloc = (clean_bytes + 4ull * max_r + 16 + 15) / 16 * 16;
        const unsigned long long base = atomicAdd(&P.s.counters[0], (unsigned long long)alloc);
        if (base + alloc > P.s.clean_cap) hdr_status(H, ESSL_ST_CAPACITY, R_SCRATCH, -1);
        H.clean_off = base;
        H.rst_off = (uint32_t)(clean_bytes / 4);
        // dequantisation tables (the reference checks them after decoding)
        for (int i = 0; i < PS.ncomp; i++) {
          const int tq = PS.comp_tq[i];
          if (tq > 15 || PS.quant_pos[tq] < 0) { H.quant_missing = tq; break; }
        }
      }
    }
  }
  __syncthreads();
  if (H.status == 0) {
    for (int e = tid; e < PS.ncomp * 64; e += kNT) {
      const int c = e >> 6, k = e & 63;
      const int tq = PS.comp_tq[c];
      const int pos = tq <= 15 ? PS.quant_pos[tq] : -1;
      int v = 0;
      if (pos >= 0) v = PS.quant_pq[tq] == 1 ? ((raw[pos + 2 * k] << 8) | raw[pos + 2 * k + 1]) : raw[pos + k];
      G->q[c][c_zz[k]] = v;
    }
  }

  if (tid == 0) S.ph[2] = clock64();
  // ---- destuff (decode_kernels.py:27-61), in place in shared memory (the
  //      clean stream overwrites the scan bytes it came from: every kept byte
  //      moves to a position <= its own), then one coalesced copy to the
  //      global clean region ---------------------------------------------------
  uint8_t *gclean = P.s.clean + H.clean_off;
  uint8_t *clean = SMEM ? dyn + (PS.scan_start & ~15) : gclean;
  if (tid == 0) {
    S.save_lo = SMEM && H.status == 0 && !H.multiscan ? (PS.scan_start & ~15) : 0;
    S.save_hi = SMEM && H.status == 0 && !H.multiscan ? PS.scan_start : 0;
  }
  if (SMEM && tid < 16 && H.status == 0 && !H.multiscan && (PS.scan_start & ~15) + tid < PS.scan_start)
    S.save[tid] = raw[(PS.scan_start & ~15) + tid];
  __syncthreads();
  if (H.status == 0 && !H.multiscan) {
    // Rounds of kNT x 16 bytes: thread t owns bytes [16t, 16t+16) of the
    // round (16-byte shared loads, conflict-free); a block scan per round
    // places the kept bytes.
    const int seg0 = PS.scan_start, seg1 = PS.scan_end;
    constexpr int kRound = kNT * 16;
    // where destuff_scan stops: found by the entropy-end pass (first FF not
    // followed by 00 / RSTn), or the segment's last byte when that is an FF
    // (decode_kernels.py:37-38: `if i + 1 >= n: break`)
    if (tid == 0) {
      int st = min(S.dstop, seg1);
      if (st == seg1 && seg1 > seg0 && raw[seg1 - 1] == 0xFF) st = seg1 - 1;
      S.stop = st;
      S.carry = 0;
    }
    __syncthreads();
    const int rbeg = seg0 & ~15;  // rounds start 16-byte aligned (uint4 loads)
    const int stop = S.stop;
    const int max_r = PS.scan_ri ? H.max_restarts + 2 : 0;
    uint32_t *rst_tab = reinterpret_cast<uint32_t *>(gclean) + H.rst_off;
    uint32_t kbase = 0, rbase = 0;
    for (int r0 = rbeg; r0 < stop; r0 += kRound) {
      const int g0 = r0 + tid * 16;
      const int a = max(g0, seg0), e = min(g0 + 16, stop);
      // this thread's 16 input bytes, the byte before and the byte after, in
      // registers before any thread of the round writes
      uint32_t w[4] = {0, 0, 0, 0};
      int prev = 0, next = 0;
      if (g0 < stop) {
        if (SMEM) {
          const uint4 v = *reinterpret_cast<const uint4 *>(raw + g0);
          w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
        } else {
#pragma unroll
          for (int q = 0; q < 16; q++) w[q >> 2] |= (uint32_t)raw[g0 + q] << (8 * (q & 3));
        }
        prev = tid == 0 ? S.carry : (g0 > 0 ? raw[g0 - 1] : 0);  // (thread 0: saved by the last round)
        next = raw[g0 + 16];
      }
      // bit masks over the group (bit q = byte g0 + q): destuff_scan keeps a
      // byte unless it follows an FF (the 00 of FF00, the marker byte of an
      // RSTn) or is the FF of an RSTn, which records a restart offset
      uint32_t range = 0, keep = 0, rstm = 0;
      bool fast = false;
      if (a < e) {
        range = ((1u << (e - g0)) - 1u) & ~((1u << (a - g0)) - 1u);
        uint32_t ffm, rsm;
        group_masks(w, ffm, rsm);
        fast = ffm == 0 && !(a > seg0 && prev == 0xFF) && range == 0xFFFFu;
        // (i > seg0 && previous byte FF); the segment's first byte never is
        uint32_t second = ((ffm << 1) | (prev == 0xFF ? 1u : 0u)) & 0xFFFFu;
        if (a == seg0) second &= ~(1u << (a - g0));
        rstm = ffm & ((rsm >> 1) | (is_rst(next) ? 0x8000u : 0u)) & range;
        keep = range & ~second & ~rstm;
      }
      uint32_t cnt[4] = {(uint32_t)__popc(keep), (uint32_t)__popc(rstm), 0, 0}, tot[4];
      block_scan4(S.warp_tot, cnt, tot);  // (barriers: every read above is done)
      if (tid == kNT - 1) S.carry = (w[3] >> 24) & 0xFF;  // the round's last input byte
      uint32_t kept = kbase + cnt[0], nrst = rbase + cnt[1];
      if (fast) {
#pragma unroll
        for (int q = 0; q < 16; q++) clean[kept + q] = (uint8_t)(w[q >> 2] >> (8 * (q & 3)));
      } else {
        const uint32_t base = kept;
#pragma unroll 1
        for (uint32_t m = rstm; m; m &= m - 1) {  // restart offsets (clean position of the marker)
          const int q = __ffs(m) - 1;
          if ((int)nrst < max_r) rst_tab[nrst] = base + __popc(keep & ((1u << q) - 1u));
          nrst++;
        }
#pragma unroll
        for (int q = 0; q < 16; q++) {  // (predicated stores: no per-byte branches)
          if ((keep >> q) & 1u) clean[kept++] = (uint8_t)(w[q >> 2] >> (8 * (q & 3)));
        }
      }
      kbase += tot[0];
      rbase += tot[1];
      __syncthreads();  // writes of this round before the next round's reads
    }
    const uint32_t tk = kbase, tr = rbase;
    __syncthreads();
    // 0xFF padding past the end (_br_fill), >= 2 whole words; the clean
    // stream goes to global as big-endian words (the bit reader's order)
    // (48 bytes: at least two whole words and one whole 16-byte chunk)
    if (tid < 48) clean[tk + tid] = 0xFF;
    __syncthreads();
    const int nwords = (int)((tk + 48) / 4);
    if (tid == 0) {
      const uint64_t clean_bytes = ((uint64_t)(PS.scan_end - PS.scan_start) + 64 + 15) / 16 * 16;
      ESSL_CHECK(g_check_dec, (uint64_t)(nwords + 3) / 4 * 16 <= clean_bytes, CK_CLEAN);
      ESSL_CHECK(g_check_dec, H.clean_off + clean_bytes <= P.s.clean_cap, CK_CLEAN);
    }
    if (SMEM) {
      const int n16 = (nwords + 3) / 4;
      const uint4 *src = reinterpret_cast<const uint4 *>(clean);
      uint4 *dst = reinterpret_cast<uint4 *>(gclean);
      for (int i = tid; i < n16; i += kNT) {
        uint4 v = src[i];
        v.x = __byte_perm(v.x, 0, 0x0123); v.y = __byte_perm(v.y, 0, 0x0123);
        v.z = __byte_perm(v.z, 0, 0x0123); v.w = __byte_perm(v.w, 0, 0x0123);
        dst[i] = v;
      }
    } else {
      uint32_t *w = reinterpret_cast<uint32_t *>(gclean);
      for (int i = tid; i < nwords; i += kNT) w[i] = __byte_perm(w[i], 0, 0x0123);
    }
    if (tid == 0) {
      H.clean_bits = tk * 8;
      H.wmax = (uint32_t)nwords - 1;
      H.cpad = (tk + 15) / 16;
      H.clean_words = (tk + 3) / 4;
      H.n_restarts = (int)tr;
      if (PS.scan_ri == 0 && tr > 0) hdr_status(H, ESSL_ST_MALFORMED, R_RST_NO_DRI, seg0);
      else if ((int)tr > H.max_restarts + 2) hdr_status(H, ESSL_ST_MALFORMED, R_TOO_MANY_RST, seg0);
    }
  }
  __syncthreads();
  if (tid == 0) S.ph[3] = clock64();

  // ---- Huffman tables (codec.py:272-304): DC slots first, then AC ----------
  // 1. thread 0 maps the scan's slots to distinct (class, id) tables;
  // 2. each table is looked up in the context's table cache (slot t = the
  //    t-th distinct table; same class + DHT counts + symbols -> copy);
  // 3. thread 0 derives the canonical first/lim/vptr of the tables that
  //    missed (and the kFastBits-bit prefixes of their long codes, which get
  //    second-level sub-tables); 4. all threads fill the lookup tables.
  __shared__ int s_tpos[kMaxTables], s_ttot[kMaxTables], s_tdc[kMaxTables], s_hit[kMaxTables];
  if (tid == 0 && H.status == 0) {
    int ntab = 0;
    int slot_dc[4] = {0, 0, 0, 0}, slot_ac[4] = {0, 0, 0, 0};
    for (int pass = 0; pass < 2 && H.status == 0; pass++) {
      for (int s = 0; s < H.ns && H.status == 0; s++) {
        const int pos = pass == 0 ? PS.slot_dpos[s] : PS.slot_apos[s];
        const int tot = pass == 0 ? PS.slot_dtot[s] : PS.slot_atot[s];
        if (pos < 0) { hdr_status(H, ESSL_ST_HUFFTABLE, R_HUFF_UNDEFINED, -1); break; }
        if (tot > 256) { hdr_status(H, ESSL_ST_HUFFTABLE, R_HUFF_TOO_MANY, -1); break; }
        int ti = -1;
        for (int t = 0; t < ntab; t++) if (s_tpos[t] == pos) ti = t;
        if (ti < 0) {
          ti = ntab++;
          s_tpos[ti] = pos;
          s_ttot[ti] = tot;
          s_tdc[ti] = pass == 0;
        }
        if (pass == 0) slot_dc[s] = ti; else slot_ac[s] = ti;
      }
    }
    H.ntab = ntab;
    uint32_t w = 0;
    for (int q = 0; q < 3; q++) w |= (uint32_t)(slot_dc[q] & 15) << (4 * q);
    for (int q = 0; q < 3; q++) w |= (uint32_t)(slot_ac[q] & 15) << (4 * (q + 3));
    H.tab_index_word = w;
  }
  __syncthreads();
  TabCacheSlot *cache = reinterpret_cast<TabCacheSlot *>(P.s.tabcache);
  if (H.status == 0) {
    for (int t = 0; t < H.ntab; t++) {
      const int len = 16 + s_ttot[t], pos = s_tpos[t];
      TabCacheSlot &C = cache[t];
      unsigned int st;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(st) : "l"(&C.state) : "memory");
      bool eq = st == 2u && C.len == len && C.is_dc == s_tdc[t];
      for (int i = tid; eq && i < len; i += kNT) eq = C.key[i] == seg_byte(S, raw, pos + i);
      const int hit = __syncthreads_and(eq);
      // a hit is used in place (slots are written once, never replaced)
      if (tid == 0) {
        s_hit[t] = hit;
        H.tab_ptr[t] = hit ? reinterpret_cast<uint64_t>(&C.tab) : reinterpret_cast<uint64_t>(&G->tab[t]);
      }
    }
  }
  __syncthreads();
  if (tid == 0 && H.status == 0) {
    for (int ti = 0; ti < H.ntab && H.status == 0; ti++) {
      if (s_hit[ti]) continue;
      const int pos = s_tpos[ti];
      HuffTab &T = G->tab[ti];
      int code = 0, vi = 0;
      T.lim[0] = 0; T.first[0] = 0; T.vptr[0] = 0;
      int nsub = 0, last = -1;
      for (int L = 1; L <= 16; L++) {
        const int cnt = seg_byte(S, raw, pos + L - 1);
        T.first[L] = code;
        T.vptr[L] = (int16_t)vi;
        if (cnt && code + cnt > (1 << L)) { hdr_status(H, ESSL_ST_HUFFTABLE, R_HUFF_OVERFLOW, -1); break; }
        // distinct kFastBits-bit prefixes of the long codes, in code order
        if (L > kFastBits)
          for (int c = code; c < code + cnt; c++) {
            const int pf = c >> (L - kFastBits);
            if (pf != last) {
              if (nsub < kSubTabs) S.sub_pf[ti][nsub] = (uint16_t)pf;
              nsub++;
              last = pf;
            }
          }
        code += cnt;
        vi += cnt;
        T.lim[L] = code;
        code <<= 1;
      }
      T.dht_pos = pos;
      T.nvals = s_ttot[ti];
      T.is_dc = s_tdc[ti];
      T.nsub = nsub;  // > kSubTabs: overflow, long codes use the canonical walk
    }
  }
  __syncthreads();
  if (H.status == 0) {
    const int ntab = H.ntab;
    for (int e = tid; e < ntab * 256; e += kNT) {
      if (s_hit[e >> 8]) continue;
      HuffTab &T = G->tab[e >> 8];
      const int v = e & 255;
      T.vals[v] = v < T.nvals ? seg_byte(S, raw, T.dht_pos + 16 + v) : (uint8_t)0;
    }
    __syncthreads();
    for (int t = 0; t < ntab; t++) {
      if (s_hit[t]) continue;
      HuffTab &T = G->tab[t];
      int lim[17], first[17], vptr[17];
#pragma unroll
      for (int L = 1; L <= 16; L++) {
        lim[L] = T.lim[L];
        first[L] = T.first[L];
        vptr[L] = T.vptr[L];
      }
      const bool dc = T.is_dc;
      const int nsub = T.nsub;
      for (int e = tid; e < (1 << kFastBits); e += kNT) {
        uint32_t ent = 0;
        bool found = false;
#pragma unroll
        for (int L = kFastBits; L >= 1; L--) {  // prefix-free: at most one length matches
          const int c = e >> (kFastBits - L);
          if (c < lim[L] && c >= first[L]) {
            ent = huff_entry(dc, T.vals[vptr[L] + c - first[L]], L);
            found = true;
          }
        }
        if (!found) {
          if (nsub > kSubTabs) {
            ent = (uint32_t)kSubCanon << 5;  // canonical walk decides (incl. invalid)
          } else {
            for (int q = 0; q < nsub; q++)
              if (S.sub_pf[t][q] == e) ent = (uint32_t)(q + 1) << 5;  // sub-table q
            // ent == 0: no code has this prefix (invalid)
          }
        }
        T.fast[e] = (uint16_t)ent;
      }
      // sub-tables: the (16 - kFastBits) bits after each long-code prefix
      const int ns = min(nsub, kSubTabs);
      for (int e = tid; e < (ns << kSubBits); e += kNT) {
        const int code16 = ((int)S.sub_pf[t][e >> kSubBits] << kSubBits) | (e & ((1 << kSubBits) - 1));
        uint32_t ent = 0;
#pragma unroll
        for (int L = 16; L > kFastBits; L--) {
          const int c = code16 >> (16 - L);
          if (c < lim[L] && c >= first[L]) ent = huff_entry(dc, T.vals[vptr[L] + c - first[L]], L);
        }
        T.sub[e] = (uint16_t)ent;
      }
    }
  }
  __syncthreads();
  // ---- publish newly built tables to empty cache slots ----------------------
  if (H.status == 0) {
    __shared__ int s_claim;
    for (int t = 0; t < H.ntab; t++) {
      if (s_hit[t]) continue;
      if (tid == 0) s_claim = atomicCAS(&cache[t].state, 0u, 1u) == 0u;
      __syncthreads();
      if (s_claim) {
        TabCacheSlot &C = cache[t];
        const HuffTab &T = G->tab[t];
        const int len = 16 + T.nvals;
        for (int i = tid; i < len; i += kNT) C.key[i] = seg_byte(S, raw, T.dht_pos + i);
        const int4 *src = reinterpret_cast<const int4 *>(&T);
        int4 *dst = reinterpret_cast<int4 *>(&C.tab);
        for (int i = tid; i < (int)(sizeof(HuffTab) / 16); i += kNT) dst[i] = src[i];
        if (tid == 0) { C.len = len; C.is_dc = T.is_dc; }
        __threadfence();
        __syncthreads();
        if (tid == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&C.state), "r"(2u) : "memory");
      }
      __syncthreads();
    }
  }
  // ---- hand over: header (+ used tables) to global ---------------------------
  {
    const int words = (int)(sizeof(DecodeHead) / 16);  // the tables are already in G
    const int4 *src = reinterpret_cast<const int4 *>(&H);
    int4 *dst = reinterpret_cast<int4 *>(G);
    for (int i = tid; i < words; i += kNT) dst[i] = src[i];
  }
  if (tid == 0) {
    info->dbg[0] = S.t0;
    info->dbg[1] = clock64();
    for (int i = 0; i < 4; i++) info->dbg[12 + i] = S.ph[i];
  }
}

// ===========================================================================
// k_entropy: entropy decode, one warp per image
// ===========================================================================
struct __align__(128) EntSmem {
  uint32_t ring[kLanes][kRingWords];  // (128-byte aligned: RingReader::skip masks addresses)
  uint32_t stage[kLanes][kGroup + 1];  // list entries of the current group (rows padded: no bank conflicts)
  DecodeHead h;
  uint16_t tab[kSmemTabs][1 << kFastBits];  // first-level tables (<= kSmemTabs used)
  LaneRec lane[kLanes];
  int status, reason, offset;
  uint32_t p_final;
  int coef_range, red;
  unsigned int dbg_units, dbg_guess, dbg_umax, dbg_ext;
  unsigned long long lbase;
  int fmt;
  int ms_nscan, ms_nlevel, ms_range;
  long long t_ph[8];
};

static_assert(sizeof(LaneTail) <= sizeof(uint32_t) * (kGroup + 1), "LaneTail fits a staging row");
__device__ __forceinline__ LaneTail &tail_of(EntSmem &S, int lane) {
  return *reinterpret_cast<LaneTail *>(&S.stage[lane][0]);
}

__device__ __forceinline__ void ent_status(EntSmem &S, int st, int reason, int off) {
  if (S.status == 0) {
    S.status = st;
    S.reason = reason;
    S.offset = off;
  }
}

// Zero the image's crop-window coefficients (the re-decoding paths scatter
// nonzeros into it).  Called by every thread of the CTA.
__device__ void zero_window(const DecodeHead &H, int16_t *coef, int lane) {
  uint64_t total = 0;
  for (int c = 0; c < 3; c++) total += (uint64_t)H.wbh[c] * H.wbw[c] * 64;
  int4 *z = reinterpret_cast<int4 *>(coef + H.coef_base);
  for (uint64_t i = lane; i < total / 8; i += kLanes) z[i] = make_int4(0, 0, 0, 0);
}

// ===========================================================================
// Multi-scan streams (progressive, or sequential with several scans): the
// reference's full-decode fallback (codec.py:352-399 _decode_scans_full,
// decode_kernels.py:111-385) on the GPU.  Every scan is decoded in full into
// the image's full coefficient arrays (int16 [BH][BW][64] per component,
// carved by k_prep); k_idct then reconstructs the crop window from them.
// Scans that touch disjoint coefficients (other components, other spectral
// bands) are independent, so the CTA's lanes decode them in parallel waves
// (a scan waits for every earlier scan it shares a component and band with;
// refinement scans therefore follow the scans they refine).  Errors are the
// reference's: the first failing scan in file order decides, with the same
// message and offset.
// ===========================================================================
constexpr int kMsMaxScans = 64;
constexpr int kMsMaxTabs = 16;

struct MsScan {
  int32_t start, end, ri;       // entropy-coded bytes [start, end) of the payload; DRI in force
  int32_t err, reason, off;     // pre-decode error (status, reason, offset) or 0
  int32_t level;                // dependency wave
  int32_t status, errp;         // decode result: status (0/1/3/4) and failing bit position
  int32_t dpos[3], apos[3];     // DHT definitions in force at the SOS (payload offsets, -1: none)
  uint8_t ns, ss, se, ah, al, pad0;
  uint8_t comp[3];
  int8_t dt[3], at[3];          // decoder index of the used tables (-1: unused)
  uint8_t pad1;
};

struct MsTab {  // canonical Huffman decoder of one DHT definition (codec.py:272-295)
  int32_t maxcode[18];   // largest code of each length (-1: none)
  int32_t mincode[17];
  int16_t valptr[17];
  int16_t pad;
  int32_t vals;          // payload offset of the symbol values
};
static_assert(sizeof(MsScan) * kMsMaxScans + sizeof(MsTab) * kMsMaxTabs <= kSmemTabs * 2048,
              "multi-scan state must fit the shared first-level table area");

// Clean-stream bit reader over the RAW scan bytes (destuff_scan semantics,
// decode_kernels.py:27-61, on the fly): FF00 -> FF, RSTn skipped, any other
// FFxx ends the data; past the end the reader supplies 0xFF (_br_fill).  p is
// the number of clean bits consumed (the reference's 8*vpos - cnt).
struct MsReader {
  const uint8_t *raw;
  int rpos, rend;
  bool ended;
  uint64_t buf;  // left-aligned
  int n;
  uint32_t p;
  __device__ __forceinline__ uint32_t next_byte() {
#pragma unroll 1
    while (!ended) {
      if (rpos >= rend) { ended = true; break; }
      const uint32_t b = raw[rpos];
      if (b != 0xFF) { rpos++; return b; }
      if (rpos + 1 >= rend) { ended = true; break; }
      const uint32_t m = raw[rpos + 1];
      if (m == 0x00) { rpos += 2; return 0xFF; }
      if (m >= 0xD0 && m <= 0xD7) { rpos += 2; continue; }
      ended = true;
    }
    return 0xFF;
  }
  __device__ __forceinline__ void anchor(int raw_pos, uint32_t clean_bit) {
    rpos = raw_pos;
    ended = false;
    buf = 0;
    n = 0;
    p = clean_bit;
  }
  __device__ __forceinline__ void fill(int need) {
#pragma unroll 1
    while (n < need) {
      buf |= (uint64_t)next_byte() << (56 - n);
      n += 8;
    }
  }
  __device__ __forceinline__ uint32_t peek16() { fill(32); return (uint32_t)(buf >> 48); }
  __device__ __forceinline__ void skip(int k) { buf <<= k; n -= k; p += k; }
  __device__ __forceinline__ uint32_t bits(int k) {  // _gb (k <= 16)
    if (k == 0) return 0;
    fill(32);
    const uint32_t v = (uint32_t)(buf >> (64 - k));
    skip(k);
    return v;
  }
  // _hd: the symbol, or -1 for a code the table does not assign
  __device__ __forceinline__ int sym(const MsTab &T, const uint8_t *payload) {
    const uint32_t c16 = peek16();
#pragma unroll 1
    for (int L = 1; L <= 16; L++) {
      const int code = (int)(c16 >> (16 - L));
      if (code <= T.maxcode[L]) {
        skip(L);
        return payload[T.vals + T.valptr[L] + code - T.mincode[L]];
      }
    }
    return -1;
  }
};

// Restart-interval cursor: the clean offset and raw position just after the
// next RSTn of the scan (restarts[] of destuff_scan, found incrementally).
struct MsRst {
  int raw;       // raw position to search from
  uint32_t clean;  // clean bytes before `raw`
  __device__ __forceinline__ bool next(const uint8_t *d, int end, int &raw_after, uint32_t &clean_at) {
#pragma unroll 1
    while (raw < end) {
      const uint32_t b = d[raw];
      if (b != 0xFF) { raw++; clean++; continue; }
      if (raw + 1 >= end) return false;
      const uint32_t m = d[raw + 1];
      if (m == 0x00) { raw += 2; clean++; continue; }
      if (m >= 0xD0 && m <= 0xD7) {
        raw += 2;
        raw_after = raw;
        clean_at = clean;
        return true;
      }
      return false;
    }
    return false;
  }
};

__device__ __forceinline__ bool ms_store(int16_t *c, int v) {
  *c = (int16_t)v;
  return v >= -32768 && v <= 32767;
}

// One scan, one thread (decode_scan_baseline / _dc_first / _dc_refine /
// _ac_first / _ac_refine).  Returns the status; errp = the clean bit position
// of the failing symbol (status 1).
__device__ int ms_decode_scan(const DecodeHead &H, const MsScan &sc, const MsTab *tabs,
                              const uint8_t *payload, int16_t *coef, bool progressive,
                              uint32_t &errp, int &range_bad) {
  MsReader r;
  r.raw = payload;
  r.rend = sc.end;
  r.anchor(sc.start, 0);
  MsRst rc{sc.start, 0};
  int nrst_used = 0;
  const int ns = sc.ns;
  // _scan_units (codec.py:333-349): one component steps over its true block
  // grid, an interleaved scan over the frame's MCUs with each component's
  // sampling factors
  int gx = H.gx, gy = H.gy;
  int hh[3] = {1, 1, 1}, vv[3] = {1, 1, 1};
  if (ns == 1) {
    gx = H.bw[sc.comp[0]];
    gy = H.bh[sc.comp[0]];
  } else {
    for (int s = 0; s < ns && s < 3; s++) { hh[s] = H.comp_hv[sc.comp[s]] >> 4; vv[s] = H.comp_hv[sc.comp[s]] & 15; }
  }
  int32_t pred[3] = {0, 0, 0};
  int eobrun = 0;
  const int ri = sc.ri;
  const bool is_dc = progressive && sc.ss == 0;
  uint64_t ms_total = 0;  // (the image's full arrays, for ESSL_CHECK)
  for (int c = 0; c < H.ncomp; c++) ms_total += (uint64_t)H.gy * (H.comp_hv[c] & 15) * H.coef_pitch[c] * 64;
  const int16_t *ms_end = coef + H.coef_base + ms_total;
  (void)ms_end;
  const int al = sc.al, ss = sc.ss, se = sc.se;
  const int p1 = 1 << al, m1 = -(1 << al);
  int unit = 0;
  auto restart = [&]() -> bool {  // at an interval boundary: jump to the next RSTn (status 3 if none)
    int ra;
    uint32_t cl;
    if (!rc.next(payload, sc.end, ra, cl)) return false;
    nrst_used++;
    r.anchor(ra, 8u * cl);
    pred[0] = pred[1] = pred[2] = 0;
    eobrun = 0;
    return true;
  };
  for (int my = 0; my < gy; my++) {
    for (int mx = 0; mx < gx; mx++, unit++) {
      if (ri > 0 && unit > 0 && unit % ri == 0 && !restart()) return 3;
      if (!progressive || is_dc) {
        // MCU of blocks: baseline (DC + AC) or progressive DC
        for (int s = 0; s < ns; s++) {
          const int c = sc.comp[s];
          const int pitch = H.coef_pitch[c];
          int16_t *base = coef + H.coef_off[c];
          for (int by = 0; by < vv[s]; by++)
            for (int bx = 0; bx < hh[s]; bx++) {
              int16_t *blk = base + ((uint64_t)(my * vv[s] + by) * pitch + (mx * hh[s] + bx)) * 64;
              ESSL_CHECK(g_check_dec, blk >= coef + H.coef_base && blk + 64 <= ms_end, CK_MS_COEF);
              if (progressive && sc.ah != 0) {  // DC refine: one bit
                if (r.bits(1)) range_bad |= !ms_store(blk, blk[0] | p1);
                continue;
              }
              const uint32_t pstart = r.p;
              const int t = r.sym(tabs[sc.dt[s]], payload);
              if (t < 0 || t > 15) { errp = pstart; return 1; }
              const uint32_t v = r.bits(t);
              pred[s] += extend_bits(v, t);
              if (progressive) {  // DC first
                range_bad |= !ms_store(blk, pred[s] * p1);
                continue;
              }
              range_bad |= !ms_store(blk, pred[s]);
              for (int k = 1; k < 64;) {  // decode_kernels.py:155-177
                const uint32_t q0 = r.p;
                const int rs = r.sym(tabs[sc.at[s]], payload);
                if (rs < 0) { errp = q0; return 1; }
                const int run = rs >> 4, sz = rs & 15;
                if (sz == 0) {
                  if (run == 15) { k += 16; continue; }
                  break;
                }
                k += run;
                if (k > 63) { errp = q0; return 1; }
                range_bad |= !ms_store(blk + c_zz[k], extend_bits(r.bits(sz), sz));
                k++;
              }
            }
        }
        continue;
      }
      // progressive AC, one component, one block per unit
      const int c = sc.comp[0];
      int16_t *blk = coef + H.coef_off[c] + ((uint64_t)my * H.coef_pitch[c] + mx) * 64;
      ESSL_CHECK(g_check_dec, blk >= coef + H.coef_base && blk + 64 <= ms_end, CK_MS_COEF);
      const MsTab &T = tabs[sc.at[0]];
      if (sc.ah == 0) {  // AC first (decode_kernels.py:259-309)
        if (eobrun > 0) { eobrun--; continue; }
        for (int k = ss; k <= se;) {
          const uint32_t q0 = r.p;
          const int rs = r.sym(T, payload);
          if (rs < 0) { errp = q0; return 1; }
          const int run = rs >> 4, sz = rs & 15;
          if (sz == 0) {
            if (run != 15) {
              eobrun = (1 << run) - 1 + (int)r.bits(run);
              break;
            }
            k += 16;
            continue;
          }
          k += run;
          if (k > se) { errp = q0; return 1; }
          range_bad |= !ms_store(blk + c_zz[k], extend_bits(r.bits(sz), sz) * p1);
          k++;
        }
        continue;
      }
      // AC refine (decode_kernels.py:312-385)
      int k = ss;
      if (eobrun == 0) {
        while (k <= se) {
          const uint32_t q0 = r.p;
          const int rs = r.sym(T, payload);
          if (rs < 0) { errp = q0; return 1; }
          int run = rs >> 4;
          const int sz = rs & 15;
          int newval = 0;
          if (sz == 0) {
            if (run != 15) {
              eobrun = (1 << run) + (int)r.bits(run);
              break;
            }
          } else {
            newval = r.bits(1) ? p1 : m1;
          }
          while (k <= se) {
            int16_t *cp = blk + c_zz[k];
            const int cur = *cp;
            if (cur != 0) {
              if (r.bits(1) && (cur & p1) == 0) range_bad |= !ms_store(cp, cur + (cur >= 0 ? p1 : m1));
            } else {
              if (run == 0) break;
              run--;
            }
            k++;
          }
          if (newval != 0 && k <= se) range_bad |= !ms_store(blk + c_zz[k], newval);
          k++;
        }
      }
      if (eobrun > 0) {
        while (k <= se) {
          int16_t *cp = blk + c_zz[k];
          const int cur = *cp;
          if (cur != 0 && r.bits(1) && (cur & p1) == 0) range_bad |= !ms_store(cp, cur + (cur >= 0 ? p1 : m1));
          k++;
        }
        eobrun--;
      }
    }
  }
  (void)nrst_used;
  // _check_consumed: bits consumed beyond the clean length -> truncated
  uint32_t clean_len = 0;
  {
    MsRst cnt{sc.start, 0};
    int ra;
    uint32_t cl;
    while (cnt.next(payload, sc.end, ra, cl)) {}
    // cnt stopped at the end of the clean data: clean bytes counted so far
    clean_len = cnt.clean;
  }
  if (r.p > 8u * clean_len) return 4;
  return 0;
}

// Parse of every scan of a multi-scan stream (thread 0; parse_stream,
// codec.py:124-251 -- the stream passed k_prep's marker walk already) plus
// each scan's pre-decode checks in the reference's order (_scan_units,
// _destuff, the progressive scan rules, _huff_lut / _lut_stack,
// codec.py:333-399) and the dependency wave of every scan.
__device__ void ms_parse(const DecodeHead &H, const uint8_t *d, int n, MsScan *scans, MsTab *tabs,
                         int &nscan_out, int &nlevel_out) {
  int huff_pos[2][16];
  for (int i = 0; i < 16; i++) huff_pos[0][i] = huff_pos[1][i] = -1;
  int tab_pos[kMsMaxTabs];
  int ntab = 0, nscan = 0, ri = 0, pos = 2;
  auto tab_of = [&](int tpos) -> int {  // canonical decoder of the DHT definition at tpos
    if (tpos < 0) return -1;
    for (int t = 0; t < ntab; t++)
      if (tab_pos[t] == tpos) return t;
    if (ntab >= kMsMaxTabs) return -2;
    const int t = ntab++;
    tab_pos[t] = tpos;
    MsTab &T = tabs[t];
    int code = 0, vi = 0;
    T.pad = 0;
    for (int L = 1; L <= 16; L++) {
      const int cnt = d[tpos + L - 1];
      T.mincode[L] = code;
      T.valptr[L] = (int16_t)vi;
      if (cnt && code + cnt > (1 << L)) T.pad = 1;  // code overflow (codec.py:287-288)
      code += cnt;
      vi += cnt;
      T.maxcode[L] = cnt ? code - 1 : -1;
      code <<= 1;
    }
    T.maxcode[17] = 0x7FFFFFFF;
    T.vals = tpos + 16;
    return t;
  };
  while (pos < n && nscan <= kMsMaxScans) {
    if (d[pos] != 0xFF) break;
    while (pos < n && d[pos] == 0xFF) pos++;
    if (pos >= n) break;
    const int marker = d[pos++];
    if (marker == 0xD9) break;
    if (marker == 0x01 || (marker >= 0xD0 && marker <= 0xD7)) continue;
    if (pos + 2 > n) break;
    const int seglen = (d[pos] << 8) | d[pos + 1];
    const int body = pos + 2, end = pos + seglen;
    if (marker == 0xC4) {
      int p = body;
      while (p + 17 <= end) {
        const int tc = d[p] >> 4, th = d[p] & 15;
        int tot = 0;
        for (int i = 0; i < 16; i++) tot += d[p + 1 + i];
        if (tc < 2) huff_pos[tc][th] = p + 1;
        p += 17 + tot;
      }
    } else if (marker == 0xDD) {
      ri = (d[body] << 8) | d[body + 1];
    } else if (marker == 0xDA) {
      if (nscan >= kMsMaxScans) { nscan++; break; }
      MsScan &S = scans[nscan];
      const int ns = d[body];
      int p = body + 1;
      S.ns = (uint8_t)ns;
      for (int s = 0; s < ns && s < 3; s++) {
        const int cs = d[p], td = d[p + 1] >> 4, ta = d[p + 1] & 15;
        int idx = 0;
        for (int i = 0; i < H.ncomp; i++)
          if (H.comp_id[i] == cs) { idx = i; break; }
        S.comp[s] = (uint8_t)idx;
        S.dpos[s] = huff_pos[0][td];
        S.apos[s] = huff_pos[1][ta];
        S.dt[s] = S.at[s] = -1;
        p += 2;
      }
      p = body + 1 + 2 * ns;
      S.ss = d[p]; S.se = d[p + 1]; S.ah = d[p + 2] >> 4; S.al = d[p + 2] & 15;
      S.ri = ri;
      S.start = end;
      // _entropy_end (codec.py:109-121)
      int q = end;
      while (true) {
        while (q < n && d[q] != 0xFF) q++;
        if (q >= n || q + 1 >= n) { q = n; break; }
        const int m = d[q + 1];
        if (m == 0x00 || (m >= 0xD0 && m <= 0xD7) || m == 0xFF) { q += m != 0xFF ? 2 : 1; continue; }
        break;
      }
      S.end = q;
      S.err = 0; S.reason = 0; S.off = -1; S.status = 0; S.errp = 0;
      nscan++;
      pos = q;
      continue;
    }
    pos = end;
  }
  // pre-decode checks and waves
  int nlevel = 0;
  const int nsc = min(nscan, kMsMaxScans);
  for (int j = 0; j < nsc; j++) {
    MsScan &S = scans[j];
    auto fail = [&](int st, int reason, int off) {
      if (!S.err) { S.err = st; S.reason = reason; S.off = off; }
    };
    if (S.ns != 1 && S.ns != H.ncomp) {
      fail(ESSL_ST_MALFORMED, R_PARTIAL_INTERLEAVE, -1);
    } else {
      // _destuff: restart markers of the scan
      int gx = H.gx, gy = H.gy;
      if (S.ns == 1) { gx = H.bw[S.comp[0]]; gy = H.bh[S.comp[0]]; }
      const int max_r = S.ri ? (gx * gy) / S.ri : 0;
      MsRst rc{S.start, 0};
      int ra, nr = 0;
      uint32_t cl;
      while (rc.next(d, S.end, ra, cl)) nr++;
      if (S.ri == 0 && nr > 0) fail(ESSL_ST_MALFORMED, R_RST_NO_DRI, S.start);
      else if (nr > max_r + 2) fail(ESSL_ST_MALFORMED, R_TOO_MANY_RST, S.start);
      auto need = [&](int tpos) -> int8_t {  // _huff_lut of a table the scan uses
        const int t = tab_of(tpos);
        if (t == -2) fail(ESSL_ST_UNSUPPORTED, R_TOO_MANY_SCANS, -1);
        else if (t < 0) fail(ESSL_ST_HUFFTABLE, R_HUFF_UNDEFINED, -1);
        else if (tabs[t].pad) fail(ESSL_ST_HUFFTABLE, R_HUFF_OVERFLOW, -1);
        return (int8_t)t;
      };
      if (!H.progressive) {
        for (int s = 0; s < S.ns; s++) S.dt[s] = need(S.dpos[s]);
        for (int s = 0; s < S.ns; s++) S.at[s] = need(S.apos[s]);
      } else if (S.ss == 0) {
        if (S.se != 0) fail(ESSL_ST_MALFORMED, R_PROG_DC_SE, -1);
        else if (S.ah == 0)
          for (int s = 0; s < S.ns; s++) S.dt[s] = need(S.dpos[s]);
      } else {
        if (S.ns != 1) fail(ESSL_ST_MALFORMED, R_PROG_AC_NCOMP, -1);
        else S.at[0] = need(S.apos[0]);
      }
    }
    // wave: after every earlier scan sharing a component and a coefficient
    int lv = 0;
    const int lo = H.progressive ? S.ss : 0, hi = H.progressive ? S.se : 63;
    for (int i = 0; i < j; i++) {
      const MsScan &O = scans[i];
      const int olo = H.progressive ? O.ss : 0, ohi = H.progressive ? O.se : 63;
      bool share = false;
      for (int a = 0; a < S.ns && a < 3; a++)
        for (int b = 0; b < O.ns && b < 3; b++) share |= S.comp[a] == O.comp[b];
      if (share && olo <= hi && lo <= ohi) lv = max(lv, O.level + 1);
    }
    S.level = lv;
    nlevel = max(nlevel, lv + 1);
    if (S.err) {  // the reference stops at the first failing scan
      nscan_out = j + 1;
      nlevel_out = nlevel;
      return;
    }
  }
  nscan_out = nscan > kMsMaxScans ? -1 : nsc;
  nlevel_out = nlevel;
}

// The multi-scan decode of one image by its k_entropy CTA.
__device__ void multiscan_body(const DecodeParams &P, EntSmem &S, int img, int lane) {
  DecodeHead &H = S.h;
  MsScan *scans = reinterpret_cast<MsScan *>(&S.tab[0][0]);
  MsTab *tabs = reinterpret_cast<MsTab *>(reinterpret_cast<uint8_t *>(&S.tab[0][0]) +
                                          sizeof(MsScan) * kMsMaxScans);
  const essl_sample smp = P.samples[img];
  const uint8_t *d = P.blob + smp.offset;
  const int n = (int)smp.length;
  int16_t *coef = P.s.coef;
  // every coefficient starts at zero (_alloc_coefs)
  uint64_t total = 0;
  for (int c = 0; c < H.ncomp; c++)
    total += (uint64_t)H.gy * (H.comp_hv[c] & 15) * H.coef_pitch[c] * 64;
  int4 *z = reinterpret_cast<int4 *>(coef + H.coef_base);
  for (uint64_t i = lane; i < total / 8; i += kLanes) z[i] = make_int4(0, 0, 0, 0);
  if (lane == 0) {
    int ns, nl;
    ms_parse(H, d, n, scans, tabs, ns, nl);
    S.ms_nscan = ns;
    S.ms_nlevel = nl;
    S.ms_range = 0;
  }
  __syncthreads();
  const int nscan = S.ms_nscan;
  if (nscan < 0) {
    if (lane == 0) ent_status(S, ESSL_ST_UNSUPPORTED, R_TOO_MANY_SCANS, -1);
    return;
  }
  // waves of independent scans, one lane per scan
  for (int w = 0; w < S.ms_nlevel; w++) {
    int rank = 0;
    for (int j = 0; j < nscan; j++) {
      MsScan &sc = scans[j];
      if (sc.level != w || sc.err) continue;
      if ((rank++ % kLanes) != lane) continue;
      uint32_t errp = 0;
      int bad = 0;
      sc.status = ms_decode_scan(H, sc, tabs, d, coef, H.progressive, errp, bad);
      sc.errp = (int32_t)errp;
      if (bad) S.ms_range = 1;
    }
    __syncthreads();
  }
  if (lane == 0) {  // the first failing scan in file order (_check_consumed, codec.py:323-330)
    for (int j = 0; j < nscan; j++) {
      const MsScan &sc = scans[j];
      if (sc.err) {
        ent_status(S, sc.err, sc.reason, sc.off);
        break;
      }
      if (sc.status == 1) {
        const uint32_t vpos = (sc.errp + 25u + 7u) / 8u;
        ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, sc.start + (int)min(vpos, (uint32_t)(sc.end - sc.start)));
        break;
      }
      if (sc.status == 3) { ent_status(S, ESSL_ST_MISSING_RST, 0, sc.start); break; }
      if (sc.status == 4) { ent_status(S, ESSL_ST_TRUNCATED, 0, sc.end); break; }
    }
    if (S.ms_range) S.coef_range = 1;
    S.fmt = 0;
  }
}

// Decode of one image by the CTA: restart intervals, serial mode, or the
// checkpoint-merge parallel decode; SH: the clean stream is staged in shared
// memory.
template <bool SH>
__device__ __forceinline__ void entropy_body(const DecodeParams &P, EntSmem &S, const EntCtx &C0,
                                             int img, int lane, uint32_t &dbg_nseq,
                                             uint32_t &dbg_cont) {
  EntCtx C = C0;
  DecodeHead &H = S.h;
  LaneRec &R = S.lane[lane];
  LaneTail &T = tail_of(S, lane);
  int16_t *coef = P.s.coef;
  const uint32_t *rst_tab = C.words + H.rst_off;
  WriteOut wo;
  wo.range = 0;
#define PHASE(i) do { if (lane == 0) S.t_ph[i] = clock64(); } while (0)
  if (S.status == 0 && H.multiscan) {
    multiscan_body(P, S, img, lane);
  } else if (S.status == 0 && H.scan_ri > 0) {
    // DRI: restart intervals decode independently from exact entry states
    // (decode_kernels.py:130-138); lanes take intervals round-robin.
    const uint32_t ri = H.scan_ri;
    const uint32_t lim_mcu = (uint32_t)H.row_stop * H.gx;
    const uint32_t nint = (lim_mcu + ri - 1) / ri;
    if (lane == 0) S.red = 0x7FFFFFFF;
    zero_window(H, coef, lane);
    __syncthreads();
    for (uint32_t j = lane; j < nint; j += kLanes) {
      if (j >= 1 && (int)(j - 1) >= H.n_restarts) {  // status 3
        atomicMin(&S.red, (int)(2 * j + 1));
        continue;
      }
      const uint32_t p0 = j == 0 ? 0 : 8u * rst_tab[j - 1];
      const uint32_t b0 = j * ri * H.bpm;
      const uint32_t b1 = min((j + 1) * ri, lim_mcu) * H.bpm;
      int32_t pr[3] = {0, 0, 0};
      write_run<SH>(C, H, coef, p0, 0, b0, b1 - b0, pr, wo, &S.p_final);
      if (wo.err) atomicMin(&S.red, (int)(2 * j));
      if (wo.range) S.coef_range = 1;
    }
    __syncthreads();
    if (lane == 0) {
      const int code = S.red;
      if (code != 0x7FFFFFFF) {
        const uint32_t j = code >> 1;
        if (code & 1) {
          ent_status(S, ESSL_ST_MISSING_RST, 0, H.scan_start);
        } else {
          const uint32_t p0 = j == 0 ? 0 : 8u * rst_tab[j - 1];
          const uint32_t errp = tail_run<SH>(C, p0, 0, 0, 0xFFFFFFFFu);
          ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, corrupt_offset(H, errp));
        }
      } else if (S.p_final != kNoEnd && S.p_final > H.clean_bits) {
        ent_status(S, ESSL_ST_TRUNCATED, 0, H.scan_end);
      }
    }
  } else if (S.status == 0 && P.mode == ESSL_DECODE_SERIAL) {
    zero_window(H, coef, lane);
    __syncthreads();
    if (lane == 0) {
      int32_t pred[3] = {0, 0, 0};
      write_run<SH>(C, H, coef, 0, 0, 0, H.limit_blocks, pred, wo, &S.p_final);
      if (wo.err) ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, corrupt_offset(H, wo.errp));
      else if (S.p_final > H.clean_bits) ent_status(S, ESSL_ST_TRUNCATED, 0, H.scan_end);
      if (wo.range) S.coef_range = 1;
    }
  } else if (S.status == 0) {
    // ---- checkpoint-merge parallel decode, each unit decoded once ---------
    const uint32_t cbits = C.cbits;
    // N2 (codec.py:494-498): the crop needs blocks [0, limit) only.  Phase 1
    // covers the bits up to an estimate of where block `limit` ends (the
    // limit's share of all blocks, plus a margin); if the exact path has not
    // reached the limit there, the last lane's path is extended serially.
    const uint32_t total_blocks = (uint32_t)H.gx * (uint32_t)H.gy * (uint32_t)H.bpm;
    uint32_t end_bits = cbits;
    if (P.early_exit && C.limit < total_blocks) {
      const uint64_t est = (uint64_t)cbits * C.limit / total_blocks;
      end_bits = (uint32_t)min((uint64_t)cbits, est + cbits / 32 + 512);
    }
    C.cend = end_bits;
    int nseq = (int)((end_bits + P.seq_bits - 1) / (uint32_t)P.seq_bits);
    nseq = max(1, min(nseq, kLanes));
    const uint32_t slen = (end_bits + nseq - 1) / nseq;
    const uint32_t warm = min((uint32_t)P.warm_bits, slen * 4);
    // unit lists + block records: one region per lane, carved per image.
    // Lists hold every decoded unit; slot cap is a sink for overflow and the
    // slot after the last unit holds a sentinel.  (No room: one-entry sinks,
    // the image falls back to a serial re-decode.)
    const uint32_t cap = ((slen + warm + kContBits) / 4 + 64 + 3) & ~3u;
    const uint32_t bcap = cap / 2 + 8;  // a block has >= 2 units (DC + an AC unit)
    // list: cap entries + a kGroup-slot sink (+ sentinel / pad); records: bcap +
    // a kGroup-slot sink (the pool is sized for this stride: api.cu list_cap)
    const uint32_t stride = cap + kGroup + 8 + ((2 * (bcap + kGroup + 2) + 3) & ~3u);
    if (lane == 0) {
      const unsigned long long need = (unsigned long long)nseq * stride;
      const unsigned long long b = atomicAdd(&P.s.counters[3], need + 4);
      const unsigned long long b4 = (b + 3) & ~3ull;
      S.lbase = b4 + need > P.s.list_cap ? ~0ull : b4;
      S.red = 0;
    }
    __syncthreads();
    if (S.lbase == ~0ull) {
      // no room in the list pool: serial decode (the ESSL_DECODE_SERIAL path)
      zero_window(H, coef, lane);
      __syncthreads();
      if (lane == 0) {
        int32_t pred[3] = {0, 0, 0};
        write_run<SH>(C, H, coef, 0, 0, 0, H.limit_blocks, pred, wo, &S.p_final);
        if (wo.err) ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, corrupt_offset(H, wo.errp));
        else if (S.p_final > H.clean_bits) ent_status(S, ESSL_ST_TRUNCATED, 0, H.scan_end);
        if (wo.range) S.coef_range = 1;
      }
      return;
    }
    const unsigned long long lreg = S.lbase + (unsigned long long)lane * stride;
    uint32_t *list = P.s.list + lreg;
    uint2 *bsl = reinterpret_cast<uint2 *>(P.s.list + lreg + cap + kGroup + 8);
    // every lane's block records (the continuations' merge targets): lane j's
    // at bsl0 + j * bstride
    const uint2 *bsl0 = reinterpret_cast<const uint2 *>(P.s.list + S.lbase + cap + kGroup + 8);
    const uint32_t bstride = stride / 2;
    if (lane < nseq) {
      const uint32_t sbeg = lane * slen;
      const uint32_t send = lane == nseq - 1 ? end_bits : min(end_bits, (lane + 1) * slen);
      const uint32_t p0 = lane == 0 ? 0u : (sbeg > warm ? sbeg - warm : 0u);
      run_path<false, SH>(C, lane, nseq, p0, sbeg, send, list, cap, bsl, bcap, bsl0, bstride, S.lane, R,
                          &T, &S.dbg_units);
    }
    __syncthreads();
    PHASE(2);
    const bool cont = lane < nseq - 1 && !(lane == 0 && R.err);
    if (cont)
      run_path<true, SH>(C, lane, nseq, 0, 0, 0, list, cap, bsl, bcap, bsl0, bstride, S.lane, R, &T,
                         &S.dbg_units);
    T.w_nb = 0;  // (every lane; the resolution sets the owners' segments)
    dbg_nseq = (uint32_t)nseq;
    if (cont) atomicMax(&S.red, (int)(T.cp - R.xp));
    __syncthreads();
    dbg_cont = (uint32_t)S.red;
    if (P.dbg_lanes) {
      int32_t *o = P.dbg_lanes + ((size_t)img * kLanes + lane) * 8;
      o[0] = nseq; o[1] = (int32_t)R.xp; o[2] = (int32_t)R.xb; o[3] = (int32_t)R.nck;
      o[4] = R.err; o[5] = cont ? (int32_t)T.cp : -1; o[6] = cont ? T.cst : -1;
      o[7] = cont ? (int32_t)T.cj : -1;
    }
    PHASE(3);
    // resolution: follow the exact path from lane 0 through the merges
    if (lane == 0) {
      uint32_t A = 0, sord = 0, sp = 0, sb = 0, snb = 0;
      int o = 0;
      const uint32_t limit = C.limit;
      S.fmt = 1;
#pragma unroll 1
      for (int hop = 0; hop < nseq; hop++) {
        LaneRec &L = S.lane[o];
        LaneTail &TL = tail_of(S, o);
        const uint32_t own = L.nblk - snb;
        TL.w_ord = sord; TL.w_p = sp; TL.w_b = sb; TL.w_A = A;
        if (L.ovf) S.fmt = 0;  // an owner's list overflowed: serial re-decode
        if (L.err) {  // error on the exact path (phase 1 of lane 0)
          TL.w_nb = min(own, limit - A);
          if (A + own < limit) ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, corrupt_offset(H, L.errp));
          break;
        }
        const bool last = o == nseq - 1;
        // a path that ends without a merge: the last lane's, or a continuation
        // that ran to the end of the covered range
        const bool open_end = last || TL.cst == 2;
        uint32_t seg = own + (last ? 0u : TL.cn);
        PathEnd X = last ? PathEnd{L.xp, L.xk, L.xb, L.xbe} : PathEnd{TL.cp, (int)TL.ek, (int)TL.eb, TL.cbe};
        if (open_end && A + seg < limit && X.p < cbits) {
          // it stopped at the estimated end before the crop's last needed
          // block: extend the exact path, appending to this lane's lists
          const unsigned long long lr = S.lbase + (unsigned long long)o * stride;
          uint32_t *lo = P.s.list + lr;
          uint2 *bo = reinterpret_cast<uint2 *>(P.s.list + lr + cap + kGroup + 8);
          uint32_t added = 0;
          int ovf = 0;
          const int xs = extend_path<SH>(C, lo, cap, bo, bcap, L.nlist, L.nbs, X, limit - (A + seg), added, ovf);
          S.dbg_ext += 1;
          seg += added;
          if (ovf) {
            L.ovf = 1;
            S.fmt = 0;
          }
          if (xs == 1) {
            TL.w_nb = min(seg, limit - A);
            ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, corrupt_offset(H, X.p));
            break;
          }
        }
        TL.w_nb = min(seg, limit - A);
        const uint32_t end_p = X.p;
        const int end_be = X.be;
        if (A + seg >= limit) {
          // the block reaching the limit ends past the data (_check_consumed)
          if (A + seg == limit && end_be && end_p > cbits) ent_status(S, ESSL_ST_TRUNCATED, 0, H.scan_end);
          break;
        }
        if (open_end) {
          // the data ends before the crop's last MCU row: continue serially
          // into the 0xFF padding to classify corrupt (1) vs truncated (4)
          const uint32_t errp = tail_run<SH>(C, end_p, X.k, X.b, limit - (A + seg));
          if (errp != kNoEnd) ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, corrupt_offset(H, errp));
          else ent_status(S, ESSL_ST_TRUNCATED, 0, H.scan_end);
          break;
        }
        if (TL.cst == 1) {
          ent_status(S, ESSL_ST_CORRUPT_HUFFMAN, 0, corrupt_offset(H, TL.cp));
          break;
        }
        A += seg;
        // merged into record cm of lane cj: the exact path continues there,
        // after cm complete blocks of that lane's list
        const uint32_t pb = TL.cpb;  // == bsl0[TL.cj * bstride + TL.cm].y
        o = (int)TL.cj;
        sord = TL.cm; sp = pb >> 6; sb = pb & 63; snb = TL.cm;
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // (lane 0's serial readers: the rings are reused below)
    __syncthreads();
    PHASE(4);
    const bool own = S.status == 0 && T.w_nb > 0;
    int range = 0;
    if (S.status == 0 && S.fmt == 1) {
      // block tables: each segment's DC continues from the earlier segments'
      // DC sums (segments are in lane order)
      int32_t sum[3] = {0, 0, 0};
      if (own) seg_dc_sums(C, list, bsl, T.w_ord, (int)T.w_b, T.w_nb, sum);
      int32_t *dcs = reinterpret_cast<int32_t *>(&S.ring[0][0]);  // (the read rings are idle now: run_path drained its copies)
      for (int q = 0; q < 3; q++) dcs[lane * 3 + q] = sum[q];
      __syncthreads();
      if (own) {
        int32_t base[3] = {0, 0, 0};
        for (int t = 0; t < lane; t++)
          for (int q = 0; q < 3; q++) base[q] += dcs[t * 3 + q];
        seg_table(C, H, coef, list, bsl, T.w_ord, (uint32_t)lreg, (int)T.w_b, T.w_A, T.w_nb,
                  min(R.nbs, bcap), R.nlist, base, range);
      }
    } else if (S.status == 0) {
      // fallback (an owner's unit list overflowed): serial re-decode into
      // the zeroed coefficient window
      zero_window(H, coef, lane);
      __syncthreads();
      if (lane == 0) {
        int32_t pred[3] = {0, 0, 0};
        write_run<SH>(C, H, coef, 0, 0, 0, C.limit, pred, wo, nullptr);
        range = wo.range;
      }
    }
    if (range) S.coef_range = 1;
  }
#undef PHASE
}

__global__ void __launch_bounds__(kLanes, 9) k_entropy(DecodeParams P) {
  TraceScope trace_(P.trace, ESSL_K_ENTROPY);
  __shared__ EntSmem S;
  const int img = blockIdx.x;
  const int lane = threadIdx.x;
  ImgInfo *info = P.s.info + img;
  const DecodeHdr *G = hdr_of(P.s, img);
  DecodeHead &H = S.h;
#define PHASE(i) do { if (lane == 0) S.t_ph[i] = clock64(); } while (0)
  if (lane < 8) S.t_ph[lane] = 0;
  __syncthreads();
  PHASE(0);
  {
    const int head = (int)(sizeof(DecodeHead) / 16);
    const int4 *src = reinterpret_cast<const int4 *>(G);
    int4 *dst = reinterpret_cast<int4 *>(&H);
    for (int i = lane; i < head; i += kLanes) dst[i] = src[i];
  }
  __syncthreads();
  if (H.status == 0 && H.ntab <= kSmemTabs) {  // the first-level tables of the used Huffman tables
    constexpr int per = (int)(kTabStride / 16);
    for (int i = lane; i < H.ntab * per; i += kLanes) {
      const int t = i / per, w = i % per;
      reinterpret_cast<int4 *>(S.tab[t])[w] =
          reinterpret_cast<const int4 *>(reinterpret_cast<const HuffTab *>(H.tab_ptr[t])->fast)[w];
    }
  }
  if (lane == 0) {
    S.status = H.status; S.reason = H.reason; S.offset = H.offset;
    S.coef_range = 0;
    S.p_final = kNoEnd;
    S.fmt = 0;
    S.dbg_units = 0; S.dbg_guess = 0; S.dbg_umax = 0; S.dbg_ext = 0;
  }
  LaneRec &R = S.lane[lane];
  R.nck = 0;
  __syncthreads();
  PHASE(1);

  EntCtx C;
  C.gtab = H.tab_ptr;
  C.tabs_s = (uint32_t)__cvta_generic_to_shared(S.tab);
  C.zz_s = (uint32_t)__cvta_generic_to_shared(H.zz);
  {
    const uint32_t w = H.tab_index_word;
    const uint32_t sz = kTabStride;
    C.d0 = (w & 15) * sz; C.d1 = ((w >> 4) & 15) * sz; C.d2 = ((w >> 8) & 15) * sz;
    C.a0 = ((w >> 12) & 15) * sz; C.a1 = ((w >> 16) & 15) * sz; C.a2 = ((w >> 20) & 15) * sz;
  }
  C.c1 = H.slot_nb[0];
  C.c2 = H.slot_nb[0] + H.slot_nb[1];
  C.bpm = H.bpm;
  C.gx = H.gx;
  C.cbits = H.clean_bits;
  C.limit = H.limit_blocks;
  C.cend = H.clean_bits;
  C.list_lo = P.s.list;
  C.list_hi = P.s.list + P.s.list_cap + 4 * kLanes;
  C.coef_lo = P.s.coef;
  C.coef_hi = P.s.coef + P.s.coef_cap;
  C.words = reinterpret_cast<const uint32_t *>(P.s.clean + H.clean_off);
  C.wmax = H.wmax;
  uint32_t dbg_nseq = 0, dbg_cont = 0;
  // per-lane read rings (cp.async) unless the validation option asks for
  // plain global reads
  const bool staged = P.stage_bytes != 0 && H.ntab <= kSmemTabs;
  C.ring_s = (uint32_t)__cvta_generic_to_shared(&S.ring[lane][0]);
  C.stage_s = (uint32_t)__cvta_generic_to_shared(&S.stage[lane][0]);
  C.cpad = H.cpad;
  __syncthreads();
  if (staged) entropy_body<true>(P, S, C, img, lane, dbg_nseq, dbg_cont);
  else entropy_body<false>(P, S, C, img, lane, dbg_nseq, dbg_cont);
  __syncthreads();
  PHASE(5);
  if (lane == 0 && S.status == 0 && S.coef_range) ent_status(S, ESSL_ST_UNSUPPORTED, R_COEF_RANGE, -1);
  if (lane == 0 && S.status == 0 && H.quant_missing >= 0)
    ent_status(S, ESSL_ST_QUANT, 0, H.quant_missing);  // codec.py:405-409
  __syncthreads();

  // ---- crop-plane allocation + per-image results ----------------------------
  if (lane == 0) {
    if (S.status == 0) {
      uint64_t total = 0;
      uint64_t off[3];
      for (int c = 0; c < 3; c++) {
        off[c] = total;
        total += (uint64_t)H.wbh[c] * 8 * H.wbw[c] * 8;
      }
      const unsigned long long base = atomicAdd(&P.s.counters[2], (unsigned long long)((total + 15) / 16 * 16));
      if (base + total > P.s.plane_cap) {
        ent_status(S, ESSL_ST_CAPACITY, R_SCRATCH, -1);
      } else {
        for (int c = 0; c < 3; c++) {
          info->plane_off[c] = base + off[c];
          info->plane_pitch[c] = H.wbw[c] * 8;
          info->wby0[c] = H.wby0[c]; info->wbx0[c] = H.wbx0[c];
          info->wbh[c] = H.wbh[c]; info->wbw[c] = H.wbw[c];
          info->coef_off[c] = H.coef_off[c] + ((uint64_t)H.wby0[c] * H.coef_pitch[c] + H.wbx0[c]) * 64 *
                                                 (H.multiscan ? 1 : 0);
          info->coef_pitch[c] = H.coef_pitch[c];
        }
      }
    }
    info->status = S.status;
    info->reason = S.reason;
    info->offset = S.offset;
    info->fmt = S.fmt;
    for (int i = 0; i < 6; i++) info->dbg[2 + i] = S.t_ph[i];
    info->dbg[10] = dbg_nseq | ((long long)S.dbg_ext << 32);
    info->dbg[11] = dbg_cont;
    const uint32_t su = S.dbg_units, sg = S.dbg_guess, mu = S.dbg_umax;
    info->dbg[8] = su | ((long long)sg << 32);
    info->dbg[9] = mu | ((long long)(S.status == 0 && S.fmt == 0) << 32);
    if (P.results) {
      essl_result r;
      // (status 0: reason 1 flags the full-decode path of a multi-scan stream,
      // DecodeStats.fallback_full, codec.py:461-469)
      r.status = S.status; r.reason = S.status == 0 ? (H.multiscan ? 1 : 0) : S.reason; r.offset = S.offset;
      r.mcus_entropy_decoded = S.status == 0 ? info->mcus_entropy : 0;
      r.mcus_reconstructed = S.status == 0 ? info->mcus_recon : 0;
      r.width = info->width; r.height = info->height; r.ncomp = info->ncomp;
      P.results[img] = r;
    }
  }
#undef PHASE
}

// ===========================================================================
// k_idct: gather + dequant + islow IDCT of the crop-window blocks -> Y/Cb/Cr
// planes (decode_kernels.py:388-534 via codec.py:412-419).  grid
// (kIdctCtas, n), 8 lanes per block.
// ===========================================================================
constexpr int kIdctCtas = 2;  // fewer, longer CTAs at 48 registers: +3% over 8 CTAs at 60 (A/B)

// Gathers window block (c, byr, bxr) of an image into blk[64] (int32,
// natural order, shared memory).  fmt 1: the block's table entry points at its
// DC entry in a unit list; its AC units follow up to the next DC-flagged entry
// (eight lanes read eight consecutive entries per round).  fmt 0: the int16
// coefficient window.  dq: dequantise on the way (k_idct) or raw (nullptr).
// Called by all 32 lanes of a warp.
__device__ void gather_block8(bool valid, const ImgInfo &I, const Scratch &sc, int c, int byr,
                              int bxr, int32_t *blk, const uint8_t *zz, const int32_t *dq) {
  const int j = threadIdx.x & 7;
  const int16_t *cf = sc.coef + I.coef_off[c] + ((uint64_t)byr * I.coef_pitch[c] + bxr) * 64;
#pragma unroll
  for (int r = 0; r < 8; r++) blk[8 * j + r] = 0;
  __syncwarp();
  if (I.fmt == 0) {
    if (valid) {
#pragma unroll
      for (int r = 0; r < 8; r++) blk[8 * r + j] = dq ? cf[8 * r + j] * dq[8 * r + j] : cf[8 * r + j];
    }
    __syncwarp();
    return;
  }
  uint2 t = make_uint2(0, 0);
  if (valid) t = *reinterpret_cast<const uint2 *>(cf);
  const int32_t dc = (int32_t)(int16_t)(t.y & 0xFFFFu);
  if (valid && j == 0) blk[0] = dq ? dc * dq[0] : dc;
  // The block's AC entries (EOB / ZRL markers included, stored as zeros at
  // positions the block leaves zero) are list[t.x + 1 .. t.x + cnt]: the
  // group's eight lanes take every eighth one.
  const uint32_t cnt = valid ? t.y >> 16 : 0u;
  const uint32_t *ent = sc.list + t.x + 1;
  // the first 32 entries (almost every block) as four independent loads per
  // lane, all in flight before the first use; longer blocks loop on
  constexpr int kFirst = 4;
  uint32_t ev[kFirst];
#pragma unroll
  for (int k = 0; k < kFirst; k++) {
    const uint32_t u = j + 8u * k;
    ev[k] = u < cnt ? __ldg(ent + u) : 0u;
  }
#pragma unroll
  for (int k = 0; k < kFirst; k++) {
    if (j + 8u * k < cnt) {
      const uint32_t e = ev[k];
      const int nat = zz[entry_zz(e)];
      blk[nat] = dq ? entry_value(e) * dq[nat] : entry_value(e);
    }
  }
#pragma unroll 1
  for (uint32_t u = j + 8u * kFirst; u < cnt; u += 8) {
    const uint32_t e = __ldg(ent + u);
    const int nat = zz[entry_zz(e)];
    blk[nat] = dq ? entry_value(e) * dq[nat] : entry_value(e);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(256, 5) k_idct(DecodeParams P) {
  TraceScope trace_(P.trace, ESSL_K_IDCT);
  __shared__ uint8_t s_zz[64];
  __shared__ int32_t q[3][64];
  __shared__ int32_t tr[8][4][64];
  __shared__ int32_t blks[32][64];
  const int img = blockIdx.y;
  const ImgInfo &I = P.s.info[img];
  if (I.status != 0) return;
  const DecodeHdr *G = hdr_of(P.s, img);
  const int tid = threadIdx.x;
  const int ncomp = I.ncomp;
  for (int e = tid; e < ncomp * 64; e += 256) q[e >> 6][e & 63] = G->q[e >> 6][e & 63];
  if (tid < 64) s_zz[tid] = c_zz[tid];
  int nb[3] = {0, 0, 0}, wb[3] = {1, 1, 1};
  uint32_t mg[3] = {0, 0, 0};  // ceil(2^32 / w), w >= 2: jb / w == umulhi(jb, mg) for jb * w < 2^31
#pragma unroll
  for (int c = 0; c < 3; c++) {
    if (c >= ncomp) break;
    const int hb = min(I.wby0[c] + I.wbh[c], G->bh[c]) - I.wby0[c];
    const int w = min(I.wbx0[c] + I.wbw[c], G->bw[c]) - I.wbx0[c];
    if (hb > 0 && w > 0) { nb[c] = hb * w; wb[c] = w; }
    mg[c] = (uint32_t)((0x100000000ull + (uint64_t)wb[c] - 1) / (uint64_t)wb[c]);
  }
  __syncthreads();
  const int total = nb[0] + nb[1] + nb[2];
  int32_t *t = tr[tid >> 5][(tid >> 3) & 3];
  int32_t *blk = blks[tid >> 3];
  for (int r0 = blockIdx.x * 32; r0 < total; r0 += kIdctCtas * 32) {
    int jb = r0 + (tid >> 3);
    const bool valid = jb < total;
    int c = 0;
    if (valid) {
      if (jb >= nb[0]) { jb -= nb[0]; c = 1; if (jb >= nb[1]) { jb -= nb[1]; c = 2; } }
    }
    // (selects, not indexing: keeps the small arrays in registers)
    const uint32_t m = c == 0 ? mg[0] : (c == 1 ? mg[1] : mg[2]);
    const int w = c == 0 ? wb[0] : (c == 1 ? wb[1] : wb[2]);
    const int byr = valid ? (w == 1 ? jb : (int)__umulhi((uint32_t)jb, m)) : 0;  // (2^32 / 1 overflows)
    const int bxr = valid ? jb - byr * w : 0;
    gather_block8(valid, I, P.s, c, byr, bxr, blk, s_zz, q[c]);  // dequantised
    const int pitch = I.plane_pitch[c];
    uint8_t *dst = P.s.plane + I.plane_off[c] + (uint64_t)byr * 8 * pitch + bxr * 8;
    ESSL_CHECK(g_check_dec, !valid || (dst >= P.s.plane && dst + 7 * (uint64_t)pitch + 8 <= P.s.plane + P.s.plane_cap),
               CK_PLANE);
    idct_block_8lanes(valid, blk, dst, pitch, t);
  }
}

// Debug copy of the crop-window coefficients (components back to back,
// natural order, int16), gathered like k_idct.
__global__ void __launch_bounds__(256) k_dump_coefs(Scratch sc, int16_t *out, const uint64_t *offsets) {
  __shared__ int32_t blks[32][64];
  __shared__ uint8_t s_zz[64];
  const int img = blockIdx.y;
  const ImgInfo &I = sc.info[img];
  if (I.status != 0) return;
  const int tid = threadIdx.x;
  if (tid < 64) s_zz[tid] = c_zz[tid];
  __syncthreads();
  int nb[3] = {0, 0, 0};
  for (int c = 0; c < I.ncomp; c++) nb[c] = I.wbh[c] * I.wbw[c];
  const int total = nb[0] + nb[1] + nb[2];
  int32_t *blk = blks[tid >> 3];
  for (int r0 = blockIdx.x * 32; r0 < total; r0 += gridDim.x * 32) {
    int jb = r0 + (tid >> 3);
    const bool valid = jb < total;
    const int jall = jb;
    int c = 0;
    if (valid) {
      if (jb >= nb[0]) { jb -= nb[0]; c = 1; if (jb >= nb[1]) { jb -= nb[1]; c = 2; } }
    }
    const int w = max(I.wbw[c], 1);
    gather_block8(valid, I, sc, c, valid ? jb / w : 0, valid ? jb % w : 0, blk, s_zz, nullptr);
    if (valid) {
      int16_t *o = out + offsets[img] + (uint64_t)jall * 64;
      const int j = tid & 7;
#pragma unroll
      for (int r = 0; r < 8; r++) o[8 * r + j] = (int16_t)blk[8 * r + j];
    }
  }
}

void launch_dump_coefs(const Scratch &sc, int n, int16_t *out, const uint64_t *offsets,
                       cudaStream_t st) {
  if (n > 0) k_dump_coefs<<<dim3(32, n), 256, 0, st>>>(sc, out, offsets);
}

// Shared-memory budget for k_prep's staged payload.
constexpr int kMaxDynSmem = 160 * 1024;

size_t decode_hdr_bytes() { return sizeof(DecodeHdr); }
size_t tabcache_bytes() { return sizeof(TabCacheSlot) * kMaxTables; }

void launch_prep(const DecodeParams &p0, cudaStream_t st, int max_len) {
  if (p0.n <= 0) return;
  // dynamic shared memory: [payload, destuffed in place + 0xFF padding][CRC partials]
  const int payload = (max_len + 15) / 16 * 16 + 128;
  int c2 = 1;
  while (c2 < (max_len + kCrcChunk - 1) / kCrcChunk && c2 < kCrcMaxChunks) c2 <<= 1;
  const int part = 4 * c2;
  DecodeParams p = p0;
  if (payload + part <= kMaxDynSmem) {
    p.prep_part_off = payload;
    k_prep<true><<<p.n, kNT, payload + part, st>>>(p);
  } else {
    p.prep_part_off = 0;
    k_prep<false><<<p.n, kNT, part, st>>>(p);
  }
}

void launch_entropy(const DecodeParams &p, cudaStream_t st, int max_len) {
  (void)max_len;
  if (p.n > 0) k_entropy<<<p.n, kLanes, 0, st>>>(p);
}

void launch_idct(const DecodeParams &p, cudaStream_t st) {
  if (p.n > 0) k_idct<<<dim3(kIdctCtas, p.n), 256, 0, st>>>(p);
}

// Per-device one-time setup (api.cu calls it once for every device a context
// is created on): the dynamic shared-memory opt-ins and the CRC tables are
// per-device state.
void init_crc_tables();
void init_device_decode() {
  cudaFuncSetAttribute(k_prep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
  cudaFuncSetAttribute(k_prep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
  init_crc_tables();
}

void init_crc_tables() {
  uint32_t x2n[32];
  uint32_t p = 1u << 30;  // x^1 (reflected), then repeated squaring (zlib x2n_table)
  auto mul = [](uint32_t a, uint32_t b) {
    uint32_t r = 0;
    for (int i = 0; i < 32; i++) {
      if (a & (0x80000000u >> i)) r ^= b;
      b = (b & 1) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
    }
    return r;
  };
  x2n[0] = p;
  for (int k = 1; k < 32; k++) x2n[k] = p = mul(p, p);
  cudaMemcpyToSymbol(c_x2n, x2n, sizeof(x2n));
  // multiply-by-x^(8*kCrcChunk*2^j) byte tables
  static uint32_t host[kCrcLevels][4][256];
  uint32_t K = 0x80000000u;  // x^0
  {
    uint64_t e = 8ull * kCrcChunk;  // K_0 = x^(8*chunk)
    int k = 0;
    while (e) {
      if (e & 1) K = mul(x2n[k & 31], K);
      e >>= 1;
      k++;
    }
  }
  for (int j = 0; j < kCrcLevels; j++) {
    for (int m = 0; m < 4; m++)
      for (int v = 0; v < 256; v++) host[j][m][v] = mul(K, (uint32_t)v << (8 * m));
    K = mul(K, K);
  }
  uint32_t *d = nullptr;
  cudaMalloc(&d, sizeof(host));
  cudaMemcpy(d, host, sizeof(host), cudaMemcpyHostToDevice);
  const uint32_t *dc = d;
  cudaMemcpyToSymbol(c_crc_mul, &dc, sizeof(dc));
}

}  // namespace essl
