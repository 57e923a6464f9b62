/* Warp-cost model of k_entropy's speculative decode (round-2 analysis tool):
 * for each JPEG (baseline, no DRI), 64 lanes over equal subsequences, lane i
 * starting W warm-up bits early from the guess (k=0, b=0) with a re-guess
 * strategy (0: one bit on with b=0, as the kernel; 1/2: retry the next
 * block-in-MCU phase at the last / first block start), and the previous
 * lane's continuation running until lane i's path has synced.  Prints the
 * per-warp maxima of warm-up, subsequence and continuation units (the warp
 * executes its slowest lane) for each W.
 * Build: gcc -O2 -include stdint.h tools/lane_sim.c -o /tmp/lane_sim -lm
 * Run:   /tmp/lane_sim a.jpg b.jpg ...   (e.g. encode_jpeg(synth_image(...), 95)) */
#include "../oracle/essl_oracle.c"
#include <stdio.h>

static int unit(BR *br, int32_t **ld, int32_t **la, const int *bslot, int bpm, int *k, int *b) {
  int s = bslot[*b];
  if (*k == 0) {
    int sym = br_hd(br, ld[s]); if (sym < 0 || sym > 15) return -1;
    br_gb(br, sym); *k = 1; return 0;
  }
  int rs = br_hd(br, la[s]); if (rs < 0) return -1;
  int r = rs >> 4, sz = rs & 15;
  if (sz == 0) { if (r == 15) { *k += 16; if (*k >= 64) { *k = 0; *b = (*b + 1) % bpm; } return 0; }
    *k = 0; *b = (*b + 1) % bpm; return 0; }
  *k += r; if (*k > 63) return -1; br_gb(br, sz); *k += 1;
  if (*k >= 64) { *k = 0; *b = (*b + 1) % bpm; }
  return 0;
}
static uint8_t *g_clean; static int64_t g_clen;
static void seek(BR *r, int64_t p) { BR t = {g_clean, g_clen, p >> 3, 0, 0}; *r = t; br_fill(r); r->cnt -= p & 7; }
static int64_t pos(BR *r) { return 8 * r->vpos - r->cnt; }


typedef struct { int64_t p; int k, b; } St;
/* decode forward from the current state with strategy st until position >= stop at a block start
   (mode 0) or unit boundary >= stop (mode 1). returns units decoded; updates state. */
static int32_t **LD, **LA; static int *BS; static int BPM;
typedef struct { BR r; int k, b; int64_t firstbs; int firstb, tries; int st; } Dec;
static void dec_init(Dec *D, int64_t p, int st) { seek(&D->r, p); D->k = 0; D->b = 0; D->firstbs = -1; D->tries = 0; D->st = st; }
static int dec_step(Dec *D) {  /* one unit (or a restart); returns 1 if a unit was decoded */
  int64_t p = pos(&D->r);
  if (D->k == 0 && D->firstbs < 0) { D->firstbs = p; D->firstb = D->b; }
  if (D->k == 0 && D->st == 1) { D->firstbs = p; D->firstb = D->b; }
  if (unit(&D->r, LD, LA, BS, BPM, &D->k, &D->b)) {
    if ((D->st == 2 || D->st == 1) && D->firstbs >= 0 && ++D->tries < BPM) { seek(&D->r, D->firstbs); D->k = 0; D->b = (D->firstb + 1) % BPM; D->firstb = D->b; }
    else { seek(&D->r, p + 1); D->k = 0; D->b = 0; D->firstbs = -1; D->tries = 0; }
  }
  return 1;
}
int main(int argc, char **argv) {
  int Ws[] = {0, 256, 512, 1024, 1536, 2048, 3072}; int nW = 7;
  double acc[4][7][3] = {{{0}}}; int nimg = 0; double totunits = 0;
  for (int a = 1; a < argc; a++) {
    FILE *fp = fopen(argv[a], "rb"); static uint8_t d[1 << 22];
    int n = fread(d, 1, sizeof d, fp); fclose(fp);
    Frame f; Err e; if (parse_stream(d, n, &f, &e)) continue;
    Scan *sc = &f.scan; if (sc->ri || f.progressive) continue;
    uint8_t *clean = malloc(n); int64_t rst[4]; int nr;
    int64_t clen = orc_destuff(d + sc->start, 0, sc->end - sc->start, clean, rst, 0, &nr, NULL);
    g_clean = clean; g_clen = clen;
    static int32_t *ld[4], *la[4];
    for (int s = 0; s < sc->ns; s++) { ld[s] = malloc(65536*4); la[s] = malloc(65536*4); huff_lut(&sc->dc[s], ld[s], &e); huff_lut(&sc->ac[s], la[s], &e); }
    static int bslot[64]; int bpm = 0;
    for (int s = 0; s < sc->ns; s++) { int hh = sc->ns > 1 ? f.comps[sc->comp[s]].h : 1, vv = sc->ns > 1 ? f.comps[sc->comp[s]].v : 1; for (int q = 0; q < hh * vv; q++) bslot[bpm++] = s; }
    LD = ld; LA = la; BS = bslot; BPM = bpm;
    int64_t nb = clen * 8 + 64; int8_t *tk = malloc(nb); int8_t *tb = malloc(nb); int32_t *tu = malloc(nb * 4); memset(tk, -1, nb);
    BR br = {clean, clen, 0, 0, 0}; int k = 0, b = 0; int32_t u = 0; int64_t endp = 0;
    for (;;) { int64_t p = pos(&br); if (p >= clen * 8) break; tk[p] = k; tb[p] = b; tu[p] = u++; endp = p; if (unit(&br, ld, la, bslot, bpm, &k, &b)) break; }
    /* unit index of the first true unit boundary at or after q */
    nimg++; totunits += u;
    int64_t bits = endp; int L = 64; int64_t slen = (bits + L - 1) / L;
    for (int st = 0; st <= 2; st += 1) for (int wi = 0; wi < nW; wi++) {
      int W = Ws[wi];
      for (int w0 = 0; w0 < L; w0 += 32) {
        double mw = 0, mp = 0, mc = 0;
        for (int i = w0; i < w0 + 32; i++) {
          int64_t sbeg = i * slen, send = (i + 1) * slen; if (send > bits) send = bits;
          int64_t p0 = i == 0 ? 0 : (sbeg > W ? sbeg - W : 0);
          Dec D; dec_init(&D, p0, st);
          long wu = 0, pu = 0;
          if (i > 0) while (!(D.k == 0 && pos(&D.r) >= sbeg)) { dec_step(&D); wu++; if (pos(&D.r) >= bits) break; }
          /* phase 1: decode to send; record sync */
          int64_t syncp = -1;
          for (;;) { int64_t p = pos(&D.r); if (syncp < 0 && p < nb && tk[p] == D.k && tb[p] == D.b && D.k == 0) syncp = p; if (p >= send) break; dec_step(&D); pu++; }
          /* continuation of lane i-1 = true units from sbeg to merge point (first synced block start) */
          long cu = 0;
          if (i > 0) { int64_t m = syncp < 0 ? send : syncp; int64_t q = sbeg; while (q < nb && tk[q] < 0) q++; int64_t q2 = m; while (q2 < nb && tk[q2] < 0) q2++; cu = tu[q2] - tu[q] + 1; }
          if (wu > mw) mw = wu; if (pu > mp) mp = pu;
          /* continuation belongs to lane i-1's warp; approximate: same warp */
          if (cu > mc) mc = cu;
        }
        acc[st][wi][0] += mw; acc[st][wi][1] += mp; acc[st][wi][2] += mc;
      }
    }
  }
  printf("images %d, true units/image %.0f (per lane %.0f)\n", nimg, totunits / nimg, totunits / nimg / 64);
  for (int st = 0; st <= 2; st += 1) for (int wi = 0; wi < nW; wi++) {
    double w = acc[st][wi][0] / nimg / 2, p = acc[st][wi][1] / nimg / 2, c = acc[st][wi][2] / nimg / 2;
    printf("strat %d W %4d: per-warp warm %.0f phase1 %.0f cont %.0f total %.0f\n", st, Ws[wi], w, p, c, w + p + c);
  }
}
