/* Design experiment for the speculative (self-synchronising) entropy
 * decoder: how many bits does a decoder started at an arbitrary bit
 * position with a guessed state (k=0, block 0) need before it lands on
 * the true path's (bitpos, k, block-in-MCU) state?  Reads JPEG streams
 * (baseline, no DRI) and prints the distribution.
 * Build: gcc -O2 tools/sync_experiment.c -o /tmp/syncx -lm -lpthread */
#include "../oracle/essl_oracle.c"
#include <stdio.h>

typedef struct { int k, b; } St;

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

int main(int argc, char **argv) {
  long hist[64] = {0}; long tot = 0, nosync = 0;
  for (int a = 1; a < argc; a++) {
    FILE *fp = fopen(argv[a], "rb"); static uint8_t d[1 << 22];
    int n = fread(d, 1, sizeof d, fp); fclose(fp);
    Frame f; Err e; if (parse_stream(d, n, &f, &e)) continue;
    Scan *sc = &f.scan; if (sc->ri || f.progressive) continue;
    uint8_t *clean = malloc(n); int64_t rst[4]; int nr;
    int64_t clen = orc_destuff(d + sc->start, 0, sc->end - sc->start, clean, rst, 0, &nr, NULL);
    int32_t *ld[4], *la[4];
    for (int s = 0; s < sc->ns; s++) { ld[s] = malloc(65536*4); la[s] = malloc(65536*4); huff_lut(&sc->dc[s], ld[s], &e); huff_lut(&sc->ac[s], la[s], &e); }
    int bslot[64], bpm = 0;
    for (int s = 0; s < sc->ns; s++) { int hh = sc->ns > 1 ? f.comps[sc->comp[s]].h : 1, vv = sc->ns > 1 ? f.comps[sc->comp[s]].v : 1; for (int q = 0; q < hh * vv; q++) bslot[bpm++] = s; }
    int64_t nb = clen * 8 + 64; int8_t *tk = malloc(nb); int8_t *tb = malloc(nb); memset(tk, -1, nb);
    BR br = {clean, clen, 0, 0, 0}; int k = 0, b = 0;
    for (;;) { int64_t p = 8 * br.vpos - br.cnt; if (p >= clen * 8) break; tk[p] = k; tb[p] = b; if (unit(&br, ld, la, bslot, bpm, &k, &b)) break; }
    for (int64_t p0 = 1; p0 < clen * 8 - 4096; p0 += 97) {
      BR r2 = {clean, clen, p0 >> 3, 0, 0}; br_fill(&r2); r2.cnt -= p0 & 7;
      int k2 = 0, b2 = 0; int64_t p = p0; int synced = 0;
      while (p < p0 + 4096) {
        if (tk[p] == k2 && tb[p] == b2) { synced = 1; break; }
        if (unit(&r2, ld, la, bslot, bpm, &k2, &b2)) { k2 = 0; b2 = 0; r2.cnt -= 1; }
        p = 8 * r2.vpos - r2.cnt;
      }
      tot++; if (!synced) nosync++; else { int bin = (p - p0) / 64; if (bin > 63) bin = 63; hist[bin]++; }
    }
  }
  long c = 0; printf("starts=%ld nosync(4096b)=%ld\n", tot, nosync);
  for (int i = 0; i < 64; i++) { c += hist[i]; if (hist[i]) printf("<=%4d bits: cum %.4f\n", (i + 1) * 64, (double)c / tot); }
}
