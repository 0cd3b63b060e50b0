/* Lane -> node map search for the 3-D STP kernel (one n^3 cell per 128-thread
 * CTA) under the measured shared-memory wavefront rule (tools/probes/lds_wf.cu):
 *   wavefronts of a warp-wide LDS.64 = max( max over lane quads of
 *   ceil(distinct addresses in the quad / 2), max over the 16 bank pairs of the
 *   distinct addresses mapping to it ).
 * Flux buffers are stored in lane order (pos[node] = lane), so stores are
 * conflict-free; the search minimises the summed wavefronts of the 3 n
 * derivative loads (axis a, index l) over the 4 warps by simulated annealing.
 *   gcc -O2 -o perm3d perm3d.c -lm && ./perm3d N [iters] [seed]
 * prints the row-major baseline, the best cost and the permutation. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static int N, NPC, L;          /* L = 128 lanes */
static int perm[128], pos[512];

static int warp_cost(int w) {
  int total = 0;
  for (int a = 0; a < 3; ++a)
    for (int l = 0; l < N; ++l) {
      int addr[32];
      for (int t = 0; t < 32; ++t) {
        int nd = perm[w * 32 + t];
        if (nd < 0) { addr[t] = -1; continue; }
        int c[3] = {nd / (N * N), (nd / N) % N, nd % N};
        c[a] = l;
        addr[t] = pos[(c[0] * N + c[1]) * N + c[2]];
      }
      int wf = 1;
      for (int q = 0; q < 8; ++q) {   /* distinct per quad */
        int d = 0, seen[4];
        for (int u = 0; u < 4; ++u) {
          int x = addr[q * 4 + u];
          if (x < 0) continue;
          int f = 0;
          for (int v = 0; v < d; ++v) f |= seen[v] == x;
          if (!f) seen[d++] = x;
        }
        int need = (d + 1) / 2;
        if (need > wf) wf = need;
      }
      int bank[16][32], nb[16];
      memset(nb, 0, sizeof nb);
      for (int t = 0; t < 32; ++t) {
        int x = addr[t];
        if (x < 0) continue;
        int b = x & 15, f = 0;
        for (int v = 0; v < nb[b]; ++v) f |= bank[b][v] == x;
        if (!f) bank[b][nb[b]++] = x;
      }
      for (int b = 0; b < 16; ++b)
        if (nb[b] > wf) wf = nb[b];
      total += wf;
    }
  return total;
}

static void set_pos(void) {
  for (int t = 0; t < L; ++t)
    if (perm[t] >= 0) pos[perm[t]] = t;
}

static int cost(void) {
  int c = 0;
  for (int w = 0; w < L / 32; ++w) c += warp_cost(w);
  return c;
}

int main(int argc, char** argv) {
  N = argc > 1 ? atoi(argv[1]) : 5;
  long iters = argc > 2 ? atol(argv[2]) : 2000000;
  srand(argc > 3 ? atoi(argv[3]) : 1);
  NPC = N * N * N;
  L = ((NPC + 31) / 32) * 32;
  for (int t = 0; t < L; ++t) perm[t] = t < NPC ? t : -1;
  /* row-major baseline with row-major storage */
  for (int nd = 0; nd < NPC; ++nd) pos[nd] = nd;
  int base = cost();
  set_pos();
  int cur = cost(), best = cur;
  int bestp[128];
  memcpy(bestp, perm, sizeof perm);
  double T0 = 2.0;
  for (long it = 0; it < iters; ++it) {
    double T = T0 * (1.0 - (double)it / iters) + 1e-3;
    int x = rand() % L, y = rand() % L;
    if (x == y || (perm[x] < 0 && perm[y] < 0)) continue;
    int wx = x / 32, wy = y / 32;
    int before = warp_cost(wx) + (wy != wx ? warp_cost(wy) : 0);
    int t = perm[x]; perm[x] = perm[y]; perm[y] = t;
    set_pos();
    /* storage moves with the lanes: every warp's loads may change */
    int after = cost();
    int delta = after - cur;
    (void)before;
    if (delta <= 0 || exp(-delta / T) > (double)rand() / RAND_MAX) {
      cur = after;
      if (cur < best) { best = cur; memcpy(bestp, perm, sizeof perm); }
    } else {
      t = perm[x]; perm[x] = perm[y]; perm[y] = t;
      set_pos();
    }
  }
  printf("N=%d row-major wavefronts %d (per load %.3f), best %d (per load %.3f)\n", N, base,
         (double)base / (L / 32 * 3 * N), best, (double)best / (L / 32 * 3 * N));
  for (int t = 0; t < L; ++t) printf("%d%s", bestp[t], t + 1 < L ? "," : "\n");
  return 0;
}
