/* evaluate a given lane->node map (stdin: 128 comma-separated ints) under the perm3d.c model */
#define main perm3d_main
#include "perm3d.c"
#undef main
int main(int argc, char** argv) {
  N = atoi(argv[1]); NPC = N * N * N; L = ((NPC + 31) / 32) * 32;
  for (int t = 0; t < L; ++t) if (scanf("%d,", &perm[t]) != 1) return 1;
  int lanestore = argc > 2 && atoi(argv[2]);
  if (lanestore) set_pos(); else for (int nd = 0; nd < NPC; ++nd) pos[nd] = nd;
  for (int w = 0; w < L / 32; ++w) printf("warp %d: %d\n", w, warp_cost(w));
  printf("total %d per load %.3f\n", cost(), (double)cost() / (L / 32 * 3 * N));
  return 0;
}
