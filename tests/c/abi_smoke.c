/* Native use of the C ABI (no Python): a two-sequence context stepped over
 * a constant-shift pair, the fused KITTI export checked against the known
 * shift, and es_matching_cost checked against a brute-force 3x3 SAD written
 * here (sgm.py:160-196 semantics: edge-replicated window, border cost
 * 9*255 where the match column leaves the image, +inf outside [lo, hi]).
 * Built and run by tests/test_gpu_c_abi.py; exit code 0 = pass. */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "egostereo_b200.h"

#define CHECK(call)                                                          \
  do {                                                                       \
    int st_ = (call);                                                        \
    if (st_ != ES_OK) {                                                      \
      fprintf(stderr, "%s failed (%d): %s\n", #call, st_, es_last_error());  \
      return 1;                                                              \
    }                                                                        \
  } while (0)

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

int main(void) {
  const int W = 96, H = 40, D_MAX = 15, B = 2, SHIFT = 5;
  es_rig rig = {64.0, 0.5, (W - 1) / 2.0, (H - 1) / 2.0, W, H, D_MAX};
  es_params prm = {3, 7.0, 86.0, 10.0, 0.25, 1.0, 200.0, 0.5, 3.0, 3.0, 1, 1, 1, 1.0, 0};
  unsigned char* img = malloc((size_t)B * 2 * H * W);
  srand(7);
  for (int s = 0; s < B; ++s) {
    unsigned char* left = img + (size_t)s * 2 * H * W;
    unsigned char* right = left + (size_t)H * W;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W + SHIFT; ++x) {
        const unsigned char v = (unsigned char)(rand() & 255);
        if (x < W) left[y * W + x] = v;               /* left(x) = base(x) */
        if (x >= SHIFT) right[y * W + x - SHIFT] = v;  /* right(x) = base(x + shift) */
      }
  }
  /* ---- context: frame 0 full range, frame 1 with identity motion -------- */
  es_ctx* ctx = NULL;
  CHECK(es_ctx_create(0, &rig, &prm, B, &ctx));
  double hm[B * 2 * 16];
  unsigned char given[B];
  memset(hm, 0, sizeof hm);
  for (int k = 0; k < B * 2; ++k)
    for (int i = 0; i < 4; ++i) hm[k * 16 + i * 5] = 1.0;   /* identity homographies */
  memset(given, 0, sizeof given);
  CHECK(es_ctx_step(ctx, img, 0, hm, given, 1));
  memset(given, 1, sizeof given);
  CHECK(es_ctx_step(ctx, img, 0, hm, given, 1));
  unsigned short* kitti = malloc(sizeof(unsigned short) * B * H * W);
  CHECK(es_ctx_export_all(ctx, ES_FUSED_KITTI, 0, kitti, 1));
  long good = 0, total = 0;
  for (int s = 0; s < B; ++s)
    for (int y = 2; y < H - 2; ++y)
      for (int x = SHIFT + 2; x < W - 2; ++x) {
        total += 1;
        good += kitti[((size_t)s * H + y) * W + x] == SHIFT * 256;
      }
  uint64_t cl = 0, cr = 0;
  CHECK(es_ctx_cells(ctx, 0, &cl, &cr));
  CHECK(es_ctx_destroy(ctx));
  printf("fused interior pixels at the true shift: %ld / %ld; frame-1 searched cells %llu\n", good,
         total, (unsigned long long)cl);
  if (good < total * 95 / 100) return 2;
  if (cl >= (uint64_t)W * H * (D_MAX + 1)) return 3;   /* frame 1 must search less */

  /* ---- stage API: matching cost vs brute force ----------------------------- */
  const int n = H * W, D = D_MAX + 1;
  int64_t* lo = malloc(sizeof(int64_t) * n);
  int64_t* hi = malloc(sizeof(int64_t) * n);
  for (int i = 0; i < n; ++i) {
    lo[i] = (i * 7) % 9;
    hi[i] = lo[i] + (i * 3) % 7;
  }
  float* vol = malloc(sizeof(float) * n * D);
  for (int view = 0; view < 2; ++view) {
    const unsigned char* ref = img + (size_t)view * H * W;
    const unsigned char* oth = img + (size_t)(1 - view) * H * W;
    CHECK(es_matching_cost(img, img + (size_t)H * W, H, W, lo, hi, D_MAX, 3, view, vol));
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        for (int d = 0; d < D; ++d) {
          const int i = y * W + x;
          float want;
          const int xm = view == 0 ? x - d : x + d;
          if (d < lo[i] || d > hi[i]) want = INFINITY;
          else if (xm < 0 || xm > W - 1) want = 9.0f * 255.0f;
          else {
            int sad = 0;
            for (int oy = -1; oy <= 1; ++oy)
              for (int ox = -1; ox <= 1; ++ox) {
                const int yy = clampi(y + oy, 0, H - 1), xx = clampi(x + ox, 0, W - 1);
                const int xo = clampi(view == 0 ? xx - d : xx + d, 0, W - 1);
                sad += abs((int)ref[yy * W + xx] - (int)oth[yy * W + xo]);
              }
            want = (float)sad;
          }
          const float got = vol[(size_t)i * D + d];
          if (!(got == want || (isinf(got) && isinf(want)))) {
            fprintf(stderr, "cost mismatch view %d (%d,%d,%d): %f vs %f\n", view, x, y, d, got, want);
            return 4;
          }
        }
  }
  printf("es_matching_cost == brute-force SAD on %d x %d x %d, both views\n", H, W, D);
  free(vol);
  free(lo);
  free(hi);
  free(kitti);
  free(img);
  return 0;
}
