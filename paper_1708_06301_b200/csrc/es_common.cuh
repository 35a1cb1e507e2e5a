// Common device types and helpers for the egostereo B200 hot path.
//
// Data layout in HBM (per sequence s, view v; "sv" = 2*s + v):
//   images      uint8  [B][2][H][W]               (left = 0, right = 1)
//   state d, p  f64    [B][2][H][W], valid uint8   (double-buffered)
//   meta        uint2  [B][2][H][W]  .x = lo | hi << 16, .y = pair offset
//   volumes     u16    pairs [B][2][H][rowcap]     (rowcap = W * npairs_max)
// A pixel's interval [lo, hi] is stored as whole u16 pairs j = lo>>1 .. hi>>1
// (pair j holds d = 2j, 2j+1), row-ragged: each image row owns a fixed
// window of rowcap pairs and packs its pixels' pairs contiguously inside it.
// Halves outside [lo, hi] hold the U16 "infinity" 0x8000.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace es {

constexpr uint32_t INF16 = 0x8000u;            // u16 +inf sentinel
constexpr uint32_t INF16x2 = 0x80008000u;
constexpr uint32_t NO_SRC = 0xFFFFFFFFu;

struct Rig {
  double f, b, cx, cy;
  int W, H, d_max;
};

struct Params {
  int window;
  float p1, p2;          // float32 penalties (numpy float32 arithmetic)
  uint32_t p1i, p2i;     // integer penalties for the u16 path
  double s_max, r_min, tau_lr, tau_sad;
  double q, gamma_f, gamma_e;
  int edge_window, edge_reject, fill_holes;
  double p_init;
};

// error bits (per sequence; shifted left by 2 * view so the host can report
// them in the reference's order: left view first, and within a view the
// warp's PointAtInfinityError before propagate_variance's ValueError,
// prediction.py:100-109, 129-145)
constexpr int ERR_POINT_AT_INFINITY = 1;
constexpr int ERR_NONPOSITIVE_D = 2;

__host__ __device__ inline int npairs_max(int d_max) { return (d_max >> 1) + 1; }

// Storage of one pixel: its pairs start at an offset o + (j0 & 3) inside an
// allocation of pixel_slots() pairs at an offset o that is a multiple of 4,
// so (offset - j0) is a multiple of 4: the 8-cell block b (cells 8b .. 8b+7,
// pairs 4b .. 4b+3) of any pixel is one aligned 16-byte word inside the
// pixel's own allocation, and the pairs 2k, 2k+1 one aligned 8-byte word.
// Padding slots (before / after the interval pairs) are written +inf by the
// cost pass, so aligned accesses that overlap them read +inf.
__host__ __device__ inline uint32_t pad_before(int lo) { return ((uint32_t)lo >> 1) & 3u; }
__host__ __device__ inline uint32_t pixel_slots(int lo, int hi) {
  const uint32_t j0 = (uint32_t)lo >> 1, j1 = (uint32_t)hi >> 1;
  return (j1 - j0 + 1 + pad_before(lo) + 3) & ~3u;
}
// pairs reserved per image row (a multiple of 4: rows start 16-byte aligned);
// a pixel never needs more than the full range rounded up to 4 pairs
__host__ __device__ inline size_t row_capacity(int W, int d_max) {
  const size_t per = (size_t)((npairs_max(d_max) + 3) & ~3);
  return (size_t)W * per;
}

__device__ __forceinline__ uint32_t lo_of(uint2 m) { return m.x & 0xFFFFu; }
__device__ __forceinline__ uint32_t hi_of(uint2 m) { return m.x >> 16; }

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(max(v, lo), hi); }

// numpy's float64 -> int64 conversion of floor/ceil/rint results on x86:
// out-of-range and NaN become INT64_MIN.
__device__ __forceinline__ long long np_to_i64(double v) {
  if (!(v >= -9.2233720368547758e18 && v < 9.2233720368547758e18)) return (long long)0x8000000000000000ULL;
  return (long long)v;
}

// The reference's (N,K) @ (K,M) float64 products (``hom @ H.T``,
// geometry.py:110; ``dir_cam @ R.T``, synth.py:175) run through OpenBLAS
// dgemm, whose kernel accumulates k = 0, 1, ... with fused multiply-adds:
// acc = a0*b0; acc = fma(a_k, b_k, acc).  Measured bit-exact against numpy
// in the build container (OpenBLAS 0.3.30, Haswell kernel) on 10^6 points;
// the TU is otherwise compiled with -fmad=false, so every other a*b+c rounds
// twice as numpy's elementwise ops do.
__device__ __forceinline__ double dgemm_dot3(double a0, double b0, double a1, double b1,
                                             double a2, double b2) {
  return __fma_rn(a2, b2, __fma_rn(a1, b1, __dmul_rn(a0, b0)));
}

// Warp a pixel through a disparity-space homography exactly as the reference
// does (geometry.py:95-159): hom = (x-cx, y-cy, d, 1), out = hom @ H.T in
// dgemm order (the k = 3 term is fma(1, h3, acc) = acc + h3).  Returns
// false when the fourth homogeneous component vanishes (PointAtInfinityError).
__device__ __forceinline__ bool warp_point(const double* __restrict__ Hm, double x, double y,
                                           double d, double cx, double cy, double& xp,
                                           double& yp, double& dp) {
  double px = x - cx, py = y - cy;
  double o[4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
    o[r] = __dadd_rn(dgemm_dot3(px, Hm[4 * r + 0], py, Hm[4 * r + 1], d, Hm[4 * r + 2]),
                     Hm[4 * r + 3]);
  if (fabs(o[3]) < 1e-12) return false;
  xp = o[0] / o[3] + cx;
  yp = o[1] / o[3] + cy;
  dp = o[2] / o[3];
  return true;
}

// widen/clamp an interval exactly as sgm.py:114-126
__device__ __forceinline__ void interval_of(double d, double p, bool valid, int d_max, int& lo,
                                            int& hi) {
  if (!valid) {
    lo = 0;
    hi = d_max;
    return;
  }
  const double s3 = 3.0 * sqrt(fmax(p, 0.0));
  long long l = np_to_i64(floor(d - s3));
  long long h = np_to_i64(ceil(d + s3));
  l = l < 0 ? 0 : (l > d_max ? d_max : l);
  h = h < 0 ? 0 : (h > d_max ? d_max : h);
  for (int k = 0; k < 2; ++k) {
    if ((h - l) < 2 && l > 0) --l;
    if ((h - l) < 2 && h < d_max) ++h;
  }
  lo = (int)l;
  hi = (int)h;
}

// block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024)
template <int NT>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* smem32,
                                                         uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem32[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < NT / 32 ? smem32[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) smem32[lane] = w;
  }
  __syncthreads();
  uint32_t base = wid ? smem32[wid - 1] : 0u;
  total = smem32[NT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

}  // namespace es
