// Evaluation metrics on the device: bad-pixel counts, bad mask, error image
// and density (reference metrics.py:39-117), batched over maps.
//
// bad (metrics.py:62-66): err = |est - gt|; "or": err > 3 || err > 0.05 gt;
// "and": both; counted over pixels valid in both maps.  Arithmetic is the
// reference's float64 (the product 0.05 * gt rounded once, no contraction:
// the library is compiled with -fmad=false).
#include <algorithm>

#include "es_common.cuh"
#include "es_kernels.h"

namespace es {

constexpr double ABS_THRESHOLD = 3.0;    // metrics.py:20
constexpr double REL_THRESHOLD = 0.05;   // metrics.py:21

__device__ __forceinline__ bool is_bad(double e, double g, int mode) {
  const double err = fabs(e - g);
  const bool over_abs = err > ABS_THRESHOLD;
  const bool over_rel = err > REL_THRESHOLD * g;
  return mode == 0 ? (over_abs || over_rel) : (over_abs && over_rel);
}

// counts[m][4] += (gt valid, jointly valid, bad, estimate valid)
__global__ void __launch_bounds__(256) k_metrics(MetricsArgs a) {
  const int m = blockIdx.y;
  const double* est = a.est + (size_t)m * a.stride_e;
  const uint8_t* ev = a.est_valid + (size_t)m * a.stride_e;
  const double* gt = a.gt + (size_t)m * a.stride_g;
  const uint8_t* gv = a.gt_valid + (size_t)m * a.stride_g;
  uint32_t c_gt = 0, c_both = 0, c_bad = 0, c_ev = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n;
       i += (size_t)gridDim.x * blockDim.x) {
    const bool g = gv[i] != 0, e = ev[i] != 0;
    const bool both = g && e;
    const bool bad = both && is_bad(est[i], gt[i], a.mode);
    c_gt += g;
    c_both += both;
    c_bad += bad;
    c_ev += e;
    if (a.mask) a.mask[(size_t)m * a.n + i] = bad;
    if (a.rgb) {
      // metrics.py:106-117: blue within threshold, red bad, black no data
      uint8_t* px = a.rgb + ((size_t)m * a.n + i) * 3;
      px[0] = bad ? 220 : (both ? 40 : 0);
      px[1] = bad ? 50 : (both ? 90 : 0);
      px[2] = bad ? 40 : (both ? 220 : 0);
    }
  }
  c_gt = __reduce_add_sync(0xffffffffu, c_gt);
  c_both = __reduce_add_sync(0xffffffffu, c_both);
  c_bad = __reduce_add_sync(0xffffffffu, c_bad);
  c_ev = __reduce_add_sync(0xffffffffu, c_ev);
  if ((threadIdx.x & 31) == 0) {
    unsigned long long* c = a.counts + (size_t)m * 4;
    atomicAdd(c + 0, (unsigned long long)c_gt);
    atomicAdd(c + 1, (unsigned long long)c_both);
    atomicAdd(c + 2, (unsigned long long)c_bad);
    atomicAdd(c + 3, (unsigned long long)c_ev);
  }
}

void launch_metrics(const MetricsArgs& a, int n_maps, cudaStream_t st) {
  const unsigned blocks = (unsigned)std::min<size_t>((a.n + 255) / 256, 148 * 8 / (size_t)std::max(n_maps, 1) + 1);
  k_metrics<<<dim3(blocks, n_maps), 256, 0, st>>>(a);
}

}  // namespace es
