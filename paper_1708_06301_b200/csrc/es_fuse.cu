// K6: left-right + SAD consistency checks fused with the per-pixel Kalman
// update, plus the stage-level kernels behind the drop-in functions.
//
// Reference: sgm.py:347-396 (lr_consistency, sad_check), pipeline.py:85-87
// (_masked), pipeline.py:144-158, fusion.py:45-79 (fuse_maps).
//
// In the frame step the SAD check reads the raw cost C(x, y, d*) that K3
// already wrote: sad_check's window SAD at rint(d*) = d* is exactly the
// un-bordered cost of the winning cell, and its off-image test coincides
// with the LR check's partner-in-image test.  All float64 arithmetic follows
// numpy's order (no FMA: the library is compiled with -fmad=false).
#include "es_common.cuh"
#include "es_kernels.h"

namespace es {

__device__ __forceinline__ void kalman(double dp, double pp, bool vp, double dm, double rm, bool vm,
                                       double p_init, double& od, double& op, bool& ov) {
  const bool both = vp && vm;
  const bool adopt = vm && !vp;
  od = 0.0;
  op = 0.0;
  if (both) {
    const double k = pp / (pp + rm);
    od = dp + k * (dm - dp);
    op = (1.0 - k) * pp;
  } else if (adopt) {
    od = dm;
    op = p_init;
  }
  ov = both || adopt;
}

__global__ void k_checks_fuse(FuseArgs a) {
  const int sv = blockIdx.y;
  const int view = sv & 1;
  const size_t HW = (size_t)a.W * a.H;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  bool nv = false;
  if (i < (int)HW) {
    const int x = i % a.W;
    const size_t o = sv * HW + i;
    const size_t po = (sv ^ 1) * HW + (i - x);   // partner view, same row
    const int d = a.dstar[o];
    const bool vm = a.mvalid[o] != 0;
    bool keep = false;
    if (vm) {
      const int xo = view == 0 ? x - d : x + d;
      if (xo >= 0 && xo < a.W && a.mvalid[po + xo] &&
          fabs((double)d - (double)a.dstar[po + xo]) <= a.tau_lr) {
        const uint2 mt = a.meta[o];
        const uint32_t w = a.C[sv * a.volcap + mt.y + ((d >> 1) - (int)(lo_of(mt) >> 1))];
        const uint32_t sad = (d & 1) ? (w >> 16) : (w & 0xFFFFu);
        keep = (double)sad <= a.tau_sad;
      }
    }
    a.keep[o] = keep;
    double nd, np;
    kalman(a.pd[o], a.pp[o], a.pv[o] != 0, keep ? (double)d : 0.0, a.r[o], keep, a.p_init, nd,
           np, nv);
    a.nd[o] = nd;
    a.np_[o] = np;
    a.nv[o] = nv;
  }
  // have_state of the next frame (pipeline.py:122): one flag per sequence,
  // one atomic per block
  if (__syncthreads_or(nv) && threadIdx.x == 0 && a.any_valid)
    atomicOr(a.any_valid + (sv >> 1), 1);
}

void launch_checks_fuse(const FuseArgs& a, int n_seq, cudaStream_t st) {
  const int HW = a.W * a.H;
  k_checks_fuse<<<dim3((HW + 255) / 256, 2 * n_seq), 256, 0, st>>>(a);
}

// ---------------------------------------------------------------- stage-level

__global__ void k_lr(const double* dl, const uint8_t* vl, const double* dr, const uint8_t* vr,
                     int W, int H, double tau, uint8_t* kl, uint8_t* kr) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H) return;
  const int x = i % W;
  const int row = i - x;
  for (int side = 0; side < 2; ++side) {
    const double* ds = side ? dr : dl;
    const uint8_t* vs = side ? vr : vl;
    const double* dd = side ? dl : dr;
    const uint8_t* vd = side ? vl : vr;
    const long long xo = (long long)x + (side ? 1 : -1) * np_to_i64(rint(ds[i]));
    const bool inb = xo >= 0 && xo < W;
    const int xc = (int)(xo < 0 ? 0 : (xo > W - 1 ? W - 1 : xo));
    const bool k = vs[i] && inb && vd[row + xc] && fabs(ds[i] - dd[row + xc]) <= tau;
    (side ? kr : kl)[i] = k;
  }
}

void launch_lr(const double* dl, const uint8_t* vl, const double* dr, const uint8_t* vr, int W,
               int H, double tau, uint8_t* kl, uint8_t* kr, cudaStream_t st) {
  k_lr<<<(W * H + 255) / 256, 256, 0, st>>>(dl, vl, dr, vr, W, H, tau, kl, kr);
}

__global__ void k_sad_check(const uint8_t* left, const uint8_t* right, const double* dmap,
                            const uint8_t* vmap, int W, int H, int window, double tau, int view,
                            uint8_t* keep) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H) return;
  const int x = i % W, y = i / W;
  bool k = false;
  if (vmap[i]) {
    const long long d = np_to_i64(rint(dmap[i]));
    const int sign = view == 0 ? -1 : 1;
    const long long c = (long long)x + sign * d;
    if (c >= 0 && c <= W - 1) {
      const uint8_t* ref = view == 0 ? left : right;
      const uint8_t* oth = view == 0 ? right : left;
      const int r = window >> 1;
      long long sad = 0;
      for (int oy = -r; oy <= r; ++oy) {
        const int yy = clampi(y + oy, 0, H - 1);
        for (int ox = -r; ox <= r; ++ox) {
          const int xx = clampi(x + ox, 0, W - 1);
          long long xm = (long long)xx + sign * d;
          xm = xm < 0 ? 0 : (xm > W - 1 ? W - 1 : xm);
          sad += abs((int)ref[(size_t)yy * W + xx] - (int)oth[(size_t)yy * W + xm]);
        }
      }
      k = (double)sad <= tau;
    }
  }
  keep[i] = k;
}

void launch_sad_check(const uint8_t* left, const uint8_t* right, const double* d, const uint8_t* v,
                      int W, int H, int window, double tau, int view, uint8_t* keep,
                      cudaStream_t st) {
  k_sad_check<<<(W * H + 255) / 256, 256, 0, st>>>(left, right, d, v, W, H, window, tau, view, keep);
}

__global__ void k_fuse(const double* dp, const double* pp, const uint8_t* vp, const double* dm,
                       const double* rm, const uint8_t* vm, int n, double p_init, double* od,
                       double* op, uint8_t* ov) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d, p;
  bool v;
  kalman(dp[i], pp[i], vp[i] != 0, dm[i], rm[i], vm[i] != 0, p_init, d, p, v);
  od[i] = d;
  op[i] = p;
  ov[i] = v;
}

void launch_fuse(const double* dp, const double* pp, const uint8_t* vp, const double* dm,
                 const double* rm, const uint8_t* vm, int n, double p_init, double* od,
                 double* op, uint8_t* ov, cudaStream_t st) {
  k_fuse<<<(n + 255) / 256, 256, 0, st>>>(dp, pp, vp, dm, rm, vm, n, p_init, od, op, ov);
}

// one simultaneous zoom-hole pass along an axis (prediction.py:148-166);
// final_pass zeroes d at invalid pixels (prediction.py:183)
__global__ void k_fill_axis(const double* d, const double* p, const uint8_t* v, int W, int H,
                            int axis, double gamma_f, double q, double* od, double* op,
                            uint8_t* ov, int final_pass) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H) return;
  const int x = i % W, y = i / W;
  double dd = d[i], pp = p[i];
  bool vv = v[i] != 0;
  const int step = axis == 1 ? 1 : W;
  const bool has_nb = axis == 1 ? (x > 0 && x < W - 1) : (y > 0 && y < H - 1);
  if (!vv && has_nb && v[i - step] && v[i + step] && fabs(d[i - step] - d[i + step]) < gamma_f) {
    dd = 0.5 * (d[i - step] + d[i + step]);
    pp = fmax(p[i - step], p[i + step]) + q;
    vv = true;
  }
  od[i] = (final_pass && !vv) ? 0.0 : dd;
  op[i] = pp;
  ov[i] = vv;
}

void launch_fill_axis(const double* d, const double* p, const uint8_t* v, int W, int H, int axis,
                      double gamma_f, double q, double* od, double* op, uint8_t* ov, int final_pass,
                      cudaStream_t st) {
  k_fill_axis<<<(W * H + 255) / 256, 256, 0, st>>>(d, p, v, W, H, axis, gamma_f, q, od, op, ov,
                                                   final_pass);
}

__global__ void k_intervals_only(const double* d, const double* p, const uint8_t* v, int n,
                                 int d_max, int64_t* lo, int64_t* hi) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int l, h;
  interval_of(d[i], p[i], v[i] != 0, d_max, l, h);
  lo[i] = l;
  hi[i] = h;
}

void launch_intervals_only(const double* d, const double* p, const uint8_t* v, int n, int d_max,
                           int64_t* lo, int64_t* hi, cudaStream_t st) {
  k_intervals_only<<<(n + 255) / 256, 256, 0, st>>>(d, p, v, n, d_max, lo, hi);
}

}  // namespace es
