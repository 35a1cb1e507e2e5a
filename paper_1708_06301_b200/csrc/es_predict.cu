// K1 + K2: forward warp with a deterministic two-phase z-buffer, Kalman
// predict of the variance, zoom-hole fill, search intervals and the
// row-ragged pair offsets.
//
// Reference: prediction.py:50-183, geometry.py:95-159, sgm.py:95-127.
//
// z-buffer (prediction.py:113-121): the surviving source of a target pixel
// is the one with the largest warped disparity d', ties to the smallest
// row-major source index.  Phase 1 (k_warp_zmax) takes atomicMax over the
// IEEE bits of d' (> 0, so bit order == numeric order); phase 2
// (k_warp_zidx) takes atomicMin over the source index among sources whose
// d' equals the phase-1 maximum.  Every kernel that needs a source's warped
// values recomputes them with the same code, so results are identical to a
// serial row-major splat regardless of scheduling.
#include "es_common.cuh"
#include "es_kernels.h"

namespace es {

// edge test (prediction.py:50-64): valid pixel whose valid-neighbour
// disparity range over the (2r+1)^2 window exceeds gamma_e
__device__ __forceinline__ bool is_edge(const double* __restrict__ d, const uint8_t* __restrict__ v,
                                        int x, int y, int W, int H, int r, double gamma_e) {
  double hi = -INFINITY, lo = INFINITY;
  for (int oy = -r; oy <= r; ++oy) {
    int yy = y + oy;
    if (yy < 0 || yy >= H) continue;
    for (int ox = -r; ox <= r; ++ox) {
      int xx = x + ox;
      if (xx < 0 || xx >= W) continue;
      size_t k = (size_t)yy * W + xx;
      if (v[k]) {
        double dv = d[k];
        hi = fmax(hi, dv);
        lo = fmin(lo, dv);
      }
    }
  }
  return (hi - lo) > gamma_e;
}

// warp one source pixel; returns true if it lands (keep test of
// prediction.py:104-106) and fills target index and d'
__device__ __forceinline__ bool warp_src(const double* __restrict__ Hm, const Rig& rig, int sx, int sy,
                                         double d, uint32_t& tgt, double& dp, bool& at_inf) {
  double xp, yp;
  at_inf = !warp_point(Hm, (double)sx, (double)sy, d, rig.cx, rig.cy, xp, yp, dp);
  if (at_inf) return false;
  double tx = rint(xp), ty = rint(yp);
  bool keep = (tx >= 0.0) && (tx < (double)rig.W) && (ty >= 0.0) && (ty < (double)rig.H) &&
              (dp > 0.0) && (dp <= (double)rig.d_max);
  if (!keep) return false;
  tgt = (uint32_t)ty * (uint32_t)rig.W + (uint32_t)tx;
  return true;
}

__global__ void k_warp_zmax(PredArgs a) {
  const int sv = blockIdx.y;
  const int s = sv >> 1;
  if (!a.have_pred[s]) return;
  const size_t HW = (size_t)a.rig.W * a.rig.H;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int)HW) return;
  const double* d = a.sd + sv * HW;
  const uint8_t* v = a.sv + sv * HW;
  uint32_t tgt = NO_SRC;
  double dp = 0.0;
  if (v[i]) {
    const int x = i % a.rig.W, y = i / a.rig.W;
    if (!(a.prm.edge_reject &&
          is_edge(d, v, x, y, a.rig.W, a.rig.H, a.prm.edge_window, a.prm.gamma_e))) {
      bool at_inf;
      const double di = d[i];
      if (warp_src(a.Hm + 16 * sv, a.rig, x, y, di, tgt, dp, at_inf)) {
        if (!(di > 0.0)) atomicOr(a.err + s, ERR_NONPOSITIVE_D << (2 * (sv & 1)));
        atomicMax(a.zkey + sv * HW + tgt, (unsigned long long)__double_as_longlong(dp));
      } else {
        tgt = NO_SRC;
        if (at_inf) atomicOr(a.err + s, ERR_POINT_AT_INFINITY << (2 * (sv & 1)));
      }
    }
  }
  // the landing of every source, so later passes never recompute the warp
  a.wt[sv * HW + i] = tgt;
  a.wd[sv * HW + i] = dp;
}

// k_warp_zmax on 32x8 pixel tiles: the tile's (32+2r)x(8+2r) neighbourhood
// of d and valid is staged in shared memory once, so the edge test
// (prediction.py:50-64) reads its window on chip instead of 9 global loads
// per pixel.  The window radius R (edge_window, 0 = no edge rejection) is a
// template parameter: the tile geometry and the window loop are compile-time
// (a runtime radius cost integer divisions in the staging loop and a
// rolled window walk; prediction stage 2.52 -> 2.22 ms per B = 64 step)
constexpr int ZT_W = 32, ZT_H = 8, ZT_RMAX = 2;

template <int R>
__global__ void __launch_bounds__(ZT_W * ZT_H) k_warp_zmax_tile(PredArgs a) {
  constexpr int r = R;
  constexpr int TW = ZT_W + 2 * r, TH = ZT_H + 2 * r;
  __shared__ double td[TH * TW];
  __shared__ uint8_t tv[TH * TW];
  const int sv = blockIdx.z;
  const int s = sv >> 1;
  if (!a.have_pred[s]) return;
  const int W = a.rig.W, H = a.rig.H;
  const size_t HW = (size_t)W * H;
  const int bx = blockIdx.x * ZT_W, by = blockIdx.y * ZT_H;
  const double* d = a.sd + sv * HW;
  const uint8_t* v = a.sv + sv * HW;
  const int tid = threadIdx.y * ZT_W + threadIdx.x;
  for (int k = tid; k < TW * TH; k += ZT_W * ZT_H) {
    const int xx = bx - r + k % TW, yy = by - r + k / TW;
    const bool in = xx >= 0 && xx < W && yy >= 0 && yy < H;
    const size_t g = (size_t)yy * W + xx;
    tv[k] = in ? v[g] : 0;
    td[k] = in ? d[g] : 0.0;
  }
  __syncthreads();
  const int x = bx + threadIdx.x, y = by + threadIdx.y;
  if (x >= W || y >= H) return;
  const int i = y * W + x;
  const int c = (threadIdx.y + r) * TW + threadIdx.x + r;
  uint32_t tgt = NO_SRC;
  double dp = 0.0;
  if (tv[c]) {
    bool edge = false;
    if (R > 0) {
      // off-image neighbours are ignored (cval = -+inf), invalid ones too
      double hi = -INFINITY, lo = INFINITY;
#pragma unroll
      for (int oy = -r; oy <= r; ++oy)
#pragma unroll
        for (int ox = -r; ox <= r; ++ox) {
          const int k = c + oy * TW + ox;
          if (tv[k]) {
            hi = fmax(hi, td[k]);
            lo = fmin(lo, td[k]);
          }
        }
      edge = (hi - lo) > a.prm.gamma_e;
    }
    if (!edge) {
      bool at_inf;
      const double di = td[c];
      if (warp_src(a.Hm + 16 * sv, a.rig, x, y, di, tgt, dp, at_inf)) {
        if (!(di > 0.0)) atomicOr(a.err + s, ERR_NONPOSITIVE_D << (2 * (sv & 1)));
        atomicMax(a.zkey + sv * HW + tgt, (unsigned long long)__double_as_longlong(dp));
      } else {
        tgt = NO_SRC;
        if (at_inf) atomicOr(a.err + s, ERR_POINT_AT_INFINITY << (2 * (sv & 1)));
      }
    }
  }
  a.wt[sv * HW + i] = tgt;
  a.wd[sv * HW + i] = dp;
}

__global__ void k_warp_zidx(PredArgs a) {
  const int sv = blockIdx.y;
  const int s = sv >> 1;
  if (!a.have_pred[s]) return;
  const size_t HW = (size_t)a.rig.W * a.rig.H;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int)HW) return;
  const uint32_t tgt = a.wt[sv * HW + i];
  if (tgt == NO_SRC) return;
  const double dp = a.wd[sv * HW + i];
  if ((unsigned long long)__double_as_longlong(dp) == a.zkey[sv * HW + tgt])
    atomicMin(a.zidx + sv * HW + tgt, (uint32_t)i);
}

// predicted (d', p', valid) at target pixel t from the z-buffer winner
// (prediction.py:67-77,123-125: p' = (d'/d)^2 p + q)
__device__ __forceinline__ void resolve(const PredArgs& a, int sv, uint32_t t, double& od,
                                        double& op, bool& ov) {
  const size_t HW = (size_t)a.rig.W * a.rig.H;
  const uint32_t src = a.zidx[sv * HW + t];
  od = 0.0;
  op = 0.0;
  ov = false;
  if (src == NO_SRC) return;
  const double d = a.sd[sv * HW + src];
  const double p = a.sp[sv * HW + src];
  const double dp = a.wd[sv * HW + src];
  const double ratio = dp / d;
  od = dp;
  op = ratio * ratio * p + a.prm.q;
  ov = true;
}

// horizontal zoom-hole pass (prediction.py:148-166, axis=1) fused with the
// z-buffer resolve; writes the intermediate maps
__global__ void k_resolve_fill_h(PredArgs a) {
  const int sv = blockIdx.y;
  const int s = sv >> 1;
  if (!a.have_pred[s]) return;
  const int W = a.rig.W;
  const size_t HW = (size_t)W * a.rig.H;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int)HW) return;
  const int x = i % W;
  double d, p;
  bool v;
  resolve(a, sv, i, d, p, v);
  if (a.prm.fill_holes && !v && x > 0 && x < W - 1) {
    double da, pa, db, pb;
    bool va, vb;
    resolve(a, sv, i - 1, da, pa, va);
    resolve(a, sv, i + 1, db, pb, vb);
    if (va && vb && fabs(da - db) < a.prm.gamma_f) {
      d = 0.5 * (da + db);
      p = fmax(pa, pb) + a.prm.q;
      v = true;
    }
  }
  a.hd[sv * HW + i] = d;
  a.hp[sv * HW + i] = p;
  a.hv[sv * HW + i] = v;
}

// vertical pass (axis=0) + final predicted maps + search intervals + the
// row-ragged pair offsets.  One CTA per image row: pass 1 visits the row's
// pixels at a stride of NT (coalesced loads / stores) and keeps each pixel's
// slot count in shared memory; pass 2 scans contiguous chunks of the row.
template <int NT>
__global__ void __launch_bounds__(NT) k_fill_v_intervals(PredArgs a) {
  extern __shared__ uint16_t slots[];   // [W]
  __shared__ uint32_t scan_smem[32];
  __shared__ unsigned long long cells_smem;
  const int sv = blockIdx.y;
  const int s = sv >> 1;
  const int y = blockIdx.x;
  const int W = a.rig.W, H = a.rig.H, d_max = a.rig.d_max;
  const size_t HW = (size_t)W * H;
  const bool pred = a.have_pred[s] != 0;
  if (threadIdx.x == 0) cells_smem = 0ull;
  // pass 1: final predicted values, intervals, slot counts
  uint32_t my_cells = 0;
  const size_t row = sv * HW + (size_t)y * W;
  for (int x = threadIdx.x; x < W; x += NT) {
    const size_t i = row + x;
    double d = 0.0, p = 0.0;
    bool v = false;
    if (pred) {
      d = a.hd[i];
      p = a.hp[i];
      v = a.hv[i] != 0;
      if (a.prm.fill_holes && !v && y > 0 && y < H - 1) {
        const bool va = a.hv[i - W] != 0, vb = a.hv[i + W] != 0;
        const double da = a.hd[i - W], db = a.hd[i + W];
        if (va && vb && fabs(da - db) < a.prm.gamma_f) {
          d = 0.5 * (da + db);
          p = fmax(a.hp[i - W], a.hp[i + W]) + a.prm.q;
          v = true;
        }
      }
      if (!v) d = 0.0;
    }
    a.pd[i] = d;
    a.pp[i] = p;
    a.pv[i] = v;
    int lo, hi;
    interval_of(d, p, v, d_max, lo, hi);
    slots[x] = (uint16_t)pixel_slots(lo, hi);
    my_cells += (uint32_t)(hi - lo + 1);
    a.meta[i].x = (uint32_t)lo | ((uint32_t)hi << 16);
  }
  my_cells = __reduce_add_sync(0xffffffffu, my_cells);
  if ((threadIdx.x & 31) == 0) atomicAdd(&cells_smem, (unsigned long long)my_cells);
  __syncthreads();
  // pass 2: offsets (first pair at a 4-aligned slot offset + (j0 & 3))
  const int per = (W + NT - 1) / NT;
  const int x0 = min((int)threadIdx.x * per, W);
  const int x1 = min(x0 + per, W);
  uint32_t my_pairs = 0;
  for (int x = x0; x < x1; ++x) my_pairs += slots[x];
  uint32_t total;
  uint32_t base = block_exclusive_scan<NT>(my_pairs, scan_smem, total);
  const uint32_t rowbase = (uint32_t)(y * row_capacity(W, d_max));
  for (int x = x0; x < x1; ++x) {
    const size_t i = row + x;
    const int lo = a.meta[i].x & 0xFFFFu;
    a.meta[i].y = rowbase + base + pad_before(lo);
    base += slots[x];
  }
  if (threadIdx.x == 0) {
    atomicAdd(a.cells + sv, cells_smem);
    if (a.cells_acc) atomicAdd(a.cells_acc, cells_smem);
  }
}

// meta from caller-supplied intervals (stage-level matching_cost / variance)
template <int NT>
__global__ void __launch_bounds__(NT) k_meta_from_intervals(const int64_t* __restrict__ lo_in,
                                                            const int64_t* __restrict__ hi_in,
                                                            int W, int H, int d_max,
                                                            uint2* __restrict__ meta) {
  __shared__ uint32_t scan_smem[32];
  const int y = blockIdx.x;
  const int per = (W + NT - 1) / NT;
  const int x0 = threadIdx.x * per;
  const int x1 = min(x0 + per, W);
  uint32_t my_pairs = 0;
  for (int x = x0; x < x1; ++x) {
    const size_t i = (size_t)y * W + x;
    const uint32_t lo = (uint32_t)lo_in[i], hi = (uint32_t)hi_in[i];
    my_pairs += pixel_slots((int)lo, (int)hi);
    meta[i].x = lo | (hi << 16);
  }
  uint32_t total;
  uint32_t base = block_exclusive_scan<NT>(my_pairs, scan_smem, total);
  const uint32_t rowbase = (uint32_t)(y * row_capacity(W, d_max));
  for (int x = x0; x < x1; ++x) {
    const size_t i = (size_t)y * W + x;
    const uint32_t m = meta[i].x;
    const int lo = m & 0xFFFFu, hi = m >> 16;
    meta[i].y = rowbase + base + pad_before(lo);
    base += pixel_slots(lo, hi);
  }
}

// stage-level edge mask (reject_edges)
__global__ void k_edges(const double* __restrict__ d, const uint8_t* __restrict__ v, int W, int H,
                        int r, double gamma_e, uint8_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W * H) return;
  out[i] = v[i] && is_edge(d, v, i % W, i / W, W, H, r, gamma_e);
}

// ---------------------------------------------------------------- launchers

void launch_predict(const PredArgs& a, int n_sv, cudaStream_t st) {
  const int HW = a.rig.W * a.rig.H;
  dim3 grid((HW + 255) / 256, n_sv);
  cudaMemsetAsync(a.zkey, 0, sizeof(unsigned long long) * (size_t)HW * n_sv, st);
  cudaMemsetAsync(a.zidx, 0xFF, sizeof(uint32_t) * (size_t)HW * n_sv, st);
  // edge_window 0 with edge rejection on keeps the generic kernel (a 1x1
  // window still compares 0 > gamma_e)
  if (!a.prm.edge_reject || (a.prm.edge_window >= 1 && a.prm.edge_window <= ZT_RMAX)) {
    dim3 tg((a.rig.W + ZT_W - 1) / ZT_W, (a.rig.H + ZT_H - 1) / ZT_H, n_sv);
    if (!a.prm.edge_reject) k_warp_zmax_tile<0><<<tg, dim3(ZT_W, ZT_H), 0, st>>>(a);
    else if (a.prm.edge_window == 1) k_warp_zmax_tile<1><<<tg, dim3(ZT_W, ZT_H), 0, st>>>(a);
    else k_warp_zmax_tile<2><<<tg, dim3(ZT_W, ZT_H), 0, st>>>(a);
  } else {
    k_warp_zmax<<<grid, 256, 0, st>>>(a);
  }
  k_warp_zidx<<<grid, 256, 0, st>>>(a);
  k_resolve_fill_h<<<grid, 256, 0, st>>>(a);
}

void launch_fill_v_intervals(const PredArgs& a, int n_sv, cudaStream_t st) {
  cudaMemsetAsync(a.cells, 0, sizeof(unsigned long long) * n_sv, st);
  k_fill_v_intervals<256><<<dim3(a.rig.H, n_sv), 256, sizeof(uint16_t) * a.rig.W, st>>>(a);
}

void launch_meta_from_intervals(const int64_t* lo, const int64_t* hi, int W, int H, int d_max,
                                uint2* meta, cudaStream_t st) {
  k_meta_from_intervals<256><<<H, 256, 0, st>>>(lo, hi, W, H, d_max, meta);
}

void launch_edges(const double* d, const uint8_t* v, int W, int H, int r, double gamma_e,
                  uint8_t* out, cudaStream_t st) {
  k_edges<<<(W * H + 255) / 256, 256, 0, st>>>(d, v, W, H, r, gamma_e, out);
}

}  // namespace es
