// Synthetic stereo renderer for the benchmark sequences (configs 2-5).
//
// Restates the reference's ray caster (synth.py:87-218) bit-exactly:
// per-pixel rays through the rectified pinhole rig, whose world directions
// ``dir_cam @ R.T`` (synth.py:175) are formed in OpenBLAS dgemm order
// (dgemm_dot3, es_common.cuh); fronto-parallel planes, optionally bounded
// (synth.py:27-38,147-163), and axis-aligned boxes by slab intersection
// (synth.py:41-50,130-170); the two-octave value-noise texture with the
// splitmix-style uint64 lattice hash (synth.py:87-127); background intensity
// where nothing is hit; ground-truth disparity f*b/Z.  Every other float64
// operation is one IEEE op in numpy's order (the TU is built -fmad=false).
// This is input generation, off the hot path: it
// replaces ~1.5 s/frame of numpy ray casting, and because its bytes equal
// synth.render_frame's, the bench and the full-size parity tests consume
// exactly the images the reference renders (tests/test_gpu_render.py).
#include "es_common.cuh"
#include "es_kernels.h"

namespace es {

__device__ __forceinline__ double lattice_hash(long long ix, long long iy, long long iz,
                                               long long seed) {
  unsigned long long h = (unsigned long long)ix * 0x9E3779B97F4A7C15ull;
  h ^= (unsigned long long)iy * 0xC2B2AE3D27D4EB4Full;
  h ^= (unsigned long long)iz * 0x165667B19E3779F9ull;
  h ^= (unsigned long long)seed * 0x27D4EB2F165667C5ull;
  h ^= h >> 30;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 27;
  h *= 0x94D049BB133111EBull;
  h ^= h >> 31;
  return (double)(h >> 11) / 9007199254740992.0;
}

__device__ double value_noise(double px, double py, double pz, long long seed) {
  const double bx = floor(px), by = floor(py), bz = floor(pz);
  double fx = px - bx, fy = py - by, fz = pz - bz;
  fx = fx * fx * (3.0 - 2.0 * fx);
  fy = fy * fy * (3.0 - 2.0 * fy);
  fz = fz * fz * (3.0 - 2.0 * fz);
  const long long ix = (long long)bx, iy = (long long)by, iz = (long long)bz;
  double out = 0.0;
  for (int c = 0; c < 8; ++c) {
    const int ox = c & 1, oy = (c >> 1) & 1, oz = (c >> 2) & 1;
    const double h = lattice_hash(ix + ox, iy + oy, iz + oz, seed);
    const double wx = ox ? fx : 1.0 - fx;
    const double wy = oy ? fy : 1.0 - fy;
    const double wz = oz ? fz : 1.0 - fz;
    out += h * wx * wy * wz;
  }
  return out;
}

__device__ __forceinline__ void slab(double c, double d, double lo, double hi, double& tmin,
                                     double& tmax) {
  if (d == 0.0) {
    const bool inside = c >= lo && c <= hi;
    tmin = inside ? -INFINITY : INFINITY;
    tmax = inside ? INFINITY : -INFINITY;
    return;
  }
  const double inv = 1.0 / d;
  const double t1 = (lo - c) * inv, t2 = (hi - c) * inv;
  tmin = fmin(t1, t2);
  tmax = fmax(t1, t2);
}

// one primitive record: [kind, p0..p5, flags]
//   kind 0 box:   x0 x1 y0 y1 z0 z1
//   kind 1 plane: z x0 x1 y0 y1 -, flags bit 0..3 = x0 x1 y0 y1 present
__device__ __forceinline__ double intersect(const double* pr, const double* o, const double* d) {
  if (pr[0] != 0.0) {
    const double dz = d[2];
    double t = (pr[1] - o[2]) / dz;
    if (fabs(dz) < 1e-15) t = INFINITY;
    const double px = o[0] + t * d[0];
    const double py = o[1] + t * d[1];
    const int fl = (int)pr[7];
    bool ok = t > 1e-6;
    if (fl & 1) ok &= px >= pr[2];
    if (fl & 2) ok &= px <= pr[3];
    if (fl & 4) ok &= py >= pr[4];
    if (fl & 8) ok &= py <= pr[5];
    return ok ? t : INFINITY;
  }
  double t0x, t1x, t0y, t1y, t0z, t1z;
  slab(o[0], d[0], pr[1], pr[2], t0x, t1x);
  slab(o[1], d[1], pr[3], pr[4], t0y, t1y);
  slab(o[2], d[2], pr[5], pr[6], t0z, t1z);
  const double tn = fmax(fmax(t0x, t0y), t0z);
  const double tf = fmin(fmin(t1x, t1y), t1z);
  return (tn <= tf && tn > 1e-6) ? tn : INFINITY;
}

__global__ void k_render(RenderArgs a) {
  const int W = a.rig.W, H = a.rig.H;
  const size_t HW = (size_t)W * H;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int)HW) return;
  const int seq = blockIdx.y >> 1, view = blockIdx.y & 1;
  const double* T = a.poses + 16 * seq;
  const double* prims = a.prims + (size_t)seq * a.n_prim * 8;
  const int x = i % W, y = i / W;
  const double dcx = ((double)x - a.rig.cx) / a.rig.f, dcy = ((double)y - a.rig.cy) / a.rig.f;
  double dir[3], cen[3];
  for (int r = 0; r < 3; ++r) {
    dir[r] = dgemm_dot3(dcx, T[4 * r + 0], dcy, T[4 * r + 1], 1.0, T[4 * r + 2]);
    // c_right = c_left + R @ (b, 0, 0): the zero terms are exact
    cen[r] = T[4 * r + 3] + (view ? T[4 * r + 0] * a.rig.b : 0.0);
  }
  double tbest = INFINITY;
  for (int k = 0; k < a.n_prim; ++k) tbest = fmin(tbest, intersect(prims + 8 * k, cen, dir));
  const bool hit = isfinite(tbest);
  double inten = (double)a.background;
  if (hit) {
    const double s = a.texture_scale;
    const double qx = (cen[0] + tbest * dir[0]) / s;
    const double qy = (cen[1] + tbest * dir[1]) / s;
    const double qz = (cen[2] + tbest * dir[2]) / s;
    const long long seed = a.seeds[seq];
    const double v = 0.65 * value_noise(qx, qy, qz, seed) +
                     0.35 * value_noise(2.0 * qx, 2.0 * qy, 2.0 * qz, seed + 1);
    inten = 20.0 + 215.0 * fmin(fmax(v, 0.0), 1.0);
  }
  const double q = fmin(fmax(rint(inten), 0.0), 255.0);
  const size_t o = (size_t)blockIdx.y * HW + i;
  a.img[o] = (uint8_t)q;
  if (a.gt) {
    const double disp = hit ? (a.rig.f * a.rig.b) / tbest : 0.0;
    a.gt[o] = (hit && disp <= a.rig.d_max) ? disp : 0.0;
  }
}

void launch_render(const RenderArgs& a, int n_seq, cudaStream_t st) {
  const int HW = a.rig.W * a.rig.H;
  k_render<<<dim3((HW + 127) / 128, 2 * n_seq), 128, 0, st>>>(a);
}

}  // namespace es
