// K4, fused column + diagonal pass: the six vertical / diagonal SGM path
// directions in two row sweeps (down: (0,+1), (+1,+1), (-1,+1); up: (0,-1),
// (-1,-1), (+1,-1)), one thread-block cluster per view.
//
// Reference: sgm.py:199-272 (_path_step, _scan_vertical, aggregate_paths).
// Every direction of a sweep takes its predecessor in the previous row of
// the sweep: column x itself (A), column x-1 (B) or column x+1 (C).  The
// cluster's CTAs own contiguous column ranges of the view; each CTA keeps the
// path state of its columns in shared memory (absolute disparity layout, the
// u16x2 words of k_sgm_grp4), A in place and B / C double-buffered by row
// parity, plus one halo column on each side that the neighbouring CTA pushes
// through distributed shared memory after computing its edge column.  One
// cluster barrier per row orders the halo pushes and the buffer flip.  Per
// searched cell the pass reads the cost once and read-modify-writes the
// partial sum once for three directions (k_sgm_grp4 does both per direction).
//
// Work inside a CTA: a warp takes groups of 4 adjacent columns (8 lanes per
// column, 4 words per lane per 64-cell chunk); per group it loads every old
// state word it needs (own words and the d-1 / d+1 edge words of the three
// predecessor columns), then computes and stores, so the in-place A state is
// never read after it is overwritten.  Arithmetic, +inf convention and the
// chunk union are those of k_sgm_grp4.
#include <cstdlib>

#include "es_common.cuh"
#include "es_kernels.h"

namespace es {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int VG = 8;                 // lanes per column
constexpr int VPPL = 4;               // words (u16 pairs) per lane per chunk
constexpr int VCW = VG * VPPL;        // words per chunk (64 cells)
constexpr int VNCH = 2;               // chunks per column: d_max <= 127
constexpr int VNW = VCW * VNCH;       // state words per column
constexpr int VNG = 32 / VG;          // columns per warp group
constexpr int VC = 8;                 // CTAs per cluster (one cluster per view)
constexpr int VWARPS = 16;
constexpr int VSLOT = 5 * VNW + 10;   // smem words per column slot (A, 2 B, 2 C, 5 m pairs)

__host__ __device__ inline void vd_range(int W, int k, int& c0, int& nc) {
  const int ng = (W + VNG - 1) / VNG;
  const int g0 = (int)((long long)ng * k / VC), g1 = (int)((long long)ng * (k + 1) / VC);
  c0 = g0 * VNG;
  nc = (g1 - g0) * VNG;   // the last CTA may own columns past W (inactive)
}
__host__ __device__ inline int vd_maxcols(int W) {
  const int ng = (W + VNG - 1) / VNG;
  return ((ng + VC - 1) / VC) * VNG;
}
inline size_t vd_smem_bytes(int W) { return sizeof(uint32_t) * (size_t)(vd_maxcols(W) + 2) * VSLOT; }

__device__ __forceinline__ uint4 lds4(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ void sts4(uint32_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  *reinterpret_cast<uint4*>(p) = make_uint4(a, b, c, d);
}

// store 16 bytes into the same shared-memory offset of CTA `rank` of the cluster
__device__ __forceinline__ void st_cluster4(const uint32_t* local, int rank, uint4 v) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};"
               :: "r"(ra), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_cluster2(const uint32_t* local, int rank, uint32_t x, uint32_t y) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("st.shared::cluster.v2.u32 [%0], {%1, %2};" :: "r"(ra), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// one path update of a lane's 4 words: L = C + min(Lp(d), min(Lp(d-1), Lp(d+1)) + P1, m + P2) - m
__device__ __forceinline__ void vd_path(const uint32_t (&P)[VPPL], uint32_t el, uint32_t er,
                                        uint32_t mp2, uint32_t ng, uint32_t p1x2,
                                        const uint32_t* cn, uint32_t (&L)[VPPL]) {
  uint32_t X[VPPL + 1];
  X[0] = __byte_perm(el, P[0], 0x5432);
#pragma unroll
  for (int k = 1; k < VPPL; ++k) X[k] = __byte_perm(P[k - 1], P[k], 0x5432);
  X[VPPL] = __byte_perm(P[VPPL - 1], er, 0x5432);
#pragma unroll
  for (int k = 0; k < VPPL; ++k) {
    const uint32_t cand = __viaddmin_u16x2(__vminu2(X[k], X[k + 1]), p1x2, __vminu2(P[k], mp2));
    L[k] = __vadd2(cn[k], __vadd2(cand, ng));
  }
}

template <bool UP>
__global__ void __cluster_dims__(VC, 1, 1) __launch_bounds__(VWARPS * 32, 1) k_sgm_vd(SgmArgs a) {
  extern __shared__ __align__(16) uint32_t vsm[];
  const int W = a.W, H = a.H;
  if (a.select) {   // uniform over the cluster (one view)
    const double frac = (double)a.cells[blockIdx.y] / ((double)W * H * (a.d_max + 1));
    if ((a.select == 1) == (frac > a.split)) return;
  }
  const int k = blockIdx.x;   // rank in the cluster (grid.x == cluster size)
  int c0, nc;
  vd_range(W, k, c0, nc);
  const int NS = vd_maxcols(W) + 2;   // column slots: halo, owned columns, halo
  uint32_t* SA = vsm;                 // [NS][VNW]        column path (in place)
  uint32_t* SB = SA + NS * VNW;       // [2][NS][VNW]     predecessor x-1
  uint32_t* SC = SB + 2 * NS * VNW;   // [2][NS][VNW]     predecessor x+1
  uint32_t* MA = SC + 2 * NS * VNW;   // [NS][2]          (m + P2, -m) splats
  uint32_t* MB = MA + 2 * NS;         // [2][NS][2]
  uint32_t* MC = MB + 4 * NS;         // [2][NS][2]
  for (int i = threadIdx.x; i < NS * VSLOT; i += blockDim.x) vsm[i] = INF16x2;
  // halo slots: CTA k-1 writes this CTA's left halo (slot 0), CTA k+1 the
  // right one (slot nc + 1); off-image halos keep the +inf / no-m init
  cluster_sync_all();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gl = lane & (VG - 1), q = lane / VG;
  const size_t HW = (size_t)W * H;
  const uint2* __restrict__ meta = a.meta + (size_t)blockIdx.y * HW;
  const uint32_t* __restrict__ C = reinterpret_cast<const uint32_t*>(a.C) + (size_t)blockIdx.y * a.volcap;
  uint32_t* S = reinterpret_cast<uint32_t*>(a.S) + (size_t)blockIdx.y * a.volcap;
  const uint32_t p1x2 = a.p1i * 0x10001u;
  const int ngroups = nc / VNG;
  int ncl = 0, ncr = 0, tmp;
  if (k > 0) vd_range(W, k - 1, tmp, ncl);
  if (k + 1 < VC) vd_range(W, k + 1, tmp, ncr);
  (void)ncl;

  for (int t = 0; t < H; ++t) {
    const int y = UP ? H - 1 - t : t;
    const int nw = t & 1, ow = nw ^ 1;
    for (int g = warp; g < ngroups; g += VWARPS) {
      const int lc = g * VNG + q;
      const int x = c0 + lc;
      const int slot = lc + 1;
      // pixel metadata (grp4 encoding)
      uint2 mt = make_uint2(0xFFFFFFFFu, 0u);
      if (x < W) mt = meta[(size_t)y * W + x];
      int base = 0, relb = 0, clo = VNCH, chi = -1;
      uint32_t spanp = 0u;
      if (mt.x != 0xFFFFFFFFu) {
        const int j0 = (int)((mt.x & 0xFFFFu) >> 1), j1 = (int)((mt.x >> 16) >> 1);
        base = (int)(mt.y - (uint32_t)j0) + VPPL * gl;
        relb = VPPL * gl - j0 + VPPL - 1;
        spanp = (uint32_t)(j1 - j0 + VPPL);
        clo = j0 / VCW;
        chi = j1 / VCW;
      }
      const int ulo = __reduce_min_sync(FULL, clo), uhi = __reduce_max_sync(FULL, chi);
      // ---- load phase: every old word this group needs
      uint32_t PA[VNCH][VPPL], PB[VNCH][VPPL], PC[VNCH][VPPL];
      uint32_t eA[VNCH][2], eB[VNCH][2], eC[VNCH][2];
      uint32_t cn[VNCH][VPPL], sn[VNCH][VPPL];
      const uint32_t* a_col = SA + slot * VNW;
      const uint32_t* b_col = SB + (ow * NS + slot - 1) * VNW;
      const uint32_t* c_col = SC + (ow * NS + slot + 1) * VNW;
#pragma unroll
      for (int c = 0; c < VNCH; ++c) {
        if (c < ulo || c > uhi) continue;
        const int w0 = c * VCW + gl * VPPL;
        const bool p = (uint32_t)(relb + c * VCW) < spanp;
        {
          const uint32_t* src = p ? C + base + c * VCW : nullptr;
          uint32_t v0 = INF16x2, v1 = INF16x2, v2 = INF16x2, v3 = INF16x2;
          if (p) {
            asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "l"(src));
          }
          cn[c][0] = v0; cn[c][1] = v1; cn[c][2] = v2; cn[c][3] = v3;
          uint32_t s0 = 0, s1 = 0, s2 = 0, s3 = 0;
          if (p) {
            asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3) : "l"(S + base + c * VCW));
          }
          sn[c][0] = s0; sn[c][1] = s1; sn[c][2] = s2; sn[c][3] = s3;
        }
        const uint4 va = lds4(a_col + w0), vb = lds4(b_col + w0), vc = lds4(c_col + w0);
        PA[c][0] = va.x; PA[c][1] = va.y; PA[c][2] = va.z; PA[c][3] = va.w;
        PB[c][0] = vb.x; PB[c][1] = vb.y; PB[c][2] = vb.z; PB[c][3] = vb.w;
        PC[c][0] = vc.x; PC[c][1] = vc.y; PC[c][2] = vc.z; PC[c][3] = vc.w;
        const bool hasl = w0 > 0, hasr = w0 + VPPL < VNW;
        eA[c][0] = hasl ? a_col[w0 - 1] : INF16x2;
        eB[c][0] = hasl ? b_col[w0 - 1] : INF16x2;
        eC[c][0] = hasl ? c_col[w0 - 1] : INF16x2;
        eA[c][1] = hasr ? a_col[w0 + VPPL] : INF16x2;
        eB[c][1] = hasr ? b_col[w0 + VPPL] : INF16x2;
        eC[c][1] = hasr ? c_col[w0 + VPPL] : INF16x2;
      }
      const uint2 mA = *reinterpret_cast<const uint2*>(MA + 2 * slot);
      const uint2 mB = *reinterpret_cast<const uint2*>(MB + 2 * (ow * NS + slot - 1));
      const uint2 mC = *reinterpret_cast<const uint2*>(MC + 2 * (ow * NS + slot + 1));
      __syncwarp();
      // ---- compute and store phase
      uint32_t* a_out = SA + slot * VNW;
      uint32_t* b_out = SB + (nw * NS + slot) * VNW;
      uint32_t* c_out = SC + (nw * NS + slot) * VNW;
      uint32_t nA = INF16x2, nB = INF16x2, nC = INF16x2;
#pragma unroll
      for (int c = 0; c < VNCH; ++c) {
        const int w0 = c * VCW + gl * VPPL;
        if (c < ulo || c > uhi) {
          sts4(a_out + w0, INF16x2, INF16x2, INF16x2, INF16x2);
          sts4(b_out + w0, INF16x2, INF16x2, INF16x2, INF16x2);
          sts4(c_out + w0, INF16x2, INF16x2, INF16x2, INF16x2);
          continue;
        }
        uint32_t LA[VPPL], LB[VPPL], LC[VPPL], Ss[VPPL];
        vd_path(PA[c], eA[c][0], eA[c][1], mA.x, mA.y, p1x2, cn[c], LA);
        vd_path(PB[c], eB[c][0], eB[c][1], mB.x, mB.y, p1x2, cn[c], LB);
        vd_path(PC[c], eC[c][0], eC[c][1], mC.x, mC.y, p1x2, cn[c], LC);
#pragma unroll
        for (int i = 0; i < VPPL; ++i) Ss[i] = __vadd2(sn[c][i], __vadd2(LA[i], __vadd2(LB[i], LC[i])));
        const bool p = (uint32_t)(relb + c * VCW) < spanp;
        if (p) {
          asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};"
                       :: "l"(S + base + c * VCW), "r"(Ss[0]), "r"(Ss[1]), "r"(Ss[2]), "r"(Ss[3])
                       : "memory");
        }
        sts4(a_out + w0, LA[0], LA[1], LA[2], LA[3]);
        sts4(b_out + w0, LB[0], LB[1], LB[2], LB[3]);
        sts4(c_out + w0, LC[0], LC[1], LC[2], LC[3]);
        nA = __vimin3_u16x2(nA, __vminu2(LA[0], LA[1]), __vminu2(LA[2], LA[3]));
        nB = __vimin3_u16x2(nB, __vminu2(LB[0], LB[1]), __vminu2(LB[2], LB[3]));
        nC = __vimin3_u16x2(nC, __vminu2(LC[0], LC[1]), __vminu2(LC[2], LC[3]));
      }
      uint32_t hA = min(nA & 0xFFFFu, nA >> 16), hB = min(nB & 0xFFFFu, nB >> 16),
               hC = min(nC & 0xFFFFu, nC >> 16);
#pragma unroll
      for (int o = VG / 2; o; o >>= 1) {
        hA = min(hA, __shfl_xor_sync(FULL, hA, o));
        hB = min(hB, __shfl_xor_sync(FULL, hB, o));
        hC = min(hC, __shfl_xor_sync(FULL, hC, o));
      }
      const bool act = spanp != 0u;
      const uint32_t ma = act ? (hA + a.p2i) * 0x10001u : INF16x2;
      const uint32_t na = act ? ((0x10000u - hA) & 0xFFFFu) * 0x10001u : INF16x2;
      const uint32_t mb = act ? (hB + a.p2i) * 0x10001u : INF16x2;
      const uint32_t nb = act ? ((0x10000u - hB) & 0xFFFFu) * 0x10001u : INF16x2;
      const uint32_t mc = act ? (hC + a.p2i) * 0x10001u : INF16x2;
      const uint32_t ncv = act ? ((0x10000u - hC) & 0xFFFFu) * 0x10001u : INF16x2;
      if (gl == 0) {
        *reinterpret_cast<uint2*>(MA + 2 * slot) = make_uint2(ma, na);
        *reinterpret_cast<uint2*>(MB + 2 * (nw * NS + slot)) = make_uint2(mb, nb);
        *reinterpret_cast<uint2*>(MC + 2 * (nw * NS + slot)) = make_uint2(mc, ncv);
      }
      // halo pushes: the first owned column's x+1-predecessor state feeds
      // CTA k-1's right halo; the last owned column's x-1-predecessor state
      // feeds CTA k+1's left halo (same offsets in every CTA)
      if (lc == 0 && k > 0) {
        const int hs = ncl + 1;
#pragma unroll
        for (int c = 0; c < VNCH; ++c) {
          const int w0 = c * VCW + gl * VPPL;
          st_cluster4(SC + (nw * NS + hs) * VNW + w0, k - 1, lds4(c_out + w0));
        }
        if (gl == 0) st_cluster2(MC + 2 * (nw * NS + hs), k - 1, mc, ncv);
      }
      if (lc == nc - 1 && k + 1 < VC) {
#pragma unroll
        for (int c = 0; c < VNCH; ++c) {
          const int w0 = c * VCW + gl * VPPL;
          st_cluster4(SB + (nw * NS + 0) * VNW + w0, k + 1, lds4(b_out + w0));
        }
        if (gl == 0) st_cluster2(MB + 2 * (nw * NS + 0), k + 1, mb, nb);
      }
      __syncwarp();
    }
    cluster_sync_all();
  }
  (void)ncr;
}

}  // namespace

bool vd_supported(int W, int d_max) {
  static int ok = -1;
  if (npairs_max(d_max) > VNW || W < VC * VNG) return false;
  const size_t smem = vd_smem_bytes(W);
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (smem > (size_t)optin) return false;
  if (ok < 0) {
    ok = cudaFuncSetAttribute(k_sgm_vd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                 cudaSuccess &&
         cudaFuncSetAttribute(k_sgm_vd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
                 cudaSuccess;
  }
  return ok == 1;
}

void launch_vd(const SgmArgs& a, bool up, int n_sv, cudaStream_t st) {
  const size_t smem = vd_smem_bytes(a.W);
  auto k = up ? k_sgm_vd<true> : k_sgm_vd<false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<dim3(VC, n_sv), VWARPS * 32, smem, st>>>(a);
}

}  // namespace es
