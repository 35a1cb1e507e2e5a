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
// Work inside a CTA: a warp takes groups of 8 adjacent columns (4 lanes per
// column, 4 words per lane per 32-cell chunk); per group it loads every old
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
constexpr int VG = 4;                 // lanes per column
constexpr int VPPL = 4;               // words (u16 pairs) per lane per chunk
constexpr int VCW = VG * VPPL;        // words per chunk (32 cells)
constexpr int VNCH = 4;               // chunks per column: d_max <= 127
constexpr int VNW = VCW * VNCH;       // state words per column
constexpr int VNG = 32 / VG;          // columns per warp group
constexpr int VC = 9;                 // CTAs per cluster (one cluster per view; 9 x 1-CTA SMs pack 15 clusters = 135 SMs)
constexpr int VGPW = 2;               // column groups per warp (static, every row)
constexpr int VMAXW = 10;             // warps per CTA at most: 20 groups = 160 columns per CTA
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
// state slots plus four halo mbarriers (left / right x row parity)
inline size_t vd_smem_bytes(int W) {
  return sizeof(uint32_t) * (size_t)(vd_maxcols(W) + 2) * VSLOT + 32 + sizeof(int) * VMAXW;
}

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
// remote arrive (release at cluster scope) on the same mbarrier of CTA `rank`
__device__ __forceinline__ void mbar_arrive_remote(const uint64_t* local, int rank) {
  const unsigned la = (unsigned)__cvta_generic_to_shared(local);
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(ra) : "memory");
}
__device__ __forceinline__ void mbar_wait(const uint64_t* bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
}
// pause between polls of a neighbour's progress (frees issue slots for the
// warps that have work; 32 ns measured best of 0 / 32 / 200)
#ifndef ES_VD_SLEEP
#define ES_VD_SLEEP 32
#endif
__device__ __forceinline__ void vd_backoff() {
#if defined(ES_VD_SLEEP) && ES_VD_SLEEP > 0
  __nanosleep(ES_VD_SLEEP);
#endif
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

// operands of one (group, row) work item, loaded one item ahead
struct VdOps {
  uint2 mt;
  uint32_t cn[VNCH][VPPL];
  uint32_t sn[VNCH][VPPL];
};

template <bool UP, bool INIT>
__global__ void __cluster_dims__(VC, 1, 1) __launch_bounds__(VMAXW * 32, 1) k_sgm_vd(SgmArgs a) {
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
  uint32_t* SA = vsm;                 // [VNCH][NS][VCW]     column path (in place)
  uint32_t* SB = SA + NS * VNW;       // [2][VNCH][NS][VCW]  predecessor x-1
  uint32_t* SC = SB + 2 * NS * VNW;   // [2][VNCH][NS][VCW]  predecessor x+1
  uint32_t* MA = SC + 2 * NS * VNW;   // [NS][2]          (m + P2, -m) splats
  uint32_t* MB = MA + 2 * NS;         // [2][NS][2]
  uint32_t* MC = MB + 4 * NS;         // [2][NS][2]
  const int CS = NS * VCW;            // chunk stride of a state buffer (words)
  const int PS = VNCH * CS;           // parity stride of the B / C buffers
  uint64_t* hbar = reinterpret_cast<uint64_t*>(vsm + NS * VSLOT);   // [L0, L1, R0, R1]
  volatile int* done = reinterpret_cast<volatile int*>(hbar + 4);   // [warp]: rows completed
  for (int i = threadIdx.x; i < NS * VSLOT; i += blockDim.x) vsm[i] = INF16x2;
  if (threadIdx.x < VMAXW) done[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < 4; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
                   :: "r"((unsigned)__cvta_generic_to_shared(hbar + b)), "r"(VG) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // halo slots: CTA k-1 writes this CTA's left halo (slot 0), CTA k+1 the
  // right one (slot nc + 1), each followed by one arrive per writing lane on
  // this CTA's left / right mbarrier of that row's parity; off-image halos
  // keep the +inf / no-m init
  cluster_sync_all();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gl = lane & (VG - 1), q = lane / VG;
  const size_t HW = (size_t)W * H;
  const uint2* __restrict__ meta = a.meta + (size_t)blockIdx.y * HW;
  const uint32_t* __restrict__ C = reinterpret_cast<const uint32_t*>(a.C) + (size_t)blockIdx.y * a.volcap;
  uint32_t* S = reinterpret_cast<uint32_t*>(a.S) + (size_t)blockIdx.y * a.volcap;
  const uint32_t p1x2 = a.p1i * 0x10001u;
  const int ngroups = nc / VNG;
  // a warp owns VGPW consecutive column groups, the same in every row
  const int g_first = warp * VGPW;
  const int g_end = min(g_first + VGPW, ngroups);
  const int n_items = g_end > g_first ? g_end - g_first : 0;
  int ncl = 0, tmp;
  if (k > 0) vd_range(W, k - 1, tmp, ncl);

  // work items: (row t, group i) in sweep order; metadata is loaded two
  // items ahead, cost and partial-sum words one item ahead
  auto load_meta = [&](int item) -> uint2 {
    uint2 m = make_uint2(0xFFFFFFFFu, 0u);
    if (n_items == 0) return m;
    const int t = item / n_items, g = g_first + item % n_items;
    const int x = c0 + g * VNG + q;
    if (t < H && x < W) m = meta[(size_t)(UP ? H - 1 - t : t) * W + x];
    return m;
  };
  auto fetch = [&](uint2 mt, VdOps& o) {
    o.mt = mt;
    int base = 0, relb = 0;
    uint32_t spanp = 0u;
    if (mt.x != 0xFFFFFFFFu) {
      const int j0 = (int)((mt.x & 0xFFFFu) >> 1), j1 = (int)((mt.x >> 16) >> 1);
      base = (int)(mt.y - (uint32_t)j0) + VPPL * gl;
      relb = VPPL * gl - j0 + VPPL - 1;
      spanp = (uint32_t)(j1 - j0 + VPPL);
    }
#pragma unroll
    for (int c = 0; c < VNCH; ++c) {
      const bool p = (uint32_t)(relb + c * VCW) < spanp;
      uint32_t v0 = INF16x2, v1 = INF16x2, v2 = INF16x2, v3 = INF16x2;
      asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}\n"
                   : "+r"(v0), "+r"(v1), "+r"(v2), "+r"(v3) : "l"(C + base + c * VCW), "r"((int)p));
      o.cn[c][0] = v0; o.cn[c][1] = v1; o.cn[c][2] = v2; o.cn[c][3] = v3;
      uint32_t s0 = 0u, s1 = 0u, s2 = 0u, s3 = 0u;
      if constexpr (!INIT) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}\n"
                     : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3) : "l"(S + base + c * VCW), "r"((int)p));
      }
      o.sn[c][0] = s0; o.sn[c][1] = s1; o.sn[c][2] = s2; o.sn[c][3] = s3;
    }
  };

  VdOps cur, nxt;
  fetch(load_meta(0), cur);
  uint2 m1 = load_meta(1);
  const int total = n_items * H;
  int item = 0;
  const bool reads_left = g_first == 0 && n_items > 0 && k > 0;
  const bool reads_right = n_items > 0 && g_end == ngroups && k + 1 < VC;
  for (int t = 0; t < H; ++t) {
    const int nw = t & 1, ow = nw ^ 1;
    if (t > 0) {
      // the neighbouring warps' columns of row t-1 (this CTA): both have
      // finished row t-1, so its state is complete and they no longer read
      // the buffers row t overwrites
      if (lane == 0) {
        const int nwarps = blockDim.x >> 5;
        if (warp > 0) while (done[warp - 1] < t) vd_backoff();
        if (warp + 1 < nwarps) while (done[warp + 1] < t) vd_backoff();
        __threadfence_block();
      }
      __syncwarp();
      // the neighbouring CTAs' edge columns of row t-1 (a barrier per
      // parity: a neighbour is never two pushes ahead on the same one)
      const unsigned ph = (unsigned)(((t - 1) >> 1) & 1);
      if (reads_left) mbar_wait(hbar + ((t - 1) & 1), ph);
      if (reads_right) mbar_wait(hbar + 2 + ((t - 1) & 1), ph);
    }
    for (int i = 0; i < n_items; ++i, ++item) {
      const uint2 m2 = load_meta(item + 2);
      if (item + 1 < total) fetch(m1, nxt);   // next group, or the next row's first
      m1 = m2;
      const int g = g_first + i;
      const int lc = g * VNG + q;
      const int slot = lc + 1;
      const uint2 mt = cur.mt;
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
      // state layout [parity][chunk][slot][VCW words]: a warp's 8 columns of
      // one chunk are 512 contiguous bytes (conflict-free 16-byte accesses)
      const uint32_t* a_col = SA + slot * VCW;
      const uint32_t* b_col = SB + ow * PS + (slot - 1) * VCW;
      const uint32_t* c_col = SC + ow * PS + (slot + 1) * VCW;
      // d-1 / d+1 edge words of every chunk, before any in-place store
      uint32_t e[VNCH][6];
#pragma unroll
      for (int c = 0; c < VNCH; ++c) {
        const int w0 = gl * VPPL;
        // d-1 of the lane's first word: the previous lane's last word, or the
        // previous chunk's last word; d+1 of its last word likewise
        const int wl = gl > 0 ? c * CS + w0 - 1 : (c > 0 ? (c - 1) * CS + VCW - 1 : 0);
        const int wr = gl < VG - 1 ? c * CS + w0 + VPPL : (c + 1 < VNCH ? (c + 1) * CS : 0);
        e[c][0] = a_col[wl]; e[c][1] = a_col[wr];
        e[c][2] = b_col[wl]; e[c][3] = b_col[wr];
        e[c][4] = c_col[wl]; e[c][5] = c_col[wr];
        if (gl == 0 && c == 0) e[c][0] = e[c][2] = e[c][4] = INF16x2;
        if (gl == VG - 1 && c + 1 == VNCH) e[c][1] = e[c][3] = e[c][5] = INF16x2;
      }
      const uint2 mA = *reinterpret_cast<const uint2*>(MA + 2 * slot);
      const uint2 mB = *reinterpret_cast<const uint2*>(MB + 2 * (ow * NS + slot - 1));
      const uint2 mC = *reinterpret_cast<const uint2*>(MC + 2 * (ow * NS + slot + 1));
      __syncwarp();
      uint32_t* a_out = SA + slot * VCW;
      uint32_t* b_out = SB + nw * PS + slot * VCW;
      uint32_t* c_out = SC + nw * PS + slot * VCW;
      uint32_t nA = INF16x2, nB = INF16x2, nC = INF16x2;
#pragma unroll
      for (int c = 0; c < VNCH; ++c) {
        const int w0 = c * CS + gl * VPPL;
        if (c < ulo || c > uhi) {
          sts4(a_out + w0, INF16x2, INF16x2, INF16x2, INF16x2);
          sts4(b_out + w0, INF16x2, INF16x2, INF16x2, INF16x2);
          sts4(c_out + w0, INF16x2, INF16x2, INF16x2, INF16x2);
          continue;
        }
        uint32_t P[VPPL], LA[VPPL], LB[VPPL], LC[VPPL], Ss[VPPL];
        uint4 v = lds4(a_col + w0);
        P[0] = v.x; P[1] = v.y; P[2] = v.z; P[3] = v.w;
        vd_path(P, e[c][0], e[c][1], mA.x, mA.y, p1x2, cur.cn[c], LA);
        v = lds4(b_col + w0);
        P[0] = v.x; P[1] = v.y; P[2] = v.z; P[3] = v.w;
        vd_path(P, e[c][2], e[c][3], mB.x, mB.y, p1x2, cur.cn[c], LB);
        v = lds4(c_col + w0);
        P[0] = v.x; P[1] = v.y; P[2] = v.z; P[3] = v.w;
        vd_path(P, e[c][4], e[c][5], mC.x, mC.y, p1x2, cur.cn[c], LC);
#pragma unroll
        for (int r = 0; r < VPPL; ++r) {
          Ss[r] = __vadd2(LA[r], __vadd2(LB[r], LC[r]));
          if constexpr (!INIT) Ss[r] = __vadd2(cur.sn[c][r], Ss[r]);
        }
        const bool p = (uint32_t)(relb + c * VCW) < spanp;
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.v4.u32 [%0], {%1, %2, %3, %4};\n\t}\n"
                     :: "l"(S + base + c * VCW), "r"(Ss[0]), "r"(Ss[1]), "r"(Ss[2]), "r"(Ss[3]), "r"((int)p)
                     : "memory");
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
          const int w0 = c * CS + gl * VPPL;
          st_cluster4(SC + nw * PS + hs * VCW + w0, k - 1, lds4(c_out + w0));
        }
        if (gl == 0) st_cluster2(MC + 2 * (nw * NS + hs), k - 1, mc, ncv);
        mbar_arrive_remote(hbar + 2 + nw, k - 1);   // CTA k-1's right mbarrier
      }
      if (lc == nc - 1 && k + 1 < VC) {
#pragma unroll
        for (int c = 0; c < VNCH; ++c) {
          const int w0 = c * CS + gl * VPPL;
          st_cluster4(SB + nw * PS + w0, k + 1, lds4(b_out + w0));
        }
        if (gl == 0) st_cluster2(MB + 2 * (nw * NS + 0), k + 1, mb, nb);
        mbar_arrive_remote(hbar + nw, k + 1);       // CTA k+1's left mbarrier
      }
      __syncwarp();
      cur = nxt;
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      done[warp] = t + 1;
    }
  }
  cluster_sync_all();   // no CTA leaves while a neighbour may still push into it
}

}  // namespace

bool vd_supported(int W, int d_max) {
  if (npairs_max(d_max) > VNW || W < VC * VNG) return false;
  if (vd_maxcols(W) / VNG > VMAXW * VGPW) return false;
  const size_t smem = vd_smem_bytes(W);
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return false;
  if (smem > (size_t)optin) return false;
  // per (kernel, device) and checked (es_api.cu ensure_*)
  for (auto k : {k_sgm_vd<false, false>, k_sgm_vd<true, false>, k_sgm_vd<false, true>,
                 k_sgm_vd<true, true>})
    if (!ensure_attr((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ||
        !ensure_smem((const void*)k, smem))
      return false;
  return true;
}

void launch_vd(const SgmArgs& a, bool up, bool init, int n_sv, cudaStream_t st) {
  const size_t smem = vd_smem_bytes(a.W);
  auto k = up ? (init ? k_sgm_vd<true, true> : k_sgm_vd<true, false>)
              : (init ? k_sgm_vd<false, true> : k_sgm_vd<false, false>);
  // attributes were set by vd_supported (the caller's precondition)
  const int nwarps = (vd_maxcols(a.W) / VNG + VGPW - 1) / VGPW;
  k<<<dim3(VC, n_sv), nwarps * 32, smem, st>>>(a);
}

}  // namespace es
