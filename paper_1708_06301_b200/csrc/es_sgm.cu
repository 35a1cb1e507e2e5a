// K4 + K5: 8-path SGM aggregation over the ragged cost volume, then
// winner-take-all and the matching-variance walk.
//
// Reference: sgm.py:199-272 (_path_step, _scan_vertical, _scan_horizontal,
// aggregate_paths), sgm.py:275-344 (select_disparity, matching_variance_map).
//
// Paths are independent chains of pixels: rows (H), columns (V), x-y = const
// (D1) and x+y = const (D2).  Kernels, in production order:
//   k_sgm_grp4  (u16, production): a warp walks 32/G chains in lockstep, G
//               lanes per chain, every lane owning one aligned 16-byte word
//               (8 cells) of each absolute chunk; see its own comment and
//               DESIGN.md section 4.  Launched as six jobs per step over two
//               (or four) partial sums by launch_aggregate_parts.
//   k_sgm_vd    (u16, opt-in ES_SGM_VD=1 / 2, es_sgm_vd.cu): the three
//               directions of one row sweep over columns and diagonals in one
//               thread-block cluster per view; parity-green, not yet faster
//               than the grp4 jobs (profiles/r01/SUMMARY_vd.md).
//   k_sgm_grp3  (u16): the previous production kernel, A/B baseline
//               (ES_SGM_G4=0).
//   k_sgm       (u16 / f32): one warp per chain, lane l holding pair
//               c*32 + l of chunk c; the f32 path (non-integer penalties or
//               arbitrary user volumes) and the per-direction launches in
//               the reference's summation order use it.
// Then k_wta_runs (u16 sums) / k_wta_var (f32 or caller winners) select the
// disparity and walk the matching variance.
//
// Arithmetic policies:
//   U16 (default integer penalties, small windows): two cells per 32-bit word,
//     VIMNMX.U16x2 / VIADDMNMX.U16x2 / VIADD.16x2.  "+inf" is 0x8000; sums
//     are exact because every finite value is <= window^2*255 + P2 and the
//     8-path sum stays < 2^16 (host-checked), while out-of-interval values
//     stay in [0x8000, 0x8000 + P2] and are never selected.
//   F32 (any other penalties / volumes): float2 per lane, numpy's float32
//     operation order, 8 single-direction launches in the reference's
//     summation order (H->, H<-, dy=+1 dx=-1,0,1, dy=-1 dx=-1,0,1).
#include <cstdlib>
#include <type_traits>

#include "es_common.cuh"
#include "es_kernels.h"

namespace es {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SGM_WARPS = 4;

// ------------------------------------------------------------ policies

struct U16A {
  using P = uint32_t;
  __device__ static __forceinline__ P inf() { return INF16x2; }
  __device__ static __forceinline__ P load_cost(const void* C, size_t k) {
    return __ldg(reinterpret_cast<const uint32_t*>(C) + k);
  }
  __device__ static __forceinline__ P step(P cv, P pv, P pl, P pr, const SgmArgs& a, P mP2,
                                           P negm) {
    const P left = __byte_perm(pl, pv, 0x5432);
    const P right = __byte_perm(pv, pr, 0x5432);
    const P nb = __vminu2(left, right);
    const P p1 = a.p1i | (a.p1i << 16);
    const P cand = __vminu2(__viaddmin_u16x2(nb, p1, pv), mP2);
    return __vadd2(cv, __vadd2(cand, negm));
  }
  __device__ static __forceinline__ P vmin(P a, P b) { return __vminu2(a, b); }
  __device__ static __forceinline__ uint32_t warp_min(P v) {
    return __reduce_min_sync(FULL, min(v & 0xFFFFu, v >> 16));
  }
  __device__ static __forceinline__ P splat_m_p2(uint32_t m, const SgmArgs& a) {
    const uint32_t s = m + a.p2i;
    return s | (s << 16);
  }
  __device__ static __forceinline__ P negm(uint32_t m) {
    const uint32_t n = (0x10000u - m) & 0xFFFFu;
    return n | (n << 16);
  }
  __device__ static __forceinline__ void store_sum(void* S, size_t k, P L, bool init) {
    uint32_t* s = reinterpret_cast<uint32_t*>(S) + k;
    *s = init ? L : __vadd2(*s, L);
  }
};

struct F32A {
  using P = float2;
  __device__ static __forceinline__ P inf() { return make_float2(INFINITY, INFINITY); }
  __device__ static __forceinline__ P load_cost_u16(const void* C, size_t k) {
    const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(C) + k);
    const uint32_t a = w & 0xFFFFu, b = w >> 16;
    return make_float2(a >= INF16 ? INFINITY : (float)a, b >= INF16 ? INFINITY : (float)b);
  }
  __device__ static __forceinline__ P step(P cv, P pv, P pl, P pr, const SgmArgs& a, P mP2,
                                           P m) {
    // numpy order (sgm.py:205-209): cand = min(prev, m+p2), then the two
    // neighbour terms prev[d-1]+p1, prev[d+1]+p1; out = cost + (cand - m)
    const float l0 = pl.y, l1 = pv.x;   // prev[d-1] for the two cells
    const float r0 = pv.y, r1 = pr.x;   // prev[d+1]
    float c0 = fminf(pv.x, mP2.x), c1 = fminf(pv.y, mP2.y);
    c0 = fminf(c0, __fadd_rn(l0, a.p1));
    c1 = fminf(c1, __fadd_rn(l1, a.p1));
    c0 = fminf(c0, __fadd_rn(r0, a.p1));
    c1 = fminf(c1, __fadd_rn(r1, a.p1));
    return make_float2(__fadd_rn(cv.x, __fsub_rn(c0, m.x)), __fadd_rn(cv.y, __fsub_rn(c1, m.y)));
  }
  __device__ static __forceinline__ P vmin(P a, P b) {
    return make_float2(fminf(a.x, b.x), fminf(a.y, b.y));
  }
  __device__ static __forceinline__ float warp_min(P v) {
    float x = fminf(v.x, v.y);
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fminf(x, __shfl_xor_sync(FULL, x, o));
    return x;
  }
  __device__ static __forceinline__ P splat_m_p2(float m, const SgmArgs& a) {
    const float s = __fadd_rn(m, a.p2);
    return make_float2(s, s);
  }
  __device__ static __forceinline__ P negm(float m) { return make_float2(m, m); }
  __device__ static __forceinline__ void store_sum(void* S, size_t k, P L, bool init) {
    float2* s = reinterpret_cast<float2*>(S) + k;
    if (init) {
      *s = L;
    } else {
      float2 o = *s;
      *s = make_float2(__fadd_rn(o.x, L.x), __fadd_rn(o.y, L.y));
    }
  }
};

__device__ __forceinline__ uint32_t shfl_u(uint32_t v, int src) { return __shfl_sync(FULL, v, src); }
__device__ __forceinline__ float2 shfl_u(float2 v, int src) {
  return make_float2(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src));
}

// chain geometry: start pixel, step, length for (family, sweep, chain)
__device__ __forceinline__ void chain_geom(int fam, int bwd, int c, int W, int H, int& x0, int& y0,
                                           int& sx, int& sy, int& len) {
  if (fam == FAM_H) {
    sy = 0;
    y0 = c;
    len = W;
    sx = bwd ? -1 : 1;
    x0 = bwd ? W - 1 : 0;
  } else if (fam == FAM_V) {
    sx = 0;
    x0 = c;
    len = H;
    sy = bwd ? -1 : 1;
    y0 = bwd ? H - 1 : 0;
  } else {
    int ya, yb;   // y range of the diagonal
    if (fam == FAM_D1) {   // x - y = u
      const int u = c - (H - 1);
      ya = max(0, -u);
      yb = min(H - 1, W - 1 - u);
      len = yb - ya + 1;
      y0 = bwd ? yb : ya;
      x0 = u + y0;
      sy = bwd ? -1 : 1;
      sx = sy;
    } else {               // x + y = s
      const int s = c;
      ya = max(0, s - (W - 1));
      yb = min(H - 1, s);
      len = yb - ya + 1;
      y0 = bwd ? yb : ya;
      x0 = s - y0;
      sy = bwd ? -1 : 1;
      sx = -sy;
    }
  }
}

template <class A, int NCH, bool COST_F32>
__global__ void __launch_bounds__(SGM_WARPS * 32) k_sgm(SgmArgs a, int fam, int sweeps, int init) {
  using P = typename A::P;
  const int lane = threadIdx.x & 31;
  const int chain = blockIdx.x * SGM_WARPS + (threadIdx.x >> 5);
  const int W = a.W, H = a.H;
  const int nchains = fam == FAM_H ? H : (fam == FAM_V ? W : W + H - 1);
  if (chain >= nchains) return;
  const size_t HW = (size_t)W * H;
  const uint2* meta = a.meta + (size_t)blockIdx.y * HW;
  const size_t vbase = (size_t)blockIdx.y * a.volcap;
  bool first_sweep = true;
  for (int bwd = 0; bwd < 2; ++bwd) {
    if (!(sweeps & (1 << bwd))) continue;
    const bool init_sum = init && first_sweep;
    first_sweep = false;
    int x, y, sx, sy, len;
    chain_geom(fam, bwd, chain, W, H, x, y, sx, sy, len);
    P prev[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) prev[c] = A::inf();
    decltype(A::warp_min(A::inf())) m = 0;
    for (int t = 0; t < len; ++t, x += sx, y += sy) {
      const uint2 mt = meta[(size_t)y * W + x];
      const int j0 = (int)(lo_of(mt) >> 1), j1 = (int)(hi_of(mt) >> 1);
      const int clo = j0 >> 5, chi = j1 >> 5;
      const P mP2 = A::splat_m_p2(m, a);
      const P ng = A::negm(m);
      P cur[NCH];
      P nmin = A::inf();
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (c < clo || c > chi) {
          cur[c] = A::inf();
          continue;
        }
        const int j = c * 32 + lane;
        const bool in = j >= j0 && j <= j1;
        const size_t k = vbase + mt.y + (size_t)(j - j0);
        P cv = A::inf();
        if (in) {
          if constexpr (COST_F32) {
            cv = __ldg(reinterpret_cast<const float2*>(a.C) + k);
          } else if constexpr (sizeof(P) == 4) {
            cv = A::load_cost(a.C, k);
          } else {
            cv = F32A::load_cost_u16(a.C, k);
          }
        }
        P L;
        if (t == 0) {
          L = cv;
        } else {
          const P srcl = lane == 31 ? (c > 0 ? prev[c > 0 ? c - 1 : 0] : A::inf()) : prev[c];
          const P pl = shfl_u(srcl, (lane + 31) & 31);
          const P srcr = lane == 0 ? (c + 1 < NCH ? prev[c + 1 < NCH ? c + 1 : c] : A::inf()) : prev[c];
          const P pr = shfl_u(srcr, (lane + 1) & 31);
          L = A::step(cv, prev[c], pl, pr, a, mP2, ng);
        }
        cur[c] = L;
        nmin = A::vmin(nmin, L);
        if (in) A::store_sum(a.S, k, L, init_sum);
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c) prev[c] = cur[c];
      m = A::warp_min(nmin);
    }
  }
}

// ------------------------------------------------------------ grouped (u16)
//
// The production u16 kernel.  A warp walks NG = 32/G chains in lockstep, G
// lanes per chain; lane g of a chain's group holds pair c*G + g of chunk c
// (2G cells per chunk, absolute disparity).  Per step the warp loops only
// over the union of its chains' chunk ranges, so reduced intervals cost one
// or two chunks.  Chain metadata is loaded G steps at a time (one load per
// lane) and broadcast with a shuffle; the next step's cost and partial sums
// are loaded into registers while the current step computes, so the
// recurrence's critical path has no global-memory latency.  Diagonal chains
// are walked row by row (inactive on rows where they leave the image).

constexpr int GRP_WARPS = 4;

__device__ __forceinline__ bool grp_pixel(int fam, int bwd, int c, int t, int W, int H, int& x,
                                          int& y) {
  if (fam == FAM_H) {
    y = c;
    x = bwd ? W - 1 - t : t;
    return c < H;
  }
  y = bwd ? H - 1 - t : t;
  if (fam == FAM_V) {
    x = c;
    return c < W;
  }
  x = fam == FAM_D1 ? c - (H - 1) + y : c - y;
  return x >= 0 && x < W && c < W + H - 1;
}

// per-step scalars of one chain for k_sgm_grp3
struct GrpStep {          // per-step scalars of one chain (uniform in its group)
  uint32_t my;            // pair offset of the pixel
  int j0;                 // first pair
  uint32_t span;          // number of pairs (0: no pixel)
  uint32_t um;            // warp-uniform chunk mask (union over the warp's chains)
};

// ------------------------------------------------------------ grouped, 2 pairs/lane
//
// The round's previous production kernel, kept as the A/B baseline of
// k_sgm_grp4 (ES_SGM_G4=0): operands fetched two steps ahead into two
// alternating register sets, metadata batches broadcast by shuffle, and every
// lane owns two
// consecutive pairs (4 cells): lane g of chunk c holds pairs
// c*2G + 2g and c*2G + 2g + 1.  The shuffles, selects, chunk-mask tests and
// address arithmetic are shared by four cells, and the byte permute that
// forms "right neighbours of the first pair" is also "left neighbours of the
// second pair".

// global-space accesses with predication in PTX: no generic addressing and
// no divergent branch around the conditional stores
__device__ __forceinline__ uint32_t ld_pred(const uint32_t* p, bool pred, uint32_t dflt) {
  uint32_t v = dflt;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.u32 %0, [%1];\n\t}\n"
      : "+r"(v)
      : "l"(p), "r"((int)pred));
  return v;
}
__device__ __forceinline__ uint32_t ldc_pred(const uint32_t* p, bool pred, uint32_t dflt) {
  uint32_t v = dflt;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}\n"
      : "+r"(v)
      : "l"(p), "r"((int)pred));
  return v;
}
// 8-byte variants: a lane's two pairs are one aligned word of its pixel's
// allocation (see pixel_slots), so one access serves both
__device__ __forceinline__ uint2 ld2_pred(const uint32_t* p, bool pred) {
  uint32_t a = 0u, b = 0u;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.global.v2.u32 {%0, %1}, [%2];\n\t}\n"
      : "+r"(a), "+r"(b)
      : "l"(p), "r"((int)pred));
  return make_uint2(a, b);
}
__device__ __forceinline__ uint2 ldc2_pred(const uint32_t* p, bool pred) {
  uint32_t a = INF16x2, b = INF16x2;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.global.nc.v2.u32 {%0, %1}, [%2];\n\t}\n"
      : "+r"(a), "+r"(b)
      : "l"(p), "r"((int)pred));
  return make_uint2(a, b);
}
__device__ __forceinline__ void st2_pred(uint32_t* p, uint32_t a, uint32_t b, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.u32 [%0], {%1, %2};\n\t}\n" ::"l"(p),
      "r"(a), "r"(b), "r"((int)pred)
      : "memory");
}

__device__ __forceinline__ void st_pred(uint32_t* p, uint32_t v, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.u32 [%0], %1;\n\t}\n" ::"l"(p),
               "r"(v), "r"((int)pred)
               : "memory");
}

template <int G, int NCH>
// measured: capping the 4-lane instance at 128 registers (4 blocks/SM) wins
// more from occupancy than it loses to one spilled word; the 8-lane instance
// is fastest uncapped
__global__ void __launch_bounds__(GRP_WARPS * 32, (G == 4 ? 4 : 1)) k_sgm_grp3(SgmArgs a, int fam, int sweeps,
                                                              int init) {
  constexpr int NG = 32 / G;
  constexpr int CW = 2 * G;   // pairs per chunk
  constexpr uint32_t NONE = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int gbase = lane & ~(G - 1);
  const int W = a.W, H = a.H;
  const int nchains = fam == FAM_H ? H : (fam == FAM_V ? W : W + H - 1);
  const int c0 = (blockIdx.x * GRP_WARPS + (threadIdx.x >> 5)) * NG;
  if (c0 >= nchains) return;
  if (a.select) {
    const double frac = (double)a.cells[blockIdx.y] / ((double)W * H * (a.d_max + 1));
    if ((a.select == 1) == (frac > a.split)) return;
  }
  const int ch = c0 + grp;
  const size_t HW = (size_t)W * H;
  const uint2* __restrict__ meta = a.meta + (size_t)blockIdx.y * HW;
  const uint32_t* __restrict__ C =
      reinterpret_cast<const uint32_t*>(a.C) + (size_t)blockIdx.y * a.volcap;
  uint32_t* S = reinterpret_cast<uint32_t*>(a.S) + (size_t)blockIdx.y * a.volcap;
  // keep the per-view bases in registers: one IMAD.WIDE per access instead of
  // re-deriving blockIdx.y * volcap under register pressure
#ifndef ES_GRP3_NOPIN
  asm volatile("" : "+l"(C));
  asm volatile("" : "+l"(S));
#endif
  const uint32_t p1x2 = a.p1i * 0x10001u;
  const uint32_t p2 = a.p2i;
  const int len = fam == FAM_H ? W : H;
  const int src_l = gbase | ((gl + G - 1) & (G - 1));
  const int src_r = gbase | ((gl + 1) & (G - 1));
  auto umask = [](int lo, int hi) -> uint32_t {
    return hi < lo ? 0u : ((hi >= 31 ? 0xFFFFFFFFu : ((2u << hi) - 1u)) & ~((1u << lo) - 1u));
  };
  bool first_sweep = true;
  for (int bwd = 0; bwd < 2; ++bwd) {
    if (!(sweeps & (1 << bwd))) continue;
    const bool init_sum = init && first_sweep;
    first_sweep = false;
    auto load_meta = [&](int tb) -> uint2 {
      int x, y;
      const int t = tb + gl;
      if (t < len && grp_pixel(fam, bwd, ch, t, W, H, x, y)) return meta[(size_t)y * W + x];
      return make_uint2(NONE, 0u);
    };
    // three meta batches in flight: a batch is loaded 2G steps before use
    uint2 mb_cur = load_meta(0);
    uint2 mb_next = load_meta(G);
    uint2 mb_next2 = load_meta(2 * G);
    int tb = 0;
    auto info = [&](int tp) -> GrpStep {
      GrpStep s{0u, 0, 0u, 0u};
      int clo = NCH, chi = -1;
      if (tp < len) {
        if (tp == tb + G) {
          tb += G;
          mb_cur = mb_next;
          mb_next = mb_next2;
          mb_next2 = load_meta(tb + 2 * G);
        }
        const int r = tp - tb;
        const uint32_t mx = __shfl_sync(FULL, mb_cur.x, gbase | r);
        s.my = __shfl_sync(FULL, mb_cur.y, gbase | r);
        if (mx != NONE) {
          s.j0 = (int)((mx & 0xFFFFu) >> 1);
          const int j1 = (int)((mx >> 16) >> 1);
          s.span = (uint32_t)(j1 - s.j0 + 1);
          clo = s.j0 / CW;
          chi = j1 / CW;
        }
      }
      s.um = umask(__reduce_min_sync(FULL, clo), __reduce_max_sync(FULL, chi));
      return s;
    };
    // operands of chunk c for one step: two pairs per lane
    auto fetch = [&](const GrpStep& s, uint32_t (&cn)[2 * NCH], uint32_t (&sn)[2 * NCH], int c) {
      const uint32_t rel = (uint32_t)(c * CW + 2 * gl - s.j0);
      const bool in0 = rel < s.span, in1 = rel + 1 < s.span;
      // offsets wrap in 32 bits (rel = -1: first pair just below the
      // interval); k0 is even, so both pairs are one aligned 8-byte word
      const uint32_t k0 = s.my + rel;
#ifndef ES_GRP3_SCALAR
      // raw words: the out-of-interval half is masked where it is used, so
      // nothing here waits for the load
      const bool any = in0 || in1;
      const uint2 cv = ldc2_pred(C + k0, any);
      cn[2 * c] = cv.x;
      cn[2 * c + 1] = cv.y;
      const uint2 sv = ld2_pred(S + k0, any && !init_sum);
      sn[2 * c] = sv.x;
      sn[2 * c + 1] = sv.y;
#else
      cn[2 * c] = ldc_pred(C + k0, in0, INF16x2);
      cn[2 * c + 1] = ldc_pred(C + (uint32_t)(k0 + 1u), in1, INF16x2);
      sn[2 * c] = ld_pred(S + k0, in0 && !init_sum, 0u);
      sn[2 * c + 1] = ld_pred(S + (uint32_t)(k0 + 1u), in1 && !init_sum, 0u);
#endif
    };
    uint32_t prev[2 * NCH], cA[2 * NCH], sA[2 * NCH], cB[2 * NCH], sB[2 * NCH];
    GrpStep s0 = info(0);
    GrpStep s1 = info(1);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      prev[2 * c] = INF16x2;
      prev[2 * c + 1] = INF16x2;
      fetch(s0, cA, sA, c);
      fetch(s1, cB, sB, c);
    }
    uint32_t m = 0;
    bool was_active = false;
    auto step = [&](const GrpStep& cur, const GrpStep& nn, uint32_t (&cn)[2 * NCH],
                    uint32_t (&sn)[2 * NCH]) {
      const bool act = cur.span != 0;
      const bool first = act && !was_active;
      const uint32_t mp2 = (m + p2) * 0x10001u;
      const uint32_t ng = ((0x10000u - m) & 0xFFFFu) * 0x10001u;
      uint32_t nmin = INF16x2;
      uint32_t left_old = INF16x2;   // previous chunk's second pair, before overwrite
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint32_t pa = prev[2 * c], pb = prev[2 * c + 1];
        if ((cur.um >> c) & 1u) {
          // left neighbour of pair a: the previous lane's pair b (or the
          // previous chunk's last one); right neighbour of pair b: the next
          // lane's pair a (or the next chunk's first one)
          const uint32_t srcl = gl == G - 1 ? left_old : pb;
          const uint32_t srcr =
              gl == 0 ? (c + 1 < NCH ? prev[c + 1 < NCH ? 2 * c + 2 : 0] : INF16x2) : pa;
          const uint32_t pl = __shfl_sync(FULL, srcl, src_l);
          const uint32_t pr = __shfl_sync(FULL, srcr, src_r);
          const uint32_t mid = __byte_perm(pa, pb, 0x5432);
          const uint32_t nba = __vminu2(__byte_perm(pl, pa, 0x5432), mid);
          const uint32_t nbb = __vminu2(mid, __byte_perm(pb, pr, 0x5432));
          const uint32_t ca = __vminu2(__viaddmin_u16x2(nba, p1x2, pa), mp2);
          const uint32_t cb = __vminu2(__viaddmin_u16x2(nbb, p1x2, pb), mp2);
          const uint32_t rel = (uint32_t)(c * CW + 2 * gl - cur.j0);
#ifndef ES_GRP3_SCALAR
          // no mask: the out-of-interval pair of a word is the pixel's own
          // padding slot, which the cost pass fills with +inf (es_common.cuh)
#ifdef ES_GRP3_MASK
          const uint32_t cwa = rel < cur.span ? cn[2 * c] : INF16x2;
          const uint32_t cwb = rel + 1 < cur.span ? cn[2 * c + 1] : INF16x2;
#else
          const uint32_t cwa = cn[2 * c], cwb = cn[2 * c + 1];
#endif
#else
          const uint32_t cwa = cn[2 * c], cwb = cn[2 * c + 1];
#endif
          const uint32_t La = first ? cwa : __vadd2(cwa, __vadd2(ca, ng));
          const uint32_t Lb = first ? cwb : __vadd2(cwb, __vadd2(cb, ng));
          prev[2 * c] = La;
          prev[2 * c + 1] = Lb;
          nmin = __vminu2(nmin, __vminu2(La, Lb));
          // one 8-byte store; a half outside the interval lands in the
          // pixel's own padding / out-of-interval slot, which nothing reads
#ifndef ES_GRP3_SCALAR
          st2_pred(S + (uint32_t)(cur.my + rel), init_sum ? La : __vadd2(sn[2 * c], La),
                   init_sum ? Lb : __vadd2(sn[2 * c + 1], Lb),
                   rel < cur.span || rel + 1 < cur.span);
#else
          st_pred(S + (uint32_t)(cur.my + rel), init_sum ? La : __vadd2(sn[2 * c], La),
                  rel < cur.span);
          st_pred(S + (uint32_t)(cur.my + rel + 1u), init_sum ? Lb : __vadd2(sn[2 * c + 1], Lb),
                  rel + 1 < cur.span);
#endif
        } else {
          prev[2 * c] = INF16x2;
          prev[2 * c + 1] = INF16x2;
        }
        left_old = pb;
        if ((nn.um >> c) & 1u) fetch(nn, cn, sn, c);
      }
      // per-chain minimum: xor butterfly inside each G-lane group
      uint32_t hm = min(nmin & 0xFFFFu, nmin >> 16);
#pragma unroll
      for (int o = G / 2; o; o >>= 1) hm = min(hm, __shfl_xor_sync(FULL, hm, o));
      m = hm;
      was_active = act;
    };
    for (int t = 0; t < len; t += 2) {
      const GrpStep s2 = info(t + 2);
      step(s0, s2, cA, sA);
      if (t + 1 >= len) break;
      const GrpStep s3 = info(t + 3);
      step(s1, s3, cB, sB);
      s0 = s2;
      s1 = s3;
    }
  }
}

template <int G>
static void launch_grp3(const SgmArgs& a, int nch_pairs, int fam, int sweeps, int init, int n_sv,
                        cudaStream_t st) {
  const int nchains = fam == FAM_H ? a.H : (fam == FAM_V ? a.W : a.W + a.H - 1);
  constexpr int per_block = GRP_WARPS * (32 / G);
  dim3 grid((nchains + per_block - 1) / per_block, n_sv);
  const int nch = (nch_pairs + 2 * G - 1) / (2 * G);
  auto go = [&](auto kern) { kern<<<grid, GRP_WARPS * 32, 0, st>>>(a, fam, sweeps, init); };
  if (nch <= 2) go(k_sgm_grp3<G, 2>);
  else if (nch <= 4) go(k_sgm_grp3<G, 4>);
  else if (nch <= 8) go(k_sgm_grp3<G, 8>);
  else go(k_sgm_grp3<G, 16>);
}

// ------------------------------------------------------------ grouped, PPL pairs/lane
//
// The production u16 kernel.  As k_sgm_grp3 (a warp walks 32/G chains in
// lockstep, G lanes per chain, absolute chunks, union-of-chunks loop, operands
// fetched two steps ahead into alternating register sets) with the per-chunk
// overhead cut down:
//  * every lane owns PPL consecutive pairs (2*PPL cells) of a chunk, one
//    aligned 8- or 16-byte word of the pixel's allocation (pixel_slots keeps
//    (offset - j0) a multiple of 4), so one load / store serves them all;
//  * per step each lane forms one signed base offset; chunk c's operands are
//    at base + c*CW, an immediate offset, and one compare gives the chunk's
//    predicate;
//  * no select for a chain's first pixel: a chain that is inactive holds
//    +inf-ish values (>= 0x8000) and mp2 = ng = 0x8000, so its first active
//    pixel computes min(...) = 0x8000 and L = C + 0x8000 + 0x8000 = C;
//  * no select for the first family's forward sweep: the predicated partial
//    sum load leaves 0.
constexpr int G4_WARPS = 4;
#ifndef G4_PF_WORDS
#define G4_PF_WORDS 128   // k_sgm_row: row-stream L2 prefetch distance in 32-bit words (0: off)
#endif

struct G4Step {
  int base;         // pair offset (this view) of the lane's pairs in chunk 0
  int relb;         // PPL*gl - j0 + PPL - 1: chunk c has a pair in [j0, j1] iff
  uint32_t spanp;   //   (unsigned)(relb + c*CW) < spanp = span + PPL - 1
  uint32_t um;      // warp-uniform chunk mask (union over the warp's chains)
};

template <int PPL>
struct Vec;
template <>
struct Vec<2> {
  __device__ static __forceinline__ void ld_any(const uint32_t* p, bool pred, uint32_t* o) {
    uint32_t a, b;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.global.v2.u32 {%0, %1}, [%2];\n\t}\n"
                 : "=r"(a), "=r"(b) : "l"(p), "r"((int)pred));
    o[0] = a; o[1] = b;
  }
  __device__ static __forceinline__ void ldc(const uint32_t* p, bool pred, uint32_t* o) {
    uint32_t a = INF16x2, b = INF16x2;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.global.nc.v2.u32 {%0, %1}, [%2];\n\t}\n"
                 : "+r"(a), "+r"(b) : "l"(p), "r"((int)pred));
    o[0] = a; o[1] = b;
  }
  __device__ static __forceinline__ void ld(const uint32_t* p, bool pred, uint32_t* o) {
    uint32_t a = 0u, b = 0u;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.global.v2.u32 {%0, %1}, [%2];\n\t}\n"
                 : "+r"(a), "+r"(b) : "l"(p), "r"((int)pred));
    o[0] = a; o[1] = b;
  }
  __device__ static __forceinline__ void st(uint32_t* p, bool pred, const uint32_t* v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.u32 [%0], {%1, %2};\n\t}\n"
                 :: "l"(p), "r"(v[0]), "r"(v[1]), "r"((int)pred) : "memory");
  }
};
template <>
struct Vec<4> {
  // predicated load that leaves the registers undefined when off (callers
  // only use them under the same predicate)
  __device__ static __forceinline__ void ld_any(const uint32_t* p, bool pred, uint32_t* o) {
    uint32_t a, b, c, d;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}\n"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p), "r"((int)pred));
    o[0] = a; o[1] = b; o[2] = c; o[3] = d;
  }
  __device__ static __forceinline__ void ldc(const uint32_t* p, bool pred, uint32_t* o) {
    uint32_t a = INF16x2, b = INF16x2, c = INF16x2, d = INF16x2;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}\n"
                 : "+r"(a), "+r"(b), "+r"(c), "+r"(d) : "l"(p), "r"((int)pred));
    o[0] = a; o[1] = b; o[2] = c; o[3] = d;
  }
  __device__ static __forceinline__ void ld(const uint32_t* p, bool pred, uint32_t* o) {
    uint32_t a = 0u, b = 0u, c = 0u, d = 0u;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.global.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}\n"
                 : "+r"(a), "+r"(b), "+r"(c), "+r"(d) : "l"(p), "r"((int)pred));
    o[0] = a; o[1] = b; o[2] = c; o[3] = d;
  }
  __device__ static __forceinline__ void st(uint32_t* p, bool pred, const uint32_t* v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.v4.u32 [%0], {%1, %2, %3, %4};\n\t}\n"
                 :: "l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"((int)pred) : "memory");
  }
};

template <int G, int NCH, int PPL, int MINB>
__global__ void __launch_bounds__(G4_WARPS * 32, MINB) k_sgm_grp4(SgmArgs a, int fam, int init, int sweeps) {
  constexpr int NG = 32 / G;
  constexpr int CW = PPL * G;      // pairs per chunk
  constexpr int NW = PPL * NCH;    // words per lane
  constexpr uint32_t NONE = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int grp = lane / G;
  const int gbase = lane & ~(G - 1);
  const int W = a.W, H = a.H;
  const int nchains = fam == FAM_H ? H : (fam == FAM_V ? W : W + H - 1);
  const int c0 = (blockIdx.x * G4_WARPS + (threadIdx.x >> 5)) * NG;
  if (c0 >= nchains) return;
  if (a.select) {
    const double frac = (double)a.cells[blockIdx.y] / ((double)W * H * (a.d_max + 1));
    if ((a.select == 1) == (frac > a.split)) return;
  }
  const int ch = c0 + grp;
  const size_t HW = (size_t)W * H;
  const uint2* __restrict__ meta = a.meta + (size_t)blockIdx.y * HW;
  const uint32_t* __restrict__ C =
      reinterpret_cast<const uint32_t*>(a.C) + (size_t)blockIdx.y * a.volcap;
  uint32_t* S = reinterpret_cast<uint32_t*>(a.S) + (size_t)blockIdx.y * a.volcap;
  asm volatile("" : "+l"(C));
  asm volatile("" : "+l"(S));
  const int len = fam == FAM_H ? W : H;
  const int src_l = gbase | ((gl + G - 1) & (G - 1));
  const int src_r = gbase | ((gl + 1) & (G - 1));
  auto umask = [](int lo, int hi) -> uint32_t {
    return hi < lo ? 0u : ((hi >= 31 ? 0xFFFFFFFFu : ((2u << hi) - 1u)) & ~((1u << lo) - 1u));
  };
  // one specialised body per partial-sum mode: the first family's forward
  // sweep stores L (no partial-sum load); every other sweep loads the
  // partial sum only where it stores, so its loads need no default value
  auto sweep = [&](const int bwd, auto load_sum_tag) {
    constexpr bool load_sum = decltype(load_sum_tag)::value;
    // chain metadata: every lane loads its chain's pixel itself, four steps
    // ahead, into the register set of the step's parity (no register
    // rotation, so nothing waits on a load before its use)
    auto load_meta = [&](int t) -> uint2 {
      int x, y;
      if (t < len && grp_pixel(fam, bwd, ch, t, W, H, x, y)) return meta[(size_t)y * W + x];
      return make_uint2(NONE, 0u);
    };
    auto info = [&](uint2 mt) -> G4Step {
      G4Step s{0, 0, 0u, 0u};
      int clo = NCH, chi = -1;
      if (mt.x != NONE) {
        const int j0 = (int)((mt.x & 0xFFFFu) >> 1);
        const int j1 = (int)((mt.x >> 16) >> 1);
        s.base = (int)(mt.y - (uint32_t)j0) + PPL * gl;
        s.relb = PPL * gl - j0 + PPL - 1;
        s.spanp = (uint32_t)(j1 - j0 + PPL);
        clo = j0 / CW;
        chi = j1 / CW;
      }
      s.um = umask(__reduce_min_sync(FULL, clo), __reduce_max_sync(FULL, chi));
      return s;
    };
    auto pred_of = [&](const G4Step& s, int c) -> bool {
      return (uint32_t)(s.relb + c * CW) < s.spanp;
    };
    auto fetch = [&](const G4Step& s, uint32_t (&cn)[NW], uint32_t (&sn)[NW], int c) {
      const bool p = pred_of(s, c);
      Vec<PPL>::ldc(C + s.base + c * CW, p, &cn[c * PPL]);
      if constexpr (load_sum) Vec<PPL>::ld_any(S + s.base + c * CW, p, &sn[c * PPL]);
    };
    uint32_t prev[NW], cA[NW], sA[NW], cB[NW], sB[NW];
    uint2 mA = load_meta(0), mB = load_meta(1);
    G4Step s0 = info(mA);
    G4Step s1 = info(mB);
    mA = load_meta(2);
    mB = load_meta(3);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
#pragma unroll
      for (int k = 0; k < PPL; ++k) prev[c * PPL + k] = INF16x2;
      fetch(s0, cA, sA, c);
      fetch(s1, cB, sB, c);
    }
    uint32_t mp2 = INF16x2, ng = INF16x2;   // no predecessor: L = C
    const uint32_t p1x2 = a.p1i * 0x10001u;
    auto step = [&](const G4Step& cur, const G4Step& nn, uint32_t (&cn)[NW], uint32_t (&sn)[NW]) {
      uint32_t nmin = INF16x2;
      uint32_t left_old = INF16x2;   // previous chunk's last word, before overwrite
      uint32_t* Sb = S + cur.base;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        uint32_t P[PPL];
#pragma unroll
        for (int k = 0; k < PPL; ++k) P[k] = prev[c * PPL + k];
        if ((cur.um >> c) & 1u) {
          const uint32_t srcl = gl == G - 1 ? left_old : P[PPL - 1];
          const uint32_t srcr = gl == 0 ? (c + 1 < NCH ? prev[(c + 1 < NCH ? c + 1 : 0) * PPL] : INF16x2) : P[0];
          const uint32_t pl = __shfl_sync(FULL, srcl, src_l);
          const uint32_t pr = __shfl_sync(FULL, srcr, src_r);
          uint32_t X[PPL + 1];
          X[0] = __byte_perm(pl, P[0], 0x5432);
#pragma unroll
          for (int k = 1; k < PPL; ++k) X[k] = __byte_perm(P[k - 1], P[k], 0x5432);
          X[PPL] = __byte_perm(P[PPL - 1], pr, 0x5432);
          uint32_t L[PPL], Ssum[PPL];
#pragma unroll
          for (int k = 0; k < PPL; ++k) {
            // L = C + min(Lp(d), Lp(d-1)+P1, Lp(d+1)+P1, m+P2) - m   (sgm.py:205-215)
            const uint32_t cand = __viaddmin_u16x2(__vminu2(X[k], X[k + 1]), p1x2, __vminu2(P[k], mp2));
            L[k] = __vadd2(cn[c * PPL + k], __vadd2(cand, ng));
            Ssum[k] = load_sum ? __vadd2(sn[c * PPL + k], L[k]) : L[k];
            prev[c * PPL + k] = L[k];
          }
          if (PPL == 4) {
            nmin = __vimin3_u16x2(nmin, L[0], L[1]);
            nmin = __vimin3_u16x2(nmin, L[PPL - 2], L[PPL - 1]);
          } else {
            nmin = __vimin3_u16x2(nmin, L[0], L[PPL - 1]);
          }
          // halves outside [lo, hi] land in the pixel's own padding /
          // out-of-interval slots, which nothing reads
          Vec<PPL>::st(Sb + c * CW, pred_of(cur, c), Ssum);
        } else {
#pragma unroll
          for (int k = 0; k < PPL; ++k) prev[c * PPL + k] = INF16x2;
        }
        left_old = P[PPL - 1];
        if ((nn.um >> c) & 1u) fetch(nn, cn, sn, c);
      }
      // per-chain minimum: xor butterfly inside each G-lane group
      uint32_t hm = min(nmin & 0xFFFFu, nmin >> 16);
#pragma unroll
      for (int o = G / 2; o; o >>= 1) hm = min(hm, __shfl_xor_sync(FULL, hm, o));
      const bool act = cur.spanp != 0u;
      mp2 = act ? (hm + a.p2i) * 0x10001u : INF16x2;
      ng = act ? ((0x10000u - hm) & 0xFFFFu) * 0x10001u : INF16x2;
    };
    for (int t = 0; t < len; t += 2) {
      const G4Step s2 = info(mA);
      mA = load_meta(t + 4);
      step(s0, s2, cA, sA);
      if (t + 1 >= len) break;
      const G4Step s3 = info(mB);
      mB = load_meta(t + 5);
      step(s1, s3, cB, sB);
      s0 = s2;
      s1 = s3;
    }
  };
  // sweeps: bit 0 forward, bit 1 backward; the first sweep into a fresh
  // partial sum (init) stores instead of accumulating
  bool fresh = init != 0;
  for (int bwd = 0; bwd < 2; ++bwd) {
    if (!((sweeps >> bwd) & 1)) continue;
    if (fresh) sweep(bwd, std::false_type{});
    else sweep(bwd, std::true_type{});
    fresh = false;
  }
}

// ------------------------------------------------------------ row chains, operands through a cp.async ring
//
// k_sgm_grp4's recurrence with its operand path replaced.  grp4 fetches the
// cost / partial-sum words into registers two steps ahead, but ptxas tracks
// every global load of that kernel on ONE scoreboard, so the first use of
// any loaded register drains all loads in flight and the two-step lead
// collapses (ncu: 28% of the row jobs' stall samples on a step's first
// metadata test).  Here each lane copies its own 16-byte words of the pixel
// RL steps ahead into a lane-private slot of a per-warp shared-memory ring
// with cp.async (one commit group per step, cp.async.wait_group RL: a true
// RL-step lead that no other load can shorten), reads them back with LDS at
// use, and only the 8-byte metadata loads remain on the LDG scoreboard.
// Words outside the pixel's interval read a 16-byte +inf pad instead of
// their (unwritten) slot.
#ifndef ROW_RL
#define ROW_RL 2          // steps of lead; the ring has RL + 1 slots
#endif
#ifndef ROW_CTA_WARPS
#define ROW_CTA_WARPS 4
#endif
#ifndef ROW_MINB
#define ROW_MINB 4
#endif
constexpr int ROW_WARPS = ROW_CTA_WARPS;
template <int NCH, bool LOAD_SUM>
constexpr size_t row_smem() {
  // [warp][slot][chunk][C (, S)][lane] 16-byte words + one +inf pad
  return (size_t)ROW_WARPS * (ROW_RL + 1) * NCH * (LOAD_SUM ? 2 : 1) * 32 * 16 + 16;
}

template <int NCH, bool LOAD_SUM>
__global__ void __launch_bounds__(ROW_WARPS * 32, ROW_MINB) k_sgm_row(SgmArgs a, int bwd, int pfon) {
  static_assert(ROW_RL == 2, "the walk below is unrolled for a three-slot ring");
  constexpr int G = 4, PPL = 4, NG = 32 / G, CW = PPL * G, NW = PPL * NCH;
  constexpr int CHB = (LOAD_SUM ? 2 : 1) * 512;   // bytes per chunk of a slot (cost words, then partial-sum words)
  constexpr int SLOTB = NCH * CHB;             // bytes per ring slot
  constexpr int NSLOT = ROW_RL + 1;
  constexpr uint32_t NONE = 0xFFFFFFFFu;
  extern __shared__ __align__(16) uint8_t rsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gl = lane & (G - 1), grp = lane / G, gbase = lane & ~(G - 1);
  const int W = a.W, H = a.H;
  const int c0 = (blockIdx.x * ROW_WARPS + wid) * NG;
  if (threadIdx.x < 4) reinterpret_cast<uint32_t*>(rsm + (size_t)ROW_WARPS * NSLOT * SLOTB)[threadIdx.x] = INF16x2;
  __syncthreads();
  if (c0 >= H) return;
  if (a.select) {
    const double frac = (double)a.cells[blockIdx.y] / ((double)W * H * (a.d_max + 1));
    if ((a.select == 1) == (frac > a.split)) return;
  }
  const int y = c0 + grp;
  const size_t HW = (size_t)W * H;
  const uint32_t* __restrict__ C = reinterpret_cast<const uint32_t*>(a.C) + (size_t)blockIdx.y * a.volcap;
  uint32_t* S = reinterpret_cast<uint32_t*>(a.S) + (size_t)blockIdx.y * a.volcap;
  const int src_l = gbase | ((gl + G - 1) & (G - 1));
  const int src_r = gbase | ((gl + 1) & (G - 1));
  const unsigned ring_s = (unsigned)__cvta_generic_to_shared(rsm) + (unsigned)(wid * NSLOT * SLOTB) + 16u * lane;
  const unsigned inf_s = (unsigned)__cvta_generic_to_shared(rsm) + (unsigned)(ROW_WARPS * NSLOT * SLOTB);
  // the row's metadata, walked with a running pointer (rows past the image:
  // the lane group idles on NONE pixels)
  const int mdir = bwd ? -1 : 1;
  const uint2* mptr = a.meta + (size_t)blockIdx.y * HW + (size_t)min(y, H - 1) * W + (bwd ? W - 1 : 0);
  const int mlen = y < H ? W : 0;
  int mt_next = 0;   // step of the next metadata load
  const bool rowpf = G4_PF_WORDS > 0 && pfon;
  int pf = -1;
  auto load_meta = [&]() -> uint2 {
    uint2 m = make_uint2(NONE, 0u);
    if (mt_next < mlen) {
      if (rowpf && gl == 0 && (mt_next & 15) == 0 && mt_next + 32 < mlen)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(mptr + 32 * mdir));
      m = *mptr;
    }
    mptr += mdir;
    ++mt_next;
    return m;
  };
  auto info = [&](uint2 mt) -> G4Step {
    G4Step s{0, 0, 0u, 0u};
    int clo = NCH, chi = -1;
    if (mt.x != NONE) {
      const int j0 = (int)((mt.x & 0xFFFFu) >> 1);
      const int j1 = (int)((mt.x >> 16) >> 1);
      s.base = (int)(mt.y - (uint32_t)j0) + PPL * gl;
      s.relb = PPL * gl - j0 + PPL - 1;
      s.spanp = (uint32_t)(j1 - j0 + PPL);
      clo = j0 / CW;
      chi = j1 / CW;
      if (rowpf) {
        // L2 prefetch of the row's packed stream ahead of this pixel, four
        // 128-byte lines (one per lane of the group) at a time
        const int as = (int)(mt.y - ((uint32_t)j0 & 3u));   // allocation start (words)
        if (!bwd) {
          if (pf < 0) pf = as;
          if (pf < as + G4_PF_WORDS) {
            const int o = pf + 32 * gl;
            if ((size_t)o < a.volcap) {
              asm volatile("prefetch.global.L2 [%0];" ::"l"(C + o));
              if (LOAD_SUM) asm volatile("prefetch.global.L2 [%0];" ::"l"(S + o));
            }
            pf += 128;
          }
        } else {
          if (pf < 0) pf = as + 128;
          if (pf > as - G4_PF_WORDS) {
            const int o = pf - 32 * (gl + 1);
            if (o >= 0) {
              asm volatile("prefetch.global.L2 [%0];" ::"l"(C + o));
              if (LOAD_SUM) asm volatile("prefetch.global.L2 [%0];" ::"l"(S + o));
            }
            pf -= 128;
          }
        }
      }
    }
    uint32_t um = 0u;
    const int ulo = __reduce_min_sync(FULL, clo), uhi = __reduce_max_sync(FULL, chi);
    if (uhi >= ulo) um = ((2u << uhi) - 1u) & ~((1u << ulo) - 1u);
    s.um = um;
    return s;
  };
  auto pred_of = [&](const G4Step& s, int c) -> bool { return (uint32_t)(s.relb + c * CW) < s.spanp; };
  // the lane's words of pixel `s` into ring slot `slot` (one commit group)
  auto issue = [&](const G4Step& s, unsigned slot) {
#pragma unroll
    for (int c = 0; c < NCH; ++c)
      if ((s.um >> c) & 1u) {
        const int p = pred_of(s, c);
        const unsigned dst = slot + (unsigned)(c * CHB);
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q cp.async.cg.shared.global [%0], [%1], 16;\n\t}\n"
                     ::"r"(dst), "l"(C + s.base + c * CW), "r"(p) : "memory");
        if (LOAD_SUM)
          asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q cp.async.cg.shared.global [%0], [%1], 16;\n\t}\n"
                       ::"r"(dst + 512u), "l"(S + s.base + c * CW), "r"(p) : "memory");
      }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  uint32_t prev[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) prev[w] = INF16x2;
  uint32_t mp2 = INF16x2, ng = INF16x2;   // no predecessor: L = C
  const uint32_t p1x2 = a.p1i * 0x10001u;
  // pixel t lives in ring slot t % 3 with its decoded step in s[t % 3] and
  // its metadata register m[t % 3]; at step t the pixel t + 2 is decoded and
  // issued, the metadata of t + 5 requested, and pixel t computed
  G4Step s0 = info(load_meta());
  issue(s0, ring_s);
  G4Step s1 = info(load_meta());
  issue(s1, ring_s + SLOTB);
  G4Step s2{0, 0, 0u, 0u};
  uint2 m2 = load_meta(), m0 = load_meta(), m1 = load_meta();
  auto step = [&](const G4Step& cur, unsigned slot_use, G4Step& nx, uint2& mreg, unsigned slot_fill) {
    nx = info(mreg);
    mreg = load_meta();
    issue(nx, slot_fill);
    asm volatile("cp.async.wait_group 2;" ::: "memory");
    uint32_t nmin = INF16x2;
    uint32_t left_old = INF16x2;
    uint32_t* Sb = S + cur.base;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      uint32_t P[PPL];
#pragma unroll
      for (int k = 0; k < PPL; ++k) P[k] = prev[c * PPL + k];
      if ((cur.um >> c) & 1u) {
        const bool p = pred_of(cur, c);
        const unsigned src = slot_use + (unsigned)(c * CHB);
        uint32_t cn[PPL], sn[PPL];
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(cn[0]), "=r"(cn[1]), "=r"(cn[2]), "=r"(cn[3]) : "r"(p ? src : inf_s));
        if (LOAD_SUM)
          asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(sn[0]), "=r"(sn[1]), "=r"(sn[2]), "=r"(sn[3]) : "r"(src + 512u));
        const uint32_t srcl = gl == G - 1 ? left_old : P[PPL - 1];
        const uint32_t srcr = gl == 0 ? (c + 1 < NCH ? prev[(c + 1 < NCH ? c + 1 : 0) * PPL] : INF16x2) : P[0];
        const uint32_t pl = __shfl_sync(FULL, srcl, src_l);
        const uint32_t pr = __shfl_sync(FULL, srcr, src_r);
        uint32_t X[PPL + 1];
        X[0] = __byte_perm(pl, P[0], 0x5432);
#pragma unroll
        for (int k = 1; k < PPL; ++k) X[k] = __byte_perm(P[k - 1], P[k], 0x5432);
        X[PPL] = __byte_perm(P[PPL - 1], pr, 0x5432);
        uint32_t L[PPL], Ssum[PPL];
#pragma unroll
        for (int k = 0; k < PPL; ++k) {
          // L = C + min(Lp(d), Lp(d-1)+P1, Lp(d+1)+P1, m+P2) - m   (sgm.py:205-215)
          const uint32_t cand = __viaddmin_u16x2(__vminu2(X[k], X[k + 1]), p1x2, __vminu2(P[k], mp2));
          L[k] = __vadd2(cn[k], __vadd2(cand, ng));
          Ssum[k] = LOAD_SUM ? __vadd2(sn[k], L[k]) : L[k];
          prev[c * PPL + k] = L[k];
        }
        nmin = __vimin3_u16x2(nmin, L[0], L[1]);
        nmin = __vimin3_u16x2(nmin, L[PPL - 2], L[PPL - 1]);
        Vec<PPL>::st(Sb + c * CW, p, Ssum);
      } else {
#pragma unroll
        for (int k = 0; k < PPL; ++k) prev[c * PPL + k] = INF16x2;
      }
      left_old = P[PPL - 1];
    }
    uint32_t hm = min(nmin & 0xFFFFu, nmin >> 16);
#pragma unroll
    for (int o = G / 2; o; o >>= 1) hm = min(hm, __shfl_xor_sync(FULL, hm, o));
    const bool act = cur.spanp != 0u;
    mp2 = act ? (hm + a.p2i) * 0x10001u : INF16x2;
    ng = act ? ((0x10000u - hm) & 0xFFFFu) * 0x10001u : INF16x2;
  };
  for (int t = 0; t < W; t += 3) {
    step(s0, ring_s, s2, m2, ring_s + 2 * SLOTB);
    if (t + 1 >= W) break;
    step(s1, ring_s + SLOTB, s0, m0, ring_s);
    if (t + 2 >= W) break;
    step(s2, ring_s + 2 * SLOTB, s1, m1, ring_s + SLOTB);
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

static void launch_row(const SgmArgs& a, int bwd, int init, int pfon, int n_sv, cudaStream_t st) {
  const int nchains = a.H;
  constexpr int per_block = ROW_WARPS * 8;
  dim3 grid((nchains + per_block - 1) / per_block, n_sv);
  const int nch = (npairs_max(a.d_max) + 15) / 16;
  auto go = [&](auto kern, size_t smem) {
    ensure_smem((const void*)kern, smem);
    kern<<<grid, ROW_WARPS * 32, smem, st>>>(a, bwd, pfon);
  };
  if (nch <= 1) { if (init) go(k_sgm_row<1, false>, row_smem<1, false>()); else go(k_sgm_row<1, true>, row_smem<1, true>()); }
  else if (nch <= 2) { if (init) go(k_sgm_row<2, false>, row_smem<2, false>()); else go(k_sgm_row<2, true>, row_smem<2, true>()); }
  else { if (init) go(k_sgm_row<4, false>, row_smem<4, false>()); else go(k_sgm_row<4, true>, row_smem<4, true>()); }
}

template <int G, int PPL, int MINB>
static void launch_grp4(const SgmArgs& a, int fam, int init, int n_sv, cudaStream_t st,
                        int sweeps = 3) {
  const int nchains = fam == FAM_H ? a.H : (fam == FAM_V ? a.W : a.W + a.H - 1);
  constexpr int per_block = G4_WARPS * (32 / G);
  dim3 grid((nchains + per_block - 1) / per_block, n_sv);
  const int nch = (npairs_max(a.d_max) + PPL * G - 1) / (PPL * G);
  auto go = [&](auto kern) { kern<<<grid, G4_WARPS * 32, 0, st>>>(a, fam, init, sweeps); };
  if (nch <= 1) go(k_sgm_grp4<G, 1, PPL, MINB>);
  else if (nch <= 2) go(k_sgm_grp4<G, 2, PPL, MINB>);
  else if (nch <= 4) go(k_sgm_grp4<G, 4, PPL, MINB>);
  else go(k_sgm_grp4<G, 8, PPL, MINB>);
}

template <class A, bool CF32>
static void launch_family(const SgmArgs& a, int nch, int fam, int sweeps, int init, int n_sv,
                          cudaStream_t st) {
  const int nchains = fam == FAM_H ? a.H : (fam == FAM_V ? a.W : a.W + a.H - 1);
  dim3 grid((nchains + SGM_WARPS - 1) / SGM_WARPS, n_sv);
  const int bs = SGM_WARPS * 32;
  switch (nch) {
    case 1: k_sgm<A, 1, CF32><<<grid, bs, 0, st>>>(a, fam, sweeps, init); break;
    case 2: k_sgm<A, 2, CF32><<<grid, bs, 0, st>>>(a, fam, sweeps, init); break;
    case 3: k_sgm<A, 3, CF32><<<grid, bs, 0, st>>>(a, fam, sweeps, init); break;
    case 4: k_sgm<A, 4, CF32><<<grid, bs, 0, st>>>(a, fam, sweeps, init); break;
    default: k_sgm<A, 8, CF32><<<grid, bs, 0, st>>>(a, fam, sweeps, init); break;
  }
}

static void launch_grp4_g(int G, const SgmArgs& a, int fam, int init, int n_sv, cudaStream_t st,
                          int sweeps = 3) {
#ifndef G4_MINB
#define G4_MINB 4
#endif
  if (G <= 4) launch_grp4<4, 4, G4_MINB>(a, fam, init, n_sv, st, sweeps);
  else if (G == 8) launch_grp4<8, 4, 1>(a, fam, init, n_sv, st, sweeps);
  else if (G == 16) launch_grp4<16, 4, 1>(a, fam, init, n_sv, st, sweeps);
  else launch_grp4<32, 4, 1>(a, fam, init, n_sv, st, sweeps);
}

// the single-direction row jobs of the per-direction schedules (small
// batches) run k_sgm_row as well (B = 8: 1397 -> 1430 frames/s, B = 16: 1480
// -> 1489).  ES_SGM_ROW = 0: grp4 everywhere, 1: k_sgm_row in the sweep
// schedules only, 2 (default): everywhere
static bool row_small(int fam, int sweeps, int widen, int d_max) {
  static const int row_env = getenv("ES_SGM_ROW") ? atoi(getenv("ES_SGM_ROW")) : 2;
  return row_env >= 2 && fam == FAM_H && (sweeps == 1 || sweeps == 2) && widen == 0 &&
         npairs_max(d_max) <= 64;
}

// u16 aggregation with the per-(seq, view) regime choice: views with reduced
// intervals run the narrow variant on st_lo[p], wide ones the wide variant on
// st_hi[p]; each (seq, view) is handled by exactly one of them, so the two
// never touch the same volume and run concurrently.  Jobs into the same
// partial sum are ordered on its stream pair.
int launch_aggregate_parts(const SgmArgs& a, int n_sv, int parts, void* const* S,
                            const cudaStream_t* st_lo, const cudaStream_t* st_hi) {
  // parts partial sums: family k accumulates into S[k % parts] on streams
  // st_lo/st_hi[k % parts]; each (seq, view) uses exactly one of lo / hi
  const int np = npairs_max(a.d_max);
  const int fams[4] = {FAM_H, FAM_V, FAM_D1, FAM_D2};
  static const int g4 = getenv("ES_SGM_G4") ? atoi(getenv("ES_SGM_G4")) : 1;   // A/B switch
  // lanes per chain: G = 4 (8 chains per warp) from two sequences up -- the
  // split job schedules keep enough warps in flight -- and G = 8 for a single
  // sequence; D = 256 doubles G so the register-resident chunk arrays stay at
  // <= 4 words x 4 chunks (measured)
  static const int widen_env = getenv("ES_SGM_WIDEN") ? atoi(getenv("ES_SGM_WIDEN")) : -1;
  int widen = widen_env >= 0 ? widen_env : (n_sv <= 2 && np <= 64 ? 1 : 0);
  if (np > 64) widen += 1;
  static const int split_env = getenv("ES_SGM_SPLITH") ? atoi(getenv("ES_SGM_SPLITH")) : 1;
  // the fused sweep runs one CTA (a whole SM) per (sequence, view) for a
  // fixed ~9.4 ms per launch at 1242x375: it pays from 64 views up (B = 32:
  // 1569 vs 1495 frames/s, B = 48: 1598 vs 1542; B = 24: 1347 vs 1477,
  // B = 16: 1086 vs 1481 -- measured); smaller batches keep the
  // per-direction jobs (ES_SGM_SWEEP=0 / 1 force it off / on)
  static const int sweep_env = getenv("ES_SGM_SWEEP") ? atoi(getenv("ES_SGM_SWEEP")) : -1;
  // (views of all contexts sharing the device count: contexts of ~32 views
  // pack the SMs better than one large context -- B = 64: 2005 frames/s as
  // 4 x 16 sequences vs 1937 as 2 x 32 and 1715 as one; B = 24: 1539 as
  // 2 x 12 vs 1262 -- pipeline.default_groups; a context on its own below
  // 64 views keeps the per-direction jobs)
  const bool use_sweep =
      sweep_env < 0 ? (n_sv >= 64 || (n_sv >= 24 && a.shared_views >= 48)) : sweep_env > 0;
  if (g4 && use_sweep && a.sweep_ring && (parts == 2 || parts == 4) && sweep_lanes(a.d_max)) {
    // fused vertical + diagonal sweeps (es_sgm_sweep.cu): each partial sum
    // takes one row job and one three-direction sweep: S0 = rows ->, then
    // the dy = +1 sweep; S1 = rows <-, then the dy = -1 sweep (parts == 4:
    // the sweeps write S2 / S3 concurrently with the row jobs instead)
    const int ns = sweep_strips(a.W, a.d_max, a.H);
    const size_t ringw = sweep_ring_words(a.W, a.d_max, a.H);
    // the sweeps keep one CTA per view and leave SMs idle (128 views on 148
    // SMs): with parts == 2 the second stream runs its sweep FIRST, so the
    // first stream's row job fills those SMs while it runs (and the second
    // stream's row job those of the first stream's sweep)
    // (with fewer views than SMs both sweeps fit side by side after both row
    // jobs: 64 views, measured 1604 vs 1558 frames/s at B = 32 and 1840 vs
    // 1796 with two B = 32 contexts; 128 views: sweep first on stream 1)
    static const int order_env = getenv("ES_SGM_SWEEP_ORDER") ? atoi(getenv("ES_SGM_SWEEP_ORDER")) : -1;
    const int order = order_env >= 0 ? order_env : (n_sv >= 128 ? 1 : 0);
    for (int p = 0; p < 2; ++p) {
      SgmArgs lo = a, hi = a;
      lo.select = 1;
      hi.select = 2;
      lo.S = S[p];
      hi.S = S[p];
      const int sp = parts == 4 ? p + 2 : p;
      SweepArgs v;
      v.a = a;
      v.a.S = S[sp];
      v.up = p;
      v.nstrips = ns;
      v.total = n_sv * ns;
      v.ring = a.sweep_ring + (size_t)p * n_sv * ringw;
      cudaStream_t vs = st_lo[sp];
      const bool sweep_first = parts == 2 && ((p == 1 && order) || order == 2);
      if (sweep_first) launch_sweep(v, true, vs);
      // both regime variants of the row job on one stream
      static const int row_env = getenv("ES_SGM_ROW") ? atoi(getenv("ES_SGM_ROW")) : 2;
      if (row_env && widen == 0 && npairs_max(a.d_max) <= 64)
        launch_row(lo, p, sweep_first ? 0 : 1, 1, n_sv, st_lo[p]);
      else
        launch_grp4_g(4 << widen, lo, FAM_H, sweep_first ? 0 : 1, n_sv, st_lo[p], p == 0 ? 1 : 2);
      launch_grp4_g(8 << widen, hi, FAM_H, sweep_first ? 0 : 1, n_sv, st_lo[p], p == 0 ? 1 : 2);
      if (!sweep_first) launch_sweep(v, parts == 4, vs);
    }
    return parts;
  }
  static const int vd3_env = getenv("ES_SGM_VD") ? atoi(getenv("ES_SGM_VD")) : 0;
  if (g4 && parts == 4 && vd3_env == 3 && vd_supported(a.W, a.d_max)) {
    // three live partial sums: S2 = the cluster pass of the dy = +1
    // directions (writing, no dependency), concurrent with S0 = rows ->,
    // columns up, x-y diagonal up and S1 = rows <-, x+y diagonal up
    SgmArgs lo2 = a, hi2 = a;
    lo2.select = 1;
    hi2.select = 2;
    lo2.S = S[2];
    hi2.S = S[2];
    launch_vd(lo2, false, true, n_sv, st_lo[2]);
    launch_vd(hi2, false, true, n_sv, st_hi[2]);
    struct Job { int part, fam, sweeps, init; };
    const Job jobs[5] = {{0, FAM_H, 1, 1}, {1, FAM_H, 2, 1}, {0, FAM_V, 2, 0},
                         {1, FAM_D2, 2, 0}, {0, FAM_D1, 2, 0}};
    for (const Job& j : jobs) {
      SgmArgs lo = a, hi = a;
      lo.select = 1;
      hi.select = 2;
      lo.S = S[j.part];
      hi.S = S[j.part];
      launch_grp4_g(4 << widen, lo, j.fam, j.init, n_sv, st_lo[j.part], j.sweeps);
      launch_grp4_g(8 << widen, hi, j.fam, j.init, n_sv, st_hi[j.part], j.sweeps);
    }
    return 3;
  }
  if (g4 && parts == 4 && split_env) {
    // small batches are latency-bound on the longest chain walk (a row's
    // 2W steps): the row family's two sweeps run as separate jobs into their
    // own partial sums, so the critical path is max(W, 3H) steps instead of
    // 2W (jobs: S0 = rows ->, S1 = rows <-, S2 = columns + x-y diagonals ->,
    // S3 = x-y diagonals <- + x+y diagonals)
    struct Job { int part, fam, sweeps, init; };
    const Job jobs[6] = {{0, FAM_H, 1, 1}, {1, FAM_H, 2, 1}, {2, FAM_V, 3, 1},
                         {3, FAM_D1, 2, 1}, {2, FAM_D1, 1, 0}, {3, FAM_D2, 3, 0}};
    for (const Job& j : jobs) {
      SgmArgs lo = a, hi = a;
      lo.select = 1;
      hi.select = 2;
      lo.S = S[j.part];
      hi.S = S[j.part];
      if (row_small(j.fam, j.sweeps, widen, a.d_max))
        launch_row(lo, j.sweeps == 2, j.init, n_sv >= 48, n_sv, st_lo[j.part]);
      else
        launch_grp4_g(4 << widen, lo, j.fam, j.init, n_sv, st_lo[j.part], j.sweeps);
      launch_grp4_g(8 << widen, hi, j.fam, j.init, n_sv, st_hi[j.part], j.sweeps);
    }
    return parts;
  }
  static const int vd_env = getenv("ES_SGM_VD") ? atoi(getenv("ES_SGM_VD")) : 0;
  if (g4 && parts == 2 && vd_env && vd_supported(a.W, a.d_max)) {
    // fused column + diagonal passes: S0 = rows ->, then the three dy = +1
    // directions; S1 = the three dy = -1 directions, then rows <-.  The
    // cluster passes leave SMs idle (whole 8-SM clusters per GPC); each runs
    // beside the other stream's row job.
    for (int p = 0; p < 2; ++p) {
      SgmArgs lo = a, hi = a;
      lo.select = 1;
      hi.select = 2;
      lo.S = S[p];
      hi.S = S[p];
      if (p == 0) {
        launch_grp4_g(4 << widen, lo, FAM_H, 1, n_sv, st_lo[p], 1);
        launch_grp4_g(8 << widen, hi, FAM_H, 1, n_sv, st_hi[p], 1);
        launch_vd(lo, false, false, n_sv, st_lo[p]);
        launch_vd(hi, false, false, n_sv, st_hi[p]);
      } else if (vd_env == 2) {
        // mixed: the dy = -1 directions as grp4 jobs beside the cluster pass
        const int fam_sw[4][3] = {{FAM_H, 2, 1}, {FAM_V, 2, 0}, {FAM_D1, 2, 0}, {FAM_D2, 2, 0}};
        for (const auto& j : fam_sw) {
          launch_grp4_g(4 << widen, lo, j[0], j[2], n_sv, st_lo[p], j[1]);
          launch_grp4_g(8 << widen, hi, j[0], j[2], n_sv, st_hi[p], j[1]);
        }
      } else {
        launch_vd(lo, true, true, n_sv, st_lo[p]);
        launch_vd(hi, true, true, n_sv, st_hi[p]);
        launch_grp4_g(4 << widen, lo, FAM_H, 0, n_sv, st_lo[p], 2);
        launch_grp4_g(8 << widen, hi, FAM_H, 0, n_sv, st_hi[p], 2);
      }
    }
    return parts;
  }
  static const int split2_env = getenv("ES_SGM_SPLIT2") ? atoi(getenv("ES_SGM_SPLIT2")) : 1;
  if (g4 && parts == 2 && split2_env) {
    // two partial sums: the row family's sweeps (the longest chains) run on
    // both streams at once, so every stream carries one long and one short
    // half: S0 = rows ->, columns, x+y diagonals ->; S1 = rows <-, x-y
    // diagonals, x+y diagonals <-
    struct Job { int part, fam, sweeps, init; };
    const Job jobs[6] = {{0, FAM_H, 1, 1}, {1, FAM_H, 2, 1}, {0, FAM_V, 3, 0},
                         {1, FAM_D1, 3, 0}, {0, FAM_D2, 1, 0}, {1, FAM_D2, 2, 0}};
    for (const Job& j : jobs) {
      SgmArgs lo = a, hi = a;
      lo.select = 1;
      hi.select = 2;
      lo.S = S[j.part];
      hi.S = S[j.part];
      if (row_small(j.fam, j.sweeps, widen, a.d_max))
        launch_row(lo, j.sweeps == 2, j.init, n_sv >= 48, n_sv, st_lo[j.part]);
      else
        launch_grp4_g(4 << widen, lo, j.fam, j.init, n_sv, st_lo[j.part], j.sweeps);
      launch_grp4_g(8 << widen, hi, j.fam, j.init, n_sv, st_hi[j.part], j.sweeps);
    }
    return parts;
  }
  if (g4) {
    for (int k = 0; k < 4; ++k) {
      const int p = k % parts;
      SgmArgs lo = a, hi = a;
      lo.select = 1;
      hi.select = 2;
      lo.S = S[p];
      hi.S = S[p];
      const int init = k < parts;
      launch_grp4_g(4 << widen, lo, fams[k], init, n_sv, st_lo[p]);
      launch_grp4_g(8 << widen, hi, fams[k], init, n_sv, st_hi[p]);
    }
    return parts;
  }
  for (int k = 0; k < 4; ++k) {
    const int p = k % parts;
    SgmArgs lo = a, hi = a;
    lo.select = 1;
    hi.select = 2;
    lo.S = S[p];
    hi.S = S[p];
    const int init = k < parts;   // first family into this partial sum
    // lanes per chain: reduced intervals 4 lanes while the full range fits
    // 8 chunks of 2G pairs (D <= 128), wide ones twice that; larger D widens
    // both so the register-resident chunk arrays never exceed 8 (16 for the
    // widest instance) -- at NCH 16 the 4-lane instance spills (measured,
    // config 4: D = 256)
    if (np <= 64) {
      launch_grp3<4>(lo, np, fams[k], 3, init, n_sv, st_lo[p]);
      launch_grp3<8>(hi, np, fams[k], 3, init, n_sv, st_hi[p]);
    } else if (np <= 128) {
      launch_grp3<8>(lo, np, fams[k], 3, init, n_sv, st_lo[p]);
      launch_grp3<16>(hi, np, fams[k], 3, init, n_sv, st_hi[p]);
    } else {
      launch_grp3<16>(lo, np, fams[k], 3, init, n_sv, st_lo[p]);
      launch_grp3<32>(hi, np, fams[k], 3, init, n_sv, st_hi[p]);
    }
  }
  return parts;
}

void launch_aggregate(const SgmArgs& a, int arith, int n_sv, cudaStream_t st) {
  int nch = (npairs_max(a.d_max) + 31) / 32;
  if (nch > 4) nch = 8;
  static const bool v1 = getenv("ES_SGM_V1") != nullptr;   // A/B switch for profiling
  static const int g4 = getenv("ES_SGM_G4") ? atoi(getenv("ES_SGM_G4")) : 1;   // A/B switch
  if (arith == ARITH_U16 && !v1 && g4 && !a.lanes) {
    const int fams[4] = {FAM_H, FAM_V, FAM_D1, FAM_D2};
    const int widen = (n_sv <= 2 ? 2 : (n_sv <= 8 ? 1 : 0)) + (npairs_max(a.d_max) > 64);
    for (int k = 0; k < 4; ++k) launch_grp4_g(4 << widen, a, fams[k], k == 0, n_sv, st);
  } else if (arith == ARITH_U16) {
    launch_family<U16A, false>(a, nch, FAM_H, 3, 1, n_sv, st);
    launch_family<U16A, false>(a, nch, FAM_V, 3, 0, n_sv, st);
    launch_family<U16A, false>(a, nch, FAM_D1, 3, 0, n_sv, st);
    launch_family<U16A, false>(a, nch, FAM_D2, 3, 0, n_sv, st);
  } else {
    // reference order: H->, H<-, (-1,+1), (0,+1), (+1,+1), (-1,-1), (0,-1), (+1,-1)
    static const int order[8][2] = {{FAM_H, 1}, {FAM_H, 2}, {FAM_D2, 1}, {FAM_V, 1},
                                    {FAM_D1, 1}, {FAM_D1, 2}, {FAM_V, 2}, {FAM_D2, 2}};
    for (int k = 0; k < 8; ++k) {
      if (a.cost_f32)
        launch_family<F32A, true>(a, nch, order[k][0], order[k][1], k == 0, n_sv, st);
      else
        launch_family<F32A, false>(a, nch, order[k][0], order[k][1], k == 0, n_sv, st);
    }
  }
}

// ------------------------------------------------------------ WTA + variance

// One warp per pixel: argmin over the interval (ties -> smaller d,
// sgm.py:282), then the outward walk of sgm.py:319-344 by lane 0.
template <bool F32>
__global__ void __launch_bounds__(256) k_wta_var(WtaArgs a) {
  const int lane = threadIdx.x & 31;
  const size_t HW = (size_t)a.W * a.H;
  const size_t pix = (size_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (pix >= HW) return;
  const int svl = blockIdx.y;
  const uint2 mt = a.meta[svl * HW + pix];
  const int lo = lo_of(mt), hi = hi_of(mt);
  const int j0 = lo >> 1, j1 = hi >> 1;
  const size_t base = svl * a.volcap + mt.y;
  float bestv = INFINITY;
  int bestd = 0x7fffffff;
  if (a.dstar_in == nullptr) {
    for (int j = j0 + lane; j <= j1; j += 32) {
      float v0, v1;
      if constexpr (F32) {
        const float2 w = reinterpret_cast<const float2*>(a.S)[base + (j - j0)];
        v0 = w.x;
        v1 = w.y;
      } else {
        const uint32_t w = reinterpret_cast<const uint32_t*>(a.S)[base + (j - j0)];
        v0 = (float)(w & 0xFFFFu);
        v1 = (float)(w >> 16);
      }
      const int d0 = 2 * j, d1 = 2 * j + 1;
      if (d0 >= lo && d0 <= hi && (v0 < bestv || (v0 == bestv && d0 < bestd))) { bestv = v0; bestd = d0; }
      if (d1 >= lo && d1 <= hi && (v1 < bestv || (v1 == bestv && d1 < bestd))) { bestv = v1; bestd = d1; }
    }
  #pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(FULL, bestv, o);
      const int od = __shfl_xor_sync(FULL, bestd, o);
      if (ov < bestv || (ov == bestv && od < bestd)) { bestv = ov; bestd = od; }
    }
    if (bestd == 0x7fffffff) bestd = 0;   // all +inf: numpy argmin -> index 0
  }
  if (lane != 0) return;
  auto cell = [&](int d) -> float {
    const int jj = (d >> 1) - j0;
    if constexpr (F32) {
      const float2 w = reinterpret_cast<const float2*>(a.S)[base + jj];
      return (d & 1) ? w.y : w.x;
    } else {
      const uint32_t w = reinterpret_cast<const uint32_t*>(a.S)[base + jj];
      return (float)((d & 1) ? (w >> 16) : (w & 0xFFFFu));
    }
  };
  if (a.dstar_in) {
    bestd = a.dstar_in[svl * HW + pix];
    bestv = (bestd >= lo && bestd <= hi) ? cell(bestd) : INFINITY;
  }
  const float cstar = bestv;
  long long count = 0;
  double s = 0.0;
  const bool inside = bestd >= lo && bestd <= hi;   // false only for all-inf pixels
  for (int d = bestd - 1; inside && d >= lo; --d) {
    s += (double)__fsub_rn(cell(d), cstar);
    if (!(s < a.s_max)) break;
    ++count;
  }
  s = 0.0;
  for (int d = bestd + 1; inside && d <= hi; ++d) {
    s += (double)__fsub_rn(cell(d), cstar);
    if (!(s < a.s_max)) break;
    ++count;
  }
  const size_t o = svl * HW + pix;
  a.dstar[o] = (uint16_t)bestd;
  a.valid[o] = bestd > 0;
  a.r[o] = fmax((double)count, a.r_min);
}

template <int N>
struct SumRows {
  const uint32_t* p[N];
  __device__ __forceinline__ uint32_t operator()(int k) const {   // total at pair offset k
    uint32_t w = p[0][k];
#pragma unroll
    for (int i = 1; i < N; ++i) w = __vadd2(w, p[i][k]);
    return w;
  }
};

template <int N>
__device__ __forceinline__ SumRows<N> sum_rows(const WtaArgs& a, size_t off) {
  SumRows<N> r;
  r.p[0] = reinterpret_cast<const uint32_t*>(a.S) + off;
#pragma unroll
  for (int i = 1; i < N; ++i) r.p[i] = reinterpret_cast<const uint32_t*>(a.Sx[i - 1]) + off;
  return r;
}

template <int N>
__device__ __forceinline__ void wta_finish(const WtaArgs& a, const SumRows<N>& s, int lo, int hi,
                                           int j0, uint32_t best, size_t o) {
  const int dstar = (int)(best & 0xFFFFu);
  const uint32_t cstar = best >> 16;
  auto cell = [&](int d) -> uint32_t {
    const uint32_t w = s((d >> 1) - j0);
    return (d & 1) ? (w >> 16) : (w & 0xFFFFu);
  };
  long long count = 0;
  double acc = 0.0;
  for (int d = dstar - 1; d >= lo; --d) {
    acc += (double)(cell(d) - cstar);
    if (!(acc < a.s_max)) break;
    ++count;
  }
  acc = 0.0;
  for (int d = dstar + 1; d <= hi; ++d) {
    acc += (double)(cell(d) - cstar);
    if (!(acc < a.s_max)) break;
    ++count;
  }
  a.dstar[o] = (uint16_t)dstar;
  a.valid[o] = dstar > 0;
  a.r[o] = fmax((double)count, a.r_min);
}

// u16 sums, run-table schedule (as k_cost_runs): a warp owns 32 consecutive
// pixels of a view, lane l streams runs l, l+32, ... of their allocations
// (one coalesced 16-byte word per partial sum, 8 cells), forms
// (value << 16 | d) keys for the cells inside [lo, hi], reduces them over the
// pixel's lanes with a segmented shuffle minimum and a shared-memory
// atomicMin (pixels whose runs span iterations), and finally every lane
// walks outward from its own pixel's winner (sgm.py:282, 319-344) over
// L1-resident data.
constexpr int WR_WARPS = 8;

template <int N, int U>
__global__ void __launch_bounds__(WR_WARPS * 32, 4) k_wta_runs(WtaArgs a, int rmax, int n_sv) {
  extern __shared__ uint32_t wsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* key = wsm + wid * 32;
  uint8_t* tab = reinterpret_cast<uint8_t*>(wsm + WR_WARPS * 32) + wid * 32 * rmax;
  const size_t HW = (size_t)a.W * a.H;
  // work items: (view, 32-pixel group), taken in a grid-wide stride so a grid
  // of whole waves (launch_wta_variance) ends together whatever the batch
  const uint32_t ngroups = (uint32_t)((HW + 31) / 32);
  const size_t nitems = (size_t)ngroups * (size_t)n_sv;
  const size_t istride = (size_t)gridDim.x * WR_WARPS;
  // metadata of the lane's pixel of item `it` (requested one item ahead: ncu
  // had 11% of this kernel's stall samples on its first use)
  auto item_meta = [&](size_t it) -> uint2 {
    if (it >= nitems) return make_uint2(0u, 0u);
    const size_t sv = it / ngroups;
    const size_t px = (it - sv * ngroups) * 32 + lane;
    return px < HW ? a.meta[sv * HW + px] : make_uint2(0u, 0u);
  };
  uint2 mt_next = item_meta((size_t)blockIdx.x * WR_WARPS + wid);
  for (size_t it = (size_t)blockIdx.x * WR_WARPS + wid; it < nitems; it += istride) {
    const int svl = (int)(it / ngroups);
    const size_t g = it - (size_t)svl * ngroups;
    const uint4* Sv[N];
    Sv[0] = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(a.S) + (size_t)svl * a.volcap);
#pragma unroll
    for (int i = 1; i < N; ++i)
      Sv[i] = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(a.Sx[i - 1]) + (size_t)svl * a.volcap);
    const size_t pix = g * 32 + lane;
    const uint2 mt = mt_next;
    mt_next = item_meta(it + istride);
    int lo = 0, hi = -1, nrun = 0;
    uint32_t run0 = 0;
    if (pix < HW) {
      lo = (int)lo_of(mt);
      hi = (int)hi_of(mt);
      run0 = (mt.y - pad_before(lo)) >> 2;
      nrun = (int)(pixel_slots(lo, hi) >> 2);
    }
    int incl = nrun;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const int excl = incl - nrun;
    const int total = __shfl_sync(FULL, incl, 31);
    for (int j = 0; j < nrun; ++j) tab[excl + j] = (uint8_t)lane;
    key[lane] = 0xFFFFFFFFu;
    __syncwarp();
    // U runs per lane per iteration: all partial-sum loads of them are in
    // flight before either is reduced; keys go to the pixel's slot with a
    // shared-memory atomicMin (ties resolve to the smaller d by the key)
    for (int r0 = 0; r0 < total; r0 += 32 * U) {
      int p[U], plo[U], phi[U], pex[U];
      uint32_t prun[U];
      bool live[U];
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + 32 * u + lane;
        live[u] = r < total;
        p[u] = live[u] ? tab[r] : 31;
        plo[u] = __shfl_sync(FULL, lo, p[u]);
        phi[u] = __shfl_sync(FULL, hi, p[u]);
        pex[u] = __shfl_sync(FULL, excl, p[u]);
        prun[u] = __shfl_sync(FULL, run0, p[u]);
        w[u] = make_uint4(0u, 0u, 0u, 0u);
        if (live[u]) {
          const int j = r - pex[u];
          w[u] = Sv[0][prun[u] + j];
#pragma unroll
          for (int i = 1; i < N; ++i) {
            const uint4 v = Sv[i][prun[u] + j];
            w[u] = make_uint4(__vadd2(w[u].x, v.x), __vadd2(w[u].y, v.y), __vadd2(w[u].z, v.z),
                              __vadd2(w[u].w, v.w));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!live[u]) continue;
        const int j = r0 + 32 * u + lane - pex[u];
        const uint32_t d0 = (uint32_t)((plo[u] & ~7) + 8 * j);
        const uint32_t ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
        uint32_t k[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          k[2 * q] = (ww[q] << 16) | (d0 + 2 * q);
          k[2 * q + 1] = (ww[q] & 0xFFFF0000u) | (d0 + 2 * q + 1);
        }
        if ((int)d0 < plo[u] || (int)d0 + 7 > phi[u]) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if ((int)d0 + i < plo[u] || (int)d0 + i > phi[u]) k[i] = 0xFFFFFFFFu;
        }
        const uint32_t best =
            min(min(min(k[0], k[1]), min(k[2], k[3])), min(min(k[4], k[5]), min(k[6], k[7])));
        atomicMin(&key[p[u]], best);
      }
    }
    __syncwarp();
    if (pix < HW) {
      const SumRows<N> s = sum_rows<N>(a, (size_t)svl * a.volcap + mt.y);
      wta_finish(a, s, lo, hi, lo >> 1, key[lane], (size_t)svl * HW + pix);
    }
    __syncwarp();
  }
}

void launch_wta_variance(const WtaArgs& a, int n_sv, cudaStream_t st) {
  if (a.arith == ARITH_U16 && a.dstar_in == nullptr) {
    const size_t HW = (size_t)a.W * a.H;
    const int nparts = 1 + (a.Sx[0] != nullptr) + (a.Sx[1] != nullptr) + (a.Sx[2] != nullptr);
    const int rmax = (npairs_max(a.d_max) + 3) / 4;
    const size_t smem = sizeof(uint32_t) * WR_WARPS * 32 + (size_t)WR_WARPS * 32 * rmax;
    const size_t groups = (HW + 31) / 32;
    // a 1-D grid of whole waves (4 resident blocks of 8 warps per SM at 64
    // registers) striding over (view, group) items: the round-1 grid of ~19
    // blocks per view was 2.05 waves at 64 views, i.e. a third, nearly empty
    // wave.  Measured at B = 64 (stage ms per step): 1 wave 4.6, 2 waves
    // 3.7, 4 waves 3.65, 8 waves 3.47 (old grid 3.9).
    static const int waves = getenv("ES_WTA_WAVES") ? std::max(1, atoi(getenv("ES_WTA_WAVES"))) : 8;
    const size_t items = groups * (size_t)n_sv;
    const unsigned nblk = (unsigned)std::min<size_t>((items + WR_WARPS - 1) / WR_WARPS,
                                                     (size_t)device_sms() * 4 * waves);
    dim3 grid(nblk);
    auto go = [&](auto kern) {
      ensure_smem((const void*)kern, smem);
      kern<<<grid, WR_WARPS * 32, smem, st>>>(a, rmax, n_sv);
    };
    // runs in flight per lane: four for narrow views, two for wide ones
    // (measured: 1242 px rows 3.49 -> 3.21 ms with four; 2048 px rows 4.75 ->
    // 5.11 ms)
    if (a.W <= 1536) {
      if (nparts == 1) go(k_wta_runs<1, 4>);
      else if (nparts == 2) go(k_wta_runs<2, 4>);
      else if (nparts == 3) go(k_wta_runs<3, 4>);
      else go(k_wta_runs<4, 4>);
    } else {
      if (nparts == 1) go(k_wta_runs<1, 2>);
      else if (nparts == 2) go(k_wta_runs<2, 2>);
      else if (nparts == 3) go(k_wta_runs<3, 2>);
      else go(k_wta_runs<4, 2>);
    }
    return;
  }
  const size_t HW = (size_t)a.W * a.H;
  dim3 grid((unsigned)((HW + 7) / 8), n_sv);
  if (a.arith == ARITH_U16) k_wta_var<false><<<grid, 256, 0, st>>>(a);
  else k_wta_var<true><<<grid, 256, 0, st>>>(a);
}

// ------------------------------------------------------------ converters

__global__ void k_export_dense(const uint2* __restrict__ meta, const void* __restrict__ vol,
                               int vol_f32, int W, int H, int D, float* __restrict__ out,
                               const void* __restrict__ vol2, const void* __restrict__ vol3,
                               const void* __restrict__ vol4) {
  const size_t HW = (size_t)W * H;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= HW * D) return;
  const size_t pix = idx / D;
  const int d = (int)(idx % D);
  const uint2 mt = meta[pix];
  const int lo = lo_of(mt), hi = hi_of(mt);
  float v = INFINITY;
  if (d >= lo && d <= hi) {
    const size_t k = (size_t)mt.y + (size_t)((d >> 1) - (lo >> 1));
    if (vol_f32 == EXPORT_F32) {
      const float2 w = reinterpret_cast<const float2*>(vol)[k];
      v = (d & 1) ? w.y : w.x;
    } else {
      uint32_t w = reinterpret_cast<const uint32_t*>(vol)[k];
      if (vol2) w = __vadd2(w, reinterpret_cast<const uint32_t*>(vol2)[k]);
      if (vol3) w = __vadd2(w, reinterpret_cast<const uint32_t*>(vol3)[k]);
      if (vol4) w = __vadd2(w, reinterpret_cast<const uint32_t*>(vol4)[k]);
      const uint32_t h = (d & 1) ? (w >> 16) : (w & 0xFFFFu);
      // u16 costs use 0x8000 as +inf; u16 sums are always finite in-interval
      v = (vol_f32 == EXPORT_U16_COST && h >= INF16) ? INFINITY : (float)h;
    }
  }
  out[idx] = v;
}

void launch_export_dense(const uint2* meta, const void* vol, int vol_f32, int W, int H, int d_max,
                         float* out, cudaStream_t st, const void* vol2, const void* vol3,
                         const void* vol4) {
  const size_t n = (size_t)W * H * (d_max + 1);
  k_export_dense<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(meta, vol, vol_f32, W, H, d_max + 1,
                                                               out, vol2, vol3, vol4);
}

// dense (H, W, D) float32 -> ragged pairs (u16 when as_f32 == 0)
__global__ void k_import_dense(const float* __restrict__ dense, const uint2* __restrict__ meta,
                               int W, int H, int D, int as_f32, void* __restrict__ vol) {
  const size_t pix = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= (size_t)W * H) return;
  const uint2 mt = meta[pix];
  const int lo = lo_of(mt), hi = hi_of(mt);
  // the pixel's padding slots hold +inf too (read by the aggregation's
  // aligned multi-pair accesses, es_common.cuh)
  const uint32_t a0 = mt.y - pad_before(lo), a1 = a0 + pixel_slots(lo, hi);
  const uint32_t k0 = mt.y, k1 = mt.y + (uint32_t)((hi >> 1) - (lo >> 1) + 1);
  for (uint32_t k = a0; k < a1; ++k) {
    if (k >= k0 && k < k1) continue;
    if (as_f32) reinterpret_cast<float2*>(vol)[k] = make_float2(INFINITY, INFINITY);
    else reinterpret_cast<uint32_t*>(vol)[k] = INF16x2;
  }
  for (int j = lo >> 1; j <= (hi >> 1); ++j) {
    const size_t k = (size_t)mt.y + (size_t)(j - (lo >> 1));
    float v[2];
    for (int h = 0; h < 2; ++h) {
      const int d = 2 * j + h;
      v[h] = (d >= lo && d <= hi) ? dense[pix * D + d] : INFINITY;
    }
    if (as_f32) {
      reinterpret_cast<float2*>(vol)[k] = make_float2(v[0], v[1]);
    } else {
      uint32_t w = 0;
      for (int h = 0; h < 2; ++h) w |= (isinf(v[h]) ? INF16 : (uint32_t)v[h]) << (16 * h);
      reinterpret_cast<uint32_t*>(vol)[k] = w;
    }
  }
}

void launch_import_dense(const float* dense, const uint2* meta, int W, int H, int D, int as_f32,
                         void* vol, cudaStream_t st) {
  const size_t HW = (size_t)W * H;
  k_import_dense<<<(unsigned)((HW + 127) / 128), 128, 0, st>>>(dense, meta, W, H, D, as_f32, vol);
}

// per-pixel hull [first finite d, last finite d] of a dense volume, plus
// flags: bit0 = some finite value is negative, non-integral or >= limit;
// bit1 = some pixel has no finite value; bit2 = NaN present; bit3 = +inf
// strictly inside a pixel's hull
__global__ void k_hull(const float* __restrict__ dense, int W, int H, int D, int64_t* lo,
                       int64_t* hi, unsigned int* flags, float limit) {
  const size_t pix = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= (size_t)W * H) return;
  int first = -1, last = -1, nfin = 0;
  unsigned f = 0;
  for (int d = 0; d < D; ++d) {
    const float v = dense[pix * D + d];
    if (isnan(v)) f |= 4u;
    if (isfinite(v)) {
      if (first < 0) first = d;
      last = d;
      ++nfin;
      if (v < 0.0f || v != floorf(v) || v >= limit) f |= 1u;
    }
  }
  if (first < 0) {
    f |= 2u;
    first = 0;
    last = 0;
  }
  else if (nfin != last - first + 1) {
    f |= 8u;   // +inf inside the hull: the u16 path cannot represent it
  }
  lo[pix] = first;
  hi[pix] = last;
  if (f) atomicOr(flags, f);
}

void launch_hull(const float* dense, int W, int H, int D, int64_t* lo, int64_t* hi,
                 unsigned int* flags, float limit, cudaStream_t st) {
  const size_t HW = (size_t)W * H;
  k_hull<<<(unsigned)((HW + 127) / 128), 128, 0, st>>>(dense, W, H, D, lo, hi, flags, limit);
}

}  // namespace es
