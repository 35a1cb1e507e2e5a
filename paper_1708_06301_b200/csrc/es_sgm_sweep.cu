// K4, fused vertical + diagonal row sweep: the three directions of one row
// sweep (down: (0,+1), (+1,+1), (-1,+1); up: (0,-1), (+1,-1), (-1,-1)) in ONE
// pass over the ragged volume: the cost words of a row are read once, the
// partial sum is read-modify-written once, and the three path states stay in
// registers.  Reference: sgm.py:199-237,257-272 (_path_step, _scan_vertical,
// aggregate_paths).
//
// Work decomposition: sheared strips.  A "strip" is NG = 32/G adjacent
// DIAGONAL chains of one view, walked by one warp over the whole sweep --
// lane group q follows the pixels x = xb + q + t of rows y = t (down) or
// y = H-1-t (up), i.e. the (+1,+1) resp. (+1,-1) path itself (state B, kept
// in place).  Each lane holds PPL = 4 u16x2 words of every 32G-cell chunk
// (absolute disparity layout of k_sgm_grp4).  In that frame the other two
// directions' predecessors are the chains one and two to the RIGHT at the
// previous step: the column path A (pred (x, y-+1)) comes from lane group
// q+1 and the anti-diagonal C (pred (x+1, y-+1)) from group q+2, both by warp
// shuffles.  Every cross-warp dependency is one-sided: a strip needs only its
// right neighbour strip's first two chains of the previous step.
//
// Schedule: one CTA per (sequence, view), 16 warps.  The view's strips are
// taken right to left in rounds of 16: in round r warp w walks strip
// 16r + w (counted from the right).  Warp w's producer is warp w-1 of the
// same round, one or two steps ahead -- hand-over through a 4-slot ring in
// shared memory and per-warp progress words (fence.cta only); warp 0's
// producer is warp 15 of the previous round, which finished that strip long
// before -- hand-over through a per-view buffer in global memory holding all
// steps (double-buffered by round parity).  Nothing waits on another CTA.
//
// Operands: the row's cost words (and partial-sum words) of the strip's NG
// pixels are one contiguous byte range of the row-ragged volume; one elected
// lane stages the next row's ranges into shared memory with cp.async.bulk
// (completion on a per-slot mbarrier) while the warp computes the current row.
//
// Arithmetic, +inf convention, chunk union and first-pixel handling are
// those of k_sgm_grp4: u16x2 words, 0x8000 = +inf,
// wrapping adds; an off-image predecessor (first row, x-1 < 0, x+1 >= W)
// holds +inf with m + P2 = -m = 0x8000, which yields L = C.
#include <cstdlib>

#include "es_common.cuh"
#include "es_kernels.h"

namespace es {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SW_PPL = 4;      // words per lane per chunk
constexpr uint32_t SW_NONE = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t sw_umask(int lo, int hi) {
  return hi < lo ? 0u : ((hi >= 31 ? 0xFFFFFFFFu : ((2u << hi) - 1u)) & ~((1u << lo) - 1u));
}

// one path update of a lane's 4 words (k_sgm_grp4's recurrence):
// L = C + min(Lp(d), min(Lp(d-1), Lp(d+1)) + P1, m + P2) - m
__device__ __forceinline__ void sw_path(const uint32_t* P, uint32_t el, uint32_t er, uint32_t mp2,
                                        uint32_t ng, uint32_t p1x2, const uint32_t* cn,
                                        uint32_t* L) {
  uint32_t X[SW_PPL + 1];
  X[0] = __byte_perm(el, P[0], 0x5432);
#pragma unroll
  for (int k = 1; k < SW_PPL; ++k) X[k] = __byte_perm(P[k - 1], P[k], 0x5432);
  X[SW_PPL] = __byte_perm(P[SW_PPL - 1], er, 0x5432);
#pragma unroll
  for (int k = 0; k < SW_PPL; ++k) {
    const uint32_t cand = __viaddmin_u16x2(__vminu2(X[k], X[k + 1]), p1x2, __vminu2(P[k], mp2));
    L[k] = __vadd2(cn[k], __vadd2(cand, ng));
  }
}

template <int G, int NCH>
struct SW {
  static constexpr int NG = 32 / G;             // chains per strip
  static constexpr int CW = SW_PPL * G;         // words per chunk
  static constexpr int NW = SW_PPL * NCH;       // state words per lane
  static constexpr int BUFW = NG * NCH * CW;    // staged words per step (upper bound)
  static constexpr int REC = 3 * G * NW + 8;    // hand-over record: A0, C0, C1 + 6 splats
};
#ifndef SW_CTA_WARPS
#define SW_CTA_WARPS 16
#endif
constexpr int SW_WARPS = SW_CTA_WARPS;   // warps per CTA = strips per round
#ifndef SW_RS_SLOTS
#define SW_RS_SLOTS 2
#endif
// shared-memory ring slots per warp pair (2 measured best: the staging
// buffers and rings share the SM's 256 KB with the L1 that serves the
// metadata loads; 8 slots cost 3 ms per step)
constexpr int SW_RS = SW_RS_SLOTS;

static_assert((SW_RS & (SW_RS - 1)) == 0, "ring slots: a power of two");
constexpr int SW_LRS = SW_RS == 1 ? 0 : (SW_RS == 2 ? 1 : (SW_RS == 4 ? 2 : 3));

// dynamic shared memory, in 32-bit words: per-warp operand staging
// [2 slots][cost, sum][BUFW], the per-warp staging mbarriers (2 each), the
// hand-over mbarriers (full, empty) of every ring slot of the SW_WARPS - 1
// warp pairs, the rings [pair][slot][REC], the progress words and one +inf
// record
template <int G, int NCH>
struct SwLayout {
  using T = SW<G, NCH>;
  static constexpr size_t bars = (size_t)SW_WARPS * 4 * T::BUFW;
  static constexpr size_t hbar = bars + SW_WARPS * 4;
  static constexpr size_t rings = (hbar + (size_t)(SW_WARPS - 1) * SW_RS * 4 + 3) & ~(size_t)3;
  static constexpr size_t progs = rings + (size_t)(SW_WARPS - 1) * SW_RS * T::REC;
  static constexpr size_t inf = progs + ((SW_WARPS + 3) & ~3);
  // warp 0's records from the last warp of the previous round, staged from
  // the global buffer by TMA one step ahead: [2][REC] + 2 mbarriers
  static constexpr size_t head = inf + T::REC;
  static constexpr size_t headbar = head + 2 * (size_t)T::REC;
  static constexpr size_t words = headbar + 4;
};

template <int G, int NCH>
constexpr size_t sweep_smem() {
  return sizeof(uint32_t) * SwLayout<G, NCH>::words;
}

__device__ __forceinline__ void spin_ge(const volatile int* p, int v) {
  while (*p < v) __nanosleep(8);
}

// predicated vector accesses (no branch, registers keep their value when the
// predicate is off): the hand-over records enter / leave through lanes of
// chains 0 and 1 only
__device__ __forceinline__ void lds4_if(bool p, unsigned a, uint32_t* r) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n\t}\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]) : "r"(a), "r"((int)p) : "memory");
}
__device__ __forceinline__ void lds2_if(bool p, unsigned a, uint32_t& x, uint32_t& y) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.shared.v2.u32 {%0, %1}, [%2];\n\t}\n"
               : "+r"(x), "+r"(y) : "r"(a), "r"((int)p) : "memory");
}
__device__ __forceinline__ void sts4_if(bool p, unsigned a, uint32_t x, uint32_t y, uint32_t z, uint32_t u) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t}\n"
               :: "r"(a), "r"(x), "r"(y), "r"(z), "r"(u), "r"((int)p) : "memory");
}
__device__ __forceinline__ void sts2_if(bool p, unsigned a, uint32_t x, uint32_t y) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.shared.v2.u32 [%0], {%1, %2};\n\t}\n"
               :: "r"(a), "r"(x), "r"(y), "r"((int)p) : "memory");
}
__device__ __forceinline__ void stg4_if(bool p, uint32_t* a, uint32_t x, uint32_t y, uint32_t z, uint32_t u) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.v4.u32 [%0], {%1, %2, %3, %4};\n\t}\n"
               :: "l"(a), "r"(x), "r"(y), "r"(z), "r"(u), "r"((int)p) : "memory");
}
__device__ __forceinline__ void stg2_if(bool p, uint32_t* a, uint32_t x, uint32_t y) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.v2.u32 [%0], {%1, %2};\n\t}\n"
               :: "l"(a), "r"(x), "r"(y), "r"((int)p) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned b, unsigned parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(done) : "r"(b), "r"(parity) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}

template <int G, int NCH, bool INIT>
#ifdef SW_MAXREG
__global__ void __maxnreg__(SW_MAXREG) k_sgm_sweep(SweepArgs v) {
#else
__global__ void __launch_bounds__(SW_WARPS * 32, 1) k_sgm_sweep(SweepArgs v) {
#endif
  using T = SW<G, NCH>;
  constexpr int NG = T::NG, CW = T::CW, NW = T::NW, PPL = SW_PPL, REC = T::REC;
  constexpr int BUFW = T::BUFW;
  extern __shared__ __align__(16) uint32_t sm5[];
  // pipeline position of the warp: the schedulers pick the highest warp id
  // first, so the chain head (position 0, free-running) is the highest warp
  const int lane = threadIdx.x & 31;
#ifdef SW_FWD_ORDER
  const int w = threadIdx.x >> 5;
#else
  const int w = SW_WARPS - 1 - (int)(threadIdx.x >> 5);
#endif
  const int gl = lane & (G - 1), q = lane / G;
  const int gbase = lane & ~(G - 1);
  const int src_l = gbase | ((gl + G - 1) & (G - 1));
  const int src_r = gbase | ((gl + 1) & (G - 1));
  using LY = SwLayout<G, NCH>;
  uint32_t* buf = sm5 + w * (4 * BUFW);   // [2 slots][cost, sum][BUFW]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm5 + LY::bars) + 2 * w;
  volatile int* progs = reinterpret_cast<volatile int*>(sm5 + LY::progs);
  // a whole hand-over record of +inf (states and splats): read instead of the
  // producer's record where its pixel is off the image; its first 4 words
  // also pad cost reads outside a pixel's interval
  uint32_t* infpad = sm5 + LY::inf;
  const unsigned sm_s = (unsigned)__cvta_generic_to_shared(sm5);
  const unsigned inf_s = sm_s + 4u * (unsigned)LY::inf;
  // ring of warp pair (p, p+1) slot s at ring_s + 4 * (p * RS + s) * REC;
  // its full / empty mbarriers at hbar_s + 16 * (p * RS + s) (+ 8)
  const unsigned ring_s = sm_s + 4u * (unsigned)LY::rings;
  const unsigned hbar_s = sm_s + 4u * (unsigned)LY::hbar;
  const unsigned head_s = sm_s + 4u * (unsigned)LY::head;
  const unsigned headbar_s = sm_s + 4u * (unsigned)LY::headbar;

  const SgmArgs& a = v.a;
  const int W = a.W, H = a.H;
  const int sv = blockIdx.x;
  const int ns = v.nstrips;
  const bool up = v.up != 0;
  const size_t HW = (size_t)W * H;
  const uint2* __restrict__ meta = a.meta + (size_t)sv * HW;
  const uint32_t* Cg = reinterpret_cast<const uint32_t*>(a.C) + (size_t)sv * a.volcap;
  uint32_t* Sg = reinterpret_cast<uint32_t*>(a.S) + (size_t)sv * a.volcap;
  // [round parity][step][REC] records, then one +inf record
  uint32_t* gbuf = v.ring + (size_t)sv * (2 * (size_t)H + 1) * REC;
  uint32_t* ginf = gbuf + 2 * (size_t)H * REC;
  const uint32_t p1x2 = a.p1i * 0x10001u;

  const unsigned bar0 = (unsigned)__cvta_generic_to_shared(bars);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < (SW_WARPS - 1) * SW_RS) {
    // all 32 lanes of the writing (reading) warp arrive: each lane's own
    // predicated stores (loads) are released by its own arrive
    const unsigned b = hbar_s + 16u * threadIdx.x;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(b) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;" ::"r"(b + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 2) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(headbar_s + 8u * threadIdx.x) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < SW_WARPS) progs[threadIdx.x] = 0;
  for (int i = threadIdx.x; i < REC; i += blockDim.x) {
    infpad[i] = INF16x2;
    ginf[i] = INF16x2;
  }
  __syncthreads();

  auto in_img = [&](int x) { return x >= 0 && x < W; };
  auto wait_slot = [&](int slot, unsigned parity) {
    const unsigned b = bar0 + 8u * (unsigned)slot;
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(b), "r"(parity) : "memory");
  };
  auto publish = [&](int value) {
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      progs[w] = value;
    }
  };

  int it_all = 0;   // steps walked by this warp (mbarrier slot / phase)
  int nr = 0, nw = 0;   // hand-over records read from / written to the shared rings
  int nh = 0, nhr = 0;  // warp 0: global records staged / consumed
  int head_seen = -1;   // warp 0, lane 0: last progress value read from the last warp
  const int rounds = (ns + SW_WARPS - 1) / SW_WARPS;
  for (int r = 0; r < rounds; ++r) {
#ifdef SW_ROUND_BARRIER
    // every warp has finished round r-1: the shared ring slots and the
    // global buffer of round r-2's parity are free again
    __syncthreads();
#endif
    const int kk = r * SW_WARPS + w;
    if (kk >= ns) continue;
    const int k = ns - 1 - kk;
    const int xb0 = -(H - 1) + k * NG;                 // chain of lane group 0 (x at step 0)
    const int t0 = max(0, -(xb0 + NG - 1)), t1 = min(H - 1, W - 1 - xb0);
    const int xbc = xb0 - NG;                          // consumer strip (kk + 1)
    const int t0c = max(0, -(xbc + NG - 1)), t1c = min(H - 1, W - 1 - xbc);
    const bool has_prod = kk > 0, has_cons = kk + 1 < ns;
    const int xbp = xb0 + NG;                          // producer strip (kk - 1)
    const int t0p = max(0, -(xbp + NG - 1)), t1p = min(H - 1, W - 1 - xbp);
    const int pbase = (r - 1) * 65536;                 // global producer: last warp, round r-1
    const int rbase = r * 65536;
    if (t0 > t1) {
      publish(rbase + H);
      continue;
    }
    // hand-over records: between warps of a round through the shared ring of
    // the warp pair (full / empty mbarriers, records numbered per pair across
    // rounds), from the last warp to warp 0 of the next round through a
    // per-view global buffer (progress words; one record per step, double-
    // buffered by round parity)
    const uint32_t* prod_gl = gbuf + (size_t)((r - 1) & 1) * H * REC;
    uint32_t* own_gl = gbuf + (size_t)(r & 1) * H * REC;
    if (r > 0 && has_cons && w == SW_WARPS - 1) {
      // the global buffer of this round's parity was read by warp 0 in round
      // r-1, which publishes rbase + H when done
      if (lane == 0) {
        spin_ge(progs + 0, (r - 1) * 65536 + H);
        __threadfence_block();
      }
      __syncwarp();
    }

#ifdef SW_META_SLOW
    auto load_meta = [&](int t) -> uint2 {
      const int x = xb0 + q + t;
      if (t <= t1 && in_img(x)) return meta[(size_t)(up ? H - 1 - t : t) * W + x];
      return make_uint2(SW_NONE, 0u);
    };
#else
    // the lane's chain pixel at step t is meta_q[t * mstride] for t in
    // [mlo, mhi] (x = xb0 + q + t inside the image, t <= t1): one multiply-
    // add and a range test per step
    const int mstride = up ? 1 - W : 1 + W;
    const uint2* meta_q = meta + (up ? (ptrdiff_t)(H - 1) * W : 0) + (xb0 + q);
    const int mlo = max(0, -(xb0 + q)), mhi = min(t1, W - 1 - xb0 - q);
    auto load_meta = [&](int t) -> uint2 {
      if (t >= mlo && t <= mhi) return meta_q[(ptrdiff_t)t * mstride];
      return make_uint2(SW_NONE, 0u);
    };
#endif
    auto issue = [&](uint2 mt, int slot) -> uint32_t {
      __syncwarp();   // every lane is done reading this slot (two steps ago)
      uint32_t st = 0xFFFFFFFFu, en = 0u;
      if (mt.x != SW_NONE) {
        const int lo = (int)(mt.x & 0xFFFFu), hi = (int)(mt.x >> 16);
        st = mt.y - pad_before(lo);
        en = st + pixel_slots(lo, hi);
      }
      st = __reduce_min_sync(FULL, st);
      en = __reduce_max_sync(FULL, en);
      if (lane == 0) {
        const uint32_t bytes = (en - st) * 4u;
        const unsigned b = bar0 + 8u * (unsigned)slot;
        uint32_t* dst = buf + slot * 2 * BUFW;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     ::"r"(b), "r"(INIT ? bytes : 2u * bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(Cg + st), "r"(bytes), "r"(b)
                     : "memory");
        if (!INIT)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"((unsigned)__cvta_generic_to_shared(dst + BUFW)), "l"(Sg + st), "r"(bytes),
                       "r"(b) : "memory");
      }
      return st;
    };

    uint32_t A[NW], B[NW], Cs[NW];
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) A[ww] = B[ww] = Cs[ww] = INF16x2;
    uint32_t a_p2 = INF16x2, a_ng = INF16x2, b_p2 = INF16x2, b_ng = INF16x2, c_p2 = INF16x2,
             c_ng = INF16x2;
    // warp 0: stage the global record of step tr (read at step tr + 1) into
    // shared memory; the last warp of round r-1 wrote it long before
    auto stage_head = [&](int tr) {
      if (lane == 0) {
        // the producer runs ~360 steps ahead: its progress word is read (and
        // the fences paid) only when the last value seen does not cover tr
        if (head_seen < pbase + tr + 1) {
          do {
            head_seen = progs[SW_WARPS - 1];
            if (head_seen < pbase + tr + 1) __nanosleep(8);
          } while (head_seen < pbase + tr + 1);
          __threadfence_block();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const unsigned b = headbar_s + 8u * (unsigned)(nh & 1);
        const unsigned dst = head_s + 4u * (unsigned)((nh & 1) * REC);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4u * REC)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(prod_gl + (size_t)tr * REC), "r"(4u * REC), "r"(b) : "memory");
      }
      ++nh;
    };
    if (w == 0 && has_prod && t0 >= 1 && t0 - 1 >= t0p && t0 - 1 <= t1p) stage_head(t0 - 1);

    uint2 m0 = load_meta(t0), m1 = load_meta(t0 + 1);
    uint32_t org = issue(m0, it_all & 1);
    uint32_t pm = 0u;   // chunks computed at the previous step (warp-uniform)

    for (int t = t0; t <= t1; ++t, ++it_all) {
      const int slot = it_all & 1;
      const uint2 mt = m0;
      const uint2 m2 = load_meta(t + 2);
      uint32_t org_next = 0;
      if (t + 1 <= t1) org_next = issue(m1, slot ^ 1);

      // ---- inputs: A from chain q+1, C from chain q+2 (previous step).  The
      // producer strip's chains 0 and 1 at step t-1 enter through this
      // strip's lanes of chains 0 and 1 (whose own states were handed on at
      // step t-1): predicated loads of the hand-over record, then one
      // rotation by G (A) and 2G (C) lanes.
      const bool need0 = has_prod && t >= 1 && in_img(xb0 + NG + t - 1);
      const bool need1 = has_prod && t >= 1 && in_img(xb0 + NG + t);
      const bool fed = need0 || need1;
      const bool rec_in = has_prod && t - 1 >= t0p && t - 1 <= t1p;
      const bool okq = q == 0 ? need0 : need1;   // lanes of chain 0: A0, C0; chain 1: C1
      if (w > 0) {
        unsigned rec = inf_s, ebar = 0;
        if (rec_in) {
          const int n = nr++;
          const unsigned slot_i = (unsigned)((w - 1) * SW_RS + (n & (SW_RS - 1)));
          mb_wait(hbar_s + 16u * slot_i, (unsigned)(n >> SW_LRS) & 1u);
          rec = ring_s + 4u * slot_i * (unsigned)REC;
          ebar = hbar_s + 16u * slot_i + 8u;
        }
        const unsigned ra = (need0 ? rec : inf_s) + 4u * (unsigned)(gl * NW);
        const unsigned rc = (okq ? rec : inf_s) + 4u * (unsigned)((1 + q) * G * NW + gl * NW);
#pragma unroll
        for (int ww = 0; ww < NW; ww += 4) {
          lds4_if(q == 0, ra + 4u * ww, &A[ww]);
          lds4_if(q < 2, rc + 4u * ww, &Cs[ww]);
        }
        lds2_if(q == 0, (need0 ? rec : inf_s) + 4u * (3 * G * NW), a_p2, a_ng);
        lds2_if(q < 2, (okq ? rec : inf_s) + 4u * (3 * G * NW + 2 + 2 * q), c_p2, c_ng);
        if (rec_in) mb_arrive(ebar);
      } else {
        unsigned rec = inf_s;
        if (rec_in) {
          const int n = nhr++;
          mb_wait(headbar_s + 8u * (unsigned)(n & 1), (unsigned)(n >> 1) & 1u);
          rec = head_s + 4u * (unsigned)((n & 1) * REC);
        }
        const unsigned ra = (need0 ? rec : inf_s) + 4u * (unsigned)(gl * NW);
        const unsigned rc = (okq ? rec : inf_s) + 4u * (unsigned)((1 + q) * G * NW + gl * NW);
#pragma unroll
        for (int ww = 0; ww < NW; ww += 4) {
          lds4_if(q == 0, ra + 4u * ww, &A[ww]);
          lds4_if(q < 2, rc + 4u * ww, &Cs[ww]);
        }
        lds2_if(q == 0, (need0 ? rec : inf_s) + 4u * (3 * G * NW), a_p2, a_ng);
        lds2_if(q < 2, (okq ? rec : inf_s) + 4u * (3 * G * NW + 2 + 2 * q), c_p2, c_ng);
        // every lane has read the slot before it is staged again (next step)
        __syncwarp();
        if (has_prod && t + 1 <= t1 && t >= t0p && t <= t1p) stage_head(t);
      }
      const int srcA = (lane + G) & 31, srcC = (lane + 2 * G) & 31;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) {
        A[ww] = __shfl_sync(FULL, A[ww], srcA);
        Cs[ww] = __shfl_sync(FULL, Cs[ww], srcC);
      }
      const uint32_t ap2 = __shfl_sync(FULL, a_p2, srcA), ang = __shfl_sync(FULL, a_ng, srcA);
      const uint32_t cp2 = __shfl_sync(FULL, c_p2, srcC), cng = __shfl_sync(FULL, c_ng, srcC);

      // ---- this step's pixel of the lane's chain
      int base = 0, relb = 0, clo = NCH, chi = -1;
      uint32_t spanp = 0u;
      if (mt.x != SW_NONE) {
        const int j0 = (int)((mt.x & 0xFFFFu) >> 1), j1 = (int)((mt.x >> 16) >> 1);
        base = (int)(mt.y - (uint32_t)j0 - org) + PPL * gl;
        relb = PPL * gl - j0 + PPL - 1;
        spanp = (uint32_t)(j1 - j0 + PPL);
        clo = j0 / CW;
        chi = j1 / CW;
      }
      const uint32_t um = sw_umask(__reduce_min_sync(FULL, clo), __reduce_max_sync(FULL, chi));
      wait_slot(slot, (unsigned)((it_all >> 1) & 1));
      const uint32_t* cb = buf + slot * 2 * BUFW;
      const uint32_t* sb = cb + BUFW;
      uint32_t* Srow = Sg + org;

      uint32_t nA = INF16x2, nB = INF16x2, nC = INF16x2;
      uint32_t lA = INF16x2, lB = INF16x2, lC = INF16x2;   // previous chunk's last word (old)
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        uint32_t PA[PPL], PB[PPL], PC[PPL];
#pragma unroll
        for (int kk2 = 0; kk2 < PPL; ++kk2) {
          PA[kk2] = A[c * PPL + kk2];
          PB[kk2] = B[c * PPL + kk2];
          PC[kk2] = Cs[c * PPL + kk2];
        }
        if ((um >> c) & 1u) {
          const int CN = c + 1 < NCH ? c + 1 : 0;
          const uint32_t rA = gl == 0 ? (c + 1 < NCH ? A[CN * PPL] : INF16x2) : PA[0];
          const uint32_t rB = gl == 0 ? (c + 1 < NCH ? B[CN * PPL] : INF16x2) : PB[0];
          const uint32_t rC = gl == 0 ? (c + 1 < NCH ? Cs[CN * PPL] : INF16x2) : PC[0];
          const uint32_t elA = __shfl_sync(FULL, gl == G - 1 ? lA : PA[PPL - 1], src_l);
          const uint32_t elB = __shfl_sync(FULL, gl == G - 1 ? lB : PB[PPL - 1], src_l);
          const uint32_t elC = __shfl_sync(FULL, gl == G - 1 ? lC : PC[PPL - 1], src_l);
          const uint32_t erA = __shfl_sync(FULL, rA, src_r);
          const uint32_t erB = __shfl_sync(FULL, rB, src_r);
          const uint32_t erC = __shfl_sync(FULL, rC, src_r);
          const bool p = (uint32_t)(relb + c * CW) < spanp;
          // words outside the pixel's interval read the INF pad
          const uint4 u = *reinterpret_cast<const uint4*>(p ? cb + base + c * CW : infpad);
          const uint32_t cn[PPL] = {u.x, u.y, u.z, u.w};
          uint32_t LA[PPL], LB[PPL], LC[PPL];
          sw_path(PA, elA, erA, ap2, ang, p1x2, cn, LA);
          sw_path(PB, elB, erB, b_p2, b_ng, p1x2, cn, LB);
          sw_path(PC, elC, erC, cp2, cng, p1x2, cn, LC);
#pragma unroll
          for (int kk2 = 0; kk2 < PPL; ++kk2) {
            A[c * PPL + kk2] = LA[kk2];
            B[c * PPL + kk2] = LB[kk2];
            Cs[c * PPL + kk2] = LC[kk2];
          }
          nA = __vimin3_u16x2(nA, __vminu2(LA[0], LA[1]), __vminu2(LA[2], LA[3]));
          nB = __vimin3_u16x2(nB, __vminu2(LB[0], LB[1]), __vminu2(LB[2], LB[3]));
          nC = __vimin3_u16x2(nC, __vminu2(LC[0], LC[1]), __vminu2(LC[2], LC[3]));
        }
        lA = PA[PPL - 1];
        lB = PB[PPL - 1];
        lC = PC[PPL - 1];
      }
      // chunks outside this step's union must hold +inf; only those computed
      // at the previous step, or refilled from the hand-over record, can hold
      // anything else (warp-uniform test, no per-chunk default moves)
      const uint32_t clr = ~um & (pm | (fed ? 0xFFFFFFFFu : 0u));
#pragma unroll
      for (int c = 0; c < NCH; ++c)
        if ((clr >> c) & 1u) {
#pragma unroll
          for (int kk2 = 0; kk2 < PPL; ++kk2)
            A[c * PPL + kk2] = B[c * PPL + kk2] = Cs[c * PPL + kk2] = INF16x2;
        }
      pm = um;
      uint32_t hA = min(nA & 0xFFFFu, nA >> 16), hB = min(nB & 0xFFFFu, nB >> 16),
               hC = min(nC & 0xFFFFu, nC >> 16);
#pragma unroll
      for (int o = G / 2; o; o >>= 1) {
        hA = min(hA, __shfl_xor_sync(FULL, hA, o));
        hB = min(hB, __shfl_xor_sync(FULL, hB, o));
        hC = min(hC, __shfl_xor_sync(FULL, hC, o));
      }
      const bool act = spanp != 0u;
      a_p2 = act ? (hA + a.p2i) * 0x10001u : INF16x2;
      a_ng = act ? ((0x10000u - hA) & 0xFFFFu) * 0x10001u : INF16x2;
      b_p2 = act ? (hB + a.p2i) * 0x10001u : INF16x2;
      b_ng = act ? ((0x10000u - hB) & 0xFFFFu) * 0x10001u : INF16x2;
      c_p2 = act ? (hC + a.p2i) * 0x10001u : INF16x2;
      c_ng = act ? ((0x10000u - hC) & 0xFFFFu) * 0x10001u : INF16x2;

      // ---- hand chains 0 and 1 to the consumer strip (it reads step t at
      // its step t + 1): predicated stores by the lanes of chains 0 and 1
      if (has_cons && t + 1 <= t1c && t + 1 >= t0c) {
        if (w < SW_WARPS - 1) {
          const int n = nw++;
          const unsigned slot_i = (unsigned)(w * SW_RS + (n & (SW_RS - 1)));
          // the slot's previous record (n - RS) has been read
          mb_wait(hbar_s + 16u * slot_i + 8u, ((unsigned)(n >> SW_LRS) & 1u) ^ 1u);
          const unsigned rec = ring_s + 4u * slot_i * (unsigned)REC;
          const unsigned wa = rec + 4u * (unsigned)(gl * NW);
          const unsigned wc = rec + 4u * (unsigned)((1 + q) * G * NW + gl * NW);
#pragma unroll
          for (int ww = 0; ww < NW; ww += 4) {
            sts4_if(q == 0, wa + 4u * ww, A[ww], A[ww + 1], A[ww + 2], A[ww + 3]);
            sts4_if(q < 2, wc + 4u * ww, Cs[ww], Cs[ww + 1], Cs[ww + 2], Cs[ww + 3]);
          }
          sts4_if(q == 0 && gl == 0, rec + 4u * (3 * G * NW), a_p2, a_ng, c_p2, c_ng);
          sts2_if(q == 1 && gl == 0, rec + 4u * (3 * G * NW + 4), c_p2, c_ng);
          mb_arrive(hbar_s + 16u * slot_i);
        } else {
          uint32_t* rec = own_gl + (size_t)t * REC;
          uint32_t* wa = rec + gl * NW;
          uint32_t* wc = rec + (1 + q) * G * NW + gl * NW;
#pragma unroll
          for (int ww = 0; ww < NW; ww += 4) {
            stg4_if(q == 0, wa + ww, A[ww], A[ww + 1], A[ww + 2], A[ww + 3]);
            stg4_if(q < 2, wc + ww, Cs[ww], Cs[ww + 1], Cs[ww + 2], Cs[ww + 3]);
          }
          stg4_if(q == 0 && gl == 0, rec + 3 * G * NW, a_p2, a_ng, c_p2, c_ng);
          stg2_if(q == 1 && gl == 0, rec + 3 * G * NW + 4, c_p2, c_ng);
        }
      }
      // the consumer of the global records (warp 0 of the next round) is
      // hundreds of steps behind: progress is published every 16th step and
      // at the end of the round
      if (w == SW_WARPS - 1 && (t & 15) == 15) publish(rbase + t + 1);
      // ---- partial sums of the step's three directions
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (((um >> c) & 1u) && (uint32_t)(relb + c * CW) < spanp) {
          uint32_t Sx[PPL];
#pragma unroll
          for (int kk2 = 0; kk2 < PPL; ++kk2)
            Sx[kk2] = __vadd2(A[c * PPL + kk2], __vadd2(B[c * PPL + kk2], Cs[c * PPL + kk2]));
          if (!INIT) {
            const uint4 w4 = *reinterpret_cast<const uint4*>(sb + base + c * CW);
            Sx[0] = __vadd2(w4.x, Sx[0]);
            Sx[1] = __vadd2(w4.y, Sx[1]);
            Sx[2] = __vadd2(w4.z, Sx[2]);
            Sx[3] = __vadd2(w4.w, Sx[3]);
          }
          *reinterpret_cast<uint4*>(Srow + base + c * CW) = make_uint4(Sx[0], Sx[1], Sx[2], Sx[3]);
        }
      }
      m0 = m1;
      m1 = m2;
      org = org_next;
    }
    publish(rbase + H);
  }
}

template <int G, int NCH>
void launch_sweep_t(const SweepArgs& v, bool init, int n_sv, cudaStream_t st) {
  const size_t smem = sweep_smem<G, NCH>();
  auto k = init ? k_sgm_sweep<G, NCH, true> : k_sgm_sweep<G, NCH, false>;
  ensure_smem((const void*)k, smem);
  k<<<n_sv, SW_WARPS * 32, smem, st>>>(v);
}

}  // namespace

int sweep_lanes(int d_max) {
  const int np = npairs_max(d_max);
  return np <= 64 ? 4 : (np <= 128 ? 8 : 0);
}

int sweep_strips(int W, int d_max, int H) {
  const int G = sweep_lanes(d_max);
  const int NG = G ? 32 / G : 1;
  return G ? (W + H - 1 + NG - 1) / NG : 0;
}

size_t sweep_ring_words(int W, int d_max, int H) {
  const int G = sweep_lanes(d_max);
  if (!G) return 0;
  // two round parities x H steps + one +inf record, REC = 3 * G * NW + 8
  // words (NW = 16 at most)
  (void)W;
  return (size_t)(2 * H + 1) * (3 * G * 16 + 8);
}

void launch_sweep(const SweepArgs& v, bool init, cudaStream_t st) {
  const int np = npairs_max(v.a.d_max);
  const int n_sv = v.total / v.nstrips;
  if (np <= 16) launch_sweep_t<4, 1>(v, init, n_sv, st);
  else if (np <= 32) launch_sweep_t<4, 2>(v, init, n_sv, st);
  else if (np <= 64) launch_sweep_t<4, 4>(v, init, n_sv, st);
  else launch_sweep_t<8, 4>(v, init, n_sv, st);
}

}  // namespace es
