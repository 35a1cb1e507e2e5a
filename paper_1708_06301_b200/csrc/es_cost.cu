// K3: windowed SAD matching cost over the row-ragged interval layout.
//
// Reference: sgm.py:130-196 (matching_cost, _shifted_abs_diff, _box_sum) and
// tests/reference_sgm.py:24-47.  For view "left", cell (x, y, d) is
//   sum_{oy,ox} |L(cy', cx') - R(cy', clamp(cx' - d))|,
//   cy' = clamp(y + oy), cx' = clamp(x + ox)      (edge replication)
// and the border cost window^2 * 255 when x < d; "right" mirrors the match
// (other column clamp(cx' + d), border when x > W-1-d).
//
// One CTA per image row.  The window's rows are staged in shared memory as
// column words: byte k of word w of column x is row y - r + 4w + k (clamped),
// so one VABSDIFF4.U8.ACC sums four rows of one window column.  The CTA
// sweeps the row's packed u16 pairs; each thread finds its pixel by binary
// search over the row's pair offsets (also staged in shared memory), so
// stores are fully coalesced whatever the interval widths.
#include <cstdlib>

#include "es_common.cuh"
#include "es_kernels.h"

namespace es {

constexpr int COST_NT = 256;
constexpr unsigned FULL = 0xffffffffu;

template <int NW>
__global__ void __launch_bounds__(COST_NT) k_cost(CostArgs a) {
  extern __shared__ uint32_t sm[];
  const int W = a.W, H = a.H;
  const int y = blockIdx.x;
  const int svl = blockIdx.y;
  const int svg = a.view0 + svl;
  const int view = svg & 1, seq = svg >> 1;
  const int r = a.window >> 1;
  uint32_t* refcol = sm;                 // [NW][W]
  uint32_t* othcol = sm + NW * W;        // [NW][W]
  uint32_t* rowoff = sm + 2 * NW * W;    // [W]
  uint32_t* rowlh = rowoff + W;          // [W] lo | hi << 16
  const size_t HW = (size_t)W * H;
  const uint8_t* ref = a.img + ((size_t)seq * 2 + view) * HW;
  const uint8_t* oth = a.img + ((size_t)seq * 2 + (view ^ 1)) * HW;
  const uint2* meta = a.meta + (size_t)svl * HW + (size_t)y * W;
  const uint32_t rowbase = (uint32_t)(y * row_capacity(W, a.d_max));
  for (int x = threadIdx.x; x < W; x += COST_NT) {
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      uint32_t rw = 0, ow = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int row = 4 * w + k;
        if (row < a.window) {
          const int yy = clampi(y - r + row, 0, H - 1);
          rw |= (uint32_t)ref[(size_t)yy * W + x] << (8 * k);
          ow |= (uint32_t)oth[(size_t)yy * W + x] << (8 * k);
        }
      }
      refcol[w * W + x] = rw;
      othcol[w * W + x] = ow;
    }
    const uint2 m = meta[x];
    rowoff[x] = m.y - rowbase;
    rowlh[x] = m.x;
  }
  __syncthreads();
  // the row's slots up to the end of the last pixel's allocation (its
  // trailing padding slot included: padding holds +inf)
  const uint32_t last = rowlh[W - 1];
  const uint32_t row_pairs = rowoff[W - 1] - pad_before(last & 0xFFFFu) +
                             pixel_slots(last & 0xFFFFu, last >> 16);
  const uint32_t border = (uint32_t)(a.window * a.window * 255);
  uint32_t* C = a.C + (size_t)svl * a.volcap + rowbase;
  const int sign = view == 0 ? -1 : 1;
  for (uint32_t q = threadIdx.x; q < row_pairs; q += COST_NT) {
    int lo_i = 0, hi_i = W - 1;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i + 1) >> 1;
      if (rowoff[mid] <= q) lo_i = mid; else hi_i = mid - 1;
    }
    const int x = lo_i;
    const uint32_t lh = rowlh[x];
    const int lo = lh & 0xFFFF, hi = lh >> 16;
    const int j = (lo >> 1) + (int)(q - rowoff[x]);
    uint32_t out = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int d = 2 * j + h;
      uint32_t c = INF16;
      if (d >= lo && d <= hi) {
        const int xm = x + sign * d;
        if (xm < 0 || xm > W - 1) {
          c = border;
        } else {
          uint32_t sad = 0;
          for (int ox = -r; ox <= r; ++ox) {
            const int xx = clampi(x + ox, 0, W - 1);
            const int xo = clampi(xx + sign * d, 0, W - 1);
#pragma unroll
            for (int w = 0; w < NW; ++w) sad = __vsadu4(refcol[w * W + xx], othcol[w * W + xo]) + sad;
          }
          c = sad;
        }
      }
      out |= c << (16 * h);
    }
    C[q] = out;
  }
}

// Window 3, run-table schedule.  Every pixel's allocation is a whole number
// of aligned 4-pair runs (8 cells, one 16-byte word; es_common.cuh), and a
// row's allocations are consecutive, so a warp that owns 32 consecutive
// pixels owns a contiguous range of runs.  The warp scans its pixels' run
// counts, writes the owning lane of every run into a per-warp table in
// shared memory, and then lane l computes runs l, l+32, ...: stores are
// fully coalesced 16-byte words and no thread searches for its pixel.  A run
// needs the three reference columns of its pixel and ten columns of the
// other image (3 VABSDIFF4 per cell on three rows packed in bytes); runs
// that touch the image border or the interval ends take the per-cell path.
constexpr int CR_WARPS = 8;

// columns of edge replication on each side of the other image's row buffer:
// covers every match column x + ox +- d of a run (|d| <= d_max, run of 8)
__host__ __device__ inline int cost_pad_cols(int d_max) { return ((d_max + 8) & ~7) + 8; }

template <int SIGN>
__device__ __forceinline__ void cost_runs_row(const CostArgs& a, int rmax);

// byte offset of the TMA row buffers in the dynamic shared memory: after the
// packed columns (words) and the run tables (bytes), 16-byte aligned
__host__ __device__ inline size_t cost_rows_offset(int W, int padc, int rmax) {
  const size_t cols = sizeof(uint32_t) * (2 * (size_t)W + 2 * (size_t)padc);
  return (((cols + 15) & ~(size_t)15) + (size_t)CR_WARPS * 32 * rmax + 15) & ~(size_t)15;
}

__global__ void __launch_bounds__(CR_WARPS * 32) k_cost_runs(CostArgs a, int rmax) {
  // the match direction is a compile-time constant of each specialised body
  if (((a.view0 + (int)blockIdx.y) & 1) == 0) cost_runs_row<-1>(a, rmax);
  else cost_runs_row<1>(a, rmax);
}

template <int SIGN>
__device__ __forceinline__ void cost_runs_row(const CostArgs& a, int rmax) {
  extern __shared__ uint32_t sm[];
  const int W = a.W, H = a.H;
  const int y = blockIdx.x;
  const int svl = blockIdx.y;
  const int svg = a.view0 + svl;
  const int view = svg & 1, seq = svg >> 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int PADC = cost_pad_cols(a.d_max);
  uint32_t* refcol = sm;                                   // [W]
  uint32_t* othpad = sm + W;                               // [W + 2 PADC], column k at k + PADC
  uint8_t* tab = reinterpret_cast<uint8_t*>(sm + 2 * W + 2 * PADC) + wid * 32 * rmax;
  const size_t HW = (size_t)W * H;
  const uint8_t* ref = a.img + ((size_t)seq * 2 + view) * HW;
  const uint8_t* oth = a.img + ((size_t)seq * 2 + (view ^ 1)) * HW;
  const uint2* meta = a.meta + (size_t)svl * HW + (size_t)y * W;
  const uint32_t rowbase = (uint32_t)(y * row_capacity(W, a.d_max));
  const int y0 = max(y - 1, 0), y2 = min(y + 1, H - 1);
  // the metadata of the warp's first 32 pixels is requested before the image
  // rows are staged (and every later group's one iteration ahead): ncu had
  // 12% of this kernel's stall samples on the first use of a metadata word
  // loaded at the top of its own iteration
  uint2 mt_next = make_uint2(0u, 0u);
  if (wid * 32 + lane < W) mt_next = meta[wid * 32 + lane];
  if (a.tma) {
    // TMA: the three rows of both images land in shared memory as byte rows
    // by six bulk copies (16-byte-aligned supersets of the rows, one elected
    // thread, one mbarrier); the packed columns are then built on chip
    const int RS = (W + 31) & ~15;
    uint8_t* rows = reinterpret_cast<uint8_t*>(sm) + cost_rows_offset(W, PADC, rmax);
    uint64_t* bar = reinterpret_cast<uint64_t*>(rows + 6 * (size_t)RS);
    const uint8_t* src[6] = {ref + (size_t)y0 * W, ref + (size_t)y * W, ref + (size_t)y2 * W,
                             oth + (size_t)y0 * W, oth + (size_t)y * W, oth + (size_t)y2 * W};
    const unsigned bar_s = (unsigned)__cvta_generic_to_shared(bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t bytes = 0;
      for (int r = 0; r < 6; ++r) {
        const uintptr_t g = reinterpret_cast<uintptr_t>(src[r]);
        bytes += (uint32_t)((((g & 15) + W) + 15) & ~(uintptr_t)15);
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_s), "r"(bytes)
                   : "memory");
      for (int r = 0; r < 6; ++r) {
        const uintptr_t g = reinterpret_cast<uintptr_t>(src[r]);
        const uint32_t size = (uint32_t)((((g & 15) + W) + 15) & ~(uintptr_t)15);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"((unsigned)__cvta_generic_to_shared(rows + r * RS)), "l"(g & ~(uintptr_t)15),
            "r"(size), "r"(bar_s) : "memory");
      }
    }
    {
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(done) : "r"(bar_s) : "memory");
    }
    const uint8_t* rr[6];
    for (int r = 0; r < 6; ++r) rr[r] = rows + r * RS + (reinterpret_cast<uintptr_t>(src[r]) & 15);
    for (int x = threadIdx.x; x < W; x += CR_WARPS * 32)
      refcol[x] = (uint32_t)rr[0][x] | ((uint32_t)rr[1][x] << 8) | ((uint32_t)rr[2][x] << 16);
    for (int k = threadIdx.x; k < W + 2 * PADC; k += CR_WARPS * 32) {
      const int x = clampi(k - PADC, 0, W - 1);
      othpad[k] = (uint32_t)rr[3][x] | ((uint32_t)rr[4][x] << 8) | ((uint32_t)rr[5][x] << 16);
    }
  } else {
    for (int x = threadIdx.x; x < W; x += CR_WARPS * 32)
      refcol[x] = (uint32_t)ref[(size_t)y0 * W + x] | ((uint32_t)ref[(size_t)y * W + x] << 8) |
                  ((uint32_t)ref[(size_t)y2 * W + x] << 16);
    for (int k = threadIdx.x; k < W + 2 * PADC; k += CR_WARPS * 32) {
      const int x = clampi(k - PADC, 0, W - 1);
      othpad[k] = (uint32_t)oth[(size_t)y0 * W + x] | ((uint32_t)oth[(size_t)y * W + x] << 8) |
                  ((uint32_t)oth[(size_t)y2 * W + x] << 16);
    }
  }
  __syncthreads();
  const uint32_t border = 9u * 255u;
  uint4* C4 = reinterpret_cast<uint4*>(a.C + (size_t)svl * a.volcap + rowbase);
  constexpr int sign = SIGN;
  for (int gx = wid * 32; gx < W; gx += CR_WARPS * 32) {
    const int x = gx + lane;
    int lo = 0, hi = -1, nrun = 0;
    uint32_t run0 = 0;   // row-relative run index of the pixel's allocation
    const uint2 mt = mt_next;
    if (x + CR_WARPS * 32 < W) mt_next = meta[x + CR_WARPS * 32];
    if (x < W) {
      lo = (int)lo_of(mt);
      hi = (int)hi_of(mt);
      run0 = (mt.y - rowbase - pad_before(lo)) >> 2;
      nrun = (int)(pixel_slots(lo, hi) >> 2);
    }
    int incl = nrun;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const int excl = incl - nrun;
    const uint32_t grun0 = __shfl_sync(FULL, run0, 0);
    // interval ends (+inf) and off-image match centres (border cost) of one
    // pixel's run, packed for the 16-byte store
    auto finish = [&](int px, int plo, int phi, int dbase, uint32_t (&c)[8]) -> uint4 {
      const int xm_far = px + sign * (dbase + 7), xm_near = px + sign * dbase;
      const bool fix = dbase < plo || dbase + 7 > phi || xm_far < 0 || xm_far > W - 1 ||
                       xm_near < 0 || xm_near > W - 1;
      if (__any_sync(FULL, fix)) {
        // 8-bit masks over the run's cells: outside [lo, hi] (+inf wins) and
        // match centre off the image (cells above a threshold, both views)
        const int lo_c = max(plo - dbase, 0);
        const int hi_c = min(phi - dbase, 7);
        const int bt = min(max(sign < 0 ? px - dbase : W - 1 - px - dbase, -1), 7);
        const uint32_t inv = ((1u << lo_c) - 1u) | (0xFFu & (0xFFu << (hi_c + 1)));
        const uint32_t bor = 0xFFu & (0xFFu << (bt + 1));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if ((bor >> i) & 1u) c[i] = border;
          if ((inv >> i) & 1u) c[i] = INF16;
        }
      }
      return make_uint4(c[0] | (c[1] << 16), c[2] | (c[3] << 16), c[4] | (c[5] << 16),
                        c[6] | (c[7] << 16));
    };

    // ---- pairs: pixels gx+2i and gx+2i+1 over their common 8-cell blocks.
    // Cell (x, d) sums the column SADs e(x-1, d) + e(x, d) + e(x+1, d), cell
    // (x+1, d) e(x, d) + e(x+1, d) + e(x+2, d): the middle two are shared, so
    // a pair run costs 4 VABSDIFF4 per two cells instead of 6.
    const int b0 = lo >> 3, b1 = b0 + nrun - 1;       // the pixel's 8-cell blocks
    const int pb0 = __shfl_xor_sync(FULL, b0, 1), pb1 = __shfl_xor_sync(FULL, b1, 1);
    const int pnrun = __shfl_xor_sync(FULL, nrun, 1);
    const int xa = gx + (lane & ~1);
    const int cb0 = max(b0, pb0), cb1 = min(b1, pb1);
    const bool pairable = nrun > 0 && pnrun > 0 && xa >= 1 && xa + 2 <= W - 1 && cb0 <= cb1;
    const int npair = ((lane & 1) == 0 && pairable) ? cb1 - cb0 + 1 : 0;
    int pincl = npair;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, pincl, o);
      if (lane >= o) pincl += v;
    }
    const int pexcl = pincl - npair;
    const int ptotal = __shfl_sync(FULL, pincl, 31);
    for (int j = 0; j < npair; ++j) tab[pexcl + j] = (uint8_t)lane;
    __syncwarp();
    for (int r0 = 0; r0 < ptotal; r0 += 32) {
      const int r = r0 + lane;
      const bool live = r < ptotal;
      const int p = tab[live ? r : 0];                 // idle lanes: a valid pair
      const int pa_lo = __shfl_sync(FULL, lo, p), pa_hi = __shfl_sync(FULL, hi, p);
      const int pb_lo = __shfl_sync(FULL, lo, p + 1), pb_hi = __shfl_sync(FULL, hi, p + 1);
      const int pa_ex = __shfl_sync(FULL, excl, p), pb_ex = __shfl_sync(FULL, excl, p + 1);
      const int pcb0 = __shfl_sync(FULL, cb0, p), ppex = __shfl_sync(FULL, pexcl, p);
      const int blk = pcb0 + (live ? r - ppex : 0);
      const int dbase = 8 * blk;
      const int px = gx + p;
      const uint32_t r0c = refcol[px - 1], r1c = refcol[px], r2c = refcol[px + 1],
                     r3c = refcol[px + 2];
      const int cbase = sign < 0 ? px - 1 - (dbase + 7) : px - 1 + dbase;
      const uint32_t* ob = othpad + PADC + cbase;
      uint32_t o[11];
#pragma unroll
      for (int k = 0; k < 11; ++k) o[k] = ob[k];
      uint32_t ca[8], cbv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // left view: cell dbase+i of pixel x uses columns cbase + 7-i .. 9-i,
        // of pixel x+1 one column further; right view: cbase + i .. i+2
        const int k = sign < 0 ? 7 - i : i;
        const uint32_t m = __vsadu4(r2c, o[k + 2]) + __vsadu4(r1c, o[k + 1]);
        ca[i] = __vsadu4(r0c, o[k]) + m;
        cbv[i] = __vsadu4(r3c, o[k + 3]) + m;
      }
      const uint4 wa = finish(px, pa_lo, pa_hi, dbase, ca);
      const uint4 wb = finish(px + 1, pb_lo, pb_hi, dbase, cbv);
      if (live) {
        C4[grun0 + pa_ex + (blk - (pa_lo >> 3))] = wa;
        C4[grun0 + pb_ex + (blk - (pb_lo >> 3))] = wb;
      }
    }
    __syncwarp();

    // ---- single runs: every block of a pixel outside its pair's common
    // range (all of them for unpaired pixels and image-edge pixels)
    const int nl = pairable ? cb0 - b0 : nrun;           // blocks left of the common range
    const int nsing = pairable ? nrun - (cb1 - cb0 + 1) : nrun;
    int sincl = nsing;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, sincl, o);
      if (lane >= o) sincl += v;
    }
    const int sexcl = sincl - nsing;
    const int stotal = __shfl_sync(FULL, sincl, 31);
    for (int j = 0; j < nsing; ++j) tab[sexcl + j] = (uint8_t)lane;
    __syncwarp();
    for (int r0 = 0; r0 < stotal; r0 += 32) {
      const int r = r0 + lane;
      const bool live = r < stotal;
      const int p = tab[live ? r : 0];
      const int plo = __shfl_sync(FULL, lo, p);
      const int phi = __shfl_sync(FULL, hi, p);
      const int pex = __shfl_sync(FULL, excl, p);
      const int psx = __shfl_sync(FULL, sexcl, p);
      const int pnl = __shfl_sync(FULL, nl, p);
      const int pcb1 = __shfl_sync(FULL, cb1, p);
      const int j = live ? r - psx : 0;
      const int blk = j < pnl ? (plo >> 3) + j : pcb1 + 1 + (j - pnl);
      const int dbase = 8 * blk;
      const int px = gx + p;
      uint32_t c[8];
      if (px >= 1 && px <= W - 2) {
        // interior pixel: the window's columns x-1..x+1 are unclamped, so the
        // clamped match column of (ox, d) is the edge-replicated buffer entry
        // x + ox + sign*d, shared by neighbouring cells
        const uint32_t r0c = refcol[px - 1], r1c = refcol[px], r2c = refcol[px + 1];
        const int cbase = sign < 0 ? px - 1 - (dbase + 7) : px - 1 + dbase;
        const uint32_t* ob = othpad + PADC + cbase;
        uint32_t o[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) o[k] = ob[k];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int k = sign < 0 ? 7 - i : i;
          c[i] = __vsadu4(r2c, o[k + 2]) + (__vsadu4(r1c, o[k + 1]) + __vsadu4(r0c, o[k]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int d = dbase + i;
          uint32_t sad = 0;
#pragma unroll
          for (int ox = -1; ox <= 1; ++ox) {
            const int xx = clampi(px + ox, 0, W - 1);
            sad = __vsadu4(refcol[xx], othpad[PADC + clampi(xx + sign * d, 0, W - 1)]) + sad;
          }
          c[i] = sad;
        }
      }
      const uint4 wv = finish(px, plo, phi, dbase, c);
      if (live) C4[grun0 + pex + (blk - (plo >> 3))] = wv;
    }
    __syncwarp();
  }
}

void launch_cost(const CostArgs& a, int n_sv, cudaStream_t st) {
  if (a.window == 3) {
    const int rmax = (npairs_max(a.d_max) + 3) / 4;   // runs per pixel, at most
    dim3 grid(a.H, n_sv);
    size_t smem = sizeof(uint32_t) * (2 * (size_t)a.W + 2 * (size_t)cost_pad_cols(a.d_max)) +
                  (size_t)CR_WARPS * 32 * rmax;
    if (a.tma)   // 16-byte-aligned byte rows + mbarrier
      smem = cost_rows_offset(a.W, cost_pad_cols(a.d_max), rmax) + 6 * (size_t)((a.W + 31) & ~15) + 16;
    ensure_smem((const void*)k_cost_runs, smem);
    k_cost_runs<<<grid, CR_WARPS * 32, smem, st>>>(a, rmax);
    return;
  }
  const int nw = (a.window + 3) / 4;
  dim3 grid(a.H, n_sv);
  const size_t smem = sizeof(uint32_t) * ((size_t)2 * nw * a.W + 2 * (size_t)a.W);
  switch (nw) {
    case 1:
      ensure_smem((const void*)k_cost<1>, smem);
      k_cost<1><<<grid, COST_NT, smem, st>>>(a);
      break;
    case 2:
      ensure_smem((const void*)k_cost<2>, smem);
      k_cost<2><<<grid, COST_NT, smem, st>>>(a);
      break;
    default:
      ensure_smem((const void*)k_cost<3>, smem);
      k_cost<3><<<grid, COST_NT, smem, st>>>(a);
      break;
  }
}

}  // namespace es
