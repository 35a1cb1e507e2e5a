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

// Runs of COST_R consecutive pairs per thread: one binary search per run,
// pixel state carried across pairs, and for window 3 a clamp-free fast path
// (interior match columns) where the pair's two cells share four columns of
// the other image: 4 LDS + 6 VABSDIFF4 per pair.
constexpr int COST_R = 4;

__global__ void __launch_bounds__(COST_NT) k_cost_w3(CostArgs a) {
  extern __shared__ uint32_t sm[];
  const int W = a.W, H = a.H;
  const int y = blockIdx.x;
  const int svl = blockIdx.y;
  const int svg = a.view0 + svl;
  const int view = svg & 1, seq = svg >> 1;
  uint32_t* refcol = sm;            // [W]
  uint32_t* othcol = sm + W;        // [W]
  uint32_t* rowoff = sm + 2 * W;    // [W + 1]
  uint32_t* rowlh = sm + 3 * W + 1; // [W]
  const size_t HW = (size_t)W * H;
  const uint8_t* ref = a.img + ((size_t)seq * 2 + view) * HW;
  const uint8_t* oth = a.img + ((size_t)seq * 2 + (view ^ 1)) * HW;
  const uint2* meta = a.meta + (size_t)svl * HW + (size_t)y * W;
  const uint32_t rowbase = (uint32_t)(y * row_capacity(W, a.d_max));
  const int y0 = max(y - 1, 0), y2 = min(y + 1, H - 1);
  for (int x = threadIdx.x; x < W; x += COST_NT) {
    refcol[x] = (uint32_t)ref[(size_t)y0 * W + x] | ((uint32_t)ref[(size_t)y * W + x] << 8) |
                ((uint32_t)ref[(size_t)y2 * W + x] << 16);
    othcol[x] = (uint32_t)oth[(size_t)y0 * W + x] | ((uint32_t)oth[(size_t)y * W + x] << 8) |
                ((uint32_t)oth[(size_t)y2 * W + x] << 16);
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
  if (threadIdx.x == 0) rowoff[W] = row_pairs;
  __syncthreads();
  const uint32_t border = 9u * 255u;
  uint32_t* C = a.C + (size_t)svl * a.volcap + rowbase;
  const int sign = view == 0 ? -1 : 1;
  for (uint32_t q0 = threadIdx.x * COST_R; q0 < row_pairs; q0 += COST_NT * COST_R) {
    int lo_i = 0, hi_i = W - 1;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i + 1) >> 1;
      if (rowoff[mid] <= q0) lo_i = mid; else hi_i = mid - 1;
    }
    int x = lo_i;
    uint32_t beg = rowoff[x], end = rowoff[x + 1];
    uint32_t lh = rowlh[x];
    uint32_t r0 = refcol[max(x - 1, 0)], r1 = refcol[x], r2 = refcol[min(x + 1, W - 1)];
    uint32_t out[COST_R];
#pragma unroll
    for (int r = 0; r < COST_R; ++r) {
      const uint32_t q = q0 + r;
      out[r] = INF16x2;
      if (q >= row_pairs) continue;
      if (q >= end) {   // next pixel (every pixel owns >= 1 pair)
        ++x;
        beg = end;
        end = rowoff[x + 1];
        lh = rowlh[x];
        r0 = refcol[max(x - 1, 0)];
        r1 = refcol[x];
        r2 = refcol[min(x + 1, W - 1)];
      }
      const int lo = lh & 0xFFFF, hi = lh >> 16;
      const int d0 = 2 * ((lo >> 1) + (int)(q - beg));
      // match columns of the two cells: x + ox + sign*d, ox in {-1,0,1},
      // d in {d0, d0+1}; interior when all four lie inside the image
      const int cmin = sign < 0 ? x - 1 - (d0 + 1) : x - 1 + d0;
      const int cmax = sign < 0 ? x + 1 - d0 : x + 1 + d0 + 1;
      uint32_t c0, c1;
      if (x >= 1 && x <= W - 2 && cmin >= 0 && cmax <= W - 1) {
        // left view: cell d uses columns x-1-d .. x+1-d; cell d+1 one to the left
        const int b = sign < 0 ? x - 2 - d0 : x - 1 + d0;   // lowest of the 4 columns
        const uint32_t o0 = othcol[b], o1 = othcol[b + 1], o2 = othcol[b + 2], o3 = othcol[b + 3];
        if (sign < 0) {
          c0 = __vsadu4(r0, o1) + __vsadu4(r1, o2) + __vsadu4(r2, o3);
          c1 = __vsadu4(r0, o0) + __vsadu4(r1, o1) + __vsadu4(r2, o2);
        } else {
          c0 = __vsadu4(r0, o0) + __vsadu4(r1, o1) + __vsadu4(r2, o2);
          c1 = __vsadu4(r0, o1) + __vsadu4(r1, o2) + __vsadu4(r2, o3);
        }
      } else {
        uint32_t cc[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int d = d0 + h;
          const int xm = x + sign * d;
          if (xm < 0 || xm > W - 1) {
            cc[h] = border;
          } else {
            uint32_t sad = 0;
#pragma unroll
            for (int ox = -1; ox <= 1; ++ox) {
              const int xx = clampi(x + ox, 0, W - 1);
              sad = __vsadu4(refcol[xx], othcol[clampi(xx + sign * d, 0, W - 1)]) + sad;
            }
            cc[h] = sad;
          }
        }
        c0 = cc[0];
        c1 = cc[1];
      }
      // off-image centres take the border cost; cells outside [lo, hi] are +inf
      if ((unsigned)(x + sign * d0) > (unsigned)(W - 1)) c0 = border;
      if ((unsigned)(x + sign * (d0 + 1)) > (unsigned)(W - 1)) c1 = border;
      // (padding slots lie wholly outside [lo, hi])
      if (d0 < lo || d0 > hi) c0 = INF16;
      if (d0 + 1 < lo || d0 + 1 > hi) c1 = INF16;
      out[r] = c0 | (c1 << 16);
    }
    if (q0 + COST_R <= row_pairs && ((rowbase + q0) & 3u) == 0 && ((a.volcap * svl) & 3u) == 0) {
      *reinterpret_cast<uint4*>(C + q0) = make_uint4(out[0], out[1], out[2], out[3]);
    } else {
#pragma unroll
      for (int r = 0; r < COST_R; ++r)
        if (q0 + r < row_pairs) C[q0 + r] = out[r];
    }
  }
}

void launch_cost(const CostArgs& a, int n_sv, cudaStream_t st) {
  if (a.window == 3 && getenv("ES_COST_V1") == nullptr) {
    dim3 grid(a.H, n_sv);
    const size_t smem = sizeof(uint32_t) * (4 * (size_t)a.W + 1);
    cudaFuncSetAttribute(k_cost_w3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_cost_w3<<<grid, COST_NT, smem, st>>>(a);
    return;
  }
  const int nw = (a.window + 3) / 4;
  dim3 grid(a.H, n_sv);
  const size_t smem = sizeof(uint32_t) * ((size_t)2 * nw * a.W + 2 * (size_t)a.W);
  switch (nw) {
    case 1:
      cudaFuncSetAttribute(k_cost<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_cost<1><<<grid, COST_NT, smem, st>>>(a);
      break;
    case 2:
      cudaFuncSetAttribute(k_cost<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_cost<2><<<grid, COST_NT, smem, st>>>(a);
      break;
    default:
      cudaFuncSetAttribute(k_cost<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_cost<3><<<grid, COST_NT, smem, st>>>(a);
      break;
  }
}

}  // namespace es
