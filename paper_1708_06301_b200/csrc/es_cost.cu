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
  const uint32_t rowbase = (uint32_t)y * (uint32_t)(W * npairs_max(a.d_max));
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
  const uint32_t last = rowlh[W - 1];
  const uint32_t row_pairs = rowoff[W - 1] + ((last >> 16) >> 1) - ((last & 0xFFFFu) >> 1) + 1;
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

void launch_cost(const CostArgs& a, int n_sv, cudaStream_t st) {
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
