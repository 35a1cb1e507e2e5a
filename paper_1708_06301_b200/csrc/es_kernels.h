// Kernel argument blocks and launcher declarations (internal to the library).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "es_common.cuh"

namespace es {

// kernel attributes, set once per (kernel, device, value) and checked:
// cudaFuncAttributeMaxDynamicSharedMemorySize is raised only when a launch
// needs more than already granted; false (and the CUDA error left for the
// caller's cudaGetLastError) when the device refuses
bool ensure_smem(const void* kernel, size_t bytes);
bool ensure_attr(const void* kernel, cudaFuncAttribute attr, int value);
// SM count of the current device (cached per device; 148 on a B200)
int device_sms();

// ---- prediction (es_predict.cu); all arrays are [n_sv][H][W] ------------
struct PredArgs {
  Rig rig;
  Params prm;
  const double* Hm;          // [n_sv][16] row-major homographies
  const uint8_t* have_pred;  // [n_seq] 1 = warp the state this frame
  const double* sd;          // previous state
  const double* sp;
  const uint8_t* sv;
  unsigned long long* zkey;  // z-buffer phase 1 (bits of max d')
  uint32_t* zidx;            // z-buffer phase 2 (min source index)
  uint32_t* wt;              // per source: landing pixel (NO_SRC: not splatted)
  double* wd;                // per source: warped disparity d'
  double* hd;                // after the horizontal fill pass
  double* hp;
  uint8_t* hv;
  double* pd;                // final predicted maps
  double* pp;
  uint8_t* pv;
  uint2* meta;               // lo | hi << 16, pair offset
  unsigned long long* cells; // [n_sv] searched cells (sum of widths)
  int* err;                  // [n_seq] error bits
  unsigned long long* cells_acc = nullptr;  // optional running total over steps
};

void launch_predict(const PredArgs& a, int n_sv, cudaStream_t st);
void launch_fill_v_intervals(const PredArgs& a, int n_sv, cudaStream_t st);
void launch_meta_from_intervals(const int64_t* lo, const int64_t* hi, int W, int H, int d_max,
                                uint2* meta, cudaStream_t st);
void launch_edges(const double* d, const uint8_t* v, int W, int H, int r, double gamma_e,
                  uint8_t* out, cudaStream_t st);

// ---- cost (es_cost.cu) ----------------------------------------------------
struct CostArgs {
  int W, H, d_max, window;
  const uint8_t* img;   // [n_seq][2][H][W]
  const uint2* meta;    // [n_sv][H][W]
  uint32_t* C;          // [n_sv][volcap] u16 pairs
  size_t volcap;        // pairs per (seq, view)
  int view0;            // view of sv_local 0
  int tma = 0;          // 1: img has >= 16 readable bytes past its end, so the
                        //    image rows may be staged by 16-byte-aligned bulk copies
};
void launch_cost(const CostArgs& a, int n_sv, cudaStream_t st);

// ---- aggregation + WTA (es_sgm.cu) ----------------------------------------
enum Family { FAM_H = 0, FAM_V = 1, FAM_D1 = 2, FAM_D2 = 3 };
enum Arith { ARITH_U16 = 0, ARITH_F32 = 1 };

struct SgmArgs {
  int W, H, d_max;
  const uint2* meta;
  const void* C;        // u16 pairs (cost_f32 == 0) or float pairs
  void* S;              // u16 pairs (ARITH_U16) or float pairs (ARITH_F32)
  size_t volcap;        // pairs per (seq, view)
  int cost_f32;
  uint32_t p1i, p2i;
  float p1, p2;
  int lanes = 0;        // forced lanes per chain of the u16 kernel (0 = heuristic)
  // device-side regime choice: with cells != nullptr both regime variants
  // launch and each (seq, view) runs in the one matching its search fraction
  // (<= split: narrow variant, > split: wide variant)
  const unsigned long long* cells = nullptr;
  double split = 0.3;
  int select = 0;       // internal: 0 all, 1 fraction <= split, 2 fraction > split
  // fused vertical + diagonal sweeps (launch_aggregate_parts): the
  // round-boundary hand-over buffers of the two sweeps (null: grp4 jobs only)
  uint32_t* sweep_ring = nullptr;   // [2][n_sv][sweep_ring_words]
  // views of all contexts sharing the device with this launch (0: n_sv)
  int shared_views = 0;
};
// full 8-path aggregation; the u16 path runs 4 family launches (both sweeps
// each), the f32 path runs the 8 directions in the reference's order
void launch_aggregate(const SgmArgs& a, int arith, int n_sv, cudaStream_t st);
// u16 only, a.cells required: the 4 path families accumulate into `parts`
// (1, 2 or 4) partial sums S[k % parts]; reduced-interval (seq, view)s run on
// st_lo[p], wide ones on st_hi[p]; all streams may run concurrently
// returns the number of partial sums holding the total (<= parts)
int launch_aggregate_parts(const SgmArgs& a, int n_sv, int parts, void* const* S,
                           const cudaStream_t* st_lo, const cudaStream_t* st_hi);
// fused column + diagonal pass (es_sgm_vd.cu): the three directions of one
// row sweep (up = 0: dy = +1, up = 1: dy = -1) in one cluster per view,
// read-modify-writing (init: writing) the u16 partial sum a.S
bool vd_supported(int W, int d_max);
void launch_vd(const SgmArgs& a, bool up, bool init, int n_sv, cudaStream_t st);

// fused vertical + diagonal row sweep (es_sgm_sweep.cu): the three
// directions of one row sweep (up = 0: dy = +1, up = 1: dy = -1) in one pass,
// one CTA per (sequence, view), sheared diagonal strips of 32/G chains per warp
struct SweepArgs {
  SgmArgs a;
  int up;                 // 0: top -> bottom, 1: bottom -> top
  int nstrips;            // strips per view (sweep_strips)
  int total;              // n_sv * nstrips
  uint32_t* ring;         // [n_sv][sweep_ring_words]: round-boundary hand-over records
};
int sweep_lanes(int d_max);                           // G (0: d_max too large)
int sweep_strips(int W, int d_max, int H);
size_t sweep_ring_words(int W, int d_max, int H);     // per (seq, view)
void launch_sweep(const SweepArgs& v, bool init, cudaStream_t st);

struct WtaArgs {
  int W, H;
  const uint2* meta;
  const void* S;
  size_t volcap;
  int arith;
  double s_max, r_min;
  uint16_t* dstar;      // [n_sv][H][W]
  double* r;
  uint8_t* valid;
  const uint16_t* dstar_in = nullptr;  // optional caller winners (variance only)
  const void* Sx[3] = {nullptr, nullptr, nullptr};  // further u16 partial sums (added to S)
  const unsigned long long* cells = nullptr;   // unused by k_wta_runs
  int d_max = 0;
  double split = 0.3;
  int select = 0;
};
void launch_wta_variance(const WtaArgs& a, int n_sv, cudaStream_t st);

// dense <-> ragged converters for parity export and stage-level APIs
enum ExportMode { EXPORT_U16_COST = 0, EXPORT_F32 = 1, EXPORT_U16_SUM = 2 };
void launch_export_dense(const uint2* meta, const void* vol, int vol_f32, int W, int H, int d_max,
                         float* out, cudaStream_t st, const void* vol2 = nullptr,
                         const void* vol3 = nullptr, const void* vol4 = nullptr);
void launch_import_dense(const float* dense, const uint2* meta, int W, int H, int D, int as_f32,
                         void* vol, cudaStream_t st);
void launch_hull(const float* dense, int W, int H, int D, int64_t* lo, int64_t* hi,
                 unsigned int* flags, float limit, cudaStream_t st);

// ---- checks + Kalman update (es_fuse.cu) ----------------------------------
struct FuseArgs {
  int W, H, window;
  double tau_lr, tau_sad, p_init;
  const uint2* meta;       // [n_sv]
  const uint32_t* C;       // [n_sv] u16 pairs (raw SAD)
  size_t volcap;
  const uint16_t* dstar;   // [n_sv]
  const uint8_t* mvalid;
  const double* r;
  const double* pd;        // predicted
  const double* pp;
  const uint8_t* pv;
  double* nd;              // new state
  double* np_;
  uint8_t* nv;
  uint8_t* keep;           // [n_sv]
  int* any_valid = nullptr;  // [n_seq] set when the new state has a valid pixel
};
void launch_checks_fuse(const FuseArgs& a, int n_seq, cudaStream_t st);

void launch_lr(const double* dl, const uint8_t* vl, const double* dr, const uint8_t* vr, int W,
               int H, double tau, uint8_t* kl, uint8_t* kr, cudaStream_t st);
void launch_sad_check(const uint8_t* left, const uint8_t* right, const double* d, const uint8_t* v,
                      int W, int H, int window, double tau, int view, uint8_t* keep,
                      cudaStream_t st);
void launch_fuse(const double* dp, const double* pp, const uint8_t* vp, const double* dm,
                 const double* rm, const uint8_t* vm, int n, double p_init, double* od,
                 double* op, uint8_t* ov, cudaStream_t st);
void launch_fill_axis(const double* d, const double* p, const uint8_t* v, int W, int H, int axis,
                      double gamma_f, double q, double* od, double* op, uint8_t* ov, int final_pass,
                      cudaStream_t st);
void launch_intervals_only(const double* d, const double* p, const uint8_t* v, int n, int d_max,
                           int64_t* lo, int64_t* hi, cudaStream_t st);

// ---- evaluation metrics (es_metrics.cu) --------------------------------------
struct MetricsArgs {
  const double* est;          // [n_maps][stride_e]
  const uint8_t* est_valid;
  const double* gt;           // [n_maps][stride_g]
  const uint8_t* gt_valid;
  size_t n, stride_e, stride_g;
  int mode;                   // 0 "or", 1 "and"
  unsigned long long* counts; // [n_maps][4]: gt valid, jointly valid, bad, estimate valid
  uint8_t* mask = nullptr;    // optional [n_maps][n]
  uint8_t* rgb = nullptr;     // optional [n_maps][n][3]
};
void launch_metrics(const MetricsArgs& a, int n_maps, cudaStream_t st);

// ---- synthetic renderer (es_render.cu) -------------------------------------
struct RenderArgs {
  Rig rig;
  const double* prims;   // [n_seq][n_prim][8]: kind, 6 parameters, plane bound flags
  int n_prim;
  const double* poses;   // [n_seq][16] world-from-camera (left camera)
  const long long* seeds;  // [n_seq] texture seed
  double texture_scale;
  int background;
  uint8_t* img;          // [n_seq][2][H][W]
  double* gt;            // optional [n_seq][2][H][W] (nullptr to skip)
};
void launch_render(const RenderArgs& a, int n_seq, cudaStream_t st);

}  // namespace es
