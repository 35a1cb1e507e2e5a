// C ABI (include/egostereo_b200.h): pipeline contexts and stage entry points.
#include <array>
#include <map>
#include <tuple>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/egostereo_b200.h"
#include "es_common.cuh"
#include "es_kernels.h"

using namespace es;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ES_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

bool is_integral(double v) { return v == (double)(long long)v; }

int check_params(const es_params* p) {
  if (p->window < 3 || p->window % 2 == 0) return fail(ES_ERR_VALUE, "window must be odd and >= 3");
  if (!(0 < p->p1 && p->p1 <= p->p2)) return fail(ES_ERR_VALUE, "penalties must satisfy 0 < P1 <= P2");
  if (p->s_max <= 0) return fail(ES_ERR_VALUE, "s_max must be positive");
  if (p->r_min <= 0) return fail(ES_ERR_VALUE, "r_min must be positive");
  if (p->window > 11) return fail(ES_ERR_UNSUPPORTED, "device cost storage supports window <= 11");
  return ES_OK;
}

int check_rig(const es_rig* r) {
  if (r->f <= 0 || r->b <= 0 || r->d_max < 1 || r->d_max >= r->width || r->width < 2 ||
      r->height < 2)
    return fail(ES_ERR_VALUE, "invalid StereoRig");
  if (r->d_max > 511) return fail(ES_ERR_UNSUPPORTED, "device path supports d_max <= 511");
  // pair offsets inside one view's volume are 32-bit; the aggregation forms
  // signed per-lane bases from them
  if ((double)row_capacity(r->width, r->d_max) * r->height >= 2147483647.0)
    return fail(ES_ERR_UNSUPPORTED, "volume exceeds 2^31 pairs per view");
  return ES_OK;
}

Params to_params(const es_params* p) {
  Params q;
  q.window = p->window;
  q.p1 = (float)p->p1;
  q.p2 = (float)p->p2;
  q.p1i = (uint32_t)p->p1;
  q.p2i = (uint32_t)p->p2;
  q.s_max = p->s_max;
  q.r_min = p->r_min;
  q.tau_lr = p->tau_lr;
  q.tau_sad = p->tau_sad;
  q.q = p->q;
  q.gamma_f = p->gamma_f;
  q.gamma_e = p->gamma_e;
  q.edge_window = p->edge_window;
  q.edge_reject = p->edge_reject;
  q.fill_holes = p->fill_holes;
  q.p_init = p->p_init;
  return q;
}

// u16 arithmetic is exact iff penalties are integers and the 8-path sum of
// the largest finite path value fits below the 0x8000 sentinel band
int choose_arith(double p1, double p2, double cmax) {
  if (!is_integral(p1) || !is_integral(p2)) return ARITH_F32;
  if (cmax + p2 >= 0x8000 - p1 - p2) return ARITH_F32;
  if (8.0 * (cmax + p2) > 65535.0) return ARITH_F32;
  if (p2 >= 0x4000) return ARITH_F32;
  return ARITH_U16;
}

Rig to_rig(const es_rig* r) {
  Rig g;
  g.f = r->f;
  g.b = r->b;
  g.cx = r->cx;
  g.cy = r->cy;
  g.W = r->width;
  g.H = r->height;
  g.d_max = r->d_max;
  return g;
}

template <class T>
int dalloc(T** p, size_t n) {
  cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (n ? n : 1));
  if (e != cudaSuccess) return fail(ES_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  return ES_OK;
}

// ---- small conversion kernels for materialisation -------------------------
__global__ void k_meta_to_lohi(const uint2* meta, size_t n, int64_t* lo, int64_t* hi) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (lo) lo[i] = meta[i].x & 0xFFFFu;
  if (hi) hi[i] = meta[i].x >> 16;
}
__global__ void k_u16_to_f64(const uint16_t* a, size_t n, double* o) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = (double)a[i];
}
// kitti_io.write_disparity_png encoding (kitti_io.py:38-46).  Fused
// disparities never exceed d_max, and for d_max <= 255 round(256 d) <= 65535;
// above that the reference's writer raises ValueError for large values, so
// the export refuses contexts with d_max > 255 instead of saturating.
static const char* kKittiRange =
    "KITTI 16-bit disparity encoding holds d < 256: d_max > 255 cannot be exported";
__global__ void k_kitti(const double* d, const uint8_t* v, size_t n, uint16_t* o) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double raw = rint(d[i] * 256.0);
  o[i] = v[i] ? (uint16_t)fmin(fmax(raw, 1.0), 65535.0) : (uint16_t)0;
}

// the same for every sequence of a batch: sequence s at d + s * stride
__global__ void k_kitti_batch(const double* d, const uint8_t* v, size_t n, size_t stride,
                              uint16_t* o) {
  const size_t s = blockIdx.y;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = d[s * stride + i];
  const bool ok = v[s * stride + i] != 0;
  const double raw = rint(x * 256.0);
  o[s * n + i] = ok ? (uint16_t)fmin(fmax(raw, 1.0), 65535.0) : (uint16_t)0;
}
// warp_point on principal-point-relative (x, y, d) triples (geometry.py:95-115)
__global__ void k_warp_points(const double* Hm, const double* pts, int n, double* out, int* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xp, yp, dp;
  if (!warp_point(Hm, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], 0.0, 0.0, xp, yp, dp)) {
    atomicOr(err, 1);
    return;
  }
  out[3 * i] = xp;
  out[3 * i + 1] = yp;
  out[3 * i + 2] = dp;
}

}  // namespace

namespace es {
bool ensure_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = granted[{kernel, dev}];
  if (bytes <= cur || bytes <= 48 * 1024) return true;
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess)
    return false;
  cur = bytes;
  return true;
}
bool ensure_attr(const void* kernel, cudaFuncAttribute attr, int value) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, int> set;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(kernel, dev, (int)attr);
  auto it = set.find(key);
  if (it != set.end() && it->second == value) return true;
  if (cudaFuncSetAttribute(kernel, attr, value) != cudaSuccess) return false;
  set[key] = value;
  return true;
}
int device_sms() {
  static std::mutex mu;
  static std::map<int, int> sms;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  auto it = sms.find(dev);
  if (it != sms.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  sms[dev] = n;
  return n;
}
}  // namespace es

struct es_ctx {
  int device = 0;
  es_rig rig_c;
  es_params prm_c;
  Rig rig;
  Params prm;
  int B = 1;
  int arith = ARITH_U16;
  size_t HW = 0, volcap = 0;
  cudaStream_t st = nullptr;
  // concurrent SGM: families accumulate into `parts` u16 partial sums (S and
  // Sx[0..parts-2]); reduced- and wide-interval variants of partial p run on
  // streams lo[p] / hi[p] (lo[0] = st)
  int parts = 1;
  uint32_t* Sx[3] = {nullptr, nullptr, nullptr};
  cudaStream_t sx[7] = {};
  int parts_live = 1;                  // partial sums holding the last step's total
  int shared_batch = 0;                // es_ctx_shared_batch: sequences of all cooperating contexts
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  uint8_t* img = nullptr;
  double* sd[2] = {nullptr, nullptr};
  double* sp[2] = {nullptr, nullptr};
  uint8_t* sv[2] = {nullptr, nullptr};
  int cur = 0;
  double *hd = nullptr, *hp = nullptr;
  uint8_t* hv = nullptr;
  double *pd = nullptr, *pp = nullptr;
  uint8_t* pv = nullptr;
  unsigned long long* zkey = nullptr;
  uint32_t* zidx = nullptr;
  uint32_t* wt = nullptr;
  double* wd = nullptr;
  uint2* meta = nullptr;
  uint32_t *C = nullptr, *S = nullptr;
  uint16_t* dstar = nullptr;
  double* r = nullptr;
  uint8_t *mvalid = nullptr, *keep = nullptr;
  double* Hm = nullptr;
  uint8_t* have_pred = nullptr;
  int* err = nullptr;
  int* anyv = nullptr;
  unsigned long long* cells = nullptr;
  // fused vertical + diagonal sweeps: round-boundary hand-over buffers of
  // the two sweeps (es_sgm_sweep.cu)
  uint32_t* sw_ring = nullptr;
  // pinned host mirrors
  double* h_Hm = nullptr;
  uint8_t* h_have = nullptr;
  int* h_err = nullptr;
  int* h_anyv = nullptr;
  unsigned long long* h_cells = nullptr;
  std::vector<long long> frame;
  std::vector<int> have_state;
  bool pending = false;
  // an error surfaced from deferred steps: their state was already
  // committed, so the filter state is not the reference's; steps are refused
  // until es_ctx_reset
  bool poisoned = false;
  // pinned argument staging ring (deferred steps may still be reading a slot)
  static constexpr int RING = 4;
  int ring_pos = 0;
  cudaEvent_t ring_ev[RING] = {};
  // per-stage CUDA-event profiling: predict, intervals, cost, aggregate,
  // wta+variance, checks+fuse
  static constexpr int NSTAGE = 6;
  bool profiling = false;
  std::vector<std::array<cudaEvent_t, NSTAGE + 1>> prof;
  uint16_t* kitti = nullptr;   // batched KITTI export staging (2 slots)
  // host<->device copy overlap: input images are double-buffered (img,
  // img2) and uploaded on cp_in; KITTI exports are copied out on cp_out, so
  // both transfers overlap the neighbouring steps' kernels
  uint8_t* img2 = nullptr;
  uint8_t* img_cur = nullptr;  // buffer the current step's kernels read
  int img_slot = 0;
  int kitti_slot = 0;
  cudaStream_t cp_in = nullptr, cp_out = nullptr;
  cudaEvent_t ev_img_free[2] = {}, ev_img_ready = nullptr, ev_kitti_ready = nullptr,
              ev_kitti_free[2] = {};
  unsigned long long* cells_acc = nullptr;   // searched cells summed over steps
  int lanes = 0;               // SGM lanes per chain (0 = heuristic)
  double last_fraction = 1.0;  // search fraction of the last synced step

  void note_fraction() {
    unsigned long long cells = 0;
    for (int s = 0; s < 2 * B; ++s) cells += h_cells[s];
    last_fraction = (double)cells / ((double)HW * 2 * B * (rig.d_max + 1));
  }
};

namespace {

int ctx_free(es_ctx* c) {
  if (!c) return ES_OK;
  cudaSetDevice(c->device);
  void* ptrs[] = {c->img, c->sd[0], c->sd[1], c->sp[0], c->sp[1], c->sv[0], c->sv[1], c->hd,
                  c->hp, c->hv, c->pd, c->pp, c->pv, c->zkey, c->zidx, c->wt, c->wd, c->meta,
                  c->C, c->S,
                  c->Sx[0], c->Sx[1], c->Sx[2], c->dstar, c->r, c->mvalid, c->keep, c->Hm,
                  c->have_pred, c->err, c->anyv,
                  c->cells, c->kitti, c->cells_acc, c->img2, c->sw_ring};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  void* hptrs[] = {c->h_Hm, c->h_have, c->h_err, c->h_anyv, c->h_cells};
  for (void* p : hptrs)
    if (p) cudaFreeHost(p);
  for (cudaEvent_t e : c->ring_ev)
    if (e) cudaEventDestroy(e);
  for (auto& a : c->prof)
    for (cudaEvent_t e : a) cudaEventDestroy(e);
  if (c->st) cudaStreamDestroy(c->st);
  for (cudaStream_t s : c->sx)
    if (s) cudaStreamDestroy(s);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (cudaEvent_t e : {c->ev_img_free[0], c->ev_img_free[1], c->ev_img_ready, c->ev_kitti_ready,
                        c->ev_kitti_free[0], c->ev_kitti_free[1]})
    if (e) cudaEventDestroy(e);
  if (c->cp_in) cudaStreamDestroy(c->cp_in);
  if (c->cp_out) cudaStreamDestroy(c->cp_out);
  delete c;
  return ES_OK;
}

PredArgs pred_args(es_ctx* c) {
  PredArgs a;
  a.rig = c->rig;
  a.prm = c->prm;
  a.Hm = c->Hm;
  a.have_pred = c->have_pred;
  a.sd = c->sd[c->cur];
  a.sp = c->sp[c->cur];
  a.sv = c->sv[c->cur];
  a.zkey = c->zkey;
  a.zidx = c->zidx;
  a.wt = c->wt;
  a.wd = c->wd;
  a.hd = c->hd;
  a.hp = c->hp;
  a.hv = c->hv;
  a.pd = c->pd;
  a.pp = c->pp;
  a.pv = c->pv;
  a.meta = c->meta;
  a.cells = c->cells;
  a.err = c->err;
  a.cells_acc = c->cells_acc;
  return a;
}

int commit_errors(es_ctx* c) {
  // the first failing sequence, and in it the reference's order: left view
  // (bits 0-1) before right (bits 2-3), point at infinity before d <= 0
  for (int s = 0; s < c->B; ++s) {
    const int bits = c->h_err[s];
    for (int view = 0; view < 2; ++view) {
      const int b = (bits >> (2 * view)) & 3;
      if (b & ERR_POINT_AT_INFINITY)
        return fail(ES_ERR_POINT_AT_INFINITY, "warped point has ~zero fourth homogeneous component");
      if (b & ERR_NONPOSITIVE_D) return fail(ES_ERR_NONPOSITIVE_D, "previous disparity must be positive");
    }
  }
  return ES_OK;
}

}  // namespace

extern "C" {

const char* es_last_error(void) { return g_err.c_str(); }
int es_version(void) { return 1; }
int es_device_count(int* n) {
  CK(cudaGetDeviceCount(n));
  return ES_OK;
}

int es_ctx_create(int device, const es_rig* rig, const es_params* prm, int batch, es_ctx** out) {
  *out = nullptr;
  if (int e = check_rig(rig)) return e;
  if (int e = check_params(prm)) return e;
  if (batch < 1) return fail(ES_ERR_VALUE, "batch must be >= 1");
  CK(cudaSetDevice(device));
  es_ctx* c = new es_ctx();
  c->device = device;
  c->rig_c = *rig;
  c->prm_c = *prm;
  c->rig = to_rig(rig);
  c->prm = to_params(prm);
  c->B = batch;
  c->arith = choose_arith(prm->p1, prm->p2, (double)prm->window * prm->window * 255.0);
  c->HW = (size_t)rig->width * rig->height;
  c->volcap = (size_t)rig->height * row_capacity(rig->width, rig->d_max);
  const size_t n = c->HW * 2 * batch;
  const size_t vol_words = c->volcap * 2 * batch * (c->arith == ARITH_F32 ? 2 : 1);
  int e = ES_OK;
  // image buffers carry 64 bytes of tail padding: the cost kernel stages
  // rows with 16-byte-aligned bulk copies that may read past the last row
  if (!e) e = dalloc(&c->img, n + 64);
  if (!e) e = dalloc(&c->img2, n + 64);
  // KITTI export staging (2 slots): allocated here, never inside a step, so
  // an export never triggers the implicit device synchronisation of cudaMalloc
  if (!e) e = dalloc(&c->kitti, 2 * (size_t)batch * c->HW);
  for (int k = 0; k < 2 && !e; ++k) {
    e = dalloc(&c->sd[k], n);
    if (!e) e = dalloc(&c->sp[k], n);
    if (!e) e = dalloc(&c->sv[k], n);
  }
  if (!e) e = dalloc(&c->hd, n);
  if (!e) e = dalloc(&c->hp, n);
  if (!e) e = dalloc(&c->hv, n);
  if (!e) e = dalloc(&c->pd, n);
  if (!e) e = dalloc(&c->pp, n);
  if (!e) e = dalloc(&c->pv, n);
  if (!e) e = dalloc(&c->zkey, n);
  if (!e) e = dalloc(&c->zidx, n);
  if (!e) e = dalloc(&c->wt, n);
  if (!e) e = dalloc(&c->wd, n);
  if (!e) e = dalloc(&c->meta, n);
  if (!e) e = dalloc(&c->C, c->volcap * 2 * batch);
  if (!e) e = dalloc(&c->S, vol_words);
  if (c->arith == ARITH_U16) {
    // small batches are latency-bound: one partial sum (and stream) per path
    // family; large ones use two (measured)
    const char* pe = getenv("ES_SGM_PARTS");
    c->parts = pe ? atoi(pe) : (batch <= 8 ? 4 : 2);
    if (c->parts != 1 && c->parts != 2 && c->parts != 4) c->parts = 2;
    for (int p = 0; p + 1 < c->parts && !e; ++p) e = dalloc(&c->Sx[p], vol_words);
    const int n_sv = 2 * batch;
    if (!e && sweep_lanes(rig->d_max) && (c->parts == 2 || c->parts == 4)) {
      e = dalloc(&c->sw_ring, 2 * (size_t)n_sv * sweep_ring_words(rig->width, rig->d_max, rig->height));
    }
  }
  if (!e) e = dalloc(&c->dstar, n);
  if (!e) e = dalloc(&c->r, n);
  if (!e) e = dalloc(&c->mvalid, n);
  if (!e) e = dalloc(&c->keep, n);
  if (!e) e = dalloc(&c->Hm, 32 * (size_t)batch);
  if (!e) e = dalloc(&c->have_pred, batch);
  if (!e) e = dalloc(&c->err, batch);
  if (!e) e = dalloc(&c->anyv, batch);
  if (!e) e = dalloc(&c->cells, 2 * (size_t)batch);
  if (!e) e = dalloc(&c->cells_acc, 1);
  if (!e && cudaMemset(c->cells_acc, 0, sizeof(unsigned long long)) != cudaSuccess)
    e = fail(ES_ERR_CUDA, "cudaMemset failed");
  if (e) {
    ctx_free(c);
    return e;
  }
  bool ev_ok = true;
  for (auto& e : c->ring_ev)
    ev_ok = ev_ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
  if (!ev_ok ||
      cudaMallocHost(&c->h_Hm, sizeof(double) * 32 * batch * es_ctx::RING) != cudaSuccess ||
      cudaMallocHost(&c->h_have, (size_t)batch * es_ctx::RING) != cudaSuccess ||
      cudaMallocHost(&c->h_err, sizeof(int) * batch) != cudaSuccess ||
      cudaMallocHost(&c->h_anyv, sizeof(int) * batch) != cudaSuccess ||
      cudaMallocHost(&c->h_cells, sizeof(unsigned long long) * 2 * batch) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->sx[0], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->sx[1], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->sx[2], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->sx[3], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->sx[4], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->sx[5], cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->sx[6], cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cp_in, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cp_out, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_img_free[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_img_free[1], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_img_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_kitti_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_kitti_free[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_kitti_free[1], cudaEventDisableTiming) != cudaSuccess) {
    ctx_free(c);
    return fail(ES_ERR_CUDA, "pinned host / stream allocation failed");
  }
  c->frame.assign(batch, -1);
  c->have_state.assign(batch, 0);
  if (int e2 = es_ctx_reset(c)) {
    ctx_free(c);
    return e2;
  }
  *out = c;
  return ES_OK;
}

int es_ctx_destroy(es_ctx* ctx) { return ctx_free(ctx); }

int es_ctx_reset(es_ctx* c) {
  CK(cudaSetDevice(c->device));
  const size_t n = c->HW * 2 * c->B;
  for (int k = 0; k < 2; ++k) {
    CK(cudaMemsetAsync(c->sd[k], 0, sizeof(double) * n, c->st));
    CK(cudaMemsetAsync(c->sp[k], 0, sizeof(double) * n, c->st));
    CK(cudaMemsetAsync(c->sv[k], 0, n, c->st));
  }
  CK(cudaStreamSynchronize(c->st));
  for (int s = 0; s < c->B; ++s) {
    c->frame[s] = -1;
    c->have_state[s] = 0;
  }
  c->poisoned = false;
  c->pending = false;
  return ES_OK;
}

int es_ctx_sync(es_ctx* c) {
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->st));
  CK(cudaStreamSynchronize(c->cp_out));
  if (c->pending) {
    c->pending = false;
    for (int s = 0; s < c->B; ++s) c->have_state[s] = c->h_anyv[s] != 0;
    c->note_fraction();
    const int e = commit_errors(c);   // error bits accumulated over the deferred steps
    if (e) c->poisoned = true;
    return e;
  }
  return ES_OK;
}

int es_ctx_step(es_ctx* c, const uint8_t* images, int images_dev, const double* Hm,
                const uint8_t* motion_given, int sync) {
  CK(cudaSetDevice(c->device));
  const int B = c->B;
  const size_t HW = c->HW;
  const int n_sv = 2 * B;
  if (c->poisoned)
    return fail(ES_ERR_VALUE, "context state is invalid after an error in a deferred step; "
                              "call es_ctx_reset");
  if (c->pending && sync) {
    // a previous deferred step: surface its errors first
    if (int e = es_ctx_sync(c)) return e;
  }
  // host-side decision: predict iff motion given, state non-empty, not baseline
  // (pipeline.py:122-123).  With deferred steps the state is assumed non-empty;
  // an empty state predicts nothing, which yields full-range intervals anyway.
  // pinned staging slot for this step's small arguments; a slot is reused
  // only after the copy that last read it has executed
  const int slot = c->ring_pos;
  c->ring_pos = (c->ring_pos + 1) % es_ctx::RING;
  CK(cudaEventSynchronize(c->ring_ev[slot]));
  double* h_Hm = c->h_Hm + (size_t)slot * 32 * B;
  uint8_t* h_have = c->h_have + (size_t)slot * B;
  for (int s = 0; s < B; ++s) {
    const bool have = c->pending ? true : (c->have_state[s] != 0);
    h_have[s] = (motion_given && motion_given[s] && have && !c->prm_c.baseline) ? 1 : 0;
  }
  if (Hm) memcpy(h_Hm, Hm, sizeof(double) * 32 * B);
  else memset(h_Hm, 0, sizeof(double) * 32 * B);
  cudaEvent_t* ev = nullptr;
  if (c->profiling) {
    c->prof.emplace_back();
    ev = c->prof.back().data();
    for (int k = 0; k <= es_ctx::NSTAGE; ++k) CK(cudaEventCreate(&ev[k]));
  }
  auto mark = [&](int k) {
    if (ev) cudaEventRecord(ev[k], c->st);
  };
  // this step's images go to the buffer the step before last read; its
  // upload waits only for that step's cost kernel, not for the previous step
  const int ib = c->img_slot;
  c->img_slot ^= 1;
  c->img_cur = ib ? c->img2 : c->img;
  CK(cudaStreamWaitEvent(c->cp_in, c->ev_img_free[ib], 0));
  CK(cudaMemcpyAsync(c->img_cur, images, HW * 2 * B,
                     images_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->cp_in));
  CK(cudaEventRecord(c->ev_img_ready, c->cp_in));
  CK(cudaStreamWaitEvent(c->st, c->ev_img_ready, 0));
  CK(cudaMemcpyAsync(c->Hm, h_Hm, sizeof(double) * 32 * B, cudaMemcpyHostToDevice, c->st));
  CK(cudaMemcpyAsync(c->have_pred, h_have, B, cudaMemcpyHostToDevice, c->st));
  CK(cudaEventRecord(c->ring_ev[slot], c->st));
  // error bits accumulate across deferred steps until a sync reads them
  if (!c->pending) CK(cudaMemsetAsync(c->err, 0, sizeof(int) * B, c->st));
  CK(cudaMemsetAsync(c->anyv, 0, sizeof(int) * B, c->st));

  PredArgs pa = pred_args(c);
  mark(0);
  launch_predict(pa, n_sv, c->st);
  mark(1);
  launch_fill_v_intervals(pa, n_sv, c->st);
  mark(2);

  CostArgs ca;
  ca.W = c->rig.W;
  ca.H = c->rig.H;
  ca.d_max = c->rig.d_max;
  ca.window = c->prm.window;
  ca.img = c->img_cur;
  ca.meta = c->meta;
  ca.C = c->C;
  ca.volcap = c->volcap;
  ca.view0 = 0;
  static const bool no_tma = getenv("ES_COST_NO_TMA") != nullptr;   // A/B switch
  ca.tma = no_tma ? 0 : 1;
  launch_cost(ca, n_sv, c->st);
  CK(cudaEventRecord(c->ev_img_free[ib], c->st));   // the images' last reader
  mark(3);

  SgmArgs sa;
  sa.W = c->rig.W;
  sa.H = c->rig.H;
  sa.d_max = c->rig.d_max;
  sa.meta = c->meta;
  sa.C = c->C;
  sa.S = c->S;
  sa.volcap = c->volcap;
  sa.cost_f32 = 0;
  sa.p1i = c->prm.p1i;
  sa.p2i = c->prm.p2i;
  sa.p1 = c->prm.p1;
  sa.p2 = c->prm.p2;
  // regime variants: each (seq, view) runs in the variant matching its
  // search fraction, chosen on the device from this frame's searched-cell
  // count (<= split: G lanes per chain, > split: 2G; measured)
  sa.lanes = c->lanes;
  sa.cells = c->cells;
  sa.sweep_ring = c->sw_ring;
  sa.shared_views = 2 * c->shared_batch;
  static const double split = getenv("ES_SGM_SPLIT") ? atof(getenv("ES_SGM_SPLIT")) : 0.6;
  sa.split = split;
  if (c->arith == ARITH_U16 && !c->lanes) {
    // fork: the partial sums' families and the two regime variants run on
    // 2 * parts concurrent streams; each touches its own (seq, view) x sum
    const int P = c->parts;
    void* S[4] = {c->S, c->Sx[0], c->Sx[1], c->Sx[2]};
    const cudaStream_t lo[4] = {c->st, c->sx[1], c->sx[3], c->sx[5]};
    const cudaStream_t hi[4] = {c->sx[0], c->sx[2], c->sx[4], c->sx[6]};
    CK(cudaEventRecord(c->ev_fork, c->st));
    for (int p = 0; p < P; ++p) {
      if (p) CK(cudaStreamWaitEvent(lo[p], c->ev_fork, 0));
      CK(cudaStreamWaitEvent(hi[p], c->ev_fork, 0));
    }
    const int live = launch_aggregate_parts(sa, n_sv, P, S, lo, hi);
    for (int p = 0; p < P; ++p) {
      for (cudaStream_t s : {lo[p], hi[p]}) {
        if (s == c->st) continue;
        CK(cudaEventRecord(c->ev_join, s));
        CK(cudaStreamWaitEvent(c->st, c->ev_join, 0));
      }
    }
    c->parts_live = live;
  } else {
    launch_aggregate(sa, c->arith, n_sv, c->st);
    c->parts_live = 1;
  }
  mark(4);

  WtaArgs wa;
  wa.W = c->rig.W;
  wa.H = c->rig.H;
  wa.meta = c->meta;
  wa.S = c->S;
  for (int p = 1; p < c->parts_live; ++p) wa.Sx[p - 1] = c->Sx[p - 1];
  wa.volcap = c->volcap;
  wa.arith = c->arith;
  wa.s_max = c->prm.s_max;
  wa.r_min = c->prm.r_min;
  wa.dstar = c->dstar;
  wa.r = c->r;
  wa.valid = c->mvalid;
  wa.cells = c->cells;
  wa.d_max = c->rig.d_max;
  launch_wta_variance(wa, n_sv, c->st);
  mark(5);

  const int nxt = c->cur ^ 1;
  FuseArgs fa;
  fa.W = c->rig.W;
  fa.H = c->rig.H;
  fa.window = c->prm.window;
  fa.tau_lr = c->prm.tau_lr;
  fa.tau_sad = c->prm.tau_sad;
  fa.p_init = c->prm.p_init;
  fa.meta = c->meta;
  fa.C = c->C;
  fa.volcap = c->volcap;
  fa.dstar = c->dstar;
  fa.mvalid = c->mvalid;
  fa.r = c->r;
  fa.pd = c->pd;
  fa.pp = c->pp;
  fa.pv = c->pv;
  fa.nd = c->sd[nxt];
  fa.np_ = c->sp[nxt];
  fa.nv = c->sv[nxt];
  fa.keep = c->keep;
  fa.any_valid = c->anyv;
  launch_checks_fuse(fa, B, c->st);
  mark(6);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(c->h_err, c->err, sizeof(int) * B, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(c->h_anyv, c->anyv, sizeof(int) * B, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(c->h_cells, c->cells, sizeof(unsigned long long) * 2 * B,
                     cudaMemcpyDeviceToHost, c->st));
  if (sync) {
    CK(cudaStreamSynchronize(c->st));
    if (int e = commit_errors(c)) return e;   // state not committed
    c->note_fraction();
    c->cur = nxt;
    for (int s = 0; s < B; ++s) {
      c->frame[s] += 1;
      c->have_state[s] = c->h_anyv[s] != 0;
    }
  } else {
    c->cur = nxt;
    for (int s = 0; s < B; ++s) c->frame[s] += 1;
    c->pending = true;
  }
  return ES_OK;
}

int es_ctx_frame(es_ctx* c, int seq, int64_t* frame) {
  if (seq < 0 || seq >= c->B) return fail(ES_ERR_VALUE, "sequence index out of range");
  *frame = c->frame[seq];
  return ES_OK;
}

int es_ctx_cells_acc(es_ctx* c, uint64_t* total, int reset) {
  CK(cudaSetDevice(c->device));
  unsigned long long v = 0;
  CK(cudaMemcpyAsync(&v, c->cells_acc, sizeof(v), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  *total = v;
  if (reset) CK(cudaMemsetAsync(c->cells_acc, 0, sizeof(v), c->st));
  return ES_OK;
}

int es_ctx_shared_batch(es_ctx* c, int total_batch) {
  if (total_batch < 0) return fail(ES_ERR_VALUE, "total_batch must be >= 0");
  c->shared_batch = total_batch;
  return ES_OK;
}

int es_ctx_profile(es_ctx* c, int enable) {
  c->profiling = enable != 0;
  return ES_OK;
}

int es_ctx_stage_times(es_ctx* c, double* ms, int64_t* steps) {
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->st));
  for (int k = 0; k < es_ctx::NSTAGE; ++k) ms[k] = 0.0;
  for (auto& a : c->prof) {
    for (int k = 0; k < es_ctx::NSTAGE; ++k) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, a[k], a[k + 1]));
      ms[k] += t;
    }
    for (cudaEvent_t e : a) cudaEventDestroy(e);
  }
  *steps = (int64_t)c->prof.size();
  c->prof.clear();
  return ES_OK;
}

int es_ctx_have_state(es_ctx* c, int seq, int64_t* have) {
  if (seq < 0 || seq >= c->B) return fail(ES_ERR_VALUE, "sequence index out of range");
  *have = c->pending ? 1 : c->have_state[seq];
  return ES_OK;
}

int es_ctx_cells(es_ctx* c, int seq, uint64_t* l, uint64_t* r) {
  if (seq < 0 || seq >= c->B) return fail(ES_ERR_VALUE, "sequence index out of range");
  CK(cudaStreamSynchronize(c->st));
  *l = c->h_cells[2 * seq];
  *r = c->h_cells[2 * seq + 1];
  return ES_OK;
}

int es_ctx_stream(es_ctx* c, void** stream) {
  *stream = (void*)c->st;
  return ES_OK;
}

int es_ctx_device_ptr(es_ctx* c, int what, int seq, int view, void** p) {
  if (seq < 0 || seq >= c->B || view < 0 || view > 1) return fail(ES_ERR_VALUE, "bad index");
  const size_t o = ((size_t)seq * 2 + view) * c->HW;
  switch (what) {
    case ES_PRED_D: *p = c->pd + o; break;
    case ES_PRED_P: *p = c->pp + o; break;
    case ES_PRED_VALID: *p = c->pv + o; break;
    case ES_MEAS_VALID: *p = c->mvalid + o; break;
    case ES_MEAS_R: *p = c->r + o; break;
    case ES_KEEP: *p = c->keep + o; break;
    case ES_FUSED_D: *p = c->sd[c->cur] + o; break;
    case ES_FUSED_P: *p = c->sp[c->cur] + o; break;
    case ES_FUSED_VALID: *p = c->sv[c->cur] + o; break;
    default: return fail(ES_ERR_VALUE, "map has no direct device pointer");
  }
  return ES_OK;
}

int es_ctx_export(es_ctx* c, int what, int seq, int view, void* out) {
  CK(cudaSetDevice(c->device));
  if (seq < 0 || seq >= c->B || view < 0 || view > 1) return fail(ES_ERR_VALUE, "bad index");
  const size_t HW = c->HW;
  const size_t o = ((size_t)seq * 2 + view) * HW;
  const unsigned nb = (unsigned)((HW + 255) / 256);
  void* src = nullptr;
  size_t bytes = 0;
  void* tmp = nullptr;
  switch (what) {
    case ES_LO:
    case ES_HI: {
      CK(cudaMallocAsync(&tmp, sizeof(int64_t) * HW, c->st));
      k_meta_to_lohi<<<nb, 256, 0, c->st>>>(c->meta + o, HW,
                                             what == ES_LO ? (int64_t*)tmp : nullptr,
                                             what == ES_HI ? (int64_t*)tmp : nullptr);
      src = tmp;
      bytes = sizeof(int64_t) * HW;
      break;
    }
    case ES_MEAS_D: {
      CK(cudaMallocAsync(&tmp, sizeof(double) * HW, c->st));
      k_u16_to_f64<<<nb, 256, 0, c->st>>>(c->dstar + o, HW, (double*)tmp);
      src = tmp;
      bytes = sizeof(double) * HW;
      break;
    }
    case ES_FUSED_KITTI: {
      if (c->rig.d_max > 255) return fail(ES_ERR_VALUE, kKittiRange);
      CK(cudaMallocAsync(&tmp, sizeof(uint16_t) * HW, c->st));
      k_kitti<<<nb, 256, 0, c->st>>>(c->sd[c->cur] + o, c->sv[c->cur] + o, HW, (uint16_t*)tmp);
      src = tmp;
      bytes = sizeof(uint16_t) * HW;
      break;
    }
    case ES_COST_DENSE:
    case ES_TOTAL_DENSE: {
      const size_t n = HW * (c->rig.d_max + 1);
      CK(cudaMallocAsync(&tmp, sizeof(float) * n, c->st));
      const size_t sv = (size_t)seq * 2 + view;
      if (what == ES_COST_DENSE)
        launch_export_dense(c->meta + o, c->C + sv * c->volcap, 0, c->rig.W, c->rig.H,
                            c->rig.d_max, (float*)tmp, c->st);
      else
        launch_export_dense(c->meta + o,
                            c->arith == ARITH_F32 ? (void*)((float2*)c->S + sv * c->volcap)
                                                  : (void*)(c->S + sv * c->volcap),
                            c->arith == ARITH_F32 ? EXPORT_F32 : EXPORT_U16_SUM, c->rig.W,
                            c->rig.H, c->rig.d_max, (float*)tmp, c->st,
                            c->parts_live > 1 ? (const void*)(c->Sx[0] + sv * c->volcap) : nullptr,
                            c->parts_live > 2 ? (const void*)(c->Sx[1] + sv * c->volcap) : nullptr,
                            c->parts_live > 3 ? (const void*)(c->Sx[2] + sv * c->volcap) : nullptr);
      src = tmp;
      bytes = sizeof(float) * n;
      break;
    }
    default: {
      void* p;
      if (int e = es_ctx_device_ptr(c, what, seq, view, &p)) return e;
      src = p;
      const bool u8 = what == ES_PRED_VALID || what == ES_MEAS_VALID || what == ES_KEEP ||
                      what == ES_FUSED_VALID;
      bytes = HW * (u8 ? 1 : sizeof(double));
    }
  }
  CK(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, c->st));
  if (tmp) CK(cudaFreeAsync(tmp, c->st));
  CK(cudaStreamSynchronize(c->st));
  return ES_OK;
}

}  // extern "C"

extern "C" int es_ctx_export_all(es_ctx* c, int what, int view, void* out, int sync) {
  CK(cudaSetDevice(c->device));
  if (view < 0 || view > 1) return fail(ES_ERR_VALUE, "bad view");
  const size_t HW = c->HW;
  const int B = c->B;
  if (what == ES_FUSED_KITTI) {
    if (c->rig.d_max > 255) return fail(ES_ERR_VALUE, kKittiRange);
    // encode on the compute stream into one of two staging slots, copy out
    // on cp_out: the transfer overlaps the next step's kernels
    const int kb = c->kitti_slot;
    c->kitti_slot ^= 1;
    uint16_t* stage = c->kitti + (size_t)kb * HW * B;
    CK(cudaStreamWaitEvent(c->st, c->ev_kitti_free[kb], 0));
    k_kitti_batch<<<dim3((unsigned)((HW + 255) / 256), B), 256, 0, c->st>>>(
        c->sd[c->cur] + (size_t)view * HW, c->sv[c->cur] + (size_t)view * HW, HW, 2 * HW, stage);
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev_kitti_ready, c->st));
    CK(cudaStreamWaitEvent(c->cp_out, c->ev_kitti_ready, 0));
    CK(cudaMemcpyAsync(out, stage, sizeof(uint16_t) * HW * B, cudaMemcpyDeviceToHost, c->cp_out));
    CK(cudaEventRecord(c->ev_kitti_free[kb], c->cp_out));
    if (sync) CK(cudaStreamSynchronize(c->cp_out));
  } else {
    void* p;
    if (int e = es_ctx_device_ptr(c, what, 0, view, &p)) return e;
    const bool u8 = what == ES_PRED_VALID || what == ES_MEAS_VALID || what == ES_KEEP ||
                    what == ES_FUSED_VALID;
    const size_t es = u8 ? 1 : sizeof(double);
    CK(cudaMemcpy2DAsync(out, HW * es, p, 2 * HW * es, HW * es, B, cudaMemcpyDeviceToHost, c->st));
  }
  if (sync) CK(cudaStreamSynchronize(c->st));
  return ES_OK;
}

// ------------------------------------------------------------ stage level

namespace {
// stage-level scratch: stream-ordered allocations from the device's default
// memory pool, which keeps up to 4 GB of freed blocks cached (release
// threshold raised once per device), so repeated stage calls neither pay
// cudaMalloc / cudaFree nor their implicit device synchronisations
void keep_pool_cached() {
  static std::mutex mu;
  static uint64_t done = 0;   // bit per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  std::lock_guard<std::mutex> lock(mu);
  if (done >> dev & 1) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = 4ull << 30;   // bounded: big contexts still get their memory
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done |= 1ull << dev;
}

struct Scratch {
  std::vector<void*> ptrs;
  Scratch() { keep_pool_cached(); }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, 0);
  }
  template <class T>
  T* get(size_t n) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), 0) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return (T*)p;
  }
  template <class T>
  T* up(const T* h, size_t n) {
    T* d = get<T>(n);
    if (d && n) cudaMemcpy(d, h, sizeof(T) * n, cudaMemcpyHostToDevice);
    return d;
  }
};
#define NEED(p) \
  if (!(p)) return fail(ES_ERR_CUDA, "device allocation failed")
#define DONE()                                   \
  do {                                           \
    CK(cudaGetLastError());                      \
    CK(cudaDeviceSynchronize());                 \
  } while (0)

int check_lohi(const int64_t* lo, const int64_t* hi, size_t n, int d_max) {
  for (size_t i = 0; i < n; ++i)
    if (lo[i] < 0 || hi[i] > d_max || lo[i] > hi[i])
      return fail(ES_ERR_VALUE, "intervals must satisfy 0 <= lo <= hi <= d_max");
  return ES_OK;
}
}  // namespace

extern "C" int es_search_intervals(const double* d, const double* p, const uint8_t* v, int H, int W,
                        int d_max, int64_t* lo, int64_t* hi) {
  const size_t n = (size_t)H * W;
  Scratch s;
  double* dd = s.up(d, n);
  double* dp = s.up(p, n);
  uint8_t* dv = s.up(v, n);
  int64_t* dl = s.get<int64_t>(n);
  int64_t* dh = s.get<int64_t>(n);
  NEED(dd && dp && dv && dl && dh);
  launch_intervals_only(dd, dp, dv, (int)n, d_max, dl, dh, 0);
  DONE();
  CK(cudaMemcpy(lo, dl, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hi, dh, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

extern "C" int es_matching_cost(const uint8_t* left, const uint8_t* right, int H, int W, const int64_t* lo,
                     const int64_t* hi, int d_max, int window, int view, float* out) {
  const size_t n = (size_t)H * W;
  if (window < 3 || window % 2 == 0) return fail(ES_ERR_VALUE, "window must be odd and >= 3");
  if (window > 11) return fail(ES_ERR_UNSUPPORTED, "device cost storage supports window <= 11");
  if (d_max > 511 || d_max < 0) return fail(ES_ERR_UNSUPPORTED, "device path supports d_max <= 511");
  if (int e = check_lohi(lo, hi, n, d_max)) return e;
  Scratch s;
  uint8_t* img = s.get<uint8_t>(2 * n);
  NEED(img);
  CK(cudaMemcpy(img, left, n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(img + n, right, n, cudaMemcpyHostToDevice));
  int64_t* dl = s.up(lo, n);
  int64_t* dh = s.up(hi, n);
  uint2* meta = s.get<uint2>(n);
  const size_t volcap = (size_t)H * row_capacity(W, d_max);
  uint32_t* C = s.get<uint32_t>(volcap);
  float* dense = s.get<float>(n * (d_max + 1));
  NEED(dl && dh && meta && C && dense);
  launch_meta_from_intervals(dl, dh, W, H, d_max, meta, 0);
  CostArgs ca;
  ca.W = W;
  ca.H = H;
  ca.d_max = d_max;
  ca.window = window;
  ca.img = img;
  ca.meta = meta;
  ca.C = C;
  ca.volcap = volcap;
  ca.view0 = view;
  launch_cost(ca, 1, 0);
  launch_export_dense(meta, C, 0, W, H, d_max, dense, 0);
  DONE();
  CK(cudaMemcpy(out, dense, sizeof(float) * n * (d_max + 1), cudaMemcpyDeviceToHost));
  return ES_OK;
}

namespace {
// upload a dense volume into the ragged layout over each pixel's finite hull
int stage_volume(Scratch& s, const float* vol, int H, int W, int D, uint2** meta_out,
                 void** rag_out, int* f32_out, unsigned* flags_out) {
  const size_t n = (size_t)H * W;
  const int d_max = D - 1;
  float* dense = s.up(vol, n * D);
  int64_t* dl = s.get<int64_t>(n);
  int64_t* dh = s.get<int64_t>(n);
  unsigned* flags = s.get<unsigned>(1);
  uint2* meta = s.get<uint2>(n);
  NEED(dense && dl && dh && flags && meta);
  CK(cudaMemset(flags, 0, sizeof(unsigned)));
  launch_hull(dense, W, H, D, dl, dh, flags, (float)INF16, 0);
  launch_meta_from_intervals(dl, dh, W, H, d_max, meta, 0);
  DONE();
  unsigned f = 0;
  CK(cudaMemcpy(&f, flags, sizeof(unsigned), cudaMemcpyDeviceToHost));
  const int f32 = f != 0;   // anything but clean finite integer costs -> f32 storage
  const size_t volcap = (size_t)H * row_capacity(W, d_max);
  void* rag = f32 ? (void*)s.get<float2>(volcap) : (void*)s.get<uint32_t>(volcap);
  NEED(rag);
  launch_import_dense(dense, meta, W, H, D, f32, rag, 0);
  DONE();
  *meta_out = meta;
  *rag_out = rag;
  *f32_out = f32;
  *flags_out = f;
  return ES_OK;
}

int aggregate_staged(Scratch& s, uint2* meta, void* rag, int f32, unsigned flags, const float* vol,
                     int H, int W, int D, double p1, double p2, void** S_out, int* arith_out) {
  const size_t volcap = (size_t)H * row_capacity(W, D - 1);
  double cmax = 0;
  if (!f32) {
    // integer costs: bound by the largest value present
    const size_t n = (size_t)H * W * D;
    for (size_t i = 0; i < n; ++i)
      if (std::isfinite(vol[i]) && vol[i] > cmax) cmax = vol[i];
  }
  int arith = f32 ? ARITH_F32 : choose_arith(p1, p2, cmax);
  if (flags & 2u) arith = ARITH_F32;
  void* S = arith == ARITH_F32 ? (void*)s.get<float2>(volcap) : (void*)s.get<uint32_t>(volcap);
  NEED(S);
  void* C = rag;
  int cost_f32 = f32;
  if (arith == ARITH_F32 && !f32) cost_f32 = 0;
  SgmArgs sa;
  sa.W = W;
  sa.H = H;
  sa.d_max = D - 1;
  sa.meta = meta;
  sa.C = C;
  sa.S = S;
  sa.volcap = volcap;
  sa.cost_f32 = cost_f32;
  sa.p1i = (uint32_t)p1;
  sa.p2i = (uint32_t)p2;
  sa.p1 = (float)p1;
  sa.p2 = (float)p2;
  launch_aggregate(sa, arith, 1, 0);
  DONE();
  *S_out = S;
  *arith_out = arith;
  return ES_OK;
}
}  // namespace

extern "C" {

int es_aggregate_paths(const float* vol, int H, int W, int D, double p1, double p2, float* out) {
  if (D - 1 > 511) return fail(ES_ERR_UNSUPPORTED, "device path supports d_max <= 511");
  if (!(0 < p1 && p1 <= p2)) return fail(ES_ERR_VALUE, "penalties must satisfy 0 < P1 <= P2");
  Scratch s;
  uint2* meta;
  void* rag;
  int f32;
  unsigned flags;
  if (int e = stage_volume(s, vol, H, W, D, &meta, &rag, &f32, &flags)) return e;
  if (flags & 6u) return fail(ES_ERR_UNSUPPORTED, "volume has an all-inf pixel or NaN");
  void* S;
  int arith;
  if (int e = aggregate_staged(s, meta, rag, f32, flags, vol, H, W, D, p1, p2, &S, &arith)) return e;
  const size_t n = (size_t)H * W * D;
  float* dense = s.get<float>(n);
  NEED(dense);
  launch_export_dense(meta, S, arith == ARITH_F32 ? EXPORT_F32 : EXPORT_U16_SUM, W, H, D - 1,
                      dense, 0);
  DONE();
  CK(cudaMemcpy(out, dense, sizeof(float) * n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_select_disparity(const float* vol, int H, int W, int D, double* d, uint8_t* valid) {
  if (D - 1 > 511) return fail(ES_ERR_UNSUPPORTED, "device path supports d_max <= 511");
  Scratch s;
  uint2* meta;
  void* rag;
  int f32;
  unsigned flags;
  if (int e = stage_volume(s, vol, H, W, D, &meta, &rag, &f32, &flags)) return e;
  if (flags & 4u) return fail(ES_ERR_UNSUPPORTED, "volume has NaN");
  const size_t n = (size_t)H * W;
  uint16_t* ds = s.get<uint16_t>(n);
  double* r = s.get<double>(n);
  uint8_t* v = s.get<uint8_t>(n);
  double* dd = s.get<double>(n);
  NEED(ds && r && v && dd);
  WtaArgs wa;
  wa.W = W;
  wa.H = H;
  wa.meta = meta;
  wa.S = rag;
  wa.volcap = (size_t)H * row_capacity(W, D - 1);
  wa.d_max = D - 1;
  wa.arith = f32 ? ARITH_F32 : ARITH_U16;
  wa.s_max = 1.0;
  wa.r_min = 1.0;
  wa.dstar = ds;
  wa.r = r;
  wa.valid = v;
  launch_wta_variance(wa, 1, 0);
  k_u16_to_f64<<<(unsigned)((n + 255) / 256), 256>>>(ds, n, dd);
  DONE();
  CK(cudaMemcpy(d, dd, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(valid, v, n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_matching_variance_map(const float* vol, const int64_t* lo, const int64_t* hi,
                             const double* d, int H, int W, int D, double s_max, double r_min,
                             double* r_out) {
  // caller winners d (select_disparity's output in the reference pipeline)
  const size_t n = (size_t)H * W;
  if (int e = check_lohi(lo, hi, n, D - 1)) return e;
  Scratch s;
  int64_t* dl = s.up(lo, n);
  int64_t* dh = s.up(hi, n);
  uint2* meta = s.get<uint2>(n);
  float* dense = s.up(vol, n * D);
  NEED(dl && dh && meta && dense);
  launch_meta_from_intervals(dl, dh, W, H, D - 1, meta, 0);
  const size_t volcap = (size_t)H * row_capacity(W, D - 1);
  float2* rag = s.get<float2>(volcap);
  NEED(rag);
  launch_import_dense(dense, meta, W, H, D, 1, rag, 0);
  std::vector<uint16_t> hd(n);
  for (size_t i = 0; i < n; ++i) {
    if (!(d[i] >= 0 && d[i] < D) || d[i] != (double)(int)d[i])
      return fail(ES_ERR_UNSUPPORTED, "matching_variance_map: disparities must be integers in [0, D)");
    hd[i] = (uint16_t)d[i];
  }
  uint16_t* ds_in = s.up(hd.data(), n);
  uint16_t* ds = s.get<uint16_t>(n);
  double* r = s.get<double>(n);
  uint8_t* v = s.get<uint8_t>(n);
  NEED(ds_in && ds && r && v);
  WtaArgs wa;
  wa.dstar_in = ds_in;
  wa.W = W;
  wa.H = H;
  wa.meta = meta;
  wa.S = rag;
  wa.volcap = volcap;
  wa.arith = ARITH_F32;
  wa.s_max = s_max;
  wa.r_min = r_min;
  wa.dstar = ds;
  wa.r = r;
  wa.valid = v;
  launch_wta_variance(wa, 1, 0);
  DONE();
  CK(cudaMemcpy(r_out, r, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_lr_consistency(const double* dl, const uint8_t* vl, const double* dr, const uint8_t* vr,
                      int H, int W, double tau, uint8_t* kl, uint8_t* kr) {
  const size_t n = (size_t)H * W;
  Scratch s;
  double* a = s.up(dl, n);
  uint8_t* b = s.up(vl, n);
  double* c = s.up(dr, n);
  uint8_t* d = s.up(vr, n);
  uint8_t* o1 = s.get<uint8_t>(n);
  uint8_t* o2 = s.get<uint8_t>(n);
  NEED(a && b && c && d && o1 && o2);
  launch_lr(a, b, c, d, W, H, tau, o1, o2, 0);
  DONE();
  CK(cudaMemcpy(kl, o1, n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(kr, o2, n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_sad_check(const uint8_t* left, const uint8_t* right, const double* d, const uint8_t* v,
                 int H, int W, int window, double tau, int view, uint8_t* keep) {
  const size_t n = (size_t)H * W;
  Scratch s;
  uint8_t* l = s.up(left, n);
  uint8_t* r = s.up(right, n);
  double* dd = s.up(d, n);
  uint8_t* dv = s.up(v, n);
  uint8_t* o = s.get<uint8_t>(n);
  NEED(l && r && dd && dv && o);
  launch_sad_check(l, r, dd, dv, W, H, window, tau, view, o, 0);
  DONE();
  CK(cudaMemcpy(keep, o, n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_fuse_maps(const double* dp, const double* pp, const uint8_t* vp, const double* dm,
                 const double* rm, const uint8_t* vm, int n, double p_init, double* od,
                 double* op, uint8_t* ov) {
  Scratch s;
  double* a = s.up(dp, n);
  double* b = s.up(pp, n);
  uint8_t* c = s.up(vp, n);
  double* d = s.up(dm, n);
  double* e = s.up(rm, n);
  uint8_t* f = s.up(vm, n);
  double* g = s.get<double>(n);
  double* h = s.get<double>(n);
  uint8_t* k = s.get<uint8_t>(n);
  NEED(a && b && c && d && e && f && g && h && k);
  launch_fuse(a, b, c, d, e, f, n, p_init, g, h, k, 0);
  DONE();
  CK(cudaMemcpy(od, g, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(op, h, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ov, k, n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_predict_view(const double* d, const double* p, const uint8_t* valid, const double* Hm,
                    const es_rig* rig, const es_params* prm, double* od, double* op, uint8_t* ov) {
  const size_t n = (size_t)rig->width * rig->height;
  Scratch s;
  PredArgs a;
  a.rig = to_rig(rig);
  a.prm = to_params(prm);
  a.prm.fill_holes = 0;   // _predict_view alone: fill is a separate stage
  uint8_t one = 1;
  a.Hm = s.up(Hm, 16);
  a.have_pred = s.up(&one, 1);
  a.sd = s.up(d, n);
  a.sp = s.up(p, n);
  a.sv = s.up(valid, n);
  a.zkey = s.get<unsigned long long>(n);
  a.zidx = s.get<uint32_t>(n);
  a.wt = s.get<uint32_t>(n);
  a.wd = s.get<double>(n);
  a.hd = s.get<double>(n);
  a.hp = s.get<double>(n);
  a.hv = s.get<uint8_t>(n);
  a.pd = nullptr;
  a.pp = nullptr;
  a.pv = nullptr;
  a.meta = nullptr;
  a.cells = nullptr;
  a.err = s.get<int>(1);
  NEED(a.Hm && a.have_pred && a.sd && a.sp && a.sv && a.zkey && a.zidx && a.wt && a.wd && a.hd &&
       a.hp && a.hv &&
       a.err);
  CK(cudaMemset(a.err, 0, sizeof(int)));
  launch_predict(a, 1, 0);
  DONE();
  int err = 0;
  CK(cudaMemcpy(&err, a.err, sizeof(int), cudaMemcpyDeviceToHost));
  if (err & ERR_POINT_AT_INFINITY)
    return fail(ES_ERR_POINT_AT_INFINITY, "warped point has ~zero fourth homogeneous component");
  if (err & ERR_NONPOSITIVE_D) return fail(ES_ERR_NONPOSITIVE_D, "previous disparity must be positive");
  CK(cudaMemcpy(od, a.hd, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(op, a.hp, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ov, a.hv, n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_fill_zoom_holes(const double* d, const double* p, const uint8_t* valid, int H, int W,
                       double gamma_f, double q, double* od, double* op, uint8_t* ov) {
  const size_t n = (size_t)H * W;
  Scratch s;
  double* d0 = s.up(d, n);
  double* p0 = s.up(p, n);
  uint8_t* v0 = s.up(valid, n);
  double* d1 = s.get<double>(n);
  double* p1 = s.get<double>(n);
  uint8_t* v1 = s.get<uint8_t>(n);
  NEED(d0 && p0 && v0 && d1 && p1 && v1);
  launch_fill_axis(d0, p0, v0, W, H, 1, gamma_f, q, d1, p1, v1, 0, 0);
  launch_fill_axis(d1, p1, v1, W, H, 0, gamma_f, q, d0, p0, v0, 1, 0);
  DONE();
  CK(cudaMemcpy(od, d0, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(op, p0, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ov, v0, n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_reject_edges(const double* d, const uint8_t* valid, int H, int W, double gamma_e,
                    int edge_window, uint8_t* out) {
  const size_t n = (size_t)H * W;
  Scratch s;
  double* dd = s.up(d, n);
  uint8_t* dv = s.up(valid, n);
  uint8_t* o = s.get<uint8_t>(n);
  NEED(dd && dv && o);
  launch_edges(dd, dv, W, H, edge_window, gamma_e, o, 0);
  DONE();
  CK(cudaMemcpy(out, o, n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

}  // extern "C"

namespace {
// sgm._box_sum (sgm.py:130-136): exact integer window sums over a
// (2r+1)^2 window with edge replication; one thread per output
__global__ void k_box_sum(const long long* a, int H, int W, int r, long long* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= H * W) return;
  const int x = i % W, y = i / W;
  long long s = 0;
  for (int dy = -r; dy <= r; ++dy) {
    const long long* row = a + (size_t)min(max(y + dy, 0), H - 1) * W;
    for (int dx = -r; dx <= r; ++dx) s += row[min(max(x + dx, 0), W - 1)];
  }
  out[i] = s;
}

// sgm.matching_variance (sgm.py:287-316), the scalar walk in float64 over
// one pixel's interval costs: rel = c - c[center]; count neighbours while the
// running sum stays below s_max, outward on each side (one thread)
__global__ void k_variance_scalar(const double* c, int n, int center, double s_max,
                                  double r_min, double* out) {
  const double cs = c[center];
  int cnt = 0;
  double s = 0.0;
  for (int i = center - 1; i >= 0; --i) {
    s += c[i] - cs;
    if (s >= s_max) break;
    ++cnt;
  }
  s = 0.0;
  for (int i = center + 1; i < n; ++i) {
    s += c[i] - cs;
    if (s >= s_max) break;
    ++cnt;
  }
  *out = fmax((double)cnt, r_min);
}
}  // namespace

extern "C" {

int es_box_sum(const int64_t* a, int H, int W, int radius, int64_t* out) {
  if (H < 1 || W < 1 || radius < 0) return fail(ES_ERR_VALUE, "box_sum: bad shape or radius");
  const size_t n = (size_t)H * W;
  Scratch s;
  long long* da = (long long*)s.up(a, n);
  long long* dout = s.get<long long>(n);
  NEED(da && dout);
  k_box_sum<<<(unsigned)((n + 255) / 256), 256>>>(da, H, W, radius, dout);
  DONE();
  CK(cudaMemcpy(out, dout, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_matching_variance_scalar(const double* costs, int n, int center, double s_max,
                                double r_min, double* r) {
  if (n < 1 || center < 0 || center >= n)
    return fail(ES_ERR_VALUE, "selected disparity outside the interval");
  Scratch s;
  double* dc = s.up(costs, (size_t)n);
  double* dr = s.get<double>(1);
  NEED(dc && dr);
  k_variance_scalar<<<1, 1>>>(dc, n, center, s_max, r_min, dr);
  DONE();
  CK(cudaMemcpy(r, dr, sizeof(double), cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_warp_points(const double* Hm, const double* pts, int n, double* out) {
  Scratch s;
  double* dH = s.up(Hm, 16);
  double* dp = s.up(pts, 3 * (size_t)n);
  double* dout = s.get<double>(3 * (size_t)n);
  int* err = s.get<int>(1);
  NEED(dH && dp && dout && err);
  CK(cudaMemset(err, 0, sizeof(int)));
  k_warp_points<<<(n + 255) / 256, 256>>>(dH, dp, n, dout, err);
  DONE();
  int e = 0;
  CK(cudaMemcpy(&e, err, sizeof(int), cudaMemcpyDeviceToHost));
  if (e) return fail(ES_ERR_POINT_AT_INFINITY, "warped point has ~zero fourth homogeneous component");
  CK(cudaMemcpy(out, dout, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
  return ES_OK;
}

int es_render_prims(const es_rig* rig, const double* prims, int n_prim, const double* poses,
                    const int64_t* seeds, int n_seq, double texture_scale, int background,
                    uint8_t* out_dev, double* gt_dev, void* stream) {
  Scratch s;
  RenderArgs a;
  a.rig = to_rig(rig);
  a.prims = s.up(prims, (size_t)n_seq * n_prim * 8);
  a.n_prim = n_prim;
  a.poses = s.up(poses, (size_t)n_seq * 16);
  a.seeds = (const long long*)s.up(seeds, (size_t)n_seq);
  a.texture_scale = texture_scale;
  a.background = background;
  a.img = out_dev;
  a.gt = gt_dev;
  NEED(a.prims && a.poses && a.seeds);
  launch_render(a, n_seq, (cudaStream_t)stream);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  return ES_OK;
}

int es_render(const es_rig* rig, const double* boxes, int n_box, const double* poses,
              const int64_t* seeds, int n_seq, double texture_scale, int background,
              uint8_t* out_dev, double* gt_dev, void* stream) {
  if (n_box < 0 || n_seq < 0) return fail(ES_ERR_VALUE, "es_render: negative count");
  std::vector<double> prims((size_t)n_seq * n_box * 8, 0.0);
  for (size_t k = 0; k < (size_t)n_seq * n_box; ++k)
    for (int j = 0; j < 6; ++j) prims[8 * k + 1 + j] = boxes[6 * k + j];
  return es_render_prims(rig, prims.data(), n_box, poses, seeds, n_seq, texture_scale,
                         background, out_dev, gt_dev, stream);
}

}  // extern "C"

// ---- evaluation metrics (metrics.py:39-117) ----------------------------------
extern "C" int es_bad_pixel_counts(const double* est, const uint8_t* est_valid, const double* gt,
                                   const uint8_t* gt_valid, int64_t n, int n_maps, int mode,
                                   uint64_t* counts, uint8_t* mask, uint8_t* rgb) {
  if (n < 0 || n_maps < 0) return fail(ES_ERR_VALUE, "bad map size");
  if (mode != 0 && mode != 1) return fail(ES_ERR_VALUE, "mode must be 'or' or 'and'");
  if (n_maps == 0) return ES_OK;
  const size_t N = (size_t)n * n_maps;
  Scratch s;
  MetricsArgs a;
  a.est = s.up(est, N);
  a.est_valid = s.up(est_valid, N);
  a.gt = s.up(gt, N);
  a.gt_valid = s.up(gt_valid, N);
  a.counts = s.get<unsigned long long>(4 * (size_t)n_maps);
  a.mask = mask ? s.get<uint8_t>(N) : nullptr;
  a.rgb = rgb ? s.get<uint8_t>(3 * N) : nullptr;
  NEED(a.est && a.est_valid && a.gt && a.gt_valid && a.counts && (!mask || a.mask) &&
       (!rgb || a.rgb));
  a.n = (size_t)n;
  a.stride_e = a.stride_g = (size_t)n;
  a.mode = mode;
  CK(cudaMemset(a.counts, 0, sizeof(unsigned long long) * 4 * n_maps));
  if (n) launch_metrics(a, n_maps, 0);
  DONE();
  CK(cudaMemcpy(counts, a.counts, sizeof(uint64_t) * 4 * n_maps, cudaMemcpyDeviceToHost));
  if (mask) CK(cudaMemcpy(mask, a.mask, N, cudaMemcpyDeviceToHost));
  if (rgb) CK(cudaMemcpy(rgb, a.rgb, 3 * N, cudaMemcpyDeviceToHost));
  return ES_OK;
}

extern "C" int es_ctx_metrics(es_ctx* c, int view, const double* gt_dev, const uint8_t* gt_valid_dev,
                              int64_t gt_stride, int mode, uint64_t* counts) {
  if (view < 0 || view > 1) return fail(ES_ERR_VALUE, "view must be 0 or 1");
  if (mode != 0 && mode != 1) return fail(ES_ERR_VALUE, "mode must be 'or' or 'and'");
  CK(cudaSetDevice(c->device));
  unsigned long long* dc = nullptr;
  CK(cudaMallocAsync((void**)&dc, sizeof(unsigned long long) * 4 * c->B, c->st));
  CK(cudaMemsetAsync(dc, 0, sizeof(unsigned long long) * 4 * c->B, c->st));
  MetricsArgs a;
  a.est = c->sd[c->cur] + (size_t)view * c->HW;
  a.est_valid = c->sv[c->cur] + (size_t)view * c->HW;
  a.gt = gt_dev;
  a.gt_valid = gt_valid_dev;
  a.n = c->HW;
  a.stride_e = 2 * c->HW;
  a.stride_g = (size_t)gt_stride;
  a.mode = mode;
  a.counts = dc;
  launch_metrics(a, c->B, c->st);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(counts, dc, sizeof(uint64_t) * 4 * c->B, cudaMemcpyDeviceToHost, c->st));
  CK(cudaFreeAsync(dc, c->st));
  CK(cudaStreamSynchronize(c->st));
  return ES_OK;
}

// make the compute stream wait for every transfer issued so far (so an event
// recorded on it afterwards covers the last export's device->host copy)
extern "C" int es_ctx_fence(es_ctx* c) {
  CK(cudaSetDevice(c->device));
  CK(cudaEventRecord(c->ev_join, c->cp_out));
  CK(cudaStreamWaitEvent(c->st, c->ev_join, 0));
  return ES_OK;
}
