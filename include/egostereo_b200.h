/* egostereo_b200.h -- C ABI of the B200-native egostereo hot path.
 *
 * Drop-in boundary for the reference package egostereo (arXiv 1708.06301,
 * /root/reference/pkg/src/egostereo).  The reference has no FFI: its
 * operator API is its Python function surface, which the host package
 * paper_1708_06301_b200 mirrors name for name and implements by calling the
 * entry points below through ctypes.
 *
 * Conventions
 *   - plain C types only; every array is row-major (H, W) unless noted;
 *     "host" pointers are ordinary (preferably pinned) CPU memory, "dev"
 *     pointers are CUDA device memory on the context's / current device;
 *   - every call returns an es_status; es_last_error() returns a
 *     thread-local message for the last failure on the calling thread;
 *   - the library owns its device buffers; callers own host arrays;
 *   - distinct contexts may be used from distinct threads concurrently.
 */
#ifndef EGOSTEREO_B200_H
#define EGOSTEREO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ES_OK = 0,
  ES_ERR_VALUE = 1,              /* ValueError (shapes, parameters)              */
  ES_ERR_POINT_AT_INFINITY = 2,  /* geometry.PointAtInfinityError                */
  ES_ERR_NONPOSITIVE_D = 3,      /* prediction.propagate_variance ValueError     */
  ES_ERR_CUDA = 4,               /* RuntimeError: CUDA failure                    */
  ES_ERR_UNSUPPORTED = 5         /* configuration outside the device envelope    */
} es_status;

/* StereoRig (core.py:18-55) */
typedef struct {
  double f, b, cx, cy;
  int32_t width, height, d_max;
} es_rig;

/* SgmParams (sgm.py:28-60) + PredictionParams (prediction.py:23-47) +
 * FusionParams (fusion.py:19-27) + PipelineParams.baseline (pipeline.py:75-82) */
typedef struct {
  int32_t window;
  double p1, p2, s_max, r_min, tau_lr, tau_sad;
  double q, gamma_f, gamma_e;
  int32_t edge_window, edge_reject, fill_holes;
  double p_init;
  int32_t baseline;
} es_params;

typedef struct es_ctx es_ctx;

const char* es_last_error(void);
int es_version(void);
int es_device_count(int* n);

/* ---- pipeline contexts: DisparityPipeline (pipeline.py:90-170), batched over
 *      `batch` independent sequences that advance one frame per call ------- */
int es_ctx_create(int device, const es_rig* rig, const es_params* prm, int batch, es_ctx** out);
int es_ctx_destroy(es_ctx* ctx);
/* DisparityPipeline.reset (pipeline.py:98-99) for every sequence */
int es_ctx_reset(es_ctx* ctx);
/* DisparityPipeline.process_frame (pipeline.py:108-170) for all sequences.
 *   images      [batch][2][H][W] uint8 (left, right); host or dev (images_dev)
 *   homographies [batch][2][16] f64: disparity_homography(rig, T) for the
 *               left view and disparity_homography(rig, right_motion(rig, T))
 *               for the right view (geometry.py:62-92); ignored where
 *               motion_given[s] == 0
 *   motion_given [batch] uint8: motion is not None for sequence s
 *   sync        1: wait, check errors, commit state only on success (the
 *                  reference raises before it updates its state)
 *               0: enqueue only; the step's state is committed before its
 *                  error bits are known.  Errors surface in es_ctx_sync (or
 *                  the next synced step) in the reference's order -- first
 *                  failing sequence, left view before right, point at
 *                  infinity before d <= 0 -- and then leave the context
 *                  POISONED: further steps return ES_ERR_VALUE until
 *                  es_ctx_reset.                                          */
int es_ctx_step(es_ctx* ctx, const uint8_t* images, int images_dev, const double* homographies,
                const uint8_t* motion_given, int sync);
int es_ctx_sync(es_ctx* ctx);
/* make the context's compute stream wait for every host<->device transfer
 * issued so far (input uploads run on a copy stream, es_ctx_export_all's
 * KITTI copies on another), so an event recorded on the compute stream
 * afterwards also covers the last export */
int es_ctx_fence(es_ctx* ctx);
/* frame counter of sequence s (FilterState.frame) and searched cells per view */
int es_ctx_frame(es_ctx* ctx, int seq, int64_t* frame);
int es_ctx_cells(es_ctx* ctx, int seq, uint64_t* cells_left, uint64_t* cells_right);
/* searched cells summed over all sequences, views and steps since the last
 * reset (syncs the context stream) */
int es_ctx_cells_acc(es_ctx* ctx, uint64_t* total, int reset);
/* pipeline.py:122 have_state of sequence s after the last synced step */
int es_ctx_have_state(es_ctx* ctx, int seq, int64_t* have);
/* per-stage CUDA-event timing on the context's stream: when enabled every
 * step records events around its 6 stages (predict, intervals, cost,
 * aggregate, wta+variance, checks+fuse); es_ctx_stage_times syncs, returns the
 * summed milliseconds per stage over the recorded steps and clears them */
int es_ctx_profile(es_ctx* ctx, int enable);
int es_ctx_stage_times(es_ctx* ctx, double* ms6, int64_t* steps);
/* scheduling hint for a batch split over several contexts of one device
 * (BatchedPipeline groups): total_batch = sequences of ALL cooperating
 * contexts.  The SGM aggregation picks its GPU-filling schedule (fused
 * vertical+diagonal sweeps, one SM per view) when the contexts together
 * bring at least 64 views, although this context alone would not.  Results
 * do not depend on it.  0 (default): this context's own batch decides. */
int es_ctx_shared_batch(es_ctx* ctx, int total_batch);

/* FrameResult materialisation (pipeline.py:53-72) of the last step into
 * host memory; `what` selects the map, `view` 0 = left, 1 = right. */
enum {
  ES_PRED_D = 0, ES_PRED_P, ES_PRED_VALID,         /* f64, f64, u8       */
  ES_LO, ES_HI,                                    /* int64              */
  ES_MEAS_D, ES_MEAS_VALID, ES_MEAS_R,             /* f64, u8, f64       */
  ES_KEEP,                                         /* u8                 */
  ES_FUSED_D, ES_FUSED_P, ES_FUSED_VALID,          /* f64, f64, u8       */
  ES_COST_DENSE, ES_TOTAL_DENSE,                   /* f32 (H, W, d_max+1) */
  ES_FUSED_KITTI                                   /* u16 round(256 d), 0 = invalid */
};
int es_ctx_export(es_ctx* ctx, int what, int seq, int view, void* host_out);
/* one map of one view for all `batch` sequences into host_out [batch][H][W]
 * (no dense volumes); sync = 0 only enqueues the work (ES_FUSED_KITTI: the
 * encode on the context stream, the copy on the export stream -- see
 * es_ctx_fence / es_ctx_sync); host_out must stay valid until then */
int es_ctx_export_all(es_ctx* ctx, int what, int view, void* host_out, int sync);
/* device pointer of a per-sequence map (what as above, no dense volumes) */
int es_ctx_device_ptr(es_ctx* ctx, int what, int seq, int view, void** dev_ptr);
/* stream the context launches on (cudaStream_t) */
int es_ctx_stream(es_ctx* ctx, void** stream);

/* ---- stage-level entry points (host arrays in, host arrays out) --------- */
/* sgm.search_intervals (sgm.py:105-127) */
int es_search_intervals(const double* d, const double* p, const uint8_t* valid, int H, int W,
                        int d_max, int64_t* lo, int64_t* hi);
/* sgm.matching_cost (sgm.py:160-196): dense f32 (H, W, d_max+1), +inf outside */
int es_matching_cost(const uint8_t* left, const uint8_t* right, int H, int W, const int64_t* lo,
                     const int64_t* hi, int d_max, int window, int view, float* out);
/* sgm.aggregate_paths (sgm.py:257-272) on a dense f32 volume */
int es_aggregate_paths(const float* vol, int H, int W, int D, double p1, double p2, float* out);
/* sgm.select_disparity (sgm.py:275-284) */
int es_select_disparity(const float* vol, int H, int W, int D, double* d, uint8_t* valid);
/* sgm.matching_variance_map (sgm.py:319-344) */
int es_matching_variance_map(const float* vol, const int64_t* lo, const int64_t* hi,
                             const double* d, int H, int W, int D, double s_max, double r_min,
                             double* r);
/* sgm.lr_consistency (sgm.py:347-370) */
int es_lr_consistency(const double* dl, const uint8_t* vl, const double* dr, const uint8_t* vr,
                      int H, int W, double tau_lr, uint8_t* keep_l, uint8_t* keep_r);
/* sgm.sad_check (sgm.py:373-396) */
int es_sad_check(const uint8_t* left, const uint8_t* right, const double* d, const uint8_t* valid,
                 int H, int W, int window, double tau_sad, int view, uint8_t* keep);
/* fusion.fuse_maps (fusion.py:45-79) */
int es_fuse_maps(const double* dp, const double* pp, const uint8_t* vp, const double* dm,
                 const double* rm, const uint8_t* vm, int n, double p_init, double* od,
                 double* op, uint8_t* ov);
/* prediction._predict_view (prediction.py:80-126) with an explicit H */
int es_predict_view(const double* d, const double* p, const uint8_t* valid, const double* Hm,
                    const es_rig* rig, const es_params* prm, double* od, double* op, uint8_t* ov);
/* prediction.fill_zoom_holes (prediction.py:169-183) */
int es_fill_zoom_holes(const double* d, const double* p, const uint8_t* valid, int H, int W,
                       double gamma_f, double q, double* od, double* op, uint8_t* ov);
/* prediction.reject_edges (prediction.py:50-64) */
int es_reject_edges(const double* d, const uint8_t* valid, int H, int W, double gamma_e,
                    int edge_window, uint8_t* out);

/* sgm._box_sum (sgm.py:130-136): exact integer (2r+1)^2 window sums with
 * edge replication, a (H, W) -> out (H, W) */
int es_box_sum(const int64_t* a, int H, int W, int radius, int64_t* out);
/* sgm.matching_variance (sgm.py:287-316): the scalar float64 walk over one
 * pixel's n interval costs from index center */
int es_matching_variance_scalar(const double* costs, int n, int center, double s_max,
                                double r_min, double* r);

/* geometry.warp_point (geometry.py:95-115) on n principal-point-relative
 * (x, y, d) triples; out (n, 3) */
int es_warp_points(const double* Hm, const double* pts, int n, double* out);

/* ---- evaluation metrics (metrics.py:39-117) -------------------------------
 * metrics.bad_pixel_rate / bad_pixel_mask / error_image / density on n_maps
 * host maps of n pixels ([n_maps][n], f64 values + u8 valid); mode 0 = "or"
 * (|err| > 3 px OR > 5 %), 1 = "and" (KITTI 2015).
 *   counts [n_maps][4]: ground-truth valid, jointly valid, bad, estimate valid
 *   mask   optional [n_maps][n] u8 (bad_pixel_mask), rgb optional
 *          [n_maps][n][3] u8 (error_image); NULL to skip                    */
int es_bad_pixel_counts(const double* est, const uint8_t* est_valid, const double* gt,
                        const uint8_t* gt_valid, int64_t n, int n_maps, int mode,
                        uint64_t* counts, uint8_t* mask, uint8_t* rgb);
/* the same counts for every sequence's fused map of `view` in a context,
 * against device ground truth (sequence s at gt_dev + s * gt_stride, H*W
 * values); counts is host [batch][4]; enqueued on the context's stream
 * behind any deferred step and synchronised once (one 32*batch-byte read) */
int es_ctx_metrics(es_ctx* ctx, int view, const double* gt_dev, const uint8_t* gt_valid_dev,
                   int64_t gt_stride, int mode, uint64_t* counts);

/* ---- synthetic input renderer (synth.py:87-218 restated bit-exactly) -----
 * Not on the hot path: generates the bench / parity inputs on the device;
 * its bytes equal synth.render_frame's (tests/test_gpu_render.py).
 * prims [n_seq][n_prim][8] records: [0, x0, x1, y0, y1, z0, z1, 0] = Box
 * (synth.py:41-50); [1, z, x0, x1, y0, y1, 0, flags] = Plane (synth.py:27-38),
 * flags bits 0..3 = bound x0, x1, y0, y1 present (None otherwise);
 * poses [n_seq][16] world-from-camera, seeds [n_seq] texture seeds; out_dev
 * images [n_seq][2][H][W] (device); gt_dev optional [n_seq][2][H][W] f64 */
int es_render_prims(const es_rig* rig, const double* prims, int n_prim, const double* poses,
                    const int64_t* seeds, int n_seq, double texture_scale, int background,
                    uint8_t* out_dev, double* gt_dev, void* stream);
/* boxes only: boxes [n_seq][n_box][6] (x0, x1, y0, y1, z0, z1) */
int es_render(const es_rig* rig, const double* boxes, int n_box, const double* poses,
              const int64_t* seeds, int n_seq, double texture_scale, int background,
              uint8_t* out_dev, double* gt_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EGOSTEREO_B200_H */
