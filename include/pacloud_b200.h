/*
 * pacloud_b200 -- C ABI of the B200 (sm_100a) hot path of 4D SlingBAG.
 *
 * Every entry point takes plain device pointers and sizes, is asynchronous on
 * the caller's CUDA stream (`pc_stream_t` is a cudaStream_t; NULL = legacy
 * default stream), allocates nothing persistent, and returns PC_OK or a
 * nonzero status (argument error / CUDA launch error).  Data errors travel
 * through device flag words that the host reads with the loss, once per
 * iteration.  Each function cites the reference (read-only, pkg/src/pacloud)
 * interface it replaces; the host-side mirror of the reference's Python
 * signatures lives in paper_2412_03898_b200/ and INTEGRATION.md shows the
 * ctypes binding a maintainer would add to the reference.
 *
 * Layouts (row-major, frame-major):
 *   ball states   mu_t (F,B,3) f64, a0_t (F,B) f32, p0_t (F,B) f32
 *   traces        (F,M,T) f32           (SignalSet.data is (M,K,T) upstream)
 *   state grads   G (F,B,5) f32 in state order (a0, p0, mu_x, mu_y, mu_z)
 *   parameters    f64 master copies; gradients f32; Adam moments f64
 */
#ifndef PACLOUD_B200_H
#define PACLOUD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void *pc_stream_t;

#define PC_OK 0
#define PC_ERR_ARGUMENT 1
#define PC_ERR_CUDA 2
#define PC_ERR_UNSUPPORTED 3

/* coord_mode (core.py:21-24 COORD_MODES) */
#define PC_COORD_MULTIPLICATIVE 0
#define PC_COORD_ADDITIVE 1
#define PC_COORD_RADIAL 2

/* basis_kind: reference Gaussian basis (deformation.py:57-99) or the
 * builder-defined cubic-polynomial + Fourier basis of BASELINE configs 2-5 */
#define PC_BASIS_GAUSS 0
#define PC_BASIS_POLYFOURIER 1

/* SensorArray (core.py:295-354) plus the radiator knobs
 * (radiator.py:195-197: support_sigmas, exact). */
typedef struct pc_array {
    const double *positions; /* device, (M,3) mm */
    int32_t n_sensors;       /* M */
    int32_t n_samples;       /* T */
    double sound_speed;      /* mm/us */
    double t_start;          /* us */
    double dt;               /* us, 1/sample_rate (core.py:345-347) */
    double support_sigmas;   /* radiator.py:31 DEFAULT_SUPPORT_SIGMAS */
    int32_t exact;           /* evaluate every sample (radiator.py:100-102) */
    int32_t sensor_offset;   /* global index of local sensor 0 (sensor
                                sharding; 0 for a whole array) */
    const int32_t *sensor_order; /* device, (M,) processing order of the
                                    sensors (spatially clustered) or NULL;
                                    outputs stay in sensor index order */
    int32_t n_sensors_total; /* sensors of the whole array (0 = n_sensors) */
    int32_t frame_offset;    /* global position of local frame 0 in the
                                iteration's frame list (frame sharding) */
} pc_array_t;

/* Coincidence word (radiator.py:97-99): the kernels atomicMin
 *   ((frame_offset + f) * B + b) * n_sensors_total + sensor_offset + m
 * over every pair (f, b, m) with R < 1e-9 into a device int64 that holds
 * INT64_MAX on entry; one frame of a whole array gives b * M + m. */

/* DynamicCloud (core.py:166-259), device f64 arrays.
 * Gaussian basis: theta/sigma (B,N) shared or (B,5,N) per-channel.
 * Poly+Fourier basis: theta/sigma unused (may be NULL), N = 4 + 2*harmonics. */
typedef struct pc_cloud {
    const double *p0;    /* (B,)   */
    const double *a0;    /* (B,)   */
    const double *mu;    /* (B,3)  */
    const double *theta; /* (B,N) or (B,5,N) */
    const double *sigma; /* same shape as theta */
    const double *omega; /* (B,5,N) */
    int64_t n_balls;
    int32_t n_basis;
    int32_t per_channel; /* theta/sigma are (B,5,N) */
    int32_t basis_kind;  /* PC_BASIS_* */
    int32_t reserved;
} pc_cloud_t;

/* Parameter-gradient outputs (radiator.py:245-263 CloudGrads), device f32. */
typedef struct pc_cloud_grads {
    float *p0;    /* (B,)  */
    float *a0;    /* (B,)  */
    float *mu;    /* (B,3) */
    float *theta; /* like cloud.theta (unused for poly+Fourier) */
    float *sigma;
    float *omega; /* (B,5,N) */
} pc_cloud_grads_t;

/* ---- deformation ------------------------------------------------------ */

/* Replaces deformation.py:184-204 cloud_states_at, batched over F frames
 * (the reference calls it once per frame, reconstruction.py:305).
 * a0_floor NaN disables the clamp (a0_floor=None); any other value clamps
 * a0_t = max(a0 (1 + H0), a0_floor) as deformation.py:202-203 does.  H
 * (F,B,5) f32 receives the channel sums for pc_deform_backward (may be
 * NULL), with H[...,0] = NaN where the floor clamped (the backward's
 * subgradient flag, deformation.py:257-264, decided here in fp64). */
int pc_deform_states(const pc_cloud_t *cloud, const double *t_frames_dev,
                     int32_t n_frames, int32_t coord_mode, double a0_floor,
                     double *mu_t, float *a0_t, float *p0_t, float *H,
                     pc_stream_t stream);

/* pc_deform_states with float64 a0_t / p0_t (the drop-in cloud_states_at
 * returns the reference's float64 CloudState, deformation.py:31-54). */
int pc_deform_states_f64(const pc_cloud_t *cloud, const double *t_frames_dev,
                         int32_t n_frames, int32_t coord_mode, double a0_floor,
                         double *mu_t, double *a0_t, double *p0_t,
                         pc_stream_t stream);

/* Replaces deformation.py:219-267 cloud_state_grads at one frame time
 * (materialised Jacobians, f64; API compatibility -- the fused engine never
 * materialises them). */
int pc_deform_jacobian(const pc_cloud_t *cloud, double t, int32_t coord_mode,
                       double a0_floor, double *d_base, double *d_omega,
                       double *d_theta, double *d_sigma, pc_stream_t stream);

/* Replaces deformation.py:57-70 eval_basis: out[i] = exp(-(t - theta)^2 /
 * (2 sigma^2)) over n already-broadcast device fp64 values. */
int pc_eval_basis(const double *t, const double *theta, const double *sigma,
                  int64_t n, double *out, pc_stream_t stream);

/* Replaces deformation.py:73-84 eval_H: out[0] = sum_n omega[n] *
 * eval_basis(t, theta[n], sigma[n]) (index order, fp64; device arrays). */
int pc_eval_h(double t, const double *omega, const double *theta,
              const double *sigma, int32_t n, double *out, pc_stream_t stream);

/* Replaces radiator.py:278-294 (accumulate_frame_grads' chain rule) for one
 * frame: G (B,5) f32 through a materialised Jacobian bundle into f64 grads.
 * omega_row: host int[5] (deformation.py:87-90); shared: theta is (B,N). */
int pc_assemble_grads(const float *G, int64_t n_balls, int32_t n_basis,
                      const double *d_base, const double *d_omega,
                      const double *d_theta, const double *d_sigma,
                      const int32_t *omega_row_host, int32_t shared,
                      int32_t with_theta_sigma, double *g_p0, double *g_a0,
                      double *g_mu, double *g_theta, double *g_sigma,
                      double *g_omega, pc_stream_t stream);

/* Fused deformation backward over F frames: the chain rule of
 * radiator.py:278-294 through deformation.py:219-267, summed over frames as
 * reconstruction.py:303-316 does, without materialising any Jacobian.
 * G and H are (F,B,5) from pc_residual_state_grads / pc_deform_states.
 * Gradients are overwritten. */
int pc_deform_backward(const pc_cloud_t *cloud, const double *t_frames_dev,
                       int32_t n_frames, int32_t coord_mode, double a0_floor,
                       const float *G, const float *H,
                       const pc_cloud_grads_t *grads, pc_stream_t stream);

/* ---- radiator ---------------------------------------------------------- */

/* Launch plan of pc_forward_traces for this problem: plan[0] = samples per
 * shared-memory time segment, plan[1] = segments, plan[2] = ball chunks
 * (> 1 adds a chunk-combine launch), plan[3] = kernel launches per call. */
int pc_forward_plan(int64_t n_balls, int32_t n_frames, const pc_array_t *array,
                    int32_t *plan);

/* Which forward kernel pc_forward_traces runs for this array: 0 = register-run
 * forward (default), 1 = shared-memory-trace forward (PC_FWD_LEGACY=1 or a
 * trace too long for the run kernel), 2 = register-run forward with the ball
 * tiles staged by cp.async.bulk (TMA) behind an mbarrier (PC_FWD_TMA=1).  All
 * three replace radiator.py:86-118.  -1 for a NULL array. */
int pc_forward_variant(const pc_array_t *array);

/* Scratch bytes pc_forward_traces needs for this problem (0 = none). */
size_t pc_forward_workspace_bytes(int64_t n_balls, int32_t n_frames,
                                  const pc_array_t *array);

/* Replaces radiator.py:86-118 _forward_traces (+ forward_frame :195-216),
 * batched over F frames, with the residual and L2 loss of
 * reconstruction.py:312-313 fused: if `observed` (F,M,T) is non-NULL, `out`
 * receives predicted - observed and loss_per_frame[f] = 0.5*sum r^2 (f64);
 * otherwise `out` receives the predicted traces.  `out` is overwritten.
 * coincident: device int64, must hold INT64_MAX on entry; receives the
 * smallest coincidence word (see pc_array_t) of any pair with R < 1e-9
 * (radiator.py:97-99). */
int pc_forward_traces(const double *mu_t, const float *a0_t,
                      const float *p0_t, int64_t n_balls, int32_t n_frames,
                      const pc_array_t *array, const float *observed,
                      float *out, double *loss_per_frame,
                      int64_t *coincident, void *workspace,
                      size_t workspace_bytes, pc_stream_t stream);

/* The residual/loss epilogue of pc_forward_traces as its own call, for
 * callers that overlap the observed-trace upload with the forward sweep
 * (reconstruction.py:312-313): out = predicted - observed (out may alias
 * predicted) and, if loss_per_frame is non-NULL, loss_per_frame[f] =
 * 0.5*sum r^2 (f64, fixed-order reduction; loss_partial = F*M doubles of
 * scratch). */
int pc_residual_loss(const float *predicted, const float *observed, float *out,
                     double *loss_partial, double *loss_per_frame,
                     int32_t n_frames, int32_t n_sensors, int32_t n_samples,
                     pc_stream_t stream);

/* Replaces radiator.py:121-174 _residual_state_grads (+ frame_state_grads
 * :219-242), batched over F frames: G (F,B,5) f32 is overwritten with the
 * gradient of 0.5*||residual||^2 w.r.t. (a0_t, p0_t, mu_t). */
int pc_residual_state_grads(const double *mu_t, const float *a0_t,
                            const float *p0_t, int64_t n_balls,
                            int32_t n_frames, const pc_array_t *array,
                            const float *residual, float *G,
                            int64_t *coincident, pc_stream_t stream);

/* Replaces radiator.py:36-55 pressure_kernel (out) and :58-83
 * pressure_kernel_grad (d_p0, d_a0, d_R; all three or none), elementwise in
 * fp64 over n already-broadcast device values of R, t, p0, a0 (sound speed
 * v > 0).  Input validation (R > 0, a0 > 0) is the caller's, as the
 * reference raises before evaluating. */
int pc_pressure_kernel(const double *R, const double *t, const double *p0,
                       const double *a0, int64_t n, double sound_speed,
                       double *out, double *d_p0, double *d_a0, double *d_R,
                       pc_stream_t stream);

/* ---- evaluation --------------------------------------------------------- */

/* Scratch bytes of pc_voxelize. */
size_t pc_voxelize_workspace_bytes(int64_t n_balls);

/* Replaces evaluation.py:46-93 _splat_balls / voxelize: out (nx,ny,nz) f32,
 * C order, = sum_b p0_b exp(-|x - mu_b|^2 / (2 a0_b^2)) at voxel centres
 * origin + i*spacing, limited to each ball's support cube unless exact.
 * mu (B,3), a0, p0 (B) f64 on the device; origin[3] and dims[3] host arrays
 * (dims <= 32767).  bad_a0: device int32, set to 1 if any a0 <= 0. */
int pc_voxelize(const double *mu, const double *a0, const double *p0,
                int64_t n_balls, const double *origin, double spacing,
                const int32_t *dims, double support_sigmas, int32_t exact,
                float *out, int32_t *bad_a0, void *workspace,
                size_t workspace_bytes, pc_stream_t stream);

/* Replaces reconstruction.py:397-398 (ubp_reconstruct filter):
 * filtered (M,T) f32 = 2 p - 2 t dp/dt, dp/dt = numpy.gradient along time
 * (central differences, one-sided ends), t_j = t_start + j / sample_rate;
 * traces (M,T) f64 on the device. */
int pc_ubp_filter(const double *traces, int32_t n_sensors, int32_t n_samples,
                  double t_start, double sample_rate, float *filtered,
                  pc_stream_t stream);

/* Replaces reconstruction.py:352-377 _backproject: out (nx,ny,nz) f32, C
 * order, = (1/M) sum_m lerp(filtered_m, (|x - s_m| / v - t_start) / dt) at
 * voxel centres origin + i*spacing (index truncated, clamped to T-2).
 * positions (M,3) f64 on the device; origin[3], dims[3] host arrays. */
int pc_backproject(const float *filtered, const double *positions,
                   int32_t n_sensors, int32_t n_samples, double sound_speed,
                   double t_start, double dt, const double *origin,
                   double spacing, const int32_t *dims, float *out,
                   pc_stream_t stream);

/* ---- loss and optimiser ------------------------------------------------- */

/* Replaces reconstruction.py:28-35 l2_loss: out[0] = 0.5*sum (p-o)^2 (f64,
 * fixed-order reduction). */
int pc_l2_loss(const double *predicted, const double *observed, int64_t n,
               double *out, pc_stream_t stream);

/* Non-finite scan (reconstruction.py:60-61): flags[s] |= 1 when segment s of
 * x (f32) holds a NaN/Inf.  seg_off is a host array of n_seg+1 offsets. */
int pc_check_finite(const float *x, int32_t n_seg, const int64_t *seg_off,
                    int32_t *flags, pc_stream_t stream);

/* float64-gradient variants (the drop-in adam_step / sgd_step take the
 * caller's float64 gradient, reconstruction.py:57-76). */
int pc_check_finite_f64(const double *x, int32_t n_seg, const int64_t *seg_off,
                        int32_t *flags, pc_stream_t stream);
int pc_adam_segments_f64(double *params, const double *grads, double *m,
                         double *v, int32_t n_seg, const int64_t *seg_off,
                         const double *seg_lr, const int32_t *seg_step,
                         const double *seg_floor, pc_stream_t stream);
int pc_sgd_segments_f64(double *params, const double *grads, int32_t n_seg,
                        const int64_t *seg_off, const double *seg_lr,
                        const double *seg_floor, pc_stream_t stream);

/* Replaces reconstruction.py:57-69 adam_step (+ the floors of :153-157) for
 * n_seg parameter segments of one flat buffer in one launch.  Per segment:
 * learning rate, step count t (after increment) and lower floor
 * (-inf = none).  seg_off / seg_lr / seg_step / seg_floor are host arrays;
 * at most PC_MAX_SEGMENTS segments. */
#define PC_MAX_SEGMENTS 16
int pc_adam_segments(double *params, const float *grads, double *m,
                     double *v, int32_t n_seg, const int64_t *seg_off,
                     const double *seg_lr, const int32_t *seg_step,
                     const double *seg_floor, pc_stream_t stream);

/* The iteration's update without a host round trip: Adam (optimizer 0) or
 * SGD (1) over n_seg segments like pc_adam_segments / pc_sgd_segments, with
 * each segment's (lr, step t) read from hyper_dev (device, 2*n_seg doubles)
 * and the reference's guard semantics decided on the device: nothing is
 * updated if *coincident_dev != INT64_MAX or *loss_dev is not finite
 * (radiator.py:186-192, reconstruction.py:317-318); otherwise the segments
 * (one per parameter array, in the reference's update order: pressure, std,
 * coords, then deform's theta, sigma, omega) before the first segment with a
 * non-finite flag (flags_dev, from pc_check_finite) are updated -- adam_step
 * raises per ARRAY before touching it (reconstruction.py:60-61, 88-93,
 * 320-327) -- and the floors (seg_floor) apply only when every segment was
 * stepped (the raise skips _clamp_floors, :328).  seg_group (host, the
 * segment's group index) is kept for the caller's bookkeeping.  seg_off /
 * seg_floor / seg_group are host arrays. */
int pc_update_guarded(double *params, const float *grads, double *m,
                      double *v, int32_t n_seg, const int64_t *seg_off,
                      const double *seg_floor, const int32_t *seg_group,
                      const double *hyper_dev, const int32_t *flags_dev,
                      const double *loss_dev, const int64_t *coincident_dev,
                      int32_t optimizer, pc_stream_t stream);

/* Replaces reconstruction.py:72-76 sgd_step over segments. */
int pc_sgd_segments(double *params, const float *grads, int32_t n_seg,
                    const int64_t *seg_off, const double *seg_lr,
                    const double *seg_floor, pc_stream_t stream);

/* ---- prune / densify compaction ----------------------------------------- */

/* Workspace bytes for pc_prune_mask / pc_compact_index on B balls. */
size_t pc_compact_workspace_bytes(int64_t n_balls);

/* reconstruction.py:217-220: keep[b] = p0[b] > rel_threshold*max(p0, 0);
 * n_keep (device int64) receives the survivor count. */
int pc_prune_mask(const double *p0, int64_t n_balls, double rel_threshold,
                  uint8_t *keep, int64_t *n_keep, void *workspace,
                  size_t workspace_bytes, pc_stream_t stream);

/* Stable compaction order (reconstruction.py:95-100 boolean gather):
 * index[0..n_keep) = ascending b with keep[b]; then, if `append` is non-NULL,
 * index[n_keep..n_keep+n_append) = ascending b with append[b] (children of
 * the config-5 split, appended after the survivors in parent order).
 * n_out (device int64) = n_keep + n_append. */
int pc_compact_index(const uint8_t *keep, const uint8_t *append,
                     int64_t n_balls, int64_t *index, int64_t *n_out,
                     void *workspace, size_t workspace_bytes,
                     pc_stream_t stream);

/* Config-5 densify masks (builder-defined rule; the
 * reference has pruning only, reconstruction.py:217-226):
 *   keep[b]  = !(p0[b] < p0_min)
 *   split[b] = keep[b] && |g[b]| > threshold       (g = dL/dp0, f32)
 * `threshold` (device double) is the numpy 'linear' percentile of |g|
 * (pc_abs_quantile_f32).  counts (device int64[2]) receive (#keep, #split). */
int pc_densify_masks(const double *p0, const float *g, int64_t n_balls,
                     double p0_min, const double *threshold, uint8_t *keep,
                     uint8_t *split, int64_t *counts, pc_stream_t stream);

/* Workspace bytes of pc_abs_quantile_f32 (independent of n). */
size_t pc_abs_quantile_workspace_bytes(void);

/* numpy.percentile(|g|, q, method='linear') of a device f32 array, on the
 * device (no host round trip): the caller passes numpy's virtual-index
 * split k = floor((n-1) q/100), gamma = (n-1) q/100 - k (0 <= gamma < 1,
 * k < n); the order statistics x_(k), x_(k+1) of |g| come from a radix
 * select and are combined by numpy's _lerp
 * (numpy/lib/_function_base_impl.py) in round-to-nearest fp64.  The result
 * is written to *threshold (device double).  g must be finite. */
int pc_abs_quantile_f32(const float *g, int64_t n, int64_t k, double gamma,
                        double *threshold, void *workspace,
                        size_t workspace_bytes, pc_stream_t stream);

/* Densify flags after pc_compact_index(keep, split) (index[0, n_keep) =
 * survivors, index[n_keep, n_out) = children's parents, n_out possibly
 * truncated by a ball cap): child[i] = i >= n_keep; halve[i] = child[i] or
 * survivor i's child is in [n_keep, n_out).  has_child: scratch of n_balls
 * bytes. */
int pc_densify_flags(const int64_t *index, int64_t n_balls, int64_t n_keep,
                     int64_t n_out, uint8_t *has_child, uint8_t *halve,
                     uint8_t *child, pc_stream_t stream);

/* After the gather of a densify step (new order = survivors then children):
 * p0[i] *= 0.5 where halve[i] (split parents and their children; halve may
 * be NULL: the clone rule keeps p0) and mu[i,0] += shift * a0[i] where
 * child[i]. */
int pc_densify_apply(double *p0, double *mu, const double *a0,
                     const uint8_t *halve, const uint8_t *child,
                     int64_t n_balls, double shift, pc_stream_t stream);

/* dst[i, :] = src[index[i], :] for i < n_rows (row_bytes a multiple of 4). */
int pc_gather_rows(const void *src, void *dst, const int64_t *index,
                   int64_t n_rows, int64_t row_bytes, pc_stream_t stream);

/* Library version string (static). */
const char *pc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PACLOUD_B200_H */
