/* spst.h — C ABI of the B200-native SPST hot path (libspst.so).
 *
 * Replaces, for one device, the compute behind the reference's public Python entry points
 * (paths relative to /root/reference/pkg/src/tilestyle/):
 *   localized.py:162  stats_pass        -> spst_forward + spst_stats_ptrs + spst_finalize
 *   localized.py:187  build_problem     -> spst_bind + spst_forward + spst_capture_content
 *   localized.py:227  loss_grad         -> spst_forward, spst_finalize, spst_content_sqdiff,
 *                                          spst_backward
 *   localized.py:283  loss_grad_global  -> same calls with the whole image as one grid
 *   lbfgs.py:68       two_loop_direction-> spst_vec_* step kernels (device scalars)
 *   lbfgs.py:99       minimize          -> spst_vec_axpy / spst_vec_sy / spst_vec_absmax
 *   tensorops.py:136  resize_down       -> spst_resize_down
 *   tensorops.py:158  resize_bilinear   -> spst_resize_bilinear
 *   metrics.py:24     psnr              -> spst_metric_sqdiff
 *   metrics.py:55     ssim              -> spst_metric_ssim
 * The reference has no FFI for this path (it is pure NumPy); the Python package
 * paper_2212_13459_b200 binds these symbols with ctypes.
 *
 * Conventions: all pointers named *_dev are device pointers; images are HWC float32; status
 * codes map 1:1 onto the reference's exception taxonomy (errors.py:4-33). No C++ exception
 * crosses this boundary; spst_last_error() returns the message of the last failure.
 * A context is bound to one device and one stream and is not thread-safe.
 */
#ifndef SPST_H_
#define SPST_H_

#ifdef __cplusplus
extern "C" {
#endif

#define SPST_ABI_VERSION 1

#define SPST_OK 0
#define SPST_ERR_SHAPE 1       /* errors.ShapeError    */
#define SPST_ERR_GEOMETRY 2    /* errors.GeometryError */
#define SPST_ERR_CONFIG 3      /* errors.ConfigError   */
#define SPST_ERR_NONFINITE 4   /* errors.NonFiniteError */
#define SPST_ERR_CUDA 5        /* RuntimeError (CUDA failure) */
#define SPST_ERR_OOM 6         /* MemoryError          */
#define SPST_ERR_UNSUPPORTED 7 /* NotImplementedError: layer graph outside the device path */
#define SPST_ERR_EMPTY 8       /* errors.EmptyError    */

#define SPST_LAYER_CONV 0
#define SPST_LAYER_RELU 1
#define SPST_LAYER_AVGPOOL 2
#define SPST_LAYER_MAXPOOL 3

typedef struct spst_ctx spst_ctx;

int spst_abi_version(void);
const char* spst_status_string(int status);

/* ---------------------------------------------------------------- extractor context ----
 * extractor.py:72-106 ExtractorSpec + extractor.py:257-280 load_weights.
 * layers: n_layers kinds (SPST_LAYER_*); conv layers carry cin/cout and float64 weights
 * (cout, cin, 3, 3) + bias (cout); style_layers / content_layer are layer indices of relu
 * layers; mean3/scale3/bgr is the Preprocess record (extractor.py:58-62). */
int spst_create(int device, int n_layers, const int* kinds, const int* cin, const int* cout,
                const double* const* weights, const double* const* biases, int n_style,
                const int* style_layers, int content_layer, int bgr, const double* mean3,
                const double* scale3, spst_ctx** out);
void spst_destroy(spst_ctx* ctx);
const char* spst_last_error(const spst_ctx* ctx);
int spst_set_stream(spst_ctx* ctx, void* cuda_stream);
/* Tensor-core precision of the conv layers (SURVEY.md §7 step 3 precision knob): 0 = fp16x3
 * (hi/lo split operands, three MMA passes, fp32-class -- the default and the parity mode);
 * 1 = fp16 (hi*hi only, one pass: ~1e-3 relative per layer, opt-in speed mode that does NOT
 * meet the gradient parity bar).  Statistics (Gram) stay fp16x3 in both. */
int spst_set_precision(spst_ctx* ctx, int mode);

/* Geometry (localized.py:116-120 make_grid, tiling.py:57-72). h, w: unpadded image. The
 * padded grid is (Hp, Wp) = dims rounded up to the deepest stride. This context evaluates
 * padded rows [grid_r0, grid_r1) as one zero-padded image and owns rows [own_r0, own_r1)
 * (statistics, content loss and gradient are restricted to owned rows; the rows outside
 * are the receptive-field halo). A single device binds grid = own = [0, Hp). */
int spst_bind(spst_ctx* ctx, int h, int w, int grid_r0, int grid_r1, int own_r0, int own_r1);
/* Window binding (2-D): the context evaluates the padded-image rectangle [grid_r0, grid_r1) x
 * [grid_c0, grid_c1) as one zero-padded image -- the reference's padded block (tiling.py:57-72,
 * localized.py:153-155) -- and owns [own_r0, own_r1) x [own_c0, own_c1) inside it: the block's
 * inner rectangle, whose tap-space crop (tiling.py:75-88) feeds the statistics and the content
 * loss and whose pixels receive the gradient.  Bounds are multiples of the deepest stride (an
 * owned end may equal the padded size).  spst_bind(rows) = full-width window. */
int spst_bind_window(spst_ctx* ctx, int h, int w, int grid_r0, int grid_r1, int grid_c0, int grid_c1,
                     int own_r0, int own_r1, int own_c0, int own_c1);
int spst_window_dims(const spst_ctx* ctx, int* rows, int* cols);
int spst_unbind(spst_ctx* ctx); /* release the bound workspace */
int spst_padded_dims(const spst_ctx* ctx, int* Hp, int* Wp);
int spst_tap_info(const spst_ctx* ctx, int tap, int* channels, int* stride, long long* owned_pixels);
long long spst_workspace_bytes(const spst_ctx* ctx);

/* Forward pass of image x_dev (h x w x 3 f32). flags bit0: keep the state the backward needs.
 * Leaves per style tap the owned-row partial sums S = sum F F^T (C x C f64) and s = sum F
 * (C f64) in device buffers exposed by spst_stats_ptrs (for an NCCL all-reduce). */
int spst_forward(spst_ctx* ctx, const float* x_dev, int flags);
/* As spst_forward with the image addressed as x_dev + (y * pitch + x) * 3 for global pixel
 * (y, x) (pitch >= w pixels): a window's rows may live in a smaller buffer whose pointer is
 * offset accordingly. */
int spst_forward_pitched(spst_ctx* ctx, const float* x_dev, long long pitch, int flags);
int spst_stats_ptrs(spst_ctx* ctx, int tap, double** S_dev, double** s_dev);

/* Content target (localized.py:205-212): copy the content-tap features of the last forward. */
int spst_capture_content(spst_ctx* ctx);
/* The captured content target of the bound window (HL16 bytes on the device, and its scale):
 * a windowed evaluation keeps one target per window (the reference's ContentStore tiles,
 * localized.py:84-109) and swaps it in with spst_set_content_target (device copy). */
int spst_content_target(spst_ctx* ctx, void** buf_dev, long long* bytes, float* scale);
int spst_set_content_target(spst_ctx* ctx, const void* buf_dev, float scale);
/* sum over owned rows of (V - V_u)^2 at the content tap, into out_dev (1 f64). */
int spst_content_sqdiff(spst_ctx* ctx, double* out_dev);

/* Style reference of tap t (stats.py:22-31 LayerStats) and its TapWeights (stats.py:81-86). */
int spst_set_style_ref(spst_ctx* ctx, int tap, const double* gram, const double* mean,
                       const double* std, double w_gram, double w_mean, double w_std);
/* Finalize global statistics from the (all-reduced) sums with global pixel counts n[tap]
 * (stats.py:59-66), write per tap the three weighted loss terms (stats.py:117-124) to
 * terms_host[3*tap..], and prepare the closed-form feature gradients (stats.py:127-165).
 * degenerate_host[tap] = 1 when a zero-std channel has a nonzero reference std. */
int spst_finalize(spst_ctx* ctx, const long long* n, double* terms_host, int* degenerate_host);
/* 1 if the last spst_finalize had to re-run the forward (its deferred range check failed):
 * anything launched behind that forward (spst_content_sqdiff) must be launched again. */
int spst_forward_redone(spst_ctx* ctx);
/* Reverse pass (extractor.py:200-214 + localized.py:246-279): pixel gradient of the loss on
 * owned rows written into grad_dev (h x w x 3 f32; rows outside the owned range untouched).
 * two_lambda = 2 * lambda_c (0 disables the content term). */
int spst_backward(spst_ctx* ctx, double two_lambda, float* grad_dev);
/* As spst_backward with the gradient written at grad_dev + (y * pitch + x) * 3 for the owned
 * pixels (y, x) of the window. */
int spst_backward_pitched(spst_ctx* ctx, double two_lambda, float* grad_dev, long long pitch);
/* Asynchronous form: launches the backward and returns; its end-of-pass range check is
 * deferred to spst_backward_resolve (or any later call on the context), which waits for the
 * pass and re-runs it in careful mode if needed (*redone = 1: the gradient was rewritten, so
 * work launched on it in between must be repeated).  One host synchronisation per gradient
 * instead of two when the caller has its own read-back to make (L-BFGS's curvature dots). */
int spst_backward_async(spst_ctx* ctx, double two_lambda, float* grad_dev, long long pitch);
int spst_backward_resolve(spst_ctx* ctx, int* redone);

/* ---------------------------------------------------------------- launch timer ---------
 * Measurement hook (no reference counterpart): when enabled, every tensor-core launch is
 * bracketed by CUDA events on the context stream.  spst_timing_read returns, per class
 * (0 conv3x3_tc N=128, 1 conv3x3_tc N=64, 2 Gram, 3 unused), the summed device ms, the
 * algorithmic FLOPs of those launches (real channel counts, one pass) and the launch count.
 * spst_timing_enable resets the totals. */
int spst_timing_enable(spst_ctx* ctx, int on);
/* Kernels launched by this library since it was loaded (all contexts and the context-free
 * entry points); bench.py reads it around its timed region. */
long long spst_launch_count(void);
int spst_timing_read(spst_ctx* ctx, double* ms4, double* flops4, long long* launches4);

/* ---------------------------------------------------------------- vector kernels ---------
 * lbfgs.py:68-142. Reductions accumulate in f64 with a fixed order (deterministic). The
 * partial buffer must hold spst_vec_partials() doubles per reduced quantity. */
int spst_vec_partials(void);
/* f64 selects float64 vectors (1) or float32 vectors (0). */
int spst_vec_dots(int f64, const void* a0, const void* b0, const void* a1, const void* b1,
                  const void* a2, const void* b2, long long n, double* partial_dev,
                  double* out_dev, void* stream);
int spst_vec_absmax(int f64, const void* a, long long n, double* partial_dev, double* out_dev,
                    void* stream);
/* q_out = cscale * (q_in + coef_dev[0] * v); partial <w, q_out> (v, w may be NULL). */
int spst_vec_axpy_dot(int f64, const void* q_in, void* q_out, const void* v,
                      const double* coef_dev, double cscale, const void* w, long long n,
                      double* partial_dev, void* stream);
/* finished dot -> mode 0: alpha = rho*dot, coef = -alpha; mode 1: coef = alpha - rho*dot */
int spst_vec_twoloop_scalar(const double* dot_dev, double rho, int mode, double* alpha_dev,
                            double* coef_dev, void* stream);
int spst_vec_sum_partials(const double* partial_dev, int n_quantities, double* out_dev, void* stream);
/* lbfgs.py:68-83 two_loop_direction as ONE call (single-device runs): out = -H g from the m
 * curvature pairs (s_vecs/y_vecs oldest first, rho_i = 1/<y_i,s_i>, gamma = <s,y>/<y,y> of the
 * newest pair).  2m+1 kernels, each an axpy+dot step that also finishes its dot product in
 * fixed block order and applies the scalar update (bit-identical to the step-by-step calls
 * above); alpha_dev holds m doubles, coef_dev one, ticket_dev one zero-initialised counter. */
int spst_vec_two_loop(int f64, const void* g, void* out, const void* const* s_vecs,
                      const void* const* y_vecs, const double* rho, double gamma, int m, long long n,
                      double* partial_dev, double* alpha_dev, unsigned int* ticket_dev, double* coef_dev,
                      void* stream);
int spst_vec_axpy(int f64, const void* x, const void* d, double t, long long n, void* out, void* stream);
int spst_vec_sy(int f64, const void* xt, const void* x, const void* gt, const void* g, long long n,
                void* s, void* y, double* partial_dev, double* out_dev /*[3]: ys, ss, yy*/,
                void* stream);

/* ---------------------------------------------------------------- metrics --------------- *
 * metrics.py:24-31 psnr: out_dev[0] = sum over n elements of (a-b)^2 (f64, fixed order).
 * metrics.py:55-73 ssim: out_dev[0] = sum of the SSIM map of the Rec.601 luma of two (h, w, c)
 *   images (c = 1 or 3), 11x11 Gaussian window sigma 1.5, valid mode, K1/K2 = 0.01/0.03; the
 *   caller divides by (h-10)(w-10).  h, w >= 11 else SPST_ERR_SHAPE.
 * partial_dev holds spst_vec_partials() doubles.  sqdiff: f64 selects float64 for both inputs;
 * ssim: f64 is a mask (bit 0: a is float64, bit 1: b is float64), each luma is formed in its
 * image's own dtype as the reference's NumPy code does. */
int spst_metric_sqdiff(int f64, const void* a, const void* b, long long n, double* partial_dev,
                       double* out_dev, void* stream);
int spst_metric_ssim(int f64, const void* a, const void* b, int h, int w, int c, double* partial_dev,
                     double* out_dev, void* stream);

/* ---------------------------------------------------------------- resampling ------------ */
int spst_resize_down(const float* in, int h, int w, int c, int factor, float* out, void* stream);
int spst_resize_bilinear(const float* in, int h, int w, int c, int oh, int ow, float* out,
                         void* stream);
/* Same with f32 (f64 = 0) or f64 (f64 = 1) images: the reference's dtype="f64" path. */
int spst_resize_down_typed(int f64, const void* in_dev, int h, int w, int c, int f, void* out_dev,
                           void* stream);
int spst_resize_bilinear_typed(int f64, const void* in_dev, int h, int w, int c, int oh, int ow,
                               void* out_dev, void* stream);

/* Relu output of conv stage `stage` (a tap layer) from the last forward, unpacked to a
 * (C_out x H x W) f32 device buffer on the context stream (extractor.py:171-197 forward_taps). */
int spst_stage_features(spst_ctx* ctx, int stage, float* out_dev);
/* out[c,p] = sum_d A[c,d] V[d,p] + r[c] V[c,p] + b[c] on a (C x P) slab (f32 or f64, device
 * pointers, f64 accumulation): the pointwise style feature gradient of stats.py:127-165 given the
 * global statistics, for direct calls of style_layer_loss_grad (loss_grad fuses it instead). */
int spst_feature_affine(int f64, const void* A, const void* r, const void* b, int C, long long P,
                        const void* V, void* out, void* stream);
/* out = c (a - b) (stats.py:168-174 content_loss_grad's gradient). */
int spst_vec_scaled_diff(int f64, const void* a, const void* b, double c, long long n, void* out,
                         void* stream);

/* ---------------------------------------------------------------- unit-test hooks -------
 * One tensor-core conv layer on host arrays (x: cin x H x W f32, weight cout x cin x 3 x 3,
 * bias cout; f64). mode 0: y = relu(conv(x)) (cout x H x W); mode 1: y = avgpool(relu(conv))
 * (cout x H/2 x W/2); mode 2: y = conv^T(x) input gradient (x has cout channels, y cin);
 * mode 3: relu mask bits of mode 0 as floats; mode 4: y = maxpool(relu(conv)); mode 5: the
 * first-argmax index (0-3, row-major in the window) of mode 4 as floats. Returns through y_host. */
int spst_debug_conv(int device, int mode, int cin, int cout, int H, int W, const float* x_host,
                    const double* weight, const double* bias, float* y_host);
/* ReLU mask of conv stage `stage` (0-based conv index) from the last forward, as bytes
 * (C_out x H x W, 1 = pre-activation > 0) — lets tests evaluate the f64 oracle on the device's
 * activation pattern. */
int spst_debug_mask(spst_ctx* ctx, int stage, unsigned char* out_host);
/* Stored relu output of conv stage `stage` from the last forward (C_out x H x W f32, local
 * grid). Pool stages keep their full-resolution output only at taps unless the context was
 * bound with SPST_DEBUG_STORE_ALL=1 in the environment (error-budget diagnostics). */
int spst_debug_stage_out(spst_ctx* ctx, int stage, float* out_host);
/* Gram of a (C x P) f32 feature matrix through the tensor-core Gram kernel, S = F F^T (f64). */
int spst_debug_gram(int device, int C, long long P, const float* f_host, double* S_host);

#ifdef __cplusplus
}
#endif
#endif /* SPST_H_ */
