// common.cuh — shared host/device definitions of the SPST device runtime.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cuda_fp16.h>

namespace spst {

constexpr int kSMs = 148;

// Process-wide count of kernels launched by this library (spst_launch_count); every launch
// site is written `note_launch(), kernel<<<...>>>(...)`.
void note_launch();

// Activation storage ("HL16"): fp16 hi plane-set followed by fp16 lo plane-set, each laid out
// [C_p/8][H][W][8] (8 channels = 16 B per pixel per kgroup).  The stored value is x * 2^e,
// split so that hi + lo carries ~22 mantissa bits.  Mask storage: uint32 [C_p/32][H][W],
// bit j of word g = (pre-activation of channel 32g+j > 0).
struct HL16 {
  __half* hi = nullptr;   // lo = hi + planes * H * W * 8
  int C_p = 0, H = 0, W = 0;
  float scale = 1.f;      // 2^e
  __host__ __device__ size_t plane_elems() const { return (size_t)H * W * 8; }
  __host__ __device__ __half* lo() const { return hi + (size_t)(C_p / 8) * plane_elems(); }
  __host__ __device__ size_t bytes() const { return (size_t)C_p * H * W * 4; }
};

enum EpiKind : int {
  EPI_FWD = 0,        // relu(acc*s + bias) -> mask bits, full-res store (optional), channel sums
  EPI_FWD_POOL = 1,   // as EPI_FWD plus 2x2 average pool of the two tile rows
  EPI_BWD = 2,        // (acc*s + bvec + content + addend) * mask -> store
  EPI_BWD_POOL = 3,   // pool adjoint: spread (acc*s)/4 onto 2x2 hi-res pixels (+addend) * hi-res mask
};

// Parameters of one tcgen05 3x3 implicit-GEMM launch (forward or input-gradient).
struct ConvArgs {
  CUtensorMap tm_r_hi, tm_r_lo;  // K operand: input activations as u64 (2W, H, C_p/8), box 136 x 1 x 1
  CUtensorMap tm_v_hi, tm_v_lo;  // extra-K operand: tap features at the output pixels (box 8 x 128 x 2 x 4)
  const uint8_t* wgt;            // [ntile][kc][pass][tap][kg][n][8] fp16
  const uint8_t* xwgt;           // [ntile][xkc][pass][kg(4)][n][8] fp16 (extra K, 32 ch per chunk)
  float x_rescale;               // extra-K chunk partials are multiplied by this when drained
  int H, W;                      // output (== input) spatial dims of the GEMM grid
  int n_kc, n_xkc;               // conv K-chunks (16 ch each), extra K-chunks (32 ch each)
  int n_ntiles;                  // output channel tiles
  int tiles_x, tiles_y;          // 128-px column blocks, 2-row row blocks
  float acc_scale;               // 2^-(e_in + f)
  float out_scale;               // 2^e_out
  int epi;
  // epilogue operands
  const float* bias;             // [C_out_p] (fwd bias or bwd bvec), may be null
  const uint32_t* mask_in;       // bwd: mask of the relu whose output gradient we produce
  uint32_t* mask_out;            // fwd: mask bits of this conv's relu
  HL16 out;                      // full-res output (fwd relu output / bwd gradient)
  HL16 out_pool;                 // fwd pooled output
  HL16 content_v, content_u;     // bwd content term operands (same grid as out)
  float content_coef;            // 2*lambda (0 = none)
  HL16 addend;                   // bwd addend at out's grid (hi == nullptr: none)
  int store_full;                // fwd pool: also store full-res relu output
  // channel sums of the relu output over rows [sum_r0, sum_r1) (fwd, tap layers)
  float* colsum_partial;         // [tiles_y*tiles_x][C_out_p], nullable
  int sum_r0, sum_r1, sum_c0, sum_c1;
  unsigned int* amax;            // max |output| (unscaled) as float bits
  // max pooling (reference tensorops.py:113-129): fwd writes, bwd reads the first-argmax index
  // (row-major in the 2x2 window) of every pooled element, 2 bits: uint32 [C_p/16][H/2][W/2]
  int pool_max;
  uint32_t* pool_arg;
  int drain;                     // K-chunks per TMEM accumulation group (1 or 2)
  int pass0;                     // first MMA pass: 0 = fp16x3 (hi*lo, lo*hi, hi*hi), 2 = fp16 (hi*hi only)
  float comp[4];                 // round-toward-zero bias factor per group relative to `fine`:
                                 // [conv 1, conv 2, extra 1, extra 2 chunks]
  float fine;                    // common relative correction applied once to the drained sum
};

struct GramArgs {
  // owned rectangle of the tap tensor viewed as u64 (2 x w_own, rows, kg); box = one KPX-pixel
  // run of one row (x16 / x8 kgroups); the run past w_own is TMA zero fill
  CUtensorMap tm_hi, tm_lo;
  int C_p;                       // channels (padded)
  int rows, w_own;               // owned rectangle (tap pixels)
  int px_per_split;              // pixels (KPX-pixel stages x KPX) per CTA partial
  int n_ctile;                   // channel tiles of 128
  float* partial;                // [split][pair][128][128]
  float comp[2];                 // round-toward-zero bias factor of a 1- / 2-stage accumulator relative to fine_*
  float fine_diag, fine_off;     // common relative correction of diagonal / off-diagonal entries
};

// Expected relative round-toward-zero bias of one TMEM accumulation group in units of
// kappa (see conv_tc.cu): per chunk `small` correction MMAs, then `large` hi*hi MMAs.
double rz_weight(int small, int large, int chunks);
// kappa of mixed-sign sums (convs; set_gram_comp holds the same-sign Gram constants)
double rz_kappa();

constexpr int kFirstC = 64;  // first-layer output channels supported by the SIMT kernels (padded)

// Preprocessed, replicate-padded image as the first conv's K operand: one 8-channel HL16 plane
// (3 channels + 5 zeros); the conv's second 8-channel K group reads out of bounds (TMA zero fill).
struct ImageHLArgs {
  const float* img;   // global pixel (y, x) at img + (y * pitch + x) * 3 (f32 HWC)
  long long pitch;    // pixels per image row of the buffer
  int h, w;           // unpadded global dims
  int row_off;        // global padded row of local row 0
  int col_off;        // global padded column of local column 0
  int Hl, Wp;         // local grid rows x columns
  int perm[3];
  float mean[3], scale[3];
  HL16 out;           // C_p = 8
  unsigned int* amax; // max |preprocessed value| (float bits)
};

struct FirstConvBwdArgs {
  HL16 g;             // gradient at the first conv's output (masked), C_p channels
  float wgt[kFirstC * 27];
  int C_out;
  int perm[3];
  float scale[3];
  float* gimg;        // (Hl, Wp, 3) f32 local padded grid
};

// Adjoint of the first conv on tcgen05 (first_bwd_tc.cu): taps folded into N (27 of 32).
struct FirstBwdTcArgs {
  CUtensorMap tm_hi, tm_lo;  // g0 (64 channels) as u64 (2W, H, 8): box 256 x 1 x 8 (128 px)
  const void* wslab;         // [hi|lo][kg 8][n 32][8] fp16: W[k][c][dy][dx] x 2^wexp at n = c*9+dy*3+dx
  int H, W;                  // local padded grid
  float acc_scale;           // 1 / (g0 scale x 2^wexp)
  int perm[3];
  float scale[3];
  float* gimg;               // (H, W, 3) f32
};
cudaError_t launch_first_bwd_tc(const FirstBwdTcArgs& a, cudaStream_t st);

struct StyleCoefArgs {
  const double* S;      // [C][C] global sum of outer products
  const double* s;      // [C] global channel sums
  double n;             // global pixel count n_p
  const double* Gr;     // style reference gram [C][C]
  const double* mur;    // [C]
  const double* sdr;    // [C]
  double wg, wm, ws;    // TapWeights
  int C;
  double* mu;           // [C]
  double* sd;           // [C]
  double* ratio;        // [C]
  float* bvec;          // [C_p] (zero padded)
  double* row_loss;     // [C] sum_j (G-Gr)^2 per row
  double* row_mmax;     // [C] max_j |M_kj| per row
  double* ms_loss;      // [2]: sum (mu-mur)^2, sum (sd-sdr)^2
  int* degenerate;      // set to 1 when sd < eps and sdr > eps
  // extra-K weight slab for the backward kernel: [ntile][xkc][pass][kg][n][8] fp16
  __half* xw;
  int N, n_xkc, xkg;    // slab layout [N-tile][xkc][pass][kg(xkg)][n][8]
  float xscale;         // 2^f_M
};

struct AxpyDotArgs {
  const void* q_in;     // f32 or f64 vectors (kernel template parameter)
  void* q_out;
  const void* v;        // axpy vector (nullable)
  const double* coef;   // device scalar: coefficient of v
  double cscale;        // host-known multiplier of the whole result (gamma or -1)
  const void* w;        // dot vector (nullable)
  long long n;
  double* partial;
  // fused step (spst_vec_two_loop): the last block to finish sums the partials in block order
  // (as finish_sums_kernel) and applies the two-loop scalar update (as twoloop_scalar_kernel)
  double* alpha_i = nullptr;     // non-null enables the fused finish
  unsigned int* ticket = nullptr;  // zero-initialised counter, reset by the last block
  double rho = 0.0;
  int mode = 0;
};

// Whole two-loop in one cooperative launch (spst_vec_two_loop on one device)
constexpr int kTwoLoopMaxHist = 128;
struct TwoLoopArgs {
  const void* g;
  void* out;
  const void* s[kTwoLoopMaxHist];  // oldest first
  const void* y[kTwoLoopMaxHist];
  double rho[kTwoLoopMaxHist];
  double gamma;
  int m;
  long long n;
  double* partial;  // 2 x red_blocks() doubles
};
cudaError_t launch_two_loop_coop(int f64, const TwoLoopArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- launchers
cudaError_t launch_conv_tc(const ConvArgs& a, int N, int grid, cudaStream_t stream);
int conv_tc_smem_bytes(int N);
int conv_tc_rows(int N);   // output rows per tile (MT)
int conv_tc_xkg(int N);    // kgroups per extra-K chunk
cudaError_t launch_gram_tc(const GramArgs& a, int n_splits, cudaStream_t stream);
cudaError_t launch_gram64_tc(const GramArgs& a, int n_splits, int C, double inv_scale2, double* S,
                             cudaStream_t stream);
cudaError_t launch_gram_reduce(const float* partial, int n_splits, int n_ctile, int C, double inv_scale2,
                               double* S, cudaStream_t stream);
cudaError_t launch_image_hl(const ImageHLArgs& a, cudaStream_t st);
cudaError_t launch_first_conv_bwd(const FirstConvBwdArgs& a, cudaStream_t st);
// grad: global pixel (y, x) at grad + (y * pitch + x) * 3; writes the owned rectangle
// [r0, r1) x [c0, c1) (clipped to the image) from the local grid gimg (Hl x Wl, origin
// (row_off, col_off)), folding the replicate-pad rows/columns onto the last image row/column.
struct FoldArgs {
  const float* gimg;
  int Hl, Wl, row_off, col_off, h, w, r0, r1, c0, c1;
  float* grad;
  long long pitch;
};
cudaError_t launch_fold_grad(const FoldArgs& a, cudaStream_t st);
cudaError_t launch_pool2_hl(const HL16& in, const HL16& out, unsigned int* amax, cudaStream_t st);
cudaError_t launch_colsum_reduce(const float* partial, int rows, int C, int stride, double* sums, double* mid,
                                 cudaStream_t st);
constexpr int kColsumMid = 256;  // doubles per channel of colsum scratch
cudaError_t launch_style_vec(const StyleCoefArgs& a, cudaStream_t st);
cudaError_t launch_style_mat(const StyleCoefArgs& a, cudaStream_t st);
cudaError_t launch_content_sqdiff(const HL16& v, const HL16& u, int C, int r0, int r1, int c0, int c1,
                                  double* partial, double* out, cudaStream_t st);
cudaError_t launch_dots(int f64, const void* a0, const void* b0, const void* a1, const void* b1, const void* a2,
                        const void* b2, long long n, double* partial, double* out, cudaStream_t st);
cudaError_t launch_absmax(int f64, const void* a, long long n, double* partial, double* out, cudaStream_t st);
cudaError_t launch_axpy_dot(int f64, const AxpyDotArgs& a, cudaStream_t st);
cudaError_t launch_twoloop_scalar(const double* dot, double rho, int mode, double* alpha_i, double* coef,
                                  cudaStream_t st);
cudaError_t launch_sum_partials(const double* partial, int nk, double* out, cudaStream_t st);
cudaError_t launch_axpy(int f64, const void* x, const void* d, double t, long long n, void* out, cudaStream_t st);
cudaError_t launch_sy(int f64, const void* xt, const void* x, const void* gt, const void* g, long long n, void* s,
                      void* y, double* partial, double* out, cudaStream_t st);
cudaError_t launch_resize_down(int f64, const void* in, int h, int w, int c, int f, void* out, cudaStream_t st);
cudaError_t launch_resize_bilinear(int f64, const void* in, int h, int w, int c, int oh, int ow, void* out,
                                   cudaStream_t st);
int red_blocks();
// api.cu (reference stats.py:127-174 on a standalone slab)
cudaError_t launch_feature_affine(int f64, const void* A, const void* r, const void* b, int C, long long P,
                                  const void* V, void* out, cudaStream_t st);
cudaError_t launch_scaled_diff(int f64, const void* a, const void* b, double c, long long n, void* out,
                               cudaStream_t st);
// metrics.cu (reference metrics.py): partial holds red_blocks() doubles; out = fixed-order sum
cudaError_t launch_metric_sqdiff(bool f64, const void* a, const void* b, long long n, double* partial, double* out,
                                 cudaStream_t st);
cudaError_t launch_metric_ssim(int f64_mask, const void* a, const void* b, int h, int w, int c, double* partial,
                               double* out, cudaStream_t st);

}  // namespace spst
