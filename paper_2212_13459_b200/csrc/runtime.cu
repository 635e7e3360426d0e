// runtime.cu — native runtime behind the C ABI (include/spst.h): network plan, weight
// staging into tensor-core layouts, HBM workspace, TMA descriptors, and the forward /
// finalize / backward schedules of Algorithm 1 (reference localized.py:162-311), plus the
// exported vector and resampling kernels.
//
// Range management for the fp16 hi/lo operands: every stored tensor carries a power-of-two
// scale chosen from the max |value| observed the previous time it was written (kernels
// record it with atomicMax).  The first time a tensor is produced the stage is checked
// immediately and re-run with the measured exponent if the stored range was off; later
// evaluations run without host syncs and fall back to that careful mode only if a range
// check at the end of the pass fails.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/spst.h"
#include "common.cuh"
#include "sm100.cuh"

using namespace spst;

namespace {

constexpr int kMaxPxPerSplit = 65536;  // Gram pixels per CTA partial (register-accumulated)
constexpr float kTargetLog2 = 11.f;  // stored |max| ~ 2^11 (fp16 max 65504 ~ 2^16)
constexpr float kOverflow = 30000.f;
constexpr float kUnderflow = 64.f;

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool get_encoder() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

// conv K operand: halo window box (8 ch, 130 px, 4 rows, 2 kg); extra-K operand: (8, 128, 2, 4)
bool map_act(CUtensorMap* m, const __half* base, int n_kg, int H, int W, int mt, bool extra, int xkg) {
  cuuint64_t dims[4] = {8, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n_kg};
  cuuint64_t strides[3] = {16, (cuuint64_t)W * 16, (cuuint64_t)H * W * 16};
  cuuint32_t box[4] = {8, extra ? 128u : 130u, extra ? (cuuint32_t)mt : (cuuint32_t)(mt + 2),
                       extra ? (cuuint32_t)xkg : 2u};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Same activation viewed as u64 (4 fp16) elements: (2W, H, kg); one box is a 68-pixel strip of one
// 8-channel plane row (1088 contiguous bytes), so TMA moves it as one long row.
bool map_rows(CUtensorMap* m, const __half* base, int n_kg, int H, int W) {
  cuuint64_t dims[3] = {2 * (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n_kg};
  cuuint64_t strides[2] = {(cuuint64_t)W * 16, (cuuint64_t)H * W * 16};
  cuuint32_t box[3] = {136, 1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// First-conv adjoint operand: a 64-channel HL16 tensor as u64 (2W, H, 8); one box is a 128-px
// row segment of all 8 planes (16 KB, [plane][px][8]).
bool map_rows128(CUtensorMap* m, const __half* base, int H, int W) {
  cuuint64_t dims[3] = {2 * (cuuint64_t)W, (cuuint64_t)H, 8};
  cuuint64_t strides[2] = {(cuuint64_t)W * 16, (cuuint64_t)H * W * 16};
  cuuint32_t box[3] = {256, 1, 8};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Gram operand: the owned rectangle of the HL16 planes viewed as u64 (2 w_own, rows, kg); box =
// one run of 64 px (128 channels: x 16 kg) or 128 px (64 channels: x 8 kg) of one row, landing
// as the dense [kg][px][8] MN-major operand; the run past w_own is TMA zero fill.
bool map_gram(CUtensorMap* m, const __half* base, int w_own, int rows, int W, int H, int n_kg) {
  cuuint64_t dims[3] = {2 * (cuuint64_t)w_own, (cuuint64_t)rows, (cuuint64_t)n_kg};
  cuuint64_t strides[2] = {(cuuint64_t)W * 16, (cuuint64_t)H * W * 16};
  const bool c64 = n_kg == 8;
  cuuint32_t box[3] = {c64 ? 256u : 128u, 1, c64 ? 8u : 16u};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, (void*)base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// Gram accumulators (gram_tc.cu): 128 channels = 8 correction + 4 hi*hi MMAs per 64-px stage;
// 64 channels = 8 hi*hi MMAs per 128-px stage (corrections in separate columns); two stages each.
// Tap features are ReLU outputs (>= 0), so every Gram entry is a same-sign sum: besides the
// result truncation, every addend's alignment truncation biases the same way.  kappa per
// kernel and entry kind, measured on B200 with tools/rz_calibrate.py (relu-like operands;
// checked on VGG-19 taps with tools/error_budget.py).
// The K dimension of a Gram accumulation is pixels: a row narrower than the stage (deep taps of
// small images, e.g. 16 px at relu5_1 of a 256x256 image) or a row's last partial stage is TMA
// zero fill, and zero addends truncate nothing.  The weights therefore count only the K=16 steps
// that carry real pixels, averaged over the row's stages by pixel count (g.w_own must be set).
void set_gram_comp(GramArgs& g, int C_p, bool nonneg = true) {
  const bool c64 = C_p == 64;
  const int kpx = c64 ? 128 : 64, steps = kpx / 16;
  // 128 channels: 2 correction + 1 hi*hi MMA per real K step; 64 channels: 1 hi*hi MMA
  auto W = [&](int r, int chunks) { return spst::rz_weight(c64 ? 0 : 2 * r, r, chunks); };
  const int w_own = std::max(1, g.w_own);
  const int full = w_own / kpx, rem = w_own % kpx, r_rem = (rem + 15) / 16;
  auto Wavg = [&](int chunks) {
    return ((double)full * kpx * W(steps, chunks) + (rem ? (double)rem * W(r_rem, chunks) : 0.0)) / w_own;
  };
  const double w1 = Wavg(1), w2 = Wavg(2);
  const double on = spst::rz_kappa() > 0.0 ? 1.0 : 0.0;  // SPST_RZ_KAPPA=0 disables every compensation
  const double kd = on * (c64 ? 7.3e-8 : 5.2e-8), ko = on * (nonneg ? (c64 ? 4.9e-8 : 3.8e-8) : spst::rz_kappa());
  g.fine_diag = (float)(kd * w2);
  g.fine_off = (float)(ko * w2);
  // a split's last accumulator may hold one stage: the remainder relative to fine
  g.comp[0] = (float)(1.0 + ko * (w1 - w2));
  g.comp[1] = 1.f;
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}
// K-chunks per TMEM accumulation group (conv_tc.cu): the forward decides the ReLU masks, so it
// drains every chunk; the backward (no sign decisions) groups two.  SPST_FWD_DRAIN /
// SPST_BWD_DRAIN override (1 or 2).
int fwd_drain() {
  static const int d = std::min(2, std::max(1, env_int("SPST_FWD_DRAIN", 1)));
  return d;
}
int bwd_drain() {
  static const int d = std::min(2, std::max(1, env_int("SPST_BWD_DRAIN", 2)));
  return d;
}

// comp[] / fine of a conv launch (conv_tc.cu): a conv chunk is 18 correction MMAs then 9 hi*hi
// MMAs per output row; an extra-K chunk xkg correction then xkg/2 hi*hi MMAs.  `fine` carries
// the full conv group's correction; comp[] the difference of every other group composition.
void set_conv_comp(ConvArgs& a, int N) {
  const double k = rz_kappa();
  const int xkg = conv_tc_xkg(N);
  const int sc = a.pass0 == 0 ? 18 : 0, sx = a.pass0 == 0 ? xkg : 0;  // correction MMAs per chunk
  const double wf = rz_weight(sc, 9, a.drain);
  a.fine = (float)(k * wf);
  a.comp[0] = (float)(1.0 + k * (rz_weight(sc, 9, 1) - wf));
  a.comp[1] = (float)(1.0 + k * (rz_weight(sc, 9, 2) - wf));
  a.comp[2] = (float)(1.0 + k * (rz_weight(sx, xkg / 2, 1) - wf));
  a.comp[3] = (float)(1.0 + k * (rz_weight(sx, xkg / 2, 2) - wf));
}
// enough (split x pair) CTAs for two waves, splits of 1K..64K pixels (multiples of 128)
int gram_px_per_split(long long px, int pairs) {
  const long long want_splits = std::max<long long>(1, (2 * kSMs + pairs - 1) / pairs);
  long long per = (px + want_splits - 1) / want_splits;
  per = std::max<long long>(1024, std::min<long long>(kMaxPxPerSplit, per));
  return (int)((per + 255) / 256 * 256);  // whole 64- and 256-pixel stages
}
int ntile_for(int C_p) { return (C_p % 128 == 0) ? 128 : 64; }
float pow2f(int e) { return std::ldexp(1.0f, e); }
int choose_exp(float amax) {
  if (!(amax > 0.f) || !std::isfinite(amax)) return 0;
  int e = (int)std::floor(kTargetLog2 - std::log2(amax));
  return std::max(-40, std::min(90, e));
}
bool range_bad(float amax, float scale) {
  return !std::isfinite(amax) || amax * scale > kOverflow || (amax > 0.f && amax * scale < kUnderflow);
}
float bits_to_float(unsigned int u) {
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
void split_host(double v, __half& hi, __half& lo) {
  hi = __float2half_rn((float)v);
  lo = __float2half_rn((float)(v - (double)__half2float(hi)));
}

struct TapState {
  int stage = -1;
  double *S = nullptr, *s = nullptr, *Gr = nullptr, *mur = nullptr, *sdr = nullptr;
  double *mu = nullptr, *sd = nullptr, *ratio = nullptr, *row_loss = nullptr, *row_mmax = nullptr,
         *ms_loss = nullptr;
  int* degenerate = nullptr;
  float* bvec = nullptr;
  __half* xw = nullptr;
  double wg = 0, wm = 0, ws = 0, n = 0, mmax = 0;
  bool has_ref = false;
  float* gram_partial = nullptr;
  int gram_splits = 0;
  int gram_px = 1024;
  float* colsum_partial = nullptr;
  int colsum_rows = 0;
  double* colsum_mid = nullptr;
};

// launch-timer classes: 0 conv3x3_tc N=128, 1 conv3x3_tc N=64, 2 Gram (tc kernel + reduce)
constexpr int kTimerClasses = 4;

struct Expo {
  int e = 0;
  bool known = false;
};

struct Stage {
  int cin = 0, cout = 0, cin_p = 0, cout_p = 0;
  bool pool_after = false;
  bool pool_max = false;         // max instead of average pooling after this stage
  uint32_t* pool_arg = nullptr;  // first-argmax bits of the max pool (2 per element)
  int style = -1;
  bool content = false;
  int stride = 1;
  std::vector<double> w, b;
  int wexp = 0;
  float* bias_d = nullptr;
  uint8_t* wf_d = nullptr;
  uint8_t* w1b_d = nullptr;  // first stage only: adjoint slab of first_bwd_tc_kernel
  uint8_t* wb_d = nullptr;
  int H = 0, W = 0;
  HL16 out, pooled;
  bool has_out = false, store_out = false;
  uint32_t* mask = nullptr;
  Expo out_e, pool_e, g_e, add_e;
  float g_written = 1.f;
};

}  // namespace

struct spst_ctx {
  int code = SPST_OK;
  std::string msg;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::vector<Stage> stages;
  std::vector<TapState> taps;
  int content_stage = -1;
  int perm[3] = {0, 1, 2};
  float mean[3] = {0, 0, 0}, scale[3] = {1, 1, 1};
  int deepest_stride = 1;
  std::vector<void*> persistent;  // weights
  std::vector<void*> allocs;      // bound workspace
  long long alloc_bytes = 0;
  bool bound = false;
  int h = 0, w = 0, Hp = 0, Wp = 0, grid_r0 = 0, grid_r1 = 0, own_r0 = 0, own_r1 = 0;
  int grid_c0 = 0, grid_c1 = 0, own_c0 = 0, own_c1 = 0;  // window columns (padded-image coordinates)
  long long x_pitch = 0, g_pitch = 0;                     // pixels per row of the image / gradient buffers
  unsigned int* amax_d = nullptr;  // [stages][4]: out, pooled, grad, addend; [4 * stages]: image
  HL16 img;                        // first conv's K operand (8-channel HL16 image), see image_hl_kernel
  Expo img_e;
  // opt-in launch timer (spst_timing_*): CUDA events around each tensor-core launch on `stream`
  struct LaunchTimer {
    cudaEvent_t a = nullptr, b = nullptr;
    int cls = 0;
    double flops = 0;
  };
  bool timing = false;
  std::vector<LaunchTimer> tpool;
  size_t tused = 0;
  double t_ms[kTimerClasses] = {}, t_flops[kTimerClasses] = {};
  long long t_n[kTimerClasses] = {};
  double* fin_d = nullptr;  // per-tap loss outputs (bind_alloc)
  HL16 gbuf[2];
  size_t gbuf_elems = 0;
  HL16 addend;
  size_t addend_elems = 0;
  float* gimg = nullptr;
  HL16 content_u;
  bool content_captured = false;
  double* content_partial = nullptr;
  __half* zero_xw = nullptr;
  bool fwd_done = false, finalized = false;
  int precision = 0;  // SPST_PRECISION_*: 0 fp16x3 (fp32-class, default), 1 fp16 (one MMA pass, opt-in)
  // Deferred end-of-pass range checks (fast path): the forward's check is resolved by the next
  // call that needs its results (finalize's one read-back, or capture / stats / features), the
  // backward's by spst_backward_resolve -- one host synchronisation per pass pair instead of
  // one per pass.  Pinned read-back buffers so the copies stay asynchronous.
  bool fwd_pending = false, fwd_redone = false, bwd_pending = false;
  const float* fwd_x = nullptr;
  double bwd_lambda = 0.0;
  float* bwd_grad = nullptr;
  unsigned int* amax_pin = nullptr;  // [4 * stages + 4]
  double* fin_pin = nullptr;
  size_t fin_count = 0;

  int fail(int c, const std::string& m) {
    code = c;
    msg = m;
    return c;
  }
  int cuda(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return SPST_OK;
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? SPST_ERR_OOM : SPST_ERR_CUDA,
                std::string(where) + ": " + cudaGetErrorString(e));
  }
  // Bound (per image size) buffers come from a per-context stream-ordered pool that keeps freed
  // memory reserved: a multiscale run re-binds at every scale and would otherwise return and
  // re-map tens of GB through the driver each time.  Persistent buffers (weights) use cudaMalloc.
  cudaMemPool_t pool = nullptr;
  bool pool_ready() {
    if (pool) return true;
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      pool = nullptr;
      return false;
    }
    uint64_t keep_all = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep_all);
    return true;
  }
  template <typename T>
  T* dalloc(size_t n, bool keep = false) {
    void* p = nullptr;
    if (n == 0) n = 1;
    const cudaError_t e = (!keep && pool_ready()) ? cudaMallocFromPoolAsync(&p, n * sizeof(T), pool, stream)
                                                  : cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    (keep ? persistent : allocs).push_back(p);
    if (!keep) alloc_bytes += (long long)(n * sizeof(T));
    return reinterpret_cast<T*>(p);
  }
  void release_bound() {
    if (stream) cudaStreamSynchronize(stream);
    cudaDeviceSynchronize();
    for (void* p : allocs) pool ? cudaFreeAsync(p, stream) : cudaFree(p);
    if (pool) cudaStreamSynchronize(stream);
    allocs.clear();
    alloc_bytes = 0;
    fin_d = nullptr;
    bound = false;
    fwd_done = finalized = content_captured = false;
    for (auto& t : taps) {
      t.S = t.s = t.mu = t.sd = t.ratio = t.row_loss = t.row_mmax = t.ms_loss = nullptr;
      t.degenerate = nullptr;
      t.bvec = nullptr;
      t.xw = nullptr;
      t.gram_partial = nullptr;
      t.colsum_partial = nullptr;
    }
  }
};

#define CK(call)                               \
  do {                                         \
    int _r = ctx->cuda((call), #call);         \
    if (_r) return _r;                         \
  } while (0)
#define TRY(call)          \
  do {                     \
    int _r = (call);       \
    if (_r) return _r;     \
  } while (0)

namespace {
std::atomic<long long> g_launches{0};
}  // namespace
void spst::note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

double spst::rz_weight(int small, int large, int chunks) {
  const double n = (double)large * chunks;
  double w = 0.0;
  int m = 0;
  for (int c = 0; c < chunks; ++c) {
    w += small * (m / n);
    for (int j = 0; j < large; ++j) w += (++m) / n;
  }
  return w;
}

// Round-toward-zero compensation constants (conv_tc.cu), measured on B200 with
// tools/rz_calibrate.py: mixed-sign sums lose ~kappa x (MMAs weighted by the partial-sum
// growth) -- one truncation of the result per MMA, 0.5 x E[ulp/|x|] -- while same-sign sums
// (Gram entries of ReLU features) also lose every addend's alignment truncation (set_gram_comp).
// SPST_RZ_KAPPA overrides (0 disables all compensation).
double spst::rz_kappa() {
  static const double k = [] {
    const char* e = getenv("SPST_RZ_KAPPA");
    return e && *e ? atof(e) : 3.3e-8;
  }();
  return k;
}


namespace {

// ------------------------------------------------------------------------------------------
// weight staging: [nt][kc][pass][tap][kg][n][8]
//   fwd: n -> output channel, k -> input channel
//   bwd: adjoint conv: n -> input channel, k -> output channel, taps flipped (2-dy, 2-dx)
// ------------------------------------------------------------------------------------------
std::vector<__half> stage_slabs(const Stage& s, bool bwd, int N) {
  const int K_p = bwd ? s.cout_p : s.cin_p;
  const int N_p = bwd ? s.cin_p : s.cout_p;
  const int nkc = K_p / 16, nnt = N_p / N;
  std::vector<__half> out((size_t)nnt * nkc * 2 * 9 * 2 * N * 8);
  const double sc = std::ldexp(1.0, s.wexp);
  // N=128: [pass][tap][kg][n][8].  N=64 (row-pair MMAs, see conv_tc.cu):
  // [pass][dx][kg][2-dy][n][8], so [W_dy2 ; W_dy1 ; W_dy0] is contiguous per (pass, dx, kg).
  const bool rowpair = N == 64;
  for (int nt = 0; nt < nnt; ++nt)
    for (int kc = 0; kc < nkc; ++kc)
      for (int pass = 0; pass < 2; ++pass)
        for (int tap = 0; tap < 9; ++tap)
          for (int kg = 0; kg < 2; ++kg)
            for (int n = 0; n < N; ++n)
              for (int e = 0; e < 8; ++e) {
                const size_t chunk = (size_t)(nt * nkc + kc) * 2 * 9 * 2 * N * 8;
                const int tdy = tap / 3, tdx = tap % 3;
                const size_t idx =
                    chunk + (rowpair ? (((((size_t)pass * 3 + tdx) * 2 + kg) * 3 + (2 - tdy)) * N + n) * 8 + e
                                     : ((((size_t)pass * 9 + tap) * 2 + kg) * N + n) * 8 + e);
                const int ng = nt * N + n, kk = kc * 16 + kg * 8 + e;
                const int dy = tap / 3, dx = tap % 3;
                const int co = bwd ? kk : ng, ci = bwd ? ng : kk;
                const int ty = bwd ? 2 - dy : dy, tx = bwd ? 2 - dx : dx;
                double v = 0.0;
                if (co < s.cout && ci < s.cin) v = s.w[(((size_t)co * s.cin + ci) * 3 + ty) * 3 + tx] * sc;
                __half hi, lo;
                split_host(v, hi, lo);
                out[idx] = pass == 0 ? hi : lo;
              }
  return out;
}

int parse_net(spst_ctx* ctx, int n_layers, const int* kinds, const int* cin, const int* cout,
              const double* const* weights, const double* const* biases, int n_style, const int* style_layers,
              int content_layer) {
  int last = content_layer;
  for (int i = 0; i < n_style; ++i) last = std::max(last, style_layers[i]);
  if (last < 0 || last >= n_layers) return ctx->fail(SPST_ERR_CONFIG, "tap layer index out of range");
  int i = 0, stride = 1, prev_c = 3;
  while (i <= last) {
    if (kinds[i] != SPST_LAYER_CONV)
      return ctx->fail(SPST_ERR_UNSUPPORTED,
                       "device path expects (conv, relu[, pool]) groups; layer " + std::to_string(i) + " breaks it");
    if (i + 1 >= n_layers || kinds[i + 1] != SPST_LAYER_RELU)
      return ctx->fail(SPST_ERR_UNSUPPORTED, "every conv must be followed by a relu on the device path");
    Stage s;
    s.cin = cin[i];
    s.cout = cout[i];
    if (s.cin != prev_c) return ctx->fail(SPST_ERR_SHAPE, "conv input channels do not chain");
    if (ctx->stages.empty() && s.cout > kFirstC)
      return ctx->fail(SPST_ERR_UNSUPPORTED, "first conv layer supports at most 64 output channels");
    s.cin_p = ctx->stages.empty() ? 16 : round_up(s.cin, 64);  // image: one 16-channel K chunk
    s.cout_p = round_up(s.cout, 64);
    s.stride = stride;
    s.w.assign(weights[i], weights[i] + (size_t)s.cout * s.cin * 9);
    s.b.assign(biases[i], biases[i] + s.cout);
    double mx = 0;
    for (double v : s.w) mx = std::max(mx, std::fabs(v));
    s.wexp = mx > 0 ? (int)std::floor(std::log2(16384.0 / mx)) : 0;
    const int relu_idx = i + 1;
    for (int t = 0; t < n_style; ++t)
      if (style_layers[t] == relu_idx) s.style = t;
    s.content = content_layer == relu_idx;
    i += 2;
    if (i <= last && (kinds[i] == SPST_LAYER_AVGPOOL || kinds[i] == SPST_LAYER_MAXPOOL)) {
      s.pool_max = kinds[i] == SPST_LAYER_MAXPOOL;
      s.pool_after = true;
      stride *= 2;
      ++i;
    }
    prev_c = s.cout;
    ctx->stages.push_back(std::move(s));
  }
  ctx->taps.assign(n_style, TapState());
  for (int t = 0; t < n_style; ++t) {
    bool found = false;
    for (size_t k = 0; k < ctx->stages.size(); ++k)
      if (ctx->stages[k].style == t) {
        ctx->taps[t].stage = (int)k;
        found = true;
      }
    if (!found) return ctx->fail(SPST_ERR_CONFIG, "style tap " + std::to_string(t) + " is not a conv relu");
  }
  ctx->content_stage = -1;
  for (size_t k = 0; k < ctx->stages.size(); ++k)
    if (ctx->stages[k].content) ctx->content_stage = (int)k;
  // deepest stride among taps (extractor.py:95-96)
  ctx->deepest_stride = 1;
  for (auto& t : ctx->taps) ctx->deepest_stride = std::max(ctx->deepest_stride, ctx->stages[t.stage].stride);
  if (ctx->content_stage >= 0)
    ctx->deepest_stride = std::max(ctx->deepest_stride, ctx->stages[ctx->content_stage].stride);
  // the trailing pool of the last stage (if any) is never evaluated
  ctx->stages.back().pool_after = false;
  return SPST_OK;
}

int upload_weights(spst_ctx* ctx) {
  for (size_t k = 0; k < ctx->stages.size(); ++k) {
    Stage& s = ctx->stages[k];
    std::vector<float> b32(s.cout_p, 0.f);
    for (int c = 0; c < s.cout; ++c) b32[c] = (float)s.b[c];
    s.bias_d = ctx->dalloc<float>(s.cout_p, true);
    if (!s.bias_d) return ctx->fail(SPST_ERR_OOM, "bias upload");
    CK(cudaMemcpy(s.bias_d, b32.data(), b32.size() * 4, cudaMemcpyHostToDevice));
    auto wf = stage_slabs(s, false, ntile_for(s.cout_p));
    s.wf_d = ctx->dalloc<uint8_t>(wf.size() * 2, true);
    if (!s.wf_d) return ctx->fail(SPST_ERR_OOM, "forward weight slabs");
    CK(cudaMemcpy(s.wf_d, wf.data(), wf.size() * 2, cudaMemcpyHostToDevice));
    if (k == 0) {  // adjoint slab of the first conv: [hi|lo][kg][n = c*9+dy*3+dx (32)][8 k]
      std::vector<__half> w1b(2 * 8 * 32 * 8, __float2half(0.f));
      const double sc = std::ldexp(1.0, s.wexp);
      for (int kk = 0; kk < std::min(s.cout, 64); ++kk)
        for (int c = 0; c < s.cin; ++c)
          for (int t = 0; t < 9; ++t) {
            __half hi, lo;
            split_host(s.w[((size_t)kk * s.cin + c) * 9 + t] * sc, hi, lo);
            const int n = c * 9 + t;
            const size_t off = ((size_t)(kk / 8) * 32 + n) * 8 + kk % 8;
            w1b[off] = hi;
            w1b[8 * 32 * 8 + off] = lo;
          }
      s.w1b_d = ctx->dalloc<uint8_t>(w1b.size() * 2, true);
      if (!s.w1b_d) return ctx->fail(SPST_ERR_OOM, "first-layer adjoint slab");
      CK(cudaMemcpy(s.w1b_d, w1b.data(), w1b.size() * 2, cudaMemcpyHostToDevice));
    }
    if (k > 0) {
      auto wb = stage_slabs(s, true, ntile_for(s.cin_p));
      s.wb_d = ctx->dalloc<uint8_t>(wb.size() * 2, true);
      if (!s.wb_d) return ctx->fail(SPST_ERR_OOM, "backward weight slabs");
      CK(cudaMemcpy(s.wb_d, wb.data(), wb.size() * 2, cudaMemcpyHostToDevice));
    }
  }
  return SPST_OK;
}

HL16 hl_shape(int C_p, int H, int W) {
  HL16 t;
  t.C_p = C_p;
  t.H = H;
  t.W = W;
  t.scale = 1.f;
  return t;
}

// ------------------------------------------------------------------------------------------
// one tensor-core conv / GEMM launch
// ------------------------------------------------------------------------------------------
struct ConvLaunch {
  const HL16* in = nullptr;      // conv K operand (nullptr: extra-K only)
  const uint8_t* wslab = nullptr;
  const HL16* v = nullptr;       // extra-K operand
  const __half* xw = nullptr;
  int H = 0, W = 0;              // GEMM grid (conv output grid)
  float acc_scale = 1.f;
  double flops = 0;              // algorithmic FLOPs (real channels, one pass) for the launch timer
  int drain = 1;                 // K-chunks per TMEM accumulation group
  ConvArgs a{};
};

spst_ctx::LaunchTimer* timer_begin(spst_ctx* ctx, int cls, double flops) {
  if (!ctx->timing) return nullptr;
  if (ctx->tused == ctx->tpool.size()) {
    spst_ctx::LaunchTimer t;
    if (cudaEventCreate(&t.a) != cudaSuccess || cudaEventCreate(&t.b) != cudaSuccess) return nullptr;
    ctx->tpool.push_back(t);
  }
  spst_ctx::LaunchTimer* t = &ctx->tpool[ctx->tused++];
  t->cls = cls;
  t->flops = flops;
  cudaEventRecord(t->a, ctx->stream);
  return t;
}
void timer_end(spst_ctx* ctx, spst_ctx::LaunchTimer* t) {
  if (t) cudaEventRecord(t->b, ctx->stream);
}
// fold the recorded launches into the per-class totals (the stream has been synchronized)
void timer_collect(spst_ctx* ctx) {
  for (size_t i = 0; i < ctx->tused; ++i) {
    const auto& t = ctx->tpool[i];
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.a, t.b) == cudaSuccess) {
      ctx->t_ms[t.cls] += ms;
      ctx->t_flops[t.cls] += t.flops;
      ctx->t_n[t.cls] += 1;
    }
  }
  ctx->tused = 0;
}

int run_conv(spst_ctx* ctx, ConvLaunch& L) {
  ConvArgs& a = L.a;
  const HL16* in = L.in ? L.in : L.v;
  const HL16* v = L.v ? L.v : in;
  const int N = ntile_for(a.out.C_p);
  const int mt = conv_tc_rows(N);
  if (!map_rows(&a.tm_r_hi, in->hi, in->C_p / 8, in->H, in->W) ||
      !map_rows(&a.tm_r_lo, in->lo(), in->C_p / 8, in->H, in->W) ||
      !map_act(&a.tm_v_hi, v->hi, v->C_p / 8, v->H, v->W, mt, true, conv_tc_xkg(N)) ||
      !map_act(&a.tm_v_lo, v->lo(), v->C_p / 8, v->H, v->W, mt, true, conv_tc_xkg(N)))
    return ctx->fail(SPST_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  a.wgt = L.in ? L.wslab : nullptr;
  a.n_kc = L.in ? (L.in->C_p + 15) / 16 : 0;  // an 8-channel input reads its 2nd K group as TMA zero fill
  a.xwgt = reinterpret_cast<const uint8_t*>(L.xw);
  a.n_xkc = L.xw ? v->C_p / (8 * conv_tc_xkg(N)) : 0;
  a.H = L.H;
  a.W = L.W;
  a.n_ntiles = a.out.C_p / N;
  a.tiles_x = (L.W + 127) / 128;
  a.tiles_y = (L.H + mt - 1) / mt;
  a.acc_scale = L.acc_scale;
  a.drain = L.drain;
  a.pass0 = ctx->precision == 1 ? 2 : 0;
  if (a.n_kc + a.n_xkc == 0) return ctx->fail(SPST_ERR_CONFIG, "empty GEMM");
  const int tiles = a.tiles_x * a.tiles_y * a.n_ntiles;
  set_conv_comp(a, N);
  const int grid = std::min(tiles, kSMs);  // persistent: one CTA per SM
  auto* tm = timer_begin(ctx, N == 128 ? 0 : 1, L.flops);
  CK(launch_conv_tc(a, N, grid, ctx->stream));
  timer_end(ctx, tm);
  return SPST_OK;
}

float read_amax(spst_ctx* ctx, int slot) {
  unsigned int v = 0;
  cudaMemcpyAsync(&v, ctx->amax_d + slot, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  return bits_to_float(v);
}

// ------------------------------------------------------------------------------------------
// forward (extractor.py:171-197) + statistics (localized.py:162-184, stats.py:43-50)
// ------------------------------------------------------------------------------------------
int forward_stage(spst_ctx* ctx, int k, const float* x) {
  Stage& s = ctx->stages[k];
  const int own0 = (ctx->own_r0 - ctx->grid_r0) / s.stride, own1 = (ctx->own_r1 - ctx->grid_r0) / s.stride;
  const int ownc0 = (ctx->own_c0 - ctx->grid_c0) / s.stride, ownc1 = (ctx->own_c1 - ctx->grid_c0) / s.stride;
  TapState* tap = s.style >= 0 ? &ctx->taps[s.style] : nullptr;
  s.out.scale = pow2f(s.out_e.e);
  s.pooled.scale = pow2f(s.pool_e.e);
  CK(cudaMemsetAsync(ctx->amax_d + 4 * k, 0, 8, ctx->stream));
  if (k == 0) {
    ImageHLArgs ia{};
    ia.img = x;
    ia.h = ctx->h;
    ia.w = ctx->w;
    ia.row_off = ctx->grid_r0;
    ia.col_off = ctx->grid_c0;
    ia.pitch = ctx->x_pitch;
    ia.Hl = s.H;
    ia.Wp = s.W;
    for (int c = 0; c < 3; ++c) {
      ia.perm[c] = ctx->perm[c];
      ia.mean[c] = ctx->mean[c];
      ia.scale[c] = ctx->scale[c];
    }
    ctx->img.scale = pow2f(ctx->img_e.e);
    ia.out = ctx->img;
    ia.amax = ctx->amax_d + 4 * ctx->stages.size();
    CK(cudaMemsetAsync(ia.amax, 0, 4, ctx->stream));
    CK(launch_image_hl(ia, ctx->stream));
  }
  const HL16& in = k == 0 ? ctx->img : (ctx->stages[k - 1].pool_after ? ctx->stages[k - 1].pooled : ctx->stages[k - 1].out);
  ConvLaunch L;
  L.in = &in;
  L.wslab = s.wf_d;
  L.H = s.H;
  L.W = s.W;
  L.acc_scale = 1.f / (in.scale * pow2f(s.wexp));
  L.flops = 2.0 * s.H * s.W * s.cout * 9.0 * s.cin;
  L.drain = fwd_drain();
  ConvArgs& a = L.a;
  a.epi = s.pool_after ? EPI_FWD_POOL : EPI_FWD;
  a.bias = s.bias_d;
  a.mask_out = s.mask;
  a.out = s.out;
  a.out_pool = s.pooled;
  a.pool_max = s.pool_after && s.pool_max;
  a.pool_arg = s.pool_arg;
  a.store_full = s.store_out ? 1 : 0;
  a.colsum_partial = tap ? tap->colsum_partial : nullptr;
  a.sum_r0 = own0;
  a.sum_r1 = own1;
  a.sum_c0 = ownc0;
  a.sum_c1 = ownc1;
  a.amax = ctx->amax_d + 4 * k;
  return run_conv(ctx, L);
}

int stage_stats(spst_ctx* ctx, int k) {
  Stage& s = ctx->stages[k];
  if (s.style < 0) return SPST_OK;
  TapState& t = ctx->taps[s.style];
  CK(launch_colsum_reduce(t.colsum_partial, t.colsum_rows, s.cout, s.cout_p, t.s, t.colsum_mid, ctx->stream));
  const int own0 = (ctx->own_r0 - ctx->grid_r0) / s.stride, own1 = (ctx->own_r1 - ctx->grid_r0) / s.stride;
  const int ownc0 = (ctx->own_c0 - ctx->grid_c0) / s.stride, ownc1 = (ctx->own_c1 - ctx->grid_c0) / s.stride;
  const long long o0 = (long long)own0 * s.W + ownc0;
  GramArgs g{};
  if (!map_gram(&g.tm_hi, s.out.hi + o0 * 8, ownc1 - ownc0, own1 - own0, s.W, s.H, s.cout_p / 8) ||
      !map_gram(&g.tm_lo, s.out.lo() + o0 * 8, ownc1 - ownc0, own1 - own0, s.W, s.H, s.cout_p / 8))
    return ctx->fail(SPST_ERR_CUDA, "cuTensorMapEncodeTiled failed (gram)");
  g.C_p = s.cout_p;
  g.rows = own1 - own0;
  g.w_own = ownc1 - ownc0;
  g.px_per_split = t.gram_px;
  const long long p0 = 0, p1 = (long long)g.rows * g.w_own;  // owned pixels (launch timer)
  g.n_ctile = (s.cout_p + 127) / 128;
  g.partial = t.gram_partial;
  set_gram_comp(g, s.cout_p);
  const double inv2 = 1.0 / ((double)s.out.scale * (double)s.out.scale);
  auto* tm = timer_begin(ctx, 2, 2.0 * (double)(p1 - p0) * s.cout * s.cout);
  if (s.cout_p == 64) {
    CK(launch_gram64_tc(g, t.gram_splits, s.cout, inv2, t.S, ctx->stream));
  } else {
    CK(launch_gram_tc(g, t.gram_splits, ctx->stream));
    CK(launch_gram_reduce(t.gram_partial, t.gram_splits, g.n_ctile, s.cout, inv2, t.S, ctx->stream));
  }
  timer_end(ctx, tm);
  return SPST_OK;
}

bool stage_ranges_ok(spst_ctx* ctx, int k, float m0, float m1) {
  const Stage& s = ctx->stages[k];
  bool ok = true;
  if (s.has_out && range_bad(m0, s.out.scale)) ok = false;
  if (s.pool_after && range_bad(m1, s.pooled.scale)) ok = false;
  return ok;
}

int forward_check(spst_ctx* ctx);

// SPST_DEBUG_HOST_US=1: host microseconds spent in each phase of a forward (launch-overhead probe)
static double host_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int do_forward(spst_ctx* ctx, const float* x, bool careful) {
  const int n = (int)ctx->stages.size();
  static const bool dbg_us = env_int("SPST_DEBUG_HOST_US", 0) != 0;
  const double t0 = dbg_us ? host_us() : 0.0;
  for (int k = 0; k < n; ++k) {
    Stage& s = ctx->stages[k];
    const bool check = careful || (s.has_out && !s.out_e.known) || (s.pool_after && !s.pool_e.known) ||
                       (k == 0 && !ctx->img_e.known);
    for (int attempt = 0; attempt < 6; ++attempt) {
      TRY(forward_stage(ctx, k, x));
      if (!check) break;
      bool img_ok = true;
      if (k == 0) {  // the image operand is range-checked like every stored tensor
        const float mi = read_amax(ctx, 4 * n);
        img_ok = !range_bad(mi, ctx->img.scale);
        ctx->img_e = {choose_exp(mi), true};
      }
      const float m0 = read_amax(ctx, 4 * k), m1 = read_amax(ctx, 4 * k + 1);
      const bool ok = stage_ranges_ok(ctx, k, m0, m1) && img_ok;
      if (s.has_out) s.out_e = {choose_exp(m0), true};
      if (s.pool_after) s.pool_e = {choose_exp(m1), true};
      if (ok) break;
    }
  }
  const double t1 = dbg_us ? host_us() : 0.0;
  for (int k = 0; k < n; ++k) TRY(stage_stats(ctx, k));
  CK(cudaMemcpyAsync(ctx->amax_pin, ctx->amax_d, 16 * n + 16, cudaMemcpyDeviceToHost, ctx->stream));
  if (dbg_us) fprintf(stderr, "[spst] forward host us: convs %.1f stats+copy %.1f\n", t1 - t0, host_us() - t1);
  if (!careful) {  // fast path: checked when the results are first needed (resolve_forward)
    ctx->fwd_pending = true;
    return 0;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return forward_check(ctx);
}

// end-of-pass range check of the forward (the read-back in amax_pin has completed)
int forward_check(spst_ctx* ctx) {
  const int n = (int)ctx->stages.size();
  timer_collect(ctx);
  bool bad = false;
  {
    const float mi = bits_to_float(ctx->amax_pin[4 * n]);
    if (range_bad(mi, ctx->img.scale)) bad = true;  // stale exponents (new problem / dims): redo carefully
    if (mi > 0 && std::isfinite(mi)) ctx->img_e = {choose_exp(mi), true};
  }
  for (int k = 0; k < n; ++k) {
    Stage& s = ctx->stages[k];
    const float m0 = bits_to_float(ctx->amax_pin[4 * k]), m1 = bits_to_float(ctx->amax_pin[4 * k + 1]);
    if (s.has_out && range_bad(m0, s.out.scale)) bad = true;
    if (s.pool_after && range_bad(m1, s.pooled.scale)) bad = true;
    static const bool dbg = env_int("SPST_DEBUG_RANGES", 0) != 0;
    if (dbg && ((s.has_out && range_bad(m0, s.out.scale)) || (s.pool_after && range_bad(m1, s.pooled.scale))))
      fprintf(stderr, "[spst] fwd stage %d out of range: amax %.3e x scale %.3e, pooled %.3e x %.3e\n", k, m0,
              s.out.scale, m1, s.pooled.scale);
    // exponents for the next write; the data now stored keep the scale they were written with
    if (s.has_out && m0 > 0 && std::isfinite(m0)) s.out_e = {choose_exp(m0), true};
    if (s.pool_after && m1 > 0 && std::isfinite(m1)) s.pool_e = {choose_exp(m1), true};
  }
  return bad ? 1 : 0;
}

// Resolve a deferred forward check: wait for the pass, check its ranges, and re-run it in
// careful mode if a stored tensor left its representable range (sets fwd_redone).
int resolve_forward(spst_ctx* ctx) {
  ctx->fwd_redone = false;
  if (!ctx->fwd_pending) return SPST_OK;
  ctx->fwd_pending = false;
  CK(cudaStreamSynchronize(ctx->stream));
  if (forward_check(ctx) == 0) return SPST_OK;
  int r = do_forward(ctx, ctx->fwd_x, true);
  if (r == 1) return ctx->fail(SPST_ERR_NONFINITE, "activation range could not be represented (non-finite?)");
  if (r) return r;
  ctx->fwd_redone = true;
  return SPST_OK;
}

// ------------------------------------------------------------------------------------------
// backward (extractor.py:200-214 with the tap gradients of stats.py:127-174)
// ------------------------------------------------------------------------------------------
StyleCoefArgs coef_args(spst_ctx* ctx, TapState& t) {
  const Stage& s = ctx->stages[t.stage];
  StyleCoefArgs a{};
  a.S = t.S;
  a.s = t.s;
  a.n = t.n;
  a.Gr = t.Gr;
  a.mur = t.mur;
  a.sdr = t.sdr;
  a.wg = t.wg;
  a.wm = t.wm;
  a.ws = t.ws;
  a.C = s.cout;
  a.mu = t.mu;
  a.sd = t.sd;
  a.ratio = t.ratio;
  a.bvec = t.bvec;
  a.row_loss = t.row_loss;
  a.row_mmax = t.row_mmax;
  a.ms_loss = t.ms_loss;
  a.degenerate = t.degenerate;
  a.N = ntile_for(s.cout_p);
  a.xkg = conv_tc_xkg(a.N);
  a.n_xkc = s.cout_p / (8 * a.xkg);
  return a;
}

// tap gradient slab for stage k with extra-K scale 2^xexp
int write_xw(spst_ctx* ctx, int k, int xexp) {
  Stage& s = ctx->stages[k];
  if (s.style < 0) return SPST_OK;
  TapState& t = ctx->taps[s.style];
  StyleCoefArgs a = coef_args(ctx, t);
  a.xw = t.xw;
  a.xscale = pow2f(xexp);
  CK(cudaMemsetAsync(t.xw, 0, (size_t)s.cout_p * s.cout_p * 2 * sizeof(__half), ctx->stream));
  CK(launch_style_mat(a, ctx->stream));
  return SPST_OK;
}

int gemm_only_xexp(spst_ctx* ctx, int k) {
  const Stage& s = ctx->stages[k];
  if (s.style < 0) return 0;
  const double mm = ctx->taps[s.style].mmax;
  return mm > 0 ? (int)std::floor(std::log2(16384.0 / mm)) : 0;
}

// tap gradient (V M + b + content) of stage k into `out` (GEMM with extra-K only)
int tap_grad_gemm(spst_ctx* ctx, int k, HL16 out, bool with_mask, double two_lambda, int slot) {
  Stage& s = ctx->stages[k];
  const int xexp = gemm_only_xexp(ctx, k);
  TRY(write_xw(ctx, k, xexp));
  ConvLaunch L;
  L.v = &s.out;
  L.xw = s.style >= 0 ? ctx->taps[s.style].xw : ctx->zero_xw;
  L.H = s.H;
  L.W = s.W;
  L.acc_scale = 1.f / (s.out.scale * pow2f(xexp));
  L.flops = s.style >= 0 ? 2.0 * s.H * s.W * s.cout * s.cout : 0.0;  // style GEMM V M (content-only: none)
  L.drain = bwd_drain();
  ConvArgs& a = L.a;
  a.x_rescale = 1.f;
  a.epi = EPI_BWD;
  a.bias = s.style >= 0 ? ctx->taps[s.style].bvec : nullptr;
  a.mask_in = with_mask ? s.mask : nullptr;
  a.out = out;
  if (s.content && two_lambda != 0.0) {
    a.content_v = s.out;
    a.content_u = ctx->content_u;
    a.content_coef = (float)two_lambda;
  }
  a.amax = ctx->amax_d + slot;
  return run_conv(ctx, L);
}

// produce g_k (gradient at stage k's conv output) into gbuf[dst] from g_{k+1} in gbuf[src]
int backward_stage(spst_ctx* ctx, int k, int src, int dst, double two_lambda) {
  Stage& s = ctx->stages[k];
  Stage& nx = ctx->stages[k + 1];
  HL16 gin = ctx->gbuf[src];  // shape set by the caller
  HL16 gout = hl_shape(s.cout_p, s.H, s.W);
  gout.hi = ctx->gbuf[dst].hi;
  gout.scale = pow2f(s.g_e.e);
  s.g_written = gout.scale;
  const bool is_tap = s.style >= 0 || (s.content && two_lambda != 0.0);
  ConvLaunch L;
  L.in = &gin;
  L.wslab = nx.wb_d;
  L.H = nx.H;
  L.W = nx.W;
  // the input gradient carries the scale it was WRITTEN with (gin.scale = stage k+1's g_written);
  // g_e may already hold the exponent chosen for the next write (careful mode updates it per
  // stage), so it must not be used here
  const int acc_e = (int)std::lround(std::log2((double)gin.scale)) + nx.wexp;
  L.acc_scale = 1.f / pow2f(acc_e);
  L.flops = 2.0 * nx.H * nx.W * nx.cin * 9.0 * nx.cout;  // input-gradient GEMM of conv k+1
  L.drain = bwd_drain();
  ConvArgs& a = L.a;
  a.x_rescale = 1.f;
  a.out = gout;
  a.mask_in = s.mask;
  a.amax = ctx->amax_d + 4 * k + 2;
  bool use_addend = false;
  if (s.pool_after) {
    a.epi = EPI_BWD_POOL;
    a.pool_max = s.pool_max;
    a.pool_arg = s.pool_arg;
    use_addend = is_tap;
  } else {
    a.epi = EPI_BWD;
    if (s.style >= 0) {
      // V*M enters as extra K-steps of the same GEMM; its chunks carry their own scale 2^(eV+xexp)
      // and are rescaled to the conv accumulator's 2^acc_e when the epilogue drains them
      const int xexp = gemm_only_xexp(ctx, k);
      TRY(write_xw(ctx, k, xexp));
      L.v = &s.out;
      L.xw = ctx->taps[s.style].xw;
      L.flops += 2.0 * s.H * s.W * s.cout * s.cout;  // fused style GEMM V M
      a.x_rescale = (float)std::ldexp(1.0, acc_e - xexp) / s.out.scale;
      a.bias = ctx->taps[s.style].bvec;
    }
    if (s.content && two_lambda != 0.0 && !use_addend) {
      a.content_v = s.out;
      a.content_u = ctx->content_u;
      a.content_coef = (float)two_lambda;
    }
  }
  if (use_addend) {
    HL16 ad = hl_shape(s.cout_p, s.H, s.W);
    ad.hi = ctx->addend.hi;
    for (int attempt = 0; attempt < 6; ++attempt) {
      ad.scale = pow2f(s.add_e.e);
      CK(cudaMemsetAsync(ctx->amax_d + 4 * k + 3, 0, 4, ctx->stream));
      TRY(tap_grad_gemm(ctx, k, ad, false, two_lambda, 4 * k + 3));
      const float m = read_amax(ctx, 4 * k + 3);
      const bool ok = !range_bad(m, ad.scale);
      s.add_e = {choose_exp(m), true};
      if (ok) break;
    }
    a.addend = ad;
    a.bias = nullptr;
    L.v = nullptr;
    L.xw = nullptr;
  }
  CK(cudaMemsetAsync(ctx->amax_d + 4 * k + 2, 0, 4, ctx->stream));
  return run_conv(ctx, L);
}

int backward_check(spst_ctx* ctx, bool careful);

int do_backward(spst_ctx* ctx, double two_lambda, float* grad, bool careful) {
  const int n = (int)ctx->stages.size();
  const int Lst = n - 1;
  Stage& sl = ctx->stages[Lst];
  int cur = 0;
  // deepest tap: g_L = mask * tapgrad (extractor.py:204-209 for the first tap met in reverse)
  for (int attempt = 0; attempt < 6; ++attempt) {
    HL16 g = hl_shape(sl.cout_p, sl.H, sl.W);
    g.hi = ctx->gbuf[cur].hi;
    g.scale = pow2f(sl.g_e.e);
    sl.g_written = g.scale;
    ctx->gbuf[cur] = g;
    CK(cudaMemsetAsync(ctx->amax_d + 4 * Lst + 2, 0, 4, ctx->stream));
    TRY(tap_grad_gemm(ctx, Lst, g, true, two_lambda, 4 * Lst + 2));
    if (!(careful || !sl.g_e.known)) break;
    const float m = read_amax(ctx, 4 * Lst + 2);
    const bool ok = !range_bad(m, g.scale);
    if (m > 0) sl.g_e = {choose_exp(m), true};
    if (ok || m == 0.f) break;
  }
  for (int k = Lst - 1; k >= 0; --k) {
    Stage& s = ctx->stages[k];
    const bool check = careful || !s.g_e.known;
    for (int attempt = 0; attempt < 6; ++attempt) {
      TRY(backward_stage(ctx, k, cur, cur ^ 1, two_lambda));
      if (!check) break;
      const float m = read_amax(ctx, 4 * k + 2);
      const bool ok = !range_bad(m, s.g_written);
      if (m > 0) s.g_e = {choose_exp(m), true};
      if (ok || m == 0.f) break;
    }
    HL16 g = hl_shape(s.cout_p, s.H, s.W);
    g.hi = ctx->gbuf[cur ^ 1].hi;
    g.scale = s.g_written;
    cur ^= 1;
    ctx->gbuf[cur] = g;
  }
  // first conv adjoint + preprocess adjoint, then fold the replicate padding
  Stage& s0 = ctx->stages[0];
  static const bool simt_first_bwd = [] {
    const char* e = getenv("SPST_FIRSTBWD_SIMT");
    return e && atoi(e) != 0;
  }();
  if (!simt_first_bwd && s0.cin == 3 && ctx->gbuf[cur].C_p == 64) {
    const HL16& g0 = ctx->gbuf[cur];
    FirstBwdTcArgs fb{};
    if (!map_rows128(&fb.tm_hi, g0.hi, g0.H, g0.W) || !map_rows128(&fb.tm_lo, g0.lo(), g0.H, g0.W))
      return ctx->fail(SPST_ERR_CUDA, "cuTensorMapEncodeTiled failed (first-conv adjoint)");
    fb.wslab = s0.w1b_d;
    fb.H = g0.H;
    fb.W = g0.W;
    fb.acc_scale = 1.f / (g0.scale * pow2f(s0.wexp));
    for (int c = 0; c < 3; ++c) {
      fb.perm[c] = ctx->perm[c];
      fb.scale[c] = ctx->scale[c];
    }
    fb.gimg = ctx->gimg;
    CK(launch_first_bwd_tc(fb, ctx->stream));
  } else {
  FirstConvBwdArgs b{};
  b.g = ctx->gbuf[cur];
  for (int i = 0; i < kFirstC * 27; ++i) b.wgt[i] = i < (int)s0.w.size() ? (float)s0.w[i] : 0.f;
  b.C_out = s0.cout;
  for (int c = 0; c < 3; ++c) {
    b.perm[c] = ctx->perm[c];
    b.scale[c] = ctx->scale[c];
  }
  b.gimg = ctx->gimg;
  CK(launch_first_conv_bwd(b, ctx->stream));
  }
  FoldArgs fa{};
  fa.gimg = ctx->gimg;
  fa.Hl = s0.H;
  fa.Wl = s0.W;
  fa.row_off = ctx->grid_r0;
  fa.col_off = ctx->grid_c0;
  fa.h = ctx->h;
  fa.w = ctx->w;
  fa.r0 = ctx->own_r0;
  fa.r1 = std::min(ctx->own_r1, ctx->h);
  fa.c0 = ctx->own_c0;
  fa.c1 = std::min(ctx->own_c1, ctx->w);
  fa.grad = grad;
  fa.pitch = ctx->g_pitch;
  CK(launch_fold_grad(fa, ctx->stream));
  // end-of-pass range check: deferred on the fast path (resolve_backward)
  CK(cudaMemcpyAsync(ctx->amax_pin, ctx->amax_d, 16 * n, cudaMemcpyDeviceToHost, ctx->stream));
  if (!careful) {
    ctx->bwd_pending = true;
    return 0;
  }
  CK(cudaStreamSynchronize(ctx->stream));
  return backward_check(ctx, careful);
}

int backward_check(spst_ctx* ctx, bool careful) {
  const int n = (int)ctx->stages.size();
  timer_collect(ctx);
  bool bad = false;
  static const bool dbg = env_int("SPST_DEBUG_RANGES", 0) != 0;
  for (int k = 0; k < n; ++k) {
    Stage& s = ctx->stages[k];
    const float m = bits_to_float(ctx->amax_pin[4 * k + 2]);
    if (dbg)
      fprintf(stderr, "[spst] bwd stage %d careful %d: amax %.3e written scale %.3e (stored max %.3e)\n", k,
              (int)careful, m, s.g_written, m * s.g_written);
    if (range_bad(m, s.g_written)) bad = true;
    if (m > 0 && std::isfinite(m)) s.g_e = {choose_exp(m), true};
  }
  return bad ? 1 : 0;
}

int resolve_backward(spst_ctx* ctx, int* redone) {
  if (redone) *redone = 0;
  if (!ctx->bwd_pending) return SPST_OK;
  ctx->bwd_pending = false;
  CK(cudaStreamSynchronize(ctx->stream));
  if (backward_check(ctx, false) == 0) return SPST_OK;
  int r = do_backward(ctx, ctx->bwd_lambda, ctx->bwd_grad, true);
  if (r == 1) return ctx->fail(SPST_ERR_NONFINITE, "gradient range could not be represented (non-finite?)");
  if (r) return r;
  if (redone) *redone = 1;
  return SPST_OK;
}

// a pass's results are about to be replaced or released: settle every deferred check first
int settle(spst_ctx* ctx) {
  TRY(resolve_backward(ctx, nullptr));
  return resolve_forward(ctx);
}

int bind_alloc(spst_ctx* ctx) {
  const int n = (int)ctx->stages.size();
  const int Hl = ctx->grid_r1 - ctx->grid_r0, Wl = ctx->grid_c1 - ctx->grid_c0;
  size_t gmax = 0, admax = 0;
  int max_cp = 64;
  for (int k = 0; k < n; ++k) {
    Stage& s = ctx->stages[k];
    s.H = Hl / s.stride;
    s.W = Wl / s.stride;
    static const bool store_all = [] {  // diagnostics (tools/error_budget.py): keep every relu output
      const char* e = getenv("SPST_DEBUG_STORE_ALL");
      return e && atoi(e) != 0;
    }();
    const bool tap = s.style >= 0 || s.content;
    s.has_out = !s.pool_after || tap || store_all;
    s.store_out = s.pool_after && (tap || store_all);
    s.out = hl_shape(s.cout_p, s.H, s.W);
    if (s.has_out) {
      s.out.hi = ctx->dalloc<__half>((size_t)s.cout_p * s.H * s.W * 2);
      if (!s.out.hi) return ctx->fail(SPST_ERR_OOM, "activation buffer");
    }
    s.pooled = hl_shape(s.cout_p, s.H / 2, s.W / 2);
    if (s.pool_after) {
      s.pooled.hi = ctx->dalloc<__half>((size_t)s.cout_p * (s.H / 2) * (s.W / 2) * 2);
      if (!s.pooled.hi) return ctx->fail(SPST_ERR_OOM, "pooled buffer");
      if (s.pool_max) {
        s.pool_arg = ctx->dalloc<uint32_t>((size_t)(s.cout_p / 16) * (s.H / 2) * (s.W / 2));
        if (!s.pool_arg) return ctx->fail(SPST_ERR_OOM, "max-pool argmax buffer");
      }
    }
    s.mask = ctx->dalloc<uint32_t>((size_t)(s.cout_p / 32) * s.H * s.W);
    if (!s.mask) return ctx->fail(SPST_ERR_OOM, "mask buffer");
    gmax = std::max(gmax, (size_t)s.cout_p * s.H * s.W * 2);
    if (tap) admax = std::max(admax, (size_t)s.cout_p * s.H * s.W * 2);
    max_cp = std::max(max_cp, s.cout_p);
    if (s.style >= 0) {
      TapState& t = ctx->taps[s.style];
      const int C = s.cout, Cp = s.cout_p;
      t.S = ctx->dalloc<double>((size_t)C * C);
      t.s = ctx->dalloc<double>(Cp);
      t.mu = ctx->dalloc<double>(C);
      t.sd = ctx->dalloc<double>(C);
      t.ratio = ctx->dalloc<double>(C);
      t.bvec = ctx->dalloc<float>(Cp);
      t.xw = ctx->dalloc<__half>((size_t)Cp * Cp * 2);
      const int own_rows = (ctx->own_r1 - ctx->own_r0) / s.stride, own_cols = (ctx->own_c1 - ctx->own_c0) / s.stride;
      const int kpx = Cp == 64 ? 128 : 64;  // pixels per Gram stage (gram_tc.cu)
      const long long own_px = (long long)own_rows * ((own_cols + kpx - 1) / kpx) * kpx;
      const int nct = (Cp + 127) / 128;
      t.gram_px = gram_px_per_split(own_px, nct * (nct + 1) / 2);
      t.gram_splits = (int)std::max<long long>(1, (own_px + t.gram_px - 1) / t.gram_px);
      t.gram_partial = ctx->dalloc<float>((size_t)t.gram_splits * (nct * (nct + 1) / 2) * 128 * 128);
      const int mt = conv_tc_rows(ntile_for(s.cout_p));
      t.colsum_rows = ((s.W + 127) / 128) * ((s.H + mt - 1) / mt) * 2 * mt;
      t.colsum_partial = ctx->dalloc<float>((size_t)t.colsum_rows * Cp);
      t.colsum_mid = ctx->dalloc<double>((size_t)kColsumMid * Cp);
      if (!t.S || !t.s || !t.mu || !t.sd || !t.ratio ||
          !t.bvec || !t.xw || !t.gram_partial || !t.colsum_partial || !t.colsum_mid)
        return ctx->fail(SPST_ERR_OOM, "statistics buffers");
      CK(cudaMemsetAsync(t.bvec, 0, Cp * 4, ctx->stream));
      CK(cudaMemsetAsync(t.s, 0, Cp * 8, ctx->stream));
      if (!t.Gr) {  // reference buffers persist across binds
        t.Gr = ctx->dalloc<double>((size_t)C * C, true);
        t.mur = ctx->dalloc<double>(C, true);
        t.sdr = ctx->dalloc<double>(C, true);
        if (!t.Gr || !t.mur || !t.sdr) return ctx->fail(SPST_ERR_OOM, "reference statistics");
        CK(cudaMemsetAsync(t.Gr, 0, (size_t)C * C * 8, ctx->stream));
        CK(cudaMemsetAsync(t.mur, 0, C * 8, ctx->stream));
        CK(cudaMemsetAsync(t.sdr, 0, C * 8, ctx->stream));
      }
    }
  }
  // per-tap loss outputs in one block: [row_loss C][row_mmax C][ms_loss 2][degenerate 1] per tap,
  // so spst_finalize reads every tap with one copy and one synchronisation
  {
    size_t total = 0;
    for (auto& t : ctx->taps) total += 2 * (size_t)ctx->stages[t.stage].cout + 3;
    ctx->fin_d = ctx->dalloc<double>(total);
    if (!ctx->fin_d) return ctx->fail(SPST_ERR_OOM, "statistics buffers");
    if (ctx->fin_count < total) {
      if (ctx->fin_pin) cudaFreeHost(ctx->fin_pin);
      ctx->fin_pin = nullptr;
      ctx->fin_count = 0;
      CK(cudaMallocHost(&ctx->fin_pin, total * sizeof(double)));
      ctx->fin_count = total;
    }
    size_t off = 0;
    for (auto& t : ctx->taps) {
      const int C = ctx->stages[t.stage].cout;
      t.row_loss = ctx->fin_d + off;
      t.row_mmax = t.row_loss + C;
      t.ms_loss = t.row_mmax + C;
      t.degenerate = reinterpret_cast<int*>(t.ms_loss + 2);
      off += 2 * (size_t)C + 3;
    }
    CK(cudaMemsetAsync(ctx->fin_d, 0, total * sizeof(double), ctx->stream));
  }
  for (int b = 0; b < 2; ++b) {
    ctx->gbuf[b] = hl_shape(64, 1, 1);
    ctx->gbuf[b].hi = ctx->dalloc<__half>(gmax);
    if (!ctx->gbuf[b].hi) return ctx->fail(SPST_ERR_OOM, "gradient buffers");
  }
  ctx->gbuf_elems = gmax;
  ctx->addend = hl_shape(64, 1, 1);
  ctx->addend.hi = ctx->dalloc<__half>(std::max<size_t>(admax, 16));
  ctx->addend_elems = admax;
  ctx->gimg = ctx->dalloc<float>((size_t)Hl * Wl * 3);
  ctx->amax_d = ctx->dalloc<unsigned int>(4 * n + 4);
  ctx->img = hl_shape(8, Hl, Wl);
  ctx->img.hi = ctx->dalloc<__half>((size_t)8 * Hl * Wl * 2);
  if (!ctx->img.hi) return ctx->fail(SPST_ERR_OOM, "image operand");
  ctx->content_partial = ctx->dalloc<double>(red_blocks() + 8);
  ctx->zero_xw = ctx->dalloc<__half>((size_t)max_cp * max_cp * 2);
  if (!ctx->addend.hi || !ctx->gimg || !ctx->amax_d || !ctx->content_partial || !ctx->zero_xw)
    return ctx->fail(SPST_ERR_OOM, "workspace");
  CK(cudaMemsetAsync(ctx->zero_xw, 0, (size_t)max_cp * max_cp * 2 * sizeof(__half), ctx->stream));
  CK(cudaMemsetAsync(ctx->amax_d, 0, 16 * n + 16, ctx->stream));
  if (ctx->content_stage >= 0) {
    const Stage& s = ctx->stages[ctx->content_stage];
    ctx->content_u = hl_shape(s.cout_p, s.H, s.W);
    ctx->content_u.hi = ctx->dalloc<__half>((size_t)s.cout_p * s.H * s.W * 2);
    if (!ctx->content_u.hi) return ctx->fail(SPST_ERR_OOM, "content target");
  }
  CK(cudaStreamSynchronize(ctx->stream));  // pool allocations and clears are stream-ordered
  return SPST_OK;
}

// ------------------------------------------------------------------------------------------
// debug helpers: CHW f32 <-> HL16
// ------------------------------------------------------------------------------------------
__global__ void pack_hl_kernel(const float* x, int C, HL16 t) {
  const long long n = (long long)t.C_p * t.H * t.W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / ((long long)t.H * t.W));
    const long long p = i % ((long long)t.H * t.W);
    const float v = c < C ? x[(size_t)c * t.H * t.W + p] : 0.f;
    HalfPair hp = split_f16(v * t.scale);
    const size_t off = (((size_t)(c >> 3)) * t.H * t.W + p) * 8 + (c & 7);
    t.hi[off] = hp.hi;
    t.lo()[off] = hp.lo;
  }
}

__global__ void unpack_hl_kernel(HL16 t, int C, float* x) {
  const long long n = (long long)C * t.H * t.W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / ((long long)t.H * t.W));
    const long long p = i % ((long long)t.H * t.W);
    const size_t off = (((size_t)(c >> 3)) * t.H * t.W + p) * 8 + (c & 7);
    x[i] = (__half2float(t.hi[off]) + __half2float(t.lo()[off])) / t.scale;
  }
}

__global__ void unpack_mask_kernel(const uint32_t* m, int C, int H, int W, float* x) {
  const long long n = (long long)C * H * W;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / ((long long)H * W));
    const long long p = i % ((long long)H * W);
    x[i] = (float)((m[(size_t)(c >> 5) * H * W + p] >> (c & 31)) & 1u);
  }
}

}  // namespace

// ==========================================================================================
// C ABI
// ==========================================================================================
extern "C" {

int spst_abi_version(void) { return SPST_ABI_VERSION; }

const char* spst_status_string(int s) {
  switch (s) {
    case SPST_OK: return "ok";
    case SPST_ERR_SHAPE: return "shape error";
    case SPST_ERR_GEOMETRY: return "geometry error";
    case SPST_ERR_CONFIG: return "config error";
    case SPST_ERR_NONFINITE: return "non-finite value";
    case SPST_ERR_CUDA: return "CUDA error";
    case SPST_ERR_OOM: return "out of device memory";
    case SPST_ERR_UNSUPPORTED: return "unsupported on the device path";
    case SPST_ERR_EMPTY: return "empty statistics";
    default: return "unknown status";
  }
}

int spst_create(int device, int n_layers, const int* kinds, const int* cin, const int* cout,
                const double* const* weights, const double* const* biases, int n_style, const int* style_layers,
                int content_layer, int bgr, const double* mean3, const double* scale3, spst_ctx** out) {
  *out = nullptr;
  spst_ctx* ctx = new spst_ctx();
  *out = ctx;
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return ctx->fail(SPST_ERR_CUDA, "cudaSetDevice failed (no CUDA device?)");
  }
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return ctx->fail(SPST_ERR_CUDA, "libspst is built for sm_100a (B200); device is sm_" +
                                                            std::to_string(prop.major) + std::to_string(prop.minor));
  if (!get_encoder()) return ctx->fail(SPST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (bgr) {
    ctx->perm[0] = 2;
    ctx->perm[2] = 0;
  }
  for (int c = 0; c < 3; ++c) {
    ctx->mean[c] = (float)mean3[c];
    ctx->scale[c] = (float)scale3[c];
  }
  TRY(parse_net(ctx, n_layers, kinds, cin, cout, weights, biases, n_style, style_layers, content_layer));
  TRY(upload_weights(ctx));
  CK(cudaMallocHost(&ctx->amax_pin, (4 * ctx->stages.size() + 4) * sizeof(unsigned int)));
  return SPST_OK;
}

void spst_destroy(spst_ctx* ctx) {
  if (!ctx) return;
  for (auto& t : ctx->tpool) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  if (ctx->bound) settle(ctx);
  ctx->release_bound();
  if (ctx->amax_pin) cudaFreeHost(ctx->amax_pin);
  if (ctx->fin_pin) cudaFreeHost(ctx->fin_pin);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  for (void* p : ctx->persistent) cudaFree(p);
  delete ctx;
}

const char* spst_last_error(const spst_ctx* ctx) { return ctx ? ctx->msg.c_str() : "null context"; }

long long spst_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int spst_timing_enable(spst_ctx* ctx, int on) {
  if (!ctx) return SPST_ERR_CONFIG;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return SPST_ERR_CUDA;
  ctx->tused = 0;
  for (int c = 0; c < kTimerClasses; ++c) ctx->t_ms[c] = ctx->t_flops[c] = 0, ctx->t_n[c] = 0;
  ctx->timing = on != 0;
  return SPST_OK;
}

int spst_timing_read(spst_ctx* ctx, double* ms, double* flops, long long* launches) {
  if (!ctx) return SPST_ERR_CONFIG;
  if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return SPST_ERR_CUDA;
  timer_collect(ctx);
  for (int c = 0; c < kTimerClasses; ++c) {
    ms[c] = ctx->t_ms[c];
    flops[c] = ctx->t_flops[c];
    launches[c] = ctx->t_n[c];
  }
  return SPST_OK;
}

int spst_set_precision(spst_ctx* ctx, int mode) {
  if (mode != 0 && mode != 1) return ctx->fail(SPST_ERR_CONFIG, "precision mode must be 0 (fp16x3) or 1 (fp16)");
  ctx->precision = mode;
  return SPST_OK;
}

int spst_set_stream(spst_ctx* ctx, void* stream) {
  ctx->stream = reinterpret_cast<cudaStream_t>(stream);
  return SPST_OK;
}

int spst_bind_window(spst_ctx* ctx, int h, int w, int grid_r0, int grid_r1, int grid_c0, int grid_c1, int own_r0,
                     int own_r1, int own_c0, int own_c1) {
  const int ds = ctx->deepest_stride;
  if (h < 1 || w < 1) return ctx->fail(SPST_ERR_SHAPE, "image dims must be >= 1");
  const int Hp = round_up(h, ds), Wp = round_up(w, ds);
  if (grid_r0 % ds || grid_r1 % ds || own_r0 % ds || (own_r1 % ds && own_r1 != Hp) || grid_c0 % ds ||
      grid_c1 % ds || own_c0 % ds || (own_c1 % ds && own_c1 != Wp))
    return ctx->fail(SPST_ERR_GEOMETRY, "window bounds must be multiples of the deepest stride");
  if (!(0 <= grid_r0 && grid_r0 <= own_r0 && own_r0 < own_r1 && own_r1 <= grid_r1 && grid_r1 <= Hp))
    return ctx->fail(SPST_ERR_GEOMETRY, "row ranges must nest: 0 <= grid_r0 <= own_r0 < own_r1 <= grid_r1 <= Hp");
  if (!(0 <= grid_c0 && grid_c0 <= own_c0 && own_c0 < own_c1 && own_c1 <= grid_c1 && grid_c1 <= Wp))
    return ctx->fail(SPST_ERR_GEOMETRY,
                     "column ranges must nest: 0 <= grid_c0 <= own_c0 < own_c1 <= grid_c1 <= Wp");
  if (ctx->bound && ctx->h == h && ctx->w == w && ctx->grid_r0 == grid_r0 && ctx->grid_r1 == grid_r1 &&
      ctx->own_r0 == own_r0 && ctx->own_r1 == own_r1 && ctx->grid_c0 == grid_c0 && ctx->grid_c1 == grid_c1 &&
      ctx->own_c0 == own_c0 && ctx->own_c1 == own_c1)
    return SPST_OK;
  if (ctx->bound) TRY(settle(ctx));
  ctx->release_bound();
  ctx->h = h;
  ctx->w = w;
  ctx->Hp = Hp;
  ctx->Wp = Wp;
  ctx->grid_r0 = grid_r0;
  ctx->grid_r1 = grid_r1;
  ctx->own_r0 = own_r0;
  ctx->own_r1 = own_r1;
  ctx->grid_c0 = grid_c0;
  ctx->grid_c1 = grid_c1;
  ctx->own_c0 = own_c0;
  ctx->own_c1 = own_c1;
  int r = bind_alloc(ctx);
  if (r) {
    ctx->release_bound();
    return r;
  }
  ctx->bound = true;
  return SPST_OK;
}

int spst_bind(spst_ctx* ctx, int h, int w, int grid_r0, int grid_r1, int own_r0, int own_r1) {
  const int Wp = round_up(w, ctx->deepest_stride);
  return spst_bind_window(ctx, h, w, grid_r0, grid_r1, 0, Wp, own_r0, own_r1, 0, Wp);
}

int spst_window_dims(const spst_ctx* ctx, int* rows, int* cols) {
  *rows = ctx->grid_r1 - ctx->grid_r0;
  *cols = ctx->grid_c1 - ctx->grid_c0;
  return SPST_OK;
}

int spst_unbind(spst_ctx* ctx) {
  ctx->release_bound();
  return SPST_OK;
}

int spst_padded_dims(const spst_ctx* ctx, int* Hp, int* Wp) {
  *Hp = ctx->Hp;
  *Wp = ctx->Wp;
  return SPST_OK;
}

int spst_tap_info(const spst_ctx* ctx, int tap, int* channels, int* stride, long long* owned_pixels) {
  if (tap < 0 || tap >= (int)ctx->taps.size()) return SPST_ERR_CONFIG;
  const Stage& s = ctx->stages[ctx->taps[tap].stage];
  *channels = s.cout;
  *stride = s.stride;
  *owned_pixels =
      ctx->bound ? (long long)((ctx->own_r1 - ctx->own_r0) / s.stride) * ((ctx->own_c1 - ctx->own_c0) / s.stride) : 0;
  return SPST_OK;
}

long long spst_workspace_bytes(const spst_ctx* ctx) { return ctx->alloc_bytes; }

int spst_forward_pitched(spst_ctx* ctx, const float* x, long long pitch, int flags) {
  (void)flags;
  if (!ctx->bound) return ctx->fail(SPST_ERR_CONFIG, "spst_bind must precede spst_forward");
  static const bool dbg_us = env_int("SPST_DEBUG_HOST_US", 0) != 0;
  const double t0 = dbg_us ? host_us() : 0.0;
  TRY(settle(ctx));
  if (dbg_us) fprintf(stderr, "[spst] forward host us: settle %.1f\n", host_us() - t0);
  ctx->fwd_x = x;
  if (pitch < std::min(ctx->grid_c1, ctx->w) - ctx->grid_c0)
    return ctx->fail(SPST_ERR_SHAPE, "image pitch below the window's image columns");
  ctx->x_pitch = pitch;
  int r = do_forward(ctx, x, false);
  if (r == 1) r = do_forward(ctx, x, true);
  if (r == 1) return ctx->fail(SPST_ERR_NONFINITE, "activation range could not be represented (non-finite?)");
  if (r) return r;
  ctx->fwd_done = true;
  ctx->finalized = false;
  return SPST_OK;
}

int spst_forward(spst_ctx* ctx, const float* x, int flags) {
  if (!ctx->bound) return ctx->fail(SPST_ERR_CONFIG, "spst_bind must precede spst_forward");
  return spst_forward_pitched(ctx, x, ctx->w, flags);
}

int spst_stats_ptrs(spst_ctx* ctx, int tap, double** S, double** s) {
  if (tap < 0 || tap >= (int)ctx->taps.size() || !ctx->bound) return ctx->fail(SPST_ERR_CONFIG, "bad tap / unbound");
  TRY(resolve_forward(ctx));
  *S = ctx->taps[tap].S;
  *s = ctx->taps[tap].s;
  return SPST_OK;
}

int spst_capture_content(spst_ctx* ctx) {
  if (ctx->content_stage < 0) return ctx->fail(SPST_ERR_CONFIG, "network has no content tap");
  if (!ctx->fwd_done) return ctx->fail(SPST_ERR_CONFIG, "no forward to capture");
  TRY(resolve_forward(ctx));
  const Stage& s = ctx->stages[ctx->content_stage];
  CK(cudaMemcpyAsync(ctx->content_u.hi, s.out.hi, s.out.bytes(), cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->content_u.scale = s.out.scale;
  ctx->content_captured = true;
  return SPST_OK;
}

int spst_content_target(spst_ctx* ctx, void** buf, long long* bytes, float* scale) {
  if (ctx->content_stage < 0 || !ctx->bound) return ctx->fail(SPST_ERR_CONFIG, "no content tap / unbound");
  TRY(settle(ctx));
  *buf = ctx->content_u.hi;
  *bytes = (long long)ctx->content_u.bytes();
  *scale = ctx->content_u.scale;
  return SPST_OK;
}

int spst_set_content_target(spst_ctx* ctx, const void* buf, float scale) {
  if (ctx->content_stage < 0 || !ctx->bound) return ctx->fail(SPST_ERR_CONFIG, "no content tap / unbound");
  if (buf != ctx->content_u.hi)
    CK(cudaMemcpyAsync(ctx->content_u.hi, buf, ctx->content_u.bytes(), cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->content_u.scale = scale;
  ctx->content_captured = true;
  return SPST_OK;
}

int spst_content_sqdiff(spst_ctx* ctx, double* out) {
  if (!ctx->content_captured) return ctx->fail(SPST_ERR_CONFIG, "content target not captured");
  const Stage& s = ctx->stages[ctx->content_stage];
  const int r0 = (ctx->own_r0 - ctx->grid_r0) / s.stride, r1 = (ctx->own_r1 - ctx->grid_r0) / s.stride;
  const int c0 = (ctx->own_c0 - ctx->grid_c0) / s.stride, c1 = (ctx->own_c1 - ctx->grid_c0) / s.stride;
  CK(launch_content_sqdiff(s.out, ctx->content_u, s.cout, r0, r1, c0, c1, ctx->content_partial, out, ctx->stream));
  return SPST_OK;
}

int spst_set_style_ref(spst_ctx* ctx, int tap, const double* gram, const double* mean, const double* std_,
                       double wg, double wm, double ws) {
  if (tap < 0 || tap >= (int)ctx->taps.size()) return ctx->fail(SPST_ERR_CONFIG, "bad tap index");
  TapState& t = ctx->taps[tap];
  const int C = ctx->stages[t.stage].cout;
  if (!t.Gr) {
    t.Gr = ctx->dalloc<double>((size_t)C * C, true);
    t.mur = ctx->dalloc<double>(C, true);
    t.sdr = ctx->dalloc<double>(C, true);
    if (!t.Gr || !t.mur || !t.sdr) return ctx->fail(SPST_ERR_OOM, "reference statistics");
  }
  CK(cudaMemcpy(t.Gr, gram, (size_t)C * C * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t.mur, mean, (size_t)C * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t.sdr, std_, (size_t)C * 8, cudaMemcpyHostToDevice));
  t.wg = wg;
  t.wm = wm;
  t.ws = ws;
  t.has_ref = true;
  return SPST_OK;
}

int spst_finalize(spst_ctx* ctx, const long long* n, double* terms, int* degenerate) {
  if (!ctx->fwd_done) return ctx->fail(SPST_ERR_CONFIG, "spst_forward must precede spst_finalize");
  TRY(resolve_backward(ctx, nullptr));
  size_t total = 0;
  for (auto& t : ctx->taps) total += 2 * (size_t)ctx->stages[t.stage].cout + 3;
  // the style coefficients and loss terms are launched behind the forward; ONE read-back
  // settles both the forward's deferred range check and the terms
  bool redone = false;
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t i = 0; i < ctx->taps.size(); ++i) {
      TapState& t = ctx->taps[i];
      if (n[i] <= 0) return ctx->fail(SPST_ERR_EMPTY, "no feature pixels accumulated");
      t.n = (double)n[i];
      StyleCoefArgs a = coef_args(ctx, t);
      CK(cudaMemsetAsync(t.degenerate, 0, 4, ctx->stream));
      CK(launch_style_vec(a, ctx->stream));
      CK(launch_style_mat(a, ctx->stream));
    }
    if (total) CK(cudaMemcpyAsync(ctx->fin_pin, ctx->fin_d, total * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    const bool pending = ctx->fwd_pending;
    TRY(resolve_forward(ctx));  // synchronises the stream when a check was pending
    if (!pending) CK(cudaStreamSynchronize(ctx->stream));
    if (!ctx->fwd_redone) break;  // (a redone forward changed the statistics: recompute)
    redone = true;
  }
  ctx->fwd_redone = redone;  // tells the caller to recompute what it launched behind the forward
  for (size_t i = 0; i < ctx->taps.size(); ++i) {
    TapState& t = ctx->taps[i];
    const int C = ctx->stages[t.stage].cout;
    const double* buf = ctx->fin_pin + (t.row_loss - ctx->fin_d);
    int deg = 0;
    std::memcpy(&deg, buf + 2 * C + 2, sizeof(int));
    double g = 0, mm = 0;
    for (int c = 0; c < C; ++c) {
      g += buf[c];
      mm = std::max(mm, buf[C + c]);
    }
    t.mmax = mm;
    terms[3 * i + 0] = t.wg * g;
    terms[3 * i + 1] = t.wm * buf[2 * C];
    terms[3 * i + 2] = t.ws * buf[2 * C + 1];
    if (degenerate) degenerate[i] = deg;
  }
  ctx->finalized = true;
  return SPST_OK;
}

int spst_forward_redone(spst_ctx* ctx) { return ctx->fwd_redone ? 1 : 0; }

int spst_backward(spst_ctx* ctx, double two_lambda, float* grad) {
  return spst_backward_pitched(ctx, two_lambda, grad, ctx->w);
}

int spst_backward_async(spst_ctx* ctx, double two_lambda, float* grad, long long pitch) {
  if (!ctx->finalized) return ctx->fail(SPST_ERR_CONFIG, "spst_finalize must precede spst_backward");
  if (pitch < std::min(ctx->own_c1, ctx->w) - ctx->own_c0)
    return ctx->fail(SPST_ERR_SHAPE, "gradient pitch below the owned image columns");
  TRY(resolve_backward(ctx, nullptr));
  ctx->g_pitch = pitch;
  if (two_lambda != 0.0 && ctx->content_stage >= 0 && !ctx->content_captured)
    return ctx->fail(SPST_ERR_CONFIG, "content weight is nonzero but no content target was captured");
  ctx->bwd_lambda = two_lambda;
  ctx->bwd_grad = grad;
  int r = do_backward(ctx, two_lambda, grad, false);
  if (r == 1) r = do_backward(ctx, two_lambda, grad, true);
  if (r == 1) return ctx->fail(SPST_ERR_NONFINITE, "gradient range could not be represented (non-finite?)");
  return r;
}

int spst_backward_resolve(spst_ctx* ctx, int* redone) { return resolve_backward(ctx, redone); }

int spst_backward_pitched(spst_ctx* ctx, double two_lambda, float* grad, long long pitch) {
  TRY(spst_backward_async(ctx, two_lambda, grad, pitch));
  return resolve_backward(ctx, nullptr);
}

// ------------------------------------------------------------------------------------ vectors
int spst_vec_partials(void) { return red_blocks(); }

int spst_vec_dots(int f64, const void* a0, const void* b0, const void* a1, const void* b1, const void* a2,
                  const void* b2, long long n, double* partial, double* out, void* stream) {
  return launch_dots(f64, a0, b0, a1, b1, a2, b2, n, partial, out, (cudaStream_t)stream) == cudaSuccess
             ? SPST_OK
             : SPST_ERR_CUDA;
}

int spst_vec_absmax(int f64, const void* a, long long n, double* partial, double* out, void* stream) {
  return launch_absmax(f64, a, n, partial, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK : SPST_ERR_CUDA;
}

int spst_vec_axpy_dot(int f64, const void* q_in, void* q_out, const void* v, const double* coef, double cscale,
                      const void* w, long long n, double* partial, void* stream) {
  AxpyDotArgs a{q_in, q_out, v, coef, cscale, w, n, partial};
  return launch_axpy_dot(f64, a, (cudaStream_t)stream) == cudaSuccess ? SPST_OK : SPST_ERR_CUDA;
}

int spst_vec_twoloop_scalar(const double* dot, double rho, int mode, double* alpha, double* coef, void* stream) {
  return launch_twoloop_scalar(dot, rho, mode, alpha, coef, (cudaStream_t)stream) == cudaSuccess ? SPST_OK
                                                                                                : SPST_ERR_CUDA;
}

int spst_vec_two_loop(int f64, const void* g, void* out, const void* const* s_vecs, const void* const* y_vecs,
                      const double* rho, double gamma, int m, long long n, double* partial, double* alpha,
                      unsigned int* ticket, double* coef, void* stream) {
  // the sequence of lbfgs.py _two_loop issued from C as 2m+1 fused kernels: each axpy+dot step
  // also finishes its dot (fixed block order) and applies the scalar update in its last block,
  // so the results equal the 3-kernel-per-step form bit for bit.  Pairs oldest first.
  if (m < 1 || n < 0 || !g || !out || !ticket) return SPST_ERR_SHAPE;
  cudaStream_t st = (cudaStream_t)stream;
  static const bool per_step = [] {
    const char* e = getenv("SPST_TWOLOOP_STEPS");
    return e && atoi(e) != 0;
  }();
  if (!per_step && m <= kTwoLoopMaxHist) {  // one cooperative launch (same bits as the steps below)
    TwoLoopArgs ta{};
    ta.g = g;
    ta.out = out;
    for (int i = 0; i < m; ++i) {
      ta.s[i] = s_vecs[i];
      ta.y[i] = y_vecs[i];
      ta.rho[i] = rho[i];
    }
    ta.gamma = gamma;
    ta.m = m;
    ta.n = n;
    ta.partial = partial;
    const cudaError_t e = launch_two_loop_coop(f64, ta, st);
    if (e == cudaSuccess) return SPST_OK;
    if (e != cudaErrorNotSupported) return SPST_ERR_CUDA;
  }
  auto step = [&](const void* qi, const void* v, double cscale, const void* w, int i, int mode) -> bool {
    AxpyDotArgs a{qi, out, v, coef, cscale, w, n, partial};
    if (w) {
      a.alpha_i = alpha + i;
      a.ticket = ticket;
      a.rho = rho[i];
      a.mode = mode;
    }
    return launch_axpy_dot(f64, a, st) == cudaSuccess;
  };
  // loop 1, newest -> oldest: alpha_i = rho_i <s_i, q>; q -= alpha_i y_i
  if (!step(g, nullptr, 1.0, s_vecs[m - 1], m - 1, 0)) return SPST_ERR_CUDA;
  for (int i = m - 1; i > 0; --i)
    if (!step(out, y_vecs[i], 1.0, s_vecs[i - 1], i - 1, 0)) return SPST_ERR_CUDA;
  // q = gamma (q - alpha_0 y_0); beta_0 = rho_0 <y_0, q>
  if (!step(out, y_vecs[0], gamma, y_vecs[0], 0, 1)) return SPST_ERR_CUDA;
  // loop 2, oldest -> newest: q += (alpha_i - beta_i) s_i
  for (int i = 0; i < m - 1; ++i)
    if (!step(out, s_vecs[i], 1.0, y_vecs[i + 1], i + 1, 1)) return SPST_ERR_CUDA;
  if (!step(out, s_vecs[m - 1], -1.0, nullptr, 0, 0)) return SPST_ERR_CUDA;
  return SPST_OK;
}

int spst_vec_sum_partials(const double* partial, int nk, double* out, void* stream) {
  return launch_sum_partials(partial, nk, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK : SPST_ERR_CUDA;
}

int spst_metric_sqdiff(int f64, const void* a, const void* b, long long n, double* partial, double* out,
                       void* stream) {
  if (n < 0 || !a || !b || !partial || !out) return SPST_ERR_SHAPE;
  return launch_metric_sqdiff(f64 != 0, a, b, n, partial, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK
                                                                                                  : SPST_ERR_CUDA;
}

int spst_metric_ssim(int f64, const void* a, const void* b, int h, int w, int c, double* partial, double* out,
                     void* stream) {
  if (h < 11 || w < 11 || (c != 1 && c != 3) || !a || !b || !partial || !out) return SPST_ERR_SHAPE;
  return launch_metric_ssim(f64, a, b, h, w, c, partial, out, (cudaStream_t)stream) == cudaSuccess
             ? SPST_OK
             : SPST_ERR_CUDA;
}

int spst_vec_axpy(int f64, const void* x, const void* d, double t, long long n, void* out, void* stream) {
  return launch_axpy(f64, x, d, t, n, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK : SPST_ERR_CUDA;
}

int spst_vec_sy(int f64, const void* xt, const void* x, const void* gt, const void* g, long long n, void* s, void* y,
                double* partial, double* out, void* stream) {
  return launch_sy(f64, xt, x, gt, g, n, s, y, partial, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK
                                                                                                : SPST_ERR_CUDA;
}

int spst_resize_down(const float* in, int h, int w, int c, int f, float* out, void* stream) {
  return spst_resize_down_typed(0, in, h, w, c, f, out, stream);
}

int spst_resize_bilinear(const float* in, int h, int w, int c, int oh, int ow, float* out, void* stream) {
  return spst_resize_bilinear_typed(0, in, h, w, c, oh, ow, out, stream);
}

int spst_resize_down_typed(int f64, const void* in, int h, int w, int c, int f, void* out, void* stream) {
  if (f < 1) return SPST_ERR_SHAPE;
  return launch_resize_down(f64, in, h, w, c, f, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK : SPST_ERR_CUDA;
}

int spst_resize_bilinear_typed(int f64, const void* in, int h, int w, int c, int oh, int ow, void* out,
                               void* stream) {
  if (oh < 1 || ow < 1) return SPST_ERR_SHAPE;
  return launch_resize_bilinear(f64, in, h, w, c, oh, ow, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK
                                                                                                   : SPST_ERR_CUDA;
}

// ------------------------------------------------------------------------------------ debug
int spst_debug_mask(spst_ctx* ctx, int stage, unsigned char* out_host) {
  if (!ctx->fwd_done || stage < 0 || stage >= (int)ctx->stages.size())
    return ctx->fail(SPST_ERR_CONFIG, "no forward / bad stage");
  TRY(settle(ctx));
  const Stage& s = ctx->stages[stage];
  const size_t n = (size_t)(s.cout_p / 32) * s.H * s.W;
  std::vector<uint32_t> bits(n);
  CK(cudaMemcpyAsync(bits.data(), s.mask, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const size_t plane = (size_t)s.H * s.W;
  for (int c = 0; c < s.cout; ++c)
    for (size_t p = 0; p < plane; ++p) out_host[c * plane + p] = (bits[(c >> 5) * plane + p] >> (c & 31)) & 1u;
  return SPST_OK;
}

int spst_stage_features(spst_ctx* ctx, int stage, float* out_dev) {
  if (!ctx->fwd_done || stage < 0 || stage >= (int)ctx->stages.size())
    return ctx->fail(SPST_ERR_CONFIG, "no forward / bad stage");
  TRY(resolve_forward(ctx));
  const Stage& s = ctx->stages[stage];
  if (!s.has_out) return ctx->fail(SPST_ERR_CONFIG, "stage output is not a stored tap");
  note_launch(), unpack_hl_kernel<<<512, 256, 0, ctx->stream>>>(s.out, s.cout, out_dev);
  CK(cudaGetLastError());
  return SPST_OK;
}

int spst_feature_affine(int f64, const void* A, const void* r, const void* b, int C, long long P, const void* V,
                        void* out, void* stream) {
  if (C < 1 || P < 0 || !A || !r || !b || !V || !out) return SPST_ERR_SHAPE;
  return launch_feature_affine(f64, A, r, b, C, P, V, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK
                                                                                              : SPST_ERR_CUDA;
}

int spst_vec_scaled_diff(int f64, const void* a, const void* b, double c, long long n, void* out, void* stream) {
  if (n < 0 || !a || !b || !out) return SPST_ERR_SHAPE;
  return launch_scaled_diff(f64, a, b, c, n, out, (cudaStream_t)stream) == cudaSuccess ? SPST_OK : SPST_ERR_CUDA;
}

int spst_debug_stage_out(spst_ctx* ctx, int stage, float* out_host) {
  if (!ctx->fwd_done || stage < 0 || stage >= (int)ctx->stages.size())
    return ctx->fail(SPST_ERR_CONFIG, "no forward / bad stage");
  TRY(settle(ctx));
  const Stage& s = ctx->stages[stage];
  if (!s.has_out) return ctx->fail(SPST_ERR_CONFIG, "stage output not stored (set SPST_DEBUG_STORE_ALL=1)");
  const size_t n = (size_t)s.cout * s.H * s.W;
  float* d = ctx->dalloc<float>(n);
  if (!d) return ctx->fail(SPST_ERR_OOM, "debug buffer");
  note_launch(), unpack_hl_kernel<<<512, 256, 0, ctx->stream>>>(s.out, s.cout, d);
  CK(cudaMemcpyAsync(out_host, d, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return SPST_OK;
}

int spst_debug_conv(int device, int mode, int cin, int cout, int H, int W, const float* x_host,
                    const double* weight, const double* bias, float* y_host) {
  if (cudaSetDevice(device) != cudaSuccess || !get_encoder()) return SPST_ERR_CUDA;
  spst_ctx holder;
  spst_ctx* ctx = &holder;
  Stage s;
  s.cin = cin;
  s.cout = cout;
  s.cin_p = round_up(cin, 64);
  s.cout_p = round_up(cout, 64);
  s.w.assign(weight, weight + (size_t)cout * cin * 9);
  s.b.assign(bias, bias + cout);
  double mx = 0;
  for (double v : s.w) mx = std::max(mx, std::fabs(v));
  s.wexp = mx > 0 ? (int)std::floor(std::log2(16384.0 / mx)) : 0;
  const bool bwd = mode == 2;
  const int Kc = bwd ? cout : cin, Kp = bwd ? s.cout_p : s.cin_p, Np = bwd ? s.cin_p : s.cout_p;
  const int Nc = bwd ? cin : cout;
  auto slab = stage_slabs(s, bwd, ntile_for(Np));
  uint8_t* slab_d = ctx->dalloc<uint8_t>(slab.size() * 2);
  float* xd = ctx->dalloc<float>((size_t)Kc * H * W);
  HL16 in = hl_shape(Kp, H, W);
  in.hi = ctx->dalloc<__half>((size_t)Kp * H * W * 2);
  HL16 out = hl_shape(Np, H, W);
  out.hi = ctx->dalloc<__half>((size_t)Np * H * W * 2);
  out.scale = 1.f;
  HL16 pooled = hl_shape(Np, H / 2, W / 2);
  pooled.hi = ctx->dalloc<__half>((size_t)Np * std::max(1, H / 2) * std::max(1, W / 2) * 2);
  float* bd = ctx->dalloc<float>(Np);
  uint32_t* mask = ctx->dalloc<uint32_t>((size_t)(Np / 32) * H * W);
  float* yd = ctx->dalloc<float>((size_t)Nc * H * W);
  uint32_t* parg = ctx->dalloc<uint32_t>((size_t)(Np / 16) * std::max(1, H / 2) * std::max(1, W / 2));
  if (!slab_d || !xd || !in.hi || !out.hi || !pooled.hi || !bd || !mask || !yd || !parg) return SPST_ERR_OOM;
  std::vector<float> b32(Np, 0.f);
  if (!bwd)
    for (int c = 0; c < cout; ++c) b32[c] = (float)bias[c];
  CK(cudaMemcpy(bd, b32.data(), Np * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(slab_d, slab.data(), slab.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(xd, x_host, (size_t)Kc * H * W * 4, cudaMemcpyHostToDevice));
  note_launch(), pack_hl_kernel<<<512, 256>>>(xd, Kc, in);
  ConvLaunch L;
  L.in = &in;
  L.wslab = slab_d;
  L.H = H;
  L.W = W;
  L.acc_scale = 1.f / (in.scale * pow2f(s.wexp));
  L.a.out = out;
  L.a.out_pool = pooled;
  L.a.bias = bwd ? nullptr : bd;
  L.a.mask_out = mask;
  L.a.epi = bwd ? EPI_BWD : ((mode == 1 || mode == 4 || mode == 5) ? EPI_FWD_POOL : EPI_FWD);
  L.a.pool_max = (mode == 4 || mode == 5) ? 1 : 0;
  L.a.pool_arg = parg;
  L.a.store_full = 0;
  L.drain = bwd ? bwd_drain() : fwd_drain();
  TRY(run_conv(ctx, L));
  CK(cudaDeviceSynchronize());
  if (mode == 1 || mode == 4) {
    note_launch(), unpack_hl_kernel<<<512, 256>>>(pooled, Nc, yd);
    CK(cudaMemcpy(y_host, yd, (size_t)Nc * (H / 2) * (W / 2) * 4, cudaMemcpyDeviceToHost));
  } else if (mode == 5) {  // first-argmax index (0-3) of every pooled element, as floats
    const size_t plane = (size_t)(H / 2) * (W / 2);
    std::vector<uint32_t> bits((size_t)(Np / 16) * plane);
    CK(cudaMemcpy(bits.data(), parg, bits.size() * 4, cudaMemcpyDeviceToHost));
    for (int c = 0; c < Nc; ++c)
      for (size_t q = 0; q < plane; ++q) y_host[c * plane + q] = (float)((bits[(c >> 4) * plane + q] >> (2 * (c & 15))) & 3u);
  } else if (mode == 3) {
    note_launch(), unpack_mask_kernel<<<512, 256>>>(mask, Nc, H, W, yd);
    CK(cudaMemcpy(y_host, yd, (size_t)Nc * H * W * 4, cudaMemcpyDeviceToHost));
  } else {
    note_launch(), unpack_hl_kernel<<<512, 256>>>(out, Nc, yd);
    CK(cudaMemcpy(y_host, yd, (size_t)Nc * H * W * 4, cudaMemcpyDeviceToHost));
  }
  CK(cudaDeviceSynchronize());
  ctx->release_bound();
  return SPST_OK;
}

int spst_debug_gram(int device, int C, long long P, const float* f_host, double* S_host) {
  if (cudaSetDevice(device) != cudaSuccess || !get_encoder()) return SPST_ERR_CUDA;
  spst_ctx holder;
  spst_ctx* ctx = &holder;
  const int Cp = round_up(C, 64);
  HL16 t = hl_shape(Cp, 1, (int)P);
  t.hi = ctx->dalloc<__half>((size_t)Cp * P * 2);
  float* fd = ctx->dalloc<float>((size_t)C * P);
  const int nct = (Cp + 127) / 128;
  const int per = gram_px_per_split(P, nct * (nct + 1) / 2);
  const int splits = (int)std::max<long long>(1, (P + per - 1) / per);
  float* part = ctx->dalloc<float>((size_t)splits * (nct * (nct + 1) / 2) * 128 * 128);
  double* Sd = ctx->dalloc<double>((size_t)C * C);
  if (!t.hi || !fd || !part || !Sd) return SPST_ERR_OOM;
  CK(cudaMemcpy(fd, f_host, (size_t)C * P * 4, cudaMemcpyHostToDevice));
  note_launch(), pack_hl_kernel<<<512, 256>>>(fd, C, t);
  GramArgs g{};
  if (!map_gram(&g.tm_hi, t.hi, (int)P, 1, (int)P, 1, Cp / 8) || !map_gram(&g.tm_lo, t.lo(), (int)P, 1, (int)P, 1, Cp / 8))
    return SPST_ERR_CUDA;
  g.C_p = Cp;
  g.rows = 1;
  g.w_own = (int)P;
  g.px_per_split = per;
  g.n_ctile = nct;
  g.partial = part;
  bool nonneg = true;  // ReLU-like operands get the same-sign compensation of real taps
  for (long long i = 0; i < (long long)C * P && nonneg; ++i) nonneg = f_host[i] >= 0.f;
  set_gram_comp(g, Cp, nonneg);
  if (Cp == 64) {
    CK(launch_gram64_tc(g, splits, C, 1.0, Sd, nullptr));
  } else {
    CK(launch_gram_tc(g, splits, nullptr));
    CK(launch_gram_reduce(part, splits, nct, C, 1.0, Sd, nullptr));
  }
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(S_host, Sd, (size_t)C * C * 8, cudaMemcpyDeviceToHost));
  ctx->release_bound();
  return SPST_OK;
}

}  // extern "C"
