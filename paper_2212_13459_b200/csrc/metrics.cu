// metrics.cu — evaluation metrics on device (reference metrics.py).
//
//   psnr  (metrics.py:24-31): 10 log10(1 / mean((a-b)^2)) in f64  -> spst_metric_sqdiff
//   ssim  (metrics.py:55-73): mean local SSIM of the Rec.601 luma, 11x11 Gaussian window
//                             (sigma 1.5), valid mode, K1/K2 = 0.01/0.03 -> spst_metric_ssim
//
// Both are HBM-bound stencils/reductions.  They compute in f64 like the reference (SSIM's
// E[x^2] - mu^2 cancels badly in fp32) and reduce with a fixed block->partial assignment and a
// fixed-order final sum (finish_sums_kernel), so results are deterministic.  The luma follows
// the reference's dtype rule: NumPy multiplies an f32 image by Python-float weights in f32
// (weak scalars), so f32 inputs get f32 luma (separately rounded multiply and adds), f64
// inputs f64 luma; both are then widened to f64.
#include <cuda_runtime.h>

#include <cmath>

#include "common.cuh"

namespace spst {

constexpr int kSsimWin = 11;
constexpr int kSsimTW = 32, kSsimTH = 16;  // output tile
constexpr int kSsimIW = kSsimTW + kSsimWin - 1, kSsimIH = kSsimTH + kSsimWin - 1;

__constant__ double c_gauss[kSsimWin];

template <typename T>
__global__ void __launch_bounds__(256) sqdiff_partial_kernel(const T* a, const T* b, long long n,
                                                             double* partial) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    s = fma(d, d, s);
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

template <typename T>
__device__ __forceinline__ double luma_at(const T* img, int w, int c, int y, int x);
template <>
__device__ __forceinline__ double luma_at<float>(const float* img, int w, int c, int y, int x) {
  const float* p = img + ((size_t)y * w + x) * c;
  if (c == 1) return (double)p[0];
  const float l = __fadd_rn(__fadd_rn(__fmul_rn(0.299f, p[0]), __fmul_rn(0.587f, p[1])), __fmul_rn(0.114f, p[2]));
  return (double)l;
}
template <>
__device__ __forceinline__ double luma_at<double>(const double* img, int w, int c, int y, int x) {
  const double* p = img + ((size_t)y * w + x) * c;
  if (c == 1) return p[0];
  return __dadd_rn(__dadd_rn(__dmul_rn(0.299, p[0]), __dmul_rn(0.587, p[1])), __dmul_rn(0.114, p[2]));
}

// One block per output tile (grid-stride over tiles, fixed assignment): stage the luma window
// of both images, filter rows (5 moments), then columns, then the SSIM map; the block's sum of
// its tiles' SSIM values is partial[blockIdx.x].
template <typename TA, typename TB>
__global__ void __launch_bounds__(256) ssim_partial_kernel(const TA* a, const TB* b, int h, int w, int c,
                                                           double* partial) {
  extern __shared__ double sm[];
  double* la = sm;                          // [IH][IW]
  double* lb = la + kSsimIH * kSsimIW;      // [IH][IW]
  double* hz = lb + kSsimIH * kSsimIW;      // [5][IH][TW]
  const int oh = h - (kSsimWin - 1), ow = w - (kSsimWin - 1);
  const int tiles_x = (ow + kSsimTW - 1) / kSsimTW, tiles_y = (oh + kSsimTH - 1) / kSsimTH;
  const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
  double acc = 0.0;
  for (int t = blockIdx.x; t < tiles_x * tiles_y; t += gridDim.x) {
    const int ox = (t % tiles_x) * kSsimTW, oy = (t / tiles_x) * kSsimTH;
    __syncthreads();
    for (int i = threadIdx.x; i < kSsimIH * kSsimIW; i += blockDim.x) {
      const int yy = oy + i / kSsimIW, xx = ox + i % kSsimIW;
      const bool in = yy < h && xx < w;
      la[i] = in ? luma_at<TA>(a, w, c, yy, xx) : 0.0;  // each image's luma in its own dtype
      lb[i] = in ? luma_at<TB>(b, w, c, yy, xx) : 0.0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSsimIH * kSsimTW; i += blockDim.x) {
      const int r = i / kSsimTW, col = i % kSsimTW;
      double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
#pragma unroll
      for (int j = 0; j < kSsimWin; ++j) {
        const double x = la[r * kSsimIW + col + j], y = lb[r * kSsimIW + col + j], k = c_gauss[j];
        sx = fma(k, x, sx);
        sy = fma(k, y, sy);
        sxx = fma(k, x * x, sxx);
        syy = fma(k, y * y, syy);
        sxy = fma(k, x * y, sxy);
      }
      const int plane = kSsimIH * kSsimTW;
      hz[i] = sx;
      hz[plane + i] = sy;
      hz[2 * plane + i] = sxx;
      hz[3 * plane + i] = syy;
      hz[4 * plane + i] = sxy;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSsimTH * kSsimTW; i += blockDim.x) {
      const int r = i / kSsimTW, col = i % kSsimTW;
      if (oy + r >= oh || ox + col >= ow) continue;
      const int plane = kSsimIH * kSsimTW;
      double m[5] = {0, 0, 0, 0, 0};
#pragma unroll
      for (int j = 0; j < kSsimWin; ++j) {
        const double k = c_gauss[j];
        const int o = (r + j) * kSsimTW + col;
#pragma unroll
        for (int q = 0; q < 5; ++q) m[q] = fma(k, hz[q * plane + o], m[q]);
      }
      const double mx = m[0], my = m[1];
      const double vx = m[2] - mx * mx, vy = m[3] - my * my, cxy = m[4] - mx * my;
      const double num = (2 * mx * my + c1) * (2 * cxy + c2);
      const double den = (mx * mx + my * my + c1) * (vx + vy + c2);
      acc += num / den;
    }
  }
  __syncthreads();
  double* red = sm;  // reuse: 256 doubles
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s2 = 128; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2) red[threadIdx.x] += red[threadIdx.x + s2];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

cudaError_t launch_metric_sqdiff(bool f64, const void* a, const void* b, long long n, double* partial, double* out,
                                 cudaStream_t st) {
  if (f64)
    note_launch(), sqdiff_partial_kernel<double><<<red_blocks(), 256, 0, st>>>((const double*)a, (const double*)b, n, partial);
  else
    note_launch(), sqdiff_partial_kernel<float><<<red_blocks(), 256, 0, st>>>((const float*)a, (const float*)b, n, partial);
  return launch_sum_partials(partial, 1, out, st);
}

template <typename TA, typename TB>
static void launch_ssim_typed(const void* a, const void* b, int h, int w, int c, double* partial, size_t smem,
                              cudaStream_t st) {
  cudaFuncSetAttribute(ssim_partial_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  note_launch(), ssim_partial_kernel<TA, TB><<<red_blocks(), 256, smem, st>>>((const TA*)a, (const TB*)b, h, w, c, partial);
}

cudaError_t launch_metric_ssim(int f64_mask, const void* a, const void* b, int h, int w, int c, double* partial,
                               double* out, cudaStream_t st) {
  static bool init = false;
  if (!init) {  // Gaussian window, normalised (metrics.py:43-46)
    double k[kSsimWin], s = 0.0;
    for (int i = 0; i < kSsimWin; ++i) {
      const double t = i - (kSsimWin - 1) / 2.0;
      k[i] = std::exp(-(t * t) / (2.0 * 1.5 * 1.5));
      s += k[i];
    }
    for (int i = 0; i < kSsimWin; ++i) k[i] /= s;
    cudaError_t e = cudaMemcpyToSymbol(c_gauss, k, sizeof(k));
    if (e != cudaSuccess) return e;
    init = true;
  }
  const size_t smem = (size_t)(2 * kSsimIH * kSsimIW + 5 * kSsimIH * kSsimTW) * sizeof(double);
  switch (f64_mask & 3) {
    case 0: launch_ssim_typed<float, float>(a, b, h, w, c, partial, smem, st); break;
    case 1: launch_ssim_typed<double, float>(a, b, h, w, c, partial, smem, st); break;
    case 2: launch_ssim_typed<float, double>(a, b, h, w, c, partial, smem, st); break;
    default: launch_ssim_typed<double, double>(a, b, h, w, c, partial, smem, st); break;
  }
  return launch_sum_partials(partial, 1, out, st);
}

}  // namespace spst
