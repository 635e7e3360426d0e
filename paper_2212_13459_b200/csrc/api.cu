// api.cu — device kernels behind the reference's per-tap public helpers that are not on the
// fused hot path (reference stats.py:127-174 style_layer_loss_grad / content_loss_grad when
// called directly on a feature slab).  Inside loss_grad the same math is fused into the
// backward conv (conv_tc.cu); these serve the drop-in API on arbitrary (C, h, w) slabs.
#include <algorithm>

#include "common.cuh"

namespace spst {

// out[c, p] = sum_d A[c, d] V[d, p] + r[c] V[c, p] + b[c] over a (C, P) slab.  A block owns
// 8 channels x 128 pixels; the 8 rows of A stream through shared memory in 64-column chunks
// and each V element read serves the block's 8 output channels.  f64 accumulation.
template <typename T>
__global__ void __launch_bounds__(128) feature_affine_kernel(const T* A, const T* r, const T* b, int C, long long P,
                                                             const T* V, T* out) {
  __shared__ double sA[8][64];
  const int c0 = blockIdx.y * 8;
  const long long p = (long long)blockIdx.x * 128 + threadIdx.x;
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  for (int d0 = 0; d0 < C; d0 += 64) {
    __syncthreads();
    for (int e = threadIdx.x; e < 8 * 64; e += 128) {
      const int i = e / 64, d = d0 + e % 64;
      sA[i][e % 64] = (c0 + i < C && d < C) ? (double)A[(size_t)(c0 + i) * C + d] : 0.0;
    }
    __syncthreads();
    if (p < P) {
      const int dn = min(64, C - d0);
      for (int dd = 0; dd < dn; ++dd) {
        const double v = (double)V[(size_t)(d0 + dd) * P + p];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(sA[i][dd], v, acc[i]);
      }
    }
  }
  if (p >= P) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = c0 + i;
    if (c >= C) break;
    const double v = (double)V[(size_t)c * P + p];
    out[(size_t)c * P + p] = (T)(acc[i] + (double)r[c] * v + (double)b[c]);
  }
}

template <typename T>
__global__ void scaled_diff_kernel(const T* a, const T* b, double c, long long n, T* out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = (T)c * (a[i] - b[i]);
}

cudaError_t launch_feature_affine(int f64, const void* A, const void* r, const void* b, int C, long long P,
                                  const void* V, void* out, cudaStream_t st) {
  if (C <= 0 || P < 0) return cudaErrorInvalidValue;
  if (P == 0) return cudaSuccess;
  dim3 grid((unsigned)((P + 127) / 128), (unsigned)((C + 7) / 8));
  if (f64)
    note_launch(), feature_affine_kernel<double><<<grid, 128, 0, st>>>(
        (const double*)A, (const double*)r, (const double*)b, C, P, (const double*)V, (double*)out);
  else
    note_launch(), feature_affine_kernel<float><<<grid, 128, 0, st>>>(
        (const float*)A, (const float*)r, (const float*)b, C, P, (const float*)V, (float*)out);
  return cudaGetLastError();
}

cudaError_t launch_scaled_diff(int f64, const void* a, const void* b, double c, long long n, void* out,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 4LL * kSMs * 8);
  if (f64)
    note_launch(), scaled_diff_kernel<double><<<blocks, 256, 0, st>>>((const double*)a, (const double*)b, c, n,
                                                                       (double*)out);
  else
    note_launch(), scaled_diff_kernel<float><<<blocks, 256, 0, st>>>((const float*)a, (const float*)b, c, n,
                                                                      (float*)out);
  return cudaGetLastError();
}

}  // namespace spst
