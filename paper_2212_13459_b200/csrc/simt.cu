// simt.cu — the HBM-bound and tiny kernels of the SPST path (no tensor-core work):
//   * first conv layer (3 input channels, K = 27) fused with replicate padding
//     (tensorops.py:201-209), preprocessing (extractor.py:151-155), bias, ReLU, mask bits
//     and tap channel sums; and its adjoint fused with preprocess_backward (158-164)
//   * fold of replicate-pad gradients (tensorops.py:212-229)
//   * standalone 2x2 average pool (tensorops.py:99-101) for nets whose first ReLU is pooled
//   * statistics finalisation and the closed-form style coefficients (stats.py:59-66,
//     117-165), content squared distance (localized.py:257-267)
//   * deterministic f64 reductions, L-BFGS vector passes (lbfgs.py:68-142)
//   * area downsampling and half-pixel bilinear resampling (tensorops.py:136-185)
#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "sm100.cuh"

namespace spst {
namespace cg = cooperative_groups;

// ------------------------------------------------------------------------------------------
// first conv (C_in = 3)
// ------------------------------------------------------------------------------------------

constexpr int FC_BX = 32, FC_BY = 8;

// Image -> first-conv operand (reference extractor.py preprocessing + the replicate padding of
// localized.py): v_c = (img[perm c] - mean_c) / scale_c at the clamped global pixel, split into
// fp16 hi/lo at scale out.scale.  One thread per grid pixel, 16 B hi + 16 B lo per pixel.
__global__ void __launch_bounds__(256) image_hl_kernel(const __grid_constant__ ImageHLArgs a) {
  float m = 0.f;
  // grid-stride over (rows: y, columns: x) -- no per-pixel index division
  for (int y = blockIdx.y; y < a.Hl; y += gridDim.y)
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < a.Wp; x += gridDim.x * blockDim.x) {
    const long long i = (long long)y * a.Wp + x;
    const int gy = min(y + a.row_off, a.h - 1), gx = min(x + a.col_off, a.w - 1);
    const float* px = a.img + ((long long)gy * a.pitch + gx) * 3;
    __align__(16) __half hh[8];
    __align__(16) __half ll[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float v = 0.f;
      if (c < 3) v = (px[a.perm[c]] - a.mean[c]) / a.scale[c];
      m = fmaxf(m, fabsf(v));
      HalfPair p = split_f16(v * a.out.scale);
      hh[c] = p.hi;
      ll[c] = p.lo;
    }
    reinterpret_cast<uint4*>(a.out.hi)[i] = *reinterpret_cast<uint4*>(hh);
    reinterpret_cast<uint4*>(a.out.lo())[i] = *reinterpret_cast<uint4*>(ll);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(a.amax, __float_as_uint(m));
}

__global__ void __launch_bounds__(256) first_conv_bwd_kernel(const __grid_constant__ FirstConvBwdArgs a) {
  constexpr int CH = 16;
  __shared__ float tile[CH][FC_BY + 2][FC_BX + 2];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * FC_BX, y0 = blockIdx.y * FC_BY;
  const int H = a.g.H, W = a.g.W;
  const float inv = 1.f / a.g.scale;
  float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int c0 = 0; c0 < kFirstC; c0 += CH) {
    if (c0 >= a.g.C_p) break;
    __syncthreads();
    for (int i = threadIdx.x; i < (CH / 8) * (FC_BY + 2) * (FC_BX + 2); i += blockDim.x) {
      const int kg = i / ((FC_BY + 2) * (FC_BX + 2));
      const int r = (i / (FC_BX + 2)) % (FC_BY + 2);
      const int cc = i % (FC_BX + 2);
      const int yy = y0 - 1 + r, xx = x0 - 1 + cc;
      float v8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (yy >= 0 && yy < H && xx >= 0 && xx < W) {
        const size_t off = ((size_t)((c0 >> 3) + kg) * H + yy) * W + xx;
        uint4 hv = reinterpret_cast<const uint4*>(a.g.hi)[off];
        uint4 lv = reinterpret_cast<const uint4*>(a.g.lo())[off];
        const __half* hh = reinterpret_cast<const __half*>(&hv);
        const __half* ll = reinterpret_cast<const __half*>(&lv);
#pragma unroll
        for (int e = 0; e < 8; ++e) v8[e] = (__half2float(hh[e]) + __half2float(ll[e])) * inv;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) tile[kg * 8 + e][r][cc] = v8[e];
    }
    __syncthreads();
    // g_in[y][x][ci] = sum_{co,dy,dx} g[co][y+1-dy][x+1-dx] * W[co][ci][dy][dx]
#pragma unroll
    for (int co = 0; co < CH; ++co)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
          const float gv = tile[co][ty + 2 - dy][tx + 2 - dx];
#pragma unroll
          for (int ci = 0; ci < 3; ++ci) acc[ci] = fmaf(gv, a.wgt[(c0 + co) * 27 + ci * 9 + dy * 3 + dx], acc[ci]);
        }
  }
  const int y = y0 + ty, x = x0 + tx;
  if (y < H && x < W) {
    float* o = a.gimg + ((size_t)y * W + x) * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) o[a.perm[c]] = acc[c] / a.scale[c];
  }
}

// grad over the owned rectangle from the local padded-grid gradient (FoldArgs, common.cuh).
__global__ void fold_grad_kernel(const FoldArgs a) {
  const int gx = a.c0 + blockIdx.x * blockDim.x + threadIdx.x;  // grid (column blocks, rows): no index division
  if (gx >= a.c1) return;
  const int lx = gx - a.col_off;
  for (int gy = a.r0 + blockIdx.y; gy < a.r1; gy += gridDim.y) {
    const int ly = gy - a.row_off;
    const float* g = a.gimg;
    float acc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] = g[((size_t)ly * a.Wl + lx) * 3 + c];
    // local rows / columns beyond the image (replicate padding) fold onto row h-1 / column w-1
    if (gy == a.h - 1)
      for (int yy = ly + 1; yy < a.Hl; ++yy)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += g[((size_t)yy * a.Wl + lx) * 3 + c];
    if (gx == a.w - 1)
      for (int xx = lx + 1; xx < a.Wl; ++xx)
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[c] += g[((size_t)ly * a.Wl + xx) * 3 + c];
    if (gy == a.h - 1 && gx == a.w - 1)
      for (int yy = ly + 1; yy < a.Hl; ++yy)
        for (int xx = lx + 1; xx < a.Wl; ++xx)
#pragma unroll
          for (int c = 0; c < 3; ++c) acc[c] += g[((size_t)yy * a.Wl + xx) * 3 + c];
    float* o = a.grad + ((long long)gy * a.pitch + gx) * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) o[c] = acc[c];
  }
}

// 2x2 average pool HL16 -> HL16 (used when the first conv's ReLU is followed by a pool).
__global__ void pool2_hl_kernel(HL16 in, HL16 out, unsigned int* amax) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long n = (long long)(in.C_p / 8) * out.H * out.W;
  float m = 0.f;
  if (i < n) {
    const int kg = (int)(i / ((long long)out.H * out.W));
    const int rem = (int)(i % ((long long)out.H * out.W));
    const int py = rem / out.W, px = rem % out.W;
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const float inv = 1.f / in.scale;
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const size_t off = ((size_t)kg * in.H + 2 * py + dy) * in.W + 2 * px + dx;
        uint4 hv = reinterpret_cast<const uint4*>(in.hi)[off];
        uint4 lv = reinterpret_cast<const uint4*>(in.lo())[off];
        const __half* hh = reinterpret_cast<const __half*>(&hv);
        const __half* ll = reinterpret_cast<const __half*>(&lv);
#pragma unroll
        for (int e = 0; e < 8; ++e) s[e] += (__half2float(hh[e]) + __half2float(ll[e])) * inv;
      }
    __align__(16) __half oh[8];
    __align__(16) __half ol[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float v = s[e] * 0.25f;
      m = fmaxf(m, fabsf(v));
      HalfPair p = split_f16(v * out.scale);
      oh[e] = p.hi;
      ol[e] = p.lo;
    }
    const size_t off = ((size_t)kg * out.H + py) * out.W + px;
    reinterpret_cast<uint4*>(out.hi)[off] = *reinterpret_cast<uint4*>(oh);
    reinterpret_cast<uint4*>(out.lo())[off] = *reinterpret_cast<uint4*>(ol);
  }
  if (amax) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(amax, __float_as_uint(m));
  }
}

// sums[c] = sum_r partial[r][c] in f64, fixed row order
// Two-level deterministic column sums: stage 1 reduces row chunks (fixed strided order per
// thread, fixed tree across threadIdx.y), stage 2 sums the chunk partials in chunk order.
constexpr int kColsumChunks = 256;

__global__ void colsum_stage1_kernel(const float* partial, int rows, int C, int stride, int rows_per,
                                     double* mid) {
  __shared__ double red[8][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * rows_per, r1 = min(r0 + rows_per, rows);
  double acc = 0.0;
  if (c < C)
    for (int r = r0 + threadIdx.y; r < r1; r += 8) acc += (double)partial[(size_t)r * stride + c];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < C) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i][threadIdx.x];
    mid[(size_t)blockIdx.y * C + c] = t;
  }
}

__global__ void colsum_stage2_kernel(const double* mid, int chunks, int C, double* sums) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double acc = 0.0;
  for (int b = 0; b < chunks; ++b) acc += mid[(size_t)b * C + c];
  sums[c] = acc;
}

// ------------------------------------------------------------------------------------------
// statistics finalisation + style coefficients (one tap)
// ------------------------------------------------------------------------------------------

constexpr double kStdEps = 1e-8;

__global__ void style_vec_kernel(StyleCoefArgs a) {
  __shared__ double red[2][256];
  double lm = 0.0, ls = 0.0;
  for (int c = threadIdx.x; c < a.C; c += blockDim.x) {
    const double g = a.S[(size_t)c * a.C + c] / a.n;
    const double m = a.s[c] / a.n;
    const double sd = sqrt(fmax(g - m * m, 0.0));
    a.mu[c] = m;
    a.sd[c] = sd;
    const bool dead = sd < kStdEps;
    if (dead && a.sdr[c] > kStdEps) *a.degenerate = 1;
    const double r = dead ? 0.0 : (sd - a.sdr[c]) / sd;
    a.ratio[c] = r;
    double b = 0.0;
    if (a.wm != 0.0) b += (2.0 * a.wm / a.n) * (m - a.mur[c]);
    if (a.ws != 0.0) b -= (2.0 * a.ws / a.n) * m * r;
    a.bvec[c] = (float)b;
    lm += (m - a.mur[c]) * (m - a.mur[c]);
    ls += (sd - a.sdr[c]) * (sd - a.sdr[c]);
  }
  red[0][threadIdx.x] = lm;
  red[1][threadIdx.x] = ls;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t0 = 0.0, t1 = 0.0;
    for (int i = 0; i < blockDim.x; ++i) {
      t0 += red[0][i];
      t1 += red[1][i];
    }
    a.ms_loss[0] = t0;
    a.ms_loss[1] = t1;
  }
}

// one block per row k: M[k][n] = (4wg/n)(G-Gr)[k][n] + delta_kn (2ws/n) ratio[n]
__global__ void style_mat_kernel(StyleCoefArgs a) {
  __shared__ double red[256];
  __shared__ double redm[256];
  const int k = blockIdx.x;
  double acc = 0.0, mm = 0.0;
  const int kc = k / (8 * a.xkg), kg = (k >> 3) % a.xkg, e = k & 7;
  for (int n = threadIdx.x; n < a.C; n += blockDim.x) {
    const double g = a.S[(size_t)k * a.C + n] / a.n;
    const double d = g - a.Gr[(size_t)k * a.C + n];
    acc += d * d;
    double mv = (a.wg != 0.0) ? (4.0 * a.wg / a.n) * d : 0.0;
    if (n == k && a.ws != 0.0) mv += (2.0 * a.ws / a.n) * a.ratio[n];
    mm = fmax(mm, fabs(mv));
    if (a.xw) {
      const float v = (float)(mv * (double)a.xscale);
      HalfPair p = split_f16(v);
      const int nt = n / a.N, nl = n % a.N;
      const size_t base = ((size_t)nt * a.n_xkc + kc) * 2;
      a.xw[(((base + 0) * a.xkg + kg) * a.N + nl) * 8 + e] = p.hi;
      a.xw[(((base + 1) * a.xkg + kg) * a.N + nl) * 8 + e] = p.lo;
    }
  }
  red[threadIdx.x] = acc;
  redm[threadIdx.x] = mm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0, m = 0.0;
    for (int i = 0; i < blockDim.x; ++i) {
      t += red[i];
      m = fmax(m, redm[i]);
    }
    a.row_loss[k] = t;
    a.row_mmax[k] = m;
  }
}

// ------------------------------------------------------------------------------------------
// content squared distance over local rows [r0, r1): sum (V - Vu)^2 (f64 partials)
// ------------------------------------------------------------------------------------------
// ------------------------------------------------------------------------------------------
// deterministic reductions and L-BFGS vector passes
// ------------------------------------------------------------------------------------------
constexpr int kRedBlocks = 2 * kSMs;
constexpr int kRedThreads = 512;

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  T t = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  return t;
}

// content distance sum over owned rows of (V/s_v - U/s_u)^2 (reference localized.py:257-267):
// grid (x: blocks per kgroup plane, y: kgroup), so each block walks one contiguous run of
// 16-byte pixels (no per-element index division) with two pixels' four loads in flight per
// thread.  HBM-bound: 4 x 16 B read per pixel and kgroup.
__device__ __forceinline__ double sqdiff8(uint4 vh, uint4 vl, uint4 uh, uint4 ul, float iv, float iu, int nvalid) {
  const __half* a0 = reinterpret_cast<const __half*>(&vh);
  const __half* a1 = reinterpret_cast<const __half*>(&vl);
  const __half* b0 = reinterpret_cast<const __half*>(&uh);
  const __half* b1 = reinterpret_cast<const __half*>(&ul);
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    if (e >= nvalid) continue;
    const float dv = (__half2float(a0[e]) + __half2float(a1[e])) * iv - (__half2float(b0[e]) + __half2float(b1[e])) * iu;
    acc += (double)dv * (double)dv;
  }
  return acc;
}

__global__ void __launch_bounds__(kRedThreads) content_sqdiff_kernel(HL16 v, HL16 u, int C, int r0, int r1,
                                                                     int c0, int c1, double* partial) {
  __shared__ double sh[32];
  const int kg = blockIdx.y;
  const int wc = c1 - c0;
  if (wc != v.W) {  // owned rectangle narrower than the grid (windowed evaluation): row/column loop
    double acc = 0.0;
    const int nvalid = min(8, C - kg * 8);
    const float iv = 1.f / v.scale, iu = 1.f / u.scale;
    const long long n = (long long)(r1 - r0) * wc;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
      const size_t o = ((size_t)kg * v.H + r0 + i / wc) * v.W + c0 + i % wc;
      acc += sqdiff8(reinterpret_cast<const uint4*>(v.hi)[o], reinterpret_cast<const uint4*>(v.lo())[o],
                     reinterpret_cast<const uint4*>(u.hi)[o], reinterpret_cast<const uint4*>(u.lo())[o], iv, iu,
                     nvalid);
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
    return;
  }
  const long long per_plane = (long long)(r1 - r0) * v.W;
  const size_t base = (size_t)kg * v.H * v.W + (size_t)r0 * v.W;
  const uint4* vh = reinterpret_cast<const uint4*>(v.hi) + base;
  const uint4* vl = reinterpret_cast<const uint4*>(v.lo()) + base;
  const uint4* uh = reinterpret_cast<const uint4*>(u.hi) + base;
  const uint4* ul = reinterpret_cast<const uint4*>(u.lo()) + base;
  const int nvalid = min(8, C - kg * 8);
  const float iv = 1.f / v.scale, iu = 1.f / u.scale;
  const long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < per_plane; i += 2 * stride) {
    const uint4 a0 = vh[i], a1 = vl[i], b0 = uh[i], b1 = ul[i];
    const uint4 c0 = vh[i + stride], c1 = vl[i + stride], d0 = uh[i + stride], d1 = ul[i + stride];
    acc += sqdiff8(a0, a1, b0, b1, iv, iu, nvalid);
    acc += sqdiff8(c0, c1, d0, d1, iv, iu, nvalid);
  }
  if (i < per_plane) acc += sqdiff8(vh[i], vl[i], uh[i], ul[i], iv, iu, nvalid);
  const double t = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.y * gridDim.x + blockIdx.x] = t;
}


// partial dot products for up to 3 simultaneous pairs: <a0,b0>, <a1,b1>, <a2,b2>
template <typename T>
__global__ void __launch_bounds__(kRedThreads) dot3_partial_kernel(const T* a0, const T* b0, const T* a1,
                                                                   const T* b1, const T* a2, const T* b2,
                                                                   long long n, double* partial) {
  __shared__ double sh[32];
  double s0 = 0, s1 = 0, s2 = 0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  long long start = 0;
  if constexpr (sizeof(T) == 4) {  // float4 body
    const long long n4 = n / 4;
    for (long long i = tid; i < n4; i += nth) {
      const float4 x = reinterpret_cast<const float4*>(a0)[i], y = reinterpret_cast<const float4*>(b0)[i];
      s0 += (double)x.x * y.x + (double)x.y * y.y + (double)x.z * y.z + (double)x.w * y.w;
      if (a1) {
        const float4 u = reinterpret_cast<const float4*>(a1)[i], v = reinterpret_cast<const float4*>(b1)[i];
        s1 += (double)u.x * v.x + (double)u.y * v.y + (double)u.z * v.z + (double)u.w * v.w;
      }
      if (a2) {
        const float4 u = reinterpret_cast<const float4*>(a2)[i], v = reinterpret_cast<const float4*>(b2)[i];
        s2 += (double)u.x * v.x + (double)u.y * v.y + (double)u.z * v.z + (double)u.w * v.w;
      }
    }
    start = n4 * 4;
  }
  for (long long i = start + tid; i < n; i += nth) {
    s0 += (double)a0[i] * (double)b0[i];
    if (a1) s1 += (double)a1[i] * (double)b1[i];
    if (a2) s2 += (double)a2[i] * (double)b2[i];
  }
  double t = block_sum(s0, sh);
  __syncthreads();
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  if (a1) {
    t = block_sum(s1, sh);
    __syncthreads();
    if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = t;
  }
  if (a2) {
    t = block_sum(s2, sh);
    __syncthreads();
    if (threadIdx.x == 0) partial[2 * gridDim.x + blockIdx.x] = t;
  }
}

// out[k] = sum_b partial[k*nb + b], k < nk (fixed order)
// The library's one fixed reduction order for block partials (whole warp; every lane returns
// the total): lane l sums p[l], p[l+32], ... in order, then a fixed xor butterfly.  Used by the
// finish kernel, the fused two-loop finish and the cooperative two-loop, so all agree bitwise.
__device__ __forceinline__ double warp_fixed_sum(const double* p, int nb) {
  const int l = threadIdx.x & 31;
  double acc = 0.0;
  for (int b = l; b < nb; b += 32) acc += __ldcg(p + b);  // L2: other blocks wrote these this launch
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  return acc;
}

// out[k] = fixed-order sum of partial[k*nb .. k*nb+nb), one warp per quantity
__global__ void finish_sums_kernel(const double* partial, int nb, int nk, double* out) {
  const int k = threadIdx.x >> 5;
  if (k >= nk) return;
  const double t = warp_fixed_sum(partial + (size_t)k * nb, nb);
  if ((threadIdx.x & 31) == 0) out[k] = t;
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads) absmax_partial_kernel(const T* a, long long n, double* partial) {
  __shared__ double sh[32];
  double m = 0.0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  long long start = 0;
  if constexpr (sizeof(T) == 4) {  // 16-byte loads when aligned (max is exact in any order)
    if ((reinterpret_cast<uintptr_t>(a) & 15) == 0) {
      const long long n4 = n / 4;
      float mf = 0.f;
      for (long long i = tid; i < n4; i += nth) {
        const float4 q = reinterpret_cast<const float4*>(a)[i];
        mf = fmaxf(mf, fmaxf(fmaxf(fabsf(q.x), fabsf(q.y)), fmaxf(fabsf(q.z), fabsf(q.w))));
      }
      m = mf;
      start = n4 * 4;
    }
  }
  for (long long i = start + tid; i < n; i += nth) m = fmax(m, fabs((double)a[i]));
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmax(t, sh[i]);
    partial[blockIdx.x] = t;
  }
}

__global__ void finish_max_kernel(const double* partial, int nb, double* out) {
  double m = 0.0;
  for (int b = 0; b < nb; ++b) m = fmax(m, partial[b]);
  *out = m;
}

// Two-loop step body (one block's slice): q_out = cscale * (q_in + c * v); returns the block's
// partial <w, q_out> in thread 0 (0 elsewhere).  Shared by the per-step and cooperative kernels so
// both produce identical bits.
template <typename T>
__device__ __forceinline__ double axpy_dot_body(const T* qi, T* qo, const T* v, T c, T cs, const T* w, long long n,
                                                double* sh) {
  double s = 0.0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  long long start = 0;
  if constexpr (sizeof(T) == 4) {  // float4 body
    const long long n4 = n / 4;
    for (long long i = tid; i < n4; i += nth) {
      float4 q = reinterpret_cast<const float4*>(qi)[i];
      if (v) {
        const float4 vv = reinterpret_cast<const float4*>(v)[i];
        q.x = q.x + c * vv.x;
        q.y = q.y + c * vv.y;
        q.z = q.z + c * vv.z;
        q.w = q.w + c * vv.w;
      }
      q.x *= cs;
      q.y *= cs;
      q.z *= cs;
      q.w *= cs;
      reinterpret_cast<float4*>(qo)[i] = q;
      if (w) {
        const float4 ww = reinterpret_cast<const float4*>(w)[i];
        s += (double)ww.x * q.x + (double)ww.y * q.y + (double)ww.z * q.z + (double)ww.w * q.w;
      }
    }
    start = n4 * 4;
  }
  for (long long i = start + tid; i < n; i += nth) {
    T q = qi[i];
    if (v) q = q + c * v[i];
    q = q * cs;
    qo[i] = q;
    if (w) s += (double)w[i] * (double)q;
  }
  return w ? block_sum(s, sh) : 0.0;
}

// Two-loop step: q_out = cscale * (q_in + coef[0] * v); partial <w, q_out>.
template <typename T>
__global__ void __launch_bounds__(kRedThreads) axpy_dot_kernel(AxpyDotArgs a) {
  __shared__ double sh[32];
  const T* qi = reinterpret_cast<const T*>(a.q_in);
  T* qo = reinterpret_cast<T*>(a.q_out);
  const T* v = reinterpret_cast<const T*>(a.v);
  const T* w = reinterpret_cast<const T*>(a.w);
  const T c = v ? (T)(*a.coef) : (T)0;
  const double t = axpy_dot_body<T>(qi, qo, v, c, (T)a.cscale, w, a.n, sh);
  if (w) {
    if (threadIdx.x == 0) a.partial[blockIdx.x] = t;
    if (a.alpha_i) {  // fused finish: the last block reduces in block order, then the scalar step
      __shared__ bool last;
      __threadfence();
      if (threadIdx.x == 0) last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
      __syncthreads();
      if (last && threadIdx.x < 32) {
        __threadfence();
        const double dot = warp_fixed_sum(a.partial, gridDim.x);
        if (threadIdx.x == 0) {
          double* coef = const_cast<double*>(a.coef);  // read by every block at entry, written here last
          if (a.mode == 0) {
            *a.alpha_i = a.rho * dot;
            *coef = -(*a.alpha_i);
          } else {
            *coef = *a.alpha_i - a.rho * dot;
          }
          *a.ticket = 0u;
        }
      }
    }
  }
}

// The whole two-loop (lbfgs.py:68-83) in one cooperative launch: each step is the body above,
// then one grid barrier; every block sums the partials in block order and applies the scalar
// update itself (alpha kept in shared memory), so the result equals the per-step kernels bit for
// bit.  Partials are double-buffered, so one barrier per step suffices.
template <typename T>
__global__ void __launch_bounds__(kRedThreads, 2) two_loop_coop_kernel(const __grid_constant__ TwoLoopArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[32];
  __shared__ double alpha[kTwoLoopMaxHist];
  __shared__ double sdot;
  T* out = reinterpret_cast<T*>(a.out);
  double coef = 0.0;
  int par = 0;
  auto step = [&](const T* qi, const T* v, double cscale, const T* w, int i, int mode) {
    const T c = v ? (T)coef : (T)0;
    const double t = axpy_dot_body<T>(qi, out, v, c, (T)cscale, w, a.n, sh);
    if (!w) return;
    double* P = a.partial + par * gridDim.x;
    if (threadIdx.x == 0) P[blockIdx.x] = t;
    grid.sync();
    if (threadIdx.x < 32) {
      const double dot = warp_fixed_sum(P, gridDim.x);
      if (threadIdx.x != 0) {
      } else if (mode == 0) {
        alpha[i] = a.rho[i] * dot;
        sdot = -alpha[i];
      } else {
        sdot = alpha[i] - a.rho[i] * dot;
      }
    }
    __syncthreads();
    coef = sdot;
    __syncthreads();  // sdot is rewritten by the next step
    par ^= 1;
  };
  const int m = a.m;
  const T* g = reinterpret_cast<const T*>(a.g);
  auto S = [&](int i) { return reinterpret_cast<const T*>(a.s[i]); };
  auto Y = [&](int i) { return reinterpret_cast<const T*>(a.y[i]); };
  step(g, nullptr, 1.0, S(m - 1), m - 1, 0);
  for (int i = m - 1; i > 0; --i) step(out, Y(i), 1.0, S(i - 1), i - 1, 0);
  step(out, Y(0), a.gamma, Y(0), 0, 1);
  for (int i = 0; i < m - 1; ++i) step(out, S(i), 1.0, Y(i + 1), i + 1, 1);
  step(out, S(m - 1), -1.0, nullptr, 0, 0);
}

// two-loop scalar bookkeeping from a finished (and possibly all-reduced) dot product
// mode 0: alpha_i = rho * dot, coef = -alpha_i;  mode 1: coef = alpha_i - rho * dot
__global__ void twoloop_scalar_kernel(const double* dot, double rho, int mode, double* alpha_i, double* coef) {
  if (mode == 0) {
    *alpha_i = rho * (*dot);
    *coef = -(*alpha_i);
  } else {
    *coef = *alpha_i - rho * (*dot);
  }
}

// x_out = x + t*d (numpy weak-scalar semantics: t has x's dtype, product rounded then sum)
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// two separate roundings (no FMA contraction), as numpy evaluates x + t * d
template <typename T>
__global__ void axpy_kernel(const T* x, const T* d, T t, long long n, T* out) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  long long start = 0;
  if constexpr (sizeof(T) == 4) {
    const long long n4 = n / 4;
    for (long long i = tid; i < n4; i += nth) {
      const float4 a = reinterpret_cast<const float4*>(x)[i], b = reinterpret_cast<const float4*>(d)[i];
      reinterpret_cast<float4*>(out)[i] = make_float4(add_rn(a.x, mul_rn(t, b.x)), add_rn(a.y, mul_rn(t, b.y)),
                                                      add_rn(a.z, mul_rn(t, b.z)), add_rn(a.w, mul_rn(t, b.w)));
    }
    start = n4 * 4;
  }
  for (long long i = start + tid; i < n; i += nth) out[i] = add_rn(x[i], mul_rn(t, d[i]));
}

// s = xt - x, y = gt - g and partials of <y,s>, <s,s>, <y,y>
template <typename T>
__global__ void __launch_bounds__(kRedThreads) sy_kernel(const T* xt, const T* x, const T* gt, const T* g,
                                                         long long n, T* s, T* y, double* partial) {
  __shared__ double sh[32];
  double ys = 0, ss = 0, yy = 0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long long)gridDim.x * blockDim.x;
  long long start = 0;
  if constexpr (sizeof(T) == 4) {
    const long long n4 = n / 4;
    for (long long i = tid; i < n4; i += nth) {
      const float4 a = reinterpret_cast<const float4*>(xt)[i], b = reinterpret_cast<const float4*>(x)[i];
      const float4 c = reinterpret_cast<const float4*>(gt)[i], d = reinterpret_cast<const float4*>(g)[i];
      const float4 si = make_float4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
      const float4 yi = make_float4(c.x - d.x, c.y - d.y, c.z - d.z, c.w - d.w);
      reinterpret_cast<float4*>(s)[i] = si;
      reinterpret_cast<float4*>(y)[i] = yi;
      ys += (double)yi.x * si.x + (double)yi.y * si.y + (double)yi.z * si.z + (double)yi.w * si.w;
      ss += (double)si.x * si.x + (double)si.y * si.y + (double)si.z * si.z + (double)si.w * si.w;
      yy += (double)yi.x * yi.x + (double)yi.y * yi.y + (double)yi.z * yi.z + (double)yi.w * yi.w;
    }
    start = n4 * 4;
  }
  for (long long i = start + tid; i < n; i += nth) {
    const T si = xt[i] - x[i];
    const T yi = gt[i] - g[i];
    s[i] = si;
    y[i] = yi;
    ys += (double)yi * si;
    ss += (double)si * si;
    yy += (double)yi * yi;
  }
  double t = block_sum(ys, sh);
  __syncthreads();
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
  t = block_sum(ss, sh);
  __syncthreads();
  if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = t;
  t = block_sum(yy, sh);
  __syncthreads();
  if (threadIdx.x == 0) partial[2 * gridDim.x + blockIdx.x] = t;
}

// ------------------------------------------------------------------------------------------
// resampling (HWC f32)
// ------------------------------------------------------------------------------------------
// T = float: the reference's f32 images; T = double: its f64 path (same formulas in double)
template <typename T>
__global__ void resize_down_kernel(const T* in, int h, int w, int c, int f, T* out) {
  const int oh = (h + f - 1) / f, ow = (w + f - 1) / f;
  const long long n = (long long)oh * ow * c;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(i % c);
    const long long p = i / c;
    const int oy = (int)(p / ow), ox = (int)(p % ow);
    const int y0 = oy * f, y1 = min(y0 + f, h), x0 = ox * f, x1 = min(x0 + f, w);
    // reference order: rows of each column summed first (reduceat axis 0), then columns
    T tot = 0;
    for (int xx = x0; xx < x1; ++xx) {
      T col = 0;
      for (int yy = y0; yy < y1; ++yy) col += in[((size_t)yy * w + xx) * c + ch];
      tot += col;
    }
    const T area = (T)(y1 - y0) * (T)(x1 - x0);
    out[i] = tot / area;
  }
}

template <typename T>
__device__ __forceinline__ void bilin_axis(int i, int n_in, int n_out, int& i0, int& i1, T& t) {
  double s = ((double)i + 0.5) * ((double)n_in / (double)n_out) - 0.5;
  s = fmin(fmax(s, 0.0), (double)n_in - 1.0);
  i0 = (int)floor(s);
  i1 = min(i0 + 1, n_in - 1);
  t = (T)(s - (double)i0);
}

__device__ __forceinline__ float mul_t(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_t(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double mul_t(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_t(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void resize_bilinear_kernel(const T* in, int h, int w, int c, int oh, int ow, T* out) {
  const long long n = (long long)oh * ow * c;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int ch = (int)(i % c);
    const long long p = i / c;
    const int oy = (int)(p / ow), ox = (int)(p % ow);
    int y0, y1, x0, x1;
    T ty, tx;
    bilin_axis(oy, h, oh, y0, y1, ty);
    bilin_axis(ox, w, ow, x0, x1, tx);
    const T omy = (T)1 - ty, omx = (T)1 - tx;
    const T r0 = add_t(mul_t(in[((size_t)y0 * w + x0) * c + ch], omy), mul_t(in[((size_t)y1 * w + x0) * c + ch], ty));
    const T r1 = add_t(mul_t(in[((size_t)y0 * w + x1) * c + ch], omy), mul_t(in[((size_t)y1 * w + x1) * c + ch], ty));
    out[i] = add_t(mul_t(r0, omx), mul_t(r1, tx));
  }
}

// ------------------------------------------------------------------------------------------
// launch helpers
// ------------------------------------------------------------------------------------------
cudaError_t launch_image_hl(const ImageHLArgs& a, cudaStream_t st) {
  const int bx = (a.Wp + 255) / 256;  // column blocks per row; ~148 x 8 blocks in total
  const dim3 grid(bx, std::max(1, std::min(a.Hl, 148 * 8 / bx)));
  note_launch(), image_hl_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_first_conv_bwd(const FirstConvBwdArgs& a, cudaStream_t st) {
  dim3 grid((a.g.W + FC_BX - 1) / FC_BX, (a.g.H + FC_BY - 1) / FC_BY);
  note_launch(), first_conv_bwd_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fold_grad(const FoldArgs& a, cudaStream_t st) {
  if (a.r1 <= a.r0 || a.c1 <= a.c0) return cudaSuccess;
  const dim3 grid((a.c1 - a.c0 + 255) / 256, std::min(a.r1 - a.r0, 65535));
  note_launch(), fold_grad_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pool2_hl(const HL16& in, const HL16& out, unsigned int* amax, cudaStream_t st) {
  const long long n = (long long)(in.C_p / 8) * out.H * out.W;
  note_launch(), pool2_hl_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, out, amax);
  return cudaGetLastError();
}

cudaError_t launch_colsum_reduce(const float* partial, int rows, int C, int stride, double* sums, double* mid,
                                 cudaStream_t st) {
  const int rows_per = (rows + kColsumChunks - 1) / kColsumChunks;
  const int chunks = (rows + rows_per - 1) / rows_per;
  note_launch(), colsum_stage1_kernel<<<dim3((C + 31) / 32, chunks), dim3(32, 8), 0, st>>>(partial, rows, C, stride, rows_per, mid);
  note_launch(), colsum_stage2_kernel<<<(C + 127) / 128, 128, 0, st>>>(mid, chunks, C, sums);
  return cudaGetLastError();
}

cudaError_t launch_style_vec(const StyleCoefArgs& a, cudaStream_t st) {
  note_launch(), style_vec_kernel<<<1, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_style_mat(const StyleCoefArgs& a, cudaStream_t st) {
  note_launch(), style_mat_kernel<<<a.C, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double* partial, int nk, double* out, cudaStream_t st) {
  note_launch(), finish_sums_kernel<<<1, 32 * nk, 0, st>>>(partial, kRedBlocks, nk, out);
  return cudaGetLastError();
}

cudaError_t launch_content_sqdiff(const HL16& v, const HL16& u, int C, int r0, int r1, int c0, int c1,
                                  double* partial, double* out, cudaStream_t st) {
  const int nkg = (C + 7) / 8;  // kgroups holding real channels
  if (nkg > kRedBlocks) return cudaErrorInvalidValue;
  const dim3 grid(std::max(1, kRedBlocks / nkg), nkg);  // <= kRedBlocks partials
  note_launch(), content_sqdiff_kernel<<<grid, kRedThreads, 0, st>>>(v, u, C, r0, r1, c0, c1, partial);
  note_launch(), finish_sums_kernel<<<1, 32, 0, st>>>(partial, (int)(grid.x * grid.y), 1, out);
  return cudaGetLastError();
}

cudaError_t launch_dots(int f64, const void* a0, const void* b0, const void* a1, const void* b1, const void* a2,
                        const void* b2, long long n, double* partial, double* out, cudaStream_t st) {
  if (f64)
    note_launch(), dot3_partial_kernel<double><<<kRedBlocks, kRedThreads, 0, st>>>(
        (const double*)a0, (const double*)b0, (const double*)a1, (const double*)b1, (const double*)a2,
        (const double*)b2, n, partial);
  else
    note_launch(), dot3_partial_kernel<float><<<kRedBlocks, kRedThreads, 0, st>>>((const float*)a0, (const float*)b0,
                                                                   (const float*)a1, (const float*)b1,
                                                                   (const float*)a2, (const float*)b2, n, partial);
  const int nk = 1 + (a1 != nullptr) + (a2 != nullptr);
  note_launch(), finish_sums_kernel<<<1, 32 * nk, 0, st>>>(partial, kRedBlocks, nk, out);
  return cudaGetLastError();
}

cudaError_t launch_absmax(int f64, const void* a, long long n, double* partial, double* out, cudaStream_t st) {
  if (f64)
    note_launch(), absmax_partial_kernel<double><<<kRedBlocks, kRedThreads, 0, st>>>((const double*)a, n, partial);
  else
    note_launch(), absmax_partial_kernel<float><<<kRedBlocks, kRedThreads, 0, st>>>((const float*)a, n, partial);
  note_launch(), finish_max_kernel<<<1, 1, 0, st>>>(partial, kRedBlocks, out);
  return cudaGetLastError();
}

// cooperative two-loop; returns cudaErrorNotSupported when co-residency of the reduction grid
// is not available (the caller then issues the per-step kernels)
cudaError_t launch_two_loop_coop(int f64, const TwoLoopArgs& a, cudaStream_t st) {
  if (a.m < 1 || a.m > kTwoLoopMaxHist) return cudaErrorNotSupported;
  const void* fn = f64 ? (const void*)two_loop_coop_kernel<double> : (const void*)two_loop_coop_kernel<float>;
  // co-residency of the grid, queried once per device and precision (the query costs tens of
  // microseconds of host time per L-BFGS iteration otherwise, with the GPU idle behind it)
  constexpr int kMaxDev = 64;
  static int ok_cache[kMaxDev][2] = {};  // 0 unknown, 1 cooperative launch fits, 2 it does not
  int dev = 0;
  cudaGetDevice(&dev);
  int& ok = ok_cache[dev < kMaxDev ? dev : 0][f64 ? 1 : 0];
  if (ok == 0) {
    int coop = 0, per_sm = 0, sms = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kRedThreads, 0);
    ok = (coop && per_sm * sms >= kRedBlocks) ? 1 : 2;
  }
  if (ok != 1) {
    cudaGetLastError();
    return cudaErrorNotSupported;
  }
  void* args[] = {const_cast<TwoLoopArgs*>(&a)};
  note_launch();
  return cudaLaunchCooperativeKernel(fn, dim3(kRedBlocks), dim3(kRedThreads), args, 0, st);
}

cudaError_t launch_axpy_dot(int f64, const AxpyDotArgs& a, cudaStream_t st) {
  if (f64)
    note_launch(), axpy_dot_kernel<double><<<kRedBlocks, kRedThreads, 0, st>>>(a);
  else
    note_launch(), axpy_dot_kernel<float><<<kRedBlocks, kRedThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_twoloop_scalar(const double* dot, double rho, int mode, double* alpha_i, double* coef,
                                  cudaStream_t st) {
  note_launch(), twoloop_scalar_kernel<<<1, 1, 0, st>>>(dot, rho, mode, alpha_i, coef);
  return cudaGetLastError();
}



cudaError_t launch_axpy(int f64, const void* x, const void* d, double t, long long n, void* out, cudaStream_t st) {
  if (f64)
    note_launch(), axpy_kernel<double><<<4 * kSMs, 512, 0, st>>>((const double*)x, (const double*)d, t, n, (double*)out);
  else
    note_launch(), axpy_kernel<float><<<4 * kSMs, 512, 0, st>>>((const float*)x, (const float*)d, (float)t, n, (float*)out);
  return cudaGetLastError();
}

cudaError_t launch_sy(int f64, const void* xt, const void* x, const void* gt, const void* g, long long n, void* s,
                      void* y, double* partial, double* out, cudaStream_t st) {
  if (f64)
    note_launch(), sy_kernel<double><<<kRedBlocks, kRedThreads, 0, st>>>((const double*)xt, (const double*)x, (const double*)gt,
                                                          (const double*)g, n, (double*)s, (double*)y, partial);
  else
    note_launch(), sy_kernel<float><<<kRedBlocks, kRedThreads, 0, st>>>((const float*)xt, (const float*)x, (const float*)gt,
                                                         (const float*)g, n, (float*)s, (float*)y, partial);
  note_launch(), finish_sums_kernel<<<1, 96, 0, st>>>(partial, kRedBlocks, 3, out);
  return cudaGetLastError();
}

cudaError_t launch_resize_down(int f64, const void* in, int h, int w, int c, int f, void* out, cudaStream_t st) {
  if (f64)
    note_launch(), resize_down_kernel<double><<<4 * kSMs, 256, 0, st>>>((const double*)in, h, w, c, f, (double*)out);
  else
    note_launch(), resize_down_kernel<float><<<4 * kSMs, 256, 0, st>>>((const float*)in, h, w, c, f, (float*)out);
  return cudaGetLastError();
}

cudaError_t launch_resize_bilinear(int f64, const void* in, int h, int w, int c, int oh, int ow, void* out,
                                   cudaStream_t st) {
  if (f64)
    note_launch(), resize_bilinear_kernel<double><<<4 * kSMs, 256, 0, st>>>((const double*)in, h, w, c, oh, ow,
                                                                             (double*)out);
  else
    note_launch(), resize_bilinear_kernel<float><<<4 * kSMs, 256, 0, st>>>((const float*)in, h, w, c, oh, ow,
                                                                            (float*)out);
  return cudaGetLastError();
}

int red_blocks() { return kRedBlocks; }

}  // namespace spst
