// umma_probe.cu — hardware probe for the descriptor conventions the conv/Gram kernels rely on.
// Standalone (no torch): nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I.. umma_probe.cu -o probe
// Checks: (1) K-major SWIZZLE_NONE A/B, (2) row-shifted A views (start address + r*16 B),
// (3) MN-major A/B (Gram layout), (4) 4-D TMA load of the CHW8 layout with OOB zero fill,
// (5) accumulation rounding of fp32 TMEM accumulators over long K.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>
#include "../paper_2212_13459_b200/csrc/sm100.cuh"

using namespace spst;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

// A: [M_ROWS_ALLOC][K] row-major fp16 (global), B: [N][K] row-major fp16.
// amode 0: A K-major interleave; amode 1: A MN-major interleave (A stored [K][M] in global).
// bmode likewise. shift: A view starts at row `shift` (K-major only).
template <int N>
__global__ void probe_gemm(const __half* A, const __half* B, float* D, int K, int amode, int bmode, int shift,
                           int mrows_alloc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  uint8_t* sa = smem;
  uint8_t* sb = smem + ((mrows_alloc * 16 * 16 + 1023) / 1024) * 1024;  // K chunk 16 per pass
  if (warp_id() == 0) tmem_alloc<256>(&tslot);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tbase = tslot;
  const uint32_t idesc = make_idesc_f16(128, N, 0, amode, bmode);
  uint32_t phase = 0;
  for (int k0 = 0; k0 < K; k0 += 16) {
    // stage A chunk rows [0,mrows_alloc) x k [k0,k0+16)
    for (int i = tid; i < mrows_alloc * 16; i += blockDim.x) {
      int m = i / 16, k = i % 16;
      __half v = amode == 0 ? A[(size_t)m * K + k0 + k] : A[(size_t)(k0 + k) * mrows_alloc + m];
      uint32_t off;
      if (amode == 0)  // K-major: [kg(2)][m][8]
        off = (k / 8) * (mrows_alloc * 16) + m * 16 + (k % 8) * 2;
      else  // MN-major: [mg][kk(16)][8]: core = 8 m (contig) x 8 k (16 B stride); LBO(k-group)=128, SBO(m-group)=256
        off = (m / 8) * 256 + (k / 8) * 128 + (k % 8) * 16 + (m % 8) * 2;
      *reinterpret_cast<__half*>(sa + off) = v;
    }
    for (int i = tid; i < N * 16; i += blockDim.x) {
      int n = i / 16, k = i % 16;
      __half v = bmode == 0 ? B[(size_t)n * K + k0 + k] : B[(size_t)(k0 + k) * N + n];
      uint32_t off;
      if (bmode == 0)
        off = (k / 8) * (N * 16) + n * 16 + (k % 8) * 2;
      else
        off = (n / 8) * 256 + (k / 8) * 128 + (k % 8) * 16 + (n % 8) * 2;
      *reinterpret_cast<__half*>(sb + off) = v;
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      uint64_t ad, bd;
      if (amode == 0)
        ad = make_sdesc(smem_u32(sa) + shift * 16, mrows_alloc * 16, 128);
      else
        ad = make_sdesc(smem_u32(sa), 128, 256);
      if (bmode == 0)
        bd = make_sdesc(smem_u32(sb), N * 16, 128);
      else
        bd = make_sdesc(smem_u32(sb), 128, 256);
      umma_f16(tbase, ad, bd, idesc, k0 > 0);
      umma_commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    tc_fence_after();
    __syncthreads();
  }
  // read TMEM: 4 warps x 32 lanes
  int w = tid / 32;
  if (w < 4) {
    for (int c = 0; c < N; c += 32) {
      float v[32];
      tmem_ld32(tbase + ((uint32_t)(w * 32) << 16) + c, v);
      int m = w * 32 + (tid & 31);
      for (int j = 0; j < 32; ++j) D[m * N + c + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<256>(tbase);
}

__global__ void probe_tma(const __grid_constant__ CUtensorMap tmap, uint16_t* out, int x0, int y0, int kg0,
                          int boxbytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, boxbytes);
    tma_load_4d(smem, &tmap, &bar, 0, x0, y0, kg0);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < boxbytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(smem)[i];
}

static float h2f(__half h) { return __half2float(h); }

int main() {
  std::mt19937 rng(42);
  std::uniform_real_distribution<float> U(-1.f, 1.f);
  int fails = 0;
  // ---------------- (1)(2)(3) GEMM probes
  for (int amode = 0; amode < 2; ++amode)
    for (int bmode = 0; bmode < 2; ++bmode)
      for (int shift : {0, 1, 7, 131}) {
        if (amode == 1 && shift) continue;
        const int N = 64, K = 64;
        int mrows = amode == 0 ? 128 + 136 : 128;
        std::vector<__half> A((size_t)mrows * K), B((size_t)N * K);
        for (auto& v : A) v = __float2half(U(rng));
        for (auto& v : B) v = __float2half(U(rng));
        // reference uses logical A[m][k] (for MN-major, global stores A as [k][m])
        auto Aat = [&](int m, int k) { return amode == 0 ? h2f(A[(size_t)m * K + k]) : h2f(A[(size_t)k * mrows + m]); };
        auto Bat = [&](int n, int k) { return bmode == 0 ? h2f(B[(size_t)n * K + k]) : h2f(B[(size_t)k * N + n]); };
        __half *dA, *dB;
        float* dD;
        CK(cudaMalloc(&dA, A.size() * 2));
        CK(cudaMalloc(&dB, B.size() * 2));
        CK(cudaMalloc(&dD, 128 * N * 4));
        CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
        int smem = 64 * 1024 + 4096;
        CK(cudaFuncSetAttribute(probe_gemm<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        probe_gemm<N><<<1, 128, smem>>>(dA, dB, dD, K, amode, bmode, shift, mrows);
        CK(cudaDeviceSynchronize());
        std::vector<float> D(128 * N);
        CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
        double maxerr = 0;
        for (int m = 0; m < 128; ++m)
          for (int n = 0; n < N; ++n) {
            double r = 0;
            for (int k = 0; k < K; ++k) r += (double)Aat(m + shift, k) * Bat(n, k);
            maxerr = fmax(maxerr, fabs(r - D[m * N + n]));
          }
        bool ok = maxerr < 1e-3;
        fails += !ok;
        printf("gemm amode=%d bmode=%d shift=%d maxerr=%.3g %s\n", amode, bmode, shift, maxerr, ok ? "OK" : "FAIL");
        cudaFree(dA);
        cudaFree(dB);
        cudaFree(dD);
      }
  // ---------------- (5) accumulation rounding: A in [0.5,1], B = 1, long K
  {
    const int N = 64, K = 8192, mrows = 128;
    std::uniform_real_distribution<float> P(0.5f, 1.f);
    std::vector<__half> A((size_t)mrows * K), B((size_t)N * K);
    for (auto& v : A) v = __float2half(P(rng));
    for (auto& v : B) v = __float2half(1.0f);
    __half *dA, *dB;
    float* dD;
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dD, 128 * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    int smem = 64 * 1024 + 4096;
    probe_gemm<N><<<1, 128, smem>>>(dA, dB, dD, K, 0, 0, 0, mrows);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(128 * N);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double bias = 0, bias_rn = 0, mabs = 0;
    for (int m = 0; m < 128; ++m) {
      double exact = 0;
      float seq = 0.f;
      for (int k = 0; k < K; ++k) {
        exact += h2f(A[(size_t)m * K + k]);
        seq += h2f(A[(size_t)m * K + k]);
      }
      bias += (D[m * N] - exact) / exact;
      bias_rn += (seq - exact) / exact;
      mabs += fabs(D[m * N] - exact) / exact;
    }
    printf("accum K=%d: mean rel err tensor=%.3g (|.|=%.3g)  sequential-fp32-RN=%.3g\n", K, bias / 128, mabs / 128,
           bias_rn / 128);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  // ---------------- (4) TMA 4-D CHW8 box with OOB zero fill
  {
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    const int W = 200, H = 7, KG = 4;
    std::vector<uint16_t> T((size_t)KG * H * W * 8);
    for (size_t i = 0; i < T.size(); ++i) T[i] = (uint16_t)(i * 7 + 1);
    uint16_t* dT;
    CK(cudaMalloc(&dT, T.size() * 2));
    CK(cudaMemcpy(dT, T.data(), T.size() * 2, cudaMemcpyHostToDevice));
    CUtensorMap tm;
    cuuint64_t dims[4] = {8, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)KG};
    cuuint64_t strides[3] = {16, (cuuint64_t)W * 16, (cuuint64_t)H * W * 16};
    cuuint32_t box[4] = {8, 130, 4, 2};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, dT, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode result %d\n", (int)r);
    int boxbytes = 8 * 130 * 4 * 2 * 2;
    uint16_t* dout;
    CK(cudaMalloc(&dout, boxbytes));
    int x0 = 120, y0 = -1, kg0 = 3;  // kg 3,4 -> 4 is OOB
    CK(cudaFuncSetAttribute(probe_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, boxbytes + 1024));
    probe_tma<<<1, 128, boxbytes + 1024>>>(tm, dout, x0, y0, kg0, boxbytes);
    CK(cudaDeviceSynchronize());
    std::vector<uint16_t> out(boxbytes / 2);
    CK(cudaMemcpy(out.data(), dout, boxbytes, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int kg = 0; kg < 2; ++kg)
      for (int ry = 0; ry < 4; ++ry)
        for (int px = 0; px < 130; ++px)
          for (int e = 0; e < 8; ++e) {
            int gx = x0 + px, gy = y0 + ry, gk = kg0 + kg;
            uint16_t want = (gx >= 0 && gx < W && gy >= 0 && gy < H && gk < KG)
                                ? T[(((size_t)gk * H + gy) * W + gx) * 8 + e]
                                : 0;
            uint16_t got = out[(((size_t)kg * 4 + ry) * 130 + px) * 8 + e];
            bad += want != got;
          }
    printf("tma 4d box: %d mismatches %s\n", bad, bad ? "FAIL" : "OK");
    fails += bad != 0;
  }
  printf("PROBE %s\n", fails ? "FAILED" : "PASSED");
  return fails ? 1 : 0;
}
