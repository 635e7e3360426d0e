// mma_rate.cu — tcgen05.mma issue-rate microbenchmark (kind::f16, M=128 / M=256 pair).
// One CTA (or CTA pair) per SM, one thread issues R back-to-back MMAs into one TMEM accumulator,
// cycling the A start address over 9 row shifts like the conv's tap loop.  Optional concurrent
// 1-D bulk copies into a separate smem region model the TMA refill traffic of the real kernel.
// Reports cycles per MMA vs the math floor 128*N/256 (M=128) and the noise bytes/cycle.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mma_rate.cu -o tools/mma_rate -lcuda
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../paper_2212_13459_b200/csrc/sm100.cuh"

using namespace spst;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

enum { SS = 0, TS = 1, PAIR = 2, SSW = 3, TSW = 4, SSH = 5, TSH = 6 };  // *H: descriptors hoisted, unrolled x3  // *W: whole warp runs the loop, elect.sync issues
constexpr int ROWS = 256;            // A rows staged (shift window)
constexpr int A_BYTES = 2 * ROWS * 16;
constexpr int B_BYTES = 2 * (256 + 64) * 16;
constexpr int NOISE_CHUNK = 32768;

__device__ __forceinline__ void umma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_f16_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_f16_ts_elect(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// shift: 0 none, 1 A by 0..2 rows (16 B steps, the conv's dx taps), 2 A by 8-row steps (128 B),
// 3 B by 0..2 rows, 4 A by 0..2 rows and B by 8-row steps
template <int N, int MODE>
__global__ void __launch_bounds__(384, 1) rate_kernel(int R, const uint8_t* noise_src, long long* out_cycles,
                                                      long long* out_noise, int shift, int lsu, uint4* gdst) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + A_BYTES;
  uint8_t* sn = smem + A_BYTES + B_BYTES;
  __shared__ uint64_t done_bar, noise_bar;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (A_BYTES + B_BYTES) / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;  // fp16 1.0 pairs
  if (threadIdx.x == 0) {
    mbar_init(&done_bar, 1);
    mbar_init(&noise_bar, 1);
    stop = 0;
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if constexpr (MODE == PAIR)
      tmem_alloc_pair<512>(&tslot);
    else
      tmem_alloc<512>(&tslot);
  }
  tc_fence_before();
  if constexpr (MODE == PAIR)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  const bool leader = MODE != PAIR || cluster_ctarank() == 0;
  if ((MODE == SS || MODE == TS || MODE == PAIR) && warp == 0 && lane == 0 && leader) {
    const uint32_t idesc = make_idesc_f16(MODE == PAIR ? 256 : 128, N, 0, 0, 0);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const int NB = MODE == PAIR ? N / 2 : N;  // B rows held by this CTA
    const long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int sh = i % 3;
      const uint32_t ash = shift == 1 || shift == 4 ? sh : shift == 2 ? 8 * sh : 0;
      const uint32_t bsh = shift == 3 ? sh : shift == 4 ? 8 * sh : 0;
      const uint64_t adesc = make_sdesc(a0 + ash * 16, ROWS * 16, 128);
      const uint64_t bdesc = make_sdesc(b0 + bsh * 16, (NB + 64) * 16, 128);
      if constexpr (MODE == SS) umma_f16(tbase, adesc, bdesc, idesc, i > 0);
      if constexpr (MODE == TS) umma_f16_ts(tbase, tbase + 256, bdesc, idesc, i > 0);
      if constexpr (MODE == PAIR) umma_f16_pair(tbase, adesc, bdesc, idesc, i > 0);
    }
    if constexpr (MODE == PAIR)
      umma_commit_pair(&done_bar);
    else
      umma_commit(&done_bar);
    mbar_wait(&done_bar, 0);
    const long long t1 = clock64();
    out_cycles[blockIdx.x] = t1 - t0;
    stop = 1;
  } else if ((MODE == SSW || MODE == TSW) && warp == 0) {
    const uint32_t idesc = make_idesc_f16(128, N, 0, 0, 0);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int sh = i % 3;
      const uint32_t ash = shift == 1 || shift == 4 ? sh : shift == 2 ? 8 * sh : 0;
      const uint32_t bsh = shift == 3 ? sh : shift == 4 ? 8 * sh : 0;
      const uint64_t adesc = make_sdesc(a0 + ash * 16, ROWS * 16, 128);
      const uint64_t bdesc = make_sdesc(b0 + bsh * 16, (N + 64) * 16, 128);
      if constexpr (MODE == SSW) umma_f16_elect(tbase, adesc, bdesc, idesc, i > 0);
      if constexpr (MODE == TSW) umma_f16_ts_elect(tbase, tbase + 256, bdesc, idesc, i > 0);
    }
    if (lane == 0) {
      umma_commit(&done_bar);
      mbar_wait(&done_bar, 0);
      const long long t1 = clock64();
      out_cycles[blockIdx.x] = t1 - t0;
      stop = 1;
    }
    __syncwarp();
  } else if ((MODE == SSH || MODE == TSH) && warp == 0) {
    const uint32_t idesc = make_idesc_f16(128, N, 0, 0, 0);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
    const uint32_t s1 = shift == 1 || shift == 4 ? 1 : shift == 2 ? 8 : 0;
    const uint64_t ad0 = make_sdesc(a0, ROWS * 16, 128), ad1 = make_sdesc(a0 + s1 * 16, ROWS * 16, 128),
                   ad2 = make_sdesc(a0 + 2 * s1 * 16, ROWS * 16, 128);
    const uint32_t t1 = shift == 3 ? 1 : shift == 4 ? 8 : 0;
    const uint64_t bd0 = make_sdesc(b0, (N + 64) * 16, 128), bd1 = make_sdesc(b0 + t1 * 16, (N + 64) * 16, 128),
                   bd2 = make_sdesc(b0 + 2 * t1 * 16, (N + 64) * 16, 128);
    const long long t0 = clock64();
    for (int i = 0; i < R; i += 3) {
      if constexpr (MODE == SSH) {
        umma_f16_elect(tbase, ad0, bd0, idesc, 1u);
        umma_f16_elect(tbase, ad1, bd1, idesc, 1u);
        umma_f16_elect(tbase, ad2, bd2, idesc, 1u);
      } else {
        umma_f16_ts_elect(tbase, tbase + 256, bd0, idesc, 1u);
        umma_f16_ts_elect(tbase, tbase + 256, bd1, idesc, 1u);
        umma_f16_ts_elect(tbase, tbase + 256, bd2, idesc, 1u);
      }
    }
    if (lane == 0) {
      umma_commit(&done_bar);
      mbar_wait(&done_bar, 0);
      const long long t2 = clock64();
      out_cycles[blockIdx.x] = t2 - t0;
      stop = 1;
    }
    __syncwarp();
  } else if (MODE == PAIR && warp == 0 && lane == 0) {
    mbar_wait(&done_bar, 0);
    out_cycles[blockIdx.x] = 0;
    stop = 1;
  } else if (warp >= 2 && lsu) {
    // LSU noise: lsu=1 st.global.v4 (coalesced 512 B per warp), 2 ld.shared.v4, 3 local spills
    long long n = 0;
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    const size_t base = ((size_t)blockIdx.x * 320 + (threadIdx.x - 64)) ;
    const uint4* sh = reinterpret_cast<const uint4*>(sn);
    uint4 loc[24];
    for (int i = 0; i < 24; ++i) loc[i] = v;
    while (!stop) {
#pragma unroll 4
      for (int k = 0; k < 64; ++k) {
        if (lsu == 1) gdst[(base + (size_t)k * 148 * 320) & ((1u << 22) - 1)] = v;
        else if (lsu == 2) {
          uint4 t;
          asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(t.x), "=r"(t.y), "=r"(t.z), "=r"(t.w)
                       : "r"(smem_u32(sh + ((threadIdx.x * 7 + k * 32) & 2047))));
          v.x += t.x;
        }
        else { loc[(k + v.x) % 24].y += v.x; v.x += loc[(k * 5 + v.y) % 24].x; }
      }
      n += 64;
    }
    if (v.x == 12345u) out_noise[0] = v.y + loc[3].y;
    if (lane == 0 && warp == 2) out_noise[blockIdx.x] = n;
  } else if (warp == 1 && lane == 0 && noise_src) {
    long long bytes = 0;
    uint32_t ph = 0;
    const uint8_t* src = noise_src + (size_t)(blockIdx.x % 64) * 2 * NOISE_CHUNK;
    while (!stop) {
      mbar_arrive_expect_tx(&noise_bar, 2 * NOISE_CHUNK);
      bulk_load(sn, src, NOISE_CHUNK, &noise_bar);
      bulk_load(sn + NOISE_CHUNK, src + NOISE_CHUNK, NOISE_CHUNK, &noise_bar);
      mbar_wait(&noise_bar, ph);
      ph ^= 1;
      bytes += 2 * NOISE_CHUNK;
    }
    out_noise[blockIdx.x] = bytes;
  }
  tc_fence_before();
  if constexpr (MODE == PAIR)
    cluster_sync_all();
  else
    __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if constexpr (MODE == PAIR)
      tmem_dealloc_pair<512>(tbase);
    else
      tmem_dealloc<512>(tbase);
  }
}

static uint4* g_dst = nullptr;
template <int N, int MODE>
void run(int R, bool noise, const uint8_t* nsrc, int shift, int lsu = 0) {
  auto k = rate_kernel<N, MODE>;
  const int smem = A_BYTES + B_BYTES + 2 * NOISE_CHUNK + 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int grid = 148;
  long long *cyc, *nb;
  CK(cudaMalloc(&cyc, grid * 8));
  CK(cudaMalloc(&nb, grid * 8));
  CK(cudaMemset(cyc, 0, grid * 8));
  CK(cudaMemset(nb, 0, grid * 8));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(lsu ? 384 : 128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = MODE == PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) CK(cudaLaunchKernelEx(&cfg, k, R, noise ? nsrc : nullptr, cyc, nb, shift, lsu, g_dst));
  CK(cudaDeviceSynchronize());
  std::vector<long long> hc(grid), hn(grid);
  CK(cudaMemcpy(hc.data(), cyc, grid * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hn.data(), nb, grid * 8, cudaMemcpyDeviceToHost));
  long long mx = 0, nsum = 0;
  int cnt = 0;
  for (int i = 0; i < grid; ++i) {
    mx = std::max(mx, hc[i]);
    if (hc[i]) {
      nsum += hn[i];
      ++cnt;
    }
  }
  const double per = (double)mx / R;
  const double floor_c = (MODE == PAIR ? 256.0 : 128.0) * N / (256.0 * (MODE == PAIR ? 2 : 1));
  const double smem_rd = MODE == TS || MODE == TSW || MODE == TSH ? N * 32.0 : (MODE == PAIR ? 128 * 32.0 + N / 2 * 32.0 : 128 * 32.0 + N * 32.0);
  printf("lsu=%d shift=%d %-5s N=%3d noise=%d: %7.1f cyc/MMA (math floor %5.1f, eff %5.1f%%), operand smem bytes/MMA %6.0f -> %5.1f B/cyc, noise %5.1f B/cyc\n",
         lsu, shift, MODE == SS ? "SS" : MODE == TS ? "TS" : MODE == SSW ? "SSW" : MODE == TSW ? "TSW" : MODE == SSH ? "SSH" : MODE == TSH ? "TSH" : "PAIR", N, (int)noise, per, floor_c, 100.0 * floor_c / per, smem_rd,
         smem_rd / per, noise ? (double)nsum / cnt / mx : 0.0);
  fflush(stdout);
  CK(cudaFree(cyc));
  CK(cudaFree(nb));
}

int main() {
  uint8_t* nsrc;
  CK(cudaMalloc(&nsrc, 64 * 2 * NOISE_CHUNK));
  CK(cudaMemset(nsrc, 0, 64 * 2 * NOISE_CHUNK));
  const int R = 1 << 15;
  const int RR = 3 * (1 << 13);
  CK(cudaMalloc(&g_dst, (size_t)16 << 22));
  for (int lsu = 0; lsu < 4; ++lsu) {
    run<128, SSH>(RR, false, nsrc, 1, lsu);
    run<64, SSH>(RR, false, nsrc, 1, lsu);
    run<128, TSH>(RR, false, nsrc, 1, lsu);
  }
  printf("ok\n");
  return 0;
}
