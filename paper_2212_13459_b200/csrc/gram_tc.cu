// gram_tc.cu — tcgen05 Gram partials S = sum_p F_p F_p^T of a tap tensor (reference
// stats.py:43-50 StatsAccumulator.accumulate, `flat @ flat.T` in f64).
//
// The tap tensor is stored HL16 ([kg][P][8] fp16 hi/lo planes), which is exactly the
// MN-major SWIZZLE_NONE operand layout (8 channels contiguous, pixels at 16 B stride), so the
// same TMA box feeds both the A (channel tile c1) and the B (channel tile c2) operand.
// A CTA owns one upper-triangle (c1, c2) tile pair and a pixel split of at most
// `px_per_split` pixels; its fp32 TMEM accumulator therefore never sums more than that many
// terms, and splits are combined in f64 in a fixed order (gram_reduce), so the result is
// deterministic and independent of the launch geometry.
#include "common.cuh"
#include "sm100.cuh"

namespace spst {

struct GramCfg {
  static constexpr int KPX = 64;                       // pixels per stage
  static constexpr int T_BYTES = 16 * KPX * 16;        // 128 channels x 64 px fp16 (16 KB)
  static constexpr int STAGE = 4 * T_BYTES;            // A hi/lo + B hi/lo
  static constexpr int STAGES = 3;
  static constexpr int SMEM = STAGES * STAGE + 1024;
};

__global__ void __launch_bounds__(192, 1) gram_tc_kernel(const __grid_constant__ GramArgs a) {
  using C = GramCfg;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[C::STAGES], empty_bar[C::STAGES], done_bar;
  __shared__ uint32_t tmem_slot;
  const uint32_t warp = warp_id(), lane = lane_id();

  // decode the upper-triangle pair index
  int pair = blockIdx.y, c1 = 0;
  while (pair >= a.n_ctile - c1) {
    pair -= a.n_ctile - c1;
    ++c1;
  }
  const int c2 = c1 + pair;
  const bool diag = c1 == c2;
  const long long p0 = a.p_begin + (long long)blockIdx.x * a.px_per_split;
  const long long p1 = min(p0 + a.px_per_split, a.p_end);
  const int n_chunks = (int)((p1 - p0 + C::KPX - 1) / C::KPX);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.tm_hi);
    tma_prefetch_desc(&a.tm_lo);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<128>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = (diag ? 2 : 4) * C::T_BYTES;
      for (int c = 0; c < n_chunks; ++c) {
        const int s = c % C::STAGES;
        mbar_wait(&empty_bar[s], ((c / C::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * C::STAGE;
        mbar_arrive_expect_tx(&full_bar[s], bytes);
        // coordinates relative to the map base (which starts at p_begin)
        const int px = (int)(p0 - a.p_begin) + c * C::KPX;
        tma_load_3d(st, &a.tm_hi, &full_bar[s], 0, px, 16 * c1);
        tma_load_3d(st + C::T_BYTES, &a.tm_lo, &full_bar[s], 0, px, 16 * c1);
        if (!diag) {
          tma_load_3d(st + 2 * C::T_BYTES, &a.tm_hi, &full_bar[s], 0, px, 16 * c2);
          tma_load_3d(st + 3 * C::T_BYTES, &a.tm_lo, &full_bar[s], 0, px, 16 * c2);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc_f16(128, 128, 0, 1, 1);
      for (int c = 0; c < n_chunks; ++c) {
        const int s = c % C::STAGES;
        mbar_wait(&full_bar[s], (c / C::STAGES) & 1);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * C::STAGE);
        const uint32_t ah = st, al = st + C::T_BYTES;
        const uint32_t bh = diag ? ah : st + 2 * C::T_BYTES, bl = diag ? al : st + 3 * C::T_BYTES;
#pragma unroll
        for (int k = 0; k < C::KPX / 16; ++k) {
          const uint32_t off = k * 256;  // 16 px = two 8-px core-matrix groups of 128 B
          const uint64_t dah = make_sdesc(ah + off, 128, C::KPX * 16);
          const uint64_t dal = make_sdesc(al + off, 128, C::KPX * 16);
          const uint64_t dbh = make_sdesc(bh + off, 128, C::KPX * 16);
          const uint64_t dbl = make_sdesc(bl + off, 128, C::KPX * 16);
          umma_f16(tmem, dah, dbh, idesc, (c > 0 || k > 0) ? 1u : 0u);
          umma_f16(tmem, dah, dbl, idesc, 1u);
          umma_f16(tmem, dal, dbh, idesc, 1u);
        }
        umma_commit(&empty_bar[s]);
      }
      umma_commit(&done_bar);
    }
  } else {
    const uint32_t q = warp & 3;
    mbar_wait(&done_bar, 0);
    tc_fence_after();
    const int pairs = a.n_ctile * (a.n_ctile + 1) / 2;
    float* dst = a.partial + (((size_t)blockIdx.x * pairs + blockIdx.y) * 128 + q * 32 + lane) * 128;
    for (int cb = 0; cb < 4; ++cb) {
      float v[32];
      if (n_chunks > 0) {
        tmem_ld32(tmem + ((q * 32u) << 16) + cb * 32, v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(dst + cb * 32 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<128>(tmem);
}

// S[c1][c2] (f64, C x C) = sum over splits of the fp32 partial tiles, fixed split order.
__global__ void gram_reduce_kernel(const float* partial, int n_splits, int n_ctile, int C, double inv_scale2,
                                   double* S) {
  const int i = blockIdx.y;  // row channel
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C || j >= C || j < i) return;
  const int t1 = i / 128, t2 = j / 128;
  const int pair = t1 * n_ctile - t1 * (t1 - 1) / 2 + (t2 - t1);
  const int pairs = n_ctile * (n_ctile + 1) / 2;
  double acc = 0.0;
  for (int s = 0; s < n_splits; ++s)
    acc += (double)partial[(((size_t)s * pairs + pair) * 128 + (i & 127)) * 128 + (j & 127)];
  acc *= inv_scale2;
  S[(size_t)i * C + j] = acc;
  S[(size_t)j * C + i] = acc;
}

int gram_tc_smem_bytes() { return GramCfg::SMEM; }

cudaError_t launch_gram_tc(const GramArgs& a, int n_splits, cudaStream_t stream) {
  cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, GramCfg::SMEM);
  dim3 grid(n_splits, a.n_ctile * (a.n_ctile + 1) / 2);
  gram_tc_kernel<<<grid, 192, GramCfg::SMEM, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gram_reduce(const float* partial, int n_splits, int n_ctile, int C, double inv_scale2,
                               double* S, cudaStream_t stream) {
  dim3 grid((C + 127) / 128, C);
  gram_reduce_kernel<<<grid, 128, 0, stream>>>(partial, n_splits, n_ctile, C, inv_scale2, S);
  return cudaGetLastError();
}

}  // namespace spst
