// gram_tc.cu — tcgen05 Gram partials S = sum_p F_p F_p^T of a tap tensor (reference
// stats.py:43-50 StatsAccumulator.accumulate, `flat @ flat.T` in f64).
//
// The tap tensor is stored HL16 ([kg][P][8] fp16 hi/lo planes), which is exactly the
// MN-major SWIZZLE_NONE operand layout (8 channels contiguous, pixels at 16 B stride), so the
// same TMA box feeds both the A (channel tile c1) and the B (channel tile c2) operand.
// A CTA owns one upper-triangle (c1, c2) tile pair and a split of at most `px_per_split`
// pixels of the owned rectangle (row-major runs of KPX pixels); its fp32 TMEM accumulator therefore never sums more than that many
// terms, and splits are combined in f64 in a fixed order (gram_reduce), so the result is
// deterministic and independent of the launch geometry.
#include "common.cuh"
#include "sm100.cuh"

namespace spst {

struct GramCfg {
  static constexpr int KPX = 64;                       // pixels per smem stage
  static constexpr int T_BYTES = 16 * KPX * 16;        // 128 channels x 64 px fp16 (16 KB)
  static constexpr int STAGE = 4 * T_BYTES;            // A hi/lo + B hi/lo
  static constexpr int STAGES = 3;
  static constexpr int DRAIN = 2;                      // stages per TMEM accumulator (128 px)
  static constexpr int NBUF = 4;                       // 4 x 128 TMEM columns
  static constexpr int SMEM = STAGES * STAGE + 1024;
};

// The tensor core sums at most DRAIN*KPX pixels into one fresh TMEM accumulator; the 4
// epilogue warps (one row of the 128x128 tile per thread) drain every accumulator into fp32
// registers with round-to-nearest adds, so the partial is accurate to ~fp32 regardless of
// how many pixels a CTA covers.
__global__ void __launch_bounds__(192, 1) gram_tc_kernel(const __grid_constant__ GramArgs a) {
  using C = GramCfg;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[C::STAGES], empty_bar[C::STAGES], cfull_bar[C::NBUF], cempty_bar[C::NBUF];
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
  // stage g of the owned rectangle = (row g / xblocks, KPX-pixel block g % xblocks)
  const int xblocks = (a.w_own + C::KPX - 1) / C::KPX;
  const long long total = (long long)a.rows * xblocks;
  const long long g0 = (long long)blockIdx.x * (a.px_per_split / C::KPX);
  const long long g1 = min(g0 + a.px_per_split / C::KPX, total);
  const int n_stages = g1 > g0 ? (int)(g1 - g0) : 0;
  const int n_drains = (n_stages + C::DRAIN - 1) / C::DRAIN;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.tm_hi);
    tma_prefetch_desc(&a.tm_lo);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(&cfull_bar[b], 1);
      mbar_init(&cempty_bar[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = (diag ? 2 : 4) * C::T_BYTES;
      for (int c = 0; c < n_stages; ++c) {
        const int s = c % C::STAGES;
        mbar_wait(&empty_bar[s], ((c / C::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * C::STAGE;
        mbar_arrive_expect_tx(&full_bar[s], bytes);
        const long long gs = g0 + c;
        const int row = (int)(gs / xblocks), px = (int)(gs % xblocks) * C::KPX;
        tma_load_3d(st, &a.tm_hi, &full_bar[s], 2 * px, row, 16 * c1);  // u64 view: 64 px = 128 elements
        tma_load_3d(st + C::T_BYTES, &a.tm_lo, &full_bar[s], 2 * px, row, 16 * c1);
        if (!diag) {
          tma_load_3d(st + 2 * C::T_BYTES, &a.tm_hi, &full_bar[s], 2 * px, row, 16 * c2);
          tma_load_3d(st + 3 * C::T_BYTES, &a.tm_lo, &full_bar[s], 2 * px, row, 16 * c2);
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp, one elected lane issues (umma_f16_ws)
      const uint32_t idesc = make_idesc_f16(128, 128, 0, 1, 1);
      for (int c = 0; c < n_stages; ++c) {
        const int dr = c / C::DRAIN;
        const uint32_t b = dr % C::NBUF;
        if (c % C::DRAIN == 0) mbar_wait(&cempty_bar[b], ((dr / C::NBUF) & 1) ^ 1);
        const int s = c % C::STAGES;
        mbar_wait(&full_bar[s], (c / C::STAGES) & 1);
        __syncwarp();
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * C::STAGE);
        const uint32_t ah = st, al = st + C::T_BYTES;
        const uint32_t bh = diag ? ah : st + 2 * C::T_BYTES, bl = diag ? al : st + 3 * C::T_BYTES;
        const uint32_t d = tmem + b * 128;
        // correction passes before the hi*hi pass (see conv_tc.cu)
#pragma unroll
        for (int pass = 0; pass < 3; ++pass)
#pragma unroll
          for (int k = 0; k < C::KPX / 16; ++k) {
            const uint32_t off = k * 256;  // 16 px = two 8-px core-matrix groups of 128 B
            const uint64_t da = make_sdesc((pass == 1 ? al : ah) + off, 128, C::KPX * 16);
            const uint64_t db = make_sdesc((pass == 0 ? bl : bh) + off, 128, C::KPX * 16);
            umma_f16_ws(d, da, db, idesc, (c % C::DRAIN > 0 || pass > 0 || k > 0) ? 1u : 0u);
          }
        umma_commit_ws(&empty_bar[s]);
        if (c % C::DRAIN == C::DRAIN - 1 || c == n_stages - 1) umma_commit_ws(&cfull_bar[b]);
      }
    }
  } else {
    const uint32_t q = warp & 3;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.f;
    for (int dr = 0; dr < n_drains; ++dr) {
      const uint32_t b = dr % C::NBUF;
      mbar_wait(&cfull_bar[b], (dr / C::NBUF) & 1);
      tc_fence_after();
      // undo the expected round-toward-zero bias of this accumulator (conv_tc.cu)
      const float cm = a.comp[min(C::DRAIN, n_stages - dr * C::DRAIN) - 1];
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        float v[32];
        tmem_ld32(tmem + ((q * 32u) << 16) + b * 128 + cb * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[cb * 32 + j] = fmaf(v[j], cm, acc[cb * 32 + j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty_bar[b]);
    }
    {  // common part of the round-toward-zero compensation (diagonal entries: same-sign sums)
      const int r = q * 32 + lane;
#pragma unroll
      for (int j = 0; j < 128; ++j) acc[j] = fmaf(acc[j], (diag && j == r) ? a.fine_diag : a.fine_off, acc[j]);
    }
    const int pairs = a.n_ctile * (a.n_ctile + 1) / 2;
    float* dst = a.partial + (((size_t)blockIdx.x * pairs + blockIdx.y) * 128 + q * 32 + lane) * 128;
#pragma unroll
    for (int j = 0; j < 128; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------------------------------
// C_p = 64 variant.  A = [V_hi ; V_lo] stacked along M (rows 0-63 hi channels, 64-127 lo
// channels: the lo planes sit right after the hi planes in smem at the same plane stride, so
// one MN-major descriptor spans both), B = V_hi (acc1) or V_lo (acc2), N = 64.  Then
//   rows 0-63  of acc1 = hi.hi, rows 64-127 of acc1 = lo.hi, rows 0-63 of acc2 = hi.lo
// and G = acc1[r] + acc1[64+r] + acc2[r] (lo.lo dropped), i.e. two M128xN64 MMAs per K-step
// instead of three M128xN128 ones on a half-empty tile.
struct Gram64Cfg {
  static constexpr int KPX = 128;                      // pixels per stage (one 2 KB TMA row per plane)
  static constexpr int PLANE = KPX * 16;               // one 8-channel plane (2 KB)
  static constexpr int STAGE = 16 * PLANE;             // 8 hi + 8 lo planes (32 KB)
  static constexpr int STAGES = 6;
  static constexpr int DRAIN = 2;                      // stages per TMEM accumulator (256 px)
  static constexpr int NBUF = 4;                       // 4 x (acc1 64 + acc2 64) TMEM columns
  static constexpr int SMEM = STAGES * STAGE + 1024;
};

__global__ void __launch_bounds__(192, 1) gram64_tc_kernel(const __grid_constant__ GramArgs a) {
  using C = Gram64Cfg;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[C::STAGES], empty_bar[C::STAGES], cfull_bar[C::NBUF], cempty_bar[C::NBUF];
  __shared__ uint32_t tmem_slot;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int xblocks = (a.w_own + C::KPX - 1) / C::KPX;
  const long long total = (long long)a.rows * xblocks;
  const long long g0 = (long long)blockIdx.x * (a.px_per_split / C::KPX);
  const long long g1 = min(g0 + a.px_per_split / C::KPX, total);
  const int n_stages = g1 > g0 ? (int)(g1 - g0) : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.tm_hi);
    tma_prefetch_desc(&a.tm_lo);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(&cfull_bar[b], 1);
      mbar_init(&cempty_bar[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int c = 0; c < n_stages; ++c) {
        const int s = c % C::STAGES;
        mbar_wait(&empty_bar[s], ((c / C::STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * C::STAGE;
        mbar_arrive_expect_tx(&full_bar[s], C::STAGE);
        const long long gs = g0 + c;
        const int row = (int)(gs / xblocks), px = (int)(gs % xblocks) * C::KPX;
        tma_load_3d(st, &a.tm_hi, &full_bar[s], 2 * px, row, 0);  // u64 view: 128 px = 256 elements
        tma_load_3d(st + 8 * C::PLANE, &a.tm_lo, &full_bar[s], 2 * px, row, 0);
      }
    }
  } else if (warp == 1) {
    {  // whole warp, one elected lane issues (umma_f16_ws)
      const uint32_t idesc = make_idesc_f16(128, 64, 0, 1, 1);
      for (int c = 0; c < n_stages; ++c) {
        const int dr = c / C::DRAIN;
        const uint32_t b = dr % C::NBUF;
        if (c % C::DRAIN == 0) mbar_wait(&cempty_bar[b], ((dr / C::NBUF) & 1) ^ 1);
        const int s = c % C::STAGES;
        mbar_wait(&full_bar[s], (c / C::STAGES) & 1);
        __syncwarp();
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * C::STAGE);
        const uint64_t da0 = make_sdesc(st, 128, C::PLANE);                // [hi;lo] x 16 px
        const uint64_t dh0 = make_sdesc(st, 128, C::PLANE);                // hi, N = 64
        const uint64_t dl0 = make_sdesc(st + 8 * C::PLANE, 128, C::PLANE); // lo, N = 64
        const uint32_t d1 = tmem + b * 128, d2 = d1 + 64;
#pragma unroll 4
        for (int k = 0; k < C::KPX / 16; ++k) {
          const uint64_t off = (uint64_t)((k * 256) >> 4);  // 16 px = two 128-B core-matrix groups
          const uint32_t acc = (c % C::DRAIN > 0 || k > 0) ? 1u : 0u;
          umma_f16_ws(d2, da0 + off, dl0 + off, idesc, acc);  // small (x lo) first
          umma_f16_ws(d1, da0 + off, dh0 + off, idesc, acc);
        }
        umma_commit_ws(&empty_bar[s]);
        if (c % C::DRAIN == C::DRAIN - 1 || c == n_stages - 1) umma_commit_ws(&cfull_bar[b]);
      }
    }
  } else {
    const uint32_t q = warp & 3;
    const int row = q * 32 + lane;  // 0-63: hi rows, 64-127: lo rows
    float acc[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) acc[i] = 0.f;
    const int n_drains = (n_stages + C::DRAIN - 1) / C::DRAIN;
    for (int c = 0; c < n_drains; ++c) {
      const uint32_t b = c % C::NBUF;
      mbar_wait(&cfull_bar[b], (c / C::NBUF) & 1);
      tc_fence_after();
      const uint32_t ta = tmem + ((q * 32u) << 16) + b * 128;
      // rows 0-63 of acc1 hold the hi*hi sums: undo their expected round-toward-zero bias
      const float cm = row < 64 ? a.comp[min(C::DRAIN, n_stages - c * C::DRAIN) - 1] : 1.f;
      float v0[32], v1[32];
      tmem_ld32x2(ta, ta + 32, v0, v1);  // acc1 (x hi)
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        acc[j] = fmaf(v0[j], cm, acc[j]);
        acc[32 + j] = fmaf(v1[j], cm, acc[32 + j]);
      }
      if (row < 64) {  // acc2 (x lo) only matters for the hi rows
        tmem_ld32x2(ta + 64, ta + 96, v0, v1);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          acc[j] += v0[j];
          acc[32 + j] += v1[j];
        }
      } else {
        __syncwarp();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty_bar[b]);
    }
    if (row < 64) {  // common part of the round-toward-zero compensation of the hi*hi sums
#pragma unroll
      for (int j = 0; j < 64; ++j) acc[j] = fmaf(acc[j], j == row ? a.fine_diag : a.fine_off, acc[j]);
    }
    float* dst = a.partial + ((size_t)blockIdx.x * 128 + row) * 64;
#pragma unroll
    for (int j = 0; j < 64; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// G[i][j] = sum over splits of partial rows i (hi.hi + hi.lo) and 64 + i (lo.hi), fixed order
__global__ void gram64_reduce_kernel(const float* partial, int n_splits, int C, double inv_scale2, double* S) {
  const int i = blockIdx.x, j = threadIdx.x;
  if (i >= C || j >= C || j < i) return;  // upper triangle, mirrored: S is exactly symmetric
  double acc = 0.0;
  for (int s = 0; s < n_splits; ++s)
    acc += (double)partial[((size_t)s * 128 + i) * 64 + j] + (double)partial[((size_t)s * 128 + 64 + i) * 64 + j];
  S[(size_t)i * C + j] = acc * inv_scale2;
  S[(size_t)j * C + i] = acc * inv_scale2;
}

cudaError_t launch_gram64_tc(const GramArgs& a, int n_splits, int C, double inv_scale2, double* S,
                             cudaStream_t stream) {
  cudaFuncSetAttribute(gram64_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Gram64Cfg::SMEM);
  note_launch(), gram64_tc_kernel<<<n_splits, 192, Gram64Cfg::SMEM, stream>>>(a);
  note_launch(), gram64_reduce_kernel<<<C, 64, 0, stream>>>(a.partial, n_splits, C, inv_scale2, S);
  return cudaGetLastError();
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
  note_launch(), gram_tc_kernel<<<grid, 192, GramCfg::SMEM, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_gram_reduce(const float* partial, int n_splits, int n_ctile, int C, double inv_scale2,
                               double* S, cudaStream_t stream) {
  dim3 grid((C + 127) / 128, C);
  note_launch(), gram_reduce_kernel<<<grid, 128, 0, stream>>>(partial, n_splits, n_ctile, C, inv_scale2, S);
  return cudaGetLastError();
}

}  // namespace spst
