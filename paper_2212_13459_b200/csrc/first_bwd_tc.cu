// first_bwd_tc.cu — adjoint of the first conv + preprocess on tcgen05 (reference extractor.py
// 200-214 through tensorops.py:58-74 conv2d_backward_input for C_in = 3, and the
// preprocess_backward of extractor.py:158-164).
//
// g_in[y][x][c] = sum_{k,dy,dx} g0[k][y+1-dy][x+1-dx] W[k][c][dy][dx] has only 3 outputs per
// pixel, so it is computed with the taps folded into N instead of into K:
//   out27[p][(c,dy,dx)] = sum_k g0[p][k] W[k][c][dy][dx]        (M = 128 px, N = 32, K = 64)
// an unshifted GEMM per image row, followed by a 3x3 gather of out27 in the epilogue:
//   g_in(y, x, c) = sum_{dy,dx} out27[y+1-dy][x+1-dx][(c,dy,dx)].
// Tile: 6 output rows x 126 output px, computed over 8 rows x 128 px (the halo).  Each epilogue
// lane (one computed column) folds the dy terms of its own column per dx; the dx gather is a
// +-1-lane exchange (shuffles, shared memory across warp edges).
//
// Numerics as the conv kernel: g0 fp16 hi/lo x W fp16 hi/lo, 3 passes (hi*lo, lo*hi, hi*hi),
// a fresh TMEM slice per row (12 accumulation steps), fp32 epilogue.
#include <algorithm>

#include "common.cuh"
#include "sm100.cuh"

namespace spst {

namespace {
constexpr int kRows = 8;                  // computed rows per tile (6 outputs + 2 halo)
constexpr int kOutRows = kRows - 2;
constexpr int kOutCols = 126;             // output columns per tile (128 computed - 2 halo)
constexpr int kPlane = 128 * 16;          // one 8-channel plane of a 128-px row (2 KB)
constexpr int kRowBytes = 8 * kPlane;     // 64 channels of one row, hi or lo (16 KB)
constexpr int kStage = 2 * kRowBytes;     // hi + lo (32 KB)
constexpr int kStages = 4;
constexpr int kBBytes = 2 * 8 * 32 * 16;  // hi/lo x 8 k-groups x 32 n x 8 k (8 KB)
constexpr int kSmem = kStages * kStage + kBBytes + 1024;
constexpr int kBuf = 2;                   // TMEM tile buffers (8 rows x 32 columns each)
}  // namespace

__global__ void __launch_bounds__(192, 1) first_bwd_tc_kernel(const __grid_constant__ FirstBwdTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sB = smem + kStages * kStage;
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], b_bar, cfull_bar[kBuf], cempty_bar[kBuf];
  __shared__ uint32_t tmem_slot;
  __shared__ float edge[4][2][kOutRows * 3];  // per warp: lane 0's S[dx=0] and lane 31's S[dx=2]

  const uint32_t warp = warp_id(), lane = lane_id();
  const int tiles_x = (a.W + kOutCols - 1) / kOutCols, tiles_y = (a.H + kOutRows - 1) / kOutRows;
  const int n_tiles = tiles_x * tiles_y;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.tm_hi);
    tma_prefetch_desc(&a.tm_lo);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&b_bar, 1);
    for (int b = 0; b < kBuf; ++b) {
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
    if (lane == 0) {  // ----------------------------------------------------- TMA producer
      mbar_arrive_expect_tx(&b_bar, kBBytes);
      bulk_load(sB, a.wslab, kBBytes, &b_bar);
      uint32_t g = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int x0 = (t % tiles_x) * kOutCols, y0 = (t / tiles_x) * kOutRows;
        for (int q = 0; q < kRows; ++q, ++g) {
          const int s = g % kStages;
          mbar_wait(&empty_bar[s], ((g / kStages) & 1) ^ 1);
          uint8_t* st = smem + s * kStage;
          mbar_arrive_expect_tx(&full_bar[s], kStage);
          // u64 view (2W, H, 8): 128 px x 8 planes from column x0-1, row y0-1+q (OOB -> zero)
          tma_load_3d(st, &a.tm_hi, &full_bar[s], 2 * (x0 - 1), y0 - 1 + q, 0);
          tma_load_3d(st + kRowBytes, &a.tm_lo, &full_bar[s], 2 * (x0 - 1), y0 - 1 + q, 0);
        }
      }
    }
  } else if (warp == 1) {  // ----------------------------------------------- MMA issuer (warp-wide)
    const uint32_t idesc = make_idesc_f16(128, 32, 0, 0, 0);
    mbar_wait(&b_bar, 0);
    const uint64_t bhi = make_sdesc(smem_u32(sB), 32 * 16, 128);
    const uint64_t blo = make_sdesc(smem_u32(sB) + kBBytes / 2, 32 * 16, 128);
    uint32_t g = 0, tcount = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tcount) {
      const uint32_t b = tcount % kBuf;
      mbar_wait(&cempty_bar[b], ((tcount / kBuf) & 1) ^ 1);
      __syncwarp();
      for (int q = 0; q < kRows; ++q, ++g) {
        const int s = g % kStages;
        mbar_wait(&full_bar[s], (g / kStages) & 1);
        __syncwarp();
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * kStage);
        const uint64_t ahi = make_sdesc(st, kPlane, 128), alo = make_sdesc(st + kRowBytes, kPlane, 128);
        const uint32_t d = tmem + b * 256 + q * 32;
#pragma unroll
        for (int pass = 0; pass < 3; ++pass)  // corrections first (see conv_tc.cu)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ad = (pass == 1 ? alo : ahi) + (uint64_t)((ks * 2 * kPlane) >> 4);
            const uint64_t bd = (pass == 0 ? blo : bhi) + (uint64_t)((ks * 2 * 32 * 16) >> 4);
            umma_f16_ws(d, ad, bd, idesc, (pass | ks) ? 1u : 0u);
          }
        umma_commit_ws(&empty_bar[s]);
      }
      umma_commit_ws(&cfull_bar[b]);
    }
  } else {  // ------------------------------------------------------------- epilogue (4 warps)
    const uint32_t q4 = warp & 3;  // TMEM lane quarter = 32 computed columns
    const int L = (int)(q4 * 32 + lane);
    uint32_t tcount = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tcount) {
      const int x0 = (t % tiles_x) * kOutCols, y0 = (t / tiles_x) * kOutRows;
      const uint32_t b = tcount % kBuf;
      mbar_wait(&cfull_bar[b], (tcount / kBuf) & 1);
      tc_fence_after();
      // S[dx][r][c] = sum_dy out27[row r + 2 - dy][own column][(c, dy, dx)]
      float S[3][kOutRows][3];
#pragma unroll
      for (int i = 0; i < 3 * kOutRows * 3; ++i) (&S[0][0][0])[i] = 0.f;
#pragma unroll
      for (int q = 0; q < kRows; ++q) {
        float v[32];
        tmem_ld32(tmem + ((q4 * 32u) << 16) + b * 256 + q * 32, v);
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
          const int r = q + dy - 2;
          if (r < 0 || r >= kOutRows) continue;
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) S[dx][r][c] += v[c * 9 + dy * 3 + dx];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&cempty_bar[b]);
      // dx gather: out(L) = S0(L+1) + S1(L) + S2(L-1); warp edges through shared memory
      if (lane == 0 || lane == 31) {
#pragma unroll
        for (int r = 0; r < kOutRows; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c) edge[q4][lane == 31][r * 3 + c] = lane == 0 ? S[0][r][c] : S[2][r][c];
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
      const int xo = L - 1, x = x0 + xo;
#pragma unroll
      for (int r = 0; r < kOutRows; ++r) {
        float o[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float right = __shfl_down_sync(0xffffffffu, S[0][r][c], 1);
          float left = __shfl_up_sync(0xffffffffu, S[2][r][c], 1);
          if (lane == 31) right = q4 < 3 ? edge[q4 + 1][0][r * 3 + c] : 0.f;
          if (lane == 0) left = q4 > 0 ? edge[q4 - 1][1][r * 3 + c] : 0.f;
          o[c] = (right + S[1][r][c] + left) * a.acc_scale;
        }
        const int y = y0 + r;
        if (xo >= 0 && xo < kOutCols && x < a.W && y < a.H) {
          float* dst = a.gimg + ((size_t)y * a.W + x) * 3;
#pragma unroll
          for (int c = 0; c < 3; ++c) dst[a.perm[c]] = o[c] / a.scale[c];
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // edge[] is rewritten by the next tile
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

cudaError_t launch_first_bwd_tc(const FirstBwdTcArgs& a, cudaStream_t st) {
  cudaFuncSetAttribute(first_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  const int tiles = ((a.W + kOutCols - 1) / kOutCols) * ((a.H + kOutRows - 1) / kOutRows);
  note_launch(), first_bwd_tc_kernel<<<std::min(tiles, kSMs), 192, kSmem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace spst
