// conv_tc.cu — tcgen05/TMEM implicit-GEMM 3x3 convolution for sm_100a.
//
// One kernel serves the forward pass (reference tensorops.py:33-55 conv2d_forward fused with
// relu_forward 81-82, avgpool_forward 99-101 and the relu mask needed by relu_backward 85-88)
// and the input-gradient pass (tensorops.py:58-74 conv2d_backward_input, run as a forward
// conv with transposed, flipped weights, fused with relu_backward, avgpool_backward 104-110,
// the tap-gradient injection of extractor.py:200-214 and the style/content feature gradients
// of stats.py:127-174 — the style gradient V*M enters as extra K-steps).
//
// GEMM view: M = output pixels (a CTA tile is 2 rows x 128 px = two M=128 accumulators),
// N = output channels (64/128 per tile), K = 9 taps x input channels.
//
// Numerics ("fp16x3 + compensated register accumulation"): operands are fp16 hi/lo pairs with
// power-of-two tensor scales; each 16-channel K-chunk issues hi*lo + lo*hi + hi*hi over the 9
// taps into a FRESH TMEM accumulator shared by at most D chunks (ConvArgs::drain: 1 in the
// forward, whose ReLU signs must be fp32-class, 2 in the backward), and the epilogue warps
// drain it into fp32 registers (round-to-nearest adds), multiplying out the expected
// round-toward-zero shrink of the tensor core's accumulation (comp[] / fine, see below and
// DESIGN.md §5).  The tensor core never carries a long running sum.
//
// Warp roles (320 threads, persistent over output tiles, one CTA per SM):
//   warp 0      TMA producer: per K-chunk the 4-row halo window of hi and lo activations as
//               32 u64-view strips of 68 px (one per lane; OOB zero fill = conv zero padding)
//               + the 9-tap weight slab (one 1-D bulk copy)
//   warp 1      MMA issuer: the whole warp runs the loop (descriptors stay in uniform
//               registers), one elected lane issues 9 taps x 2 rows x 3 passes per chunk
//               (64-channel layers: row-pair MMAs, see the N == 64 branch); a tap shift is a
//               descriptor start-address offset into the halo window
//   warps 2..9  two epilogue warpgroups; group g drains channel half g of both rows of every
//               accumulation group into registers, then runs the fused pointwise epilogue
#include "common.cuh"
#include "sm100.cuh"

namespace spst {

// RES ("resident weights", 64-channel GEMMs whose conv slab fits): the whole weight slab is
// loaded once per CTA behind two activation-only stages, instead of re-streaming 37 KB per
// chunk per tile -- those layers were bound by their operand loads.
// Epilogue warps of the N=64 kernels.  16 (four warpgroups of 16 channels) was measured and
// rejected: conv1_1 7.56 vs 4.95 ms, conv1_2 9.28 vs 8.86 ms (16-bit mask halves, more
// partial-warp work) -- those layers are bound by their A-window stages, not by epilogue issue.
#ifndef SPST_N64_EPIW
#define SPST_N64_EPIW 8
#endif
template <int N, bool RES = false>
struct ConvCfg {
  static constexpr int MT = 2;                      // output rows per tile (M = MT x 128 px)
  static constexpr int PITCH = 136;                 // 128 output px + 2 halo px, padded to 17 x 128 B
  static constexpr int STRIP = 68;                  // TMA strip (px): two per row at px 0 and 64
  static constexpr int RIN = MT + 2;                // output rows + 2 halo rows
  static constexpr int A_PLANE = RIN * PITCH * 16;  // one 8-channel plane of the window
  static constexpr int A_HALF = 2 * A_PLANE;        // 16 channels
  static constexpr int A_BYTES = 2 * A_HALF;        // hi + lo
  static constexpr int B_TAP = 2 * N * 16;          // 16 channels x N outputs (fp16)
  static constexpr int B_BYTES = 2 * 9 * B_TAP;     // hi/lo x 9 taps
  // extra-K (style-gradient) chunk: 8*XKG channels of the tap features at the tile's own pixels.
  // N=128: 64 channels (24 MMAs, ~1.5k cycles -- enough to hide the next stage's load); its
  // 64 KB operand runs into the weight area, so the slab sits behind it (XB_OFF).
  static constexpr int XKG = MT == 2 ? (N == 128 ? 8 : 4) : 2;
  static constexpr int XA_PLANE = MT * 128 * 16;    // extra-K operand: MT rows x 128 px, 8 ch
  static constexpr int XA_HALF = XKG * XA_PLANE;
  static constexpr int XB_BYTES = 2 * XKG * N * 16; // extra-K slab: hi/lo x XKG kgroups
  // (a resident-mode stage holds an activation window or an extra-K operand + its slab)
  static constexpr int STAGE_BYTES = RES ? (A_BYTES > 2 * XA_HALF + XB_BYTES ? A_BYTES : 2 * XA_HALF + XB_BYTES)
                                         : A_BYTES + B_BYTES;
  static constexpr int STAGE = ((STAGE_BYTES + 1023) / 1024) * 1024;
  static constexpr int STAGES = (N == 128 || RES) ? 2 : 3;
  static constexpr int RES_OFF = STAGES * STAGE;     // resident slab (RES only)
  static constexpr int RES_MAX = RES ? 147456 : 0;   // up to 4 chunks of N=64 (C_in <= 64)
  static constexpr int NBUF = 512 / (MT * N);       // TMEM chunk buffers (MT rows x N each)
  // epilogue warps: 8 = two warpgroups, one channel half each (SPST_N64_EPIW for N=64)
  static constexpr int EPIW = N == 64 ? SPST_N64_EPIW : 8;
  static constexpr int THREADS = 64 + 32 * EPIW;
  static constexpr int TMEM_COLS = 512;
  static constexpr int SMEM = STAGES * STAGE + RES_MAX + 1024;
  static constexpr int CPG = MT == 2 ? N / (EPIW / 4) : N;  // channels per epilogue warpgroup
  static constexpr int NCH = CPG < 32 ? CPG : 32;   // channels per epilogue_ch call
  static constexpr int XB_OFF = (RES || 2 * XA_HALF > A_BYTES) ? 2 * XA_HALF : A_BYTES;  // extra-K slab offset
  static_assert(XB_OFF + XB_BYTES <= STAGE, "extra-K operand and slab must fit one stage");
  static_assert(SMEM + 2048 <= 232448, "dynamic + static shared memory must fit 227 KB");
  static_assert(2 * STRIP * 16 == PITCH * 16 && (PITCH * 16) % 128 == 0 && A_PLANE % 128 == 0, "strip layout");
};

// Chunk schedule of a tile: the n_kc conv chunks, then the n_xkc extra-K (style gradient)
// chunks.  (An interleaved schedule measured slower: its index math sits in the single-thread
// MMA issue loop, which is on the critical path.)
__device__ __forceinline__ bool chunk_is_extra(int c, int n_kc, int& idx) {
  const bool e = c >= n_kc;
  idx = e ? c - n_kc : c;
  return e;
}

// TMEM accumulation groups: up to D (a.drain, 1 or 2) consecutive chunks of the same kind
// (conv / extra-K, which carry different scales) share one fresh TMEM buffer before the
// epilogue drains it into fp32 registers.
//
// Numerics of the in-TMEM accumulation (measured): every MMA rounds its result
// toward zero to fp32, so a group's partial is biased toward zero by ~kappa * w relative, with
// w = sum over the group's MMAs of (hi*hi MMAs issued so far / hi*hi MMAs in the group) and
// kappa ~ E[truncated fraction] x E[ulp/|x|] ~ 0.5 x 0.72 x 2^-23 (fitted on B200: 3.2e-8).
// Uncompensated, that bias has the same sign at every layer and the forward's relative error
// grows linearly with depth (2.2e-7 per conv with one chunk per group, 7e-7 with two).  The
// host passes the expected factor 1 + kappa w: its common part a.fine is applied once to the
// drained sum, the per-group-composition remainder in a.comp[] by the drain.  What is left is
// the unbiased (sqrt-growing) part: fp32-class.
__device__ __forceinline__ void chunk_group(int D, int c, int n_kc, int n_chunks, bool& first, bool& last) {
  const int j = c < n_kc ? c : c - n_kc;
  const int end = c < n_kc ? n_kc : n_chunks;
  first = D == 1 || (j & 1) == 0;
  last = D == 1 || (j & 1) == 1 || c == end - 1;
}
__host__ __device__ constexpr int n_groups(int D, int n_kc, int n_xkc) {
  return (n_kc + D - 1) / D + (n_xkc + D - 1) / D;
}

// 8 channels of one pixel -> hi/lo planes: hi = RN(v s), lo = RN(v s - hi), two floats per
// F2FP conversion (packed: 1 % faster than per-element conversions on the N=128 epilogue too,
// r02 A/B 131.3 -> 130.0 ms/evaluation of conv3x3_tc<128>).
__device__ __forceinline__ void store_hl8(const HL16& t, int kg, int y, int x, const float* v8, float s) {
  const size_t off = ((size_t)kg * t.H + y) * t.W + x;
  uint4 h, l;
  uint32_t* hp = &h.x;
  uint32_t* lp = &l.x;
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    const float a = v8[e] * s, b = v8[e + 1] * s;
    const __half2 hi = __floats2half2_rn(a, b);
    const float2 back = __half22float2(hi);
    const __half2 lo = __floats2half2_rn(a - back.x, b - back.y);
    hp[e / 2] = *reinterpret_cast<const uint32_t*>(&hi);
    lp[e / 2] = *reinterpret_cast<const uint32_t*>(&lo);
  }
  reinterpret_cast<uint4*>(t.hi)[off] = h;
  reinterpret_cast<uint4*>(t.lo())[off] = l;
}

__device__ __forceinline__ void load_hl8(const HL16& t, int kg, int y, int x, float* v8) {
  size_t off = ((size_t)kg * t.H + y) * t.W + x;
  uint4 hv = reinterpret_cast<const uint4*>(t.hi)[off];
  uint4 lv = reinterpret_cast<const uint4*>(t.lo())[off];
  const __half* h = reinterpret_cast<const __half*>(&hv);
  const __half* l = reinterpret_cast<const __half*>(&lv);
  float inv = 1.f / t.scale;
#pragma unroll
  for (int e = 0; e < 8; ++e) v8[e] = (__half2float(h[e]) + __half2float(l[e])) * inv;
}

// After the loop, lane l holds in v[0] the sum over the warp's 32 lanes of column l.
__device__ __forceinline__ float warp_transpose_sum(float (&v)[32]) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
    for (int i = 0; i < off; ++i) {
      float send = (lane & off) ? v[i] : v[i + off];
      float keep = (lane & off) ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// lane l < NCH gets the sum over the warp's 32 lanes of column l (NCH = 32: warp_transpose_sum;
// NCH = 16: the same butterfly from offset 8, then the two half-warps are added)
template <int NCH>
__device__ __forceinline__ float warp_transpose_sum_n(float (&v)[NCH]) {
  if constexpr (NCH == 32) {
    return warp_transpose_sum(v);
  } else {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int off = NCH / 2; off >= 1; off >>= 1) {
#pragma unroll
      for (int i = 0; i < off; ++i) {
        float send = (lane & off) ? v[i] : v[i + off];
        float keep = (lane & off) ? v[i + off] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// 32 columns of TMEM added into acc[0..31] (fp32 round-to-nearest adds)
__device__ __forceinline__ void tmem_add32(uint32_t taddr, float* acc, float scale) {
  float v[32];
  tmem_ld32(taddr, v);
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = fmaf(v[i], scale, acc[i]);
}

// Fused pointwise epilogue for NCH (32, or 16 with 16 epilogue warps) channels of one pixel in
// both rows (v0: row y0, v1: y0+1).  ch0 is a multiple of NCH.
// mpre (nullable): the tile's ReLU mask words for these 32 channels, loaded at tile start (EPI_BWD:
// [row]; EPI_BWD_POOL: [row * 4 + i * 2 + jx]); bpre (nullable): the channels' bias in registers.
template <int N, int NCH>
__device__ __forceinline__ void epilogue_ch(const ConvArgs& a, float* v0, float* v1, int ch0, int x, int y0,
                                            int tile_xy, uint32_t q, float& amax0, float& amax1,
                                            const uint32_t* mpre = nullptr, const float* bpre = nullptr) {
  static_assert(NCH == 16 || NCH == 32, "16 or 32 channels per call");
  const uint32_t lane = lane_id();
  constexpr int KG = NCH / 8;
  if (a.epi == EPI_FWD || a.epi == EPI_FWD_POOL) {
    uint32_t bits0 = 0, bits1 = 0;
#pragma unroll
    for (int j = 0; j < NCH; ++j) {
      const float bj = bpre ? bpre[j] : (a.bias ? __ldg(a.bias + ch0 + j) : 0.f);
      const float p0 = fmaf(v0[j], a.acc_scale, bj);
      const float p1 = fmaf(v1[j], a.acc_scale, bj);
      bits0 |= (p0 > 0.f ? 1u : 0u) << j;
      bits1 |= (p1 > 0.f ? 1u : 0u) << j;
      v0[j] = fmaxf(p0, 0.f);
      v1[j] = fmaxf(p1, 0.f);
    }
    const bool ok0 = x < a.W && y0 < a.H, ok1 = x < a.W && y0 + 1 < a.H;
    if (a.mask_out) {
      const size_t w0 = ((size_t)(ch0 >> 5) * a.H + y0) * a.W + x, w1 = w0 + a.W;
      if constexpr (NCH == 32) {
        if (ok0) a.mask_out[w0] = bits0;
        if (ok1) a.mask_out[w1] = bits1;
      } else {  // a 16-channel half of the 32-bit mask word (little endian)
        uint16_t* m16 = reinterpret_cast<uint16_t*>(a.mask_out);
        const int h = (ch0 >> 4) & 1;
        if (ok0) m16[2 * w0 + h] = (uint16_t)bits0;
        if (ok1) m16[2 * w1 + h] = (uint16_t)bits1;
      }
    }
    if (a.epi == EPI_FWD || a.store_full) {
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        if (ok0) store_hl8(a.out, (ch0 >> 3) + k, y0, x, v0 + 8 * k, a.out.scale);
        if (ok1) store_hl8(a.out, (ch0 >> 3) + k, y0 + 1, x, v1 + 8 * k, a.out.scale);
      }
      if constexpr (N == 64) {  // (the N=128 kernel's codegen prefers the select form)
        if (ok0) {
#pragma unroll
          for (int j = 0; j < NCH; ++j) amax0 = fmaxf(amax0, v0[j]);
        }
        if (ok1) {
#pragma unroll
          for (int j = 0; j < NCH; ++j) amax0 = fmaxf(amax0, v1[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          amax0 = fmaxf(amax0, ok0 ? v0[j] : 0.f);
          amax0 = fmaxf(amax0, ok1 ? v1[j] : 0.f);
        }
      }
    }
    if (a.colsum_partial) {
      const bool inx = x >= a.sum_c0 && x < a.sum_c1;
      const bool in0 = ok0 && inx && y0 >= a.sum_r0 && y0 < a.sum_r1;
      const bool in1 = ok1 && inx && y0 + 1 >= a.sum_r0 && y0 + 1 < a.sum_r1;
      float s[NCH];
#pragma unroll
      for (int j = 0; j < NCH; ++j) s[j] = (in0 ? v0[j] : 0.f) + (in1 ? v1[j] : 0.f);
      const float tot = warp_transpose_sum_n<NCH>(s);
      if (lane < NCH) a.colsum_partial[((size_t)tile_xy * 4 + q) * (size_t)(a.n_ntiles * N) + ch0 + lane] = tot;
    }
    if (a.epi == EPI_FWD_POOL) {
      float pv[NCH];
      const int px = x >> 1, py = y0 >> 1;
      if (a.pool_max) {
        // first-argmax over the window in row-major order (x, y0), (x+1, y0), (x, y0+1),
        // (x+1, y0+1): strict '>' keeps the first of equal values (np.argmax)
        uint32_t arg0 = 0, arg1 = 0;
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const float b = __shfl_xor_sync(0xffffffffu, v0[j], 1), d = __shfl_xor_sync(0xffffffffu, v1[j], 1);
          float m = v0[j];
          uint32_t idx = 0;
          if (b > m) m = b, idx = 1;
          if (v1[j] > m) m = v1[j], idx = 2;
          if (d > m) m = d, idx = 3;
          pv[j] = m;
          if (j < 16) arg0 |= idx << (2 * j);
          else arg1 |= idx << (2 * (j - 16));
        }
        if ((lane & 1) == 0 && px < a.out_pool.W && py < a.out_pool.H) {
          const size_t plane = (size_t)a.out_pool.H * a.out_pool.W, o = (size_t)py * a.out_pool.W + px;
          a.pool_arg[(size_t)(ch0 >> 4) * plane + o] = arg0;
          if constexpr (NCH == 32) a.pool_arg[(size_t)((ch0 >> 4) + 1) * plane + o] = arg1;
        }
      } else {
#pragma unroll
        for (int j = 0; j < NCH; ++j) {
          const float s2 = v0[j] + v1[j];
          pv[j] = (s2 + __shfl_xor_sync(0xffffffffu, s2, 1)) * 0.25f;
        }
      }
      if ((lane & 1) == 0 && px < a.out_pool.W && py < a.out_pool.H) {
#pragma unroll
        for (int k = 0; k < KG; ++k) store_hl8(a.out_pool, (ch0 >> 3) + k, py, px, pv + 8 * k, a.out_pool.scale);
#pragma unroll
        for (int j = 0; j < NCH; ++j) amax1 = fmaxf(amax1, pv[j]);
      }
    }
  } else if (a.epi == EPI_BWD) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float* v = r ? v1 : v0;
      const int y = y0 + r;
      if (x >= a.W || y >= a.H) continue;
#pragma unroll
      for (int j = 0; j < NCH; ++j)
        v[j] = fmaf(v[j], a.acc_scale, bpre ? bpre[j] : (a.bias ? __ldg(a.bias + ch0 + j) : 0.f));
      if (a.content_coef != 0.f) {
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          float cv[8], cu[8];
          load_hl8(a.content_v, (ch0 >> 3) + k, y, x, cv);
          load_hl8(a.content_u, (ch0 >> 3) + k, y, x, cu);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[8 * k + e] = fmaf(a.content_coef, cv[e] - cu[e], v[8 * k + e]);
        }
      }
      if (a.addend.hi) {
#pragma unroll
        for (int k = 0; k < KG; ++k) {
          float ad[8];
          load_hl8(a.addend, (ch0 >> 3) + k, y, x, ad);
#pragma unroll
          for (int e = 0; e < 8; ++e) v[8 * k + e] += ad[e];
        }
      }
      if (a.mask_in) {
        const uint32_t bits =
            (mpre ? mpre[r] : a.mask_in[((size_t)(ch0 >> 5) * a.H + y) * a.W + x]) >> (ch0 & 16);
#pragma unroll
        for (int j = 0; j < NCH; ++j) v[j] = ((bits >> j) & 1u) ? v[j] : 0.f;
      }
#pragma unroll
      for (int j = 0; j < NCH; ++j) amax0 = fmaxf(amax0, fabsf(v[j]));
#pragma unroll
      for (int k = 0; k < KG; ++k) store_hl8(a.out, (ch0 >> 3) + k, y, x, v + 8 * k, a.out.scale);
    }
  } else {  // EPI_BWD_POOL: out is the 2x finer grid
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float* v = r ? v1 : v0;
      const int y = y0 + r;
      if (x >= a.W || y >= a.H) continue;
      // avg: spread g/4 onto the window (tensorops.py:104-110); max: g to the forward's
      // first argmax only (tensorops.py:117-129)
      uint32_t arg0 = 0, arg1 = 0;
      if (a.pool_max) {
        const size_t plane = (size_t)a.H * a.W, o = (size_t)y * a.W + x;
        arg0 = a.pool_arg[(size_t)(ch0 >> 4) * plane + o];
        if constexpr (NCH == 32) arg1 = a.pool_arg[(size_t)((ch0 >> 4) + 1) * plane + o];
      }
      const float sc = a.pool_max ? a.acc_scale : a.acc_scale * 0.25f;
#pragma unroll
      for (int j = 0; j < NCH; ++j) v[j] *= sc;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int jx = 0; jx < 2; ++jx) {
          const int yy = 2 * y + i, xx = 2 * x + jx;
          float w[NCH];
          if (a.pool_max) {
            const uint32_t want = 2 * i + jx;
#pragma unroll
            for (int j = 0; j < NCH; ++j) {
              const uint32_t idx = ((j < 16 ? arg0 : arg1) >> (2 * (j & 15))) & 3u;
              w[j] = idx == want ? v[j] : 0.f;
            }
          } else {
#pragma unroll
            for (int j = 0; j < NCH; ++j) w[j] = v[j];
          }
          if (a.addend.hi) {
#pragma unroll
            for (int k = 0; k < KG; ++k) {
              float ad[8];
              load_hl8(a.addend, (ch0 >> 3) + k, yy, xx, ad);
#pragma unroll
              for (int e = 0; e < 8; ++e) w[8 * k + e] += ad[e];
            }
          }
          if (a.mask_in) {
            const uint32_t bits =
                (mpre ? mpre[r * 4 + i * 2 + jx] : a.mask_in[((size_t)(ch0 >> 5) * a.out.H + yy) * a.out.W + xx]) >>
                (ch0 & 16);
#pragma unroll
            for (int j = 0; j < NCH; ++j) w[j] = ((bits >> j) & 1u) ? w[j] : 0.f;
          }
#pragma unroll
          for (int j = 0; j < NCH; ++j) amax0 = fmaxf(amax0, fabsf(w[j]));
#pragma unroll
          for (int k = 0; k < KG; ++k) store_hl8(a.out, (ch0 >> 3) + k, yy, xx, w + 8 * k, a.out.scale);
        }
    }
  }
}

// Work decomposition: unit t = (spatial tile, n-tile), n-tile fastest, so consecutive CTAs
// share the spatial tile's halo window in L2.  (A clustered variant that multicast the weight
// slab to 2/4/8 CTAs measured slower: the shared stage release couples the CTAs.)
struct TileId {
  int nt, cx, ry;
};

__device__ __forceinline__ TileId decode_tile(const ConvArgs& a, int t) {
  TileId id;
  id.nt = t % a.n_ntiles;
  const int sp = t / a.n_ntiles;
  id.cx = sp % a.tiles_x;
  id.ry = sp / a.tiles_x;
  return id;
}

template <int N, bool RES>
__global__ void __launch_bounds__(ConvCfg<N, RES>::THREADS, 1) conv3x3_tc_kernel(const __grid_constant__ ConvArgs a) {
  using C = ConvCfg<N, RES>;
  static_assert(!RES || (N == 64 && C::MT == 2), "the split lo/hi stages are wired into the row-pair path");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[C::STAGES], empty_bar[C::STAGES];
  // RES: a stage's lo half has its own barriers (full_lo / empty_lo; full_bar / empty_bar then
  // guard the hi half): the lo planes feed only the first correction pass, so they are released
  // -- and the next chunk's lo planes fetched -- a third of a chunk early
  __shared__ uint64_t full_lo[RES ? C::STAGES : 1], empty_lo[RES ? C::STAGES : 1];
  __shared__ uint64_t cfull_bar[C::NBUF], cempty_bar[C::NBUF], res_bar;
  __shared__ uint32_t tmem_slot;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int n_tiles = a.tiles_x * a.tiles_y * a.n_ntiles;
  const int first = (int)blockIdx.x;
  const int step = (int)gridDim.x;
  const int n_chunks = a.n_kc + a.n_xkc;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&a.tm_r_hi);
    tma_prefetch_desc(&a.tm_r_lo);
    tma_prefetch_desc(&a.tm_v_hi);
    tma_prefetch_desc(&a.tm_v_lo);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
      if constexpr (RES) {
        mbar_init(&full_lo[s], 1);
        mbar_init(&empty_lo[s], 1);
      }
    }
    for (int b = 0; b < C::NBUF; ++b) {
      mbar_init(&cfull_bar[b], 1);
      mbar_init(&cempty_bar[b], C::EPIW);
    }
    mbar_init(&res_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    // The A window is fetched as 8*RIN strips of 68 pixels (1088 contiguous bytes) -- one per
    // lane -- through a u64 view of the activation: a box with a 16-byte inner dimension costs
    // the TMA unit one row per pixel and was measured to throttle the MMA pipe. The two strips
    // of a row start at px 0 and 64 (128-B aligned smem) and overlap by 4 px.
    static_assert(8 * C::RIN <= 32, "one A strip per producer lane");
    const int s_hl = lane / (4 * C::RIN), s_p = (lane / (2 * C::RIN)) & 1, s_r = (lane >> 1) % C::RIN, s_h = lane & 1;
    const uint32_t s_off = s_hl * C::A_HALF + s_p * C::A_PLANE + (s_r * C::PITCH + s_h * 64) * 16;
    const void* s_map = s_hl ? (const void*)&a.tm_r_lo : (const void*)&a.tm_r_hi;
    if constexpr (RES) {  // the whole conv slab (one N-tile), once per CTA
      if (lane == 0) {
        mbar_arrive_expect_tx(&res_bar, (uint32_t)a.n_kc * C::B_BYTES);
        bulk_load(smem + C::RES_OFF, a.wgt, (uint32_t)a.n_kc * C::B_BYTES, &res_bar);
      }
    }
    uint32_t g = 0;
    for (int t = first; t < n_tiles; t += step) {
      const TileId id = decode_tile(a, t);
      const int nt = id.nt;
      const int x0 = id.cx * 128;
      const int y0 = id.ry * C::MT;
      for (int c = 0; c < n_chunks; ++c, ++g) {
        const int s = g % C::STAGES;
        const uint32_t eph = ((g / C::STAGES) & 1) ^ 1;
        uint8_t* st = smem + s * C::STAGE;
        int ci;
        const bool extra = chunk_is_extra(c, a.n_kc, ci);
        if constexpr (RES) {
          // lo half first (consumed by the first pass), then the hi half; an extra-K chunk
          // occupies the whole stage and arrives on full_bar only
          mbar_wait(&empty_lo[s], eph);
          if (!extra) {
            if (lane == 0) mbar_arrive_expect_tx(&full_lo[s], C::A_HALF);
            __syncwarp();
            if (lane < 8 * C::RIN && s_hl == 1)
              tma_load_3d(st + s_off, s_map, &full_lo[s], 2 * (x0 - 1) + 128 * s_h, y0 - 1 + s_r, 2 * ci + s_p);
          }
          mbar_wait(&empty_bar[s], eph);
          if (!extra) {
            if (lane == 0) mbar_arrive_expect_tx(&full_bar[s], C::A_HALF);
            __syncwarp();
            if (lane < 8 * C::RIN && s_hl == 0)
              tma_load_3d(st + s_off, s_map, &full_bar[s], 2 * (x0 - 1) + 128 * s_h, y0 - 1 + s_r, 2 * ci + s_p);
          } else if (lane == 0) {
            mbar_arrive(&full_lo[s]);
            mbar_arrive_expect_tx(&full_bar[s], 2 * C::XA_HALF + C::XB_BYTES);
            tma_load_4d(st, &a.tm_v_hi, &full_bar[s], 0, x0, y0, C::XKG * ci);
            tma_load_4d(st + C::XA_HALF, &a.tm_v_lo, &full_bar[s], 0, x0, y0, C::XKG * ci);
            bulk_load(st + C::XB_OFF, a.xwgt + ((size_t)nt * a.n_xkc + ci) * C::XB_BYTES, C::XB_BYTES, &full_bar[s]);
          }
          continue;
        }
        mbar_wait(&empty_bar[s], eph);
        if (!extra) {
          if (lane == 0) mbar_arrive_expect_tx(&full_bar[s], C::A_BYTES + (RES ? 0 : C::B_BYTES));
          __syncwarp();
          if (lane < 8 * C::RIN)
            tma_load_3d(st + s_off, s_map, &full_bar[s], 2 * (x0 - 1) + 128 * s_h, y0 - 1 + s_r, 2 * ci + s_p);
        } else if (lane == 0) {  // extra K (tap features): only the tile's own MT x 128 pixels
          mbar_arrive_expect_tx(&full_bar[s], 2 * C::XA_HALF + C::XB_BYTES);
          tma_load_4d(st, &a.tm_v_hi, &full_bar[s], 0, x0, y0, C::XKG * ci);
          tma_load_4d(st + C::XA_HALF, &a.tm_v_lo, &full_bar[s], 0, x0, y0, C::XKG * ci);
        }
        if (lane == 0 && (extra || !RES)) {
          const uint8_t* bsrc = extra ? a.xwgt + ((size_t)nt * a.n_xkc + ci) * C::XB_BYTES
                                      : a.wgt + ((size_t)nt * a.n_kc + ci) * C::B_BYTES;
          const uint32_t bbytes = extra ? C::XB_BYTES : C::B_BYTES;
          const uint32_t boff = extra ? C::XB_OFF : C::A_BYTES;
          bulk_load(st + boff, bsrc, bbytes, &full_bar[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer (whole warp,
    // one elected lane issues; see umma_f16_ws)
    {
      const uint32_t idesc = make_idesc_f16(128, N, 0, 0, 0);
      if constexpr (RES) mbar_wait(&res_bar, 0);
      uint32_t g = 0, gq = 0;  // chunk counter (smem stages), group counter (TMEM buffers)
      for (int t = first; t < n_tiles; t += step) {
        for (int c = 0; c < n_chunks; ++c, ++g) {
          bool gfirst, glast;
          chunk_group(a.drain, c, a.n_kc, n_chunks, gfirst, glast);
          const uint32_t b = gq % C::NBUF;
          if (gfirst) mbar_wait(&cempty_bar[b], ((gq / C::NBUF) & 1) ^ 1);
          const int s = g % C::STAGES;
          const uint32_t fph = (g / C::STAGES) & 1;
          int ci;
          const bool extra = chunk_is_extra(c, a.n_kc, ci);
          if constexpr (RES) {
            mbar_wait(&full_lo[s], fph);
            if (extra) mbar_wait(&full_bar[s], fph);
          } else {
            mbar_wait(&full_bar[s], fph);
          }
          __syncwarp();
          tc_fence_after();
          const uint32_t st = smem_u32(smem + s * C::STAGE);
          const uint32_t bb = RES ? smem_u32(smem + C::RES_OFF) + (uint32_t)ci * C::B_BYTES : st + C::A_BYTES;
          const uint32_t dcol = tmem_base + b * C::MT * N;
          // descriptor arithmetic: start-address field = addr >> 4 in the low bits, so an
          // offset of k bytes is an add of k >> 4 on the precomputed 64-bit descriptor
          if (extra) {
            // V[MT rows x 128 px, 8*XKG ch] x M[8*XKG x N]: XKG/2 K=16 steps per pass
            const uint64_t bdesc0 = make_sdesc(st + C::XB_OFF, N * 16, 128);
            const uint64_t adesc0 = make_sdesc(st, C::XA_PLANE, 128);
            for (int pass = 0; pass < 3; ++pass)
#pragma unroll
              for (int ks = 0; ks < C::XKG / 2; ++ks) {
                if (pass < a.pass0) continue;  // one-pass (fp16) mode: hi*hi only
                const uint64_t bd = bdesc0 + (uint64_t)((((pass == 0 ? C::XKG : 0) + 2 * ks) * N * 16) >> 4);
#pragma unroll
                for (int mt = 0; mt < C::MT; ++mt) {
                  const uint64_t ad =
                      adesc0 + (uint64_t)(((pass == 1 ? C::XA_HALF : 0) + mt * 128 * 16 + 2 * ks * C::XA_PLANE) >> 4);
                  umma_f16_ws(dcol + mt * N, ad, bd, idesc, (!gfirst || pass != a.pass0 || ks) ? 1u : 0u);
                }
              }
          } else if constexpr (N == 64 && C::MT == 2) {
            // Row-pair MMAs: window row r feeds output row 0 through tap dy=r and output row 1
            // through dy=r-1, so rows r=1,2 are ONE N=128 MMA A_r x [W_r ; W_{r-1}] writing both
            // rows' columns (row 0: 0-63, row 1: 64-127); r=0 / r=3 are N=64 MMAs for one row.
            // Slab per (pass, dx, kgroup): [W_dy2 ; W_dy1 ; W_dy0] (192 rows), so every B
            // operand is a contiguous window.  The first MMA of a group is r=1 (initialises both
            // rows); an SS N=64 MMA is smem-read bound (48 cycles), this pairing saves 22 %.
            const uint32_t idesc2 = make_idesc_f16(128, 2 * N, 0, 0, 0);
            constexpr int ROWS3 = 3 * N;                       // rows of one (pass, dx, kg) slab
            const uint64_t bdesc0 = make_sdesc(bb, ROWS3 * 16, 128);
            const uint64_t adesc0 = make_sdesc(st, C::A_PLANE, 128);
            // issue order q: RES runs lo*hi first (then hi*lo, hi*hi) so the lo half can be
            // released after q = 0; both orders put the corrections before the large products
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              if constexpr (RES) {
                if (q == 1) {  // lo planes consumed: release them, wait for the hi planes
                  umma_commit_ws(&empty_lo[s]);
                  mbar_wait(&full_bar[s], fph);
                  __syncwarp();
                  tc_fence_after();
                }
              }
              const int pass = RES ? (q == 0 ? 1 : (q == 1 ? 0 : 2)) : q;
              if (pass < a.pass0) continue;  // one-pass (fp16) mode: hi*hi only
              const uint64_t bp = bdesc0 + (uint64_t)(((pass == 0 ? 9 : 0) * C::B_TAP) >> 4);
              const uint64_t ap = adesc0 + (uint64_t)((pass == 1 ? C::A_HALF : 0) >> 4);
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
                const uint64_t bx = bp + (uint64_t)((dx * 2 * ROWS3 * 16) >> 4);
                const uint64_t a0 = ap + (uint64_t)((dx * 16) >> 4), rowp = (uint64_t)((C::PITCH * 16) >> 4);
                const uint32_t first = (gfirst && q == a.pass0 && dx == 0) ? 0u : 1u;
                umma_f16_ws(dcol, a0 + rowp, bx + (uint64_t)((N * 16) >> 4), idesc2, first);  // r=1
                umma_f16_ws(dcol, a0, bx + (uint64_t)((2 * N * 16) >> 4), idesc, 1u);         // r=0
                umma_f16_ws(dcol, a0 + 2 * rowp, bx, idesc2, 1u);                              // r=2
                umma_f16_ws(dcol + N, a0 + 3 * rowp, bx, idesc, 1u);                           // r=3
              }
            }
          } else {
            const uint64_t bdesc0 = make_sdesc(bb, N * 16, 128);
            const uint64_t adesc0 = make_sdesc(st, C::A_PLANE, 128);
            // Small correction products first (hi*lo, lo*hi), then the large hi*hi products: the
            // tensor core truncates each accumulation to the running sum's exponent, so keeping
            // the sum small while the corrections go in cuts the chunk's rounding error ~3x.
#pragma unroll
            for (int pass = 0; pass < 3; ++pass) {
              if (pass < a.pass0) continue;  // one-pass (fp16) mode: hi*hi only
              const uint64_t bp = bdesc0 + (uint64_t)(((pass == 0 ? 9 : 0) * C::B_TAP) >> 4);
              const uint64_t ap = adesc0 + (uint64_t)((pass == 1 ? C::A_HALF : 0) >> 4);
#pragma unroll
              for (int tap = 0; tap < 9; ++tap) {
                const int dy = tap / 3, dx = tap % 3;
                const uint64_t bd = bp + (uint64_t)((tap * C::B_TAP) >> 4);
#pragma unroll
                for (int mt = 0; mt < C::MT; ++mt) {
                  const uint64_t ad = ap + (uint64_t)((((mt + dy) * C::PITCH + dx) * 16) >> 4);
                  umma_f16_ws(dcol + mt * N, ad, bd, idesc, (!gfirst || pass != a.pass0 || tap) ? 1u : 0u);  // fresh per group
                }
              }
            }
          }
          if constexpr (RES) {
            if (extra) umma_commit_ws(&empty_lo[s]);
          }
          umma_commit_ws(&empty_bar[s]);
          if (glast) {
            umma_commit_ws(&cfull_bar[b]);
            ++gq;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------------ epilogue (8 warps)
    const uint32_t q = warp & 3;            // TMEM lane quarter
    const uint32_t grp = (warp - 2) >> 2;   // MT=2: channel half; MT=4: row pair
    const int m = q * 32 + lane;
    const int rp = C::MT == 2 ? 0 : (int)grp;            // row pair handled by this warpgroup
    const int cofs = C::MT == 2 ? (int)grp * C::CPG : 0;  // first channel handled
    uint32_t g = 0;
    // max |output| over all of this thread's tiles: one atomic per warp per launch (a per-tile
    // atomic on the same two words from every SM serialised in L2)
    float amax0 = 0.f, amax1 = 0.f;
    // N=64 (one epilogue_ch call per thread and tile): bias in registers for the whole launch,
    // ReLU mask words fetched at tile start so their latency hides behind the drains
    constexpr bool PRE = N == 64 && C::CPG == 32;
    float bpre[PRE ? 32 : 1];
    int bias_nt = -1;
    for (int t = first; t < n_tiles; t += step) {
      const TileId id = decode_tile(a, t);
      const int nt = id.nt, cx = id.cx, ry = id.ry;
      const int x0 = cx * 128, y0 = ry * C::MT + 2 * rp;
      const int x = x0 + m;
      uint32_t mpre[PRE ? 8 : 1];
      if constexpr (PRE) {
        const int ch0 = nt * N + cofs;
        if (nt != bias_nt) {
#pragma unroll
          for (int j = 0; j < 32; ++j) bpre[j] = a.bias ? __ldg(a.bias + ch0 + j) : 0.f;
          bias_nt = nt;
        }
        if (a.mask_in && a.epi == EPI_BWD) {
#pragma unroll
          for (int r = 0; r < 2; ++r)
            mpre[r] = (x < a.W && y0 + r < a.H) ? a.mask_in[((size_t)(ch0 >> 5) * a.H + y0 + r) * a.W + x] : 0u;
        } else if (a.mask_in && a.epi == EPI_BWD_POOL) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int r = k >> 2, yy = 2 * (y0 + r) + ((k >> 1) & 1), xx = 2 * x + (k & 1);
            mpre[k] = (x < a.W && y0 + r < a.H) ? a.mask_in[((size_t)(ch0 >> 5) * a.out.H + yy) * a.out.W + xx] : 0u;
          }
        }
      }
      float acc0[C::CPG], acc1[C::CPG];
#pragma unroll
      for (int i = 0; i < C::CPG; ++i) acc0[i] = acc1[i] = 0.f;
      const int D = a.drain;
      // accumulation groups as the MMA issuer forms them (chunk_group): up to D chunks of one kind
      const int ce = n_chunks;
      for (int c = 0; c < ce; ++g) {
        const bool xg = c >= a.n_kc;
        const int gsz = min(D, (xg ? ce : min(ce, a.n_kc)) - c);
        c += gsz;
        const uint32_t b = g % C::NBUF;
        mbar_wait(&cfull_bar[b], (g / C::NBUF) & 1);
        tc_fence_after();
        const uint32_t trow = tmem_base + ((q * 32u) << 16) + b * C::MT * N + 2 * rp * N + cofs;
        // extra-K groups carry their own scale; comp[] undoes the expected round-toward-zero bias
        // of the group (index: kind x 2 + chunks in the group - 1)
        const float cs = (xg ? a.x_rescale : 1.f) * a.comp[(xg ? 2 : 0) + gsz - 1];
        if constexpr (C::CPG == 32) {  // both rows in one batch: 2 loads, 1 wait
          float v0[32], v1[32];
          tmem_ld32x2(trow, trow + N, v0, v1);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            acc0[i] = fmaf(v0[i], cs, acc0[i]);
            acc1[i] = fmaf(v1[i], cs, acc1[i]);
          }
        } else if constexpr (C::CPG == 16) {
          float v0[16], v1[16];
          tmem_ld16x2(trow, trow + N, v0, v1);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            acc0[i] = fmaf(v0[i], cs, acc0[i]);
            acc1[i] = fmaf(v1[i], cs, acc1[i]);
          }
        } else {
#pragma unroll
          for (int cb = 0; cb < C::CPG / 32; ++cb) {
            tmem_add32(trow + cb * 32, acc0 + cb * 32, cs);
            tmem_add32(trow + N + cb * 32, acc1 + cb * 32, cs);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty_bar[b]);
      }
      // the common part of the round-toward-zero compensation, once per output (exact to fp32
      // rounding; a (1 + eps) factor in the per-group drains would be quantised to 2^-23)
#pragma unroll
      for (int i = 0; i < C::CPG; ++i) {
        acc0[i] = fmaf(acc0[i], a.fine, acc0[i]);
        acc1[i] = fmaf(acc1[i], a.fine, acc1[i]);
      }
      const int part_row = (ry * a.tiles_x + cx) * (C::MT / 2) + rp;
      if constexpr (PRE) {
        epilogue_ch<N, 32>(a, acc0, acc1, nt * N + cofs, x, y0, part_row, q, amax0, amax1,
                           a.mask_in ? mpre : nullptr, bpre);
      } else {
#pragma unroll
        for (int cb = 0; cb < C::CPG / C::NCH; ++cb)
          epilogue_ch<N, C::NCH>(a, acc0 + cb * C::NCH, acc1 + cb * C::NCH, nt * N + cofs + cb * C::NCH, x, y0,
                                 part_row, q, amax0, amax1);
      }
    }
    if (a.amax) {
      amax0 = warp_max(amax0);
      amax1 = warp_max(amax1);
      if (lane == 0) {
        if (amax0 > 0.f) atomicMax(a.amax, __float_as_uint(amax0));
        if (amax1 > 0.f) atomicMax(a.amax + 1, __float_as_uint(amax1));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

// ------------------------------------------------------------------------------------------
int conv_tc_smem_bytes(int N) { return N == 128 ? ConvCfg<128>::SMEM : ConvCfg<64>::SMEM; }
int conv_tc_rows(int N) { return N == 128 ? ConvCfg<128>::MT : ConvCfg<64>::MT; }
int conv_tc_xkg(int N) { return N == 128 ? ConvCfg<128>::XKG : ConvCfg<64>::XKG; }

template <int N, bool RES>
static cudaError_t launch_one(const ConvArgs& a, int grid, cudaStream_t stream) {
  auto k = conv3x3_tc_kernel<N, RES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, ConvCfg<N, RES>::SMEM);
  note_launch(), k<<<grid, ConvCfg<N, RES>::THREADS, ConvCfg<N, RES>::SMEM, stream>>>(a);
  return cudaGetLastError();
}

// resident: 64-channel GEMM whose whole conv slab (one N-tile, n_kc chunks) fits in smem
bool conv_tc_resident_ok(int N, int n_ntiles, int n_kc) {
  return N == 64 && n_ntiles == 1 && n_kc >= 1 && n_kc * ConvCfg<64, true>::B_BYTES <= ConvCfg<64, true>::RES_MAX;
}

cudaError_t launch_conv_tc(const ConvArgs& a, int N, int grid, cudaStream_t stream) {
  if (N == 128) return launch_one<128, false>(a, grid, stream);
  return conv_tc_resident_ok(N, a.n_ntiles, a.n_kc) ? launch_one<64, true>(a, grid, stream)
                                                    : launch_one<64, false>(a, grid, stream);
}

}  // namespace spst
