// Dense update and training helpers of the GCN/GIN layers.
//   ag_gemm_f32      the (agg @ W) update of models.py:99/:112 and its two
//                    backward products (H^T G, G W^T); fp32 SIMT, 128x128x8
//                    CTA tiles, 8x8 register micro-tiles, register-prefetched
//                    double buffering, deterministic split-K for the skinny
//                    H^T G case (K = V, M,N <= a few hundred).
//   ag_softmax_xent  composed loss of SURVEY.md §8c (mean masked softmax CE)
//   ag_relu_backward, ag_sgd_step
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "ag_common.cuh"

namespace ag {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8, NT = 256;

struct GemmArgs {
  int64_t M, N, K;
  const float *A;
  int64_t lda;
  int ta;
  const float *B;
  int64_t ldb;
  int tb;
  float *C;  // final output (splits == 1) or partial buffer [splits][M][N]
  int64_t ldc;
  float alpha, beta;
  int epi;
  int64_t k_per_split;
  const uint32_t *mask;  // ReLU-backward bit mask (NULL: none): out = bit ? out : 0
  int64_t ldm;           // words per mask row
};

// A(m, k) of op(A) and B(k, n) of op(B)
__device__ __forceinline__ float ldA(const GemmArgs &g, int64_t m, int64_t k) {
  if (m >= g.M || k >= g.K) return 0.0f;
  return g.ta ? __ldg(g.A + k * g.lda + m) : __ldg(g.A + m * g.lda + k);
}
__device__ __forceinline__ float ldB(const GemmArgs &g, int64_t k, int64_t n) {
  if (k >= g.K || n >= g.N) return 0.0f;
  return g.tb ? __ldg(g.B + n * g.ldb + k) : __ldg(g.B + k * g.ldb + n);
}

__global__ void __launch_bounds__(NT, 2) sgemm_kernel(GemmArgs g, int partial) {
  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
  const int64_t kbeg = static_cast<int64_t>(blockIdx.z) * g.k_per_split;
  const int64_t kend = min(g.K, kbeg + g.k_per_split);
  // loader mapping: 1024 elements of each tile, 4 per thread
  // non-transposed A: row-major [m][k]  -> thread loads (m = tid/2, k = (tid%2)*4 .. +4)
  // transposed A:     stored [k][m]     -> thread loads (k = tid/32, m = (tid%32)*4 .. +4)
  float ra[4], rb[4];
  auto load_regs = [&](int64_t k0) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (!g.ta) ra[t] = ldA(g, m0 + tid / 2, k0 + (tid % 2) * 4 + t);
      else ra[t] = ldA(g, m0 + (tid % 32) * 4 + t, k0 + tid / 32);
      if (!g.tb) rb[t] = ldB(g, k0 + tid / 32, n0 + (tid % 32) * 4 + t);
      else rb[t] = ldB(g, k0 + (tid % 2) * 4 + t, n0 + tid / 2);
    }
  };
  auto store_smem = [&](int buf) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (!g.ta) As[buf][(tid % 2) * 4 + t][tid / 2] = ra[t];
      else As[buf][tid / 32][(tid % 32) * 4 + t] = ra[t];
      if (!g.tb) Bs[buf][tid / 32][(tid % 32) * 4 + t] = rb[t];
      else Bs[buf][(tid % 2) * 4 + t][tid / 2] = rb[t];
    }
  };
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;
  const int ty = tid / 16, tx = tid % 16;
  int buf = 0;
  if (kbeg < kend) {
    load_regs(kbeg);
    store_smem(0);
    __syncthreads();
  }
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load_regs(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
      const float4 a0 = *reinterpret_cast<const float4 *>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4 *>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[buf][kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_smem(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
  // epilogue: rows ty*4+{0..3} and 64+ty*4+{0..3}; cols tx*4+{0..3}, 64+tx*4+{0..3}
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n >= g.N) continue;
      if (partial) {
        g.C[(static_cast<int64_t>(blockIdx.z) * g.M + m) * g.N + n] = acc[i][j];
      } else {
        float v = g.alpha * acc[i][j];
        if (g.beta != 0.0f) v = fmaf(g.beta, g.C[m * g.ldc + n], v);
        if (g.epi & AG_GEMM_RELU) v = fmaxf(v, 0.0f);
        if (g.mask && !relu_bit(g.mask, g.ldm, m, n)) v = 0.0f;
        g.C[m * g.ldc + n] = v;
      }
    }
  }
}

__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int splits, const float *part, float *C,
                                     int64_t ldc, float alpha, float beta, int epi,
                                     const uint32_t *mask, int64_t ldm) {
  const int64_t n = M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.0f;
    for (int p = 0; p < splits; ++p) s += part[p * n + i];  // fixed order: deterministic
    const int64_t m = i / N, c = i % N;
    float v = alpha * s;
    if (beta != 0.0f) v = fmaf(beta, C[m * ldc + c], v);
    if (epi & AG_GEMM_RELU) v = fmaxf(v, 0.0f);
    if (mask && !relu_bit(mask, ldm, m, c)) v = 0.0f;
    C[m * ldc + c] = v;
  }
}

// Mean softmax cross-entropy over the masked rows.  CTA b owns
// the contiguous row block [b*R, (b+1)*R); a warp per row; lane c holds
// logits c, c+32, ...  Each CTA reduces its rows' losses in fp64 in a fixed
// order and writes one partial; loss_final_kernel adds the partials in order,
// so the loss is deterministic for a given grid.
constexpr int kXentThreads = 256;

__global__ void __launch_bounds__(kXentThreads) xent_kernel(
    int64_t rows, int64_t C, int64_t ld, const float *logits, const int32_t *labels,
    const uint8_t *mask, float inv_n, int64_t rows_per_cta, double *partial, float *dlogits,
    int64_t ldd) {
  __shared__ double warp_sum[kXentThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = blockIdx.x * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  double acc = 0.0;
  for (int64_t r = r0 + warp; r < r1; r += kXentThreads / 32) {
    const float *z = logits + r * ld;
    float *dz = dlogits + r * ldd;
    for (int64_t c = C + lane; c < ldd; c += 32) dz[c] = 0.0f;  // pad columns stay 0
    const bool on = mask ? mask[r] != 0 : true;
    if (!on) {
      for (int64_t c = lane; c < C; c += 32) dz[c] = 0.0f;
      continue;
    }
    float mx = -INFINITY;
    for (int64_t c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float se = 0.0f;
    for (int64_t c = lane; c < C; c += 32) se += expf(z[c] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int32_t y = labels[r];
    const float inv_se = 1.0f / se;
    for (int64_t c = lane; c < C; c += 32) {
      const float p = expf(z[c] - mx) * inv_se;
      dz[c] = (p - (c == y ? 1.0f : 0.0f)) * inv_n;
    }
    if (lane == 0) acc += static_cast<double>(mx + logf(se) - z[y]);
  }
  if (lane == 0) warp_sum[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kXentThreads / 32; ++w) t += warp_sum[w];
    partial[blockIdx.x] = t;
  }
}

// Narrow logits (C <= 64): a warp per row, lane l holding logits l and l + 32
// in registers -- one coalesced pass over the row, exp computed once and kept
// for the gradient, max / sum by warp shuffles.  Loss partials as in
// xent_kernel (fp64 per lane-0 in a fixed row order, fixed-order CTA sum).
__global__ void __launch_bounds__(kXentThreads) xent_warp_kernel(
    int64_t rows, int64_t C, int64_t ld, const float *logits, const int32_t *labels,
    const uint8_t *mask, float inv_n, int64_t rows_per_cta, double *partial, float *dlogits,
    int64_t ldd) {
  constexpr int U = 4;  // rows per warp in flight (their loads issued together)
  __shared__ double warp_sum[kXentThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = blockIdx.x * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  const int c0 = lane, c1 = lane + 32;
  const bool in0 = c0 < C, in1 = c1 < C;
  double acc = 0.0;
  for (int64_t rb = r0 + warp * U; rb < r1; rb += (kXentThreads / 32) * U) {
    float z0[U], z1[U];
    int32_t y[U];
    bool on[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = rb + u;
      const bool ok = r < r1;
      const float *z = logits + (ok ? r : r0) * ld;
      z0[u] = (ok && in0) ? __ldg(z + c0) : -INFINITY;
      z1[u] = (ok && in1) ? __ldg(z + c1) : -INFINITY;
      y[u] = ok ? labels[r] : 0;
      on[u] = ok && (mask ? mask[r] != 0 : true);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t r = rb + u;
      if (r >= r1) break;
      float g0 = 0.0f, g1 = 0.0f;
      if (on[u]) {
        float mx = fmaxf(z0[u], z1[u]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float e0 = in0 ? expf(z0[u] - mx) : 0.0f, e1 = in1 ? expf(z1[u] - mx) : 0.0f;
        float se = e0 + e1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const float inv_se = 1.0f / se;
        g0 = (e0 * inv_se - (c0 == y[u] ? 1.0f : 0.0f)) * inv_n;
        g1 = (e1 * inv_se - (c1 == y[u] ? 1.0f : 0.0f)) * inv_n;
        const float zy = __shfl_sync(0xffffffffu, y[u] < 32 ? z0[u] : z1[u], y[u] & 31);
        if (lane == 0) acc += static_cast<double>(mx + logf(se) - zy);
      }
      float *dz = dlogits + r * ldd;
      if (c0 < ldd) dz[c0] = in0 ? g0 : 0.0f;  // pad columns stay 0
      if (c1 < ldd) dz[c1] = in1 ? g1 : 0.0f;
    }
  }
  if (lane == 0) warp_sum[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kXentThreads / 32; ++w) t += warp_sum[w];
    partial[blockIdx.x] = t;
  }
}

// Narrow logits (ld <= kXentLd): a thread per row.  Each CTA stages a chunk of
// kXentThreads consecutive rows (contiguous: row stride ld) in shared memory
// with coalesced float4 loads, every thread reduces its own row there (max,
// sum of exp, gradient written back in place), and the chunk is stored back
// coalesced.  Loss partials as in xent_kernel: fp64 per thread in a fixed row
// order, then a fixed-order CTA sum.
constexpr int kXentLd = 64;

__global__ void __launch_bounds__(kXentThreads) xent_rows_kernel(
    int64_t rows, int64_t C, int64_t ld, const float *logits, const int32_t *labels,
    const uint8_t *mask, float inv_n, double *partial, float *dlogits, int64_t ldd) {
  extern __shared__ float zs[];  // kXentThreads * (ld + 1)
  __shared__ double tsum[kXentThreads];
  const int t = threadIdx.x;
  double acc = 0.0;
  for (int64_t r0 = static_cast<int64_t>(blockIdx.x) * kXentThreads; r0 < rows;
       r0 += static_cast<int64_t>(gridDim.x) * kXentThreads) {
    const int64_t nr = rows - r0 < kXentThreads ? rows - r0 : static_cast<int64_t>(kXentThreads);
    const int64_t n = nr * ld;
    const int64_t lp = ld + 1;  // odd row stride in shared memory: conflict-free per-thread rows
    const float *src = logits + r0 * ld;
    const int ni = static_cast<int>(n), li = static_cast<int>(ld), lpi = li + 1;
    for (int i = t; i < ni; i += kXentThreads) zs[(i / li) * lpi + i % li] = src[i];
    __syncthreads();
    if (t < nr) {
      float *z = zs + static_cast<int64_t>(t) * lp;
      const int64_t r = r0 + t;
      if (mask && mask[r] == 0) {
        for (int64_t c = 0; c < C; ++c) z[c] = 0.0f;
      } else {
        const int ci = static_cast<int>(C);
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        int c = 0;
        for (; c + 4 <= ci; c += 4)
#pragma unroll
          for (int j = 0; j < 4; ++j) m4[j] = fmaxf(m4[j], z[c + j]);
        for (; c < ci; ++c) m4[0] = fmaxf(m4[0], z[c]);
        const float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
        const int32_t y = labels[r];
        const float zy = z[y];
        float se = 0.0f;
#pragma unroll 8
        for (int cc = 0; cc < ci; ++cc) {  // exp once, kept in place for the gradient
          const float ex = expf(z[cc] - mx);
          z[cc] = ex;
          se += ex;
        }
        acc += static_cast<double>(mx + logf(se) - zy);
        const float inv_se = 1.0f / se;
#pragma unroll 8
        for (int cc = 0; cc < ci; ++cc) z[cc] = (z[cc] * inv_se - (cc == y ? 1.0f : 0.0f)) * inv_n;
      }
    }
    __syncthreads();
    // rows of dlogits have their own stride ldd; columns >= C (the pad) are 0
    const int ldi = static_cast<int>(ldd), nd = static_cast<int>(nr * ldd);
    float *dst = dlogits + r0 * ldd;
    for (int i = t; i < nd; i += kXentThreads) {
      const int c = i % ldi;
      dst[i] = c < C ? zs[(i / ldi) * lpi + c] : 0.0f;
    }
    __syncthreads();
  }
  tsum[t] = acc;
  __syncthreads();
  if (t == 0) {
    double s = 0.0;
    for (int i = 0; i < kXentThreads; ++i) s += tsum[i];
    partial[blockIdx.x] = s;
  }
}

// One warp: lane l sums partials l, l + 32, ... in order, then a fixed
// shuffle tree -- deterministic for a given partial count, ~30x shorter than
// one thread walking every partial.
__global__ void loss_final_kernel(int n, const double *partial, double inv_n, float *out) {
  if (blockIdx.x != 0 || threadIdx.x >= 32) return;
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) t += partial[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (threadIdx.x == 0) *out = static_cast<float>(t * inv_n);
}

// bits[r][w] of a [rows][feat] (row stride ld) activation: a warp per
// (row, 32-column word), one ballot per word.
__global__ void relu_bits_kernel(int64_t rows, int64_t feat, const float *h, int64_t ld,
                                 uint32_t *bits, int64_t ldw) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = relu_words(feat);
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
       t < rows * nw; t += warps) {
    const int64_t r = t / nw, w = t % nw;
    const int64_t c = w * 32 + lane;
    const bool on = c < feat && h[r * ld + c] > 0.0f;
    const uint32_t b = __ballot_sync(0xffffffffu, on);
    if (lane == 0) bits[r * ldw + w] = b;
  }
}

// Dense diagonal blocks -> block-diagonal panels for the tensor-core dense
// block product: row r of A (panel width P = max(B, 128)) holds block
// b = r / B's row r - bB at columns bB - pb .. bB - pb + B (pb = the panel's
// first row), zeros elsewhere; a missing community (comm_slot < 0) is a zero row.
__global__ void dense_block_pack_kernel(int64_t rows, int64_t B, int64_t P,
                                        const int32_t *comm_slot, const float *blocks, float *A,
                                        int64_t lda) {
  const int64_t n = rows * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / P, c = i % P;
    const int64_t b = r / B, pb = (r / P) * P;
    const int64_t j = c - (b * B - pb);
    float v = 0.0f;
    if (j >= 0 && j < B) {
      const int32_t slot = comm_slot[b];
      if (slot >= 0) v = blocks[(static_cast<int64_t>(slot) * B + (r - b * B)) * B + j];
    }
    A[r * lda + c] = v;
  }
}

__global__ void relu_bwd_kernel(int64_t n, const float *h, float *g) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!(h[i] > 0.0f)) g[i] = 0.0f;
}

__global__ void sgd_kernel(int64_t n, float *w, const float *dw, float lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    w[i] = w[i] - lr * dw[i];
}

}  // namespace
}  // namespace ag

using namespace ag;

extern "C" int ag_gemm_f32(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                           int32_t trans_a, const float *B, int64_t ldb, int32_t trans_b,
                           float *C, int64_t ldc, float alpha, float beta, int32_t epilogue,
                           const uint32_t *mask, int64_t ldm, uint32_t *mask_out,
                           int64_t ldmo, void *stream) {
  if (M < 0 || N < 0 || K < 0) return fail(AG_ERR_VALUE, "negative GEMM sizes");
  if (M == 0 || N == 0) return AG_OK;
  if ((mask && ldm < relu_words(N)) || (mask_out && ldmo < relu_words(N)))
    return fail(AG_ERR_VALUE, "relu-bit row strides must be >= ceil(N / 32) words");
  cudaStream_t st = as_stream(stream);
  const int64_t tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  if (tiles_m > 65535) return fail(AG_ERR_VALUE, "GEMM M too large (%lld)", (long long)M);
  const int64_t tiles = tiles_m * tiles_n;
  const int64_t target = 2LL * sm_count();
  int splits = 1;
  if (tiles < target && K >= 4 * 512) {
    splits = static_cast<int>(std::min<int64_t>((target + tiles - 1) / tiles, K / 512));
    splits = std::max(1, std::min(splits, 256));
  }
  int64_t kps = (K + splits - 1) / splits;
  kps = (kps + BK - 1) / BK * BK;
  splits = static_cast<int>((K + kps - 1) / kps);
  if (splits < 1) splits = 1;
  GemmArgs g{M, N, K, A, lda, trans_a, B, ldb, trans_b, C, ldc, alpha, beta, epilogue, kps,
             mask, ldm};
  dim3 grid(static_cast<unsigned>(tiles_n), static_cast<unsigned>(tiles_m), splits);
  if (splits == 1) {
    sgemm_kernel<<<grid, NT, 0, st>>>(g, 0);
    AG_LAUNCH_CHECK("sgemm_kernel");
    return mask_out ? ag_relu_bits(M, N, C, ldc, mask_out, ldmo, stream) : AG_OK;
  }
  Scratch part;
  AG_CUDA(part.alloc(static_cast<size_t>(splits) * M * N * sizeof(float), st));
  g.C = part.as<float>();
  sgemm_kernel<<<grid, NT, 0, st>>>(g, 1);
  AG_LAUNCH_CHECK("sgemm_kernel(split)");
  splitk_reduce_kernel<<<grid_for(M * N, 256), 256, 0, st>>>(M, N, splits, part.as<float>(), C,
                                                            ldc, alpha, beta, epilogue, mask,
                                                            ldm);
  AG_LAUNCH_CHECK("splitk_reduce_kernel");
  return mask_out ? ag_relu_bits(M, N, C, ldc, mask_out, ldmo, stream) : AG_OK;
}

extern "C" int ag_softmax_xent(int64_t rows, int64_t C, int64_t ld, const float *logits,
                               const int32_t *labels, const uint8_t *mask, int64_t num_masked,
                               float *loss_out, float *dlogits, int64_t ld_dlogits,
                               void *stream) {
  if (rows < 0 || C < 1 || ld < C || ld_dlogits < C) return fail(AG_ERR_VALUE, "bad loss sizes");
  cudaStream_t st = as_stream(stream);
  const float inv_n = num_masked > 0 ? 1.0f / static_cast<float>(num_masked) : 0.0f;
  const bool narrow = ld <= kXentLd && std::getenv("AG_XENT_ROWS") != nullptr;
  if (C <= 64 && ld_dlogits <= 64 && !narrow) {
    const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64,
                                                                static_cast<int64_t>(sm_count()) * 8));
    const int64_t per = (rows + ctas - 1) / ctas;
    Scratch pw;
    AG_CUDA(pw.alloc(ctas * sizeof(double), st));
    xent_warp_kernel<<<static_cast<unsigned>(ctas), kXentThreads, 0, st>>>(
        rows, C, ld, logits, labels, mask, inv_n, std::max<int64_t>(per, 1), pw.as<double>(),
        dlogits, ld_dlogits);
    AG_LAUNCH_CHECK("xent_warp_kernel");
    loss_final_kernel<<<1, 32, 0, st>>>(static_cast<int>(ctas), pw.as<double>(),
                                        num_masked > 0 ? 1.0 / num_masked : 0.0, loss_out);
    AG_LAUNCH_CHECK("loss_final_kernel");
    return AG_OK;
  }
  int64_t ctas;
  Scratch part;
  if (narrow) {
    // rows per CTA chunk = kXentThreads; ~2 chunks per CTA in flight per SM slot
    const size_t smem = static_cast<size_t>(kXentThreads) * (ld + 1) * sizeof(float);
    ctas = std::max<int64_t>(1, std::min<int64_t>((rows + kXentThreads - 1) / kXentThreads,
                                                  static_cast<int64_t>(sm_count()) * 4));
    AG_CUDA(part.alloc(ctas * sizeof(double), st));
    AG_CUDA(cudaFuncSetAttribute(xent_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kXentThreads * (kXentLd + 1) * sizeof(float))));
    xent_rows_kernel<<<static_cast<unsigned>(ctas), kXentThreads, smem, st>>>(
        rows, C, ld, logits, labels, mask, inv_n, part.as<double>(), dlogits, ld_dlogits);
    AG_LAUNCH_CHECK("xent_rows_kernel");
  } else {
    ctas = std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64,
                                                  static_cast<int64_t>(sm_count()) * 8));
    const int64_t per = (rows + ctas - 1) / ctas;
    AG_CUDA(part.alloc(ctas * sizeof(double), st));
    xent_kernel<<<static_cast<unsigned>(ctas), kXentThreads, 0, st>>>(
        rows, C, ld, logits, labels, mask, inv_n, std::max<int64_t>(per, 1), part.as<double>(),
        dlogits, ld_dlogits);
    AG_LAUNCH_CHECK("xent_kernel");
  }
  loss_final_kernel<<<1, 32, 0, st>>>(static_cast<int>(ctas), part.as<double>(),
                                      num_masked > 0 ? 1.0 / num_masked : 0.0, loss_out);
  AG_LAUNCH_CHECK("loss_final_kernel");
  return AG_OK;
}

extern "C" int ag_relu_bits(int64_t rows, int64_t feat, const float *h, int64_t ld,
                            uint32_t *bits, int64_t ldw, void *stream) {
  if (rows < 0 || feat < 0 || ld < feat || ldw < relu_words(feat))
    return fail(AG_ERR_VALUE, "bad relu_bits sizes");
  if (rows == 0 || feat == 0) return AG_OK;
  const int64_t warps = rows * relu_words(feat);
  relu_bits_kernel<<<grid_for(warps * 32, 256), 256, 0, as_stream(stream)>>>(rows, feat, h, ld,
                                                                          bits, ldw);
  AG_LAUNCH_CHECK("relu_bits_kernel");
  return AG_OK;
}

extern "C" int ag_dense_block_pack(int64_t num_rows, int64_t block_size, int64_t panel,
                                   const int32_t *comm_slot, const float *blocks, float *A,
                                   int64_t lda, void *stream) {
  if (num_rows < 0 || block_size < 1) return fail(AG_ERR_VALUE, "bad dense block sizes");
  if (panel % 128 != 0 || (block_size <= 128 ? panel != 128 : panel != block_size) ||
      (block_size < 128 && 128 % block_size != 0) || lda < panel)
    return fail(AG_ERR_VALUE, "panel must be max(block_size, 128) with block_size dividing 128 "
                              "or a multiple of 128");
  if (num_rows == 0) return AG_OK;
  dense_block_pack_kernel<<<grid_for(num_rows * panel, 256), 256, 0, as_stream(stream)>>>(
      num_rows, block_size, panel, comm_slot, blocks, A, lda);
  AG_LAUNCH_CHECK("dense_block_pack_kernel");
  return AG_OK;
}

extern "C" int ag_relu_backward(int64_t n, const float *h, float *g, void *stream) {
  if (n == 0) return AG_OK;
  relu_bwd_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, h, g);
  AG_LAUNCH_CHECK("relu_bwd_kernel");
  return AG_OK;
}

extern "C" int ag_sgd_step(int64_t n, float *w, const float *dw, float lr, void *stream) {
  if (n == 0) return AG_OK;
  sgd_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, w, dw, lr);
  AG_LAUNCH_CHECK("sgd_kernel");
  return AG_OK;
}
