// Aggregation kernels K1-K5 of the AdaptGear path on sm_100a.
//
//   K1 ag_csr_spmm        aggregate_csr_inter          kernels.py:87-134
//   K2 ag_csr_intra_spmm  aggregate_csr_intra_blocked  kernels.py:137-189
//   K3 ag_coo_spmm        aggregate_coo_atomic         kernels.py:192-225
//   K4 ag_dense_block_spmm aggregate_dense_block       kernels.py:228-250
//   K5 ag_combine         combine                      kernels.py:253-276
//
// Floating-point contract of K1/K2 (bitwise equal to the reference):
// the reference reduces each CSR row with np.add.reduceat over
// contrib = fl(val * x[col]) (kernels.py:112-113, :187-188).  For a segment
// c[0..m) numpy computes  c[0] + P(c[1..m))  where P is numpy's pairwise sum:
//   n < 8     r = -0.0; r += a[i] sequentially
//   n <= 128  8 accumulators r[j] = a[j], r[j] += a[i+j] for full groups of 8,
//             ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n%8 tail in order
//   n > 128   m = n/2 rounded down to a multiple of 8; P(a[:m]) + P(a[m:])
// Every operation below is an explicit round-to-nearest intrinsic (__fmul_rn /
// __fadd_rn) so nvcc cannot contract it into an FMA.  The leaves of the
// pairwise tree hold 8 independent gathers each, which is also what keeps
// enough loads in flight to saturate HBM.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

#include "ag_common.cuh"
#include "ag_vec.cuh"

namespace ag {
namespace {
using namespace vec;

constexpr int kBlock = 256;
constexpr int kLeaf = 128;      // numpy PW_BLOCKSIZE
constexpr int kMaxDepth = 40;   // pairwise recursion depth bound (n < 2^31)

// Where the gathered source rows live: global X (K1) or a shared-memory slab
// of one community (K2).  row(c) returns a pointer to feature f of source c.
struct GlobalSrc {
  const float *x;
  int64_t ld;
  __device__ __forceinline__ const float *at(int32_t c, int f) const {
    return x + static_cast<int64_t>(c) * ld + f;
  }
};
struct SharedSrc {
  const float *slab;  // [B][ld]
  int32_t base;       // first source id of the community
  int ld;
  int f0;             // first feature of the staged tile
  __device__ __forceinline__ const float *at(int32_t c, int f) const {
    return slab + (c - base) * ld + (f - f0);
  }
};

template <int VEC, class Src>
__device__ __forceinline__ Vf<VEC> load_src(const Src &src, int32_t c, int f) {
  if constexpr (std::is_same<Src, GlobalSrc>::value) {
    return ldv<VEC>(src.at(c, f));
  } else {
    Vf<VEC> r;
    const float *p = src.at(c, f);
#pragma unroll
    for (int i = 0; i < VEC; ++i) r.v[i] = p[i];
    return r;
  }
}

// contrib(k) = fl(val[k] * x[col[k]])   (kernels.py:112: a.val[...,None] * x[cols])
template <int VEC, class Src>
__device__ __forceinline__ Vf<VEC> contrib(const Src &src, const int32_t *__restrict__ col,
                                           const float *__restrict__ val, int64_t k, int f) {
  int32_t c = __ldg(col + k);
  Vf<VEC> xv = load_src<VEC>(src, c, f);
  if (val != nullptr) xv = vscale<VEC>(__ldg(val + k), xv);
  return xv;
}

// One numpy pairwise leaf over a[start .. start+n), n <= 128.  For n < 8 this
// is numpy's sequential branch (r = -0.0; r += a[i]), which is exactly the
// "tail" part of the n >= 8 branch started from -0.0.
template <int VEC, class Src>
__device__ __forceinline__ Vf<VEC> pw_leaf(const Src &src, const int32_t *__restrict__ col,
                                           const float *__restrict__ val, int64_t start, int n,
                                           int f) {
  Vf<VEC> res = splat<VEC>(-0.0f);
  int m = 0;
  if (n >= 8) {
    Vf<VEC> r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = contrib<VEC>(src, col, val, start + j, f);
    m = n - (n & 7);
    for (int i = 8; i < m; i += 8) {
      int32_t cc[8];
      float cv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cc[j] = __ldg(col + start + i + j);
        cv[j] = val ? __ldg(val + start + i + j) : 1.0f;
      }
      Vf<VEC> c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = load_src<VEC>(src, cc[j], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (val) c[j] = vscale<VEC>(cv[j], c[j]);
        r[j] = vadd<VEC>(r[j], c[j]);
      }
    }
    res = vadd<VEC>(vadd<VEC>(vadd<VEC>(r[0], r[1]), vadd<VEC>(r[2], r[3])),
                    vadd<VEC>(vadd<VEC>(r[4], r[5]), vadd<VEC>(r[6], r[7])));
  }
  const int tail = n - m;
  Vf<VEC> c[7];
#pragma unroll
  for (int t = 0; t < 7; ++t)
    if (t < tail) c[t] = contrib<VEC>(src, col, val, start + m + t, f);
#pragma unroll
  for (int t = 0; t < 7; ++t)
    if (t < tail) res = vadd<VEC>(res, c[t]);
  return res;
}

// numpy pairwise_sum over a[start .. start+n): explicit post-order walk of the
// recursion tree (split at n/2 rounded down to a multiple of 8 above 128), so
// the leaf code is instantiated once.  The frame stack lives in local memory
// and is only touched once per leaf (>= 57 edges apart).
template <int VEC, class Src>
__device__ __noinline__ Vf<VEC> pw_sum(const Src src, const int32_t *__restrict__ col,
                                       const float *__restrict__ val, int64_t start, int n,
                                       int f) {
  int64_t st_start[kMaxDepth];
  int st_n[kMaxDepth];
  int st_stage[kMaxDepth];
  Vf<VEC> st_left[kMaxDepth];
  int sp = 0;
  st_start[0] = start;
  st_n[0] = n;
  st_stage[0] = 0;
  Vf<VEC> ret = splat<VEC>(0.0f);
  while (sp >= 0) {
    const int cn = st_n[sp];
    if (cn <= kLeaf) {
      ret = pw_leaf<VEC>(src, col, val, st_start[sp], cn, f);
      --sp;
      continue;
    }
    int n2 = cn / 2;
    n2 -= n2 & 7;
    const int stage = st_stage[sp];
    if (stage == 0) {
      st_stage[sp] = 1;
      st_start[sp + 1] = st_start[sp];
      st_n[sp + 1] = n2;
      st_stage[sp + 1] = 0;
      ++sp;
    } else if (stage == 1) {
      st_left[sp] = ret;
      st_stage[sp] = 2;
      st_start[sp + 1] = st_start[sp] + n2;
      st_n[sp + 1] = cn - n2;
      st_stage[sp + 1] = 0;
      ++sp;
    } else {
      ret = vadd<VEC>(st_left[sp], ret);
      --sp;
    }
  }
  return ret;
}

// Row reduction for one (row, feature chunk): sum/mean -> reduceat order,
// max -> plain max over raw source rows (weights ignored, kernels.py:108-110).
template <int VEC, bool IS_MAX, class Src>
__device__ __forceinline__ Vf<VEC> reduce_row(const Src &src, const int32_t *__restrict__ col,
                                              const float *__restrict__ val, int64_t s, int64_t e,
                                              int f) {
  const int64_t m = e - s;
  if (m <= 0) return splat<VEC>(0.0f);
  if constexpr (IS_MAX) {
    Vf<VEC> r[4];
    r[0] = load_src<VEC>(src, __ldg(col + s), f);
    r[1] = r[0]; r[2] = r[0]; r[3] = r[0];
    int64_t k = s + 1;
    for (; k + 4 <= e; k += 4) {
      Vf<VEC> c[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] = load_src<VEC>(src, __ldg(col + k + j), f);
#pragma unroll
      for (int j = 0; j < 4; ++j) r[j] = vmax<VEC>(r[j], c[j]);
    }
    for (; k < e; ++k) r[0] = vmax<VEC>(r[0], load_src<VEC>(src, __ldg(col + k), f));
    return vmax<VEC>(vmax<VEC>(r[0], r[1]), vmax<VEC>(r[2], r[3]));
  } else {
    Vf<VEC> c0 = contrib<VEC>(src, col, val, s, f);
    if (m == 1) return c0;
    Vf<VEC> p = pw_sum<VEC>(src, col, val, s + 1, static_cast<int>(m - 1), f);
    return vadd<VEC>(c0, p);
  }
}

// ---------------------------------------------------------------- K1: CSR --
struct CsrArgs {
  int64_t rows;
  int64_t feat;
  const int32_t *row_ptr;
  const int32_t *col;
  const float *val;
  const float *x;
  float *y;
  Epi ep;
};

template <int VEC, int LANES, bool IS_MAX>
__global__ void __launch_bounds__(kBlock) csr_spmm_kernel(CsrArgs a) {
  const int lane = threadIdx.x % LANES;
  const int64_t group = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / LANES;
  const int64_t ngroups = static_cast<int64_t>(gridDim.x) * (kBlock / LANES);
  const int tile = LANES * VEC;
  GlobalSrc src{a.x, a.feat};
  for (int64_t r = group; r < a.rows; r += ngroups) {
    const int64_t s = a.row_ptr[r];
    const int64_t e = a.row_ptr[r + 1];
    for (int f0 = 0; f0 < a.feat; f0 += tile) {
      const int f = f0 + lane * VEC;
      if (f >= a.feat) continue;
      Vf<VEC> acc = reduce_row<VEC, IS_MAX>(src, a.col, a.val, s, e, f);
      epilogue_store<VEC>(a.ep, a.y, r, f, acc, e > s);
    }
  }
}

// ------------------------------------------------- K2: intra-block CSR ------
struct IntraArgs {
  int64_t rows;
  int64_t feat;
  int block;     // B
  int ftile;     // staged feature columns per pass (multiple of VEC)
  const int32_t *row_ptr;
  const int32_t *col;
  const float *val;
  const float *x;
  float *y;
  Epi ep;
};

template <int VEC, int LANES, bool IS_MAX>
__global__ void __launch_bounds__(kBlock) csr_intra_kernel(IntraArgs a) {
  extern __shared__ __align__(16) float slab[];
  const int64_t ncomm = (a.rows + a.block - 1) / a.block;
  const int lane = threadIdx.x % LANES;
  const int grp = threadIdx.x / LANES;
  const int ngrp = kBlock / LANES;
  const int tile = LANES * VEC;
  for (int64_t c = blockIdx.x; c < ncomm; c += gridDim.x) {
    const int64_t r0 = c * a.block;
    const int nr = static_cast<int>(::min((int64_t)a.block, a.rows - r0));
    for (int f0 = 0; f0 < a.feat; f0 += a.ftile) {
      const int fw = static_cast<int>(::min((int64_t)a.ftile, a.feat - f0));
      // stage the community's [nr x fw] source slab (kernels.py:180-181)
      __syncthreads();
      const int vec_per_row = fw / VEC;
      for (int idx = threadIdx.x; idx < nr * vec_per_row; idx += kBlock) {
        const int i = idx / vec_per_row;
        const int j = (idx - i * vec_per_row) * VEC;
        Vf<VEC> v = ldv<VEC>(a.x + (r0 + i) * a.feat + f0 + j);
        float *d = slab + i * a.ftile + j;
#pragma unroll
        for (int t = 0; t < VEC; ++t) d[t] = v.v[t];
      }
      __syncthreads();
      SharedSrc src{slab, static_cast<int32_t>(r0), a.ftile, f0};
      for (int i = grp; i < nr; i += ngrp) {
        const int64_t r = r0 + i;
        const int64_t s = a.row_ptr[r];
        const int64_t e = a.row_ptr[r + 1];
        for (int fs = 0; fs < fw; fs += tile) {
          const int f = f0 + fs + lane * VEC;
          if (fs + lane * VEC >= fw) continue;
          Vf<VEC> acc = reduce_row<VEC, IS_MAX>(src, a.col, a.val, s, e, f);
          epilogue_store<VEC>(a.ep, a.y, r, f, acc, e > s);
        }
      }
    }
  }
}

// ----------------------------------------------------------- K3: COO -------
struct CooArgs {
  int64_t feat;
  int64_t nnz;
  int chunk;  // edges per group
  const int32_t *row;
  const int32_t *col;
  const float *val;
  const float *x;
  float *y;
};

__device__ __forceinline__ void atomic_max_f32(float *addr, float v) {
  // order-preserving integer mapping; y starts at -inf (kernels.py:212-214)
  if (v >= 0.0f) {
    atomicMax(reinterpret_cast<int *>(addr), __float_as_int(v));
  } else {
    atomicMin(reinterpret_cast<unsigned int *>(addr), __float_as_uint(v));
  }
}

template <int VEC, bool IS_MAX>
__device__ __forceinline__ void coo_flush(float *p, const Vf<VEC> &acc) {
  if constexpr (IS_MAX) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) atomic_max_f32(p + i, acc.v[i]);
  } else if constexpr (VEC == 4) {
    atomicAdd(reinterpret_cast<float4 *>(p), make_float4(acc.v[0], acc.v[1], acc.v[2], acc.v[3]));
  } else if constexpr (VEC == 2) {
    atomicAdd(reinterpret_cast<float2 *>(p), make_float2(acc.v[0], acc.v[1]));
  } else {
    atomicAdd(p, acc.v[0]);
  }
}

template <int VEC, int LANES, bool IS_MAX>
__global__ void __launch_bounds__(kBlock) coo_spmm_kernel(CooArgs a) {
  const int lane = threadIdx.x % LANES;
  const int64_t group = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / LANES;
  const int64_t ngroups = static_cast<int64_t>(gridDim.x) * (kBlock / LANES);
  const int tile = LANES * VEC;
  const int64_t nchunks = (a.nnz + a.chunk - 1) / a.chunk;
  for (int64_t ch = group; ch < nchunks; ch += ngroups) {
    const int64_t e0 = ch * a.chunk;
    const int64_t e1 = ::min((int64_t)e0 + a.chunk, a.nnz);
    for (int f0 = 0; f0 < a.feat; f0 += tile) {
      const int f = f0 + lane * VEC;
      if (f >= a.feat) continue;
      int32_t cur = __ldg(a.row + e0);
      Vf<VEC> acc = splat<VEC>(IS_MAX ? -__int_as_float(0x7f800000) : 0.0f);
      int64_t k = e0;
      for (; k < e1; k += 4) {
        int32_t rr[4];
        Vf<VEC> c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (k + j < e1) {
            rr[j] = __ldg(a.row + k + j);
            c[j] = ldv<VEC>(a.x + static_cast<int64_t>(__ldg(a.col + k + j)) * a.feat + f);
            if (!IS_MAX && a.val) c[j] = vscale<VEC>(__ldg(a.val + k + j), c[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (k + j < e1) {
            if (rr[j] != cur) {
              coo_flush<VEC, IS_MAX>(a.y + static_cast<int64_t>(cur) * a.feat + f, acc);
              cur = rr[j];
              acc = splat<VEC>(IS_MAX ? -__int_as_float(0x7f800000) : 0.0f);
            }
            acc = IS_MAX ? vmax<VEC>(acc, c[j]) : vadd<VEC>(acc, c[j]);
          }
        }
      }
      coo_flush<VEC, IS_MAX>(a.y + static_cast<int64_t>(cur) * a.feat + f, acc);
    }
  }
}

// ------------------------------------- K3 as a row gather (sum / mean) -----
// coo_atomic leaves the summation order open (the reference accumulates in
// fp64 bincount over scrambled edges, kernels.py:192-225, tested at 1e-4), and
// its COO is dst-sorted, so each destination's edges are one contiguous run.
// LANES lanes own a row (VEC columns each), load its (col, val) run LANES at a
// time coalesced, and gather 8 source rows per step with all 8 loads in flight,
// accumulating in registers: no atomics, one store per row.  For graphs whose
// sources are far apart (C4: every row reads ~300 rows spread over 16k) this is
// an L2 gather; the atomic kernel below stays for max.
template <int VEC, int LANES>
__global__ void __launch_bounds__(kBlock) coo_gather_kernel(int64_t rows, int64_t feat,
                                                            const int32_t *row_ptr,
                                                            const int32_t *col, const float *val,
                                                            const float *x, float *y) {
  const int sub = threadIdx.x & 31;
  const int lane = sub % LANES;
  const unsigned gmask =
      LANES == 32 ? 0xffffffffu : (((1u << LANES) - 1u) << (sub / LANES * LANES));
  const int64_t grp = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / LANES;
  const int64_t ngrp = static_cast<int64_t>(gridDim.x) * (kBlock / LANES);
  const int tile = LANES * VEC;
  for (int64_t r = grp; r < rows; r += ngrp) {
    const int32_t s = __ldg(row_ptr + r), e = __ldg(row_ptr + r + 1);
    for (int f0 = 0; f0 < feat; f0 += tile) {
      const int64_t f = f0 + lane * VEC;
      const bool act = f < feat;
      Vf<VEC> a0 = splat<VEC>(0.0f), a1 = a0;
      for (int32_t b = s; b < e; b += LANES) {
        int32_t mc = 0;
        float mv = 0.0f;
        if (b + lane < e) {
          mc = __ldg(col + b + lane);
          mv = val ? __ldg(val + b + lane) : 1.0f;
        }
        const int n = e - b < LANES ? e - b : LANES;
        for (int j = 0; j < n; j += 8) {
          Vf<VEC> xv[8];
          float w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int jj = j + u;
            const int32_t c = __shfl_sync(gmask, mc, jj, LANES);
            w[u] = __shfl_sync(gmask, mv, jj, LANES);
            xv[u] = (jj < n && act) ? ldv<VEC>(x + static_cast<int64_t>(c) * feat + f)
                                    : splat<VEC>(0.0f);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (j + u < n) {
              Vf<VEC> &acc = (u & 1) ? a1 : a0;
#pragma unroll
              for (int i = 0; i < VEC; ++i) acc.v[i] = fmaf(xv[u].v[i], w[u], acc.v[i]);
            }
          }
        }
      }
      if (act) stv<VEC>(y + r * feat + f, vadd<VEC>(a0, a1));
    }
  }
}

// ------------------- small graphs: the (dense_block, coo_atomic) pair as a gather --
// Both roles of that selector pair are order-free (the dense block product is a
// BLAS matmul, kernels.py:247; coo_atomic a scrambled bincount), so on a graph
// whose features fit L2 the pair runs as ONE row gather over the full CSR: a
// LANES-lane group per row (4 columns per lane), 8 source loads in flight,
// then the fused epilogue -- GIN (1 + eps) x, ReLU (+ its bit mask), or the
// ReLU-backward mask -- and one store.  The slab kernel's pipeline start-up
// (tens of microseconds filling the X ring) dominates such graphs.
template <int LANES, int NV>
__global__ void __launch_bounds__(kBlock) gather_pair_kernel(
    int64_t rows, int64_t feat, const int32_t *row_ptr, const int32_t *col, const float *val,
    const float *x, float *y, int32_t flags, float gin_scale, const uint32_t *relu_bits,
    uint32_t *relu_out, int64_t ldw) {
  // NV float4 chunks per lane per pass (chunk k covers columns f0 + 4 (lane + k LANES))
  constexpr int VEC = 4;
  const int sub = threadIdx.x & 31;
  const int lane = sub % LANES;
  const unsigned gmask =
      LANES == 32 ? 0xffffffffu : (((1u << LANES) - 1u) << (sub / LANES * LANES));
  const int64_t grp = (static_cast<int64_t>(blockIdx.x) * kBlock + threadIdx.x) / LANES;
  const int64_t ngrp = static_cast<int64_t>(gridDim.x) * (kBlock / LANES);
  const int tile = LANES * VEC * NV;
  for (int64_t r = grp; r < rows; r += ngrp) {
    const int32_t s = __ldg(row_ptr + r), e = __ldg(row_ptr + r + 1);
    for (int f0 = 0; f0 < feat; f0 += tile) {
      int64_t f[NV];
      bool act[NV];
      Vf<VEC> a0[NV], a1[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        f[k] = f0 + (lane + k * LANES) * VEC;
        act[k] = f[k] < feat;
        a0[k] = splat<VEC>(0.0f);
        a1[k] = a0[k];
      }
      for (int32_t b = s; b < e; b += LANES) {
        int32_t mc = 0;
        float mv = 0.0f;
        if (b + lane < e) {
          mc = __ldg(col + b + lane);
          mv = val ? __ldg(val + b + lane) : 1.0f;
        }
        const int n = e - b < LANES ? e - b : LANES;
        for (int j = 0; j < n; j += 8) {
          Vf<VEC> xv[8][NV];
          float w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int jj = j + u;
            const int32_t c = __shfl_sync(gmask, mc, jj, LANES);
            w[u] = __shfl_sync(gmask, mv, jj, LANES);
            const float *xr = x + static_cast<int64_t>(c) * feat;
#pragma unroll
            for (int k = 0; k < NV; ++k)
              xv[u][k] = (jj < n && act[k]) ? ldv<VEC>(xr + f[k]) : splat<VEC>(0.0f);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (j + u < n) {
#pragma unroll
              for (int k = 0; k < NV; ++k) {
                Vf<VEC> &acc = (u & 1) ? a1[k] : a0[k];
#pragma unroll
                for (int i = 0; i < VEC; ++i) acc.v[i] = fmaf(xv[u][k].v[i], w[u], acc.v[i]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        Vf<VEC> o = vadd<VEC>(a0[k], a1[k]);
        if ((flags & AG_EPI_GIN) && act[k]) {
          const Vf<VEC> xr = ldv<VEC>(x + r * feat + f[k]);
#pragma unroll
          for (int i = 0; i < VEC; ++i) o.v[i] = fmaf(gin_scale, xr.v[i], o.v[i]);
        }
        if (flags & AG_EPI_RELU) {
#pragma unroll
          for (int i = 0; i < VEC; ++i) o.v[i] = fmaxf(o.v[i], 0.0f);
        }
        if ((flags & AG_EPI_RELU_MASK) && act[k]) {
          const uint32_t nib = (__ldg(relu_bits + r * ldw + (f[k] >> 5)) >> (f[k] & 31)) & 15u;
#pragma unroll
          for (int i = 0; i < VEC; ++i)
            if (!((nib >> i) & 1u)) o.v[i] = 0.0f;
        }
        if (relu_out != nullptr) {  // 8 lanes x 4 columns = one mask word
          uint32_t wd = 0;
#pragma unroll
          for (int i = 0; i < VEC; ++i)
            if (act[k] && f[k] + i < feat && o.v[i] > 0.0f) wd |= 1u << (4 * (lane & 7) + i);
          if constexpr (LANES >= 8) {
            wd |= __shfl_xor_sync(gmask, wd, 1, LANES);
            wd |= __shfl_xor_sync(gmask, wd, 2, LANES);
            wd |= __shfl_xor_sync(gmask, wd, 4, LANES);
            if ((lane & 7) == 0 && act[k]) relu_out[r * ldw + (f[k] >> 5)] = wd;
          } else {  // fewer than 8 lanes (NV = 1): the group's lanes share one word
#pragma unroll
            for (int o2 = 1; o2 < LANES; o2 <<= 1) wd |= __shfl_xor_sync(gmask, wd, o2, LANES);
            if (lane == 0) relu_out[r * ldw + (f0 >> 5)] = wd;
          }
        }
        if (act[k]) stv<VEC>(y + r * feat + f[k], o);
      }
    }
  }
}

// ---------------------------------------------------- K4: dense blocks -----
struct DenseArgs {
  int64_t rows;
  int64_t feat;
  int block;
  const int32_t *comm_slot;
  const float *blocks;
  const uint8_t *row_touched;
  const float *x;
  float *y;
  Epi ep;
};

constexpr int kDenseRows = 16;  // output rows held in registers per pass

__global__ void __launch_bounds__(kBlock) dense_block_kernel(DenseArgs a) {
  extern __shared__ __align__(16) float sblk[];  // [kDenseRows][B]
  const int B = a.block;
  const int64_t ncomm = (a.rows + B - 1) / B;
  for (int64_t c = blockIdx.x; c < ncomm; c += gridDim.x) {
    const int64_t r0 = c * B;
    const int nr = static_cast<int>(::min((int64_t)B, a.rows - r0));
    const int slot = a.comm_slot[c];
    const float *blk = slot >= 0 ? a.blocks + static_cast<int64_t>(slot) * B * B : nullptr;
    for (int i0 = 0; i0 < nr; i0 += kDenseRows) {
      const int ni = min(kDenseRows, nr - i0);
      __syncthreads();
      if (blk) {
        for (int t = threadIdx.x; t < ni * B; t += blockDim.x) sblk[t] = blk[i0 * B + t];
      }
      __syncthreads();
      for (int64_t f = threadIdx.x; f < a.feat; f += blockDim.x) {
        float acc[kDenseRows];
#pragma unroll
        for (int i = 0; i < kDenseRows; ++i) acc[i] = 0.0f;
        if (blk) {
          for (int j = 0; j < nr; ++j) {  // padded rows j >= nr contribute 0
            const float xv = __ldg(a.x + (r0 + j) * a.feat + f);
#pragma unroll
            for (int i = 0; i < kDenseRows; ++i)
              if (i < ni) acc[i] = fmaf(sblk[i * B + j], xv, acc[i]);
          }
        }
        for (int i = 0; i < ni; ++i) {
          const bool touched = blk ? a.row_touched[static_cast<int64_t>(slot) * B + i0 + i] != 0 : false;
          Vf<1> v;
          v.v[0] = acc[i];
          epilogue_store<1>(a.ep, a.y, r0 + i0 + i, static_cast<int>(f), v, touched);
        }
      }
    }
  }
}

// ---------------------------------------------------------- K5: combine ----
__global__ void combine_kernel(int64_t rows, int64_t feat, const float *a, const uint8_t *ta,
                               const float *b, const uint8_t *tb, const int64_t *deg, int op,
                               float *out) {
  const int64_t n = rows * feat;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / feat;
    const float va = a[i], vb = b[i];
    float o;
    if (op == AG_OP_SUM) {
      o = __fadd_rn(va, vb);
    } else if (op == AG_OP_MEAN) {
      int64_t d = deg[r];
      if (d < 1) d = 1;
      o = __fdiv_rn(__fadd_rn(va, vb), static_cast<float>(d));
    } else {
      const bool x = ta[r] != 0, y = tb[r] != 0;
      o = (x && y) ? fmaxf(va, vb) : x ? va : y ? vb : 0.0f;
    }
    out[i] = o;
  }
}

// ------------------------------------------------------------ dispatch -----
inline int pick_vec(int64_t feat, const void *x, const void *y) {
  auto al = [](const void *p, int b) { return (reinterpret_cast<uintptr_t>(p) % b) == 0; };
  if (feat % 4 == 0 && al(x, 16) && al(y, 16)) return 4;
  if (feat % 2 == 0 && al(x, 8) && al(y, 8)) return 2;
  return 1;
}

inline int pick_lanes(int64_t chunks) {
  if (chunks <= 4) return 4;
  if (chunks <= 8) return 8;
  if (chunks <= 16) return 16;
  return 32;
}

template <class K>
int resident_grid(K kernel, size_t smem, int64_t work_blocks) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBlock, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t g = static_cast<int64_t>(sm_count()) * per_sm;
  if (work_blocks < g) g = work_blocks;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

template <int VEC, int LANES>
int launch_coo_gather(int64_t rows, int64_t feat, const int32_t *row_ptr, const int32_t *col,
                      const float *val, const float *x, float *y, cudaStream_t st) {
  auto k = coo_gather_kernel<VEC, LANES>;
  const int64_t work = (rows * LANES + kBlock - 1) / kBlock;
  k<<<resident_grid(k, 0, work), kBlock, 0, st>>>(rows, feat, row_ptr, col, val, x, y);
  AG_LAUNCH_CHECK("coo_gather_kernel");
  return AG_OK;
}

template <int VEC>
int launch_coo_gather_vec(int64_t rows, int64_t feat, const int32_t *row_ptr,
                          const int32_t *col, const float *val, const float *x, float *y,
                          cudaStream_t st) {
  switch (pick_lanes((feat + VEC - 1) / VEC)) {
    case 4: return launch_coo_gather<VEC, 4>(rows, feat, row_ptr, col, val, x, y, st);
    case 8: return launch_coo_gather<VEC, 8>(rows, feat, row_ptr, col, val, x, y, st);
    case 16: return launch_coo_gather<VEC, 16>(rows, feat, row_ptr, col, val, x, y, st);
    default: return launch_coo_gather<VEC, 32>(rows, feat, row_ptr, col, val, x, y, st);
  }
}

template <int LANES, int NV = 1>
int launch_gather_pair(int64_t rows, int64_t feat, const int32_t *row_ptr, const int32_t *col,
                       const float *val, const float *x, float *y, int32_t flags, float gin,
                       const uint32_t *rb, uint32_t *ro, cudaStream_t st) {
  auto k = gather_pair_kernel<LANES, NV>;
  const int64_t work = (rows * LANES + kBlock - 1) / kBlock;
  k<<<resident_grid(k, 0, work), kBlock, 0, st>>>(rows, feat, row_ptr, col, val, x, y, flags, gin,
                                                   rb, ro, relu_words(feat));
  AG_LAUNCH_CHECK("gather_pair_kernel");
  return AG_OK;
}

template <int VEC, int LANES>
int launch_csr(const CsrArgs &a, bool is_max, cudaStream_t st) {
  const int64_t work = (a.rows * LANES + kBlock - 1) / kBlock;
  if (is_max) {
    auto k = csr_spmm_kernel<VEC, LANES, true>;
    k<<<resident_grid(k, 0, work), kBlock, 0, st>>>(a);
  } else {
    auto k = csr_spmm_kernel<VEC, LANES, false>;
    k<<<resident_grid(k, 0, work), kBlock, 0, st>>>(a);
  }
  AG_LAUNCH_CHECK("csr_spmm_kernel");
  return AG_OK;
}

template <int VEC>
int launch_csr_vec(const CsrArgs &a, bool is_max, cudaStream_t st) {
  switch (pick_lanes((a.feat + VEC - 1) / VEC)) {
    case 4: return launch_csr<VEC, 4>(a, is_max, st);
    case 8: return launch_csr<VEC, 8>(a, is_max, st);
    case 16: return launch_csr<VEC, 16>(a, is_max, st);
    default: return launch_csr<VEC, 32>(a, is_max, st);
  }
}

template <int VEC, int LANES>
int launch_intra(const IntraArgs &a, bool is_max, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(a.block) * a.ftile * sizeof(float);
  const int64_t ncomm = (a.rows + a.block - 1) / a.block;
  if (is_max) {
    auto k = csr_intra_kernel<VEC, LANES, true>;
    AG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<resident_grid(k, smem, ncomm), kBlock, smem, st>>>(a);
  } else {
    auto k = csr_intra_kernel<VEC, LANES, false>;
    AG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<resident_grid(k, smem, ncomm), kBlock, smem, st>>>(a);
  }
  AG_LAUNCH_CHECK("csr_intra_kernel");
  return AG_OK;
}

template <int VEC>
int launch_intra_vec(const IntraArgs &a, bool is_max, cudaStream_t st) {
  switch (pick_lanes((a.ftile + VEC - 1) / VEC)) {
    case 4: return launch_intra<VEC, 4>(a, is_max, st);
    case 8: return launch_intra<VEC, 8>(a, is_max, st);
    case 16: return launch_intra<VEC, 16>(a, is_max, st);
    default: return launch_intra<VEC, 32>(a, is_max, st);
  }
}

template <int VEC, int LANES>
int launch_coo(const CooArgs &a, bool is_max, cudaStream_t st) {
  const int64_t nchunks = (a.nnz + a.chunk - 1) / a.chunk;
  const int64_t work = (nchunks * LANES + kBlock - 1) / kBlock;
  if (is_max) {
    auto k = coo_spmm_kernel<VEC, LANES, true>;
    k<<<resident_grid(k, 0, work), kBlock, 0, st>>>(a);
  } else {
    auto k = coo_spmm_kernel<VEC, LANES, false>;
    k<<<resident_grid(k, 0, work), kBlock, 0, st>>>(a);
  }
  AG_LAUNCH_CHECK("coo_spmm_kernel");
  return AG_OK;
}

template <int VEC>
int launch_coo_vec(const CooArgs &a, bool is_max, cudaStream_t st) {
  switch (pick_lanes((a.feat + VEC - 1) / VEC)) {
    case 4: return launch_coo<VEC, 4>(a, is_max, st);
    case 8: return launch_coo<VEC, 8>(a, is_max, st);
    case 16: return launch_coo<VEC, 16>(a, is_max, st);
    default: return launch_coo<VEC, 32>(a, is_max, st);
  }
}

int check_common(int64_t rows, int64_t feat, int32_t op, int32_t flags, const int64_t *deg) {
  if (rows < 0 || feat < 0) return fail(AG_ERR_VALUE, "negative sizes (rows=%lld, feat=%lld)",
                                        (long long)rows, (long long)feat);
  if (op < AG_OP_SUM || op > AG_OP_MAX) return fail(AG_ERR_KERNEL, "unknown op %d", op);
  if ((flags & AG_EPI_COMBINE) && op == AG_OP_MEAN && deg == nullptr)
    return fail(AG_ERR_KERNEL, "mean combine requires the full-graph degree vector");
  return AG_OK;
}

}  // namespace
}  // namespace ag

using namespace ag;

extern "C" int ag_csr_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                           const int32_t *col_idx, const float *val, const float *x, float *y,
                           int32_t op, int32_t epi_flags, const uint8_t *other_touched,
                           const int64_t *deg, float gin_scale, void *stream) {
  if (int rc = check_common(num_rows, feat, op, epi_flags, deg)) return rc;
  if (num_rows == 0 || feat == 0) return AG_OK;
  CsrArgs a{num_rows, feat, row_ptr, col_idx, val, x, y,
            Epi{op, epi_flags, other_touched, deg, x, feat, gin_scale}};
  const bool is_max = op == AG_OP_MAX;
  cudaStream_t st = as_stream(stream);
  switch (pick_vec(feat, x, y)) {
    case 4: return launch_csr_vec<4>(a, is_max, st);
    case 2: return launch_csr_vec<2>(a, is_max, st);
    default: return launch_csr_vec<1>(a, is_max, st);
  }
}

extern "C" int ag_csr_intra_spmm(int64_t num_rows, int64_t feat, int64_t block_size,
                                 int64_t tile_budget_bytes, const int32_t *row_ptr,
                                 const int32_t *col_idx, const float *val, const float *x,
                                 float *y, int32_t op, int32_t epi_flags,
                                 const uint8_t *other_touched, const int64_t *deg,
                                 float gin_scale, void *stream) {
  if (int rc = check_common(num_rows, feat, op, epi_flags, deg)) return rc;
  if (block_size < 1) return fail(AG_ERR_KERNEL, "block_size must be >= 1");
  if (num_rows == 0 || feat == 0) return AG_OK;
  const int vec = pick_vec(feat, x, y);
  // F tile as in kernels.py:169-171, rounded to the vector width and capped
  // by what one CTA can stage (the tiling never changes the values).
  int64_t ftile = (block_size * feat * 4 <= tile_budget_bytes)
                      ? feat
                      : std::max<int64_t>(1, tile_budget_bytes / (block_size * 4));
  const int64_t smem_cap = 200 * 1024;
  const int64_t cap_cols = std::max<int64_t>(1, smem_cap / (block_size * 4));
  ftile = std::min(ftile, cap_cols);
  int v = vec;
  while (v > 1 && ftile % v != 0 && ftile > v) --v;
  if (ftile < v) v = 1;
  if (v == 3) v = 2;
  if (ftile % v != 0) ftile -= ftile % v;
  if (ftile < 1) ftile = 1;
  if (block_size * 4 > smem_cap)
    return fail(AG_ERR_KERNEL, "block_size %lld too large for the staged intra kernel",
                (long long)block_size);
  IntraArgs a{num_rows, feat, static_cast<int>(block_size), static_cast<int>(ftile), row_ptr,
              col_idx, val, x, y, Epi{op, epi_flags, other_touched, deg, x, feat, gin_scale}};
  const bool is_max = op == AG_OP_MAX;
  cudaStream_t st = as_stream(stream);
  switch (v) {
    case 4: return launch_intra_vec<4>(a, is_max, st);
    case 2: return launch_intra_vec<2>(a, is_max, st);
    default: return launch_intra_vec<1>(a, is_max, st);
  }
}

extern "C" int ag_coo_spmm(int64_t num_rows, int64_t feat, int64_t num_edges, const int32_t *row,
                           const int32_t *col, const float *val, const float *x, float *y,
                           int32_t op, void *stream) {
  if (int rc = check_common(num_rows, feat, op, 0, nullptr)) return rc;
  if (num_edges == 0 || feat == 0) return AG_OK;
  CooArgs a{feat, num_edges, 32, row, col, val, x, y};
  const bool is_max = op == AG_OP_MAX;
  cudaStream_t st = as_stream(stream);
  switch (pick_vec(feat, x, y)) {
    case 4: return launch_coo_vec<4>(a, is_max, st);
    case 2: return launch_coo_vec<2>(a, is_max, st);
    default: return launch_coo_vec<1>(a, is_max, st);
  }
}

extern "C" int ag_dense_block_spmm(int64_t num_rows, int64_t feat, int64_t block_size,
                                   const int32_t *comm_slot, const float *blocks,
                                   const uint8_t *row_touched, const float *x, float *y,
                                   int32_t op, int32_t epi_flags, const uint8_t *other_touched,
                                   const int64_t *deg, float gin_scale, void *stream) {
  if (int rc = check_common(num_rows, feat, op, epi_flags, deg)) return rc;
  if (op == AG_OP_MAX)
    return fail(AG_ERR_KERNEL, "dense_block kernel does not support max aggregation");
  if (block_size < 1) return fail(AG_ERR_KERNEL, "block_size must be >= 1");
  if (num_rows == 0 || feat == 0) return AG_OK;
  const size_t smem = static_cast<size_t>(kDenseRows) * block_size * sizeof(float);
  if (smem > 200 * 1024)
    return fail(AG_ERR_KERNEL, "block_size %lld too large for dense_block", (long long)block_size);
  DenseArgs a{num_rows, feat, static_cast<int>(block_size), comm_slot, blocks, row_touched, x, y,
              Epi{op, epi_flags, other_touched, deg, x, feat, gin_scale}};
  cudaStream_t st = as_stream(stream);
  AG_CUDA(cudaFuncSetAttribute(dense_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  const int64_t ncomm = (num_rows + block_size - 1) / block_size;
  dense_block_kernel<<<resident_grid(dense_block_kernel, smem, ncomm), kBlock, smem, st>>>(a);
  AG_LAUNCH_CHECK("dense_block_kernel");
  return AG_OK;
}

extern "C" int ag_combine(int64_t num_rows, int64_t feat, const float *a, const uint8_t *touched_a,
                          const float *b, const uint8_t *touched_b, const int64_t *deg, int32_t op,
                          float *out, void *stream) {
  if (int rc = check_common(num_rows, feat, op, 0, nullptr)) return rc;
  if (op == AG_OP_MEAN && deg == nullptr)
    return fail(AG_ERR_KERNEL, "mean combine requires the full-graph degree vector");
  if (num_rows * feat == 0) return AG_OK;
  combine_kernel<<<grid_for(num_rows * feat, 256), 256, 0, as_stream(stream)>>>(
      num_rows, feat, a, touched_a, b, touched_b, deg, op, out);
  AG_LAUNCH_CHECK("combine_kernel");
  return AG_OK;
}

extern "C" int ag_coo_gather_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                                  const int32_t *col, const float *val, const float *x, float *y,
                                  void *stream) {
  if (int rc = check_common(num_rows, feat, AG_OP_SUM, 0, nullptr)) return rc;
  if (num_rows == 0 || feat == 0) return AG_OK;
  if (row_ptr == nullptr) return fail(AG_ERR_VALUE, "row_ptr is required");
  cudaStream_t st = as_stream(stream);
  switch (pick_vec(feat, x, y)) {
    case 4: return launch_coo_gather_vec<4>(num_rows, feat, row_ptr, col, val, x, y, st);
    case 2: return launch_coo_gather_vec<2>(num_rows, feat, row_ptr, col, val, x, y, st);
    default: return launch_coo_gather_vec<1>(num_rows, feat, row_ptr, col, val, x, y, st);
  }
}

extern "C" int ag_gather_pair_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                                   const int32_t *col, const float *val, const float *x,
                                   float *y, int32_t epi_flags, float gin_scale,
                                   const uint32_t *relu_bits, uint32_t *relu_out, void *stream) {
  if (num_rows < 0 || feat < 0) return fail(AG_ERR_VALUE, "negative sizes");
  constexpr int32_t kFlags = AG_EPI_GIN | AG_EPI_RELU | AG_EPI_RELU_MASK;
  if (epi_flags & ~kFlags) return fail(AG_ERR_VALUE, "ag_gather_pair_spmm takes GIN / RELU / RELU_MASK");
  if ((epi_flags & AG_EPI_RELU_MASK) && relu_bits == nullptr)
    return fail(AG_ERR_VALUE, "AG_EPI_RELU_MASK needs relu_bits");
  if (relu_out != nullptr && !(epi_flags & AG_EPI_RELU))
    return fail(AG_ERR_VALUE, "relu_out is written with AG_EPI_RELU only");
  if (num_rows == 0 || feat == 0) return AG_OK;
  if (feat % 4 || (reinterpret_cast<uintptr_t>(x) & 15) || (reinterpret_cast<uintptr_t>(y) & 15))
    return fail(AG_ERR_VALUE, "ag_gather_pair_spmm needs feat % 4 == 0 and 16-byte aligned x / y");
  cudaStream_t st = as_stream(stream);
  switch (pick_lanes(feat / 4)) {
    case 4: return launch_gather_pair<4>(num_rows, feat, row_ptr, col, val, x, y, epi_flags,
                                         gin_scale, relu_bits, relu_out, st);
    case 8: return launch_gather_pair<8>(num_rows, feat, row_ptr, col, val, x, y, epi_flags,
                                         gin_scale, relu_bits, relu_out, st);
    case 16: return launch_gather_pair<16>(num_rows, feat, row_ptr, col, val, x, y, epi_flags,
                                           gin_scale, relu_bits, relu_out, st);
    default:
      // wider than 128 columns: two float4 chunks per lane per pass (256 columns)
      if (feat > 128)
        return launch_gather_pair<32, 2>(num_rows, feat, row_ptr, col, val, x, y, epi_flags,
                                         gin_scale, relu_bits, relu_out, st);
      return launch_gather_pair<32>(num_rows, feat, row_ptr, col, val, x, y, epi_flags,
                                    gin_scale, relu_bits, relu_out, st);
  }
}
