// Small vector helpers and the fused combine epilogue shared by the
// aggregation kernels (ag_spmm.cu, ag_fused.cu).  Every float operation is an
// explicit round-to-nearest intrinsic so nvcc never contracts into an FMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "adaptgear_b200.h"

namespace ag {
namespace vec {

template <int VEC>
struct Vf {
  float v[VEC];
};

template <int VEC>
__device__ __forceinline__ Vf<VEC> ldv(const float *p) {
  Vf<VEC> r;
  if constexpr (VEC == 4) {
    float4 t = __ldg(reinterpret_cast<const float4 *>(p));
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
  } else if constexpr (VEC == 2) {
    float2 t = __ldg(reinterpret_cast<const float2 *>(p));
    r.v[0] = t.x; r.v[1] = t.y;
  } else {
    r.v[0] = __ldg(p);
  }
  return r;
}

// Plain (coherent) load: used for y, which the same kernel writes.
template <int VEC>
__device__ __forceinline__ Vf<VEC> ldv_rw(const float *p) {
  Vf<VEC> r;
  if constexpr (VEC == 4) {
    float4 t = *reinterpret_cast<const float4 *>(p);
    r.v[0] = t.x; r.v[1] = t.y; r.v[2] = t.z; r.v[3] = t.w;
  } else if constexpr (VEC == 2) {
    float2 t = *reinterpret_cast<const float2 *>(p);
    r.v[0] = t.x; r.v[1] = t.y;
  } else {
    r.v[0] = *p;
  }
  return r;
}

template <int VEC>
__device__ __forceinline__ void stv(float *p, const Vf<VEC> &r) {
  if constexpr (VEC == 4) {
    *reinterpret_cast<float4 *>(p) = make_float4(r.v[0], r.v[1], r.v[2], r.v[3]);
  } else if constexpr (VEC == 2) {
    *reinterpret_cast<float2 *>(p) = make_float2(r.v[0], r.v[1]);
  } else {
    *p = r.v[0];
  }
}

template <int VEC>
__device__ __forceinline__ Vf<VEC> splat(float s) {
  Vf<VEC> r;
#pragma unroll
  for (int i = 0; i < VEC; ++i) r.v[i] = s;
  return r;
}

template <int VEC>
__device__ __forceinline__ Vf<VEC> vadd(const Vf<VEC> &a, const Vf<VEC> &b) {
  Vf<VEC> r;
#pragma unroll
  for (int i = 0; i < VEC; ++i) r.v[i] = __fadd_rn(a.v[i], b.v[i]);
  return r;
}

template <int VEC>
__device__ __forceinline__ Vf<VEC> vmax(const Vf<VEC> &a, const Vf<VEC> &b) {
  Vf<VEC> r;
#pragma unroll
  for (int i = 0; i < VEC; ++i) r.v[i] = fmaxf(a.v[i], b.v[i]);
  return r;
}

template <int VEC>
__device__ __forceinline__ Vf<VEC> vscale(float s, const Vf<VEC> &a) {
  Vf<VEC> r;
#pragma unroll
  for (int i = 0; i < VEC; ++i) r.v[i] = __fmul_rn(s, a.v[i]);
  return r;
}

struct Epi {
  int32_t op;
  int32_t flags;
  const uint8_t *other_touched;
  const int64_t *deg;
  const float *x;  // for the GIN term
  int64_t ld;      // row stride of x and y
  float gin_scale;
  const uint32_t *relu_bits = nullptr;  // AG_EPI_RELU_MASK: zero where the mask bit is 0
};

// combine() of kernels.py:253-276 fused into the producing kernel, plus the
// GIN (1+eps)*x term of models.py:111.
template <int VEC>
__device__ __forceinline__ void epilogue_store(const Epi &ep, float *y, int64_t r, int f,
                                               Vf<VEC> acc, bool touched) {
  float *yp = y + r * ep.ld + f;
  Vf<VEC> out;
  if (!(ep.flags & AG_EPI_COMBINE)) {
    out = touched ? acc : splat<VEC>(0.0f);
  } else {
    Vf<VEC> other = ldv_rw<VEC>(yp);
    if (ep.op == AG_OP_SUM) {
      out = vadd<VEC>(acc, other);
    } else if (ep.op == AG_OP_MEAN) {
      int64_t d = ep.deg ? ep.deg[r] : 1;
      if (d < 1) d = 1;
      const float df = static_cast<float>(d);
      Vf<VEC> s = vadd<VEC>(acc, other);
#pragma unroll
      for (int i = 0; i < VEC; ++i) out.v[i] = __fdiv_rn(s.v[i], df);
    } else {
      const bool ot = ep.other_touched ? (ep.other_touched[r] != 0) : false;
      if (touched && ot) out = vmax<VEC>(acc, other);
      else if (touched) out = acc;
      else if (ot) out = other;
      else out = splat<VEC>(0.0f);
    }
  }
  if (ep.flags & AG_EPI_GIN) {
    Vf<VEC> xv = ldv<VEC>(ep.x + r * ep.ld + f);
    out = vadd<VEC>(vscale<VEC>(ep.gin_scale, xv), out);
  }
  stv<VEC>(yp, out);
}

}  // namespace vec
}  // namespace ag
