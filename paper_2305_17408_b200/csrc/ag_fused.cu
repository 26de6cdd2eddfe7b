// Decomposed aggregation in one pass (the hot path of every GCN/GIN layer).
//
// For every destination row r of a CSR whose edges are stored in ROLE ORDER
// (intra run first, then the inter edges; ag_role_csr_build), one launch
// computes
//   I = intra-role value over edges [row_ptr[r], mid[r])
//   O = inter-role value over edges [mid[r], row_ptr[r+1])
//   y[r] = combine(I, O)  [+ (1+eps) x[r] for GIN]
// bit-for-bit what the reference computes with two CSR kernels and combine()
// (kernels.py:87-189, :253-276).  Each role is reduced in np.add.reduceat's
// order: c0 + P(c1..c_{n-1}) with c = fl(val * x[col]) and P numpy's pairwise
// sum (n < 8: sequential from -0.0; n <= 128: 8 strided accumulators, the
// tree ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail in order;
// n > 128: split at n/2 rounded down to a multiple of 8 and recurse).
//
// Work decomposition (sm_100a, HBM/L2-bound gather):
//  * The feature dimension is cut into column tiles of T = 32 floats (one
//    128-byte L1 line per source row).  A CTA owns one column tile of one
//    contiguous, nnz-balanced range of rows and sweeps it front to back, so
//    the source rows of a reordered graph (the 16-row community block and its
//    neighbourhood) are re-read from the SM's L1 instead of L2.  The CTAs of
//    the ntiles column tiles of a range are adjacent in launch order and share
//    the range's topology through L2.
//  * One warp per row.  The warp is split into NG groups of 32/NG lanes; every
//    group covers the SAME T columns (float4 per lane) and owns 8/NG of the
//    8 pairwise accumulators, so a warp has NG independent row gathers in
//    flight per round and the accumulator tree's upper levels are two
//    xor-shuffles -- the exact numpy tree, no re-association.
//  * Column indices and weights are streamed 32 edges at a time into lane
//    registers (one coalesced load each) and broadcast with shuffles.
//  * Products / sums are packed FMUL2 / FADD2 (fp32x2, round-to-nearest, no
//    FMA contraction), so results stay bitwise equal to the reference.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "ag_common.cuh"
#include "ag_vec.cuh"

namespace ag {
namespace {
using namespace vec;

constexpr int kLeafN = 128;  // numpy PW_BLOCKSIZE
constexpr int kDepth = 40;
constexpr int kThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

struct GArgs {
  int64_t rows;
  int feat;
  int mask;                 // 1 intra only, 2 inter only, 3 both (combine)
  const int32_t *row_ptr;   // [rows + 1]
  const int32_t *mid;       // [rows] end of the intra run; nullptr: single role
  const int32_t *col;       // role-ordered column indices
  const float *val;         // role-ordered weights; nullptr = implicit 1.0
  const float *x;
  float *y;
  Epi ep;
  int ntiles;               // column tiles
  int ranges;               // row ranges
  int64_t cost_total;       // nnz + kRowCost * rows
  float one;                // 1.0f, passed at run time (see add2)
  int chunk_rows;           // rows per work unit
};

constexpr int64_t kRowCost = 4;  // a row's fixed cost in edge units (epilogue, topology)

// ---------------------------------------------------------- packed fp32x2 --
__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(uint64_t r, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// fl(a + b) as FFMA2(a, one, b) with a RUN-TIME one = {1.0f, 1.0f}: exact
// (a * 1 is exact, so the only rounding is the sum's), and opaque to ptxas,
// which otherwise contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 and
// changes the rounding of c = fl(val * x).
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b, uint64_t one) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(one), "l"(b));
  return d;
}

// Predicated packed add: acc = on ? fl(acc + c) : acc (no select, no branch).
__device__ __forceinline__ uint64_t add2_if(uint64_t acc, uint64_t c, uint64_t one, bool on) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q fma.rn.f32x2 %0, %0, %1, %2;\n\t}"
      : "+l"(acc)
      : "l"(one), "l"(c), "r"(static_cast<int>(on)));
  return acc;
}

// A lane's slice of one row: VEC consecutive columns as packed fp32 pairs.
template <int VEC>
struct Lv {
  static constexpr int NP = VEC / 2;
  uint64_t p[NP];
};
template <>
struct Lv<1> {
  static constexpr int NP = 0;
  float s;
};

template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_splat(float v) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    r.s = v;
  } else {
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i) r.p[i] = pk(v, v);
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_add(const Lv<VEC> &a, const Lv<VEC> &b, uint64_t one) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    r.s = __fadd_rn(a.s, b.s);
  } else {
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i) r.p[i] = add2(a.p[i], b.p[i], one);
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_add_if(const Lv<VEC> &a, const Lv<VEC> &b, uint64_t one,
                                             bool on) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    r.s = on ? __fadd_rn(a.s, b.s) : a.s;
  } else {
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i) r.p[i] = add2_if(a.p[i], b.p[i], one, on);
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_scale(const Lv<VEC> &a, uint64_t vv) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    float v, v2;
    upk(vv, v, v2);
    r.s = __fmul_rn(a.s, v);
  } else {
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i) r.p[i] = mul2(a.p[i], vv);
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_max(const Lv<VEC> &a, const Lv<VEC> &b) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    r.s = fmaxf(a.s, b.s);
  } else {
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i) {
      float a0, a1, b0, b1;
      upk(a.p[i], a0, a1);
      upk(b.p[i], b0, b1);
      r.p[i] = pk(fmaxf(a0, b0), fmaxf(a1, b1));
    }
  }
  return r;
}
// Unconditional non-coherent 16-byte loads straight into packed pairs.  Every
// caller passes a valid address (inactive lanes / discarded tail items read a
// clamped, in-bounds row), so no predicate or branch surrounds the load.
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_load(const float *p) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    r.s = __ldg(p);
  } else {
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; i += 2)
      asm("ld.global.nc.v2.b64 {%0, %1}, [%2];"
          : "=l"(r.p[i]), "=l"(r.p[i + 1])
          : "l"(p + 2 * i));
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ Vf<VEC> lv_out(const Lv<VEC> &a) {
  Vf<VEC> r;
  if constexpr (VEC == 1) {
    r.v[0] = a.s;
  } else {
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i) upk(a.p[i], r.v[2 * i], r.v[2 * i + 1]);
  }
  return r;
}

// One entry of a warp's topology window (16 bytes): the source row's offset
// into x in floats, and its weight duplicated as an fp32 pair (the FMUL2
// operand), so one broadcast LDS.128 yields everything an item needs.
constexpr int kWin = 32;  // items per window refill

__device__ __forceinline__ void win_st(uint32_t addr, uint64_t a, uint64_t b) {
  asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void win_ld(uint32_t addr, uint32_t &off, uint64_t &vv) {
  uint64_t a;
  asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(vv) : "r"(addr) : "memory");
  off = static_cast<uint32_t>(a);
}

// ------------------------------------------------------------ the warp ----
// Per-warp state, passed by value (never by address: it must stay in
// registers).  Edge indices are int32 (E < 2^31 is checked on the host).
template <int VEC, bool W>
struct RowWarp {
  uint32_t win;        // shared address of this warp's window (kWin entries)
  const int32_t *col;  // role-ordered topology
  const float *val;    // nullptr = 1.0
  const float *xl;     // x + this lane's first column (clamped in-bounds)
  uint32_t feat;
  int lane;
  uint64_t one;    // {1.0f, 1.0f} loaded at run time (see add2)
  int32_t p, end;  // window holds items [p, p + kWin)

  __device__ __forceinline__ void fill(int32_t at) {
    __syncwarp();
    p = at;
    const int32_t e = at + lane;
    if (e < end) {
      const uint32_t off = static_cast<uint32_t>(__ldg(col + e)) * feat;
      const float v = W ? __ldg(val + e) : 1.0f;
      win_st(win + lane * 16, off, pk(v, v));
    }
    __syncwarp();
  }
  // install a prefetched window [at, at + kWin) ∩ [at, end): lane l's (c, v)
  __device__ __forceinline__ void install(int32_t at, int32_t c, float v) {
    __syncwarp();
    p = at;
    if (at + lane < end) win_st(win + lane * 16, static_cast<uint32_t>(c) * feat, pk(v, v));
    __syncwarp();
  }
  __device__ __forceinline__ void ensure(int32_t lo, int n) {
    if (lo + n > p + kWin) fill(lo);
  }
  template <bool RAW>
  __device__ __forceinline__ Lv<VEC> item(int32_t e) const {
    uint32_t off;
    uint64_t vv;
    win_ld(win + static_cast<uint32_t>(e - p) * 16u, off, vv);
    const float *ptr;  // xl + off as one IMAD.WIDE.U32
    asm("mad.wide.u32 %0, %1, 4, %2;" : "=l"(ptr) : "r"(off), "l"(xl));
    const Lv<VEC> xv = lv_load<VEC>(ptr);
    if (RAW || !W) return xv;
    return lv_scale<VEC>(xv, vv);
  }

  // res + c_e0 + ... + c_{e0+t-1} in order, t < 8 (warp-uniform)
  __device__ __forceinline__ Lv<VEC> seq(Lv<VEC> res, int32_t e0, int t) {
    if (t <= 0) return res;
    ensure(e0, t);
    Lv<VEC> c[7];
#pragma unroll
    for (int i = 0; i < 7; ++i) c[i] = item<false>(e0 + (i < t ? i : 0));
#pragma unroll
    for (int i = 0; i < 7; ++i) res = lv_add_if<VEC>(res, c[i], one, i < t);
    return res;
  }

  // numpy pairwise leaf over items [e0, e0 + n), 8 <= n <= 128
  __device__ __forceinline__ Lv<VEC> leaf(int32_t e0, int n) {
    const int q = n >> 3;
    Lv<VEC> r[8];
    ensure(e0, 8);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = item<false>(e0 + j);
#pragma unroll 1
    for (int g = 1; g < q; ++g) {
      const int32_t b = e0 + 8 * g;
      ensure(b, 8);
      Lv<VEC> c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = item<false>(b + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = lv_add<VEC>(r[j], c[j], one);
    }
    const Lv<VEC> s = lv_add<VEC>(
        lv_add<VEC>(lv_add<VEC>(r[0], r[1], one), lv_add<VEC>(r[2], r[3], one), one),
        lv_add<VEC>(lv_add<VEC>(r[4], r[5], one), lv_add<VEC>(r[6], r[7], one), one), one);
    return seq(s, e0 + 8 * q, n & 7);
  }

  // recursion of numpy's pairwise sum (n > 128), post-order, explicit stack
  __device__ __forceinline__ Lv<VEC> pairwise_long(int32_t e0, int n) {
    int32_t st_e[kDepth];
    int st_n[kDepth];
    int st_stage[kDepth];
    Lv<VEC> st_left[kDepth];
    int sp = 0;
    st_e[0] = e0;
    st_n[0] = n;
    st_stage[0] = 0;
    Lv<VEC> ret = lv_splat<VEC>(0.0f);
#pragma unroll 1
    while (sp >= 0) {
      const int cn = st_n[sp];
      if (cn <= kLeafN) {
        ret = leaf(st_e[sp], cn);
        --sp;
        continue;
      }
      int n2 = cn / 2;
      n2 -= n2 & 7;
      if (st_stage[sp] == 0) {
        st_stage[sp] = 1;
        st_e[sp + 1] = st_e[sp];
        st_n[sp + 1] = n2;
        st_stage[sp + 1] = 0;
        ++sp;
      } else if (st_stage[sp] == 1) {
        st_left[sp] = ret;
        st_stage[sp] = 2;
        st_e[sp + 1] = st_e[sp] + n2;
        st_n[sp + 1] = cn - n2;
        st_stage[sp + 1] = 0;
        ++sp;
      } else {
        ret = lv_add<VEC>(st_left[sp], ret, one);
        --sp;
      }
    }
    return ret;
  }

  // one role over items [e0, e0 + n)
  template <bool IS_MAX>
  __device__ __forceinline__ Lv<VEC> role(int32_t e0, int32_t n);
};

// Roles longer than kLeafN + 1 items take the recursion out of line; the
// warp state travels by value so the hot path keeps it in registers.
template <int VEC, bool W>
__device__ __noinline__ Lv<VEC> pairwise_long_fn(RowWarp<VEC, W> w, int32_t e0, int n) {
  w.fill(e0);
  return w.pairwise_long(e0, n);
}

template <int VEC, bool W>
template <bool IS_MAX>
__device__ __forceinline__ Lv<VEC> RowWarp<VEC, W>::role(int32_t e0, int32_t n) {
  if (n <= 0) return lv_splat<VEC>(0.0f);
  ensure(e0, n < kWin ? static_cast<int>(n) : kWin);  // the row's window normally covers it
  if constexpr (IS_MAX) {
    Lv<VEC> acc = item<true>(e0);
    const int32_t rend = e0 + n;  // this role's end (end is the row's)
#pragma unroll 1
    for (int32_t b = e0 + 1; b < rend; b += 8) {
      const int cnt = rend - b < 8 ? rend - b : 8;
      ensure(b, cnt);
      Lv<VEC> c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = item<true>(b + (j < cnt ? j : 0));
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = lv_max<VEC>(acc, c[j]);  // duplicates are harmless
    }
    return acc;
  } else {
    const Lv<VEC> c0 = item<false>(e0);
    const int32_t m = n - 1;
    if (m == 0) return c0;
    if (m < 8) return lv_add<VEC>(c0, seq(lv_splat<VEC>(-0.0f), e0 + 1, m), one);
    if (m <= kLeafN) return lv_add<VEC>(c0, leaf(e0 + 1, m), one);
    return lv_add<VEC>(c0, pairwise_long_fn<VEC, W>(*this, e0 + 1, m), one);
  }
}

__device__ __forceinline__ int64_t range_start(const GArgs &a, int k) {
  if (k <= 0) return 0;
  if (k >= a.ranges) return a.rows;
  const int64_t target = a.cost_total / a.ranges * k + (a.cost_total % a.ranges) * k / a.ranges;
  int64_t lo = 0, hi = a.rows;  // first r with cost(r) >= target
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (static_cast<int64_t>(a.row_ptr[m]) + kRowCost * m < target) lo = m + 1;
    else hi = m;
  }
  return lo;
}

template <int VEC>
__device__ __forceinline__ Vf<VEC> combine2(int op, const Vf<VEC> &I, bool ti, const Vf<VEC> &O,
                                            bool to, int64_t deg) {
  if (op == AG_OP_SUM) return vadd<VEC>(I, O);
  if (op == AG_OP_MEAN) {
    const float d = static_cast<float>(deg < 1 ? 1 : deg);
    Vf<VEC> s = vadd<VEC>(I, O), r;
#pragma unroll
    for (int i = 0; i < VEC; ++i) r.v[i] = __fdiv_rn(s.v[i], d);
    return r;
  }
  if (ti && to) return vmax<VEC>(I, O);
  if (ti) return I;
  if (to) return O;
  return splat<VEC>(0.0f);
}

// One destination row (both roles, epilogue) for this lane's columns.
template <int VEC, bool IS_MAX, bool W>
__device__ __forceinline__ void do_row(const GArgs &a, RowWarp<VEC, W> &w, int64_t r, int32_t s,
                                       int32_t e, int32_t m, int64_t fcol, bool act) {
  const int64_t ld = a.feat;
  const int32_t ni = (a.mask & 1) ? m - s : 0;
  const int32_t no = (a.mask & 2) ? e - m : 0;
  const Vf<VEC> I = lv_out<VEC>(w.template role<IS_MAX>(s, ni));
  const Vf<VEC> O = lv_out<VEC>(w.template role<IS_MAX>(m, no));
  if (!act) return;
  float *yp = a.y + r * ld + fcol;
  const int64_t d = (a.ep.op == AG_OP_MEAN && a.ep.deg) ? a.ep.deg[r] : 1;
  Vf<VEC> out;
  if (a.mask == 3) {
    out = combine2<VEC>(a.ep.op, I, ni > 0, O, no > 0, d);
  } else {
    const Vf<VEC> v = (a.mask == 1) ? I : O;
    const bool t = (a.mask == 1) ? ni > 0 : no > 0;
    if (!(a.ep.flags & AG_EPI_COMBINE)) {
      out = t ? v : splat<VEC>(0.0f);
    } else if (a.ep.flags & AG_EPI_EMPTY_OTHER) {
      out = combine2<VEC>(a.ep.op, v, t, splat<VEC>(0.0f), false, d);
    } else {
      const bool ot = a.ep.other_touched ? a.ep.other_touched[r] != 0 : false;
      out = combine2<VEC>(a.ep.op, v, t, ldv_rw<VEC>(yp), ot, d);
    }
  }
  if (a.ep.flags & AG_EPI_GIN)
    out = vadd<VEC>(vscale<VEC>(a.ep.gin_scale, ldv<VEC>(a.x + r * ld + fcol)), out);
  if (a.ep.flags & AG_EPI_RELU_MASK) {
    const Vf<VEC> h = ldv<VEC>(a.ep.relu_src + r * ld + fcol);
#pragma unroll
    for (int i = 0; i < VEC; ++i) out.v[i] = h.v[i] > 0.0f ? out.v[i] : 0.0f;
  }
  stv<VEC>(yp, out);
}

// Work order.  Units are (chunk of kChunkRows consecutive rows, column tile),
// tile fastest; global warp gw takes units gw, gw + W, gw + 2W, ... (W = all
// warps of the persistent grid).  Every warp advances at about the same rate,
// so the whole GPU sweeps the row space as ONE narrow wavefront: the source
// rows the reorder keeps near each destination are re-read from L2 (and from
// L1: a CTA's warps hold adjacent chunks, i.e. one contiguous band of rows and
// both column tiles of it), and no atomics or CTA barriers are needed.
// Within its sequence a warp software-pipelines the next row's row_ptr / mid /
// first kWin (col, val) while the current row gathers.
template <int VEC, bool IS_MAX, bool W>
__global__ void __launch_bounds__(kThreads, 2) gather_kernel(GArgs a) {
  constexpr int T = 32 * VEC;
  __shared__ __align__(16) uint64_t wins[kThreads / 32][kWin * 2];
  const int warp = threadIdx.x >> 5;
  RowWarp<VEC, W> w;
  w.win = static_cast<uint32_t>(__cvta_generic_to_shared(wins[warp]));
  w.col = a.col;
  w.val = a.val;
  w.feat = static_cast<uint32_t>(a.feat);
  w.lane = threadIdx.x & 31;
  w.one = pk(a.one, a.one);
  w.p = 0;
  w.end = 0;
  const int CR = a.chunk_rows;
  const int64_t nrc = (a.rows + CR - 1) / CR;
  const int64_t nunits = nrc * a.ntiles;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  // cursor over this warp's (unit, row-in-chunk) sequence
  int64_t k = gw;
  int j = 0;
  auto row_of = [&](int64_t kk, int jj) { return (kk / a.ntiles) * CR + jj; };
  auto advance = [&](int64_t &kk, int &jj) {
    ++jj;
    if (jj == CR || row_of(kk, jj) >= a.rows) { kk += nw; jj = 0; }
  };
  int32_t ns = 0, ne = 0, nm = 0, nc = 0;
  float nv = 1.0f;
  auto prefetch = [&](int64_t kk, int jj) {
    if (kk < nunits) {
      const int64_t rr = row_of(kk, jj);
      ns = a.row_ptr[rr];
      ne = a.row_ptr[rr + 1];
      nm = a.mid ? a.mid[rr] : (a.mask == 1 ? ne : ns);
      const int32_t ed = ns + w.lane;
      nc = ed < ne ? __ldg(a.col + ed) : 0;
      nv = (W && ed < ne) ? __ldg(a.val + ed) : 1.0f;
    }
  };
  prefetch(k, j);
  int cur_tile = -1;
  int64_t fcol = 0;
  bool act = false;
#pragma unroll 1
  while (k < nunits) {
    const int tile = static_cast<int>(k % a.ntiles);
    if (tile != cur_tile) {
      cur_tile = tile;
      fcol = static_cast<int64_t>(tile) * T + w.lane * VEC;
      act = fcol < a.feat;
      w.xl = a.x + (act ? fcol : 0);
    }
    const int64_t r = row_of(k, j);
    const int32_t s = ns, e = ne, m = nm;
    w.end = e;
    w.install(s, nc, nv);
    int64_t k2 = k;
    int j2 = j;
    advance(k2, j2);
    prefetch(k2, j2);
    do_row<VEC, IS_MAX, W>(a, w, r, s, e, m, fcol, act);
    k = k2;
    j = j2;
  }
}

// -------------------------------------------------- role-ordered CSR build --
__global__ void role_csr_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *col,
                                const float *val, int64_t B, int32_t *rcol, float *rval,
                                int32_t *mid) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = row_ptr[r], e = row_ptr[r + 1];
    const int64_t cb = (r / B) * B;
    int64_t lo = s, hi = e;
    while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (col[m] < cb) lo = m + 1; else hi = m; }
    const int64_t ia = lo;
    hi = e;
    while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (col[m] < cb + B) lo = m + 1; else hi = m; }
    const int64_t ib = lo;
    int64_t t = s;
    for (int64_t k = ia; k < ib; ++k, ++t) { rcol[t] = col[k]; if (rval) rval[t] = val[k]; }
    for (int64_t k = s; k < ia; ++k, ++t) { rcol[t] = col[k]; if (rval) rval[t] = val[k]; }
    for (int64_t k = ib; k < e; ++k, ++t) { rcol[t] = col[k]; if (rval) rval[t] = val[k]; }
    mid[r] = static_cast<int32_t>(s + (ib - ia));
  }
}

int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <int VEC>
int launch_gather(GArgs a, bool is_max, cudaStream_t st) {
  constexpr int T = 32 * VEC;
  auto k = is_max ? (a.val ? gather_kernel<VEC, true, true> : gather_kernel<VEC, true, false>)
                  : (a.val ? gather_kernel<VEC, false, true> : gather_kernel<VEC, false, false>);
  // prefer L1 over shared memory: the gathers' reuse lives in L1
  AG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 8));
  int per_sm = 0;
  AG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kThreads, 0));
  if (per_sm < 1) per_sm = 1;
  a.ntiles = static_cast<int>((a.feat + T - 1) / T);
  a.chunk_rows = std::max(1, env_int("AG_GATHER_CHUNK", 16));
  const int64_t units = (a.rows + a.chunk_rows - 1) / a.chunk_rows * a.ntiles;
  const int64_t warps = (units + 0);
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;
  grid = std::max<int64_t>(1, std::min(grid, (warps + kThreads / 32 - 1) / (kThreads / 32)));
  k<<<(unsigned)grid, kThreads, 0, st>>>(a);
  AG_LAUNCH_CHECK("gather_kernel");
  return AG_OK;
}

}  // namespace
}  // namespace ag

using namespace ag;

extern "C" int ag_role_csr_build(int64_t num_rows, const int32_t *row_ptr, const int32_t *col_idx,
                                 const float *val, int64_t block_size, int32_t *role_col,
                                 float *role_val, int32_t *role_mid, void *stream) {
  if (num_rows < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (block_size < 1) return fail(AG_ERR_VALUE, "block_size must be >= 1");
  if (val != nullptr && role_val == nullptr)
    return fail(AG_ERR_VALUE, "role_val is required for a weighted CSR");
  if (num_rows == 0) return AG_OK;
  role_csr_kernel<<<grid_for(num_rows, 128), 128, 0, as_stream(stream)>>>(
      num_rows, row_ptr, col_idx, val, block_size, role_col, val ? role_val : nullptr, role_mid);
  AG_LAUNCH_CHECK("role_csr_kernel");
  return AG_OK;
}

extern "C" int ag_fused_spmm(int64_t num_rows, int64_t feat, int32_t role_mask,
                             const int32_t *row_ptr, const int32_t *role_mid,
                             const int32_t *col_idx, const float *val, int64_t num_edges,
                             const float *x, float *y, int32_t op, int32_t epi_flags,
                             const uint8_t *other_touched, const int64_t *deg, float gin_scale,
                             const float *relu_src, void *stream) {
  if (num_rows < 0 || feat < 0 || num_edges < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (op < AG_OP_SUM || op > AG_OP_MAX) return fail(AG_ERR_KERNEL, "unknown op %d", op);
  if (role_mask < 1 || role_mask > 3) return fail(AG_ERR_VALUE, "role_mask must be 1, 2 or 3");
  if (role_mid == nullptr && role_mask == 3)
    return fail(AG_ERR_VALUE, "role_mask 3 needs the role-ordered CSR (role_mid)");
  if (op == AG_OP_MEAN && deg == nullptr && (role_mask == 3 || (epi_flags & AG_EPI_COMBINE)))
    return fail(AG_ERR_KERNEL, "mean combine requires the full-graph degree vector");
  if ((epi_flags & AG_EPI_RELU_MASK) && relu_src == nullptr)
    return fail(AG_ERR_VALUE, "AG_EPI_RELU_MASK needs relu_src");
  if (num_rows == 0 || feat == 0) return AG_OK;
  if (num_rows > 2147483647LL || num_edges > 2147483647LL)
    return fail(AG_ERR_VALUE, "too many rows or edges for int32 CSR");
  if (num_rows * feat > 4294967295LL)
    return fail(AG_ERR_VALUE, "feature matrix too large for 32-bit row offsets");
  cudaStream_t st = as_stream(stream);
  GArgs a{num_rows, static_cast<int>(feat), role_mask, row_ptr, role_mid, col_idx, val, x, y,
          Epi{op, epi_flags, other_touched, deg, x, feat, gin_scale, relu_src}, 1, 1, 0, 1.0f,
          16};
  a.cost_total = num_edges + kRowCost * num_rows;
  const bool is_max = op == AG_OP_MAX;
  const bool v4 = feat % 4 == 0 && (reinterpret_cast<uintptr_t>(x) % 16) == 0 &&
                  (reinterpret_cast<uintptr_t>(y) % 16) == 0;
  if (!v4) return launch_gather<1>(a, is_max, st);
  const int vec = env_int("AG_GATHER_VEC", 4);
  if (vec == 8 && feat % 8 == 0 && feat > 128) return launch_gather<8>(a, is_max, st);
  return launch_gather<4>(a, is_max, st);
}
