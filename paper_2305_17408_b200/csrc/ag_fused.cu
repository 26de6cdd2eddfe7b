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
// Work decomposition: the "slab" kernel (sm_100a).
//  * A reordered graph keeps most sources near their destination: the
//    community's own 16-row block (intra) and, for the inter edges, a band of
//    neighbouring blocks.  One CTA per SM owns a column tile of T = 32*VEC
//    floats of one contiguous, nnz-balanced range of 16-row blocks and sweeps
//    it front to back (about two such units per CTA).
//  * X producer warp: streams the X tile of block b (16 rows x T floats) into
//    a kSlots-slot ring in shared memory, one TMA tensor load per block
//    (cp.async.bulk.tensor.2d, mbarrier complete_tx), and pulls the topology
//    ahead into L2.  X crosses HBM -> L2 -> SM once per tile.
//  * Far producer warp: bulk-copies each block's <= kFarMax distinct sources
//    outside the ring window into a kFarSlots-deep far ring.
//  * Consumer warps (14; 16 in the dense + coo mode) take the range's rows
//    round-robin.  At block k the ring holds blocks [k-H, k+H] (H picked per
//    graph, ag_slab_window); a staged source is one conflict-free 256-byte
//    shared load per warp, anything else a direct global load.  A row's
//    (code, weight) pairs are prefetched in registers one row ahead and
//    installed into a per-warp window, so the inner loop is LDS(window) +
//    LDS(x) + math.
//  * Per-block mbarriers: ready[k] (producers' arrivals + the copies' bytes),
//    done[k] (every consumer left block k); a slot is refilled only after done
//    of the last block that reads it, so warps drift freely by a few blocks.
//  * Modes (the selector pair being run): both roles bitwise (numpy order,
//    FMUL2 / FFMA2-with-a-runtime-one so nothing contracts); dense_block intra
//    on two extra "dense" warps (16 x 16 block weights x the block's X rows,
//    register-blocked, into an I-slot the consumers add); coo_atomic inter
//    (AG_EPI_INTER_COO) with fused multiply-adds in any order.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ag_common.cuh"
#include "ag_ptx.cuh"
#include "ag_vec.cuh"

namespace ag {
namespace {
using namespace vec;
using namespace ptx;

constexpr int kLeafN = 128;  // numpy PW_BLOCKSIZE
constexpr int kDepth = 40;
constexpr int kRB = 16;      // rows per ring block
// consumer warps per CTA (+ 2 producer warps): 14 -> 16 warps, 4 per SMSP at 128 registers
// for the exact-order modes; the order-free inter modes (AG_EPI_INTER_COO) need fewer
// registers: with the intra role on the dense warps (kModeDense3Coo) the consumers run
// 16 + 2 warps at 96 registers (measured faster; the exact-order code spills there)
constexpr int kConsMax = 16;
#ifndef AG_SLAB_COO_CONS
#define AG_SLAB_COO_CONS 14
#endif
// dense + coo: consumer warps (+ 2 dense warps), rows round-robin.  Measured at
// C5 F = 256: 8 / 10 / 12 / 14 warps 6.13 / 5.35 / 4.74 / 4.56 ms; 16 warps each
// owning one row of every block (no per-row block bookkeeping) 4.92 ms
constexpr int kCooCons = AG_SLAB_COO_CONS;
static_assert(kCooCons <= kConsMax, "consumer windows");
template <int MODE>
constexpr int cons_warps();
constexpr int kWin = 64;     // topology items per window refill (two per lane)
#ifndef AG_SLAB_SLOTS
#define AG_SLAB_SLOTS 43
#endif
#ifndef AG_SLAB_FAR_SLOTS
#define AG_SLAB_FAR_SLOTS 5
#endif
constexpr int kSlots = AG_SLAB_SLOTS;  // X ring capacity in blocks (window H <= (kSlots - 9) / 2 = 17)
constexpr int kFarSlots = AG_SLAB_FAR_SLOTS;  // far ring depth (measured: 43 / 5 vs 45 / 4 is 2% faster)
constexpr int kFarMax = 20;  // staged far sources per block (more: read from global)
constexpr int kRG = 1;       // consecutive rows a consumer warp takes at a time (divides kRB)
constexpr int kISlots = 4;   // dense-intra mode: per-block intra results (16 rows x tile)
constexpr int kReady = 16;   // per-block "ready" barriers (X window + far rows staged)
constexpr int kDone = 32;    // per-block "done" barriers (every consumer left the block)
constexpr int kRowSlow = 1;  // rowinfo flag: row has global sources or > kWin pairs
constexpr int kFarRow0 = kSlots * 16;  // first far-ring row (codes >= kFarRow0)
constexpr int64_t kRowCost = 4;  // a row's fixed cost in edge units (epilogue, topology)

struct GArgs {
  int64_t rows;
  int feat;
  int mask;                 // 1 intra only, 2 inter only, 3 both (combine)
  const int32_t *row_ptr;   // [rows + 1]
  const int32_t *mid;       // [rows] end of the intra run; nullptr: single role
  const int2 *cv;           // role-ordered (code, weight bits) per edge (ag_slab_codes)
  const int4 *rowinfo;      // per row {start, intra end, end, flags} (ag_slab_codes)
  const int32_t *far_cnt;   // [nblocks] staged far sources per block (<= kFarMax)
  const int32_t *far_src;   // [nblocks * kFarMax] their source rows
  int weighted;             // 0: every weight is 1.0 (multiplies skipped: exact)
  int has_mid;              // rowinfo.y is the intra-run end (role-ordered layout)
  int relu;                 // AG_EPI_RELU_MASK: y *= the relu_bits mask (ep.relu_bits)
  uint32_t *relu_out;       // AG_EPI_RELU: write y's relu bits here (or NULL)
  int64_t ldw;              // words per relu-bit row: ceil(feat / 32)
  const float *blk_w;       // dense-intra mode: [nblocks][16][16] intra weights (dst, src)
  const float *x;
  float *y;
  Epi ep;
  int ntiles;               // column tiles
  int ranges;               // row ranges (of whole blocks)
  int64_t cost_total;       // nnz + kRowCost * rows
  float one;                // 1.0f, passed at run time (see add2)
  int H;                    // window radius (blocks)
  int64_t nblocks;          // ceil(rows / 16)
  int64_t x_rows;           // rows of x (>= rows: a rank's halo rows follow its own)
  int64_t xblocks;          // ceil(x_rows / 16)
  int tma;                  // 1: TMA tensor loads; 0: cp.async element copies
  int sleep;                // producers' done waits: 1 suspend between polls, 0 spin
  uint32_t csleep;          // consumer / dense-warp waits: suspend hint (ns) per poll, 0 spin
  const int4 *brec;         // band kernel: per-block topology records (ag_band_records), or NULL
  const int32_t *brec_off;  // [nblocks + 1] record offsets in 16-byte units
  long long *trace;         // AG_SLAB_TRACE: per-block globaltimer stamps of CTA 0 (development)
  int dbg;                  // development knob (AG_SLAB_DEBUG bits, values then garbage): 1 skip the
                            // reductions, 2 far copies, 4 dense products, 8 X tiles, 16 Y stores,
                            // 32 consumer topology loads
};

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
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(b), "l"(one));
  return a;
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
__device__ __forceinline__ Lv<VEC> lv_scale(const Lv<VEC> &a, float v) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    r.s = __fmul_rn(a.s, v);
  } else {
    const uint64_t vv = pk(v, v);
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i) r.p[i] = mul2(a.p[i], vv);
  }
  return r;
}
// acc + x * v with one rounding (order-free roles only: AG_EPI_INTER_COO)
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_fma(const Lv<VEC> &x, float v, Lv<VEC> acc) {
  if constexpr (VEC == 1) {
    acc.s = __fmaf_rn(x.s, v, acc.s);
  } else {
    const uint64_t vv = pk(v, v);
#pragma unroll
    for (int i = 0; i < Lv<VEC>::NP; ++i)
      asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc.p[i]) : "l"(x.p[i]), "l"(vv));
  }
  return acc;
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
// shared-memory row slice (ring) and global row slice (far sources)
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_lds(uint32_t addr) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r.s) : "r"(addr) : "memory");
  } else if constexpr (VEC == 2) {
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(r.p[0]) : "r"(addr) : "memory");
  } else {
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(r.p[0]), "=l"(r.p[1]) : "r"(addr)
                 : "memory");
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ Lv<VEC> lv_ldg(const float *p) {
  Lv<VEC> r;
  if constexpr (VEC == 1) {
    r.s = __ldg(p);
  } else if constexpr (VEC == 2) {
    asm("ld.global.nc.b64 %0, [%1];" : "=l"(r.p[0]) : "l"(p));
  } else {
    asm("ld.global.nc.v2.b64 {%0, %1}, [%2];" : "=l"(r.p[0]), "=l"(r.p[1]) : "l"(p));
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

// Window entry (8 bytes): the source's ring byte offset (>= 0) or ~src for a
// far source (< 0), and its weight.
__device__ __forceinline__ void win_st(uint32_t addr, int32_t code, float v) {
  asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(code), "f"(v) : "memory");
}
__device__ __forceinline__ void win_ld(uint32_t addr, int32_t &code, float &v) {
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(code), "=f"(v) : "r"(addr) : "memory");
}

// ------------------------------------------------------------ the warp ----
// Per-warp state, passed by value (never by address: it must stay in
// registers).  Edge indices are int32 (E < 2^31 is checked on the host).
template <int VEC, bool W>
struct RowWarp {
  uint32_t win;        // shared address of this warp's window (kWin entries)
  uint32_t ring;       // shared address of the ring + this lane's column byte
  const int2 *cv;      // role-ordered (code, weight) pairs in global memory
  const float *xl;     // x + this lane's first column (clamped in-bounds)
  uint32_t feat;
  int lane;
  uint64_t one;        // {1.0f, 1.0f} loaded at run time (see add2)
  int32_t p, end;      // window holds items [p, p + kWin)
  uint64_t far;        // bit i: window item p + i is a far (global) source
  __device__ __forceinline__ void fill(int32_t at) {
    __syncwarp();
    p = at;
    int32_t cd[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int32_t e = at + h * 32 + lane;
      if (e < end) {
        const int2 p2 = __ldg(cv + e);
        cd[h] = p2.x;
        win_st(win + (h * 32 + lane) * 8, cd[h], __int_as_float(p2.y));
      }
    }
    far = __ballot_sync(0xffffffffu, cd[0] < 0) |
          (static_cast<uint64_t>(__ballot_sync(0xffffffffu, cd[1] < 0)) << 32);
    __syncwarp();
  }
  // install a prefetched window [at, at + kWin) ∩ [at, end): lane l's pairs
  // at + l and at + 32 + l.  Rows on the fast path have no global sources,
  // so `far` is only computed for the general path.
  template <bool FAST>
  __device__ __forceinline__ void install(int32_t at, int2 q0, int2 q1) {
    __syncwarp();
    p = at;
    const bool in0 = at + lane < end, in1 = at + 32 + lane < end;
    if (in0) win_st(win + lane * 8, q0.x, __int_as_float(q0.y));
    if (in1) win_st(win + (32 + lane) * 8, q1.x, __int_as_float(q1.y));
    if (!FAST)
      far = __ballot_sync(0xffffffffu, in0 && q0.x < 0) |
            (static_cast<uint64_t>(__ballot_sync(0xffffffffu, in1 && q1.x < 0)) << 32);
    __syncwarp();
  }
  __device__ __forceinline__ void ensure(int32_t lo, int n) {
    if (lo + n > p + kWin) fill(lo);
  }
  // NEAR: the caller checked `far` -- the item is in the ring
  template <bool RAW, bool NEAR = false>
  __device__ __forceinline__ Lv<VEC> item(int32_t e) const {
    int32_t cd;
    float v;
    win_ld(win + static_cast<uint32_t>(e - p) * 8u, cd, v);
    Lv<VEC> xv;
    if (NEAR || cd >= 0) {
      xv = lv_lds<VEC>(ring + static_cast<uint32_t>(cd) * (32u * VEC * 4u));
    } else {
      const float *ptr;  // xl + src * feat as one IMAD.WIDE.U32
      asm("mad.wide.u32 %0, %1, %2, %3;"
          : "=l"(ptr)
          : "r"(static_cast<uint32_t>(~cd)), "r"(feat * 4u), "l"(xl));
      xv = lv_ldg<VEC>(ptr);
    }
    if (RAW || !W) return xv;
    return lv_scale<VEC>(xv, v);
  }

  // ---- fast path: the whole row is in the window and every source is
  // staged in shared memory (X ring or far ring): straight-line, no checks.
  template <bool RAW>
  __device__ __forceinline__ Lv<VEC> it(int j) const {
    int32_t cd;
    float v;
    win_ld(win + static_cast<uint32_t>(j) * 8u, cd, v);
    const Lv<VEC> xv = lv_lds<VEC>(ring + static_cast<uint32_t>(cd) * (32u * VEC * 4u));
    if (RAW || !W) return xv;
    return lv_scale<VEC>(xv, v);
  }
  template <int N>
  __device__ __forceinline__ Lv<VEC> seqf_n(Lv<VEC> res, int j) const {
    Lv<VEC> c[N];
#pragma unroll
    for (int i = 0; i < N; ++i) c[i] = it<false>(j + i);
#pragma unroll
    for (int i = 0; i < N; ++i) res = lv_add<VEC>(res, c[i], one);
    return res;
  }
  __device__ __forceinline__ Lv<VEC> seqf(Lv<VEC> res, int j, int t) const {
    if (t & 4) { res = seqf_n<4>(res, j); j += 4; }
    if (t & 2) { res = seqf_n<2>(res, j); j += 2; }
    if (t & 1) res = seqf_n<1>(res, j);
    return res;
  }
  // one role over window offsets [o, o + n), o + n <= kWin
  template <bool IS_MAX>
  __device__ __forceinline__ Lv<VEC> role_fast(int o, int n) const {
    if (n <= 0) return lv_splat<VEC>(0.0f);
    if constexpr (IS_MAX) {
      Lv<VEC> acc = it<true>(o);
#pragma unroll 1
      for (int j = 1; j < n; ++j) acc = lv_max<VEC>(acc, it<true>(o + j));
      return acc;
    } else {
      const Lv<VEC> c0 = it<false>(o);
      const int m = n - 1;
      if (m == 0) return c0;
      if (m < 8) return lv_add<VEC>(c0, seqf(lv_splat<VEC>(-0.0f), o + 1, m), one);
      Lv<VEC> r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = it<false>(o + 1 + j);
      const int q = m >> 3;
#pragma unroll 1
      for (int g = 1; g < q; ++g) {
        Lv<VEC> c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = it<false>(o + 1 + 8 * g + j);
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = lv_add<VEC>(r[j], c[j], one);
      }
      const Lv<VEC> t = lv_add<VEC>(
          lv_add<VEC>(lv_add<VEC>(r[0], r[1], one), lv_add<VEC>(r[2], r[3], one), one),
          lv_add<VEC>(lv_add<VEC>(r[4], r[5], one), lv_add<VEC>(r[6], r[7], one), one), one);
      return lv_add<VEC>(c0, seqf(t, o + 1 + 8 * q, m & 7), one);
    }
  }

  // ---- order-free inter role (AG_EPI_INTER_COO: the selector's coo_atomic,
  // any summation order): fused multiply-adds into two accumulators.
  __device__ __forceinline__ void acc_it(Lv<VEC> &acc, int j) const {
    int32_t cd;
    float v;
    win_ld(win + static_cast<uint32_t>(j) * 8u, cd, v);
    const Lv<VEC> xv = lv_lds<VEC>(ring + static_cast<uint32_t>(cd) * (32u * VEC * 4u));
    acc = W ? lv_fma<VEC>(xv, v, acc) : lv_add<VEC>(acc, xv, one);
  }
  __device__ __forceinline__ Lv<VEC> role_coo_fast(int o, int n) const {
    Lv<VEC> a0 = lv_splat<VEC>(0.0f), a1 = a0;
    int j = o;
    const int e = o + n;
    // fully unrolled (n <= kWin): no loop-carried accumulator copies
#pragma unroll
    for (int c = 0; c < kWin / 8; ++c) {
      if (j + 8 > e) break;
#pragma unroll
      for (int i = 0; i < 8; i += 2) {
        acc_it(a0, j + i);
        acc_it(a1, j + i + 1);
      }
      j += 8;
    }
    if (j + 4 <= e) {
      acc_it(a0, j);
      acc_it(a1, j + 1);
      acc_it(a0, j + 2);
      acc_it(a1, j + 3);
      j += 4;
    }
    if (j + 2 <= e) {
      acc_it(a0, j);
      acc_it(a1, j + 1);
      j += 2;
    }
    if (j < e) acc_it(a0, j);
    return lv_add<VEC>(a0, a1, one);
  }
  // general path: window refills and global (far) sources
  __device__ __forceinline__ void acc_item(Lv<VEC> &acc, int32_t e) const {
    int32_t cd;
    float v;
    win_ld(win + static_cast<uint32_t>(e - p) * 8u, cd, v);
    Lv<VEC> xv;
    if (cd >= 0) {
      xv = lv_lds<VEC>(ring + static_cast<uint32_t>(cd) * (32u * VEC * 4u));
    } else {
      const float *ptr;
      asm("mad.wide.u32 %0, %1, %2, %3;"
          : "=l"(ptr)
          : "r"(static_cast<uint32_t>(~cd)), "r"(feat * 4u), "l"(xl));
      xv = lv_ldg<VEC>(ptr);
    }
    acc = W ? lv_fma<VEC>(xv, v, acc) : lv_add<VEC>(acc, xv, one);
  }
  __device__ __forceinline__ Lv<VEC> role_coo(int32_t e0, int32_t n) {
    Lv<VEC> a0 = lv_splat<VEC>(0.0f), a1 = a0;
    const int32_t rend = e0 + n;
#pragma unroll 1
    for (int32_t b = e0; b < rend; b += 8) {
      const int cnt = rend - b < 8 ? rend - b : 8;
      ensure(b, cnt);
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        if (j < cnt) acc_item(a0, b + j);
        if (j + 1 < cnt) acc_item(a1, b + j + 1);
      }
    }
    return lv_add<VEC>(a0, a1, one);
  }

  // N consecutive items [e, e + N) of the window: one uniform branch picks
  // the all-in-ring path (shared loads only) or the mixed one
  template <int N, bool RAW>
  __device__ __forceinline__ void items(int32_t e, Lv<VEC> (&c)[N]) const {
    const uint32_t fb = static_cast<uint32_t>(far >> (e - p)) & ((1u << N) - 1u);
    if (fb == 0) {
#pragma unroll
      for (int j = 0; j < N; ++j) c[j] = item<RAW, true>(e + j);
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j) c[j] = item<RAW, false>(e + j);
    }
  }
  template <int N>
  __device__ __forceinline__ Lv<VEC> seq_n(Lv<VEC> res, int32_t e) const {
    Lv<VEC> c[N];
    items<N, false>(e, c);
#pragma unroll
    for (int j = 0; j < N; ++j) res = lv_add<VEC>(res, c[j], one);
    return res;
  }
  // res + c_e0 + ... + c_{e0+t-1} in order, t < 8 (warp-uniform): chunks of
  // 4, 2, 1 so no load is wasted
  __device__ __forceinline__ Lv<VEC> seq(Lv<VEC> res, int32_t e0, int t) {
    if (t <= 0) return res;
    ensure(e0, t);
    if (t & 4) { res = seq_n<4>(res, e0); e0 += 4; }
    if (t & 2) { res = seq_n<2>(res, e0); e0 += 2; }
    if (t & 1) res = seq_n<1>(res, e0);
    return res;
  }

  // numpy pairwise leaf over items [e0, e0 + n), 8 <= n <= 128
  __device__ __forceinline__ Lv<VEC> leaf(int32_t e0, int n) {
    const int q = n >> 3;
    Lv<VEC> r[8];
    ensure(e0, 8);
    items<8, false>(e0, r);
#pragma unroll 1
    for (int g = 1; g < q; ++g) {
      const int32_t b = e0 + 8 * g;
      ensure(b, 8);
      Lv<VEC> c[8];
      items<8, false>(b, c);
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
    const int32_t rend = e0 + n;
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

// First block of row range k (ranges are balanced by nnz + kRowCost * rows).
__device__ __forceinline__ int64_t range_block(const GArgs &a, int k) {
  if (k <= 0) return 0;
  if (k >= a.ranges) return a.nblocks;
  const int64_t target = a.cost_total / a.ranges * k + (a.cost_total % a.ranges) * k / a.ranges;
  int64_t lo = 0, hi = a.rows;  // first r with cost(r) >= target
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (static_cast<int64_t>(a.row_ptr[m]) + kRowCost * m < target) lo = m + 1;
    else hi = m;
  }
  return std::min<int64_t>((lo + kRB - 1) / kRB, a.nblocks);
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

// Kernel modes: the training path (both roles, sum combine) gets its own
// instantiation without the generic epilogue's runtime dispatch.
constexpr int kModeSum3 = 0;   // role_mask 3, op sum (flags: GIN / RELU_MASK only)
constexpr int kModeAny = 1;    // any role mask, sum or mean, any flags
constexpr int kModeMax = 2;    // any role mask, max
// role mask 3, op sum, the intra role as a dense 16 x 16 block product (the
// reference's dense_block kernel, order-unpinned like its BLAS matmul) computed
// once per block by a dedicated warp; the inter role stays bitwise csr_inter
constexpr int kModeDense3 = 3;
// kModeSum3 / kModeDense3 with the inter role order-free (AG_EPI_INTER_COO)
constexpr int kModeSum3Coo = 4;
constexpr int kModeDense3Coo = 5;
__host__ __device__ constexpr bool mode_dense(int m) { return m == kModeDense3 || m == kModeDense3Coo; }
__host__ __device__ constexpr bool mode_coo(int m) { return m == kModeSum3Coo || m == kModeDense3Coo; }
template <int MODE>
constexpr int cons_warps() { return MODE == kModeDense3Coo ? kCooCons + 2 : 14; }
__host__ __device__ constexpr bool mode_sum3(int m) {
  return m == kModeSum3 || m == kModeDense3 || mode_coo(m);
}

// One destination row (both roles, epilogue) for this lane's columns.
// spread the 16 low bits of x to the even bit positions
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  return (x | (x << 1)) & 0x55555555u;
}

template <int VEC, int MODE, bool W>
__device__ __forceinline__ void do_row(const GArgs &a, RowWarp<VEC, W> &w, int64_t r, int32_t s,
                                       int32_t e, int32_t m, float *yrow, bool act, bool fast,
                                       int64_t fcol, uint32_t intra_s, uint32_t rword,
                                       uint32_t iv_bar = 0, uint32_t iv_phase = 0,
                                       bool *iv_pending = nullptr) {
  constexpr bool IS_MAX = MODE == kModeMax;
  constexpr bool SUM3 = mode_sum3(MODE);
  constexpr bool DENSE = mode_dense(MODE);
  constexpr bool COO = mode_coo(MODE);
  // dense-intra mode: the intra role comes from the dense warp's block product
  const int32_t ni = DENSE ? 0 : (SUM3 || (a.mask & 1)) ? m - s : 0;
  const int32_t no = (SUM3 || (a.mask & 2)) ? e - m : 0;
  // the row's ReLU-mask word was loaded a row ahead (the consumer pipeline)
  const bool relu = a.relu && act;
  const uint32_t rbits = relu ? rword >> (fcol & 31) : 0u;
  Vf<VEC> I, O;
  if (a.dbg & 1) {
    I = splat<VEC>(0.0f);
    O = I;
  } else if (fast) {
    I = lv_out<VEC>(w.template role_fast<IS_MAX>(0, ni));
    O = lv_out<VEC>(COO ? w.role_coo_fast(m - s, no) : w.template role_fast<IS_MAX>(m - s, no));
  } else {
    I = lv_out<VEC>(w.template role<IS_MAX>(s, ni));
    O = lv_out<VEC>(COO ? w.role_coo(m, no) : w.template role<IS_MAX>(m, no));
  }
  // inactive lanes (columns past F) run the epilogue too -- the relu-bit
  // ballots need the whole warp -- but store nothing
  float *yp = yrow;
  Vf<VEC> out;
  if constexpr (DENSE) {
    // the block's intra partials: waited for here, after this row's inter
    // reduction, so the dense warps' block product overlaps it
    if (iv_pending && *iv_pending) {
      mbar_wait_hint(iv_bar, iv_phase, a.csleep);
      *iv_pending = false;
    }
    out = vadd<VEC>(lv_out<VEC>(lv_lds<VEC>(intra_s)), O);
  } else if constexpr (SUM3) {
    out = vadd<VEC>(I, O);
  } else if (a.mask == 3) {
    const int64_t d = (a.ep.op == AG_OP_MEAN && a.ep.deg) ? a.ep.deg[r] : 1;
    out = combine2<VEC>(a.ep.op, I, ni > 0, O, no > 0, d);
  } else {
    const int64_t d = (a.ep.op == AG_OP_MEAN && a.ep.deg) ? a.ep.deg[r] : 1;
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
  if (a.ep.flags & AG_EPI_GIN) {
    // x[r] sits in the ring (its own block is always resident)
    const uint32_t rr = static_cast<uint32_t>(((r / kRB) % kSlots) * kRB + (r % kRB));
    const Vf<VEC> xr = lv_out<VEC>(lv_lds<VEC>(w.ring + rr * (32u * VEC * 4u)));
    out = vadd<VEC>(vscale<VEC>(a.ep.gin_scale, xr), out);
  }
  if (a.ep.flags & AG_EPI_RELU) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) out.v[i] = fmaxf(out.v[i], 0.0f);
  }
  if (relu) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) out.v[i] = (rbits >> i) & 1u ? out.v[i] : 0.0f;
  }
  if (a.relu_out != nullptr) {
    // y's relu bits: lane l holds columns fcol .. fcol + VEC - 1 of the tile
    uint32_t *rw = a.relu_out + r * a.ldw;
    const int64_t c0 = fcol - static_cast<int64_t>(w.lane) * VEC;  // the tile's first column
    if constexpr (VEC == 1) {
      const uint32_t b = __ballot_sync(0xffffffffu, act && out.v[0] > 0.0f);
      if (w.lane == 0) rw[c0 >> 5] = b;
    } else {
      const uint32_t b0 = __ballot_sync(0xffffffffu, act && out.v[0] > 0.0f);
      const uint32_t b1 = __ballot_sync(0xffffffffu, act && out.v[1] > 0.0f);
      const uint32_t wd = w.lane == 0 ? spread16(b0) | (spread16(b1) << 1)
                                      : spread16(b0 >> 16) | (spread16(b1 >> 16) << 1);
      if (w.lane < 2 && c0 + 32 * w.lane < a.feat) rw[(c0 >> 5) + w.lane] = wd;
    }
  }
  if (act && !(a.dbg & 16)) stv<VEC>(yp, out);
}

// Band-kernel topology records (see band_kernel): per 16-row block, a 64-byte
// header of row words, the block's inter (code, weight) pairs, and (staged
// next to them) the block's ReLU-mask words.
constexpr int kBandCap = 560;               // pairs staged per block (more: read from global)
constexpr uint32_t kRecHdr = 64;            // 16 row words
constexpr uint32_t kRecRelu = 512;          // 16 rows x up to 8 mask words (feat <= 256)
constexpr uint32_t kRecSlot = kRecHdr + kBandCap * 8 + kRecRelu;
constexpr int kTopoSlots = 8;               // band topology FIFO depth (blocks)

// Shared-memory geometry of one slab-family kernel: an X ring of SLOTS blocks
// (column tile T = 32 * VEC), the far ring, intra slots, dense-warp weights,
// the barriers, then per-warp windows (slab) or the topology FIFO (band).
template <int VEC_, int SLOTS = kSlots, bool BAND = false>
struct SlabGeom {
  static constexpr int VEC = VEC_;
  static constexpr int kSlotsN = SLOTS;
  static constexpr int kFarRow = SLOTS * kRB;  // first far-ring row (codes >= kFarRow)
  static constexpr int T = 32 * VEC;
  static constexpr uint32_t kRowBytes = T * 4;
  static constexpr uint32_t kSlotBytes = kRB * kRowBytes;
  static constexpr uint32_t kFarSlotBytes = kFarMax * kRowBytes;
  static constexpr uint32_t kIOff = SLOTS * kSlotBytes + (BAND ? 0 : kFarSlots * kFarSlotBytes);
  static constexpr uint32_t kWOff = kIOff + kISlots * kSlotBytes;  // 2 warps x 2 x 512 B weights
  static constexpr uint32_t kRingBytes = kWOff + 2 * 1024;
  static constexpr uint32_t kBarBytes = (kReady + kDone + kISlots) * 8;
  static constexpr uint32_t kWinBytes = BAND ? 0 : kConsMax * kWin * 8;
  static constexpr uint32_t kTopoBytes = BAND ? kTopoSlots * kRecSlot : 0;
  static constexpr size_t kSmem = kRingBytes + kBarBytes + kWinBytes + kTopoBytes;
  static_assert(kBarBytes % 16 == 0 && kRecSlot % 16 == 0, "16-byte aligned topology slots");
};

// Bulk L2 prefetch of [p, p + bytes), widened to 16-byte granules.
__device__ __forceinline__ void l2_prefetch(const void *p, int64_t bytes) {
  if (bytes <= 0) return;
  const uintptr_t lo = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t hi = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo),
               "r"(static_cast<uint32_t>(hi - lo))
               : "memory");
}
// One lane per block: pull block b's rows of the topology into L2 so the
// consumers' per-row loads (rowinfo, first kWin pairs) hit L2.  The block's
// pair range [e0, e1) was loaded one batch earlier (topo_bounds).
struct TopoBounds {
  int32_t e0, e1;
};
__device__ __forceinline__ TopoBounds topo_bounds(const GArgs &a, uint32_t b, uint32_t kb1) {
  TopoBounds t{0, 0};
  if (a.brec != nullptr) {  // band kernel: the block's record
    if (b < kb1) {
      t.e0 = a.brec_off[b];
      t.e1 = a.brec_off[b + 1];
    }
    return t;
  }
  if (b < kb1) {
    const int64_t r0 = static_cast<int64_t>(b) * kRB;
    t.e0 = a.row_ptr[r0];
    t.e1 = a.row_ptr[std::min<int64_t>(r0 + kRB, a.rows)];
  }
  return t;
}
__device__ __forceinline__ void prefetch_topology(const GArgs &a, uint32_t b, uint32_t kb0,
                                                  uint32_t kb1, TopoBounds tb, int64_t c0,
                                                  int64_t tile_bytes) {
  if (b < kb0 || b >= kb1) return;
  if (a.brec != nullptr) {  // band: the record and the block's far rows (read by the consumers)
    l2_prefetch(a.brec + tb.e0, static_cast<int64_t>(tb.e1 - tb.e0) * 16);
    return;
  }
  const int64_t r0 = static_cast<int64_t>(b) * kRB;
  const int64_t r1 = std::min<int64_t>(r0 + kRB, a.rows);
  l2_prefetch(a.rowinfo + r0, (r1 - r0) * 16);
  l2_prefetch(a.cv + tb.e0, static_cast<int64_t>(tb.e1 - tb.e0) * 8);
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// tx expectation without an arrival (more X blocks feed the same block)
__device__ __forceinline__ void mbar_expect_tx_only(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}

// Development trace (build with -DAG_SLAB_TRACE_BUILD, run with AG_SLAB_TRACE=1): per-block
// globaltimer stamps of CTA 0's producers / consumer warps, printed by the host.  Compiled
// out by default.
constexpr int kTraceBlocks = 64;
__device__ __forceinline__ void tstamp(const GArgs &a, uint32_t fi, int slot) {
#ifdef AG_SLAB_TRACE_BUILD
  if (a.trace != nullptr && blockIdx.x == 0 && fi < kTraceBlocks) {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    a.trace[fi * 8 + slot] = t;
  }
#endif
}

// Per-block synchronisation, relative to the range's first block kb0:
//   ready[(k - kb0) % kReady]  completes when consumer block k can run: every
//       X block of its window is in the X ring and its far rows are staged
//       (2 arrivals -- X producer, far producer -- plus the copies' bytes);
//   done[(k - kb0) % kDone]    completes when all consumers left block k.
// Phases are ((k - kb0) / n) & 1.  done completes in block order (each warp
// leaves blocks in order), so waiting on done[j] covers every block <= j.
struct BlockSync {
  uint32_t ready, done, kb0;
  int sleep;  // wait_done suspends between polls (1) or spins (0)
  __device__ __forceinline__ uint32_t rdy(uint32_t k) const {
    return ready + ((k - kb0) % kReady) * 8;
  }
  __device__ __forceinline__ uint32_t rdy_phase(uint32_t k) const {
    return ((k - kb0) / kReady) & 1u;
  }
  __device__ __forceinline__ void wait_done(uint32_t k) const {
    if (sleep) mbar_wait_sleep(done + ((k - kb0) % kDone) * 8, ((k - kb0) / kDone) & 1u);
    else mbar_wait(done + ((k - kb0) % kDone) * 8, ((k - kb0) / kDone) & 1u);
  }
};

// X producer warp: streams X blocks [Llo, Lhi) of column tile `tile` into
// the X ring slot b % kSlots, one TMA tensor tile per block (cp.async element
// copies when x is not TMA-addressable).  Block t is first needed by
// consumer block kt = max(kb0, t - H) and completes on ready[kt].  Before
// overwriting a slot it waits until no consumer block still needs the old
// block (done[t - kSlots + H]).  It also pulls the topology into L2 ahead.
template <class G>
__device__ __forceinline__ void produce_x(const GArgs &a, const CUtensorMap *map, uint32_t ring,
                                          const BlockSync &bs, uint32_t Llo, uint32_t Lhi,
                                          uint32_t kb0, uint32_t kb1, uint32_t H, int tile,
                                          int lane) {
  constexpr int VEC = G::VEC;
  constexpr int kSlots = G::kSlotsN;
  const int64_t c0 = static_cast<int64_t>(tile) * G::T;
  uint32_t slot = Llo % kSlots;
  TopoBounds tb = topo_bounds(a, Llo + lane, kb1);
  TopoBounds tb_next = topo_bounds(a, Llo + 32 + lane, kb1);
  for (uint32_t t = Llo; t < Lhi; ++t) {
    const uint32_t i = t - Llo;
    if (i % 32 == 0) {
      prefetch_topology(a, t + lane, kb0, kb1, tb, c0, std::min<int64_t>(G::T, a.feat - c0) * 4);
      tb = tb_next;
      tb_next = topo_bounds(a, t + 64 + lane, kb1);
    }
    const uint32_t kt = t > kb0 + H ? t - H : kb0;
    // the slot's previous block, and the ready barrier's previous block
    int64_t need = -1;
    if (t >= Llo + kSlots) need = int64_t(t) - kSlots + H;
    if (kt >= kb0 + kReady) need = std::max<int64_t>(need, int64_t(kt) - kReady);
    const bool last = t == kt + H || t + 1 == Lhi;  // last X block feeding ready[kt]
    const uint32_t dst = ring + slot * G::kSlotBytes;
    if (a.tma) {
      if (lane == 0) {
        if (need >= 0) bs.wait_done(static_cast<uint32_t>(need));
        const uint32_t xb = (a.dbg & 8) ? 0u : G::kSlotBytes;
        if (last) {
          tstamp(a, kt - kb0, 2);
          mbar_expect_tx(bs.rdy(kt), xb);
        }
        else if (xb) mbar_expect_tx_only(bs.rdy(kt), xb);
        if (xb) tma_load_2d(dst, map, bs.rdy(kt), static_cast<int>(c0), static_cast<int>(t * kRB));
      }
    } else {
      if (need >= 0) bs.wait_done(static_cast<uint32_t>(need));
#pragma unroll 4
      for (int rr = 0; rr < kRB; ++rr) {
        const int64_t row = static_cast<int64_t>(t) * kRB + rr;  // past x_rows: zero
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
          const int64_t c = c0 + lane * VEC + j;
          const bool ok = row < a.x_rows && c < a.feat;
          cp_async4(dst + (rr * G::T + lane * VEC + j) * 4, ok ? a.x + row * a.feat + c : a.x,
                    ok ? 4 : 0);
        }
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
      if (lane == 0 && last) mbar_arrive(bs.rdy(kt));
    }
    __syncwarp();
    if (++slot == kSlots) slot = 0;
  }
  // consumer blocks whose window ends past the last X block: arrive plainly
  const uint32_t k0 = std::max(kb0 + 1, Lhi > H ? Lhi - H : 0u);
  for (uint32_t k = k0; k < kb1; ++k) {
    if (lane == 0) {
      if (k >= kb0 + kReady) bs.wait_done(k - kReady);
      mbar_arrive(bs.rdy(k));
    }
  }
  __syncwarp();
}

// Band kernel: block f's ReLU-mask words (16 rows x ldw words, contiguous) are
// staged with its record when they fit the slot and the block is whole.
__device__ __forceinline__ bool band_relu_staged(const GArgs &a, uint32_t f) {
  return a.relu && a.ldw * kRB * 4 <= kRecRelu && int64_t(f + 1) * kRB <= a.rows;
}

// Far producer warp: for every consumer block f in [kb0, kb1), copies the
// tile columns of its staged far sources (far_src; one bulk copy per source,
// lanes in parallel; cp.async elements when x is not bulk-copyable) into
// far-ring slot f % kFarSlots once every consumer left block f - kFarSlots,
// completing on ready[f].  Look-ahead loads are consumed in place (the loop
// is unrolled by D): rotating them through moves would wait on each load.
template <class G>
__device__ __forceinline__ void produce_far(const GArgs &a, uint32_t ring, const BlockSync &bs,
                                            uint32_t kb0, uint32_t kb1, int tile, int lane) {
  constexpr int VEC = G::VEC;
  constexpr int D = 4;
  const uint32_t far_ring = ring + G::kSlotsN * G::kSlotBytes;
  const int64_t c0 = static_cast<int64_t>(tile) * G::T;
  const uint32_t tile_bytes =
      static_cast<uint32_t>(std::min<int64_t>(G::T, a.feat - c0)) * 4u;  // partial last tile
  auto far_list = [&](uint32_t f) -> int32_t {
    return (f < kb1 && lane < kFarMax) ? a.far_src[static_cast<int64_t>(f) * kFarMax + lane] : 0;
  };
  auto far_counts = [&](uint32_t f) -> int32_t { return f + lane < kb1 ? a.far_cnt[f + lane] : 0; };
  int32_t fsa[D];
#pragma unroll
  for (int u = 0; u < D; ++u) fsa[u] = far_list(kb0 + u);
  int32_t fc = far_counts(kb0), fc_next = far_counts(kb0 + 32);
  uint32_t fslot = kb0 % kFarSlots;
  for (uint32_t fb = kb0; fb < kb1; fb += D) {
#pragma unroll
    for (int u = 0; u < D; ++u) {
      const uint32_t f = fb + u;
      if (f >= kb1) break;
      const uint32_t fi = f - kb0;
      const int cnt = __shfl_sync(0xffffffffu, fc, fi & 31);
      const int32_t src = fsa[u];
      fsa[u] = far_list(f + D);
      if ((fi & 31) == 31) {
        fc = fc_next;
        fc_next = far_counts(f + 33);
      }
      const uint32_t slot_base = far_ring + fslot * G::kFarSlotBytes;
      if (++fslot == kFarSlots) fslot = 0;
      // far slot reuse: done[f - kFarSlots]
      const int64_t need = int64_t(f) - kFarSlots;
      if (a.tma) {
        if (lane == 0) {
          tstamp(a, fi, 0);
          if (need >= int64_t(kb0)) bs.wait_done(static_cast<uint32_t>(need));
          tstamp(a, fi, 1);
          mbar_expect_tx(bs.rdy(f), (a.dbg & 2) ? 0u : static_cast<uint32_t>(cnt) * tile_bytes);
        }
        __syncwarp();
        if (lane < cnt && !(a.dbg & 2))
          bulk_g2s(slot_base + lane * G::kRowBytes, a.x + static_cast<int64_t>(src) * a.feat + c0,
                   tile_bytes, bs.rdy(f));

      } else {
        if (need >= int64_t(kb0)) bs.wait_done(static_cast<uint32_t>(need));
        for (int j = 0; j < cnt; ++j) {
          const int32_t sj = __shfl_sync(0xffffffffu, src, j);
#pragma unroll
          for (int v = 0; v < VEC; ++v) {
            const int64_t c = c0 + lane * VEC + v;
            const bool ok = c < a.feat;
            cp_async4(slot_base + j * G::kRowBytes + (lane * VEC + v) * 4,
                      ok ? a.x + static_cast<int64_t>(sj) * a.feat + c : a.x, ok ? 4 : 0);
          }
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        if (lane == 0) mbar_arrive(bs.rdy(f));
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

// Band topology producer: block f's record (header + pairs, or the header
// alone when the block is unstaged) and its ReLU-mask words into topology
// slot f % kTopoSlots once every consumer left block f - kTopoSlots,
// completing on ready[f].  Record offsets are read 32 blocks at a time.
template <class G>
__device__ __forceinline__ void produce_topo(const GArgs &a, uint32_t ring, const BlockSync &bs,
                                             uint32_t kb0, uint32_t kb1, int tile, int lane) {
  const uint32_t topo = ring + G::kRingBytes + G::kBarBytes + G::kWinBytes;
  auto rec_offs = [&](uint32_t f) -> int32_t {
    return (f + lane <= a.nblocks) ? a.brec_off[f + lane] : 0;
  };
  int32_t ro = rec_offs(kb0), ro_next = rec_offs(kb0 + 32);
  // far rows of block f + kFarAhead into L2 (the consumers load them), the
  // source list loaded one block earlier
  constexpr uint32_t kFarAhead = 12;
  const int64_t c0 = static_cast<int64_t>(tile) * G::T;
  const uint32_t tile_bytes = static_cast<uint32_t>(std::min<int64_t>(G::T, a.feat - c0)) * 4u;
  const bool pf = !(a.dbg & 64);  // 64: development, no far-row prefetch
  auto far_at = [&](uint32_t f) -> int32_t {  // -1: none
    if (!pf || f >= kb1 || lane >= kFarMax) return -1;
    return lane < a.far_cnt[f] ? a.far_src[static_cast<int64_t>(f) * kFarMax + lane] : -1;
  };
  for (uint32_t f = kb0; f < kb0 + kFarAhead; ++f) {
    const int32_t src = far_at(f);
    if (src >= 0) l2_prefetch(a.x + static_cast<int64_t>(src) * a.feat + c0, tile_bytes);
  }
  int32_t fnext = far_at(kb0 + kFarAhead);
#pragma unroll 1
  for (uint32_t f = kb0; f < kb1; ++f) {
    const uint32_t fi = f - kb0;
    if (fnext >= 0) l2_prefetch(a.x + static_cast<int64_t>(fnext) * a.feat + c0, tile_bytes);
    fnext = far_at(f + kFarAhead + 1);
    const int32_t o0 = __shfl_sync(0xffffffffu, ro, fi & 31);
    const int32_t o1 = __shfl_sync(0xffffffffu, (fi & 31) == 31 ? ro_next : ro, (fi + 1) & 31);
    if ((fi & 31) == 31) {
      ro = ro_next;
      ro_next = rec_offs(f + 33);
    }
    if (lane == 0) {
      const uint32_t rb = static_cast<uint32_t>(o1 - o0) * 16u;
      const uint32_t rec_bytes = rb <= kRecHdr + kBandCap * 8 ? rb : kRecHdr;  // unstaged: header
      const uint32_t relu_bytes =
          band_relu_staged(a, f) ? static_cast<uint32_t>(kRB * a.ldw * 4) : 0u;
      tstamp(a, fi, 0);
      if (fi >= kTopoSlots) bs.wait_done(f - kTopoSlots);
      tstamp(a, fi, 1);
      const uint32_t tslot = topo + (f % kTopoSlots) * kRecSlot;
      mbar_expect_tx(bs.rdy(f), rec_bytes + relu_bytes);
      bulk_g2s(tslot, a.brec + o0, rec_bytes, bs.rdy(f));
      if (relu_bytes)
        bulk_g2s(tslot + kRecHdr + kBandCap * 8,
                 a.ep.relu_bits + static_cast<int64_t>(f) * kRB * a.ldw, relu_bytes, bs.rdy(f));
    }
    __syncwarp();
  }
}

// Dense-intra warp (kModeDense3): for every block f in [kb0, kb1), the 16 x 16
// intra weight block (cp.async, one block ahead) times the block's 16 X rows
// (already in the ring) -> the 16 intra partials of this column tile, into
// I-slot f % kISlots for the consumers' epilogues.  Register-blocked: each X
// row is read from shared memory once per block instead of once per edge.
constexpr int kDenseWarps = 2;  // each takes 16 / kDenseWarps rows of every block (measured: 2 > 1, 4)

template <class G, int ND = kDenseWarps>
__device__ __forceinline__ void dense_intra(const GArgs &a, uint32_t ring, const BlockSync &bs,
                                            uint32_t ivalid, uint32_t kb0, uint32_t kb1,
                                            int lane, int half) {
  constexpr int VEC = G::VEC;
  // this warp's own double buffer of its kRB / kDenseWarps weight rows (the
  // warps drift apart by a block, so they must not share one)
  constexpr int kRows = kRB / ND;
  constexpr uint32_t kBuf = kRows * kRB * 4;  // 512 B for 2 warps
  const uint32_t wbuf = ring + G::kWOff + half * 2 * kBuf;
  auto fetch_w = [&](uint32_t f, int buf) {  // 16 bytes per lane
    if (f < kb1 && lane * 16u < kBuf)
      cp_async16(wbuf + buf * kBuf + lane * 16,
                 a.blk_w + static_cast<int64_t>(f) * 256 + half * kRows * kRB + lane * 4);
    cp_async_commit();
  };
  fetch_w(kb0, 0);
#pragma unroll 1
  for (uint32_t f = kb0; f < kb1; ++f) {
    const uint32_t fi = f - kb0;
    const int buf = static_cast<int>(fi & 1u);
    fetch_w(f + 1, buf ^ 1);
    cp_async_wait<1>();  // this block's weights have landed
    __syncwarp();
    mbar_wait_hint(bs.rdy(f), bs.rdy_phase(f), a.csleep);  // X block f is in the ring
    if (fi >= kISlots) bs.wait_done(f - kISlots);  // the I slot's previous block is consumed
    if (a.dbg & 4) {
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(ivalid + (fi % kISlots) * 8);
        mbar_arrive(bs.done + (fi % kDone) * 8);
      }
      continue;
    }
    const uint32_t xs = ring + (f % G::kSlotsN) * G::kSlotBytes + lane * VEC * 4;
    Lv<VEC> xr[kRB];
#pragma unroll
    for (int j = 0; j < kRB; ++j) xr[j] = lv_lds<VEC>(xs + j * G::kRowBytes);
    const uint32_t is = ring + G::kIOff + (fi % kISlots) * G::kSlotBytes + lane * VEC * 4;
    const uint32_t wrow = wbuf + buf * kBuf;
#pragma unroll 2
    for (int i = half * kRows; i < (half + 1) * kRows; ++i) {
      float wv[kRB];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(wv[4 * q]), "=f"(wv[4 * q + 1]), "=f"(wv[4 * q + 2]),
                       "=f"(wv[4 * q + 3])
                     : "r"(wrow + (i - half * kRows) * 64 + q * 16));
      Lv<VEC> acc = lv_scale<VEC>(xr[0], wv[0]);
#pragma unroll
      for (int j = 1; j < kRB; ++j) {
        if constexpr (VEC == 1) {
          acc.s = __fmaf_rn(xr[j].s, wv[j], acc.s);
        } else {
          const uint64_t ww = pk(wv[j], wv[j]);
#pragma unroll
          for (int pp = 0; pp < Lv<VEC>::NP; ++pp)
            asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc.p[pp]) : "l"(xr[j].p[pp]), "l"(ww));
        }
      }
      if constexpr (VEC == 1) {
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(is + i * G::kRowBytes), "f"(acc.s) : "memory");
      } else {
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(is + i * G::kRowBytes), "l"(acc.p[0])
                     : "memory");
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (half == 0) tstamp(a, fi, 6);
      mbar_arrive(ivalid + (fi % kISlots) * 8);
      mbar_arrive(bs.done + (fi % kDone) * 8);
    }
  }
  cp_async_wait<0>();
}

template <int VEC, int MODE, bool W>
__global__ void __launch_bounds__((cons_warps<MODE>() + 2) * 32, 1)
    slab_kernel(const __grid_constant__ CUtensorMap tmap, GArgs a) {
  using G = SlabGeom<VEC>;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int64_t s_kb[2];
  const uint32_t ring = su32(smem);
  const uint32_t ready = ring + G::kRingBytes;
  const uint32_t done = ready + kReady * 8;
  const uint32_t ivalid = done + kDone * 8;  // dense-intra mode: I slot of block k written
  const uint32_t wins = ivalid + kISlots * 8;
  constexpr bool DENSE = mode_dense(MODE);
  constexpr int kCons = cons_warps<MODE>();
  constexpr int NC = DENSE ? kCons - kDenseWarps : kCons;  // consumer warps (dense warps last)
  // kModeDense3Coo defers a block's ivalid wait to the warp's first epilogue in
  // it: every consumer warp must own a row of every block, or a warp skipping
  // kISlots blocks could pass a stale-parity wait
  static_assert((NC - 1) * kRG < kRB, "every consumer warp needs a row in every block");
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t H = static_cast<uint32_t>(a.H);
  const int64_t units = static_cast<int64_t>(a.ranges) * a.ntiles;
  if (a.tma && threadIdx.x == kCons * 32) tma_prefetch_desc(&tmap);

#pragma unroll 1
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int tile = static_cast<int>(u % a.ntiles);
    const int range = static_cast<int>(u / a.ntiles);
    if (threadIdx.x == 0) {
      s_kb[0] = range_block(a, range);
      s_kb[1] = range_block(a, range + 1);
      for (int s = 0; s < kReady; ++s) mbar_init(ready + s * 8, 2);
      for (int s = 0; s < kDone; ++s) mbar_init(done + s * 8, kCons);  // (+ the dense warp)
      for (int s = 0; s < kISlots; ++s) mbar_init(ivalid + s * 8, kDenseWarps);
      fence_mbar_init();
    }
    __syncthreads();
    const uint32_t kb0 = static_cast<uint32_t>(s_kb[0]), kb1 = static_cast<uint32_t>(s_kb[1]);
    const uint32_t Llo = kb0 > H ? kb0 - H : 0u;
    const uint32_t Lhi = static_cast<uint32_t>(std::min<int64_t>(a.xblocks, int64_t(kb1) + H));
    const BlockSync bs{ready, done, kb0, a.sleep};
    if (kb0 < kb1) {
      if (warp == kCons) {
        produce_x<G>(a, &tmap, ring, bs, Llo, Lhi, kb0, kb1, H, tile, lane);
      } else if (warp == kCons + 1) {
        produce_far<G>(a, ring, bs, kb0, kb1, tile, lane);
      } else if (DENSE && warp >= kCons - kDenseWarps) {
        dense_intra<G>(a, ring, bs, ivalid, kb0, kb1, lane, warp - (kCons - kDenseWarps));
      } else {
        RowWarp<VEC, W> w;
        const int64_t fcol = static_cast<int64_t>(tile) * G::T + lane * VEC;
        const bool act = fcol < a.feat;
        w.win = wins + warp * kWin * 8;
        w.ring = ring + lane * VEC * 4;
        w.cv = a.cv;
        w.xl = a.x + (act ? fcol : 0);
        w.feat = static_cast<uint32_t>(a.feat);
        w.lane = lane;
        w.one = pk(a.one, a.one);
        w.p = 0;
        w.end = 0;
        w.far = 0;
        float *const ylane = a.y + (act ? fcol : 0);
        const uint32_t ld = static_cast<uint32_t>(a.feat);
        const uint32_t r0 = kb0 * kRB;
        const uint32_t r1 = static_cast<uint32_t>(std::min<int64_t>(int64_t(kb1) * kRB, a.rows));
        // Topology pipeline in registers: rowinfo two rows ahead, the first
        // kWin (code, weight) pairs one row ahead.  Both are issued before
        // the current row's reduction and only moved after it, so each load
        // has a full row of work to land.
        const int4 zero4 = make_int4(0, 0, 0, 0);
        const bool notopo = (a.dbg & 32) != 0;  // experiment: rows without topology loads
        auto info_at = [&](uint32_t rr) -> int4 {
          return (rr < r1 && !notopo) ? __ldg(a.rowinfo + rr) : zero4;
        };
        auto pairs_at = [&](const int4 &inf, int h) -> int2 {
          const int32_t ed = inf.x + h * 32 + lane;
          return (ed < inf.z && !notopo) ? __ldg(a.cv + ed) : make_int2(0, 0);
        };
        // rows go to warps in groups of kRG consecutive rows (one block
        // change per group instead of per row); a warp's next row:
        auto next_row = [&](uint32_t r) -> uint32_t {
          return (r % kRG != kRG - 1) ? r + 1 : r + (NC - 1) * kRG + 1;
        };
        // ReLU-backward mask words, one row ahead like the topology
        const bool relu_rows = a.relu && act;
        auto rword_at = [&](uint32_t rrow) -> uint32_t {
          return (relu_rows && rrow < r1) ? __ldg(a.ep.relu_bits + static_cast<int64_t>(rrow) * a.ldw +
                                                  (fcol >> 5))
                                          : 0u;
        };
        uint32_t rr = r0 + warp * kRG;
        int4 info = info_at(rr);
        uint32_t rw = rword_at(rr);
        int2 q0 = pairs_at(info, 0), q1 = pairs_at(info, 1);
        uint32_t rn = next_row(rr);
        int4 info1 = info_at(rn);
        uint32_t kcur = kb0;
        // entering block k: its X window and far rows (ready), and in
        // dense-intra mode its intra partials
        bool iv_pending = false;  // dense-intra: the current block's ivalid not yet waited for
        auto enter = [&](uint32_t k) {
          if (warp == 0 && lane == 0) tstamp(a, k - kb0, 3);
          mbar_wait_hint(bs.rdy(k), bs.rdy_phase(k), a.csleep);
          if (warp == 0 && lane == 0) tstamp(a, k - kb0, 4);
          // dense + coo: waited for at the first epilogue in the block (measured
          // faster); dense + csr: here (the deferred wait costs it registers)
          if (MODE == kModeDense3Coo) iv_pending = true;
          else if (DENSE)
            mbar_wait_hint(ivalid + ((k - kb0) % kISlots) * 8, ((k - kb0) / kISlots) & 1u, a.csleep);
        };
        bool entered = false;
#pragma unroll 1
        for (; rr < r1; rr = rn, rn = next_row(rn)) {
          const uint32_t k = rr / kRB;
          if (kcur != k || !entered) {  // leave the blocks before k (rows or not), enter k
            __syncwarp();
            for (; kcur != k; ++kcur)
              if (lane == 0) {
                if (warp == 0) tstamp(a, kcur - kb0, 5);
                if (warp == NC - 1) tstamp(a, kcur - kb0, 7);
                mbar_arrive(done + ((kcur - kb0) % kDone) * 8);
              }
            enter(k);
            entered = true;
          }
          const int32_t s = info.x, e = info.z;
          const int32_t m =
              (mode_sum3(MODE) || a.has_mid) ? info.y : (a.mask == 1 ? e : s);
          const bool fast = !(info.w & kRowSlow);
          w.end = e;
          if (fast) w.template install<true>(s, q0, q1);
          else w.template install<false>(s, q0, q1);
          // next row's pairs and mask word, the row after next's bounds
          const int2 n0 = pairs_at(info1, 0), n1 = pairs_at(info1, 1);
          const uint32_t rw1 = rword_at(rn);
          const int4 info2 = info_at(next_row(rn));
          float *yrow;  // ylane + rr * ld as one IMAD.WIDE.U32
          asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(yrow) : "r"(rr), "r"(ld * 4u), "l"(ylane));
          const uint32_t intra_s = ring + G::kIOff + ((k - kb0) % kISlots) * G::kSlotBytes +
                                   (rr % kRB) * G::kRowBytes + lane * VEC * 4;
          if constexpr (MODE == kModeDense3Coo)
            do_row<VEC, MODE, W>(a, w, rr, s, e, m, yrow, act, fast, fcol, intra_s, rw,
                                 ivalid + ((k - kb0) % kISlots) * 8, ((k - kb0) / kISlots) & 1u,
                                 &iv_pending);
          else
            do_row<VEC, MODE, W>(a, w, rr, s, e, m, yrow, act, fast, fcol, intra_s, rw);
          info = info1;
          info1 = info2;
          q0 = n0;
          q1 = n1;
          rw = rw1;
        }
        __syncwarp();
        for (; kcur < kb1; ++kcur)  // leave the rest of the range
          if (lane == 0) mbar_arrive(done + ((kcur - kb0) % kDone) * 8);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int s = 0; s < kReady; ++s) mbar_inval(ready + s * 8);
      for (int s = 0; s < kDone; ++s) mbar_inval(done + s * 8);
      for (int s = 0; s < kISlots; ++s) mbar_inval(ivalid + s * 8);
    }
    __syncthreads();
  }
}

// ===================================================================== band ==
// The band kernel: the order-free selector pair (dense_block intra, coo_atomic
// inter; kModeDense3Coo's semantics) with a leaner consumer.  The slab
// consumer fetches every row's rowinfo, pairs and mask word from global
// memory, installs the pairs into a per-warp window and runs a general
// epilogue: ~200 issue slots of control per row-tile, which bounds it.  Here
// the far producer also bulk-copies each block's TOPOLOGY RECORD (built once
// per graph by ag_band_records) and its ReLU-mask words into a shared-memory
// slot next to the block's far rows, completing on the same ready barrier:
//   record = 16 row words (end offset of the row's pairs | kRowGlobal) and the
//            block's inter (code, weight) pairs in row order, codes as in the
//            slab layout but for the band ring (kBandSlots blocks);
// so a consumer warp's row is: two shared-memory loads for its bounds, the
// pairs two at a time (one broadcast LDS.128 per two edges), one conflict-
// free 256-byte gather and one FFMA2 per edge, then the epilogue.  The only
// global accesses left in the consumers are the y stores.
constexpr int kBandSlots = 42;
constexpr int kBandMaxWindow = (kBandSlots - 9) / 2;  // 16 blocks
#ifndef AG_BAND_CONS
#define AG_BAND_CONS 26
#endif
#ifndef AG_BAND_DENSE
#define AG_BAND_DENSE 2
#endif
// consumer warps (rows round-robin) and dense-intra warps (each 16 / kBandDense
// rows of every block): many consumers starve a single-warp stage of issue
// slots, so the dense product is split over several warps
constexpr int kBandCons = AG_BAND_CONS;
constexpr int kBandDense = AG_BAND_DENSE;
constexpr uint32_t kRowEndMask = 0xFFFFFu;
constexpr uint32_t kRowGlobal = 1u << 30;    // the row has sources in global memory
constexpr uint32_t kBlkUnstaged = 1u << 31;  // the block has > kBandCap pairs: read them from global
using BandGeom = SlabGeom<2, kBandSlots, true>;
static_assert(BandGeom::kSmem + 256 <= 232448, "band kernel shared memory");
// a consumer's consecutive rows are kBandCons apart: it skips at most
// kBandCons / kRB blocks, fewer than the kISlots intra slots (stale-parity safe)
static_assert(kBandCons / kRB + 1 < kISlots, "consumer row stride vs intra slots");

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void lds_pair2(uint32_t addr, int32_t &c0, float &w0, int32_t &c1,
                                          float &w1) {
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(c0), "=f"(w0), "=r"(c1), "=f"(w1)
               : "r"(addr));
}
__device__ __forceinline__ void lds_pair(uint32_t addr, int32_t &c, float &w) {
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(c), "=f"(w) : "r"(addr));
}
__device__ __forceinline__ uint64_t lds_x(uint32_t xl, int32_t code) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(xl + static_cast<uint32_t>(code) * 256u));
  return v;
}
__device__ __forceinline__ void fma2(uint64_t &acc, uint64_t x, float w) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(x), "l"(pk(w, w)));
}

// One band row: the inter pairs [s, e) of record `pairs` (shared), all in the
// X ring or the far ring.
__device__ __forceinline__ uint64_t ldg_x(const float *xg, uint32_t feat, int32_t code) {
  const float *ptr;  // xg + src * feat as one IMAD.WIDE.U32
  asm("mad.wide.u32 %0, %1, %2, %3;"
      : "=l"(ptr)
      : "r"(static_cast<uint32_t>(~code)), "r"(feat * 4u), "l"(xg));
  uint64_t v;
  asm("ld.global.nc.b64 %0, [%1];" : "=l"(v) : "l"(ptr));
  return v;
}

// One band row: its nf leading far pairs (sources in global memory, loaded
// first so their latency overlaps the ring part), then the ring pairs up to e.
__device__ __forceinline__ uint64_t band_row_fast(uint32_t pairs, uint32_t xl, const float *xg,
                                                  uint32_t feat, uint32_t s, uint32_t e,
                                                  uint32_t nf) {
  uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;  // +0.0f pairs
  uint64_t fx[4];
  float fw[4];
  const uint32_t nq = nf < 4 ? nf : 4;
#pragma unroll
  for (uint32_t q = 0; q < 4; ++q) {
    fx[q] = 0;
    fw[q] = 0.0f;
    if (q < nq) {
      int32_t c;
      lds_pair(pairs + (s + q) * 8u, c, fw[q]);
      fx[q] = ldg_x(xg, feat, c);
    }
  }
#pragma unroll 1
  for (uint32_t j = s + 4; j < s + nf; ++j) {  // rows with more than 4 far sources
    int32_t c;
    float w;
    lds_pair(pairs + j * 8u, c, w);
    fma2(a1, ldg_x(xg, feat, c), w);
  }
  s += nf;
  uint32_t p = pairs + s * 8u;
  int n = static_cast<int>(e - s);
  if (n > 0 && (s & 1u)) {  // align to a pair of pairs
    int32_t c;
    float w;
    lds_pair(p, c, w);
    fma2(a0, lds_x(xl, c), w);
    p += 8;
    --n;
  }
#pragma unroll 1
  for (; n >= 8; n -= 8, p += 64) {
    int32_t c[8];
    float w[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) lds_pair2(p + 16 * q, c[2 * q], w[2 * q], c[2 * q + 1], w[2 * q + 1]);
    uint64_t x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = lds_x(xl, c[q]);
    fma2(a0, x[0], w[0]);
    fma2(a1, x[1], w[1]);
    fma2(a2, x[2], w[2]);
    fma2(a3, x[3], w[3]);
    fma2(a0, x[4], w[4]);
    fma2(a1, x[5], w[5]);
    fma2(a2, x[6], w[6]);
    fma2(a3, x[7], w[7]);
  }
  if (n >= 4) {
    int32_t c[4];
    float w[4];
    lds_pair2(p, c[0], w[0], c[1], w[1]);
    lds_pair2(p + 16, c[2], w[2], c[3], w[3]);
    uint64_t x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = lds_x(xl, c[q]);
    fma2(a0, x[0], w[0]);
    fma2(a1, x[1], w[1]);
    fma2(a2, x[2], w[2]);
    fma2(a3, x[3], w[3]);
    p += 32;
    n -= 4;
  }
  if (n >= 2) {
    int32_t c0, c1;
    float w0, w1;
    lds_pair2(p, c0, w0, c1, w1);
    const uint64_t x0 = lds_x(xl, c0), x1 = lds_x(xl, c1);
    fma2(a0, x0, w0);
    fma2(a1, x1, w1);
    p += 16;
    n -= 2;
  }
  if (n > 0) {
    int32_t c;
    float w;
    lds_pair(p, c, w);
    fma2(a2, lds_x(xl, c), w);
  }
#pragma unroll
  for (uint32_t q = 0; q < 4; ++q)
    if (q < nq) fma2(a3, fx[q], fw[q]);
  const uint64_t one = pk(1.0f, 1.0f);
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(a1), "l"(one));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a2) : "l"(a3), "l"(one));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(a2), "l"(one));
  return a0;
}

// The general band row: pairs from shared memory or (an unstaged block) from
// the global record; a source is a ring row (code >= 0) or x[~code].
__device__ __forceinline__ uint64_t band_row_slow(uint32_t pairs, const int2 *gpairs,
                                                  uint32_t xl, const float *xg, uint32_t feat,
                                                  uint32_t s, uint32_t e) {
  uint64_t a0 = 0, a1 = 0;
#pragma unroll 1
  for (uint32_t j = s; j < e; ++j) {
    int32_t c;
    float w;
    if (gpairs != nullptr) {
      const int2 q = __ldg(gpairs + j);
      c = q.x;
      w = __int_as_float(q.y);
    } else {
      lds_pair(pairs + j * 8u, c, w);
    }
    uint64_t xv;
    if (c >= 0) {
      xv = lds_x(xl, c);
    } else {
      const float *ptr;
      asm("mad.wide.u32 %0, %1, %2, %3;"
          : "=l"(ptr)
          : "r"(static_cast<uint32_t>(~c)), "r"(feat * 4u), "l"(xg));
      asm("ld.global.nc.b64 %0, [%1];" : "=l"(xv) : "l"(ptr));
    }
    fma2((j & 1u) ? a1 : a0, xv, w);
  }
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(a1), "l"(pk(1.0f, 1.0f)));
  return a0;
}

__device__ __forceinline__ void band_consume(const GArgs &a, uint32_t ring, uint32_t topo,
                                             const BlockSync &bs, uint32_t ivalid, uint32_t kb0,
                                             uint32_t kb1, int tile, int warp, int lane) {
  using G = BandGeom;
  const int64_t fcol = static_cast<int64_t>(tile) * G::T + lane * 2;
  const bool act = fcol < a.feat;
  const uint32_t xl = ring + lane * 8;
  float *const ylane = a.y + (act ? fcol : 0);
  const float *const xg = a.x + (act ? fcol : 0);
  const uint32_t feat = static_cast<uint32_t>(a.feat);
  const uint32_t wsel = static_cast<uint32_t>(fcol >> 5);
  const uint32_t r0 = kb0 * kRB;
  const uint32_t r1 = static_cast<uint32_t>(std::min<int64_t>(int64_t(kb1) * kRB, a.rows));
  uint32_t kcur = kb0;
  bool entered = false;
#pragma unroll 1
  for (uint32_t r = r0 + warp; r < r1; r += kBandCons) {
    const uint32_t k = r / kRB;
    const int i = static_cast<int>(r % kRB);
    const uint32_t fi = k - kb0;
    if (k != kcur || !entered) {  // leave the blocks before k, enter k
      __syncwarp();
      for (; kcur != k; ++kcur)
        if (lane == 0) {
          if (warp == 0) tstamp(a, kcur - kb0, 5);
          mbar_arrive(bs.done + ((kcur - kb0) % kDone) * 8);
        }
      if (warp == 0 && lane == 0) tstamp(a, fi, 3);
      mbar_wait_hint(bs.rdy(k), bs.rdy_phase(k), a.csleep);
      if (warp == 0 && lane == 0) tstamp(a, fi, 4);
      entered = true;
    }
    const uint32_t rec = topo + (k % kTopoSlots) * kRecSlot;
    const uint32_t hw = lds_u32(rec + 4 * i);
    const uint32_t s = i ? (lds_u32(rec + 4 * (i - 1)) & kRowEndMask) : 0u;
    const uint32_t e = hw & kRowEndMask;
    const uint32_t pairs = rec + kRecHdr;
    uint64_t acc;
    if (a.dbg & 1) {
      acc = 0;  // development: no reduction (values garbage)
    } else if (!(hw & (kRowGlobal | kBlkUnstaged))) {
      acc = band_row_fast(pairs, xl, xg, feat, s, e, (hw >> 20) & 0xFFu);
    } else {
      const int2 *gp = (hw & kBlkUnstaged)
                           ? reinterpret_cast<const int2 *>(a.brec + a.brec_off[k]) + kRecHdr / 8
                           : nullptr;
      acc = band_row_slow(pairs, gp, xl, xg, feat, s, e);
    }
    // the block's intra partials (dense warps)
    mbar_wait_hint(ivalid + (fi % kISlots) * 8, (fi / kISlots) & 1u, a.csleep);
    uint64_t iv;
    asm volatile("ld.shared.b64 %0, [%1];"
                 : "=l"(iv)
                 : "r"(ring + G::kIOff + (fi % kISlots) * G::kSlotBytes + i * G::kRowBytes +
                       lane * 8));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(iv), "l"(pk(1.0f, 1.0f)));
    Vf<2> out;
    upk(acc, out.v[0], out.v[1]);
    if (a.ep.flags & AG_EPI_GIN) {
      float x0, x1;
      upk(lds_x(xl, static_cast<int32_t>((k % kBandSlots) * kRB + i)), x0, x1);
      out.v[0] = __fmaf_rn(a.ep.gin_scale, x0, out.v[0]);
      out.v[1] = __fmaf_rn(a.ep.gin_scale, x1, out.v[1]);
    }
    if (a.ep.flags & AG_EPI_RELU) {
      out.v[0] = fmaxf(out.v[0], 0.0f);
      out.v[1] = fmaxf(out.v[1], 0.0f);
    }
    if (a.relu && act) {
      const uint32_t word =
          band_relu_staged(a, k)
              ? lds_u32(rec + kRecHdr + kBandCap * 8 + (static_cast<uint32_t>(i) * a.ldw + wsel) * 4)
              : __ldg(a.ep.relu_bits + static_cast<int64_t>(r) * a.ldw + wsel);
      const uint32_t rb = word >> (fcol & 31);
      if (!(rb & 1u)) out.v[0] = 0.0f;
      if (!(rb & 2u)) out.v[1] = 0.0f;
    }
    if (a.relu_out != nullptr) {
      uint32_t *rw = a.relu_out + static_cast<int64_t>(r) * a.ldw;
      const int64_t c0 = fcol - static_cast<int64_t>(lane) * 2;  // the tile's first column
      const uint32_t b0 = __ballot_sync(0xffffffffu, act && out.v[0] > 0.0f);
      const uint32_t b1 = __ballot_sync(0xffffffffu, act && out.v[1] > 0.0f);
      const uint32_t wd = lane == 0 ? spread16(b0) | (spread16(b1) << 1)
                                    : spread16(b0 >> 16) | (spread16(b1 >> 16) << 1);
      if (lane < 2 && c0 + 32 * lane < a.feat) rw[(c0 >> 5) + lane] = wd;
    }
    if (act) {
      float *yp;
      asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(yp) : "r"(r), "r"(feat * 4u), "l"(ylane));
      stv<2>(yp, out);
    }
  }
  __syncwarp();
  for (; kcur < kb1; ++kcur)  // leave the rest of the range
    if (lane == 0) mbar_arrive(bs.done + ((kcur - kb0) % kDone) * 8);
}

__global__ void __launch_bounds__((kBandCons + kBandDense + 2) * 32, 1)
    band_kernel(const __grid_constant__ CUtensorMap tmap, GArgs a) {
  using G = BandGeom;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ int64_t s_kb[2];
  const uint32_t ring = su32(smem);
  const uint32_t ready = ring + G::kRingBytes;
  const uint32_t done = ready + kReady * 8;
  const uint32_t ivalid = done + kDone * 8;
  const uint32_t topo = ring + G::kRingBytes + G::kBarBytes;
  constexpr int kCons = kBandCons + kBandDense;  // warps arriving on done
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t H = static_cast<uint32_t>(a.H);
  const int64_t units = static_cast<int64_t>(a.ranges) * a.ntiles;
  if (threadIdx.x == kCons * 32) tma_prefetch_desc(&tmap);
#pragma unroll 1
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int tile = static_cast<int>(u % a.ntiles);
    const int range = static_cast<int>(u / a.ntiles);
    if (threadIdx.x == 0) {
      s_kb[0] = range_block(a, range);
      s_kb[1] = range_block(a, range + 1);
      for (int q = 0; q < kReady; ++q) mbar_init(ready + q * 8, 2);
      for (int q = 0; q < kDone; ++q) mbar_init(done + q * 8, kCons);
      for (int q = 0; q < kISlots; ++q) mbar_init(ivalid + q * 8, kBandDense);
      fence_mbar_init();
    }
    __syncthreads();
    const uint32_t kb0 = static_cast<uint32_t>(s_kb[0]), kb1 = static_cast<uint32_t>(s_kb[1]);
    const uint32_t Llo = kb0 > H ? kb0 - H : 0u;
    const uint32_t Lhi = static_cast<uint32_t>(std::min<int64_t>(a.xblocks, int64_t(kb1) + H));
    const BlockSync bs{ready, done, kb0, a.sleep};
    if (kb0 < kb1) {
      if (warp == kCons) produce_x<G>(a, &tmap, ring, bs, Llo, Lhi, kb0, kb1, H, tile, lane);
      else if (warp == kCons + 1) produce_topo<G>(a, ring, bs, kb0, kb1, tile, lane);
      else if (warp >= kBandCons) dense_intra<G, kBandDense>(a, ring, bs, ivalid, kb0, kb1, lane, warp - kBandCons);
      else band_consume(a, ring, topo, bs, ivalid, kb0, kb1, tile, warp, lane);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 0; q < kReady; ++q) mbar_inval(ready + q * 8);
      for (int q = 0; q < kDone; ++q) mbar_inval(done + q * 8);
      for (int q = 0; q < kISlots; ++q) mbar_inval(ivalid + q * 8);
    }
    __syncthreads();
  }
}

// ---------------------------------------------- window radius (per graph) --
constexpr int kHistBins = 64;

__global__ void block_dist_hist_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *col,
                                       unsigned long long *hist) {
  __shared__ unsigned int h[kHistBins + 1];
  for (int i = threadIdx.x; i <= kHistBins; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rb = r / kRB;
    for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      int64_t d = static_cast<int64_t>(col[e] / kRB) - rb;
      if (d < 0) d = -d;
      atomicAdd(&h[d < kHistBins ? d : kHistBins], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= kHistBins; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(h[i]));
}

int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// largest window radius: >= 8 blocks of drift slack between the fastest and
// slowest consumer warp
constexpr int kMaxWindow = (kSlots - 9) / 2;

// Development trace printer (AG_SLAB_TRACE with an -DAG_SLAB_TRACE_BUILD build).
void print_trace(long long *trace, const char *name, const GArgs &a, cudaStream_t st) {
  long long h[kTraceBlocks * 8];
  if (cudaStreamSynchronize(st) != cudaSuccess ||
      cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaFree(trace);
    return;
  }
  cudaFree(trace);
  const long long t0 = h[0] ? h[0] : h[3];
  std::fprintf(stderr, "%s trace feat=%d H=%d (us; far/topo: done-wait start..end | X last | "
                       "cons0 ready-wait start..end | cons0 leave | dense ivalid | last-cons leave)\n",
               name, a.feat, a.H);
  for (int i = 0; i < kTraceBlocks; ++i) {
    auto f = [&](int j) { return h[i * 8 + j] ? (h[i * 8 + j] - t0) / 1e3 : -1.0; };
    std::fprintf(stderr, "blk %2d far %7.2f..%7.2f | X %7.2f | c0 %7.2f..%7.2f leave %7.2f | dense %7.2f | "
                         "clast leave %7.2f\n", i, f(0), f(1), f(2), f(3), f(4), f(5), f(6), f(7));
  }
}

template <int VEC>
int launch_slab(GArgs a, int mode, int window, cudaStream_t st) {
  using G = SlabGeom<VEC>;
  const bool wt = a.weighted != 0;
  auto k = mode == kModeMax
               ? (wt ? slab_kernel<VEC, kModeMax, true> : slab_kernel<VEC, kModeMax, false>)
           : mode == kModeDense3Coo
               ? (wt ? slab_kernel<VEC, kModeDense3Coo, true> : slab_kernel<VEC, kModeDense3Coo, false>)
           : mode == kModeSum3Coo
               ? (wt ? slab_kernel<VEC, kModeSum3Coo, true> : slab_kernel<VEC, kModeSum3Coo, false>)
           : mode == kModeDense3
               ? (wt ? slab_kernel<VEC, kModeDense3, true> : slab_kernel<VEC, kModeDense3, false>)
           : mode == kModeSum3
               ? (wt ? slab_kernel<VEC, kModeSum3, true> : slab_kernel<VEC, kModeSum3, false>)
               : (wt ? slab_kernel<VEC, kModeAny, true> : slab_kernel<VEC, kModeAny, false>);
  a.H = window;
  a.dbg = env_int("AG_SLAB_DEBUG", 0);
  a.sleep = env_int("AG_SLAB_SLEEP", 1);
  a.csleep = static_cast<uint32_t>(env_int("AG_SLAB_CSLEEP", 0));
  a.nblocks = (a.rows + kRB - 1) / kRB;
  a.xblocks = (a.x_rows + kRB - 1) / kRB;
  a.ntiles = static_cast<int>((a.feat + G::T - 1) / G::T);
  const size_t smem = G::kSmem;
  {
    cudaFuncAttributes fa;
    AG_CUDA(cudaFuncGetAttributes(&fa, k));
    int dev = 0, optin = 0;
    AG_CUDA(cudaGetDevice(&dev));
    AG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (smem + fa.sharedSizeBytes > static_cast<size_t>(optin))
      return fail(AG_ERR_CUDA, "slab kernel needs %zu + %zu B of shared memory, the device allows %d",
                  smem, static_cast<size_t>(fa.sharedSizeBytes), optin);
  }
  AG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int sms = sm_count();
  // ~2 units (range x tile) per CTA, ranges of >= 4 blocks
  int64_t ranges = (2LL * sms + a.ntiles - 1) / a.ntiles;
  ranges = std::max<int64_t>(1, std::min<int64_t>(ranges, a.nblocks / 4));
  a.ranges = static_cast<int>(ranges);
  const int64_t units = ranges * a.ntiles;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(units, sms)));

  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  a.tma = 0;
  a.relu = (a.ep.flags & AG_EPI_RELU_MASK) ? 1 : 0;
  a.ldw = relu_words(a.feat);
  // 2-D fp32 tensor map over [rows, feat] with row stride feat, box 16 x T
  auto encode = [&](CUtensorMap *m, const float *base, int64_t rows) -> bool {
    TmaEncodeFn enc = tma_encode_fn();
    if (!enc || reinterpret_cast<uintptr_t>(base) % 16 != 0) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.feat), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.feat) * 4};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(G::T), static_cast<cuuint32_t>(kRB)};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  if (a.feat % 4 == 0 && env_int("AG_SLAB_NO_TMA", 0) == 0 && encode(&map, a.x, a.x_rows))
    a.tma = 1;
  const int threads = (mode == kModeDense3Coo ? kCooCons + 2 : 14) * 32 + 64;
  long long *trace = nullptr;
  if (std::getenv("AG_SLAB_TRACE")) {
    AG_CUDA(cudaMalloc(&trace, kTraceBlocks * 8 * sizeof(long long)));
    AG_CUDA(cudaMemset(trace, 0, kTraceBlocks * 8 * sizeof(long long)));
    a.trace = trace;
  }
  k<<<grid, threads, smem, st>>>(map, a);
  AG_LAUNCH_CHECK("slab_kernel");
  if (trace) print_trace(trace, "slab", a, st);
  return AG_OK;
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

// Slab layout, one thread per 16-row block (edges in the given order).  Each
// edge becomes a (code, weight bits) pair: a source within `window` blocks
// of the destination's block is an X-ring row, slot-major
// ((src / 16) % kSlots) * 16 + src % 16; a farther one is staged in the far
// ring -- the block's j-th distinct far source (j < kFarMax) is row
// kFarRow0 + (block % kFarSlots) * kFarMax + j, far_src[block * kFarMax + j]
// = src -- and past kFarMax distinct far sources the code is ~src (global
// memory).  rowinfo[r] = {start, intra-run end (mid[r], or start when there
// is no role split), end, flags}; kRowSlow marks rows the fast path cannot
// take (global sources or more than kWin pairs).
__global__ void slab_code_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *col,
                                 const float *val, const int32_t *mid, int32_t window, int2 *cv,
                                 int4 *rowinfo, int32_t *far_cnt, int32_t *far_src) {
  const int64_t nb = (rows + kRB - 1) / kRB;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    int32_t staged[kFarMax];
    int j = 0;
    const int64_t r1 = std::min<int64_t>(b * kRB + kRB, rows);
    for (int64_t r = b * kRB; r < r1; ++r) {
      const int32_t s = row_ptr[r], e = row_ptr[r + 1];
      int flags = e - s > kWin ? kRowSlow : 0;
      for (int32_t ed = s; ed < e; ++ed) {
        const int32_t c = col[ed];
        const int64_t sb = c / kRB;
        const int64_t d = sb - b;
        int32_t code;
        if (d >= -window && d <= window) {
          code = static_cast<int32_t>((sb % kSlots) * kRB + c % kRB);
        } else {
          int k = 0;
          while (k < j && staged[k] != c) ++k;
          if (k == j && j < kFarMax) staged[j++] = c;
          if (k < j) {
            code = static_cast<int32_t>(kFarRow0 + (b % kFarSlots) * kFarMax + k);
          } else {
            code = ~c;
            flags |= kRowSlow;
          }
        }
        cv[ed] = make_int2(code, __float_as_int(val ? val[ed] : 1.0f));
      }
      rowinfo[r] = make_int4(s, mid ? mid[r] : s, e, flags);
    }
    far_cnt[b] = j;
    for (int k = 0; k < j; ++k) far_src[b * kFarMax + k] = staged[k];
  }
}

// The intra run of each row of a 16-row block as a dense 16 x 16 matrix
// (row = destination within the block, column = source within it; the
// reference's to_dense_blocks layout, formats.py:118-140), one thread per block.
__global__ void dense_block_weights_kernel(int64_t rows, const int32_t *row_ptr,
                                           const int32_t *mid, const int32_t *col,
                                           const float *val, float *blk_w) {
  const int64_t nb = (rows + kRB - 1) / kRB;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    float *w = blk_w + b * kRB * kRB;
    for (int i = 0; i < kRB * kRB; ++i) w[i] = 0.0f;
    const int64_t r1 = std::min<int64_t>(b * kRB + kRB, rows);
    for (int64_t r = b * kRB; r < r1; ++r)
      for (int32_t e = row_ptr[r]; e < mid[r]; ++e)
        w[(r - b * kRB) * kRB + (col[e] - b * kRB)] = val ? val[e] : 1.0f;
  }
}

// Band records, pass 1: per 16-row block, its record size in 16-byte units
// (64-byte header + 8 bytes per inter pair, padded) and the largest count.
__global__ void band_size_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *mid,
                                 int32_t *sizes, unsigned int *max_pairs) {
  const int64_t nb = (rows + kRB - 1) / kRB;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r1 = std::min<int64_t>(b * kRB + kRB, rows);
    int64_t n = 0;
    for (int64_t r = b * kRB; r < r1; ++r) n += row_ptr[r + 1] - mid[r];
    sizes[b] = static_cast<int32_t>((kRecHdr + 8 * n + 15) / 16);
    atomicMax(max_pairs, static_cast<unsigned int>(std::min<int64_t>(n, 0x7fffffff)));
  }
}

// Band records, pass 2 (one thread per block): row words and the inter pairs
// [mid[r], row_ptr[r+1]) of the role-ordered CSR as (code, weight bits), each
// row's FAR pairs first: a source within `window` blocks of the destination's
// block is a band-ring row, code ((src / 16) % kBandSlots) * 16 + src % 16;
// any other source is read from global memory by the consumer, code ~src.
// Row word i = end offset of row i's pairs | nfar << 20 (its leading far
// pairs; more than 255: kRowGlobal, the general path) | kBlkUnstaged when the
// block has more than kBandCap pairs.  far_cnt / far_src list up to kFarMax
// distinct far sources per block (the producer prefetches them into L2).
__global__ void band_record_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *col,
                                   const float *val, const int32_t *mid, int32_t window,
                                   const int32_t *rec_off, int4 *rec, int32_t *far_cnt,
                                   int32_t *far_src) {
  const int64_t nb = (rows + kRB - 1) / kRB;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t *hdr = reinterpret_cast<uint32_t *>(rec + rec_off[b]);
    int2 *pr = reinterpret_cast<int2 *>(hdr + kRecHdr / 4);
    const int64_t r1 = std::min<int64_t>(b * kRB + kRB, rows);
    int64_t n = 0;
    for (int64_t r = b * kRB; r < r1; ++r) n += row_ptr[r + 1] - mid[r];
    const uint32_t unstaged = n > kBandCap ? kBlkUnstaged : 0u;
    int32_t staged[kFarMax];
    int j = 0;
    uint32_t pos = 0;
    auto near = [&](int32_t c) {
      const int64_t d = static_cast<int64_t>(c / kRB) - b;
      return d >= -window && d <= window;
    };
    for (int i = 0; i < kRB; ++i) {
      const int64_t r = b * kRB + i;
      uint32_t nfar = 0;
      if (r < rows) {
        for (int pass = 0; pass < 2; ++pass)  // far pairs, then ring pairs
          for (int32_t ed = mid[r]; ed < row_ptr[r + 1]; ++ed) {
            const int32_t c = col[ed];
            const bool nr = near(c);
            if (nr != (pass == 1)) continue;
            int32_t code;
            if (nr) {
              code = static_cast<int32_t>(((c / kRB) % kBandSlots) * kRB + c % kRB);
            } else {
              code = ~c;
              ++nfar;
              int k = 0;
              while (k < j && staged[k] != c) ++k;
              if (k == j && j < kFarMax) staged[j++] = c;
            }
            pr[pos++] = make_int2(code, __float_as_int(val ? val[ed] : 1.0f));
          }
      }
      hdr[i] = pos | (nfar > 255 ? kRowGlobal : (nfar << 20)) | unstaged;
    }
    if (pos & 1u) pr[pos] = make_int2(0, 0);  // the 16-byte pad
    far_cnt[b] = j;
    for (int k = 0; k < j; ++k) far_src[b * kFarMax + k] = staged[k];
  }
}

int launch_band(GArgs a, int window, cudaStream_t st) {
  using G = BandGeom;
  a.H = window;
  a.dbg = env_int("AG_SLAB_DEBUG", 0);
  a.sleep = env_int("AG_SLAB_SLEEP", 1);
  a.csleep = static_cast<uint32_t>(env_int("AG_SLAB_CSLEEP", 0));
  a.nblocks = (a.rows + kRB - 1) / kRB;
  a.xblocks = (a.x_rows + kRB - 1) / kRB;
  a.ntiles = static_cast<int>((a.feat + G::T - 1) / G::T);
  a.relu = (a.ep.flags & AG_EPI_RELU_MASK) ? 1 : 0;
  a.ldw = relu_words(a.feat);
  const size_t smem = G::kSmem;
  auto k = band_kernel;
  {
    cudaFuncAttributes fa;
    AG_CUDA(cudaFuncGetAttributes(&fa, k));
    int dev = 0, optin = 0;
    AG_CUDA(cudaGetDevice(&dev));
    AG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (smem + fa.sharedSizeBytes > static_cast<size_t>(optin))
      return fail(AG_ERR_CUDA, "band kernel needs %zu + %zu B of shared memory, the device allows %d",
                  smem, static_cast<size_t>(fa.sharedSizeBytes), optin);
  }
  AG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  const int sms = sm_count();
  int64_t ranges = (2LL * sms + a.ntiles - 1) / a.ntiles;
  ranges = std::max<int64_t>(1, std::min<int64_t>(ranges, a.nblocks / 4));
  a.ranges = static_cast<int>(ranges);
  const int64_t units = ranges * a.ntiles;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(units, sms)));
  CUtensorMap map;
  std::memset(&map, 0, sizeof(map));
  TmaEncodeFn enc = tma_encode_fn();
  if (!enc) return fail(AG_ERR_CUDA, "band kernel: no cuTensorMapEncodeTiled");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.feat), static_cast<cuuint64_t>(a.x_rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.feat) * 4};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(G::T), static_cast<cuuint32_t>(kRB)};
  cuuint32_t es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(a.x), dims, strides, box,
          es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(AG_ERR_CUDA, "band kernel: tensor map encode failed");
  a.tma = 1;
  long long *trace = nullptr;
  if (std::getenv("AG_SLAB_TRACE")) {
    AG_CUDA(cudaMalloc(&trace, kTraceBlocks * 8 * sizeof(long long)));
    AG_CUDA(cudaMemset(trace, 0, kTraceBlocks * 8 * sizeof(long long)));
    a.trace = trace;
  }
  k<<<grid, (kBandCons + kBandDense + 2) * 32, smem, st>>>(map, a);
  AG_LAUNCH_CHECK("band_kernel");
  if (trace) print_trace(trace, "band", a, st);
  return AG_OK;
}

}  // namespace
}  // namespace ag

using namespace ag;

extern "C" int ag_slab_far_capacity(void) { return kFarMax; }

extern "C" int ag_slab_dense_blocks(int64_t num_rows, const int32_t *row_ptr,
                                    const int32_t *role_mid, const int32_t *role_col,
                                    const float *role_val, float *blk_w, void *stream) {
  if (num_rows < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (role_mid == nullptr) return fail(AG_ERR_VALUE, "role_mid (block size 16) is required");
  if (num_rows == 0) return AG_OK;
  const int64_t nb = (num_rows + kRB - 1) / kRB;
  dense_block_weights_kernel<<<grid_for(nb, 128), 128, 0, as_stream(stream)>>>(
      num_rows, row_ptr, role_mid, role_col, role_val, blk_w);
  AG_LAUNCH_CHECK("dense_block_weights_kernel");
  return AG_OK;
}

extern "C" int ag_slab_codes(int64_t num_rows, const int32_t *row_ptr, const int32_t *col_idx,
                             const float *val, const int32_t *role_mid, int32_t window,
                             int32_t *cv, int32_t *rowinfo, int32_t *far_cnt, int32_t *far_src,
                             void *stream) {
  if (num_rows < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (window < 0 || window > kMaxWindow)
    return fail(AG_ERR_VALUE, "window must be in [0, %d]", kMaxWindow);
  if (num_rows > 2147483647LL) return fail(AG_ERR_VALUE, "too many rows for int32 CSR");
  if (num_rows == 0) return AG_OK;
  const int64_t nb = (num_rows + kRB - 1) / kRB;
  slab_code_kernel<<<grid_for(nb, 128), 128, 0, as_stream(stream)>>>(
      num_rows, row_ptr, col_idx, val, role_mid, window, reinterpret_cast<int2 *>(cv),
      reinterpret_cast<int4 *>(rowinfo), far_cnt, far_src);
  AG_LAUNCH_CHECK("slab_code_kernel");
  return AG_OK;
}

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

extern "C" int ag_slab_window(int64_t num_rows, const int32_t *row_ptr, const int32_t *col_idx,
                              double coverage, int32_t *window, void *stream) {
  if (num_rows < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (window == nullptr) return fail(AG_ERR_VALUE, "window output is NULL");
  *window = 0;
  if (num_rows == 0) return AG_OK;
  cudaStream_t st = as_stream(stream);
  Scratch hist;
  AG_CUDA(hist.alloc((kHistBins + 1) * sizeof(unsigned long long), st));
  AG_CUDA(cudaMemsetAsync(hist.ptr, 0, (kHistBins + 1) * sizeof(unsigned long long), st));
  block_dist_hist_kernel<<<grid_for(num_rows, 256, 148LL * 8), 256, 0, st>>>(
      num_rows, row_ptr, col_idx, hist.as<unsigned long long>());
  AG_LAUNCH_CHECK("block_dist_hist_kernel");
  unsigned long long h[kHistBins + 1];
  AG_CUDA(cudaMemcpyAsync(h, hist.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  // smallest radius whose ring covers `coverage` of what the largest
  // supported radius would cover
  const int hmax = kMaxWindow;
  unsigned long long total = 0;
  for (int d = 0; d <= hmax && d < kHistBins; ++d) total += h[d];
  unsigned long long acc = 0;
  int H = 0;
  for (int d = 0; d <= hmax && d < kHistBins; ++d) {
    acc += h[d];
    H = d;
    if (static_cast<double>(acc) >= coverage * static_cast<double>(total)) break;
  }
  *window = H;
  return AG_OK;
}

extern "C" int ag_fused_spmm(int64_t num_rows, int64_t feat, int32_t role_mask,
                             const int32_t *row_ptr, const int32_t *role_mid,
                             const int32_t *cv, const int32_t *rowinfo,
                             const int32_t *far_cnt, const int32_t *far_src, int32_t weighted,
                             const float *blk_w, int64_t num_edges,
                             const float *x, float *y, int32_t op, int32_t epi_flags,
                             const uint8_t *other_touched, const int64_t *deg, float gin_scale,
                             const uint32_t *relu_bits, uint32_t *relu_out, int64_t x_rows,
                             int32_t window, void *stream) {
  if (num_rows < 0 || feat < 0 || num_edges < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (op < AG_OP_SUM || op > AG_OP_MAX) return fail(AG_ERR_KERNEL, "unknown op %d", op);
  if (role_mask < 1 || role_mask > 3) return fail(AG_ERR_VALUE, "role_mask must be 1, 2 or 3");
  if (role_mid == nullptr && role_mask == 3)
    return fail(AG_ERR_VALUE, "role_mask 3 needs the role-ordered CSR (role_mid)");
  if (op == AG_OP_MEAN && deg == nullptr && (role_mask == 3 || (epi_flags & AG_EPI_COMBINE)))
    return fail(AG_ERR_KERNEL, "mean combine requires the full-graph degree vector");
  if ((epi_flags & AG_EPI_RELU_MASK) && relu_bits == nullptr)
    return fail(AG_ERR_VALUE, "AG_EPI_RELU_MASK needs relu_bits");
  if (relu_out != nullptr && !(epi_flags & AG_EPI_RELU))
    return fail(AG_ERR_VALUE, "relu_out is written with AG_EPI_RELU only");
  if (window < 0 || window > kMaxWindow)
    return fail(AG_ERR_VALUE, "window must be in [0, %d]", kMaxWindow);
  if (x_rows < num_rows) return fail(AG_ERR_VALUE, "x_rows must be >= num_rows");
  if (num_rows == 0 || feat == 0) return AG_OK;
  if (x_rows > 2147483647LL || num_edges > 2147483647LL)
    return fail(AG_ERR_VALUE, "too many rows or edges for int32 CSR");
  cudaStream_t st = as_stream(stream);
  GArgs a{};
  a.rows = num_rows;
  a.x_rows = x_rows;
  a.feat = static_cast<int>(feat);
  a.mask = role_mask;
  a.row_ptr = row_ptr;
  a.mid = role_mid;
  a.cv = reinterpret_cast<const int2 *>(cv);
  a.rowinfo = reinterpret_cast<const int4 *>(rowinfo);
  a.far_cnt = far_cnt;
  a.far_src = far_src;
  if (!cv || !rowinfo || !far_cnt || !far_src)
    return fail(AG_ERR_VALUE, "cv / rowinfo / far_cnt / far_src (ag_slab_codes) are required");
  if ((reinterpret_cast<uintptr_t>(cv) & 7) || (reinterpret_cast<uintptr_t>(rowinfo) & 15))
    return fail(AG_ERR_VALUE, "cv must be 8-byte and rowinfo 16-byte aligned");
  a.weighted = weighted != 0;
  a.has_mid = role_mid != nullptr;
  a.blk_w = blk_w;
  constexpr int32_t kSum3Flags = AG_EPI_GIN | AG_EPI_RELU_MASK | AG_EPI_RELU | AG_EPI_INTER_COO;
  if (blk_w != nullptr &&
      (role_mask != 3 || op != AG_OP_SUM || role_mid == nullptr || (epi_flags & ~kSum3Flags) != 0))
    return fail(AG_ERR_VALUE, "dense intra blocks need role_mask 3, op sum and role_mid");
  const bool coo = (epi_flags & AG_EPI_INTER_COO) != 0;
  if (coo && (role_mask != 3 || op != AG_OP_SUM || role_mid == nullptr ||
              (epi_flags & ~kSum3Flags) != 0))
    return fail(AG_ERR_VALUE, "AG_EPI_INTER_COO needs role_mask 3, op sum and role_mid");
  a.x = x;
  a.y = y;
  a.ep = Epi{op, epi_flags, other_touched, deg, x, feat, gin_scale, relu_bits};
  a.relu_out = relu_out;
  a.cost_total = num_edges + kRowCost * num_rows;
  a.one = 1.0f;
  const bool is_max = op == AG_OP_MAX;
  const bool v2 = feat % 2 == 0 && feat > 32 && (reinterpret_cast<uintptr_t>(x) % 8) == 0 &&
                  (reinterpret_cast<uintptr_t>(y) % 8) == 0 &&
                  env_int("AG_SLAB_VEC", 2) == 2;
  const int mode = blk_w != nullptr ? (coo ? kModeDense3Coo : kModeDense3)
                 : coo ? kModeSum3Coo
                 : is_max ? kModeMax
                   : (role_mask == 3 && op == AG_OP_SUM && (epi_flags & ~kSum3Flags) == 0)
                       ? kModeSum3
                       : kModeAny;
  if (v2) return launch_slab<2>(a, mode, window, st);
  return launch_slab<1>(a, mode, window, st);
}

extern "C" int ag_band_max_window(void) { return kBandMaxWindow; }
extern "C" int ag_band_capacity(void) { return kBandCap; }

extern "C" int ag_band_sizes(int64_t num_rows, const int32_t *row_ptr, const int32_t *role_mid,
                             int32_t *sizes, int64_t *max_pairs_host, void *stream) {
  if (num_rows < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (role_mid == nullptr || sizes == nullptr || max_pairs_host == nullptr)
    return fail(AG_ERR_VALUE, "role_mid, sizes and max_pairs are required");
  *max_pairs_host = 0;
  if (num_rows == 0) return AG_OK;
  if (num_rows > 2147483647LL) return fail(AG_ERR_VALUE, "too many rows for int32 CSR");
  cudaStream_t st = as_stream(stream);
  const int64_t nb = (num_rows + kRB - 1) / kRB;
  Scratch mx;
  AG_CUDA(mx.alloc(sizeof(unsigned int), st));
  AG_CUDA(cudaMemsetAsync(mx.ptr, 0, sizeof(unsigned int), st));
  band_size_kernel<<<grid_for(nb, 128), 128, 0, st>>>(num_rows, row_ptr, role_mid, sizes,
                                                      mx.as<unsigned int>());
  AG_LAUNCH_CHECK("band_size_kernel");
  unsigned int h = 0;
  AG_CUDA(cudaMemcpyAsync(&h, mx.ptr, sizeof(h), cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  *max_pairs_host = h;
  return AG_OK;
}

extern "C" int ag_band_records(int64_t num_rows, const int32_t *row_ptr, const int32_t *role_col,
                               const float *role_val, const int32_t *role_mid, int32_t window,
                               const int32_t *rec_off, int32_t *rec, int32_t *far_cnt,
                               int32_t *far_src, void *stream) {
  if (num_rows < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (window < 0 || window > kBandMaxWindow)
    return fail(AG_ERR_VALUE, "window must be in [0, %d]", kBandMaxWindow);
  if (role_mid == nullptr || rec_off == nullptr || rec == nullptr)
    return fail(AG_ERR_VALUE, "role_mid, rec_off and rec are required");
  if (reinterpret_cast<uintptr_t>(rec) & 15) return fail(AG_ERR_VALUE, "rec must be 16-byte aligned");
  if (num_rows == 0) return AG_OK;
  const int64_t nb = (num_rows + kRB - 1) / kRB;
  band_record_kernel<<<grid_for(nb, 128), 128, 0, as_stream(stream)>>>(
      num_rows, row_ptr, role_col, role_val, role_mid, window, rec_off,
      reinterpret_cast<int4 *>(rec), far_cnt, far_src);
  AG_LAUNCH_CHECK("band_record_kernel");
  return AG_OK;
}

extern "C" int ag_band_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                            const int32_t *rec, const int32_t *rec_off, const int32_t *far_cnt,
                            const int32_t *far_src, const float *blk_w, int64_t num_edges,
                            const float *x, float *y, int32_t epi_flags, float gin_scale,
                            const uint32_t *relu_bits, uint32_t *relu_out, int64_t x_rows,
                            int32_t window, void *stream) {
  if (num_rows < 0 || feat < 0 || num_edges < 0) return fail(AG_ERR_VALUE, "negative sizes");
  constexpr int32_t kFlags = AG_EPI_GIN | AG_EPI_RELU_MASK | AG_EPI_RELU | AG_EPI_INTER_COO;
  if (epi_flags & ~kFlags) return fail(AG_ERR_VALUE, "ag_band_spmm takes GIN / RELU / RELU_MASK flags");
  if ((epi_flags & AG_EPI_RELU_MASK) && relu_bits == nullptr)
    return fail(AG_ERR_VALUE, "AG_EPI_RELU_MASK needs relu_bits");
  if (relu_out != nullptr && !(epi_flags & AG_EPI_RELU))
    return fail(AG_ERR_VALUE, "relu_out is written with AG_EPI_RELU only");
  if (window < 0 || window > kBandMaxWindow)
    return fail(AG_ERR_VALUE, "window must be in [0, %d]", kBandMaxWindow);
  if (x_rows < num_rows) return fail(AG_ERR_VALUE, "x_rows must be >= num_rows");
  if (!row_ptr || !rec || !rec_off || !far_cnt || !far_src || !blk_w)
    return fail(AG_ERR_VALUE, "row_ptr / band records / far lists / blk_w are required");
  if (num_rows == 0 || feat == 0) return AG_OK;
  if (feat % 4 != 0 || feat <= 32 || (reinterpret_cast<uintptr_t>(x) & 15) ||
      (reinterpret_cast<uintptr_t>(y) & 7) || (reinterpret_cast<uintptr_t>(rec) & 15) ||
      (relu_bits && (reinterpret_cast<uintptr_t>(relu_bits) & 15)))
    return fail(AG_ERR_VALUE, "ag_band_spmm needs feat % 4 == 0, feat > 32, 16-byte aligned x / rec / relu_bits");
  if (x_rows > 2147483647LL || num_edges > 2147483647LL)
    return fail(AG_ERR_VALUE, "too many rows or edges for int32 CSR");
  GArgs a{};
  a.rows = num_rows;
  a.x_rows = x_rows;
  a.feat = static_cast<int>(feat);
  a.mask = 3;
  a.row_ptr = row_ptr;
  a.far_cnt = far_cnt;
  a.far_src = far_src;
  a.weighted = 1;
  a.has_mid = 1;
  a.blk_w = blk_w;
  a.brec = reinterpret_cast<const int4 *>(rec);
  a.brec_off = rec_off;
  a.x = x;
  a.y = y;
  a.ep = Epi{AG_OP_SUM, epi_flags, nullptr, nullptr, x, feat, gin_scale, relu_bits};
  a.relu_out = relu_out;
  a.cost_total = num_edges + kRowCost * num_rows;
  a.one = 1.0f;
  return launch_band(a, window, as_stream(stream));
}
