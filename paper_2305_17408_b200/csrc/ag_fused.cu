// Fused single-pass decomposed aggregation (the hot path of every GCN/GIN layer).
//
// One launch computes, for every destination row r of the FULL reordered CSR,
//   I = intra-role value over the row's block-local edges (cols in [cB, cB+B))
//   O = inter-role value over the remaining edges (prefix ++ suffix of the row)
//   y[r] = combine(I, O)  [+ (1+eps) x[r] for GIN]
// which is bit-for-bit what the reference computes with two separate CSR
// kernels and combine() (kernels.py:87-189, :253-276): both role sums follow
// np.add.reduceat's order (first term + numpy pairwise, see ag_spmm.cu), the
// intra edges of a sorted row are one contiguous run, and the inter role is
// the ordered concatenation of what is left.  Compared with two launches it
// saves one full write + read of the V x F partial (2VF*4 bytes): HBM traffic
// is topology once, X once (modulo L2 misses), Y once.
//
// Layout: the "stage-aligned CSR" (built once per topology, ag_stage_layout_*)
// lists every row's edges in role order (intra run, then inter = prefix ++
// suffix) cut into 9-slot stages aligned with numpy's pairwise structure:
// slot 0 holds a role's first term c0 (only in the role's first stage), slots
// 1..8 hold one 8-wide accumulator group, empty slots hold col = -1.  The
// reduction is then branch-free per stage: the 8 accumulators start at -0.0
// (x + -0.0 == x bitwise) and take one group per stage, leaves of the >128
// recursion start on stage boundaries (split points are multiples of 8), and
// the n%8 tail is the role's last stage.
//
// Data movement (sm_100a).  Warps pull chunks of 16 consecutive rows from a
// global atomic counter, so the whole grid sweeps the row space as one tight
// wavefront and the reorder's locality keeps gathered X rows L2-resident.
// Each warp runs a producer/consumer pipeline on itself: the producer reads a
// stage's 9 (col, val) slots with one coalesced load and issues one
// cp.async.bulk (TMA) per source row into a shared-memory ring of stages,
// completing on the stage's mbarrier; the consumer reduces stage by stage.
// Products and sums use packed FMUL2 / FFMA2(acc, 1.0, c) (exact: acc*1 is
// exact, so the only rounding is that of the sum) -- half the FP issue slots.
// Feature widths the bulk path cannot serve (F % 4 != 0, F > 256) take the
// register-gather long-row kernel below.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "ag_common.cuh"
#include "ag_vec.cuh"

namespace ag {
namespace {
using namespace vec;

constexpr int kChunk = 16;   // rows per chunk (consecutive)
constexpr int kSlots = 9;    // slot 0: first term, slots 1..8: one pairwise group
constexpr int kLeafN = 128;  // numpy PW_BLOCKSIZE
constexpr int kDepth = 40;

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t addr = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// packed fp32x2: p = fl(a * s) per lane pair (FMUL2)
__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(uint64_t r, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t pmul(uint64_t a, uint64_t s) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(s));
  return d;
}
// acc + c as FFMA2(acc, 1.0, c) with a run-time 1.0 (one): exact fl(acc + c),
// and not contractible with the preceding FMUL2
__device__ __forceinline__ uint64_t padd(uint64_t acc, uint64_t one, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(acc), "l"(one), "l"(c));
  return d;
}

// ------------------------------------------------------------ arguments ----
struct FusedArgs {
  int64_t rows;
  int feat;
  int block;      // B (0: no role split, the whole row is one role)
  int mask;       // 1 intra only, 2 inter only, 3 both (combine)
  const int32_t *row_ptr;  // CSR (register-gather fallback)
  const int32_t *col;
  const float *val;        // nullptr: implicit 1.0
  const float *x;
  float *y;
  Epi ep;
  // stage-aligned layout
  const int32_t *stage_ptr;  // [rows + 1] first stage of each row
  const int2 *counts;        // [rows] items of the (intra, inter) role, mask applied
  const int32_t *scol;       // [stages * 9]; -1 = empty slot
  const float *sval;         // [stages * 9]
  unsigned int *chunk_ctr;   // dynamic chunk scheduler (zeroed per launch)
  int warps;                 // warps per CTA
  int warp_bytes;            // dynamic smem per warp
  int stages;                // ring depth (power of two)
  float one;                 // 1.0f at run time (keeps FFMA2(acc, 1, c) opaque)
};

__device__ __forceinline__ int role_stages(int n) {
  return n <= 0 ? 0 : (n == 1 ? 1 : (n - 1 + 7) >> 3);
}

__device__ __forceinline__ void lds_v2u64(uint32_t addr, uint64_t &a, uint64_t &b) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}

template <int FV>
struct Warp {
  static constexpr int W = 4 * FV;
  static constexpr int P = W / 2;  // fp32x2 pairs per lane
  const FusedArgs *a;
  uint64_t *bar;
  float *vals;        // [stages][kSlots]
  int *fifo;          // [4] chunk ids, producer -> consumer
  uint32_t ring_u32;  // shared address of the ring
  uint32_t vals_u32;
  uint32_t rowbytes;
  int lane;
  int smask;
  int64_t nchunks;
  bool act[FV];       // this lane holds feature columns in half h
  // producer
  int64_t pt;         // stages issued
  int64_t ps, pe;     // next stage to issue / end of the producer's chunk
  int pcount;         // chunk ids pushed
  bool pdone;
  // consumer
  int64_t ct;         // stages consumed
  int ccount;         // chunk ids popped
  uint32_t phase;
  int cur;
  uint32_t cur_base;  // ring address of the acquired stage's slot 0, this lane
  uint64_t one2;

  // pull the next chunk from the scheduler into the FIFO
  __device__ __forceinline__ bool prod_next_chunk() {
    if (pdone || pcount - ccount >= 4) return false;
    int c = 0;
    if (lane == 0) c = static_cast<int>(atomicAdd(a->chunk_ctr, 1u));
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= nchunks) {
      c = -1;
      pdone = true;
    }
    if (lane == 0) fifo[pcount & 3] = c;
    __syncwarp();
    ++pcount;
    if (c < 0) return false;
    const int64_t r0 = static_cast<int64_t>(c) * kChunk;
    const int64_t r1 = r0 + kChunk < a->rows ? r0 + kChunk : a->rows;
    ps = a->stage_ptr[r0];
    pe = a->stage_ptr[r1];
    return true;
  }

  __device__ __forceinline__ bool prod_seek() {
    while (ps >= pe)
      if (!prod_next_chunk()) return false;
    return true;
  }

  __device__ __forceinline__ void issue() {
    const int slot = static_cast<int>(pt) & smask;
    int32_t c = -1;
    float v = 0.0f;
    if (lane < kSlots) {
      c = __ldg(a->scol + ps * kSlots + lane);
      v = __ldg(a->sval + ps * kSlots + lane);
      vals[slot * kSlots + lane] = v;
    }
    const bool valid = c >= 0;
    const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, valid));
    if (lane == 0) mbar_expect_tx(&bar[slot], rowbytes * cnt);
    __syncwarp();
    if (valid) {
      fence_proxy_async();
      bulk_g2s(reinterpret_cast<char *>(ring_ptr()) + (slot * kSlots + lane) * rowbytes,
               a->x + static_cast<int64_t>(c) * a->feat, rowbytes, &bar[slot]);
    }
    ++pt;
    ++ps;
  }

  float *ring_base;
  __device__ __forceinline__ float *ring_ptr() const { return ring_base; }

  __device__ __forceinline__ void fill() {
    while (pt - ct < smask + 1 && prod_seek()) issue();
  }

  // consumer side ---------------------------------------------------------
  __device__ __forceinline__ int next_chunk() {
    if (ccount == pcount) prod_next_chunk();
    const int c = fifo[ccount & 3];
    ++ccount;
    fill();
    return c;
  }

  __device__ __forceinline__ void acquire() {
    cur = static_cast<int>(ct) & smask;
    mbar_wait(&bar[cur], (phase >> cur) & 1u);
    phase ^= 1u << cur;
    cur_base = ring_u32 + cur * kSlots * rowbytes + lane * 16;
  }

  __device__ __forceinline__ void release() {
    ++ct;
    __syncwarp();
    fill();
  }

  // packed contribution fl(val * x) of slot j of the acquired stage
  __device__ __forceinline__ void contrib(int j, uint64_t (&c)[P]) const {
    const float v = vals[cur * kSlots + j];
    const uint64_t v2 = pk(v, v);
    const uint32_t addr = cur_base + j * rowbytes;
#pragma unroll
    for (int h = 0; h < FV; ++h) {
      uint64_t lo = 0, hi = 0;
      if (act[h]) lds_v2u64(addr + h * 512, lo, hi);
      c[2 * h] = pmul(lo, v2);
      c[2 * h + 1] = pmul(hi, v2);
    }
  }

  __device__ __forceinline__ Vf<W> raw(int j) const {
    const uint32_t addr = cur_base + j * rowbytes;
    Vf<W> v;
#pragma unroll
    for (int h = 0; h < FV; ++h) {
      uint64_t lo = 0, hi = 0;
      if (act[h]) lds_v2u64(addr + h * 512, lo, hi);
      upk(lo, v.v[4 * h], v.v[4 * h + 1]);
      upk(hi, v.v[4 * h + 2], v.v[4 * h + 3]);
    }
    return v;
  }

  // numpy pairwise leaf over the next nl items (stage aligned)
  __device__ __forceinline__ void leaf(int nl, bool first_in_cur, uint64_t (&res)[P]) {
    const int q = nl >> 3, tail = nl & 7;
    const uint64_t nz = pk(-0.0f, -0.0f);
#pragma unroll
    for (int i = 0; i < P; ++i) res[i] = nz;
    if (q > 0) {
      uint64_t r[8][P];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) r[j][i] = nz;
#pragma unroll 1
      for (int g = 0; g < q; ++g) {
        if (g > 0 || !first_in_cur) { release(); acquire(); }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint64_t c[P];
          contrib(1 + j, c);
#pragma unroll
          for (int i = 0; i < P; ++i) r[j][i] = padd(r[j][i], one2, c[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < P; ++i)
        res[i] = padd(padd(padd(r[0][i], one2, r[1][i]), one2, padd(r[2][i], one2, r[3][i])),
                      one2,
                      padd(padd(r[4][i], one2, r[5][i]), one2, padd(r[6][i], one2, r[7][i])));
    }
    if (tail > 0) {
      if (q > 0 || !first_in_cur) { release(); acquire(); }
#pragma unroll 1
      for (int j = 0; j < tail; ++j) {
        uint64_t c[P];
        contrib(1 + j, c);
#pragma unroll
        for (int i = 0; i < P; ++i) res[i] = padd(res[i], one2, c[i]);
      }
    }
  }

  // P over the next m items: post-order walk of numpy's recursion (a single
  // leaf when m <= 128); the first leaf shares the role's first stage with c0
  __device__ __forceinline__ void pairwise(int m, uint64_t (&out)[P]) {
    int st_n[kDepth];
    int st_stage[kDepth];
    uint64_t st_left[kDepth][P];
    int sp = 0;
    bool first = true;
    st_n[0] = m;
    st_stage[0] = 0;
#pragma unroll 1
    while (sp >= 0) {
      const int cn = st_n[sp];
      if (cn <= kLeafN) {
        leaf(cn, first, out);
        first = false;
        --sp;
        continue;
      }
      int n2 = cn / 2;
      n2 -= n2 & 7;
      if (st_stage[sp] == 0) {
        st_stage[sp] = 1;
        st_n[sp + 1] = n2;
        st_stage[sp + 1] = 0;
        ++sp;
      } else if (st_stage[sp] == 1) {
#pragma unroll
        for (int i = 0; i < P; ++i) st_left[sp][i] = out[i];
        st_stage[sp] = 2;
        st_n[sp + 1] = cn - n2;
        st_stage[sp + 1] = 0;
        ++sp;
      } else {
#pragma unroll
        for (int i = 0; i < P; ++i) out[i] = padd(st_left[sp][i], one2, out[i]);
        --sp;
      }
    }
  }

  template <bool IS_MAX>
  __device__ __forceinline__ Vf<W> role(int n) {
    Vf<W> out = splat<W>(0.0f);
    if (n <= 0) return out;
    acquire();
    if constexpr (IS_MAX) {
      out = raw(0);
      int left = n - 1, k = 0;
#pragma unroll 1
      while (left > 0) {
        if (k > 0) { release(); acquire(); }
        const int cnt = left < 8 ? left : 8;
#pragma unroll 1
        for (int j = 0; j < cnt; ++j) out = vmax<W>(out, raw(1 + j));
        left -= cnt;
        ++k;
      }
      release();
      return out;
    } else {
      uint64_t c0[P];
      contrib(0, c0);
      if (n > 1) {
        uint64_t p[P];
        pairwise(n - 1, p);
#pragma unroll
        for (int i = 0; i < P; ++i) c0[i] = padd(c0[i], one2, p[i]);
      }
      release();
#pragma unroll
      for (int i = 0; i < P; ++i) upk(c0[i], out.v[2 * i], out.v[2 * i + 1]);
      return out;
    }
  }
};

template <int W>
__device__ __forceinline__ Vf<W> combine2(int op, const Vf<W> &I, bool ti, const Vf<W> &O,
                                          bool to, int64_t deg) {
  if (op == AG_OP_SUM) return vadd<W>(I, O);
  if (op == AG_OP_MEAN) {
    const float d = static_cast<float>(deg < 1 ? 1 : deg);
    Vf<W> s = vadd<W>(I, O), r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = __fdiv_rn(s.v[i], d);
    return r;
  }
  if (ti && to) return vmax<W>(I, O);
  if (ti) return I;
  if (to) return O;
  return splat<W>(0.0f);
}

template <int FV>
__device__ __forceinline__ Vf<4 * FV> load_row(const float *base, int feat, int lane) {
  Vf<4 * FV> v = splat<4 * FV>(0.0f);
#pragma unroll
  for (int h = 0; h < FV; ++h) {
    const int f = h * 128 + lane * 4;
    if (f < feat) {
      const float4 t = *reinterpret_cast<const float4 *>(base + f);
      v.v[h * 4 + 0] = t.x; v.v[h * 4 + 1] = t.y; v.v[h * 4 + 2] = t.z; v.v[h * 4 + 3] = t.w;
    }
  }
  return v;
}

template <int FV, bool IS_MAX>
__global__ void __launch_bounds__(FV == 1 ? 512 : 384) fused_kernel(FusedArgs a) {
  constexpr int W = 4 * FV;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned char *base = smem_raw + static_cast<size_t>(warp) * a.warp_bytes;
  Warp<FV> w;
  w.a = &a;
  w.bar = reinterpret_cast<uint64_t *>(base);
  w.vals = reinterpret_cast<float *>(base + 8 * a.stages);
  w.fifo = reinterpret_cast<int *>(base + 8 * a.stages + 4 * kSlots * a.stages);
  const int hdr = (8 * a.stages + 4 * kSlots * a.stages + 16 + 127) / 128 * 128;
  w.ring_base = reinterpret_cast<float *>(base + hdr);
  w.ring_u32 = smem_u32(w.ring_base);
  w.vals_u32 = smem_u32(w.vals);
  w.rowbytes = static_cast<uint32_t>(a.feat) * 4u;
  w.lane = lane;
  w.smask = a.stages - 1;
  w.nchunks = (a.rows + kChunk - 1) / kChunk;
#pragma unroll
  for (int h = 0; h < FV; ++h) w.act[h] = h * 128 + lane * 4 < a.feat;
  w.pt = 0; w.ps = 0; w.pe = 0; w.pcount = 0; w.pdone = false;
  w.ct = 0; w.ccount = 0; w.phase = 0; w.cur = 0; w.cur_base = 0;
  w.one2 = pk(a.one, a.one);
  if (lane == 0) {
    for (int i = 0; i < a.stages; ++i) mbar_init(&w.bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int64_t ld = a.feat;
  const bool need_y = a.mask != 3 && (a.ep.flags & AG_EPI_COMBINE) &&
                      !(a.ep.flags & AG_EPI_EMPTY_OTHER);
  const bool need_x = (a.ep.flags & AG_EPI_GIN) != 0;
  const bool need_ot = need_y && a.ep.other_touched != nullptr;
  const bool need_deg = a.ep.op == AG_OP_MEAN && a.ep.deg != nullptr;
#pragma unroll 1
  for (;;) {
    const int c = w.next_chunk();
    if (c < 0) break;
    const int64_t r0 = static_cast<int64_t>(c) * kChunk;
    const int nr = static_cast<int>(a.rows - r0 < kChunk ? a.rows - r0 : kChunk);
    int2 cnt = make_int2(0, 0);
    long long dg = 1;
    int ot = 0;
    if (lane < nr) {
      cnt = a.counts[r0 + lane];
      if (need_deg) dg = a.ep.deg[r0 + lane];
      if (need_ot) ot = a.ep.other_touched[r0 + lane];
    }
#pragma unroll 1
    for (int l = 0; l < nr; ++l) {
      const int64_t r = r0 + l;
      const int ni = __shfl_sync(0xffffffffu, cnt.x, l);
      const int no = __shfl_sync(0xffffffffu, cnt.y, l);
      const long long d = __shfl_sync(0xffffffffu, dg, l);
      const bool other_t = __shfl_sync(0xffffffffu, ot, l) != 0;
      Vf<W> side_y = splat<W>(0.0f), side_x = splat<W>(0.0f);
      if (need_y) side_y = load_row<FV>(a.y + r * ld, a.feat, lane);
      if (need_x) side_x = load_row<FV>(a.x + r * ld, a.feat, lane);
      Vf<W> I = splat<W>(0.0f), O = splat<W>(0.0f);
#pragma unroll 1
      for (int role = 0; role < 2; ++role) {
        const Vf<W> v = w.template role<IS_MAX>(role == 0 ? ni : no);
        if (role == 0) I = v; else O = v;
      }
      Vf<W> out;
      if (a.mask == 3) {
        out = combine2<W>(a.ep.op, I, ni > 0, O, no > 0, d);
      } else {
        const Vf<W> v = (a.mask == 1) ? I : O;
        const bool t = (a.mask == 1) ? ni > 0 : no > 0;
        if (!(a.ep.flags & AG_EPI_COMBINE)) out = t ? v : splat<W>(0.0f);
        else out = combine2<W>(a.ep.op, v, t, side_y, other_t, d);
      }
      if (need_x) out = vadd<W>(vscale<W>(a.ep.gin_scale, side_x), out);
#pragma unroll
      for (int h = 0; h < FV; ++h) {
        const int f = h * 128 + lane * 4;
        if (f < a.feat)
          *reinterpret_cast<float4 *>(a.y + r * ld + f) = make_float4(
              out.v[h * 4 + 0], out.v[h * 4 + 1], out.v[h * 4 + 2], out.v[h * 4 + 3]);
      }
    }
  }
}

// ---------------------------------------------- stage-aligned layout build --
__device__ __forceinline__ void intra_run(const int32_t *col, int64_t s, int64_t e, int64_t r,
                                          int64_t B, int64_t &ia, int64_t &ib) {
  if (B <= 0) { ia = ib = 0; return; }
  const int64_t cb = (r / B) * B;
  int64_t lo = s, hi = e;
  while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (col[m] < cb) lo = m + 1; else hi = m; }
  ia = lo - s;
  hi = e;
  while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (col[m] < cb + B) lo = m + 1; else hi = m; }
  ib = lo - s;
}

__global__ void layout_count_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *col,
                                    int64_t B, int mask, int2 *counts, int32_t *nstages) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = row_ptr[r], e = row_ptr[r + 1];
    int64_t ia, ib;
    intra_run(col, s, e, r, B, ia, ib);
    const int n1 = static_cast<int>(ib - ia);
    const int ni = (mask & 1) ? n1 : 0;
    const int no = (mask & 2) ? static_cast<int>(e - s) - n1 : 0;
    counts[r] = make_int2(ni, no);
    nstages[r] = role_stages(ni) + role_stages(no);
  }
}

__global__ void layout_fill_kernel(int64_t rows, const int32_t *row_ptr, const int32_t *col,
                                   const float *val, int64_t B, const int32_t *stage_ptr,
                                   const int2 *counts, int32_t *scol, float *sval) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = row_ptr[r], e = row_ptr[r + 1];
    int64_t ia, ib;
    intra_run(col, s, e, r, B, ia, ib);
    int64_t t = stage_ptr[r];
    const int2 cn = counts[r];
    for (int role = 0; role < 2; ++role) {
      const int n = role == 0 ? cn.x : cn.y;
      const int ns = role_stages(n);
      for (int k = 0; k < ns; ++k, ++t) {
        for (int j = 0; j < kSlots; ++j) {
          const int item = (j == 0) ? (k == 0 ? 0 : -1) : 8 * k + j;
          int32_t c = -1;
          float v = 0.0f;
          if (item >= 0 && item < n) {
            int64_t ed;
            if (role == 0) ed = s + ia + item;
            else ed = (item < ia) ? s + item : s + ib + (item - ia);
            c = col[ed];
            v = val ? val[ed] : 1.0f;
          }
          scol[t * kSlots + j] = c;
          sval[t * kSlots + j] = v;
        }
      }
    }
  }
}

// ------------------------------------------------------ long-row kernel ----
// One warp per row (from a row list, or every row), register gathers straight
// from global memory, the same role split / order / epilogue.  Serves rows
// longer than kLong and feature widths the bulk path does not cover.
struct LongArgs {
  FusedArgs f;
  const int32_t *list;  // nullptr: all rows
  int64_t count;
};

// role item k -> edge id
struct RoleMap {
  int64_t s, a, b;
  bool intra;
  __device__ __forceinline__ int64_t edge(int64_t k) const {
    if (intra) return a + k;
    return (k < a - s) ? s + k : b + (k - (a - s));
  }
};

template <int VEC>
__device__ __forceinline__ Vf<VEC> g_contrib(const LongArgs &la, const RoleMap &m, int64_t k,
                                             int f, bool raw) {
  const int64_t e = m.edge(k);
  const int32_t c = __ldg(la.f.col + e);
  Vf<VEC> v = ldv<VEC>(la.f.x + static_cast<int64_t>(c) * la.f.feat + f);
  if (!raw && la.f.val) v = vscale<VEC>(__ldg(la.f.val + e), v);
  return v;
}

template <int VEC>
__device__ __forceinline__ Vf<VEC> g_leaf(const LongArgs &la, const RoleMap &m, int64_t start,
                                          int n, int f) {
  Vf<VEC> res = splat<VEC>(-0.0f);
  int i = 0;
  if (n >= 8) {
    Vf<VEC> r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = g_contrib<VEC>(la, m, start + j, f, false);
    const int mm = n - (n & 7);
    for (i = 8; i < mm; i += 8) {
      Vf<VEC> c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = g_contrib<VEC>(la, m, start + i + j, f, false);
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = vadd<VEC>(r[j], c[j]);
    }
    res = vadd<VEC>(vadd<VEC>(vadd<VEC>(r[0], r[1]), vadd<VEC>(r[2], r[3])),
                    vadd<VEC>(vadd<VEC>(r[4], r[5]), vadd<VEC>(r[6], r[7])));
    i = mm;
  }
  Vf<VEC> c[7];
#pragma unroll
  for (int t = 0; t < 7; ++t)
    if (i + t < n) c[t] = g_contrib<VEC>(la, m, start + i + t, f, false);
#pragma unroll
  for (int t = 0; t < 7; ++t)
    if (i + t < n) res = vadd<VEC>(res, c[t]);
  return res;
}

template <int VEC>
__device__ __noinline__ Vf<VEC> g_pairwise(const LongArgs la, const RoleMap m, int64_t start,
                                           int n, int f) {
  int64_t st_start[kDepth];
  int st_n[kDepth];
  int st_stage[kDepth];
  Vf<VEC> st_left[kDepth];
  int sp = 0;
  st_start[0] = start;
  st_n[0] = n;
  st_stage[0] = 0;
  Vf<VEC> ret = splat<VEC>(0.0f);
  while (sp >= 0) {
    const int cn = st_n[sp];
    if (cn <= kLeafN) {
      ret = g_leaf<VEC>(la, m, st_start[sp], cn, f);
      --sp;
      continue;
    }
    int n2 = cn / 2;
    n2 -= n2 & 7;
    if (st_stage[sp] == 0) {
      st_stage[sp] = 1;
      st_start[sp + 1] = st_start[sp];
      st_n[sp + 1] = n2;
      st_stage[sp + 1] = 0;
      ++sp;
    } else if (st_stage[sp] == 1) {
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

template <int VEC, bool IS_MAX>
__device__ __forceinline__ Vf<VEC> g_role(const LongArgs &la, const RoleMap &m, int64_t n,
                                          int f) {
  if (n <= 0) return splat<VEC>(0.0f);
  if constexpr (IS_MAX) {
    Vf<VEC> acc = g_contrib<VEC>(la, m, 0, f, true);
    int64_t k = 1;
    for (; k + 4 <= n; k += 4) {
      Vf<VEC> c[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) c[j] = g_contrib<VEC>(la, m, k + j, f, true);
#pragma unroll
      for (int j = 0; j < 4; ++j) acc = vmax<VEC>(acc, c[j]);
    }
    for (; k < n; ++k) acc = vmax<VEC>(acc, g_contrib<VEC>(la, m, k, f, true));
    return acc;
  } else {
    Vf<VEC> c0 = g_contrib<VEC>(la, m, 0, f, false);
    if (n == 1) return c0;
    return vadd<VEC>(c0, g_pairwise<VEC>(la, m, 1, static_cast<int>(n - 1), f));
  }
}

template <int VEC, bool IS_MAX>
__global__ void __launch_bounds__(256) long_row_kernel(LongArgs la) {
  const FusedArgs &a = la.f;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t n_items = la.list ? la.count : a.rows;
  for (int64_t it = gw; it < n_items; it += nw) {
    const int64_t r = la.list ? la.list[it] : it;
    const int64_t s = a.row_ptr[r], e = a.row_ptr[r + 1];
    int64_t ra = s, rb = s;
    if (a.block > 0) {  // intra run: binary search of [cB, cB+B) in the sorted row
      const int64_t cb = (r / a.block) * a.block;
      int64_t lo = s, hi = e;
      while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (a.col[m] < cb) lo = m + 1; else hi = m; }
      ra = lo;
      hi = e;
      while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (a.col[m] < cb + a.block) lo = m + 1; else hi = m;
      }
      rb = lo;
    }
    const int64_t ni = (a.mask & 1) ? rb - ra : 0;
    const int64_t no = (a.mask & 2) ? (e - s) - (rb - ra) : 0;
    const RoleMap mi{s, ra, rb, true}, mo{s, ra, rb, false};
    for (int f0 = 0; f0 < a.feat; f0 += 32 * VEC) {
      const int f = f0 + lane * VEC;
      if (f >= a.feat) continue;
      Vf<VEC> I = g_role<VEC, IS_MAX>(la, mi, ni, f);
      Vf<VEC> O = g_role<VEC, IS_MAX>(la, mo, no, f);
      Vf<VEC> out;
      if (a.mask == 3) {
        const int64_t d = (a.ep.op == AG_OP_MEAN && a.ep.deg) ? a.ep.deg[r] : 1;
        out = combine2<VEC>(a.ep.op, I, ni > 0, O, no > 0, d);
        if (a.ep.flags & AG_EPI_GIN)
          out = vadd<VEC>(vscale<VEC>(a.ep.gin_scale, ldv<VEC>(a.x + r * a.feat + f)), out);
        stv<VEC>(a.y + r * a.feat + f, out);
      } else {
        const bool t = (a.mask == 1) ? ni > 0 : no > 0;
        if (a.ep.flags & AG_EPI_EMPTY_OTHER) {
          const int64_t d = (a.ep.op == AG_OP_MEAN && a.ep.deg) ? a.ep.deg[r] : 1;
          out = combine2<VEC>(a.ep.op, (a.mask == 1) ? I : O, t, splat<VEC>(0.0f), false, d);
          if (a.ep.flags & AG_EPI_GIN)
            out = vadd<VEC>(vscale<VEC>(a.ep.gin_scale, ldv<VEC>(a.x + r * a.feat + f)), out);
          stv<VEC>(a.y + r * a.feat + f, out);
        } else {
          epilogue_store<VEC>(a.ep, a.y, r, f, (a.mask == 1) ? I : O, t);
        }
      }
    }
  }
}

inline int pick_vec(int64_t feat, const void *x, const void *y) {
  auto al = [](const void *p, int b) { return (reinterpret_cast<uintptr_t>(p) % b) == 0; };
  if (feat % 4 == 0 && al(x, 16) && al(y, 16)) return 4;
  if (feat % 2 == 0 && al(x, 8) && al(y, 8)) return 2;
  return 1;
}

template <int VEC>
int launch_long(const LongArgs &la, bool is_max, cudaStream_t st) {
  const int64_t n = la.list ? la.count : la.f.rows;
  if (n == 0) return AG_OK;
  int64_t blocks = (n * 32 + 255) / 256;
  const int64_t cap = static_cast<int64_t>(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  if (is_max) long_row_kernel<VEC, true><<<(int)blocks, 256, 0, st>>>(la);
  else long_row_kernel<VEC, false><<<(int)blocks, 256, 0, st>>>(la);
  AG_LAUNCH_CHECK("long_row_kernel");
  return AG_OK;
}

int launch_long_any(const LongArgs &la, bool is_max, cudaStream_t st) {
  switch (pick_vec(la.f.feat, la.f.x, la.f.y)) {
    case 4: return launch_long<4>(la, is_max, st);
    case 2: return launch_long<2>(la, is_max, st);
    default: return launch_long<1>(la, is_max, st);
  }
}

template <int FV>
int launch_fused(FusedArgs a, bool is_max, cudaStream_t st) {
  a.stages = FV == 1 ? 4 : 2;
  const int hdr = (8 * a.stages + 4 * kSlots * a.stages + 16 + 127) / 128 * 128;
  const int ring = a.stages * kSlots * a.feat * 4;
  a.warp_bytes = hdr + (ring + 127) / 128 * 128;
  const int budget = 220 * 1024;
  const int max_warps = FV == 1 ? 16 : 12;
  a.warps = std::max(1, std::min(max_warps, budget / a.warp_bytes));
  a.one = 1.0f;
  const int smem = a.warps * a.warp_bytes;
  const int64_t nchunks = (a.rows + kChunk - 1) / kChunk;
  auto k = is_max ? fused_kernel<FV, true> : fused_kernel<FV, false>;
  AG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  AG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, a.warps * 32, smem));
  if (per_sm < 1) per_sm = 1;
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;
  const int64_t need = (nchunks + a.warps - 1) / a.warps;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  Scratch ctr;
  AG_CUDA(ctr.alloc(sizeof(unsigned int), st));
  AG_CUDA(cudaMemsetAsync(ctr.ptr, 0, sizeof(unsigned int), st));
  a.chunk_ctr = ctr.as<unsigned int>();
  k<<<(int)grid, a.warps * 32, smem, st>>>(a);
  AG_LAUNCH_CHECK("fused_kernel");
  return AG_OK;
}

}  // namespace
}  // namespace ag

using namespace ag;

extern "C" int ag_stage_layout_count(int64_t num_rows, const int32_t *row_ptr,
                                     const int32_t *col_idx, int64_t block_size,
                                     int32_t role_mask, int32_t *stage_ptr, int32_t *counts,
                                     int64_t *num_stages_host, void *stream) {
  *num_stages_host = 0;
  if (block_size < 0) return fail(AG_ERR_VALUE, "block_size must be >= 0");
  if (role_mask < 1 || role_mask > 3) return fail(AG_ERR_VALUE, "role_mask must be 1, 2 or 3");
  if (block_size == 0 && role_mask != 2)
    return fail(AG_ERR_VALUE, "block_size 0 (no split) requires role_mask 2");
  cudaStream_t st = as_stream(stream);
  const int64_t n = num_rows + 1;
  Scratch ns, tmp;
  AG_CUDA(ns.alloc(n * sizeof(int32_t), st));
  AG_CUDA(cudaMemsetAsync(ns.ptr, 0, n * sizeof(int32_t), st));
  if (num_rows > 0) {
    layout_count_kernel<<<grid_for(num_rows, 256), 256, 0, st>>>(
        num_rows, row_ptr, col_idx, block_size, role_mask, reinterpret_cast<int2 *>(counts),
        ns.as<int32_t>());
    AG_LAUNCH_CHECK("layout_count_kernel");
  }
  size_t bytes = 0;
  AG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, ns.as<int32_t>(), stage_ptr, (int)n, st));
  AG_CUDA(tmp.alloc(bytes, st));
  AG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, bytes, ns.as<int32_t>(), stage_ptr, (int)n, st));
  int32_t total = 0;
  AG_CUDA(cudaMemcpyAsync(&total, stage_ptr + num_rows, 4, cudaMemcpyDeviceToHost, st));
  AG_CUDA(cudaStreamSynchronize(st));
  *num_stages_host = total;
  return AG_OK;
}

extern "C" int ag_stage_layout_fill(int64_t num_rows, const int32_t *row_ptr,
                                    const int32_t *col_idx, const float *val, int64_t block_size,
                                    const int32_t *stage_ptr, const int32_t *counts,
                                    int32_t *stage_col, float *stage_val, void *stream) {
  if (num_rows == 0) return AG_OK;
  layout_fill_kernel<<<grid_for(num_rows, 128), 128, 0, as_stream(stream)>>>(
      num_rows, row_ptr, col_idx, val, block_size, stage_ptr,
      reinterpret_cast<const int2 *>(counts), stage_col, stage_val);
  AG_LAUNCH_CHECK("layout_fill_kernel");
  return AG_OK;
}

extern "C" int ag_fused_spmm(int64_t num_rows, int64_t feat, int64_t block_size,
                             int32_t role_mask, const int32_t *row_ptr, const int32_t *col_idx,
                             const float *val, const int32_t *stage_ptr, const int32_t *counts,
                             const int32_t *stage_col, const float *stage_val, const float *x,
                             float *y, int32_t op, int32_t epi_flags,
                             const uint8_t *other_touched, const int64_t *deg, float gin_scale,
                             void *stream) {
  if (num_rows < 0 || feat < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (op < AG_OP_SUM || op > AG_OP_MAX) return fail(AG_ERR_KERNEL, "unknown op %d", op);
  if (role_mask < 1 || role_mask > 3) return fail(AG_ERR_VALUE, "role_mask must be 1, 2 or 3");
  if (block_size < 0) return fail(AG_ERR_VALUE, "block_size must be >= 0");
  if (block_size == 0 && role_mask != 2)
    return fail(AG_ERR_VALUE, "block_size 0 (no split) requires role_mask 2");
  if (op == AG_OP_MEAN && deg == nullptr && (role_mask == 3 || (epi_flags & AG_EPI_COMBINE)))
    return fail(AG_ERR_KERNEL, "mean combine requires the full-graph degree vector");
  if (num_rows == 0 || feat == 0) return AG_OK;
  if (num_rows > 2147483647LL || block_size > 2147483647LL)
    return fail(AG_ERR_VALUE, "too many rows");
  cudaStream_t st = as_stream(stream);
  FusedArgs a{num_rows, static_cast<int>(feat), static_cast<int>(block_size), role_mask, row_ptr,
              col_idx, val, x, y, Epi{op, epi_flags, other_touched, deg, x, feat, gin_scale},
              stage_ptr, reinterpret_cast<const int2 *>(counts), stage_col, stage_val, nullptr,
              0, 0, 2, 1.0f};
  const bool is_max = op == AG_OP_MAX;
  const bool bulk_ok = feat % 4 == 0 && feat <= 256 && stage_ptr && counts && stage_col &&
                       stage_val && (reinterpret_cast<uintptr_t>(x) % 16) == 0 &&
                       (reinterpret_cast<uintptr_t>(y) % 16) == 0;
  if (!bulk_ok) return launch_long_any(LongArgs{a, nullptr, 0}, is_max, st);
  return feat <= 128 ? launch_fused<1>(a, is_max, st) : launch_fused<2>(a, is_max, st);
}
