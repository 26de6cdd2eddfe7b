// The dense update GEMMs of the GCN/GIN layers on the 5th-generation tensor
// cores (tcgen05, kind::tf32) with fp32-faithful 3xTF32 splitting.
//
//   forward  out = agg @ W          A = agg [M=V][K] (K-major), B = W [K][N] (N-major)
//   backward dH  = G @ W^T          A = G   [V][K]   (K-major), B = W [N][K] (K-major)
//            dW  = agg^T @ G        A = agg [K=V][M] (M-major), B = G [K][N] (N-major)
// (models.py:99, :112 `agg @ W`; the backward products are the composed
// training step of SURVEY.md §8c.)
//
// 3xTF32: every fp32 operand x is split in shared memory into hi = x with the
// low 13 mantissa bits cleared (exactly representable in tf32) and
// lo = x - hi (exact in fp32).  The tile product is accumulated in TWO fp32
// TMEM accumulators -- A_hi*B_hi (exact 22-bit products) and the correction
// A_hi*B_lo + A_lo*B_hi (~2^-11 smaller, so its own rounding is negligible) --
// which the epilogue adds in IEEE fp32.  Keeping the correction out of the
// main accumulator matters: the tensor core's fp32 accumulation truncates, and
// folding the small terms into the large sum tripled the error.  The dropped
// A_lo*B_lo term is ~2^-22 relative.
//
// Kernel anatomy (one CTA per SM, persistent over 128 x BN output tiles and,
// for the skinny dW product, K splits):
//   warp 0        TMA producer: A and B k-blocks (32 fp32 = one 128-byte
//                 swizzle row) into a 2-3 stage shared-memory ring, SWIZZLE_128B
//   warps 2-5     splitters: x -> hi (in place) and lo (second buffer), then
//                 fence.proxy.async so the tensor core sees the writes
//   warp 1        TMEM allocator + single-thread tcgen05.mma issuer (3 MMAs per
//                 K=8 step), tcgen05.commit frees ring slots / publishes tiles
//   warps 6-9     epilogue: tcgen05.ld 32x32b -> alpha/beta/ReLU -> global,
//                 double-buffered TMEM accumulators so it overlaps the next tile
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "ag_common.cuh"

namespace ag {
namespace {

constexpr int BM = 128;
// fp32 elements per k-block: one 128-byte swizzle row (SWIZZLE_128B).  BK = 16
// (SWIZZLE_64B, 4 stages of 48 KB) also works and was measured: no faster for
// K = 256 and slower for short K (twice the per-k-block barrier round trips).
#ifndef AG_TC_BK
#define AG_TC_BK 32
#endif
constexpr int BK = AG_TC_BK;
constexpr int kKRow = BK * 4;                       // bytes per K-major row
constexpr uint64_t kKLayout = BK == 32 ? 2ull : 4ull;  // SWIZZLE_128B / SWIZZLE_64B
constexpr uint32_t kKSbo = 8 * kKRow;               // 8-row swizzle atom
constexpr uint32_t kMnBox = 128 * BK;               // MN-major TMA box {32 mn, BK k} bytes
// warps: 0 TMA, 1 MMA, 2-5 splitters, 6-13 epilogue (two per TMEM lane quarter, each
// taking half of the tile's columns: the epilogue bounds short-K products)
constexpr int kEpiWarps = 8;
constexpr int kThreads = (6 + kEpiWarps) * 32;
constexpr int kConvWarp0 = 2, kEpiWarp0 = 6;
// chunked split-K (TcArgs::split_mode 2): k-blocks per tensor-core accumulation
// chunk length 1024 k-blocks = 32768 rows: products up to ~4.8M rows keep
// one accumulation per CTA (C5 dW: 33k rows per split, 3e-7 of the sum of
// |terms|, scripts/gemm_kerr.py); longer K is chunked so the truncation of
// one accumulation stays bounded.  Shorter chunks measured slower (per-chunk
// epilogue round trips and workspace): 2048 rows 2.15 ms vs 1.68 ms at C5.
constexpr int kChunkKb = 1024;

struct TcArgs {
  int64_t M, N, K;
  float *C;         // output (splits == 1) or partial workspace [splits][M][N]
  int64_t ldc;
  float alpha, beta;
  int relu;
  int m_tiles, n_tiles, splits;
  int raw_hi;  // 1: leave x in place as the hi operand (the MMA reads its tf32 bits)
  int b_presplit;  // 1: B's lo half comes from global (ag_tf32_split_lo), only A is split
  int exp;         // timing experiments (AG_TC_EXP bits; results invalid): 1 no split,
                   // 2 one MMA per k-step, 4 no epilogue stores
  const uint32_t *mask;  // ReLU-backward bit mask (NULL: none): out = bit ? out : 0
  int64_t ldm;           // words per mask row
  uint32_t *mask_out;    // (splits == 1) bits of out > 0 (the forward ReLU's mask), or NULL
  int64_t ldmo;
  int64_t k_per_split;  // multiple of BK
  // split-K products: 1 = the partial of split s goes to workspace slot s; 2 =
  // "chunked": every CTA adds each of its (short) K splits into its own slot
  // [blockIdx.x][M][N] in IEEE fp32, so no tensor-core accumulation runs over
  // more than k_per_split rows (its fp32 accumulation truncates: the error of
  // one long accumulation grows with K, measured 20x numpy's at K = 2.45M)
  int split_mode;
  // block-diagonal product (ag_block_diag_gemm_tf32x3): the B operand's K rows
  // of output tile m0 start at the panel base (m0 / bdiag) * bdiag; 0 = plain GEMM
  int64_t bdiag;
  int c_tma;            // 1: tmC maps C (direct products): the epilogue stores by TMA
  long long *trace;     // AG_TC_TRACE: per-tile clock stamps of CTA 0 (development only)
};
constexpr int kTraceTiles = 48;
// CTA 0 stamps (globaltimer, ns): [tile][0] MMA tempty-wait start, [1] its end, [2] MMA's
// last k-block issued, [3] epilogue tfull-wait start, [4] its end, [5] epilogue done;
// [6..] the MMA warp's conv waits of the tile's first two k-blocks (start, end)
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------ PTX helpers --
__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
constexpr uint32_t kWaitHintNs = 20000;
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
// Waits suspend the warp in hardware (try_wait with a time hint) until the
// phase completes instead of spinning: idle splitter / epilogue warps polling
// took a third of the issue slots the epilogue needs (ncu, C5 dH product).
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
    if (++spins > (1u << 22)) __trap();  // a lost arrival: fail instead of hanging
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity), "r"(kWaitHintNs)
        : "memory");
  }
}
// Spin wait for the single-thread critical path (TMA producer, MMA issuer).
__device__ __forceinline__ void mbar_wait_spin(uint64_t *b, uint32_t parity) {
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
    if (++spins > (1u << 26)) __trap();
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   su32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          su32(b)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
// TMA tensor store of a 32 x 32 fp32 box from shared memory (bulk group)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// the same load delivered to the same shared-memory offset (and mbarrier) of
// every CTA in `mask` of the cluster
__device__ __forceinline__ void tma_load_2d_mc(void *dst, const CUtensorMap *map, uint64_t *bar,
                                               int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t *bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(bar)),
      "h"(mask)
      : "memory");
}
// ---- 2-SM (cta_group::2) pair helpers: the leader (cluster rank 0) issues the
// M = 256 MMAs over both CTAs' shared memory; barrier arrivals from the peer
// target the leader's barriers through their cluster addresses
__device__ __forceinline__ uint32_t mapa_rank(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *b, uint32_t parity) {
  uint32_t done = 0;
  uint32_t spins = 0;
  while (!done) {
    if (++spins > (1u << 26)) __trap();
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tc_mma_tf32_2sm(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_2sm(uint64_t *bar) {  // arrives on both CTAs' barrier
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// 32 consecutive fp32 columns of this lane's TMEM row, no wait (the caller
// issues tmem_wait_ld() once for several loads)
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor (sm_100 version 1).  K-major operands use
// SWIZZLE_128B (layout 2: 8 rows x 128 B atoms, 16-byte chunks XOR row%8);
// tf32 MN-major operands must use SWIZZLE_128B_BASE32B (layout 1: 4 K-rows x
// 128 B atoms, 32-byte chunks XOR row%4), which TMA writes with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo,
                                              bool mn) {
  return (static_cast<uint64_t>((addr >> 4) & 0x3FFFu)) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) |
         ((mn ? 1ull : kKLayout) << 61);
}

// Instruction descriptor: D f32, A/B tf32, majors, N, M = 128.
__host__ __device__ constexpr uint32_t instr_desc(bool a_mn, bool b_mn, int n, int m = BM) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

template <int BN, bool ONE = false, bool P2 = false>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;   // 16 KB
  // P2 (2-SM pair): each CTA holds half of the B tile's columns
  static constexpr int B_BYTES = (P2 ? BN / 2 : BN) * BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES =
      STAGE * 4 <= 200 * 1024 ? 4 : STAGE * 3 <= 200 * 1024 ? 3 : 2;
  // two fp32 accumulators per tile (hi*hi and the hi*lo + lo*hi correction),
  // double-buffered when TMEM allows
  // ONE: the correction and hi*hi products share one accumulator (half the
  // TMEM, so a 256-wide tile is double-buffered and the epilogue overlaps the
  // next tile's MMAs); error ~3e-7 relative instead of ~1e-7
  static constexpr int NACC = ONE ? 1 : 2;
  static constexpr int ACC_BUFS = 2 * NACC * BN <= 512 ? 2 : 1;
  static constexpr int COLS = ACC_BUFS * NACC * BN;
  static constexpr int TMEM_COLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128
                                 : COLS <= 256 ? 256 : 512;
  // epilogue transpose buffers: kEpiWarps x (32 rows x 32 fp32)
  static constexpr int EPI = kEpiWarps * 32 * 32 * 4;
  static constexpr int SMEM = STAGES * STAGE + 1024 /* align */ + 256 /* barriers */ + EPI;
};

// split x (fp32) into hi (in place) and lo, n4 float4s.  RAW: only lo is
// written and x stays as the hi operand -- valid because kind::tf32 reads
// just the top 19 bits of each fp32 operand (verified bitwise against the
// masked split by tests/test_gemm_gpu.py).
template <bool RAW>
__device__ __forceinline__ void split_tile(uint32_t hi, uint32_t lo, int n4, int t, int nt) {
  // shared-space addresses: generic pointers here compile to LD.E / ST.E
  // through the generic path (long-scoreboard latency)
#pragma unroll 4
  for (int i = t; i < n4; i += nt) {
    float4 v, h, l;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(hi + i * 16)
                 : "memory");
    h.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
    l.x = __fsub_rn(v.x, h.x);
    l.y = __fsub_rn(v.y, h.y);
    l.z = __fsub_rn(v.z, h.z);
    l.w = __fsub_rn(v.w, h.w);
    if (!RAW)
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(hi + i * 16), "f"(h.x),
                   "f"(h.y), "f"(h.z), "f"(h.w)
                   : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(lo + i * 16), "f"(l.x),
                 "f"(l.y), "f"(l.z), "f"(l.w)
                 : "memory");
  }
}

// CL > 1: a cluster of CL CTAs computes CL vertically adjacent 128-row tiles
// of the same N tile in lockstep; each CTA TMA-loads 1/CL of every B k-block
// and multicasts it to all of them, so B crosses L2 once per cluster, and the
// MMA completions free the stage in every CTA (multicast commit).
template <int BN, bool A_MN, bool B_MN, bool ONE, int CL, bool P2 = false>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmBl,
                   const __grid_constant__ CUtensorMap tmC, TcArgs g) {
  using C = Cfg<BN, ONE, P2>;
  static_assert(!P2 || CL == 2, "a 2-SM pair is a cluster of two");
  extern __shared__ unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  // epilogue staging buffers first (1024-byte aligned: the TMA store's 128B
  // swizzle is a function of the absolute shared address), then the barriers
  unsigned char *epi_buf = smem + C::STAGES * C::STAGE;  // C::EPI bytes
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE + C::EPI);
  uint64_t *conv = full + C::STAGES;
  uint64_t *empty = conv + C::STAGES;
  uint64_t *tfull = empty + C::STAGES;  // [2]
  uint64_t *tempty = tfull + 2;         // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster tiles: CL consecutive M tiles x one N tile x one K split
  const int rank = static_cast<int>(blockIdx.x % CL);
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int64_t msup = (g.m_tiles + CL - 1) / CL;
  const int64_t tiles_mn = msup * g.n_tiles;
  const int64_t total = tiles_mn * g.splits;
  const int nkb_full = static_cast<int>(g.k_per_split / BK);
  constexpr uint16_t kAll = static_cast<uint16_t>((1u << CL) - 1u);
  // tile index math in 32 bits (64-bit division is a long software sequence on
  // the epilogue's critical path between tiles; tile counts are < 2^31)
  const uint32_t tmn32 = static_cast<uint32_t>(tiles_mn), nt32 = static_cast<uint32_t>(g.n_tiles);
  auto tile_m0 = [&](int64_t t) -> int64_t {
    return static_cast<int64_t>(((static_cast<uint32_t>(t) % tmn32) / nt32) * CL + rank) * BM;
  };
  auto tile_n0 = [&](int64_t t) -> int64_t {
    return static_cast<int64_t>((static_cast<uint32_t>(t) % tmn32) % nt32) * BN;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], P2 ? 8 : 4);     // P2: both CTAs' splitters arrive on the leader's
      mbar_init(&empty[s], P2 ? 1 : CL);   // P2: the leader's multicast commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], P2 ? 2 * kEpiWarps : kEpiWarps);  // P2: both CTAs' epilogues
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
  }
  if (warp == 1) {
    if constexpr (P2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "n"(C::TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();  // every CTA's barriers exist before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // k-blocks of tile t (the last split may be shorter)
  auto tile_kblocks = [&](int64_t t, int64_t &k0) -> int {
    const int64_t s = static_cast<uint32_t>(t) / tmn32;
    k0 = s * g.k_per_split;
    const int64_t k1 = std::min<int64_t>(g.K, k0 + g.k_per_split);
    const int64_t nk = (k1 - k0 + BK - 1) / BK;
    return static_cast<int>(nk < nkb_full ? nk : nkb_full);
  };

  if (warp == 0) {
    // ----------------------------------------------------- TMA producer --
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = cid; t < total; t += ncl) {
        const int m0 = static_cast<int>(tile_m0(t));
        const int n0 = static_cast<int>(tile_n0(t));
        int64_t k0;
        const int nkb = tile_kblocks(t, k0);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait_spin(&empty[stage], phase ^ 1);
          unsigned char *st = smem + stage * C::STAGE;
          unsigned char *sa = st, *sb = st + 2 * C::A_BYTES;
          if (g.exp & 32) {  // experiment: no operand traffic, handoffs only
            mbar_expect_tx(&full[stage], 0);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_expect_tx(&full[stage], C::A_BYTES + (g.b_presplit ? 2 : 1) * C::B_BYTES);
          const int kk = static_cast<int>(k0 + static_cast<int64_t>(kb) * BK);
          if (A_MN) {  // boxes {32 (m), 32 (k)}: 4 KB each, LBO apart
#pragma unroll
            for (int c = 0; c < BM / 32; ++c) tma_load_2d(sa + c * kMnBox, &tmA, &full[stage],
                                                          m0 + 32 * c, kk);
          } else {  // box {32 (k), 128 (m)}
            tma_load_2d(sa, &tmA, &full[stage], kk, m0);
          }
          // B (and its presplit lo half): this CTA's 1/CL share, multicast
          // block-diagonal mode: this tile's B rows start at its panel base
          const int kb_row = kk + (g.bdiag ? static_cast<int>((m0 / g.bdiag) * g.bdiag) : 0);
          auto load_b = [&](unsigned char *dst, const CUtensorMap *map) {
            if constexpr (P2) {  // this CTA's half of the columns, no multicast
              if (B_MN) {
#pragma unroll
                for (int c = 0; c < BN / 64; ++c)
                  tma_load_2d(dst + c * kMnBox, map, &full[stage],
                              n0 + rank * (BN / 2) + 32 * c, kb_row);
              } else {
                tma_load_2d(dst, map, &full[stage], kb_row, n0 + rank * (BN / 2));
              }
              return;
            }
            if (B_MN) {  // BN/32 boxes {32 (n), 32 (k)}: box c from CTA c % CL
#pragma unroll
              for (int c = 0; c < BN / 32; ++c) {
                if (CL == 1) tma_load_2d(dst + c * kMnBox, map, &full[stage], n0 + 32 * c, kb_row);
                else if (c % CL == rank)
                  tma_load_2d_mc(dst + c * kMnBox, map, &full[stage], n0 + 32 * c, kb_row, kAll);
              }
            } else {  // box {32 (k), BN / CL rows}: rows of 128 B, 8-row swizzle atoms
              constexpr int R = BN / CL;
              if (CL == 1) tma_load_2d(dst, map, &full[stage], kb_row, n0);
              else tma_load_2d_mc(dst + rank * R * kKRow, map, &full[stage], kb_row, n0 + rank * R,
                                  kAll);
            }
          };
          load_b(sb, &tmB);
          if (g.b_presplit) load_b(sb + C::B_BYTES, &tmBl);  // raw B is the hi half
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ----------------------------------------------------- MMA issuer ----
    // P2: the leader issues M = 256 MMAs over both CTAs; the peer's warp idles
    if (P2 && rank != 0) {
    } else {
    constexpr uint32_t idesc = instr_desc(A_MN, B_MN, BN, P2 ? 2 * BM : BM);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = cid; t < total; t += ncl) {
      int64_t k0;
      const int nkb = tile_kblocks(t, k0);
      const int ti = static_cast<int>(static_cast<uint32_t>(t - cid) / static_cast<uint32_t>(ncl));
      const bool tr = g.trace != nullptr && blockIdx.x == 0 && lane == 0 && ti < kTraceTiles;
      if (tr) g.trace[ti * 10 + 0] = gtime();
      if (P2) mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
      else mbar_wait_spin(&tempty[acc], acc_phase ^ 1);
      if (tr) g.trace[ti * 10 + 1] = gtime();
      tc_fence_after();
      const uint32_t d = tmem_base + static_cast<uint32_t>(acc * C::NACC * BN);  // hi*hi
      const uint32_t dc = ONE ? d : d + BN;                                     // correction
      for (int kb = 0; kb < nkb; ++kb) {
        if (tr && kb < 2) g.trace[ti * 10 + 6 + 2 * kb] = gtime();
        if (P2) mbar_wait_cluster(&conv[stage], phase);
        else mbar_wait_spin(&conv[stage], phase);
        if (tr && kb < 2) g.trace[ti * 10 + 7 + 2 * kb] = gtime();
        tc_fence_after();
        if (lane == 0) {
          if (tr && kb == nkb - 1) g.trace[ti * 10 + 2] = gtime();
          const uint32_t st = su32(smem + stage * C::STAGE);
          const uint32_t a_hi = st, a_lo = st + C::A_BYTES;
          const uint32_t b_hi = st + 2 * C::A_BYTES, b_lo = b_hi + C::B_BYTES;
#pragma unroll
          for (int ks = 0; ks < BK / 8; ++ks) {
            // K=8 step: K-major advances 32 B inside the swizzle row, MN-major
            // advances 8 K-rows (two 512 B atoms, 1 KB)
            const uint32_t ao = A_MN ? ks * 1024 : ks * 32;
            const uint32_t bo = B_MN ? ks * 1024 : ks * 32;
            // MN-major: LBO = next 32-element MN chunk (one 4 KB TMA box),
            // SBO = next 4-row K atom (512 B); K-major: SBO = next 8-row group
            const uint32_t albo = A_MN ? kMnBox : 16, asbo = A_MN ? 512 : kKSbo;
            const uint32_t blbo = B_MN ? kMnBox : 16, bsbo = B_MN ? 512 : kKSbo;
            const uint64_t dah = smem_desc(a_hi + ao, albo, asbo, A_MN);
            const uint64_t dal = smem_desc(a_lo + ao, albo, asbo, A_MN);
            const uint64_t dbh = smem_desc(b_hi + bo, blbo, bsbo, B_MN);
            const uint64_t dbl = smem_desc(b_lo + bo, blbo, bsbo, B_MN);
            const uint32_t first = (kb == 0 && ks == 0) ? 0u : 1u;
            if constexpr (P2) {
              tc_mma_tf32_2sm(dc, dal, dbh, idesc, first);
              tc_mma_tf32_2sm(dc, dah, dbl, idesc, 1u);
              tc_mma_tf32_2sm(d, dah, dbh, idesc, ONE ? 1u : first);
            } else {
              if (!(g.exp & 18)) {
                tc_mma_tf32(dc, dal, dbh, idesc, first);
                tc_mma_tf32(dc, dah, dbl, idesc, 1u);
              }
              if (!(g.exp & 16)) tc_mma_tf32(d, dah, dbh, idesc, ONE ? 1u : first);
            }
          }
          if constexpr (P2) {
            tc_commit_2sm(&empty[stage]);  // the stage is free in both CTAs
            if (kb == nkb - 1) tc_commit_2sm(&tfull[acc]);
          } else {
            if (CL == 1) tc_commit(&empty[stage]);
            else tc_commit_mc(&empty[stage], kAll);  // the stage is free in every CTA's view
            if (kb == nkb - 1) tc_commit(&tfull[acc]);
          }
        }
        __syncwarp();
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (nkb == 0 && lane == 0) {  // (K == 0: nothing to do)
        if constexpr (P2) tc_commit_2sm(&tfull[acc]);
        else tc_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++acc == C::ACC_BUFS) { acc = 0; acc_phase ^= 1; }
    }
    }
  } else if (warp < kEpiWarp0) {
    // ------------------------------------------------------- splitters ---
    const int t_id = threadIdx.x - kConvWarp0 * 32;
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t t = cid; t < total; t += ncl) {
      int64_t k0;
      const int nkb = tile_kblocks(t, k0);
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full[stage], phase);
        const uint32_t st = su32(smem + stage * C::STAGE);
        if (g.exp & 1) {
        } else if (g.b_presplit) {
          split_tile<true>(st, st + C::A_BYTES, C::A_BYTES / 16, t_id, 128);
        } else if (g.raw_hi) {
          split_tile<true>(st, st + C::A_BYTES, C::A_BYTES / 16, t_id, 128);
          split_tile<true>(st + 2 * C::A_BYTES, st + 2 * C::A_BYTES + C::B_BYTES, C::B_BYTES / 16,
                           t_id, 128);
        } else {
          split_tile<false>(st, st + C::A_BYTES, C::A_BYTES / 16, t_id, 128);
          split_tile<false>(st + 2 * C::A_BYTES, st + 2 * C::A_BYTES + C::B_BYTES, C::B_BYTES / 16,
                            t_id, 128);
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if constexpr (P2) mbar_arrive_cluster(mapa_rank(&conv[stage], 0));
          else mbar_arrive(&conv[stage]);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // -------------------------------------------------------- epilogue ---
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int ehalf = (warp - kEpiWarp0) >> 2;  // which half of the tile's columns
    constexpr int kHalfCols = BN >= 64 ? BN / 2 : BN;
    const int c_lo = ehalf * kHalfCols, c_hi = BN >= 64 ? c_lo + kHalfCols : (ehalf ? 0 : BN);
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = cid; t < total; t += ncl) {
      const int64_t s = static_cast<uint32_t>(t) / tmn32;
      const int64_t m0 = tile_m0(t);
      const int64_t n0 = tile_n0(t);
      if (g.mask != nullptr && g.splits == 1 && warp == kEpiWarp0 && lane == 0) {
        // pull the NEXT tile's mask rows into L2 a tile period ahead: one bulk
        // prefetch of the whole contiguous row block (per-row prefetches from
        // every lane stalled the epilogue warps)
        auto prefetch_rows = [&](int64_t tt) {
          if (tt >= total) return;
          const int64_t r0 = tile_m0(tt);
          const int64_t r1 = std::min<int64_t>(r0 + BM, g.M);
          if (r1 <= r0) return;
          const uintptr_t lo = reinterpret_cast<uintptr_t>(g.mask + r0 * g.ldm) & ~uintptr_t(15);
          const uintptr_t hi = (reinterpret_cast<uintptr_t>(g.mask + (r1 - 1) * g.ldm +
                                                            relu_words(g.N)) + 15) & ~uintptr_t(15);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo),
                       "r"(static_cast<uint32_t>(hi - lo))
                       : "memory");
        };
        if (t == cid) prefetch_rows(t);
        prefetch_rows(t + ncl);
      }
      const int ti = static_cast<int>(static_cast<uint32_t>(t - cid) / static_cast<uint32_t>(ncl));
      const bool tr = g.trace != nullptr && blockIdx.x == 0 && warp == kEpiWarp0 && lane == 0 &&
                      ti < kTraceTiles;
      // this warp's 32 rows' ReLU-mask words for its column half, lane = row:
      // loaded once per tile before the accumulator wait (their latency
      // overlaps it); the row passes below take them by shuffle.  The forward
      // mask words (mask_out) are gathered the same way and stored once.
      const int64_t myrow = m0 + q * 32 + lane;
      const int nwords = (c_hi - c_lo) / 32;
      uint32_t mw[4] = {0u, 0u, 0u, 0u}, ow[4] = {0u, 0u, 0u, 0u};
      if (g.mask != nullptr && g.splits == 1 && myrow < g.M && !(g.exp & 8)) {
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (w < nwords && n0 + c_lo + 32 * w < g.N)
            mw[w] = __ldg(g.mask + myrow * g.ldm + ((n0 + c_lo) >> 5) + w);
      }
      if (tr) g.trace[ti * 10 + 3] = gtime();
      mbar_wait(&tfull[acc], acc_phase);
      if (tr) g.trace[ti * 10 + 4] = gtime();
      tc_fence_after();
      const bool direct = g.splits == 1;
      const bool vec_ok = ((reinterpret_cast<uintptr_t>(g.C) & 15) == 0) &&
                          (direct ? (g.ldc % 4 == 0) : (g.N % 4 == 0));
      // 32-column chunks: tcgen05.ld gives each lane one row; the chunk goes
      // through this warp's shared buffer (16-byte chunks XOR-swizzled by
      // row, conflict-free both ways) so that every global access below is
      // four full 128-byte row segments per instruction (coalesced C / mask
      // reads and stores).
      const uint32_t xb = su32(epi_buf) + static_cast<uint32_t>(warp - kEpiWarp0) * (32 * 32 * 4);
      const int rsub = lane >> 3, j4 = lane & 7;  // read-back role: row rsub + 4 i, chunk j4
      // TMA-store epilogue: direct products without a C read (beta = 0)
      const bool fast = g.c_tma && direct && g.beta == 0.0f && !(g.exp & 12);
#pragma unroll 1
      for (int c = c_lo; c < c_hi; c += 32) {
        const int cw = (c - c_lo) >> 5;
        const uint32_t mwc = cw == 0 ? mw[0] : cw == 1 ? mw[1] : cw == 2 ? mw[2] : mw[3];
        uint32_t owc = 0;
        float v[32];
        {
          uint32_t rh[32], rc[32];
          const uint32_t ta = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                              static_cast<uint32_t>(acc * C::NACC * BN + c);
          tmem_ld32_nowait(ta, rh);
          if (!ONE) tmem_ld32_nowait(ta + BN, rc);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            v[i] = ONE ? __uint_as_float(rh[i])
                       : __fadd_rn(__uint_as_float(rh[i]), __uint_as_float(rc[i]));
        }
        if (fast) {
          // lane = row: alpha / ReLU / the row's backward-mask bits and its
          // forward-mask word in registers, then the 32 x 32 chunk goes out
          // as one TMA tensor store from the (128B-swizzled) shared buffer
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float r = g.alpha == 1.0f ? v[i] : g.alpha * v[i];
            if (g.relu) r = fmaxf(r, 0.0f);
            if (g.mask != nullptr && !((mwc >> i) & 1u)) r = 0.0f;
            v[i] = r;
          }
          if (g.mask_out != nullptr) {
            uint32_t wd = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) wd |= (v[i] > 0.0f ? 1u : 0u) << i;
            if (cw == 0) ow[0] = wd;
            else if (cw == 1) ow[1] = wd;
            else if (cw == 2) ow[2] = wd;
            else ow[3] = wd;
          }
          if (lane == 0) bulk_wait_read0();  // the previous chunk's store has read xb
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                             xb + lane * 128 + ((j ^ (lane & 7)) * 16)),
                         "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                         : "memory");
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmC, xb, static_cast<int>(n0 + c), static_cast<int>(m0 + q * 32));
            bulk_commit();
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                           xb + lane * 128 + ((j ^ (lane & 7)) * 16)),
                       "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                       : "memory");
        __syncwarp();
        const int64_t col = n0 + c + 4 * j4;
        const bool col4 = col + 4 <= g.N;
        const bool colok = col < g.N;
        // all eight row passes' operands first, so their loads are in flight together
        float4 o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = 4 * i + rsub;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(o[i].x), "=f"(o[i].y), "=f"(o[i].z), "=f"(o[i].w)
                       : "r"(xb + rr * 128 + ((j4 ^ (rr & 7)) * 16))
                       : "memory");
        }
        __syncwarp();  // the buffer is rewritten by the next chunk
        const int64_t grow0 = m0 + q * 32 + rsub;
        if (direct && (g.mask != nullptr || g.beta != 0.0f)) {
#pragma unroll
          for (int hf = 0; hf < 8; hf += 4) {  // four passes' loads in flight at a time
          uint32_t mk[4];
          float4 cv[4];
#pragma unroll
          for (int i0 = 0; i0 < 4; ++i0) {
            const int i = hf + i0;
            const int64_t grow = grow0 + 4 * i;
            const bool in = grow < g.M && colok;
            cv[i0] = make_float4(0.f, 0.f, 0.f, 0.f);
            // the 4 columns' bits of the row's mask word (col % 4 == 0), from
            // the lane that loaded row 4 i + rsub
            const uint32_t word = __shfl_sync(0xffffffffu, mwc, 4 * i + rsub);
            mk[i0] = (g.mask != nullptr && !(g.exp & 8)) ? (word >> (col & 31)) & 15u : 15u;
            if (in && g.beta != 0.0f) {
              const float *cp = g.C + grow * g.ldc + col;
              if (vec_ok && col4) {
                cv[i0] = *reinterpret_cast<const float4 *>(cp);
              } else {
                cv[i0].x = cp[0];
                if (col + 1 < g.N) cv[i0].y = cp[1];
                if (col + 2 < g.N) cv[i0].z = cp[2];
                if (col + 3 < g.N) cv[i0].w = cp[3];
              }
            }
          }
#pragma unroll
          for (int i0 = 0; i0 < 4; ++i0) {
            const int i = hf + i0;
            float *ov = &o[i].x;
            const float *c4 = &cv[i0].x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float r = g.alpha == 1.0f ? ov[e] : g.alpha * ov[e];
              if (g.beta != 0.0f) r = fmaf(g.beta, c4[e], r);
              if (g.relu) r = fmaxf(r, 0.0f);
              if (!((mk[i0] >> e) & 1u)) r = 0.0f;
              ov[e] = r;
            }
          }
          }
        } else if (direct) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float *ov = &o[i].x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float r = g.alpha * ov[e];
              if (g.relu) r = fmaxf(r, 0.0f);
              ov[e] = r;
            }
          }
        }
        if (direct && g.mask_out != nullptr) {
          // forward ReLU mask: the 8 lanes of a row pass hold its 32 columns
          // [n0 + c, n0 + c + 32) = one mask word (n0, c multiples of 32)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float *ov = &o[i].x;
            uint32_t nib = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (col + e < g.N && ov[e] > 0.0f) nib |= 1u << e;
            uint32_t wd = nib << (4 * j4);
            wd |= __shfl_xor_sync(0xffffffffu, wd, 1);
            wd |= __shfl_xor_sync(0xffffffffu, wd, 2);
            wd |= __shfl_xor_sync(0xffffffffu, wd, 4);
            // lane l keeps row l's word (row 4 i + (l & 3) lives in group l & 3)
            const uint32_t wrow = __shfl_sync(0xffffffffu, wd, (lane & 3) * 8);
            if ((lane >> 2) == i) owc = wrow;
          }
          if (cw == 0) ow[0] = owc;
          else if (cw == 1) ow[1] = owc;
          else if (cw == 2) ow[2] = owc;
          else ow[3] = owc;
        }
        if (!(g.exp & 4)) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int64_t grow = grow0 + 4 * i;
            if (grow >= g.M || !colok) continue;
            const int64_t slot = g.split_mode == 2 ? static_cast<int64_t>(blockIdx.x) : s;
            float *cp = direct ? g.C + grow * g.ldc + col : g.C + (slot * g.M + grow) * g.N + col;
            if (g.split_mode == 2) {  // this CTA's running sum (slot zeroed by the host)
              if (vec_ok && col4) {
                const float4 p = *reinterpret_cast<const float4 *>(cp);
                o[i].x += p.x; o[i].y += p.y; o[i].z += p.z; o[i].w += p.w;
              } else {
                o[i].x += cp[0];
                if (col + 1 < g.N) o[i].y += cp[1];
                if (col + 2 < g.N) o[i].z += cp[2];
                if (col + 3 < g.N) o[i].w += cp[3];
              }
            }
            if (vec_ok && col4) {
              *reinterpret_cast<float4 *>(cp) = o[i];
            } else {
              cp[0] = o[i].x;
              if (col + 1 < g.N) cp[1] = o[i].y;
              if (col + 2 < g.N) cp[2] = o[i].z;
              if (col + 3 < g.N) cp[3] = o[i].w;
            }
          }
        }

      }
      if (g.splits == 1 && g.mask_out != nullptr && myrow < g.M) {
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (w < nwords && n0 + c_lo + 32 * w < g.N)
            g.mask_out[myrow * g.ldmo + ((n0 + c_lo) >> 5) + w] = ow[w];
      }
      tc_fence_before();
      __syncwarp();
      if (tr) g.trace[ti * 10 + 5] = gtime();
      if (lane == 0) {
        if constexpr (P2) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
        else mbar_arrive(&tempty[acc]);
      }
      if (++acc == C::ACC_BUFS) { acc = 0; acc_phase ^= 1; }
    }
  }

  if (warp >= kEpiWarp0 && lane == 0) bulk_wait0();  // the TMA stores have completed
  tc_fence_before();
  __syncthreads();
  if (CL > 1) cluster_sync();  // no CTA leaves while a peer may still signal / write it
  if (warp == 1) {
    tc_fence_after();
    if constexpr (P2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(C::TMEM_COLS)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "n"(C::TMEM_COLS)
                   : "memory");
  }
}

// Sum of the split-K partials: a 32 x 8 block takes 32 consecutive outputs;
// thread (o, g) adds partials g, g + 8, ... of output o in fp64 (loads
// coalesced across o), then the 8 group sums are added in a fixed order --
// deterministic, and 8x the memory parallelism of one thread per output
// walking all ~150 partials.
constexpr int kSumGroups = 8;
__global__ void __launch_bounds__(32 * kSumGroups) splitk_sum_kernel(
    int64_t M, int64_t N, int splits, const float *part, float *C, int64_t ldc, float alpha,
    float beta, int relu, const uint32_t *mask, int64_t ldm) {
  __shared__ double acc[kSumGroups][32];
  const int64_t n = M * N;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32; i0 < n;
       i0 += static_cast<int64_t>(gridDim.x) * 32) {
    const int64_t i = i0 + tx;
    double s = 0.0;
    if (i < n)
      for (int p = ty; p < splits; p += kSumGroups) s += part[p * n + i];
    acc[ty][tx] = s;
    __syncthreads();
    if (ty == 0 && i < n) {
      s = 0.0;
#pragma unroll
      for (int q = 0; q < kSumGroups; ++q) s += acc[q][tx];
      const int64_t m = i / N, c = i % N;
      float v = alpha * static_cast<float>(s);
      if (beta != 0.0f) v = fmaf(beta, C[m * ldc + c], v);
      if (relu) v = fmaxf(v, 0.0f);
      if (mask && !relu_bit(mask, ldm, m, c)) v = 0.0f;
      C[m * ldc + c] = v;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- host side --
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2-D fp32 tensor map: inner dim `inner` (contiguous), outer dim `outer` with
// row stride ld (elements); box {32, box_outer}, 128-byte swizzle (32-byte
// atoms for MN-major operands), OOB -> 0.
int make_map(CUtensorMap *m, const float *base, int64_t inner, int64_t outer, int64_t ld,
             int box_outer, bool mn) {
  EncodeFn enc = encode_fn();
  if (!enc) return fail(AG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  // MN-major: box {32 (mn), BK (k)}; K-major: box {BK (k), box_outer rows}
  cuuint32_t box[2] = {static_cast<cuuint32_t>(mn ? 32 : BK), static_cast<cuuint32_t>(box_outer)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims,
                   strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                      : (BK == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(AG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return AG_OK;
}

template <int BN, bool A_MN, bool B_MN, bool ONE, int CL, bool P2 = false>
int launch_tc(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mbl,
              const CUtensorMap &mc, TcArgs g, cudaStream_t st) {
  using C = Cfg<BN, ONE, P2>;
  auto k = tc_gemm_kernel<BN, A_MN, B_MN, ONE, CL, P2>;
  AG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  const int64_t msup = (g.m_tiles + CL - 1) / CL;
  const int64_t total = msup * g.n_tiles * g.splits;
  const int grid = static_cast<int>(std::min<int64_t>(total, sm_count() / CL)) * CL;
  if (CL == 1) {
    k<<<grid, kThreads, C::SMEM, st>>>(ma, mb, mbl, mc, g);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    AG_CUDA(cudaLaunchKernelEx(&cfg, k, ma, mb, mbl, mc, g));
  }
  AG_LAUNCH_CHECK("tc_gemm_kernel");
  return AG_OK;
}

template <int BN, bool ONE, int CL>
int launch_bn1(bool a_mn, bool b_mn, const CUtensorMap &ma, const CUtensorMap &mb,
               const CUtensorMap &mbl, const CUtensorMap &mc, const TcArgs &g, cudaStream_t st) {
  if (!a_mn && b_mn) return launch_tc<BN, false, true, ONE, CL>(ma, mb, mbl, mc, g, st);
  if (!a_mn && !b_mn) return launch_tc<BN, false, false, ONE, CL>(ma, mb, mbl, mc, g, st);
  if (a_mn && b_mn) return launch_tc<BN, true, true, ONE, CL>(ma, mb, mbl, mc, g, st);
  return launch_tc<BN, true, false, ONE, CL>(ma, mb, mbl, mc, g, st);
}
// 2-SM pairs (cta_group::2, M = 256 per MMA, each CTA holding half of B):
// 256-wide tiles only
int launch_2sm(bool a_mn, bool b_mn, bool one, const CUtensorMap &ma, const CUtensorMap &mb,
               const CUtensorMap &mbl, const CUtensorMap &mc, const TcArgs &g, cudaStream_t st) {
  if (one) {
    if (!a_mn && b_mn) return launch_tc<256, false, true, true, 2, true>(ma, mb, mbl, mc, g, st);
    if (!a_mn && !b_mn) return launch_tc<256, false, false, true, 2, true>(ma, mb, mbl, mc, g, st);
    if (a_mn && b_mn) return launch_tc<256, true, true, true, 2, true>(ma, mb, mbl, mc, g, st);
    return launch_tc<256, true, false, true, 2, true>(ma, mb, mbl, mc, g, st);
  }
  if (!a_mn && b_mn) return launch_tc<256, false, true, false, 2, true>(ma, mb, mbl, mc, g, st);
  if (!a_mn && !b_mn) return launch_tc<256, false, false, false, 2, true>(ma, mb, mbl, mc, g, st);
  if (a_mn && b_mn) return launch_tc<256, true, true, false, 2, true>(ma, mb, mbl, mc, g, st);
  return launch_tc<256, true, false, false, 2, true>(ma, mb, mbl, mc, g, st);
}

template <int BN>
int launch_bn(bool a_mn, bool b_mn, const CUtensorMap &ma, const CUtensorMap &mb,
              const CUtensorMap &mbl, const CUtensorMap &mc, const TcArgs &g, int cl,
              cudaStream_t st) {
  // one shared accumulator for 256-wide row-tile products (two would fill
  // TMEM and leave the epilogue un-overlapped: measured 2.0 -> 1.65 ms for
  // V x 256 x 256, 2.6 -> 1.4 ms for the masked V x 48 x 256 dH); the split-K
  // dW products (M-major A) keep two; AG_TC_ONEACC=0/1 overrides
  const char *e = std::getenv("AG_TC_ONEACC");
  const bool one = e ? std::atoi(e) != 0 : (BN == 256 && !a_mn);
  if constexpr (BN >= 64) {
    if (cl == 2) {
      return one ? launch_bn1<BN, true, 2>(a_mn, b_mn, ma, mb, mbl, mc, g, st)
                 : launch_bn1<BN, false, 2>(a_mn, b_mn, ma, mb, mbl, mc, g, st);
    }
  }
  return one ? launch_bn1<BN, true, 1>(a_mn, b_mn, ma, mb, mbl, mc, g, st)
             : launch_bn1<BN, false, 1>(a_mn, b_mn, ma, mb, mbl, mc, g, st);
}

__global__ void tf32_split_lo_kernel(int64_t n, const float *src, float *lo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = src[i];
    lo[i] = __fsub_rn(v, __uint_as_float(__float_as_uint(v) & 0xFFFFE000u));
  }
}

}  // namespace
}  // namespace ag

using namespace ag;

extern "C" int ag_tf32_split_lo(int64_t n, const float *src, float *lo, void *stream) {
  if (n < 0) return fail(AG_ERR_VALUE, "negative size");
  if (n == 0) return AG_OK;
  tf32_split_lo_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, src, lo);
  AG_LAUNCH_CHECK("tf32_split_lo_kernel");
  return AG_OK;
}

namespace ag {
namespace {
// bdiag > 0: block-diagonal product C[m] = A[m][0:K] @ B[(m / bdiag) * bdiag + k] with B
// (N-major, not transposed) holding b_rows rows
int gemm_tc(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda, int32_t trans_a,
            const float *B, int64_t ldb, int32_t trans_b, const float *B_lo, float *C,
            int64_t ldc, float alpha, float beta, int32_t epilogue, const uint32_t *mask,
            int64_t ldm, uint32_t *mask_out, int64_t ldmo, int64_t bdiag, int64_t b_rows,
            void *stream) {
  if (M < 0 || N < 0 || K < 0) return fail(AG_ERR_VALUE, "negative GEMM sizes");
  if (M == 0 || N == 0) return AG_OK;
  const bool a_mn = trans_a != 0;  // A stored [K][M]
  const bool b_mn = trans_b == 0;  // B stored [K][N]
  auto al16 = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(A) || !al16(B) || (B_lo && !al16(B_lo)) || (lda % 4) || (ldb % 4))
    return fail(AG_ERR_VALUE, "tensor-core GEMM needs 16-byte aligned operands and row strides");
  if (M > 2147483647LL || N > 2147483647LL || K > 2147483647LL)
    return fail(AG_ERR_VALUE, "GEMM dimension too large");
  cudaStream_t st = as_stream(stream);
  if (K == 0) {  // C = beta * C (relu)
    return fail(AG_ERR_VALUE, "K == 0 is not supported by the tensor-core GEMM");
  }
  // N tile: the whole N when it fits one MMA (<= 256), padded to 16
  int bn = static_cast<int>(std::min<int64_t>(256, ((N + 15) / 16) * 16));
  bn = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
  // (256-wide tiles share one TMEM accumulator, so they double-buffer too and
  // the epilogue overlaps the next tile's MMAs at any K)
  if (const char *e = std::getenv("AG_TC_BN")) bn = std::min(bn, std::max(32, std::atoi(e)));
  TcArgs g{};
  g.M = M; g.N = N; g.K = K;
  g.alpha = alpha; g.beta = beta; g.relu = (epilogue & AG_GEMM_RELU) ? 1 : 0;
  g.mask = mask;
  g.ldm = ldm;
  g.mask_out = mask_out;
  g.ldmo = ldmo;
  if (mask_out != nullptr && ldmo < relu_words(N))
    return fail(AG_ERR_VALUE, "mask_out row stride must be >= ceil(N / 32) words");
  if (mask != nullptr && ldm < relu_words(N))
    return fail(AG_ERR_VALUE, "mask row stride must be >= ceil(N / 32) words");
  g.b_presplit = B_lo != nullptr;
  g.bdiag = bdiag;
  if (const char *e = std::getenv("AG_TC_EXP")) g.exp = std::atoi(e);
  {
    // raw hi by default: the MMA reads only an fp32 operand's top 19 bits, so
    // the splitters need not write the masked hi half back (a third less
    // shared-memory traffic in the split; bitwise equal, tests/test_slab_gpu.py)
    const char *rh = std::getenv("AG_TC_RAWHI");
    g.raw_hi = rh ? std::atoi(rh) : 1;
  }
  g.m_tiles = static_cast<int>((M + BM - 1) / BM);
  g.n_tiles = static_cast<int>((N + bn - 1) / bn);
  const int64_t tiles = static_cast<int64_t>(g.m_tiles) * g.n_tiles;
  const int sms = sm_count();
  int splits = 1;
  const int64_t kblocks = (K + BK - 1) / BK;
  if (tiles < sms / 2 && kblocks >= 16 && bdiag == 0) {  // skinny-output product (dW): split K
    splits = static_cast<int>(std::min<int64_t>(std::max<int64_t>(1, sms / tiles), kblocks / 8));
  }
  int64_t kb_per = (kblocks + splits - 1) / splits;
  g.split_mode = splits > 1 ? 1 : 0;
  if (splits > 1 && kb_per > kChunkKb) {
    // long K per split: chunk it (split_mode 2)
    if (const char *e = std::getenv("AG_TC_CHUNK_BN")) {  // development: narrower tiles
      bn = std::min(bn, std::max(32, std::atoi(e)));
      g.n_tiles = static_cast<int>((N + bn - 1) / bn);
    }
    int64_t chunk = kChunkKb;
    if (const char *e = std::getenv("AG_TC_CHUNK_KB")) chunk = std::max(8, std::atoi(e));
    // as many chunks as needed, rounded up to a multiple of the CTAs per
    // output tile so every persistent CTA gets the same number of chunks
    const int64_t per_tile = std::max<int64_t>(1, sms / (static_cast<int64_t>(g.m_tiles) * g.n_tiles));
    int64_t nsp = (kblocks + chunk - 1) / chunk;
    nsp = (nsp + per_tile - 1) / per_tile * per_tile;
    kb_per = (kblocks + nsp - 1) / nsp;
    g.split_mode = 2;
  }
  g.k_per_split = kb_per * BK;
  splits = static_cast<int>((kblocks + kb_per - 1) / kb_per);
  g.splits = splits;
  if (tiles * splits > 2147483647LL) return fail(AG_ERR_VALUE, "GEMM has too many tiles");
  // clusters of 2 CTAs share (multicast) every B k-block
  // (not for the M-major, split-K dW products: measured slower there)
  int cl = (bn >= 64 && g.m_tiles >= 2 && !a_mn) ? 2 : 1;
  if (const char *e = std::getenv("AG_TC_CL")) cl = std::atoi(e) == 2 && bn >= 64 ? 2 : 1;
  if (bdiag) cl = 1;  // neighbouring tiles read different B panels: no multicast
  // 2-SM pairs for 256-wide tiles (AG_TC_2SM=1; development until measured)
  const char *e2 = std::getenv("AG_TC_2SM");
  const bool p2 = bn == 256 && bdiag == 0 && g.m_tiles >= 2 && e2 && std::atoi(e2) == 1;
  if (p2) cl = 2;
  CUtensorMap ma, mb;
  int rc;
  // A: K-major [M][K] (inner K) or M-major [K][M] (inner M)
  if (a_mn) rc = make_map(&ma, A, M, K, lda, BK, true);
  else rc = make_map(&ma, A, K, M, lda, BM, false);
  if (rc) return rc;
  if (b_mn) rc = make_map(&mb, B, N, bdiag ? b_rows : K, ldb, BK, true);
  else rc = make_map(&mb, B, K, N, ldb, bn / cl, false);  // (p2: cl = 2, each CTA's half)
  if (rc) return rc;
  CUtensorMap mbl = mb;
  if (B_lo) {
    if (b_mn) rc = make_map(&mbl, B_lo, N, K, ldb, BK, true);
    else rc = make_map(&mbl, B_lo, K, N, ldb, bn / cl, false);
    if (rc) return rc;
  }
  Scratch ws;
  int nparts = splits;
  if (g.split_mode == 2) {
    // one zeroed slot per CTA of the persistent grid (launch_tc's grid)
    const int64_t msup = (g.m_tiles + cl - 1) / cl;
    const int64_t total = msup * g.n_tiles * static_cast<int64_t>(splits);
    nparts = static_cast<int>(std::min<int64_t>(total, sms / cl)) * cl;
    AG_CUDA(ws.alloc(static_cast<size_t>(nparts) * M * N * sizeof(float), st));
    AG_CUDA(cudaMemsetAsync(ws.ptr, 0, static_cast<size_t>(nparts) * M * N * sizeof(float), st));
    g.C = ws.as<float>();
    g.ldc = N;
  } else if (splits > 1) {
    AG_CUDA(ws.alloc(static_cast<size_t>(splits) * M * N * sizeof(float), st));
    g.C = ws.as<float>();
    g.ldc = N;
  } else {
    g.C = C;
    g.ldc = ldc;
  }
  // C as a TMA tensor (box 32 x 32, 128-byte swizzle = the epilogue's staging
  // layout) for direct products: the epilogue stores its chunks by TMA
  CUtensorMap mc = mb;
  g.c_tma = 0;
  if (g.split_mode == 0 && splits == 1 && (reinterpret_cast<uintptr_t>(C) & 15) == 0 &&
      ldc % 4 == 0 && std::getenv("AG_TC_NO_CTMA") == nullptr) {
    EncodeFn enc = encode_fn();
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldc) * 4};
    cuuint32_t box[2] = {32, 32};
    cuuint32_t es[2] = {1, 1};
    if (enc && enc(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      g.c_tma = 1;
  }
  long long *trace = nullptr;
  if (std::getenv("AG_TC_TRACE")) {
    AG_CUDA(cudaMalloc(&trace, kTraceTiles * 10 * sizeof(long long)));
    AG_CUDA(cudaMemset(trace, 0, kTraceTiles * 10 * sizeof(long long)));
    g.trace = trace;
  }
  if (p2) {
    const char *eo = std::getenv("AG_TC_ONEACC");
    rc = launch_2sm(a_mn, b_mn, eo ? std::atoi(eo) != 0 : !a_mn, ma, mb, mbl, mc, g, st);
  } else switch (bn) {
    case 32: rc = launch_bn<32>(a_mn, b_mn, ma, mb, mbl, mc, g, cl, st); break;
    case 64: rc = launch_bn<64>(a_mn, b_mn, ma, mb, mbl, mc, g, cl, st); break;
    case 128: rc = launch_bn<128>(a_mn, b_mn, ma, mb, mbl, mc, g, cl, st); break;
    default: rc = launch_bn<256>(a_mn, b_mn, ma, mb, mbl, mc, g, cl, st); break;
  }
  if (rc) return rc;
  if (trace) {
    long long h[kTraceTiles * 10];
    AG_CUDA(cudaStreamSynchronize(st));
    AG_CUDA(cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost));
    cudaFree(trace);
    const long long t0 = h[0];
    std::fprintf(stderr, "tc_gemm trace M=%lld N=%lld K=%lld bn=%d (us from first stamp)\n",
                 (long long)M, (long long)N, (long long)K, bn);
    for (int i = 0; i < kTraceTiles; ++i) {
      if (!h[i * 10]) break;
      std::fprintf(stderr, "tile %2d mma: tempty %.2f..%.2f conv0 %.2f..%.2f conv1 %.2f..%.2f last %.2f"
                   " | epi: tfull %.2f..%.2f done %.2f\n", i,
                   (h[i*10+0]-t0)/1e3, (h[i*10+1]-t0)/1e3, (h[i*10+6]-t0)/1e3, (h[i*10+7]-t0)/1e3,
                   (h[i*10+8]-t0)/1e3, (h[i*10+9]-t0)/1e3, (h[i*10+2]-t0)/1e3,
                   (h[i*10+3]-t0)/1e3, (h[i*10+4]-t0)/1e3, (h[i*10+5]-t0)/1e3);
    }
  }
  if (splits > 1) {
    splitk_sum_kernel<<<grid_for((M * N + 31) / 32, 1), 32 * kSumGroups, 0, st>>>(M, N, nparts, g.C, C, ldc, alpha,
                                                            beta, g.relu, mask, ldm);
    AG_LAUNCH_CHECK("splitk_sum_kernel");
    if (mask_out != nullptr) {
      rc = ag_relu_bits(M, N, C, ldc, mask_out, ldmo, stream);
      if (rc) return rc;
    }
  }
  return AG_OK;
}
}  // namespace
}  // namespace ag

extern "C" int ag_gemm_tf32x3(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                              int32_t trans_a, const float *B, int64_t ldb, int32_t trans_b,
                              const float *B_lo, float *C, int64_t ldc, float alpha, float beta,
                              int32_t epilogue, const uint32_t *mask, int64_t ldm,
                              uint32_t *mask_out, int64_t ldmo, void *stream) {
  return gemm_tc(M, N, K, A, lda, trans_a, B, ldb, trans_b, B_lo, C, ldc, alpha, beta, epilogue,
                 mask, ldm, mask_out, ldmo, 0, 0, stream);
}

extern "C" int ag_block_diag_gemm_tf32x3(int64_t num_rows, int64_t feat, int64_t panel,
                                         const float *A, int64_t lda, const float *x,
                                         int64_t ldx, int64_t x_rows, float *y, int64_t ldy,
                                         float beta, void *stream) {
  if (num_rows < 0 || feat < 0 || x_rows < 0) return fail(AG_ERR_VALUE, "negative sizes");
  if (panel < 128 || panel % 128 != 0 || panel > 4096)
    return fail(AG_ERR_VALUE, "panel must be a multiple of 128 in [128, 4096]");
  if (lda < panel) return fail(AG_ERR_VALUE, "lda must be >= panel");
  if (num_rows == 0 || feat == 0) return AG_OK;
  return gemm_tc(num_rows, feat, panel, A, lda, 0, x, ldx, 0, nullptr, y, ldy, 1.0f, beta, 0,
                 nullptr, 0, nullptr, 0, panel, x_rows, stream);
}
