/*
 * adaptgear_b200.h -- C ABI of the B200-native AdaptGear aggregation path.
 *
 * Everything below is `extern "C"`, takes plain pointers + sizes and an opaque
 * `void *stream` (a cudaStream_t; NULL = legacy default stream).  Pointers are
 * DEVICE pointers unless the name ends in `_host`.  Outputs are caller-allocated
 * unless stated otherwise.  Every entry point returns an AG_* status; on failure
 * ag_last_error() returns a thread-local message that the Python shim maps onto
 * the reference's exception types (ValueError / KernelError / RuntimeError).
 *
 * Reference interface each group replaces (paths relative to
 * /root/reference/pkg/src/adaptgear/):
 *   preprocessing  graph.py:47-82 (Graph.from_edges), models.py:57-73
 *                  (gcn_normalize), reorder.py:92-228 (cluster_bfs,
 *                  load_partition, apply_reorder), decompose.py:57-75,
 *                  formats.py:76-140 (to_csr / to_coo / to_dense_blocks)
 *   kernels        kernels.py:117-134 (aggregate_csr_inter),
 *                  kernels.py:137-189 (aggregate_csr_intra_blocked),
 *                  kernels.py:192-225 (aggregate_coo_atomic),
 *                  kernels.py:228-250 (aggregate_dense_block),
 *                  kernels.py:253-276 (combine), kernels.py:309-313 (backward_sum)
 *   layers         models.py:86-112 (gcn/gin_layer_forward: agg @ W)
 */
#ifndef ADAPTGEAR_B200_H
#define ADAPTGEAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (ag_last_error() holds the message) ------------------- */
#define AG_OK 0
#define AG_ERR_VALUE 1  /* -> ValueError  (bad sizes / ids / block_size)     */
#define AG_ERR_KERNEL 2 /* -> KernelError (kernel preconditions)            */
#define AG_ERR_CUDA 3   /* -> RuntimeError (CUDA runtime failure)           */

/* ---- aggregation operators: kernels.py:42-45 AggregateOp ----------------- */
#define AG_OP_SUM 0
#define AG_OP_MEAN 1
#define AG_OP_MAX 2

/* ---- epilogue flags of the aggregation kernels -------------------------- */
/* AG_EPI_COMBINE: y already holds the OTHER role's partial (inter values, or
 *   zeros for an empty partial); the kernel writes combine(this, other)
 *   exactly as kernels.py:253-276 does (sum: a+b; mean: (a+b)/f32(max(deg,1));
 *   max: touched-aware).  Without it the kernel stores the raw partial (rows
 *   with no edges get 0, kernels.py:123).
 * AG_EPI_GIN: additionally y = f32(gin_scale) * x + y  (models.py:111).
 * AG_EPI_EMPTY_OTHER (with COMBINE, ag_fused_spmm only): the other partial is
 *   the empty one (zeros, untouched) -- combine(partial, empty_partial) of
 *   aggregate_full (kernels.py:355-362) without reading y. */
#define AG_EPI_COMBINE 1
#define AG_EPI_GIN 2
#define AG_EPI_EMPTY_OTHER 4
/* Bit-packed ReLU masks ("relu bits"): for a [rows][feat] activation h, row r
 * is ldw >= ceil(feat / 32) uint32 words and bit (c % 32) of word c / 32 is
 * (h[r][c] > 0).  The forward epilogues that apply a ReLU can write them
 * (ag_gemm_* mask_out, ag_fused_spmm relu_out with AG_EPI_RELU), the backward
 * epilogues read them -- 1/32 of the bytes of re-reading h to test its sign.
 * ag_relu_bits builds them from an fp32 activation. */
int ag_relu_bits(int64_t num_rows, int64_t feat, const float *h, int64_t ld,
                 uint32_t *bits, int64_t ldw, void *stream);
/* AG_EPI_RELU_MASK (ag_fused_spmm only): after everything else,
 * y = bit ? y : 0 from relu_bits (row stride ceil(feat / 32) words) -- the
 * ReLU backward of the layer below (its output's mask), fused into the
 * transposed aggregation. */
#define AG_EPI_RELU_MASK 8
/* AG_EPI_RELU (ag_fused_spmm only): y = max(y, 0) after everything else --
 * the hidden layers' activation when the update GEMM runs before the
 * aggregation (A (H W) for a narrowing layer); with relu_out non-NULL the
 * kernel also writes y's relu bits (row stride ceil(feat / 32) words). */
#define AG_EPI_RELU 16
/* AG_EPI_INTER_COO (ag_fused_spmm, role_mask 3, op sum only): the inter role
 * is the selector's coo_atomic kernel (kernels.py:192-225), whose summation
 * order the reference leaves open (fp64 bincount over scrambled edges, tested
 * at 1e-4): the inter edges of a row are accumulated with fused fp32
 * multiply-adds in any order instead of the reduceat order.  The intra role
 * keeps its own kernel's semantics (bitwise csr_intra_blocked, or dense_block
 * with blk_w) -- the selector pairs (csr_intra_blocked | dense_block,
 * coo_atomic) in one pass. */
#define AG_EPI_INTER_COO 32

int ag_abi_version(void);
const char *ag_last_error(void);
/* Number of SMs of the current device (0 when no device is present). */
int ag_device_sm_count(void);
/* Kernels this library has launched since load (process-wide counter). */
uint64_t ag_launch_count(void);

/* ======================= preprocessing (device) ========================== */

/* Graph.from_edges (graph.py:47-82): validate endpoints against [0, V),
 * sort by key dst*V+src, drop duplicates, sum duplicate weights in fp64 in
 * input order and round to fp32.  dst/src are int64[E]; w may be NULL.
 * Outputs must hold E entries; *num_out_host receives the unique count. */
int ag_canonicalize(int64_t num_vertices, int64_t num_edges, const int64_t *dst,
                    const int64_t *src, const float *w, int32_t *dst_out,
                    int32_t *src_out, float *w_out, int64_t *num_out_host,
                    void *stream);

/* apply_reorder relabel step (reorder.py:217-228): out = perm[in] as int64. */
int ag_relabel(int64_t num_edges, const int64_t *perm, const int32_t *dst,
               const int32_t *src, int64_t *dst_out, int64_t *src_out,
               void *stream);

/* gcn_normalize (models.py:57-73) on a canonical graph: binary union with
 * self loops, in-degree of A+I, w = f32(1/sqrt(f64(deg[d])*f64(deg[s]))).
 * Outputs must hold E+V entries. */
int ag_gcn_normalize(int64_t num_vertices, int64_t num_edges,
                     const int32_t *dst, const int32_t *src, int32_t *dst_out,
                     int32_t *src_out, float *w_out, int64_t *num_out_host,
                     void *stream);

/* in_degrees (graph.py:94-96): int64 histogram of dst. */
int ag_in_degrees(int64_t num_vertices, int64_t num_edges, const int32_t *dst,
                  int64_t *deg_out, void *stream);

/* decompose (decompose.py:57-75), two phases: count intra edges, then split
 * order-preservingly (a canonical input stays canonical).  w may be NULL. */
int ag_decompose_count(int64_t num_edges, const int32_t *dst,
                       const int32_t *src, int64_t block_size,
                       int64_t *num_intra_host, void *stream);
int ag_decompose_split(int64_t num_edges, const int32_t *dst,
                       const int32_t *src, const float *w, int64_t block_size,
                       int32_t *intra_dst, int32_t *intra_src, float *intra_w,
                       int32_t *inter_dst, int32_t *inter_src, float *inter_w,
                       void *stream);

/* to_csr (formats.py:76-88): row_ptr[V+1] from canonical (sorted) dst. */
int ag_build_row_ptr(int64_t num_vertices, int64_t num_edges,
                     const int32_t *dst, int32_t *row_ptr, void *stream);

/* touched = rowlen > 0 (kernels.py:121). */
int ag_row_touched(int64_t num_rows, const int32_t *row_ptr, uint8_t *touched,
                   void *stream);

/* First edge index whose endpoints are in different B-blocks, or -1
 * (formats.py:115-123, kernels.py:154-161).  Uses CSR arrays only. */
int ag_first_off_block(int64_t num_rows, const int32_t *row_ptr,
                       const int32_t *col_idx, int64_t block_size,
                       int64_t *first_bad_host, void *stream);

/* to_dense_blocks (formats.py:105-140), two phases.  count: number k of
 * B-blocks holding >= 1 edge.  fill: community_ids[k] (ascending),
 * comm_slot[ceil(V/B)] (slot or -1), blocks[k*B*B] (zero-filled here),
 * row_touched[k*B].  Edges must be block-local (checked by the caller). */
int ag_blocks_count(int64_t num_vertices, int64_t num_edges,
                    const int32_t *dst, int64_t block_size, int64_t *k_host,
                    void *stream);
int ag_blocks_fill(int64_t num_vertices, int64_t num_edges, const int32_t *dst,
                   const int32_t *src, const float *w, int64_t block_size,
                   int64_t k, int32_t *community_ids, int32_t *comm_slot,
                   float *blocks, uint8_t *row_touched, void *stream);

/* ================== aggregation kernels (the hot path) =================== */

/* K1 aggregate_csr_inter (kernels.py:87-134).  Y[r] = sum_e val[e]*X[col[e]]
 * reduced in EXACTLY numpy's np.add.reduceat order (first term + pairwise
 * 8-accumulator blocked sum, block 128) so values are bitwise equal to the
 * reference; max reduces raw X rows.  val may be NULL (implicit 1.0).
 * x, y: fp32 [V, F] row-major.  See AG_EPI_* for the epilogue. */
int ag_csr_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                const int32_t *col_idx, const float *val, const float *x,
                float *y, int32_t op, int32_t epi_flags,
                const uint8_t *other_touched, const int64_t *deg,
                float gin_scale, void *stream);

/* K2 aggregate_csr_intra_blocked (kernels.py:137-189): one CTA per B-row
 * community; the community's B x F_tile source slab is staged in shared
 * memory once and every row of the block gathers from it.  F is tiled so
 * that B*F_tile*4 <= tile_budget_bytes (kernels.py:169-171).  Values are
 * bitwise identical to ag_csr_spmm. */
int ag_csr_intra_spmm(int64_t num_rows, int64_t feat, int64_t block_size,
                      int64_t tile_budget_bytes, const int32_t *row_ptr,
                      const int32_t *col_idx, const float *val, const float *x,
                      float *y, int32_t op, int32_t epi_flags,
                      const uint8_t *other_touched, const int64_t *deg,
                      float gin_scale, void *stream);

/* K3 aggregate_coo_atomic (kernels.py:192-225): edge-parallel over a
 * (row, col)-sorted COO; warps fold runs of equal rows in registers and
 * flush with vector atomics.  ACCUMULATES into y: the caller initialises
 * y to 0 (sum/mean) or -inf (max). */
int ag_coo_spmm(int64_t num_rows, int64_t feat, int64_t num_edges,
                const int32_t *row, const int32_t *col, const float *val,
                const float *x, float *y, int32_t op, void *stream);
/* coo_atomic (kernels.py:192-225) for sum / mean partials as a row gather:
 * the COO is dst-sorted, so row_ptr[num_rows + 1] (ag_build_row_ptr of its
 * rows) delimits each destination's edge run; a sub-warp per row gathers the
 * sources (8 loads in flight) and writes y[r] = sum of val * x[col] in an
 * unspecified order (the reference's order is open too; tested at 1e-4), with
 * no atomics.  y rows without edges are written 0.  val NULL: weights 1.0. */
int ag_coo_gather_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                       const int32_t *col, const float *val, const float *x, float *y,
                       void *stream);
/* The (dense_block, coo_atomic) selector pair on a small graph (features that
 * fit L2) as ONE order-free row gather over the full CSR (both roles' edges),
 * with ag_fused_spmm's epilogues: y = sum [+ gin_scale * x] [relu, bits to
 * relu_out] [* relu_bits].  feat % 4 == 0, x / y 16-byte aligned, row stride
 * feat; relu masks [rows][ceil(feat / 32)] words.  Order-free like the pair
 * (kernels.py:228-250 matmul, :192-225 scrambled bincount; tested at 1e-5). */
int ag_gather_pair_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                        const int32_t *col, const float *val, const float *x, float *y,
                        int32_t epi_flags, float gin_scale, const uint32_t *relu_bits,
                        uint32_t *relu_out, void *stream);

/* K4 aggregate_dense_block (kernels.py:228-250): for every B-row community c
 * with slot k = comm_slot[c] >= 0: Y[cB:cB+B] = blocks[k] @ X[cB:cB+B]
 * (ragged last block zero-padded).  Communities without a block produce an
 * untouched (zero) partial.  Rejects max (kernels.py:234-235). */
int ag_dense_block_spmm(int64_t num_rows, int64_t feat, int64_t block_size,
                        const int32_t *comm_slot, const float *blocks,
                        const uint8_t *row_touched, const float *x, float *y,
                        int32_t op, int32_t epi_flags,
                        const uint8_t *other_touched, const int64_t *deg,
                        float gin_scale, void *stream);

/* Tensor-core dense_block (K4 on tcgen05): the DenseBlockSet as
 * block-diagonal panels of width panel = max(block_size, 128) (block_size
 * divides 128 -- 8 blocks of 16 share a 128 x 128 panel, zeros off their
 * diagonal -- or is a multiple of 128), A[num_rows][lda]; then
 *   y[r] = A[r][0:panel] @ x[(r / panel) * panel + k]  (+ beta * y[r])
 * with kind::tf32 3xTF32 (fp32-faithful: ~1e-7 of the sum of |terms|; the
 * reference's BLAS matmul order is unpinned anyway, kernels.py:247).  beta 1
 * accumulates onto an inter partial already in y (combine(sum)). */
int ag_dense_block_pack(int64_t num_rows, int64_t block_size, int64_t panel,
                        const int32_t *comm_slot, const float *blocks, float *A,
                        int64_t lda, void *stream);
int ag_block_diag_gemm_tf32x3(int64_t num_rows, int64_t feat, int64_t panel,
                              const float *A, int64_t lda, const float *x, int64_t ldx,
                              int64_t x_rows, float *y, int64_t ldy, float beta,
                              void *stream);

/* Role-ordered CSR of the fused kernel, built once per (topology, B):
 * every row's edges re-listed as its intra run (cols in [floor(r/B)B, +B),
 * ascending) followed by its inter edges (the sorted row's prefix ++ suffix,
 * ascending) -- the two operand lists of the reference's intra / inter CSR
 * kernels (decompose.py:63, kernels.py:117-189).  role_col / role_val hold E
 * entries (role_val may be NULL iff val is NULL); role_mid[r] = row_ptr[r] +
 * (intra edges of row r). */
int ag_role_csr_build(int64_t num_rows, const int32_t *row_ptr,
                      const int32_t *col_idx, const float *val,
                      int64_t block_size, int32_t *role_col, float *role_val,
                      int32_t *role_mid, void *stream);

/* Fused decomposed aggregation (one launch).  For every row r,
 *   I = intra-role value over edges [row_ptr[r], role_mid[r])
 *   O = inter-role value over edges [role_mid[r], row_ptr[r+1])
 * each in the reference's np.add.reduceat order (bitwise), then
 *   role_mask 3: y = combine(I, O) (kernels.py:253-276)   [+ gin term]
 *   role_mask 1/2: a single role with the AG_EPI_* epilogue of ag_csr_spmm.
 * role_mid NULL: the whole row is the single role of role_mask 1 or 2 --
 * aggregate_csr_inter (kernels.py:117-134).  The edges are given by the slab
 * layout of ag_slab_codes over the role-ordered (or plain) CSR, built with
 * the same `window` and role_mid; `weighted` 0 means every weight is 1.0.
 * num_edges = row_ptr[num_rows] (balances the row ranges).  x has x_rows >=
 * num_rows rows (a rank's halo rows follow its own rows).
 * "Slab" kernel, one CTA per SM sweeping a column tile of an nnz-balanced
 * range of 16-row blocks: an X producer warp streams X into a shared-memory
 * ring holding the blocks within `window` blocks of the current one (TMA
 * tensor tiles), a far producer warp stages each block's out-of-window
 * sources (bulk copies), and 14 consumer warps take the range's rows
 * round-robin, reducing out of shared memory.  `window` only affects speed,
 * never values (ag_slab_window picks it per graph).  Any F (TMA when
 * F % 4 == 0 and x is 16-byte aligned, cp.async otherwise).
 * blk_w (NULL: bitwise intra role): the pair (dense_block, csr_inter) of the
 * reference's selector in one pass -- the intra role of every 16-row block as
 * a dense 16 x 16 block product (ag_slab_dense_blocks; the reference's
 * dense_block kernel, kernels.py:228-250, order-unpinned like its BLAS
 * matmul) computed once per block by a dedicated warp, the inter role bitwise;
 * needs role_mask 3, op sum and the B = 16 role-ordered layout. */
int ag_fused_spmm(int64_t num_rows, int64_t feat, int32_t role_mask,
                  const int32_t *row_ptr, const int32_t *role_mid,
                  const int32_t *cv, const int32_t *rowinfo,
                  const int32_t *far_cnt, const int32_t *far_src,
                  int32_t weighted, const float *blk_w, int64_t num_edges,
                  const float *x, float *y,
                  int32_t op, int32_t epi_flags, const uint8_t *other_touched,
                  const int64_t *deg, float gin_scale, const uint32_t *relu_bits,
                  uint32_t *relu_out, int64_t x_rows, int32_t window, void *stream);

/* Window radius (in 16-row blocks) for ag_fused_spmm over this CSR: the
 * smallest radius whose ring covers `coverage` (e.g. 0.995) of the edges the
 * largest supported radius (17) would cover, from a device histogram of
 * |src/16 - dst/16|.  Synchronous (reads the histogram back); call once per
 * topology and cache the result.  No reference counterpart: a B200 layout
 * parameter of the cached formats (formats.py:76-140). */
int ag_slab_window(int64_t num_rows, const int32_t *row_ptr,
                   const int32_t *col_idx, double coverage, int32_t *window,
                   void *stream);

/* Slab layout for ag_fused_spmm over a CSR (edges in col_idx / val order:
 * plain or role-ordered; val NULL = unweighted; role_mid NULL = no role
 * split).  cv: int32[2 * E] (8-byte aligned), pair e = (code, weight bits):
 * code = X-ring row of col_idx[e] when its 16-row block is within `window`
 * blocks of row r's block; otherwise the source is one of the block's
 * staged far sources (far_src[block * cap + j], j < cap =
 * ag_slab_far_capacity(), far_cnt[block] of them) or, past the capacity,
 * code = ~col_idx[e] (read from global memory).  rowinfo: int32[4 * V]
 * (16-byte aligned) = per row {start, intra end, end, flags}.  far_cnt:
 * int32[ceil(V / 16)], far_src: int32[that * cap]. */
int ag_slab_codes(int64_t num_rows, const int32_t *row_ptr,
                  const int32_t *col_idx, const float *val,
                  const int32_t *role_mid, int32_t window, int32_t *cv,
                  int32_t *rowinfo, int32_t *far_cnt, int32_t *far_src,
                  void *stream);
/* Dense 16 x 16 intra weights per 16-row block for ag_fused_spmm's blk_w:
 * blk_w[b][i][j] = weight of edge (16b + i <- 16b + j) from the role-ordered
 * CSR's intra runs [row_ptr[r], role_mid[r]) (role_val NULL: 1.0), zeros
 * elsewhere.  blk_w: float[ceil(num_rows / 16) * 256]. */
int ag_slab_dense_blocks(int64_t num_rows, const int32_t *row_ptr,
                         const int32_t *role_mid, const int32_t *role_col,
                         const float *role_val, float *blk_w, void *stream);
/* Staged far sources per 16-row block (the far-ring capacity). */
int ag_slab_far_capacity(void);

/* ---- band kernel: the order-free (dense_block, coo_atomic) pair ----------
 * The same selector pair as ag_fused_spmm with blk_w and AG_EPI_INTER_COO
 * (kernels.py:228-250 intra, :192-225 inter, combine :253-276), with the
 * inter topology packed per 16-row block into a RECORD that a producer warp
 * bulk-copies into an 8-deep shared-memory FIFO (no per-row global topology
 * loads in the consumers):
 *   words 0..15 : row i's end offset into the block's pairs (bits 0-19)
 *                 | nfar << 20 (the row's leading far pairs, <= 255)
 *                 | 1 << 30 if nfar > 255 (the row takes the general path)
 *                 | 1 << 31 if the block has more than ag_band_capacity()
 *                   pairs (then read from the global record, not staged)
 *   then int32 pairs (code, weight bits) of the inter edges, each row's far
 *   pairs first (role-ordered CSR [role_mid[r], row_ptr[r+1])), padded to
 *   16 bytes.  code = band-ring row ((src / 16) % 42) * 16 + src % 16 within
 *   `window` blocks, else ~src (read from global memory; far_cnt / far_src
 *   list up to ag_slab_far_capacity() of them per block for L2 prefetch).
 * ag_band_sizes: per-block record sizes in 16-byte units (int32[nb]) and the
 * largest pair count (host).  The caller scans them into rec_off
 * (int32[nb + 1], exclusive) and allocates rec (16-byte aligned,
 * rec_off[nb] * 16 bytes) for ag_band_records.  window <= ag_band_max_window().
 * ag_band_spmm: y = dense_intra(x) + coo_inter(x) [+ gin_scale * x] [relu]
 * [* relu_bits] (flags as in ag_fused_spmm: GIN, RELU (+ relu_out),
 * RELU_MASK; INTER_COO is implied); feat % 4 == 0, feat > 32, x / rec /
 * relu_bits 16-byte aligned.  Order-free like the pair it runs (tested at
 * 1e-5 against the reference pair).  An alternative to ag_fused_spmm's
 * dense + coo mode, measured slower on the C5 graph. */
int ag_band_max_window(void);
int ag_band_capacity(void);
int ag_band_sizes(int64_t num_rows, const int32_t *row_ptr, const int32_t *role_mid,
                  int32_t *sizes, int64_t *max_pairs_host, void *stream);
int ag_band_records(int64_t num_rows, const int32_t *row_ptr, const int32_t *role_col,
                    const float *role_val, const int32_t *role_mid, int32_t window,
                    const int32_t *rec_off, int32_t *rec, int32_t *far_cnt,
                    int32_t *far_src, void *stream);
int ag_band_spmm(int64_t num_rows, int64_t feat, const int32_t *row_ptr,
                 const int32_t *rec, const int32_t *rec_off, const int32_t *far_cnt,
                 const int32_t *far_src, const float *blk_w, int64_t num_edges,
                 const float *x, float *y, int32_t epi_flags, float gin_scale,
                 const uint32_t *relu_bits, uint32_t *relu_out, int64_t x_rows,
                 int32_t window, void *stream);

/* K5 combine (kernels.py:253-276) as a standalone pass. out may alias a. */
int ag_combine(int64_t num_rows, int64_t feat, const float *a,
               const uint8_t *touched_a, const float *b,
               const uint8_t *touched_b, const int64_t *deg, int32_t op,
               float *out, void *stream);

/* ======================== dense update (K7) ============================== */

/* C = alpha * op(A) @ op(B) + beta * C, fp32 row-major, optional ReLU on
 * the result (epilogue 1).  op(A) is [M,K], op(B) is [K,N]. */
#define AG_GEMM_RELU 1
/* mask (relu bits, may be NULL; ldm in words): after the epilogue,
 * C[m][n] = bit(m, n) ? C[m][n] : 0 -- the ReLU backward of the layer below
 * (its output's mask), fused into dH = G W^T.  mask_out (may be NULL; ldmo in
 * words): the relu bits of the final C (the forward ReLU's mask). */
int ag_gemm_f32(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                int32_t trans_a, const float *B, int64_t ldb, int32_t trans_b,
                float *C, int64_t ldc, float alpha, float beta,
                int32_t epilogue, const uint32_t *mask, int64_t ldm,
                uint32_t *mask_out, int64_t ldmo, void *stream);

/* The same GEMM on the tensor cores: tcgen05.mma kind::tf32 with TMA-fed,
 * 128-byte-swizzled shared-memory operands, TMEM accumulators and 3xTF32
 * operand splitting (hi*hi + hi*lo + lo*hi, fp32 accumulation) -- fp32-faithful
 * to a few ulp.  Needs 16-byte aligned A, B and lda, ldb multiples of 4 and
 * K >= 1; any M, N, K otherwise (TMA zero-fills the ragged edges).  Skinny
 * outputs (dW = H^T G, K = V) are split over K with a deterministic fixed-order
 * reduction. */
int ag_gemm_tf32x3(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                   int32_t trans_a, const float *B, int64_t ldb, int32_t trans_b,
                   const float *B_lo, float *C, int64_t ldc, float alpha, float beta,
                   int32_t epilogue, const uint32_t *mask, int64_t ldm,
                   uint32_t *mask_out, int64_t ldmo, void *stream);

/* lo[i] = src[i] - tf32_truncate(src[i]) (exact): the low half of the 3xTF32
 * split, precomputed for a small B operand that every output tile re-reads
 * (the layer weights); pass it as ag_gemm_tf32x3's B_lo (NULL: split in
 * shared memory).  src / lo share the layout. */
int ag_tf32_split_lo(int64_t n, const float *src, float *lo, void *stream);

/* ===================== training helpers (composed) ======================= */

/* Mean softmax cross-entropy over rows with mask[r] != 0 (mask may be NULL =
 * all rows).  logits / dlogits are [num_rows] x [num_classes] with row stride
 * ld >= num_classes; dlogits has its own row stride ld_dlogits >= num_classes.
 * Writes the loss (fp32 scalar, device; per-CTA fp64 partials summed in a
 * fixed order) and dlogits = (softmax - onehot) / n_masked (0 for unmasked
 * rows; columns [num_classes, ld_dlogits) are written as 0). */
int ag_softmax_xent(int64_t num_rows, int64_t num_classes, int64_t ld,
                    const float *logits, const int32_t *labels,
                    const uint8_t *mask, int64_t num_masked, float *loss_out,
                    float *dlogits, int64_t ld_dlogits, void *stream);
/* g = g * (h > 0) in place (ReLU backward). */
int ag_relu_backward(int64_t n, const float *h, float *g, void *stream);
/* w -= lr * dw. */
int ag_sgd_step(int64_t n, float *w, const float *dw, float lr, void *stream);

/* ====================== host-side preprocessing ========================== */

/* cluster_bfs (reorder.py:92-153) bit-exact, sequential, HOST arrays.
 * dst_host/src_host: canonical int32 edges.  Outputs int64[V]. */
int ag_cluster_bfs(int64_t num_vertices, int64_t num_edges,
                   const int32_t *dst_host, const int32_t *src_host,
                   int64_t comm_size, int64_t *community_out_host,
                   int64_t *permutation_out_host);

/* load_partition core (reorder.py:156-203): stable sort of community ids,
 * chunking into <= comm_size runs, renumbering.  HOST arrays. */
int ag_partition_from_ids(int64_t num_vertices, const int64_t *ids_host,
                          int64_t comm_size, int64_t *community_out_host,
                          int64_t *permutation_out_host);

/* ====================== synthetic generator (device) ===================== */

/* Candidate edges of the seeded community generator:
 * candidate i in [first, first+count) -> (dst, src) int64 in PRE-shuffle id
 * space.  Pure function of (params, i): identical to oracle/synth.py. */
int ag_synth_candidates(int64_t num_vertices, int64_t block_gen,
                        double p_intra, double p_global, int64_t window,
                        int64_t skew, uint64_t seed, int64_t first,
                        int64_t count, int64_t *dst_out, int64_t *src_out,
                        void *stream);
/* 64-bit vertex shuffle keys: key[v] = hash(seed, v). */
int ag_synth_vertex_keys(int64_t num_vertices, uint64_t seed, uint64_t *keys,
                         void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ADAPTGEAR_B200_H */
