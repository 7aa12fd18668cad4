/*
 * blast.h -- C ABI of the B200 (sm_100a) block-sparse MLP + prune-and-grow library
 * (libblast_b200.so).
 *
 * The reference (arxiv 2507.03117 "BLaST", package `blocksparse`, pure numpy)
 * has no native layer: its boundary is a set of module-level Python functions
 * over float32 arrays. Each entry point below replaces one of
 * them; the reference function it stands in for is cited per symbol as
 * pkg/src/blocksparse/<file>:<line>. A host binding only needs ctypes / cgo /
 * JNI-style calls with plain pointers: no torch types cross this boundary.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA storage),
 *    row-major, densely packed unless a leading dimension is given.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is asynchronous on that stream; no call synchronizes the host
 *    except where documented (counts returned through host pointers).
 *  - Return value: 0 on success, otherwise a BLAST_E* code; blast_last_error()
 *    returns a message. The host wrappers map codes to the reference's
 *    ValueError messages ("mismatch", "grid", ...).
 *  - dtype: BLAST_F32 computes with 3xTF32 on the tensor cores (fp32-class
 *    accuracy, <=1e-4 relative); BLAST_BF16 computes bf16 x bf16 -> fp32 accumulate.
 *  - Block matrices use the reference's BCSC layout (bcsc.py:35-109):
 *    col_ptr[gc+1] (int64), block_row_idx[nnzb] (int32 here, uint32 there; the
 *    values are identical), values[nnzb][b][b] with values[k][i][j] = W[r*b+i][c*b+j].
 *    `kmap[gr][gc]` (int32) is the inverse map: stored block index or -1.
 */
#ifndef BLAST_B200_H
#define BLAST_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { BLAST_F32 = 0, BLAST_BF16 = 1, BLAST_F64 = 2 /* norms / masks inputs only */ };
enum { BLAST_ACT_NONE = 0, BLAST_ACT_RELU = 1, BLAST_ACT_GELU = 2, BLAST_ACT_SILU = 3 };
enum {
  BLAST_OK = 0,
  BLAST_EINVAL = 1,     /* bad argument (shape, block size, dtype) */
  BLAST_EMISMATCH = 2,  /* dimension mismatch (kernels.py:70-72 "mismatch") */
  BLAST_EGRID = 3,      /* mask grid does not match matrix grid (pruner.py:178-182) */
  BLAST_ECUDA = 4,      /* CUDA runtime / launch error */
  BLAST_ENOMEM = 5,
  BLAST_EUNSUPPORTED = 6  /* configuration not covered by this entry point (nothing launched) */
};

/* Device-resident BCSC matrix (bcsc.py:35 BlockSparseMatrix) plus the cached
 * execution plans derived from it (see blast_bcsc_plan). */
typedef struct blast_bcsc {
  int64_t rows, cols;   /* logical dense shape */
  int32_t block;        /* b */
  int32_t dtype;        /* BLAST_F32 / BLAST_BF16 of `values` */
  int64_t nnzb;
  const int64_t* col_ptr;      /* [gc+1] */
  const int32_t* row_idx;      /* [nnzb] */
  const void* values;          /* [nnzb][b][b] */
  /* F32 only (3xTF32 tensor-core operands, see blast_tf32_prepare), else NULL:
   * blocks transposed (forward, K-major B) and as stored (transposed product). */
  const void* tf32_fwd_hi; const void* tf32_fwd_lo;
  const void* tf32_rt_hi;  const void* tf32_rt_lo;
  const int32_t* kmap;         /* [gr][gc] */
  /* plans: column lines (Y = X W) and row lines (Y = X W^T) */
  const int32_t* fwd_step_ptr; const int32_t* fwd_steps; const int32_t* fwd_flags;
  const int32_t* rt_step_ptr;  const int32_t* rt_steps;  const int32_t* rt_flags;
} blast_bcsc_t;

/* Fused-MLP plans over two matrices of the same grid (gate/up):
 * gu_*  : column lines, steps carry (row, k_gate, k_up)    -> fused gate+up forward
 * dx_*  : row lines,    steps carry (col, k_gate, k_up)    -> dX = dA Wg^T + dB Wu^T  */
typedef struct blast_mlp_plan {
  const int32_t* gu_step_ptr; const int32_t* gu_steps; const int32_t* gu_flags;
  const int32_t* dx_step_ptr; const int32_t* dx_steps; const int32_t* dx_flags;
} blast_mlp_plan_t;

/* Tensor-parallel group for the fused down-projection + all-reduce (SURVEY.md section 8e/8f-4,
 * blast_tp_mlp_forward). Every rank holds the same table; entry r of each array is rank r's
 * buffer as mapped into THIS process (torch symmetric memory / CUDA IPC peer pointers over
 * NVLink, or plain local buffers when the "ranks" share one device). Buffers:
 *   recv[r]  float [2][n][tiles][owned][128][b]  partial output tiles sent to owner r
 *            (tiles = ceil(m / 128); owned = ceil(lines / n), line j owned by rank j % n)
 *   flags[r] uint32 [tiles][owned]  arrival counters, zero-initialised, monotonic
 *   y[r]     [m][d] output of rank r (every rank receives the full all-reduced Y)
 *   done[r]  uint32 tiles written into y[r], zero-initialised, monotonic
 * `epoch` counts the group's fused launches (0, 1, 2, ...; identical on every rank); recv is
 * double-buffered by its parity. n <= 8. */
#define BLAST_TP_MAX 8
typedef struct blast_tp {
  int32_t n, rank;
  uint32_t epoch;
  int32_t reserved;
  float* recv[BLAST_TP_MAX];
  uint32_t* flags[BLAST_TP_MAX];
  void* y[BLAST_TP_MAX];
  uint32_t* done[BLAST_TP_MAX];
} blast_tp_t;

const char* blast_last_error(void);
int blast_version(void);
int blast_num_sms(void);

/* ---------------------------------------------------------------- format / plans */
/* Cost-balanced work lists of the persistent engine (csrc/schedule.cu): item (t, j) of a
 * product with n_tiles token tiles and n_lines output lines, assigned by batched
 * longest-processing-time over the plan's per-line stage counts (step_ptr, or the gate+up
 * counts in flags when seq_gu != 0). out[k * grid + c] = k-th item of CTA c, -1 past its end;
 * out has ceil(n_tiles * n_lines / grid) * grid entries. The engine builds and caches these
 * itself; this entry exposes them for tests. */
int blast_balanced_schedule(const int32_t* step_ptr, const int32_t* flags, int32_t n_lines,
                            int32_t n_tiles, int32_t grid, int32_t seq_gu, int32_t* out,
                            void* stream);
/* kmap from col_ptr/row_idx (inverse index of bcsc.py:205-210). */
int blast_kmap_from_bcsc(const int64_t* col_ptr, const int32_t* row_idx, int64_t grid_rows,
                         int64_t grid_cols, int32_t* kmap, void* stream);
/* Step lists of one or two block maps of the same grid. by_rows = 0: one line per block
 * column (ascending block row, kernels.py:117); by_rows = 1: one line per block row
 * (ascending block column, kernels.py:159). Buffers: step_ptr[lines+1], steps[4*gr*gc],
 * flags[lines]. kmap1 may be NULL. A step is {inner index, block of map 0 or -1, block of
 * map 1 or -1, bits}: bit 0/1 = block of map 0/1 present, bit 2/3 = its first block in the
 * line. flags: bit 0/1 = map 0/1 has a block in the line, bits 2..16 / 17..31 = its block
 * count (saturating at 2^15 - 1). */
int blast_build_plan(const int32_t* kmap0, const int32_t* kmap1, int64_t grid_rows,
                     int64_t grid_cols, int by_rows, int32_t* step_ptr, int32_t* steps,
                     int32_t* flags, void* stream);
/* 3xTF32 operand split: hi = x with the low 13 mantissa bits cleared, lo = x - hi. hi may be
 * NULL: the engine passes the raw x as the hi operand (kind::tf32 reads it truncated). */
int blast_split_tf32(const float* x, float* hi, float* lo, int64_t n, void* stream);
/* 3xTF32 weight operands of an F32 BCSC: split values[nnzb][b][b] into hi/lo, once as
 * stored (rt_*) and once with every block transposed (fwd_*): kind::tf32 reads B K-major. */
int blast_tf32_prepare(const float* values, int64_t nnzb, int32_t block, float* fwd_hi,
                       float* fwd_lo, float* rt_hi, float* rt_lo, void* stream);

/* ---------------------------------------------------------------- products */
/* Y[m, w.cols] = act(X[m, w.rows] @ W)       kernels.py:86 bspmm / :127 bspmm_fused */
int blast_bspmm(const void* x, int64_t m, const blast_bcsc_t* w, int act, void* y,
                void* stream);
/* Y = act(X @ W + bias): bias is float32 [w.cols] (or NULL), added in the epilogue before
 * the activation; pre (optional, same shape/dtype as Y) receives X @ W + bias for the
 * backward. Used by the GPT-2 MLP integration (Conv1D carries a bias; the reference
 * bspmm_fused has none, kernels.py:127). */
int blast_bspmm_ex(const void* x, int64_t m, const blast_bcsc_t* w, const float* bias, int act,
                   void* y, void* pre, void* stream);
/* Backward of a fused activation: Y[m, w.rows] = (X[m, w.cols] @ W^T) * act'(pre), where pre
 * [m, w.rows] is the saved pre-activation of the layer feeding W. */
int blast_bspmm_rt_act(const void* x, int64_t m, const blast_bcsc_t* w, int act, const void* pre,
                       void* y, void* stream);
/* Y[m, w.rows] = X[m, w.cols] @ W^T           kernels.py:143 bspmm_rt */
int blast_bspmm_rt(const void* x, int64_t m, const blast_bcsc_t* w, void* y, void* stream);
/* Elementwise activation (kernels.py:50-62 apply_nonlinearity); in-place allowed. */
int blast_activation(const void* x, void* y, int64_t n, int dtype, int act, void* stream);

/* Gated MLP forward (mlp.py:102-115):
 *   a = X Wg, b = X Wu, g = (a*sigmoid(a))*b, y = g Wd.
 * gate_pre/up_out/gated may be NULL (inference: the intermediate stays in a
 * scratch ring and is never returned). All share dtype with x. */
int blast_mlp_forward(const void* x, int64_t m, const blast_bcsc_t* gate,
                      const blast_bcsc_t* up, const blast_bcsc_t* down,
                      const blast_mlp_plan_t* plan, void* y, void* gate_pre, void* up_out,
                      void* gated, void* stream);
/* Row-parallel down projection of one TP rank fused with the all-reduce of the partial Y
 * (reference mlp.py:114 on a sharded hidden dimension):
 * y[r] (every rank r of tp) += nothing until all ranks of the group have run this call with the
 * same tp->epoch; then y[r] = sum over ranks of G_rank Wd_rank, rounded once. Partial tiles go
 * to their owner rank over peer memory as they are produced (blast_tp_t). Asynchronous: the
 * caller waits with blast_tp_wait(tp->done[rank], (epoch + 1) * tiles * lines) before using y,
 * tiles = ceil(m / 128), lines = ceil(d / b). Tensor-core engine only (b in 16/32/64/128). */
int blast_tp_down_allreduce(const void* g, int64_t m, const blast_bcsc_t* down_shard,
                            const blast_tp_t* tp, void* stream);
/* One TP rank's MLP forward (column-parallel gate/up shards, row-parallel down shard) with the
 * fused all-reduce (the K9 entry of SURVEY.md section 8b). */
int blast_tp_mlp_forward(const void* x, int64_t m, const blast_bcsc_t* gate_shard,
                         const blast_bcsc_t* up_shard, const blast_bcsc_t* down_shard,
                         const blast_mlp_plan_t* plan, const blast_tp_t* tp, void* stream);
/* Stream-ordered wait until *done (system scope) reaches target (wrapping compare); traps
 * after 20 s so a missing peer is a reported error, not a hung device. */
int blast_tp_wait(const uint32_t* done, uint32_t target, void* stream);
/* out[c] = sum_r x[r, c] (fp32) of a row-major [m, n] bf16 / f32 matrix: bias gradients of
 * layers with bias (GPT2MLP integration). Deterministic (fixed row splits, fixed order). */
int blast_column_sums(const void* x, int dtype, int64_t m, int64_t n, float* out, void* stream);
/* blast_mlp_forward on HOST buffers, the reference's boundary (mlp.py:102 takes and returns
 * ndarrays): x_host [m, e] and y_host [m, e] in the network dtype. The tokens are cut into
 * chunks of chunk_tokens rows (0: automatic) and the host->device copy of chunk c+1, the
 * MLP of chunk c and the device->host copy of chunk c-1 run concurrently on two copy
 * streams and the caller's stream. Stream-ordered: y_host is complete once `stream`
 * reaches the point of the call. Host buffers should be page-locked for overlap. */
int blast_mlp_forward_host(const void* x_host, int64_t m, const blast_bcsc_t* gate,
                           const blast_bcsc_t* up, const blast_bcsc_t* down,
                           const blast_mlp_plan_t* plan, void* y_host, int64_t chunk_tokens,
                           void* stream);
/* First half of blast_mlp_forward: gate and up products of every block column from one
 * load of each activation panel, g = (a*sigmoid(a))*b in the epilogue (mlp.py:111-113).
 * gated is required; gate_pre/up_out optional. */
int blast_mlp_gate_up(const void* x, int64_t m, const blast_bcsc_t* gate, const blast_bcsc_t* up,
                      const blast_mlp_plan_t* plan, void* gated, void* gate_pre, void* up_out,
                      void* stream);
/* Gated MLP backward, activation gradients (mlp.py:133-139, :142):
 *   dg = dY Wd^T; db = dg*s; da = (dg*b)*dsilu(a); dX = da Wg^T + db Wu^T.
 * da/db (M x h) are returned for the weight gradients. */
int blast_mlp_backward_dgrad(const void* dy, int64_t m, const void* gate_pre,
                             const void* up_out, const blast_bcsc_t* gate,
                             const blast_bcsc_t* up, const blast_bcsc_t* down,
                             const blast_mlp_plan_t* plan, void* dx, void* da, void* db,
                             void* stream);
/* Weight gradient dW = A^T @ D (mlp.py:137-141, d_gate = x^T da, d_up = x^T db,
 * d_down = g^T dy). a: [m, rows] activations, d: [m, cols] upstream gradient.
 * Block mode (dense_out == NULL): only the blocks of the BCSC structure
 * (col_ptr[gc+1], row_idx[nnzb]) -> out_blocks[nnzb][b][b] float32, BCSC order.
 * Full-grid mode (dense_out != NULL): every block -> dense_out[rows][cols] float32,
 * the reference's dense gradient. */
int blast_block_wgrad(const void* a, const void* d, int64_t m, int64_t rows, int64_t cols,
                      int32_t block, int dtype, const int64_t* col_ptr, const int32_t* row_idx,
                      int64_t nnzb, float* out_blocks, float* dense_out, void* stream);
/* The stored-block mode's work list depends only on the structure: build it once
 * (items: int4[nnzb], counts: int64[grid_cols + 1]; b = 64 or 128) and reuse it with
 * blast_block_wgrad_planned until the mask changes. Same results as blast_block_wgrad. */
int blast_wgrad_plan(const int64_t* col_ptr, int64_t grid_rows, int64_t grid_cols, int32_t block,
                     int32_t* items, int64_t* counts, void* stream);
int blast_block_wgrad_planned(const void* a, const void* d, int64_t m, int64_t rows,
                              int64_t cols, int32_t block, int dtype, const int64_t* col_ptr,
                              const int32_t* row_idx, int64_t nnzb, const int32_t* items,
                              const int64_t* counts, float* out_blocks, void* stream);

/* ---------------------------------------------------------------- prune-and-grow */
/* Frobenius norm per b x b block in float64 (pruner.py:88-98); zero-padded edges.
 * x2 may be NULL; when given, its norms go to norms2 in the same pass (W and G).
 * dtype: BLAST_F32, BLAST_BF16 or BLAST_F64 (every element squared in fp64). */
int blast_block_norms(const void* x, const void* x2, int64_t rows, int64_t cols, int32_t block,
                      int dtype, double* norms, double* norms2, void* stream);
/* Keep the k blocks with the largest norms; ties -> ascending (block col, block row)
 * (pruner.py:101-125). k computed by the caller exactly as pruner.py:111.
 * keep: uint8[gr][gc]. Scratch is internal. */
int blast_topk_mask(const double* norms, int64_t grid_rows, int64_t grid_cols, int64_t k,
                    uint8_t* keep, void* stream);
/* Two independent selections with the same k (weight and gradient norms of
 * generate_masks, pruner.py:142-143) in one launch when the grid fits one CTA's
 * shared memory (<= 24576 blocks), else two launches of blast_topk_mask. */
int blast_topk_mask2(const double* norms_a, const double* norms_b, int64_t grid_rows,
                     int64_t grid_cols, int64_t k, uint8_t* keep_a, uint8_t* keep_b,
                     void* stream);
/* regrown = grad_sel & ~kept; counts[0] = |kept|, counts[1] = |regrown| (device int64[2]).
 * (pruner.py:142-156) */
int blast_mask_difference(const uint8_t* kept, const uint8_t* grad_sel, int64_t n,
                          uint8_t* regrown, int64_t* counts, void* stream);
/* generate_masks in one call (pruner.py:128-157): fp64 block norms of W and G, each in its
 * own dtype (F32 / BF16 / F64; one pass when they match), kept = top-k(norms_w),
 * regrown = top-k(norms_g) & ~kept, counts (device int64[2]) = |kept|, |regrown|; k as
 * pruner.py:111. norms_* are [gr][gc] f64, kept / regrown uint8 [gr][gc]. When counts_host is
 * not NULL the counts are copied there and the call synchronizes the stream (the one host
 * sync of a refresh: PruneReport needs them). */
int blast_generate_masks(const void* w, int dtype_w, const void* g, int dtype_g, int64_t rows,
                         int64_t cols, int32_t block, int64_t k, double* norms_w,
                         double* norms_g, uint8_t* kept, uint8_t* regrown, int64_t* counts,
                         int64_t* counts_host, void* stream);
/* Repack step 1 (bcsc.py:200-209): store = active mask (or any-nonzero blocks when
 * mask == NULL); col_ptr (int64 [gc+1]) by column counts + scan; kmap [gr][gc].
 * nnzb is col_ptr[gc] (left on device). */
int blast_repack_index(const uint8_t* kept, const uint8_t* regrown, const void* dense,
                       int64_t rows, int64_t cols, int32_t block, int dtype, int64_t* col_ptr,
                       int32_t* kmap, void* stream);
/* Repack step 2: block_row_idx from kmap (column-major walk, bcsc.py:207-209). */
int blast_repack_rows(const int32_t* kmap, const int64_t* col_ptr, int64_t grid_rows,
                      int64_t grid_cols, int32_t* row_idx, void* stream);
/* apply_mask + gather (pruner.py:183-186, bcsc.py:210): masked = dense * expand(survive)
 * (multiply semantics: -0.0 and NaN preserved), values[kmap] = masked block, converted to
 * values_dtype. survive = kept (zero_regrown) or kept|regrown. masked_out may alias dense
 * or be NULL. */
int blast_apply_mask_gather(const void* dense, int64_t rows, int64_t cols, int32_t block,
                            int dtype, const uint8_t* kept, const uint8_t* regrown,
                            int zero_regrown, const int32_t* kmap, void* masked_out,
                            void* values, int values_dtype, void* stream);

/* ---------------------------------------------------------------- optimizer glue */
/* w = w - f32(lr) * g without FMA contraction (trainer.py:263-265). */
int blast_sgd_step(float* w, const float* g, int64_t n, float lr, void* stream);
/* out[0] += sum(g^2) in float64 (trainer.py:268-277 global norm). */
int blast_sumsq_f64(const void* x, int64_t n, int dtype, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BLAST_B200_H */
