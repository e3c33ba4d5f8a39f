/*
 * hb.h — C ABI of the B200 (sm_100a) tree-ensemble scoring library (libhb.so).
 *
 * The library implements the hot path Hummingbird (Nakandala et al., OSDI'20,
 * arXiv 2010.04804; /root/reference/PAPER.md, cited as P:<line>) compiles
 * tree ensembles into: batch scoring with the GEMM strategy (Alg. 1),
 * TreeTraversal (Alg. 2) or PerfectTreeTraversal (Alg. 3,
 * P:243-286), picked from tree depth as in Sec. 5.1.
 *
 * Conventions for every entry point
 *  - Status codes: every call returns hb_status; on failure hb_last_error()
 *    returns a thread-local, human-readable message (valid until the next
 *    failing call on the same thread).
 *  - Ownership: hb_compile deep-copies the ensemble; the caller may free it on
 *    return. The model owns its device memory on `device` until hb_free.
 *  - Device pointers: X / out of the hb_predict* family are caller-owned
 *    DEVICE pointers on the model's device (checked with
 *    cudaPointerGetAttributes; host or foreign-device pointers give
 *    HB_E_INVALID). The caller sizes `out` for the kind it asks for (see
 *    hb_output); the library cannot check a buffer's length. The only
 *    per-call device memory is scratch from a stream-ordered pool the model
 *    owns and keeps warm (cudaMallocFromPoolAsync / cudaFreeAsync on
 *    `stream`; no device-wide synchronisation; HB_E_OOM if it cannot be
 *    satisfied): the rank codes of the pre-pass (hb_model_info.rank_prepass =
 *    1; ceil(n_rows / 32) * 128 * words bytes) and the fp64 raw partials of a
 *    TT model walked in L2-resident tree chunks (hb_model_info.tt_chunk_trees
 *    > 0; n_rows * K * 8 bytes). Both are capturable in a CUDA graph.
 *  - Arithmetic: comparisons are IEEE fp32 (Alg. 1-3); every scorer
 *    sums leaf values in fp64 and forms the margin in fp64, so scores agree
 *    with an fp64 tree-order sum to ~1 fp32 ulp whatever the summation order
 *    (reading R23; the paper validates at rtol = atol = 1e-5,
 *    P:469).
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream). Calls only enqueue work and return once the launch succeeded;
 *    asynchronous kernel faults surface at the caller's synchronisation.
 *  - Threading: a compiled model is immutable; concurrent predicts on
 *    different streams are safe. hb_free must not race with in-flight work.
 *  - Layout: X is fp32 row-major, row r at X + r * ldx, ldx >= n_features.
 *    n_rows == 0 is a no-op returning HB_OK.
 */
#ifndef HB_H
#define HB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HB_ABI_VERSION 6   /* 2: hb_model_info.tt_sector; 3: tt_chunk_trees appended;
                              4: HB_OUT_RAW64 + hb_finalize64 (fp64 raw sums);
                              5: hb_model_info.rank_prepass_tma appended;
                              6: hb_model_info.rows_per_lane (was reserved0) */

typedef enum {
  HB_OK = 0,
  HB_E_INVALID = 1,      /* bad argument (NULL, sizes, pointer kind, device)      */
  HB_E_TREE = 2,         /* ensemble fails validation (message names tree/node)   */
  HB_E_UNSUPPORTED = 3,  /* valid but outside what this build supports            */
  HB_E_OOM = 4,          /* device allocation failed                              */
  HB_E_CUDA = 5          /* a CUDA runtime call or kernel launch failed           */
} hb_status;

/* Decision predicate; true => LEFT child ("< comparisons"; Alg. 2
 * Where(T_V < T_T, T_L, T_R)). LE is the sklearn/LightGBM convention.
 * IEEE fp32 compare: NaN makes the predicate false, so NaN goes RIGHT. */
typedef enum { HB_CMP_LT = 0, HB_CMP_LE = 1 } hb_cmp;

/* Ensemble reduction over the tree dimension. MEAN divides output k
 * by the number of trees feeding it in the WHOLE ensemble. */
typedef enum { HB_AGG_SUM = 0, HB_AGG_MEAN = 1 } hb_agg;

/* Post transform of the margin (Table 2: sigmoid, exp, logsumexp).
 * ISOLATION (IsolationForest, Table 1): with leaf
 * values = path length h (depth + c(leaf size) - 1) and agg = MEAN, the
 * anomaly score is 2^(-margin / post_param), post_param = c(psi) > 0. */
typedef enum {
  HB_POST_IDENTITY = 0,
  HB_POST_SIGMOID = 1,
  HB_POST_SOFTMAX = 2,
  HB_POST_ISOLATION = 3
} hb_post;

typedef enum { HB_TASK_REGRESSION = 0, HB_TASK_CLASSIFICATION = 1 } hb_task;

/* Compilation strategy (Sec. 4.1). AUTO applies the depth heuristic of
 * Sec. 5.1 with thresholds recalibrated on B200 (DESIGN.md §6.1,
 * reading R24): PTT if D_max <= 10, else TT; GEMM only when forced or when
 * env HB_GEMM_MAX_DEPTH is set (3 restores the paper's CPU rule). For AUTO
 * models, calls with n_rows <= hb_model_info.small_batch_max_rows (4096) use
 * the trees-across-threads small-batch kernel (small batches
 * favour other kernels); a forced strategy runs its own kernel at every batch
 * size (small_batch_max_rows = 0) unless env HB_SMALL_BATCH is set at compile
 * time (the test / sweep override).  */
typedef enum {
  HB_STRATEGY_AUTO = 0,
  HB_STRATEGY_GEMM = 1,
  HB_STRATEGY_TT = 2,
  HB_STRATEGY_PTT = 3
} hb_strategy;

/* What a scoring launch writes (hb_predict_ex). */
typedef enum {
  HB_OUT_PREDICT = 0,    /* regression: float[n*K] post applied; classification: int32[n] label */
  HB_OUT_PROBA = 1,      /* classification: float[n*C], C = K==1 ? 2 : K; binary gives [1-p, p]  */
  HB_OUT_RAW = 2,        /* float[n*K]: sum of leaf values of THIS model's trees (tree-shard partial) */
  HB_OUT_MARGIN = 3,     /* float[n*K]: (MEAN ? raw/ntrees_k : raw) + base, no post               */
  HB_OUT_LEAF = 4,       /* int32[n*T_model]: tree-local ORIGINAL node id of the reached leaf     */
  HB_OUT_LEAF_HASH = 5,  /* uint64[n]: sum_t mix64((uint64)t_global << 32 | leaf) mod 2^64        */
  HB_OUT_RAW64 = 6       /* double[n*K]: RAW in fp64 (the scorers accumulate in fp64), for
                            tree-shard partials that are reduced and then hb_finalize64'd   */
} hb_output;

/*
 * The ensemble, one flat array per node attribute (Tables 3/5 of P:143-204
 * describe the same per-node information as tensors).
 *  node_offset [n_trees+1]  tree t owns nodes [node_offset[t], node_offset[t+1]);
 *                           tree-local id 0 is the root.
 *  feature     [n_nodes]    0-based feature id; read at internal nodes only.
 *  threshold   [n_nodes]    fp32; read at internal nodes only; must not be NaN
 *                           (+-Inf allowed).
 *  left, right [n_nodes]    tree-local child ids; -1/-1 marks a leaf.
 *  leaf_value  [n_nodes*leaf_width]  read at leaves only; must be finite.
 *  leaf_width               1 (scalar leaves, routed by tree_output) or n_outputs
 *                           (vector leaves, e.g. RF class distributions).
 *  tree_output [n_trees]    output column of each scalar-leaf tree; NULL => t % K.
 *  base_score  [n_outputs]  margin-space constant added after aggregation; NULL => 0.
 */
typedef struct {
  int32_t n_trees;
  int32_t n_features;
  int32_t n_outputs;            /* K: 1 for regression / binary margin */
  const int64_t *node_offset;
  const int32_t *feature;
  const float *threshold;
  const int32_t *left;
  const int32_t *right;
  const float *leaf_value;
  int32_t leaf_width;
  const int32_t *tree_output;
  const float *base_score;
  int32_t cmp;                  /* hb_cmp      */
  int32_t agg;                  /* hb_agg      */
  int32_t post;                 /* hb_post     */
  int32_t task;                 /* hb_task     */
  float post_param;             /* ISOLATION: c(psi) > 0; ignored otherwise */
} hb_ensemble;

typedef struct hb_model hb_model;

typedef struct {
  int32_t strategy;             /* the strategy actually compiled (never AUTO) */
  int32_t max_depth;            /* D_max over this model's trees               */
  int32_t tree_begin;           /* first global tree id of this model          */
  int32_t n_trees;              /* trees in this model                         */
  int32_t n_trees_total;        /* trees in the ensemble it was compiled from  */
  int32_t n_features;
  int32_t n_outputs;
  int32_t leaf_width;
  int32_t device;
  int32_t x_in_smem;            /* 1 if the scorer stages X row tiles in SMEM  */
  int64_t device_bytes;         /* device memory owned by the model            */
  int64_t tree_stride_bytes;    /* bytes per tree in the compiled layout       */
  int32_t tensor_cores;         /* 1 if the scorer runs tcgen05 MMAs (GEMM)    */
  int32_t node_record_bytes;    /* node record size: 4 rank-coded PTT, 8 fp32 PTT / narrow TT,
                                   16 wide-row TT, 0 GEMM */
  int32_t kernel;               /* row-tile scorer: 0 ptt, 1 ptt rank-coded, 2 tt, 3 tt wide-row,
                                   4 gemm tcgen05, 5 gemm CUDA-core (6, 7: removed
                                   experimental TT kernels, never reported)
                                   (small batches: hb_small) */
  int32_t rows_per_cta;         /* rows one CTA owns per tile                   */
  int32_t code_cell_bits;       /* rank-coded PTT: 32 or 16-bit X code cells    */
  int32_t rank_prepass;         /* rank-coded PTT: 1 if a separate launch (rank_code_kernel)
                                   computes the X codes into stream-ordered scratch */
  int32_t tt_sector;            /* always 0 (sector-paired TT records were removed; kept for ABI layout) */
  int32_t tt_chunk_trees;       /* wide-row TT: trees per L2-resident chunk when the model is
                                   walked in several launches (0: one launch) */
  int32_t small_batch_max_rows; /* calls with n_rows <= this run the small-batch kernel
                                   (trees across threads) instead of `kernel` (ABI 4) */
  int32_t tt_walks_per_lane;    /* wide-row TT: concurrent walks per lane (ABI 4)        */
  int64_t tt_record_bytes;      /* wide-row TT: bytes of the 16-B node records the walk
                                   reads (tables of leaf ids excluded) (ABI 4)          */
  int32_t rank_prepass_tma;     /* rank_prepass: 1 if the tables are grouped for the TMA
                                   pre-pass (rank_code_tma_kernel, one 16-B box of 4 X
                                   columns per row); it runs on calls whose X is 16-B
                                   aligned with ldx % 4 == 0, the generic pre-pass
                                   kernels on the others (ABI 5)                       */
  int32_t rows_per_lane;        /* rank-coded PTT scorer: rows each lane walks (2: the top
                                   three tree levels are loaded once for a lane's two rows;
                                   pre-pass codes, D >= 3); 1 otherwise (ABI 6)          */
} hb_model_info;

/* Host-only validation of an ensemble (no CUDA calls): the tree structure
 * the paper's compilers assume (binary trees of numerical splits, P:137;
 * node tensors of Tables 3/5/6). HB_E_TREE names the
 * first offending tree/node. Rules: n_trees >= 1, n_features >= 1,
 * n_outputs >= 1, leaf_width in {1, K}; offsets monotone; each tree a rooted
 * binary tree (one parent per non-root node, no cycles, all nodes reachable,
 * left == -1 <=> right == -1); feature in range; threshold not NaN; leaf values
 * finite; tree_output in [0, K); SIGMOID => K == 1; SOFTMAX => K >= 2;
 * ISOLATION => K == 1, REGRESSION and a finite post_param > 0;
 * CLASSIFICATION => (K == 1 and SIGMOID) or K >= 2. */
hb_status hb_validate(const hb_ensemble *e);

/* Validate, select the strategy (Sec. 5.1), build its layout
 * (Tables 3/5/6; perfect padding P:243; feature-selection
 * injection P:316) and upload it to `device`. Forced PTT beyond its memory/depth budget -> HB_E_UNSUPPORTED
 * (AUTO falls back to TT). */
hb_status hb_compile(const hb_ensemble *e, int32_t strategy, int32_t device, hb_model **out);

/* Same for the tree shard [tree_begin, tree_end): the model keeps the global
 * per-output tree counts (for MEAN) and global tree ids (for leaf hashes) so
 * partial sums of shards reduce to the unsharded result.
 * For vector-free multiclass (leaf_width == 1, K > 1) tree_begin should be a
 * multiple of K to keep shards balanced (not required for correctness). */
hb_status hb_compile_range(const hb_ensemble *e, int32_t tree_begin, int32_t tree_end,
                           int32_t strategy, int32_t device, hb_model **out);

/* One fused scoring launch writing `kind` (hb_output) for rows [0, n_rows)
 * (two for rank_prepass models on more than the small-batch row count: the
 * rank-code pre-pass, then the scorer; one per L2-resident tree chunk plus a
 * finalize for chunked TT models; all on `stream`).
 * Defined by: the strategies' input/output contract, X in R^{n x |F|} in,
 * R in R^{n x |C|} out — Alg. 1 P:171-172 (GEMM), Alg. 2
 * (TreeTraversal), Alg. 3 P:262-263 (PerfectTreeTraversal) — followed by the
 * reduction over the tree dimension of an ensemble and the post
 * transforms of Table 2 (sigmoid, exp/logsumexp, argmax).
 * Arguments: X device fp32 row-major, row r at X + r * ldx (ldx >= n_features);
 * out device, sized per `kind` (hb_output); stream = cudaStream_t or NULL.
 * Errors: HB_E_INVALID (NULL model/pointers, n_rows < 0, ldx < n_features,
 * host or foreign-device pointers, bad kind), HB_E_UNSUPPORTED (PROBA on a
 * regression model), HB_E_OOM (scratch), HB_E_CUDA (launch failure). */
hb_status hb_predict_ex(const hb_model *m, const float *X, int64_t n_rows, int64_t ldx,
                        int32_t kind, void *out, void *stream);

/* Profiling form of hb_predict_ex (same arguments, same work): additionally
 * records the caller-created events `events[i]` (cudaEvent_t passed as void*)
 * on `stream` at the start of the call's launch i and one after its last
 * launch, so per-kernel durations of a multi-launch call (rank-code pre-pass
 * + scorer; tree chunks + finalize) can be read with cudaEventElapsedTime
 * without any synchronisation. n_events >= 2; at most n_events events are
 * recorded. *n_launches (if not NULL) receives the number of kernel launches
 * the call made. Used by bench.py's roofline (dominant kernel duration). */
hb_status hb_predict_ex_events(const hb_model *m, const float *X, int64_t n_rows, int64_t ldx,
                               int32_t kind, void *out, void *stream, void **events,
                               int32_t n_events, int32_t *n_launches);

/* = hb_predict_ex(HB_OUT_PREDICT): the algorithms' output R (P:172, P:210,
 * P:263) — regression: float[n*K] after the post transform; classification:
 * int32[n] class index (K == 1: 1 iff margin > 0; else argmax, lowest index on
 * ties; R22). */
hb_status hb_predict(const hb_model *m, const float *X, int64_t n_rows, int64_t ldx,
                     void *out, void *stream);
/* = hb_predict_ex(HB_OUT_PROBA): class probabilities validated in P:469
 * ("both the final scores and the probabilities"): float[n*C], C = 2 for a
 * sigmoid model ([1-p, p]), else K. HB_E_UNSUPPORTED on a regression model. */
hb_status hb_predict_proba(const hb_model *m, const float *X, int64_t n_rows, int64_t ldx,
                           float *out, void *stream);
/* = hb_predict_ex(HB_OUT_RAW): float[n*K], the per-output sum over THIS
 * model's trees of the selected leaf values — the tree-dimension reduction of
 * P:192 before MEAN / base / post; a tree shard's partial. */
hb_status hb_predict_raw(const hb_model *m, const float *X, int64_t n_rows, int64_t ldx,
                         float *out, void *stream);
/* = hb_predict_ex(HB_OUT_LEAF): int32[n*T_model], the tree-local ORIGINAL
 * node id of the leaf each (row, tree) reaches — the leaf selection of Alg. 1
 * (S == D), Alg. 2 (final T_I) and Alg. 3 (T_I - 2^D mapped
 * back through the padding); the quantity the paper's output
 * validation rests on and the bit-exact parity target. */
hb_status hb_predict_leaf(const hb_model *m, const float *X, int64_t n_rows, int64_t ldx,
                          int32_t *out, void *stream);

/* Epilogue only (P:192 reduction result -> Table 2 P:117 transforms): from
 * raw sums over ALL trees (e.g. the NCCL-reduced tree-shard partials,
 * float[n*K] on the device) write `kind` in {PREDICT, PROBA, MARGIN} using the
 * model's global per-output tree counts (MEAN), base score and post
 * transform. Errors as hb_predict_ex; HB_E_INVALID for any other kind. */
hb_status hb_finalize(const hb_model *m, const float *raw, int64_t n_rows, int32_t kind,
                      void *out, void *stream);
/* Same from fp64 raw sums (double[n*K], e.g. HB_OUT_RAW64 partials reduced
 * in fp64), so a tree-sharded result carries no fp32 rounding before the
 * margin is formed. */
hb_status hb_finalize64(const hb_model *m, const double *raw, int64_t n_rows, int32_t kind,
                        void *out, void *stream);

/* End-to-end scoring from HOST memory (the same contract as hb_predict_ex,
 * P:171-172 / P:209-210 / P:262-263, with X and out in host memory): rows are
 * streamed in chunks through double-buffered device staging (H2D copy of chunk
 * i+1 overlaps scoring of chunk i on a second stream) and results copied back.
 * Synchronous: returns when `out_host` is filled. Pinned host buffers
 * (cudaHostAlloc / torch.pin_memory) are needed for the copies to overlap.
 * kind as in hb_predict_ex except LEAF (HB_E_UNSUPPORTED). */
hb_status hb_predict_host(const hb_model *m, const float *X_host, int64_t n_rows, int64_t ldx,
                          int32_t kind, void *out_host);

hb_status hb_model_get_info(const hb_model *m, hb_model_info *info);
void hb_free(hb_model *m);
const char *hb_last_error(void);
int32_t hb_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HB_H */
