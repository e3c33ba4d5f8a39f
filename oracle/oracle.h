/*
 * oracle.h — plain, slow, obviously-correct CPU scoring of decision-tree
 * ensembles. TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. It shares
 * no code, header, table or helper with the CUDA product
 * (paper_2010_04804_b200/, include/hb.h).
 *
 * What it computes (§4.1; readings in DESIGN.md §2):
 *   for each row r and tree t: start at the root (tree-local node 0), and
 *   while the node is internal go left iff pred(X[r, feature], threshold)
 *   (cmp LT: x < t, cmp LE: x <= t; IEEE fp32 compare, NaN => false => right);
 *   the reached leaf is leaf[r][t] (its tree-local ORIGINAL node id).
 *   raw[r][k]    = sum over trees feeding k, in tree order, fp64.
 *   margin[r][k] = (agg == MEAN ? raw / ntrees_k : raw) + base[k].
 *   post: identity | sigmoid | softmax (max-subtracted) | isolation
 *   2^(-margin / c(psi)) (IsolationForest, Liu et al.; sklearn score_samples), fp64.
 *   label: K == 1 -> margin > 0 ; K >= 2 -> argmax, lowest index on ties.
 *
 * The GEMM / TreeTraversal / PerfectTreeTraversal strategies reach exactly
 * this leaf (SURVEY.md §8(c) "Why GEMM selects exactly one real leaf"); the
 * literal numpy transcriptions of Alg. 1-3 in oracle/literal.py check that.
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t n_trees, n_features, n_outputs;
  const int64_t *node_offset;   /* [n_trees+1] */
  const int32_t *feature;       /* [n_nodes]   */
  const float   *threshold;     /* [n_nodes]   */
  const int32_t *left, *right;  /* [n_nodes], -1/-1 = leaf */
  const float   *leaf_value;    /* [n_nodes * leaf_width] */
  int32_t        leaf_width;    /* 1 or n_outputs */
  const int32_t *tree_output;   /* [n_trees] or NULL => t % K (leaf_width == 1 only) */
  const float   *base_score;    /* [n_outputs] or NULL => 0 */
  int32_t cmp;                  /* 0 = LT, 1 = LE */
  int32_t agg;                  /* 0 = SUM, 1 = MEAN */
  int32_t post;                 /* 0 = identity, 1 = sigmoid, 2 = softmax, 3 = isolation */
  double post_param;            /* isolation: c(psi) */
} oracle_ensemble;

/* leaf ids: out[r * (t1 - t0) + (t - t0)] for trees t in [t0, t1). */
void oracle_leaf(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                 int32_t t0, int32_t t1, int32_t *out);

/* raw sums over trees [t0, t1): out[r * K + k], fp64, tree order. */
void oracle_raw(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                int32_t t0, int32_t t1, double *out);

/* margin from a raw sum over ALL trees: MEAN divides by the number of trees
 * feeding output k in the whole ensemble; then + base. In place allowed. */
void oracle_margin(const oracle_ensemble *e, const double *raw, int64_t n, double *margin);

/* post transform of margins (identity / sigmoid / softmax), fp64. */
void oracle_post(const oracle_ensemble *e, const double *margin, int64_t n, double *out);

/* class label from margins. */
void oracle_label(const oracle_ensemble *e, const double *margin, int64_t n, int32_t *out);

/* order-independent per-row leaf hash over trees [t0, t1):
 * h_r = sum_t mix64(((uint64)t << 32) | leaf[r][t]) mod 2^64, t global id. */
void oracle_leaf_hash(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                      int32_t t0, int32_t t1, uint64_t *out);

/* multi-threaded raw (rows split in contiguous blocks); used only to time the
 * oracle as the CPU baseline. nthreads <= 0 => all online cores. Returns the
 * thread count used. */
int oracle_raw_mt(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                  int32_t t0, int32_t t1, double *out, int nthreads);

/* raw sums AND leaf hashes over trees [t0, t1) in one walk per (row, tree),
 * rows split over nthreads pthreads (<= 0: all online cores): the same values
 * as oracle_raw + oracle_leaf_hash, for parity checks on every row of a
 * full-size config. Returns the thread count used. */
int oracle_raw_hash_mt(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                       int32_t t0, int32_t t1, double *out, uint64_t *hash, int nthreads);

/* full scoring (raw over all trees -> margin -> post), multi-threaded; the
 * thing bench.py times. out = post-transformed scores [n * K]. */
int oracle_predict_mt(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                      double *out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
