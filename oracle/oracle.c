/*
 * oracle.c — the CPU oracle. TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Compiled with plain -O2, no -ffast-math (NaN must stay NaN), no SIMD
 * intrinsics. Every function is the textbook definition written out.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <unistd.h>

/* PAPER.md P:137 ("we assume all decision nodes perform < comparisons") and
 * Alg. 2 P:232 `Where(T_V < T_T, T_L, T_R)`: predicate true => LEFT child.
 * LE is the sklearn/LightGBM convention (reading R1). A NaN makes
 * both comparisons false, so NaN goes right (reading R2). */
static int go_left(int32_t cmp, float x, float t) {
  if (cmp == 0) return x < t;
  return x <= t;
}

/* Plain tree walk from the root (tree-local id 0) to a leaf; returns the
 * leaf's tree-local id. A node is a leaf iff left == -1. */
static int32_t walk(const oracle_ensemble *e, int32_t t, const float *x) {
  int64_t base = e->node_offset[t];
  int32_t i = 0;
  while (e->left[base + i] != -1) {
    float xv = x[e->feature[base + i]];
    float th = e->threshold[base + i];
    i = go_left(e->cmp, xv, th) ? e->left[base + i] : e->right[base + i];
  }
  return i;
}

static int32_t tree_out(const oracle_ensemble *e, int32_t t) {
  if (e->tree_output) return e->tree_output[t];
  return t % e->n_outputs;
}

void oracle_leaf(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                 int32_t t0, int32_t t1, int32_t *out) {
  int32_t nt = t1 - t0;
  for (int64_t r = 0; r < n; ++r)
    for (int32_t t = t0; t < t1; ++t)
      out[r * nt + (t - t0)] = walk(e, t, X + r * ldx);
}

/* ensembles batch the per-tree results and reduce over the
 * tree dimension; regression leaves carry values ("we initialize E with label
 * values"). Here: fp64 sum in tree order of the reached leaf's value(s). */
static void raw_rows(const oracle_ensemble *e, const float *X, int64_t r0, int64_t r1,
                     int64_t ldx, int32_t t0, int32_t t1, double *out) {
  int32_t K = e->n_outputs, w = e->leaf_width;
  for (int64_t r = r0; r < r1; ++r) {
    double *o = out + r * K;
    for (int32_t k = 0; k < K; ++k) o[k] = 0.0;
    for (int32_t t = t0; t < t1; ++t) {
      int32_t leaf = walk(e, t, X + r * ldx);
      const float *v = e->leaf_value + (e->node_offset[t] + leaf) * w;
      if (w == 1) {
        o[tree_out(e, t)] += (double)v[0];
      } else {
        for (int32_t k = 0; k < K; ++k) o[k] += (double)v[k];
      }
    }
  }
}

void oracle_raw(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                int32_t t0, int32_t t1, double *out) {
  raw_rows(e, X, 0, n, ldx, t0, t1, out);
}

/* Number of trees feeding output k over the whole ensemble (for MEAN,
 * "ReduceMean over the batched dimension"). */
static void trees_per_output(const oracle_ensemble *e, double *cnt) {
  int32_t K = e->n_outputs;
  for (int32_t k = 0; k < K; ++k) cnt[k] = 0.0;
  for (int32_t t = 0; t < e->n_trees; ++t) {
    if (e->leaf_width == 1) cnt[tree_out(e, t)] += 1.0;
    else for (int32_t k = 0; k < K; ++k) cnt[k] += 1.0;
  }
}

void oracle_margin(const oracle_ensemble *e, const double *raw, int64_t n, double *margin) {
  int32_t K = e->n_outputs;
  double cnt[4096];
  double *c = K <= 4096 ? cnt : (double *)malloc(sizeof(double) * K);
  trees_per_output(e, c);
  for (int64_t r = 0; r < n; ++r)
    for (int32_t k = 0; k < K; ++k) {
      double m = raw[r * K + k];
      if (e->agg == 1) m = m / c[k];
      if (e->base_score) m = m + (double)e->base_score[k];
      margin[r * K + k] = m;
    }
  if (c != cnt) free(c);
}

/* Table 2 P:117 lists sigmoid, exp, logsumexp: sigmoid(m) = 1 / (1 + exp(-m));
 * softmax(m)_k = exp(m_k - max_j m_j) / sum_j exp(m_j - max_j m_j). */
void oracle_post(const oracle_ensemble *e, const double *margin, int64_t n, double *out) {
  int32_t K = e->n_outputs;
  for (int64_t r = 0; r < n; ++r) {
    const double *m = margin + r * K;
    double *o = out + r * K;
    if (e->post == 0) {
      for (int32_t k = 0; k < K; ++k) o[k] = m[k];
    } else if (e->post == 1) {
      for (int32_t k = 0; k < K; ++k) o[k] = 1.0 / (1.0 + exp(-m[k]));
    } else if (e->post == 3) {
      /* IsolationForest anomaly score: 2^(-E[h(x)] / c(psi)) */
      for (int32_t k = 0; k < K; ++k) o[k] = pow(2.0, -m[k] / e->post_param);
    } else {
      double mx = m[0];
      for (int32_t k = 1; k < K; ++k) if (m[k] > mx) mx = m[k];
      double s = 0.0;
      for (int32_t k = 0; k < K; ++k) s += exp(m[k] - mx);
      for (int32_t k = 0; k < K; ++k) o[k] = exp(m[k] - mx) / s;
    }
  }
}

/* Labels (reading R22): K == 1 -> 1 iff margin > 0 (sigmoid > 0.5);
 * K >= 2 -> argmax with the lowest index on ties. */
void oracle_label(const oracle_ensemble *e, const double *margin, int64_t n, int32_t *out) {
  int32_t K = e->n_outputs;
  for (int64_t r = 0; r < n; ++r) {
    const double *m = margin + r * K;
    if (K == 1) { out[r] = m[0] > 0.0 ? 1 : 0; continue; }
    int32_t best = 0;
    for (int32_t k = 1; k < K; ++k) if (m[k] > m[best]) best = k;
    out[r] = best;
  }
}

static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

void oracle_leaf_hash(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                      int32_t t0, int32_t t1, uint64_t *out) {
  for (int64_t r = 0; r < n; ++r) {
    uint64_t h = 0;
    for (int32_t t = t0; t < t1; ++t) {
      uint32_t leaf = (uint32_t)walk(e, t, X + r * ldx);
      h += mix64(((uint64_t)(uint32_t)t << 32) | leaf);
    }
    out[r] = h;
  }
}

typedef struct {
  const oracle_ensemble *e; const float *X; int64_t r0, r1, ldx; int32_t t0, t1; double *out;
} job_t;

static void *job_main(void *p) {
  job_t *j = (job_t *)p;
  raw_rows(j->e, j->X, j->r0, j->r1, j->ldx, j->t0, j->t1, j->out);
  return NULL;
}

int oracle_raw_mt(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                  int32_t t0, int32_t t1, double *out, int nthreads) {
  if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 1024) nthreads = 1024;
  if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
  pthread_t th[1024];
  job_t jobs[1024];
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].e = e; jobs[i].X = X; jobs[i].ldx = ldx; jobs[i].t0 = t0; jobs[i].t1 = t1;
    jobs[i].out = out;
    jobs[i].r0 = n * i / nthreads; jobs[i].r1 = n * (i + 1) / nthreads;
    if (nthreads == 1) job_main(&jobs[i]);
    else pthread_create(&th[i], NULL, job_main, &jobs[i]);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  return nthreads;
}

/* raw sums and leaf hashes of rows [r0, r1) in one walk per (row, tree):
 * exactly raw_rows() and oracle_leaf_hash() above, fused so the full-size
 * parity checks (every row of C3 / the C5 shard) walk each pair once. */
static void raw_hash_rows(const oracle_ensemble *e, const float *X, int64_t r0, int64_t r1,
                          int64_t ldx, int32_t t0, int32_t t1, double *out, uint64_t *hash) {
  int32_t K = e->n_outputs, w = e->leaf_width;
  for (int64_t r = r0; r < r1; ++r) {
    double *o = out + r * K;
    uint64_t h = 0;
    for (int32_t k = 0; k < K; ++k) o[k] = 0.0;
    for (int32_t t = t0; t < t1; ++t) {
      int32_t leaf = walk(e, t, X + r * ldx);
      const float *v = e->leaf_value + (e->node_offset[t] + leaf) * w;
      if (w == 1) {
        o[tree_out(e, t)] += (double)v[0];
      } else {
        for (int32_t k = 0; k < K; ++k) o[k] += (double)v[k];
      }
      h += mix64(((uint64_t)(uint32_t)t << 32) | (uint32_t)leaf);
    }
    hash[r] = h;
  }
}

typedef struct {
  const oracle_ensemble *e; const float *X; int64_t r0, r1, ldx; int32_t t0, t1;
  double *out; uint64_t *hash;
} hjob_t;

static void *hjob_main(void *p) {
  hjob_t *j = (hjob_t *)p;
  raw_hash_rows(j->e, j->X, j->r0, j->r1, j->ldx, j->t0, j->t1, j->out, j->hash);
  return NULL;
}

int oracle_raw_hash_mt(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                       int32_t t0, int32_t t1, double *out, uint64_t *hash, int nthreads) {
  if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 1024) nthreads = 1024;
  if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
  pthread_t th[1024];
  hjob_t jobs[1024];
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].e = e; jobs[i].X = X; jobs[i].ldx = ldx; jobs[i].t0 = t0; jobs[i].t1 = t1;
    jobs[i].out = out; jobs[i].hash = hash;
    jobs[i].r0 = n * i / nthreads; jobs[i].r1 = n * (i + 1) / nthreads;
    if (nthreads == 1) hjob_main(&jobs[i]);
    else pthread_create(&th[i], NULL, hjob_main, &jobs[i]);
  }
  if (nthreads > 1)
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  return nthreads;
}

int oracle_predict_mt(const oracle_ensemble *e, const float *X, int64_t n, int64_t ldx,
                      double *out, int nthreads) {
  int used = oracle_raw_mt(e, X, n, ldx, 0, e->n_trees, out, nthreads);
  oracle_margin(e, out, n, out);
  oracle_post(e, out, n, out);
  return used;
}
