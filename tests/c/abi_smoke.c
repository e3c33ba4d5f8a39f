/*
 * abi_smoke.c — a plain C consumer of include/hb.h: built
 * with gcc against the header, linked to libhb.so, it drives every entry point
 * through the C ABI on the hand-traced trees of tests/golden/hand_trees.json
 * (Alg. 1-3 I/O, P:171-172 / P:209-210 / P:262-263; reduction
 * P:192) and checks leaf ids bit-exact and scores within the R23 tolerance
 * (|got - ref| <= 1e-5 + 1e-5 |ref|).
 *
 * Input: a flat text dump of the golden file written by tests/test_c_abi.py
 * (the JSON stays the single source of truth):
 *   T F n_nodes n_rows
 *   node_offset[T+1] feature[n] threshold[n] left[n] right[n] leaf_value[n]
 *   X[n_rows*F]
 *   for cmp in (LT, LE): leaf[n_rows*T] sum[n_rows]
 * Exit status 0 = every check passed; prints one line per failure.
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "hb.h"

static int failures = 0;
#define CHECK(cond, ...)                                   \
  do {                                                     \
    if (!(cond)) {                                         \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);                        \
      fprintf(stderr, "\n");                               \
      ++failures;                                          \
    }                                                      \
  } while (0)
#define HB(call)                                                                    \
  do {                                                                              \
    hb_status st_ = (call);                                                         \
    if (st_ != HB_OK) {                                                             \
      fprintf(stderr, "FAIL %s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, st_, \
              hb_last_error());                                                     \
      ++failures;                                                                   \
    }                                                                               \
  } while (0)
#define CU(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "CUDA %s:%d: %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(2);                                                                      \
    }                                                                               \
  } while (0)

static int tol_ok(double got, double ref) { return fabs(got - ref) <= 1e-5 + 1e-5 * fabs(ref); }

static FILE *in;
static double rd(void) {
  char tok[64];
  if (fscanf(in, "%63s", tok) != 1) { fprintf(stderr, "short input\n"); exit(2); }
  return strtod(tok, NULL);
}

static void *dalloc(size_t bytes) {
  void *p = NULL;
  CU(cudaMalloc(&p, bytes ? bytes : 16));
  return p;
}

int main(int argc, char **argv) {
  if (argc != 2 || !(in = fopen(argv[1], "r"))) {
    fprintf(stderr, "usage: abi_smoke <golden.txt>\n");
    return 2;
  }
  const int T = (int)rd(), F = (int)rd(), N = (int)rd(), R = (int)rd();
  int64_t *off = malloc(sizeof(int64_t) * (T + 1));
  int32_t *feat = malloc(4 * N), *left = malloc(4 * N), *right = malloc(4 * N);
  float *thr = malloc(4 * N), *val = malloc(4 * N), *X = malloc(4 * (size_t)R * F);
  for (int i = 0; i <= T; ++i) off[i] = (int64_t)rd();
  for (int i = 0; i < N; ++i) feat[i] = (int32_t)rd();
  for (int i = 0; i < N; ++i) thr[i] = (float)rd();
  for (int i = 0; i < N; ++i) left[i] = (int32_t)rd();
  for (int i = 0; i < N; ++i) right[i] = (int32_t)rd();
  for (int i = 0; i < N; ++i) val[i] = (float)rd();
  for (int i = 0; i < R * F; ++i) X[i] = (float)rd();
  int32_t *exp_leaf[2];
  double *exp_sum[2];
  for (int c = 0; c < 2; ++c) {
    exp_leaf[c] = malloc(4 * (size_t)R * T);
    exp_sum[c] = malloc(8 * (size_t)R);
    for (int i = 0; i < R * T; ++i) exp_leaf[c][i] = (int32_t)rd();
    for (int i = 0; i < R; ++i) exp_sum[c][i] = rd();
  }
  fclose(in);

  CHECK(hb_abi_version() == HB_ABI_VERSION, "abi version %d != header %d", hb_abi_version(), HB_ABI_VERSION);

  float *dX = dalloc(4 * (size_t)R * F);
  CU(cudaMemcpy(dX, X, 4 * (size_t)R * F, cudaMemcpyHostToDevice));
  float *dF = dalloc(8 * (size_t)R);            /* float outputs (up to 2 per row) */
  double *dD = dalloc(8 * (size_t)R);           /* fp64 raw                        */
  int32_t *dL = dalloc(4 * (size_t)R * T);      /* leaf ids / labels               */
  uint64_t *dH = dalloc(8 * (size_t)R);         /* leaf hashes                     */
  float *hF = malloc(8 * (size_t)R);
  double *hD = malloc(8 * (size_t)R);
  int32_t *hL = malloc(4 * (size_t)R * T);
  uint64_t *hH = malloc(8 * (size_t)R);
  cudaStream_t s;
  CU(cudaStreamCreate(&s));

  const int strategies[4] = {HB_STRATEGY_AUTO, HB_STRATEGY_GEMM, HB_STRATEGY_TT, HB_STRATEGY_PTT};
  for (int cmp = 0; cmp < 2; ++cmp) {
    /* regression model: leaf values summed over trees, identity post */
    hb_ensemble e;
    memset(&e, 0, sizeof e);
    e.n_trees = T; e.n_features = F; e.n_outputs = 1;
    e.node_offset = off; e.feature = feat; e.threshold = thr; e.left = left; e.right = right;
    e.leaf_value = val; e.leaf_width = 1; e.tree_output = NULL; e.base_score = NULL;
    e.cmp = cmp; e.agg = HB_AGG_SUM; e.post = HB_POST_IDENTITY; e.task = HB_TASK_REGRESSION;
    HB(hb_validate(&e));
    for (int si = 0; si < 4; ++si) {
      hb_model *m = NULL;
      HB(hb_compile(&e, strategies[si], 0, &m));
      if (!m) continue;
      hb_model_info info;
      HB(hb_model_get_info(m, &info));
      CHECK(info.n_trees == T && info.n_features == F && info.n_outputs == 1, "model info");
      CHECK(si == 0 || info.strategy == strategies[si], "strategy %d compiled as %d", strategies[si], info.strategy);
      /* leaf ids: bit-exact */
      HB(hb_predict_leaf(m, dX, R, F, dL, s));
      CU(cudaStreamSynchronize(s));
      CU(cudaMemcpy(hL, dL, 4 * (size_t)R * T, cudaMemcpyDeviceToHost));
      for (int i = 0; i < R * T; ++i)
        CHECK(hL[i] == exp_leaf[cmp][i], "cmp %d strat %d leaf[%d] = %d, expected %d", cmp, si, i, hL[i], exp_leaf[cmp][i]);
      /* predict (regression) and raw: the hand-traced sums */
      HB(hb_predict(m, dX, R, F, dF, s));
      CU(cudaStreamSynchronize(s));
      CU(cudaMemcpy(hF, dF, 4 * (size_t)R, cudaMemcpyDeviceToHost));
      for (int r = 0; r < R; ++r) CHECK(tol_ok(hF[r], exp_sum[cmp][r]), "predict row %d %g vs %g", r, hF[r], exp_sum[cmp][r]);
      HB(hb_predict_raw(m, dX, R, F, dF, s));
      CU(cudaStreamSynchronize(s));
      CU(cudaMemcpy(hF, dF, 4 * (size_t)R, cudaMemcpyDeviceToHost));
      for (int r = 0; r < R; ++r) CHECK(tol_ok(hF[r], exp_sum[cmp][r]), "raw row %d", r);
      HB(hb_predict_ex(m, dX, R, F, HB_OUT_RAW64, dD, s));
      CU(cudaStreamSynchronize(s));
      CU(cudaMemcpy(hD, dD, 8 * (size_t)R, cudaMemcpyDeviceToHost));
      for (int r = 0; r < R; ++r) CHECK(tol_ok(hD[r], exp_sum[cmp][r]), "raw64 row %d", r);
      /* epilogue from raw sums: finalize (fp32) and finalize64 */
      HB(hb_finalize64(m, dD, R, HB_OUT_PREDICT, dF, s));
      CU(cudaStreamSynchronize(s));
      CU(cudaMemcpy(hF, dF, 4 * (size_t)R, cudaMemcpyDeviceToHost));
      for (int r = 0; r < R; ++r) CHECK(tol_ok(hF[r], exp_sum[cmp][r]), "finalize64 row %d", r);
      /* proba on a regression model is unsupported; the message is set */
      CHECK(hb_predict_proba(m, dX, R, F, dF, s) == HB_E_UNSUPPORTED, "proba on regression");
      CHECK(strlen(hb_last_error()) > 0, "hb_last_error empty");
      /* host pointers are rejected */
      CHECK(hb_predict(m, X, R, F, dF, s) == HB_E_INVALID, "host X accepted");
      /* end to end from host memory */
      HB(hb_predict_host(m, X, R, F, HB_OUT_PREDICT, hF));
      for (int r = 0; r < R; ++r) CHECK(tol_ok(hF[r], exp_sum[cmp][r]), "predict_host row %d", r);
      hb_free(m);
    }

    /* binary classification variant: sigmoid of the sums, base score -0.5 */
    float base = -0.5f;
    e.base_score = &base;
    e.post = HB_POST_SIGMOID;
    e.task = HB_TASK_CLASSIFICATION;
    hb_model *m = NULL;
    HB(hb_compile(&e, HB_STRATEGY_AUTO, 0, &m));
    if (m) {
      HB(hb_predict_proba(m, dX, R, F, dF, s));
      HB(hb_predict(m, dX, R, F, dL, s));
      CU(cudaStreamSynchronize(s));
      CU(cudaMemcpy(hF, dF, 8 * (size_t)R, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(hL, dL, 4 * (size_t)R, cudaMemcpyDeviceToHost));
      for (int r = 0; r < R; ++r) {
        const double mg = exp_sum[cmp][r] - 0.5, p = 1.0 / (1.0 + exp(-mg));
        CHECK(tol_ok(hF[2 * r + 1], p) && tol_ok(hF[2 * r], 1.0 - p), "proba row %d", r);
        if (fabs(mg) > 1e-4) CHECK(hL[r] == (mg > 0), "label row %d", r);
      }
      /* tree shards: raw partials of [0, 2) and [2, T) add up; finalize on the sum */
      hb_model *a = NULL, *b = NULL;
      HB(hb_compile_range(&e, 0, 2, HB_STRATEGY_AUTO, 0, &a));
      HB(hb_compile_range(&e, 2, T, HB_STRATEGY_AUTO, 0, &b));
      if (a && b) {
        float *dR2 = dalloc(4 * (size_t)R);
        HB(hb_predict_raw(a, dX, R, F, dF, s));
        HB(hb_predict_raw(b, dX, R, F, dR2, s));
        CU(cudaStreamSynchronize(s));
        float *h1 = malloc(4 * (size_t)R), *h2 = malloc(4 * (size_t)R);
        CU(cudaMemcpy(h1, dF, 4 * (size_t)R, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(h2, dR2, 4 * (size_t)R, cudaMemcpyDeviceToHost));
        for (int r = 0; r < R; ++r) h1[r] += h2[r];
        CU(cudaMemcpy(dR2, h1, 4 * (size_t)R, cudaMemcpyHostToDevice));
        HB(hb_finalize(a, dR2, R, HB_OUT_PROBA, dF, s));
        CU(cudaStreamSynchronize(s));
        CU(cudaMemcpy(hF, dF, 8 * (size_t)R, cudaMemcpyDeviceToHost));
        for (int r = 0; r < R; ++r) {
          const double p = 1.0 / (1.0 + exp(-(exp_sum[cmp][r] - 0.5)));
          CHECK(tol_ok(hF[2 * r + 1], p), "shard finalize row %d", r);
        }
        /* leaf hashes are additive over shards */
        uint64_t *hA = malloc(8 * (size_t)R);
        HB(hb_predict_ex(a, dX, R, F, HB_OUT_LEAF_HASH, dH, s));
        CU(cudaStreamSynchronize(s));
        CU(cudaMemcpy(hA, dH, 8 * (size_t)R, cudaMemcpyDeviceToHost));
        HB(hb_predict_ex(b, dX, R, F, HB_OUT_LEAF_HASH, dH, s));
        CU(cudaStreamSynchronize(s));
        CU(cudaMemcpy(hH, dH, 8 * (size_t)R, cudaMemcpyDeviceToHost));
        for (int r = 0; r < R; ++r) hA[r] += hH[r];
        HB(hb_predict_ex(m, dX, R, F, HB_OUT_LEAF_HASH, dH, s));
        CU(cudaStreamSynchronize(s));
        CU(cudaMemcpy(hH, dH, 8 * (size_t)R, cudaMemcpyDeviceToHost));
        for (int r = 0; r < R; ++r) CHECK(hA[r] == hH[r], "shard leaf hash row %d", r);
        free(h1); free(h2); free(hA);
        cudaFree(dR2);
      }
      hb_free(a);
      hb_free(b);
      hb_free(m);
    }
  }
  /* argument errors */
  hb_model *none = NULL;
  CHECK(hb_compile(NULL, 0, 0, &none) == HB_E_INVALID && none == NULL, "NULL ensemble");
  CHECK(hb_predict(NULL, dX, R, F, dF, s) == HB_E_INVALID, "NULL model");

  cudaStreamDestroy(s);
  cudaFree(dX); cudaFree(dF); cudaFree(dD); cudaFree(dL); cudaFree(dH);
  if (failures) {
    fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  printf("abi_smoke: all checks passed (%d trees, %d rows, 4 strategies x LT/LE)\n", T, R);
  return 0;
}
