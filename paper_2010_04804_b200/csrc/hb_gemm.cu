// hb_gemm.cu — GEMM strategy (Alg. 1; Table 3).
//
// Alg. 1 per tree:  T <- X.A ; T <- T < B ; S <- T.C ; T <- S == D ; R <- T.E.
// Compiled tensors (per tree, zero-padded to the max |I| / |L| over trees as
// P:192 says, with padded leaf columns masked by an unreachable D, reading R7):
//   A   as a feature-id vector (never a dense one-hot matrix: X.A by a real
//       multiply turns one Inf/NaN in a row into NaN at every node, V4),
//   B   fp32 thresholds,
//   C   {-1,0,+1} [|I| x |L|] stored as two bit masks per leaf column
//       (Lmask_j = {i : C_ij = +1}, Rmask_j = {i : C_ij = -1}),
//   D   left-edge counts (reading R5),
//   E   fp32 leaf values [|L| x w].
// The path contraction S_j = sum_i T_i C_ij is evaluated exactly as
// popc(T & Lmask_j) - popc(T & Rmask_j) and compared with D_j; exactly one
// real column matches (proof in DESIGN.md §2.2). The tensor-core variant of
// this contraction is hb_gemm_tc.cu.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "hb_device.cuh"
#include "hb_internal.h"
#include "hb_layouts.h"

namespace hb {

struct GemmParams {
  const float *X;
  int64_t n, ldx;
  const uint8_t *trees;
  uint32_t stride, off_feat, off_thr, off_lm, off_rm, off_d, off_e;
  int ni, nl;
  int n_trees_pad, n_trees, tree_begin;
  const int32_t *leafmap;
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
};

template <bool LE, int NACC>
__global__ void __launch_bounds__(128) gemm_kernel(const GemmParams p) {
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const float *xr = p.X + (row < p.n ? row : 0) * p.ldx;
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  double acc[NACC];   // fp64 accumulation (R23)
#pragma unroll
  for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
  uint64_t h = 0;
  for (int t = 0; t < p.n_trees_pad; ++t) {
    const uint8_t *rec = p.trees + (size_t)t * p.stride;
    const uint32_t *feat = reinterpret_cast<const uint32_t *>(rec + p.off_feat);
    const float *thr = reinterpret_cast<const float *>(rec + p.off_thr);
    // T <- (X.A < B): exact gathers + fp32 compares -> bit vector
    uint64_t T = 0;
    for (int i = 0; i < p.ni; ++i) {
      const float x = __ldg(xr + __ldg(feat + i));
      const float b = __ldg(thr + i);
      const bool pr = LE ? (x <= b) : (x < b);
      T |= (uint64_t)pr << i;
    }
    // S <- T.C ; T <- S == D  (integer contraction, exact)
    const uint64_t *lmk = reinterpret_cast<const uint64_t *>(rec + p.off_lm);
    const uint64_t *rmk = reinterpret_cast<const uint64_t *>(rec + p.off_rm);
    const uint32_t *D = reinterpret_cast<const uint32_t *>(rec + p.off_d);
    int sel = 0;
    for (int j = 0; j < p.nl; ++j) {
      const int S = __popcll(T & __ldg(lmk + j)) - __popcll(T & __ldg(rmk + j));
      if (S == (int)__ldg(D + j)) sel = j;
    }
    // R <- T.E : gather the selected leaf's value(s)
    const float *E = reinterpret_cast<const float *>(rec + p.off_e);
    if (p.w == 1) {
      const double v = (double)__ldg(E + sel);
      const uint32_t k0 = __ldg(reinterpret_cast<const uint32_t *>(rec));
#pragma unroll
      for (int k = 0; k < NACC; ++k)
        if (k0 == (uint32_t)k) acc[k] += v;
    } else {
#pragma unroll
      for (int k = 0; k < NACC; ++k)
        if (k < p.K) acc[k] += (double)__ldg(E + sel * p.w + k);
    }
    if (lm && t < p.n_trees) {
      const int32_t id = __ldg(p.leafmap + (size_t)t * p.nl + sel);
      if (lm == 1) {
        if (row < p.n) static_cast<int32_t *>(p.out)[row * p.n_trees + t] = id;
      } else {
        h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + t) << 32) | (uint32_t)id);
      }
    }
  }
  if (row < p.n) {
    if (lm == 2) static_cast<uint64_t *>(p.out)[row] = h;
    else if (lm == 0) dev::write_row<NACC>(p.kind, acc, p.K, p.task, p.post, p.scale, p.base, row, p.out);
  }
}

using GemmFn = void (*)(const GemmParams);

template <bool LE>
static GemmFn pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return gemm_kernel<LE, 1>;
    case 4: return gemm_kernel<LE, 4>;
    case 8: return gemm_kernel<LE, 8>;
    default: return gemm_kernel<LE, 16>;
  }
}

hb_status launch_gemm(const Model &m, const RunArgs &a) {
  if (m.gemm_tc) return launch_gemm_tc(m, a);
  const GemmGeom g = gemm_geom(m.gemm_ni, m.gemm_nl, m.leaf_width);
  GemmParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.trees = static_cast<const uint8_t *>(m.d_trees);
  p.stride = (uint32_t)g.stride;
  p.off_feat = (uint32_t)g.off_feat;
  p.off_thr = (uint32_t)g.off_thr;
  p.off_lm = (uint32_t)g.off_lm;
  p.off_rm = (uint32_t)g.off_rm;
  p.off_d = (uint32_t)g.off_d;
  p.off_e = (uint32_t)g.off_e;
  p.ni = g.ni;
  p.nl = g.nl;
  p.n_trees_pad = m.n_trees_pad;
  p.n_trees = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.leafmap = m.d_leafmap;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  GemmFn fn = m.cmp == HB_CMP_LE ? pick_nacc<true>(m.nacc) : pick_nacc<false>(m.nacc);
  const int threads = 128;
  const int64_t blocks = (a.n + threads - 1) / threads;
  if (blocks > INT32_MAX) return fail(HB_E_UNSUPPORTED, "too many rows");
  fn<<<(int)blocks, threads, 0, a.stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "gemm_kernel launch");
  return HB_OK;
}

}  // namespace hb
