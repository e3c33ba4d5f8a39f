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

namespace hb {

constexpr int kGemmMaxInternal = 64;   // T fits one 64-bit word

// per-tree record (all fields 8-B aligned):
//   u32 hdr[2] = {tree_output, 0}
//   u32 feat[NI]; f32 thr[NI]                 (NI padded to even)
//   u64 lmask[NL]; u64 rmask[NL]; u32 D[NL] (NL padded to even)
//   f32 E[NL * w]
struct GemmGeom {
  int ni, nl, w;
  size_t off_feat, off_thr, off_lm, off_rm, off_d, off_e, stride;
};

static GemmGeom gemm_geom(int ni, int nl, int w) {
  GemmGeom g;
  g.ni = (ni + 1) & ~1;
  g.nl = (nl + 1) & ~1;
  g.w = w;
  size_t o = 8;
  g.off_feat = o; o += 4 * (size_t)g.ni;
  g.off_thr = o;  o += 4 * (size_t)g.ni;
  g.off_lm = o;   o += 8 * (size_t)g.nl;
  g.off_rm = o;   o += 8 * (size_t)g.nl;
  g.off_d = o;    o += 4 * (size_t)g.nl;
  g.off_e = o;    o += 4 * (size_t)g.nl * w;
  g.stride = (o + 15) & ~size_t(15);
  return g;
}

bool gemm_supported(int depth) { return depth <= 6; }

hb_status compile_gemm(const hb_ensemble *e, int t0, int t1, Model *m) {
  const int w = e->leaf_width;
  int ni = 1, nl = 1;
  for (int t = t0; t < t1; ++t) {
    const int64_t a = e->node_offset[t], b = e->node_offset[t + 1];
    int ci = 0, cl = 0;
    for (int64_t i = a; i < b; ++i) (e->left[i] == -1 ? cl : ci)++;
    ni = std::max(ni, ci);
    nl = std::max(nl, cl);
  }
  if (ni > kGemmMaxInternal)
    return fail(HB_E_UNSUPPORTED, "GEMM: trees with more than 64 internal nodes (use PTT/TT)");
  const GemmGeom g = gemm_geom(ni, nl, w);
  const int Tpad = m->n_trees_pad;
  std::vector<uint8_t> buf((size_t)Tpad * g.stride, 0);
  std::vector<int32_t> leafmap((size_t)Tpad * g.nl, -1);
  std::vector<int> ipos, lpos, stack;
  for (int lt = 0; lt < Tpad; ++lt) {
    uint8_t *rec = buf.data() + (size_t)lt * g.stride;
    uint32_t *hdr = reinterpret_cast<uint32_t *>(rec);
    float *thr = reinterpret_cast<float *>(rec + g.off_thr);
    uint32_t *feat = reinterpret_cast<uint32_t *>(rec + g.off_feat);
    uint64_t *lm = reinterpret_cast<uint64_t *>(rec + g.off_lm);
    uint64_t *rm = reinterpret_cast<uint64_t *>(rec + g.off_rm);
    uint32_t *D = reinterpret_cast<uint32_t *>(rec + g.off_d);
    float *E = reinterpret_cast<float *>(rec + g.off_e);
    for (int i = 0; i < g.ni; ++i) thr[i] = INFINITY;  // padded nodes: C rows are 0
    for (int j = 0; j < g.nl; ++j) D[j] = 0xFFFFu;      // padded leaves: unreachable D
    if (lt >= t1 - t0) {
      D[0] = 0;  // zero tree: column 0 (C = 0, D = 0) always matches, E = 0
      continue;
    }
    const int t = t0 + lt;
    const int64_t a = e->node_offset[t];
    const int n = (int)(e->node_offset[t + 1] - a);
    hdr[0] = (uint32_t)(w == 1 ? (e->tree_output ? e->tree_output[t] : t % e->n_outputs) : 0);
    // ordered lists I and L (node-id order, Table 3)
    ipos.assign(n, -1);
    lpos.assign(n, -1);
    int ci = 0, cl = 0;
    for (int i = 0; i < n; ++i) {
      if (e->left[a + i] != -1) ipos[i] = ci++;
      else lpos[i] = cl++;
    }
    for (int i = 0; i < n; ++i) {
      if (ipos[i] >= 0) {
        feat[ipos[i]] = (uint32_t)e->feature[a + i];
        thr[ipos[i]] = e->threshold[a + i];
      } else {
        const int j = lpos[i];
        for (int k = 0; k < w; ++k) E[(size_t)j * w + k] = e->leaf_value[(a + i) * w + k];
        leafmap[(size_t)lt * g.nl + j] = i;
      }
    }
    // C: +1 for leaves in the left subtree of internal node i, -1 right.
    for (int i = 0; i < n; ++i) {
      if (ipos[i] < 0) continue;
      for (int side = 0; side < 2; ++side) {
        stack.assign(1, side == 0 ? e->left[a + i] : e->right[a + i]);
        while (!stack.empty()) {
          const int k = stack.back();
          stack.pop_back();
          if (e->left[a + k] == -1) {
            (side == 0 ? lm : rm)[lpos[k]] |= 1ull << ipos[i];
          } else {
            stack.push_back(e->left[a + k]);
            stack.push_back(e->right[a + k]);
          }
        }
      }
    }
    for (int j = 0; j < cl; ++j) D[j] = (uint32_t)__builtin_popcountll(lm[j]);
  }
  m->stride = g.stride;
  m->nslots = g.nl;
  m->gemm_ni = g.ni;
  m->gemm_nl = g.nl;
  size_t acct = 0;
  cudaError_t err = cudaMalloc(&m->d_trees, buf.size());
  if (err != cudaSuccess) return cuda_fail(err, "cudaMalloc(gemm)");
  m->device_bytes += buf.size();
  err = cudaMemcpy(m->d_trees, buf.data(), buf.size(), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) return cuda_fail(err, "cudaMemcpy(gemm)");
  err = cudaMalloc(&m->d_leafmap, leafmap.size() * 4);
  if (err != cudaSuccess) return cuda_fail(err, "cudaMalloc(gemm leafmap)");
  m->device_bytes += leafmap.size() * 4;
  err = cudaMemcpy(m->d_leafmap, leafmap.data(), leafmap.size() * 4, cudaMemcpyHostToDevice);
  if (err != cudaSuccess) return cuda_fail(err, "cudaMemcpy(gemm leafmap)");
  (void)acct;
  m->cfg = LaunchCfg();
  m->cfg.nw = 4;
  m->cfg.x_smem = 0;
  m->cfg.t_smem = 0;
  return HB_OK;
}

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
