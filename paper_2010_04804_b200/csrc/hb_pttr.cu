// hb_pttr.cu — PerfectTreeTraversal with rank-coded thresholds (sm_100a).
//
// Same algorithm as hb_ptt.cu (Alg. 3), same results bit
// for bit, with 4-byte instead of 8-byte node records:
//
//  * Compile time: for every feature f used by the model, the distinct
//    thresholds u_0 < ... < u_{m-1} (fp32 order) are collected. A node that
//    tests (f, u_k) stores k and the compact feature index.
//  * Per row tile, each X value is replaced by its rank code
//        LT: c(x) = #{j : u_j <= x}      LE: c(x) = #{j : u_j <  x}
//    and NaN by 0xFFFF. Then  x < u_k  <=>  c(x) <= k  (LE:  x <= u_k <=> c(x) <= k)
//    for every x, so the integer walk takes exactly the fp32 walk's branches.
//  * The code is computed by walking a perfect binary search tree over the u_j
//    in Eytzinger (heap) order — itself a perfect-tree traversal: after L =
//    bit_length(m) steps of  i <- 2 i + pred(e_i, x)  the rank is i - 2^L
//    (padding slots hold NaN, so pred is false there, i.e. they sort last).
//
// Why: a warp-wide LDS.64 is served in two half-warp passes, so 8-B node
// records cost >= 2 SMEM wavefronts per level; a 4-B record costs 1 when the
// level's nodes are distinct banks. The bank-conflict model of DESIGN.md §4.1
// (validated against ncu: 31.9 vs 31.1 wavefronts per warp-tree) gives 20.3
// wavefronts per warp-tree for this layout, plus ~7% for the per-tile code
// transform.
//
// Node record: u32 = (fc * 128) << 16 | k. The per-warp code tile holds
// cell[fc][lane] = (fc * 128) << 16 | c(x) as u32, so lane l always reads bank l
// (conflict-free whatever feature it needs), the cell address is one LEA.HI
// (tile + (node >> 16)), and since node and cell share the high half, "go
// left" is the single unsigned compare  node >= cell  <=>  k >= c(x)
// (n_fc <= 511 so that fc * 128 fits 16 bits).
// Leaf layout makes the leaf address equal to the final heap byte offset: tree
// record = node[2^D] (node[0] = tree_output) then leaf[2^D] (w = 1), so after D
// levels off = 4 i with i in [2^D, 2^(D+1)) and leaf(i - 2^D) sits at off.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "hb_internal.h"
#include "hb_pttr_kernel.cuh"

namespace hb {

struct RankAux {
  // per compact feature: {orig feature, L, byte offset inside its group, group}
  // per group: {byte offset in the eytzinger pool, bytes, fc_begin, fc_end}
  std::vector<uint32_t> fmeta, groups;
  std::vector<float> pool;
  int n_fc = 0, n_groups = 0;
  size_t max_feat_bytes = 0;
};

static int bit_length(uint32_t m) {
  int L = 0;
  while ((1u << L) <= m) ++L;
  return L;  // 2^L - 1 >= m
}

static void eytz_fill(const std::vector<float> &sorted, std::vector<float> &out, int L, int p,
                      size_t &next) {
  if (p >= (1 << L)) return;
  eytz_fill(sorted, out, L, 2 * p, next);
  out[p] = next < sorted.size() ? sorted[next] : NAN;
  ++next;
  eytz_fill(sorted, out, L, 2 * p + 1, next);
}

static int env_int2(const char *name, int dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoi(v);
}

// Builds the rank-coded layout; returns HB_E_UNSUPPORTED (and leaves m intact)
// when the model does not qualify (caller then uses the fp32 PTT layout).
hb_status compile_ptt_rank(const hb_ensemble *e, int t0, int t1, int D, Model *m, int nw_fp32) {
  if (env_int2("HB_PTT_RANK", -1) == 0) return HB_E_UNSUPPORTED;
  const int F = e->n_features, w = e->leaf_width;
  const TreeOrder order = ptt_order(e, t0, t1, true);
  const int Tpad = (int)order.local.size();
  // 1. distinct thresholds per feature
  std::vector<std::vector<float>> th(F);
  for (int t = t0; t < t1; ++t)
    for (int64_t i = e->node_offset[t]; i < e->node_offset[t + 1]; ++i)
      if (e->left[i] != -1) {
        float v = e->threshold[i];
        if (v == 0.f) v = 0.f;  // -0 == +0 under IEEE compare
        th[e->feature[i]].push_back(v);
      }
  std::vector<int> fc_of(F, -1);
  RankAux A;
  std::vector<std::vector<float>> sorted;
  for (int f = 0; f < F; ++f) {
    if (th[f].empty()) continue;
    std::vector<float> &v = th[f];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    if (v.size() > 65534) return HB_E_UNSUPPORTED;
    fc_of[f] = A.n_fc++;
    sorted.push_back(v);
  }
  if (A.n_fc > 1023) return HB_E_UNSUPPORTED;   // node offsets must fit 16 bits
  const int P = 1 << D;
  const size_t stride = (4 * (size_t)P + 4 * (size_t)w * P + 15) & ~size_t(15);
  // Eytzinger search arrays (grouped later by stage size)
  std::vector<std::vector<float>> ey(A.n_fc);
  std::vector<int> Ls(A.n_fc);
  for (int c = 0; c < A.n_fc; ++c) {
    const int L = bit_length((uint32_t)sorted[c].size());
    Ls[c] = L;
    ey[c].assign(std::max(4, 1 << L), NAN);   // >= 16 B, slot 0 unused
    size_t next = 0;
    eytz_fill(sorted[c], ey[c], L, 1, next);
    A.max_feat_bytes = std::max(A.max_feat_bytes, ey[c].size() * 4);
  }
  // launch configuration: X code tile NW * tile_bytes + a 2-stage ring. Every
  // consumer warp waits for every ring item, so items should be large: the
  // largest tree chunk that fits (<= 64 trees) for the most warps. Measured on
  // B200: C3 24 warps x 2 stages x 32 trees = 700M rows/s vs
  // 520M with 16-tree chunks. 32-bit cells first; 16-bit cells (half the
  // tile, one more instruction per level) when they buy more warps.
  const int force = env_int2("HB_PTT_RANK", -1);
  const int force_cw = env_int2("HB_RANK_CW", 0);
  const int force_nw = env_int2("HB_NW", 0);
  const int force_pre = env_int2("HB_RANK_PRE", -1);
  // pre: codes come from the pre-pass (hb_rank_codes.cu), the ring carries
  // tree chunks only; otherwise the ring also carries the Eytzinger arrays
  auto try_cfg = [&](int cw, bool pre, LaunchCfg &cfg) {
    if (cw == 32 && A.n_fc > 511) return false;
    const long tile = cw == 32 ? (long)A.n_fc * 128 : (long)((A.n_fc + 1) / 2) * 128;
    for (int nw : {24, 16, 12, 8, 4}) {
      if (force_nw && nw != force_nw) continue;
      const long xb = (long)nw * tile;
      const long rem = (long)kSmemBudget - xb;
      const int ns = env_int2("HB_NS", 2);
      const long per = rem / ns - 16;
      if ((!pre && per < (long)A.max_feat_bytes) || per < (long)kTreeGroup * (long)stride) continue;
      int ch = (int)std::min<long>(env_int2("HB_CH", 64), per / (long)stride) & ~(kTreeGroup - 1);
      ch = std::min(ch, Tpad);
      const long stage = pre ? (long)ch * stride : std::max<long>((long)ch * stride, (long)A.max_feat_bytes);
      cfg.nw = nw;
      cfg.ns = ns;
      cfg.ch = ch;
      cfg.x_smem = 1;
      cfg.t_smem = 1;
      cfg.stage_bytes = (int)((stage + 127) & ~127L);
      cfg.smem_bytes = (int)(xb + (long)ns * cfg.stage_bytes + 16 * ns);
      if (cfg.smem_bytes <= kSmemBudget) return true;
    }
    return false;
  };
  // 32-bit cells first; 16-bit cells (half the tile, one more instruction
  // per level) when they buy more warps
  auto pick_cw = [&](bool pre, LaunchCfg &cfg, int &cw) {
    LaunchCfg c32, c16;
    const bool ok32 = force_cw != 16 && try_cfg(32, pre, c32);
    const bool ok16 = force_cw != 32 && try_cfg(16, pre, c16);
    if (ok16 && (!ok32 || force_cw == 16 || c16.nw > c32.nw)) {
      cfg = c16;
      cw = 16;
      return true;
    }
    cfg = c32;
    cw = 32;
    return ok32;
  };
  LaunchCfg cfg;
  int cw = 32;
  bool pre = force_pre == 1;
  bool ok = !pre && pick_cw(false, cfg, cw);
  // auto: in-kernel codes only when (a) the per-tile rank
  // transform (sum_f L_f searches per row) stays small next to the walk it
  // shortens (T * D levels per row) and (b) the layout runs at least as many
  // warps as the fp32-node layout would (occupancy decides at equal bytes).
  // Otherwise the pre-pass computes the codes (cost: one more read of X, and
  // a write + read of the code words, in HBM).
  if (ok && force != 1) {
    double lsum = 0;
    for (int c = 0; c < A.n_fc; ++c) lsum += Ls[c];
    if (lsum > 0.2 * (double)Tpad * (double)std::max(D, 1)) ok = false;
    if (cfg.nw < nw_fp32) ok = false;
  }
  if (ok && force_pre == -1 && force_cw == 0) {
    // when the pre-pass layout runs 32-bit cells (one instruction less per
    // level than 16-bit ones) at no fewer warps, it wins: the scorer then
    // only copies codes and its ring carries trees only (C3: 742.8M vs 704.1M
    // rows/s; C4, whose in-kernel layout needs 16-bit cells: 107.0M vs
    // 98.9M). With 16-bit pre-pass cells it does not (C4': 404.8M vs 420.8M).
    LaunchCfg pc;
    int pcw = 32;
    if (pick_cw(true, pc, pcw) && pcw == 32 && pc.nw >= cfg.nw) {
      pre = true;
      cfg = pc;
      cw = pcw;
    }
  }
  if (!ok && force_pre != 0) {
    pre = true;
    ok = pick_cw(true, cfg, cw);
  }
  if (!ok) return HB_E_UNSUPPORTED;
  // tree records: node = (cell offset) << 16 | k
  auto cell_off = [&](int fc) -> uint32_t {
    return cw == 32 ? (uint32_t)fc * 128u : (uint32_t)(fc >> 1) * 128u + (uint32_t)(fc & 1) * 2u;
  };
  std::vector<uint8_t> buf((size_t)Tpad * stride, 0);
  std::vector<int32_t> leafmap((size_t)Tpad * P, -1);
  std::vector<int> orig(2 * P);
  const uint32_t kPad = 0x0000FFFFu;  // column 0, k = 0xFFFF >= any code: always left
  for (int lt = 0; lt < Tpad; ++lt) {
    uint8_t *rec = buf.data() + (size_t)lt * stride;
    uint32_t *node = reinterpret_cast<uint32_t *>(rec);
    float *leaf = reinterpret_cast<float *>(rec + 4 * (size_t)P);
    for (int p = 1; p < P; ++p) node[p] = kPad;
    node[0] = ptt_header(order, lt);
    if (order.local[lt] < 0) continue;   // zero tree (padding)
    const int t = t0 + order.local[lt];
    const int64_t a = e->node_offset[t];
    orig[1] = 0;
    for (int p = 1; p < P; ++p) {
      const int o = orig[p];
      if (e->left[a + o] != -1) {
        const int f = e->feature[a + o];
        float v = e->threshold[a + o];
        if (v == 0.f) v = 0.f;
        const std::vector<float> &u = sorted[fc_of[f]];
        const uint32_t k = (uint32_t)(std::lower_bound(u.begin(), u.end(), v) - u.begin());
        node[p] = (cell_off(fc_of[f]) << 16) | k;
        orig[2 * p] = e->left[a + o];
        orig[2 * p + 1] = e->right[a + o];
      } else {
        orig[2 * p] = orig[2 * p + 1] = o;
      }
    }
    for (int p = P; p < 2 * P; ++p) {
      const int o = D == 0 ? 0 : orig[p];
      const int slot = p - P;
      for (int k = 0; k < w; ++k) leaf[(size_t)slot * w + k] = e->leaf_value[(a + o) * w + k];
      leafmap[(size_t)lt * P + slot] = o;
    }
  }
  if (!pre) {
    // 5. group features into stage-sized bulk copies
    {
      size_t goff = 0, gbytes = 0;
      int gbeg = 0;
      auto close = [&](int end) {
        A.groups.insert(A.groups.end(), {(uint32_t)goff, (uint32_t)gbytes, (uint32_t)gbeg, (uint32_t)end});
        goff += gbytes;
        gbytes = 0;
        gbeg = end;
        A.n_groups++;
      };
      for (int c = 0; c < A.n_fc; ++c) {
        const size_t b = ey[c].size() * 4;
        if (gbytes + b > (size_t)cfg.stage_bytes) close(c);
        A.fmeta.insert(A.fmeta.end(), {0u, (uint32_t)Ls[c], (uint32_t)gbytes, (uint32_t)A.n_groups});
        gbytes += b;
        A.pool.insert(A.pool.end(), ey[c].begin(), ey[c].end());
      }
      if (gbytes) close(A.n_fc);
      int c = 0;
      for (int f = 0; f < F; ++f)
        if (fc_of[f] >= 0) A.fmeta[4 * c++] = (uint32_t)f;
    }
  }
  // 6. upload: trees, leafmap, aux = [fmeta | groups | pool]
  cudaError_t err;
  if ((err = cudaMalloc(&m->d_trees, buf.size())) != cudaSuccess) return cuda_fail(err, "cudaMalloc(pttr)");
  m->device_bytes += buf.size();
  if ((err = cudaMemcpy(m->d_trees, buf.data(), buf.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(err, "cudaMemcpy(pttr)");
  if ((err = cudaMalloc(&m->d_leafmap, leafmap.size() * 4)) != cudaSuccess)
    return cuda_fail(err, "cudaMalloc(pttr leafmap)");
  m->device_bytes += leafmap.size() * 4;
  if ((err = cudaMemcpy(m->d_leafmap, leafmap.data(), leafmap.size() * 4, cudaMemcpyHostToDevice)) !=
      cudaSuccess)
    return cuda_fail(err, "cudaMemcpy(pttr leafmap)");
  if (!pre) {
    const size_t fb = A.fmeta.size() * 4, gb = A.groups.size() * 4, pb = A.pool.size() * 4;
    const size_t pool_off = (fb + gb + 127) & ~size_t(127);
    std::vector<uint8_t> aux(pool_off + pb, 0);
    std::memcpy(aux.data(), A.fmeta.data(), fb);
    std::memcpy(aux.data() + fb, A.groups.data(), gb);
    std::memcpy(aux.data() + pool_off, A.pool.data(), pb);
    if ((err = cudaMalloc(&m->d_aux, aux.size())) != cudaSuccess) return cuda_fail(err, "cudaMalloc(pttr aux)");
    m->device_bytes += aux.size();
    if ((err = cudaMemcpy(m->d_aux, aux.data(), aux.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return cuda_fail(err, "cudaMemcpy(pttr aux)");
    m->aux_groups_off = fb;
    m->aux_pool_off = pool_off;
    m->rank_ngroups = A.n_groups;
  } else {
    // pre-pass bucket tables: [feat | groups | pool]
    std::vector<int> origf;
    for (int f = 0; f < F; ++f)
      if (fc_of[f] >= 0) origf.push_back(f);
    RankBuckets R;
    const hb_status st = build_rank_buckets(sorted, origf, cw, &R);
    if (st != HB_OK) return st;
    const size_t fb = R.feat.size() * 4, gb = R.groups.size() * 4;
    const size_t pool_off = (fb + gb + 127) & ~size_t(127);
    std::vector<uint8_t> aux(pool_off + R.pool.size(), 0);
    std::memcpy(aux.data(), R.feat.data(), fb);
    std::memcpy(aux.data() + fb, R.groups.data(), gb);
    std::memcpy(aux.data() + pool_off, R.pool.data(), R.pool.size());
    if ((err = cudaMalloc(&m->d_rb, aux.size())) != cudaSuccess) return cuda_fail(err, "cudaMalloc(rank tables)");
    m->device_bytes += aux.size();
    if ((err = cudaMemcpy(m->d_rb, aux.data(), aux.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return cuda_fail(err, "cudaMemcpy(rank tables)");
    m->rb_groups_off = fb;
    m->rb_pool_off = pool_off;
    m->rb_ngroups = R.n_groups;
    m->rb_smem = R.max_group_bytes;
    m->rb_smem_cap = R.smem_cap;
    m->rb_max_span = R.max_span;
    m->rb_global = R.any_global;
    m->rank_nwords = R.n_words;
    m->rank_ngroups = 0;
    // per-call code scratch: stream-ordered allocations from a model-owned
    // pool that keeps its memory (no cudaMalloc on the scoring path)
    const hb_status pst = ensure_pool(m);
    if (pst != HB_OK) return pst;
  }
  m->rank_pre = pre ? 1 : 0;
  m->rank_nfc = A.n_fc;
  m->stride = stride;
  m->nslots = P;
  m->cfg = cfg;
  m->ptt_rank = 1;
  m->n_trees_pad = Tpad;
  m->rank_cw = cw;
  return HB_OK;
}

int sm_count(int device);

hb_status launch_ptt_rank(const Model &m, const RunArgs &a) {
  PttrFn fn = m.rank_cw == 16 ? pttr_fn16(m.depth, m.cmp == HB_CMP_LE, m.nacc)
                              : pttr_fn32(m.depth, m.cmp == HB_CMP_LE, m.nacc);
  if (!fn) return fail(HB_E_UNSUPPORTED, "PTT depth out of range");
  PttrParams p;
  // pre-pass: rank codes of every (row, used feature) into stream-ordered
  // scratch, in the per-warp tile layout the scorer copies verbatim
  uint32_t *codes = nullptr;
  cudaError_t e;
  if (m.rank_pre) {
    const int64_t nblocks = (a.n + 31) / 32;
    const size_t bytes = std::max<size_t>((size_t)nblocks * m.rank_nwords * 128, 128);
    const hb_status ast = scratch_alloc(m, bytes, a.stream, reinterpret_cast<void **>(&codes));
    if (ast != HB_OK) return ast;
    const hb_status st = launch_rank_codes(m, a, codes, nblocks);
    if (st != HB_OK) {
      cudaFreeAsync(codes, a.stream);
      return st;
    }
  }
  p.codes = codes;
  p.n_words = m.rank_nwords;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.trees = static_cast<const uint8_t *>(m.d_trees);
  p.stride = (uint32_t)m.stride;
  p.n_trees_pad = m.n_trees_pad;
  p.n_trees = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.leafmap = m.d_leafmap;
  p.nslots = m.nslots;
  const uint8_t *aux = static_cast<const uint8_t *>(m.d_aux);
  p.fmeta = reinterpret_cast<const uint4 *>(aux);
  p.groups = reinterpret_cast<const uint4 *>(aux + m.aux_groups_off);
  p.pool = aux + m.aux_pool_off;
  p.n_fc = m.rank_nfc;
  p.n_groups = m.rank_ngroups;
  p.F = m.n_features;
  p.vec4 = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);
  p.x_direct = m.rank_cw == 32 && m.rank_nfc == m.n_features;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  p.prefetch = m.cfg.prefetch;
  p.nw = m.cfg.nw;
  p.ns = m.cfg.ns;
  p.ch = m.cfg.ch;
  p.stage_bytes = (uint32_t)m.cfg.stage_bytes;
  const int64_t rows_per_tile = (int64_t)m.cfg.nw * 32;
  const int64_t ntiles = (a.n + rows_per_tile - 1) / rows_per_tile;
  if (ntiles > INT32_MAX) {
    if (codes) cudaFreeAsync(codes, a.stream);
    return fail(HB_E_UNSUPPORTED, "too many rows for one launch");
  }
  p.ntiles = (int)ntiles;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count(m.device) * m.cfg.ctas_per_sm);
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m.cfg.smem_bytes);
  if (e == cudaSuccess) {
    if (codes) mark_launch(a);     // scorer starts (the pre-pass was launch 0)
    fn<<<grid, 32 * (m.cfg.nw + 1), m.cfg.smem_bytes, a.stream>>>(p);
    e = cudaGetLastError();
  }
  if (codes) cudaFreeAsync(codes, a.stream);
  if (e != cudaSuccess) return cuda_fail(e, "pttr_kernel launch");
  return HB_OK;
}

}  // namespace hb
