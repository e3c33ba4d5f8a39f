// hb_host.cpp — the C ABI (include/hb.h): validation, strategy selection
// (Sec. 5.1), layout compilation for the three strategies
// (Tables 3/5/6) and the scoring entry points.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "hb_internal.h"
#include "hb_layouts.h"

namespace hb {

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

void set_error(const std::string &s) { g_err = s; }

hb_status fail(hb_status st, const std::string &s) {
  g_err = s;
  return st;
}

hb_status cuda_fail(cudaError_t e, const char *what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? HB_E_OOM : HB_E_CUDA;
}

int sm_count(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (cache[device] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
      v = 148;
    cache[device] = v;
  }
  return cache[device];
}

// Keeps the caller's current device intact around library calls.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (dev < 0) return;           // host-only compile: no CUDA call at all
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------------ validation
struct TreeInfo {
  int depth = 0;
  int n_nodes = 0;
};

static hb_status validate_impl(const hb_ensemble *e, std::vector<TreeInfo> *info) {
  if (!e) return fail(HB_E_INVALID, "ensemble is NULL");
  const int T = e->n_trees, F = e->n_features, K = e->n_outputs, w = e->leaf_width;
  if (T < 1) return fail(HB_E_TREE, "n_trees must be >= 1");
  if (F < 1) return fail(HB_E_TREE, "n_features must be >= 1");
  if (K < 1) return fail(HB_E_TREE, "n_outputs must be >= 1");
  if (w != 1 && w != K) return fail(HB_E_TREE, "leaf_width must be 1 or n_outputs");
  if (!e->node_offset || !e->feature || !e->threshold || !e->left || !e->right || !e->leaf_value)
    return fail(HB_E_INVALID, "ensemble array pointer is NULL");
  if (e->cmp != HB_CMP_LT && e->cmp != HB_CMP_LE)
    return fail(HB_E_UNSUPPORTED, "cmp must be HB_CMP_LT or HB_CMP_LE (GT/GE would change NaN routing)");
  if (e->agg != HB_AGG_SUM && e->agg != HB_AGG_MEAN) return fail(HB_E_TREE, "bad agg");
  if (e->post < HB_POST_IDENTITY || e->post > HB_POST_ISOLATION) return fail(HB_E_TREE, "bad post");
  if (e->post == HB_POST_ISOLATION &&
      (K != 1 || e->task != HB_TASK_REGRESSION || !(e->post_param > 0.f) || !std::isfinite(e->post_param)))
    return fail(HB_E_TREE, "ISOLATION requires n_outputs == 1, REGRESSION and post_param > 0");
  if (e->task != HB_TASK_REGRESSION && e->task != HB_TASK_CLASSIFICATION)
    return fail(HB_E_TREE, "bad task");
  if (e->post == HB_POST_SIGMOID && K != 1) return fail(HB_E_TREE, "SIGMOID requires n_outputs == 1");
  if (e->post == HB_POST_SOFTMAX && K < 2) return fail(HB_E_TREE, "SOFTMAX requires n_outputs >= 2");
  if (e->task == HB_TASK_CLASSIFICATION && !((K == 1 && e->post == HB_POST_SIGMOID) || K >= 2))
    return fail(HB_E_TREE, "CLASSIFICATION requires (K == 1 and SIGMOID) or K >= 2");
  if (e->node_offset[0] != 0) return fail(HB_E_TREE, "node_offset[0] must be 0");
  if (e->tree_output && w == 1)
    for (int t = 0; t < T; ++t)
      if (e->tree_output[t] < 0 || e->tree_output[t] >= K)
        return fail(HB_E_TREE, "tree " + std::to_string(t) + ": tree_output out of range");
  if (e->base_score)
    for (int k = 0; k < K; ++k)
      if (!std::isfinite(e->base_score[k])) return fail(HB_E_TREE, "base_score must be finite");
  if (info) info->assign(T, TreeInfo());
  std::vector<int> pc, depth, queue;
  for (int t = 0; t < T; ++t) {
    const int64_t a = e->node_offset[t], b = e->node_offset[t + 1];
    const std::string where = "tree " + std::to_string(t);
    if (b <= a) return fail(HB_E_TREE, where + ": has no nodes (offsets not increasing)");
    if (b - a > (int64_t)INT32_MAX) return fail(HB_E_TREE, where + ": too many nodes");
    const int n = (int)(b - a);
    pc.assign(n, 0);
    for (int i = 0; i < n; ++i) {
      const int L = e->left[a + i], R = e->right[a + i];
      const std::string at = where + " node " + std::to_string(i);
      if ((L == -1) != (R == -1)) return fail(HB_E_TREE, at + ": exactly one child is -1");
      if (L != -1) {
        if (L < 0 || L >= n || R < 0 || R >= n) return fail(HB_E_TREE, at + ": child id out of range");
        if (L == R) return fail(HB_E_TREE, at + ": left == right");
        pc[L]++;
        pc[R]++;
        const int f = e->feature[a + i];
        if (f < 0 || f >= F) return fail(HB_E_TREE, at + ": feature out of range");
        if (std::isnan(e->threshold[a + i])) return fail(HB_E_TREE, at + ": threshold is NaN");
      } else {
        for (int k = 0; k < w; ++k)
          if (!std::isfinite(e->leaf_value[(a + i) * w + k]))
            return fail(HB_E_TREE, at + ": leaf value not finite");
      }
    }
    if (pc[0] != 0) return fail(HB_E_TREE, where + ": root (node 0) has a parent");
    for (int i = 1; i < n; ++i)
      if (pc[i] != 1)
        return fail(HB_E_TREE, where + " node " + std::to_string(i) + ": has " +
                                   std::to_string(pc[i]) + " parents (must be exactly 1)");
    depth.assign(n, -1);
    queue.clear();
    queue.push_back(0);
    depth[0] = 0;
    int maxd = 0;
    for (size_t q = 0; q < queue.size(); ++q) {
      const int i = queue[q];
      const int L = e->left[a + i];
      if (L == -1) {
        maxd = std::max(maxd, depth[i]);
        continue;
      }
      const int R = e->right[a + i];
      depth[L] = depth[R] = depth[i] + 1;
      queue.push_back(L);
      queue.push_back(R);
    }
    if ((int)queue.size() != n)
      return fail(HB_E_TREE, where + ": not all nodes reachable from the root (cycle)");
    if (info) {
      (*info)[t].depth = maxd;
      (*info)[t].n_nodes = n;
    }
  }
  return HB_OK;
}

// ------------------------------------------------------------------ layouts
static inline int tree_out(const hb_ensemble *e, int t) {
  return e->tree_output ? e->tree_output[t] : t % e->n_outputs;
}

// Record order of the PTT layouts. For per-class scalar trees (leaf_width 1,
// K > 1) records are sorted by output class (stable) and every class is padded
// with zero trees to a multiple of the kernel's tree group, so a whole ILP
// group shares one class and the kernel selects the accumulator once per group
// (DESIGN.md §4.1). Each record header carries class | (local id + 1) << 8.
TreeOrder ptt_order(const hb_ensemble *e, int t0, int t1, bool by_class) {
  TreeOrder o;
  const int K = e->n_outputs;
  if (by_class && e->leaf_width == 1 && K > 1) {
    for (int k = 0; k < K; ++k) {
      for (int t = t0; t < t1; ++t)
        if (tree_out(e, t) == k) o.local.push_back(t - t0), o.cls.push_back(k);
      while (o.local.size() % kTreeGroup) o.local.push_back(-1), o.cls.push_back(k);
    }
  } else {
    for (int t = t0; t < t1; ++t)
      o.local.push_back(t - t0), o.cls.push_back(e->leaf_width == 1 ? tree_out(e, t) : 0);
    while (o.local.size() % kTreeGroup) o.local.push_back(-1), o.cls.push_back(0);
  }
  return o;
}

uint32_t ptt_header(const TreeOrder &o, size_t r) {
  return (uint32_t)o.cls[r] | ((uint32_t)(o.local[r] + 1) << 8);
}

static inline uint32_t f2u(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

static size_t round16(size_t x) { return (x + 15) & ~size_t(15); }

// Feature-selection injection (Sec. 5.2): "for tree models,
// we update the indices of the decision variables" — used features get
// compact ids in first-use-independent (ascending) order.
struct FeatureMap {
  std::vector<int32_t> remap;    // original -> compact (-1 unused)
  std::vector<int32_t> used;     // compact -> original
  bool identity = true;
};

static int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoi(v);
}

static FeatureMap feature_map(const hb_ensemble *e, int t0, int t1) {
  FeatureMap fm;
  std::vector<char> u(e->n_features, 0);
  for (int t = t0; t < t1; ++t)
    for (int64_t i = e->node_offset[t]; i < e->node_offset[t + 1]; ++i)
      if (e->left[i] != -1) u[e->feature[i]] = 1;
  fm.remap.assign(e->n_features, -1);
  for (int f = 0; f < e->n_features; ++f)
    if (u[f]) {
      fm.remap[f] = (int32_t)fm.used.size();
      fm.used.push_back(f);
    }
  if (fm.used.empty()) fm.used.push_back(0), fm.remap[0] = 0;
  // compact only when it removes a real share of the columns: a compacted
  // tile is filled by per-column gathers through the map, the full one by
  // 16-B row loads — with 6 of 200 features unused (the paper's Fig. 8
  // shape at D3) the gather fill re-read X from DRAM twice (1.50 vs 0.82 GB
  // per launch) and doubled the step (ncu). Threshold:
  // HB_FSEL_MAX_PCT (75) percent of the columns used.
  fm.identity = (long)fm.used.size() * 100 > (long)env_int("HB_FSEL_MAX_PCT", 75) * e->n_features;
  if (fm.identity) {
    fm.used.resize(e->n_features);
    for (int f = 0; f < e->n_features; ++f) fm.remap[f] = f, fm.used[f] = f;
  }
  return fm;
}

struct HostLayout {
  std::vector<uint8_t> trees;
  std::vector<int32_t> leafmap;
  size_t stride = 0;
  int nslots = 0;
};

// PTT (Table 6, perfect padding P:243). Per tree record:
//   uint2 node[2^D]: node[0] = {tree_output, 0}; node[p] for heap position
//   p in [1, 2^D) = {N'_F, N'_T}; then float leaf[2^D][w] = N'_C.
// A leaf at depth D_k < D becomes a perfect subtree whose decision nodes
// compare feature 0 against +Inf ("free to perform arbitrary comparisons")
// and whose 2^(D-D_k) leaves copy the leaf; leafmap keeps the original id.
static void build_ptt(const hb_ensemble *e, int t0, int D, const TreeOrder &order, HostLayout *L,
                      const FeatureMap *fm = nullptr) {
  const int w = e->leaf_width;
  const int P = 1 << D;
  const int Tpad = (int)order.local.size();
  L->nslots = P;
  L->stride = round16((size_t)8 * P + (size_t)4 * w * P);
  L->trees.assign((size_t)Tpad * L->stride, 0);
  L->leafmap.assign((size_t)Tpad * P, -1);
  std::vector<int> orig(2 * P);
  const float pinf = INFINITY;
  for (int lt = 0; lt < Tpad; ++lt) {
    uint8_t *rec = L->trees.data() + (size_t)lt * L->stride;
    uint32_t *node = reinterpret_cast<uint32_t *>(rec);
    float *leaf = reinterpret_cast<float *>(rec + (size_t)8 * P);
    node[0] = ptt_header(order, lt);
    if (order.local[lt] < 0) {  // zero tree (padding of a class / the tree group)
      for (int p = 1; p < P; ++p) node[2 * p] = 0, node[2 * p + 1] = f2u(pinf);
      continue;
    }
    const int t = t0 + order.local[lt];
    const int64_t a = e->node_offset[t];
    orig[1] = 0;
    for (int p = 1; p < P; ++p) {
      const int o = orig[p];
      if (e->left[a + o] != -1) {
        node[2 * p] = (uint32_t)(fm ? fm->remap[e->feature[a + o]] : e->feature[a + o]);
        node[2 * p + 1] = f2u(e->threshold[a + o]);
        orig[2 * p] = e->left[a + o];
        orig[2 * p + 1] = e->right[a + o];
      } else {
        node[2 * p] = 0;
        node[2 * p + 1] = f2u(pinf);
        orig[2 * p] = orig[2 * p + 1] = o;
      }
    }
    for (int p = P; p < 2 * P; ++p) {
      const int o = D == 0 ? 0 : orig[p];
      const int slot = p - P;
      for (int k = 0; k < w; ++k) leaf[(size_t)slot * w + k] = e->leaf_value[(a + o) * w + k];
      L->leafmap[(size_t)lt * P + slot] = o;
    }
  }
}

// TT (Table 5). Nodes renumbered BFS with siblings adjacent so that
// N_L = N_R - 1; per tree record: 16-B header {tree_output}, uint2
// node[nslots] = {N_F | N_R << 16, N_T}, float leaf[nslots][w] = N_C. Leaves
// self-loop (N_R = self, N_T = NaN => predicate false for LT and LE). Padded
// to the max node count over trees.
static hb_status build_tt(const hb_ensemble *e, int t0, int t1, int Tpad, HostLayout *L,
                          const FeatureMap *fm = nullptr) {
  const int w = e->leaf_width;
  int maxn = 1;
  for (int t = t0; t < t1; ++t)
    maxn = std::max<int>(maxn, (int)(e->node_offset[t + 1] - e->node_offset[t]));
  if (maxn > 65535) return fail(HB_E_UNSUPPORTED, "TT: trees with more than 65535 nodes");
  if (e->n_features > 65536) return fail(HB_E_UNSUPPORTED, "TT: more than 65536 features");
  L->nslots = maxn;
  L->stride = round16(16 + (size_t)8 * maxn + (size_t)4 * w * maxn);
  L->trees.assign((size_t)Tpad * L->stride, 0);
  L->leafmap.assign((size_t)Tpad * maxn, -1);
  const uint32_t qnan = 0x7FC00000u;
  std::vector<int> neworder;
  for (int lt = 0; lt < Tpad; ++lt) {
    uint8_t *rec = L->trees.data() + (size_t)lt * L->stride;
    uint32_t *hdr = reinterpret_cast<uint32_t *>(rec);
    uint32_t *node = reinterpret_cast<uint32_t *>(rec + 16);
    float *leaf = reinterpret_cast<float *>(rec + 16 + (size_t)8 * maxn);
    // default: every slot is a self-looping zero leaf
    for (int j = 0; j < maxn; ++j) node[2 * j] = (uint32_t)j << 16, node[2 * j + 1] = qnan;
    if (lt >= t1 - t0) continue;
    const int t = t0 + lt;
    const int64_t a = e->node_offset[t];
    const int n = (int)(e->node_offset[t + 1] - a);
    hdr[0] = (uint32_t)(w == 1 ? tree_out(e, t) : 0);
    neworder.assign(1, 0);  // new id -> original id
    for (size_t q = 0; q < neworder.size(); ++q) {
      const int o = neworder[q];
      if (e->left[a + o] != -1) {
        neworder.push_back(e->left[a + o]);
        neworder.push_back(e->right[a + o]);
      }
    }
    std::vector<int> newid(n);
    for (int j = 0; j < n; ++j) newid[neworder[j]] = j;
    for (int j = 0; j < n; ++j) {
      const int o = neworder[j];
      L->leafmap[(size_t)lt * maxn + j] = o;
      if (e->left[a + o] != -1) {
        const int r = newid[e->right[a + o]];
        node[2 * j] = (uint32_t)(fm ? fm->remap[e->feature[a + o]] : e->feature[a + o]) | ((uint32_t)r << 16);
        node[2 * j + 1] = f2u(e->threshold[a + o]);
      } else {
        for (int k = 0; k < w; ++k) leaf[(size_t)j * w + k] = e->leaf_value[(a + o) * w + k];
      }
    }
  }
  return HB_OK;
}

// Wide-row TT records (tt_wide_kernel). Alg. 2's per-node
// tensors (Table 5: N_F, N_T, N_L, N_R, N_C) folded per INTERNAL node into one
// 16-B record {4 R N_F | leafL | leafR << 1, N_T, payload_L, payload_R} (4 R N_F
// = the byte offset of feature N_F's column in the kernel's R-row X tile),
// in BFS order of the internal nodes. A payload is the child's record index,
// or, when the child is a leaf (flag set), its value bits (w == 1) or its leaf
// slot (w > 1; values at vals_off). So a walk ends on the record whose chosen
// child is a leaf, carrying the value: D_k dependent loads for a leaf at depth
// D_k instead of D_k + 1 (leaf self-loop) + 1 (N_C gather). Per tree:
// 16-B header {n_records, ids_off, tree_output, vals_off}, the records, then
// ids[n_records][2] (original ids of the leaf children, read only by the LEAF /
// LEAF_HASH outputs) and the leaf values (w > 1). Trees are packed without
// padding; toff[t] is the tree's offset in 16-B units. A single-leaf tree gets
// one record {feature 0, +Inf, leaf, leaf}: both children are the leaf, so the
// compare (true for finite x, false for +Inf / NaN) cannot matter.
struct WideLayout {
  std::vector<uint32_t> words;   // the packed trees, 16-B aligned
  std::vector<uint32_t> toff;    // [Tpad] tree offset in 16-B units
};

static hb_status build_ttw(const hb_ensemble *e, int t0, int t1, int Tpad, const FeatureMap *fm,
                           int R, WideLayout *W) {
  const int w = e->leaf_width;
  const uint32_t pinf = f2u(INFINITY);
  std::vector<int> q, recid, slot;
  W->words.clear();
  W->toff.assign(Tpad, 0);
  for (int lt = 0; lt < Tpad; ++lt) {
    const size_t base = W->words.size();
    if ((base / 4) > 0xFFFFFFFFull) return fail(HB_E_UNSUPPORTED, "TT: model larger than 64 GB");
    W->toff[lt] = (uint32_t)(base / 4);
    if (lt >= t1 - t0) {   // padding tree: one record, both children a zero leaf
      W->words.insert(W->words.end(), {1u, 32u, 0u, 48u});   // header (byte offsets)
      W->words.insert(W->words.end(), {0u | 3u, pinf, 0u, 0u});
      W->words.insert(W->words.end(), {0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u});   // ids (never read)
      for (int k = 0; k < 4; ++k) W->words.push_back(0u);                  // w <= 4 zero values
      if (w > 4) W->words.resize(W->words.size() + ((size_t)w - 4 + 3) / 4 * 4, 0u);
      continue;
    }
    const int t = t0 + lt;
    const int64_t a = e->node_offset[t];
    const int n = (int)(e->node_offset[t + 1] - a);
    // BFS over internal nodes; record ids in that order, leaf slots in order
    // of appearance
    q.assign(1, 0);
    recid.assign(n, -1);
    slot.assign(n, -1);
    int nrec = 0, nleaf = 0;
    const bool root_leaf = e->left[a] == -1;
    if (!root_leaf) recid[0] = nrec++;
    for (size_t k = 0; k < q.size(); ++k) {
      const int o = q[k];
      if (e->left[a + o] == -1) {
        slot[o] = nleaf++;
        continue;
      }
      for (int c : {e->left[a + o], e->right[a + o]}) {
        if (e->left[a + c] != -1) recid[c] = nrec++;
        q.push_back(c);
      }
    }
    if (root_leaf) nrec = 1;
    const uint32_t ids_off = 4 + 4 * (uint32_t)nrec;                    // words
    const uint32_t vals_off = ids_off + ((2 * (uint32_t)nrec + 3) & ~3u);
    const size_t vals_words = w == 1 ? 0 : (((size_t)nleaf * w + 3) & ~(size_t)3);
    W->words.resize(base + vals_off + vals_words, 0u);
    uint32_t *T = W->words.data() + base;
    T[0] = (uint32_t)nrec;
    T[1] = ids_off * 4;
    T[2] = (uint32_t)(w == 1 ? tree_out(e, t) : 0);
    T[3] = vals_off * 4;
    auto payload = [&](int c) -> uint32_t {
      if (e->left[a + c] != -1) return (uint32_t)recid[c];
      return w == 1 ? f2u(e->leaf_value[a + c]) : (uint32_t)slot[c];
    };
    if (root_leaf) {
      uint32_t *r = T + 4;
      r[0] = 0u | 3u;
      r[1] = pinf;
      r[2] = r[3] = payload(0);
      T[ids_off] = T[ids_off + 1] = 0u;
    } else {
      for (int o = 0; o < n; ++o) {
        if (recid[o] < 0) continue;
        uint32_t *r = T + 4 + 4 * recid[o];
        const int L = e->left[a + o], Rc = e->right[a + o];
        const uint32_t f = (uint32_t)(fm ? fm->remap[e->feature[a + o]] : e->feature[a + o]);
        r[0] = 4u * (uint32_t)R * f | (e->left[a + L] == -1 ? 1u : 0u) | (e->left[a + Rc] == -1 ? 2u : 0u);
        r[1] = f2u(e->threshold[a + o]);
        r[2] = payload(L);
        r[3] = payload(Rc);
        T[ids_off + 2 * recid[o]] = e->left[a + L] == -1 ? (uint32_t)L : 0xFFFFFFFFu;
        T[ids_off + 2 * recid[o] + 1] = e->left[a + Rc] == -1 ? (uint32_t)Rc : 0xFFFFFFFFu;
      }
    }
    if (w > 1)
      for (int o = 0; o < n; ++o)
        if (slot[o] >= 0)
          for (int k = 0; k < w; ++k) T[vals_off + (size_t)slot[o] * w + k] = f2u(e->leaf_value[(a + o) * w + k]);
  }
  return HB_OK;
}


// Launch configuration: as many 32-row warps as SMEM allows
// for the feature-major X slices (NW * F * 128 B), the rest for a 2-4 stage
// ring of tree chunks.
static bool choose_cfg(int F, size_t stride, int Tpad, bool allow_x_global, bool allow_t_global,
                       int max_nw, LaunchCfg *c) {
  const long budget = kSmemBudget;
  const int force_nw = env_int("HB_NW", 0);      // tuning override (bench sweeps)
  for (int nw : {24, 16, 12, 8, 4}) {
    if (force_nw && nw != force_nw) continue;
    if (nw > max_nw) continue;
    const long xb = (long)nw * F * 128;
    if (xb + 2L * kTreeGroup * (long)stride > budget) continue;
    const long rem = budget - xb;
    int ns = (rem >= 3 * 8 * (long)stride) ? 3 : 2;
    if (env_int("HB_NS", 0)) ns = env_int("HB_NS", 0);
    // up to 128 trees per ring item: every item costs each warp an mbarrier
    // wait + release, which small (shallow) trees do not amortise at 32
    int ch = (int)std::min<long>(env_int("HB_CH", 128), rem / (ns * (long)stride)) & ~(kTreeGroup - 1);
    ch = std::min(ch, Tpad);
    if (ch < kTreeGroup) continue;
    c->nw = nw;
    c->ns = ns;
    c->ch = ch;
    c->x_smem = 1;
    c->t_smem = 1;
    c->smem_bytes = (int)(xb + (long)ns * ch * stride + 16 * ns);
    return true;
  }
  // X does not fit: read rows from global memory, keep the tree ring.
  if (allow_x_global) {
    const long rem = budget;
    if (2L * kTreeGroup * (long)stride <= rem) {
      int ns = (rem >= 3 * 8 * (long)stride) ? 3 : 2;
      int ch = std::min<int>((int)std::min<long>(32, rem / (ns * (long)stride)) & ~(kTreeGroup - 1), Tpad);
      c->nw = 16;
      c->ns = ns;
      c->ch = ch;
      c->x_smem = 0;
      c->t_smem = 1;
      c->smem_bytes = (int)((long)ns * ch * stride + 16 * ns);
      return true;
    }
    if (allow_t_global) {  // neither fits: both through L2/L1
      const long xb = 16L * F * 128;
      c->nw = 16;
      c->ns = 1;
      c->ch = std::min(Tpad, 32) & ~(kTreeGroup - 1);
      c->x_smem = xb <= budget ? 1 : 0;
      c->t_smem = 0;
      c->smem_bytes = c->x_smem ? (int)xb : 0;
      return true;
    }
  }
  return false;
}


// Sec. 5.1: GEMM for shallow trees, PTT up to D = 10, TT beyond,
// with the crossover "determined by ... the underlying hardware". Recalibrated
// on B200 by tools/crossover.py (profiles/r01_crossover.json):
// PTT beats TT up to D = 10 at large batches, TT wins beyond; the tcgen05 GEMM
// never beats PTT (large batches) or the small-batch kernel (small batches),
// so AUTO does not pick GEMM unless HB_GEMM_MAX_DEPTH is set (3 = the paper's
// CPU rule).
static int select_strategy(int D) {
  const int gemm_max = env_int("HB_GEMM_MAX_DEPTH", -1);
  const int ptt_max = std::min(env_int("HB_PTT_MAX_DEPTH", kPttMaxDepth), kPttMaxDepth);
  if (D <= gemm_max && gemm_supported(D)) return HB_STRATEGY_GEMM;
  if (D <= ptt_max) return HB_STRATEGY_PTT;
  return HB_STRATEGY_TT;
}

static void free_model(Model *m) {
  if (!m) return;
  void *bufs[] = {m->d_trees, m->d_leafmap, m->d_scale, m->d_base, m->d_gemm, m->d_aux,
                  m->sb_own_trees, m->sb_own_leafmap, m->d_fmap, m->d_rb, m->d_ttw, m->d_ttw_off};
  if (m->host_only) {
    for (void *b : bufs) std::free(b);
  } else {
    DeviceGuard g(m->device);
    for (void *b : bufs) cudaFree(b);
    if (m->mempool) cudaMemPoolDestroy(m->mempool);   // deferred until pending frees complete
  }
  delete m;
}

void free_model_any(Model *m) { free_model(m); }

hb_status dev_upload(Model *m, const void *src, size_t bytes, void **dst) {
  const size_t alloc = std::max<size_t>(bytes, 16);
  if (m->host_only) {
    *dst = std::malloc(alloc);
    if (!*dst) return fail(HB_E_OOM, "malloc(host-only model)");
    std::memset(*dst, 0, alloc);
    if (bytes) std::memcpy(*dst, src, bytes);
    m->device_bytes += alloc;
    return HB_OK;
  }
  cudaError_t e = cudaMalloc(dst, alloc);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(model)");
  m->device_bytes += alloc;
  if (bytes) {
    e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(model)");
  }
  return HB_OK;
}

hb_status ensure_pool(Model *m) {
  if (m->mempool || m->host_only) return HB_OK;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = m->device;
  cudaError_t err;
  if ((err = cudaMemPoolCreate(&m->mempool, &props)) != cudaSuccess) return cuda_fail(err, "cudaMemPoolCreate");
  uint64_t keep = UINT64_MAX;
  if ((err = cudaMemPoolSetAttribute(m->mempool, cudaMemPoolAttrReleaseThreshold, &keep)) != cudaSuccess)
    return cuda_fail(err, "cudaMemPoolSetAttribute");
  return HB_OK;
}

hb_status scratch_alloc(const Model &m, size_t bytes, cudaStream_t s, void **p) {
  // under stream capture the allocation becomes a graph memory node, which
  // CUDA supports for the device's default pool
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) cap = cudaStreamCaptureStatusNone;
  bytes = std::max<size_t>(bytes, 128);
  const cudaError_t e = (cap == cudaStreamCaptureStatusActive || !m.mempool)
                            ? cudaMallocAsync(p, bytes, s)
                            : cudaMallocFromPoolAsync(p, bytes, m.mempool, s);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocFromPoolAsync(scratch)");
  return HB_OK;
}

template <typename T>
static hb_status upload(Model *m, const std::vector<T> &h, T **d) {
  return dev_upload(m, h.data(), h.size() * sizeof(T), reinterpret_cast<void **>(d));
}

static hb_status compile_impl(const hb_ensemble *e, int t0, int t1, int strategy, int device,
                              Model **out, bool host_only = false) {
  if (!out) return fail(HB_E_INVALID, "out is NULL");
  *out = nullptr;
  std::vector<TreeInfo> info;
  hb_status st = validate_impl(e, &info);
  if (st != HB_OK) return st;
  if (t0 < 0 || t1 > e->n_trees || t0 >= t1) return fail(HB_E_INVALID, "bad tree range");
  if (strategy < HB_STRATEGY_AUTO || strategy > HB_STRATEGY_PTT)
    return fail(HB_E_INVALID, "bad strategy");
  const int K = e->n_outputs;
  if (K > kMaxOutputs) return fail(HB_E_UNSUPPORTED, "n_outputs > 16 is not supported by this build");
  int ndev = 0;
  if (!host_only && (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev))
    return fail(HB_E_INVALID, "device " + std::to_string(device) + " is not a CUDA device");
  DeviceGuard guard(host_only ? -1 : device);
  if (!host_only && !guard.ok) return fail(HB_E_CUDA, "cudaSetDevice failed");

  std::unique_ptr<Model, void (*)(Model *)> m(new Model(), free_model);
  m->host_only = host_only;
  m->device = device;
  m->n_trees = t1 - t0;
  m->tree_begin = t0;
  m->n_trees_total = e->n_trees;
  m->n_trees_pad = (m->n_trees + kTreeGroup - 1) / kTreeGroup * kTreeGroup;
  m->n_features = e->n_features;
  m->n_outputs = K;
  m->leaf_width = e->leaf_width;
  m->cmp = e->cmp;
  m->agg = e->agg;
  m->post = e->post;
  m->task = e->task;
  m->nacc = K == 1 ? 1 : (K <= 4 ? 4 : (K <= 8 ? 8 : 16));
  int D = 0;
  for (int t = t0; t < t1; ++t) D = std::max(D, info[t].depth);
  m->depth = D;

  int strat = strategy == HB_STRATEGY_AUTO ? select_strategy(D) : strategy;
  HostLayout L;
  if (strat == HB_STRATEGY_GEMM) {
    // tensor-core kernel for |I| <= 8, |L| <= 8 (D <= 3); CUDA-core exact
    // contraction for deeper forced-GEMM trees
    st = gemm_tc_eligible(e, t0, t1) && env_int("HB_GEMM_TC", 1) ? compile_gemm_tc(e, t0, t1, m.get())
                                                                 : compile_gemm(e, t0, t1, m.get());
    if (st != HB_OK) return st;
  } else {
    bool done = false;
    const FeatureMap fmap = feature_map(e, t0, t1);
    m->n_xf = (int)fmap.used.size();
    if (!fmap.identity) {
      st = upload(m.get(), fmap.used, &m->d_fmap);
      if (st != HB_OK) return st;
    }
    if (strat == HB_STRATEGY_PTT && D <= kPttMaxDepth) {
      // warps the fp32-node layout would get (the rank layout must match it)
      LaunchCfg fcfg;
      const size_t fstride = round16((size_t)8 * (1 << D) + (size_t)4 * e->leaf_width * (1 << D));
      const int nw_fp32 = choose_cfg(m->n_xf, fstride, m->n_trees_pad, false, false, 24, &fcfg) ? fcfg.nw : 0;
      st = compile_ptt_rank(e, t0, t1, D, m.get(), nw_fp32);   // 4-B rank-coded nodes when eligible
      if (st == HB_OK) done = true;
      else if (st != HB_E_UNSUPPORTED) return st;
    }
    if (!done && strat == HB_STRATEGY_PTT) {
      bool ok = D <= kPttMaxDepth;
      if (ok) {
        const TreeOrder order = ptt_order(e, t0, t1, true);
        m->n_trees_pad = (int)order.local.size();
        build_ptt(e, t0, D, order, &L, &fmap);
        ok = choose_cfg((int)fmap.used.size(), L.stride, m->n_trees_pad, false, false, 24, &m->cfg);
      }
      if (!ok) {
        if (strategy == HB_STRATEGY_PTT)
          return fail(HB_E_UNSUPPORTED,
                      "PTT: depth " + std::to_string(D) + " / n_features " +
                          std::to_string(e->n_features) +
                          " exceed the perfect-tree / SMEM budget (use TT or AUTO)");
        strat = HB_STRATEGY_TT;
        L = HostLayout();
        m->n_trees_pad = (m->n_trees + kTreeGroup - 1) / kTreeGroup * kTreeGroup;
      }
    }
    if (!done && strat == HB_STRATEGY_TT) {
      st = build_tt(e, t0, t1, m->n_trees_pad, &L, &fmap);
      if (st != HB_OK) return st;
      // rows that fit a 32-row-per-warp SMEM slice with room for a tree ring
      // use tt_kernel; wider rows or trees too big for SMEM use tt_wide_kernel
      const bool narrow = choose_cfg((int)fmap.used.size(), L.stride, m->n_trees_pad, false, false, 16, &m->cfg);
      const int force_wide = env_int("HB_TT_WIDE", -1);
      if (!narrow || force_wide == 1) {
        if (force_wide == 0) return fail(HB_E_UNSUPPORTED, "TT: no narrow configuration fits");
        LaunchCfg c;
        c.nw = 32;
        c.wide_rows = 0;
        const int force_r = env_int("HB_TT_WIDE_ROWS", 0);   // tuning override (32/16/8)
        for (int R : {32, 16, 8}) {
          if (force_r && R != force_r) continue;
          const size_t bytes = tt_wide_smem((int)fmap.used.size(), R, c.nw, m->nacc);
          if (bytes <= (size_t)kSmemBudget) {
            c.wide_rows = R;
            c.smem_bytes = (int)bytes;
            break;
          }
        }
        if (!c.wide_rows) return fail(HB_E_UNSUPPORTED, "TT: rows too wide for an 8-row SMEM tile");
        c.x_smem = 1;
        c.t_smem = 0;
        c.ch = kTreeGroup;
        m->cfg = c;
        m->tt_g = env_int("HB_TT_G", 4);   // walks per lane (DESIGN.md §4.3 sweep)
        WideLayout W;
        st = build_ttw(e, t0, t1, m->n_trees_pad, &fmap, m->cfg.wide_rows, &W);
        if (st != HB_OK) return st;
        // models larger than L2: walk them in tree chunks whose records stay
        // L2-resident (HB_TT_CHUNK: -1 auto, N trees, 0 off). The walk reads
        // only the 16-B records (not the leaf-id tables), so the chunk is
        // sized on record bytes: HB_TT_CHUNK_L2 (percent of L2, default 40)
        // of records per chunk when they exceed HB_TT_BIG_L2 (default 50)
        // percent of L2
        int l2_bytes = 126 * 1024 * 1024;   // B200; the host-only compile assumes it
        if (!host_only) cudaDeviceGetAttribute(&l2_bytes, cudaDevAttrL2CacheSize, device);
        double rec_bytes = 0;
        for (int lt = 0; lt < m->n_trees; ++lt) rec_bytes += 16.0 * W.words[(size_t)W.toff[lt] * 4];
        m->ttw_rec_bytes = (size_t)rec_bytes;
        const bool big = rec_bytes > 0.01 * env_int("HB_TT_BIG_L2", 50) * (double)l2_bytes;
        const int want_chunk = env_int("HB_TT_CHUNK", -1);
        if (want_chunk > 0 || (want_chunk == -1 && big)) {
          const double per_tree = std::max(1.0, rec_bytes / std::max(1, m->n_trees));
          const int autoc = (int)(0.01 * env_int("HB_TT_CHUNK_L2", 40) * (double)l2_bytes / per_tree) &
                            ~(kTreeGroup - 1);
          m->tt_chunk = std::max(kTreeGroup, want_chunk > 0 ? want_chunk : autoc);
          if (m->tt_chunk >= m->n_trees_pad) m->tt_chunk = 0;   // one chunk: one plain launch
        }
        if (m->tt_chunk) {
          st = ensure_pool(m.get());
          if (st != HB_OK) return st;
        }
        st = upload(m.get(), W.words, reinterpret_cast<uint32_t **>(&m->d_ttw));
        if (st != HB_OK) return st;
        st = upload(m.get(), W.toff, &m->d_ttw_off);
        if (st != HB_OK) return st;
        m->ttw_bytes = W.words.size() * 4;
      }
    }
    if (!done) {
      m->stride = L.stride;
      m->nslots = L.nslots;
      st = upload(m.get(), L.trees, reinterpret_cast<uint8_t **>(&m->d_trees));
      if (st != HB_OK) return st;
      st = upload(m.get(), L.leafmap, &m->d_leafmap);
      if (st != HB_OK) return st;
    }
  }
  m->strategy = strat;
  m->cfg.prefetch = env_int("HB_PREFETCH", 1);

  // small-batch path: reuse the PTT fp32 / TT records, else build PTT fp32 ones
  m->sb_nxf = m->n_features;
  if (strat == HB_STRATEGY_TT || (strat == HB_STRATEGY_PTT && !m->ptt_rank)) {
    m->sb_fmap = m->d_fmap;     // those records index the compacted tile
    m->sb_nxf = m->n_xf;
  }
  if (strat == HB_STRATEGY_TT) {
    m->sb_nrec = m->n_trees;
    m->sb_trees = m->d_trees;
    m->sb_leafmap = m->d_leafmap;
    m->sb_stride = m->stride;
    m->sb_nslots = m->nslots;
    m->sb_tt = 1;
    m->sb_depth = D;
  } else if (strat == HB_STRATEGY_PTT && !m->ptt_rank) {
    m->sb_nrec = m->n_trees_pad;
    m->sb_trees = m->d_trees;
    m->sb_leafmap = m->d_leafmap;
    m->sb_stride = m->stride;
    m->sb_nslots = m->nslots;
    m->sb_depth = D;
  } else if (D <= kPttMaxDepth) {
    HostLayout S;
    const TreeOrder order = ptt_order(e, t0, t1, true);
    build_ptt(e, t0, D, order, &S);
    m->sb_nrec = (int)order.local.size();
    uint8_t *dt = nullptr;
    st = upload(m.get(), S.trees, &dt);
    if (st != HB_OK) return st;
    m->sb_own_trees = dt;
    st = upload(m.get(), S.leafmap, &m->sb_own_leafmap);
    if (st != HB_OK) return st;
    m->sb_trees = dt;
    m->sb_leafmap = m->sb_own_leafmap;
    m->sb_stride = S.stride;
    m->sb_nslots = S.nslots;
    m->sb_depth = D;
  }

  // request/response sizes: trees-across-threads kernel (f2) for n_rows <=
  // small_max; threshold from the crossover sweep (tools/crossover.py,
  // DESIGN.md §6.2), env HB_SMALL_BATCH overrides (0: off) at compile time
  // A forced strategy is honoured at every batch size: the small-batch
  // kernel serves AUTO models only, unless HB_SMALL_BATCH is set explicitly
  const char *sbe = std::getenv("HB_SMALL_BATCH");
  const bool sb_on = strategy == HB_STRATEGY_AUTO || (sbe && *sbe);
  m->small_max = (m->sb_trees && sb_on) ? std::max(0, env_int("HB_SMALL_BATCH", 4096)) : 0;

  // global per-output tree counts (MEAN divisor) and base score
  std::vector<float> div(K, 1.f), base(K + 1, 0.f);   // base[K] = post_param
  if (e->agg == HB_AGG_MEAN) {
    std::vector<double> cnt(K, 0.0);
    for (int t = 0; t < e->n_trees; ++t) {
      if (e->leaf_width == 1) cnt[tree_out(e, t)] += 1.0;
      else for (int k = 0; k < K; ++k) cnt[k] += 1.0;
    }
    for (int k = 0; k < K; ++k) div[k] = cnt[k] > 0 ? (float)cnt[k] : 1.f;
  }
  if (e->base_score)
    for (int k = 0; k < K; ++k) base[k] = e->base_score[k];
  base[K] = e->post == HB_POST_ISOLATION ? e->post_param : 1.f;
  st = upload(m.get(), div, &m->d_scale);
  if (st != HB_OK) return st;
  st = upload(m.get(), base, &m->d_base);
  if (st != HB_OK) return st;
  *out = m.release();
  return HB_OK;
}

hb_status compile_model_host(const hb_ensemble *e, int t0, int t1, int strategy, Model **out) {
  return compile_impl(e, t0, t1, strategy, 0, out, true);
}

static const Model *M(const hb_model *m) { return reinterpret_cast<const Model *>(m); }

static hb_status check_dev_ptr(const void *p, int device, const char *what) {
  cudaPointerAttributes attr;
  cudaError_t e = cudaPointerGetAttributes(&attr, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HB_E_INVALID, std::string(what) + " is not a CUDA pointer");
  }
  if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
    return fail(HB_E_INVALID, std::string(what) + " is not a device pointer");
  if (attr.device != device)
    return fail(HB_E_INVALID, std::string(what) + " lives on device " + std::to_string(attr.device) +
                                  ", model on device " + std::to_string(device));
  return HB_OK;
}

static size_t out_row_bytes(const Model &m, int kind) {
  switch (kind) {
    case HB_OUT_PREDICT:
      return m.task == HB_TASK_CLASSIFICATION ? 4 : 4 * (size_t)m.n_outputs;
    case HB_OUT_PROBA: return m.n_outputs == 1 ? 8 : 4 * (size_t)m.n_outputs;
    case HB_OUT_RAW:
    case HB_OUT_MARGIN: return 4 * (size_t)m.n_outputs;
    case HB_OUT_LEAF: return 4 * (size_t)m.n_trees;
    case HB_OUT_LEAF_HASH: return 8;
    case HB_OUT_RAW64: return 8 * (size_t)m.n_outputs;
  }
  return 0;
}

static hb_status check_kind(const Model &m, int kind) {
  if (kind < HB_OUT_PREDICT || kind > HB_OUT_RAW64) return fail(HB_E_INVALID, "bad output kind");
  if (kind == HB_OUT_PROBA && m.task != HB_TASK_CLASSIFICATION)
    return fail(HB_E_UNSUPPORTED, "predict_proba on a regression model");
  return HB_OK;
}

static hb_status run(const Model &m, const RunArgs &a) {
  switch (m.strategy) {
    case HB_STRATEGY_PTT: return m.ptt_rank ? launch_ptt_rank(m, a) : launch_ptt(m, a);
    case HB_STRATEGY_TT: return launch_tt(m, a);
    case HB_STRATEGY_GEMM: return launch_gemm(m, a);
  }
  return fail(HB_E_INVALID, "corrupt model");
}

// NVTX ranges around compile / predict (SURVEY §5 tracing): header-only
// nvtx3, a no-op unless a profiler (ncu, nsys) injects its collector
namespace {
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
const char *kind_range(int kind) {
  // indexed by hb_output (PREDICT, PROBA, RAW, MARGIN, LEAF, LEAF_HASH, RAW64)
  static const char *names[] = {"hb_predict", "hb_predict_proba", "hb_predict_raw", "hb_predict_margin",
                                "hb_predict_leaf", "hb_predict_leaf_hash", "hb_predict_raw64"};
  return kind >= 0 && kind < (int)(sizeof(names) / sizeof(names[0])) ? names[kind] : "hb_predict";
}
}  // namespace

static hb_status predict_impl(const hb_model *hm, const float *X, int64_t n, int64_t ldx, int kind,
                              void *out, void *stream, bool check_ptrs, void **events = nullptr,
                              int nev = 0, int32_t *n_launches = nullptr) {
  NvtxRange range(kind_range(kind));
  if (n_launches) *n_launches = 0;
  if (!hm) return fail(HB_E_INVALID, "model is NULL");
  const Model &m = *M(hm);
  hb_status st = check_kind(m, kind);
  if (st != HB_OK) return st;
  if (n < 0) return fail(HB_E_INVALID, "n_rows < 0");
  if (ldx < m.n_features) return fail(HB_E_INVALID, "ldx < n_features");
  if (n == 0) return HB_OK;
  if (!X || !out) return fail(HB_E_INVALID, "X or out is NULL");
  DeviceGuard g(m.device);
  if (check_ptrs) {
    st = check_dev_ptr(X, m.device, "X");
    if (st != HB_OK) return st;
    st = check_dev_ptr(out, m.device, "out");
    if (st != HB_OK) return st;
  }
  RunArgs a{X, n, ldx, kind, out, static_cast<cudaStream_t>(stream), nullptr};
  int k = 0;
  cudaError_t ev_err = cudaSuccess;
  if (events && nev > 0) {
    a.ev = reinterpret_cast<cudaEvent_t *>(events);
    a.nev = nev;
    a.ev_k = &k;
    a.ev_err = &ev_err;
  }
  mark_launch(a);
  // request/response sizes: trees-across-threads kernel (f2); threshold from
  // the crossover sweep (tools/crossover.py)
  st = n <= m.small_max ? launch_small_batch(m, a) : run(m, a);
  mark_launch(a);
  if (n_launches) *n_launches = k > 0 ? k - 1 : 0;
  if (st == HB_OK && ev_err != cudaSuccess) return cuda_fail(ev_err, "cudaEventRecord(hb_predict_ex_events)");
  return st;
}

// ------------------------------------------------------------------ host streaming
struct HostStage {
  std::mutex mu;
  int device = -1;
  cudaStream_t s[2] = {nullptr, nullptr};
  float *x[2] = {nullptr, nullptr};
  uint8_t *o[2] = {nullptr, nullptr};
  size_t xcap = 0, ocap = 0;
  ~HostStage() {}
};

static HostStage &host_stage(int device) {
  static std::mutex mu;
  static std::deque<HostStage> stages;  // one per device, never freed
  std::lock_guard<std::mutex> lk(mu);
  for (auto &s : stages)
    if (s.device == device) return s;
  stages.emplace_back();
  stages.back().device = device;
  return stages.back();
}

static hb_status host_impl(const hb_model *hm, const float *Xh, int64_t n, int64_t ldx, int kind,
                           void *outh) {
  NvtxRange range("hb_predict_host");
  if (!hm) return fail(HB_E_INVALID, "model is NULL");
  const Model &m = *M(hm);
  hb_status st = check_kind(m, kind);
  if (st != HB_OK) return st;
  if (kind == HB_OUT_LEAF) return fail(HB_E_UNSUPPORTED, "hb_predict_host: LEAF output not supported");
  if (n < 0 || ldx < m.n_features) return fail(HB_E_INVALID, "bad n_rows / ldx");
  if (n == 0) return HB_OK;
  if (!Xh || !outh) return fail(HB_E_INVALID, "X or out is NULL");
  DeviceGuard g(m.device);
  HostStage &hs = host_stage(m.device);
  std::lock_guard<std::mutex> lk(hs.mu);
  cudaError_t e;
  for (int i = 0; i < 2; ++i)
    if (!hs.s[i] && (e = cudaStreamCreateWithFlags(&hs.s[i], cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
  const size_t orow = out_row_bytes(m, kind);
  const size_t xrow = (size_t)ldx * 4;
  // chunks of ~64 MB of X (at least 64K rows) so copies pipeline with scoring
  const int64_t chunk = std::min<int64_t>(n, std::max<int64_t>(65536, (64LL << 20) / (int64_t)xrow));
  if (hs.xcap < chunk * xrow || hs.ocap < chunk * orow) {
    for (int i = 0; i < 2; ++i) {
      cudaFree(hs.x[i]);
      cudaFree(hs.o[i]);
      hs.x[i] = nullptr;
      hs.o[i] = nullptr;
    }
    hs.xcap = hs.ocap = 0;
    for (int i = 0; i < 2; ++i) {
      if ((e = cudaMalloc(&hs.x[i], chunk * xrow)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(stage)");
      if ((e = cudaMalloc(&hs.o[i], chunk * orow)) != cudaSuccess) return cuda_fail(e, "cudaMalloc(stage)");
    }
    hs.xcap = chunk * xrow;
    hs.ocap = chunk * orow;
  }
  int ci = 0;
  for (int64_t r0 = 0; r0 < n; r0 += chunk, ci ^= 1) {
    const int64_t rows = std::min(chunk, n - r0);
    cudaStream_t s = hs.s[ci];
    if ((e = cudaMemcpyAsync(hs.x[ci], reinterpret_cast<const uint8_t *>(Xh) + r0 * xrow,
                             rows * xrow, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync(H2D)");
    RunArgs a{hs.x[ci], rows, ldx, kind, hs.o[ci], s, nullptr};
    st = run(m, a);
    if (st != HB_OK) return st;
    if ((e = cudaMemcpyAsync(static_cast<uint8_t *>(outh) + r0 * orow, hs.o[ci], rows * orow,
                             cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync(D2H)");
  }
  for (int i = 0; i < 2; ++i)
    if ((e = cudaStreamSynchronize(hs.s[i])) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  return HB_OK;
}

}  // namespace hb

// ====================================================================== C ABI
using namespace hb;

extern "C" {

hb_status hb_validate(const hb_ensemble *e) { return validate_impl(e, nullptr); }

hb_status hb_compile(const hb_ensemble *e, int32_t strategy, int32_t device, hb_model **out) {
  NvtxRange range("hb_compile");
  if (!e) return fail(HB_E_INVALID, "ensemble is NULL");
  return compile_impl(e, 0, e->n_trees, strategy, device, reinterpret_cast<Model **>(out));
}

hb_status hb_compile_range(const hb_ensemble *e, int32_t tree_begin, int32_t tree_end,
                           int32_t strategy, int32_t device, hb_model **out) {
  NvtxRange range("hb_compile_range");
  return compile_impl(e, tree_begin, tree_end, strategy, device, reinterpret_cast<Model **>(out));
}

hb_status hb_predict_ex(const hb_model *m, const float *X, int64_t n, int64_t ldx, int32_t kind,
                        void *out, void *stream) {
  return predict_impl(m, X, n, ldx, kind, out, stream, true);
}

hb_status hb_predict_ex_events(const hb_model *m, const float *X, int64_t n, int64_t ldx,
                               int32_t kind, void *out, void *stream, void **events, int32_t n_events,
                               int32_t *n_launches) {
  if (!events || n_events < 2) return fail(HB_E_INVALID, "hb_predict_ex_events: need >= 2 events");
  return predict_impl(m, X, n, ldx, kind, out, stream, true, events, n_events, n_launches);
}

hb_status hb_predict(const hb_model *m, const float *X, int64_t n, int64_t ldx, void *out,
                     void *stream) {
  return predict_impl(m, X, n, ldx, HB_OUT_PREDICT, out, stream, true);
}

hb_status hb_predict_proba(const hb_model *m, const float *X, int64_t n, int64_t ldx, float *out,
                           void *stream) {
  return predict_impl(m, X, n, ldx, HB_OUT_PROBA, out, stream, true);
}

hb_status hb_predict_raw(const hb_model *m, const float *X, int64_t n, int64_t ldx, float *out,
                         void *stream) {
  return predict_impl(m, X, n, ldx, HB_OUT_RAW, out, stream, true);
}

hb_status hb_predict_leaf(const hb_model *m, const float *X, int64_t n, int64_t ldx, int32_t *out,
                          void *stream) {
  return predict_impl(m, X, n, ldx, HB_OUT_LEAF, out, stream, true);
}

static hb_status finalize_impl(const hb_model *hm, const float *raw, const double *raw64, int64_t n,
                               int32_t kind, void *out, void *stream) {
  if (!hm) return fail(HB_E_INVALID, "model is NULL");
  const Model &m = *M(hm);
  if (kind != HB_OUT_PREDICT && kind != HB_OUT_PROBA && kind != HB_OUT_MARGIN)
    return fail(HB_E_INVALID, "hb_finalize: kind must be PREDICT, PROBA or MARGIN");
  hb_status st = check_kind(m, kind);
  if (st != HB_OK) return st;
  if (n < 0) return fail(HB_E_INVALID, "n_rows < 0");
  if (n == 0) return HB_OK;
  if ((!raw && !raw64) || !out) return fail(HB_E_INVALID, "raw or out is NULL");
  DeviceGuard g(m.device);
  if ((st = check_dev_ptr(raw ? (const void *)raw : (const void *)raw64, m.device, "raw")) != HB_OK) return st;
  if ((st = check_dev_ptr(out, m.device, "out")) != HB_OK) return st;
  RunArgs a{nullptr, n, 0, kind, out, static_cast<cudaStream_t>(stream), raw};
  a.raw_in64 = raw64;
  return launch_finalize(m, a);
}

hb_status hb_finalize(const hb_model *hm, const float *raw, int64_t n, int32_t kind, void *out,
                      void *stream) {
  return finalize_impl(hm, raw, nullptr, n, kind, out, stream);
}

hb_status hb_finalize64(const hb_model *hm, const double *raw, int64_t n, int32_t kind, void *out,
                        void *stream) {
  return finalize_impl(hm, nullptr, raw, n, kind, out, stream);
}

hb_status hb_predict_host(const hb_model *m, const float *X, int64_t n, int64_t ldx, int32_t kind,
                          void *out) {
  return host_impl(m, X, n, ldx, kind, out);
}

hb_status hb_model_get_info(const hb_model *hm, hb_model_info *info) {
  if (!hm || !info) return fail(HB_E_INVALID, "NULL argument");
  const Model &m = *M(hm);
  info->strategy = m.strategy;
  info->max_depth = m.depth;
  info->tree_begin = m.tree_begin;
  info->n_trees = m.n_trees;
  info->n_trees_total = m.n_trees_total;
  info->n_features = m.n_features;
  info->n_outputs = m.n_outputs;
  info->leaf_width = m.leaf_width;
  info->device = m.device;
  info->x_in_smem = m.cfg.x_smem;
  info->device_bytes = (int64_t)m.device_bytes;
  info->tree_stride_bytes = (int64_t)m.stride;
  info->tensor_cores = m.gemm_tc;
  info->node_record_bytes = m.strategy == HB_STRATEGY_GEMM ? 0 : m.ptt_rank ? 4 : m.cfg.wide_rows ? 16 : 8;
  if (m.strategy == HB_STRATEGY_PTT) info->kernel = m.ptt_rank ? 1 : 0;
  else if (m.strategy == HB_STRATEGY_TT)
    info->kernel = m.cfg.wide_rows ? 3 : 2;
  else info->kernel = m.gemm_tc ? 4 : 5;
  info->rows_per_cta = m.strategy == HB_STRATEGY_GEMM ? (m.gemm_tc ? 128 : 128)
                       : (m.cfg.wide_rows ? m.cfg.wide_rows : 32 * m.cfg.nw * (m.ptt_rank ? m.rank_rpl : 1));
  info->code_cell_bits = m.ptt_rank ? m.rank_cw : 0;
  info->rank_prepass = m.rank_pre;
  info->tt_sector = 0;   // sector-paired TT records were removed
  info->tt_chunk_trees = m.tt_chunk;
  info->small_batch_max_rows = m.small_max;
  info->tt_walks_per_lane = m.cfg.wide_rows ? m.tt_g : 0;
  info->tt_record_bytes = (int64_t)m.ttw_rec_bytes;
  info->rank_prepass_tma = m.rank_pre ? m.rb_tma : 0;
  info->rows_per_lane = m.strategy == HB_STRATEGY_PTT && m.ptt_rank ? m.rank_rpl : 1;
  return HB_OK;
}

void hb_free(hb_model *m) { free_model(reinterpret_cast<Model *>(m)); }

const char *hb_last_error(void) { return g_err.c_str(); }

int32_t hb_abi_version(void) { return HB_ABI_VERSION; }

}  // extern "C"
