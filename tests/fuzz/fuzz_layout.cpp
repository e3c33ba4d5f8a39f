// fuzz_layout.cpp — mutation fuzzer of the host-side boundary code, built with
// AddressSanitizer + UndefinedBehaviorSanitizer (tests/test_fuzz_host.py):
// hb_validate (include/hb.h) and the whole compile path — strategy selection,
// the PTT / TT / wide-TT / GEMM / rank-coded PTT layout builders and the
// rank-code bucket tables (paper_2010_04804_b200/csrc/hb_host.cpp,
// hb_compile.cpp) — in their host-only mode (no GPU: buffers are host memory).
//
// Per iteration:
//  1. a random VALID ensemble (random tree shapes up to depth 12, duplicate /
//     +-Inf / +-0 / denormal thresholds, 1..5 outputs, scalar or vector
//     leaves, LT or LE) must pass hb_validate and compile under every
//     strategy (HB_OK, or HB_E_UNSUPPORTED where a strategy's limits say so);
//     every layout that was built is then INTERPRETED on random rows (NaN,
//     +-Inf, ties) and must reach the leaf a plain tree walk reaches (PAPER.md
//     Alg. 1-3 reach the same leaf, SURVEY.md §8(c) P-d) with its value;
//  2. the same ensemble with one random corruption (bad child id, cycle,
//     shared child, NaN threshold, feature out of range, non-finite leaf,
//     bad enum, non-monotone offsets, ...) must be rejected by hb_validate and
//     by the compile with the same status, and must not crash.
// Any sanitizer report aborts the process (-fno-sanitize-recover=all).
//
//   fuzz_layout <iterations> <seed>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <random>
#include <vector>

#include "hb.h"
#include "hb_internal.h"
#include "hb_layouts.h"

using namespace hb;

// ---- the launch entry points hb_host.cpp references (never reached: the
// host-only model is not scored in this build)
namespace hb {
hb_status launch_ptt_rank(const Model &, const RunArgs &) { return HB_E_UNSUPPORTED; }
hb_status launch_ptt(const Model &, const RunArgs &) { return HB_E_UNSUPPORTED; }
hb_status launch_tt(const Model &, const RunArgs &) { return HB_E_UNSUPPORTED; }
hb_status launch_gemm(const Model &, const RunArgs &) { return HB_E_UNSUPPORTED; }
hb_status launch_finalize(const Model &, const RunArgs &) { return HB_E_UNSUPPORTED; }
hb_status launch_small_batch(const Model &, const RunArgs &) { return HB_E_UNSUPPORTED; }
}  // namespace hb

static std::mt19937_64 rng;
static int failures = 0;
#define REQUIRE(c, ...)                                             \
  do {                                                              \
    if (!(c)) {                                                     \
      std::fprintf(stderr, "FAIL line %d: ", __LINE__);             \
      std::fprintf(stderr, __VA_ARGS__);                            \
      std::fprintf(stderr, " (%s)\n", hb_last_error());             \
      if (++failures > 20) std::exit(1);                            \
    }                                                               \
  } while (0)

static int rnd(int n) { return (int)(rng() % (uint64_t)n); }
static float u01() { return (float)((rng() >> 40) * (1.0 / 16777216.0)); }

struct Ens {
  int T = 0, F = 0, K = 1, w = 1, cmp = 0, agg = 0, post = 0, task = 0;
  float post_param = 0.f;
  std::vector<int64_t> off;
  std::vector<int32_t> feat, left, right, tout;
  std::vector<float> thr, val, base;
  bool use_tout = false, use_base = false;
  hb_ensemble view() const {
    hb_ensemble e;
    std::memset(&e, 0, sizeof e);
    e.n_trees = T; e.n_features = F; e.n_outputs = K;
    e.node_offset = off.data(); e.feature = feat.data(); e.threshold = thr.data();
    e.left = left.data(); e.right = right.data(); e.leaf_value = val.data();
    e.leaf_width = w; e.tree_output = use_tout ? tout.data() : nullptr;
    e.base_score = use_base ? base.data() : nullptr;
    e.cmp = cmp; e.agg = agg; e.post = post; e.task = task; e.post_param = post_param;
    return e;
  }
};

static float rand_threshold(const std::vector<float> &grid) {
  const int r = rnd(100);
  if (r < 3) return INFINITY;
  if (r < 6) return -INFINITY;
  if (r < 8) return -0.0f;
  if (r < 10) return 1e-40f;                              // denormal
  if (r < 12) return std::nextafter(grid[rnd((int)grid.size())], INFINITY);
  return grid[rnd((int)grid.size())];                     // coarse grid: many ties / duplicates
}

// random rooted binary tree, node ids shuffled (root stays 0)
static void add_tree(Ens &E, int maxd, const std::vector<float> &grid) {
  const int64_t a = (int64_t)E.feat.size();
  struct N { int parent_depth; };
  std::vector<int> L(1, -1), R(1, -1), depth(1, 0);
  std::vector<int> frontier(1, 0);
  const float psplit = 0.55f + 0.4f * u01();
  for (size_t k = 0; k < frontier.size(); ++k) {
    const int i = frontier[k];
    if (depth[i] < maxd && (i == 0 ? u01() < 0.95f : u01() < psplit)) {
      const int l = (int)L.size();
      L.push_back(-1); R.push_back(-1); depth.push_back(depth[i] + 1);
      L.push_back(-1); R.push_back(-1); depth.push_back(depth[i] + 1);
      L[i] = l; R[i] = l + 1;
      frontier.push_back(l); frontier.push_back(l + 1);
    }
  }
  const int n = (int)L.size();
  std::vector<int> perm(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  std::shuffle(perm.begin() + 1, perm.end(), rng);          // new id of old node
  std::vector<int> inv(n);
  for (int i = 0; i < n; ++i) inv[perm[i]] = i;
  for (int j = 0; j < n; ++j) {
    const int o = inv[j];
    const bool leaf = L[o] < 0;
    E.left.push_back(leaf ? -1 : perm[L[o]]);
    E.right.push_back(leaf ? -1 : perm[R[o]]);
    E.feat.push_back(leaf ? (rnd(3) == 0 ? -1 : 0) : rnd(E.F));
    E.thr.push_back(leaf ? NAN : rand_threshold(grid));
  }
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < E.w; ++k)
      E.val.push_back(E.left[a + j] < 0 ? (float)(rnd(2001) - 1000) / 64.f : NAN);
  E.off.push_back((int64_t)E.feat.size());
}

static Ens random_ensemble() {
  Ens E;
  E.T = 1 + rnd(24);
  E.F = 1 + rnd(rnd(4) == 0 ? 600 : 12);
  E.cmp = rnd(2);
  const int kind = rnd(6);
  if (kind == 0) {            // regression
    E.K = 1;
  } else if (kind == 1) {     // binary
    E.K = 1; E.post = HB_POST_SIGMOID; E.task = HB_TASK_CLASSIFICATION;
  } else if (kind == 2) {     // per-class scalar trees
    E.K = 2 + rnd(4); E.post = HB_POST_SOFTMAX; E.task = HB_TASK_CLASSIFICATION;
  } else if (kind == 3) {     // vector leaves, MEAN
    E.K = 2 + rnd(4); E.w = E.K; E.agg = HB_AGG_MEAN; E.task = HB_TASK_CLASSIFICATION;
  } else if (kind == 4) {     // isolation forest
    E.K = 1; E.agg = HB_AGG_MEAN; E.post = HB_POST_ISOLATION; E.post_param = 3.5f;
  } else {                    // multi-output regression with explicit tree_output
    E.K = 1 + rnd(5); E.use_tout = true;
  }
  std::vector<float> grid;
  const int ng = 1 + rnd(12);
  for (int i = 0; i < ng; ++i) grid.push_back((float)(rnd(33) - 16) / 4.f);
  const int maxd = rnd(5) == 0 ? 12 : rnd(9);
  E.off.push_back(0);
  for (int t = 0; t < E.T; ++t) add_tree(E, maxd, grid);
  E.tout.resize(E.T);
  for (int t = 0; t < E.T; ++t) E.tout[t] = rnd(E.K);
  E.use_base = rnd(2) == 0;
  E.base.resize(E.K);
  for (int k = 0; k < E.K; ++k) E.base[k] = (float)(rnd(9) - 4) / 8.f;
  return E;
}

// ---- reference: the plain walk (Alg. 2 without tensors)
static bool pred(int cmp, float x, float t) { return cmp == 0 ? x < t : x <= t; }
static int walk(const Ens &E, int t, const float *x) {
  const int64_t a = E.off[t];
  int i = 0;
  while (E.left[a + i] != -1) i = pred(E.cmp, x[E.feat[a + i]], E.thr[a + i]) ? E.left[a + i] : E.right[a + i];
  return i;
}
static float leafv(const Ens &E, int t, int leaf, int k) { return E.val[(E.off[t] + leaf) * E.w + k]; }

static std::vector<float> random_rows(const Ens &E, int n) {
  std::vector<float> X((size_t)n * E.F);
  for (auto &v : X) {
    const int r = rnd(100);
    if (r < 4) v = NAN;
    else if (r < 7) v = (r & 1) ? INFINITY : -INFINITY;
    else if (r < 9) v = (r & 1) ? 0.f : -0.f;
    else if (r < 60) v = (float)(rnd(33) - 16) / 4.f;    // threshold grid: ties
    else v = (u01() - 0.5f) * 10.f;
  }
  return X;
}

static uint32_t f2u(float f) { uint32_t u; std::memcpy(&u, &f, 4); return u; }
static float u2f(uint32_t u) { float f; std::memcpy(&f, &u, 4); return f; }

// compact feature of the fp32 PTT / TT records -> original feature
static int orig_feature(const Model &m, int c) {
  return m.d_fmap ? m.d_fmap[c] : c;
}

// ---- interpreters of the compiled layouts (host copies in a host-only model)
static void check_ptt_fp32(const Ens &E, const Model &m, const std::vector<float> &X, int n) {
  const int D = m.depth, P = 1 << D, w = E.w;
  const uint8_t *trees = static_cast<const uint8_t *>(m.d_trees);
  for (int lt = 0; lt < m.n_trees_pad; ++lt) {
    const uint8_t *rec = trees + (size_t)lt * m.stride;
    const uint32_t *node = reinterpret_cast<const uint32_t *>(rec);
    const int local = (int)(node[0] >> 8) - 1;
    if (local < 0) continue;
    const int t = m.tree_begin + local;
    for (int r = 0; r < n; ++r) {
      const float *x = &X[(size_t)r * E.F];
      uint32_t i = 1;
      for (int l = 0; l < D; ++l) {
        const float xv = x[orig_feature(m, (int)node[2 * i])];
        i = 2 * i + (pred(E.cmp, xv, u2f(node[2 * i + 1])) ? 0 : 1);
      }
      const int slot = (int)(i - (uint32_t)P);
      const int want = walk(E, t, x);
      REQUIRE(m.d_leafmap[(size_t)lt * P + slot] == want, "PTT fp32 leaf tree %d row %d", t, r);
      const float *leaf = reinterpret_cast<const float *>(rec + (size_t)8 * P);
      for (int k = 0; k < w; ++k)
        REQUIRE(f2u(leaf[(size_t)slot * w + k]) == f2u(leafv(E, t, want, k)), "PTT fp32 value");
      if (E.w == 1 && E.K > 1)
        REQUIRE((int)(node[0] & 0xFF) == (E.use_tout ? E.tout[t] : t % E.K), "PTT class");
    }
  }
}

static void check_ptt_rank(const Ens &E, const Model &m, const std::vector<float> &X, int n, int t0, int t1) {
  // distinct thresholds per used feature, in fp32 order (-0 == +0)
  std::vector<std::vector<float>> u(E.F);
  for (int t = t0; t < t1; ++t)
    for (int64_t i = E.off[t]; i < E.off[t + 1]; ++i)
      if (E.left[i] != -1) u[E.feat[i]].push_back(E.thr[i] == 0.f ? 0.f : E.thr[i]);
  std::vector<int> fc_feat;
  for (int f = 0; f < E.F; ++f) {
    std::sort(u[f].begin(), u[f].end());
    u[f].erase(std::unique(u[f].begin(), u[f].end()), u[f].end());
    if (!u[f].empty()) fc_feat.push_back(f);
  }
  auto code = [&](int f, float x) -> uint32_t {   // the definition: c(x) = #{u <= x} (LT), #{u < x} (LE)
    if (x != x) return 0xFFFFu;
    uint32_t c = 0;
    for (float v : u[f]) c += E.cmp == 0 ? (v <= x) : (v < x);
    return c;
  };
  const int D = m.depth, P = 1 << D, w = E.w;
  const uint8_t *trees = static_cast<const uint8_t *>(m.d_trees);
  for (int lt = 0; lt < m.n_trees_pad; ++lt) {
    const uint8_t *rec = trees + (size_t)lt * m.stride;
    const uint32_t *node = reinterpret_cast<const uint32_t *>(rec);
    const int local = (int)(node[0] >> 8) - 1;
    if (local < 0) continue;
    const int t = m.tree_begin + local;
    for (int r = 0; r < n; ++r) {
      const float *x = &X[(size_t)r * E.F];
      uint32_t i = 1;
      for (int l = 0; l < D; ++l) {
        const uint32_t nd = node[i], off = nd >> 16, k = nd & 0xFFFFu;
        const int fc = m.rank_cw == 32 ? (int)(off / 128) : (int)((off / 128) * 2 + (off % 128) / 2);
        bool left;
        if (k == 0xFFFFu) left = true;                      // padding node
        else {
          REQUIRE(fc < (int)fc_feat.size(), "rank fc out of range");
          if (fc >= (int)fc_feat.size()) return;
          left = k >= code(fc_feat[fc], x[fc_feat[fc]]);
        }
        i = 2 * i + (left ? 0 : 1);
      }
      const int slot = (int)(i - (uint32_t)P);
      const int want = walk(E, t, x);
      REQUIRE(m.d_leafmap[(size_t)lt * P + slot] == want, "PTT rank leaf tree %d row %d", t, r);
      const float *leaf = reinterpret_cast<const float *>(rec + (size_t)4 * P);
      for (int k = 0; k < w; ++k)
        REQUIRE(f2u(leaf[(size_t)slot * w + k]) == f2u(leafv(E, t, want, k)), "PTT rank value");
    }
  }
  if (!m.rank_pre) {
    // in-kernel codes: per feature an Eytzinger search array (itself a
    // perfect-tree walk: L steps of i <- 2i + (u_i sorts before x), code =
    // i - 2^L) that must give the definition's code
    const uint8_t *aux = static_cast<const uint8_t *>(m.d_aux);
    const uint32_t *fmeta = reinterpret_cast<const uint32_t *>(aux);
    const uint32_t *groups = reinterpret_cast<const uint32_t *>(aux + m.aux_groups_off);
    const uint8_t *pool = aux + m.aux_pool_off;
    for (int c = 0; c < (int)fc_feat.size(); ++c) {
      const uint32_t *fm = fmeta + 4 * c;
      REQUIRE((int)fm[0] == fc_feat[c], "eytzinger feature id");
      const float *ey = reinterpret_cast<const float *>(pool + groups[4 * fm[3]] + fm[2]);
      for (int r = 0; r < n; ++r) {
        const float x = X[(size_t)r * E.F + fc_feat[c]];
        if (x != x) continue;
        uint32_t i = 1;
        for (uint32_t l = 0; l < fm[1]; ++l) i = 2 * i + (E.cmp == 0 ? (ey[i] <= x) : (ey[i] < x));
        REQUIRE(i - (1u << fm[1]) == code(fc_feat[c], x), "eytzinger code feature %d", fc_feat[c]);
      }
    }
    return;
  }
  // pre-pass bucket tables: the bucket search (bucket by the recorded map,
  // then a scan of that bucket) must give the definition's code
  const uint8_t *rb = static_cast<const uint8_t *>(m.d_rb);
  const uint32_t *feat = reinterpret_cast<const uint32_t *>(rb);
  const uint32_t *groups = reinterpret_cast<const uint32_t *>(rb + m.rb_groups_off);
  const uint8_t *pool = rb + m.rb_pool_off;
  const int per_word = m.rank_cw == 32 ? 1 : 2;
  int words_seen = 0, max_feats = 0;
  for (int g = 0; g < m.rb_ngroups; ++g) {
    const uint32_t *G = groups + 8 * g;
    REQUIRE((int)G[2] == words_seen && G[3] > G[2], "bucket groups must tile the code words");
    words_seen = (int)G[3];
    const int cb = (int)G[2] * per_word, ce = std::min((int)G[3] * per_word, (int)fc_feat.size());
    max_feats = std::max(max_feats, ce - cb);
    if (m.rb_tma) {
      // TMA pre-pass: one 16-B box {aligned 4-column block} per row holds
      // every x of the group, and the group's tables are SMEM-resident
      REQUIRE((int)G[4] == fc_feat[cb], "TMA group first column");
      for (int c = cb; c < ce; ++c)
        REQUIRE(fc_feat[c] == fc_feat[cb] + (c - cb) && (fc_feat[c] >> 2) == (fc_feat[cb] >> 2),
                "TMA group columns %d..%d not one aligned 4-column run", fc_feat[cb], fc_feat[ce - 1]);
      REQUIRE(G[1] <= kRcTmaTableMax, "TMA group tables exceed the SMEM budget");
    }
    for (int wd = (int)G[2]; wd < (int)G[3]; ++wd)
      for (int q = 0; q < per_word; ++q) {
        const int c = wd * per_word + q;
        if (c >= (int)fc_feat.size()) continue;
        const uint32_t *fm = feat + 8 * c;
        REQUIRE((int)fm[0] == fc_feat[c], "bucket feature id");
        const uint32_t B = fm[1];
        const float lo = u2f(fm[4]), hi = u2f(fm[5]), s = u2f(fm[6]);
        const uint8_t *tb = pool + G[0];
        for (int r = 0; r < n; ++r) {
          const float x = X[(size_t)r * E.F + fc_feat[c]];
          if (x != x) continue;
          volatile float xc = std::fmin(std::fmax(x, lo), hi);
          volatile float d = xc - lo;
          volatile float y = d * s;
          const uint32_t b = (uint32_t)std::fmin((float)y, (float)(B - 1u));
          uint32_t be;
          std::memcpy(&be, tb + fm[3] + 4 * b, 4);
          uint32_t base = be & 0xFFFF, cnt = be >> 16;
          const float *uu = reinterpret_cast<const float *>(tb + fm[7]);
          uint32_t got = base;
          for (uint32_t j = 0; j < cnt; ++j) got += E.cmp == 0 ? (uu[base + j] <= x) : (uu[base + j] < x);
          REQUIRE(got == code(fc_feat[c], x), "bucket code feature %d x %g: %u vs %u", fc_feat[c], x, got,
                  code(fc_feat[c], x));
          {
            // the pre-pass kernels' fixed window: S_g power-of-two steps from
            // the bucket start over 2^S_g - 1 slots, which must stay inside
            // the group's tables (NaN pads, later buckets compare false)
            uint32_t sg = 0;
            for (int c2 = cb; c2 < ce; ++c2) sg = std::max(sg, feat[8 * c2 + 2]);
            REQUIRE(fm[7] + 4 * ((size_t)base + (1u << sg) - 1) <= G[1], "TMA window past the group tables");
            uint32_t pos = base;
            for (int k = (int)sg - 1; k >= 0; --k) {
              const float v = uu[pos + (1u << k) - 1];
              if (E.cmp == 0 ? v <= x : v < x) pos += 1u << k;
            }
            REQUIRE(pos == code(fc_feat[c], x), "TMA window code feature %d x %g: %u vs %u", fc_feat[c], x, pos,
                    code(fc_feat[c], x));
          }
        }
      }
  }
  REQUIRE(words_seen == m.rank_nwords, "bucket groups cover %d of %d words", words_seen, m.rank_nwords);
  REQUIRE(m.rb_max_feats == max_feats, "rb_max_feats %d vs %d", m.rb_max_feats, max_feats);
}

static void check_tt_wide(const Ens &E, const Model &m, const std::vector<float> &X, int n) {
  const uint32_t *words = static_cast<const uint32_t *>(m.d_ttw);
  for (int lt = 0; lt < m.n_trees; ++lt) {
    const int t = m.tree_begin + lt;
    const uint32_t *T = words + (size_t)m.d_ttw_off[lt] * 4;
    const uint32_t nrec = T[0];
    for (int r = 0; r < n; ++r) {
      const float *x = &X[(size_t)r * E.F];
      uint32_t q = 0, side = 0, pay = 0;
      for (int l = 0; l <= std::max(m.depth, 1); ++l) {
        REQUIRE(q < nrec, "TT wide record index %u >= %u", q, nrec);
        if (q >= nrec) return;
        const uint32_t *d = T + 4 + 4 * q;
        // word 0 = byte offset 4 R f of the feature's column in the R-row X tile | flags
        const int R = m.cfg.wide_rows;
        REQUIRE(R > 0 && (d[0] & ~3u) % (4u * R) == 0, "TT wide feature offset");
        const bool pr = pred(E.cmp, x[orig_feature(m, (int)((d[0] & ~3u) / (4u * R)))], u2f(d[1]));
        const uint32_t nx = pr ? d[2] : d[3];
        if (d[0] & (pr ? 1u : 2u)) { side = pr ? 1 : 2; pay = nx; break; }
        q = nx;
      }
      REQUIRE(side != 0, "TT wide walk did not end within depth");
      const int want = walk(E, t, x);
      const uint32_t *ids = reinterpret_cast<const uint32_t *>(reinterpret_cast<const uint8_t *>(T) + T[1]);
      REQUIRE((int)ids[2 * q + side - 1] == want, "TT wide leaf tree %d row %d", t, r);
      if (E.w == 1) {
        REQUIRE(pay == f2u(leafv(E, t, want, 0)), "TT wide value");
        if (E.K > 1) REQUIRE((int)T[2] == (E.use_tout ? E.tout[t] : t % E.K), "TT wide class");
      } else {
        const float *v = reinterpret_cast<const float *>(reinterpret_cast<const uint8_t *>(T) + T[3]);
        for (int k = 0; k < E.w; ++k) REQUIRE(f2u(v[pay * E.w + k]) == f2u(leafv(E, t, want, k)), "TT wide vector");
      }
    }
  }
}

static void check_gemm(const Ens &E, const Model &m, const std::vector<float> &X, int n) {
  const GemmGeom g = gemm_geom(m.gemm_ni, m.gemm_nl, E.w);
  const uint8_t *trees = static_cast<const uint8_t *>(m.d_trees);
  for (int lt = 0; lt < m.n_trees; ++lt) {
    const int t = m.tree_begin + lt;
    const uint8_t *rec = trees + (size_t)lt * g.stride;
    const uint32_t *feat = reinterpret_cast<const uint32_t *>(rec + g.off_feat);
    const float *thr = reinterpret_cast<const float *>(rec + g.off_thr);
    const uint64_t *lm = reinterpret_cast<const uint64_t *>(rec + g.off_lm);
    const uint64_t *rm = reinterpret_cast<const uint64_t *>(rec + g.off_rm);
    const uint32_t *Dv = reinterpret_cast<const uint32_t *>(rec + g.off_d);
    for (int r = 0; r < n; ++r) {
      const float *x = &X[(size_t)r * E.F];
      uint64_t Tb = 0;
      for (int i = 0; i < g.ni; ++i) Tb |= (uint64_t)pred(E.cmp, x[feat[i]], thr[i]) << i;
      int matches = 0, sel = 0;
      for (int j = 0; j < g.nl; ++j) {
        const int S = __builtin_popcountll(Tb & lm[j]) - __builtin_popcountll(Tb & rm[j]);
        if (S == (int)Dv[j]) { ++matches; sel = j; }
      }
      REQUIRE(matches == 1, "GEMM: %d leaf columns match (exactly one expected, DESIGN R8)", matches);
      REQUIRE(m.d_leafmap[(size_t)lt * g.nl + sel] == walk(E, t, x), "GEMM leaf tree %d row %d", t, r);
    }
  }
}

// ---- corruptions hb_validate must reject
static bool corrupt(Ens &E) {
  const int n = (int)E.feat.size();
  std::vector<int> internal, leaves;
  for (int i = 0; i < n; ++i) (E.left[i] == -1 ? leaves : internal).push_back(i);
  switch (rnd(14)) {
    case 0: if (internal.empty()) return false; E.left[internal[rnd((int)internal.size())]] = 1 << 20; return true;
    case 1: if (internal.empty()) return false; E.right[internal[rnd((int)internal.size())]] = -1; return true;
    case 2: if (internal.empty()) return false; { int i = internal[rnd((int)internal.size())]; E.right[i] = E.left[i]; } return true;
    case 3: { // a child pointing back at the root (cycle / root with a parent)
      if (internal.empty()) return false;
      const int i = internal[rnd((int)internal.size())];
      int t = 0;
      while (E.off[t + 1] <= i) ++t;
      E.left[i] = 0;
      return true;
    }
    case 4: if (internal.empty()) return false; E.thr[internal[rnd((int)internal.size())]] = NAN; return true;
    case 5: if (internal.empty()) return false; E.feat[internal[rnd((int)internal.size())]] = E.F + rnd(5); return true;
    case 6: if (internal.empty()) return false; E.feat[internal[rnd((int)internal.size())]] = -1 - rnd(5); return true;
    case 7: E.val[(size_t)leaves[rnd((int)leaves.size())] * E.w] = rnd(2) ? INFINITY : NAN; return true;
    case 8: E.cmp = 2 + rnd(3); return true;
    case 9: E.post = 4 + rnd(3); return true;
    case 10: if (E.T < 2) return false; std::swap(E.off[1], E.off[E.T]); return E.off[1] != E.off[E.T];
    case 11: E.w = E.K + 1; return true;   // leaf_width neither 1 nor K (arrays stay large enough: w only grows reads ≤ val size? no: guarded below)
    case 12: if (!E.use_tout && E.w == 1) { E.use_tout = true; E.tout[rnd(E.T)] = E.K + rnd(3); return true; } return false;
    case 13: { // two parents for one node: point a second internal node at another's child
      if (internal.size() < 2) return false;
      const int a = internal[rnd((int)internal.size())], b = internal[rnd((int)internal.size())];
      int ta = 0, tb = 0;
      while (E.off[ta + 1] <= a) ++ta;
      while (E.off[tb + 1] <= b) ++tb;
      if (ta != tb || a == b || E.left[b] == E.left[a]) return false;
      E.left[a] = E.left[b];
      return true;
    }
  }
  return false;
}

int main(int argc, char **argv) {
  const long iters = argc > 1 ? std::atol(argv[1]) : 200;
  rng.seed(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1);
  long compiled = 0, rejected = 0, checked_rows = 0;
  long n_fp32 = 0, n_rank = 0, n_pre = 0, n_ttw = 0, n_gemm = 0, n_cw16 = 0, n_tma = 0;
  const int strategies[4] = {HB_STRATEGY_AUTO, HB_STRATEGY_PTT, HB_STRATEGY_TT, HB_STRATEGY_GEMM};
  for (long it = 0; it < iters; ++it) {
    // layout choices the compile reads from the environment: cover every
    // PTT layout (fp32 nodes; rank codes in the scorer or from the pre-pass,
    // 32- or 16-bit cells; TMA or generic pre-pass groups) and TT (narrow / wide rows, tree chunks)
    static const char *rank[] = {"-1", "0", "1"}, *pre[] = {"-1", "0", "1"}, *cw[] = {"0", "32", "16"},
                      *wide[] = {"-1", "1"}, *chunk[] = {"-1", "0", "4"}, *rctma[] = {"0", "1"};
    setenv("HB_PTT_RANK", rank[rnd(3)], 1);
    setenv("HB_RANK_PRE", pre[rnd(3)], 1);
    setenv("HB_RANK_CW", cw[rnd(3)], 1);
    setenv("HB_TT_WIDE", wide[rnd(2)], 1);
    setenv("HB_TT_CHUNK", chunk[rnd(3)], 1);
    setenv("HB_RC_TMA", rctma[rnd(2)], 1);
    Ens E = random_ensemble();
    hb_ensemble v = E.view();
    REQUIRE(hb_validate(&v) == HB_OK, "valid ensemble rejected (iteration %ld)", it);
    const int n = 24;
    const std::vector<float> X = random_rows(E, n);
    for (int s : strategies) {
      const int t0 = rnd(4) == 0 ? rnd(E.T) : 0;
      const int t1 = t0 + 1 + rnd(E.T - t0);
      Model *m = nullptr;
      const hb_status st = compile_model_host(&v, t0, t1, s, &m);
      REQUIRE(st == HB_OK || st == HB_E_UNSUPPORTED, "compile strategy %d -> %d", s, st);
      if (st != HB_OK) continue;
      ++compiled;
      if (m->strategy == HB_STRATEGY_PTT && !m->ptt_rank) check_ptt_fp32(E, *m, X, n), ++n_fp32;
      if (m->strategy == HB_STRATEGY_PTT && m->ptt_rank) check_ptt_rank(E, *m, X, n, t0, t1), ++n_rank, n_pre += m->rank_pre, n_cw16 += m->rank_cw == 16, n_tma += m->rb_tma;
      if (m->strategy == HB_STRATEGY_TT && m->d_ttw) check_tt_wide(E, *m, X, n), ++n_ttw;
      if (m->strategy == HB_STRATEGY_GEMM && !m->gemm_tc) check_gemm(E, *m, X, n), ++n_gemm;
      checked_rows += n;
      free_model_any(m);
    }
    // one corruption of the same ensemble
    Ens C = E;
    if (!corrupt(C)) continue;
    if (C.w > E.w) C.val.resize(C.val.size() / E.w * C.w, 1.f);   // keep the arrays as long as declared
    hb_ensemble cv = C.view();
    const hb_status vs = hb_validate(&cv);
    REQUIRE(vs != HB_OK, "corrupted ensemble accepted (iteration %ld)", it);
    Model *m = nullptr;
    const hb_status cs = compile_model_host(&cv, 0, C.T, HB_STRATEGY_AUTO, &m);
    REQUIRE(cs == vs && m == nullptr, "compile of a corrupted ensemble: %d vs validate %d", cs, vs);
    if (m) free_model_any(m);
    ++rejected;
  }
  std::printf("fuzz_layout: %ld iterations, %ld models compiled and interpreted (%ld row checks: "
              "PTT fp32 %ld, PTT rank %ld (pre-pass tables %ld of them TMA groups %ld, 16-bit cells %ld), wide TT %ld, "
              "GEMM %ld), %ld corruptions rejected, %d failures\n", iters, compiled, checked_rows, n_fp32, n_rank, n_pre,
              n_tma, n_cw16,
              n_ttw, n_gemm, rejected, failures);
  return failures ? 1 : 0;
}
