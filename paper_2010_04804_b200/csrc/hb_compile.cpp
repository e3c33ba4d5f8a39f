// hb_compile.cpp — host-side layout compilers of the GEMM strategy (Alg. 1,
// Table 3), the rank-coded PTT layout (Alg. 3, Tables 6) and the rank-code
// pre-pass tables. Pure host C++: every device copy goes through dev_upload
// (hb_host.cpp), so these also run in the host-only compile the fuzz build
// uses (tests/fuzz/fuzz_layout.cpp). The PTT / TT builders are in hb_host.cpp.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hb_internal.h"
#include "hb_layouts.h"

namespace hb {

// memcpy of possibly empty vectors (their data() may be null: memcpy with a
// null pointer is undefined even for 0 bytes; found by the UBSan fuzz build)
static inline void copy_bytes(void *dst, const void *src, size_t n) {
  if (n) std::memcpy(dst, src, n);
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
  hb_status st = dev_upload(m, buf.data(), buf.size(), &m->d_trees);
  if (st != HB_OK) return st;
  st = dev_upload(m, leafmap.data(), leafmap.size() * 4, reinterpret_cast<void **>(&m->d_leafmap));
  if (st != HB_OK) return st;
  m->cfg = LaunchCfg();
  m->cfg.nw = 4;
  m->cfg.x_smem = 0;
  m->cfg.t_smem = 0;
  return HB_OK;
}


static inline uint16_t bf16_bits(float f) {  // exact for {-1, 0, 1}
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16);
}

bool gemm_tc_eligible(const hb_ensemble *e, int t0, int t1) {
  for (int t = t0; t < t1; ++t) {
    const int64_t a = e->node_offset[t], b = e->node_offset[t + 1];
    int ni = 0, nl = 0;
    for (int64_t i = a; i < b; ++i) (e->left[i] == -1 ? nl : ni)++;
    if (ni > 8 || nl > 8) return false;
  }
  return true;
}

hb_status compile_gemm_tc(const hb_ensemble *e, int t0, int t1, Model *m) {
  const int w = e->leaf_width;
  const TcGeom g = tc_geom(w);
  const int T = t1 - t0;
  const int ngroups = (T + kTcTrees - 1) / kTcTrees;
  // feature-selection injection: the X tile holds used features only
  std::vector<int32_t> remap(e->n_features, -1), used;
  for (int t = t0; t < t1; ++t)
    for (int64_t i = e->node_offset[t]; i < e->node_offset[t + 1]; ++i)
      if (e->left[i] != -1) remap[e->feature[i]] = 1;
  for (int f = 0; f < e->n_features; ++f)
    if (remap[f] == 1) {
      remap[f] = (int32_t)used.size();
      used.push_back(f);
    }
  if (used.empty()) used.push_back(0), remap[0] = 0;
  // X slice of the 128-row tile in SMEM when the used columns fit next to
  // the two A tiles, the record ring and the barriers (gemm_tc_kernel)
  const TcGeom g0 = tc_geom(e->leaf_width);
  const long fixed = (long)gemm_tc_a_region(m->nacc) + 3L * (long)g0.stride + 128;
  const bool fits = 4L * (long)used.size() * 128 + fixed <= (long)kSmemBudget;
  // compact only when it removes a real share of the columns (see feature_map)
  const char *fs = std::getenv("HB_FSEL_MAX_PCT");
  const long pct = fs && *fs ? std::atol(fs) : 75;
  const bool compact = fits && (long)used.size() * 100 <= pct * e->n_features;
  if (!compact)
    for (int f = 0; f < e->n_features; ++f) remap[f] = f;
  std::vector<uint8_t> buf((size_t)ngroups * g.stride, 0);
  std::vector<int32_t> leafmap((size_t)ngroups * kTcTrees * 8, -1);
  std::vector<int> ipos, lpos, stack;
  for (int gi = 0; gi < ngroups; ++gi) {
    uint8_t *rec = buf.data() + (size_t)gi * g.stride;
    uint16_t *bimg = reinterpret_cast<uint16_t *>(rec + g.off_b);
    uint32_t *feat = reinterpret_cast<uint32_t *>(rec + g.off_feat);
    float *thr = reinterpret_cast<float *>(rec + g.off_thr);
    float *dval = reinterpret_cast<float *>(rec + g.off_d);
    uint32_t *tout = reinterpret_cast<uint32_t *>(rec + g.off_tout);
    float *E = reinterpret_cast<float *>(rec + g.off_e);
    for (int q = 0; q < kTcTrees; ++q) {
      for (int i = 0; i < 8; ++i) {
        thr[q * 8 + i] = INFINITY;
        dval[q * 8 + i] = kTcDPad;
      }
      const int lt = gi * kTcTrees + q;
      if (lt >= T) {  // zero tree: column 0 (C = 0, D = 0) always matches, E = 0
        dval[q * 8] = 0.f;
        continue;
      }
      const int t = t0 + lt;
      const int64_t a = e->node_offset[t];
      const int n = (int)(e->node_offset[t + 1] - a);
      tout[q] = (uint32_t)(w == 1 ? (e->tree_output ? e->tree_output[t] : t % e->n_outputs) : 0);
      ipos.assign(n, -1);
      lpos.assign(n, -1);
      int ci = 0, cl = 0;
      for (int i = 0; i < n; ++i) {
        if (e->left[a + i] != -1) ipos[i] = ci++;
        else lpos[i] = cl++;
      }
      for (int i = 0; i < n; ++i) {
        if (ipos[i] >= 0) {
          feat[q * 8 + ipos[i]] = (uint32_t)remap[e->feature[a + i]];
          thr[q * 8 + ipos[i]] = e->threshold[a + i];
        } else {
          for (int k = 0; k < w; ++k)
            E[((size_t)q * 8 + lpos[i]) * w + k] = e->leaf_value[(a + i) * w + k];
          leafmap[(size_t)lt * 8 + lpos[i]] = i;
        }
      }
      // C (Table 3): +1 left subtree, -1 right subtree; D_j = #left edges (R5)
      int dcount[8] = {0};
      const int pair = q >> 1, half = q & 1;
      for (int i = 0; i < n; ++i) {
        if (ipos[i] < 0) continue;
        for (int side = 0; side < 2; ++side) {
          stack.assign(1, side == 0 ? e->left[a + i] : e->right[a + i]);
          while (!stack.empty()) {
            const int k = stack.back();
            stack.pop_back();
            if (e->left[a + k] == -1) {
              const int j = lpos[k];
              // B[nrow][kcol] with nrow = leaf column (half*8 + j), kcol = node (half*8 + i)
              const int nrow = half * 8 + j, kcol = half * 8 + ipos[i];
              const int core = (nrow >> 3) * 2 + (kcol >> 3);  // SBO = 256 B = 2 cores, LBO = 128 B
              bimg[pair * 256 + core * 64 + (nrow & 7) * 8 + (kcol & 7)] =
                  bf16_bits(side == 0 ? 1.f : -1.f);
              if (side == 0) dcount[j]++;
            } else {
              stack.push_back(e->left[a + k]);
              stack.push_back(e->right[a + k]);
            }
          }
        }
      }
      for (int j = 0; j < cl; ++j) dval[q * 8 + j] = (float)dcount[j];
    }
  }
  m->stride = g.stride;
  m->nslots = 8;
  m->n_trees_pad = ngroups * kTcTrees;
  hb_status st = dev_upload(m, buf.data(), buf.size(), &m->d_trees);
  if (st != HB_OK) return st;
  st = dev_upload(m, leafmap.data(), leafmap.size() * 4, reinterpret_cast<void **>(&m->d_leafmap));
  if (st != HB_OK) return st;
  if (compact) {
    st = dev_upload(m, used.data(), used.size() * 4, reinterpret_cast<void **>(&m->d_fmap));
    if (st != HB_OK) return st;
  }
  m->n_xf = compact ? (int)used.size() : e->n_features;
  const long xb = 4L * m->n_xf * 128;
  m->cfg = LaunchCfg();
  m->cfg.nw = 16;
  m->cfg.x_smem = fits ? 1 : 0;
  m->cfg.t_smem = 1;
  m->cfg.smem_bytes = (int)((m->cfg.x_smem ? xb : 0) + fixed);
  // 16 warps per CTA, 256 TMEM columns each: up to 2 CTAs per SM (threads,
  // TMEM: 2 x 256 of 512 columns) when SMEM allows
  m->cfg.ctas_per_sm = std::max(1, std::min(2, (int)(kSmemBudget / std::max(1, m->cfg.smem_bytes))));
  m->gemm_tc = 1;
  return HB_OK;
}


namespace {
// Host twin of the bucket map in rank_code(): same fp32 operations, same
// order, no contraction (volatile intermediates).
uint32_t host_bucket(float x, float lo, float hi, float s, uint32_t B) {
  volatile float xc = std::fmin(std::fmax(x, lo), hi);
  volatile float d = xc - lo;
  volatile float y = d * s;
  const float yy = std::fmin((float)y, (float)(B - 1u));
  return (uint32_t)yy;
}

}  // namespace

// Bucket tables for the sorted distinct thresholds of each compact feature
// (sorted[c], feature id orig[c]); words group 1 (CW 32) or 2 (CW 16) features.
hb_status build_rank_buckets(const std::vector<std::vector<float>> &sorted, const std::vector<int> &orig,
                             int cw, RankBuckets *out, size_t cap_bytes, int density, bool one_per_group,
                             bool block4) {
  const float pad_nan = NAN;
  // per-CTA table budget: 48 KB -> 4 CTAs (32 warps) per SM (HB_RC_SMEM_KB overrides)
  const char *ev = std::getenv("HB_RC_SMEM_KB");
  const size_t cap = cap_bytes ? cap_bytes
                               : std::min<size_t>(kRcSmemMax, (ev && *ev ? (size_t)std::atoi(ev) : 48) * 1024);
  out->smem_cap = cap;
  const int n_fc = (int)sorted.size();
  const int per_word = cw == 32 ? 1 : 2;
  const int n_words = (n_fc + per_word - 1) / per_word;
  RankBuckets R;
  R.n_words = n_words;
  R.feat.assign((size_t)n_fc * 8, 0u);
  std::vector<std::vector<uint8_t>> tabs(n_fc);
  for (int c = 0; c < n_fc; ++c) {
    const std::vector<float> &u = sorted[c];
    const uint32_t m = (uint32_t)u.size();
    float lo = 0.f, hi = 0.f;
    bool any = false;
    for (float v : u)
      if (std::isfinite(v)) {
        if (!any) lo = v;
        hi = v;
        any = true;
      }
    // <= 2 thresholds per bucket on average (HB_RC_DENSITY=d: <= 2/d)
    static const int dens_env = [] {
      const char *e = std::getenv("HB_RC_DENSITY");
      return e && *e ? std::max(1, std::atoi(e)) : 1;
    }();
    const int dens = density > 0 ? density : dens_env;
    uint32_t B = 1;
    while (2 * B < m * (uint32_t)dens && B < 16384u) B <<= 1;
    float s = 0.f;
    if (hi > lo) {
      const float range = hi - lo;
      s = std::isfinite(range) ? (float)B / range : (float)B / FLT_MAX;
      if (!(s <= FLT_MAX)) s = FLT_MAX;     // tiny range: keep s finite (0 * s must stay 0)
      if (!(s > 0.f)) s = FLT_MIN;
    } else {
      B = 1;
    }
    std::vector<uint32_t> start(B + 1, 0);
    std::vector<uint32_t> bk(m);
    for (uint32_t j = 0; j < m; ++j) bk[j] = host_bucket(u[j], lo, hi, s, B);
    uint32_t maxocc = 0;
    {
      uint32_t j = 0;
      for (uint32_t b = 0; b <= B; ++b) {
        while (j < m && bk[j] < b) ++j;
        start[b] = j;
      }
      for (uint32_t b = 0; b < B; ++b) maxocc = std::max(maxocc, start[b + 1] - start[b]);
    }
    uint32_t S = 0;
    while ((1u << S) <= maxocc) ++S;        // bit_length(maxocc) search steps
    const size_t sbytes = (size_t)B * 4;
    const size_t ubytes = ((size_t)(m + 1) * 4);
    std::vector<uint8_t> t(sbytes + ubytes, 0);
    for (uint32_t b = 0; b < B; ++b) {
      const uint32_t v = start[b] | ((start[b + 1] - start[b]) << 16);
      std::memcpy(t.data() + 4 * b, &v, 4);
    }
    std::memcpy(t.data() + sbytes, u.data(), (size_t)m * 4);
    // pad slot(s) after the thresholds: NaN compares false against every x,
    // so a fixed-window search (TMA kernel) never counts them
    const float pad = NAN;
    std::memcpy(t.data() + sbytes + (size_t)m * 4, &pad, 4);
    tabs[c] = std::move(t);
    uint32_t *fm = R.feat.data() + (size_t)c * 8;
    fm[0] = (uint32_t)orig[c];
    fm[1] = B;
    fm[2] = S;
    fm[3] = 0;                                 // start offset: set when grouped
    std::memcpy(&fm[4], &lo, 4);
    std::memcpy(&fm[5], &hi, 4);
    std::memcpy(&fm[6], &s, 4);
    fm[7] = (uint32_t)sbytes;                  // u offset relative to start; rebased below
  }
  // Groups of whole words (pass 1), each <= cap bytes with its pads (an
  // oversized word is a group of its own and is searched from global
  // memory); one word per group for the column kernel (one_per_group). With
  // block4 (TMA pre-pass) a group is also a run of consecutive X columns
  // inside one aligned 4-column block, so one 16-B box per row holds every x
  // it searches.
  // Every pre-pass kernel searches a fixed window of 2^S_g - 1 slots from the
  // bucket's first threshold (S_g = the group's deepest search): thresholds
  // of later buckets are > x and the pads are NaN (false against every x),
  // so "u <= x" holds on a prefix of the window and its length completes the
  // code. Each table therefore ends with max(1, 2^S_g - 1) NaN slots.
  auto S_of = [&](int c) { return R.feat[(size_t)c * 8 + 2]; };
  auto padded = [&](int c, uint32_t sg) {          // table bytes with the group's pads, 16-B rounded
    const size_t pads = std::max<size_t>(1, ((size_t)1 << sg) - 1);
    return (tabs[c].size() - 4 + 4 * pads + 15) & ~size_t(15);
  };
  std::vector<int> gstart(n_words + 1, 0);         // 1 where a group starts
  {
    auto group_bytes = [&](int w0, int w1, uint32_t sg) {
      size_t b = 0;
      for (int c = w0 * per_word; c < std::min(w1 * per_word, n_fc); ++c) b += padded(c, sg);
      return b;
    };
    int first = 0;
    uint32_t sg = 0;
    for (int wd = 0; wd < n_words; ++wd) {
      uint32_t sw = 0;
      for (int q = 0; q < per_word && wd * per_word + q < n_fc; ++q) sw = std::max(sw, S_of(wd * per_word + q));
      bool split = wd == 0 || one_per_group;
      if (!split && block4) {
        const int c = wd * per_word, cfirst = first * per_word;
        for (int q = 0; q < per_word && c + q < n_fc; ++q)
          if (orig[c + q] != orig[c - 1] + 1 + q || (orig[c + q] >> 2) != (orig[cfirst] >> 2)) split = true;
      }
      if (!split && group_bytes(first, wd + 1, std::max(sg, sw)) > cap) split = true;
      if (split) {
        gstart[wd] = 1;
        first = wd;
        sg = 0;
      }
      sg = std::max(sg, sw);
    }
    gstart[n_words] = 1;
    for (int w0 = 0; w0 < n_words;) {
      int w1 = w0 + 1;
      while (!gstart[w1]) ++w1;
      uint32_t sgg = 0;
      for (int c = w0 * per_word; c < std::min(w1 * per_word, n_fc); ++c) sgg = std::max(sgg, S_of(c));
      for (int c = w0 * per_word; c < std::min(w1 * per_word, n_fc); ++c) {
        std::vector<uint8_t> &t = tabs[c];
        const size_t old = t.size(), want = old - 4 + 4 * std::max<size_t>(1, ((size_t)1 << sgg) - 1);
        t.resize(want);
        for (size_t i = old; i < want; i += 4) std::memcpy(t.data() + i, &pad_nan, 4);
      }
      w0 = w1;
    }
  }
  // groups of whole words, <= cap bytes each (an oversized word is a
  // group of its own and is searched from global memory)
  size_t goff = 0, gbytes = 0;
  int wbeg = 0;
  auto close = [&](int wend) {
    // X columns the group's features span (the staged kernel copies them)
    int clo = INT32_MAX, chi = -1;
    for (int c = wbeg * per_word; c < std::min(wend * per_word, n_fc); ++c) {
      clo = std::min(clo, orig[c]);
      chi = std::max(chi, orig[c]);
    }
    const uint32_t ncols = chi >= clo ? (uint32_t)(chi - clo + 1) : 0u;
    R.groups.insert(R.groups.end(), {(uint32_t)goff, (uint32_t)gbytes, (uint32_t)wbeg, (uint32_t)wend,
                                     (uint32_t)(chi >= clo ? clo : 0), ncols, ncols | 1u, 0u});
    R.max_span = std::max<uint32_t>(R.max_span, ncols);
    R.max_feats = std::max(R.max_feats, std::min(wend * per_word, n_fc) - wbeg * per_word);
    for (int c = wbeg * per_word + 1; c < std::min(wend * per_word, n_fc); ++c)
      if (orig[c] != orig[c - 1] + 1 || (orig[c] >> 2) != (orig[wbeg * per_word] >> 2)) R.block4_ok = false;
    if (gbytes > cap) R.any_global = true;
    R.max_group_bytes = std::max(R.max_group_bytes, gbytes <= cap ? gbytes : (size_t)0);
    goff += gbytes;
    gbytes = 0;
    wbeg = wend;
    R.n_groups++;
  };
  for (int wd = 0; wd < n_words; ++wd) {
    if (gbytes > 0 && gstart[wd]) close(wd);
    for (int q = 0; q < per_word && wd * per_word + q < n_fc; ++q) {
      const int c = wd * per_word + q;
      uint32_t *fm = R.feat.data() + (size_t)c * 8;
      fm[3] = (uint32_t)gbytes;
      fm[7] += (uint32_t)gbytes;
      const size_t tb = (tabs[c].size() + 15) & ~size_t(15);
      tabs[c].resize(tb, 0);
      R.pool.insert(R.pool.end(), tabs[c].begin(), tabs[c].end());
      gbytes += tb;
    }
  }
  if (gbytes) close(n_words);
  R.smem_cap = cap;
  *out = std::move(R);
  return HB_OK;
}


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
  // rpl: rows per lane (2: each warp holds two 32-row code blocks, pre-pass only)
  auto try_cfg = [&](int cw, bool pre, LaunchCfg &cfg, int rpl = 1) {
    if (cw == 32 && A.n_fc > 511) return false;
    const long tile = (cw == 32 ? (long)A.n_fc * 128 : (long)((A.n_fc + 1) / 2) * 128) * rpl;
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
    // 98.9M). With 16-bit pre-pass cells it did not in round 1 (C4': 404.8M
    // vs 420.8M); since the window-search pre-pass (round 2) it does when
    // the walk is long next to the feature count (C4', T*D / n_fc = 74:
    // 427.9M vs 416.8M rows/s), HB_PRE16_MIN_RATIO (64)
    LaunchCfg pc;
    int pcw = 32;
    const double walk_ratio = (double)Tpad * (double)std::max(D, 1) / std::max(1, A.n_fc);
    if (pick_cw(true, pc, pcw) && pc.nw >= cfg.nw &&
        (pcw == 32 || walk_ratio >= (double)env_int2("HB_PRE16_MIN_RATIO", 64))) {
      pre = true;
      cfg = pc;
      cw = pcw;
    }
  }
  if (!ok && force_pre != 0) {
    // The pre-pass codes every used feature of every row (n_fc searches and
    // a code write + read per row) to make the T * D node visits per row
    // cheaper: it pays only when the walk is long next to the feature count.
    // Measured (profiles/r02_crossover.json): C2 / C3 / C4
    // (T*D / n_fc = 44 / 143 / 519) gain from it; the paper's Fig. 8 shape
    // (100 trees over 200 features, T*D / n_fc = 1.5-5) loses to fp32 nodes
    // at every batch size. Below HB_PRE_MIN_RATIO (16) AUTO keeps fp32 nodes.
    const double ratio = (double)Tpad * (double)std::max(D, 1) / std::max(1, A.n_fc);
    if (force_pre == -1 && force != 1 && ratio < (double)env_int2("HB_PRE_MIN_RATIO", 16))
      return HB_E_UNSUPPORTED;
    pre = true;
    ok = pick_cw(true, cfg, cw);
  }
  if (!ok) return HB_E_UNSUPPORTED;
  // two rows per lane (pttr_kernel<RPL = 2>): the top three levels are
  // shared by a lane's two rows; pre-pass codes and D >= 3 only. AUTO for
  // scalar-output models (C3 835.7M -> 885.0M rows/s, C2 581.4M -> 596.6M);
  // with 7 per-class accumulators per row (C4) the two rows' fp64 sums spill
  // (107.3M -> 63.6M), so K > 1 keeps one row per lane. HB_PTTR_RPL: 1 / 2
  // forces
  int rpl = 1;
  const int want_rpl = env_int2("HB_PTTR_RPL", 0);
  if (pre && D >= 3 && (want_rpl == 2 || (want_rpl == 0 && m->nacc == 1))) {
    LaunchCfg c2;
    if (try_cfg(cw, true, c2, 2)) {
      cfg = c2;
      rpl = 2;
    }
  }
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
  hb_status ust = dev_upload(m, buf.data(), buf.size(), &m->d_trees);
  if (ust != HB_OK) return ust;
  ust = dev_upload(m, leafmap.data(), leafmap.size() * 4, reinterpret_cast<void **>(&m->d_leafmap));
  if (ust != HB_OK) return ust;
  if (!pre) {
    const size_t fb = A.fmeta.size() * 4, gb = A.groups.size() * 4, pb = A.pool.size() * 4;
    const size_t pool_off = (fb + gb + 127) & ~size_t(127);
    std::vector<uint8_t> aux(pool_off + pb, 0);
    copy_bytes(aux.data(), A.fmeta.data(), fb);
    copy_bytes(aux.data() + fb, A.groups.data(), gb);
    copy_bytes(aux.data() + pool_off, A.pool.data(), pb);
    ust = dev_upload(m, aux.data(), aux.size(), &m->d_aux);
    if (ust != HB_OK) return ust;
    m->aux_groups_off = fb;
    m->aux_pool_off = pool_off;
    m->rank_ngroups = A.n_groups;
  } else {
    // pre-pass bucket tables: [feat | groups | pool]
    std::vector<int> origf;
    for (int f = 0; f < F; ++f)
      if (fc_of[f] >= 0) origf.push_back(f);
    RankBuckets R;
    // at most 32 used features with 32-bit cells: the pre-pass runs the
    // single-feature column kernel (hb_rank_codes.cu), one table per CTA;
    // HB_RC_ONE_DENS / HB_RC_ONE_CAP_KB size those tables (measured, §4.6.1)
    const int nwords_colk = cw == 32 ? A.n_fc : (A.n_fc + 1) / 2;
    // 16-bit cells whose words are aligned float2 pairs of X (every feature
    // used, F even) group several words for the direct kernel's (row, word)
    // lanes instead (C4': 1.164 -> 0.922 ms, 428.3M -> 437.5M rows/s)
    const bool pairs16 = cw == 16 && A.n_fc == F && F % 2 == 0;
    const bool colk = !pairs16 && nwords_colk <= env_int2("HB_RC_ONEK_MAX_GROUPS", 32);
    // TMA pre-pass (rank_code_tma_kernel, HB_RC_TMA=0 turns it off): one
    // group per aligned 4-column block of X (fewer when the tables outgrow
    // kRcTmaTableMax), every table SMEM-resident. Only for F % 4 == 0, where
    // a contiguous X has the 16-B row pitch the tensor map needs (C3; not
    // C2 / C4 with F = 90 / 54, which keep the groupings measured for the
    // generic kernels); calls with another pitch run the generic kernels on
    // these groups
    const int tma_env = env_int2("HB_RC_TMA", -1);
    bool tma = tma_env == 1 || (tma_env == -1 && F % 4 == 0);
    hb_status st = HB_OK;
    if (tma) {
      st = build_rank_buckets(sorted, origf, cw, &R, kRcTmaTableMax, 0, false, true);
      if (st != HB_OK) return st;
      tma = R.block4_ok && !R.any_global;
    }
    if (!tma) {
      R = RankBuckets();
      st = colk ? build_rank_buckets(sorted, origf, cw, &R, (size_t)env_int2("HB_RC_ONE_CAP_KB", 48) * 1024,
                                     env_int2("HB_RC_ONE_DENS", 1), true)
                : build_rank_buckets(sorted, origf, cw, &R);
      if (st != HB_OK) return st;
    }
    m->rb_tma = tma ? 1 : 0;
    m->rb_max_feats = R.max_feats;
    const size_t fb = R.feat.size() * 4, gb = R.groups.size() * 4;
    const size_t pool_off = (fb + gb + 127) & ~size_t(127);
    std::vector<uint8_t> aux(pool_off + R.pool.size(), 0);
    copy_bytes(aux.data(), R.feat.data(), fb);
    copy_bytes(aux.data() + fb, R.groups.data(), gb);
    copy_bytes(aux.data() + pool_off, R.pool.data(), R.pool.size());
    ust = dev_upload(m, aux.data(), aux.size(), &m->d_rb);
    if (ust != HB_OK) return ust;
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
  m->rank_rpl = rpl;
  return HB_OK;
}

}  // namespace hb
