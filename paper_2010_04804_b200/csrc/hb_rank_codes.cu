// hb_rank_codes.cu — rank-code pre-pass of the rank-coded PTT scorer (sm_100a).
//
// The rank-coded PTT layout (hb_pttr.cu) walks integer codes
// c(x) = #{j : u_j <= x} (LT; LE: u_j < x) instead of fp32 values, which keeps
// every branch of PAPER.md Alg. 3 bit-identical to the fp32 walk.
// For models with many distinct thresholds per feature (C2: ~1,400 over 90
// features) the in-kernel Eytzinger search costs more than the walk it
// shortens, and its search arrays crowd the tree ring out of shared memory.
// This pre-pass computes the codes once per (row, feature) in a separate
// launch and writes them in exactly the per-warp SMEM tile layout the scorer
// uses, so the scorer's tile fill is a plain 16-B copy and its ring carries
// tree chunks only.
//
// Search: a bucket index followed by a short binary search.
//   b(x) = trunc(min((clamp(x, lo, hi) - lo) * s, B - 1))     (fp32, RN, no FMA)
// is monotone non-decreasing in x for any s > 0, so
//   u_j in a lower bucket than x  =>  u_j < x,   higher  =>  u_j > x,
// and c(x) = start[b(x)] + #{u_j in bucket b(x) : u_j <= x}. start[] is
// computed on the host by applying the same b() to every u_j, so the result is
// exact whatever rounding b() does — the fp32 compares against u_j decide.
// NaN -> 0xFFFF (sorts after every threshold: "go right", as x < t is false).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hb_internal.h"

namespace hb {

namespace {

constexpr int kRcWarps = 8;                 // warps per CTA of the pre-pass
constexpr uint32_t kRcSmemMax = 200 * 1024; // largest per-CTA table budget
constexpr int kRcBatch = 16;                // X loads in flight together per lane
constexpr int kRcRows = 4;                  // 32-row blocks per warp iteration

struct RankCodeParams {
  const float *X;
  int64_t n, ldx;
  const uint4 *feat;      // [n_fc][2] {f, B, S, start off} {lo, hi, s, u off} (offsets in group)
  const uint4 *groups;    // [n_groups][2] {pool byte offset, bytes, word_begin, word_end}
                          //              {first X column, columns spanned, staged row pitch, 0}
  const uint8_t *pool;
  int n_fc, n_words;
  int pair_loads;         // CW 16: word w = features 2w, 2w+1 = one aligned float2 of X
  uint32_t smem_cap;      // groups up to this size are staged in SMEM
  uint32_t *codes;        // [nblocks][n_words][32]
  int64_t nblocks;
  uint32_t stage_off;     // staged kernel: SMEM byte offset of the X staging buffers
};

template <bool LE>
__device__ __forceinline__ uint32_t rank_code(float x, const uint4 m0, const uint4 m1, const uint8_t *tb) {
  // branch-free: NaN clamps to lo (fmaxf), walks bucket 0 (compares false)
  // and is replaced by 0xFFFF at the end
  const float lo = __uint_as_float(m1.x), hi = __uint_as_float(m1.y), s = __uint_as_float(m1.z);
  const float xc = fminf(fmaxf(x, lo), hi);
  float y = __fmul_rn(__fsub_rn(xc, lo), s);
  y = fminf(y, (float)(m0.y - 1u));
  const uint32_t b = __float2uint_rz(y);
  // bucket entry: first threshold index | count << 16 (one load)
  const uint32_t be = reinterpret_cast<const uint32_t *>(tb + m0.w)[b];
  const float *u = reinterpret_cast<const float *>(tb + m1.w);
  uint32_t base = be & 0xFFFFu;
  uint32_t cnt = be >> 16;
#pragma unroll
  for (uint32_t k = 0; k < 16; ++k) {
    if (k >= m0.z) break;                      // S steps (warp-uniform)
    const uint32_t half = cnt >> 1;
    const float v = u[base + half];              // u has one pad slot: in range when cnt == 0
    const bool go = cnt != 0 && (LE ? v < x : v <= x);
    base = go ? base + half + 1u : base;
    cnt = go ? cnt - half - 1u : half;
  }
  return x != x ? 0xFFFFu : base;
}

template <bool LE, int CW>
__global__ void __launch_bounds__(32 * kRcWarps, 4) rank_code_kernel(const RankCodeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint4 g = __ldg(p.groups + 2 * blockIdx.y);
  const uint8_t *tb = p.pool + g.x;
  if (g.y <= p.smem_cap) {
    const uint4 *src = reinterpret_cast<const uint4 *>(tb);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < g.y / 16u; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    tb = smem;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // one warp = kRcRows 32-row blocks, all words of this group: lane = row, so
  // the strided X reads of consecutive features hit the sectors the first one
  // brought into L1, and each word store is one coalesced 128-B line. X loads
  // of kRcRows blocks x NB words are issued before the first search, so the
  // HBM latency is paid once per batch, not once per feature.
  constexpr int PW = CW == 32 ? 1 : 2;                   // features per word
  constexpr int NB = kRcBatch / (kRcRows * PW) > 0 ? kRcBatch / (kRcRows * PW) : 1;   // words per batch
  for (int64_t rb0 = ((int64_t)blockIdx.x * kRcWarps + warp) * kRcRows; rb0 < p.nblocks;
       rb0 += (int64_t)gridDim.x * kRcWarps * kRcRows) {
    // rows past n (and row blocks past the end) read row 0 and are not stored
    const float *xr[kRcRows];
#pragma unroll
    for (int i = 0; i < kRcRows; ++i) {
      const int64_t row = (rb0 + i) * 32 + lane;
      xr[i] = p.X + (row < p.n ? row : 0) * p.ldx;
    }
    for (int w0 = (int)g.z; w0 < (int)g.w; w0 += NB) {
      float xv[kRcRows][NB][PW];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int wc = min(w0 + j, (int)g.w - 1);   // clamped: loads stay unconditional
        if (PW == 2 && p.pair_loads) {
          // word = features 2w, 2w+1 = X columns 2w, 2w+1: one 8-B load
#pragma unroll
          for (int i = 0; i < kRcRows; ++i) {
            const float2 v = __ldg(reinterpret_cast<const float2 *>(xr[i] + 2 * wc));
            xv[i][j][0] = v.x;
            xv[i][j][PW - 1] = v.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < PW; ++q) {
            const uint32_t f = __ldg(reinterpret_cast<const uint32_t *>(p.feat + 2 * min(wc * PW + q, p.n_fc - 1)));
#pragma unroll
            for (int i = 0; i < kRcRows; ++i) xv[i][j][q] = __ldg(xr[i] + f);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int wd = w0 + j;
        if (wd >= (int)g.w) break;
        const int f0 = PW * wd, f1 = PW * wd + 1;
        const uint4 a0 = __ldg(p.feat + 2 * f0), a1 = __ldg(p.feat + 2 * f0 + 1);
        const bool has1 = PW == 2 && f1 < p.n_fc;
        const uint4 b0 = __ldg(p.feat + 2 * (has1 ? f1 : f0)), b1 = __ldg(p.feat + 2 * (has1 ? f1 : f0) + 1);
#pragma unroll
        for (int i = 0; i < kRcRows; ++i) {
          uint32_t word;
          if (CW == 32) {
            word = ((uint32_t)wd << 23) | rank_code<LE>(xv[i][j][0], a0, a1, tb);
          } else {
            const uint32_t c0 = rank_code<LE>(xv[i][j][0], a0, a1, tb);
            const uint32_t c1 = has1 ? rank_code<LE>(xv[i][j][PW - 1], b0, b1, tb) : 0u;
            word = c0 | (c1 << 16);
          }
          if (rb0 + i < p.nblocks) p.codes[((size_t)(rb0 + i) * p.n_words + wd) * 32 + lane] = word;
        }
      }
    }
  }
}

using RcFn = void (*)(const RankCodeParams);

RcFn rc_pick(bool le, int cw) {
  if (cw == 32) return le ? rank_code_kernel<true, 32> : rank_code_kernel<false, 32>;
  return le ? rank_code_kernel<true, 16> : rank_code_kernel<false, 16>;
}

// Staged variant: the X columns a table group needs are copied into per-warp
// SMEM buffers with cp.async (LDGSTS) — lanes walk the [rows x columns] span
// in row-major order, so one warp instruction touches a few consecutive rows
// instead of 32 (the strided lane = row loads above cost one L1 wavefront per
// lane) — kStStages stages deep, so the HBM latency overlaps the searches of
// earlier stages without holding X in registers. A stage is RB consecutive
// 32-row blocks; the search then reads x from SMEM (row pitch odd: lane = row
// is conflict free) with RB independent searches per feature in flight.
constexpr int kStStages = 3;

__device__ __forceinline__ void cp_async4(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <bool LE, int CW, int RB>
__global__ void __launch_bounds__(32 * kRcWarps, 2) rank_code_staged_kernel(const RankCodeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint4 g = __ldg(p.groups + 2 * blockIdx.y);
  const uint4 gs = __ldg(p.groups + 2 * blockIdx.y + 1);   // {col_lo, ncols, pitch, 0}
  const uint8_t *tb = p.pool + g.x;
  if (g.y <= p.smem_cap) {
    const uint4 *src = reinterpret_cast<const uint4 *>(tb);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < g.y / 16u; i += blockDim.x) dst[i] = __ldg(src + i);
    tb = smem;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncols = (int)gs.y, pitch = (int)gs.z;
  const uint32_t stage_words = (uint32_t)(RB * 32 * pitch);
  uint32_t *xs = reinterpret_cast<uint32_t *>(smem + p.stage_off) + (size_t)warp * kStStages * stage_words;
  const uint32_t xs_s = (uint32_t)__cvta_generic_to_shared(xs);
  const int drow = 32 / ncols, dcol = 32 - drow * ncols;
  const int row_l = lane / ncols, col_l = lane - row_l * ncols;
  const float *xg = p.X + gs.x;
  const int64_t nunits = (p.nblocks + RB - 1) / RB;
  const int64_t ustep = (int64_t)gridDim.x * kRcWarps;
  // copy unit u's rows (clamped to the last row: the tail block computes
  // valid, unused codes) into stage st
  auto issue = [&](int64_t u, int st) {
    if (u < nunits) {
      const int64_t r0 = u * RB * 32;
      const uint32_t d0 = xs_s + (uint32_t)st * stage_words * 4u;
      int row = row_l, col = col_l;
      for (int it = 0; it < RB * ncols; ++it) {
        const int64_t gr = min(r0 + row, p.n - 1);
        cp_async4(d0 + (uint32_t)(row * pitch + col) * 4u, xg + gr * p.ldx + col);
        col += dcol;
        row += drow;
        if (col >= ncols) {
          col -= ncols;
          ++row;
        }
      }
    }
    cp_async_commit();   // empty groups keep the wait count uniform
  };
  constexpr int PW = CW == 32 ? 1 : 2;
  int64_t u = (int64_t)blockIdx.x * kRcWarps + warp;
#pragma unroll
  for (int s = 0; s < kStStages - 1; ++s) issue(u + s * ustep, s);
  int st = 0;
  for (; u < nunits; u += ustep) {
    issue(u + (kStStages - 1) * ustep, st == 0 ? kStStages - 1 : st - 1);
    cp_async_wait<kStStages - 1>();
    __syncwarp();
    const uint32_t *xr = xs + st * stage_words + lane * pitch;
    for (int wd = (int)g.z; wd < (int)g.w; ++wd) {
      const int f0 = PW * wd, f1 = PW * wd + 1;
      const uint4 a0 = __ldg(p.feat + 2 * f0), a1 = __ldg(p.feat + 2 * f0 + 1);
      const bool has1 = PW == 2 && f1 < p.n_fc;
      const uint4 b0 = __ldg(p.feat + 2 * (has1 ? f1 : f0)), b1 = __ldg(p.feat + 2 * (has1 ? f1 : f0) + 1);
      const int c0 = (int)(a0.x - gs.x), c1 = (int)(b0.x - gs.x);
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const float x0 = __uint_as_float(xr[i * 32 * pitch + c0]);
        uint32_t word;
        if (CW == 32) {
          word = ((uint32_t)wd << 23) | rank_code<LE>(x0, a0, a1, tb);
        } else {
          const float x1 = __uint_as_float(xr[i * 32 * pitch + c1]);
          const uint32_t k0 = rank_code<LE>(x0, a0, a1, tb);
          const uint32_t k1 = has1 ? rank_code<LE>(x1, b0, b1, tb) : 0u;
          word = k0 | (k1 << 16);
        }
        const int64_t blk = u * RB + i;
        if (blk < p.nblocks) p.codes[((size_t)blk * p.n_words + wd) * 32 + lane] = word;
      }
    }
    __syncwarp();        // every lane is done with stage st before it is refilled
    st = st == kStStages - 1 ? 0 : st + 1;
  }
  cp_async_wait<0>();
}

template <bool LE, int CW>
RcFn staged_pick_rb(int rb) {
  if (rb >= 4) return rank_code_staged_kernel<LE, CW, 4>;
  if (rb == 2) return rank_code_staged_kernel<LE, CW, 2>;
  return rank_code_staged_kernel<LE, CW, 1>;
}

RcFn staged_pick(bool le, int cw, int rb) {
  if (cw == 32) return le ? staged_pick_rb<true, 32>(rb) : staged_pick_rb<false, 32>(rb);
  return le ? staged_pick_rb<true, 16>(rb) : staged_pick_rb<false, 16>(rb);
}

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
                             int cw, RankBuckets *out) {
  // per-CTA table budget: 48 KB -> 4 CTAs (32 warps) per SM (HB_RC_SMEM_KB overrides)
  const char *ev = std::getenv("HB_RC_SMEM_KB");
  const size_t cap = std::min<size_t>(kRcSmemMax, (ev && *ev ? (size_t)std::atoi(ev) : 48) * 1024);
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
    uint32_t B = 1;
    while (2 * B < m && B < 16384u) B <<= 1;     // <= 2 thresholds per bucket on average
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
    const float pad = INFINITY;
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
    if (gbytes > cap) R.any_global = true;
    R.max_group_bytes = std::max(R.max_group_bytes, gbytes <= cap ? gbytes : (size_t)0);
    goff += gbytes;
    gbytes = 0;
    wbeg = wend;
    R.n_groups++;
  };
  for (int wd = 0; wd < n_words; ++wd) {
    size_t wb = 0;
    for (int q = 0; q < per_word && wd * per_word + q < n_fc; ++q) wb += (tabs[wd * per_word + q].size() + 15) & ~size_t(15);
    if (gbytes > 0 && gbytes + wb > cap) close(wd);
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

int sm_count(int device);

hb_status launch_rank_codes(const Model &m, const RunArgs &a, uint32_t *codes, int64_t nblocks) {
  if (m.rb_ngroups == 0 || nblocks == 0) return HB_OK;   // no split uses any feature: no codes
  RankCodeParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  const uint8_t *aux = static_cast<const uint8_t *>(m.d_rb);
  p.feat = reinterpret_cast<const uint4 *>(aux);
  p.groups = reinterpret_cast<const uint4 *>(aux + m.rb_groups_off);
  p.pool = aux + m.rb_pool_off;
  p.n_fc = m.rank_nfc;
  p.n_words = m.rank_nwords;
  p.codes = codes;
  p.nblocks = nblocks;
  p.smem_cap = (uint32_t)m.rb_smem_cap;
  p.pair_loads = m.rank_cw == 16 && m.rank_nfc == m.n_features && m.n_features % 2 == 0 &&
                 a.ldx % 2 == 0 && (reinterpret_cast<uintptr_t>(a.X) & 7) == 0;
  const size_t tbytes = (m.rb_smem + 15) & ~size_t(15);
  p.stage_off = (uint32_t)tbytes;
  // staged kernel (cp.async X staging) unless the groups span too many
  // columns for the SMEM staging budget (HB_RC_STAGED=0/1 forces; HB_RC_RB
  // picks the 32-row blocks per stage)
  const char *ev = std::getenv("HB_RC_STAGED");
  const char *erb = std::getenv("HB_RC_RB");
  const size_t pitch = (size_t)(m.rb_max_span | 1u);
  const size_t stage_budget = 64 * 1024;
  int rb = 4;
  while (rb > 1 && (size_t)kRcWarps * kStStages * rb * 32 * pitch * 4 > stage_budget) rb >>= 1;
  if (erb && *erb) rb = std::atoi(erb) >= 4 ? 4 : (std::atoi(erb) >= 2 ? 2 : 1);
  const size_t staged_smem = tbytes + (size_t)kRcWarps * kStStages * rb * 32 * pitch * 4;
  // AUTO: staged when some table group is searched from global memory (its
  // table exceeds the SMEM cap): those searches are L1-latency bound and the
  // cp.async pipeline keeps X off the dependency chain (C4: 49.2 -> 46.9 ms per
  // step). SMEM-resident tables keep the direct kernel, which runs twice the
  // CTAs per SM (C2 pre-pass 0.49 ms direct vs 0.94 ms staged).
  const bool fits = staged_smem <= (size_t)kRcSmemMax + stage_budget && m.rb_max_span > 0;
  bool staged = fits && m.rb_global;
  if (ev && *ev && std::atoi(ev) >= 0) staged = fits && std::atoi(ev) != 0;   // -1: AUTO
  RcFn fn = staged ? staged_pick(m.cmp == HB_CMP_LE, m.rank_cw, rb) : rc_pick(m.cmp == HB_CMP_LE, m.rank_cw);
  const int smem = (int)(staged ? staged_smem : m.rb_smem);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(rank codes)");
  // as many CTAs as fit per SM (by SMEM, at most 4), spread over the feature
  // groups (blockIdx.y)
  const size_t per_cta = staged ? staged_smem : std::max<size_t>(m.rb_smem_cap, 1);
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(4, (220 * 1024) / per_cta));
  const int64_t want = std::max<int64_t>(1, ((int64_t)per_sm * sm_count(m.device) + m.rb_ngroups - 1) / m.rb_ngroups);
  const int64_t rows_per_cta = (int64_t)kRcWarps * (staged ? rb : kRcRows);
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(want, (nblocks + rows_per_cta - 1) / rows_per_cta));
  fn<<<dim3(gx, m.rb_ngroups), 32 * kRcWarps, smem, a.stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "rank_code_kernel launch");
  return HB_OK;
}

}  // namespace hb
