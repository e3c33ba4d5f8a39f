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
//
// Two per-group kernels, one CTA = one table group in SMEM:
//   rank_code_kernel         direct strided X loads (lane = row), for groups of
//                            several features (C2);
//   rank_code_staged_kernel  X columns staged with cp.async, for narrow groups
//                            (C3, C4) or tables searched from global memory.
// Both run the searches of a batch in lockstep (rank_codes_lockstep) and use
// a group-major grid with contiguous row slices. (A cluster variant holding
// all tables in one cluster's DSMEM was measured slower and removed, DESIGN.md
// §4.6.)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hb_device.cuh"
#include "hb_internal.h"
#include "hb_layouts.h"

namespace hb {

namespace {

constexpr int kRcWarps = 8;                 // warps per CTA of the pre-pass
constexpr int kRcBatch = 16;                // X loads in flight together per lane
constexpr int kRcRows = 4;                  // 32-row blocks per warp iteration (HB_RC_ROWS=8: eight)

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
  int gorder;             // 1 = blockIdx.x is the table group and each CTA owns a contiguous
                          // row range (the groups of the same rows run together); 0 = strided
  int rw;                 // direct kernel, pair_loads: lanes = (row, word) (rank_code_body_rw)
};

// Table reads: SMEM-resident groups are plain shared-memory loads (LDS), the
// others the read-only global path.
template <bool SM>
__device__ __forceinline__ uint32_t tab_u32(const uint8_t *tb, uint32_t off) {
  // plain loads (no asm): the compiler may schedule the independent loads of
  // a lockstep step together; tb points into shared memory when SM
  if (SM) return *reinterpret_cast<const uint32_t *>(tb + off);
  return __ldg(reinterpret_cast<const uint32_t *>(tb + off));
}

// S power-of-two window steps (2^(S-1) slots first) over NC chains, each
// step's NC loads back to back (see rank_codes_lockstep)
template <bool LE, bool SM, int NC, int S>
__device__ __forceinline__ void window_steps(const uint8_t *tb, uint32_t (&pos)[NC], const float (&x)[NC]) {
  if constexpr (S > 0) {
    constexpr uint32_t k = S - 1;
    float v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = __uint_as_float(tab_u32<SM>(tb, pos[c] + 4u * ((1u << k) - 1u)));
#pragma unroll
    for (int c = 0; c < NC; ++c) pos[c] += (LE ? v[c] < x[c] : v[c] <= x[c]) ? (4u << k) : 0u;
    window_steps<LE, SM, NC, S - 1>(tb, pos, x);
  }
}

// NC rank codes in lockstep: the bucket step of every search first, then a
// fixed window of 2^smax - 1 slots from each bucket's first threshold.
// Thresholds of later buckets are > x and every table ends with 2^S_g - 1
// NaN pads (build_rank_buckets; S_g >= smax for any set of one group's
// features), so "u <= x" (LE: u < x) holds on a prefix of the window and the
// code is the bucket start + the prefix length, found by smax power-of-two
// steps of one load, one compare and one select — all NC loads of a step
// back to back (the searches are independent: their latencies overlap).
template <bool LE, bool SM, int NC>
__device__ __forceinline__ void rank_codes_lockstep(const float (&x)[NC], const uint4 *m0, const uint4 *m1,
                                                    const int (&mi)[NC], uint32_t smax, const uint8_t *tb,
                                                    uint32_t (&code)[NC]) {
  uint32_t pos[NC], uo[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint4 a = m0[mi[c]], b = m1[mi[c]];
    const float lo = __uint_as_float(b.x), hi = __uint_as_float(b.y), sc = __uint_as_float(b.z);
    const float xc = fminf(fmaxf(x[c], lo), hi);            // NaN -> lo: walks bucket 0, replaced below
    float y = __fmul_rn(__fsub_rn(xc, lo), sc);
    y = fminf(y, (float)(a.y - 1u));
    const uint32_t bk = __float2uint_rz(y);
    const uint32_t be = tab_u32<SM>(tb, a.w + 4u * bk);   // first index | count << 16
    uo[c] = b.w;
    pos[c] = b.w + 4u * (be & 0xFFFFu);
  }
  switch (smax) {
    case 0: break;
    case 1: window_steps<LE, SM, NC, 1>(tb, pos, x); break;
    case 2: window_steps<LE, SM, NC, 2>(tb, pos, x); break;
    case 3: window_steps<LE, SM, NC, 3>(tb, pos, x); break;
    case 4: window_steps<LE, SM, NC, 4>(tb, pos, x); break;
    case 5: window_steps<LE, SM, NC, 5>(tb, pos, x); break;
    default:
      for (uint32_t sb = 4u << (smax - 1u); sb >= 4u; sb >>= 1) {
        float v[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = __uint_as_float(tab_u32<SM>(tb, pos[c] + sb - 4u));
#pragma unroll
        for (int c = 0; c < NC; ++c) pos[c] += (LE ? v[c] < x[c] : v[c] <= x[c]) ? sb : 0u;
      }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) code[c] = x[c] != x[c] ? 0xFFFFu : (pos[c] - uo[c]) >> 2;
}

template <bool LE, int CW, bool SM, int ROWS>
__device__ __forceinline__ void rank_code_body(const RankCodeParams &p, const uint4 g, const uint8_t *tb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // one warp = ROWS 32-row blocks, all words of this group: lane = row, so
  // the strided X reads of consecutive features hit the sectors the first one
  // brought into L1, and each word store is one coalesced 128-B line. X loads
  // of ROWS blocks x NB words are issued before the first search, so the
  // HBM latency is paid once per batch, not once per feature; the searches
  // then run two features x ROWS rows in lockstep.
  constexpr int PW = CW == 32 ? 1 : 2;                   // features per word
  constexpr int NB = kRcBatch / (ROWS * PW) > 0 ? kRcBatch / (ROWS * PW) : 1;   // words per batch
  constexpr int NS = NB * PW;                            // feature slots per batch (even)
  static_assert(NS % 2 == 0, "feature slots go in pairs");
  // batches of ROWS row blocks: strided over the grid (gorder 0) or one
  // contiguous slice per CTA (gorder 1, group-major grid: see the staged kernel)
  const int64_t nbat = (p.nblocks + ROWS - 1) / ROWS;
  const int64_t nparts = p.gorder ? gridDim.y : gridDim.x;
  const int64_t part = p.gorder ? blockIdx.y : blockIdx.x;
  const int64_t bend = p.gorder ? (part + 1) * nbat / nparts : nbat;
  const int64_t bstep = p.gorder ? (int64_t)kRcWarps : nparts * kRcWarps;
  for (int64_t bt = (p.gorder ? part * nbat / nparts : part * kRcWarps) + warp; bt < bend; bt += bstep) {
    const int64_t rb0 = bt * ROWS;
    // rows past n (and row blocks past the end) read row 0 and are not stored
    const float *xr[ROWS];
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const int64_t row = (rb0 + i) * 32 + lane;
      xr[i] = p.X + (row < p.n ? row : 0) * p.ldx;
    }
    for (int w0 = (int)g.z; w0 < (int)g.w; w0 += NB) {
      // feature slot s = j * PW + q: word w0 + j, compact feature PW * (w0 + j) + q
      // (clamped to a valid feature: loads stay unconditional)
      int cf[NS];
      bool ok[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int wd = w0 + s / PW, c = PW * wd + s % PW;
        ok[s] = wd < (int)g.w && c < p.n_fc;
        cf[s] = ok[s] ? c : PW * (int)g.z;
      }
      float xv[NS][ROWS];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (PW == 2 && p.pair_loads) {
          // word = features 2w, 2w+1 = X columns 2w, 2w+1: one 8-B load
          const int wc = min(w0 + j, (int)g.w - 1);
#pragma unroll
          for (int i = 0; i < ROWS; ++i) {
            const float2 v = __ldg(reinterpret_cast<const float2 *>(xr[i] + 2 * wc));
            xv[j * PW][i] = v.x;
            xv[j * PW + PW - 1][i] = v.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < PW; ++q) {
            const uint32_t f = __ldg(reinterpret_cast<const uint32_t *>(p.feat + 2 * cf[j * PW + q]));
#pragma unroll
            for (int i = 0; i < ROWS; ++i) xv[j * PW + q][i] = __ldg(xr[i] + f);
          }
        }
      }
#pragma unroll
      for (int sp = 0; sp < NS; sp += 2) {
        uint4 M0[2], M1[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          M0[e] = __ldg(p.feat + 2 * cf[sp + e]);
          M1[e] = __ldg(p.feat + 2 * cf[sp + e] + 1);
        }
        float x8[2 * ROWS];
        int mi[2 * ROWS];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int i = 0; i < ROWS; ++i) {
            x8[e * ROWS + i] = xv[sp + e][i];
            mi[e * ROWS + i] = e;
          }
        const uint32_t smax = max(ok[sp] ? M0[0].z : 0u, ok[sp + 1] ? M0[1].z : 0u);
        uint32_t code[2 * ROWS];
        rank_codes_lockstep<LE, SM, 2 * ROWS>(x8, M0, M1, mi, smax, tb, code);
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
          if (rb0 + i >= p.nblocks) continue;
          if (CW == 32) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int wd = w0 + sp + e;
              if (ok[sp + e])
                p.codes[((size_t)(rb0 + i) * p.n_words + wd) * 32 + lane] = ((uint32_t)wd << 23) | code[e * ROWS + i];
            }
          } else {
            const int wd = w0 + sp / 2;
            if (ok[sp])
              p.codes[((size_t)(rb0 + i) * p.n_words + wd) * 32 + lane] =
                  code[i] | ((ok[sp + 1] ? code[ROWS + i] : 0u) << 16);
          }
        }
      }
    }
  }
}

// 16-bit cells with every word one aligned float2 of X (pair_loads, C2): lanes
// = (row, word) instead of lane = row, so a warp's X load reads WQ adjacent
// words (8 WQ bytes) of 32 / WQ rows — a few sectors per row — instead of
// one float2 from each of 32 rows (32 sectors per load, the L1 cost that
// bound the row-per-lane body: 48M sectors + 41M SMEM wavefronts per C2
// call). WQ = min(words in the group, 4) words of 32 / WQ rows per load (a
// 3-word group: 10 rows, lanes 30-31 idle). Each lane runs 4 rows x its
// word's 2 features = 8 searches in lockstep; the window-step count is the
// warp's maximum.
template <bool LE, bool SM>
__device__ __forceinline__ void rank_code_body_rw(const RankCodeParams &p, const uint4 g, const uint8_t *tb) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int ROWS = kRcRows;                       // 32-row blocks per warp iteration
  const int nwg = (int)(g.w - g.z);
  const int WQ = min(nwg, 4);                         // words per load
  const int RI = 32 / WQ;                             // rows per load (lanes >= RI WQ idle)
  const int wo = lane % WQ, ro = lane / WQ;
  const bool lact = lane < RI * WQ;
  const int nk = (ROWS * 32 + RI - 1) / RI;           // loads per lane and batch
  const int64_t nbat = (p.nblocks + ROWS - 1) / ROWS;
  const int64_t nparts = p.gorder ? gridDim.y : gridDim.x;
  const int64_t part = p.gorder ? blockIdx.y : blockIdx.x;
  const int64_t bend = p.gorder ? (part + 1) * nbat / nparts : nbat;
  const int64_t bstep = p.gorder ? (int64_t)kRcWarps : nparts * kRcWarps;
  for (int w0 = (int)g.z; w0 < (int)g.w; w0 += WQ) {
    const int wd = w0 + wo;
    const bool wok = wd < (int)g.w;
    const int wc = wok ? wd : w0;                     // clamped: loads stay unconditional
    uint4 M0[2], M1[2];
    uint32_t sl = 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = min(2 * wc + e, p.n_fc - 1);
      M0[e] = __ldg(p.feat + 2 * c);
      M1[e] = __ldg(p.feat + 2 * c + 1);
      sl = max(sl, (wok && 2 * wc + e < p.n_fc) ? M0[e].z : 0u);
    }
    const uint32_t smax = __reduce_max_sync(0xFFFFFFFFu, sl);
    const int mi8[2 * 4] = {0, 0, 0, 0, 1, 1, 1, 1};
    for (int64_t bt = (p.gorder ? part * nbat / nparts : part * kRcWarps) + warp; bt < bend; bt += bstep) {
      const int64_t r0 = bt * ROWS * 32;
      // this lane's rows of the batch: r0 + ro + RI k, k < 4 * 32 / RI, four at a time
      // X of the next four rows is loaded before the current four are
      // searched (register double buffer: one X latency per batch, not per 4 rows)
      float2 nx[4];
      auto load4 = [&](int k0, float2 (&v)[4]) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t r = r0 + ro + (int64_t)RI * (k0 + i);
          const int64_t rr = r < p.n ? r : 0;
          v[i] = __ldg(reinterpret_cast<const float2 *>(p.X + rr * p.ldx + 2 * wc));
        }
      };
      load4(0, nx);
      for (int k0 = 0; k0 < nk; k0 += 4) {
        float x8[8];
        int64_t rw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          rw[i] = r0 + ro + (int64_t)RI * (k0 + i);
          x8[i] = nx[i].x;
          x8[4 + i] = nx[i].y;
        }
        if (k0 + 4 < nk) load4(k0 + 4, nx);
        uint32_t code[8];
        rank_codes_lockstep<LE, SM, 8>(x8, M0, M1, mi8, smax, tb, code);
        if (wok && lact) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t blk = rw[i] >> 5;
            HB_DCHECK(wd < p.n_words && 2 * wd < p.n_fc);
            if (rw[i] < p.nblocks * 32 && rw[i] < r0 + ROWS * 32)
              p.codes[((size_t)blk * p.n_words + wd) * 32 + (rw[i] & 31)] =
                  code[i] | ((2 * wd + 1 < p.n_fc ? code[4 + i] : 0u) << 16);
          }
        }
      }
    }
  }
}

template <bool LE, int CW, int ROWS>
__global__ void __launch_bounds__(32 * kRcWarps, ROWS == 4 ? 4 : 3) rank_code_kernel(const RankCodeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint4 g = __ldg(p.groups + 2 * (p.gorder ? blockIdx.x : blockIdx.y));
  const uint8_t *tb = p.pool + g.x;
  if (g.y <= p.smem_cap) {
    const uint4 *src = reinterpret_cast<const uint4 *>(tb);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < g.y / 16u; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    if (CW == 16 && ROWS == kRcRows && p.pair_loads && p.rw) rank_code_body_rw<LE, true>(p, g, smem);
    else rank_code_body<LE, CW, true, ROWS>(p, g, smem);
  } else {
    if (CW == 16 && ROWS == kRcRows && p.pair_loads && p.rw) rank_code_body_rw<LE, false>(p, g, tb);
    else rank_code_body<LE, CW, false, ROWS>(p, g, tb);
  }
}

using RcFn = void (*)(const RankCodeParams);

template <int ROWS>
RcFn rc_pick_rows(bool le, int cw) {
  if (cw == 32) return le ? rank_code_kernel<true, 32, ROWS> : rank_code_kernel<false, 32, ROWS>;
  return le ? rank_code_kernel<true, 16, ROWS> : rank_code_kernel<false, 16, ROWS>;
}

RcFn rc_pick(bool le, int cw, int rows) { return rows == 8 ? rc_pick_rows<8>(le, cw) : rc_pick_rows<4>(le, cw); }

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

template <bool LE, int CW, int RB, bool SM, bool ONE>
__device__ __forceinline__ void rank_code_staged_body(const RankCodeParams &p, const uint4 g, const uint4 gs,
                                                      const uint8_t *tb, uint8_t *smem) {
  // ONE (32-bit cells only): one feature per lockstep set, RB row blocks of
  // it — for single-feature table groups, where a feature pair would leave
  // half the chains idle
  constexpr int NSL = (CW == 32 && ONE) ? 1 : 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncols = (int)gs.y, pitch = (int)gs.z;
  const uint32_t stage_words = (uint32_t)(RB * 32 * pitch);
  uint32_t *xs = reinterpret_cast<uint32_t *>(smem + p.stage_off) + (size_t)warp * kStStages * stage_words;
  const uint32_t xs_s = (uint32_t)__cvta_generic_to_shared(xs);
  const int drow = 32 / ncols, dcol = 32 - drow * ncols;
  const int row_l = lane / ncols, col_l = lane - row_l * ncols;
  const float *xg = p.X + gs.x;
  const int64_t nunits = (p.nblocks + RB - 1) / RB;
  // unit range of this CTA: strided over the grid (gorder 0) or one
  // contiguous slice (gorder 1: the CTAs of all groups for the same rows are
  // launched together and read the same X sectors at about the same time)
  const int64_t nparts = p.gorder ? gridDim.y : gridDim.x;
  const int64_t part = p.gorder ? blockIdx.y : blockIdx.x;
  const int64_t uend = p.gorder ? (part + 1) * nunits / nparts : nunits;
  const int64_t ustep = p.gorder ? (int64_t)kRcWarps : nparts * kRcWarps;
  const int64_t ubeg = p.gorder ? part * nunits / nparts : part * kRcWarps;
  // copy unit u's rows (clamped to the last row: the tail block computes
  // valid, unused codes) into stage st
  auto issue = [&](int64_t u, int st) {
    if (u < uend) {
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
  constexpr int WS = NSL / PW;        // words per lockstep set
  int64_t u = ubeg + warp;
#pragma unroll
  for (int s = 0; s < kStStages - 1; ++s) issue(u + s * ustep, s);
  int st = 0;
  for (; u < uend; u += ustep) {
    issue(u + (kStStages - 1) * ustep, st == 0 ? kStStages - 1 : st - 1);
    cp_async_wait<kStStages - 1>();
    __syncwarp();
    const uint32_t *xr = xs + st * stage_words + lane * pitch;
    // NSL features x RB rows per lockstep search
    for (int wd = (int)g.z; wd < (int)g.w; wd += WS) {
      uint4 M0[NSL], M1[NSL];
      bool ok[2] = {true, false};
      float x8[NSL * RB];
      int mi[NSL * RB];
#pragma unroll
      for (int e = 0; e < NSL; ++e) {
        const int c = PW * wd + e;
        ok[e] = (PW == 2 ? wd : wd + e) < (int)g.w && c < p.n_fc;
        const int cc = ok[e] ? c : PW * wd;
        M0[e] = __ldg(p.feat + 2 * cc);
        M1[e] = __ldg(p.feat + 2 * cc + 1);
        const int col = (int)(M0[e].x - gs.x);
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          x8[e * RB + i] = __uint_as_float(xr[i * 32 * pitch + col]);
          mi[e * RB + i] = e;
        }
      }
      const uint32_t smax = NSL == 1 ? M0[0].z : max(M0[0].z, ok[1] ? M0[NSL - 1].z : 0u);
      uint32_t code[NSL * RB];
      rank_codes_lockstep<LE, SM, NSL * RB>(x8, M0, M1, mi, smax, tb, code);
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int64_t blk = u * RB + i;
        if (blk >= p.nblocks) continue;
        uint32_t *dst = p.codes + ((size_t)blk * p.n_words + wd) * 32 + lane;
        if (CW == 32) {
          dst[0] = ((uint32_t)wd << 23) | code[i];
          if (NSL == 2 && ok[1]) dst[32] = ((uint32_t)(wd + 1) << 23) | code[(NSL - 1) * RB + i];
        } else {
          dst[0] = code[i] | ((ok[1] ? code[(NSL - 1) * RB + i] : 0u) << 16);
        }
      }
    }
    __syncwarp();        // every lane is done with stage st before it is refilled
    st = st == kStStages - 1 ? 0 : st + 1;
  }
  cp_async_wait<0>();
}

template <bool LE, int CW, int RB, bool ONE>
__global__ void __launch_bounds__(32 * kRcWarps, 2) rank_code_staged_kernel(const RankCodeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int gi = p.gorder ? blockIdx.x : blockIdx.y;
  const uint4 g = __ldg(p.groups + 2 * gi);
  const uint4 gs = __ldg(p.groups + 2 * gi + 1);   // {col_lo, ncols, pitch, 0}
  const uint8_t *tb = p.pool + g.x;
  if (g.y <= p.smem_cap) {
    const uint4 *src = reinterpret_cast<const uint4 *>(tb);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < g.y / 16u; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
    rank_code_staged_body<LE, CW, RB, true, ONE>(p, g, gs, smem, smem);
  } else {
    rank_code_staged_body<LE, CW, RB, false, ONE>(p, g, gs, tb, smem);
  }
}

template <bool LE, int CW, bool ONE>
RcFn staged_pick_rb(int rb) {
  if (rb >= 4) return rank_code_staged_kernel<LE, CW, 4, ONE>;
  if (rb == 2) return rank_code_staged_kernel<LE, CW, 2, ONE>;
  return rank_code_staged_kernel<LE, CW, 1, ONE>;
}

RcFn staged_pick(bool le, int cw, int rb, bool one) {
  if (cw == 32) {
    if (one) return le ? staged_pick_rb<true, 32, true>(rb) : staged_pick_rb<false, 32, true>(rb);
    return le ? staged_pick_rb<true, 32, false>(rb) : staged_pick_rb<false, 32, false>(rb);
  }
  return le ? staged_pick_rb<true, 16, false>(rb) : staged_pick_rb<false, 16, false>(rb);
}

}  // namespace

// fixed-window search helpers over 32-bit shared addresses (column and TMA
// kernels; rank_codes_lockstep explains the window)
template <int OFF>
__device__ __forceinline__ float lds_f32_off(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(a), "n"(OFF));
  return v;
}

// S power-of-two steps (2^(S-1) slots first) over every chain, each step's
// loads back to back, the slot offsets immediates
template <bool LE, int NQ, int U, int S>
__device__ __forceinline__ void window_search(uint32_t (&pos)[NQ][U], const float (&x)[NQ][U]) {
  if constexpr (S > 0) {
    constexpr int k = S - 1;
    float v[NQ][U];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int i = 0; i < U; ++i) v[q][i] = lds_f32_off<4 * ((1 << k) - 1)>(pos[q][i]);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int i = 0; i < U; ++i) pos[q][i] += (LE ? v[q][i] < x[q][i] : v[q][i] <= x[q][i]) ? (4u << k) : 0u;
    window_search<LE, NQ, U, S - 1>(pos, x);
  }
}

// Single-feature table groups with 32-bit cells (C3, C4: one ~34-40 KB table
// per feature, one feature per CTA): a lean column kernel. The CTA owns one
// feature for a contiguous slice of 32-row blocks (group-major grid: the CTAs
// of all features for the same rows run together and share X's L2 sectors);
// each warp takes U = 4 blocks at a time, lane = row. The U column values are
// loaded straight into registers with 32-bit per-unit offsets (the next
// unit's loads are issued before this unit's searches, so one X latency hides
// behind a unit of work), the U searches run in lockstep over the SMEM table
// with 32-bit shared addresses, and each code word is one coalesced 128-B
// store. Same arithmetic as rank_codes_lockstep (exact, R28); what it removes
// is the generic staging loop's 64-bit index math (242 instructions per lane
// and 2 codes in the staged kernel, ncu round 2).
constexpr int kOneU = 4;

template <bool LE, int NWARP, int CW>
__global__ void __launch_bounds__(32 * NWARP, NWARP == 8 ? 4 : 2) rank_code_one_kernel(const RankCodeParams p) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int PW = CW == 32 ? 1 : 2;              // features per code word
  const int gi = blockIdx.x;                        // table group = one code word
  const uint4 g = __ldg(p.groups + 2 * gi);
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(p.pool + g.x);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < g.y / 16u; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const int wd = (int)g.z;                          // the word of this group
  const uint32_t tab = dev::smem_u32(smem);
  // per feature of the word: column, bucket map, search depth, table bases
  const float *xcol[PW];
  float lo[PW], hi[PW], sc[PW], bmax[PW];
  uint32_t sbase[PW], ubase[PW];
  bool okf[PW];
  uint32_t smax = 0;
#pragma unroll
  for (int q = 0; q < PW; ++q) {
    const int c = PW * wd + q;
    okf[q] = c < p.n_fc;
    const int cc = okf[q] ? c : PW * wd;
    const uint4 m0 = __ldg(p.feat + 2 * cc), m1 = __ldg(p.feat + 2 * cc + 1);
    xcol[q] = p.X + m0.x;
    lo[q] = __uint_as_float(m1.x);
    hi[q] = __uint_as_float(m1.y);
    sc[q] = __uint_as_float(m1.z);
    bmax[q] = (float)(m0.y - 1u);
    sbase[q] = tab + m0.w;
    ubase[q] = tab + m1.w;
    if (okf[q]) smax = max(smax, m0.z);
  }
  const uint32_t cellhi = CW == 32 ? (uint32_t)wd << 23 : 0u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's contiguous slice of units (U blocks each)
  const int64_t nunits = (p.nblocks + kOneU - 1) / kOneU;
  const int64_t ubeg = blockIdx.y * nunits / gridDim.y, uend = (blockIdx.y + 1) * nunits / gridDim.y;
  const int64_t rstride = 32 * p.ldx;               // one row block, in floats
  auto load = [&](int64_t u, float (&x)[PW][kOneU]) {
    const int64_t row0 = u * (kOneU * 32) + lane;
#pragma unroll
    for (int q = 0; q < PW; ++q) {
      const float *ptr = xcol[q] + row0 * p.ldx;
      if (row0 + (kOneU - 1) * 32 < p.n) {
#pragma unroll
        for (int i = 0; i < kOneU; ++i) x[q][i] = __ldg(ptr + i * rstride);
      } else {                                      // last unit: rows past n read row n - 1
#pragma unroll
        for (int i = 0; i < kOneU; ++i) {
          const int64_t r = min(row0 + i * 32, p.n - 1);
          x[q][i] = __ldg(xcol[q] + r * p.ldx);
        }
      }
    }
  };
  float xn[PW][kOneU];
  int64_t u = ubeg + warp;
  if (u < uend) load(u, xn);
  for (; u < uend; u += NWARP) {
    float x[PW][kOneU];
#pragma unroll
    for (int q = 0; q < PW; ++q)
#pragma unroll
      for (int i = 0; i < kOneU; ++i) x[q][i] = xn[q][i];
    if (u + NWARP < uend) load(u + NWARP, xn);   // next unit's loads in flight
    // bucket, then the fixed window (rank_codes_lockstep)
    uint32_t pos[PW][kOneU];
#pragma unroll
    for (int q = 0; q < PW; ++q)
#pragma unroll
      for (int i = 0; i < kOneU; ++i) {
        const float xc = fminf(fmaxf(x[q][i], lo[q]), hi[q]);      // NaN -> lo; replaced below
        const float y = fminf(__fmul_rn(__fsub_rn(xc, lo[q]), sc[q]), bmax[q]);
        const uint32_t be = dev::lds_u32(sbase[q] + 4u * __float2uint_rz(y));
        pos[q][i] = ubase[q] + 4u * (be & 0xFFFFu);
      }
    switch (smax) {
      case 0: break;
      case 1: window_search<LE, PW, kOneU, 1>(pos, x); break;
      case 2: window_search<LE, PW, kOneU, 2>(pos, x); break;
      case 3: window_search<LE, PW, kOneU, 3>(pos, x); break;
      case 4: window_search<LE, PW, kOneU, 4>(pos, x); break;
      case 5: window_search<LE, PW, kOneU, 5>(pos, x); break;
      default:
        for (uint32_t sb = 4u << (smax - 1u); sb >= 4u; sb >>= 1) {
#pragma unroll
          for (int q = 0; q < PW; ++q)
#pragma unroll
            for (int i = 0; i < kOneU; ++i) {
              const float v = dev::lds_f32(pos[q][i] + sb - 4u);
              pos[q][i] += (LE ? v < x[q][i] : v <= x[q][i]) ? sb : 0u;
            }
        }
    }
    uint32_t base[PW][kOneU];
#pragma unroll
    for (int q = 0; q < PW; ++q)
#pragma unroll
      for (int i = 0; i < kOneU; ++i) base[q][i] = (pos[q][i] - ubase[q]) >> 2;
    uint32_t *dst = p.codes + ((size_t)u * kOneU * p.n_words + (size_t)wd) * 32 + lane;
#pragma unroll
    for (int i = 0; i < kOneU; ++i) {
      if (u * kOneU + i < p.nblocks) {
        const uint32_t c0 = x[0][i] != x[0][i] ? 0xFFFFu : base[0][i];
        uint32_t w = cellhi | c0;
        if (PW == 2) {
          const uint32_t c1 = x[PW - 1][i] != x[PW - 1][i] ? 0xFFFFu : base[PW - 1][i];
          w |= (okf[PW - 1] ? c1 : 0u) << 16;
        }
        dst[(size_t)i * p.n_words * 32] = w;
      }
    }
  }
}

// TMA-staged pre-pass (round 2). A table group is a run of consecutive X
// columns inside one aligned 4-column block (<= 4 features, all tables in
// SMEM), so one 16-B piece of each row holds every x the group searches. The
// TMA engine copies those pieces for 64 rows at a time (a 2-D tensor box of
// {4 columns, 64 rows} over X) into per-warp rings, kRcTmaStages deep:
//  - the column kernels above gathered x with 4-B loads at a row stride,
//    one 32-B sector per lane and ~12 L1 wavefronts per warp load (C3, ncu:
//    the X gather was half of the L1 data-pipe wavefronts, 105M of 253M);
//    the TMA path spends one 16-B SMEM read per row and no LSU work on X;
//  - one box serves all the group's features: C3's 28 single-feature CTAs
//    pulled 28 sectors per row out of L2, 4-feature groups pull 7.
// Searches: NQ features x kRcTmaU row blocks per lane in lockstep (the
// bucket + binary search of rank_codes_lockstep).
__device__ __forceinline__ void tma_box_2d(uint32_t dst, const CUtensorMap *tm, int c0, int r0, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(r0), "r"(bar)
      : "memory");
}

__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

template <bool LE, int CW, int NQ>
__global__ void __launch_bounds__(32 * kRcTmaWarps, 1)
    rank_code_tma_kernel(const __grid_constant__ CUtensorMap tmx, const RankCodeParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int U = kRcTmaU, S = kRcTmaStages, NW = kRcTmaWarps;
  constexpr int PW = CW == 32 ? 1 : 2;             // features per code word
  const uint4 g = __ldg(p.groups + 2 * blockIdx.x);       // {pool off, bytes, word_begin, word_end}
  const uint4 gs = __ldg(p.groups + 2 * blockIdx.x + 1);  // {first X column, columns, ...}
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(p.pool + g.x);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < g.y / 16u; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *ring = smem + p.stage_off + (size_t)warp * S * kRcTmaStageBytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + p.stage_off + (size_t)NW * S * kRcTmaStageBytes) + warp * 2 * S;
  uint64_t *empty = full + S;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      dev::mbar_init(full + s, 1);
      dev::mbar_init(empty + s, 32);
    }
    dev::fence_mbar_init();
  }
  __syncthreads();                                 // tables and barriers
  const uint32_t tab = dev::smem_u32(smem);
  const int fbeg = PW * (int)g.z, fend = min(PW * (int)g.w, p.n_fc);
  const int c0 = (int)(gs.x & ~3u);                // box column: the aligned 4-column block
  int comp[NQ];
  float lo[NQ], hi[NQ], sc[NQ], bmax[NQ];
  uint32_t sbase[NQ], ubase[NQ];
  bool okf[NQ];
  uint32_t smax = 0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    okf[q] = fbeg + q < fend;
    const int cc = okf[q] ? fbeg + q : fbeg;
    const uint4 m0 = __ldg(p.feat + 2 * cc), m1 = __ldg(p.feat + 2 * cc + 1);
    comp[q] = (int)m0.x - c0;                      // 0..3: the x's place in the 16-B piece
    lo[q] = __uint_as_float(m1.x);
    hi[q] = __uint_as_float(m1.y);
    sc[q] = __uint_as_float(m1.z);
    bmax[q] = (float)(m0.y - 1u);
    sbase[q] = tab + m0.w;
    ubase[q] = tab + m1.w;
    if (okf[q]) smax = max(smax, m0.z);
  }
  // where the group's x sit in the box (CTA-uniform): 0 = columns 0..NQ-1,
  // 2 = columns 2, 3 (NQ = 2), 1 = anything else (per-feature selects)
  bool first_cols = true, last_cols = NQ == 2;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    first_cols = first_cols && comp[q] == q;
    last_cols = last_cols && comp[q] == 2 + q;
  }
  const int lay = first_cols ? 0 : (last_cols ? 2 : 1);
  // this CTA's contiguous slice of units (U row blocks = one box each)
  const int64_t nunits = (p.nblocks + U - 1) / U;
  const int64_t ubeg = blockIdx.y * nunits / gridDim.y, uend = (blockIdx.y + 1) * nunits / gridDim.y;
  const uint32_t ring_s = dev::smem_u32(ring);
  auto issue = [&](int64_t u, int s) {
    dev::mbar_arrive_expect_tx(full + s, kRcTmaStageBytes);
    tma_box_2d(ring_s + (uint32_t)s * kRcTmaStageBytes, &tmx, c0, (int)(u * U * 32), dev::smem_u32(full + s));
  };
  int64_t u = ubeg + warp;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (u + (int64_t)s * NW < uend) issue(u + (int64_t)s * NW, s);
  }
  for (int k = 0; u < uend; ++k, u += NW) {
    const int s = k % S;
    const uint32_t ph = (uint32_t)(k / S) & 1u;
    dev::mbar_wait(full + s, ph);
    float x[NQ][U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const float4 v = lds_f4(ring_s + (uint32_t)s * kRcTmaStageBytes + (uint32_t)(i * 32 + lane) * 16u);
      if (lay == 0) {            // the group's columns are the box's first NQ: no selects
        x[0][i] = v.x;
        x[1][i] = v.y;
        if (NQ == 4) {
          x[NQ - 2][i] = v.z;
          x[NQ - 1][i] = v.w;
        }
      } else if (NQ == 2 && lay == 2) {    // columns 2, 3 of the box
        x[0][i] = v.z;
        x[NQ - 1][i] = v.w;
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) x[q][i] = comp[q] == 0 ? v.x : comp[q] == 1 ? v.y : comp[q] == 2 ? v.z : v.w;
      }
    }
    // the stage is free once every lane holds its x (ordered before the
    // next TMA write by each lane's proxy fence + arrive; lane 0 acquires)
    dev::release_stage(empty + s, lane);
    if (lane == 0 && u + (int64_t)S * NW < uend) {
      dev::mbar_wait(empty + s, ph);
      issue(u + (int64_t)S * NW, s);
    }
    // bucket, then a fixed window of 2^smax - 1 slots from the bucket's
    // first threshold (build_rank_buckets block4 pads every table so the
    // window stays inside it): thresholds of later buckets are > x and the
    // pads are NaN, so the predicate "u <= x" is true on a prefix of the
    // window and the code is the bucket start + the prefix length, found by
    // smax power-of-two steps of one load, one compare and one select
    uint32_t pos[NQ][U];                           // SMEM byte address of the window's next slot
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const float xc = fminf(fmaxf(x[q][i], lo[q]), hi[q]);      // NaN -> lo; replaced below
        const float y = fminf(__fmul_rn(__fsub_rn(xc, lo[q]), sc[q]), bmax[q]);
        const uint32_t be = dev::lds_u32(sbase[q] + 4u * __float2uint_rz(y));
        pos[q][i] = ubase[q] + 4u * (be & 0xFFFFu);
      }
    switch (smax) {
      case 0: break;
      case 1: window_search<LE, NQ, U, 1>(pos, x); break;
      case 2: window_search<LE, NQ, U, 2>(pos, x); break;
      case 3: window_search<LE, NQ, U, 3>(pos, x); break;
      case 4: window_search<LE, NQ, U, 4>(pos, x); break;
      case 5: window_search<LE, NQ, U, 5>(pos, x); break;
      case 6: window_search<LE, NQ, U, 6>(pos, x); break;
      default:
        for (uint32_t sb = 4u << (smax - 1u); sb >= 4u; sb >>= 1) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < U; ++i) {
              const float v = dev::lds_f32(pos[q][i] + sb - 4u);
              pos[q][i] += (LE ? v < x[q][i] : v <= x[q][i]) ? sb : 0u;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int64_t blk = u * U + i;
      if (blk >= p.nblocks) continue;
      // the group's words are consecutive: one base pointer, immediate offsets
      uint32_t *dst = p.codes + ((size_t)blk * p.n_words + (size_t)(fbeg / PW)) * 32 + lane;
#pragma unroll
      for (int q = 0; q < NQ; q += PW) {
        if (!okf[q]) continue;
        const uint32_t c0v = x[q][i] != x[q][i] ? 0xFFFFu : (pos[q][i] - ubase[q]) >> 2;
        uint32_t w;
        if (CW == 32) {
          w = ((uint32_t)(fbeg + q) << 23) | c0v;
        } else {
          const uint32_t c1v = x[q + 1][i] != x[q + 1][i] ? 0xFFFFu : (pos[q + 1][i] - ubase[q + 1]) >> 2;
          w = c0v | ((okf[q + 1] ? c1v : 0u) << 16);
        }
        dst[(q / PW) * 32] = w;
      }
    }
  }
}

int sm_count(int device);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiledFn>(nullptr);
    }
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

static int env_int_rc(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

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
  p.rw = env_int_rc("HB_RC_RW", 1);
  p.pair_loads = m.rank_cw == 16 && m.rank_nfc == m.n_features && m.n_features % 2 == 0 &&
                 a.ldx % 2 == 0 && (reinterpret_cast<uintptr_t>(a.X) & 7) == 0;
  const size_t tbytes = (m.rb_smem + 15) & ~size_t(15);
  p.stage_off = (uint32_t)tbytes;
  // TMA pre-pass: X 16-B aligned with a 16-B multiple row pitch (the tensor
  // map's requirements); otherwise the generic kernels below run the same
  // groups
  const char *etma = std::getenv("HB_RC_TMA");
  if (m.rb_tma && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0 && a.ldx % 4 == 0 && a.n <= INT32_MAX - 256 &&
      !(etma && *etma && std::atoi(etma) == 0) && encode_tiled()) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)m.n_features, (cuuint64_t)a.n};
    const cuuint64_t strides[1] = {(cuuint64_t)a.ldx * 4u};
    const cuuint32_t box[2] = {4u, (cuuint32_t)(kRcTmaU * 32)};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult cr = encode_tiled()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(a.X), dims,
                                       strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(HB_E_CUDA, "cuTensorMapEncodeTiled failed for X");
    const bool le = m.cmp == HB_CMP_LE;
    using TmaFn = void (*)(const CUtensorMap, const RankCodeParams);
    TmaFn fn;
    if (m.rb_max_feats <= 2)
      fn = m.rank_cw == 16 ? (le ? rank_code_tma_kernel<true, 16, 2> : rank_code_tma_kernel<false, 16, 2>)
                           : (le ? rank_code_tma_kernel<true, 32, 2> : rank_code_tma_kernel<false, 32, 2>);
    else
      fn = m.rank_cw == 16 ? (le ? rank_code_tma_kernel<true, 16, 4> : rank_code_tma_kernel<false, 16, 4>)
                           : (le ? rank_code_tma_kernel<true, 32, 4> : rank_code_tma_kernel<false, 32, 4>);
    p.stage_off = (uint32_t)((tbytes + 127) & ~size_t(127));
    const size_t smem = p.stage_off + (size_t)kRcTmaRingBytes;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(rank codes tma)");
    // one wave: as many CTAs as fit per SM, spread over the groups
    // (blockIdx.x = group, blockIdx.y = contiguous row slice)
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * kRcTmaWarps, smem) != cudaSuccess ||
        per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
    }
    const int64_t units = (nblocks + kRcTmaU - 1) / kRcTmaU;
    const int64_t want = std::max<int64_t>(1, ((int64_t)per_sm * sm_count(m.device)) / m.rb_ngroups);   // no tail wave
    const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(want, (units + kRcTmaWarps - 1) / kRcTmaWarps));
    fn<<<dim3(m.rb_ngroups, gy), 32 * kRcTmaWarps, smem, a.stream>>>(tm, p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "rank_code_tma_kernel launch");
    return HB_OK;
  }
  // staged kernel (cp.async X staging) unless the groups span too many
  // columns for the SMEM staging budget (HB_RC_STAGED=0/1 forces; HB_RC_RB
  // picks the 32-row blocks per stage)
  const char *ev = std::getenv("HB_RC_STAGED");
  const char *erb = std::getenv("HB_RC_RB");
  const size_t pitch = (size_t)(m.rb_max_span | 1u);
  const size_t stage_budget = 64 * 1024;
  // single-feature groups (32-bit cells, one word per group): one feature
  // per lockstep set over 4 row blocks (HB_RC_ONE=0/1 forces)
  const char *eone = std::getenv("HB_RC_ONE");
  bool one = m.rank_cw == 32 && m.rb_ngroups == m.rank_nwords;
  // single-feature groups whose tables are all SMEM-resident: the lean
  // column kernel (HB_RC_ONEK=0 keeps the staged kernel)
  const char *eonek = std::getenv("HB_RC_ONEK");
  // Measured: C3 (28 single-feature groups, ~34 KB tables) 1.65 -> 1.39 ms;
  // C4 (54 groups, ~48 KB tables) 2.34 -> 2.67 ms, so the staged kernel keeps
  // models with more than 32 groups (HB_RC_ONEK=1 forces the column kernel)
  const bool one_word = m.rb_ngroups == m.rank_nwords;   // one code word per table group
  const bool onek_auto = m.rb_ngroups <= env_int_rc("HB_RC_ONEK_MAX_GROUPS", 32);
  const bool onek = eonek && *eonek ? std::atoi(eonek) != 0 : onek_auto;
  if (one_word && !m.rb_global && onek && !(ev && *ev && std::atoi(ev) >= 0)) {
    const char *ewp = std::getenv("HB_RC_ONE_WARPS");
    const int ow = ewp && *ewp && std::atoi(ewp) == 16 ? 16 : 8;
    const bool le = m.cmp == HB_CMP_LE;
    RcFn fn1 = m.rank_cw == 16
                   ? (ow == 16 ? (le ? rank_code_one_kernel<true, 16, 16> : rank_code_one_kernel<false, 16, 16>)
                               : (le ? rank_code_one_kernel<true, 8, 16> : rank_code_one_kernel<false, 8, 16>))
                   : (ow == 16 ? (le ? rank_code_one_kernel<true, 16, 32> : rank_code_one_kernel<false, 16, 32>)
                               : (le ? rank_code_one_kernel<true, 8, 32> : rank_code_one_kernel<false, 8, 32>));
    const int smem1 = (int)tbytes;
    cudaError_t e1 = cudaFuncSetAttribute(fn1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
    if (e1 != cudaSuccess) return cuda_fail(e1, "cudaFuncSetAttribute(rank codes one)");
    const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(32 / ow, (220 * 1024) / std::max<size_t>(tbytes, 1)));
    const int64_t units = (nblocks + kOneU - 1) / kOneU;
    const int64_t want = std::max<int64_t>(1, ((int64_t)per_sm * sm_count(m.device) + m.rb_ngroups - 1) / m.rb_ngroups);
    const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(want, (units + ow - 1) / ow));
    fn1<<<dim3(m.rb_ngroups, gy), 32 * ow, smem1, a.stream>>>(p);
    e1 = cudaGetLastError();
    if (e1 != cudaSuccess) return cuda_fail(e1, "rank_code_one_kernel launch");
    return HB_OK;
  }
  if (eone && *eone) one = m.rank_cw == 32 && std::atoi(eone) != 0;
  // 2 row blocks per stage: C3 13.13 ms per step (single-feature sets; 4
  // blocks: 13.39); feature pairs: 13.46 (4 blocks: 13.64)
  int rb = 2;
  while (rb > 1 && (size_t)kRcWarps * kStStages * rb * 32 * pitch * 4 > stage_budget) rb >>= 1;
  if (erb && *erb) rb = std::atoi(erb) >= 4 ? 4 : (std::atoi(erb) >= 2 ? 2 : 1);
  const size_t staged_smem = tbytes + (size_t)kRcWarps * kStStages * rb * 32 * pitch * 4;
  // AUTO: staged when the table groups are narrow (<= 2 features each, e.g.
  // C4: ~40 KB per feature, 54 single-feature groups) or some group is
  // searched from global memory. A narrow group has few searches per row
  // block, so the direct kernel waits on its strided X loads; the cp.async
  // pipeline keeps hundreds of rows in flight per warp (C4: 49.2 -> 46.4 ms
  // per step). Wider groups keep the direct kernel, which runs twice the CTAs
  // per SM (C2, 5 features per group: 0.42 ms direct vs 0.90 ms staged).
  const bool fits = staged_smem <= (size_t)kRcSmemMax + stage_budget && m.rb_max_span > 0;
  bool staged = fits && (m.rb_global || m.rank_nfc <= 2 * m.rb_ngroups);
  if (ev && *ev && std::atoi(ev) >= 0) staged = fits && std::atoi(ev) != 0;   // -1: AUTO
  const char *erows = std::getenv("HB_RC_ROWS");
  const int rows = erows && std::atoi(erows) == 8 ? 8 : kRcRows;
  RcFn fn = staged ? staged_pick(m.cmp == HB_CMP_LE, m.rank_cw, rb, one) : rc_pick(m.cmp == HB_CMP_LE, m.rank_cw, rows);
  const int smem = (int)(staged ? staged_smem : m.rb_smem);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(rank codes)");
  // as many CTAs as fit per SM (by SMEM, at most 4), spread over the feature
  // groups (blockIdx.y)
  const size_t per_cta = staged ? staged_smem : std::max<size_t>(m.rb_smem_cap, 1);
  const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(!staged && rows == 8 ? 3 : 4, (220 * 1024) / per_cta));
  const int64_t want = std::max<int64_t>(1, ((int64_t)per_sm * sm_count(m.device) + m.rb_ngroups - 1) / m.rb_ngroups);
  const int64_t rows_per_cta = (int64_t)kRcWarps * (staged ? rb : rows);
  const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(want, (nblocks + rows_per_cta - 1) / rows_per_cta));
  const char *eord = std::getenv("HB_RC_ORDER");
  // group-major grid with contiguous row slices for the staged kernel: the 28
  // single-feature groups of C3 then read X from DRAM ~1.25x instead of ~5.4x
  // (ncu: 6.1 -> 1.4 GB per launch; C3 13.12 -> 12.92 ms, C4 46.8 -> 46.0 ms)
  // (direct kernel on C2: 1.80 -> 1.78 ms per step); HB_RC_ORDER=0 reverts
  p.gorder = !(eord && *eord && std::atoi(eord) == 0);
  const dim3 grid = p.gorder ? dim3(m.rb_ngroups, gx) : dim3(gx, m.rb_ngroups);
  fn<<<grid, 32 * kRcWarps, smem, a.stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "rank_code_kernel launch");
  return HB_OK;
}

}  // namespace hb
