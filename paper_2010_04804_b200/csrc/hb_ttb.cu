// hb_ttb.cu — TreeTraversal over 2-level node blocks, for wide rows (sm_100a).
//
// Same algorithm as hb_tt.cu (Alg. 2): per (row, tree)
// a data-dependent walk from the root, T_I <- (X[r, N_F[T_I]] < N_T[T_I]) ?
// N_L[T_I] : N_R[T_I], until a leaf, whose N_C value is accumulated. What
// differs is the node layout and the schedule, both chosen for B200's memory
// system:
//
//  * Blocks. Every node array is cut into 2-level blocks: a block holds a node
//    and its two children (3 thresholds, 3 feature ids) and the 4 exits below
//    them, each either another block or a leaf, in one 32-B record = one L2
//    sector. One dependent load now advances a walk two levels (vs one 8-B
//    node per level in hb_tt.cu), halving both the latency chain and the
//    sectors per level of a deep (D = 12) tree whose nodes live in L2.
//    Record: w0..w2 thresholds (slot 0 = block root, 1 = its left child,
//    2 = right child), w3 = f0 | f1 << 16, w4 = f2 | exitmask << 16, w5 = first
//    child block, w6 = first leaf. Exit e = 2 b0 + b1 (b = 1: went right); an
//    exit with mask bit e continues to block w5 + popc(mask below e), else it
//    is leaf w6 + e - popc(mask below e). A leaf reached above the bottom of a
//    block becomes a padding slot with threshold NaN: x < NaN and x <= NaN are
//    false, so the walk goes right through it to an exit holding that leaf —
//    the paper's self-loop idea without a second record.
//  * Schedule. Each lane keeps G independent walk cursors for its row. A
//    cursor that reaches a leaf immediately starts the next tree of the lane's
//    list (persistent walks), so lanes of a warp do not wait for the deepest
//    path of a group of trees (mixed-depth trees: mean path 5.7 of D = 12).
//    The leaf value is loaded when the leaf is reached and added at the
//    cursor's next leaf, off the dependent chain.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <vector>

#include "hb_device.cuh"
#include "hb_internal.h"

namespace hb {

namespace {

struct TtbParams {
  const float *X;
  int64_t n, ldx;
  int F;                  // columns of the X tile (used features when fmap != null)
  const int32_t *fmap;    // compact column -> original feature, or null
  const uint4 *blocks;    // [nblocks][2] 32-B block records; block t = root of tree t
  const float *leaves;    // [nleaves][w]
  const int32_t *lorig;   // [nleaves] original node id (leaf / leaf-hash outputs)
  const uint32_t *cls;    // [T] output of a scalar-leaf tree
  int T, tree_begin;
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
  int ntiles;
};

constexpr int kTtbWarps = 32;
constexpr int kTtbCursors = 4;

// X tile column swizzle: row rr of feature f sits at f * R + (rr ^ h(f)), so
// the coalesced fill (consecutive threads -> consecutive f of one row) is
// bank-conflict free.
template <int R>
__device__ __forceinline__ int swz(int f) {
  constexpr int S = R == 32 ? 0 : (R == 16 ? 1 : 2);
  return (f >> S) & (R - 1);
}

// One 32-B block record per lane in a single 256-bit load (SASS LDG.E.ENL2.256):
// one L1 wavefront per distinct line instead of two for a pair of LDG.128.
__device__ __forceinline__ void ldg256(const uint4 *p, uint4 &a, uint4 &b) {
  asm("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// SYNC: the lanes of a warp move cursor g to its next tree together, once
// every lane's walk of the current one is done (rows of a tree slot stay in
// step, so the top blocks of a tree are fetched once for all of them);
// otherwise each lane's cursor moves on as soon as its own walk ends.
template <bool LE, int NACC, int R, bool SYNC>
__global__ void __launch_bounds__(32 * kTtbWarps, 1) ttb_kernel(const TtbParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int L = 32 / R;                       // tree slots per warp
  constexpr int G = kTtbCursors;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / R, r = lane % R;
  float *xs = reinterpret_cast<float *>(smem);                            // [F][R] swizzled
  float *red = xs + (size_t)p.F * R;                                      // [warps][R][NACC]
  uint64_t *hred = reinterpret_cast<uint64_t *>(red + (size_t)kTtbWarps * R * NACC);  // [warps][R]
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  const int slots = kTtbWarps * L;
  const int T = p.T;
  for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const int64_t row0 = (int64_t)tile * R;
    for (int idx = threadIdx.x; idx < R * p.F; idx += blockDim.x) {
      const int rr = idx / p.F, f = idx - rr * p.F;
      const int64_t gr = row0 + rr;
      const int fo = p.fmap ? __ldg(p.fmap + f) : f;
      xs[f * R + (rr ^ swz<R>(f))] = gr < p.n ? __ldg(p.X + gr * p.ldx + fo) : 0.f;
    }
    __syncthreads();
    const int64_t row = row0 + r;
    float acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.f;
    uint64_t h = 0;
    // cursor g walks tree tc[g] (block blk[g]); this lane's trees are
    // warp * L + sub + j * slots, handed out in order as cursors free up
    int tn = warp * L + sub;
    uint32_t blk[G];
    int tc[G];
    float pv[G];        // deferred leaf value (added at the cursor's next leaf)
    uint32_t pk[G];     // its output (per-class scalar trees)
    bool park[G];       // SYNC: walk done, waiting for the warp
#pragma unroll
    for (int g = 0; g < G; ++g) {
      park[g] = false;
      tc[g] = tn;
      blk[g] = (uint32_t)tn;
      tn += slots;
      pv[g] = 0.f;
      pk[g] = 0u;
    }
    while (true) {
      uint4 qa[G], qb[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (tc[g] < T && !park[g]) ldg256(p.blocks + 2 * (size_t)blk[g], qa[g], qb[g]);
      }
      bool live = false;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (tc[g] >= T) continue;
        live = true;
        if (park[g]) continue;
        const uint32_t f0 = qa[g].w & 0xFFFFu;
        const float x0 = xs[f0 * R + (r ^ swz<R>(f0))];
        const float t0 = __uint_as_float(qa[g].x);
        const bool b0 = !(LE ? x0 <= t0 : x0 < t0);
        const uint32_t f1 = b0 ? (qb[g].x & 0xFFFFu) : (qa[g].w >> 16);
        const float t1 = __uint_as_float(b0 ? qa[g].z : qa[g].y);
        const float x1 = xs[f1 * R + (r ^ swz<R>(f1))];
        const bool b1 = !(LE ? x1 <= t1 : x1 < t1);
        const uint32_t e = (b0 ? 2u : 0u) + (b1 ? 1u : 0u);
        const uint32_t mask = qb[g].x >> 16;
        const uint32_t pc = __popc(mask & ((1u << e) - 1u));
        if ((mask >> e) & 1u) {
          blk[g] = qb[g].y + pc;
        } else {
          const uint32_t leaf = qb[g].z + e - pc;
          if (p.w == 1) {
            if (NACC == 1) {
              acc[0] += pv[g];
            } else {
#pragma unroll
              for (int k = 0; k < NACC; ++k)
                if (pk[g] == (uint32_t)k) acc[k] += pv[g];
              pk[g] = __ldg(p.cls + tc[g]);
            }
            pv[g] = __ldg(p.leaves + leaf);
          } else {
            const float *lv = p.leaves + (size_t)leaf * p.w;
#pragma unroll
            for (int k = 0; k < NACC; ++k)
              if (k < p.K) acc[k] += __ldg(lv + k);
          }
          if (lm) {
            const int32_t id = __ldg(p.lorig + leaf);
            if (lm == 1) {
              if (row < p.n) static_cast<int32_t *>(p.out)[row * (int64_t)T + tc[g]] = id;
            } else {
              h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + tc[g]) << 32) | (uint32_t)id);
            }
          }
          if (SYNC) {
            park[g] = true;
          } else {
            tc[g] = tn;
            blk[g] = (uint32_t)tn;
            tn += slots;
          }
        }
      }
      if (SYNC) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (__all_sync(0xFFFFFFFFu, park[g] || tc[g] >= T)) {
            if (tc[g] < T) {
              tc[g] = tn;
              blk[g] = (uint32_t)tn;
              tn += slots;
            }
            park[g] = false;
          }
        }
      }
      if (!__any_sync(0xFFFFFFFFu, live)) break;
    }
    if (p.w == 1) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (NACC == 1) {
          acc[0] += pv[g];
        } else {
#pragma unroll
          for (int k = 0; k < NACC; ++k)
            if (pk[g] == (uint32_t)k) acc[k] += pv[g];
        }
      }
    }
    // combine the L tree slots of a row inside the warp, then across warps
#pragma unroll
    for (int o = R; o < 32; o <<= 1) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] += __shfl_xor_sync(0xFFFFFFFFu, acc[k], o);
      h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
    }
    if (sub == 0) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) red[(warp * R + r) * NACC + k] = acc[k];
      hred[warp * R + r] = h;
    }
    __syncthreads();
    if (warp == 0 && lane < R) {
      float tot[NACC];
#pragma unroll
      for (int k = 0; k < NACC; ++k) tot[k] = 0.f;
      uint64_t ht = 0;
      for (int w2 = 0; w2 < kTtbWarps; ++w2) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) tot[k] += red[(w2 * R + lane) * NACC + k];
        ht += hred[w2 * R + lane];
      }
      const int64_t orow = row0 + lane;
      if (orow < p.n) {
        if (lm == 2) static_cast<uint64_t *>(p.out)[orow] = ht;
        else if (lm == 0) dev::write_row<NACC>(p.kind, tot, p.K, p.task, p.post, p.scale, p.base, orow, p.out);
      }
    }
    __syncthreads();
  }
}

using TtbFn = void (*)(const TtbParams);

template <bool LE, int R, bool SYNC>
TtbFn ttb_pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return ttb_kernel<LE, 1, R, SYNC>;
    case 4: return ttb_kernel<LE, 4, R, SYNC>;
    case 8: return ttb_kernel<LE, 8, R, SYNC>;
    default: return ttb_kernel<LE, 16, R, SYNC>;
  }
}

template <bool LE, bool SYNC>
TtbFn ttb_pick_r(int R, int nacc) {
  switch (R) {
    case 32: return ttb_pick_nacc<LE, 32, SYNC>(nacc);
    case 16: return ttb_pick_nacc<LE, 16, SYNC>(nacc);
    default: return ttb_pick_nacc<LE, 8, SYNC>(nacc);
  }
}

template <bool LE>
TtbFn ttb_pick(int R, int nacc, bool sync) {
  return sync ? ttb_pick_r<LE, true>(R, nacc) : ttb_pick_r<LE, false>(R, nacc);
}

uint32_t f2u_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

}  // namespace

// Builds the block layout of trees [t0, t1) (remap: original -> X tile
// column, or null) and uploads it as [blocks | leaves | lorig | cls].
hb_status compile_tt_blocks(const hb_ensemble *e, int t0, int t1, const int32_t *remap, Model *m) {
  const int T = t1 - t0, w = e->leaf_width, K = e->n_outputs;
  const uint32_t kNaN = 0x7FC00000u;
  std::vector<uint32_t> blocks((size_t)T * 8, 0);
  std::vector<float> leaves;
  std::vector<int32_t> lorig;
  std::vector<uint32_t> cls(T, 0);
  size_t nblocks = (size_t)T;
  struct Slot {
    int node;      // original node id (local to the tree)
    bool pad;      // leaf above the block bottom: NaN threshold, always right
  };
  std::deque<std::pair<size_t, int>> q;   // (block index, block root node)
  for (int lt = 0; lt < T; ++lt) {
    const int t = t0 + lt;
    const int64_t a = e->node_offset[t];
    cls[lt] = (uint32_t)(e->tree_output ? e->tree_output[t] : t % K);
    q.clear();
    q.emplace_back((size_t)lt, 0);
    while (!q.empty()) {
      const size_t bi = q.front().first;
      const int root = q.front().second;
      q.pop_front();
      auto internal = [&](int v) { return e->left[a + v] != -1; };
      Slot s[3];
      s[0] = {root, !internal(root)};
      s[1] = s[0].pad ? s[0] : Slot{e->left[a + root], !internal(e->left[a + root])};
      s[2] = s[0].pad ? s[0] : Slot{e->right[a + root], !internal(e->right[a + root])};
      if (!s[0].pad) {
        s[1].pad = !internal(s[1].node);
        s[2].pad = !internal(s[2].node);
      }
      uint32_t thr[3], feat[3];
      int exits[4];
      for (int k = 0; k < 3; ++k) {
        const int v = s[k].node;
        if (s[k].pad) {
          thr[k] = kNaN;
          feat[k] = 0;
        } else {
          float th = e->threshold[a + v];
          thr[k] = f2u_bits(th);
          const int f = e->feature[a + v];
          feat[k] = (uint32_t)(remap ? remap[f] : f);
        }
      }
      for (int k = 1; k <= 2; ++k) {
        const int v = s[k].node;
        const int el = 2 * (k - 1);
        if (s[k].pad) {
          exits[el] = exits[el + 1] = v;
        } else {
          exits[el] = e->left[a + v];
          exits[el + 1] = e->right[a + v];
        }
      }
      uint32_t mask = 0;
      const uint32_t cbase = (uint32_t)nblocks, lbase = (uint32_t)lorig.size();
      for (int x = 0; x < 4; ++x) {
        const int v = exits[x];
        if (internal(v)) {
          mask |= 1u << x;
          q.emplace_back(nblocks++, v);
        } else {
          lorig.push_back(v);
          for (int k = 0; k < w; ++k) leaves.push_back(e->leaf_value[(a + v) * w + k]);
        }
      }
      if (nblocks > 0xFFFFFFFFull || lorig.size() > 0xFFFFFFFFull)
        return fail(HB_E_UNSUPPORTED, "TT blocks: more than 2^32 blocks or leaves");
      if (blocks.size() < nblocks * 8) blocks.resize(std::max(nblocks * 8, blocks.size() * 2), 0);
      uint32_t *b = blocks.data() + bi * 8;
      b[0] = thr[0];
      b[1] = thr[1];
      b[2] = thr[2];
      b[3] = feat[0] | (feat[1] << 16);
      b[4] = feat[2] | (mask << 16);
      b[5] = cbase;
      b[6] = lbase;
      b[7] = 0;
    }
  }
  blocks.resize(nblocks * 8);
  auto al = [](size_t x) { return (x + 127) & ~size_t(127); };
  const size_t ob = 0, ol = al(blocks.size() * 4), oo = ol + al(std::max<size_t>(leaves.size(), 1) * 4),
               oc = oo + al(std::max<size_t>(lorig.size(), 1) * 4), total = oc + al(cls.size() * 4);
  std::vector<uint8_t> buf(total, 0);
  std::memcpy(buf.data() + ob, blocks.data(), blocks.size() * 4);
  std::memcpy(buf.data() + ol, leaves.data(), leaves.size() * 4);
  std::memcpy(buf.data() + oo, lorig.data(), lorig.size() * 4);
  std::memcpy(buf.data() + oc, cls.data(), cls.size() * 4);
  cudaError_t err;
  if ((err = cudaMalloc(&m->d_ttb, total)) != cudaSuccess) return cuda_fail(err, "cudaMalloc(tt blocks)");
  m->device_bytes += total;
  if ((err = cudaMemcpy(m->d_ttb, buf.data(), total, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(err, "cudaMemcpy(tt blocks)");
  m->ttb_leaf_off = ol;
  m->ttb_lorig_off = oo;
  m->ttb_cls_off = oc;
  m->ttb_nblocks = (int64_t)nblocks;
  m->tt_blocks = 1;
  const char *sv = std::getenv("HB_TTB_SYNC");
  m->ttb_sync = (sv && *sv) ? std::atoi(sv) : 1;
  return HB_OK;
}

int sm_count(int device);

hb_status launch_tt_blocks(const Model &m, const RunArgs &a) {
  const int R = m.cfg.wide_rows;
  const bool sync = m.ttb_sync != 0;
  TtbFn fn = m.cmp == HB_CMP_LE ? ttb_pick<true>(R, m.nacc, sync) : ttb_pick<false>(R, m.nacc, sync);
  TtbParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.F = m.n_xf;
  p.fmap = m.d_fmap;
  const uint8_t *b = static_cast<const uint8_t *>(m.d_ttb);
  p.blocks = reinterpret_cast<const uint4 *>(b);
  p.leaves = reinterpret_cast<const float *>(b + m.ttb_leaf_off);
  p.lorig = reinterpret_cast<const int32_t *>(b + m.ttb_lorig_off);
  p.cls = reinterpret_cast<const uint32_t *>(b + m.ttb_cls_off);
  p.T = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  const int64_t ntiles = (a.n + R - 1) / R;
  if (ntiles > INT32_MAX) return fail(HB_E_UNSUPPORTED, "too many rows for one launch");
  p.ntiles = (int)ntiles;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count(m.device));
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m.cfg.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(ttb)");
  fn<<<grid, 32 * kTtbWarps, m.cfg.smem_bytes, a.stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "ttb_kernel launch");
  return HB_OK;
}

}  // namespace hb
