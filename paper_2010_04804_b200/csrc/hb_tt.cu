// hb_tt.cu — TreeTraversal scorer for sm_100a (Alg. 2, P:206-237;
// Table 5; fixed TREE_DEPTH iterations with leaf self-loops).
//
// Alg. 2 per (row, tree): T_I <- root; repeat TREE_DEPTH: T_F <- N_F[T_I];
// T_V <- X[r, T_F]; T_T <- N_T[T_I]; T_I <- Where(T_V < T_T, N_L[T_I],
// N_R[T_I]); R <- N_C[T_I].
//
// Compiled node record (8 B): nodes are renumbered in BFS
// order with siblings adjacent, so N_L = N_R - 1 and one record carries
// {N_F | N_R << 16, N_T}. A leaf j stores N_R = j and N_T = NaN: both LT and LE
// are false against NaN, so T_I <- N_R = j — the paper's self-loop.
// X comes from a per-warp SMEM slice when it fits, else straight from global
// memory (wide rows, e.g. Epsilon-shaped F = 2000); tree records stream through
// the same cp.async.bulk ring as PTT when a chunk fits in SMEM, else are read
// through L2/L1 (deep D = 12 trees of very large ensembles).
#include <cuda_runtime.h>

#include "hb_device.cuh"
#include "hb_internal.h"
#include "hb_layouts.h"

namespace hb {

struct TtParams {
  const float *X;
  int64_t n, ldx;
  int F, vec4, depth;     // F: columns of the X tile (used features when fmap != null)
  const int32_t *fmap;    // compact column -> original feature, or null
  const uint8_t *trees;
  uint32_t stride;
  int n_trees_pad, n_trees, tree_begin;
  const int32_t *leafmap;
  int nslots;
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
  int nw, ns, ch, ntiles, x_smem, t_smem;
  int x_prefetch;         // tt_wide_kernel: L2 prefetch of the next row tile
  const uint4 *ttw;       // tt_wide_kernel: packed 16-B records (hb_host.cpp build_ttw)
  const uint32_t *toff;   // tt_wide_kernel: tree offsets in 16-B units
  // tt_wide_kernel over one tree chunk of a model larger than L2 (launch_tt):
  int accumulate;         // RAW64 / LEAF_HASH outputs are added to, not written
  int leaf_stride;        // LEAF output row stride (the model's tree count)
  int tree_off;           // first model-local tree of this chunk (LEAF column)
};

// One Alg. 2 walk over a tree record staged in shared memory: nodes at the
// 32-bit shared address `nodes` (8-B records), this lane's X slice at `xlane`
// (xs[f * 32 + lane] -> byte offset 128 f). Explicit ld.shared (the ring is
// rewritten by the TMA engine between mbarrier phases).
template <bool LE>
__device__ __forceinline__ uint32_t tt_walk(uint32_t nodes, uint32_t xlane, int depth) {
  uint32_t i = 0;
#pragma unroll 4
  for (int l = 0; l < depth; ++l) {
    const uint2 d = dev::lds_v2(nodes + 8u * i);
    const float x = dev::lds_f32(xlane + ((d.x & 0xFFFFu) << 7));
    const float t = __uint_as_float(d.y);
    const bool pr = LE ? (x <= t) : (x < t);
    i = (d.x >> 16) - (pr ? 1u : 0u);
  }
  return i;
}

// Narrow-row TreeTraversal: the PTT kernel's structure (X slice per warp in
// SMEM, tree records streamed through a cp.async.bulk ring by a producer
// warp); AUTO uses it for TT models whose rows and records fit (the launch
// configuration always stages both in SMEM).
template <bool LE, int NACC>
__global__ void __launch_bounds__(32 * 17, 1) tt_kernel(const TtParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = p.nw, ns = p.ns, ch = p.ch;
  const size_t xbytes = (size_t)nw * p.F * 128;
  uint8_t *stages = smem + xbytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(stages + (size_t)ns * ch * p.stride);
  uint64_t *empty = full + ns;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      dev::mbar_init(&full[s], 1);
      dev::mbar_init(&empty[s], dev::ring_arrivals(nw));
    }
    dev::fence_mbar_init();
  }
  __syncthreads();
  const int nchunks = (p.n_trees_pad + ch - 1) / ch;
  const int my_tiles = (p.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

  if (warp == nw) {
    if (lane == 0) {
      const long total = (long)my_tiles * nchunks;
      dev::Ring r(ns);
      int c = 0;
      for (long it = 0; it < total; ++it, r.next(), c = (c + 1 == nchunks) ? 0 : c + 1) {
        const int s = r.s;
        dev::mbar_wait(&empty[s], r.ph ^ 1u);
        const int t0 = c * ch;
        const int nt = min(ch, p.n_trees_pad - t0);
        const uint32_t bytes = (uint32_t)nt * p.stride;
        dev::mbar_arrive_expect_tx(&full[s], bytes);
        dev::bulk_g2s(stages + (size_t)s * ch * p.stride, p.trees + (size_t)t0 * p.stride, bytes,
                      &full[s]);
      }
    }
    return;
  }

  float *xs = reinterpret_cast<float *>(smem) + (size_t)warp * p.F * 32;
  const uint32_t xlane = dev::smem_u32(xs) + 4u * (uint32_t)lane;
  const uint32_t stage0 = dev::smem_u32(stages);
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  dev::Ring ring(ns);
  for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const int64_t row = (int64_t)tile * (nw * 32) + warp * 32 + lane;
    if (p.fmap) dev::load_x_slice_map(xs, p.X, row, p.n, p.ldx, p.fmap, p.F, lane);
    else dev::load_x_slice(xs, p.X, row, p.n, p.ldx, p.F, lane, p.vec4 != 0);
    __syncwarp();
    double acc[NACC];   // fp64 accumulation (R23)
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    uint64_t h = 0;
    for (int c = 0; c < nchunks; ++c, ring.next()) {
      const int s = ring.s;
      dev::mbar_wait(&full[s], ring.ph);
      const uint32_t cb = stage0 + (uint32_t)(s * ch) * p.stride;
      const int nt = min(ch, p.n_trees_pad - c * ch);
      for (int j = 0; j < nt; j += 2) {
        const uint32_t ra = cb + (uint32_t)j * p.stride;
        const uint32_t rb = ra + p.stride;
        const uint32_t ia = tt_walk<LE>(ra + 16u, xlane, p.depth);
        const uint32_t ib = tt_walk<LE>(rb + 16u, xlane, p.depth);
        const uint32_t la = ra + 16u + 8u * (uint32_t)p.nslots;   // leaf[nslots][w]
        const uint32_t lb = rb + 16u + 8u * (uint32_t)p.nslots;
        if (p.w == 1) {
          const double va = (double)dev::lds_f32(la + 4u * ia), vb = (double)dev::lds_f32(lb + 4u * ib);
          if (NACC == 1) {
            acc[0] += va;
            acc[0] += vb;
          } else {
            const uint32_t ka = dev::lds_u32(ra);
            const uint32_t kb = dev::lds_u32(rb);
#pragma unroll
            for (int k = 0; k < NACC; ++k) {
              if (ka == (uint32_t)k) acc[k] += va;
              if (kb == (uint32_t)k) acc[k] += vb;
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < NACC; ++k)
            if (k < p.K) acc[k] += (double)dev::lds_f32(la + 4u * (ia * (uint32_t)p.w + k));
#pragma unroll
          for (int k = 0; k < NACC; ++k)
            if (k < p.K) acc[k] += (double)dev::lds_f32(lb + 4u * (ib * (uint32_t)p.w + k));
        }
        if (lm) {
          const int tg = c * ch + j;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int t = tg + q;
            if (t < p.n_trees) {
              const int32_t id = __ldg(p.leafmap + (size_t)t * p.nslots + (q ? ib : ia));
              if (lm == 1) {
                if (row < p.n) static_cast<int32_t *>(p.out)[row * p.n_trees + t] = id;
              } else {
                h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + t) << 32) | (uint32_t)id);
              }
            }
          }
        }
      }
      dev::release_stage(&empty[s], lane);
    }
    if (row < p.n) {
      if (lm == 2) {
        static_cast<uint64_t *>(p.out)[row] = h;
      } else if (lm == 0) {
        dev::write_row<NACC>(p.kind, acc, p.K, p.task, p.post, p.scale, p.base, row, p.out);
      }
    }
  }
}

// Wide-row TreeTraversal (Epsilon-shaped X, F up to thousands; deep trees
// whose records do not fit SMEM). A CTA owns R rows whose X tile lives in SMEM
// feature-major (xs[f*R + r]); lane = (tree slot, row) with 32/R tree slots per
// warp, and all warps of the CTA walk disjoint trees of the same R rows. Node
// records (16 B per internal node with both children's payloads, hb_host.cpp
// build_ttw: a walk to a leaf at depth D_k is D_k dependent loads, the last
// one carrying the leaf value) come through L1/L2 (__ldg): the R rows of a
// tree slot share their top-level requests (one sector for the root, <= 2^l
// at level l). Each lane walks G trees at once
// (memory-level parallelism); finished walks issue no loads and the group ends
// once every walk of the warp reached a leaf (the fixed TREE_DEPTH loop of
// Alg. 2 with its leaf self-loops, cut short). Per-row sums are
// combined with warp shuffles and one SMEM pass in a fixed order.
// X tile layout: plain xs[f*R + r], so the R lanes of one tree slot (distinct
// rows) always read distinct banks whatever features their walks test; only
// lanes of different tree slots on the same row can meet (<= 32/R-way). The
// fill gives the 32/R row groups of a warp different 4-feature chunks and
// rotates their store order so a warp's 32 stores hit 32 distinct banks.

// One level of Alg. 2 on the 16-B records: T_V <- X[r, N_F] (the record holds
// the column's byte offset in the X tile); go left iff pred(T_V, N_T); the
// chosen child is the next record or, when its leaf flag is set, the leaf
// payload (value bits for w == 1, leaf slot for w > 1). A finished walk
// (done != 0) issues no load; q then still names the last record.
template <bool LE>
__device__ __forceinline__ void wide_step(const uint4 *tr, uint32_t &q, uint32_t &pay, uint32_t &done,
                                          uint32_t xlane) {
  if (done == 0u) {
    HB_DCHECK(q < __ldg(&tr->x));               // record index inside the tree (header: n_records)
    const uint4 d = __ldg(tr + 1 + q);          // record q follows the 16-B tree header
    const float x = dev::lds_f32(xlane + (d.x & ~3u));
    const float t = __uint_as_float(d.y);
    const bool pr = LE ? (x <= t) : (x < t);
    pay = pr ? d.z : d.w;
    done = d.x & (pr ? 1u : 2u);
    if (done == 0u) q = pay;
  }
}

template <bool LE, int NACC, int R, int G>   // G: trees walked at once per lane
__global__ void __launch_bounds__(1024, 1) tt_wide_kernel(const TtParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int L = 32 / R;                       // tree slots per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int sub = lane / R, r = lane % R;
  float *xs = reinterpret_cast<float *>(smem);                       // [F][R]
  double *red = reinterpret_cast<double *>(xs + (((size_t)p.F * R + 1) & ~(size_t)1));  // [nwarps][R][NACC]
  uint64_t *hred = reinterpret_cast<uint64_t *>(red + (size_t)nwarps * R * NACC);       // [nwarps][R]
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  const int slots = nwarps * L;
  for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const int64_t row0 = (int64_t)tile * R;
    // X tile load: lane = (row group sub, row rr); each lane loads one
    // 4-feature chunk of its row (16 B, float4 when aligned) and stores it
    // feature-major, the store order rotated by sub (bank = chunk position)
    {
      constexpr int SUBS = 32 / R;
      const int F4 = (p.F + 3) >> 2;
      const int nblk = (F4 + SUBS - 1) / SUBS;
      const bool v4 = !p.fmap && p.vec4 && (p.F & 3) == 0;
      if (v4) {
        // U independent 16-B loads per thread in flight before the stores:
        // the fill waits one L2/HBM latency per U chunks, not per chunk
        constexpr int U = 4;
        const int total = nblk * 32;
        for (int i0 = threadIdx.x; i0 < total; i0 += U * blockDim.x) {
          float4 v[U];
          int f_[U], rr_[U], sub_[U];
          bool ok[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int idx = i0 + u * (int)blockDim.x;
            const int q = idx & 31, rr = q % R, sub = q / R;
            const int c = (idx >> 5) * SUBS + sub;
            ok[u] = idx < total && c < F4;
            f_[u] = 4 * c;
            rr_[u] = rr;
            sub_[u] = sub;
            const int64_t gr = row0 + rr;
            v[u] = ok[u] && gr < p.n ? __ldg(reinterpret_cast<const float4 *>(p.X + gr * p.ldx + 4 * c))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int jj = (j + sub_[u]) & 3;
              const float val = jj == 0 ? v[u].x : (jj == 1 ? v[u].y : (jj == 2 ? v[u].z : v[u].w));
              xs[(f_[u] + jj) * R + rr_[u]] = val;
            }
          }
        }
      } else {
        for (int idx = threadIdx.x; idx < nblk * 32; idx += blockDim.x) {
          const int q = idx & 31, rr = q % R, sub = q / R;
          const int c = (idx >> 5) * SUBS + sub;
          if (c >= F4) continue;
          const int f = 4 * c;
          const int64_t gr = row0 + rr;
          float t[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int fj = f + j;
            t[j] = (gr < p.n && fj < p.F) ? __ldg(p.X + gr * p.ldx + (p.fmap ? __ldg(p.fmap + fj) : fj)) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int jj = (j + sub) & 3;
            const float val = jj == 0 ? t[0] : (jj == 1 ? t[1] : (jj == 2 ? t[2] : t[3]));
            if (f + jj < p.F) xs[(f + jj) * R + rr] = val;
          }
        }
      }
    }
    // warm L2 with the next tile's rows while this one is walked (the fill
    // above is not overlapped with compute: one 8 KB row per lane group)
    if (threadIdx.x == 0 && p.x_prefetch)
      dev::prefetch_rows_l2(p.X, (int64_t)(tile + gridDim.x) * R, R, p.n, p.ldx);
    __syncthreads();
    const int64_t row = row0 + r;
    const uint32_t xlane = dev::smem_u32(xs) + 4u * (uint32_t)r;   // this lane's row in the X tile
    double acc[NACC];   // fp64 accumulation (R23)
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    uint64_t h = 0;
    // walk of tree t ended on record q, payload pay: add the leaf value /
    // emit the leaf's original id
    auto finish = [&](int t, const uint4 *tr, uint32_t q, uint32_t pay) {
      if (p.w == 1) {
        const double v = (double)__uint_as_float(pay);
        if (NACC == 1) {
          acc[0] += v;
        } else {
          const uint32_t k0 = __ldg(reinterpret_cast<const uint32_t *>(tr) + 2);   // tree_output
#pragma unroll
          for (int k = 0; k < NACC; ++k)
            if (k0 == (uint32_t)k) acc[k] += v;
        }
      } else {
        const float *lv = reinterpret_cast<const float *>(
            reinterpret_cast<const uint8_t *>(tr) + __ldg(reinterpret_cast<const uint32_t *>(tr) + 3));
#pragma unroll
        for (int k = 0; k < NACC; ++k)
          if (k < p.K) acc[k] += (double)__ldg(lv + pay * p.w + k);
      }
      if (lm && t < p.n_trees) {
        const uint32_t *ids = reinterpret_cast<const uint32_t *>(
            reinterpret_cast<const uint8_t *>(tr) + __ldg(reinterpret_cast<const uint32_t *>(tr) + 1));
        // the side the walk took at record q (re-evaluated: only the leaf-id
        // outputs need it, the value path does not carry it)
        const uint4 d = __ldg(tr + 1 + q);
        const float x = dev::lds_f32(xlane + (d.x & ~3u));
        const bool pr = LE ? (x <= __uint_as_float(d.y)) : (x < __uint_as_float(d.y));
        const int32_t id = (int32_t)__ldg(ids + 2 * q + (pr ? 0u : 1u));
        if (lm == 1) {
          if (row < p.n) static_cast<int32_t *>(p.out)[row * p.leaf_stride + p.tree_off + t] = id;
        } else {
          h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + t) << 32) | (uint32_t)id);
        }
      }
    };
    const int levels = p.depth > 0 ? p.depth : 1;   // a single-leaf tree still has one record
    // warp-uniform loop over groups of G tree slots (t = base + sub + g*slots)
    for (int base = warp * L; base < p.n_trees_pad; base += G * slots) {
      const uint4 *tr[G];
      uint32_t q[G], pay[G], dn[G];
      bool valid[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int t = base + sub + g * slots;
        valid[g] = t < p.n_trees_pad;                 // uniform across the warp
        tr[g] = p.ttw + __ldg(p.toff + (valid[g] ? t : base + sub));
        q[g] = 0;
        pay[g] = 0;
        dn[g] = valid[g] ? 0u : 4u;                   // no tree, nothing to walk
      }
      for (int l = 0; l < levels; ++l) {
#pragma unroll
        for (int g = 0; g < G; ++g) wide_step<LE>(tr[g], q[g], pay[g], dn[g], xlane);
        bool all = true;
#pragma unroll
        for (int g = 0; g < G; ++g) all = all && dn[g] != 0u;
        if (__all_sync(0xFFFFFFFFu, all)) break;    // every walk of the warp reached a leaf
      }
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (valid[g]) finish(base + sub + g * slots, tr[g], q[g], pay[g]);
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
      double tot[NACC];
#pragma unroll
      for (int k = 0; k < NACC; ++k) tot[k] = 0.0;
      uint64_t ht = 0;
      for (int w2 = 0; w2 < nwarps; ++w2) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) tot[k] += red[(w2 * R + lane) * NACC + k];
        ht += hred[w2 * R + lane];
      }
      const int64_t orow = row0 + lane;
      if (orow < p.n) {
        if (lm == 2) {
          uint64_t *o = static_cast<uint64_t *>(p.out) + orow;
          *o = p.accumulate ? *o + ht : ht;
        } else if (lm == 0 && p.accumulate) {      // fp64 RAW partial of a later tree chunk
#pragma unroll
          for (int k = 0; k < NACC; ++k)
            if (k < p.K) static_cast<double *>(p.out)[orow * p.K + k] += tot[k];
        } else if (lm == 0) {
          dev::write_row<NACC>(p.kind, tot, p.K, p.task, p.post, p.scale, p.base, orow, p.out);
        }
      }
    }
    __syncthreads();
  }
}

using TtFn = void (*)(const TtParams);

template <bool LE>
static TtFn pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return tt_kernel<LE, 1>;
    case 4: return tt_kernel<LE, 4>;
    case 8: return tt_kernel<LE, 8>;
    default: return tt_kernel<LE, 16>;
  }
}

int sm_count(int device);

template <bool LE, int R>
static TtFn pick_wide_nacc(int nacc, int g) {
  // 6 or 8 concurrent walks per lane: scalar outputs only (registers)
  if (nacc == 1 && g == 8) return tt_wide_kernel<LE, 1, R, 8>;
  if (nacc == 1 && g == 6) return tt_wide_kernel<LE, 1, R, 6>;
  switch (nacc) {
    case 1: return tt_wide_kernel<LE, 1, R, 4>;
    case 4: return tt_wide_kernel<LE, 4, R, 4>;
    case 8: return tt_wide_kernel<LE, 8, R, 4>;
    default: return tt_wide_kernel<LE, 16, R, 4>;
  }
}

template <bool LE>
static TtFn pick_wide(int R, int nacc, int g) {
  switch (R) {
    case 32: return pick_wide_nacc<LE, 32>(nacc, g);
    case 16: return pick_wide_nacc<LE, 16>(nacc, g);
    default: return pick_wide_nacc<LE, 8>(nacc, g);
  }
}

hb_status launch_tt(const Model &m, const RunArgs &a) {
  const bool wide = m.cfg.wide_rows > 0;
  TtFn fn = wide ? (m.cmp == HB_CMP_LE ? pick_wide<true>(m.cfg.wide_rows, m.nacc, m.tt_g)
                                      : pick_wide<false>(m.cfg.wide_rows, m.nacc, m.tt_g))
                 : (m.cmp == HB_CMP_LE ? pick_nacc<true>(m.nacc) : pick_nacc<false>(m.nacc));
  TtParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.F = m.n_xf;
  p.fmap = m.d_fmap;
  p.vec4 = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);
  p.depth = m.depth;
  p.trees = static_cast<const uint8_t *>(m.d_trees);
  p.stride = (uint32_t)m.stride;
  p.n_trees_pad = m.n_trees_pad;
  p.n_trees = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.leafmap = m.d_leafmap;
  p.nslots = m.nslots;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  p.nw = m.cfg.nw;
  p.ns = m.cfg.ns;
  p.ch = m.cfg.ch;
  p.x_smem = m.cfg.x_smem;
  p.t_smem = m.cfg.t_smem;
  p.x_prefetch = m.cfg.prefetch;
  p.ttw = static_cast<const uint4 *>(m.d_ttw);
  p.toff = m.d_ttw_off;
  p.accumulate = 0;
  p.leaf_stride = m.n_trees;
  p.tree_off = 0;
  const int64_t rows_per_tile = wide ? (int64_t)m.cfg.wide_rows : (int64_t)m.cfg.nw * 32;
  const int64_t ntiles = (a.n + rows_per_tile - 1) / rows_per_tile;
  if (ntiles > INT32_MAX) return fail(HB_E_UNSUPPORTED, "too many rows for one launch");
  p.ntiles = (int)ntiles;
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count(m.device) * m.cfg.ctas_per_sm);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       m.cfg.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tt)");
  const int threads = wide ? 32 * m.cfg.nw : 32 * (m.cfg.nw + 1);
  if (!wide && (!m.cfg.x_smem || !m.cfg.t_smem))
    return fail(HB_E_UNSUPPORTED, "tt_kernel needs its X slices and tree ring in SMEM");
  if (!(wide && m.tt_chunk > 0 && m.n_trees_pad > m.tt_chunk)) {
    fn<<<grid, threads, m.cfg.smem_bytes, a.stream>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "tt_kernel launch");
    return HB_OK;
  }
  // model larger than L2: walk it in L2-resident tree chunks (every chunk
  // re-streams X from HBM, sequentially, instead of fetching deep node
  // records from HBM at random). fp64 RAW partials accumulate in a scratch
  // buffer from the model's pool (RAW64 / LEAF_HASH: in the output itself),
  // and one finalize launch writes PREDICT / PROBA / MARGIN / RAW.
  const bool direct = a.kind == HB_OUT_RAW64 || a.kind == HB_OUT_LEAF_HASH || a.kind == HB_OUT_LEAF;
  double *raw = nullptr;
  if (!direct) {
    const hb_status st = scratch_alloc(m, (size_t)a.n * m.n_outputs * sizeof(double), a.stream,
                                       reinterpret_cast<void **>(&raw));
    if (st != HB_OK) return st;
  }
  for (int t0 = 0; t0 < m.n_trees_pad; t0 += m.tt_chunk) {
    TtParams pc = p;
    pc.toff = p.toff + t0;
    pc.n_trees_pad = std::min(m.tt_chunk, m.n_trees_pad - t0);
    pc.n_trees = std::max(0, std::min(m.tt_chunk, m.n_trees - t0));
    pc.tree_begin = m.tree_begin + t0;
    pc.leafmap = p.leafmap + (size_t)t0 * p.nslots;
    pc.tree_off = t0;
    pc.kind = direct ? a.kind : HB_OUT_RAW64;
    pc.out = direct ? a.out : static_cast<void *>(raw);
    pc.accumulate = t0 > 0 && pc.kind != HB_OUT_LEAF;
    if (t0 > 0) mark_launch(a);    // next chunk launch starts
    fn<<<grid, threads, m.cfg.smem_bytes, a.stream>>>(pc);
    e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (raw) cudaFreeAsync(raw, a.stream);
      return cuda_fail(e, "tt_wide_kernel launch (tree chunk)");
    }
  }
  if (!direct) {
    RunArgs f = a;
    f.raw_in = nullptr;
    f.raw_in64 = raw;
    mark_launch(a);                // finalize starts
    const hb_status st = launch_finalize(m, f);
    cudaFreeAsync(raw, a.stream);
    if (st != HB_OK) return st;
  }
  return HB_OK;
}

}  // namespace hb
