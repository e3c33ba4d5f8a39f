// hb_ptt.cu — PerfectTreeTraversal scorer for sm_100a (Alg. 3,
// P:259-284; perfect padding P:243; Table 6).
//
// Alg. 3 per (row, tree):  T_I <- 1;  repeat D: T_F <- N'_F[T_I];
// T_V <- X[r, T_F]; T_T <- N'_T[T_I]; T_I <- 2 T_I + (T_V < T_T ? 0 : 1);
// R <- N'_C[T_I - 2^D]. Here one lane owns one row and walks every tree with
// D unrolled ("we unroll all iterations"), two trees at a time for ILP.
//
// Data movement:
//  * X: each warp stages its 32 rows feature-major in SMEM (xs[f*32 + lane]),
//    so the data-dependent read X[r, f] is bank-conflict free.
//  * Trees: the compiled PTT records (per tree: heap-ordered {feature, thr}
//    nodes then the 2^D leaf values) stream through an NS-stage SMEM ring,
//    filled by a dedicated producer warp with cp.async.bulk (TMA bulk copy,
//    UBLKCP) and mbarrier transaction counts; consumer warps release a stage
//    with one mbarrier arrive each.
//  * Persistent CTAs (one per SM) loop over row tiles of 32*NW rows; the tree
//    stream simply restarts for every tile.
#include <cuda_runtime.h>

#include <cstdlib>

#include "hb_device.cuh"
#include "hb_internal.h"

namespace hb {

struct PttParams {
  const float *X;
  int64_t n, ldx;
  int F;                  // columns of the X slice (used features when fmap != null)
  const int32_t *fmap;    // compact column -> original feature, or null (identity)
  int vec4;
  const uint8_t *trees;
  uint32_t stride;
  int n_trees_pad, n_trees, tree_begin;
  const int32_t *leafmap;
  int nslots;
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
  int nw, ns, ch, ntiles;
  int prefetch;           // L2 prefetch of the next tile's X rows
  int interleave;         // 1: warp units interleaved over the grid (ntiles = rounds; hb_pttr_kernel.cuh)
};

template <int D, bool LE, int NACC, int G>
__global__ void __launch_bounds__(32 * 25, 1) ptt_kernel(const PttParams p) {
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
  // contiguous CTA tiles, or warp units interleaved over the grid so that a
  // partial last round leaves every SM some warps (as pttr_kernel)
  const int my_tiles = p.interleave ? p.ntiles
                                    : (p.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  auto unit_of = [&](int k) -> int64_t {
    return p.interleave ? ((int64_t)k * nw + warp) * gridDim.x + blockIdx.x
                        : ((int64_t)blockIdx.x + (int64_t)k * gridDim.x) * nw + warp;
  };

  if (warp == nw) {
    // ---------------- producer warp: stream tree chunks through the ring
    if (lane == 0) {
      const long total = (long)my_tiles * nchunks;
      dev::Ring r(ns);
      int c = 0;
      for (long it = 0; it < total; ++it, r.next(), c = (c + 1 == nchunks) ? 0 : c + 1) {
        const int s = r.s;
        dev::mbar_wait(&empty[s], r.ph ^ 1u);
        if (c == 0 && p.prefetch && !p.interleave) {
          // first item of a tile: warm L2 with this CTA's NEXT tile of X rows
          const long tile_i = it / nchunks;
          const int64_t next = (int64_t)(blockIdx.x + (tile_i + 1) * gridDim.x) * (nw * 32);
          dev::prefetch_rows_l2(p.X, next, (int64_t)nw * 32, p.n, p.ldx);
        }
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

  // ---------------- consumer warps
  float *xs = reinterpret_cast<float *>(smem) + (size_t)warp * p.F * 32;
  const uint32_t xlane = dev::smem_u32(xs) + 4u * lane;   // X[row, f] at xlane + 128 f
  const uint32_t stage0 = dev::smem_u32(stages);
  const uint32_t leaf_off = 4u << D;                      // leaf(i) at tree + leaf_off + 4 i ... (w = 1)
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  dev::Ring ring(ns);
  for (int k = 0; k < my_tiles; ++k) {
    const int64_t wrow0 = unit_of(k) * 32;
    if (p.interleave && p.prefetch && lane == 0)   // warm L2 with this warp's next rows
      dev::prefetch_rows_l2(p.X, unit_of(k + 1) * 32, 32, p.n, p.ldx);
    const int64_t row = wrow0 + lane;
    const bool active = wrow0 < p.n;        // whole warp beyond n: only keep the ring in step
    if (active) {
      if (p.fmap) dev::load_x_slice_map(xs, p.X, row, p.n, p.ldx, p.fmap, p.F, lane);
      else dev::load_x_slice(xs, p.X, row, p.n, p.ldx, p.F, lane, p.vec4 != 0);
    }
    double acc[NACC];   // fp64 accumulation (R23)
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    uint64_t h = 0;
    double cur = 0.0;     // running sum of the current class (per-class scalar trees)
    uint32_t curk = 0;

    for (int c = 0; c < nchunks; ++c, ring.next()) {
      const int s = ring.s;
      dev::mbar_wait(&full[s], ring.ph);
      if (active) {
        const uint32_t cb = stage0 + (uint32_t)(s * ch) * p.stride;
        const int nt = min(ch, p.n_trees_pad - c * ch);
        for (int j = 0; j < nt; j += G) {
          // a = absolute address of heap node i (tree + 8 i); next level:
          // a' = tree + 16 i + (pr ? 0 : 8) = 2 a + (pr ? -tree : 8 - tree)
          uint32_t tb[G], a[G], m0[G], m8[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            tb[g] = cb + (uint32_t)(j + g) * p.stride;
            a[g] = tb[g] + 8u;              // heap node 1 (the root), 8-B records
            m0[g] = 0u - tb[g];
            m8[g] = 8u - tb[g];
          }
          // Alg. 3: T_I <- 2 T_I + (X[r, N'_F[T_I]] < N'_T[T_I] ? 0 : 1), D times
#pragma unroll
          for (int l = 0; l < D; ++l) {
            uint2 nd[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
              HB_DCHECK(a[g] - tb[g] >= (8u << l) && a[g] - tb[g] < (16u << l));   // heap node of level l
              nd[g] = dev::lds_v2(a[g]);
            }
            float x[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
              HB_DCHECK(nd[g].x < (uint32_t)p.F);                                  // column of the X slice
              x[g] = dev::lds_f32(xlane + (nd[g].x << 7));
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const float t = __uint_as_float(nd[g].y);
              const bool pr = LE ? (x[g] <= t) : (x[g] < t);
              a[g] = 2u * a[g] + (pr ? m0[g] : m8[g]);
            }
          }
          uint32_t off[G];
#pragma unroll
          for (int g = 0; g < G; ++g) off[g] = a[g] - tb[g];
          // R <- N'_C[T_I - 2^D]
          double vsum = 0.0;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t slot = (off[g] >> 3) - (1u << D);
            if (p.w == 1) {
              const double v = (double)dev::lds_f32(tb[g] + leaf_off + (off[g] >> 1));
              if (NACC == 1) acc[0] += v;
              else vsum += v;
            } else {
              const uint32_t lb = tb[g] + (8u << D) + 4u * slot * (uint32_t)p.w;
#pragma unroll
              for (int k = 0; k < NACC; ++k)
                if (k < p.K) acc[k] += (double)dev::lds_f32(lb + 4u * k);
            }
          }
          if (NACC > 1 && p.w == 1) {
            // per-class records are ordered by class (hb_host.cpp ptt_order,
            // whole groups of G): sum into one running accumulator and move
            // it to acc[class] only when the class changes (K times per
            // tile; the branch is warp-uniform, every lane reads the record)
            const uint32_t k0 = dev::lds_u32(tb[0]) & 0xFFu;
            if (k0 != curk) {
#pragma unroll
              for (int k = 0; k < NACC; ++k)
                if (curk == (uint32_t)k) acc[k] += cur;
              cur = 0.0;
              curk = k0;
            }
            cur += vsum;
          }
          if (lm) {
            // record header: tree_output | (local tree id + 1) << 8 (0: padding)
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const int orig = (int)(dev::lds_u32(tb[g]) >> 8) - 1;
              if (orig < 0) continue;
              const uint32_t slot = (off[g] >> 3) - (1u << D);
              const int32_t id = __ldg(p.leafmap + (size_t)(c * ch + j + g) * p.nslots + slot);
              if (lm == 1) {
                if (row < p.n) static_cast<int32_t *>(p.out)[row * p.n_trees + orig] = id;
              } else {
                h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + orig) << 32) | (uint32_t)id);
              }
            }
          }
        }
      }
      dev::release_stage(&empty[s], lane);
    }
    if (NACC > 1 && p.w == 1) {
#pragma unroll
      for (int k = 0; k < NACC; ++k)
        if (curk == (uint32_t)k) acc[k] += cur;
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

using PttFn = void (*)(const PttParams);

template <int D, bool LE>
static PttFn pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return ptt_kernel<D, LE, 1, kTreeGroup>;
    case 4: return ptt_kernel<D, LE, 4, kTreeGroup>;
    case 8: return ptt_kernel<D, LE, 8, kTreeGroup>;
    default: return ptt_kernel<D, LE, 16, kTreeGroup>;
  }
}

template <int D>
static PttFn pick_le(bool le, int nacc) {
  return le ? pick_nacc<D, true>(nacc) : pick_nacc<D, false>(nacc);
}

static PttFn pick(int D, bool le, int nacc) {
  switch (D) {
    case 0: return pick_le<0>(le, nacc);
    case 1: return pick_le<1>(le, nacc);
    case 2: return pick_le<2>(le, nacc);
    case 3: return pick_le<3>(le, nacc);
    case 4: return pick_le<4>(le, nacc);
    case 5: return pick_le<5>(le, nacc);
    case 6: return pick_le<6>(le, nacc);
    case 7: return pick_le<7>(le, nacc);
    case 8: return pick_le<8>(le, nacc);
    case 9: return pick_le<9>(le, nacc);
    case 10: return pick_le<10>(le, nacc);
    default: return nullptr;
  }
}

int sm_count(int device);

hb_status launch_ptt(const Model &m, const RunArgs &a) {
  PttFn fn = pick(m.depth, m.cmp == HB_CMP_LE, m.nacc);
  if (!fn) return fail(HB_E_UNSUPPORTED, "PTT depth out of range");
  PttParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.F = m.n_xf;
  p.fmap = m.d_fmap;
  p.vec4 = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);
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
  p.prefetch = m.cfg.prefetch;
  p.nw = m.cfg.nw;
  p.ns = m.cfg.ns;
  p.ch = m.cfg.ch;
  const int64_t rows_per_tile = (int64_t)m.cfg.nw * 32;
  const int64_t ntiles = (a.n + rows_per_tile - 1) / rows_per_tile;
  if (ntiles > INT32_MAX) return fail(HB_E_UNSUPPORTED, "too many rows for one launch");
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count(m.device) * m.cfg.ctas_per_sm);
  p.interleave = !(std::getenv("HB_PTTR_INTERLEAVE") && std::atoi(std::getenv("HB_PTTR_INTERLEAVE")) == 0);
  if (p.interleave) {
    const int64_t units = (a.n + 31) / 32;
    p.ntiles = (int)((units + (int64_t)grid * m.cfg.nw - 1) / ((int64_t)grid * m.cfg.nw));
  } else {
    p.ntiles = (int)ntiles;
  }
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       m.cfg.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(ptt)");
  fn<<<grid, 32 * (m.cfg.nw + 1), m.cfg.smem_bytes, a.stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "ptt_kernel launch");
  return HB_OK;
}

}  // namespace hb
