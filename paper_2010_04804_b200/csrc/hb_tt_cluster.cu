// hb_tt_cluster.cu — TreeTraversal for very large ensembles on wide rows
// (C5-shaped: thousands of depth-12 trees, 2000 features), as a 4-CTA
// thread-block cluster.
//
// The wide-row TT kernel is bound by L2 latency: every row tile walks every
// tree and even the top levels miss L1. Here the trees are split over the 4
// CTAs of a cluster; each CTA keeps the TOP levels (TOPD) of its trees in SMEM
// for the whole launch, in perfect-tree form (PAPER.md P:243 padding, heap
// order — the PTT layout of Alg. 3 for the top of the tree), followed by an
// exit table mapping each top-leaf slot to the TT node (Table 5 layout, BFS,
// self-looping leaves) where the walk continues in L2 (Alg. 2) if the path is
// deeper. All 4 CTAs score the same R rows: the X tile is fetched ONCE per
// cluster with multicast bulk copies (cp.async.bulk ... .multicast::cluster,
// each CTA issuing a quarter of the rows), and the per-row partial sums of the
// 4 CTAs are combined through distributed shared memory in a fixed order
// (deterministic), then the leader CTA runs the fused epilogue.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "hb_device.cuh"
#include "hb_internal.h"

namespace hb {

constexpr int kCs = 4;            // CTAs per cluster = tree groups
constexpr int kCR = 16;           // rows per tile
constexpr int kCW = 32;           // warps per CTA

struct TcParams2 {
  const float *X;
  int64_t n, ldx;
  int F, depth, topd;
  const uint8_t *trees;           // TT records
  uint32_t stride;
  int nslots, n_trees, tree_begin;
  const uint8_t *tops;            // [kCs][per_cta][top_bytes] by cluster rank
  int per_cta;                    // trees per CTA slot range (padded)
  uint32_t top_bytes;
  const int32_t *leafmap;
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
  int ntiles;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

__device__ __forceinline__ void st_cluster_u64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}

__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                            uint16_t mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "h"(mask)
      : "memory");
}

template <bool LE, int NACC>
__global__ void __launch_bounds__(32 * kCW, 1)
    tt_cluster_kernel(const TcParams2 p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t q = cluster_rank();
  const int sub = lane / kCR, r = lane % kCR;   // 2 tree slots x 16 rows per warp
  constexpr int kSlots = 32 / kCR;
  constexpr int kG = 4;                          // trees in flight per lane
  // SMEM: xs [kCR][F] row-major (multicast target) | tops | red | part[2][kCs][kCR] | bars
  const size_t xbytes = ((size_t)kCR * p.F * 4 + 127) & ~size_t(127);
  float *xs = reinterpret_cast<float *>(smem);
  uint8_t *tops = smem + xbytes;
  const size_t tbytes = ((size_t)p.per_cta * p.top_bytes + 127) & ~size_t(127);
  float *red = reinterpret_cast<float *>(tops + tbytes);                 // [kCW][kCR][NACC]
  uint64_t *hred = reinterpret_cast<uint64_t *>(red + kCW * kCR * NACC);  // [kCW][kCR]
  float *part = reinterpret_cast<float *>(hred + kCW * kCR);              // [2][kCs][kCR][NACC]
  uint64_t *hpart = reinterpret_cast<uint64_t *>(part + 2 * kCs * kCR * NACC);  // [2][kCs][kCR]
  uint64_t *bars = hpart + 2 * kCs * kCR;                                  // [0] tops, [1] X
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);

  // this CTA's trees: local tree ids q, q + kCs, q + 2 kCs, ...
  const int my_trees = p.n_trees > (int)q ? (p.n_trees - (int)q + kCs - 1) / kCs : 0;
  if (threadIdx.x == 0) {
    dev::mbar_init(&bars[0], 1);
    dev::mbar_init(&bars[1], 1);
    dev::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)my_trees * p.top_bytes;
    dev::mbar_arrive_expect_tx(&bars[0], bytes);
    if (bytes) dev::bulk_g2s(tops, p.tops + (size_t)q * p.per_cta * p.top_bytes, bytes, &bars[0]);
  }
  const int tile0 = (int)cluster_id_x();
  auto tile_rows = [&](int tile) -> int {
    if (tile >= p.ntiles) return 0;
    const int64_t left = p.n - (int64_t)tile * kCR;
    return left < kCR ? (int)left : kCR;
  };
  if (threadIdx.x == 0 && tile0 < p.ntiles)   // arm the X barrier before anyone multicasts
    dev::mbar_arrive_expect_tx(&bars[1], (uint32_t)tile_rows(tile0) * p.F * 4u);
  cluster_sync();   // every CTA's barriers are initialised and armed before multicasts target them
  dev::mbar_wait(&bars[0], 0);

  const uint32_t xs_s = dev::smem_u32(xs);
  const uint32_t xbar_s = dev::smem_u32(&bars[1]);
  const int topn = 1 << p.topd;
  uint32_t xphase = 0;
  int it = 0;
  for (int tile = (int)cluster_id_x(); tile < p.ntiles; tile += (int)nclusters_x(), ++it) {
    const int64_t row0 = (int64_t)tile * kCR;
    const int rows = tile_rows(tile);
    if (threadIdx.x == 32 && q == 0)   // warm L2 with the cluster's next tile of X rows
      dev::prefetch_rows_l2(p.X, (int64_t)(tile + (int)nclusters_x()) * kCR, kCR, p.n, p.ldx);
    // ---- X tile: one multicast bulk copy per row, rows split over the 4 CTAs
    if (threadIdx.x == 0) {
      for (int rr = (int)q; rr < rows; rr += kCs)
        bulk_g2s_mc(xs_s + (uint32_t)(rr * p.F * 4), p.X + (row0 + rr) * p.ldx, (uint32_t)p.F * 4u,
                    xbar_s, (uint16_t)((1u << kCs) - 1));
    }
    dev::mbar_wait(&bars[1], xphase);
    xphase ^= 1u;
    const int64_t row = row0 + r;
    const float *xr = xs + (size_t)r * p.F;
    float acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.f;
    uint64_t h = 0;
    // two trees per lane in flight; the loop bound is warp-uniform
    for (int base = warp * kSlots; base < my_trees; base += kG * kSlots * kCW) {
      int jj[kG];
      bool val[kG];
      uint32_t i[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        jj[g] = base + sub + g * kSlots * kCW;
        val[g] = jj[g] < my_trees;
        i[g] = 1;
      }
      // top levels from SMEM (perfect heap, 8-B {feature, thr}; slot 0 = {class})
#pragma unroll 1
      for (int l = 0; l < p.topd; ++l) {
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          const uint32_t tb = dev::smem_u32(tops) + (uint32_t)(val[g] ? jj[g] : 0) * p.top_bytes;
          const uint2 nd = dev::lds_v2(tb + 8u * i[g]);
          const float x = xr[nd.x];
          const float t = __uint_as_float(nd.y);
          const bool pr = LE ? (x <= t) : (x < t);
          i[g] = 2u * i[g] + (pr ? 0u : 1u);
        }
      }
      // exit slot -> TT node id (bit 31: the walk already reached a leaf)
      uint32_t node[kG];
      bool done[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const uint32_t tb = dev::smem_u32(tops) + (uint32_t)(val[g] ? jj[g] : 0) * p.top_bytes;
        const uint32_t ex = dev::lds_u32(tb + 8u * (uint32_t)topn + 4u * (i[g] - (uint32_t)topn));
        node[g] = ex & 0x7FFFFFFFu;
        done[g] = (ex >> 31) != 0u;
      }
      // deep levels through L2 (Alg. 2 with self-loops, early exit)
      const uint2 *nd2[kG];
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        const int tl = (int)q + kCs * (val[g] ? jj[g] : 0);
        nd2[g] = reinterpret_cast<const uint2 *>(p.trees + (size_t)tl * p.stride + 16);
      }
      for (int l = p.topd; l < p.depth; ++l) {
        bool all_done = true;
#pragma unroll
        for (int g = 0; g < kG; ++g) all_done = all_done && done[g];
        if (__all_sync(0xFFFFFFFFu, all_done)) break;
#pragma unroll
        for (int g = 0; g < kG; ++g) {
          if (done[g]) continue;
          const uint2 d = __ldg(nd2[g] + node[g]);
          const float x = xr[d.x & 0xFFFFu];
          const float t = __uint_as_float(d.y);
          const bool pr = LE ? (x <= t) : (x < t);
          const uint32_t nx = (d.x >> 16) - (pr ? 1u : 0u);
          done[g] = nx == node[g];
          node[g] = nx;
        }
      }
#pragma unroll
      for (int g = 0; g < kG; ++g) {
        if (!val[g]) continue;
        const int tl = (int)q + kCs * jj[g];
        const float *lv = reinterpret_cast<const float *>(nd2[g] + p.nslots);
        if (p.w == 1) {
          const float v = __ldg(lv + node[g]);
          if (NACC == 1) {
            acc[0] += v;
          } else {
            const uint32_t k0 = dev::lds_u32(dev::smem_u32(tops) + (uint32_t)jj[g] * p.top_bytes);
#pragma unroll
            for (int k = 0; k < NACC; ++k)
              if (k0 == (uint32_t)k) acc[k] += v;
          }
        } else {
#pragma unroll
          for (int k = 0; k < NACC; ++k)
            if (k < p.K) acc[k] += __ldg(lv + node[g] * p.w + k);
        }
        if (lm) {
          const int32_t id = __ldg(p.leafmap + (size_t)tl * p.nslots + node[g]);
          if (lm == 1) {
            if (row < p.n) static_cast<int32_t *>(p.out)[row * p.n_trees + tl] = id;
          } else {
            h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + tl) << 32) | (uint32_t)id);
          }
        }
      }
    }
    // ---- reduce: 4 tree slots of a row (shuffles), 32 warps (SMEM), 4 CTAs (DSMEM)
#pragma unroll
    for (int o = kCR; o < 32; o <<= 1) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] += __shfl_xor_sync(0xFFFFFFFFu, acc[k], o);
      h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
    }
    if (sub == 0) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) red[(warp * kCR + r) * NACC + k] = acc[k];
      hred[warp * kCR + r] = h;
    }
    __syncthreads();
    const int pb = it & 1;   // partial buffers alternate by tile parity
    if (warp == 0 && lane < kCR) {
      float tot[NACC];
#pragma unroll
      for (int k = 0; k < NACC; ++k) tot[k] = 0.f;
      uint64_t ht = 0;
      for (int w2 = 0; w2 < kCW; ++w2) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) tot[k] += red[(w2 * kCR + lane) * NACC + k];
        ht += hred[w2 * kCR + lane];
      }
      const uint32_t pa = dev::smem_u32(part + ((pb * kCs + (int)q) * kCR + lane) * NACC);
      const uint32_t ha = dev::smem_u32(hpart + (pb * kCs + (int)q) * kCR + lane);
#pragma unroll
      for (int k = 0; k < NACC; ++k) st_cluster_f32(map_to_rank(pa + 4u * k, 0), tot[k]);
      st_cluster_u64(map_to_rank(ha, 0), ht);
    }
    if (threadIdx.x == 0) {       // arm the next tile's X barrier before the sync
      const int nt = tile + (int)nclusters_x();
      if (nt < p.ntiles) dev::mbar_arrive_expect_tx(&bars[1], (uint32_t)tile_rows(nt) * p.F * 4u);
    }
    cluster_sync();   // partials landed in the leader; every CTA is done with xs
    if (q == 0 && warp == 0 && lane < kCR) {
      const int64_t orow = row0 + lane;
      float tot[NACC];
#pragma unroll
      for (int k = 0; k < NACC; ++k) tot[k] = 0.f;
      uint64_t ht = 0;
      for (int c = 0; c < kCs; ++c) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) tot[k] += part[((pb * kCs + c) * kCR + lane) * NACC + k];
        ht += hpart[(pb * kCs + c) * kCR + lane];
      }
      if (orow < p.n) {
        if (lm == 2) static_cast<uint64_t *>(p.out)[orow] = ht;
        else if (lm == 0) dev::write_row<NACC>(p.kind, tot, p.K, p.task, p.post, p.scale, p.base, orow, p.out);
      }
    }
  }
  cluster_sync();   // no CTA exits while others may still multicast into it
}

// --------------------------------------------------------------- host side
// Top-region layout per tree (top_bytes = 12 * 2^TOPD, 16-B aligned):
//   uint2 node[2^TOPD]: node[0] = {class, 0}; node[p] = {feature, thr} for heap
//   p in [1, 2^TOPD) (perfect padding: feature 0, +Inf, both children map to
//   the same TT node); then u32 exit[2^TOPD]: TT node id | (leaf ? 1 << 31 : 0).
hb_status compile_tt_cluster(const hb_ensemble *e, int t0, int t1, Model *m, const int32_t *fremap,
                             const std::vector<uint8_t> &tt_trees) {
  const int T = t1 - t0;
  const int per_cta = (T + kCs - 1) / kCs;
  const long xbytes = ((long)kCR * m->n_xf * 4 + 127) & ~127L;
  const long fixed = xbytes + (long)kCW * kCR * (4L * m->nacc + 8) + 2L * kCs * kCR * (4L * m->nacc + 8) + 64;
  int topd = 0;
  for (int d = std::min(m->depth, 6); d >= 2; --d) {
    const long tb = 12L << d;
    if (fixed + (((long)per_cta * tb + 127) & ~127L) <= kSmemBudget) {
      topd = d;
      break;
    }
  }
  if (topd == 0 || (m->n_xf * 4) % 16 != 0) return HB_E_UNSUPPORTED;
  const int P = 1 << topd;
  const uint32_t top_bytes = (uint32_t)(12 * P);
  std::vector<uint8_t> tops((size_t)kCs * per_cta * top_bytes, 0);
  std::vector<int> cur(2 * P);
  const size_t stride = m->stride;
  for (int lt = 0; lt < T; ++lt) {
    const int q = lt % kCs, j = lt / kCs;
    uint8_t *rec = tops.data() + ((size_t)q * per_cta + j) * top_bytes;
    uint32_t *node = reinterpret_cast<uint32_t *>(rec);
    uint32_t *exits = reinterpret_cast<uint32_t *>(rec + 8 * P);
    // the TT record of this tree: BFS nodes {f | R << 16, thr}; leaf: R == self
    const uint32_t *tn = reinterpret_cast<const uint32_t *>(tt_trees.data() + (size_t)lt * stride + 16);
    node[0] = *reinterpret_cast<const uint32_t *>(tt_trees.data() + (size_t)lt * stride);
    cur[1] = 0;
    for (int p = 1; p < P; ++p) {
      const int o = cur[p];
      const uint32_t a = tn[2 * o];
      const bool leaf = (int)(a >> 16) == o;
      if (!leaf) {
        node[2 * p] = a & 0xFFFFu;
        node[2 * p + 1] = tn[2 * o + 1];
        cur[2 * p] = (int)(a >> 16) - 1;
        cur[2 * p + 1] = (int)(a >> 16);
      } else {
        node[2 * p] = 0;
        const float pinf = INFINITY;
        std::memcpy(&node[2 * p + 1], &pinf, 4);
        cur[2 * p] = cur[2 * p + 1] = o;
      }
    }
    for (int p = P; p < 2 * P; ++p) {
      const int o = cur[p];
      const bool leaf = (int)(tn[2 * o] >> 16) == o;
      exits[p - P] = (uint32_t)o | (leaf ? 0x80000000u : 0u);
    }
  }
  (void)fremap;
  cudaError_t err;
  if ((err = cudaMalloc(&m->d_tops, tops.size())) != cudaSuccess) return cuda_fail(err, "cudaMalloc(tops)");
  m->device_bytes += tops.size();
  if ((err = cudaMemcpy(m->d_tops, tops.data(), tops.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(err, "cudaMemcpy(tops)");
  m->cl_topd = topd;
  m->cl_per_cta = per_cta;
  m->cl_top_bytes = top_bytes;
  m->cl_smem = (int)(fixed + (((long)per_cta * top_bytes + 127) & ~127L));
  return HB_OK;
}

template <bool LE>
static void *pick_cl(int nacc) {
  switch (nacc) {
    case 1: return (void *)tt_cluster_kernel<LE, 1>;
    case 4: return (void *)tt_cluster_kernel<LE, 4>;
    case 8: return (void *)tt_cluster_kernel<LE, 8>;
    default: return (void *)tt_cluster_kernel<LE, 16>;
  }
}

int sm_count(int device);

// returns HB_E_UNSUPPORTED when this call cannot use the cluster kernel
// (unaligned X rows); the caller then runs tt_wide_kernel
hb_status launch_tt_cluster(const Model &m, const RunArgs &a) {
  if ((reinterpret_cast<uintptr_t>(a.X) & 15) != 0 || (a.ldx % 4) != 0 || m.d_fmap != nullptr)
    return HB_E_UNSUPPORTED;
  TcParams2 p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.F = m.n_features;
  p.depth = m.depth;
  p.topd = m.cl_topd;
  p.trees = static_cast<const uint8_t *>(m.d_trees);
  p.stride = (uint32_t)m.stride;
  p.nslots = m.nslots;
  p.n_trees = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.tops = static_cast<const uint8_t *>(m.d_tops);
  p.per_cta = m.cl_per_cta;
  p.top_bytes = (uint32_t)m.cl_top_bytes;
  p.leafmap = m.d_leafmap;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  const int64_t ntiles = (a.n + kCR - 1) / kCR;
  if (ntiles > INT32_MAX) return fail(HB_E_UNSUPPORTED, "too many rows");
  p.ntiles = (int)ntiles;
  const int nclusters = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, sm_count(m.device) / kCs));
  void *fn = m.cmp == HB_CMP_LE ? pick_cl<true>(m.nacc) : pick_cl<false>(m.nacc);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m.cl_smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(tt_cluster)");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nclusters * kCs);
  cfg.blockDim = dim3(32 * kCW);
  cfg.dynamicSmemBytes = m.cl_smem;
  cfg.stream = a.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void *args[] = {&p};
  e = cudaLaunchKernelExC(&cfg, fn, args);
  if (e != cudaSuccess) return cuda_fail(e, "tt_cluster_kernel launch");
  return HB_OK;
}

}  // namespace hb
