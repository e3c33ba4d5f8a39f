// hb_small.cu — small-batch / request-response scoring (
// PAPER.md Sec. 6.1.1 "request/response" P:355-362 and the batch-size study
// P:424-430, where GEMM wins at small batches on the paper's hardware).
//
// The row-per-lane scorers need ~10^5 rows to fill 148 SMs; a single row would
// be walked by one warp through all trees (hundreds of microseconds). Here the
// parallel dimension is the TREE: one CTA owns a row, its threads walk
// disjoint trees (two at a time) through L2-resident records, and a block
// reduction in a fixed order feeds the usual fused epilogue. One launch, no
// scratch. Works on the PTT fp32-node layout (D <= 10; built in addition for
// rank-coded PTT and GEMM models) and on the TT layout (deep trees).
#include <cuda_runtime.h>

#include "hb_device.cuh"
#include "hb_internal.h"

namespace hb {

struct SbParams {
  const float *X;
  int64_t n, ldx;
  const int32_t *fmap;       // compact column -> original feature, or null
  int F, depth, tt;          // tt: 1 = TT records (16-B header, self-loops), 0 = PTT fp32 records
  const uint8_t *trees;
  uint32_t stride;
  int n_rec, n_trees, tree_begin, nslots;   // n_rec: records (PTT: class-ordered + padding)
  const int32_t *leafmap;
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
};

template <bool LE>
__device__ __forceinline__ uint32_t sb_walk_ptt(const uint2 *node, const float *xs, int D) {
  uint32_t i = 1;
  for (int l = 0; l < D; ++l) {
    const uint2 nd = __ldg(node + i);
    const float x = xs[nd.x];
    const float t = __uint_as_float(nd.y);
    const bool pr = LE ? (x <= t) : (x < t);
    i = 2u * i + (pr ? 0u : 1u);
  }
  return i - (1u << D);   // leaf slot
}

template <bool LE>
__device__ __forceinline__ uint32_t sb_walk_tt(const uint2 *node, const float *xs, int D) {
  uint32_t i = 0;
  for (int l = 0; l < D; ++l) {
    const uint2 nd = __ldg(node + i);
    const float x = xs[nd.x & 0xFFFFu];
    const float t = __uint_as_float(nd.y);
    const bool pr = LE ? (x <= t) : (x < t);
    const uint32_t nx = (nd.x >> 16) - (pr ? 1u : 0u);
    if (nx == i) break;     // self-looping leaf: further iterations are no-ops
    i = nx;
  }
  return i;
}

template <bool LE, int NACC>
__global__ void __launch_bounds__(256) small_batch_kernel(const SbParams p) {
  extern __shared__ __align__(16) float sb_smem[];
  float *xs = sb_smem;                              // [F]
  double *red = reinterpret_cast<double *>(xs + ((p.F + 3) & ~3));   // [8 warps][NACC]
  uint64_t *hred = reinterpret_cast<uint64_t *>(red + 8 * NACC);     // [8]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  for (int64_t row = blockIdx.x; row < p.n; row += gridDim.x) {
    for (int f = threadIdx.x; f < p.F; f += blockDim.x)
      xs[f] = __ldg(p.X + row * p.ldx + (p.fmap ? __ldg(p.fmap + f) : f));
    __syncthreads();
    double acc[NACC];   // fp64 accumulation (R23)
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    uint64_t h = 0;
    for (int t = threadIdx.x; t < p.n_rec; t += blockDim.x) {
      const uint8_t *rec = p.trees + (size_t)t * p.stride;
      uint32_t slot;
      const float *leaf;
      const uint32_t hdr = __ldg(reinterpret_cast<const uint32_t *>(rec));
      uint32_t kout;
      int orig;
      if (p.tt) {
        slot = sb_walk_tt<LE>(reinterpret_cast<const uint2 *>(rec + 16), xs, p.depth);
        leaf = reinterpret_cast<const float *>(rec + 16 + 8 * (size_t)p.nslots);
        kout = hdr;
        orig = t;
      } else {
        // PTT header: class | (local tree id + 1) << 8, 0 = padding record
        orig = (int)(hdr >> 8) - 1;
        if (orig < 0) continue;
        slot = sb_walk_ptt<LE>(reinterpret_cast<const uint2 *>(rec), xs, p.depth);
        leaf = reinterpret_cast<const float *>(rec + (8u << p.depth));
        kout = hdr & 0xFFu;
      }
      if (p.w == 1) {
        const double v = (double)__ldg(leaf + slot);
#pragma unroll
        for (int k = 0; k < NACC; ++k)
          if (kout == (uint32_t)k) acc[k] += v;
      } else {
#pragma unroll
        for (int k = 0; k < NACC; ++k)
          if (k < p.K) acc[k] += (double)__ldg(leaf + slot * p.w + k);
      }
      if (lm) {
        const int32_t id = __ldg(p.leafmap + (size_t)t * p.nslots + slot);
        if (lm == 1) static_cast<int32_t *>(p.out)[row * p.n_trees + orig] = id;
        else h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + orig) << 32) | (uint32_t)id);
      }
    }
    // fixed-order block reduction: warp shuffles, then warp 0 over 8 warps
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) acc[k] += __shfl_xor_sync(0xFFFFFFFFu, acc[k], o);
      h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
    }
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) red[warp * NACC + k] = acc[k];
      hred[warp] = h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot[NACC];
#pragma unroll
      for (int k = 0; k < NACC; ++k) tot[k] = 0.0;
      uint64_t ht = 0;
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) tot[k] += red[w2 * NACC + k];
        ht += hred[w2];
      }
      if (lm == 2) static_cast<uint64_t *>(p.out)[row] = ht;
      else if (lm == 0) dev::write_row<NACC>(p.kind, tot, p.K, p.task, p.post, p.scale, p.base, row, p.out);
    }
    __syncthreads();
  }
}

using SbFn = void (*)(const SbParams);

template <bool LE>
static SbFn pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return small_batch_kernel<LE, 1>;
    case 4: return small_batch_kernel<LE, 4>;
    case 8: return small_batch_kernel<LE, 8>;
    default: return small_batch_kernel<LE, 16>;
  }
}

int sm_count(int device);

hb_status launch_small_batch(const Model &m, const RunArgs &a) {
  SbParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.F = m.sb_nxf;
  p.fmap = m.sb_fmap;
  p.depth = m.sb_tt ? m.depth : m.sb_depth;
  p.tt = m.sb_tt;
  p.trees = static_cast<const uint8_t *>(m.sb_trees);
  p.stride = (uint32_t)m.sb_stride;
  p.n_rec = m.sb_nrec;
  p.n_trees = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.nslots = m.sb_nslots;
  p.leafmap = m.sb_leafmap;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  const int threads = 256;
  const size_t smem = (size_t)((m.sb_nxf + 3) & ~3) * 4 + 8 * 16 * 8 + 8 * 8;
  if (smem > (size_t)kSmemBudget) return fail(HB_E_UNSUPPORTED, "small-batch path: row too wide");
  const int64_t grid = std::min<int64_t>(a.n, (int64_t)sm_count(m.device) * 16);
  SbFn fn = m.cmp == HB_CMP_LE ? pick_nacc<true>(m.nacc) : pick_nacc<false>(m.nacc);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(small_batch)");
  fn<<<(int)grid, threads, smem, a.stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "small_batch_kernel launch");
  return HB_OK;
}

}  // namespace hb
