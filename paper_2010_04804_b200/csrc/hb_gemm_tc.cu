// hb_gemm_tc.cu — GEMM strategy on the 5th-generation tensor cores (tcgen05).
//
// PAPER.md Alg. 1, Table 3, batched over trees:
//   T <- X.A ; T <- T < B ; S <- T.C ; T <- S == D ; R <- T.E
// Only the path contraction S = T.C runs on the tensor cores; the node
// evaluation gathers X[r, feature] and compares in fp32 (reading R3: a dense
// X.A would be poisoned by Inf/NaN and a tf32/bf16 product would flip
// compares), and R = T.E is a gather of the single selected leaf.
//
// Exactness: T in {0,1} and C in {-1,0,+1} are exact in bf16; |S| <= 8 is exact
// in the fp32 TMEM accumulator. So S == D is decided on exact integers and the
// selected leaf is bit-identical to the walk (tests: exhaustive 2^7 patterns).
//
// Tiling: one CTA = 4 warps = 128 rows = UMMA M (TMEM lane =
// row). Trees with |I| <= 8 and |L| <= 8 (D <= 3, the depths AUTO sends here)
// are taken in PAIRS: one kind::f16 UMMA of shape M128 x N16 x K16 evaluates
// the block-diagonal [C_a 0; 0 C_b] for two trees at once. A group of 8 pairs
// (16 trees) occupies a 128 x 128 bf16 A tile (8 K-slabs of 4 KB, canonical
// K-major core-matrix layout, no swizzle) and 128 TMEM columns. Per group:
//   1. every thread evaluates its row's 16 x 8 node predicates -> bf16 bits
//      into the A tile (16-B stores, one core-matrix row each),
//   2. fence.proxy.async + barrier; one thread issues 8 tcgen05.mma and a
//      tcgen05.commit to an mbarrier,
//   3. every warp tcgen05.ld's its 32 lanes x 16 columns per pair, compares
//      with D, gathers E and accumulates.
// Group records (the B images, thresholds, features, D, E) are pre-built on
// the host in their exact SMEM image and double-buffered with cp.async.bulk.
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "hb_device.cuh"
#include "hb_internal.h"
#include "hb_layouts.h"

namespace hb {

// ------------------------------------------------------------------ device
namespace tc {

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SM100 shared-memory matrix descriptor: start>>4 [0,14), LBO>>4 [16,30),
  // SBO>>4 [32,46), version = 1 [46,48), base offset 0, layout SWIZZLE_NONE (0).
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// kind::f16 instruction descriptor: A = B = bf16, D = f32, both K-major,
// N = 16 (n_dim = N >> 3), M = 128 (m_dim = M >> 4).
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(0)
      : "memory");
}

__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   dev::smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace tc

struct TcParams {
  const float *X;
  int64_t n, ldx;
  int F, vec4, x_smem;
  const int32_t *fmap;   // compact X column -> original feature, or null
  const uint8_t *groups;
  uint32_t stride, off_feat, off_thr, off_d, off_tout, off_e;
  int ngroups, n_trees, tree_begin;
  const int32_t *leafmap;
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
  int ntiles;
  int prefetch;          // L2 prefetch of the CTA's next X row tile
  uint32_t a_region;     // bytes of the A-tile region (also the tile-end reduction scratch)
};

constexpr int kTcThreads = 512;   // 4 row quarters x 4 tree quarters
constexpr int kTcStages = 3;      // group-record ring: epilogue(i-1), MMA(i), landing(i+1)

// Software pipeline per CTA: iteration i builds the A tile
// of group i (node predicates, CUDA cores), issues its 8 UMMAs into TMEM
// buffer i & 1 (tensor cores, asynchronous), then runs the epilogue of group
// i - 1 from the other TMEM buffer while the tensor cores work. Records come
// through a 3-stage cp.async.bulk ring (record i - 1: D / E of the epilogue,
// i: B operand of the MMA, i + 1: landing). Thread (row, part): row = tid %
// 128 (TMEM lane), part = tid / 128 owns trees 4 part .. 4 part + 3 of every
// group in the A build and pairs 2 part, 2 part + 1 in the epilogue; the 4
// parts' per-row sums are combined in SMEM in a fixed order at the tile end.
template <bool LE, int NACC>
__global__ void __launch_bounds__(kTcThreads, 1) gemm_tc_kernel(const TcParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = tid & (kTcRows - 1), part = tid >> 7, quarter = r >> 5;
  const size_t xbytes = p.x_smem ? (size_t)4 * p.F * 128 : 0;     // xs[quarter][F][32]
  uint8_t *atiles = smem + xbytes;                                 // 2 x kTcPairs x 4 KB
  uint8_t *recbuf = atiles + p.a_region;                           // kTcStages x stride
  uint64_t *bars = reinterpret_cast<uint64_t *>(recbuf + (size_t)kTcStages * p.stride);
  uint64_t *rec_full = bars;                // [kTcStages] group record landed
  uint64_t *mma_done = bars + kTcStages;    // [2] MMA of TMEM buffer b finished
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + kTcStages + 2);
  double *red = reinterpret_cast<double *>(atiles);                // tile-end reduction (aliases A)
  uint64_t *hred = reinterpret_cast<uint64_t *>(atiles + (size_t)4 * kTcRows * NACC * 8);

  if (tid == 0) {
    for (int i = 0; i < kTcStages; ++i) dev::mbar_init(&rec_full[i], 1);
    dev::mbar_init(&mma_done[0], 1);
    dev::mbar_init(&mma_done[1], 1);
    dev::fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     dev::smem_u32(tmem_slot)),
                 "n"(2 * kTcCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  float *xs = reinterpret_cast<float *>(smem) + (size_t)quarter * p.F * 32;
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  const uint32_t a_base = dev::smem_u32(atiles);
  const int my_tiles = (p.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const uint32_t total = (uint32_t)my_tiles * p.ngroups;
  // record ring: item `it` (global over this CTA's tiles x groups) in stage it % 3
  auto issue_rec = [&](uint32_t it) {
    if (it < total) {
      const int st = (int)(it % kTcStages);
      const int gi = (int)(it % (uint32_t)p.ngroups);
      dev::mbar_arrive_expect_tx(&rec_full[st], p.stride);
      dev::bulk_g2s(recbuf + (size_t)st * p.stride, p.groups + (size_t)gi * p.stride, p.stride,
                    &rec_full[st]);
    }
  };
  if (tid == 0) issue_rec(0);
  uint32_t it = 0;          // record / MMA item counter
  uint32_t mma_ph[2] = {0u, 0u};

  for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const int64_t row0 = (int64_t)tile * kTcRows;
    const int64_t row = row0 + r;
    // ---- X slice of this tile: quarter q of the rows, features split over the 4 parts
    const float *xrow;
    int xstride;
    if (p.x_smem) {
      const float *xr = p.X + (row < p.n ? row : 0) * p.ldx;
      if (p.vec4 && !p.fmap) {
        // this thread's 16-B chunks j = part, part + 4, ...: 4 loads in flight
        // before their stores (one memory latency per 4 chunks)
        const int F4 = p.F >> 2;
        int j = part;
        for (; j + 12 < F4; j += 16) {
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            v[u] = row < p.n ? __ldg(reinterpret_cast<const float4 *>(xr + 4 * (j + 4 * u)))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int f = 4 * (j + 4 * u);
            xs[(f + 0) * 32 + lane] = v[u].x;
            xs[(f + 1) * 32 + lane] = v[u].y;
            xs[(f + 2) * 32 + lane] = v[u].z;
            xs[(f + 3) * 32 + lane] = v[u].w;
          }
        }
        for (; 4 * j < p.F; j += 4) {
          const int f = 4 * j;
          if (f + 4 <= p.F) {
            const float4 v = row < p.n ? __ldg(reinterpret_cast<const float4 *>(xr + f))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
            xs[(f + 0) * 32 + lane] = v.x;
            xs[(f + 1) * 32 + lane] = v.y;
            xs[(f + 2) * 32 + lane] = v.z;
            xs[(f + 3) * 32 + lane] = v.w;
          } else {
            for (int c = f; c < p.F; ++c) xs[c * 32 + lane] = row < p.n ? __ldg(xr + c) : 0.f;
          }
        }
      } else {
        for (int c = part; c < p.F; c += 4)
          xs[c * 32 + lane] = row < p.n ? __ldg(xr + (p.fmap ? __ldg(p.fmap + c) : c)) : 0.f;
      }
      if (tid == 0 && p.prefetch)
        dev::prefetch_rows_l2(p.X, (int64_t)(tile + gridDim.x) * kTcRows, kTcRows, p.n, p.ldx);
      xrow = xs + lane;
      xstride = 32;
      __syncthreads();   // the 4 parts filled different columns of each row's slice
    } else {
      xrow = p.X + (row < p.n ? row : 0) * p.ldx;
      xstride = 1;
    }
    double acc[NACC];   // fp64 accumulation (R23)
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    uint64_t h = 0;
    // previous group's item (its epilogue runs in the next iteration)
    uint32_t prev_it = 0;
    int prev_gi = -1;

    // epilogue of group gi (item pit): T <- S == D ; R <- T.E for this
    // thread's pairs 2 part, 2 part + 1 (16 TMEM columns each)
    auto epilogue = [&](uint32_t pit, int gi) {
      const int b = (int)(pit & 1u);
      dev::mbar_wait(&mma_done[b], mma_ph[b]);
      mma_ph[b] ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint8_t *rec = recbuf + (size_t)(pit % kTcStages) * p.stride;
      const float *dval = reinterpret_cast<const float *>(rec + p.off_d);
      const uint32_t *tout = reinterpret_cast<const uint32_t *>(rec + p.off_tout);
      const float *E = reinterpret_cast<const float *>(rec + p.off_e);
#pragma unroll
      for (int sp = 0; sp < 2; ++sp) {
        const int s = 2 * part + sp;
        float S[16];
        tc::ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * kTcCols + s * 16), S);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int q = 2 * s + hh;
          int sel = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (S[hh * 8 + j] == dval[q * 8 + j]) sel = j;
          if (p.w == 1) {
            const double v = (double)E[q * 8 + sel];
            if (NACC == 1) {
              acc[0] += v;
            } else {
              const uint32_t k0 = tout[q];
#pragma unroll
              for (int k = 0; k < NACC; ++k)
                if (k0 == (uint32_t)k) acc[k] += v;
            }
          } else {
#pragma unroll
            for (int k = 0; k < NACC; ++k)
              if (k < p.K) acc[k] += (double)E[(q * 8 + sel) * p.w + k];
          }
          if (lm) {
            const int t = gi * kTcTrees + q;
            if (t < p.n_trees) {
              const int32_t id = __ldg(p.leafmap + (size_t)t * 8 + sel);
              if (lm == 1) {
                if (row < p.n) static_cast<int32_t *>(p.out)[row * p.n_trees + t] = id;
              } else {
                h += dev::mix64(((uint64_t)(uint32_t)(p.tree_begin + t) << 32) | (uint32_t)id);
              }
            }
          }
        }
      }
    };

    for (int gi = 0; gi < p.ngroups; ++gi, ++it) {
      const int st = (int)(it % kTcStages);
      const int b = (int)(it & 1u);
      dev::mbar_wait(&rec_full[st], (it / kTcStages) & 1u);
      const uint8_t *rec = recbuf + (size_t)st * p.stride;
      const uint32_t *feat = reinterpret_cast<const uint32_t *>(rec + p.off_feat);
      const float *thr = reinterpret_cast<const float *>(rec + p.off_thr);
      // 1. T <- (X.A < B) for this thread's 4 trees -> bf16 {0,1} into A
      //    tile b. Pair s is K-slab s: row r, k-chunk c (= tree 2s + c) at
      //    s * 4096 + (r >> 3) * 256 + c * 128 + (r & 7) * 16.
      uint8_t *atile = atiles + (size_t)b * kTcPairs * 4096;
#pragma unroll
      for (int qq = 0; qq < 4; ++qq) {
        const int q = 4 * part + qq;
        uint32_t bits[4];
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          uint32_t v = 0;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int i = i2 * 2 + hh;
            const float x = xrow[feat[q * 8 + i] * xstride];
            const float t = thr[q * 8 + i];
            const bool pr = LE ? (x <= t) : (x < t);
            v |= (pr ? 0x3F80u : 0u) << (16 * hh);
          }
          bits[i2] = v;
        }
        uint8_t *dst = atile + (size_t)(q >> 1) * 4096 + (r >> 3) * 256 + (q & 1) * 128 + (r & 7) * 16;
        *reinterpret_cast<uint4 *>(dst) = make_uint4(bits[0], bits[1], bits[2], bits[3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();   // A tile b built; epilogue(i - 2) done with TMEM buffer b and record i - 2
      asm volatile("tcgen05.fence::after_thread_sync;");
      // 2. S <- T.C on the tensor cores (asynchronous): one M128 x N16 x K16
      //    UMMA per pair into TMEM buffer b; then refill the ring stage that
      //    held record i - 2 with record i + 1
      if (tid == 0) {
        const uint32_t b_base = dev::smem_u32(rec);
        const uint32_t ab = a_base + (uint32_t)b * kTcPairs * 4096u;
#pragma unroll
        for (int s = 0; s < kTcPairs; ++s) {
          const uint64_t ad = tc::smem_desc(ab + s * 4096, 128, 256);
          const uint64_t bd = tc::smem_desc(b_base + s * 512, 128, 256);
          tc::mma_bf16(tmem + (uint32_t)(b * kTcCols + s * 16), ad, bd);
        }
        tc::commit(&mma_done[b]);
        issue_rec(it + 1);
      }
      // 3. epilogue of the previous group while the tensor cores work
      if (prev_gi >= 0) epilogue(prev_it, prev_gi);
      prev_it = it;
      prev_gi = gi;
    }
    // drain: the last group's epilogue
    if (prev_gi >= 0) epilogue(prev_it, prev_gi);
    // ---- combine the 4 parts of every row in a fixed order
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();   // every A tile consumed (all MMAs waited): reuse it for the reduction
    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
    for (int k = 0; k < NACC; ++k) red[((size_t)part * kTcRows + r) * NACC + k] = acc[k];
    hred[part * kTcRows + r] = h;
    __syncthreads();
    if (part == 0) {
#pragma unroll
      for (int k = 0; k < NACC; ++k) {
        double t = 0.0;
        for (int q = 0; q < 4; ++q) t += red[((size_t)q * kTcRows + r) * NACC + k];
        acc[k] = t;
      }
      uint64_t ht = 0;
      for (int q = 0; q < 4; ++q) ht += hred[q * kTcRows + r];
      if (row < p.n) {
        if (lm == 2) static_cast<uint64_t *>(p.out)[row] = ht;
        else if (lm == 0) dev::write_row<NACC>(p.kind, acc, p.K, p.task, p.post, p.scale, p.base, row, p.out);
      }
    }
    __syncthreads();   // reduction scratch and X slice free for the next tile
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * kTcCols));
}

using TcFn = void (*)(const TcParams);

template <bool LE>
static TcFn pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return gemm_tc_kernel<LE, 1>;
    case 4: return gemm_tc_kernel<LE, 4>;
    case 8: return gemm_tc_kernel<LE, 8>;
    default: return gemm_tc_kernel<LE, 16>;
  }
}

int sm_count(int device);

hb_status launch_gemm_tc(const Model &m, const RunArgs &a) {
  const TcGeom g = tc_geom(m.leaf_width);
  TcParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.vec4 = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);
  p.x_smem = m.cfg.x_smem;
  p.F = m.n_xf;
  p.fmap = m.d_fmap;
  p.groups = static_cast<const uint8_t *>(m.d_trees);
  p.stride = (uint32_t)g.stride;
  p.off_feat = (uint32_t)g.off_feat;
  p.off_thr = (uint32_t)g.off_thr;
  p.off_d = (uint32_t)g.off_d;
  p.off_tout = (uint32_t)g.off_tout;
  p.off_e = (uint32_t)g.off_e;
  p.ngroups = m.n_trees_pad / kTcTrees;
  p.n_trees = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.leafmap = m.d_leafmap;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  const int64_t ntiles = (a.n + kTcRows - 1) / kTcRows;
  if (ntiles > INT32_MAX) return fail(HB_E_UNSUPPORTED, "too many rows");
  p.ntiles = (int)ntiles;
  p.prefetch = m.cfg.prefetch;
  p.a_region = (uint32_t)gemm_tc_a_region(m.nacc);
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count(m.device) * m.cfg.ctas_per_sm);
  TcFn fn = m.cmp == HB_CMP_LE ? pick_nacc<true>(m.nacc) : pick_nacc<false>(m.nacc);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       m.cfg.smem_bytes);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(gemm_tc)");
  fn<<<grid, kTcThreads, m.cfg.smem_bytes, a.stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "gemm_tc_kernel launch");
  return HB_OK;
}

}  // namespace hb
