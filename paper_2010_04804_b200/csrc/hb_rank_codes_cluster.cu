// hb_rank_codes_cluster.cu — rank-code pre-pass over a thread-block cluster
// (sm_100a): the bucket tables of all features live in the distributed shared
// memory of one cluster (<= 8 CTAs, one table group each), X is read from HBM
// once per cluster and every value is sent to the CTA that owns its feature.
//
// Same codes as hb_rank_codes.cu (Alg. 3
// walked on integer codes, reading R28): c(x) = #{j : u_j <= x} (LT; LE:
// u_j < x), NaN -> 0xFFFF, found by a bucket index and a short binary search
// whose steps run in lockstep (rank_codes_lockstep).
//
// Why a cluster: the per-group kernels read, for every table group, the
// group's columns of every row — for narrow groups (C3: 28 features of ~34 KB
// tables, one per group) that is one 32-B sector per row and group, i.e. ~8x
// the X bytes through L2, with 32 rows per load instruction. Here a cluster
// tile of TR rows is split into CL row slices; CTA c reads its slice with
// coalesced row-major loads and stores each value into the owner CTA's
// staging buffer (st.shared::cluster); after one cluster barrier every CTA
// searches its own features for all TR rows from SMEM.
//
// Staging layout (per CTA, two stages): xs[stage][row][j], row pitch = odd
// number of words >= the group's feature count, so the owner's reads (lane =
// row) are conflict free and consecutive features of one row are consecutive
// words for the senders.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "hb_internal.h"

namespace hb {

namespace {

constexpr int kClWarps = 16;        // warps per CTA
constexpr int kClMaxF = 128;        // X columns one lane scatters: lane + 32 q, q < 4
constexpr int kClBatch = 8;         // rows whose X loads are in flight together per warp
// ROWS (template): 32-row blocks per warp per tile = lockstep searches per
// feature; a cluster tile is kClWarps * ROWS * 32 rows (1024 or 512)

struct RcClusterParams {
  const float *X;
  int64_t n, ldx;
  int F;                     // X columns scanned (owner map entries)
  const uint4 *feat;         // [n_fc][2] (offsets relative to the group's pool base)
  const uint4 *groups;       // [CL][2] {pool off, bytes, word_begin, word_end} {pitch, nf, 0, 0}
  const uint8_t *pool;
  const int32_t *own;        // [F] owner << 16 | local feature index, or -1 (column unused)
  int n_fc, n_words, cl;
  uint32_t stage_off;        // SMEM byte offset of the staging buffers
  uint32_t stage_words;      // words per stage (kClTile * max pitch)
  uint32_t *codes;           // [nblocks][n_words][32]
  int64_t nblocks;
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
__device__ __forceinline__ uint32_t map_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// lockstep bucket search, tables in this CTA's SMEM (see hb_rank_codes.cu)
template <bool LE, int NC>
__device__ __forceinline__ void codes_lockstep(const float (&x)[NC], const uint4 *m0, const uint4 *m1,
                                               const int (&mi)[NC], uint32_t smax, const uint8_t *tab,
                                               uint32_t (&code)[NC]) {
  uint32_t base[NC], cnt[NC], uo[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint4 a = m0[mi[c]], b = m1[mi[c]];
    const float lo = __uint_as_float(b.x), hi = __uint_as_float(b.y), sc = __uint_as_float(b.z);
    const float xc = fminf(fmaxf(x[c], lo), hi);            // NaN -> lo: walks bucket 0, replaced below
    float y = __fmul_rn(__fsub_rn(xc, lo), sc);
    y = fminf(y, (float)(a.y - 1u));
    const uint32_t bk = __float2uint_rz(y);
    const uint32_t be = *reinterpret_cast<const uint32_t *>(tab + a.w + 4u * bk);   // first index | count << 16
    base[c] = be & 0xFFFFu;
    cnt[c] = be >> 16;
    uo[c] = b.w;
  }
  for (uint32_t k = 0; k < smax; ++k) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const uint32_t half = cnt[c] >> 1;
      const float v = *reinterpret_cast<const float *>(tab + uo[c] + 4u * (base[c] + half));
      // branch-free (the load is unconditional: u has a pad slot), so the
      // NC chains of one step overlap instead of each waiting on its load
      const uint32_t go = (uint32_t)(LE ? v < x[c] : v <= x[c]) & (uint32_t)(cnt[c] != 0);
      base[c] += go * (half + 1u);
      cnt[c] = go ? cnt[c] - half - 1u : half;
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) code[c] = x[c] != x[c] ? 0xFFFFu : base[c];
}

template <bool LE, int CW, int ROWS>
__global__ void __launch_bounds__(32 * kClWarps, 1) rank_code_cluster_kernel(const RcClusterParams p) {
  constexpr int kClRows = ROWS;
  constexpr int kClTile = kClWarps * ROWS * 32;
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t crank = cluster_rank();
  const uint4 g = __ldg(p.groups + 2 * crank);
  const uint4 gx = __ldg(p.groups + 2 * crank + 1);
  const int pitch = (int)gx.x;
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(p.pool + g.x);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (uint32_t i = threadIdx.x; i < g.y / 16u; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  const uint32_t tsm = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t xs0 = tsm + p.stage_off;             // same offset in every CTA of the cluster
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this lane's X columns: owner CTA, local feature index, owner's row pitch
  int32_t own[kClMaxF / 32];
  uint32_t opitch[kClMaxF / 32];
#pragma unroll
  for (int q = 0; q < kClMaxF / 32; ++q) {
    const int f = lane + 32 * q;
    own[q] = f < p.F ? __ldg(p.own + f) : -1;
    opitch[q] = own[q] >= 0 ? __ldg(reinterpret_cast<const uint32_t *>(p.groups + 2 * ((uint32_t)own[q] >> 16) + 1)) : 1u;
  }
  // every CTA has started and holds its tables before any DSMEM store
  cluster_sync();
  constexpr int PW = CW == 32 ? 1 : 2;
  constexpr int WS = 2 / PW;                          // words per feature pair
  const int64_t ntiles = (p.n + kClTile - 1) / kClTile;
  int st = 0;
  for (int64_t tile = cluster_id_x(); tile < ntiles; tile += nclusters_x(), st ^= 1) {
    const int64_t row0 = tile * kClTile;
    const uint32_t stage = xs0 + (uint32_t)st * p.stage_words * 4u;
    // ---- scatter this CTA's rows (every cl-th row of the tile) to the owners'
    // staging buffers: lane = column (lane + 32 q), kClBatch rows of loads in
    // flight before the remote stores
    for (int i0 = 0;; i0 += kClBatch) {
      const int tr0 = (int)crank + p.cl * (warp + kClWarps * i0);
      if (tr0 >= kClTile) break;
      float v[kClBatch][kClMaxF / 32];
#pragma unroll
      for (int b = 0; b < kClBatch; ++b) {
        const int trow = (int)crank + p.cl * (warp + kClWarps * (i0 + b));
        const int64_t grow = min(row0 + min(trow, kClTile - 1), p.n - 1);   // tail rows: valid, unused codes
        const float *xr = p.X + grow * p.ldx;
#pragma unroll
        for (int q = 0; q < kClMaxF / 32; ++q)
          v[b][q] = (own[q] >= 0) ? __ldg(xr + lane + 32 * q) : 0.f;
      }
#pragma unroll
      for (int b = 0; b < kClBatch; ++b) {
        const int trow = (int)crank + p.cl * (warp + kClWarps * (i0 + b));
        if (trow >= kClTile) break;
#pragma unroll
        for (int q = 0; q < kClMaxF / 32; ++q)
          if (own[q] >= 0)
            st_cluster_f32(map_rank(stage + 4u * ((uint32_t)trow * opitch[q] + ((uint32_t)own[q] & 0xFFFFu)),
                                    (uint32_t)own[q] >> 16), v[b][q]);
      }
    }
    cluster_sync();
    // ---- search: this CTA's features x the tile's rows (lane = row)
    const int64_t blk0 = row0 / 32 + warp * kClRows;
    for (int wd = (int)g.z; wd < (int)g.w; wd += WS) {
      uint4 M0[2], M1[2];
      bool ok[2];
      int jl[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = PW * wd + e;
        ok[e] = (PW == 2 ? wd : wd + e) < (int)g.w && c < p.n_fc;
        const int cc = ok[e] ? c : PW * wd;
        M0[e] = __ldg(p.feat + 2 * cc);
        M1[e] = __ldg(p.feat + 2 * cc + 1);
        jl[e] = cc - PW * (int)g.z;
      }
      float x8[2 * kClRows];
      int mi[2 * kClRows];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int i = 0; i < kClRows; ++i) {
          const int trow = (warp * kClRows + i) * 32 + lane;
          x8[e * kClRows + i] = __uint_as_float(lds32(stage + 4u * ((uint32_t)trow * pitch + jl[e])));
          mi[e * kClRows + i] = e;
        }
      const uint32_t smax = max(M0[0].z, ok[1] ? M0[1].z : 0u);
      uint32_t code[2 * kClRows];
      codes_lockstep<LE, 2 * kClRows>(x8, M0, M1, mi, smax, smem, code);
#pragma unroll
      for (int i = 0; i < kClRows; ++i) {
        const int64_t blk = blk0 + i;
        if (blk >= p.nblocks) continue;
        uint32_t *dst = p.codes + ((size_t)blk * p.n_words + wd) * 32 + lane;
        if (CW == 32) {
          dst[0] = ((uint32_t)wd << 23) | code[i];
          if (ok[1]) dst[32] = ((uint32_t)(wd + 1) << 23) | code[kClRows + i];
        } else {
          dst[0] = code[i] | ((ok[1] ? code[kClRows + i] : 0u) << 16);
        }
      }
    }
    // the next tile scatters into the other stage; this stage is rewritten two
    // tiles later, after the next cluster barrier (all reads above precede it)
  }
  cluster_sync();   // no CTA leaves while peers may still store into its SMEM
}

using RcClFn = void (*)(const RcClusterParams);

template <int ROWS>
RcClFn cl_pick_rows(bool le, int cw) {
  if (cw == 32) return le ? rank_code_cluster_kernel<true, 32, ROWS> : rank_code_cluster_kernel<false, 32, ROWS>;
  return le ? rank_code_cluster_kernel<true, 16, ROWS> : rank_code_cluster_kernel<false, 16, ROWS>;
}

RcClFn cl_pick(bool le, int cw, int tile) { return tile == 2048 ? cl_pick_rows<4>(le, cw) : cl_pick_rows<2>(le, cw); }

}  // namespace

int sm_count(int device);

// staging bytes per CTA (two stages) for a cluster tile of `tile` rows
size_t rank_cluster_stage_bytes(uint32_t max_pitch, int tile) { return (size_t)2 * tile * max_pitch * 4; }

hb_status launch_rank_codes_cluster(const Model &m, const RunArgs &a, uint32_t *codes, int64_t nblocks) {
  RcClusterParams p;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.F = m.n_features;
  const uint8_t *aux = static_cast<const uint8_t *>(m.d_rbc);
  p.feat = reinterpret_cast<const uint4 *>(aux);
  p.groups = reinterpret_cast<const uint4 *>(aux + m.rbc_groups_off);
  p.own = reinterpret_cast<const int32_t *>(aux + m.rbc_own_off);
  p.pool = aux + m.rbc_pool_off;
  p.n_fc = m.rank_nfc;
  p.n_words = m.rank_nwords;
  p.cl = m.rbc_cl;
  p.codes = codes;
  p.nblocks = nblocks;
  const size_t tbytes = (m.rbc_smem + 15) & ~size_t(15);
  p.stage_off = (uint32_t)tbytes;
  const int tile = m.rbc_tile;
  p.stage_words = (uint32_t)tile * m.rbc_max_pitch;
  const size_t smem = tbytes + rank_cluster_stage_bytes(m.rbc_max_pitch, tile);
  RcClFn fn = cl_pick(m.cmp == HB_CMP_LE, m.rank_cw, tile);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(rank codes cluster)");
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)m.rbc_cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(32 * kClWarps);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = a.stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // persistent: as many clusters as can be co-resident, capped by the tiles
  int max_clusters = 0;
  cfg.gridDim = dim3((unsigned)(m.rbc_cl * std::max(1, sm_count(m.device) / m.rbc_cl)));
  e = cudaOccupancyMaxActiveClusters(&max_clusters, fn, &cfg);
  if (e != cudaSuccess || max_clusters <= 0) {
    cudaGetLastError();
    max_clusters = std::max(1, sm_count(m.device) / m.rbc_cl);
  }
  const int64_t ntiles = (a.n + tile - 1) / tile;
  const int64_t ncl = std::max<int64_t>(1, std::min<int64_t>(max_clusters, ntiles));
  cfg.gridDim = dim3((unsigned)(ncl * m.rbc_cl));
  e = cudaLaunchKernelEx(&cfg, fn, p);
  if (e != cudaSuccess) return cuda_fail(e, "rank_code_cluster_kernel launch");
  return HB_OK;
}

}  // namespace hb
