// hb_pttr_kernel.cuh — the rank-coded PTT scorer (kernel template); host
// side and launch in hb_pttr.cu, instantiations in hb_pttr_k32.cu / hb_pttr_k16.cu
// (two translation units so the build parallelises).
#pragma once
#include <cuda_runtime.h>

#include "hb_device.cuh"
#include "hb_internal.h"

namespace hb {

struct PttrParams {
  const float *X;
  int64_t n, ldx;
  const uint8_t *trees;
  uint32_t stride;
  int n_trees_pad, n_trees, tree_begin;
  const int32_t *leafmap;
  int nslots;
  const uint4 *fmeta;     // [n_fc] {orig f, L, offset in group, group}
  const uint4 *groups;    // [n_groups] {pool byte offset, bytes, fc_begin, fc_end}
  const uint8_t *pool;
  int n_fc, n_groups;
  int F, vec4, x_direct;  // x_direct: all F features used -> stage X into the cells, recode in place
  const float *scale, *base;
  int K, w, task, post, kind;
  void *out;
  int nw, ns, ch, ntiles;
  int prefetch;           // L2 prefetch of the next tile's X rows (code words with the pre-pass)
  uint32_t stage_bytes;
  const uint32_t *codes;  // pre-pass output [row block][n_words][32] (null: codes computed in-kernel)
  int n_words;
  int interleave;         // 1: warp units interleaved over the grid (ntiles = rounds, every CTA
                          // runs all of them; the last round's rows spread over every SM)
};

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void sts_u16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((uint16_t)v));
}

// CW = code cell width. 32: cell(fc, lane) = (fc*128) << 16 | c(x) (u32), node
// = (fc*128) << 16 | k, left <=> node >= cell. 16: codes of features 2m, 2m+1
// share lane l's 32-bit word (bank l) of row m; node = off16 << 16 | k with
// off16 = (fc>>1)*128 + (fc&1)*2, left <=> (node & 0xFFFF) >= c(x): half the
// tile, one more instruction per level.
//
// RPL = rows per lane. RPL = 2 (codes from the pre-pass only, D >= 3): a warp
// owns 64 rows, lane l rows l and l + 32 (two consecutive 32-row code blocks
// in SMEM). The top three levels are shared by the two rows: the root with
// one LDS, nodes 2-3 with one LDS.64 and nodes 4-7 with one LDS.128, all
// broadcasts (one wavefront each), then selected per row; below level 2 each
// row walks on its own. The kernel is bound by SMEM wavefronts (~20.3 per
// warp-tree at one row per lane, three of them for levels 0-2), so sharing
// the top levels saves wavefronts: ncu on C3 38.7 instead of 2 x 20.3 per
// 64 rows and tree, scorer 11.35 -> 10.69 ms.
template <int D, bool LE, int NACC, int G, int CW, int RPL = 1>
__global__ void __launch_bounds__(32 * 25, 1) pttr_kernel(const PttrParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = p.nw, ns = p.ns, ch = p.ch;
  const uint32_t tile_bytes = CW == 32 ? (uint32_t)p.n_fc * 128u : (uint32_t)((p.n_fc + 1) / 2) * 128u;
  const size_t xbytes = (size_t)nw * tile_bytes * RPL;
  uint8_t *stages = smem + xbytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(stages + (size_t)ns * p.stage_bytes);
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
  const int items = p.n_groups + nchunks;          // per tile: feature groups, then tree chunks
  // row tiles of this CTA. Contiguous tiles: tile t = blockIdx.x + k grid,
  // warp w owns unit t nw + w. Interleaved units (p.interleave): round k,
  // warp w owns unit (k nw + w) grid + blockIdx.x, so a partial last round
  // leaves every SM some warps instead of leaving whole SMs idle.
  const int my_tiles = p.interleave ? p.ntiles
                                    : (p.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  auto unit_of = [&](int k) -> int64_t {
    return p.interleave ? ((int64_t)k * nw + warp) * gridDim.x + blockIdx.x
                        : ((int64_t)blockIdx.x + (int64_t)k * gridDim.x) * nw + warp;
  };

  if (warp == nw) {
    if (lane == 0) {
      const long total = (long)my_tiles * items;
      dev::Ring r(ns);
      int q = 0;
      for (long it = 0; it < total; ++it, r.next(), q = (q + 1 == items) ? 0 : q + 1) {
        const int s = r.s;
        dev::mbar_wait(&empty[s], r.ph ^ 1u);
        if (q == 0 && p.prefetch && !p.interleave) {
          // first item of a tile: warm L2 with this CTA's NEXT tile of X rows
          // (of code words, which are contiguous per tile, with the pre-pass)
          const long tile_i = it / items;
          const int64_t next = (int64_t)(blockIdx.x + (tile_i + 1) * gridDim.x) * (nw * 32 * RPL);
          if (p.codes) {
            const int64_t nb = (p.n + 31) / 32, b0 = next / 32;
            if (b0 < nb)
              dev::prefetch_rows_l2(reinterpret_cast<const float *>(p.codes), b0,
                                    min((int64_t)nw * RPL, nb - b0), nb, (int64_t)p.n_words * 32);
          } else {
            dev::prefetch_rows_l2(p.X, next, (int64_t)nw * 32, p.n, p.ldx);
          }
        }
        const uint8_t *src;
        uint32_t bytes;
        if (q < p.n_groups) {
          const uint4 g = __ldg(p.groups + q);
          src = p.pool + g.x;
          bytes = g.y;
        } else {
          const int t0 = (q - p.n_groups) * ch;
          src = p.trees + (size_t)t0 * p.stride;
          bytes = (uint32_t)min(ch, p.n_trees_pad - t0) * p.stride;
        }
        dev::mbar_arrive_expect_tx(&full[s], bytes);
        dev::bulk_g2s(stages + (size_t)s * p.stage_bytes, src, bytes, &full[s]);
      }
    }
    return;
  }

  if constexpr (RPL == 2) {
    static_assert(D >= 3, "RPL = 2 shares levels 0-2");
    // pre-pass codes only (host: rank_pre, no feature groups in the ring)
    const uint32_t codesA = dev::smem_u32(smem) + (uint32_t)warp * 2u * tile_bytes + 4u * lane;
    const uint32_t codesB = codesA + tile_bytes;
    const uint32_t stage0 = dev::smem_u32(stages);
    const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
    // go left <=> k >= c(x) (node and 32-bit cell share the high half; 16-bit
    // cells compare the low half)
    auto left_of = [&](uint32_t nd, uint32_t cbase) -> bool {
      HB_DCHECK((nd >> 16) < tile_bytes);               // code cell inside this row block's tile
      if (CW == 32) return nd >= dev::lds_u32(cbase + (nd >> 16));
      return (nd & 0xFFFFu) >= lds_u16(cbase + (nd >> 16));
    };
    dev::Ring ring(ns);
    for (int k = 0; k < my_tiles; ++k) {
      const int64_t wrow0 = unit_of(k) * 64;
      const int64_t rowA = wrow0 + lane, rowB = rowA + 32;
      const bool active = wrow0 < p.n;
      if (p.interleave && p.prefetch && lane == 0) {
        // warm L2 with this warp's next unit of code words
        const int64_t nb = (p.n + 31) / 32, b1 = (unit_of(k + 1) * 64) >> 5;
        if (b1 < nb)
          dev::prefetch_rows_l2(reinterpret_cast<const float *>(p.codes), b1, min((int64_t)2, nb - b1), nb,
                                (int64_t)p.n_words * 32);
      }
      __syncwarp();   // previous tile's cell reads done before the fill (WAR)
      if (active) {
        const int nblk = wrow0 + 32 < p.n ? 2 : 1;
        HB_DCHECK((wrow0 >> 5) + nblk <= (p.n + 31) / 32);   // pre-pass blocks that exist
        const uint4 *src = reinterpret_cast<const uint4 *>(p.codes + (size_t)(wrow0 >> 5) * p.n_words * 32);
        const uint32_t dst = codesA - 4u * lane;
        for (int i = lane; i < nblk * p.n_words * 8; i += 32) {
          const uint4 v = __ldg(src + i);
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16u * i), "r"(v.x), "r"(v.y),
                       "r"(v.z), "r"(v.w));
        }
        __syncwarp();
      }
      double accA[NACC], accB[NACC];
#pragma unroll
      for (int k = 0; k < NACC; ++k) accA[k] = accB[k] = 0.0;
      uint64_t hA = 0, hB = 0;
      double curA = 0.0, curB = 0.0;
      uint32_t curk = 0;
      for (int c = 0; c < nchunks; ++c, ring.next()) {
        const int s = ring.s;
        dev::mbar_wait(&full[s], ring.ph);
        if (active) {
          const uint32_t cb = stage0 + (uint32_t)s * p.stage_bytes;
          const int nt = min(ch, p.n_trees_pad - c * ch);
          for (int j = 0; j < nt; j += G) {
            uint32_t tb[G], aA[G], aB[G];
#pragma unroll
            for (int g = 0; g < G; ++g) tb[g] = cb + (uint32_t)(j + g) * p.stride;
            // levels 0-2 shared by the two rows: one broadcast load per level
            uint32_t r0[G];
#pragma unroll
            for (int g = 0; g < G; ++g) r0[g] = dev::lds_u32(tb[g] + 4u);
            bool a0[G], b0[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
              a0[g] = left_of(r0[g], codesA);
              b0[g] = left_of(r0[g], codesB);
            }
            uint2 n23[G];
#pragma unroll
            for (int g = 0; g < G; ++g) n23[g] = dev::lds_v2(tb[g] + 8u);
            bool a1[G], b1[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
              a1[g] = left_of(a0[g] ? n23[g].x : n23[g].y, codesA);
              b1[g] = left_of(b0[g] ? n23[g].x : n23[g].y, codesB);
            }
            uint4 n47[G];
#pragma unroll
            for (int g = 0; g < G; ++g)
              asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                           : "=r"(n47[g].x), "=r"(n47[g].y), "=r"(n47[g].z), "=r"(n47[g].w)
                           : "r"(tb[g] + 16u));
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const uint32_t ndA = a0[g] ? (a1[g] ? n47[g].x : n47[g].y) : (a1[g] ? n47[g].z : n47[g].w);
              const uint32_t ndB = b0[g] ? (b1[g] ? n47[g].x : n47[g].y) : (b1[g] ? n47[g].z : n47[g].w);
              const bool a2 = left_of(ndA, codesA), b2 = left_of(ndB, codesB);
              // heap node 8 + 4(!l0) + 2(!l1) + (!l2) at tree + 4 i
              aA[g] = tb[g] + 32u + (a0[g] ? 0u : 16u) + (a1[g] ? 0u : 8u) + (a2 ? 0u : 4u);
              aB[g] = tb[g] + 32u + (b0[g] ? 0u : 16u) + (b1[g] ? 0u : 8u) + (b2 ? 0u : 4u);
            }
            // levels 3 .. D-1: each row on its own (a' = 2 a - tree + (left ? 0 : 4))
#pragma unroll
            for (int l = 3; l < D; ++l) {
              uint32_t ndA[G], ndB[G];
#pragma unroll
              for (int g = 0; g < G; ++g) {
                HB_DCHECK(aA[g] - tb[g] >= (4u << l) && aA[g] - tb[g] < (8u << l));   // heap node of level l
                HB_DCHECK(aB[g] - tb[g] >= (4u << l) && aB[g] - tb[g] < (8u << l));
                ndA[g] = dev::lds_u32(aA[g]);
                ndB[g] = dev::lds_u32(aB[g]);
              }
#pragma unroll
              for (int g = 0; g < G; ++g) {
                const bool la = left_of(ndA[g], codesA), lb = left_of(ndB[g], codesB);
                aA[g] = 2u * aA[g] - tb[g] + (la ? 0u : 4u);
                aB[g] = 2u * aB[g] - tb[g] + (lb ? 0u : 4u);
              }
            }
            double vsA = 0.0, vsB = 0.0;
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const uint32_t offA = aA[g] - tb[g], offB = aB[g] - tb[g];
              HB_DCHECK(offA >= (4u << D) && offA < (8u << D) && offB >= (4u << D) && offB < (8u << D));
              if (p.w == 1) {
                const double vA = (double)dev::lds_f32(tb[g] + offA);
                const double vB = (double)dev::lds_f32(tb[g] + offB);
                if (NACC == 1) {
                  accA[0] += vA;
                  accB[0] += vB;
                } else {
                  vsA += vA;
                  vsB += vB;
                }
              } else {
                const uint32_t lbA = tb[g] + (4u << D) + 4u * ((offA >> 2) - (1u << D)) * (uint32_t)p.w;
                const uint32_t lbB = tb[g] + (4u << D) + 4u * ((offB >> 2) - (1u << D)) * (uint32_t)p.w;
#pragma unroll
                for (int k = 0; k < NACC; ++k)
                  if (k < p.K) {
                    accA[k] += (double)dev::lds_f32(lbA + 4u * k);
                    accB[k] += (double)dev::lds_f32(lbB + 4u * k);
                  }
              }
            }
            if (NACC > 1 && p.w == 1) {
              // class-ordered records (see the one-row path below)
              const uint32_t k0 = dev::lds_u32(tb[0]) & 0xFFu;
              if (k0 != curk) {
#pragma unroll
                for (int k = 0; k < NACC; ++k)
                  if (curk == (uint32_t)k) {
                    accA[k] += curA;
                    accB[k] += curB;
                  }
                curA = curB = 0.0;
                curk = k0;
              }
              curA += vsA;
              curB += vsB;
            }
            if (lm) {
#pragma unroll
              for (int g = 0; g < G; ++g) {
                const int orig = (int)(dev::lds_u32(tb[g]) >> 8) - 1;
                if (orig < 0) continue;
                const size_t lmb = (size_t)(c * ch + j + g) * p.nslots;
                const int32_t idA = __ldg(p.leafmap + lmb + (((aA[g] - tb[g]) >> 2) - (1u << D)));
                const int32_t idB = __ldg(p.leafmap + lmb + (((aB[g] - tb[g]) >> 2) - (1u << D)));
                if (lm == 1) {
                  if (rowA < p.n) static_cast<int32_t *>(p.out)[rowA * p.n_trees + orig] = idA;
                  if (rowB < p.n) static_cast<int32_t *>(p.out)[rowB * p.n_trees + orig] = idB;
                } else {
                  const uint64_t th = (uint64_t)(uint32_t)(p.tree_begin + orig) << 32;
                  hA += dev::mix64(th | (uint32_t)idA);
                  hB += dev::mix64(th | (uint32_t)idB);
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
          if (curk == (uint32_t)k) {
            accA[k] += curA;
            accB[k] += curB;
          }
      }
      if (lm == 2) {
        if (rowA < p.n) static_cast<uint64_t *>(p.out)[rowA] = hA;
        if (rowB < p.n) static_cast<uint64_t *>(p.out)[rowB] = hB;
      } else if (lm == 0) {
        if (rowA < p.n) dev::write_row<NACC>(p.kind, accA, p.K, p.task, p.post, p.scale, p.base, rowA, p.out);
        if (rowB < p.n) dev::write_row<NACC>(p.kind, accB, p.K, p.task, p.post, p.scale, p.base, rowB, p.out);
      }
    }
    return;
  }

  const uint32_t codes = dev::smem_u32(smem) + (uint32_t)warp * tile_bytes + 4u * lane;
  const uint32_t stage0 = dev::smem_u32(stages);
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  dev::Ring ring(ns);
  for (int k = 0; k < my_tiles; ++k) {
    const int64_t wrow0 = unit_of(k) * 32;
    const int64_t row = wrow0 + lane;
    const bool active = wrow0 < p.n;
    if (p.interleave && p.prefetch && lane == 0) {
      // warm L2 with this warp's next unit: code words, or its X rows
      const int64_t r1 = unit_of(k + 1) * 32;
      if (p.codes) {
        const int64_t nb = (p.n + 31) / 32;
        if ((r1 >> 5) < nb)
          dev::prefetch_rows_l2(reinterpret_cast<const float *>(p.codes), r1 >> 5, 1, nb, (int64_t)p.n_words * 32);
      } else {
        dev::prefetch_rows_l2(p.X, r1, 32, p.n, p.ldx);
      }
    }
    const float *xr = p.X + (row < p.n ? row : 0) * p.ldx;
    // the tile fills below write other lanes' cells: every lane is done
    // reading the previous tile's (WAR within the warp; racecheck)
    __syncwarp();
    if (p.codes) {
      // codes from the pre-pass: this warp's block is already in tile layout
      if (active) {
        const uint4 *src = reinterpret_cast<const uint4 *>(p.codes + (size_t)(wrow0 >> 5) * p.n_words * 32);
        const uint32_t dst = codes - 4u * lane;
        for (int i = lane; i < p.n_words * 8; i += 32) {
          const uint4 v = __ldg(src + i);
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(dst + 16u * i), "r"(v.x), "r"(v.y),
                       "r"(v.z), "r"(v.w));
        }
        __syncwarp();
      }
    } else if (CW == 32 && p.x_direct && active) {
      // fp32 X slice straight into the code cells (cell(f, lane) = xs[f*32 + lane])
      dev::load_x_slice(reinterpret_cast<float *>(smem) + (size_t)warp * p.n_fc * 32, p.X, row, p.n,
                        p.ldx, p.F, lane, p.vec4 != 0);
    }

    // ---- rank codes of this warp's 32 rows, one feature group per stage
    for (int gq = 0; gq < p.n_groups; ++gq, ring.next()) {
      const int s = ring.s;
      dev::mbar_wait(&full[s], ring.ph);
      if (active) {
        const uint4 g = __ldg(p.groups + gq);
        const uint32_t gb = stage0 + (uint32_t)s * p.stage_bytes;
        // four independent searches per lane (memory-level parallelism); the
        // per-feature depth L is warp-uniform, so the guards do not diverge
        for (int fc = (int)g.z; fc < (int)g.w; fc += 4) {
          uint32_t i[4], eb[4], L[4];
          float x[4];
          uint32_t lmax = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool valid = fc + q < (int)g.w;
            const uint4 fm = __ldg(p.fmeta + (valid ? fc + q : fc));
            x[q] = (CW == 32 && p.x_direct) ? dev::lds_f32(codes + (uint32_t)(valid ? fc + q : fc) * 128u)
                                            : __ldg(xr + fm.x);
            eb[q] = gb + fm.z;
            L[q] = valid ? fm.y : 0u;
            i[q] = 1u;
            lmax = max(lmax, L[q]);
          }
          for (uint32_t l = 0; l < lmax; ++l) {
            // branch-free: finished searches re-read a valid slot and keep i
            float u[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) u[q] = dev::lds_f32(eb[q] + (l < L[q] ? 4u * i[q] : 4u));
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const bool pr = LE ? (u[q] < x[q]) : (u[q] <= x[q]);   // u sorts before x
              const uint32_t nx = 2u * i[q] + (pr ? 1u : 0u);
              i[q] = l < L[q] ? nx : i[q];
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (fc + q < (int)g.w) {
              const uint32_t code = (x[q] != x[q]) ? 0xFFFFu : i[q] - (1u << L[q]);
              const uint32_t c = (uint32_t)(fc + q);
              if (CW == 32) dev::sts_u32(codes + c * 128u, (c << 23) | code);
              else sts_u16(codes + (c >> 1) * 128u + (c & 1u) * 2u, code);
            }
        }
      }
      dev::release_stage(&empty[s], lane);
    }

    // fp64 accumulators: every fp32 leaf value is added exactly enough that
    // the sum matches the oracle's fp64 sum to ~1e-16 relative whatever the
    // order (R23), at one F2F + DADD per (row, tree)
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 0.0;
    uint64_t h = 0;
    double cur = 0.0;     // running sum of the current class (per-class scalar trees)
    uint32_t curk = 0;
    for (int c = 0; c < nchunks; ++c, ring.next()) {
      const int s = ring.s;
      dev::mbar_wait(&full[s], ring.ph);
      if (active) {
        const uint32_t cb = stage0 + (uint32_t)s * p.stage_bytes;
        const int nt = min(ch, p.n_trees_pad - c * ch);
        for (int j = 0; j < nt; j += G) {
          // a = absolute address of heap node i (tree + 4 i); next level:
          // a' = tree + 8 i + (left ? 0 : 4) = 2 a + (left ? -tree : 4 - tree)
          uint32_t tb[G], a[G], m0[G], m4[G];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            tb[g] = cb + (uint32_t)(j + g) * p.stride;
            a[g] = tb[g] + 4u;                 // heap node 1 (root), 4-B records
            m0[g] = 0u - tb[g];
            m4[g] = 4u - tb[g];
          }
#pragma unroll
          for (int l = 0; l < D; ++l) {
            uint32_t nd[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
              HB_DCHECK(a[g] - tb[g] >= (4u << l) && a[g] - tb[g] < (8u << l));   // heap node of level l
              nd[g] = dev::lds_u32(a[g]);
            }
            uint32_t xc[G];
#pragma unroll
            for (int g = 0; g < G; ++g) HB_DCHECK((nd[g] >> 16) < tile_bytes);   // code cell in the tile
#pragma unroll
            for (int g = 0; g < G; ++g)
              xc[g] = CW == 32 ? dev::lds_u32(codes + (nd[g] >> 16)) : lds_u16(codes + (nd[g] >> 16));
#pragma unroll
            for (int g = 0; g < G; ++g) {
              // k >= c(x)  <=>  x < u_k
              const bool left = CW == 32 ? nd[g] >= xc[g] : (nd[g] & 0xFFFFu) >= xc[g];
              a[g] = 2u * a[g] + (left ? m0[g] : m4[g]);
            }
          }
          uint32_t off[G];
#pragma unroll
          for (int g = 0; g < G; ++g) off[g] = a[g] - tb[g];
          double vsum = 0.0;
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const uint32_t slot = (off[g] >> 2) - (1u << D);
            if (p.w == 1) {
              const double v = (double)dev::lds_f32(tb[g] + off[g]);
              if (NACC == 1) acc[0] += v;
              else vsum += v;
            } else {
              const uint32_t lb = tb[g] + (4u << D) + 4u * slot * (uint32_t)p.w;
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
              const uint32_t slot = (off[g] >> 2) - (1u << D);
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

using PttrFn = void (*)(const PttrParams);

template <int CW, int D, bool LE, int RPL>
static PttrFn pttr_pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return pttr_kernel<D, LE, 1, kTreeGroup, CW, RPL>;
    case 4: return pttr_kernel<D, LE, 4, kTreeGroup, CW, RPL>;
    case 8: return pttr_kernel<D, LE, 8, kTreeGroup, CW, RPL>;
    default: return pttr_kernel<D, LE, 16, kTreeGroup, CW, RPL>;
  }
}

template <int CW, int D, int RPL>
static PttrFn pttr_pick_le(bool le, int nacc) {
  return le ? pttr_pick_nacc<CW, D, true, RPL>(nacc) : pttr_pick_nacc<CW, D, false, RPL>(nacc);
}

template <int CW>
static PttrFn pttr_pick(int D, bool le, int nacc) {
  switch (D) {
    case 0: return pttr_pick_le<CW, 0, 1>(le, nacc);
    case 1: return pttr_pick_le<CW, 1, 1>(le, nacc);
    case 2: return pttr_pick_le<CW, 2, 1>(le, nacc);
    case 3: return pttr_pick_le<CW, 3, 1>(le, nacc);
    case 4: return pttr_pick_le<CW, 4, 1>(le, nacc);
    case 5: return pttr_pick_le<CW, 5, 1>(le, nacc);
    case 6: return pttr_pick_le<CW, 6, 1>(le, nacc);
    case 7: return pttr_pick_le<CW, 7, 1>(le, nacc);
    case 8: return pttr_pick_le<CW, 8, 1>(le, nacc);
    case 9: return pttr_pick_le<CW, 9, 1>(le, nacc);
    case 10: return pttr_pick_le<CW, 10, 1>(le, nacc);
    default: return nullptr;
  }
}

// two rows per lane (pre-pass codes, D >= 3)
template <int CW>
static PttrFn pttr_pick_rpl2(int D, bool le, int nacc) {
  switch (D) {
    case 3: return pttr_pick_le<CW, 3, 2>(le, nacc);
    case 4: return pttr_pick_le<CW, 4, 2>(le, nacc);
    case 5: return pttr_pick_le<CW, 5, 2>(le, nacc);
    case 6: return pttr_pick_le<CW, 6, 2>(le, nacc);
    case 7: return pttr_pick_le<CW, 7, 2>(le, nacc);
    case 8: return pttr_pick_le<CW, 8, 2>(le, nacc);
    case 9: return pttr_pick_le<CW, 9, 2>(le, nacc);
    case 10: return pttr_pick_le<CW, 10, 2>(le, nacc);
    default: return nullptr;
  }
}

PttrFn pttr_fn32(int D, bool le, int nacc);
PttrFn pttr_fn16(int D, bool le, int nacc);
PttrFn pttr_fn32_rpl2(int D, bool le, int nacc);
PttrFn pttr_fn16_rpl2(int D, bool le, int nacc);

}  // namespace hb
