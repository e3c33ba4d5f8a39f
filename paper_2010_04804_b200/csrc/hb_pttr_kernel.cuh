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
template <int D, bool LE, int NACC, int G, int CW>
__global__ void __launch_bounds__(32 * 25, 1) pttr_kernel(const PttrParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = p.nw, ns = p.ns, ch = p.ch;
  const uint32_t tile_bytes = CW == 32 ? (uint32_t)p.n_fc * 128u : (uint32_t)((p.n_fc + 1) / 2) * 128u;
  const size_t xbytes = (size_t)nw * tile_bytes;
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
  const int my_tiles = (p.ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;

  if (warp == nw) {
    if (lane == 0) {
      const long total = (long)my_tiles * items;
      dev::Ring r(ns);
      int q = 0;
      for (long it = 0; it < total; ++it, r.next(), q = (q + 1 == items) ? 0 : q + 1) {
        const int s = r.s;
        dev::mbar_wait(&empty[s], r.ph ^ 1u);
        if (q == 0 && p.prefetch) {
          // first item of a tile: warm L2 with this CTA's NEXT tile of X rows
          // (of code words, which are contiguous per tile, with the pre-pass)
          const long tile_i = it / items;
          const int64_t next = (int64_t)(blockIdx.x + (tile_i + 1) * gridDim.x) * (nw * 32);
          if (p.codes) {
            const int64_t nb = (p.n + 31) / 32, b0 = next / 32;
            if (b0 < nb)
              dev::prefetch_rows_l2(reinterpret_cast<const float *>(p.codes), b0,
                                    min((int64_t)nw, nb - b0), nb, (int64_t)p.n_words * 32);
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

  const uint32_t codes = dev::smem_u32(smem) + (uint32_t)warp * tile_bytes + 4u * lane;
  const uint32_t stage0 = dev::smem_u32(stages);
  const int lm = p.kind == HB_OUT_LEAF ? 1 : (p.kind == HB_OUT_LEAF_HASH ? 2 : 0);
  dev::Ring ring(ns);
  for (int tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
    const int64_t wrow0 = (int64_t)tile * (nw * 32) + warp * 32;
    const int64_t row = wrow0 + lane;
    const bool active = wrow0 < p.n;
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
            for (int g = 0; g < G; ++g) nd[g] = dev::lds_u32(a[g]);
            uint32_t xc[G];
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

template <int CW, int D, bool LE>
static PttrFn pttr_pick_nacc(int nacc) {
  switch (nacc) {
    case 1: return pttr_kernel<D, LE, 1, kTreeGroup, CW>;
    case 4: return pttr_kernel<D, LE, 4, kTreeGroup, CW>;
    case 8: return pttr_kernel<D, LE, 8, kTreeGroup, CW>;
    default: return pttr_kernel<D, LE, 16, kTreeGroup, CW>;
  }
}

template <int CW, int D>
static PttrFn pttr_pick_le(bool le, int nacc) {
  return le ? pttr_pick_nacc<CW, D, true>(nacc) : pttr_pick_nacc<CW, D, false>(nacc);
}

template <int CW>
static PttrFn pttr_pick(int D, bool le, int nacc) {
  switch (D) {
    case 0: return pttr_pick_le<CW, 0>(le, nacc);
    case 1: return pttr_pick_le<CW, 1>(le, nacc);
    case 2: return pttr_pick_le<CW, 2>(le, nacc);
    case 3: return pttr_pick_le<CW, 3>(le, nacc);
    case 4: return pttr_pick_le<CW, 4>(le, nacc);
    case 5: return pttr_pick_le<CW, 5>(le, nacc);
    case 6: return pttr_pick_le<CW, 6>(le, nacc);
    case 7: return pttr_pick_le<CW, 7>(le, nacc);
    case 8: return pttr_pick_le<CW, 8>(le, nacc);
    case 9: return pttr_pick_le<CW, 9>(le, nacc);
    case 10: return pttr_pick_le<CW, 10>(le, nacc);
    default: return nullptr;
  }
}

PttrFn pttr_fn32(int D, bool le, int nacc);
PttrFn pttr_fn16(int D, bool le, int nacc);

}  // namespace hb
