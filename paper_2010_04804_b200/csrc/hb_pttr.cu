// hb_pttr.cu — PerfectTreeTraversal with rank-coded thresholds (sm_100a).
//
// Same algorithm as hb_ptt.cu (Alg. 3), same results bit
// for bit, with 4-byte instead of 8-byte node records:
//
//  * Compile time: for every feature f used by the model, the distinct
//    thresholds u_0 < ... < u_{m-1} (fp32 order) are collected. A node that
//    tests (f, u_k) stores k and the compact feature index.
//  * Per row tile, each X value is replaced by its rank code
//        LT: c(x) = #{j : u_j <= x}      LE: c(x) = #{j : u_j <  x}
//    and NaN by 0xFFFF. Then  x < u_k  <=>  c(x) <= k  (LE:  x <= u_k <=> c(x) <= k)
//    for every x, so the integer walk takes exactly the fp32 walk's branches.
//  * The code is computed by walking a perfect binary search tree over the u_j
//    in Eytzinger (heap) order — itself a perfect-tree traversal: after L =
//    bit_length(m) steps of  i <- 2 i + pred(e_i, x)  the rank is i - 2^L
//    (padding slots hold NaN, so pred is false there, i.e. they sort last).
//
// Why: a warp-wide LDS.64 is served in two half-warp passes, so 8-B node
// records cost >= 2 SMEM wavefronts per level; a 4-B record costs 1 when the
// level's nodes are distinct banks. The bank-conflict model of DESIGN.md §4.1
// (validated against ncu: 31.9 vs 31.1 wavefronts per warp-tree) gives 20.3
// wavefronts per warp-tree for this layout, plus ~7% for the per-tile code
// transform.
//
// Node record: u32 = (fc * 128) << 16 | k. The per-warp code tile holds
// cell[fc][lane] = (fc * 128) << 16 | c(x) as u32, so lane l always reads bank l
// (conflict-free whatever feature it needs), the cell address is one LEA.HI
// (tile + (node >> 16)), and since node and cell share the high half, "go
// left" is the single unsigned compare  node >= cell  <=>  k >= c(x)
// (n_fc <= 511 so that fc * 128 fits 16 bits).
// Leaf layout makes the leaf address equal to the final heap byte offset: tree
// record = node[2^D] (node[0] = tree_output) then leaf[2^D] (w = 1), so after D
// levels off = 4 i with i in [2^D, 2^(D+1)) and leaf(i - 2^D) sits at off.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hb_internal.h"
#include "hb_layouts.h"
#include "hb_pttr_kernel.cuh"

namespace hb {

int sm_count(int device);

hb_status launch_ptt_rank(const Model &m, const RunArgs &a) {
  const bool le = m.cmp == HB_CMP_LE;
  PttrFn fn = m.rank_rpl == 2 ? (m.rank_cw == 16 ? pttr_fn16_rpl2(m.depth, le, m.nacc) : pttr_fn32_rpl2(m.depth, le, m.nacc))
                              : (m.rank_cw == 16 ? pttr_fn16(m.depth, le, m.nacc) : pttr_fn32(m.depth, le, m.nacc));
  if (!fn) return fail(HB_E_UNSUPPORTED, "PTT depth out of range");
  PttrParams p;
  // pre-pass: rank codes of every (row, used feature) into stream-ordered
  // scratch, in the per-warp tile layout the scorer copies verbatim
  uint32_t *codes = nullptr;
  cudaError_t e;
  if (m.rank_pre) {
    const int64_t nblocks = (a.n + 31) / 32;
    const size_t bytes = std::max<size_t>((size_t)nblocks * m.rank_nwords * 128, 128);
    const hb_status ast = scratch_alloc(m, bytes, a.stream, reinterpret_cast<void **>(&codes));
    if (ast != HB_OK) return ast;
    const hb_status st = launch_rank_codes(m, a, codes, nblocks);
    if (st != HB_OK) {
      cudaFreeAsync(codes, a.stream);
      return st;
    }
  }
  p.codes = codes;
  p.n_words = m.rank_nwords;
  p.X = a.X;
  p.n = a.n;
  p.ldx = a.ldx;
  p.trees = static_cast<const uint8_t *>(m.d_trees);
  p.stride = (uint32_t)m.stride;
  p.n_trees_pad = m.n_trees_pad;
  p.n_trees = m.n_trees;
  p.tree_begin = m.tree_begin;
  p.leafmap = m.d_leafmap;
  p.nslots = m.nslots;
  const uint8_t *aux = static_cast<const uint8_t *>(m.d_aux);
  p.fmeta = reinterpret_cast<const uint4 *>(aux);
  p.groups = reinterpret_cast<const uint4 *>(aux + m.aux_groups_off);
  p.pool = aux + m.aux_pool_off;
  p.n_fc = m.rank_nfc;
  p.n_groups = m.rank_ngroups;
  p.F = m.n_features;
  p.vec4 = ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && (a.ldx % 4 == 0);
  p.x_direct = m.rank_cw == 32 && m.rank_nfc == m.n_features;
  p.scale = m.d_scale;
  p.base = m.d_base;
  p.K = m.n_outputs;
  p.w = m.leaf_width;
  p.task = m.task;
  p.post = m.post;
  p.kind = a.kind;
  p.out = a.out;
  p.prefetch = m.cfg.prefetch;
  // consumer warps of this launch: the persistent grid walks ceil(tiles / SMs)
  // rounds of row tiles, so a call whose tiles leave the last round part
  // empty runs up to 2 fewer warps per CTA when that costs fewer warp-rounds
  // (rounds x warps; SMEM sized for cfg.nw holds any smaller count). E.g.
  // C3's 1.25M rows per GPU at 8 GPUs: 24 warps x 64 rows = 5.5 rounds ->
  // 22 warps, 6.0 rounds: 796.4M -> 834.5M rows/s. Deeper trims lose more
  // per-warp throughput than they save (C2 at 18 warps: 597M -> 563M).
  // HB_NW_TRIM=0 keeps cfg.nw.
  const int sms = sm_count(m.device) * m.cfg.ctas_per_sm;
  int nw = m.cfg.nw;
  // interleaved warp units (HB_PTTR_INTERLEAVE, default on) spread a partial
  // last round over every SM, which makes the warp trim below unnecessary
  p.interleave = !(std::getenv("HB_PTTR_INTERLEAVE") && std::atoi(std::getenv("HB_PTTR_INTERLEAVE")) == 0);
  if (!p.interleave && !(std::getenv("HB_NW_TRIM") && std::atoi(std::getenv("HB_NW_TRIM")) == 0)) {
    int64_t best = INT64_MAX;
    for (int w = m.cfg.nw; w >= std::max(1, m.cfg.nw - 2); --w) {
      const int64_t rows = (int64_t)w * 32 * m.rank_rpl;
      const int64_t rounds = ((a.n + rows - 1) / rows + sms - 1) / sms;
      if (rounds * w < best) {
        best = rounds * w;
        nw = w;
      }
    }
  }
  p.nw = nw;
  p.ns = m.cfg.ns;
  p.ch = m.cfg.ch;
  p.stage_bytes = (uint32_t)m.cfg.stage_bytes;
  const int64_t rows_per_tile = (int64_t)nw * 32 * m.rank_rpl;
  int64_t ntiles = (a.n + rows_per_tile - 1) / rows_per_tile;
  if (ntiles > INT32_MAX) {
    if (codes) cudaFreeAsync(codes, a.stream);
    return fail(HB_E_UNSUPPORTED, "too many rows for one launch");
  }
  const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count(m.device) * m.cfg.ctas_per_sm);
  // interleaved warp units: ntiles becomes the number of rounds every CTA runs
  if (p.interleave) {
    const int64_t unit_rows = 32 * (int64_t)m.rank_rpl;
    const int64_t units = (a.n + unit_rows - 1) / unit_rows;
    ntiles = (units + (int64_t)grid * nw - 1) / ((int64_t)grid * nw);
  }
  p.ntiles = (int)ntiles;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, m.cfg.smem_bytes);
  if (e == cudaSuccess) {
    if (codes) mark_launch(a);     // scorer starts (the pre-pass was launch 0)
    fn<<<grid, 32 * (nw + 1), m.cfg.smem_bytes, a.stream>>>(p);
    e = cudaGetLastError();
  }
  if (codes) cudaFreeAsync(codes, a.stream);
  if (e != cudaSuccess) return cuda_fail(e, "pttr_kernel launch");
  return HB_OK;
}

}  // namespace hb
