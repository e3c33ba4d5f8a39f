// hb_layouts.h — compiled-layout geometry shared by the host compilers
// (hb_compile.cpp, hb_host.cpp) and the CUDA kernels that read the layouts.
// Host-only C++ (no device code), so the compilers build with a plain host
// compiler too (the ASan/UBSan fuzz build, tests/fuzz/).
#pragma once

#include <stddef.h>
#include <stdint.h>

namespace hb {

// ---- GEMM strategy, CUDA-core kernel (hb_gemm.cu)
constexpr int kGemmMaxInternal = 64;   // T fits one 64-bit word

// per-tree record (all fields 8-B aligned):
//   u32 hdr[2] = {tree_output, 0}
//   u32 feat[NI]; f32 thr[NI]                 (NI padded to even)
//   u64 lmask[NL]; u64 rmask[NL]; u32 D[NL] (NL padded to even)
//   f32 E[NL * w]
struct GemmGeom {
  int ni, nl, w;
  size_t off_feat, off_thr, off_lm, off_rm, off_d, off_e, stride;
};

inline GemmGeom gemm_geom(int ni, int nl, int w) {
  GemmGeom g;
  g.ni = (ni + 1) & ~1;
  g.nl = (nl + 1) & ~1;
  g.w = w;
  size_t o = 8;
  g.off_feat = o; o += 4 * (size_t)g.ni;
  g.off_thr = o;  o += 4 * (size_t)g.ni;
  g.off_lm = o;   o += 8 * (size_t)g.nl;
  g.off_rm = o;   o += 8 * (size_t)g.nl;
  g.off_d = o;    o += 4 * (size_t)g.nl;
  g.off_e = o;    o += 4 * (size_t)g.nl * w;
  g.stride = (o + 15) & ~size_t(15);
  return g;
}


// ---- GEMM strategy, tensor-core kernel (hb_gemm_tc.cu)
constexpr int kTcPairs = 8;                 // pairs of trees per group
constexpr int kTcTrees = 2 * kTcPairs;      // 16 trees per group
constexpr int kTcCols = 16 * kTcPairs;      // TMEM columns per group
constexpr int kTcRows = 128;                // rows per CTA tile (UMMA M)
constexpr float kTcDPad = 99.f;             // unreachable D for padded leaf columns

// Group record (SMEM image), all offsets 16-B aligned:
//   bimg  [kTcPairs][512 B]   B operand: per pair 16 (N) x 16 (K) bf16, K-major
//                             core matrices (8 rows x 16 B), LBO = 128, SBO = 256
//   feat  [kTcTrees][8] u32   feature id of internal node i (pads: 0)
//   thr   [kTcTrees][8] f32   threshold (pads: +Inf)
//   dval  [kTcTrees][8] f32   D_j (pads: 99)
//   tout  [kTcTrees]    u32   tree_output
//   e     [kTcTrees][8][w] f32
struct TcGeom {
  int w;
  size_t off_b, off_feat, off_thr, off_d, off_tout, off_e, stride;
};

inline TcGeom tc_geom(int w) {
  TcGeom g;
  g.w = w;
  size_t o = 0;
  g.off_b = o;    o += 512 * kTcPairs;
  g.off_feat = o; o += 4 * 8 * kTcTrees;
  g.off_thr = o;  o += 4 * 8 * kTcTrees;
  g.off_d = o;    o += 4 * 8 * kTcTrees;
  g.off_tout = o; o += 4 * kTcTrees;
  g.off_e = o;    o += 4 * 8 * (size_t)kTcTrees * w;
  g.stride = (o + 127) & ~size_t(127);
  return g;
}


// gemm_tc_kernel SMEM: two A tiles (kTcPairs K-slabs of 4 KB each), reused
// at the tile end as the scratch of the 4-part per-row reduction (fp64 sums
// + leaf hash per part and row)
inline size_t gemm_tc_a_region(int nacc) {
  const size_t a = 2 * (size_t)kTcPairs * 4096, red = 4 * (size_t)kTcRows * (8 * (size_t)nacc + 8);
  return a > red ? a : red;
}

// ---- rank-code pre-pass (hb_rank_codes.cu)
constexpr uint32_t kRcSmemMax = 200 * 1024;  // largest per-CTA table budget
// TMA pre-pass (hb_rank_codes.cu rank_code_tma_kernel): per-warp rings of
// kRcTmaStages boxes of kRcTmaU x 32 rows x 16 B next to the group's tables
constexpr int kRcTmaWarps = 16;
constexpr int kRcTmaU = 2;
constexpr int kRcTmaStages = 3;
constexpr uint32_t kRcTmaStageBytes = kRcTmaU * 32 * 16;
constexpr uint32_t kRcTmaRingBytes = kRcTmaWarps * kRcTmaStages * (kRcTmaStageBytes + 16);
constexpr uint32_t kRcTmaTableMax = 227 * 1024 - kRcTmaRingBytes - 128;

// ---- wide-row TT (hb_tt.cu)
// SMEM of tt_wide_kernel for R rows: X tile + fp64 per-warp row sums + hashes
inline size_t tt_wide_smem(int F, int R, int nwarps, int nacc) {
  return ((((size_t)F * R + 1) & ~(size_t)1) * 4) + (size_t)nwarps * R * (8 * (size_t)nacc + 8);
}

}  // namespace hb
