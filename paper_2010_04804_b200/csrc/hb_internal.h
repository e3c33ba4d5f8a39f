// hb_internal.h — model object, compiled layouts and kernel entry points of
// libhb.so. Not part of the ABI (include/hb.h is).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "hb.h"

namespace hb {

constexpr int kMaxOutputs = 16;       // NACC upper bound of the fused epilogue
constexpr int kPttMaxDepth = 10;      // P:308 "PTT when D <= 10"; template range 0..10
constexpr int kTreeGroup = 4;         // trees walked concurrently per lane (ILP)
constexpr int kSmemBudget = 227 * 1024 - 2048;

// Kernel launch configuration chosen at compile time from F and the per-tree
// record size.
struct LaunchCfg {
  int nw = 16;          // compute warps per CTA (32 rows each)
  int ns = 2;           // tree-chunk pipeline stages
  int ch = 2;           // trees per chunk (multiple of kTreeGroup)
  int x_smem = 1;       // X row tile staged in SMEM (feature-major per warp)
  int t_smem = 1;       // tree chunks staged in SMEM via cp.async.bulk
  int smem_bytes = 0;   // dynamic SMEM per CTA
  int ctas_per_sm = 1;
  int wide_rows = 0;    // TT only: >0 selects tt_wide_kernel with this many rows per CTA
  int stage_bytes = 0;  // PTT rank layout: bytes per ring stage
  int prefetch = 1;     // producer warms L2 with the next tile's X rows
};

struct Model {
  int device = 0;
  int strategy = HB_STRATEGY_PTT;
  int depth = 0;            // D_max of this model's trees
  int n_trees = 0;          // real trees in this model
  int n_trees_pad = 0;      // padded to a multiple of kTreeGroup (zero trees)
  int tree_begin = 0;
  int n_trees_total = 0;
  int n_features = 0;
  int n_outputs = 0;
  int leaf_width = 1;
  int cmp = 0, agg = 0, post = 0, task = 0;
  int nacc = 1;             // accumulator template bucket >= n_outputs

  // compiled layout
  size_t stride = 0;        // bytes per tree record (multiple of 16)
  int nslots = 0;           // PTT: 2^D leaf slots; TT: max node count
  void *d_trees = nullptr;  // n_trees_pad * stride bytes
  int32_t *d_leafmap = nullptr;   // [n_trees_pad * nslots] original node id
  float *d_scale = nullptr; // [K]: 1/ntrees_k (MEAN) or 1 (SUM)
  float *d_base = nullptr;  // [K]
  // GEMM-only tensors (Table 3 form, see hb_gemm.cu)
  void *d_gemm = nullptr;
  size_t gemm_bytes = 0;
  int gemm_ni = 0, gemm_nl = 0;
  int gemm_tc = 0;          // 1: tensor-core (tcgen05) GEMM kernel
  // PTT with rank-coded thresholds (hb_pttr.cu)
  int ptt_rank = 0;
  int rank_cw = 32;          // code cell width (32 or 16 bits)
  int rank_rpl = 1;          // rows per lane of pttr_kernel (2: top levels shared by two rows)
  void *d_aux = nullptr;    // [fmeta | groups | eytzinger pool]
  size_t aux_groups_off = 0, aux_pool_off = 0;
  int rank_nfc = 0, rank_ngroups = 0;
  // rank-code pre-pass (hb_rank_codes.cu): codes computed by a separate launch
  // into a per-call scratch buffer (stream-ordered pool), scorer ring carries
  // tree chunks only
  int rank_pre = 0;
  int rank_nwords = 0;       // 32-bit code words per row (n_fc or ceil(n_fc / 2))
  void *d_rb = nullptr;      // [feat | groups | bucket tables]
  size_t rb_groups_off = 0, rb_pool_off = 0, rb_smem = 0, rb_smem_cap = 0;
  int rb_ngroups = 0;
  uint32_t rb_max_span = 0;  // widest X column span of a table group (staged pre-pass)
  bool rb_global = false;    // some table group is searched from global memory
  // groups are runs of consecutive X columns inside one aligned 4-column
  // block (rank_code_tma_kernel: one 16-B TMA box per row); widest group
  int rb_tma = 0, rb_max_feats = 0;
  cudaMemPool_t mempool = nullptr;   // per-call scratch (rank codes, TT chunk partials)

  // small-batch path (hb_small.cu): PTT fp32 or TT records walked by
  // trees-across-threads; may alias d_trees / d_leafmap
  const void *sb_trees = nullptr;
  const int32_t *sb_leafmap = nullptr;
  void *sb_own_trees = nullptr;
  int32_t *sb_own_leafmap = nullptr;
  size_t sb_stride = 0;
  int sb_nslots = 0, sb_tt = 0, sb_depth = 0;
  int sb_nrec = 0;                    // records in sb_trees (PTT: class-ordered, padded)
  const int32_t *sb_fmap = nullptr;   // feature map of the small-batch records
  int sb_nxf = 0;
  int small_max = 0;                  // n_rows <= small_max -> small-batch kernel

  // feature-selection injection: fp32 PTT / TT records index a
  // compacted X tile holding only the model's used features
  int32_t *d_fmap = nullptr;   // [n_xf] compact column -> original feature (null: identity)
  int n_xf = 0;

  int tt_chunk = 0;          // tt_wide_kernel: trees per L2-resident chunk (0: one launch)
  int tt_g = 4;              // tt_wide_kernel: concurrent walks per lane (4; 6, 8 for K = 1)
  // tt_wide_kernel records (hb_host.cpp build_ttw): packed trees of 16-B
  // internal-node records + per-tree offsets in 16-B units
  void *d_ttw = nullptr;
  uint32_t *d_ttw_off = nullptr;
  size_t ttw_bytes = 0;
  size_t ttw_rec_bytes = 0;  // node-record bytes the walk reads (sum over trees)

  size_t device_bytes = 0;
  LaunchCfg cfg;
  // host-only compile (compile_model_host, the ASan/UBSan fuzz build): every
  // "device" buffer is host memory (malloc) and no CUDA call is made
  bool host_only = false;
};

// thread-local error text
void set_error(const std::string &s);
hb_status fail(hb_status st, const std::string &s);
hb_status cuda_fail(cudaError_t e, const char *what);

// arguments of one scoring launch
struct RunArgs {
  const float *X;
  int64_t n, ldx;
  int kind;                 // hb_output
  void *out;
  cudaStream_t stream;
  const float *raw_in;      // finalize only: fp32 raw sums (hb_finalize)
  const double *raw_in64 = nullptr;   // finalize only: fp64 raw sums (hb_finalize64, tree chunks)
  // hb_predict_ex_events: caller events recorded on `stream` at the start of
  // every launch and after the last one (per-kernel durations, no sync)
  cudaEvent_t *ev = nullptr;
  int nev = 0;
  int *ev_k = nullptr;
  cudaError_t *ev_err = nullptr;   // first cudaEventRecord failure of the call
};

// record the next profiling event of a call (no-op without events)
inline void mark_launch(const RunArgs &a) {
  if (a.ev && a.ev_k && *a.ev_k < a.nev) {
    const cudaError_t e = cudaEventRecord(a.ev[(*a.ev_k)++], a.stream);
    if (e != cudaSuccess && a.ev_err && *a.ev_err == cudaSuccess) *a.ev_err = e;
  }
}

bool gemm_supported(int depth);
hb_status compile_gemm(const hb_ensemble *e, int t0, int t1, Model *m);
bool gemm_tc_eligible(const hb_ensemble *e, int t0, int t1);
hb_status compile_gemm_tc(const hb_ensemble *e, int t0, int t1, Model *m);
hb_status launch_gemm_tc(const Model &m, const RunArgs &a);
// record order of the PTT layouts (hb_host.cpp ptt_order)
struct TreeOrder {
  std::vector<int> local;   // per record: local tree id (t - t0), -1 = zero tree
  std::vector<int> cls;     // per record: output class
};
TreeOrder ptt_order(const hb_ensemble *e, int t0, int t1, bool by_class);
uint32_t ptt_header(const TreeOrder &o, size_t r);
hb_status compile_ptt_rank(const hb_ensemble *e, int t0, int t1, int D, Model *m, int nw_fp32);
hb_status launch_ptt_rank(const Model &m, const RunArgs &a);
// rank-code pre-pass tables (hb_rank_codes.cu)
struct RankBuckets {
  std::vector<uint32_t> feat;     // [n_fc][8] {f, B, S, start off, lo, hi, s, u off}
  std::vector<uint32_t> groups;   // [n_groups][8] {pool off, bytes, word_begin, word_end,
                                  //                col_lo, ncols, staged pitch, 0}
  std::vector<uint8_t> pool;
  int n_groups = 0, n_words = 0;
  size_t max_group_bytes = 0;     // largest SMEM-resident group
  size_t smem_cap = 0;            // groups up to this size are staged in SMEM
  uint32_t max_span = 0;          // widest X column span of one group
  bool any_global = false;        // some group's table exceeds the cap (searched from global memory)
  int max_feats = 0;              // most features in one group
  bool block4_ok = true;          // every group is consecutive columns inside one 4-column block
};
hb_status build_rank_buckets(const std::vector<std::vector<float>> &sorted, const std::vector<int> &orig,
                             int cw, RankBuckets *out, size_t cap_bytes = 0, int density = 0,
                             bool one_per_group = false, bool block4 = false);
hb_status launch_rank_codes(const Model &m, const RunArgs &a, uint32_t *codes, int64_t nblocks);

hb_status launch_ptt(const Model &m, const RunArgs &a);
hb_status launch_tt(const Model &m, const RunArgs &a);
hb_status launch_gemm(const Model &m, const RunArgs &a);
hb_status launch_finalize(const Model &m, const RunArgs &a);
hb_status launch_small_batch(const Model &m, const RunArgs &a);
// copy a compiled layout to the model's device (host memory for host-only
// models); accounts the bytes in m->device_bytes
hb_status dev_upload(Model *m, const void *src, size_t bytes, void **dst);
// the whole compile (validation, strategy, layouts) without a GPU, for the
// sanitizer fuzz build; the model's buffers are host memory
hb_status compile_model_host(const hb_ensemble *e, int t0, int t1, int strategy, Model **out);
void free_model_any(Model *m);
// model-owned stream-ordered scratch (hb_host.cpp): a pool created at compile
// time with release threshold UINT64_MAX, so per-call allocations reuse warm
// memory; under stream capture the device default pool is used instead
hb_status ensure_pool(Model *m);
hb_status scratch_alloc(const Model &m, size_t bytes, cudaStream_t s, void **p);

}  // namespace hb
