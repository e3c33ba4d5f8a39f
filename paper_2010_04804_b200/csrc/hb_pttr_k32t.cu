// Instantiations of the rank-coded PTT scorer, 32-bit code cells, with the
// opt-in LDS.128 top-of-tree load (HB_PTTR_TOP=1).
#include "hb_pttr_kernel.cuh"

namespace hb {
PttrFn pttr_fn32_top(int D, bool le, int nacc) { return pttr_pick<32, true>(D, le, nacc); }
}  // namespace hb
