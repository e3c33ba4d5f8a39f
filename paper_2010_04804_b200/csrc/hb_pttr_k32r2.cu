// Instantiations of the rank-coded PTT scorer, 32-bit code cells, two rows per lane.
#include "hb_pttr_kernel.cuh"

namespace hb {
PttrFn pttr_fn32_rpl2(int D, bool le, int nacc) { return pttr_pick_rpl2<32>(D, le, nacc); }
}  // namespace hb
