// Instantiations of the rank-coded PTT scorer, 16-bit code cells, two rows per lane.
#include "hb_pttr_kernel.cuh"

namespace hb {
PttrFn pttr_fn16_rpl2(int D, bool le, int nacc) { return pttr_pick_rpl2<16>(D, le, nacc); }
}  // namespace hb
