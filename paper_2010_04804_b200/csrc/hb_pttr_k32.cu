// Instantiations of the rank-coded PTT scorer, 32-bit code cells.
#include "hb_pttr_kernel.cuh"

namespace hb {
PttrFn pttr_fn32(int D, bool le, int nacc) { return pttr_pick<32>(D, le, nacc); }
}  // namespace hb
