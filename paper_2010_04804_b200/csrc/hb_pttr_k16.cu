// Instantiations of the rank-coded PTT scorer, 16-bit code cells.
#include "hb_pttr_kernel.cuh"

namespace hb {
PttrFn pttr_fn16(int D, bool le, int nacc) { return pttr_pick<16>(D, le, nacc); }
}  // namespace hb
