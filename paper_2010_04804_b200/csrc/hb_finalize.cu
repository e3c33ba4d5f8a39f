// hb_finalize.cu — stand-alone epilogue for raw sums that
// were produced elsewhere, e.g. tree-shard partials reduced with one NCCL
// reduce. Same arithmetic as the scorers' fused epilogue.
#include <cuda_runtime.h>

#include "hb_device.cuh"
#include "hb_internal.h"

namespace hb {

template <int NACC, typename RawT>
__global__ void finalize_kernel(const RawT *__restrict__ raw, int64_t n, int K, int task, int post,
                                int kind, const float *__restrict__ scale,
                                const float *__restrict__ base, void *out) {
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = k < K ? (double)raw[row * K + k] : 0.0;
    dev::write_row<NACC>(kind, acc, K, task, post, scale, base, row, out);
  }
}

int sm_count(int device);

hb_status launch_finalize(const Model &m, const RunArgs &a) {
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((a.n + threads - 1) / threads,
                                           (int64_t)sm_count(m.device) * 8);
  // raw sums in fp32 (hb_finalize) or fp64 (hb_finalize64, tree-chunk partials)
  auto go = [&](auto fn, auto *raw) {
    fn<<<(int)blocks, threads, 0, a.stream>>>(raw, a.n, m.n_outputs, m.task, m.post, a.kind,
                                             m.d_scale, m.d_base, a.out);
  };
  if (a.raw_in64) {
    switch (m.nacc) {
      case 1: go(finalize_kernel<1, double>, a.raw_in64); break;
      case 4: go(finalize_kernel<4, double>, a.raw_in64); break;
      case 8: go(finalize_kernel<8, double>, a.raw_in64); break;
      default: go(finalize_kernel<16, double>, a.raw_in64); break;
    }
  } else {
    switch (m.nacc) {
      case 1: go(finalize_kernel<1, float>, a.raw_in); break;
      case 4: go(finalize_kernel<4, float>, a.raw_in); break;
      case 8: go(finalize_kernel<8, float>, a.raw_in); break;
      default: go(finalize_kernel<16, float>, a.raw_in); break;
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "finalize_kernel launch");
  return HB_OK;
}

}  // namespace hb
