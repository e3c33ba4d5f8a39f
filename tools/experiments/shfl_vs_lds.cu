// Do warp shuffles and shared-memory loads share one per-SM data pipe?
// A: N LDS per thread; B: N SHFL.idx; C: N LDS + N SHFL interleaved (independent).
// If C ~ max(A, B) they use separate pipes; if C ~ A + B they contend.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(1024) k(int iters, unsigned *out) {
  __shared__ unsigned s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  unsigned a = lane, b = lane * 7, c = lane * 3, d = lane * 5;
  unsigned v = lane * 13;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE != 1) {
        a = s[(a & 127) * 32 + lane];      // conflict-free LDS, bank = lane
        b = s[(b & 127) * 32 + lane];
      }
      if (MODE != 0) {
        c = __shfl_sync(0xffffffffu, v + c, (c + lane) & 31);
        d = __shfl_sync(0xffffffffu, v ^ d, (d ^ lane) & 31);
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
int main() {
  unsigned *out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 2;
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<blocks, 1024>>>(iters, out);
      if (mode == 1) k<1><<<blocks, 1024>>>(iters, out);
      if (mode == 2) k<2><<<blocks, 1024>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 2.0 * 8 * iters * blocks * 1024 / 32;   // warp-instr per kind
      printf("mode %s: %.3f ms, %.3f warp-ops/clk/SM per kind @1.965GHz\n",
             mode == 0 ? "LDS     " : mode == 1 ? "SHFL    " : "LDS+SHFL", ms,
             ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  return 0;
}
