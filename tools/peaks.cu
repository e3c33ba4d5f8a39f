// peaks.cu — on-chip bandwidth microbenchmarks for the roofline denominators
// MEASURED_PEAKS.json lacks: shared-memory load bandwidth
// (conflict-free LDS.128, all SMs) and L2 read bandwidth (working set well
// inside L2). Not part of the scoring path; used by bench.py.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(1024, 1) smem_bw_kernel(int iters, float *sink) {
  extern __shared__ float4 buf[];
  const int n = 4096;  // 64 KB
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  float4 acc = make_float4(0, 0, 0, 0);
  int idx = threadIdx.x;
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    float4 v = buf[(idx + it * 32) & (n - 1)];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x + acc.y + acc.z + acc.w == -1.f) sink[threadIdx.x] = acc.x;
}

__global__ void l2_bw_kernel(const float4 *__restrict__ src, int64_t n4, int reps, float *sink) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(src + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  if (acc.x + acc.y + acc.z + acc.w == -1.f) sink[threadIdx.x] = acc.x;
}

static double time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// returns GB/s of shared-memory loads across the whole GPU (best of reps)
extern "C" double hbpeaks_smem_gbs(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float *sink;
  cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(smem_bw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int iters = 1 << 16;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  smem_bw_kernel<<<sms, 1024, 65536>>>(256, sink);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    smem_bw_kernel<<<sms, 1024, 65536>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    const double bytes = (double)sms * 1024 * iters * 16;
    best = fmax(best, bytes / (time_ms(a, b) * 1e-3) / 1e9);
  }
  cudaFree(sink);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

// L2 read bandwidth with a 32 MB working set read repeatedly.
extern "C" double hbpeaks_l2_gbs(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t bytes = 32ll << 20;
  float4 *src;
  float *sink;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 0, bytes);
  cudaMalloc(&sink, 4096);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 20;
  l2_bw_kernel<<<sms * 4, 512>>>(src, bytes / 16, 1, sink);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    l2_bw_kernel<<<sms * 4, 512>>>(src, bytes / 16, reps, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    best = fmax(best, (double)bytes * reps / (time_ms(a, b) * 1e-3) / 1e9);
  }
  cudaFree(src);
  cudaFree(sink);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
