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

// Dependent random 16-B gathers through the read-only path (the access
// pattern of a tree walk whose records come from L2: every load's address
// depends on the previous load). Each thread runs G independent chains over
// a random single-cycle permutation of a `bytes` buffer (L2-resident when
// bytes << L2) for `steps` steps, the chains of a thread issued back to back
// like tt_wide_kernel's G walks. Launch shape = tt_wide_kernel's (one
// 1024-thread CTA per SM). Returns dependent loads per second.
template <int G>
__global__ void __launch_bounds__(1024, 1) l2_chase_kernel(const uint4 *__restrict__ buf, uint32_t n,
                                                           int steps, uint32_t *sink) {
  uint32_t idx[G];
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int g = 0; g < G; ++g) idx[g] = (t * 2654435761u + (uint32_t)g * 40503u) % n;
  for (int s = 0; s < steps; ++s) {
#pragma unroll
    for (int g = 0; g < G; ++g) idx[g] = __ldg(buf + idx[g]).x;
  }
  uint32_t acc = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) acc ^= idx[g];
  if (acc == 0xFFFFFFFFu) sink[threadIdx.x] = acc;
}

extern "C" double hbpeaks_l2_chase(int device, long long bytes, int chains) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const uint32_t n = (uint32_t)(bytes / 16);
  // single random cycle (Sattolo's shuffle), LCG-driven: every chain visits
  // the whole buffer in random order
  uint32_t *next = (uint32_t *)malloc((size_t)n * 4);
  for (uint32_t i = 0; i < n; ++i) next[i] = i;
  uint64_t z = 0x9E3779B97F4A7C15ull;
  for (uint32_t i = n - 1; i > 0; --i) {
    z = z * 6364136223846793005ull + 1442695040888963407ull;
    const uint32_t j = (uint32_t)((z >> 33) % i);
    const uint32_t tmp = next[i]; next[i] = next[j]; next[j] = tmp;
  }
  uint4 *h = (uint4 *)malloc((size_t)n * 16);
  for (uint32_t i = 0; i < n; ++i) h[i] = make_uint4(next[i], i, 0, 0);
  uint4 *buf;
  uint32_t *sink;
  cudaMalloc(&buf, (size_t)n * 16);
  cudaMemcpy(buf, h, (size_t)n * 16, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 4096);
  free(next);
  free(h);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int steps = 2048;
  auto launch = [&](int s) {
    if (chains >= 8) l2_chase_kernel<8><<<sms, 1024>>>(buf, n, s, sink);
    else if (chains >= 4) l2_chase_kernel<4><<<sms, 1024>>>(buf, n, s, sink);
    else if (chains >= 2) l2_chase_kernel<2><<<sms, 1024>>>(buf, n, s, sink);
    else l2_chase_kernel<1><<<sms, 1024>>>(buf, n, s, sink);
  };
  launch(64);
  double best = 0;
  const int g = chains >= 8 ? 8 : chains >= 4 ? 4 : chains >= 2 ? 2 : 1;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a);
    launch(steps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    const double loads = (double)sms * 1024 * g * steps;
    best = fmax(best, loads / (time_ms(a, b) * 1e-3));
  }
  cudaFree(buf);
  cudaFree(sink);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
