// hb_device.cuh — device helpers shared by the scoring kernels: mbarrier /
// cp.async.bulk (TMA bulk-copy engine) wrappers and the fused epilogue.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hb.h"

// Device-side bounds checks of the checked build (libhb_checked.so, -DHB_CHECKED;
// DESIGN.md §7.1): a failed check prints its site and traps, so the launch
// fails with cudaErrorLaunchFailure. Compiled out of the product library.
#ifdef HB_CHECKED
#include <cstdio>
#define HB_DCHECK(c)                                                                  \
  do {                                                                                \
    if (!(c)) {                                                                       \
      printf("HB_DCHECK failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                      \
      __trap();                                                                       \
    }                                                                                 \
  } while (0)
#else
#define HB_DCHECK(c) ((void)0)
#endif

namespace hb {
namespace dev {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Consumer release of a ring stage that the TMA engine will overwrite: every
// consumer thread orders its own generic-proxy reads of the stage before the
// async-proxy writes of the next fill (fence.proxy.async) and arrives on the
// stage's `empty` barrier (release semantics), which the producer acquires
// before issuing the next cp.async.bulk into the stage. The barrier counts
// kRingArrivals(nw) = 32 arrivals per consumer warp (each reading thread
// signals for itself, as CUTLASS's PipelineTmaAsync consumers do; an elected
// lane after __syncwarp is equivalent under the memory model but invisible to
// compute-sanitizer racecheck, which then reported the ring reuse).
__device__ __forceinline__ void release_stage(uint64_t *bar, int lane) {
  (void)lane;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}

__device__ __forceinline__ constexpr uint32_t ring_arrivals(int nw) { return 32u * (uint32_t)nw; }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared through the TMA engine; completion is
// signalled on `bar` as transaction bytes (SASS: UBLKCP).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Explicit 32-bit shared-memory loads (volatile: the ring buffers are
// rewritten by the TMA engine between mbarrier phases, so they must not be
// hoisted or merged across iterations; ILP comes from manual interleaving).
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

__device__ __forceinline__ void sts_u32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}

// Warm L2 with the X rows of a CTA's next row tile (TMA bulk prefetch, no
// SMEM, no completion tracking); [first, first + rows) rows of stride ldx.
__device__ __forceinline__ void prefetch_rows_l2(const float *X, int64_t first, int64_t rows,
                                                 int64_t n, int64_t ldx) {
  if (first >= n) return;
  rows = min(rows, n - first);
  const char *a = reinterpret_cast<const char *>(X + first * ldx);
  const char *b = reinterpret_cast<const char *>(X + (first + rows) * ldx);
  const char *p = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15));
  while (p < b) {
    const int64_t left = ((int64_t)(b - p) + 15) & ~int64_t(15);
    const uint32_t bytes = (uint32_t)(left < 65536 ? left : 65536);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
    p += bytes;
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Position in an NS-stage mbarrier ring (stage index + phase parity),
// advanced incrementally: no 64-bit division in the hot loops.
struct Ring {
  int s = 0;
  uint32_t ph = 0;
  int ns;
  __device__ __forceinline__ explicit Ring(int n) : ns(n) {}
  __device__ __forceinline__ void next() {
    if (++s == ns) {
      s = 0;
      ph ^= 1u;
    }
  }
};

// Per-lane X row staging: lane `lane` of a warp owns row `row`; the warp's
// slice is feature-major xs[f * 32 + lane] so that every later data-dependent
// read X[row, f] hits bank `lane` (conflict-free whatever f each lane needs).
__device__ __forceinline__ void load_x_slice(float *xs, const float *__restrict__ X, int64_t row,
                                             int64_t n, int64_t ldx, int F, int lane, bool vec4) {
  if (row < n) {
    const float *xr = X + row * ldx;
    int f = 0;
    if (vec4) {
      // 8 independent 16-B loads in flight per lane before their stores: the
      // slice waits one memory latency per 32 columns, not per 4 (wide rows,
      // e.g. the Fig. 8 shape's 200 columns, are load-latency bound otherwise)
      for (; f + 32 <= F; f += 32) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const float4 *>(xr + f + 4 * u));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          xs[(f + 4 * u + 0) * 32 + lane] = v[u].x;
          xs[(f + 4 * u + 1) * 32 + lane] = v[u].y;
          xs[(f + 4 * u + 2) * 32 + lane] = v[u].z;
          xs[(f + 4 * u + 3) * 32 + lane] = v[u].w;
        }
      }
      for (; f + 4 <= F; f += 4) {
        float4 v = __ldg(reinterpret_cast<const float4 *>(xr + f));
        xs[(f + 0) * 32 + lane] = v.x;
        xs[(f + 1) * 32 + lane] = v.y;
        xs[(f + 2) * 32 + lane] = v.z;
        xs[(f + 3) * 32 + lane] = v.w;
      }
    }
    for (; f < F; ++f) xs[f * 32 + lane] = __ldg(xr + f);
  } else {
    for (int f = 0; f < F; ++f) xs[f * 32 + lane] = 0.f;
  }
}

// Same, for a compacted feature set (feature-selection injection):
// slice column c holds X[row, fmap[c]] for the model's used features only.
__device__ __forceinline__ void load_x_slice_map(float *xs, const float *__restrict__ X, int64_t row,
                                                 int64_t n, int64_t ldx,
                                                 const int32_t *__restrict__ fmap, int nx, int lane) {
  const float *xr = X + (row < n ? row : 0) * ldx;
  for (int c = 0; c < nx; ++c) xs[c * 32 + lane] = row < n ? __ldg(xr + __ldg(fmap + c)) : 0.f;
}

// Fused epilogue for one row (a10/a11 of SURVEY §8; P:192 reduction, Table 2
// P:117 transforms). The accumulators are fp64 (every scorer sums its fp32
// leaf values in fp64), so the margin m_k = acc_k / div_k + base_k is formed
// in fp64 as in the oracle and rounded once; labels take the argmax of the
// fp64 margins; softmax exponentiates the fp64 differences m_k - max_j m_j.
template <int NACC>
__device__ __forceinline__ void write_row(int kind, const double (&acc)[NACC], int K, int task,
                                          int post, const float *__restrict__ scale /* divisor: ntrees_k (MEAN) or 1 */,
                                          const float *__restrict__ base, int64_t row, void *out) {
  if (kind == HB_OUT_RAW) {
    float *o = static_cast<float *>(out) + row * K;
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      if (k < K) o[k] = (float)acc[k];
    return;
  }
  if (kind == HB_OUT_RAW64) {
    double *o = static_cast<double *>(out) + row * K;
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      if (k < K) o[k] = acc[k];
    return;
  }
  double m[NACC];
#pragma unroll
  for (int k = 0; k < NACC; ++k)
    m[k] = (k < K) ? acc[k] / (double)__ldg(scale + k) + (double)__ldg(base + k) : 0.0;
  if (kind == HB_OUT_MARGIN) {
    float *o = static_cast<float *>(out) + row * K;
#pragma unroll
    for (int k = 0; k < NACC; ++k)
      if (k < K) o[k] = (float)m[k];
    return;
  }
  if (kind == HB_OUT_PREDICT && task == HB_TASK_CLASSIFICATION) {
    int32_t lab = 0;
    if (K == 1) {
      lab = m[0] > 0.0 ? 1 : 0;
    } else {
      double best = m[0];
#pragma unroll
      for (int k = 1; k < NACC; ++k)
        if (k < K && m[k] > best) { best = m[k]; lab = k; }
    }
    static_cast<int32_t *>(out)[row] = lab;
    return;
  }
  // post transform (PREDICT for regression, PROBA for classification)
  float p[NACC];
  if (post == HB_POST_SIGMOID) {
#pragma unroll
    for (int k = 0; k < NACC; ++k) p[k] = 1.f / (1.f + expf(-(float)m[k]));
  } else if (post == HB_POST_SOFTMAX) {
    double mx = m[0];
#pragma unroll
    for (int k = 1; k < NACC; ++k)
      if (k < K) mx = fmax(mx, m[k]);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NACC; ++k) {
      p[k] = (k < K) ? expf((float)(m[k] - mx)) : 0.f;
      s += p[k];
    }
#pragma unroll
    for (int k = 0; k < NACC; ++k) p[k] = p[k] / s;
  } else if (post == HB_POST_ISOLATION) {
    // 2^(-mean path length / c(psi)); c(psi) is stored after the K base scores
    const double c = (double)__ldg(base + K);
#pragma unroll
    for (int k = 0; k < NACC; ++k) p[k] = exp2f((float)(-m[k] / c));
  } else {
#pragma unroll
    for (int k = 0; k < NACC; ++k) p[k] = (float)m[k];
  }
  if (kind == HB_OUT_PROBA && K == 1) {
    float2 v = make_float2(1.f - p[0], p[0]);
    reinterpret_cast<float2 *>(out)[row] = v;
    return;
  }
  float *o = static_cast<float *>(out) + row * K;
#pragma unroll
  for (int k = 0; k < NACC; ++k)
    if (k < K) o[k] = p[k];
}

}  // namespace dev
}  // namespace hb
