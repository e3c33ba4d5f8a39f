// synth_dev.cu — device twin of synth/xgen.py (same counter-based formula,
// written separately; tests check host == device bits). Input generation
// only: none of the scoring arithmetic lives here.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t sx_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void sx_gen_kernel(uint64_t seed, int64_t n, int F, int64_t ldx, int grid,
                              uint32_t special_q24, int64_t row_offset, float *out) {
  const int64_t total = n * (int64_t)F;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / F;
    const int f = (int)(idx - r * F);
    const uint64_t c = (uint64_t)(row_offset + r) * (uint64_t)F + (uint64_t)f;
    const uint64_t z = sx_mix64(seed * 0x9E3779B97F4A7C15ULL + c * 0xD1B54A32D192ED03ULL);
    float x;
    if (grid == 0) x = (float)((int)(z & 0xFFFFu) - 32768) * (1.0f / 4096.0f);
    else x = (float)((int)(z & 0x3Fu) - 32) * 0.25f;
    if (special_q24 && (z >> 40) < special_q24) {
      switch ((int)((z >> 16) % 5)) {
        case 0: x = __int_as_float(0x7FC00000); break;
        case 1: x = __int_as_float(0x7F800000); break;
        case 2: x = __int_as_float(0xFF800000); break;
        case 3: x = -0.0f; break;
        default: x = 0.0f; break;
      }
    }
    out[r * ldx + f] = x;
  }
}

extern "C" int hbsynth_gen_X(uint64_t seed, int64_t n, int F, int64_t ldx, int grid,
                             uint32_t special_q24, int64_t row_offset, float *out, void *stream) {
  if (n <= 0) return 0;
  if (ldx > F) cudaMemsetAsync(out, 0, (size_t)n * ldx * 4, (cudaStream_t)stream);
  const int64_t total = n * (int64_t)F;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  sx_gen_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(seed, n, F, ldx, grid, special_q24,
                                                              row_offset, out);
  return (int)cudaGetLastError();
}
