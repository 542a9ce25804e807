// Shared-memory counter updates at random words: ATOMS.ADD with its result used
// (K7's form) against RED-style (result unused) and against conflict-free
// addresses.  One warp per block, 8 KB accumulators, as K7 runs them.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o atoms_vs_red atoms_vs_red.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int MODE>  // 0 atom (result used), 1 red, 2 atom conflict-free, 3 red conflict-free
__global__ void __launch_bounds__(32) k(uint32_t iters, uint32_t* out) {
  __shared__ uint32_t acc[2048];
  const int lane = threadIdx.x;
  for (int t = lane; t < 2048; t += 32) acc[t] = 0;
  __syncwarp();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(acc);
  uint32_t cr = 0, h = mix(blockIdx.x * 977u + lane);
  for (uint32_t i = 0; i < iters; ++i) {
    uint32_t a[8];
    h = h * 1664525u + 1013904223u;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      // one cheap address per update (a rotate + a mask), so the loop is not issue-bound
      uint32_t w = __funnelshift_r(h, h, 3 * j + 1) & (2047u << 2);
      if (MODE >= 2) w = (w & ~(31u << 2)) | (lane << 2);  // lane-distinct banks
      a[j] = base + w;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t d = 1u;
      if (MODE == 0 || MODE == 2) {
        uint32_t old;
        asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(a[j]), "r"(d) : "memory");
        cr |= old;
      } else {
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[j]), "r"(d) : "memory");
      }
    }
  }
  __syncwarp();
  uint32_t s = cr;
  for (int t = lane; t < 2048; t += 32) s += acc[t];
  if (s == 0x12345678u) out[0] = s;
}

template <int MODE>
float run(uint32_t iters, uint32_t* out, int blocks) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<blocks, 32>>>(iters, out);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 32>>>(iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  uint32_t* out; cudaMalloc(&out, 4);
  const int blocks = 148 * 16; const uint32_t iters = 4096;
  const double n = double(blocks) * iters * 8 * 32;
  const char* names[4] = {"atom random", "red random", "atom conflict-free", "red conflict-free"};
  float ms[4] = {run<0>(iters, out, blocks), run<1>(iters, out, blocks), run<2>(iters, out, blocks), run<3>(iters, out, blocks)};
  for (int i = 0; i < 4; ++i)
    printf("%-20s %.3f ms  %.1f G updates/s  %.2f cycles per warp instruction per SM (1.965 GHz)\n", names[i], ms[i], n / ms[i] / 1e6,
           ms[i] * 1e-3 * 1.965e9 * 148 / (n / 32));
  return 0;
}
