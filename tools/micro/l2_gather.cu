// Microbenchmark: achievable L2->SM bandwidth for K1's access pattern -- warps
// reading random 512-byte row segments (float4 per lane) of an L2-resident
// panel -- against the same volume streamed sequentially.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2_gather.cu -o l2_gather
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

template <int kB>
__global__ void gather(const float* __restrict__ y, const uint32_t* __restrict__ idx, uint64_t nidx,
                       uint32_t rows, uint32_t n, float* out) {
  const int lane = threadIdx.x & 31;
  float4 acc = make_float4(0, 0, 0, 0);
  const uint64_t w0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t t = w0 * kB; t < nidx; t += nw * kB) {
    float4 v[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      const uint32_t k = idx[(t + q) % nidx];
      v[q] = __ldg(reinterpret_cast<const float4*>(y + size_t(k) * n) + lane);
    }
#pragma unroll
    for (int q = 0; q < kB; ++q) {
      acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w;
    }
  }
  if (acc.x == 123.f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
  const uint32_t rows = 16384;
  for (uint32_t n : {128u, 15000u, 60000u, 60032u}) {  // row stride (floats); 128 columns read
  const uint64_t nidx = 1 << 24;
  float* y; uint32_t* idx; float* out;
  cudaMalloc(&y, size_t(rows) * n * 4);
  cudaMemset(y, 0, size_t(rows) * n * 4);
  if (n == 128u) cudaMalloc(&idx, nidx * 4);
  if (n == 128u) cudaMalloc(&out, 4);
  std::vector<uint32_t> h(nidx);
  uint64_t s = 88172645463325252ull;
  for (auto& x : h) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = uint32_t(s % rows); }
  cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSm : {6, 8}) {
    for (int kb : {1, 2, 4}) {
      auto run = [&] {
        if (kb == 1) gather<1><<<sms * blocksPerSm, 256>>>(y, idx, nidx, rows, n, out);
        if (kb == 4) gather<4><<<sms * blocksPerSm, 256>>>(y, idx, nidx, rows, n, out);
        if (kb == 2) gather<2><<<sms * blocksPerSm, 256>>>(y, idx, nidx, rows, n, out);
      };
      run();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      const double bytes = double(nidx) * 512;
      printf("stride %6u blocks/SM %2d batch %d: %.3f ms  %.2f TB/s (random 512 B row segments, 16384 rows)\n",
             n, blocksPerSm, kb, ms, bytes / ms / 1e9);
    }
  }
  cudaFree(y);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
