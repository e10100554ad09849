// L2 gather-bandwidth probe (diagnostic): warps read 128-byte segments at
// random segment indices out of a working set of W bytes, which is first
// touched once so it sits in L2 when W < L2.  Reports GB/s delivered to the
// SMs for W in 8 MB .. 512 MB.  Models the decoder's band pass (each output
// 128-B segment gathers ~19 neighbour segments).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__global__ void gather_k(const float4* __restrict__ data, const int* __restrict__ idx, long long nidx,
                         float* out) {
  // each lane reads 16 B of a 128-B segment: 8 lanes per segment, 4 segments per warp instr
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long long s = warp * 4; s < nidx; s += nw * 4) {
    int seg = __ldg(idx + s + (lane >> 3));
    float4 v = __ldcg(data + (long long)seg * 8 + (lane & 7));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const long long nidx = 1ll << 27;  // 128 M segment reads = 16 GB
  int* idx;
  cudaMalloc(&idx, nidx * 4);
  float4* data;
  const long long maxW = 512ll << 20;
  cudaMalloc(&data, maxW);
  cudaMemset(data, 0, maxW);
  float* out;
  cudaMalloc(&out, 4);
  std::vector<int> h(nidx);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (long long W : {8ll << 20, 16ll << 20, 32ll << 20, 48ll << 20, 64ll << 20, 96ll << 20, 128ll << 20, 512ll << 20}) {
    const int nseg = (int)(W / 128);
    std::mt19937 rng(7);
    for (long long i = 0; i < nidx; ++i) h[i] = rng() % nseg;
    cudaMemcpy(idx, h.data(), nidx * 4, cudaMemcpyHostToDevice);
    for (int blocks : {148 * 4, 148 * 8}) {
      gather_k<<<blocks, 256>>>(data, idx, nidx, out);
      cudaEventRecord(a);
      gather_k<<<blocks, 256>>>(data, idx, nidx, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("W=%4lld MB blocks=%d: %.3f ms, gathered %.1f GB/s (+idx %.1f GB/s)\n", W >> 20, blocks, ms,
             nidx * 128.0 / ms / 1e6, nidx * 4.0 / ms / 1e6);
    }
  }
  return 0;
}
