// Peak fp64 throughput on this GPU: DMMA (mma.sync m8n8k4 f64) vs DFMA, and
// a fragment-layout check of m8n8k4 against a scalar product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void dmma_loop(double* out, int iters) {
  double c[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) dmma(c[q], a, b);
  double s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double c[16] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 16; ++q) c[q] = fma(a, b, c[q]);
  double s = 0;
  for (int q = 0; q < 16; ++q) s += c[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// layout check: A 8x4 row-major, B 4x8 (col-major "col"), C 8x8
__global__ void layout(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a = A[g * 4 + t];      // row g, k t
  double b = B[t * 8 + g];      // k t, col g
  double c[2] = {0, 0};
  dmma(c, a, b);
  C[g * 8 + 2 * t] = c[0];
  C[g * 8 + 2 * t + 1] = c[1];
}

int main() {
  double *out, *A, *B, *C;
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  cudaMallocManaged(&A, 32 * 8);
  cudaMallocManaged(&B, 32 * 8);
  cudaMallocManaged(&C, 64 * 8);
  for (int i = 0; i < 32; ++i) A[i] = i + 1, B[i] = 0.5 * i - 3;
  layout<<<1, 32>>>(A, B, C);
  cudaDeviceSynchronize();
  double err = 0;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int k = 0; k < 4; ++k) s += A[i * 4 + k] * B[k * 8 + j];
      err += fabs(s - C[i * 8 + j]);
    }
  printf("m8n8k4 layout check: abs err %g\n", err);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int threads : {256, 512}) {
      cudaEventRecord(e0);
      dmma_loop<<<148 * (1024 / threads), threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 256.0 * 8 * iters * (148.0 * 1024 / 32);
      printf("DMMA %d thr: %.1f TFLOP/s\n", threads, flops / ms / 1e9);
      cudaEventRecord(e0);
      dfma_loop<<<148 * (1024 / threads), threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double f2 = 2.0 * 16 * iters * (148.0 * 1024);
      printf("DFMA %d thr: %.1f TFLOP/s\n", threads, f2 / ms / 1e9);
    }
  }
  return 0;
}
