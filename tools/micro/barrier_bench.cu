// Grid-barrier microbenchmark (148 co-resident CTAs): the library's
// volatile-spin barrier vs cooperative_groups grid.sync vs an
// acquire/release barrier with backoff.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ void bar_volatile(unsigned* count, unsigned* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x;
    volatile unsigned* vg = gen;
    const unsigned g = *vg;
    __threadfence();
    if (atomicAdd(count, 1u) == nb - 1) {
      *count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vg == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
// Sense-free counting barrier: the counter only grows; CTA waits until it
// reaches the next multiple of nb.
__device__ __forceinline__ void bar_acqrel(unsigned* count, unsigned& epoch, int sleep) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x;
    epoch += nb;
    atom_add_release(count, 1u);
    while (ld_acquire(count) < epoch) {
      if (sleep) __nanosleep(sleep);
    }
  }
  __syncthreads();
}

__global__ void k_volatile(unsigned* b, int iters) {
  for (int i = 0; i < iters; ++i) bar_volatile(b, b + 1);
}
__global__ void k_cg(int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
}
__global__ void k_acqrel(unsigned* b, int iters, int sleep) {
  unsigned epoch = 0;
  for (int i = 0; i < iters; ++i) bar_acqrel(b, epoch, sleep);
}

int main() {
  unsigned* b;
  cudaMalloc(&b, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int threads : {256, 512}) {
    for (int variant = 0; variant < 5; ++variant) {
      cudaMemset(b, 0, 64);
      int it = iters;
      int sleep = variant == 3 ? 32 : (variant == 4 ? 100 : 0);
      void* a0[] = {&b, &it};
      void* a1[] = {&it};
      void* a2[] = {&b, &it, &sleep};
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(b, 0, 64);
        cudaEventRecord(e0);
        if (variant == 0) cudaLaunchCooperativeKernel((void*)k_volatile, sms, threads, a0, 0, 0);
        if (variant == 1) cudaLaunchCooperativeKernel((void*)k_cg, sms, threads, a1, 0, 0);
        if (variant >= 2) cudaLaunchCooperativeKernel((void*)k_acqrel, sms, threads, a2, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("threads %d variant %d (%s) : %.3f us per barrier (%s)\n", threads, variant,
             variant == 0 ? "volatile" : variant == 1 ? "cg.sync" : variant == 2 ? "acqrel" : "acqrel+sleep",
             ms * 1000.f / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
