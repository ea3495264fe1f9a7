// Grid-barrier micro-benchmark (B200): cost per barrier of the EDT engines'
// software grid barrier (edt.cuh grid_barrier) vs variants, for the round
// engines' launch shapes.  Development evidence (profiles/r02_ubench_barrier.txt).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_bar scripts/ubench_grid_barrier.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// variant 0: the engines' barrier (acq_rel arrival, release generation, 16 ns polls)
// variant 1: same, polls back off to 256 ns
// variant 2: cooperative_groups grid.sync()
// variant 3: two-level: CTAs arrive on one of 8 sub-counters (blockIdx % 8); the
//            last arriver of a sub-counter arrives on the root
template <int V>
__global__ void bar_kernel(unsigned *ctl, int iters) {
  unsigned *count = ctl, *gen = ctl + 64, *sub = ctl + 128;
  unsigned g = threadIdx.x == 0 ? ld_acquire(gen) : 0u;
  for (int i = 0; i < iters; i++) {
    if (V == 2) {
      cooperative_groups::this_grid().sync();
      continue;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      bool last = false;
      if (V == 3) {
        const unsigned ng = 8, k = blockIdx.x % ng;
        const unsigned members = (gridDim.x - k + ng - 1) / ng;
        unsigned a;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(a) : "l"(sub + 32 * k) : "memory");
        if (a == members - 1) {
          asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(sub + 32 * k) : "memory");
          unsigned b;
          asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(b) : "l"(count) : "memory");
          last = b == (gridDim.x < ng ? gridDim.x : ng) - 1;
        }
      } else {
        unsigned a;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(a) : "l"(count) : "memory");
        last = a == gridDim.x - 1;
      }
      if (last) {
        asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
      } else {
        unsigned ns = 16;
        while (ld_acquire(gen) == g) {
          __nanosleep(ns);
          if (V == 1 && ns < 256) ns *= 2;
        }
      }
      g++;
    }
    __syncthreads();
  }
}

template <int V>
float run(int blocks, int threads, unsigned *ctl, int iters) {
  void *args[] = {&ctl, &iters};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  for (int rep = 0; rep < 2; rep++) {
    cudaMemset(ctl, 0, 4096);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void *)bar_kernel<V>, dim3(blocks), dim3(threads), args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  return ms * 1000.f / iters;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *ctl;
  cudaMalloc(&ctl, 4096);
  const int iters = 2000;
  for (auto shape : {std::pair<int, int>{4, 256}, {2, 512}, {1, 1024}, {1, 256}}) {
    const int blocks = sms * shape.first, threads = shape.second;
    printf("%4d CTAs x %4d threads: engines' barrier %.2f us | backoff %.2f us | cg grid.sync %.2f us | two-level %.2f us\n",
           blocks, threads, run<0>(blocks, threads, ctl, iters), run<1>(blocks, threads, ctl, iters),
           run<2>(blocks, threads, ctl, iters), run<3>(blocks, threads, ctl, iters));
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
