// Microbenchmarks for the recon tile engine's candidate shared bottlenecks on
// B200 (development evidence, profiles/r02_ubench_limits.txt):
//   1. same-address atomics: every warp's lane 0 does returned atomicAdd /
//      fire-and-forget RED on ONE global word (the ring head / pending
//      counters of the tile queue);
//   2. box-pattern loads: every warp reads 34 rows x 64 bytes (or 96 bytes,
//      the sector footprint) at random 32x32-tile positions of a large u8
//      image -- the register engine's J + I staging, minus everything else.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench_engine_limits.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void atom_ret(unsigned *p, int iters, unsigned *sink) {
  unsigned acc = 0;
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < iters; i++) {
      unsigned v;
      asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(p) : "memory");
      acc += v;
    }
  if (acc == 0xdeadbeef) *sink = acc;
}
__global__ void atom_red(unsigned *p, int iters) {
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < iters; i++) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
// spread: each warp hits its own line (no contention) -- the latency floor
__global__ void atom_ret_spread(unsigned *p, int iters, unsigned *sink) {
  unsigned acc = 0;
  unsigned *q = p + 64 * (blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32);
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < iters; i++) {
      unsigned v;
      asm volatile("atom.relaxed.gpu.global.add.u32 %0, [%1], 1;" : "=r"(v) : "l"(q) : "memory");
      acc += v;
    }
  if (acc == 0xdeadbeef) *sink = acc;
}

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}
// each lane reads `bytes` of one box row (16-byte vector loads), 34 rows per
// tile for two images; tiles at random positions
__global__ void box_loads(const uint8_t *J, const uint8_t *I, int W, int H, int tiles_per_warp,
                          int bytes, unsigned *sink) {
  const int lane = threadIdx.x & 31;
  const unsigned wid = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int ntx = W / 32, nty = H / 32;
  unsigned acc = 0;
  for (int k = 0; k < tiles_per_warp; k++) {
    const unsigned t = hash32(wid * 7919u + k) % (unsigned)(ntx * nty);
    const int tx = t % ntx, ty = t / ntx;
    int x0 = tx * 32 - 16;
    if (x0 < 0) x0 = 0;
    if (x0 + bytes > W) x0 = W - bytes;
    for (int r = lane; r < 34; r += 32) {
      int y = ty * 32 - 1 + r;
      y = y < 0 ? 0 : (y >= H ? H - 1 : y);
      const uint4 *pj = reinterpret_cast<const uint4 *>(J + (size_t)y * W + x0);
      const uint4 *pi = reinterpret_cast<const uint4 *>(I + (size_t)y * W + x0);
      for (int c = 0; c < bytes / 16; c++) {
        uint4 a = __ldcg(pj + c), b = __ldcg(pi + c);
        acc += a.x ^ b.y ^ a.z ^ b.w;
      }
    }
  }
  if (acc == 0x12345678) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned *ctr, *sink;
  cudaMalloc(&ctr, 1 << 20);
  cudaMalloc(&sink, 64);
  cudaMemset(ctr, 0, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const int blocks = sms * 5, threads = 128, iters = 2000;
  const double nwarps = blocks * threads / 32.0;
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(a);
    atom_ret<<<blocks, threads>>>(ctr, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("same-address returned atomicAdd: %.0f warps x %d: %.3f ms -> %.3f G atomics/s, %.2f us/atomic/warp\n",
                    nwarps, iters, ms, nwarps * iters / ms * 1e-6, ms * 1e3 / iters);
    cudaEventRecord(a);
    atom_red<<<blocks, threads>>>(ctr, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("same-address RED.ADD:            %.0f warps x %d: %.3f ms -> %.3f G atomics/s\n", nwarps,
                    iters, ms, nwarps * iters / ms * 1e-6);
    cudaEventRecord(a);
    atom_ret_spread<<<blocks, threads>>>(ctr, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("per-warp-address returned atomic: %.0f warps x %d: %.3f ms -> %.3f G atomics/s, %.2f us/atomic/warp\n",
                    nwarps, iters, ms, nwarps * iters / ms * 1e-6, ms * 1e3 / iters);
  }
  for (int n : {4096, 16384, 65536}) {
    uint8_t *J, *I;
    size_t bytes = (size_t)n * n;
    if (cudaMalloc(&J, bytes) != cudaSuccess || cudaMalloc(&I, bytes) != cudaSuccess) {
      printf("alloc %d failed\n", n);
      return 1;
    }
    cudaMemset(J, 1, bytes);
    cudaMemset(I, 2, bytes);
    for (int bw : {32, 64, 96}) {
      const int tpw = n >= 65536 ? 400 : 100;
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        box_loads<<<blocks, threads>>>(J, I, n, n, tpw, bw, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      const double tiles = nwarps * tpw;
      printf("%5d^2 box loads %2d B/row: %.0f tiles in %.3f ms -> %.1f M tiles/s, useful %.0f GB/s (2 x 34 x %d B)\n",
             n, bw, tiles, ms, tiles / ms * 1e-3, tiles * 2 * 34 * bw / ms * 1e-6, bw);
    }
    cudaFree(J);
    cudaFree(I);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
