// iwpp_common.cuh -- shared device helpers for the sm_100a IWPP kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/iwpp_b200.h"

#define IWPP_CUDA_TRY(expr)                                                   \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) return iwpp::set_cuda_error(_e, #expr, __FILE__, __LINE__); \
  } while (0)

namespace iwpp {

int set_error(int status, const char *fmt, ...);
int set_cuda_error(cudaError_t e, const char *what, const char *file, int line);
int device_sm_count();

constexpr int kWarp = 32;

// Neighbourhoods in the reference's raster order (K.22-25).

// Offsets packed as 2-bit fields (value + 1) so a dynamic k never indexes
// a local array (which would spill to the stack).
template <int CONN>
struct Nbr;
template <>
struct Nbr<8> {
  static constexpr int N = 8;
  __device__ __forceinline__ static int dx(int k) { return (int)((0x9224u >> (2 * k)) & 3u) - 1; }
  __device__ __forceinline__ static int dy(int k) { return (int)((0xa940u >> (2 * k)) & 3u) - 1; }
};
template <>
struct Nbr<4> {
  static constexpr int N = 4;
  __device__ __forceinline__ static int dx(int k) { return (int)((0x61u >> (2 * k)) & 3u) - 1; }
  __device__ __forceinline__ static int dy(int k) { return (int)((0x94u >> (2 * k)) & 3u) - 1; }
};

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated reservation: every lane with `want` gets a distinct slot
// (returned), one atomicAdd per warp on `counter` (the TQ -> BQ/GBQ step of
// the paper's hierarchical queue).  Must be called by
// all lanes in `active`.
template <typename CounterT>
__device__ __forceinline__ CounterT warp_reserve(CounterT *counter, unsigned count,
                                                 unsigned active) {
  // inclusive scan of `count` across the active lanes
  unsigned lane = lane_id();
  unsigned incl = count;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned v = __shfl_up_sync(active, incl, o);
    if (lane >= (unsigned)o) incl += v;
  }
  unsigned total = __shfl_sync(active, incl, 31);
  CounterT base = 0;
  if (lane == 31 && total) base = atomicAdd(counter, (CounterT)total);
  base = __shfl_sync(active, base, 31);
  return base + (CounterT)(incl - count);
}

// L2-coherent loads/stores for data other CTAs mutate concurrently
// (L1 is not coherent across SMs).
template <typename T>
__device__ __forceinline__ T ld_cg(const T *p) {
  return __ldcg(p);
}
__device__ __forceinline__ uint8_t ld_cg(const uint8_t *p) {
  return (uint8_t)__ldcg((const unsigned char *)p);
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Acquire/release fence at GPU scope (MEMBAR.ALL.GPU): enough for the
// message-passing patterns of the engines (publish data, then a flag / queue
// slot; observe the flag, then read the data).  __threadfence() is a
// sequentially consistent fence (MEMBAR.SC.GPU), which is costlier.
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Predicated shared-memory atomics (no branch around the atomic, so a run of
// them issues back to back).  A predicated-off call returns INT_MAX (max) /
// all-ones (or), which callers treat as "no effect".
__device__ __forceinline__ int smem_atomic_max_if(int *p, int v, unsigned pred) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p);
  int old = 0x7fffffff;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q atom.shared.max.s32 %0, [%1], %2;\n\t}"
      : "+r"(old)
      : "r"(a), "r"(v), "r"(pred)
      : "memory");
  return old;
}
__device__ __forceinline__ unsigned smem_atomic_or_if(unsigned *p, unsigned v, unsigned pred) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p);
  unsigned old = 0xffffffffu;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q atom.shared.or.b32 %0, [%1], %2;\n\t}"
      : "+r"(old)
      : "r"(a), "r"(v), "r"(pred)
      : "memory");
  return old;
}

// Predicated global 64-bit atomicMin (predicated off: returns all-ones and
// touches nothing).
__device__ __forceinline__ unsigned long long gmem_atomic_min_if(unsigned long long *p,
                                                                 unsigned long long v,
                                                                 unsigned pred) {
  unsigned long long old = ~0ull;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q atom.global.min.u64 %0, [%1], %2;\n\t}"
      : "+l"(old)
      : "l"(p), "l"(v), "r"(pred)
      : "memory");
  return old;
}

// Element traits: the engines keep values as int32 in shared memory so the
// hardware atomicMax covers every element kind (u8/u16 widen losslessly).
template <typename T>
struct Elem;
template <>
struct Elem<uint8_t> {
  static constexpr int code = IWPP_U8;
  static constexpr uint8_t lo = 0;  // smallest value (the "outside" sentinel mask)
};
template <>
struct Elem<uint16_t> {
  static constexpr int code = IWPP_U16;
  static constexpr uint16_t lo = 0;
};
template <>
struct Elem<int32_t> {
  static constexpr int code = IWPP_I32;
  static constexpr int32_t lo = INT32_MIN;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Carve a caller-provided workspace into aligned pieces.
struct Carver {
  char *base;
  size_t off = 0;
  explicit Carver(void *b) : base((char *)b) {}
  template <typename T>
  T *take(size_t n) {
    off = align_up(off, 256);
    T *p = base ? (T *)(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
};

}  // namespace iwpp
