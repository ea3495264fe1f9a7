// imgio.cu -- device side of the image I/O path (reference: gridwave/imgio.py).
//
// Files are read into pinned host memory, copied to HBM as raw bytes and
// decoded here, so a whole-slide PGM goes disk -> PCIe -> HBM without a host
// pass over the samples:
//   * iwpp_pgm_decode  P5 raster -> samples (imgio.py:62-110): 8-bit copy,
//                      16-bit big-endian byte swap, maxval 1 -> {0, 255};
//                      the largest raw sample is returned for the
//                      "sample exceeds maxval" check (imgio.py:105-106);
//   * iwpp_pgm_encode  samples -> P5 raster (imgio.py:113-130);
//   * iwpp_gen_marker  max(mask - h, 0) (imgio.py:216-228);
//   * iwpp_quantize_u8 the CLI's quantized EDT view min(rint(d), 255)
//                      (cli.py:98-101).
// All are HBM-streaming kernels: 16 bytes per thread per iteration, grid =
// a multiple of the SM count.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "iwpp_common.cuh"

namespace iwpp {
namespace io {

constexpr int kThreads = 256;

static int grid_for(int64_t units) {
  const int64_t per = kThreads;
  int64_t g = (units + per - 1) / per;
  const int64_t cap = (int64_t)device_sm_count() * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

__device__ __forceinline__ void block_max_to(unsigned v, unsigned *out) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// 8-bit samples: 16 per thread-iteration
__global__ void decode8_kernel(uint8_t *dst, const uint8_t *src, int64_t n, int binary,
                               unsigned *maxv) {
  const int64_t n16 = n >> 4;
  unsigned m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 w = reinterpret_cast<const uint4 *>(src)[i];
    unsigned *u = reinterpret_cast<unsigned *>(&w);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const unsigned x = u[k];
      m = max(m, max(max(x & 0xffu, (x >> 8) & 0xffu), max((x >> 16) & 0xffu, x >> 24)));
      if (binary) {
        // nonzero byte -> 0xff: OR-fold each byte onto its low bit, spread
        unsigned nz = x | (x >> 4);
        nz |= nz >> 2;
        nz |= nz >> 1;
        nz &= 0x01010101u;
        u[k] = nz * 0xffu;
      }
    }
    reinterpret_cast<uint4 *>(dst)[i] = w;
  }
  for (int64_t i = (n16 << 4) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned x = src[i];
    m = max(m, x);
    dst[i] = binary ? (x ? 0xffu : 0u) : (uint8_t)x;
  }
  block_max_to(m, maxv);
}

// 16-bit big-endian samples: 8 per thread-iteration
__global__ void decode16_kernel(uint16_t *dst, const uint8_t *src, int64_t n, unsigned *maxv) {
  const int64_t n8 = n >> 3;
  unsigned m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 w = reinterpret_cast<const uint4 *>(src)[i];
    unsigned *u = reinterpret_cast<unsigned *>(&w);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const unsigned x = __byte_perm(u[k], 0, 0x2301);  // swap the bytes of each half
      u[k] = x;
      m = max(m, max(x & 0xffffu, x >> 16));
    }
    reinterpret_cast<uint4 *>(dst)[i] = w;
  }
  for (int64_t i = (n8 << 3) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned x = ((unsigned)src[2 * i] << 8) | src[2 * i + 1];
    m = max(m, x);
    dst[i] = (uint16_t)x;
  }
  block_max_to(m, maxv);
}

__global__ void encode16_kernel(uint8_t *dst, const uint16_t *src, int64_t n) {
  const int64_t n8 = n >> 3;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 w = reinterpret_cast<const uint4 *>(src)[i];
    unsigned *u = reinterpret_cast<unsigned *>(&w);
#pragma unroll
    for (int k = 0; k < 4; k++) u[k] = __byte_perm(u[k], 0, 0x2301);
    reinterpret_cast<uint4 *>(dst)[i] = w;
  }
  for (int64_t i = (n8 << 3) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    dst[2 * i] = (uint8_t)(src[i] >> 8);
    dst[2 * i + 1] = (uint8_t)src[i];
  }
}

template <typename T>
__global__ void marker_int_kernel(T *out, const T *mask, int64_t n, long long h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = (long long)mask[i] - h;
    out[i] = (T)(v > 0 ? v : 0);
  }
}

// np.maximum(a - float32(h), float32(0)): NaN propagates; ties keep the
// first operand (so -0.0 stays -0.0)
__global__ void marker_f32_kernel(float *out, const float *mask, int64_t n, float h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float d = mask[i] - h;
    out[i] = (d >= 0.f || d != d) ? d : 0.f;
  }
}

// np.minimum(np.rint(d), 255).astype(uint8) for finite d >= 0
__global__ void quantize_u8_kernel(uint8_t *out, const float *d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float r = fminf(rintf(d[i]), 255.f);
    out[i] = (uint8_t)(r > 0.f ? r : 0.f);
  }
}

}  // namespace io
}  // namespace iwpp

using namespace iwpp;

extern "C" {

int iwpp_pgm_decode(void *dst, const void *raster, int64_t n, int bytes_per_sample, int binary,
                    void *workspace, int64_t *max_sample_host, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || (bytes_per_sample != 1 && bytes_per_sample != 2) ||
      (binary && bytes_per_sample != 1))
    return set_error(IWPP_E_CONTRACT, "pgm_decode: bad arguments (n=%lld, bytes=%d, binary=%d)",
                     (long long)n, bytes_per_sample, binary);
  if ((uintptr_t)dst % 16 || (uintptr_t)raster % 16)
    return set_error(IWPP_E_CONTRACT, "pgm_decode: buffers must be 16-byte aligned");
  unsigned *maxv = (unsigned *)workspace;
  IWPP_CUDA_TRY(cudaMemsetAsync(maxv, 0, sizeof *maxv, st));
  if (n > 0) {
    if (bytes_per_sample == 1)
      io::decode8_kernel<<<io::grid_for((n >> 4) + 1), io::kThreads, 0, st>>>(
          (uint8_t *)dst, (const uint8_t *)raster, n, binary, maxv);
    else
      io::decode16_kernel<<<io::grid_for((n >> 3) + 1), io::kThreads, 0, st>>>(
          (uint16_t *)dst, (const uint8_t *)raster, n, maxv);
    IWPP_CUDA_TRY(cudaGetLastError());
  }
  if (max_sample_host) {
    unsigned v = 0;
    IWPP_CUDA_TRY(cudaMemcpyAsync(&v, maxv, sizeof v, cudaMemcpyDeviceToHost, st));
    IWPP_CUDA_TRY(cudaStreamSynchronize(st));
    *max_sample_host = v;
  }
  return IWPP_OK;
}

int iwpp_pgm_encode(void *raster, const void *src, int64_t n, int bytes_per_sample, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || (bytes_per_sample != 1 && bytes_per_sample != 2))
    return set_error(IWPP_E_CONTRACT, "pgm_encode: bad arguments");
  if (n == 0) return IWPP_OK;
  if (bytes_per_sample == 1) {
    IWPP_CUDA_TRY(cudaMemcpyAsync(raster, src, (size_t)n, cudaMemcpyDeviceToDevice, st));
    return IWPP_OK;
  }
  if ((uintptr_t)raster % 16 || (uintptr_t)src % 16)
    return set_error(IWPP_E_CONTRACT, "pgm_encode: buffers must be 16-byte aligned");
  io::encode16_kernel<<<io::grid_for((n >> 3) + 1), io::kThreads, 0, st>>>(
      (uint8_t *)raster, (const uint16_t *)src, n);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int iwpp_gen_marker(void *marker, const void *mask, int64_t n, int dtype, double h, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || h < 0) return set_error(IWPP_E_CONTRACT, "h must be >= 0");
  if (n == 0) return IWPP_OK;
  const int g = io::grid_for(n);
  switch (dtype) {
    case IWPP_U8:
      io::marker_int_kernel<uint8_t><<<g, io::kThreads, 0, st>>>((uint8_t *)marker,
                                                                 (const uint8_t *)mask, n,
                                                                 (long long)h);
      break;
    case IWPP_U16:
      io::marker_int_kernel<uint16_t><<<g, io::kThreads, 0, st>>>((uint16_t *)marker,
                                                                  (const uint16_t *)mask, n,
                                                                  (long long)h);
      break;
    case IWPP_I32:
      io::marker_int_kernel<int32_t><<<g, io::kThreads, 0, st>>>((int32_t *)marker,
                                                                 (const int32_t *)mask, n,
                                                                 (long long)h);
      break;
    case IWPP_F32:
      io::marker_f32_kernel<<<g, io::kThreads, 0, st>>>((float *)marker, (const float *)mask, n,
                                                        (float)h);
      break;
    default:
      return set_error(IWPP_E_CONTRACT, "gen_marker: unsupported dtype %d", dtype);
  }
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int iwpp_quantize_u8(uint8_t *out, const float *dist, int64_t n, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0) return set_error(IWPP_E_CONTRACT, "quantize_u8: n < 0");
  if (n == 0) return IWPP_OK;
  io::quantize_u8_kernel<<<io::grid_for(n), io::kThreads, 0, st>>>(out, dist, n);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

}  // extern "C"
