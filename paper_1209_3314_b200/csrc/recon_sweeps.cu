// recon_sweeps.cu -- full-image scan sweeps, seed scan and contract check.
//
// Row sweeps (K.115-139 recon_rows_forward/backward): the recurrence
//   J'[x] = max(J[x], min(J'[x-1], I[x])) = clamp(J'[x-1], J[x], I[x])
// is a composition of clamp functions f_x(v) = min(I_x, max(J_x, v)), and
// clamps are closed under composition:
//   g o f = (clamp(l_f, l_g, h_g), clamp(h_f, l_g, h_g)).
// So one warp computes a whole row sweep exactly with a shuffle scan over
// (l, h) pairs -- fully parallel instead of the reference's sequential walk,
// with 16-byte vector loads per lane.  Forward and backward passes run in
// one kernel; the backward pass re-reads the row from L2.
//
// Seed scan (K.193-217): active pixels (p can raise a neighbour q:
// J(q) < J(p) and J(q) < I(q)) emitted with warp-aggregated compaction.

#include <climits>

#include "iwpp_common.cuh"
#include "recon_sweeps.cuh"

namespace iwpp {
namespace recon {

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(hi, max(lo, v)); }

template <typename T>
struct VecLoad {
  static constexpr int V = 16 / sizeof(T);
};

template <typename T, bool VEC>
__device__ __forceinline__ void load_seg(const T *Jr, const T *Ir, int x0, int W, int (&j)[VecLoad<T>::V],
                                         int (&m)[VecLoad<T>::V]) {
  constexpr int V = VecLoad<T>::V;
  if (VEC && x0 + V <= W) {
    uint4 a = __ldcg(reinterpret_cast<const uint4 *>(Jr + x0));
    uint4 b = __ldg(reinterpret_cast<const uint4 *>(Ir + x0));
    const T *pa = reinterpret_cast<const T *>(&a);
    const T *pb = reinterpret_cast<const T *>(&b);
#pragma unroll
    for (int e = 0; e < V; e++) {
      j[e] = (int)pa[e];
      m[e] = (int)pb[e];
    }
  } else {
#pragma unroll
    for (int e = 0; e < V; e++) {
      int x = x0 + e;
      if (x < W) {
        j[e] = (int)Jr[x];
        m[e] = (int)Ir[x];
      } else {
        j[e] = INT_MIN;  // identity clamp
        m[e] = INT_MAX;
      }
    }
  }
}

template <typename T, bool VEC>
__device__ __forceinline__ void store_seg(T *Jr, int x0, int W, const int (&j)[VecLoad<T>::V]) {
  constexpr int V = VecLoad<T>::V;
  if (VEC && x0 + V <= W) {
    uint4 a;
    T *pa = reinterpret_cast<T *>(&a);
#pragma unroll
    for (int e = 0; e < V; e++) pa[e] = (T)j[e];
    *reinterpret_cast<uint4 *>(Jr + x0) = a;
  } else {
#pragma unroll
    for (int e = 0; e < V; e++)
      if (x0 + e < W) Jr[x0 + e] = (T)j[e];
  }
}

template <typename T, bool VEC>
__global__ void __launch_bounds__(256) row_sweep_kernel(T *__restrict__ J, const T *__restrict__ I,
                                                        int W, int H, int dirs,
                                                        unsigned long long *changed) {
  constexpr int V = VecLoad<T>::V;
  constexpr int SEG = 32 * V;
  const unsigned FULL = 0xffffffffu;
  int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (row >= H) return;
  T *Jr = J + (size_t)row * W;
  const T *Ir = I + (size_t)row * W;
  int j[V], m[V];
  bool ch = false;
  // forward (west neighbour)
  int carry = INT_MIN;
  for (int s0 = 0; s0 < W && (dirs & 1); s0 += SEG) {
    int x0 = s0 + lane * V;
    load_seg<T, VEC>(Jr, Ir, x0, W, j, m);
    int l = INT_MIN, h = INT_MAX;
#pragma unroll
    for (int e = 0; e < V; e++) {
      l = clampi(l, j[e], m[e]);
      h = clampi(h, j[e], m[e]);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int ol = __shfl_up_sync(FULL, l, o), oh = __shfl_up_sync(FULL, h, o);
      if (lane >= o) {
        int nl = clampi(ol, l, h), nh = clampi(oh, l, h);
        l = nl;
        h = nh;
      }
    }
    int el = __shfl_up_sync(FULL, l, 1), eh = __shfl_up_sync(FULL, h, 1);
    if (lane == 0) {
      el = INT_MIN;
      eh = INT_MAX;
    }
    int v = clampi(carry, el, eh);
#pragma unroll
    for (int e = 0; e < V; e++) {
      v = clampi(v, j[e], m[e]);
      ch |= v != j[e];
      j[e] = v;
    }
    store_seg<T, VEC>(Jr, x0, W, j);
    carry = __shfl_sync(FULL, v, 31);
  }
  __syncwarp();
  // backward (east neighbour)
  carry = INT_MIN;
  int nseg = (W + SEG - 1) / SEG;
  for (int si = nseg - 1; si >= 0 && (dirs & 2); si--) {
    int x0 = si * SEG + lane * V;
    load_seg<T, VEC>(Jr, Ir, x0, W, j, m);
    int l = INT_MIN, h = INT_MAX;
#pragma unroll
    for (int e = V - 1; e >= 0; e--) {
      l = clampi(l, j[e], m[e]);
      h = clampi(h, j[e], m[e]);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int ol = __shfl_down_sync(FULL, l, o), oh = __shfl_down_sync(FULL, h, o);
      if (lane + o < 32) {
        int nl = clampi(ol, l, h), nh = clampi(oh, l, h);
        l = nl;
        h = nh;
      }
    }
    int el = __shfl_down_sync(FULL, l, 1), eh = __shfl_down_sync(FULL, h, 1);
    if (lane == 31) {
      el = INT_MIN;
      eh = INT_MAX;
    }
    int v = clampi(carry, el, eh);
#pragma unroll
    for (int e = V - 1; e >= 0; e--) {
      v = clampi(v, j[e], m[e]);
      ch |= v != j[e];
      j[e] = v;
    }
    store_seg<T, VEC>(Jr, x0, W, j);
    carry = __shfl_sync(FULL, v, 0);
  }
  if (changed && __any_sync(FULL, ch) && lane == 0) *changed = 1;
}

// Column sweeps, vertical neighbour (K.142-190; the diagonal terms are left
// to the tile engine): per column the same clamp recurrence, computed
// exactly along full columns in three bandwidth-bound passes:
//   A. per (column, 64-row segment): the composite clamp (l, h) of the segment
//   B. per column: exclusive scan of the segment composites -> carry-in
//   C. per (column, segment): re-walk the segment from its carry-in
// Thread = one column, warp = 32 consecutive columns (coalesced rows).
constexpr int kColSeg = 64;

template <typename T, bool DOWN>
__global__ void __launch_bounds__(128) col_composite_kernel(const T *__restrict__ J,
                                                            const T *__restrict__ I, int W, int H,
                                                            int2 *__restrict__ comp) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, seg = blockIdx.y;
  if (x >= W) return;
  int y0 = seg * kColSeg, y1 = min(H, y0 + kColSeg);
  int l = INT_MIN, h = INT_MAX;  // identity
#pragma unroll 8
  for (int k = 0; k < y1 - y0; k++) {
    int y = DOWN ? y0 + k : y1 - 1 - k;
    size_t g = (size_t)y * W + x;
    int j = (int)__ldcg(J + g), m = (int)__ldg(I + g);
    l = clampi(l, j, m);  // f_y o (running composite)
    h = clampi(h, j, m);
  }
  comp[(size_t)seg * W + x] = make_int2(l, h);
}

template <bool DOWN>
__global__ void __launch_bounds__(128) col_carry_kernel(const int2 *__restrict__ comp, int W,
                                                        int nseg, int *__restrict__ carry) {
  int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  int v = INT_MIN;
  for (int k = 0; k < nseg; k++) {
    int seg = DOWN ? k : nseg - 1 - k;
    carry[(size_t)seg * W + x] = v;
    int2 c = comp[(size_t)seg * W + x];
    v = clampi(v, c.x, c.y);
  }
}

template <typename T, bool DOWN>
__global__ void __launch_bounds__(128) col_apply_kernel(T *__restrict__ J, const T *__restrict__ I,
                                                        int W, int H,
                                                        const int *__restrict__ carry) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, seg = blockIdx.y;
  if (x >= W) return;
  int y0 = seg * kColSeg, y1 = min(H, y0 + kColSeg);
  int v = carry[(size_t)seg * W + x];
#pragma unroll 8
  for (int k = 0; k < y1 - y0; k++) {
    int y = DOWN ? y0 + k : y1 - 1 - k;
    size_t g = (size_t)y * W + x;
    int j = (int)J[g];
    v = clampi(v, j, (int)__ldg(I + g));
    if (v != j) J[g] = (T)v;
  }
}

size_t col_scratch_bytes(int64_t W, int64_t H) {
  size_t nseg = (size_t)((H + kColSeg - 1) / kColSeg);
  return align_up(nseg * W * sizeof(int2), 256) + align_up(nseg * W * sizeof(int), 256);
}

template <typename T>
static int cols_impl(void *Jv, const void *Iv, int W, int H, void *scratch, cudaStream_t st) {
  T *J = (T *)Jv;
  const T *I = (const T *)Iv;
  int nseg = (H + kColSeg - 1) / kColSeg;
  Carver c(scratch);
  int2 *comp = c.take<int2>((size_t)nseg * W);
  int *carry = c.take<int>((size_t)nseg * W);
  dim3 g2((W + 127) / 128, nseg), g1((W + 127) / 128);
  col_composite_kernel<T, true><<<g2, 128, 0, st>>>(J, I, W, H, comp);
  col_carry_kernel<true><<<g1, 128, 0, st>>>(comp, W, nseg, carry);
  col_apply_kernel<T, true><<<g2, 128, 0, st>>>(J, I, W, H, carry);
  col_composite_kernel<T, false><<<g2, 128, 0, st>>>(J, I, W, H, comp);
  col_carry_kernel<false><<<g1, 128, 0, st>>>(comp, W, nseg, carry);
  col_apply_kernel<T, false><<<g2, 128, 0, st>>>(J, I, W, H, carry);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

template <typename T, int CONN>
__global__ void seed_scan_kernel(const T *__restrict__ J, const T *__restrict__ I, int W, int H,
                                 int64_t *__restrict__ out, unsigned long long *n_out) {
  const unsigned FULL = 0xffffffffu;
  size_t n = (size_t)W * H;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n;
       base += stride) {
    size_t p = base + (threadIdx.x & 31u);
    bool want = false;
    if (p < n) {
      int py = (int)(p / (unsigned)W), px = (int)(p - (size_t)py * W);
      int v = (int)J[p];
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
        if (qx >= 0 && qx < W && qy >= 0 && qy < H) {
          size_t q = (size_t)qy * W + qx;
          int vq = (int)J[q];
          if (vq < v && vq < (int)I[q]) want = true;
        }
      }
    }
    unsigned long long pos = warp_reserve(n_out, want ? 1u : 0u, FULL);
    if (want) out[pos] = (int64_t)p;
  }
}

template <typename T>
__global__ void check_le_kernel(const T *__restrict__ J, const T *__restrict__ I, size_t n,
                                unsigned long long *viol) {
  unsigned long long c = 0;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x)
    c += !(J[p] <= I[p]);  // a NaN anywhere is a violation (recon.py:60, np.all(m <= i))
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(viol, c);
}

// u8 fast path: 16 bytes per thread with byte-SIMD compares
__global__ void check_le_u8x16_kernel(const uint4 *__restrict__ J, const uint4 *__restrict__ I,
                                      size_t n16, unsigned long long *viol) {
  unsigned long long c = 0;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n16;
       p += (size_t)gridDim.x * blockDim.x) {
    uint4 a = __ldg(J + p), b = __ldg(I + p);
    // __vcmpgtu4: 0xff per byte where a > b
    c += __popc(__vcmpgtu4(a.x, b.x)) + __popc(__vcmpgtu4(a.y, b.y)) +
         __popc(__vcmpgtu4(a.z, b.z)) + __popc(__vcmpgtu4(a.w, b.w));
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(viol, c / 8);
}

static int grid_cap(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  size_t cap = (size_t)device_sm_count() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

template <typename T>
static int rows_impl(void *J, const void *I, int W, int H, cudaStream_t st, int dirs = 3,
                     unsigned long long *changed = nullptr) {
  constexpr int V = VecLoad<T>::V;
  bool vec = ((size_t)W * sizeof(T)) % 16 == 0 && ((uintptr_t)J % 16 == 0) && ((uintptr_t)I % 16 == 0);
  (void)V;
  int blocks = (H * 32 + 255) / 256;
  if (vec)
    row_sweep_kernel<T, true><<<blocks, 256, 0, st>>>((T *)J, (const T *)I, W, H, dirs, changed);
  else
    row_sweep_kernel<T, false><<<blocks, 256, 0, st>>>((T *)J, (const T *)I, W, H, dirs, changed);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int sweep_rows(void *J, const void *I, int W, int H, int dtype, cudaStream_t st, int dirs,
               unsigned long long *changed) {
  switch (dtype) {
    case IWPP_U8:
    case IWPP_BIN: return rows_impl<uint8_t>(J, I, W, H, st, dirs, changed);
    case IWPP_U16: return rows_impl<uint16_t>(J, I, W, H, st, dirs, changed);
    case IWPP_I32: return rows_impl<int32_t>(J, I, W, H, st, dirs, changed);
  }
  return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
}

int sweep_cols(void *J, const void *I, int W, int H, int dtype, void *scratch, cudaStream_t st) {
  switch (dtype) {
    case IWPP_U8:
    case IWPP_BIN: return cols_impl<uint8_t>(J, I, W, H, scratch, st);
    case IWPP_U16: return cols_impl<uint16_t>(J, I, W, H, scratch, st);
    case IWPP_I32: return cols_impl<int32_t>(J, I, W, H, scratch, st);
  }
  return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
}

int seed_scan(const void *J, const void *I, int W, int H, int dtype, int conn, int64_t *out,
              unsigned long long *n_out, cudaStream_t st) {
  size_t n = (size_t)W * H;
  int g = grid_cap(n, 256);
#define SS(T)                                                                                     \
  if (conn == 8)                                                                                  \
    seed_scan_kernel<T, 8><<<g, 256, 0, st>>>((const T *)J, (const T *)I, W, H, out, n_out);      \
  else                                                                                            \
    seed_scan_kernel<T, 4><<<g, 256, 0, st>>>((const T *)J, (const T *)I, W, H, out, n_out);
  switch (dtype) {
    case IWPP_U8:
    case IWPP_BIN: SS(uint8_t); break;
    case IWPP_U16: SS(uint16_t); break;
    case IWPP_I32: SS(int32_t); break;
    default: return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
  }
#undef SS
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int check_le(const void *J, const void *I, size_t n, int dtype, unsigned long long *viol,
             cudaStream_t st) {
  int g = grid_cap(n, 256);
  switch (dtype) {
    case IWPP_U8:
    case IWPP_BIN:
      if (n % 16 == 0 && (uintptr_t)J % 16 == 0 && (uintptr_t)I % 16 == 0)
        check_le_u8x16_kernel<<<grid_cap(n / 16, 256), 256, 0, st>>>((const uint4 *)J, (const uint4 *)I,
                                                                     n / 16, viol);
      else
        check_le_kernel<uint8_t><<<g, 256, 0, st>>>((const uint8_t *)J, (const uint8_t *)I, n, viol);
      break;
    case IWPP_U16: check_le_kernel<uint16_t><<<g, 256, 0, st>>>((const uint16_t *)J, (const uint16_t *)I, n, viol); break;
    case IWPP_I32: check_le_kernel<int32_t><<<g, 256, 0, st>>>((const int32_t *)J, (const int32_t *)I, n, viol); break;
    case IWPP_F32: check_le_kernel<float><<<g, 256, 0, st>>>((const float *)J, (const float *)I, n, viol); break;
    default: return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
  }
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

// f32 <-> order-preserving int32: non-negative floats keep their bits,
// negative floats flip the magnitude bits, so signed-int order = float order
// (the engines then run their int32 path: hardware atomicMax, same fixed
// point).  -0.0 maps to +0.0 (they compare equal as floats).  NaN never
// reaches the engine: the marker <= mask contract rejects it.
__global__ void f32_to_ord_kernel(const uint32_t *__restrict__ src, int32_t *__restrict__ dst,
                                  size_t n) {
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    uint32_t b = src[p];
    if (b == 0x80000000u) b = 0u;
    dst[p] = (int32_t)b >= 0 ? (int32_t)b : (int32_t)(b ^ 0x7FFFFFFFu);
  }
}
__global__ void ord_to_f32_kernel(const int32_t *__restrict__ src, uint32_t *__restrict__ dst,
                                  size_t n) {
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    int32_t v = src[p];
    dst[p] = v >= 0 ? (uint32_t)v : ((uint32_t)v ^ 0x7FFFFFFFu);
  }
}

int f32_to_ord(const void *src, void *dst, size_t n, cudaStream_t st) {
  f32_to_ord_kernel<<<grid_cap(n, 256), 256, 0, st>>>((const uint32_t *)src, (int32_t *)dst, n);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}
int ord_to_f32(const void *src, void *dst, size_t n, cudaStream_t st) {
  ord_to_f32_kernel<<<grid_cap(n, 256), 256, 0, st>>>((const int32_t *)src, (uint32_t *)dst, n);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

}  // namespace recon
}  // namespace iwpp
