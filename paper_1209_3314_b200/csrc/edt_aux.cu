// edt_aux.cu -- the EDT's public helpers on the device:
//
//  * init_packed / edt_init (edt.py:187-202): vr = own index on background,
//    INF (-1) on foreground (K.edt_assign, K.339-347), plus the contour seeds
//    -- background cells with an in-bounds foreground neighbour -- compacted
//    in raster order (K.edt_contour_seeds, K.350-373).  Ordered compaction in
//    three passes over 2048-pixel chunks: count, scan the chunk counts, write.
//  * edt_exact_bruteforce (edt.py:313-323, oracles.bruteforce_sqdist,
//    oracles.py:57-73): the exact squared Euclidean distance to the nearest
//    background cell.  The reference minimises over every background cell
//    (quadratic); the same minimum is computed here by the separable exact
//    transform (Meijster et al.): a column pass gives each cell's vertical
//    distance g to the nearest background cell of its column, a row pass
//    takes the lower envelope of the parabolas (x - i)^2 + g(i)^2.  Integer
//    arithmetic throughout, so the result is the exact minimum, identical to
//    brute force (tests/test_gpu_edt.py checks both against each other).
#include <stdint.h>

#include "iwpp_common.cuh"

namespace iwpp {
namespace edtaux {

constexpr int kChunk = 2048;        // pixels per chunk (one CTA)
constexpr int kThreads = 256;       // 8 consecutive pixels per thread
constexpr int kPer = kChunk / kThreads;

template <int CONN>
__device__ __forceinline__ bool is_contour(const uint8_t *__restrict__ mask, int W, int H, int x,
                                           int y) {
  if (mask[(size_t)y * W + x] != 0) return false;
#pragma unroll
  for (int k = 0; k < Nbr<CONN>::N; k++) {
    const int nx = x + Nbr<CONN>::dx(k), ny = y + Nbr<CONN>::dy(k);
    if (nx >= 0 && nx < W && ny >= 0 && ny < H && mask[(size_t)ny * W + nx] != 0) return true;
  }
  return false;
}

// per-thread flags of its 8 pixels (bit i = pixel base + i is a seed)
template <int CONN>
__device__ __forceinline__ unsigned chunk_flags(const uint8_t *__restrict__ mask, int W, int H,
                                                size_t n, size_t base) {
  unsigned f = 0;
#pragma unroll
  for (int i = 0; i < kPer; i++) {
    const size_t p = base + i;
    if (p < n) {
      const int y = (int)(p / (size_t)W), x = (int)(p - (size_t)y * W);
      if (is_contour<CONN>(mask, W, H, x, y)) f |= 1u << i;
    }
  }
  return f;
}

// exclusive block scan of one value per thread (kThreads), returns the total
__device__ __forceinline__ unsigned block_excl_scan(unsigned v, unsigned &total) {
  __shared__ unsigned warp_sums[kThreads / 32];
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (unsigned)o) incl += t;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  unsigned off = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; w++) {
    const unsigned s = warp_sums[w];
    off += (unsigned)w < wid ? s : 0u;
    tot += s;
  }
  __syncthreads();
  total = tot;
  return off + incl - v;
}

template <int CONN>
__global__ void __launch_bounds__(kThreads) contour_count_kernel(const uint8_t *__restrict__ mask,
                                                                 int W, int H,
                                                                 unsigned *__restrict__ counts) {
  const size_t n = (size_t)W * H;
  const size_t base = (size_t)blockIdx.x * kChunk + (size_t)threadIdx.x * kPer;
  const unsigned c = __popc(chunk_flags<CONN>(mask, W, H, n, base));
  unsigned total;
  block_excl_scan(c, total);
  if (threadIdx.x == 0) counts[blockIdx.x] = total;
}

// exclusive scan of the chunk counts in one CTA (1024 threads, each a
// contiguous run); offsets[nchunks] = the total
__global__ void __launch_bounds__(1024) chunk_scan_kernel(const unsigned *__restrict__ counts,
                                                          long long nchunks,
                                                          unsigned long long *__restrict__ offsets) {
  __shared__ unsigned long long part[1024];
  const long long per = (nchunks + 1023) / 1024;
  const long long lo = (long long)threadIdx.x * per, hi = min(nchunks, lo + per);
  unsigned long long s = 0;
  for (long long i = lo; i < hi; i++) s += counts[i];
  part[threadIdx.x] = s;
  __syncthreads();
  // Hillis-Steele over the 1024 partial sums
  for (int o = 1; o < 1024; o <<= 1) {
    unsigned long long t = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0ull;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  unsigned long long run = part[threadIdx.x] - s;
  for (long long i = lo; i < hi; i++) {
    offsets[i] = run;
    run += counts[i];
  }
  if (threadIdx.x == 1023) offsets[nchunks] = part[1023];
}

template <int CONN>
__global__ void __launch_bounds__(kThreads) init_write_kernel(const uint8_t *__restrict__ mask,
                                                              int W, int H,
                                                              const unsigned long long *__restrict__ offsets,
                                                              int64_t *__restrict__ vr,
                                                              int64_t *__restrict__ seeds) {
  const size_t n = (size_t)W * H;
  const size_t base = (size_t)blockIdx.x * kChunk + (size_t)threadIdx.x * kPer;
  const unsigned f = chunk_flags<CONN>(mask, W, H, n, base);
  unsigned total;
  const unsigned off = block_excl_scan(__popc(f), total);
  if (vr) {
#pragma unroll
    for (int i = 0; i < kPer; i++) {
      const size_t p = base + i;
      if (p < n) vr[p] = mask[p] == 0 ? (int64_t)p : (int64_t)-1;
    }
  }
  if (seeds) {
    unsigned long long o = offsets[blockIdx.x] + off;
    for (unsigned g = f; g; g &= g - 1) seeds[o++] = (int64_t)(base + (unsigned)__ffs(g) - 1);
  }
}

// ---------------------------------------------------------------- exact EDT

constexpr int32_t kInfG = 1 << 30;

// column pass: g[y][x] = |y - nearest background row in column x| (kInfG if
// the column has none).  One thread per column; rows are coalesced across
// the warp.
__global__ void exact_cols_kernel(const uint8_t *__restrict__ mask, int W, int H,
                                  int32_t *__restrict__ g) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  int32_t d = kInfG;
  for (int y = 0; y < H; y++) {
    const size_t p = (size_t)y * W + x;
    d = mask[p] == 0 ? 0 : (d >= kInfG ? kInfG : d + 1);
    g[p] = d;
  }
  d = g[(size_t)(H - 1) * W + x];
  for (int y = H - 2; y >= 0; y--) {
    const size_t p = (size_t)y * W + x;
    const int32_t here = g[p];
    d = d >= kInfG ? kInfG : d + 1;
    if (d < here) g[p] = d;
    else d = here;
  }
}

__device__ __forceinline__ long long floor_div(long long a, long long b) {  // b > 0
  long long q = a / b;
  return (a % b != 0 && a < 0) ? q - 1 : q;
}

// row pass: lower envelope of f_i(u) = (u - i)^2 + g(i)^2 over the columns
// i with finite g (one thread per row).  The stack of (segment start t,
// parabola index s) is kept in the row's own d2 output: entry q is never
// needed after cell u >= t[q] >= q is written (t is strictly increasing from
// 0), and the scan reads entry q into registers before writing cell u.
__global__ void exact_rows_kernel(const int32_t *__restrict__ g, int W, int H,
                                  int64_t *__restrict__ d2, float *__restrict__ dist) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y >= H) return;
  const int32_t *gr = g + (size_t)y * W;
  int64_t *row = d2 + (size_t)y * W;
  auto f = [&](long long u, long long i, long long gi) { return (u - i) * (u - i) + gi * gi; };
  int q = -1;
  long long sq = 0, tq = 0, gsq = 0;  // top of the stack, cached
  for (int u = 0; u < W; u++) {
    const long long gu = gr[u];
    if (gu >= kInfG) continue;
    while (q >= 0 && f(tq, sq, gsq) > f(tq, u, gu)) {
      q--;
      if (q >= 0) {
        const uint64_t e = (uint64_t)row[q];
        sq = (long long)(e >> 32);
        tq = (long long)(e & 0xffffffffu);
        gsq = gr[sq];
      }
    }
    if (q < 0) {
      q = 0;
      sq = u, tq = 0, gsq = gu;
      row[0] = (int64_t)(((uint64_t)u << 32) | 0u);
    } else {
      const long long w = 1 + floor_div(u * (long long)u - sq * sq + gu * gu - gsq * gsq, 2 * (u - sq));
      if (w < W) {
        q++;
        sq = u, tq = w, gsq = gu;
        row[q] = (int64_t)(((uint64_t)u << 32) | (uint64_t)w);
      }
    }
  }
  if (q < 0) {  // no background anywhere (caller reports NO_BACKGROUND)
    for (int u = 0; u < W; u++) {
      row[u] = (int64_t)1 << 62;
      if (dist) dist[(size_t)y * W + u] = __double2float_rn(__dsqrt_rn((double)((int64_t)1 << 62)));
    }
    return;
  }
  for (int u = W - 1; u >= 0; u--) {
    const long long d = f(u, sq, gsq);
    const bool pop = u == tq;
    row[u] = d;
    if (dist) dist[(size_t)y * W + u] = __double2float_rn(__dsqrt_rn((double)d));
    if (pop && u > 0) {
      q--;
      const uint64_t e = (uint64_t)row[q];
      sq = (long long)(e >> 32);
      tq = (long long)(e & 0xffffffffu);
      gsq = gr[sq];
    }
  }
}

}  // namespace edtaux
}  // namespace iwpp

using namespace iwpp;

extern "C" {

size_t iwpp_edt_init_workspace_bytes(int64_t W, int64_t H) {
  const size_t nch = ((size_t)W * H + edtaux::kChunk - 1) / edtaux::kChunk;
  return align_up(nch * 4, 256) + align_up((nch + 1) * 8, 256) + 256;
}

int iwpp_edt_init(const uint8_t *mask, int64_t W, int64_t H, int conn, int64_t *vr, int64_t *seeds,
                  int64_t *n_seeds_host, void *workspace, size_t workspace_bytes, void *stream) {
  if (W < 1 || H < 1 || W > (1 << 30) || H > (1 << 30) || W * H > ((int64_t)1 << 36))
    return set_error(IWPP_E_CONTRACT, "bad image dimensions %lld x %lld", (long long)W, (long long)H);
  if (conn != 4 && conn != 8)
    return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8, got %d", conn);
  if (workspace_bytes < iwpp_edt_init_workspace_bytes(W, H))
    return set_error(IWPP_E_WORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const long long nch = ((long long)W * H + edtaux::kChunk - 1) / edtaux::kChunk;
  Carver c(workspace);
  unsigned *counts = c.take<unsigned>((size_t)nch);
  unsigned long long *offs = c.take<unsigned long long>((size_t)nch + 1);
  if (seeds || n_seeds_host) {
    if (conn == 8) edtaux::contour_count_kernel<8><<<(unsigned)nch, edtaux::kThreads, 0, st>>>(mask, (int)W, (int)H, counts);
    else edtaux::contour_count_kernel<4><<<(unsigned)nch, edtaux::kThreads, 0, st>>>(mask, (int)W, (int)H, counts);
    IWPP_CUDA_TRY(cudaGetLastError());
    edtaux::chunk_scan_kernel<<<1, 1024, 0, st>>>(counts, nch, offs);
    IWPP_CUDA_TRY(cudaGetLastError());
  }
  if (conn == 8) edtaux::init_write_kernel<8><<<(unsigned)nch, edtaux::kThreads, 0, st>>>(mask, (int)W, (int)H, offs, vr, seeds);
  else edtaux::init_write_kernel<4><<<(unsigned)nch, edtaux::kThreads, 0, st>>>(mask, (int)W, (int)H, offs, vr, seeds);
  IWPP_CUDA_TRY(cudaGetLastError());
  if (n_seeds_host) {
    unsigned long long n = 0;
    IWPP_CUDA_TRY(cudaMemcpyAsync(&n, offs + nch, sizeof n, cudaMemcpyDeviceToHost, st));
    IWPP_CUDA_TRY(cudaStreamSynchronize(st));
    *n_seeds_host = (int64_t)n;
  }
  return IWPP_OK;
}

size_t iwpp_edt_exact_workspace_bytes(int64_t W, int64_t H) {
  return align_up((size_t)W * H * 4, 256) + align_up((size_t)W * H * 8, 256) + 512;
}

int iwpp_edt_exact(const uint8_t *mask, int64_t W, int64_t H, int64_t *d2, float *dist,
                   void *workspace, size_t workspace_bytes, void *stream) {
  if (W < 1 || H < 1 || W > (1 << 30) || H > (1 << 30) || W * H > ((int64_t)1 << 36))
    return set_error(IWPP_E_CONTRACT, "bad image dimensions %lld x %lld", (long long)W, (long long)H);
  const size_t need = align_up((size_t)W * H * 4, 256) + (d2 ? 0 : align_up((size_t)W * H * 8, 256)) + 256;
  if (workspace_bytes < need) return set_error(IWPP_E_WORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  Carver c(workspace);
  int32_t *g = c.take<int32_t>((size_t)W * H);
  int64_t *out = d2 ? d2 : c.take<int64_t>((size_t)W * H);
  edtaux::exact_cols_kernel<<<(unsigned)((W + 127) / 128), 128, 0, st>>>(mask, (int)W, (int)H, g);
  IWPP_CUDA_TRY(cudaGetLastError());
  edtaux::exact_rows_kernel<<<(unsigned)((H + 63) / 64), 64, 0, st>>>(g, (int)W, (int)H, out, dist);
  IWPP_CUDA_TRY(cudaGetLastError());
  // background present iff column-pass found one anywhere: check one row's
  // first cell (every cell is FAR iff there is no background at all)
  int64_t first = 0;
  IWPP_CUDA_TRY(cudaMemcpyAsync(&first, out, sizeof first, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  if (first == ((int64_t)1 << 62))
    return set_error(IWPP_E_NO_BACKGROUND, "no background reachable: distance map undefined");
  return IWPP_OK;
}

}  // extern "C"
