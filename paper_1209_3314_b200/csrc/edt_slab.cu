// edt_slab.cu -- one horizontal slab of a multi-GPU EDT.
//
// The reference's synchronous rule needs one exchange per round
// (tiles.py:10-15, 305-331; edt_bp_sweep K.493-522 offers the wave-start
// value across the cut).  Each rank owns rows [y0, y0+h) of the global
// image and runs the key engine one round per launch:
//   * its own frontier items offer to its own cells;
//   * the neighbours' boundary frontier items ("halo items": the cells of
//     the adjacent rows that are in the frontier, with their round-start
//     sources) offer into its boundary row -- the cross-cut offers;
//   * after the round, the cells of its first / last row that changed (=
//     its boundary frontier items of the next round) are extracted into
//     dense rows (source or INF per column) for the neighbours.
// Keys use GLOBAL (y, x) coordinates, so the (d2, packed index) tie-break is
// the single-device one and the slab result is identical cell for cell.

#include "edt.cuh"

namespace iwpp {
namespace edt {

struct Slab {
  unsigned long long *keys;  // 2 per local cell, double-buffered
  uint32_t *F[2];            // frontier (global yx codes)
  unsigned *cnt;             // [3]
  unsigned long long *counters;
  int W, h, y0;
};

static Slab carve_slab(Carver &c, int64_t W, int64_t h) {
  size_t n = (size_t)W * h;
  Slab s;
  s.keys = c.take<unsigned long long>(2 * n);
  s.F[0] = c.take<uint32_t>(n);
  s.F[1] = c.take<uint32_t>(n);
  s.cnt = c.take<unsigned>(4);
  s.counters = c.take<unsigned long long>(EC_N);
  return s;
}

size_t slab_bytes(int64_t W, int64_t h) {
  Carver c(nullptr);
  carve_slab(c, W, h);
  return c.off + 256;
}

// mask_ext: (h + 2) rows, row 0 / h+1 = the neighbours' rows (ignored when
// has_up / has_down is 0: the image ends there).
template <int CONN>
__global__ void slab_init_kernel(const uint8_t *__restrict__ mask_ext, Slab s, int has_up,
                                 int has_down, int H, unsigned long long *out_up, unsigned long long *out_dn) {
  const unsigned FULL = 0xffffffffu;
  const int W = s.W, h = s.h;
  size_t n = (size_t)W * h;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n;
       base += stride) {
    size_t p = base + (threadIdx.x & 31u);
    bool push = false;
    uint32_t yx = 0;
    int ly = 0, px = 0;
    if (p < n) {
      ly = (int)(p / (unsigned)W);
      px = (int)(p - (size_t)ly * W);
      int gy = s.y0 + ly;
      yx = ((uint32_t)gy << 16) | (uint32_t)px;
      bool bg = mask_ext[(size_t)(ly + 1) * W + px] == 0;
      unsigned long long k = bg ? (unsigned long long)yx : KINF;
      reinterpret_cast<ulonglong2 *>(s.keys)[p] = make_ulonglong2(k, k);
      if (bg) {
#pragma unroll
        for (int k8 = 0; k8 < Nbr<CONN>::N; k8++) {
          int qx = px + Nbr<CONN>::dx(k8), qly = ly + Nbr<CONN>::dy(k8);
          int qgy = s.y0 + qly;
          bool in = qx >= 0 && qx < W && qgy >= 0 && qgy < H && (qly >= 0 || has_up) &&
                    (qly < h || has_down);
          if (in && mask_ext[(size_t)(qly + 1) * W + qx] != 0) push = true;
        }
      }
      if (ly == 0 && out_up) out_up[px] = push ? (unsigned long long)yx : KINF;
      if (ly == h - 1 && out_dn) out_dn[px] = push ? (unsigned long long)yx : KINF;
    }
    unsigned pos = warp_reserve(&s.cnt[0], push ? 1u : 0u, FULL);
    if (push) s.F[0][pos] = yx;
  }
}

// offers of one item (global px, gy) with source src to its in-slab
// neighbours; returns the bitmask of neighbours it made change
template <int CONN>
__device__ __forceinline__ unsigned slab_offers(const Slab &s, int px, int gy, uint32_t src, int kr,
                                                int kw) {
  unsigned long long rq[Nbr<CONN>::N], nk[Nbr<CONN>::N];
  unsigned cand = 0;
#pragma unroll
  for (int k = 0; k < Nbr<CONN>::N; k++) {
    int qx = px + Nbr<CONN>::dx(k), qly = gy + Nbr<CONN>::dy(k) - s.y0;
    bool in = qx >= 0 && qx < s.W && qly >= 0 && qly < s.h;
    rq[k] = in ? __ldcg(s.keys + 2 * ((size_t)qly * s.W + qx) + kr) : 0ull;
  }
#pragma unroll
  for (int k = 0; k < Nbr<CONN>::N; k++) {
    int qx = px + Nbr<CONN>::dx(k), qy = gy + Nbr<CONN>::dy(k);
    long long dx = qx - (int)(src & 0xffffu), dy = qy - (int)(src >> 16);
    unsigned long long d2 = (unsigned long long)(dx * dx + dy * dy);
    if (d2 >> 32) {  // beyond the key range: flag it (the caller raises), never offer
      atomicOr(reinterpret_cast<unsigned long long *>(&s.counters[EC_RANGE]), 1ull);
      nk[k] = KINF;
    } else {
      nk[k] = (d2 << 32) | src;
    }
    if (nk[k] < rq[k]) cand |= 1u << k;
  }
  unsigned mask = 0;
#pragma unroll
  for (int k = 0; k < Nbr<CONN>::N; k++) {
    int qx = px + Nbr<CONN>::dx(k), qly = gy + Nbr<CONN>::dy(k) - s.y0;
    unsigned on = (cand >> k) & 1u;
    unsigned long long old =
        gmem_atomic_min_if(s.keys + 2 * ((size_t)qly * s.W + qx) + kw, nk[k], on);
    if (on && old >= rq[k]) mask |= 1u << k;
  }
  return mask;
}

template <int CONN>
__global__ void __launch_bounds__(kRoundThreads) slab_round_kernel(Slab s, int r,
                                                                   const unsigned long long *halo_up,
                                                                   const unsigned long long *halo_dn) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u;
  __shared__ uint32_t bq[kEdtBq];
  __shared__ unsigned bq_n, bq_base;
  const unsigned n = s.cnt[r % 3];
  const int kr = r & 1, kw = kr ^ 1;
  const uint32_t *cur = s.F[r & 1];
  uint32_t *nxt = s.F[(r + 1) & 1];
  unsigned *ncnt = &s.cnt[(r + 1) % 3];
  if (threadIdx.x == 0) bq_n = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) s.cnt[(r + 2) % 3] = 0;
  __syncthreads();
  const unsigned halo_items = (halo_up ? s.W : 0) + (halo_dn ? s.W : 0);
  const unsigned total = n + halo_items;
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < total;
       base += stride) {
    unsigned i = base + lane;
    unsigned mask = 0;
    int px = 0, gy = 0;
    if (i < n) {  // own frontier item
      uint32_t pyx = __ldcg(cur + i);
      gy = (int)(pyx >> 16);
      px = (int)(pyx & 0xffffu);
      size_t p = (size_t)(gy - s.y0) * s.W + px;
      unsigned long long kp = __ldcg(s.keys + 2 * p + kr);
      atomicMin(s.keys + 2 * p + kw, kp);  // the building key lags on the frontier
      if (kp != KINF) mask = slab_offers<CONN>(s, px, gy, (uint32_t)kp, kr, kw);
    } else if (i < total) {  // a neighbour's boundary frontier item
      unsigned j = i - n;
      const bool up = halo_up && j < (unsigned)s.W;
      const unsigned long long *row = up ? halo_up : halo_dn;
      if (!up && halo_up) j -= s.W;
      px = (int)j;
      gy = up ? s.y0 - 1 : s.y0 + s.h;
      unsigned long long src = __ldcg(row + j);
      if (src != KINF) mask = slab_offers<CONN>(s, px, gy, (uint32_t)src, kr, kw);
    }
    unsigned c = __popc(mask);
    unsigned pos = warp_reserve(&bq_n, c, FULL);
    while (mask) {
      int k = __ffs(mask) - 1;
      mask &= mask - 1;
      int qx = px + Nbr<CONN>::dx(k), qy = gy + Nbr<CONN>::dy(k);
      uint32_t item = ((uint32_t)qy << 16) | (uint32_t)qx;
      if (pos < kEdtBq)
        bq[pos] = item;
      else
        nxt[atomicAdd(ncnt, 1u)] = item;
      pos++;
    }
  }
  __syncthreads();
  unsigned m = min(bq_n, (unsigned)kEdtBq);
  if (threadIdx.x == 0 && m) bq_base = atomicAdd(ncnt, m);
  __syncthreads();
  for (unsigned i = threadIdx.x; i < m; i += blockDim.x) nxt[bq_base + i] = bq[i];
}

// the next round's boundary frontier items (cells of the first / last row
// whose key changed this round) as dense rows of sources (INF32 = none)
__global__ void slab_extract_kernel(Slab s, int r, unsigned long long *out_up, unsigned long long *out_dn) {
  const int kr = r & 1, kw = kr ^ 1;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < s.W; x += gridDim.x * blockDim.x) {
    if (out_up) {
      unsigned long long a = __ldcg(s.keys + 2 * (size_t)x + kr), b = __ldcg(s.keys + 2 * (size_t)x + kw);
      out_up[x] = b < a ? (unsigned long long)(uint32_t)b : KINF;
    }
    if (out_dn) {
      size_t p = (size_t)(s.h - 1) * s.W + x;
      unsigned long long a = __ldcg(s.keys + 2 * p + kr), b = __ldcg(s.keys + 2 * p + kw);
      out_dn[x] = b < a ? (unsigned long long)(uint32_t)b : KINF;
    }
  }
}

__global__ void slab_finalize_kernel(Slab s, int fb, int64_t *vr, float *dist) {
  size_t n = (size_t)s.W * s.h;
  unsigned long long ninf = 0;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    unsigned long long k = __ldcg(s.keys + 2 * p + fb);
    if (k == KINF) {
      ninf++;
      if (vr) vr[p] = -1;
      if (dist) dist[p] = 0.f;
      continue;
    }
    uint32_t src = (uint32_t)k;
    if (vr) vr[p] = (int64_t)(src >> 16) * s.W + (src & 0xffffu);
    if (dist) dist[p] = __double2float_rn(__dsqrt_rn((double)(k >> 32)));
  }
  for (int o = 16; o; o >>= 1) ninf += __shfl_xor_sync(0xffffffffu, ninf, o);
  if ((threadIdx.x & 31) == 0 && ninf) atomicAdd(&s.counters[EC_NINF], ninf);
}

static int grid_cap(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  size_t cap = (size_t)device_sm_count() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

int slab_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H, int conn,
              int has_up, int has_down, void *ws, unsigned long long *out_up,
              unsigned long long *out_dn, cudaStream_t st) {
  Carver c(ws);
  Slab s = carve_slab(c, W, h);
  s.W = (int)W;
  s.h = (int)h;
  s.y0 = (int)y0;
  IWPP_CUDA_TRY(cudaMemsetAsync(s.cnt, 0, sizeof(unsigned) * 4, st));
  IWPP_CUDA_TRY(cudaMemsetAsync(s.counters, 0, sizeof(unsigned long long) * EC_N, st));
  int g = grid_cap((size_t)W * h, 256);
  if (conn == 8)
    slab_init_kernel<8><<<g, 256, 0, st>>>(mask_ext, s, has_up, has_down, (int)H, out_up, out_dn);
  else
    slab_init_kernel<4><<<g, 256, 0, st>>>(mask_ext, s, has_up, has_down, (int)H, out_up, out_dn);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int slab_round(void *ws, int64_t W, int64_t h, int64_t y0, int conn, int64_t r,
               const unsigned long long *halo_up, const unsigned long long *halo_dn,
               unsigned long long *out_up, unsigned long long *out_dn, int64_t *n_next_host,
               cudaStream_t st) {
  Carver c(ws);
  Slab s = carve_slab(c, W, h);
  s.W = (int)W;
  s.h = (int)h;
  s.y0 = (int)y0;
  int blocks = device_sm_count() * kRoundBlocksPerSm;
  if (conn == 8)
    slab_round_kernel<8><<<blocks, kRoundThreads, 0, st>>>(s, (int)r, halo_up, halo_dn);
  else
    slab_round_kernel<4><<<blocks, kRoundThreads, 0, st>>>(s, (int)r, halo_up, halo_dn);
  IWPP_CUDA_TRY(cudaGetLastError());
  slab_extract_kernel<<<grid_cap((size_t)W, 256), 256, 0, st>>>(s, (int)r, out_up, out_dn);
  IWPP_CUDA_TRY(cudaGetLastError());
  if (n_next_host) {
    unsigned v = 0;
    IWPP_CUDA_TRY(cudaMemcpyAsync(&v, &s.cnt[(r + 1) % 3], sizeof v, cudaMemcpyDeviceToHost, st));
    IWPP_CUDA_TRY(cudaStreamSynchronize(st));
    *n_next_host = v;
  }
  return IWPP_OK;
}

int slab_finalize(void *ws, int64_t W, int64_t h, int64_t y0, int64_t rounds, int64_t *vr,
                  float *dist, int64_t *n_inf_host, int64_t *range_err_host, cudaStream_t st) {
  Carver c(ws);
  Slab s = carve_slab(c, W, h);
  s.W = (int)W;
  s.h = (int)h;
  s.y0 = (int)y0;
  IWPP_CUDA_TRY(cudaMemsetAsync(&s.counters[EC_NINF], 0, sizeof(unsigned long long), st));
  slab_finalize_kernel<<<grid_cap((size_t)W * h, 256), 256, 0, st>>>(s, (int)(rounds & 1), vr,
                                                                     dist);
  IWPP_CUDA_TRY(cudaGetLastError());
  unsigned long long v[EC_N];
  IWPP_CUDA_TRY(cudaMemcpyAsync(v, s.counters, sizeof v, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  if (n_inf_host) *n_inf_host = (int64_t)v[EC_NINF];
  if (range_err_host) *range_err_host = (int64_t)v[EC_RANGE];
  return IWPP_OK;
}

}  // namespace edt
}  // namespace iwpp
