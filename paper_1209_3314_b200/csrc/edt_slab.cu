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

#include <cstring>

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

// ===========================================================================
// Device-resident multi-slab rounds (no host round trip per round).
//
// The per-round host loop above (launch, extract, count copy + sync, NCCL
// send/recv, all-reduce) costs tens of microseconds per round.  Here every
// rank runs ONE persistent kernel for all its rounds; boundary items and the
// frontier counts move by stores / atomics into the ranks' mailboxes:
//   * mailbox (per rank, in that rank's memory; written by its neighbours
//     and by every rank): two tagged entry rows per side and parity --
//     entry x = (tag << 32) | src, tag = consuming round + 1 (0 = empty), so
//     only the changed boundary cells are written (no full-row traffic) and
//     stale entries are ignored -- plus per-slot count sums and arrivals;
//   * round r of a rank (its CTAs): offers of its own frontier and of the
//     valid halo entries into its rows (raster offers + next-frontier bitmap
//     for large frontiers, returned atomics + block queues for small ones),
//     group barrier, next-frontier list (bitmap compaction, or the queue as
//     pushed) with the first / last row's new frontier cells written into
//     the neighbours' mailboxes (final keys: the round's offers are done),
//     group barrier, then the count exchange: the group's lead CTA adds its
//     count into every rank's slot and arrives (release, system scope);
//     every CTA waits for G arrivals on its own mailbox (acquire) and reads
//     the global next-frontier size -- 0 ends the run everywhere at once.
// Ranks may be G groups of CTAs of one cooperative launch on one GPU (the
// virtual mode: mailboxes in the same memory, the single-GPU tests and the
// protocol's cost measurement) or one launch per GPU with the neighbours'
// mailboxes mapped over NVLink (peer pointers).  The code is the same:
// every mailbox access is system-scoped.
constexpr int kMgMaxRanks = 16;

struct MgSlab {
  Slab s;
  uint32_t *fb;              // next-frontier bitmap, h rows x ceil(W/32) words
  unsigned *bar;             // group barrier: [0] arrivals, [kBarGen] generation
  unsigned long long *mb_self;               // my mailbox
  unsigned long long *mb_up, *mb_dn;         // the neighbours' mailboxes (null at the edge)
  unsigned long long *mb_all[kMgMaxRanks];   // every rank's mailbox (count exchange)
  int H, has_up, has_down, rank, G;
  int cta0, ncta;            // this slab's CTAs in the launch
};

// mailbox layout (u64 units): [4][W] entry rows (side * 2 + parity; side 0 =
// from the rank above, 1 = from below), then 3 slots x (sum, arrivals) on
// their own lines
inline size_t mg_mailbox_words(int64_t W) { return 4 * (size_t)W + 3 * 2 * 16; }
__device__ __forceinline__ unsigned long long *mb_row(unsigned long long *mb, int W, int side, int par) {
  return mb + (size_t)(side * 2 + par) * W;
}
__device__ __forceinline__ unsigned *mb_sum(unsigned long long *mb, int W, int slot) {
  return reinterpret_cast<unsigned *>(mb + 4 * (size_t)W + slot * 32);
}
__device__ __forceinline__ unsigned *mb_arr(unsigned long long *mb, int W, int slot) {
  return reinterpret_cast<unsigned *>(mb + 4 * (size_t)W + slot * 32 + 16);
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// group barrier over the slab's CTAs (as edt.cuh grid_barrier)
__device__ __forceinline__ void mg_barrier(const MgSlab &m, unsigned &g) {
  grid_barrier(&m.bar[0], &m.bar[kBarGen], (unsigned)m.ncta, g);
}

// count exchange after round r - 1 (slot r % 3): the lead CTA adds this
// slab's next-frontier size to every rank's slot, arrives, waits for the G
// arrivals on its own mailbox (system scope) and hands the global size to
// the slab's other CTAs through a local generation word (GPU scope: one
// remote-coherent poller per slab, not one per CTA)
constexpr int kXGen = 128, kXTotal = 160;  // m.bar words (own lines)
// a rank that waits this long for its peers' arrivals gives up (a peer died
// or never launched): the run ends on every CTA of the slab with an error
// instead of hanging the GPU
constexpr unsigned long long kMgWatchdogNs = 20ull * 1000 * 1000 * 1000;
constexpr unsigned long long kMgLost = 1ull << 40;
__device__ unsigned mg_count_exchange(const MgSlab &m, int r, unsigned n_mine, int lead, unsigned &xg) {
  __shared__ unsigned total;
  const int slot = r % 3;
  if (threadIdx.x == 0) {
    if (lead) {
      fence_sys();  // this slab's halo entries (their writers fenced them before the barrier)
      for (int g = 0; g < m.G; g++)
        if (n_mine) atomicAdd_system(mb_sum(m.mb_all[g], m.s.W, slot), n_mine);
      fence_sys();
      for (int g = 0; g < m.G; g++)
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(mb_arr(m.mb_all[g], m.s.W, slot))
                     : "memory");
      unsigned ns = 32;
      unsigned long long t0, now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      bool lost = false;
      while (ld_acquire_sys(mb_arr(m.mb_self, m.s.W, slot)) < (unsigned)m.G) {
        __nanosleep(ns);
        if (ns < 128) ns *= 2;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        if (now - t0 > kMgWatchdogNs) {  // a peer never arrived: end the run with an error
          lost = true;
          break;
        }
      }
      if (lost) atomicOr(&m.s.counters[EC_BAD], kMgLost);
      const unsigned t = lost ? 0u : ld_acquire_sys(mb_sum(m.mb_self, m.s.W, slot));
      // slot (r + 2) % 3 was last used after round r - 2: everyone has passed it
      *mb_sum(m.mb_self, m.s.W, (r + 2) % 3) = 0;
      *mb_arr(m.mb_self, m.s.W, (r + 2) % 3) = 0;
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(&m.bar[kXTotal]), "r"(t) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&m.bar[kXGen]) : "memory");
      total = t;
    } else {
      while (ld_acquire(&m.bar[kXGen]) == xg) __nanosleep(32);
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(total) : "l"(&m.bar[kXTotal]) : "memory");
    }
    xg++;
  }
  __syncthreads();
  return total;
}

// the new frontier cell (gx, ly) of a boundary row: its item for the
// neighbour's next round (consumer round rc, final key k)
__device__ __forceinline__ void mg_emit(const MgSlab &m, int ly, int gx, unsigned long long k, int rc,
                                        bool &wrote) {
  const unsigned long long e = ((unsigned long long)(rc + 1) << 32) | (uint32_t)k;
  if (ly == 0 && m.mb_up) {
    st_relaxed_sys64(mb_row(m.mb_up, m.s.W, 1, rc & 1) + gx, e);  // I am below my up-neighbour
    wrote = true;
  }
  if (ly == m.s.h - 1 && m.mb_dn) {
    st_relaxed_sys64(mb_row(m.mb_dn, m.s.W, 0, rc & 1) + gx, e);
    wrote = true;
  }
}

// round-start keys: read through L2 (IWPP_MG_L1KEYS=1: through L1; the
// buffer is read-only within a round and every barrier invalidates L1)
#if IWPP_MG_L1KEYS
#define MG_LDK(p) (*(p))
#else
#define MG_LDK(p) __ldcg(p)
#endif
// all local slabs travel as one kernel parameter (no device allocation)
struct MgArgs {
  MgSlab slab[kMgMaxRanks];
  int n;
};

template <int CONN>
__global__ void __launch_bounds__(kRoundThreads, kRoundBlocksPerSm) mg_rounds_kernel(const __grid_constant__ MgArgs args,
                                                                  long long max_rounds) {
  const unsigned FULL = 0xffffffffu;
  int si = 0;
  while (si + 1 < args.n && (int)blockIdx.x >= args.slab[si + 1].cta0) si++;
  const MgSlab &m = args.slab[si];
  const Slab &s = m.s;
  const int W = s.W, h = s.h, y0 = s.y0;
  const int WW = (W + 31) >> 5;
  const unsigned cta = blockIdx.x - m.cta0, ncta = (unsigned)m.ncta;
  const int lead = cta == 0;
  const unsigned lane = threadIdx.x & 31u;
  unsigned bar_g = grid_barrier_gen(&m.bar[kBarGen]);
  unsigned xg = threadIdx.x == 0 ? ld_acquire(&m.bar[kXGen]) : 0u;
  __shared__ uint32_t bq[kEdtBq];
  __shared__ unsigned bq_n, blk_base, wsum[kRoundThreads / 32];
  unsigned long long *K = s.keys;
  // this CTA's run of bitmap words (compaction)
  const unsigned nwords = (unsigned)WW * (unsigned)h;
  const unsigned per = ((nwords + ncta - 1) / ncta + 3) / 4 * 4;
  const unsigned w_lo = min(nwords, cta * per), w_hi = min(nwords, w_lo + per);
  unsigned total = mg_count_exchange(m, 0, ld_acquire(&s.cnt[0]), lead, xg);
  int r = 0;
  for (; total; r++) {
    if (max_rounds >= 0 && r >= max_rounds) {
      if (lead && threadIdx.x == 0) s.counters[EC_LIMIT] = 1;
      break;
    }
    const unsigned n = ld_acquire(&s.cnt[r % 3]);
    const int kr = r & 1, kw = kr ^ 1;
    const uint32_t *cur = s.F[r & 1];
    uint32_t *nxt = s.F[(r + 1) & 1];
    unsigned *ncnt = &s.cnt[(r + 1) % 3];
    if (lead && threadIdx.x == 0) s.cnt[(r + 2) % 3] = 0;
    const bool raster = n >= kRasterMinFrontier;
    // phase 1: own items [0, n), then the halo entries of both sides
    const unsigned nh = (m.has_up ? (unsigned)W : 0u) + (m.has_down ? (unsigned)W : 0u);
    const unsigned ntot = n + nh;
    if (threadIdx.x == 0) bq_n = 0;
    __syncthreads();
    const unsigned stride = ncta * blockDim.x;
    for (unsigned base = cta * blockDim.x + (threadIdx.x & ~31u); base < ntot; base += stride) {
      const unsigned i = base + lane;
      int px = 0, gy = 0;
      unsigned long long kp = KINF;
      bool own = false;
      if (i < n) {
        const uint32_t pyx = __ldcg(cur + i);
        gy = (int)(pyx >> 16);
        px = (int)(pyx & 0xffffu);
        own = true;
        kp = MG_LDK(K + 2 * ((size_t)(gy - y0) * W + px) + kr);  // round-start: read-only this round
      } else if (i < ntot) {
        unsigned j = i - n;
        const bool up = m.has_up && j < (unsigned)W;
        if (!up && m.has_up) j -= W;
        px = (int)j;
        gy = up ? y0 - 1 : y0 + h;
        const unsigned long long e = ld_relaxed_sys64(mb_row(m.mb_self, W, up ? 0 : 1, r & 1) + j);
        if ((unsigned)(e >> 32) == (unsigned)(r + 1)) kp = (uint32_t)e;  // a valid item: its source
      }
      unsigned long long rq[Nbr<CONN>::N], nk[Nbr<CONN>::N];
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        const int qx = px + Nbr<CONN>::dx(k), qly = gy + Nbr<CONN>::dy(k) - y0;
        const bool in = kp != KINF && qx >= 0 && qx < W && qly >= 0 && qly < h;
        rq[k] = in ? MG_LDK(K + 2 * ((size_t)qly * W + qx) + kr) : 0ull;
      }
      if (own) atomicMin(K + 2 * ((size_t)(gy - y0) * W + px) + kw, kp);  // resync the building key
      unsigned cand = 0;
      const uint32_t src = (uint32_t)kp;
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        const int qx = px + Nbr<CONN>::dx(k), qy = gy + Nbr<CONN>::dy(k);
        bool ok = true;
        nk[k] = make_key_checked(qx, qy, src, ok);
        if (kp != KINF && !ok) s.counters[EC_RANGE] = 1;
        if (kp != KINF && ok && nk[k] < rq[k]) cand |= 1u << k;
      }
      unsigned mask = 0;
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        const int qx = px + Nbr<CONN>::dx(k), qly = gy + Nbr<CONN>::dy(k) - y0;
        const unsigned on = (cand >> k) & 1u;
        unsigned long long *q = K + 2 * ((size_t)(on ? qly : 0) * W + (on ? qx : 0)) + kw;
        if (raster) {
          if (on) atomicMin(q, nk[k]);
          const unsigned waddr = on ? (unsigned)qly * (unsigned)WW + ((unsigned)qx >> 5) : 0xffffffffu;
          const unsigned grp = __match_any_sync(FULL, waddr);
          const unsigned orb = __reduce_or_sync(grp, on ? (1u << (qx & 31)) : 0u);
          if (on && lane == (unsigned)(__ffs(grp) - 1)) atomicOr(m.fb + waddr, orb);
        } else {
          const unsigned long long old = gmem_atomic_min_if(q, nk[k], on);
          if (on && old >= rq[k]) mask |= 1u << k;
        }
      }
      if (!raster) {  // transition rule: one push per changed cell
        const unsigned c = __popc(mask);
        unsigned pos = warp_reserve(&bq_n, c, FULL);
        while (mask) {
          const int k = __ffs(mask) - 1;
          mask &= mask - 1;
          const int qx = px + Nbr<CONN>::dx(k), qy = gy + Nbr<CONN>::dy(k);
          const uint32_t item = ((uint32_t)qy << 16) | (uint32_t)qx;
          if (pos < kEdtBq)
            bq[pos] = item;
          else
            nxt[atomicAdd(ncnt, 1u)] = item;
          pos++;
        }
      }
    }
    if (!raster) {
      __syncthreads();
      const unsigned mq = min(bq_n, (unsigned)kEdtBq);
      if (threadIdx.x == 0 && mq) blk_base = atomicAdd(ncnt, mq);
      __syncthreads();
      for (unsigned i = threadIdx.x; i < mq; i += blockDim.x) nxt[blk_base + i] = bq[i];
    }
    mg_barrier(m, bar_g);
    // phase 2: the next list (raster: compact this CTA's bitmap words) and
    // the boundary rows' new frontier items for the neighbours
    bool wrote = false;
    if (raster) {
      // 4 words per thread per pass (one 16-byte load), one block scan and
      // one global atomic per pass (as the single-image raster engine)
      for (unsigned wb = w_lo; wb < w_hi; wb += blockDim.x * 4) {
        const unsigned wi = wb + threadIdx.x * 4;
        unsigned w4[4];
        const bool full = wi + 4 <= w_hi;
        if (full) {
          const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(m.fb + wi));
          w4[0] = v.x, w4[1] = v.y, w4[2] = v.z, w4[3] = v.w;
        } else {
#pragma unroll
          for (unsigned k = 0; k < 4; k++) w4[k] = wi + k < w_hi ? __ldcg(m.fb + wi + k) : 0u;
        }
        const unsigned c = __popc(w4[0]) + __popc(w4[1]) + __popc(w4[2]) + __popc(w4[3]);
        unsigned incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_up_sync(FULL, incl, o);
          if (lane >= (unsigned)o) incl += v;
        }
        if (lane == 31) wsum[threadIdx.x >> 5] = incl;
        __syncthreads();
        if (threadIdx.x == 0) {
          unsigned t = 0;
          for (int k = 0; k < kRoundThreads / 32; k++) {
            const unsigned v = wsum[k];
            wsum[k] = t;
            t += v;
          }
          blk_base = t ? atomicAdd(ncnt, t) : 0u;
        }
        __syncthreads();
        unsigned o = blk_base + wsum[threadIdx.x >> 5] + incl - c;
        if (c) {
          if (full) {
            *reinterpret_cast<uint4 *>(m.fb + wi) = make_uint4(0u, 0u, 0u, 0u);
          } else {
            for (unsigned k = 0; k < 4; k++)
              if (w4[k]) m.fb[wi + k] = 0u;
          }
#pragma unroll
          for (unsigned k = 0; k < 4; k++) {
            unsigned w = w4[k];
            if (!w) continue;
            const unsigned ly = (wi + k) / (unsigned)WW, x0 = (wi + k - ly * (unsigned)WW) * 32;
            while (w) {
              const int bb = __ffs(w) - 1;
              w &= w - 1;
              const int gx = (int)x0 + bb;
              nxt[o++] = ((uint32_t)(y0 + ly) << 16) | (uint32_t)gx;
              if (ly == 0 || ly == (unsigned)h - 1)
                mg_emit(m, (int)ly, gx, __ldcg(K + 2 * ((size_t)ly * W + gx) + kw), r + 1, wrote);
            }
          }
        }
        __syncthreads();
      }
    } else {
      const unsigned nn = ld_acquire(ncnt);  // complete after the barrier
      for (unsigned i = cta * blockDim.x + threadIdx.x; i < nn; i += stride) {
        const uint32_t pyx = __ldcg(nxt + i);
        const int ly = (int)(pyx >> 16) - y0, gx = (int)(pyx & 0xffffu);
        if (ly == 0 || ly == h - 1) mg_emit(m, ly, gx, __ldcg(K + 2 * ((size_t)ly * W + gx) + kw), r + 1, wrote);
      }
    }
    if (__syncthreads_or(wrote) && threadIdx.x == 0) fence_sys();  // peer entries before the arrival
    mg_barrier(m, bar_g);
    total = mg_count_exchange(m, r + 1, ld_acquire(ncnt), lead, xg);
  }
  if (lead && threadIdx.x == 0) {
    s.counters[EC_ROUNDS] = (unsigned long long)r;
    s.counters[EC_FINAL] = (unsigned long long)(r & 1);
  }
}

// the initial boundary items (slab_init's dense rows) into the neighbours'
// mailboxes, consumer round 0
__global__ void mg_seed_mail_kernel(const unsigned long long *out_up, const unsigned long long *out_dn,
                                    int W, unsigned long long *mb_up, unsigned long long *mb_dn) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < W; x += gridDim.x * blockDim.x) {
    if (mb_up && out_up[x] != KINF) st_relaxed_sys64(mb_row(mb_up, W, 1, 0) + x, (1ull << 32) | (uint32_t)out_up[x]);
    if (mb_dn && out_dn[x] != KINF) st_relaxed_sys64(mb_row(mb_dn, W, 0, 0) + x, (1ull << 32) | (uint32_t)out_dn[x]);
  }
  __syncthreads();
  if (threadIdx.x == 0) fence_sys();
}

size_t mg_slab_bytes(int64_t W, int64_t h) {
  Carver c(nullptr);
  carve_slab(c, W, h);
  c.take<uint32_t>((size_t)((W + 31) / 32) * h);
  c.take<unsigned>(256);
  c.take<unsigned long long>(2 * (size_t)W);
  return c.off + 256;
}
size_t mg_mailbox_bytes(int64_t W) { return mg_mailbox_words(W) * sizeof(unsigned long long); }

static void carve_mg(void *ws, int64_t W, int64_t h, Slab &s, uint32_t *&fb, unsigned *&bar,
                     unsigned long long *&rows) {
  Carver c(ws);
  s = carve_slab(c, W, h);
  fb = c.take<uint32_t>((size_t)((W + 31) / 32) * h);
  bar = c.take<unsigned>(256);
  rows = c.take<unsigned long long>(2 * (size_t)W);
  s.W = (int)W;
  s.h = (int)h;
}

int mg_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H, int conn, int has_up,
            int has_down, void *ws, void *mailbox, void *mb_up, void *mb_dn, cudaStream_t st) {
  Slab s;
  uint32_t *fb;
  unsigned *bar;
  unsigned long long *rows;
  carve_mg(ws, W, h, s, fb, bar, rows);
  IWPP_CUDA_TRY(cudaMemsetAsync(fb, 0, sizeof(uint32_t) * ((W + 31) / 32) * (size_t)h, st));
  IWPP_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned) * 256, st));
  (void)mailbox;  // cleared by the caller before any rank seeds (collective order)
  int rc = slab_init(mask_ext, W, h, y0, H, conn, has_up, has_down, ws, rows, rows + W, st);
  if (rc) return rc;
  mg_seed_mail_kernel<<<grid_cap((size_t)W, 256), 256, 0, st>>>(
      rows, rows + W, (int)W, (unsigned long long *)mb_up, (unsigned long long *)mb_dn);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int mg_run(const iwpp_edt_mg_slab *d, int nlocal, int conn, long long max_rounds, int64_t *rounds_host,
           cudaStream_t st) {
  if (nlocal < 1 || nlocal > kMgMaxRanks) return set_error(IWPP_E_CONTRACT, "1..16 local slabs");
  MgArgs args;  // the kernel parameter, staged on this host thread's stack
  memset(&args, 0, sizeof args);
  args.n = nlocal;
  MgSlab *hs = args.slab;
  static int per_sm[2] = {0, 0};
  int &ps = per_sm[conn == 8];
  if (ps == 0) {
    IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &ps, conn == 8 ? (const void *)mg_rounds_kernel<8> : (const void *)mg_rounds_kernel<4>, kRoundThreads,
        0));
    if (ps < 1) ps = 1;
    if (ps > kRoundBlocksPerSm) ps = kRoundBlocksPerSm;
  }
  const int nb = device_sm_count() * ps;
  if (nb < nlocal) return set_error(IWPP_E_CONTRACT, "more local slabs than resident CTAs");
  for (int i = 0; i < nlocal; i++) {
    MgSlab &m = hs[i];
    unsigned long long *rows;
    carve_mg(d[i].workspace, d[i].W, d[i].h, m.s, m.fb, m.bar, rows);
    m.s.y0 = (int)d[i].y0;
    m.H = (int)d[i].H;
    m.has_up = d[i].has_up;
    m.has_down = d[i].has_down;
    m.rank = d[i].rank;
    m.G = d[i].world;
    if (m.G < 1 || m.G > kMgMaxRanks) return set_error(IWPP_E_CONTRACT, "world must be 1..16");
    m.mb_self = (unsigned long long *)d[i].mailbox[d[i].rank];
    m.mb_up = d[i].has_up ? (unsigned long long *)d[i].mailbox[d[i].rank - 1] : nullptr;
    m.mb_dn = d[i].has_down ? (unsigned long long *)d[i].mailbox[d[i].rank + 1] : nullptr;
    for (int g = 0; g < kMgMaxRanks; g++)
      m.mb_all[g] = g < m.G ? (unsigned long long *)d[i].mailbox[g] : nullptr;
    // CTAs in proportion to the slab heights
    m.cta0 = (int)((long long)nb * i / nlocal);
    m.ncta = (int)((long long)nb * (i + 1) / nlocal) - m.cta0;
  }
  void *kargs[] = {&args, &max_rounds};
  const void *k = conn == 8 ? (const void *)mg_rounds_kernel<8> : (const void *)mg_rounds_kernel<4>;
  cudaError_t e = cudaLaunchCooperativeKernel(k, dim3(nb), dim3(kRoundThreads), kargs, 0, st);
  unsigned long long cnt[EC_N] = {0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(cnt, hs[0].s.counters, sizeof cnt, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_error(IWPP_E_CUDA, "mg rounds: %s", cudaGetErrorString(e));
  if (rounds_host) *rounds_host = (int64_t)cnt[EC_ROUNDS];
  if (cnt[EC_BAD] & kMgLost)
    return set_error(IWPP_E_CUDA, "multi-slab EDT: a peer rank never arrived (watchdog, %llu s)",
                     kMgWatchdogNs / 1000000000ull);
  if (cnt[EC_LIMIT]) return set_error(IWPP_E_ENGINE_LIMIT, "no fixed point within %lld rounds", max_rounds);
  return IWPP_OK;
}

}  // namespace edt
}  // namespace iwpp
