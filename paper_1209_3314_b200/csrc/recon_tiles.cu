// recon_tiles.cu -- persistent tile engine for morphological reconstruction.
//
// Replaces the reference's wavefront phase (recon_wavefront K.220-270,
// run_parallel/round shares engine.py:251-364, K.273-303) and its seed
// detection (recon_seed_scan K.193-217) with one persistent sm_100a kernel.
//
// Queue hierarchy (the paper's TQ/BQ/GBQ, re-designed):
//   TQ  : per-thread register bitmask of raised neighbours (<= 8 bits)
//   BQ  : per-CTA shared-memory pixel queue (two level buffers); pushes are
//         warp-aggregated (shfl scan + one shared atomicAdd per warp)
//   GBQ : global MPMC ring of *tile* ids.  A tile enters it when one of its
//         halo pixels is raised by a neighbouring tile (border exchange,
//         the BP step of tiles.py:342-359 done asynchronously).
// Persistent blocks pop tiles, load tile+halo into shared memory, detect
// the tile's active pixels (full-neighbourhood predicate, K.193-217), run
// the BQ propagation to the tile's local fixed point with shared-memory
// atomicMax (the update rule J(q) <- min(J(p), I(q)) under the condition
// J(q) < J(p) and J(q) != I(q), recon.py:92-101), write the tile back and
// activate neighbour tiles whose pixels the changed border can still raise.
// BQ overflow drops work, raises a flag and re-seeds the tile by a full
// rescan (the drop/rescan/re-execute contract of engine.py:274-303).
// Termination: a global count of tiles that are queued or running; the
// engine is done when the ring is empty and that count is 0.
//
// The fixed point is unique (engine.py:9-18), so this asynchronous schedule
// is bit-exact with recon_fh.

#include <climits>

#include "iwpp_common.cuh"
#include "recon_tiles.cuh"

namespace iwpp {
namespace recon {

// tile states
constexpr unsigned ST_IDLE = 0, ST_QUEUED = 1, ST_RUNNING = 2, ST_DIRTY = 3;

struct SmemLayout {
  int *J;          // PN  (int32 working values; INT_MIN = outside image)
  int *I;          // PN
  uint16_t *q[2];  // QCAP each
  int *ring0;      // 4*TW border-ring values as written back last time
};

__host__ __device__ constexpr size_t smem_bytes() {
  return sizeof(int) * PN * 2 + sizeof(uint16_t) * QCAP * 2 + sizeof(int) * 4 * TW + 64;
}

__device__ __forceinline__ int ring_index(int lx, int ly) {
  // interior border ring position of an interior cell on the tile edge,
  // -1 when the cell is not on the ring
  if (ly == 1) return lx - 1;
  if (ly == TH) return TW + lx - 1;
  if (lx == 1) return 2 * TW + ly - 1;
  if (lx == TW) return 3 * TW + ly - 1;
  return -1;
}

__device__ __forceinline__ bool interior(int lx, int ly) {
  return lx >= 1 && lx <= TW && ly >= 1 && ly <= TH;
}

struct EngineArgs {
  void *J;
  const void *I;
  int W, H;
  int ntx, nty;
  unsigned ntiles;
  unsigned qlimit;  // block-queue capacity actually used (<= QCAP)
  TileQueue q;
};

// --- global tile queue ---------------------------------------------------

__device__ __forceinline__ void ring_push(const TileQueue &q, unsigned t) {
  unsigned pos = atomicAdd(q.tail, 1u);
  st_release64(&q.ring[pos & q.mask], ((unsigned long long)pos << 32) | t);
}

// returns tile id or -1 when the ring is momentarily empty
__device__ __forceinline__ int ring_pop(const TileQueue &q) {
  for (;;) {
    unsigned h = ld_relaxed(q.head);
    unsigned t = ld_relaxed(q.tail);
    if ((int)(t - h) <= 0) return -1;
    if (atomicCAS(q.head, h, h + 1) != h) continue;
    unsigned long long *slot = &q.ring[h & q.mask];
    unsigned long long v;
    while (((v = ld_acquire64(slot)) >> 32) != h) __nanosleep(20);
    return (int)(v & 0xffffffffu);
  }
}

__device__ __forceinline__ void activate(const TileQueue &q, unsigned t) {
  unsigned s = ld_relaxed(&q.state[t]);
  for (;;) {
    if (s == ST_QUEUED || s == ST_DIRTY) return;
    if (s == ST_IDLE) {
      unsigned old = atomicCAS(&q.state[t], ST_IDLE, ST_QUEUED);
      if (old == ST_IDLE) {
        atomicAdd(q.pending, 1u);
        ring_push(q, t);
        return;
      }
      s = old;
    } else {  // RUNNING
      unsigned old = atomicCAS(&q.state[t], ST_RUNNING, ST_DIRTY);
      if (old == ST_RUNNING) return;
      s = old;
    }
  }
}

// --- tile processing -----------------------------------------------------

template <typename T>
__device__ __forceinline__ void load_cell(const EngineArgs &a, SmemLayout &s, int i, int x0,
                                          int y0) {
  int ly = i / PW, lx = i - ly * PW;
  int gx = x0 + lx - 1, gy = y0 + ly - 1;
  if (gx >= 0 && gx < a.W && gy >= 0 && gy < a.H) {
    size_t g = (size_t)gy * a.W + gx;
    s.J[i] = (int)ld_cg((const T *)a.J + g);
    s.I[i] = (int)__ldg((const T *)a.I + g);
  } else {
    s.J[i] = INT_MIN;
    s.I[i] = INT_MIN;
  }
}

// Detect active pixels (p can raise an interior neighbour) into q[0]
// (K.193-217 restricted to the tile, halo cells act as sources only).
// Returns the number queued (clipped to qlimit; *s_over set if clipped).
template <int CONN>
__device__ unsigned detect_seeds(SmemLayout &s, unsigned *s_n, unsigned *s_over, unsigned qlimit) {
  const unsigned FULL = 0xffffffffu;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int base = warp * 32; base < PN; base += blockDim.x) {
    int p = base + lane;
    bool want = false;
    if (p < PN) {
      int v = s.J[p];
      int py = p / PW, px = p - py * PW;
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
        if (interior(qx, qy)) {
          int qq = qy * PW + qx;
          int vq = s.J[qq];
          if (vq < v && vq < s.I[qq]) want = true;
        }
      }
    }
    unsigned pos = warp_reserve(s_n, want ? 1u : 0u, FULL);
    if (want) {
      if (pos < qlimit)
        s.q[0][pos] = (uint16_t)p;
      else
        *s_over = 1;
    }
  }
  __syncthreads();
  unsigned n = *s_n;
  return n < qlimit ? n : qlimit;
}

// BQ propagation to the tile-local fixed point (level-synchronous inside
// the CTA; K.220-270 semantics with atomicMax merges, recon.py:92-101).
// Dropped work (BQ overflow) is recovered by a full rescan of the tile.
template <int CONN>
__device__ void tile_fixpoint(SmemLayout &s, unsigned *s_n, unsigned *s_over, unsigned *s_changed,
                              unsigned qlimit, unsigned long long &pushes,
                              unsigned long long &overflows, unsigned long long &seeds) {
  const unsigned FULL = 0xffffffffu;
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int cur = 0;
  unsigned n = 0;
  bool rescan = true;
  for (;;) {
    if (n == 0) {
      if (!rescan) break;
      if (threadIdx.x == 0) {
        s_n[0] = 0;
        *s_over = 0;
      }
      __syncthreads();
      n = detect_seeds<CONN>(s, &s_n[0], s_over, qlimit);
      rescan = *s_over != 0;
      if (threadIdx.x == 0) {
        seeds += n;
        if (rescan) overflows++;
      }
      cur = 0;
      __syncthreads();
      if (n == 0) break;
    }
    if (threadIdx.x == 0) {
      s_n[1 - cur] = 0;
      *s_over = 0;
    }
    __syncthreads();
    const uint16_t *in = s.q[cur];
    uint16_t *out = s.q[1 - cur];
    for (unsigned base = warp * 32; base < n; base += blockDim.x) {
      unsigned i = base + lane;
      unsigned mask = 0;
      int p = 0;
      if (i < n) {
        p = in[i];
        int v = s.J[p];
        int py = p / PW, px = p - py * PW;
#pragma unroll
        for (int k = 0; k < Nbr<CONN>::N; k++) {
          int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
          if (interior(qx, qy)) {
            int qq = qy * PW + qx;
            int vq = s.J[qq];
            int iq = s.I[qq];
            if (vq < v && vq < iq) {
              int nv = v < iq ? v : iq;
              int old = atomicMax(&s.J[qq], nv);
              if (old < nv) mask |= 1u << k;
            }
          }
        }
      }
      unsigned cnt = __popc(mask);
      unsigned pos = warp_reserve(&s_n[1 - cur], cnt, FULL);
      if (cnt) {
        *s_changed = 1;
        int py = p / PW, px = p - py * PW;
        while (mask) {
          int k = __ffs(mask) - 1;
          mask &= mask - 1;
          if (pos < qlimit)
            out[pos] = (uint16_t)((py + Nbr<CONN>::dy(k)) * PW + px + Nbr<CONN>::dx(k));
          else
            *s_over = 1;
          pos++;
        }
      }
    }
    __syncthreads();
    unsigned nn = s_n[1 - cur];
    if (*s_over) {
      rescan = true;
      if (threadIdx.x == 0) overflows++;
      nn = qlimit;
    }
    if (threadIdx.x == 0) pushes += nn;
    cur = 1 - cur;
    n = nn;
    __syncthreads();
  }
}

template <typename T, int CONN>
__global__ void __launch_bounds__(kTileThreads) tile_engine_kernel(EngineArgs a,
                                                                   unsigned long long *counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SmemLayout s;
  s.J = (int *)smem_raw;
  s.I = s.J + PN;
  s.q[0] = (uint16_t *)(s.I + PN);
  s.q[1] = s.q[0] + QCAP;
  s.ring0 = (int *)(s.q[1] + QCAP);
  __shared__ int s_tile;
  __shared__ unsigned s_n[2], s_over, s_changed, s_dirs;

  unsigned long long n_tiles = 0, n_reruns = 0, n_push = 0, n_over = 0, n_seeds = 0;

  for (;;) {
    if (threadIdx.x == 0) {
      int t;
      for (;;) {
        t = ring_pop(a.q);
        if (t >= 0) {
          atomicExch(&a.q.state[t], ST_RUNNING);
          __threadfence();
          break;
        }
        if (ld_acquire(a.q.pending) == 0) break;
        __nanosleep(64);
      }
      s_tile = t;
    }
    __syncthreads();
    const int t = s_tile;
    if (t < 0) break;
    const int tx = t % a.ntx, ty = t / a.ntx;
    const int x0 = tx * TW, y0 = ty * TH;

    // full load of tile + halo
    for (int i = threadIdx.x; i < PN; i += blockDim.x) load_cell<T>(a, s, i, x0, y0);
    __syncthreads();
    for (int r = threadIdx.x; r < 4 * TW; r += blockDim.x) {
      int side = r / TW, k = r - side * TW;
      int lx = side < 2 ? k + 1 : (side == 2 ? 1 : TW);
      int ly = side < 2 ? (side == 0 ? 1 : TH) : k + 1;
      s.ring0[r] = s.J[ly * PW + lx];
    }
    bool first = true;
    for (;;) {  // re-run loop while neighbours dirtied this tile
      if (threadIdx.x == 0) {
        s_n[0] = 0;
        s_n[1] = 0;
        s_changed = 0;
        s_dirs = 0;
        n_tiles++;
        if (!first) n_reruns++;
      }
      __syncthreads();
      tile_fixpoint<CONN>(s, s_n, &s_over, &s_changed, a.qlimit, n_push, n_over, n_seeds);
      __syncthreads();
      if (s_changed) {
        // write back the interior
        for (int i = threadIdx.x; i < TW * TH; i += blockDim.x) {
          int ly = i / TW + 1, lx = i % TW + 1;
          int gx = x0 + lx - 1, gy = y0 + ly - 1;
          if (gx < a.W && gy < a.H) ((T *)a.J)[(size_t)gy * a.W + gx] = (T)s.J[ly * PW + lx];
        }
        __threadfence();
        // which neighbour tiles can the changed border still raise?
        for (int h = threadIdx.x; h < 2 * PW + 2 * TH; h += blockDim.x) {
          int lx, ly;
          if (h < PW) {
            lx = h;
            ly = 0;
          } else if (h < 2 * PW) {
            lx = h - PW;
            ly = TH + 1;
          } else if (h < 2 * PW + TH) {
            lx = 0;
            ly = h - 2 * PW + 1;
          } else {
            lx = TW + 1;
            ly = h - 2 * PW - TH + 1;
          }
          int hi = ly * PW + lx;
          int vh = s.J[hi];
          if (vh == INT_MIN && s.I[hi] == INT_MIN) continue;  // outside the image
          if (!(vh < s.I[hi])) continue;
          bool need = false;
#pragma unroll
          for (int k = 0; k < Nbr<CONN>::N; k++) {
            int bx = lx + Nbr<CONN>::dx(k), by = ly + Nbr<CONN>::dy(k);
            if (interior(bx, by)) {
              int ri = ring_index(bx, by);
              int vb = s.J[by * PW + bx];
              if (vb != s.ring0[ri] && vh < vb) need = true;
            }
          }
          if (need) {
            int dxi = lx == 0 ? 0 : (lx == TW + 1 ? 2 : 1);
            int dyi = ly == 0 ? 0 : (ly == TH + 1 ? 2 : 1);
            atomicOr(&s_dirs, 1u << (dyi * 3 + dxi));
          }
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_dirs) {
          unsigned d = s_dirs;
          while (d) {
            int b = __ffs(d) - 1;
            d &= d - 1;
            int ntxi = tx + (b % 3) - 1, ntyi = ty + (b / 3) - 1;
            if (ntxi >= 0 && ntxi < a.ntx && ntyi >= 0 && ntyi < a.nty)
              activate(a.q, (unsigned)(ntyi * a.ntx + ntxi));
          }
        }
        // the ring as now published
        for (int r = threadIdx.x; r < 4 * TW; r += blockDim.x) {
          int side = r / TW, k = r - side * TW;
          int lx = side < 2 ? k + 1 : (side == 2 ? 1 : TW);
          int ly = side < 2 ? (side == 0 ? 1 : TH) : k + 1;
          s.ring0[r] = s.J[ly * PW + lx];
        }
      }
      __syncthreads();
      // finish: RUNNING -> IDLE, or re-run if a neighbour dirtied us
      if (threadIdx.x == 0) {
        unsigned old = atomicCAS(&a.q.state[t], ST_RUNNING, ST_IDLE);
        if (old == ST_RUNNING) {
          __threadfence();
          atomicSub(a.q.pending, 1u);
          s_tile = -1;
        } else {
          atomicExch(&a.q.state[t], ST_RUNNING);
          __threadfence();
        }
      }
      __syncthreads();
      if (s_tile < 0) break;
      // re-run: refresh the halo only (the interior is ours and current)
      for (int h = threadIdx.x; h < 2 * PW + 2 * TH; h += blockDim.x) {
        int lx, ly;
        if (h < PW) {
          lx = h;
          ly = 0;
        } else if (h < 2 * PW) {
          lx = h - PW;
          ly = TH + 1;
        } else if (h < 2 * PW + TH) {
          lx = 0;
          ly = h - 2 * PW + 1;
        } else {
          lx = TW + 1;
          ly = h - 2 * PW - TH + 1;
        }
        load_cell<T>(a, s, ly * PW + lx, x0, y0);
      }
      first = false;
      __syncthreads();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    atomicAdd(&counters[CNT_TILES], n_tiles);
    atomicAdd(&counters[CNT_RERUNS], n_reruns);
    atomicAdd(&counters[CNT_PUSHES], n_push);
    atomicAdd(&counters[CNT_OVERFLOW], n_over);
    atomicAdd(&counters[CNT_SEEDS], n_seeds);
  }
}

__global__ void tile_queue_init_kernel(TileQueue q, unsigned ntiles, unsigned long long *counters) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  for (unsigned t = i; t < ntiles; t += gridDim.x * blockDim.x) {
    q.state[t] = ST_QUEUED;
    q.ring[t] = ((unsigned long long)t << 32) | t;
  }
  for (unsigned t = ntiles + i; t <= q.mask; t += gridDim.x * blockDim.x) q.ring[t] = ~0ull;
  if (i == 0) {
    *q.head = 0;
    *q.tail = ntiles;
    *q.pending = ntiles;
  }
  if (i < CNT_N) counters[i] = 0;
}

size_t tile_queue_bytes(unsigned ntiles) {
  unsigned cap = 1;
  while (cap < 2 * ntiles + 2) cap <<= 1;
  return align_up(sizeof(unsigned) * ntiles, 256) + align_up(sizeof(unsigned long long) * cap, 256) +
         256 * 2;
}

TileQueue carve_tile_queue(Carver &c, unsigned ntiles) {
  unsigned cap = 1;
  while (cap < 2 * ntiles + 2) cap <<= 1;
  TileQueue q;
  q.state = c.take<unsigned>(ntiles);
  q.ring = c.take<unsigned long long>(cap);
  q.mask = cap - 1;
  unsigned *ctr = c.take<unsigned>(4);
  q.head = ctr;
  q.tail = ctr + 1;
  q.pending = ctr + 2;
  return q;
}

template <typename T, int CONN>
static int launch_engine(void *J, const void *I, int W, int H, TileQueue q,
                         unsigned long long *counters, int max_blocks, int qcap, cudaStream_t st) {
  int ntx = (W + TW - 1) / TW, nty = (H + TH - 1) / TH;
  unsigned ntiles = (unsigned)ntx * nty;
  size_t smem = smem_bytes();
  auto kern = tile_engine_kernel<T, CONN>;
  IWPP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTileThreads, smem));
  if (per_sm < 1) per_sm = 1;
  int blocks = device_sm_count() * per_sm;
  if (max_blocks > 0 && blocks > max_blocks) blocks = max_blocks;
  if ((unsigned)blocks > ntiles) blocks = (int)ntiles;
  tile_queue_init_kernel<<<(ntiles + 255) / 256 > 1024 ? 1024 : (ntiles + 255) / 256 + 1, 256, 0, st>>>(
      q, ntiles, counters);
  IWPP_CUDA_TRY(cudaGetLastError());
  unsigned qlimit = (qcap > 0 && qcap < QCAP) ? (unsigned)qcap : (unsigned)QCAP;
  EngineArgs a{J, I, W, H, ntx, nty, ntiles, qlimit, q};
  kern<<<blocks, kTileThreads, smem, st>>>(a, counters);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int run_tile_engine(void *J, const void *I, int W, int H, int dtype, int conn, TileQueue q,
                    unsigned long long *counters, int max_blocks, int qcap, cudaStream_t st) {
#define DISPATCH(T)                                                                           \
  return conn == 8 ? launch_engine<T, 8>(J, I, W, H, q, counters, max_blocks, qcap, st)      \
                   : launch_engine<T, 4>(J, I, W, H, q, counters, max_blocks, qcap, st)
  switch (dtype) {
    case IWPP_U8:
      DISPATCH(uint8_t);
    case IWPP_U16:
      DISPATCH(uint16_t);
    case IWPP_I32:
      DISPATCH(int32_t);
  }
#undef DISPATCH
  return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
}

}  // namespace recon
}  // namespace iwpp
