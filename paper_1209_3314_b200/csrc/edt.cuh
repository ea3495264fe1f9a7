// edt.cuh -- level-synchronous EDT engine interface (see edt.cu).
#pragma once
#include "iwpp_common.cuh"

namespace iwpp {
namespace edt {

constexpr uint32_t INF32 = 0xFFFFFFFFu;
constexpr uint32_t SEED_STAMP = 0xFFFFFFFEu;
#ifndef IWPP_EDT_ROUND_THREADS
#define IWPP_EDT_ROUND_THREADS 256
#endif
#ifndef IWPP_EDT_ROUND_BLOCKS
#define IWPP_EDT_ROUND_BLOCKS 4
#endif
constexpr int kRoundThreads = IWPP_EDT_ROUND_THREADS;
constexpr int kRoundBlocksPerSm = IWPP_EDT_ROUND_BLOCKS;
constexpr int kEdtBq = 6144;  // per-block next-frontier buffer (shared memory, 24 KB)
// rounds whose frontier is smaller than this run as queue rounds (returned
// atomics + block queues) instead of raster rounds (bitmap + compaction)
#ifndef IWPP_RASTER_MIN
#define IWPP_RASTER_MIN 262144
#endif
constexpr unsigned kRasterMinFrontier = IWPP_RASTER_MIN;

enum { EC_ROUNDS = 0, EC_VISITS, EC_NINF, EC_LIMIT, EC_FINAL, EC_BAD, EC_RANGE, EC_LASTCHG, EC_N = 8 };

struct EdtState {
  int keymode;               // 1: 64-bit keys (d2 << 32 | src), 0: 32-bit sources + CAS
  int keycheck;              // keymode on an image whose d2 may exceed 32 bits: every offer
                             // checks the range and flags EC_RANGE instead of wrapping
  unsigned long long *keys;  // keymode: 2 keys per cell (AoS, double-buffered)
  uint32_t *buf[2];          // !keymode: source per cell, (sy << 16 | sx), double-buffered
  uint32_t *stamp;           // !keymode: round stamp per cell (frontier dedupe)
  uint32_t *F[2];            // frontier queues (yx codes)
  unsigned *cnt;             // [3] frontier sizes (triple-buffered)
  unsigned *bar;             // grid barrier: [0] arrivals, [kBarGen] generation
  unsigned long long *counters;
  // block engine (edt_block.cu)
  int block;                 // keymode runs on the temporally blocked engine
  int raster;                // keymode runs on the raster-frontier engine
  unsigned long long *plane[2];  // block engine: two key planes (no interleave)
  uint32_t *fbits[2];        // frontier bitmaps (row-major, ceil(W/32) words per row)
  unsigned *rplane;          // per region: (pass << 1) | plane holding its current keys
  unsigned *fstamp[2];       // per region: pass for which fbits[b] holds its frontier
  unsigned *astamp;          // per region: last pass it was activated for
  unsigned *rflag;           // per region: holds seeds (init)
  unsigned *alist[3];        // active region lists (triple-buffered)
  unsigned *acnt, *wc;       // [3] list sizes, [3] work counters
  unsigned long long *diag;  // [16] block-engine diagnostics (IWPP_TRACE)
  unsigned long long *rtrace;  // per-round (globaltimer, frontier) pairs or null (IWPP_EDT_RTRACE)
};

// Images the 32-bit (y,x) source code can address.
inline bool size_supported(int64_t W, int64_t H) {
  return W >= 1 && H >= 1 && W <= 65536 && H <= 65536;
}
// The CAS engine's INF code (all ones) must not be a cell's own code.
inline bool cas_supported(int64_t W, int64_t H) {
  return size_supported(W, H) && !(W == 65536 && H == 65536);
}
// Engine selection (tests / diagnostics): 0 auto, 1 force the CAS engine,
// 2 force range-checked keys.
enum {
  ENGINE_AUTO = 0, ENGINE_CAS = 1, ENGINE_KEYCHECK = 2, ENGINE_QUEUE = 3, ENGINE_BLOCK = 4,
  ENGINE_QUEUE_PF = 5,    // queue engine, next frontier by warp reservations in global memory
  ENGINE_QUEUE_NAIVE = 6, // queue engine, one global atomic per pushed item
  ENGINE_RASTER = 7       // raster-frontier engine (bitmap + compaction, no returned atomics)
};

extern thread_local int g_engine_override;
// The key engine needs every squared distance to fit 32 bits.
inline bool key_mode_ok(int64_t W, int64_t H) {
  return (uint64_t)(W - 1) * (W - 1) + (uint64_t)(H - 1) * (H - 1) < (1ull << 32);
}

// key = (d2(q, src) << 32) | src_yx: the reference's total order at q
// (K.320-336) as a plain unsigned order; INF (no source) = all ones.
constexpr unsigned long long KINF = ~0ull;

__device__ __forceinline__ unsigned long long make_key(int qx, int qy, uint32_t src) {
  int sy = (int)(src >> 16), sx = (int)(src & 0xffffu);
  unsigned dx = (unsigned)abs(qx - sx), dy = (unsigned)abs(qy - sy);
  unsigned d2 = dx * dx + dy * dy;  // < 2^32 by key_mode_ok
  return ((unsigned long long)d2 << 32) | src;
}
// Range-checked key: d2 in 64 bits; *ok = false when it needs more than 32.
__device__ __forceinline__ unsigned long long make_key_checked(int qx, int qy, uint32_t src,
                                                               bool &ok) {
  int sy = (int)(src >> 16), sx = (int)(src & 0xffffu);
  unsigned long long dx = (unsigned)abs(qx - sx), dy = (unsigned)abs(qy - sy);
  unsigned long long d2 = dx * dx + dy * dy;
  ok = (d2 >> 32) == 0;
  return (d2 << 32) | src;
}

// Software grid barrier for the persistent cooperative kernels.
// Thread 0's view of the barrier generation, read once at kernel start
// (every block reads it before its first arrival, so no block can have
// advanced it yet) and then tracked locally: one round trip less per barrier.
constexpr int kBarGen = 64;  // generation word offset (its own 256-byte line)

__device__ __forceinline__ unsigned grid_barrier_gen(const unsigned *gen) {
  return threadIdx.x == 0 ? ld_acquire(gen) : 0u;
}

__device__ __forceinline__ void grid_barrier(unsigned *count, unsigned *gen, unsigned nblocks,
                                             unsigned &g) {
  // Arrival is an acq_rel RMW (publishes this block's writes, and the last
  // arriver acquires everyone's); the release is a release add on the
  // generation, which the waiters acquire.  No sequentially consistent
  // fences (MEMBAR.SC) on the round's critical path.
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned arrived;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(count) : "memory");
    if (arrived == nblocks - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
    } else {
      while (ld_acquire(gen) == g) __nanosleep(16);
    }
    g++;
  }
  __syncthreads();
}

size_t state_bytes(int64_t W, int64_t H);

// slab engine (edt_slab.cu): one round per launch, halo items from the
// neighbours, boundary frontier rows out (source or KINF per column)
size_t slab_bytes(int64_t W, int64_t h);
int slab_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H, int conn,
              int has_up, int has_down, void *ws, unsigned long long *out_up,
              unsigned long long *out_dn, cudaStream_t st);
int slab_round(void *ws, int64_t W, int64_t h, int64_t y0, int conn, int64_t r,
               const unsigned long long *halo_up, const unsigned long long *halo_dn,
               unsigned long long *out_up, unsigned long long *out_dn, int64_t *n_next_host,
               cudaStream_t st);
int slab_finalize(void *ws, int64_t W, int64_t h, int64_t y0, int64_t rounds, int64_t *vr,
                  float *dist, int64_t *n_inf_host, int64_t *range_err_host, cudaStream_t st);
// device-resident multi-slab rounds (edt_slab.cu; iwpp_edt_mg_*)
size_t mg_slab_bytes(int64_t W, int64_t h);
size_t mg_mailbox_bytes(int64_t W);
int mg_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H, int conn, int has_up,
            int has_down, void *ws, void *mailbox, void *mb_up, void *mb_dn, cudaStream_t st);
int mg_run(const iwpp_edt_mg_slab *slabs, int nlocal, int conn, long long max_rounds, int64_t *rounds_host,
           cudaStream_t st);
EdtState carve_state(Carver &c, int64_t W, int64_t H, bool cas = false);
int read_counters(const EdtState &s, unsigned long long *c, cudaStream_t st);
int reset_control(const EdtState &s, cudaStream_t st);
// r0 (out, may be null): 1 when round 0 ran in the init (raster engine) --
// then launch_rounds must start at r0
int launch_init(const uint8_t *mask, int W, int H, int conn, const EdtState &s, cudaStream_t st,
                int *r0 = nullptr);
int launch_import(const int64_t *vr, const int64_t *seeds, int64_t n_seeds, int W, int H,
                  const EdtState &s, cudaStream_t st);
int launch_rounds(int W, int H, int conn, const EdtState &s, long long max_rounds,
                  cudaStream_t st, int r0 = 0);
int launch_finalize_auto(const EdtState &s, int W, int H, int64_t *vr, float *dist, int64_t *d2,
                         cudaStream_t st);
// block engine (edt_block.cu)
constexpr int kBlockShift = 6;
constexpr int kBlockC = 1 << kBlockShift;  // region side (central cells)
constexpr int kBlockK = 8;                 // halo width = local rounds per pass
constexpr int kBlockThreads = 512;
constexpr int kBlockMinCtas = 2;
inline int64_t block_regions(int64_t W, int64_t H) {
  return ((W + kBlockC - 1) / kBlockC) * ((H + kBlockC - 1) / kBlockC);
}
int block_init(const uint8_t *mask, const int64_t *vr, const int64_t *seeds, int64_t n_seeds,
               int W, int H, int conn, const EdtState &s, cudaStream_t st);
int block_rounds(int W, int H, int conn, const EdtState &s, long long max_rounds, cudaStream_t st);
int block_finalize(const EdtState &s, int W, int H, int64_t *vr, float *dist, int64_t *d2,
                   cudaStream_t st);
int launch_finalize_vr(const int64_t *vr, int W, int H, float *dist, int64_t *d2,
                       unsigned long long *counters, cudaStream_t st);

}  // namespace edt
}  // namespace iwpp
