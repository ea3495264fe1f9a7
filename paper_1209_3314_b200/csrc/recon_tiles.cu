// recon_tiles.cu -- persistent warp-per-tile engine for morphological
// reconstruction by dilation.
//
// Replaces the reference's scan + wavefront phases (recon_raster_pass /
// recon_antiraster_pass K.38-112, recon_rows/cols K.115-190, recon_seed_scan
// K.193-217, recon_wavefront K.220-270, the round engine engine.py:251-364)
// with one persistent sm_100a kernel.  Every warp is an independent worker
// that owns one 32x32 tile (+ 1-pixel halo) at a time in its own slice of
// shared memory -- no CTA barriers anywhere, ~20 tiles in flight per SM.
// Per tile activation:
//
//   1. load tile + halo (16-byte vector loads of the rows, L2-coherent)
//   2. halo offers: every (halo -> border cell) pair is applied once, so the
//      halo never has to be queued (values only grow: an applied offer stays
//      satisfied) and all queue items are interior cells
//   3. sweeps (first visit, or a wide front entering): lane = line, each
//      lane walks its row W->E / E->W, then its column N->S / S->N with
//      v <- clamp(v, J, I) -- the paper's raster / anti-raster scan phase in
//      its axis-decomposed form (Alg. 5)
//   4. initial-wavefront detection fused into the last walk: a cell is
//      active iff it can raise a neighbour (J(q) < J(p), J(q) < I(q)), i.e.
//      J(p) > min over N(p) of the "raisable" values -- a 3x3 (8-conn) /
//      cross (4-conn) min filter, sliding row window in registers,
//      ballot-compacted into the warp's pixel queue
//   5. propagation to the tile's fixed point: the warp drains its pixel
//      queue 32 items per step; each lane offers its cell's value to its 8
//      (4) neighbours with predicated shared atomicMax
//      (J(q) <- min(J(p), I(q)) iff J(q) < J(p) and J(q) != I(q),
//      recon.py:92-101); pushes are placed by bit-plane ballots (no atomics)
//   6. write the interior back and activate the neighbour tiles whose cells
//      the changed border can still raise.
//
// Sentinels instead of bounds checks: halo cells and cells outside the image
// carry I = min(T) in the propagation arrays (never raisable); cells outside
// the image also carry J = min(T) (raise nothing).  The halo's real mask
// values live apart (Ih) for the activation test.
//
// Queue hierarchy (the paper's TQ/BQ/GBQ):
//   TQ  : per-lane register bitmask of raised neighbours (<= 8 bits)
//   BQ  : per-warp shared-memory pixel ring, ballot/popc placement
//   GBQ : global MPMC ring of tile ids (ticket pop, per-tile state bits);
//         a tile whose halo a neighbour raised re-enters it -- the BP border
//         exchange of tiles.py:342-359, asynchronous, no wave barriers.
// BQ overflow (user-forced small capacity, QueueConfig.gbq_capacity) drops
// work and re-seeds the tile by a full rescan -- the drop / rescan /
// re-execute contract of engine.py:274-303.
// Termination: a global count of queued+running tiles reaches 0.
//
// The fixed point is unique (engine.py:9-18), so this asynchronous schedule
// is bit-exact with recon_fh.

#include <climits>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include <cooperative_groups.h>
#include <type_traits>
#include <vector>
#include <cuda.h>  // CUtensorMap (the encoder is fetched from the driver at run time)

#include "iwpp_common.cuh"
#include "recon_tiles.cuh"

namespace iwpp {
namespace recon {

constexpr unsigned FULL = 0xffffffffu;
constexpr unsigned ST_Q = 1, ST_R = 2, ST_V = 4;
constexpr int RING = 4 * TS + 4;  // halo cells

template <typename T>
struct alignas(16) WarpSmem {
  int J[PNS];
  alignas(16) T I[PNS];    // interior: mask; halo / outside the image: min(T)
  alignas(16) T Ih[RING];  // the halo's real mask values (activation test)
  alignas(16) uint16_t ring[RQ];  // pixel queue (absolute positions mod RQ)
  int ring0[4 * TS];              // border ring as last published
};

struct EngineArgs {
  void *J;
  const void *I;
  int W, H;
  int ntx, nty;
  unsigned qlimit;       // pixel-queue capacity actually used (<= RQ)
  unsigned halo_thresh;  // re-activation front above which to sweep first
  int sweeps;            // sweep passes on a tile's first visit
  int vec;               // rows are 16-byte aligned
  uint8_t *dirty;        // per tile row: written by this run (nullable)
  int WW;                // binary engine: words per bit-plane row
  TileQueue q;
  unsigned long long ntx_m;  // ceil(2^40 / ntx) (0: divide): tile id -> (tx, ty)
};

// tile id -> (tx, ty) without an integer division (exact while ntx < 2^14
// and t < 2^26; the launcher sets ntx_m = 0 beyond that)
__device__ __forceinline__ void tile_xy(const EngineArgs &a, unsigned t, int &tx, int &ty) {
  if (a.ntx_m) {
    ty = (int)((t * a.ntx_m) >> 40);
    tx = (int)(t - (unsigned)ty * (unsigned)a.ntx);
  } else {
    tx = (int)(t % (unsigned)a.ntx);
    ty = (int)(t / (unsigned)a.ntx);
  }
}

__device__ __forceinline__ int sidx(int lx, int ly) { return ly * PS + lx; }
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return min(hi, max(lo, v)); }
template <int CONN>
__device__ __forceinline__ int noff(int k) {  // neighbour k as a shared-memory index offset
  return Nbr<CONN>::dy(k) * PS + Nbr<CONN>::dx(k);
}

// halo cell h in [0, RING) -> (lx, ly): top row, bottom row, left, right
__device__ __forceinline__ void halo_cell(int h, int &lx, int &ly) {
  if (h < PW) {
    lx = h;
    ly = 0;
  } else if (h < 2 * PW) {
    lx = h - PW;
    ly = TS + 1;
  } else if (h < 2 * PW + TS) {
    lx = 0;
    ly = h - 2 * PW + 1;
  } else {
    lx = TS + 1;
    ly = h - 2 * PW - TS + 1;
  }
}

// border-ring slot of an interior edge cell (corners map to the rows)
__device__ __forceinline__ int ring_index(int lx, int ly) {
  if (ly == 1) return lx - 1;
  if (ly == TS) return TS + lx - 1;
  if (lx == 1) return 2 * TS + ly - 1;
  return 3 * TS + ly - 1;  // lx == TS
}
__device__ __forceinline__ void ring_cell(int r, int &lx, int &ly) {
  int side = r / TS, k = r - side * TS;
  lx = side < 2 ? k + 1 : (side == 2 ? 1 : TS);
  ly = side < 2 ? (side == 0 ? 1 : TS) : k + 1;
}

// --- global tile queue (GBQ) -------------------------------------------------

__device__ __forceinline__ void ring_push(const TileQueue &q, unsigned t) {
  unsigned pos = atomicAdd(q.tail, 1u);
  st_release64(&q.ring[pos & q.mask], ((unsigned long long)pos << 32) | t);
}

// Ticket pop: one fetch-and-add per pop (no CAS retry storms on the head),
// then wait until the slot carries the ticket's tag.  Returns -1 once the
// engine has terminated (no tile queued or running: nothing can be pushed
// any more, and a filled slot would imply a queued tile).  Idle workers back
// off to ~1 us so they do not steal issue slots from busy ones.
constexpr int kBinCtasPerSm = 4;

#ifndef IWPP_POP_MAX_SLEEP_NS
#define IWPP_POP_MAX_SLEEP_NS 2048
#endif
constexpr unsigned kPopMaxSleepNs = IWPP_POP_MAX_SLEEP_NS;
#ifndef IWPP_PENDING_POLL_NS
#define IWPP_PENDING_POLL_NS 1024
#endif
constexpr unsigned kPendingPollNs = IWPP_PENDING_POLL_NS;

template <unsigned PollNs = kPendingPollNs>
__device__ __forceinline__ int ring_pop(const TileQueue &q, unsigned long long *idle = nullptr) {
  unsigned ticket = atomicAdd(q.head, 1u);
  unsigned long long *slot = &q.ring[ticket & q.mask];
  for (unsigned ns = 32;; ns = ns < kPopMaxSleepNs ? ns * 2 : kPopMaxSleepNs) {
    unsigned long long v = ld_acquire64(slot);
    if ((unsigned)(v >> 32) == ticket) return (int)(v & 0xffffffffu);
    if (idle) ++*idle;  // queue-occupancy evidence: polls that found the slot empty
    // the termination test reads the hot pending line: only once the
    // slot has stayed empty for a few polls (PollNs; the binary engine's
    // narrow fronts keep most warps idle and measured best polling at once)
    if constexpr (PollNs <= 32) {
      if (ld_acquire(q.pending) == 0) return -1;
    } else {
      if (ns >= PollNs && ld_acquire(q.pending) == 0) return -1;
    }
    __nanosleep(ns);
  }
}

// Activation trace (development builds with -DIWPP_ATRACE; queue-occupancy
// and concurrency evidence): lane 0 of the register engine appends one
// record per tile activation -- globaltimer at pop start / tile taken / boxes
// loaded / fixed point / activation end (ns, low 32 bits), the tile, the
// SM, the Jacobi steps and the ring depth (tail - ticket) seen at the pop.
struct ATraceRec {
  unsigned t_pop, t_take, t_load, t_fix, t_end, tile, sm_steps, depth;
};
#ifdef IWPP_ATRACE
__device__ ATraceRec *g_atrace;
__device__ unsigned g_atrace_n, g_atrace_cap;
__device__ __forceinline__ unsigned gtime32() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (unsigned)t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
constexpr bool kATrace = true;
#else
__device__ __forceinline__ unsigned gtime32() { return 0; }
__device__ __forceinline__ unsigned smid() { return 0; }
constexpr bool kATrace = false;
#endif

// Tile state bits: Q = queued, or re-run requested while running; R =
// running; V = never processed (set only by the initial fill).
//   activate : old = atomicOr(Q); old == 0 (idle) -> we own the push
//   pop      : old = acquire exchange to R (sees every border write
//              made before a request that found Q already set)
//   finish   : CAS(R -> 0), after a changed tile fenced its stores (the
//              next owner loads them); failure means Q was set meanwhile -> re-run
// Returns true when the caller now owns an idle tile's activation (it must
// either push it or process it itself); pending already counts it.
// Take a tile (state <- R) with acquire semantics: the borders published
// before any request this consumes are visible afterwards.  An acquire RMW
// (ATOM + L1 invalidate) rather than RMW + fence.acq_rel.  (A changed tile
// fences its own stores before its finish, so nothing unfenced is pending.)
#ifndef IWPP_STATE_ACQ
#define IWPP_STATE_ACQ 1
#endif
#ifndef IWPP_CTR_SPREAD
#define IWPP_CTR_SPREAD 1
#endif
#ifndef IWPP_FUSED_INIT
#define IWPP_FUSED_INIT 1
#endif
// below this many tiles a cooperative launch costs more than the init kernel
constexpr unsigned kFusedInitMinTiles = 128;
__device__ __forceinline__ unsigned state_take(unsigned *p) {
#if IWPP_STATE_ACQ
  unsigned old;
  asm volatile("atom.acquire.gpu.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(ST_R) : "memory");
  // Consume the returned value here: with the result unused, ptxas emits the
  // exchange with no destination and nothing waits for it, so a TMA box load
  // (async proxy) issued next could read a border published before the
  // request this exchange consumes from before it became visible.
  if (old > (ST_Q | ST_R | ST_V)) __trap();
  return old;
#else
  const unsigned old = atomicExch(p, ST_R);
  fence_acq_rel();
  return old;
#endif
}

// the claim alone: the caller accounts for pending itself
__device__ __forceinline__ bool activate_claim_nopend(const TileQueue &q, unsigned t) {
  return atomicOr(&q.state[t], ST_Q) == 0;
}

__device__ __forceinline__ bool activate_claim(const TileQueue &q, unsigned t) {
  unsigned old = atomicOr(&q.state[t], ST_Q);
  if (old == 0) {
    atomicAdd(q.pending, 1u);
    return true;
  }
  return false;
}

// --- loads / stores (warp) -----------------------------------------------------

template <typename T>
__device__ void load_halo(const EngineArgs &a, WarpSmem<T> &s, int x0, int y0, int lane) {
  constexpr int LO = (int)Elem<T>::lo;
  constexpr int NH = (RING + 31) / 32;
  // all of the lane's halo loads first (independent), then the stores
  int jv[NH];
  T iv[NH];
#pragma unroll
  for (int k = 0; k < NH; k++) {
    const int h = lane + 32 * k;
    jv[k] = LO;
    iv[k] = Elem<T>::lo;
    if (h < RING) {
      int lx, ly;
      halo_cell(h, lx, ly);
      const int gx = x0 + lx - 1, gy = y0 + ly - 1;
      if (gx >= 0 && gx < a.W && gy >= 0 && gy < a.H) {
        const size_t g = (size_t)gy * a.W + gx;
        jv[k] = (int)ld_cg((const T *)a.J + g);
        iv[k] = __ldg((const T *)a.I + g);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < NH; k++) {
    const int h = lane + 32 * k;
    if (h < RING) {
      int lx, ly;
      halo_cell(h, lx, ly);
      const int i = sidx(lx, ly);
      s.I[i] = Elem<T>::lo;  // never raisable from inside the tile
      s.J[i] = jv[k];
      s.Ih[h] = iv[k];
    }
  }
}

// lane = row; full-width aligned rows go by 16-byte vectors
template <typename T>
__device__ void load_tile(const EngineArgs &a, WarpSmem<T> &s, int x0, int y0, int lane) {
  constexpr int E = 16 / sizeof(T), CPR = TS / E;
  constexpr int LO = (int)Elem<T>::lo;
  const int ly = lane + 1, gy = y0 + lane;
  if (a.vec && x0 + TS <= a.W && gy < a.H) {
    const T *pj = (const T *)a.J + (size_t)gy * a.W + x0;
    const T *pi = (const T *)a.I + (size_t)gy * a.W + x0;
#pragma unroll
    for (int c = 0; c < CPR; c++) {
      uint4 vj = __ldcg(reinterpret_cast<const uint4 *>(pj) + c);
      uint4 vi = __ldg(reinterpret_cast<const uint4 *>(pi) + c);
      const T *ej = reinterpret_cast<const T *>(&vj);
      const T *ei = reinterpret_cast<const T *>(&vi);
#pragma unroll
      for (int e = 0; e < E; e++) {
        s.J[sidx(1 + c * E + e, ly)] = (int)ej[e];
        s.I[sidx(1 + c * E + e, ly)] = ei[e];
      }
    }
  } else {
    for (int lx = 1; lx <= TS; lx++) {
      int gx = x0 + lx - 1, i = sidx(lx, ly);
      if (gx < a.W && gy < a.H) {
        size_t g = (size_t)gy * a.W + gx;
        s.J[i] = (int)ld_cg((const T *)a.J + g);
        s.I[i] = __ldg((const T *)a.I + g);
      } else {  // outside the image: raises nothing, never raised
        s.J[i] = LO;
        s.I[i] = Elem<T>::lo;
      }
    }
  }
  load_halo<T>(a, s, x0, y0, lane);
}

template <typename T>
__device__ void store_tile(const EngineArgs &a, WarpSmem<T> &s, int x0, int y0, int limx,
                           int limy, int lane) {
  constexpr int E = 16 / sizeof(T), CPR = TS / E;
  const int ly = lane + 1, gy = y0 + lane;
  if (ly > limy) return;
  T *pj = (T *)a.J + (size_t)gy * a.W + x0;
  if (a.vec && x0 + TS <= a.W) {
#pragma unroll
    for (int c = 0; c < CPR; c++) {
      uint4 v;
      T *ev = reinterpret_cast<T *>(&v);
#pragma unroll
      for (int e = 0; e < E; e++) ev[e] = (T)s.J[sidx(1 + c * E + e, ly)];
      reinterpret_cast<uint4 *>(pj)[c] = v;
    }
  } else {
    for (int lx = 1; lx <= limx; lx++) pj[lx - 1] = (T)s.J[sidx(lx, ly)];
  }
}

// --- halo offers ---------------------------------------------------------------
//
// Apply every (halo h -> border cell q) offer once: J(q) <- max(J(q),
// min(J(h), I(q))).  Sides run one after the other (a corner cell belongs to
// two sides), lane = position along the side.  Returns, per lane, a bitmask
// of the sides whose border cell this lane raised.
template <int CONN, typename T>
__device__ unsigned halo_offers(WarpSmem<T> &s, int lane) {
  const int k = lane + 1;
  unsigned raised = 0;
  // (q, halo row/col offset direction): top, bottom, left, right
#pragma unroll
  for (int side = 0; side < 4; side++) {
    int qx, qy, hx, hy, sx, sy;  // q, the facing halo cell, step along the side
    if (side == 0) { qx = k; qy = 1; hx = k; hy = 0; sx = 1; sy = 0; }
    else if (side == 1) { qx = k; qy = TS; hx = k; hy = TS + 1; sx = 1; sy = 0; }
    else if (side == 2) { qx = 1; qy = k; hx = 0; hy = k; sx = 0; sy = 1; }
    else { qx = TS; qy = k; hx = TS + 1; hy = k; sx = 0; sy = 1; }
    int q = sidx(qx, qy);
    int best = s.J[sidx(hx, hy)];
    if (CONN == 8) {
      best = max(best, s.J[sidx(hx - sx, hy - sy)]);
      best = max(best, s.J[sidx(hx + sx, hy + sy)]);
    }
    int jq = s.J[q], iq = (int)s.I[q];
    int nv = min(best, iq);
    if (nv > jq) {
      s.J[q] = nv;
      raised |= 1u << side;
    }
    __syncwarp();
  }
  return raised;
}

// queue a ballot of cells (one per lane) at the warp tail; returns the new tail
__device__ __forceinline__ unsigned push_ballot(uint16_t *ring, unsigned t, bool want, int p,
                                                unsigned qlimit) {
  unsigned k = __ballot_sync(FULL, want);
  unsigned pos = t + __popc(k & lanemask_lt());
  if (want && pos < qlimit) ring[pos & (RQ - 1)] = (uint16_t)p;
  return t + __popc(k);
}

__device__ __forceinline__ unsigned queue_halo_raised(uint16_t *ring, unsigned t, unsigned raised,
                                                      unsigned qlimit, int lane) {
  const int k = lane + 1;
  t = push_ballot(ring, t, raised & 1u, sidx(k, 1), qlimit);
  t = push_ballot(ring, t, raised & 2u, sidx(k, TS), qlimit);
  t = push_ballot(ring, t, raised & 4u, sidx(1, k), qlimit);
  t = push_ballot(ring, t, raised & 8u, sidx(TS, k), qlimit);
  return t;
}

// --- sweeps (the paper's scan phase, Alg. 5 axis decomposition) ---------------
//
// lane = line; the lane walks its 32 cells with v <- clamp(v, J, I) from the
// cell before the line: rows W->E then E->W (K.115-139), then columns N->S
// then S->N (K.142-190, vertical neighbour).  Straight-line code: compile-
// time stride, a chunk's loads issued together, unconditional stores.  A
// clamp through a sentinel cell (I = min(T)) can never raise an in-image cell.
template <int STEP, typename T>
__device__ __forceinline__ bool walk_line(WarpSmem<T> &s, int first, int carry_idx) {
  constexpr int C = 8;
  int v = s.J[carry_idx];
  bool chg = false;
#pragma unroll 1
  for (int k0 = 0; k0 < TS; k0 += C) {
    int j[C], m[C];
#pragma unroll
    for (int c = 0; c < C; c++) {
      j[c] = s.J[first + (k0 + c) * STEP];
      m[c] = (int)s.I[first + (k0 + c) * STEP];
    }
#pragma unroll
    for (int c = 0; c < C; c++) {
      int nv = clampi(v, j[c], m[c]);
      chg |= nv != j[c];
      s.J[first + (k0 + c) * STEP] = nv;
      v = nv;
    }
  }
  return chg;
}

// Column walk, lane = column.  8-connectivity takes the three cells of the
// previous row (K.142-190: {NW, N, NE} forward, {SW, S, SE} backward): the
// diagonal values come from the neighbouring lanes' registers (lanes 0 / 31
// read the side halo column), so a diagonal wavefront crosses the tile in
// one walk instead of being left to the queue.
template <int CONN, int DIR, typename T>
__device__ __forceinline__ bool walk_col(WarpSmem<T> &s, int lane) {
  if (CONN == 4) {
    const int k = lane + 1;
    return DIR > 0 ? walk_line<PS>(s, sidx(k, 1), sidx(k, 0))
                   : walk_line<-PS>(s, sidx(k, TS), sidx(k, TS + 1));
  }
  const int x = lane + 1;
  const int y0 = DIR > 0 ? 1 : TS, yc = DIR > 0 ? 0 : TS + 1;
  const bool edge = lane == 0 || lane == 31;
  const int side = lane == 0 ? 0 : TS + 1;
  int v = s.J[sidx(x, yc)];
  int sv = edge ? s.J[sidx(side, yc)] : INT_MIN;
  bool chg = false;
  constexpr int C = 8;
#pragma unroll 1
  for (int k0 = 0; k0 < TS; k0 += C) {
    int j[C], m[C], sn[C];
#pragma unroll
    for (int c = 0; c < C; c++) {
      const int y = y0 + DIR * (k0 + c);
      j[c] = s.J[sidx(x, y)];
      m[c] = (int)s.I[sidx(x, y)];
      sn[c] = edge ? s.J[sidx(side, y)] : INT_MIN;
    }
#pragma unroll
    for (int c = 0; c < C; c++) {
      int l = __shfl_up_sync(FULL, v, 1), r = __shfl_down_sync(FULL, v, 1);
      if (lane == 0) l = sv;
      if (lane == 31) r = sv;
      const int nv = clampi(max(v, max(l, r)), j[c], m[c]);
      chg |= nv != j[c];
      s.J[sidx(x, y0 + DIR * (k0 + c))] = nv;
      v = nv;
      sv = sn[c];
    }
  }
  return chg;
}

template <int CONN, typename T>
__device__ bool sweep_pass(WarpSmem<T> &s, int lane) {
  const int k = lane + 1;
  bool chg = walk_line<1>(s, sidx(1, k), sidx(0, k));
  chg |= walk_line<-1>(s, sidx(TS, k), sidx(TS + 1, k));
  __syncwarp();
  chg |= walk_col<CONN, 1>(s, lane);
  __syncwarp();
  chg |= walk_col<CONN, -1>(s, lane);
  __syncwarp();
  return __any_sync(FULL, chg);
}

// --- detection -----------------------------------------------------------------
//
// Raisable value m(q) = J(q) if J(q) < I(q) else +inf (halo and outside cells
// are never raisable by construction).  p is active iff J(p) > min over N(p)
// of m.  lane = column; lr = min(m left, m right) by shuffles (the halo
// columns' m is +inf).

__device__ __forceinline__ int lr_of(int m, int lane) {
  int l = __shfl_up_sync(FULL, m, 1), r = __shfl_down_sync(FULL, m, 1);
  if (lane == 0) l = INT_MAX;
  if (lane == 31) r = INT_MAX;
  return min(l, r);
}

template <int CONN>
__device__ __forceinline__ int window_lo(int m_n, int lr_n, int m_c, int lr_c, int m_p, int lr_p) {
  return CONN == 8 ? min(min(min(m_p, lr_p), min(m_c, lr_c)), min(m_n, lr_n))
                   : min(min(lr_c, m_p), m_n);
}

// Full detection over the interior (rows stream through a 3-row window).
template <int CONN, typename T>
__device__ unsigned detect_full(WarpSmem<T> &s, unsigned t, unsigned qlimit, int lane) {
  const int x = lane + 1;
  auto mrow = [&](int y, int &m, int &j) {
    int i = sidx(x, y);
    j = s.J[i];
    m = j < (int)s.I[i] ? j : INT_MAX;
  };
  int m_p = INT_MAX, lr_p = INT_MAX, m_c, lr_c, j_c, jd;
  mrow(0, m_c, jd);  // row 0 is halo: m = +inf
  lr_c = lr_of(m_c, lane);
  m_p = m_c;
  lr_p = lr_c;
  mrow(1, m_c, j_c);
  lr_c = lr_of(m_c, lane);
#pragma unroll 4
  for (int y = 1; y <= TS; y++) {
    int m_n, j_n;
    mrow(y + 1, m_n, j_n);
    int lr_n = lr_of(m_n, lane);
    t = push_ballot(s.ring, t, j_c > window_lo<CONN>(m_n, lr_n, m_c, lr_c, m_p, lr_p),
                    sidx(x, y), qlimit);
    m_p = m_c;
    lr_p = lr_c;
    m_c = m_n;
    lr_c = lr_n;
    j_c = j_n;
  }
  return t;
}

// One sweep pass whose last walk (columns S->N, lane = column) also does the
// detection: once the walk has finalised row y, rows y..y+2 are final, so
// the centre row y+1 is evaluated one step behind the walk.
template <int CONN, typename T>
__device__ bool sweep_detect(WarpSmem<T> &s, unsigned &t, unsigned qlimit, int lane) {
  const int k = lane + 1, x = k;
  bool chg = walk_line<1>(s, sidx(1, k), sidx(0, k));
  chg |= walk_line<-1>(s, sidx(TS, k), sidx(TS + 1, k));
  __syncwarp();
  chg |= walk_col<CONN, 1>(s, lane);
  __syncwarp();
  int v = s.J[sidx(x, TS + 1)];
  const bool edge = lane == 0 || lane == 31;
  const int side = lane == 0 ? 0 : TS + 1;
  int sv = edge ? s.J[sidx(side, TS + 1)] : INT_MIN;
  // window (n, c, p) = rows (y, y+1, y+2); start with c = row TS+1 (halo),
  // p = beyond: both +inf
  int m_c = INT_MAX, lr_c = INT_MAX, j_c = 0, m_p = INT_MAX, lr_p = INT_MAX;
  constexpr int C = 8;
#pragma unroll 1
  for (int k0 = 0; k0 < TS; k0 += C) {
    int j[C], mm[C];
    int sn[C];
#pragma unroll
    for (int c = 0; c < C; c++) {
      j[c] = s.J[sidx(x, TS - k0 - c)];
      mm[c] = (int)s.I[sidx(x, TS - k0 - c)];
      sn[c] = (CONN == 8 && edge) ? s.J[sidx(side, TS - k0 - c)] : INT_MIN;
    }
#pragma unroll
    for (int c = 0; c < C; c++) {
      const int y = TS - k0 - c;
      int in = v;
      if (CONN == 8) {  // {SW, S, SE} of the row below (K.142-190 backward)
        int l = __shfl_up_sync(FULL, v, 1), r = __shfl_down_sync(FULL, v, 1);
        if (lane == 0) l = sv;
        if (lane == 31) r = sv;
        in = max(v, max(l, r));
        sv = sn[c];
      }
      int nv = clampi(in, j[c], mm[c]);
      chg |= nv != j[c];
      s.J[sidx(x, y)] = nv;
      v = nv;
      int m_n = nv < mm[c] ? nv : INT_MAX;
      int lr_n = lr_of(m_n, lane);
      if (y + 1 <= TS)  // centre y+1 (rows y..y+2 final)
        t = push_ballot(s.ring, t, j_c > window_lo<CONN>(m_n, lr_n, m_c, lr_c, m_p, lr_p),
                        sidx(x, y + 1), qlimit);
      m_p = m_c;
      lr_p = lr_c;
      m_c = m_n;
      lr_c = lr_n;
      j_c = nv;
    }
  }
  // centre row 1: rows 0 (halo: +inf), 1, 2
  t = push_ballot(s.ring, t, j_c > window_lo<CONN>(INT_MAX, INT_MAX, m_c, lr_c, m_p, lr_p),
                  sidx(x, 1), qlimit);
  return __any_sync(FULL, chg);
}

// --- propagation to the tile's fixed point ---------------------------------------
//
// The warp drains its ring 32 items per step.  Items are interior cells, so
// all 8 (4) neighbours lie in the padded tile: no bounds checks.  Each lane
// loads its neighbours, then issues its predicated atomicMax offers back to
// back; a neighbour it raised is pushed.  __syncwarp orders one step's
// merges before the next step's reads.
template <int CONN, typename T>
__device__ void tile_fixpoint(WarpSmem<T> &s, unsigned qlimit, bool full, int sweeps,
                              unsigned halo_thresh, int lane, bool &changed,
                              unsigned long long &pushes, unsigned long long &overflows,
                              unsigned long long &seeds, unsigned long long *ph) {
  const bool l0 = lane == 0;
  unsigned h = 0, t = 0;
  bool rescan = true, pending = false, swept = false, offered = false;
  for (;;) {
    if (rescan) {
      long long d0 = pclock(l0);
      unsigned n = 0;
      if (!offered) {  // halo -> border offers, once per activation
        offered = true;
        unsigned raised = halo_offers<CONN>(s, lane);
        changed |= __any_sync(FULL, raised != 0);
        if (!full) {
          n = queue_halo_raised(s.ring, 0, raised, qlimit, lane);
          if (sweeps > 0 && n > halo_thresh) full = true;  // a wide front: sweep it in
        }
      }
      if (full && !swept && sweeps > 0) {
        swept = true;
        n = 0;
        for (int sp = 1; sp < sweeps; sp++) changed |= sweep_pass<CONN>(s, lane);
        changed |= sweep_detect<CONN>(s, n, qlimit, lane);
        if (kPhases && l0) ph[2] += clock64() - d0;
      } else if (full) {
        swept = true;
        n = detect_full<CONN>(s, 0, qlimit, lane);
        if (kPhases && l0) ph[3] += clock64() - d0;
      }
      __syncwarp();
      full = true;  // later rescans (overflow recovery) are always full
      rescan = false;
      pending = n > qlimit;
      if (pending) n = qlimit;
      if (l0) {
        seeds += n;
        if (pending) overflows++;
      }
      h = 0;
      t = n;
      if (n == 0) break;
    }
    // one step: up to 32 items
    const unsigned b = min(t - h, 32u);
    const bool act = (unsigned)lane < b;
    const int p = act ? s.ring[(h + lane) & (RQ - 1)] : sidx(1, 1);
    const int v = act ? s.J[p] : INT_MIN;
    int nv[Nbr<CONN>::N];
    unsigned cand = 0;
#pragma unroll
    for (int k = 0; k < Nbr<CONN>::N; k++) {
      int qq = p + noff<CONN>(k);
      int vq = s.J[qq], iq = (int)s.I[qq];
      nv[k] = min(v, iq);
      if (vq < v && vq < iq) cand |= 1u << k;
    }
    unsigned mask = 0;
#pragma unroll
    for (int k = 0; k < Nbr<CONN>::N; k++) {
      int old = smem_atomic_max_if(&s.J[p + noff<CONN>(k)], nv[k], (cand >> k) & 1u);
      if (old < nv[k]) mask |= 1u << k;  // predicated-off lanes return INT_MAX
    }
    changed |= __any_sync(FULL, mask != 0);
    // placement: exclusive prefix of the per-lane counts from bit-plane ballots
    const unsigned c = __popc(mask);
    const unsigned b0 = __ballot_sync(FULL, c & 1u), b1 = __ballot_sync(FULL, c & 2u);
    const unsigned b2 = __ballot_sync(FULL, c & 4u), b3 = __ballot_sync(FULL, c & 8u);
    const unsigned lt = lanemask_lt();
    const unsigned pre =
        __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt) + 8 * __popc(b3 & lt);
    const unsigned tot = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2) + 8 * __popc(b3);
    const unsigned hb = h + b;
    unsigned pos = t + pre;
    while (mask) {
      int k = __ffs(mask) - 1;
      mask &= mask - 1;
      if (pos - hb < qlimit) s.ring[pos & (RQ - 1)] = (uint16_t)(p + noff<CONN>(k));
      pos++;
    }
    if (l0) pushes += tot;
    h = hb;
    t += tot;
    __syncwarp();
    if (t - h > qlimit) {  // dropped pushes: discard and rescan the tile
      if (l0) overflows++;
      rescan = true;
      continue;
    }
    if (h == t) {
      if (!pending) break;
      rescan = true;
    }
  }
}

// --- the persistent kernel ------------------------------------------------------

template <typename T, int CONN>
__global__ void __launch_bounds__(kCtaThreads, kCtaMinBlocks)
    tile_engine_kernel(EngineArgs a, unsigned long long *counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpSmem<T> &s = reinterpret_cast<WarpSmem<T> *>(smem_raw)[warp];
  const bool l0 = lane == 0;

  unsigned long long n_tiles = 0, n_reruns = 0, n_push = 0, n_over = 0, n_seeds = 0;
  unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};

  int next_tile = -1;  // a claimed neighbour this warp continues with
  for (;;) {
    long long c_pop = pclock(l0);
    int t = -1;
    unsigned first = 0;
    if (l0) {
      t = next_tile >= 0 ? next_tile : ring_pop(a.q);
      if (t >= 0) {
        unsigned old = state_take(&a.q.state[t]);
        first = old & ST_V;
      }
    }
    t = __shfl_sync(FULL, t, 0);
    next_tile = -1;
    if (t < 0) break;
    bool full = __shfl_sync(FULL, first, 0) != 0;
    int tx, ty;
    tile_xy(a, (unsigned)t, tx, ty);
    const int x0 = tx * TS, y0 = ty * TS;
    const int limx = min(TS, a.W - x0), limy = min(TS, a.H - y0);
    long long c_load = pclock(l0);
    if (kPhases && l0) ph[0] += c_load - c_pop;

    load_tile<T>(a, s, x0, y0, lane);
    __syncwarp();
    for (int r = lane; r < 4 * TS; r += 32) {
      int lx, ly;
      ring_cell(r, lx, ly);
      s.ring0[r] = s.J[sidx(lx, ly)];
    }
    __syncwarp();
    if (kPhases && l0) ph[1] += clock64() - c_load;
    bool rerun = false;
    for (;;) {  // re-run while neighbours request it
      n_tiles += l0;
      n_reruns += l0 && rerun;
      long long c_fix = pclock(l0);
      unsigned long long sd0 = ph[2] + ph[3];
      bool changed = false;
      tile_fixpoint<CONN>(s, a.qlimit, full, a.sweeps, a.halo_thresh, lane, changed, n_push,
                          n_over, n_seeds, ph);
      full = false;
      changed = __any_sync(FULL, changed);
      long long c_st = pclock(l0);
      if (kPhases && l0) ph[4] += (c_st - c_fix) - (ph[2] + ph[3] - sd0);
      if (changed) {
        __syncwarp();
        store_tile<T>(a, s, x0, y0, limx, limy, lane);
        if (a.dirty && l0) a.dirty[ty] = 1;
        // Which neighbour tiles can the changed border still raise?  Per
        // side, lane = position along it: cv = the border cell's value if it
        // changed since last published (else -inf); a halo cell needs its
        // tile re-run iff it can still be raised (J < real I) by the max cv
        // of its interior neighbours (lanes l-1..l+1 for 8-conn).  Cells
        // outside the image hold J = I = min(T): never "need".
        const int k = lane + 1;
        auto cv_of = [&](int bx, int by) -> int {
          int vb = s.J[sidx(bx, by)];
          return vb != s.ring0[ring_index(bx, by)] ? vb : INT_MIN;
        };
        auto nb3 = [&](int c) -> int {
          if (CONN == 4) return c;
          int u = __shfl_up_sync(FULL, c, 1), d = __shfl_down_sync(FULL, c, 1);
          if (lane == 0) u = INT_MIN;
          if (lane == 31) d = INT_MIN;
          return max(c, max(u, d));
        };
        auto need_h = [&](int hx, int hy, int hidx, int c) -> bool {
          int vh = s.J[sidx(hx, hy)];
          return vh < (int)s.Ih[hidx] && vh < c;
        };
        const int ct = cv_of(k, 1), cb = cv_of(k, TS), cl = cv_of(1, k), cr = cv_of(TS, k);
        const int nt = nb3(ct), nbm = nb3(cb), nl = nb3(cl), nr = nb3(cr);
        unsigned dirs = 0;
        if (__any_sync(FULL, need_h(k, 0, k, nt))) dirs |= 1u << 1;                     // N
        if (__any_sync(FULL, need_h(k, TS + 1, PW + k, nbm))) dirs |= 1u << 7;          // S
        if (__any_sync(FULL, need_h(0, k, 2 * PW + k - 1, nl))) dirs |= 1u << 3;        // W
        if (__any_sync(FULL, need_h(TS + 1, k, 2 * PW + TS + k - 1, nr))) dirs |= 1u << 5;  // E
        if (CONN == 8) {  // corners touch one interior cell each
          bool c0 = lane == 0 && need_h(0, 0, 0, ct);
          bool c2 = lane == 31 && need_h(TS + 1, 0, TS + 1, ct);
          bool c6 = lane == 0 && need_h(0, TS + 1, PW, cb);
          bool c8 = lane == 31 && need_h(TS + 1, TS + 1, PW + TS + 1, cb);
          if (__any_sync(FULL, c0)) dirs |= 1u << 0;
          if (__any_sync(FULL, c2)) dirs |= 1u << 2;
          if (__any_sync(FULL, c6)) dirs |= 1u << 6;
          if (__any_sync(FULL, c8)) dirs |= 1u << 8;
        }
        fence_acq_rel();  // publish the interior before any neighbour is (re)queued
        __syncwarp();
        // one lane per direction claims the neighbour; the warp keeps one
        // claimed idle neighbour as its own continuation (no queue round
        // trip on a wavefront's critical path) and pushes the rest
        bool own = false;
        unsigned ntile = 0;
        if (lane < 9 && ((dirs >> lane) & 1u)) {
          int ntxi = tx + (lane % 3) - 1, ntyi = ty + (lane / 3) - 1;
          if (ntxi >= 0 && ntxi < a.ntx && ntyi >= 0 && ntyi < a.nty) {
            ntile = (unsigned)(ntyi * a.ntx + ntxi);
            own = activate_claim_nopend(a.q, ntile);
          }
        }
        unsigned ownmask = __ballot_sync(FULL, own);
        int keep = (ownmask && next_tile < 0) ? __ffs(ownmask) - 1 : -1;
        // the kept continuation inherits this tile's pending count (no +1 here,
        // no -1 at this tile's finish); a pushed tile counts before its push
        if (own && lane != keep) {
          atomicAdd(a.q.pending, 1u);
          ring_push(a.q, ntile);
        }
        if (keep >= 0) next_tile = __shfl_sync(FULL, (int)ntile, keep);
        for (int r = lane; r < 4 * TS; r += 32) {
          int lx, ly;
          ring_cell(r, lx, ly);
          s.ring0[r] = s.J[sidx(lx, ly)];
        }
      }
      // finish: R -> idle, or re-run if a neighbour requested it meanwhile
      int done = 0;
      if (l0) {
        unsigned old = atomicCAS(&a.q.state[t], ST_R, 0u);
        if (old == ST_R) {
          // no fence: pending is only ever changed by RMWs, whose per-location
          // order already puts our activations' increments before this
          if (next_tile < 0) atomicSub(a.q.pending, 1u);  // (else passed on, above)
          done = 1;
        } else {
          state_take(&a.q.state[t]);  // consume the request (acquire)
        }
      }
      done = __shfl_sync(FULL, done, 0);
      if (kPhases && l0) ph[5] += clock64() - c_st;
      if (done) break;
      __syncwarp();
      load_halo<T>(a, s, x0, y0, lane);  // the interior is ours and current
      __syncwarp();
      rerun = true;
    }
  }
  if (l0) {
    atomicAdd(&counters[CNT_TILES], n_tiles);
    atomicAdd(&counters[CNT_RERUNS], n_reruns);
    atomicAdd(&counters[CNT_PUSHES], n_push);
    atomicAdd(&counters[CNT_OVERFLOW], n_over);
    atomicAdd(&counters[CNT_SEEDS], n_seeds);
    if (kPhases)
      for (int i = 0; i < 6; i++) atomicAdd(&counters[CNT_PH_POP + i], ph[i]);
  }
}

// --- register engine (u8) -------------------------------------------------------
//
// One warp holds one 32 x 32 u8 tile in registers: lane = row, 8 words of 4
// packed pixels for J and for I.  The tile's fixed point (given its halo) is
// reached by Jacobi steps on the packed bytes,
//     J <- max(J, min(I, max over N(p) of J)),
// with the 3 x 3 (8-conn) / cross (4-conn) maximum built from byte-SIMD max
// (vmaxu4), funnel shifts for the row neighbours and shfl for the rows above
// and below.  Each step is a valid set of raise operations of the reference
// rule (recon.py:92-101, K.220-270), so the unique fixed point is unchanged;
// on random marker/mask pairs a tile converges in ~8 steps of ~100
// instructions, with no shared memory at all.  The queue protocol (pop,
// activation of the neighbours a changed border can still raise, finish,
// re-run) is the same as the shared-memory engine's.
struct RegHalo {
  unsigned row[8];           // lane 0: the row above the tile; lane 31: the row below
  unsigned l, r, lI, rI;     // the cells left / right of my row (J, I)
  unsigned cl, cr, clI, crI; // lane 0: corners above; lane 31: corners below
};

__device__ __forceinline__ void reg_load_row(const uint8_t *base, int W, int x0, int gy, int H,
                                             bool vec, bool cg, unsigned *w) {
  if (gy < 0 || gy >= H) {
#pragma unroll
    for (int k = 0; k < 8; k++) w[k] = 0;
    return;
  }
  const uint8_t *p = base + (size_t)gy * W + x0;
  if (vec && x0 + TS <= W) {
    const uint4 a = cg ? __ldcg(reinterpret_cast<const uint4 *>(p)) : __ldg(reinterpret_cast<const uint4 *>(p));
    const uint4 b = cg ? __ldcg(reinterpret_cast<const uint4 *>(p) + 1)
                       : __ldg(reinterpret_cast<const uint4 *>(p) + 1);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    return;
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
    unsigned v = 0;
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const int x = x0 + 4 * k + b;
      if (x < W) v |= (unsigned)(cg ? ld_cg(p + 4 * k + b) : __ldg(p + 4 * k + b)) << (8 * b);
    }
    w[k] = v;
  }
}

__device__ __forceinline__ unsigned reg_cell(const uint8_t *base, int W, int H, int gx, int gy,
                                             bool cg) {
  if (gx < 0 || gx >= W || gy < 0 || gy >= H) return 0u;
  const uint8_t *p = base + (size_t)gy * W + gx;
  return cg ? (unsigned)ld_cg(p) : (unsigned)__ldg(p);
}

__device__ __forceinline__ void reg_load_halo(const EngineArgs &a, int x0, int y0, int lane,
                                              RegHalo &h) {
  const uint8_t *J = (const uint8_t *)a.J, *I = (const uint8_t *)a.I;
  const int gy = y0 + lane;
  const int hy = lane == 0 ? y0 - 1 : (lane == 31 ? y0 + TS : -1);
  h.l = reg_cell(J, a.W, a.H, x0 - 1, gy, true);
  h.r = reg_cell(J, a.W, a.H, x0 + TS, gy, true);
  h.lI = reg_cell(I, a.W, a.H, x0 - 1, gy, false);
  h.rI = reg_cell(I, a.W, a.H, x0 + TS, gy, false);
  h.cl = reg_cell(J, a.W, a.H, x0 - 1, hy, true);
  h.cr = reg_cell(J, a.W, a.H, x0 + TS, hy, true);
  h.clI = reg_cell(I, a.W, a.H, x0 - 1, hy, false);
  h.crI = reg_cell(I, a.W, a.H, x0 + TS, hy, false);
  reg_load_row(J, a.W, x0, hy, a.H, a.vec, true, h.row);
}

// Per-warp shared memory of the register engine (keeps registers for the
// Jacobi state): lanes 0 / 31 park the halo row's I and their row as last
// published (the activation test's inputs).
struct RegWarpSmem {
  unsigned rowI[2][8];
  unsigned ob[2][8];
};

// 16-bit lane SIMD (VIMNMX.U16x2: one instruction for two pixels)
__device__ __forceinline__ unsigned max2(unsigned a, unsigned b) {
  unsigned r;
  asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ unsigned min2(unsigned a, unsigned b) {
  unsigned r;
  asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// One Jacobi step J <- min(I, 3x3 / cross max of J) on the even / odd split
// (TRACK: accumulate the changed bits into ch).
template <int CONN, bool TRACK>
__device__ __forceinline__ void reg_step(unsigned (&e)[8], unsigned (&o)[8], const unsigned (&ie)[8],
                                         const unsigned (&io)[8], unsigned &ch) {
  unsigned ve[8], vo[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    // lanes 0 / 31 see themselves: harmless under max
    const unsigned ue = __shfl_up_sync(FULL, e[k], 1), de = __shfl_down_sync(FULL, e[k], 1);
    const unsigned uo = __shfl_up_sync(FULL, o[k], 1), dn = __shfl_down_sync(FULL, o[k], 1);
    ve[k] = CONN == 8 ? max2(e[k], max2(ue, de)) : max2(ue, de);
    vo[k] = CONN == 8 ? max2(o[k], max2(uo, dn)) : max2(uo, dn);
  }
  if (CONN == 8) {
    // 3x3 max = horizontal max of the vertical maxima
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const unsigned lE = __funnelshift_l(k ? vo[k - 1] : 0u, vo[k], 16);
      const unsigned rO = __funnelshift_r(ve[k], k < 7 ? ve[k + 1] : 0u, 16);
      const unsigned dE = max2(ve[k], max2(lE, vo[k]));
      const unsigned dO = max2(vo[k], max2(ve[k], rO));
      const unsigned nE = min2(ie[k], dE), nO = min2(io[k], dO);  // D >= J (centre included)
      if (TRACK) ch |= (nE ^ e[k]) | (nO ^ o[k]);
      e[k] = nE;
      o[k] = nO;
    }
  } else {
    unsigned prevo = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const unsigned lE = __funnelshift_l(prevo, o[k], 16);
      const unsigned rO = __funnelshift_r(e[k], k < 7 ? e[k + 1] : 0u, 16);
      const unsigned dE = max2(max2(ve[k], e[k]), max2(lE, o[k]));
      const unsigned dO = max2(max2(vo[k], o[k]), max2(e[k], rO));
      prevo = o[k];  // the old odd word, for word k + 1
      const unsigned nE = min2(ie[k], dE), nO = min2(io[k], dO);
      if (TRACK) ch |= (nE ^ e[k]) | (nO ^ o[k]);
      e[k] = nE;
      o[k] = nO;
    }
  }
}

// Jacobi steps to the tile's fixed point; returns the number of steps.
// The row's 32 pixels are split into even / odd pixels, two per word as
// 16-bit lanes: e[k] = (p[4k], p[4k+2]), o[k] = (p[4k+1], p[4k+3]).  Then a
// pixel's left / right neighbours are the other parity's word (same word or
// one funnel shift away) and every max/min is one VIMNMX.U16x2.
template <int CONN>
__device__ __forceinline__ int reg_fixpoint(unsigned *j, const unsigned *m, const RegHalo &h,
                                            int lane, bool &changed) {
  constexpr unsigned LO8 = 0x00FF00FFu;
  unsigned e[8], o[8], ie[8], io[8];
#pragma unroll
  for (int k = 0; k < 8; k++) {
    e[k] = j[k] & LO8;
    o[k] = (j[k] >> 8) & LO8;
    ie[k] = m[k] & LO8;
    io[k] = (m[k] >> 8) & LO8;
  }
  // The halo is constant during the iteration: its whole effect on the
  // tile's fixed point is the lower bound min(I, halo dilation) on the edge
  // pixels.  Apply it once; the steps below then see a closed tile.
  unsigned hlv = h.l, hrv = h.r;
  if (CONN == 8) {
    unsigned lu = __shfl_up_sync(FULL, h.l, 1), ld = __shfl_down_sync(FULL, h.l, 1);
    unsigned ru = __shfl_up_sync(FULL, h.r, 1), rd = __shfl_down_sync(FULL, h.r, 1);
    if (lane == 0) { lu = h.cl; ru = h.cr; }
    if (lane == 31) { ld = h.cl; rd = h.cr; }
    hlv = max(h.l, max(lu, ld));
    hrv = max(h.r, max(ru, rd));
  }
  e[0] = max2(e[0], min2(ie[0], hlv));
  o[7] = max2(o[7], min2(io[7], hrv << 16));
  if (lane == 0 || lane == 31) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
      const unsigned he = h.row[k] & LO8, ho = (h.row[k] >> 8) & LO8;
      unsigned dE = he, dO = ho;
      if (CONN == 8) {
        const unsigned hoP = k ? (h.row[k - 1] >> 8) & LO8 : (h.cl << 16);
        const unsigned heN = k < 7 ? h.row[k + 1] & LO8 : h.cr;
        dE = max2(he, max2(__funnelshift_l(hoP, ho, 16), ho));
        dO = max2(ho, max2(he, __funnelshift_r(he, heN, 16)));
      }
      e[k] = max2(e[k], min2(ie[k], dE));
      o[k] = max2(o[k], min2(io[k], dO));
    }
  }
  // Jacobi steps in pairs, the change test on the second step of a pair
  // only: a pair whose second step changes nothing ends at a fixed point
  // (costs at most one extra step; saves the test and the loop-carried
  // register copies of every other step)
  int steps = 0;
  for (;;) {
    unsigned ch = 0;
    reg_step<CONN, false>(e, o, ie, io, ch);
    reg_step<CONN, true>(e, o, ie, io, ch);
    steps += 2;
    if (!__any_sync(FULL, ch != 0)) break;
  }
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const unsigned nj = e[k] | (o[k] << 8);
    changed |= nj != j[k];
    j[k] = nj;
  }
  return steps;
}

// --- TMA staging of a tile (register engine, u8) --------------------------------
//
// One elected lane loads the tile plus its one-pixel halo of J and of I as
// two 64 x 34-byte boxes with cp.async.bulk.tensor (out-of-image cells come
// back as 0, the u8 sentinel), completion on a per-warp mbarrier; the lanes
// then read their rows from shared memory.  A box's start column must be
// 16-byte aligned, so box column c is image column x0 - 16 + c (the tile at
// c = 16..47, the halo at 15 and 48); row r is image row y0 - 1 + r.
constexpr int kBoxW = 64, kBoxH = TS + 2, kBoxBytes = kBoxW * kBoxH, kBoxX = 16;

struct alignas(128) TmaWarpSmem {
  uint8_t J[kBoxBytes];
  uint8_t pad0[(128 - kBoxBytes % 128) % 128];
  uint8_t I[kBoxBytes];
  uint8_t pad1[(128 - kBoxBytes % 128) % 128];
  unsigned long long bar;
  alignas(16) uint8_t nrow[2 * TS];  // the new top / bottom row (need test)
};

__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_box(const CUtensorMap *map, void *dst, unsigned long long *bar,
                                             int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// lane 0: issue the J (and, for a fresh tile, I) boxes of tile (x0, y0);
// every lane then waits for them.  `phase` toggles per use.
__device__ __forceinline__ void tma_stage(const CUtensorMap *mJ, const CUtensorMap *mI, TmaWarpSmem &t,
                                          int x0, int y0, bool withI, unsigned &phase, int lane) {
  __syncwarp();  // the previous boxes have been read (WAR on the staging buffers)
  if (lane == 0) {
    // other SMs' stores, acquired through the tile state, must be visible
    // to the async proxy that performs the box reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(&t.bar, withI ? 2u * kBoxBytes : (unsigned)kBoxBytes);
    tma_load_box(mJ, t.J, &t.bar, x0 - kBoxX, y0 - 1);
    if (withI) tma_load_box(mI, t.I, &t.bar, x0 - kBoxX, y0 - 1);
  }
  mbar_wait(&t.bar, phase);
  phase ^= 1u;
}

// rows from the staged boxes: my row's words + halo bytes; lanes 0 / 31 also
// take the halo row above / below and its corners
__device__ __forceinline__ void tma_row(const uint8_t *box, int r, unsigned *w) {
  const uint4 *p = reinterpret_cast<const uint4 *>(box + r * kBoxW + kBoxX);
  const uint4 a = p[0], b = p[1];
  w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
  w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

// The need test of the rows above / below (which neighbour tile can my
// changed border still raise?), one lane per column: lanes 0 / 31 park the
// new top / bottom row in shared memory; column x then tests the halo cell
// above / below it against the changed border cells at x-1..x+1 (x for
// 4-conn): J(q) < I(q) and J(q) < the changed value.  The border as loaded
// and the halo rows are in this tile's boxes.  Returns bit 0 = N, bit 1 = S.
template <int CONN>
__device__ __forceinline__ unsigned tma_need_rows(TmaWarpSmem &t, const unsigned *j, int lane) {
  if (lane == 0 || lane == 31) {
    uint4 *d = reinterpret_cast<uint4 *>(t.nrow + (lane == 31 ? TS : 0));
    d[0] = make_uint4(j[0], j[1], j[2], j[3]);
    d[1] = make_uint4(j[4], j[5], j[6], j[7]);
  }
  __syncwarp();
  const int c = kBoxX + lane;
  const unsigned nt = t.nrow[lane], nb = t.nrow[TS + lane];
  const unsigned ct = nt != t.J[kBoxW + c] ? nt : 0u;
  const unsigned cb = nb != t.J[TS * kBoxW + c] ? nb : 0u;
  unsigned dt = ct, db = cb;
  if (CONN == 8) {  // lanes 0 / 31 see themselves: harmless under max
    dt = max(ct, max(__shfl_up_sync(FULL, ct, 1), __shfl_down_sync(FULL, ct, 1)));
    db = max(cb, max(__shfl_up_sync(FULL, cb, 1), __shfl_down_sync(FULL, cb, 1)));
  }
  const unsigned hjt = t.J[c], hit = t.I[c];
  const unsigned hjb = t.J[(TS + 1) * kBoxW + c], hib = t.I[(TS + 1) * kBoxW + c];
  const bool n = hjt < hit && hjt < dt, sth = hjb < hib && hjb < db;
  __syncwarp();  // nrow is rewritten by the next test
  return (__any_sync(FULL, n) ? 1u : 0u) | (__any_sync(FULL, sth) ? 2u : 0u);
}

// the two box descriptors travel as a __grid_constant__ kernel parameter
// (no upload, no tensormap proxy fence)
struct alignas(64) BoxMaps {
  CUtensorMap m[2];
};

__device__ __forceinline__ void tile_queue_init(const TileQueue &q, int ntx, int nty,
                                                unsigned long long *counters, int keep);

// fused init with a separate marker: the grid copies it into J before the
// grid-wide sync (16-byte vectors, 4 in flight per thread; the marker is read
// once, so streaming loads; J stays in L2 for the first box reads)
__device__ __forceinline__ void copy_marker(const EngineArgs &a, const void *M) {
  const size_t n = (size_t)a.W * a.H;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  const uint8_t *src = static_cast<const uint8_t *>(M);
  uint8_t *dst = static_cast<uint8_t *>(a.J);
  size_t done = 0;
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
    const size_t nv = n / 16;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    size_t i = tid;
    for (; i + 3 * nt < nv; i += 4 * nt) {
      const uint4 v0 = __ldcs(s4 + i), v1 = __ldcs(s4 + i + nt), v2 = __ldcs(s4 + i + 2 * nt),
                  v3 = __ldcs(s4 + i + 3 * nt);
      d4[i] = v0;
      d4[i + nt] = v1;
      d4[i + 2 * nt] = v2;
      d4[i + 3 * nt] = v3;
    }
    for (; i < nv; i += nt) d4[i] = __ldcs(s4 + i);
    done = nv * 16;
  }
  for (size_t i = done + tid; i < n; i += nt) dst[i] = src[i];
}

// fused_init: the launch is cooperative and the kernel builds the initial
// queue itself (all tiles, INIT_FULL) before one grid-wide sync, instead of
// a separate init kernel
template <int CONN>
__global__ void __launch_bounds__(kCtaThreads, kRegCtaMinBlocks)
    tile_engine_reg_kernel(EngineArgs a, unsigned long long *counters,
                           const __grid_constant__ BoxMaps maps, int use_tma, int fused_init,
                           const void *M) {
  if (fused_init) {
    if (M) copy_marker(a, M);
    tile_queue_init(a.q, a.ntx, a.nty, counters, 0);
    cooperative_groups::this_grid().sync();
  }
  __shared__ RegWarpSmem wsm[kWarpsPerCta];
  __shared__ TmaWarpSmem tsm[kWarpsPerCta];
  TmaWarpSmem &ts = tsm[threadIdx.x >> 5];
  const CUtensorMap *tmJ = &maps.m[0], *tmI = &maps.m[1];
  unsigned tphase = 0;
  if (use_tma && (threadIdx.x & 31) == 0) {
    mbar_init(&ts.bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int lane = threadIdx.x & 31;
  const bool l0 = lane == 0;
  const bool edge = lane == 0 || lane == 31;
  const int sel = lane == 31;
  RegWarpSmem &ws = wsm[threadIdx.x >> 5];
  unsigned long long n_tiles = 0, n_reruns = 0, n_steps = 0, n_idle = 0;
  unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
  int next_tile = -1;
  for (;;) {
    long long c_pop = pclock(l0);
    ATraceRec rec;
    if (kATrace) {
      rec.t_pop = gtime32();
      rec.depth = kATrace && l0 ? *(volatile unsigned *)a.q.tail - *(volatile unsigned *)a.q.head : 0u;
    }
    int t = -1;
    unsigned took = 0;  // (diagnostics) the state word the take consumed
    if (l0) {
      t = next_tile >= 0 ? next_tile : ring_pop(a.q, &n_idle);
      if (t >= 0) took = state_take(&a.q.state[t]);
    }
    (void)took;
    t = __shfl_sync(FULL, t, 0);
    if (kATrace) {
      rec.t_take = gtime32();
      rec.tile = (unsigned)t | (next_tile >= 0 ? 0x80000000u : 0u);  // top bit: continuation
      rec.sm_steps = smid() << 16;
    }
    next_tile = -1;
    if (t < 0) break;
    int tx, ty;
    tile_xy(a, (unsigned)t, tx, ty);
    const int x0 = tx * TS, y0 = ty * TS;
    long long c_load = pclock(l0);
    if (kPhases && l0) ph[0] += c_load - c_pop;

    unsigned j[8], m[8];
    RegHalo h;
    if (use_tma) {
      tma_stage(tmJ, tmI, ts, x0, y0, true, tphase, lane);
      const int hr = lane == 0 ? 0 : TS + 1;  // halo row (lanes 0 / 31)
      tma_row(ts.J, lane + 1, j);
      tma_row(ts.I, lane + 1, m);
      tma_row(ts.J, hr, h.row);
      h.l = ts.J[(lane + 1) * kBoxW + kBoxX - 1];
      h.r = ts.J[(lane + 1) * kBoxW + kBoxX + TS];
      h.lI = ts.I[(lane + 1) * kBoxW + kBoxX - 1];
      h.rI = ts.I[(lane + 1) * kBoxW + kBoxX + TS];
      h.cl = ts.J[hr * kBoxW + kBoxX - 1];
      h.cr = ts.J[hr * kBoxW + kBoxX + TS];
      h.clI = ts.I[hr * kBoxW + kBoxX - 1];
      h.crI = ts.I[hr * kBoxW + kBoxX + TS];
      // (the need test reads the border as loaded and the halo rows' mask
      // from the boxes: tma_need_rows)
    } else {
      reg_load_row((const uint8_t *)a.J, a.W, x0, y0 + lane, a.H, a.vec, true, j);
      reg_load_row((const uint8_t *)a.I, a.W, x0, y0 + lane, a.H, a.vec, false, m);
      reg_load_halo(a, x0, y0, lane, h);
      // the border as last published (lanes 0 / 31: whole rows; every lane: its ends)
      if (edge) {
        const int hy = lane == 0 ? y0 - 1 : y0 + TS;
        unsigned hI[8];
        reg_load_row((const uint8_t *)a.I, a.W, x0, hy, a.H, a.vec, false, hI);
#pragma unroll
        for (int k = 0; k < 8; k++) {
          ws.rowI[sel][k] = hI[k];
          ws.ob[sel][k] = j[k];
        }
      }
    }
    unsigned obl = j[0] & 0xffu, obr = j[7] >> 24;
    __syncwarp();
    if (kPhases && l0) ph[1] += clock64() - c_load;
    if (kATrace) rec.t_load = gtime32();
    bool rerun = false;
    for (;;) {  // re-run while neighbours request it
      n_tiles += l0;
      n_reruns += l0 && rerun;
      long long c_fix = pclock(l0);
      bool changed = false;
      const int steps = reg_fixpoint<CONN>(j, m, h, lane, changed);
      if (l0) n_steps += steps;
#ifdef IWPP_COUNT_NOCHANGE
      // diagnostics: [8] first visits, [9] later activations, [10] re-runs
      // that changed nothing; [11] later activations that changed something
      {
        const bool ch = __any_sync(FULL, changed);
        if (l0 && !rerun && (took & ST_V)) ph[0] += 1;
        if (l0 && !rerun && !(took & ST_V)) ph[1] += 1;
        if (l0 && rerun && !ch) ph[2] += 1;
        if (l0 && !rerun && !(took & ST_V) && ch) ph[3] += 1;
      }
#endif
      if (kATrace) {
        rec.t_fix = gtime32();
        rec.sm_steps += steps;
      }
      changed = __any_sync(FULL, changed);
      long long c_st = pclock(l0);
      if (kPhases && l0) ph[2] += c_st - c_fix;
      if (changed) {
        // store my row
        const int gy = y0 + lane;
        if (gy < a.H) {
          uint8_t *p = (uint8_t *)a.J + (size_t)gy * a.W + x0;
          if (a.vec && x0 + TS <= a.W) {
            reinterpret_cast<uint4 *>(p)[0] = make_uint4(j[0], j[1], j[2], j[3]);
            reinterpret_cast<uint4 *>(p)[1] = make_uint4(j[4], j[5], j[6], j[7]);
          } else {
            // (static indices: a dynamic j[] index puts the tile row in local memory)
#pragma unroll
            for (int k = 0; k < 8; k++)
#pragma unroll
              for (int b = 0; b < 4; b++)
                if (x0 + 4 * k + b < a.W) p[4 * k + b] = (uint8_t)(j[k] >> (8 * b));
          }
        }
        if (a.dirty && l0) a.dirty[ty] = 1;
        // which neighbours can the changed border still raise (J < I, J < the
        // max of the adjacent changed border cells)?
        unsigned need_row = 0;  // lanes 0 / 31: the row above / below
        unsigned need_ns = 0;   // (TMA staging) bit 0 / 1: N / S
        if (use_tma) {
          need_ns = tma_need_rows<CONN>(ts, j, lane);
        } else if (edge) {
          unsigned cv[8];
#pragma unroll
          for (int k = 0; k < 8; k++) cv[k] = j[k] & __vcmpne4(j[k], ws.ob[sel][k]);
#pragma unroll
          for (int k = 0; k < 8; k++) {
            unsigned D = cv[k];
            if (CONN == 8) {
              const unsigned L = __funnelshift_l(k ? cv[k - 1] : 0u, cv[k], 8);
              const unsigned R = __funnelshift_r(cv[k], k < 7 ? cv[k + 1] : 0u, 8);
              D = __vmaxu4(D, __vmaxu4(L, R));
            }
            need_row |= __vcmpltu4(h.row[k], ws.rowI[sel][k]) & __vcmpltu4(h.row[k], D);
          }
        }
        // changed row ends (or 0)
        const unsigned jl = j[0] & 0xffu, jr = j[7] >> 24;
        const unsigned cl = jl != obl ? jl : 0u, cr = jr != obr ? jr : 0u;
        unsigned dl = cl, dr = cr;
        if (CONN == 8) {
          unsigned lu = __shfl_up_sync(FULL, cl, 1), ld = __shfl_down_sync(FULL, cl, 1);
          unsigned ru = __shfl_up_sync(FULL, cr, 1), rd = __shfl_down_sync(FULL, cr, 1);
          if (lane == 0) lu = ru = 0;
          if (lane == 31) ld = rd = 0;
          dl = max(cl, max(lu, ld));
          dr = max(cr, max(ru, rd));
        }
        unsigned dirs = ((need_ns & 1u) << 1) | ((need_ns & 2u) << 6);
        if (!use_tma) {
          if (__any_sync(FULL, l0 && need_row)) dirs |= 1u << 1;             // N
          if (__any_sync(FULL, lane == 31 && need_row)) dirs |= 1u << 7;     // S
        }
        if (__any_sync(FULL, h.l < h.lI && h.l < dl)) dirs |= 1u << 3;    // W
        if (__any_sync(FULL, h.r < h.rI && h.r < dr)) dirs |= 1u << 5;    // E
        if (CONN == 8) {  // corners: one interior cell each
          const bool cwl = h.cl < h.clI && h.cl < cl, cwr = h.cr < h.crI && h.cr < cr;
          if (__any_sync(FULL, l0 && cwl)) dirs |= 1u << 0;
          if (__any_sync(FULL, l0 && cwr)) dirs |= 1u << 2;
          if (__any_sync(FULL, lane == 31 && cwl)) dirs |= 1u << 6;
          if (__any_sync(FULL, lane == 31 && cwr)) dirs |= 1u << 8;
        }
        if (edge && !use_tma)
#pragma unroll
          for (int k = 0; k < 8; k++) ws.ob[sel][k] = j[k];
        obl = jl;
        obr = jr;
        // publish the tile before any neighbour is (re)queued, and before
        // this tile's finish: the finish CAS is what lets a later activation
        // pop the tile again, and its next owner must load these values (a
        // stale interior could be recomputed lower and overwrite them)
        fence_acq_rel();
        __syncwarp();
        bool own = false;
        unsigned ntile = 0;
        if (lane < 9 && ((dirs >> lane) & 1u)) {
          int ntxi = tx + (lane % 3) - 1, ntyi = ty + (lane / 3) - 1;
          if (ntxi >= 0 && ntxi < a.ntx && ntyi >= 0 && ntyi < a.nty) {
            ntile = (unsigned)(ntyi * a.ntx + ntxi);
            own = activate_claim_nopend(a.q, ntile);
          }
        }
        unsigned ownmask = __ballot_sync(FULL, own);
        int keep = (ownmask && next_tile < 0) ? __ffs(ownmask) - 1 : -1;
        // the kept continuation inherits this tile's pending count (no +1 here,
        // no -1 at this tile's finish); a pushed tile counts before its push
        if (own && lane != keep) {
          atomicAdd(a.q.pending, 1u);
          ring_push(a.q, ntile);
        }
        if (keep >= 0) next_tile = __shfl_sync(FULL, (int)ntile, keep);
      }
      int done = 0;
      if (l0) {
        unsigned old = atomicCAS(&a.q.state[t], ST_R, 0u);
        if (old == ST_R) {
          // no fence: pending is only ever changed by RMWs, whose per-location
          // order already puts our activations' increments before this
          if (next_tile < 0) atomicSub(a.q.pending, 1u);  // (else passed on, above)
          done = 1;
        } else {
          state_take(&a.q.state[t]);  // consume the request (acquire)
        }
      }
      done = __shfl_sync(FULL, done, 0);
      if (kPhases && l0) ph[5] += clock64() - c_st;
#ifdef IWPP_ATRACE
      if (l0 && done) {
        rec.t_end = gtime32();
        const unsigned i = atomicAdd(&g_atrace_n, 1u);
        if (i < g_atrace_cap) g_atrace[i] = rec;
      }
#endif
      if (done) break;
      if (use_tma) {  // the interior is ours and current: refresh the J halo only
        tma_stage(tmJ, tmI, ts, x0, y0, false, tphase, lane);
        const int hr = lane == 0 ? 0 : TS + 1;
        tma_row(ts.J, hr, h.row);
        h.l = ts.J[(lane + 1) * kBoxW + kBoxX - 1];
        h.r = ts.J[(lane + 1) * kBoxW + kBoxX + TS];
        h.cl = ts.J[hr * kBoxW + kBoxX - 1];
        h.cr = ts.J[hr * kBoxW + kBoxX + TS];
      } else {
        reg_load_halo(a, x0, y0, lane, h);  // the interior is ours and current
      }
      rerun = true;
    }
  }
  if (l0) {
    atomicAdd(&counters[CNT_TILES], n_tiles);
    atomicAdd(&counters[CNT_RERUNS], n_reruns);
    atomicAdd(&counters[CNT_STEPS], n_steps);
    atomicAdd(&counters[CNT_IDLE_POLLS], n_idle);
#ifdef IWPP_COUNT_NOCHANGE
    for (int i = 0; i < 4; i++) atomicAdd(&counters[CNT_PH_POP + i], ph[i]);
#endif
    if (kPhases)
      for (int i = 0; i < 6; i++) atomicAdd(&counters[CNT_PH_POP + i], ph[i]);
  }
}


// --- level-synchronous tile rounds (register engine, u8) ------------------------
//
// The queue engine above pays a chain of L2 round trips per tile activation
// (ticket, slot, acquire exchange, box load, publish fence, claims, finish
// CAS).  This engine runs the same per-tile fixed point in rounds instead:
//   round 0      every tile once, from the marker (2 x 2 colour order, so
//                the tiles running at the same time are not neighbours);
//   round r > 0  exactly the tiles a neighbour flagged in round r - 1 (its
//                changed border can still raise one of their cells: the same
//                need test as the queue engine's activation);
// with one grid barrier per round and no per-tile protocol (no state word,
// no publish fence, no finish CAS).  Tiles of one round run concurrently
// and may read a neighbour's border before or after that neighbour writes
// it; values only grow between the marker and the result, and a neighbour
// that changes its border after we read it flags us for the next round, so
// the last round leaves every tile at its fixed point under its final halo:
// the unique fixed point (engine.py:9-18), exactly.  Round 0 is the
// reference's scan phase; the later rounds are its wavefront phase
// (K.220-270), level-synchronous like run_parallel's rounds
// (engine.py:251-364) at tile granularity, with the round's front as a
// deduplicated tile list (the GBQ of one round).
//
// Work split: entry i of a round's list goes to warp i mod nw, so every
// warp gets the same number of tiles (+-1) and knows its next tile while it
// processes the current one: the next tile's TMA boxes load into a second
// staging buffer meanwhile.  Flagging a tile = returned atomicOr on the next
// round's bitmap (dedupe) + a warp-aggregated push onto the next list.
struct RoundsArgs {
  unsigned *bm0, *bm1;      // round bitmaps (one bit per tile)
  unsigned *list0, *list1;  // round tile lists (ntiles entries each)
  unsigned *len;            // 3 list lengths (round % 3), 64 words apart
  unsigned *bar_count, *bar_gen;
};
constexpr int kLenStride = 64;

__device__ __forceinline__ void rounds_barrier(unsigned *count, unsigned *gen, unsigned nblocks,
                                               unsigned &g) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned arrived;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(count) : "memory");
    if (arrived == nblocks - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(gen) : "memory");
    } else {
      while (ld_acquire(gen) == g) __nanosleep(32);
    }
    g++;
  }
  __syncthreads();
}

// round 0's tile order: the 2 x 2 colour classes one after the other, each
// in raster order (the queue engine's initial queue order)
struct ColourOrder {
  unsigned cx[4], base[4];
  unsigned long long m[4];  // ceil(2^40 / cx): exact for cx < 2^14, r < 2^26
  __device__ ColourOrder(int ntx, int nty) {
    unsigned acc = 0;
#pragma unroll
    for (int c = 0; c < 4; c++) {
      cx[c] = (ntx - (c & 1) + 1) / 2;
      const unsigned cy = (nty - (c >> 1) + 1) / 2;
      base[c] = acc;
      acc += cx[c] * cy;
      m[c] = cx[c] ? ((1ull << 40) + cx[c] - 1) / cx[c] : 0;
    }
  }
  __device__ __forceinline__ unsigned tile(unsigned i, int ntx) const {
    const int c = (i >= base[1]) + (i >= base[2]) + (i >= base[3]);
    // (selects, not dynamic indices: the tables stay in registers)
    unsigned b = base[0], x = cx[0];
    unsigned long long mm = m[0];
#pragma unroll
    for (int k = 1; k < 4; k++)
      if (c == k) b = base[k], x = cx[k], mm = m[k];
    const unsigned r = i - b;
    const unsigned ry = (unsigned)((r * mm) >> 40), rx = r - ry * x;
    return (2 * ry + (c >> 1)) * (unsigned)ntx + 2 * rx + (c & 1);
  }
};

template <int CONN>
__global__ void __launch_bounds__(kCtaThreads, kRegCtaMinBlocks)
    tile_rounds_reg_kernel(EngineArgs a, RoundsArgs r, unsigned long long *counters,
                           const __grid_constant__ BoxMaps maps, int keep_counters, int rtrace,
                           int max_rounds) {
  __shared__ TmaWarpSmem tsm[kWarpsPerCta][2];
  __shared__ unsigned s_len;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned nw = gridDim.x * kWarpsPerCta;
  const unsigned gw = blockIdx.x * kWarpsPerCta + wib;
  const unsigned ntiles = (unsigned)a.ntx * a.nty;
  const unsigned nwords = (ntiles + 31) / 32;
  unsigned long long t_start = 0;
  if (rtrace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
  {  // clear both bitmaps and the control words, then one grid-wide sync
    const unsigned i0 = blockIdx.x * blockDim.x + threadIdx.x, st = gridDim.x * blockDim.x;
    for (unsigned i = i0; i < nwords; i += st) {
      r.bm0[i] = 0;
      r.bm1[i] = 0;
    }
    if (i0 < 3) r.len[i0 * kLenStride] = 0;
    if (i0 == 0) *r.bar_count = 0;
    if (!keep_counters && i0 < CNT_N) counters[i0] = 0;
  }
  cooperative_groups::this_grid().sync();
  unsigned bar_g = threadIdx.x == 0 ? ld_acquire(r.bar_gen) : 0u;

  if (lane == 0) {
    mbar_init(&tsm[wib][0].bar);
    mbar_init(&tsm[wib][1].bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const CUtensorMap *tmJ = &maps.m[0], *tmI = &maps.m[1];
  unsigned phase = 0;  // bit b: the parity of staging buffer b
  const bool l0 = lane == 0;
  unsigned long long n_tiles = 0, n_reruns = 0, n_steps = 0;
  const ColourOrder corder(a.ntx, a.nty);

  auto issue = [&](unsigned t, int bi) {  // lane 0: both boxes of tile t into buffer bi
    if (l0) {
      int tx, ty;
      tile_xy(a, t, tx, ty);
      TmaWarpSmem &ts = tsm[wib][bi];
      mbar_expect_tx(&ts.bar, 2u * kBoxBytes);
      tma_load_box(tmJ, ts.J, &ts.bar, tx * TS - kBoxX, ty * TS - 1);
      tma_load_box(tmI, ts.I, &ts.bar, tx * TS - kBoxX, ty * TS - 1);
    }
  };

  unsigned n = ntiles;  // this round's list length
  for (unsigned round = 0;; round++) {
    const unsigned *list = (round & 1) ? r.list1 : r.list0;
    unsigned *nlist = (round & 1) ? r.list0 : r.list1;
    unsigned *bcur = (round & 1) ? r.bm1 : r.bm0;
    unsigned *bnxt = (round & 1) ? r.bm0 : r.bm1;
    unsigned *nlen = &r.len[((round + 1) % 3) * kLenStride];
    // other SMs' stores of the previous round (ordered by the barrier) must be
    // visible to the async proxy that performs the box reads
    if (l0) asm volatile("fence.proxy.async.global;" ::: "memory");
    // the length counter of round + 2 was last read after round - 1's barrier
    if (blockIdx.x == 0 && threadIdx.x == 0) r.len[((round + 2) % 3) * kLenStride] = 0;
    auto entry = [&](unsigned i) -> unsigned {
      return round == 0 ? corder.tile(i, a.ntx) : ld_relaxed(&list[i]);
    };
    unsigned i = gw;
    unsigned t = i < n ? entry(i) : 0u;
    unsigned tn = i + nw < n ? entry(i + nw) : 0u;  // list entries load one tile ahead
    int bi = 0;
    if (i < n) issue(t, bi);
    while (i < n) {
      const unsigned i2 = i + nw;
      const unsigned tnn = i2 + nw < n ? entry(i2 + nw) : 0u;
      if (round > 0 && l0) bcur[t >> 5] = 0;  // consumed (bnxt of round + 1)
      __syncwarp();  // the other buffer's previous tile is done (WAR)
      if (i2 < n) issue(tn, bi ^ 1);
      TmaWarpSmem &ts = tsm[wib][bi];
      mbar_wait(&ts.bar, (phase >> bi) & 1u);
      phase ^= 1u << bi;
      int tx, ty;
      tile_xy(a, t, tx, ty);
      const int x0 = tx * TS, y0 = ty * TS;
      unsigned j[8], m[8];
      RegHalo h;
      const int hr = lane == 0 ? 0 : TS + 1;  // halo row (lanes 0 / 31)
      tma_row(ts.J, lane + 1, j);
      tma_row(ts.I, lane + 1, m);
      tma_row(ts.J, hr, h.row);
      h.l = ts.J[(lane + 1) * kBoxW + kBoxX - 1];
      h.r = ts.J[(lane + 1) * kBoxW + kBoxX + TS];
      h.lI = ts.I[(lane + 1) * kBoxW + kBoxX - 1];
      h.rI = ts.I[(lane + 1) * kBoxW + kBoxX + TS];
      h.cl = ts.J[hr * kBoxW + kBoxX - 1];
      h.cr = ts.J[hr * kBoxW + kBoxX + TS];
      h.clI = ts.I[hr * kBoxW + kBoxX - 1];
      h.crI = ts.I[hr * kBoxW + kBoxX + TS];
      const unsigned obl = j[0] & 0xffu, obr = j[7] >> 24;
      n_tiles += l0;
      n_reruns += l0 && round > 0;
      bool changed = false;
      const int steps = reg_fixpoint<CONN>(j, m, h, lane, changed);
      if (l0) n_steps += steps;
      if (__any_sync(FULL, changed)) {
        const int gy = y0 + lane;
        if (gy < a.H) {
          uint8_t *p = (uint8_t *)a.J + (size_t)gy * a.W + x0;
          reinterpret_cast<uint4 *>(p)[0] = make_uint4(j[0], j[1], j[2], j[3]);
          if (x0 + TS <= a.W)  // (else W % 32 == 16: the last tile column holds 16 pixels)
            reinterpret_cast<uint4 *>(p)[1] = make_uint4(j[4], j[5], j[6], j[7]);
        }
        // which neighbours can the changed border still raise?
        const unsigned need_ns = tma_need_rows<CONN>(ts, j, lane);
        const unsigned jl = j[0] & 0xffu, jr = j[7] >> 24;
        const unsigned cl = jl != obl ? jl : 0u, cr = jr != obr ? jr : 0u;
        unsigned dl = cl, dr = cr;
        if (CONN == 8) {
          unsigned lu = __shfl_up_sync(FULL, cl, 1), ld = __shfl_down_sync(FULL, cl, 1);
          unsigned ru = __shfl_up_sync(FULL, cr, 1), rd = __shfl_down_sync(FULL, cr, 1);
          if (lane == 0) lu = ru = 0;
          if (lane == 31) ld = rd = 0;
          dl = max(cl, max(lu, ld));
          dr = max(cr, max(ru, rd));
        }
        unsigned dirs = ((need_ns & 1u) << 1) | ((need_ns & 2u) << 6);  // N, S
        if (__any_sync(FULL, h.l < h.lI && h.l < dl)) dirs |= 1u << 3;   // W
        if (__any_sync(FULL, h.r < h.rI && h.r < dr)) dirs |= 1u << 5;   // E
        if (CONN == 8) {
          const bool cwl = h.cl < h.clI && h.cl < cl, cwr = h.cr < h.crI && h.cr < cr;
          if (__any_sync(FULL, l0 && cwl)) dirs |= 1u << 0;
          if (__any_sync(FULL, l0 && cwr)) dirs |= 1u << 2;
          if (__any_sync(FULL, lane == 31 && cwl)) dirs |= 1u << 6;
          if (__any_sync(FULL, lane == 31 && cwr)) dirs |= 1u << 8;
        }
        // flag: first setter of the tile's bit pushes it onto the next list
        bool push = false;
        unsigned nt = 0;
        if (lane < 9 && ((dirs >> lane) & 1u)) {
          const int nx = tx + (lane % 3) - 1, ny = ty + (lane / 3) - 1;
          if (nx >= 0 && nx < a.ntx && ny >= 0 && ny < a.nty) {
            nt = (unsigned)(ny * a.ntx + nx);
            const unsigned bit = 1u << (nt & 31);
            push = !(atomicOr(&bnxt[nt >> 5], bit) & bit);
          }
        }
        const unsigned pm = __ballot_sync(FULL, push);
        if (pm) {
          unsigned base = 0;
          if (l0) base = atomicAdd(nlen, (unsigned)__popc(pm));
          base = __shfl_sync(FULL, base, 0);
          if (push) nlist[base + __popc(pm & ((1u << lane) - 1))] = nt;
        }
      }
      i = i2;
      t = tn;
      tn = tnn;
      bi ^= 1;
    }
    rounds_barrier(r.bar_count, r.bar_gen, gridDim.x, bar_g);
    if (threadIdx.x == 0) {
      s_len = ld_relaxed(nlen);
      if (rtrace && blockIdx.x == 0 && round < 37) {
        unsigned long long now;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
        r.len[(3 + round) * kLenStride] = (unsigned)(now - t_start);  // trace: ns at round end
      }
    }
    __syncthreads();
    n = s_len;
    const bool limit = n != 0 && max_rounds > 0 && round + 1 >= (unsigned)max_rounds;
    if (n == 0 || limit) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(&counters[CNT_ROUNDS], round + 1);
        if (limit) counters[CNT_LIMIT] = 1;
      }
      break;
    }
  }
  if (l0) {
    atomicAdd(&counters[CNT_TILES], n_tiles);
    atomicAdd(&counters[CNT_RERUNS], n_reruns);
    atomicAdd(&counters[CNT_STEPS], n_steps);
  }
}

// --- register engine, 16 / 32-bit kinds (u16, int32; f32 via the ordered map) ---
//
// Same design as the u8 register engine: one warp per 32 x 32 tile, lane =
// row, the row's 32 values in registers (widened to int), Jacobi steps
// J <- min(I, max over the 3 x 3 / cross neighbourhood) to the tile's fixed
// point, the same queue protocol.  The tile and its halo are staged in
// shared memory first (TMA box when rows are 16-byte aligned, else a
// cooperative copy); the halo rows / columns and the last published border
// (the activation test's inputs) are read from that box, so registers hold
// only the 2 x 32 row values.
template <typename T>
struct R32 {
  static constexpr int OFF = 16 / (int)sizeof(T);  // box columns left of the tile
  static constexpr int BW = TS + 2 * OFF;          // box width (elements, 16-byte rows)
  static constexpr int LO = (int)Elem<T>::lo;      // the sentinel (outside the image)
};

template <typename T>
struct alignas(128) Box32Smem {
  static constexpr int BYTES = (TS + 2) * R32<T>::BW * (int)sizeof(T);
  T J[TS + 2][R32<T>::BW];
  uint8_t pad0[(128 - BYTES % 128) % 128];  // TMA destinations are 128-byte aligned
  T I[TS + 2][R32<T>::BW];
  uint8_t pad1[(128 - BYTES % 128) % 128];
  unsigned long long bar;
};

// stage the J (and I) box of tile (x0, y0); cells outside the image hold LO
// f32 as order-preserving int32 (the same map as recon_sweeps.cu's
// f32_to_ord: -0.0 -> +0.0, negative floats flip their magnitude bits)
__device__ __forceinline__ int f32_ord(int b) {
  if (b == INT_MIN) b = 0;
  return b >= 0 ? b : (b ^ 0x7fffffff);
}
__device__ __forceinline__ int f32_unord(int v) { return v >= 0 ? v : (v ^ 0x7fffffff); }

template <typename T, bool ORD = false>
__device__ __forceinline__ void box32_stage(const EngineArgs &a, const CUtensorMap *maps, int use_tma,
                                            Box32Smem<T> &b, int x0, int y0, bool withI,
                                            unsigned &phase, int lane) {
  constexpr int OFF = R32<T>::OFF, BW = R32<T>::BW;
  constexpr int BYTES = (TS + 2) * BW * (int)sizeof(T);
  __syncwarp();  // the previous box contents have been read
  const bool edge = x0 - OFF < 0 || y0 - 1 < 0 || x0 + TS + OFF > a.W || y0 + TS + 1 > a.H;
  if (use_tma) {
    if (lane == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      mbar_expect_tx(&b.bar, withI ? 2u * BYTES : (unsigned)BYTES);
      tma_load_box(maps, &b.J[0][0], &b.bar, x0 - OFF, y0 - 1);
      if (withI) tma_load_box(maps + 1, &b.I[0][0], &b.bar, x0 - OFF, y0 - 1);
    }
    mbar_wait(&b.bar, phase);
    phase ^= 1u;
    if (ORD) {  // f32 bit patterns -> ordered ints, in place
      int *bj = reinterpret_cast<int *>(&b.J[0][0]), *bi = reinterpret_cast<int *>(&b.I[0][0]);
      for (int i = lane; i < (TS + 2) * BW; i += 32) {
        bj[i] = f32_ord(bj[i]);
        if (withI) bi[i] = f32_ord(bi[i]);
      }
      __syncwarp();
    }
    if (edge && Elem<T>::lo != 0) {  // TMA fills with 0: patch the sentinel in
      for (int i = lane; i < (TS + 2) * BW; i += 32) {
        const int r = i / BW, c = i - r * BW, gx = x0 - OFF + c, gy = y0 - 1 + r;
        if (gx < 0 || gx >= a.W || gy < 0 || gy >= a.H) {
          b.J[r][c] = Elem<T>::lo;
          if (withI) b.I[r][c] = Elem<T>::lo;
        }
      }
    }
  } else {
    const T *J = (const T *)a.J, *I = (const T *)a.I;
    for (int i = lane; i < (TS + 2) * BW; i += 32) {
      const int r = i / BW, c = i - r * BW, gx = x0 - OFF + c, gy = y0 - 1 + r;
      const bool in = gx >= 0 && gx < a.W && gy >= 0 && gy < a.H;
      const size_t g = (size_t)gy * a.W + gx;
      if (ORD) {
        b.J[r][c] = in ? (T)f32_ord((int)ld_cg(J + g)) : Elem<T>::lo;
        if (withI) b.I[r][c] = in ? (T)f32_ord((int)__ldg(I + g)) : Elem<T>::lo;
      } else {
        b.J[r][c] = in ? ld_cg(J + g) : Elem<T>::lo;
        if (withI) b.I[r][c] = in ? __ldg(I + g) : Elem<T>::lo;
      }
    }
  }
  __syncwarp();
}

template <int CONN, typename T>
__device__ __forceinline__ int reg32_fixpoint(int *j, const int *m, const Box32Smem<T> &b, int lane,
                                              bool &changed) {
  constexpr int OFF = R32<T>::OFF, LO = R32<T>::LO;
  const int row = lane + 1;
  // The halo is constant during the iteration, so its whole effect on the
  // tile's fixed point is the lower bound min(I, halo dilation) on the edge
  // pixels: apply it once, then iterate with the tile closed (shuffles only).
  {
    int hl = (int)b.J[row][OFF - 1], hr = (int)b.J[row][OFF + TS];
    if (CONN == 8) {
      hl = max(hl, max((int)b.J[row - 1][OFF - 1], (int)b.J[row + 1][OFF - 1]));
      hr = max(hr, max((int)b.J[row - 1][OFF + TS], (int)b.J[row + 1][OFF + TS]));
    }
    bool ch = false;
    int nj = max(j[0], min(m[0], hl));
    ch |= nj != j[0];
    j[0] = nj;
    nj = max(j[TS - 1], min(m[TS - 1], hr));
    ch |= nj != j[TS - 1];
    j[TS - 1] = nj;
    if (lane == 0 || lane == 31) {
      const int hrow = lane == 0 ? 0 : TS + 1;
#pragma unroll
      for (int k = 0; k < TS; k++) {
        int h = (int)b.J[hrow][OFF + k];
        if (CONN == 8) h = max(h, max((int)b.J[hrow][OFF + k - 1], (int)b.J[hrow][OFF + k + 1]));
        nj = max(j[k], min(m[k], h));
        ch |= nj != j[k];
        j[k] = nj;
      }
    }
    changed |= ch;
  }
  int steps = 0;
  for (;;) {
    steps++;
    bool ch = false;
    // rows lane-1 / lane+1 (lanes 0 / 31 see themselves: harmless under max)
    auto vert = [&](int k) -> int {
      const int u = __shfl_up_sync(FULL, j[k], 1), d = __shfl_down_sync(FULL, j[k], 1);
      return CONN == 8 ? max(j[k], max(u, d)) : max(u, d);
    };
    if (CONN == 8) {
      int left = LO, vc = vert(0);  // left: max over the 3 rows at k-1, Gauss-Seidel in the row
#pragma unroll
      for (int k = 0; k < TS; k++) {
        const int vn = k + 1 < TS ? vert(k + 1) : LO;
        const int nj = min(m[k], max(vc, max(left, vn)));  // >= j[k]: the centre is included
        ch |= nj != j[k];
        j[k] = nj;
        left = max(vc, nj);
        vc = vn;
      }
    } else {
      int prev = LO;  // the updated left neighbour (Gauss-Seidel in the row)
#pragma unroll
      for (int k = 0; k < TS; k++) {
        const int right = k + 1 < TS ? j[k + 1] : LO;
        const int D = max(max(prev, right), vert(k));
        const int nj = max(j[k], min(m[k], D));
        ch |= nj != j[k];
        j[k] = nj;
        prev = nj;
      }
    }
    if (!__any_sync(FULL, ch)) break;
    changed = true;
  }
  return steps;
}

template <typename T, int CONN, bool ORD = false>
__global__ void __launch_bounds__(kCtaThreads, kReg32CtaMinBlocks)
    tile_engine_reg32_kernel(EngineArgs a, unsigned long long *counters,
                             const __grid_constant__ BoxMaps maps, int use_tma, int fused_init) {
  constexpr int OFF = R32<T>::OFF, LO = R32<T>::LO;
  if (fused_init) {  // cooperative launch: build the initial queue here
    tile_queue_init(a.q, a.ntx, a.nty, counters, 0);
    cooperative_groups::this_grid().sync();
  }
  const CUtensorMap *tmaps = &maps.m[0];
  __shared__ Box32Smem<T> bsm[kWarpsPerCta];
  Box32Smem<T> &b = bsm[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const bool l0 = lane == 0, l31 = lane == 31;
  unsigned phase = 0;
  if (use_tma && l0) {
    mbar_init(&b.bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned long long n_tiles = 0, n_reruns = 0, n_steps = 0;
  unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
  int next_tile = -1;
  for (;;) {
    long long c_pop = pclock(l0);
    int t = -1;
    if (l0) {
      t = next_tile >= 0 ? next_tile : ring_pop(a.q);
      if (t >= 0) {
        state_take(&a.q.state[t]);
      }
    }
    t = __shfl_sync(FULL, t, 0);
    next_tile = -1;
    if (t < 0) break;
    int tx, ty;
    tile_xy(a, (unsigned)t, tx, ty);
    const int x0 = tx * TS, y0 = ty * TS;
    long long c_load = pclock(l0);
    if (kPhases && l0) ph[0] += c_load - c_pop;
    box32_stage<T, ORD>(a, tmaps, use_tma, b, x0, y0, true, phase, lane);
    int j[TS], m[TS];
#pragma unroll
    for (int k = 0; k < TS; k++) {
      j[k] = (int)b.J[lane + 1][OFF + k];
      m[k] = (int)b.I[lane + 1][OFF + k];
    }
    if (kPhases && l0) ph[1] += clock64() - c_load;
    bool rerun = false;
    for (;;) {
      n_tiles += l0;
      n_reruns += l0 && rerun;
      long long c_fix = pclock(l0);
      bool changed = false;
      const int steps = reg32_fixpoint<CONN, T>(j, m, b, lane, changed);
      if (l0) n_steps += steps;
      changed = __any_sync(FULL, changed);
      long long c_st = pclock(l0);
      if (kPhases && l0) ph[2] += c_st - c_fix;
      if (changed) {
        const int gy = y0 + lane;
        if (gy < a.H) {  // store my row
          T *p = (T *)a.J + (size_t)gy * a.W + x0;
          if (a.vec && x0 + TS <= a.W) {
            constexpr int E = 16 / (int)sizeof(T);
#pragma unroll
            for (int v = 0; v < TS / E; v++) {
              uint4 w;
              T *e = reinterpret_cast<T *>(&w);
#pragma unroll
              for (int q = 0; q < E; q++) e[q] = (T)(ORD ? f32_unord(j[v * E + q]) : j[v * E + q]);
              reinterpret_cast<uint4 *>(p)[v] = w;
            }
          } else {
#pragma unroll
            for (int k = 0; k < TS; k++)
              if (x0 + k < a.W) p[k] = (T)(ORD ? f32_unord(j[k]) : j[k]);
          }
        }
        if (a.dirty && l0) a.dirty[ty] = 1;
        // the box still holds the border as last published (loaded at the
        // start of the activation / refreshed on re-runs)
        const int row = lane + 1, ob_row = l0 ? 1 : TS, h_row = l0 ? 0 : TS + 1;
        bool need_row = false;
        if (l0 || l31) {
          int cp = LO, cc = j[0] != (int)b.J[ob_row][OFF] ? j[0] : LO;
#pragma unroll
          for (int k = 0; k < TS; k++) {
            const int cn = k + 1 < TS ? (j[k + 1] != (int)b.J[ob_row][OFF + k + 1] ? j[k + 1] : LO) : LO;
            const int D = CONN == 8 ? max(cc, max(cp, cn)) : cc;
            const int hJ = (int)b.J[h_row][OFF + k], hI = (int)b.I[h_row][OFF + k];
            need_row |= hJ < hI && hJ < D;
            cp = cc;
            cc = cn;
          }
        }
        const int cl = j[0] != (int)b.J[row][OFF] ? j[0] : LO;
        const int cr = j[TS - 1] != (int)b.J[row][OFF + TS - 1] ? j[TS - 1] : LO;
        int dl = cl, dr = cr;
        if (CONN == 8) {
          int u = __shfl_up_sync(FULL, cl, 1), d = __shfl_down_sync(FULL, cl, 1);
          if (l0) u = LO;
          if (l31) d = LO;
          dl = max(cl, max(u, d));
          u = __shfl_up_sync(FULL, cr, 1);
          d = __shfl_down_sync(FULL, cr, 1);
          if (l0) u = LO;
          if (l31) d = LO;
          dr = max(cr, max(u, d));
        }
        const int hlJ = (int)b.J[row][OFF - 1], hlI = (int)b.I[row][OFF - 1];
        const int hrJ = (int)b.J[row][OFF + TS], hrI = (int)b.I[row][OFF + TS];
        unsigned dirs = 0;
        if (__any_sync(FULL, l0 && need_row)) dirs |= 1u << 1;   // N
        if (__any_sync(FULL, l31 && need_row)) dirs |= 1u << 7;  // S
        if (__any_sync(FULL, hlJ < hlI && hlJ < dl)) dirs |= 1u << 3;  // W
        if (__any_sync(FULL, hrJ < hrI && hrJ < dr)) dirs |= 1u << 5;  // E
        if (CONN == 8) {
          const int cJl = (int)b.J[h_row][OFF - 1], cIl = (int)b.I[h_row][OFF - 1];
          const int cJr = (int)b.J[h_row][OFF + TS], cIr = (int)b.I[h_row][OFF + TS];
          const bool cwl = cJl < cIl && cJl < cl, cwr = cJr < cIr && cJr < cr;
          if (__any_sync(FULL, l0 && cwl)) dirs |= 1u << 0;
          if (__any_sync(FULL, l0 && cwr)) dirs |= 1u << 2;
          if (__any_sync(FULL, l31 && cwl)) dirs |= 1u << 6;
          if (__any_sync(FULL, l31 && cwr)) dirs |= 1u << 8;
        }
        // the published border becomes the reference for the next check
        __syncwarp();
        b.J[row][OFF] = (T)j[0];
        b.J[row][OFF + TS - 1] = (T)j[TS - 1];
        if (l0 || l31)
#pragma unroll
          for (int k = 0; k < TS; k++) b.J[ob_row][OFF + k] = (T)j[k];
        fence_acq_rel();  // publish before any neighbour is (re)queued and before the finish
        __syncwarp();
        bool own = false;
        unsigned ntile = 0;
        if (lane < 9 && ((dirs >> lane) & 1u)) {
          int ntxi = tx + (lane % 3) - 1, ntyi = ty + (lane / 3) - 1;
          if (ntxi >= 0 && ntxi < a.ntx && ntyi >= 0 && ntyi < a.nty) {
            ntile = (unsigned)(ntyi * a.ntx + ntxi);
            own = activate_claim_nopend(a.q, ntile);
          }
        }
        unsigned ownmask = __ballot_sync(FULL, own);
        int keep = (ownmask && next_tile < 0) ? __ffs(ownmask) - 1 : -1;
        // the kept continuation inherits this tile's pending count (no +1 here,
        // no -1 at this tile's finish); a pushed tile counts before its push
        if (own && lane != keep) {
          atomicAdd(a.q.pending, 1u);
          ring_push(a.q, ntile);
        }
        if (keep >= 0) next_tile = __shfl_sync(FULL, (int)ntile, keep);
      }
      int done = 0;
      if (l0) {
        unsigned old = atomicCAS(&a.q.state[t], ST_R, 0u);
        if (old == ST_R) {
          if (next_tile < 0) atomicSub(a.q.pending, 1u);  // (else passed on, above)
          done = 1;
        } else {
          state_take(&a.q.state[t]);  // consume the request (acquire)
        }
      }
      done = __shfl_sync(FULL, done, 0);
      if (kPhases && l0) ph[5] += clock64() - c_st;
      if (done) break;
      box32_stage<T, ORD>(a, tmaps, use_tma, b, x0, y0, false, phase, lane);  // J halo (+ our rows)
      rerun = true;
    }
  }
  if (l0) {
    atomicAdd(&counters[CNT_TILES], n_tiles);
    atomicAdd(&counters[CNT_RERUNS], n_reruns);
    atomicAdd(&counters[CNT_STEPS], n_steps);
    if (kPhases)
      for (int i = 0; i < 6; i++) atomicAdd(&counters[CNT_PH_POP + i], ph[i]);
  }
}

// --- binary engine (bit planes) ------------------------------------------------
//
// The "binary" element kind (grid.py binary, imfill).  iwpp_recon packs the
// 0 / 255 marker and mask into bit planes (one bit per pixel, ceil(W/32)
// words per row) and unpacks the result afterwards, so the engine moves
// 1/8 of the bytes and does no byte arithmetic.  A warp owns a 128 x 128
// tile -- lane = rows lane + 32 q (q = 0..3), four words per row -- and a
// Jacobi step
//     J <- I & (J | J_up | J_down | the same shifted by one column)
// plus whole row and column run fills is a few hundred instructions for
// 16384 pixels.  Binary fills are long narrow fronts crossing the image tile
// by tile; 128-pixel tiles quarter the tile hops of 32-pixel tiles on that
// critical path.  Same queue protocol, on a 128-pixel tile grid.

__device__ __forceinline__ unsigned bitw(const uint32_t *P, int WW, int H, int wx, int gy, bool cg) {
  if (gy < 0 || gy >= H || wx < 0 || wx >= WW) return 0u;
  const uint32_t *p = P + (size_t)gy * WW + wx;
  return cg ? __ldcg(p) : __ldg(p);
}

constexpr int BNR = TSB / 32;  // rows per lane: lane + 32 q, q = 0 .. BNR - 1
constexpr int BNW = TSB / 32;  // 32-bit words per tile row
static_assert(BNR == 4 && BNW == 4, "the binary engine's masks assume 128 x 128 tiles");

struct BinHalo {
  unsigned row[BNW], rowI[BNW];  // lane 0: the row above; lane 31: the row below
  unsigned l, r, lI, rI;         // bit q: the cell left / right of row lane + 32 q (J, I)
  unsigned cl, cr, clI, crI;     // lane 0: corners above; lane 31: corners below
};

// the tile (rows lane + 32 q, words wx .. wx + 3) and its halo: every load
// issued before any is used (16-byte loads when the plane's rows allow)
__device__ __forceinline__ void bin_load(const EngineArgs &a, int x0, int y0, int lane, bool tile,
                                         unsigned (&jt)[BNR][BNW], unsigned (&mt)[BNR][BNW],
                                         BinHalo &h) {
  const uint32_t *J = (const uint32_t *)a.J, *I = (const uint32_t *)a.I;
  const int WW = a.WW, wx = x0 >> 5;
  const bool vec = (WW & 3) == 0 && wx + BNW <= WW;
  const int hy = lane == 0 ? y0 - 1 : (lane == 31 ? y0 + TSB : -1);
  if (tile) {
#pragma unroll
    for (int q = 0; q < BNR; q++) {
      const int gy = y0 + lane + 32 * q;
      if (vec && gy < a.H) {
        const uint4 vj = __ldcg(reinterpret_cast<const uint4 *>(J + (size_t)gy * WW + wx));
        const uint4 vi = __ldg(reinterpret_cast<const uint4 *>(I + (size_t)gy * WW + wx));
        jt[q][0] = vj.x; jt[q][1] = vj.y; jt[q][2] = vj.z; jt[q][3] = vj.w;
        mt[q][0] = vi.x; mt[q][1] = vi.y; mt[q][2] = vi.z; mt[q][3] = vi.w;
      } else {
#pragma unroll
        for (int w = 0; w < BNW; w++) {
          jt[q][w] = bitw(J, WW, a.H, wx + w, gy, true);
          mt[q][w] = bitw(I, WW, a.H, wx + w, gy, false);
        }
      }
    }
  }
  unsigned jl[BNR], jr[BNR], il[BNR], ir[BNR];
#pragma unroll
  for (int q = 0; q < BNR; q++) {
    const int gy = y0 + lane + 32 * q;
    jl[q] = bitw(J, WW, a.H, wx - 1, gy, true);
    jr[q] = bitw(J, WW, a.H, wx + BNW, gy, true);
    il[q] = bitw(I, WW, a.H, wx - 1, gy, false);
    ir[q] = bitw(I, WW, a.H, wx + BNW, gy, false);
  }
#pragma unroll
  for (int w = 0; w < BNW; w++) {
    h.row[w] = bitw(J, WW, a.H, wx + w, hy, true);
    h.rowI[w] = bitw(I, WW, a.H, wx + w, hy, false);
  }
  const unsigned jhl = bitw(J, WW, a.H, wx - 1, hy, true), jhr = bitw(J, WW, a.H, wx + BNW, hy, true);
  const unsigned ihl = bitw(I, WW, a.H, wx - 1, hy, false), ihr = bitw(I, WW, a.H, wx + BNW, hy, false);
  h.l = h.r = h.lI = h.rI = 0;
#pragma unroll
  for (int q = 0; q < BNR; q++) {
    h.l |= (jl[q] >> 31) << q;
    h.r |= (jr[q] & 1u) << q;
    h.lI |= (il[q] >> 31) << q;
    h.rI |= (ir[q] & 1u) << q;
  }
  h.cl = jhl >> 31; h.cr = jhr & 1u; h.clI = ihl >> 31; h.crI = ihr & 1u;
}

// TMA staging of a binary tile (bit planes with W % 128 == 0): one box per
// plane of 12 words x 130 rows -- image words wx - 4 .. wx + 7 (16-byte
// aligned start; the tile is words 4..7, its halo words 3 and 8) and rows
// y0 - 1 .. y0 + 128 -- instead of ~60 scattered per-lane loads; cells
// outside the image arrive as 0, the plane's own outside value.
constexpr int kBinBoxW = 12, kBinBoxH = TSB + 2, kBinBoxX = 4;
struct alignas(128) BinBoxSmem {  // (TMA destinations 128-byte aligned)
  uint32_t J[kBinBoxH][kBinBoxW];
  uint8_t pad0[(128 - kBinBoxH * kBinBoxW * 4 % 128) % 128];
  uint32_t I[kBinBoxH][kBinBoxW];
  uint8_t pad1[(128 - kBinBoxH * kBinBoxW * 4 % 128) % 128];
  unsigned long long bar;
};
static_assert(offsetof(BinBoxSmem, I) % 128 == 0, "TMA destination alignment");

__device__ __forceinline__ void bin_load_box(const CUtensorMap *maps, BinBoxSmem &b, int x0, int y0,
                                             int lane, bool tile, unsigned &phase,
                                             unsigned (&jt)[BNR][BNW], unsigned (&mt)[BNR][BNW],
                                             BinHalo &h) {
  constexpr unsigned BYTES = kBinBoxH * kBinBoxW * 4;
  __syncwarp();  // the previous boxes have been read
  if (lane == 0) {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    mbar_expect_tx(&b.bar, tile ? 2u * BYTES : BYTES);
    tma_load_box(maps, &b.J[0][0], &b.bar, (x0 >> 5) - kBinBoxX, y0 - 1);
    if (tile) tma_load_box(maps + 1, &b.I[0][0], &b.bar, (x0 >> 5) - kBinBoxX, y0 - 1);
  }
  mbar_wait(&b.bar, phase);
  phase ^= 1u;
  h.l = h.r = h.lI = h.rI = 0;
#pragma unroll
  for (int q = 0; q < BNR; q++) {
    const int r = lane + 32 * q + 1;
    if (tile) {
      const uint4 vj = *reinterpret_cast<const uint4 *>(&b.J[r][kBinBoxX]);
      const uint4 vi = *reinterpret_cast<const uint4 *>(&b.I[r][kBinBoxX]);
      jt[q][0] = vj.x; jt[q][1] = vj.y; jt[q][2] = vj.z; jt[q][3] = vj.w;
      mt[q][0] = vi.x; mt[q][1] = vi.y; mt[q][2] = vi.z; mt[q][3] = vi.w;
    }
    h.l |= (b.J[r][kBinBoxX - 1] >> 31) << q;
    h.r |= (b.J[r][kBinBoxX + BNW] & 1u) << q;
    h.lI |= (b.I[r][kBinBoxX - 1] >> 31) << q;
    h.rI |= (b.I[r][kBinBoxX + BNW] & 1u) << q;
  }
  const int hr = lane == 0 ? 0 : kBinBoxH - 1;  // halo row (lanes 0 / 31)
#pragma unroll
  for (int w = 0; w < BNW; w++) {
    h.row[w] = b.J[hr][kBinBoxX + w];
    h.rowI[w] = b.I[hr][kBinBoxX + w];
  }
  h.cl = b.J[hr][kBinBoxX - 1] >> 31;
  h.cr = b.J[hr][kBinBoxX + BNW] & 1u;
  h.clI = b.I[hr][kBinBoxX - 1] >> 31;
  h.crI = b.I[hr][kBinBoxX + BNW] & 1u;
}

// Vertical neighbours of a column of per-row bits packed as bit q = row
// lane + 32 q (the rows above / below within the tile; `in_up` / `in_dn`:
// lane 0's bit 0 above / lane 31's bit BNR-1 below come from outside).
__device__ __forceinline__ unsigned bits_up(unsigned b, int lane, unsigned in_up) {
  const unsigned R = __shfl_sync(FULL, b, (lane + 31) & 31);  // lane - 1 (lane 0: lane 31)
  return lane == 0 ? (((R << 1) & ((1u << BNR) - 2u)) | in_up) : R;
}
__device__ __forceinline__ unsigned bits_dn(unsigned b, int lane, unsigned in_dn) {
  const unsigned S = __shfl_sync(FULL, b, (lane + 1) & 31);  // lane + 1 (lane 31: lane 0)
  return lane == 31 ? ((S >> 1) | (in_dn << (BNR - 1))) : S;
}

// 3x3 (8-conn) / cross (4-conn) horizontal dilation of a 128-bit row with
// the halo bits at its ends
__device__ __forceinline__ void bin_hdil(const unsigned (&v)[BNW], unsigned hl, unsigned hr,
                                         unsigned (&d)[BNW]) {
#pragma unroll
  for (int w = 0; w < BNW; w++)
    d[w] = v[w] | (v[w] << 1) | (v[w] >> 1) | (w ? v[w - 1] >> 31 : hl) |
           (w < BNW - 1 ? v[w + 1] << 31 : hr << 31);
}

// Row run fill: every mask bit joined to a set bit by a run of mask bits,
// in one step.  For seeds s within mask m, m + s carries from a run's
// lowest seed to the run's top (and one bit past it, outside m), so
// ((m + s) ^ m) | s, masked by m, is the run above each lowest seed; the
// other direction is the same on the bit-reversed row.  Rows are 128 bits:
// one add-with-carry chain.
#ifndef IWPP_BIN_RUNFILL
#define IWPP_BIN_RUNFILL 1
#endif
__device__ __forceinline__ void up_fill128(const unsigned (&s)[BNW], const unsigned (&m)[BNW],
                                           unsigned (&f)[BNW]) {
  unsigned t0, t1, t2, t3;
  asm("add.cc.u32 %0, %4, %8;\n\t"
      "addc.cc.u32 %1, %5, %9;\n\t"
      "addc.cc.u32 %2, %6, %10;\n\t"
      "addc.u32 %3, %7, %11;"
      : "=r"(t0), "=r"(t1), "=r"(t2), "=r"(t3)
      : "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "r"(s[0]), "r"(s[1]), "r"(s[2]), "r"(s[3]));
  f[0] = ((t0 ^ m[0]) | s[0]) & m[0];
  f[1] = ((t1 ^ m[1]) | s[1]) & m[1];
  f[2] = ((t2 ^ m[2]) | s[2]) & m[2];
  f[3] = ((t3 ^ m[3]) | s[3]) & m[3];
}
__device__ __forceinline__ void row_fill(unsigned (&x)[BNW], const unsigned (&m)[BNW]) {
  unsigned f[BNW], rs[BNW], rm[BNW], g[BNW];
  up_fill128(x, m, f);
#pragma unroll
  for (int w = 0; w < BNW; w++) {
    rs[w] = __brev(x[BNW - 1 - w]);
    rm[w] = __brev(m[BNW - 1 - w]);
  }
  up_fill128(rs, rm, g);
#pragma unroll
  for (int w = 0; w < BNW; w++) x[w] = f[w] | __brev(g[BNW - 1 - w]);
}

// Column run fill over the tile's 128 rows, one word of columns: a
// Kogge-Stone segmented scan down and up the lanes inside each 32-row
// quarter (g |= p & g[lane - d], p &= p[lane - d]; p: the mask all along
// the span), then the carries across the quarters (a quarter's top rows
// take the fill of the row above it where the mask runs unbroken from
// there; the same upwards).
#ifndef IWPP_BIN_COLFILL
#define IWPP_BIN_COLFILL 1
#endif
__device__ __forceinline__ void col_fill(unsigned (&x)[BNR], const unsigned (&m)[BNR], int lane) {
  unsigned g[BNR], p[BNR], h[BNR], r[BNR];
#pragma unroll
  for (int q = 0; q < BNR; q++) {
    g[q] = h[q] = x[q];
    p[q] = r[q] = m[q];
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
    for (int q = 0; q < BNR; q++) {
      const unsigned gu = __shfl_up_sync(FULL, g[q], d), pu = __shfl_up_sync(FULL, p[q], d);
      const unsigned hd = __shfl_down_sync(FULL, h[q], d), rd = __shfl_down_sync(FULL, r[q], d);
      if (lane >= d) g[q] |= p[q] & gu, p[q] &= pu;
      if (lane + d < 32) h[q] |= r[q] & hd, r[q] &= rd;
    }
  }
#pragma unroll
  for (int q = 1; q < BNR; q++) g[q] |= p[q] & __shfl_sync(FULL, g[q - 1], 31);
#pragma unroll
  for (int q = BNR - 2; q >= 0; q--) h[q] |= r[q] & __shfl_sync(FULL, h[q + 1], 0);
#pragma unroll
  for (int q = 0; q < BNR; q++) x[q] = g[q] | h[q];
}

template <int CONN>
__device__ __forceinline__ int bin_fixpoint(unsigned (&A)[BNR][BNW], const unsigned (&M)[BNR][BNW],
                                            const BinHalo &h, int lane, bool &changed) {
  // halo column bits (bit q: row lane + 32 q), vertically dilated for 8-conn
  unsigned hl = h.l, hr = h.r;
  if (CONN == 8) {
    hl = h.l | bits_up(h.l, lane, h.cl) | bits_dn(h.l, lane, h.cl);
    hr = h.r | bits_up(h.r, lane, h.cr) | bits_dn(h.r, lane, h.cr);
  }
  int steps = 0;
  for (;;) {
    steps++;
    unsigned N[BNR][BNW];
    // rows above / below: the neighbouring lane, across quarters through
    // lanes 0 / 31, and the halo rows at the tile's top / bottom
#pragma unroll
    for (int w = 0; w < BNW; w++) {
      unsigned R[BNR], S[BNR];
#pragma unroll
      for (int q = 0; q < BNR; q++) {
        R[q] = __shfl_sync(FULL, A[q][w], (lane + 31) & 31);
        S[q] = __shfl_sync(FULL, A[q][w], (lane + 1) & 31);
      }
#pragma unroll
      for (int q = 0; q < BNR; q++) {
        const unsigned up = lane == 0 ? (q ? R[q - 1] : h.row[w]) : R[q];
        const unsigned dn = lane == 31 ? (q < BNR - 1 ? S[q + 1] : h.row[w]) : S[q];
        N[q][w] = CONN == 8 ? (A[q][w] | up | dn) : (up | dn);
      }
    }
#pragma unroll
    for (int q = 0; q < BNR; q++) {
      unsigned D[BNW];
      if (CONN == 8) {
        bin_hdil(N[q], (hl >> q) & 1u, (hr >> q) & 1u, D);
      } else {
        bin_hdil(A[q], (h.l >> q) & 1u, (h.r >> q) & 1u, D);
#pragma unroll
        for (int w = 0; w < BNW; w++) D[w] |= N[q][w];
      }
#pragma unroll
      for (int w = 0; w < BNW; w++) N[q][w] = M[q][w] & D[w];
    }
    // The plain step is the fixed-point test: if it adds nothing, no mask
    // cell touches a set cell, so the run fills below cannot add anything
    // either.  Only a step that changes something pays for the fills.
    unsigned ch = 0;
#pragma unroll
    for (int q = 0; q < BNR; q++)
#pragma unroll
      for (int w = 0; w < BNW; w++) ch |= N[q][w] ^ A[q][w];
    if (!__any_sync(FULL, ch != 0)) break;
    if (IWPP_BIN_RUNFILL) {  // whole row runs in one step
#pragma unroll
      for (int q = 0; q < BNR; q++) row_fill(N[q], M[q]);
    }
    if (IWPP_BIN_COLFILL) {  // and whole column runs of the tile
#pragma unroll
      for (int w = 0; w < BNW; w++) {
        unsigned x[BNR], m[BNR];
#pragma unroll
        for (int q = 0; q < BNR; q++) x[q] = N[q][w], m[q] = M[q][w];
        col_fill(x, m, lane);
#pragma unroll
        for (int q = 0; q < BNR; q++) N[q][w] = x[q];
      }
    }
#pragma unroll
    for (int q = 0; q < BNR; q++)
#pragma unroll
      for (int w = 0; w < BNW; w++) A[q][w] = N[q][w];
    changed = true;
  }
  return steps;
}

template <int CONN>
__global__ void __launch_bounds__(kCtaThreads, 3)
    tile_engine_bin_kernel(EngineArgs a, unsigned long long *counters,
                           const __grid_constant__ BoxMaps maps, int use_tma) {
  extern __shared__ __align__(128) unsigned char bin_dsmem[];  // use_tma: one BinBoxSmem per warp
  const int lane = threadIdx.x & 31;
  const bool l0 = lane == 0, l31 = lane == 31;
  BinBoxSmem &bx = reinterpret_cast<BinBoxSmem *>(bin_dsmem)[threadIdx.x >> 5];
  unsigned tphase = 0;
  if (use_tma && l0) {
    mbar_init(&bx.bar);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned long long n_tiles = 0, n_reruns = 0, n_steps = 0;
  unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
  int next_tile = -1;
  for (;;) {
    long long c_pop = pclock(l0);
    int t = -1;
    if (l0) {
      t = next_tile >= 0 ? next_tile : ring_pop<32>(a.q);
      if (t >= 0) {
        state_take(&a.q.state[t]);
      }
    }
    t = __shfl_sync(FULL, t, 0);
    next_tile = -1;
    if (t < 0) break;
    int tx, ty;
    tile_xy(a, (unsigned)t, tx, ty);
    const int x0 = tx * TSB, y0 = ty * TSB;
    long long c_load = pclock(l0);
    if (kPhases && l0) ph[0] += c_load - c_pop;
    unsigned A[BNR][BNW], M[BNR][BNW], O[BNR][BNW];  // O: as last published
    BinHalo h;
    if (use_tma)
      bin_load_box(&maps.m[0], bx, x0, y0, lane, true, tphase, A, M, h);
    else
      bin_load(a, x0, y0, lane, true, A, M, h);
#pragma unroll
    for (int q = 0; q < BNR; q++)
#pragma unroll
      for (int w = 0; w < BNW; w++) O[q][w] = A[q][w];
    if (kPhases && l0) ph[1] += clock64() - c_load;
    bool rerun = false;
    for (;;) {
      n_tiles += l0;
      n_reruns += l0 && rerun;
      long long c_fix = pclock(l0);
      bool changed = false;
      const int steps = bin_fixpoint<CONN>(A, M, h, lane, changed);
      if (l0) n_steps += steps;
      changed = __any_sync(FULL, changed);
      long long c_st = pclock(l0);
      if (kPhases && l0) ph[2] += c_st - c_fix;
      if (changed) {
        uint32_t *Jw = (uint32_t *)a.J;
        const int wx = x0 >> 5;
#pragma unroll
        for (int q = 0; q < BNR; q++) {
          const int gy = y0 + lane + 32 * q;
          if (gy < a.H) {
#pragma unroll
            for (int w = 0; w < BNW; w++)
              if (A[q][w] != O[q][w]) Jw[(size_t)gy * a.WW + wx + w] = A[q][w];
          }
        }
        if (a.dirty && l0) a.dirty[ty] = 1;
        // newly set border cells; a neighbour needs a re-run where such a
        // cell (dilated along the border for 8-conn) meets a halo cell with
        // J = 0, I = 1
        unsigned need_row = 0;  // lane 0: top row vs the row above; lane 31: bottom vs below
        {
          const int qe = l0 ? 0 : BNR - 1;
          unsigned c[BNW];
#pragma unroll
          for (int w = 0; w < BNW; w++) c[w] = (qe == 0 ? A[0][w] & ~O[0][w] : A[BNR - 1][w] & ~O[BNR - 1][w]);
#pragma unroll
          for (int w = 0; w < BNW; w++) {
            unsigned d = c[w];
            if (CONN == 8)
              d |= (c[w] << 1) | (c[w] >> 1) | (w ? c[w - 1] >> 31 : 0u) | (w < BNW - 1 ? c[w + 1] << 31 : 0u);
            need_row |= d & h.rowI[w] & ~h.row[w];
          }
        }
        unsigned cl = 0, cr = 0;  // bit q: row lane + 32 q's left / right cell newly set
#pragma unroll
        for (int q = 0; q < BNR; q++) {
          cl |= ((A[q][0] & ~O[q][0]) & 1u) << q;
          cr |= ((A[q][BNW - 1] & ~O[q][BNW - 1]) >> 31) << q;
        }
        unsigned dl = cl, dr = cr;
        if (CONN == 8) {
          dl |= bits_up(cl, lane, 0u) | bits_dn(cl, lane, 0u);
          dr |= bits_up(cr, lane, 0u) | bits_dn(cr, lane, 0u);
        }
        unsigned dirs = 0;
        if (__any_sync(FULL, l0 && need_row)) dirs |= 1u << 1;   // N
        if (__any_sync(FULL, l31 && need_row)) dirs |= 1u << 7;  // S
        if (__any_sync(FULL, dl & h.lI & ~h.l)) dirs |= 1u << 3;  // W
        if (__any_sync(FULL, dr & h.rI & ~h.r)) dirs |= 1u << 5;  // E
        if (CONN == 8) {  // corners: one interior cell each
          const unsigned c0l = cl & 1u, c0r = cr & 1u, c3l = (cl >> (BNR - 1)) & 1u, c3r = (cr >> (BNR - 1)) & 1u;
          if (__any_sync(FULL, l0 && (c0l & h.clI & ~h.cl))) dirs |= 1u << 0;
          if (__any_sync(FULL, l0 && (c0r & h.crI & ~h.cr))) dirs |= 1u << 2;
          if (__any_sync(FULL, l31 && (c3l & h.clI & ~h.cl))) dirs |= 1u << 6;
          if (__any_sync(FULL, l31 && (c3r & h.crI & ~h.cr))) dirs |= 1u << 8;
        }
#pragma unroll
        for (int q = 0; q < BNR; q++)
#pragma unroll
          for (int w = 0; w < BNW; w++) O[q][w] = A[q][w];
        // publish the tile before any neighbour is (re)queued, and before
        // this tile's finish: the finish CAS is what lets a later activation
        // pop the tile again, and its next owner must load these values (a
        // stale interior could be recomputed lower and overwrite them)
        fence_acq_rel();
        __syncwarp();
        bool own = false;
        unsigned ntile = 0;
        if (lane < 9 && ((dirs >> lane) & 1u)) {
          int ntxi = tx + (lane % 3) - 1, ntyi = ty + (lane / 3) - 1;
          if (ntxi >= 0 && ntxi < a.ntx && ntyi >= 0 && ntyi < a.nty) {
            ntile = (unsigned)(ntyi * a.ntx + ntxi);
            own = activate_claim_nopend(a.q, ntile);
          }
        }
        unsigned ownmask = __ballot_sync(FULL, own);
        int keep = (ownmask && next_tile < 0) ? __ffs(ownmask) - 1 : -1;
        // the kept continuation inherits this tile's pending count (no +1 here,
        // no -1 at this tile's finish); a pushed tile counts before its push
        if (own && lane != keep) {
          atomicAdd(a.q.pending, 1u);
          ring_push(a.q, ntile);
        }
        if (keep >= 0) next_tile = __shfl_sync(FULL, (int)ntile, keep);
      }
      int done = 0;
      if (l0) {
        unsigned old = atomicCAS(&a.q.state[t], ST_R, 0u);
        if (old == ST_R) {
          if (next_tile < 0) atomicSub(a.q.pending, 1u);  // (else passed on, above)
          done = 1;
        } else {
          state_take(&a.q.state[t]);  // consume the request (acquire)
        }
      }
      done = __shfl_sync(FULL, done, 0);
      if (kPhases && l0) ph[5] += clock64() - c_st;
      if (done) break;
      if (use_tma)  // the tile is ours: halo only
        bin_load_box(&maps.m[0], bx, x0, y0, lane, false, tphase, A, M, h);
      else
        bin_load(a, x0, y0, lane, false, A, M, h);
      rerun = true;
    }
  }
  if (l0) {
    atomicAdd(&counters[CNT_TILES], n_tiles);
    atomicAdd(&counters[CNT_RERUNS], n_reruns);
    atomicAdd(&counters[CNT_STEPS], n_steps);
    if (kPhases)
      for (int i = 0; i < 6; i++) atomicAdd(&counters[CNT_PH_POP + i], ph[i]);
  }
}

// 0 / 255 bytes <-> bit planes: one thread per 32-pixel word (32-bit index
// math; rows 16-byte aligned -> two 16-byte loads / stores per word)
__device__ __forceinline__ unsigned pack_bits(const unsigned *w) {
  unsigned b = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const unsigned t = (w[k] | (w[k] << 1) | (w[k] << 2) | (w[k] << 3) | (w[k] << 4) |
                        (w[k] << 5) | (w[k] << 6) | (w[k] << 7)) & 0x80808080u;  // byte != 0
    b |= ((t * 0x00204081u) >> 28) << (4 * k);
  }
  return b;
}

// blockIdx.y selects the plane: (src, bits) or (src2, bits2) -- the marker
// and the mask are packed by one launch
__global__ void bin_pack_kernel(const uint8_t *__restrict__ src0, int W, int H,
                                uint32_t *__restrict__ bits0, int vec0,
                                const uint8_t *__restrict__ src2, uint32_t *__restrict__ bits2, int vec2) {
  const uint8_t *__restrict__ src = blockIdx.y ? src2 : src0;
  uint32_t *__restrict__ bits = blockIdx.y ? bits2 : bits0;
  const int vec = blockIdx.y ? vec2 : vec0;
  const unsigned WW = (unsigned)(W + 31) >> 5;
  const unsigned nw = WW * (unsigned)H;
  for (unsigned wi = blockIdx.x * blockDim.x + threadIdx.x; wi < nw; wi += gridDim.x * blockDim.x) {
    const unsigned y = wi / WW, x0 = (wi - y * WW) * 32;
    const uint8_t *p = src + (size_t)y * W + x0;
    unsigned w[8];
    if (vec && x0 + 32 <= (unsigned)W) {
      const uint4 a = __ldg(reinterpret_cast<const uint4 *>(p)), b = __ldg(reinterpret_cast<const uint4 *>(p) + 1);
      w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; k++) {
        unsigned v = 0;
        for (int e = 0; e < 4; e++)
          if (x0 + 4 * k + e < (unsigned)W) v |= (unsigned)p[4 * k + e] << (8 * e);
        w[k] = v;
      }
    }
    bits[wi] = pack_bits(w);
  }
}

__device__ __forceinline__ unsigned unpack_nibble(unsigned b, int k) {  // 4 bits -> 4 bytes of 0 / 255
  return ((((b >> (4 * k)) & 0xFu) * 0x00204081u) & 0x01010101u) * 0xFFu;
}

// One 32-pixel word per lane.  When rows are whole words (W % 32 == 0) and
// the output is 16-byte aligned, a warp's 32 words are 1 KB of contiguous
// output: store j writes chunk lane + 32 j (half lane & 1 of the word of lane
// lane / 2 + 16 j, fetched by one shuffle), so each store instruction fills
// 512 contiguous bytes -- whole sectors instead of half sectors.
__global__ void bin_unpack_kernel(const uint32_t *__restrict__ bits, int W, int H,
                                  uint8_t *__restrict__ dst, int vec) {
  const unsigned WW = (unsigned)(W + 31) >> 5;
  const unsigned nw = WW * (unsigned)H;
  const int lane = threadIdx.x & 31;
  const bool lin = vec && (W & 31) == 0;
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < nw; base += stride) {
    const unsigned wi = base + lane;
    if (lin && base + 32 <= nw) {  // (warp-uniform)
      const unsigned b = bits[wi];
      uint4 *out = reinterpret_cast<uint4 *>(dst + (size_t)base * 32);
      const int h = lane & 1;
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const unsigned bs = __shfl_sync(0xffffffffu, b, (lane >> 1) + 16 * j);
        const unsigned v = h ? bs >> 16 : bs;
        out[lane + 32 * j] = make_uint4(unpack_nibble(v, 0), unpack_nibble(v, 1), unpack_nibble(v, 2),
                                        unpack_nibble(v, 3));
      }
      continue;
    }
    if (wi >= nw) continue;
    const unsigned y = wi / WW, x0 = (wi - y * WW) * 32;
    const unsigned b = bits[wi];
    unsigned w[8];
#pragma unroll
    for (int k = 0; k < 8; k++) w[k] = unpack_nibble(b, k);
    uint8_t *p = dst + (size_t)y * W + x0;
    if (vec && x0 + 32 <= (unsigned)W) {
      reinterpret_cast<uint4 *>(p)[0] = make_uint4(w[0], w[1], w[2], w[3]);
      reinterpret_cast<uint4 *>(p)[1] = make_uint4(w[4], w[5], w[6], w[7]);
    } else {
      for (unsigned x = 0; x < 32 && x0 + x < (unsigned)W; x++) p[x] = (uint8_t)(w[x >> 2] >> (8 * (x & 3)));
    }
  }
}

size_t bin_plane_words(int64_t W, int64_t H) { return (size_t)((W + 31) / 32) * (size_t)H; }

int bin_pack(const void *src, int W, int H, uint32_t *bits, cudaStream_t st, const void *src2,
             uint32_t *bits2) {
  size_t threads = bin_plane_words(W, H);
  size_t blocks = (threads + 255) / 256, cap = (size_t)device_sm_count() * (src2 ? 8 : 16);
  const int vec = W % 16 == 0 && (uintptr_t)src % 16 == 0;
  const int vec2 = W % 16 == 0 && (uintptr_t)src2 % 16 == 0;
  const dim3 grid((unsigned)(blocks < cap ? blocks : cap), src2 ? 2u : 1u);
  bin_pack_kernel<<<grid, 256, 0, st>>>((const uint8_t *)src, W, H, bits, vec, (const uint8_t *)src2,
                                        bits2, vec2);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}
int bin_unpack(const uint32_t *bits, int W, int H, void *dst, cudaStream_t st) {
  size_t threads = bin_plane_words(W, H);
  size_t blocks = (threads + 255) / 256, cap = (size_t)device_sm_count() * 16;
  const int vec = W % 16 == 0 && (uintptr_t)dst % 16 == 0;
  bin_unpack_kernel<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, st>>>(bits, W, H, (uint8_t *)dst,
                                                                             vec);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

// Initial GBQ: every tile, ordered by 2x2 colour class (then raster) so the
// first wave of concurrently running tiles are never neighbours.
__device__ __forceinline__ void tile_queue_init(const TileQueue &q, int ntx, int nty,
                                                unsigned long long *counters, int keep) {
  unsigned ntiles = (unsigned)ntx * nty;
  unsigned stride = gridDim.x * blockDim.x;
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned cx[4], cy[4], base[4];
#pragma unroll
  for (int c = 0; c < 4; c++) {
    cx[c] = (ntx - (c & 1) + 1) / 2;
    cy[c] = (nty - (c >> 1) + 1) / 2;
    base[c] = c == 0 ? 0 : base[c - 1] + cx[c - 1] * cy[c - 1];
  }
  // banded: the colour order runs band by band (B tile rows, B even), so the
  // four colour passes over a band find its boxes in L2 on a whole slide
  const unsigned B = (q.band && q.band < (unsigned)nty) ? q.band : (unsigned)nty;
  for (unsigned t = i; t < ntiles; t += stride) {
    unsigned tx = t % ntx, ty = t / ntx;
    unsigned c = (tx & 1) | ((ty & 1) << 1);
    unsigned slot;
    // (selects, not dynamic indices: the arrays stay in registers)
    unsigned bc = base[0], xc = cx[0];
#pragma unroll
    for (int k = 1; k < 4; k++)
      if (c == (unsigned)k) bc = base[k], xc = cx[k];
    if (B == (unsigned)nty) {
      slot = bc + (ty >> 1) * xc + (tx >> 1);
    } else {
      const unsigned r0 = ty / B * B, rows = min(B, (unsigned)nty - r0);
      unsigned bb = 0;
#pragma unroll
      for (int k = 0; k < 3; k++)
        if ((unsigned)k < c) bb += cx[k] * ((rows - (k >> 1) + 1) / 2);
      slot = r0 * (unsigned)ntx + bb + ((ty - r0) >> 1) * xc + (tx >> 1);
    }
    q.state[t] = ST_Q | ST_V;
    q.ring[slot] = ((unsigned long long)slot << 32) | t;
  }
  for (unsigned t = ntiles + i; t <= q.mask; t += stride) q.ring[t] = ~0ull;
  if (i == 0) {
    *q.head = 0;
    *q.tail = ntiles;
    *q.pending = ntiles;
  }
  if (!keep && i < CNT_N) counters[i] = 0;
}

__global__ void tile_queue_init_kernel(TileQueue q, int ntx, int nty, unsigned long long *counters,
                                       int keep) {
  tile_queue_init(q, ntx, nty, counters, keep);
}

// Re-activation fill for slab runs (multi-GPU waves): only the tile rows
// holding or touching a changed halo row are queued -- the first tile row
// for the top halo, the last two for the bottom one -- as first visits
// (the halo row may lie inside a tile, so full detection is needed there);
// the rest of the slab is already at its local fixed point.
__device__ __forceinline__ bool rows_sel(int ty, int nty, int top, int bottom) {
  return (top && ty == 0) || (bottom && ty >= nty - 2);
}

__global__ void tile_queue_init_rows_kernel(TileQueue q, int ntx, int nty, int top, int bottom,
                                            unsigned long long *counters) {
  unsigned ntiles = (unsigned)ntx * nty;
  unsigned stride = gridDim.x * blockDim.x;
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned nrows = 0;
  for (int ty = 0; ty < nty; ty++) {
    if (ty > 0 && ty < nty - 2) ty = nty - 2;  // only rows 0, nty-2, nty-1 can be selected
    nrows += rows_sel(ty, nty, top, bottom);
  }
  unsigned nq = (unsigned)ntx * nrows;
  for (unsigned t = i; t < ntiles; t += stride) {
    int tx = (int)(t % ntx), ty = (int)(t / ntx);
    bool sel = rows_sel(ty, nty, top, bottom);
    q.state[t] = sel ? (ST_Q | ST_V) : 0u;
    if (sel) {
      unsigned before = 0;  // selected rows above ty
      for (int r = 0; r < ty; r++) {
        if (r > 0 && r < nty - 2) r = nty - 2;
        if (r < ty) before += rows_sel(r, nty, top, bottom);
      }
      unsigned slot = before * ntx + tx;
      q.ring[slot] = ((unsigned long long)slot << 32) | t;
    }
  }
  for (unsigned t = nq + i; t <= q.mask; t += stride) q.ring[t] = ~0ull;
  if (i == 0) {
    *q.head = 0;
    *q.tail = nq;
    *q.pending = nq;
  }
  if (i < CNT_N) counters[i] = 0;
}

// INIT_CONTINUE: queue tile rows [lo, hi] (first visits, 2x2 colour order)
// after the previous run's tickets.  Single CTA: it reads the previous run's
// head/tail before publishing the new ones.  Slots are not cleared: every
// stale slot holds a tag below `base`, so no later ticket can match it
// before the ring wraps a full 2^32 tickets.
__global__ void tile_queue_continue_kernel(TileQueue q, int ntx, int lo, int hi,
                                           unsigned long long *counters, int keep) {
  __shared__ unsigned base;
  if (threadIdx.x == 0) {
    unsigned h = *q.head, t = *q.tail;
    base = (int)(h - t) > 0 ? h : t;
  }
  __syncthreads();
  const int nty = hi - lo + 1;
  const unsigned nq = (unsigned)ntx * nty;
  unsigned cx[4], cy[4], cb[4];
  for (int c = 0; c < 4; c++) {
    cx[c] = (ntx - (c & 1) + 1) / 2;
    cy[c] = (nty - (c >> 1) + 1) / 2;
    cb[c] = c == 0 ? 0 : cb[c - 1] + cx[c - 1] * cy[c - 1];
  }
  for (unsigned i = threadIdx.x; i < nq; i += blockDim.x) {
    unsigned tx = i % ntx, tyr = i / ntx;
    unsigned c = (tx & 1) | ((tyr & 1) << 1);
    unsigned pos = base + cb[c] + (tyr >> 1) * cx[c] + (tx >> 1);
    unsigned t = (unsigned)(lo + tyr) * ntx + tx;
    q.state[t] = ST_Q | ST_V;
    q.ring[pos & q.mask] = ((unsigned long long)pos << 32) | t;
  }
  if (!keep && threadIdx.x < CNT_N) counters[threadIdx.x] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    *q.head = base;
    *q.tail = base + nq;
    *q.pending = nq;
  }
}

size_t tile_queue_bytes(unsigned ntiles) {
  Carver c(nullptr);
  carve_tile_queue(c, ntiles);
  return c.off + 256;
}

TileQueue carve_tile_queue(Carver &c, unsigned ntiles) {
  unsigned cap = 1;
  // >= 2x the tiles plus the tickets waiting workers can hold, so a slot is
  // never refilled before its ticket holder has read it
  while (cap < 2 * ntiles + 65536) cap <<= 1;
  TileQueue q;
  q.state = c.take<unsigned>(ntiles);
  q.ring = c.take<unsigned long long>(cap);
  q.mask = cap - 1;
  // head, tail and pending are the engine's hottest atomics: one 256-byte
  // line each, so they do not serialise in one L2 slice
  constexpr int kCtrStride = IWPP_CTR_SPREAD ? 64 : 1;
  unsigned *ctr = c.take<unsigned>(3 * kCtrStride + 1);
  q.tmaps = c.take<unsigned char>(2 * 128);  // 256-byte aligned by the carver
  q.head = ctr;
  q.tail = ctr + kCtrStride;
  q.pending = ctr + 2 * kCtrStride;
  return q;
}

// A 2D u8 tensor map of a (H, W) image with 48 x 34 boxes (TMA staging of
// the register engine).  The encoder comes from the driver at run time (no
// link-time libcuda dependency).  Needs 16-byte aligned rows.
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool make_box_map(CUtensorMap *map, const void *base, int W, int H, int esize, int boxW,
                         int boxH = kBoxH) {
  static EncodeTiledFn encode = nullptr;
  static int tried = 0;
  if (!tried) {
    tried = 1;
    if (!getenv("IWPP_NO_TMA")) {
      void *fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        encode = (EncodeTiledFn)fn;
    }
  }
  if (!encode || ((size_t)W * esize) % 16 != 0 || (uintptr_t)base % 16 != 0) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
  const cuuint64_t strides[1] = {(cuuint64_t)W * esize};
  const cuuint32_t box[2] = {(cuuint32_t)boxW, (cuuint32_t)boxH};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = esize == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                              : CU_TENSOR_MAP_DATA_TYPE_INT32;
  return encode(map, dt, 2, const_cast<void *>(base), dims, strides, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the register engine covers u8 (and binary); the shared-memory engine stays
// for u16 / int32 / f32 and whenever its knobs are asked for (queue capacity
// for the forced-overflow path, in-tile sweep counts)
template <typename T>
static bool use_reg_engine(const EngineOpts &o) {
  if (o.engine == ENGINE_SMEM) return false;
  if (o.engine == ENGINE_REG || o.engine == ENGINE_ROUNDS) return true;
  return o.qcap <= 0 && o.sweeps_set == 0;
}

static bool use_bin_engine(bool binary, const EngineOpts &o) {
  return binary && o.engine != ENGINE_SMEM && o.engine != ENGINE_REG && o.qcap <= 0 &&
         o.sweeps_set == 0;
}

bool f32_in_engine(const EngineOpts &o) { return use_reg_engine<int32_t>(o); }

// activation trace control (IWPP_ATRACE builds only; see ATraceRec)
int atrace_control(void *buf, unsigned cap, unsigned *n_out) {
#ifdef IWPP_ATRACE
  if (buf) {
    ATraceRec *p = (ATraceRec *)buf;
    unsigned z = 0;
    if (cudaMemcpyToSymbol(g_atrace, &p, sizeof p) != cudaSuccess ||
        cudaMemcpyToSymbol(g_atrace_cap, &cap, sizeof cap) != cudaSuccess ||
        cudaMemcpyToSymbol(g_atrace_n, &z, sizeof z) != cudaSuccess)
      return IWPP_E_CUDA;
  }
  if (n_out && cudaMemcpyFromSymbol(n_out, g_atrace_n, sizeof *n_out) != cudaSuccess) return IWPP_E_CUDA;
  return (int)sizeof(ATraceRec);
#else
  (void)buf, (void)cap, (void)n_out;
  return IWPP_E_CONTRACT;
#endif
}

int tile_side(int dtype, const EngineOpts &o) {
  return use_bin_engine(dtype == IWPP_BIN, o) ? TSB : TS;
}


// the 16 / 32-bit register engine (no u8 instantiation)
template <typename T, int CONN, bool ORD>
static int launch_reg32_kernel(const EngineArgs &a, unsigned long long *counters, const TileQueue &q,
                               const void *J, const void *I, int W, int H, const EngineOpts &o,
                               unsigned max_b, int fused_init, cudaStream_t st);

template <typename T, int CONN>
static int launch_reg32(const EngineArgs &a, unsigned long long *counters, const TileQueue &q,
                        const void *J, const void *I, int W, int H, const EngineOpts &o,
                        unsigned max_b, int fused_init, cudaStream_t st, bool ord = false) {
  if constexpr (std::is_same<T, int32_t>::value) {
    if (ord) return launch_reg32_kernel<T, CONN, true>(a, counters, q, J, I, W, H, o, max_b, fused_init, st);
  }
  return launch_reg32_kernel<T, CONN, false>(a, counters, q, J, I, W, H, o, max_b, fused_init, st);
}

template <typename T, int CONN, bool ORD>
static int launch_reg32_kernel(const EngineArgs &a, unsigned long long *counters, const TileQueue &q,
                               const void *J, const void *I, int W, int H, const EngineOpts &o,
                               unsigned max_b, int fused_init, cudaStream_t st) {
  if constexpr (sizeof(T) == 1) {
    return set_error(IWPP_E_CONTRACT, "no 8-bit register32 engine");
  } else {
    static int r32_blocks = 0;
    if (r32_blocks == 0) {
      int per_sm = 0;
      IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, tile_engine_reg32_kernel<T, CONN, ORD>, kCtaThreads, 0));
      r32_blocks = device_sm_count() * (per_sm < 1 ? 1 : per_sm);
    }
    int rb = r32_blocks;
    if (o.max_blocks > 0 && rb > o.max_blocks) rb = o.max_blocks;
    if ((unsigned)rb > max_b) rb = (int)max_b;
    BoxMaps maps;
    memset(&maps, 0, sizeof maps);
    int use_tma = q.tmaps && make_box_map(&maps.m[0], J, W, H, sizeof(T), R32<T>::BW) &&
                  make_box_map(&maps.m[1], I, W, H, sizeof(T), R32<T>::BW);
    if (fused_init) {
      int fi = 1;
      void *args[] = {const_cast<EngineArgs *>(&a), &counters, &maps, &use_tma, &fi};
      IWPP_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)tile_engine_reg32_kernel<T, CONN, ORD>,
                                                dim3(rb), dim3(kCtaThreads), args, 0, st));
    } else {
      tile_engine_reg32_kernel<T, CONN, ORD><<<rb, kCtaThreads, 0, st>>>(a, counters, maps, use_tma, 0);
    }
    IWPP_CUDA_TRY(cudaGetLastError());
    return IWPP_OK;
  }
}

template <typename T, int CONN>
static int launch_engine(void *J, const void *I, int W, int H, TileQueue q,
                         unsigned long long *counters, const EngineOpts &o, cudaStream_t st,
                         bool binary = false, bool f32 = false) {
  const int ts = use_bin_engine(binary, o) ? TSB : TS;
  int ntx = (W + ts - 1) / ts, nty = (H + ts - 1) / ts;
  unsigned ntiles = (unsigned)ntx * nty;
  size_t smem = sizeof(WarpSmem<T>) * kWarpsPerCta;
  auto kern = tile_engine_kernel<T, CONN>;
  static int per_sm_cache = 0;
  if (per_sm_cache == 0) {
    IWPP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCtaThreads, smem));
    per_sm_cache = per_sm < 1 ? 1 : per_sm;
  }
  int blocks = device_sm_count() * per_sm_cache;
  if (o.max_blocks > 0 && blocks > o.max_blocks) blocks = o.max_blocks;
  unsigned max_b = (ntiles + kWarpsPerCta - 1) / kWarpsPerCta;
  if ((unsigned)blocks > max_b) blocks = (int)max_b;
  unsigned ib = (q.mask + 1 + 255) / 256;
  if (ib > 1024) ib = 1024;
  // the u8 register engine builds a full initial queue itself (cooperative
  // launch): one launch less per call
  const int fused_init = IWPP_FUSED_INIT && !use_bin_engine(binary, o) &&
                         use_reg_engine<T>(o) && o.init_mode != INIT_CONTINUE && !o.rows_mode &&
                         !o.keep_counters && ntiles >= kFusedInitMinTiles;
  // a separate marker (o.src): the fused u8 register engine (not the rounds
  // engine) copies it in its prologue; every other path copies it here
  bool src_in_kernel = o.src && fused_init && sizeof(T) == 1 && !use_bin_engine(binary, o);
  if (o.src && !src_in_kernel)
    IWPP_CUDA_TRY(cudaMemcpyAsync(J, o.src, (size_t)W * H * sizeof(T), cudaMemcpyDeviceToDevice, st));
  if (fused_init) {
    // (the engine kernel initialises the queue)
  } else if (o.init_mode == INIT_CONTINUE) {
    int lo = o.sel_lo < 0 ? 0 : o.sel_lo;
    int hi = (o.sel_hi < 0 || o.sel_hi >= nty) ? nty - 1 : o.sel_hi;
    if (lo > hi) return IWPP_OK;  // nothing to queue
    tile_queue_continue_kernel<<<1, 1024, 0, st>>>(q, ntx, lo, hi, counters, o.keep_counters);
  } else if (o.rows_mode) {
    tile_queue_init_rows_kernel<<<ib, 256, 0, st>>>(q, ntx, nty, o.rows_mode & 1,
                                                     (o.rows_mode >> 1) & 1, counters);
  } else {
    tile_queue_init_kernel<<<ib, 256, 0, st>>>(q, ntx, nty, counters, o.keep_counters);
  }
  IWPP_CUDA_TRY(cudaGetLastError());
  unsigned qlimit = (o.qcap > 0 && o.qcap < RQ) ? (unsigned)o.qcap : (unsigned)RQ;
  unsigned hth = o.halo_thresh >= 0 ? (unsigned)o.halo_thresh : kHaloSweepThreshold;
  bool vec = ((size_t)W * sizeof(T)) % 16 == 0 && (uintptr_t)J % 16 == 0 && (uintptr_t)I % 16 == 0;
  const unsigned long long ntx_m =
      (ntx < (1 << 14) && nty < (1 << 23) && ntiles < (1u << 26)) ? ((1ull << 40) + ntx - 1) / ntx
                                                                  : 0ull;
  // whole slides: colour order band by band (IWPP_BAND = tile rows per band,
  // 0 = image-wide).  Auto, when marker + mask exceed 2 x L2: the smallest
  // band whose colour classes still hold 2x the resident warps (smaller
  // bands put neighbours in flight together: re-runs), measured 64K^2 u8 c8
  // 24.9 -> 23.9 ms (band 16), 16K^2 1.55 -> 1.50 ms (band 32 ~ auto 48)
  {
    static int band_env = -2;
    if (band_env == -2) band_env = getenv("IWPP_BAND") ? atoi(getenv("IWPP_BAND")) : -1;
    const size_t img2 = (size_t)W * H * sizeof(T) * 2;
    unsigned band = 0;
    if (band_env >= 0) {
      band = (unsigned)(band_env & ~1);
    } else if (img2 > ((size_t)256 << 20) && !use_bin_engine(binary, o)) {  // (bit planes fit L2)
      const unsigned warps = (unsigned)device_sm_count() * 20u;
      band = (8u * warps + (unsigned)ntx - 1) / (unsigned)ntx;
      band = (band + 1) & ~1u;
      if (band < 8) band = 8;
    }
    q.band = band;
  }
  EngineArgs a{J, I, W, H, ntx, nty, qlimit, hth, o.sweeps, vec ? 1 : 0, o.dirty, (W + 31) / 32, q, ntx_m};
  if (o.ev_begin) IWPP_CUDA_TRY(cudaEventRecord((cudaEvent_t)o.ev_begin, st));
  if (use_bin_engine(binary, o)) {
    // TMA boxes when the plane's rows are 16-byte multiples (W % 128 == 0)
    BoxMaps maps;
    const int WW = (W + 31) / 32;
    int use_tma = (WW % 4 == 0) && !getenv("IWPP_BIN_NO_TMA") &&
                  make_box_map(&maps.m[0], J, WW, H, 4, kBinBoxW, kBinBoxH) &&
                  make_box_map(&maps.m[1], I, WW, H, 4, kBinBoxW, kBinBoxH);
    const size_t dsm = use_tma ? kWarpsPerCta * sizeof(BinBoxSmem) : 0;
    static int bin_blocks = 0;
    if (bin_blocks == 0) {
      int per_sm = 0;
      IWPP_CUDA_TRY(cudaFuncSetAttribute(tile_engine_bin_kernel<CONN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kWarpsPerCta * sizeof(BinBoxSmem))));
      IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_engine_bin_kernel<CONN>,
                                                                  kCtaThreads, kWarpsPerCta * sizeof(BinBoxSmem)));
      // more resident warps than this only adds idle pollers on the tile
      // ring (binary fills are narrow fronts): measured best at 4 CTAs/SM
      int cap = kBinCtasPerSm;
      if (const char *e = getenv("IWPP_BIN_CTAS")) cap = atoi(e);
      if (per_sm > cap) per_sm = cap;
      bin_blocks = device_sm_count() * (per_sm < 1 ? 1 : per_sm);
    }
    int bb = bin_blocks;
    if (o.max_blocks > 0 && bb > o.max_blocks) bb = o.max_blocks;
    if ((unsigned)bb > max_b) bb = (int)max_b;
    tile_engine_bin_kernel<CONN><<<bb, kCtaThreads, dsm, st>>>(a, counters, maps, use_tma);
  } else if (sizeof(T) > 1 && use_reg_engine<T>(o)) {  // 16 / 32-bit register engine
    const int rc = launch_reg32<T, CONN>(a, counters, q, J, I, W, H, o, max_b, fused_init, st, f32);
    if (rc) return rc;
  } else if (use_reg_engine<T>(o)) {
    static int reg_blocks = 0;
    if (reg_blocks == 0) {
      int per_sm = 0;
      IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tile_engine_reg_kernel<CONN>,
                                                                  kCtaThreads, 0));
      reg_blocks = device_sm_count() * (per_sm < 1 ? 1 : per_sm);
    }
    int rb = reg_blocks;
    if (o.max_blocks > 0 && rb > o.max_blocks) rb = o.max_blocks;
    if ((unsigned)rb > max_b) rb = (int)max_b;
    BoxMaps maps;
    memset(&maps, 0, sizeof maps);
    int use_tma = vec && q.tmaps && make_box_map(&maps.m[0], J, W, H, 1, kBoxW) &&
                  make_box_map(&maps.m[1], I, W, H, 1, kBoxW);
    if (getenv("IWPP_TRACE")) fprintf(stderr, "[iwpp] reg engine %dx%d use_tma=%d vec=%d fused=%d\n", W, H, use_tma, (int)vec, fused_init);
    // level-synchronous rounds: a plain full run (no slab rows, no pipelined
    // continuation, no dirty flags) with TMA staging
    static int rounds_env = -1;
    // (AUTO keeps the queue engine: measured 0.125 vs 0.130-0.137 ms at 4K^2
    // u8 c8, 26.7 vs 28.5 ms at 64K^2; IWPP_RECON_ROUNDS=1 makes AUTO pick
    // the rounds engine)
    if (rounds_env < 0) rounds_env = getenv("IWPP_RECON_ROUNDS") ? atoi(getenv("IWPP_RECON_ROUNDS")) : 0;
    const bool rounds = use_tma && ntx_m && o.init_mode != INIT_CONTINUE && !o.rows_mode && !o.dirty &&
                        (o.engine == ENGINE_ROUNDS || (o.engine == ENGINE_AUTO && rounds_env));
    if (src_in_kernel && rounds) {  // (the rounds engine has no marker prologue)
      IWPP_CUDA_TRY(cudaMemcpyAsync(J, o.src, (size_t)W * H, cudaMemcpyDeviceToDevice, st));
      src_in_kernel = false;
    }
    const void *msrc = src_in_kernel ? o.src : nullptr;
    if (rounds) {
      static int rd_per_sm = 0;
      if (rd_per_sm == 0) {
        IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rd_per_sm, tile_rounds_reg_kernel<CONN>,
                                                                    kCtaThreads, 0));
        if (rd_per_sm < 1) rd_per_sm = 1;
      }
      int nb = device_sm_count() * rd_per_sm;
      if (o.max_blocks > 0 && nb > o.max_blocks) nb = o.max_blocks;
      if ((unsigned)nb > max_b) nb = (int)max_b;
      RoundsArgs ra;
      unsigned *w32 = reinterpret_cast<unsigned *>(q.ring);  // the ring is free in this mode
      const size_t nwd = (ntiles + 31) / 32;
      ra.len = w32;                      // [0, 3): lengths; [3, 3 + rounds): trace
      ra.bar_count = w32 + 40 * kLenStride;
      ra.bar_gen = w32 + 41 * kLenStride;
      ra.bm0 = w32 + 42 * kLenStride;
      ra.bm1 = ra.bm0 + (nwd + 63) / 64 * 64;
      ra.list0 = ra.bm1 + (nwd + 63) / 64 * 64;
      ra.list1 = ra.list0 + (ntiles + 63) / 64 * 64;
      int kc = o.keep_counters ? 1 : 0;
      static int rtrace = getenv("IWPP_RECON_RTRACE") ? 1 : 0;
      int mr = o.max_rounds;
      void *args[] = {&a, &ra, &counters, &maps, &kc, &rtrace, &mr};
      IWPP_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)tile_rounds_reg_kernel<CONN>, dim3(nb),
                                                dim3(kCtaThreads), args, 0, st));
      if (rtrace) {  // diagnostics: per-round end times (IWPP_RECON_RTRACE)
        std::vector<unsigned> tr(40 * kLenStride);
        IWPP_CUDA_TRY(cudaMemcpyAsync(tr.data(), ra.len, tr.size() * 4, cudaMemcpyDeviceToHost, st));
        IWPP_CUDA_TRY(cudaStreamSynchronize(st));
        for (int k = 0; k < 37 && tr[(3 + k) * kLenStride]; k++)
          fprintf(stderr, "[rounds] round %d ends at %.2f us\n", k, tr[(3 + k) * kLenStride] * 1e-3);
        IWPP_CUDA_TRY(cudaMemsetAsync(ra.len, 0, 40 * kLenStride * 4, st));
      }
    } else if (fused_init) {
      int fi = fused_init;
      void *args[] = {&a, &counters, &maps, &use_tma, &fi, &msrc};
      IWPP_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)tile_engine_reg_kernel<CONN>, dim3(rb),
                                                dim3(kCtaThreads), args, 0, st));
    } else {
      tile_engine_reg_kernel<CONN><<<rb, kCtaThreads, 0, st>>>(a, counters, maps, use_tma, 0, nullptr);
    }
  } else {
    kern<<<blocks, kCtaThreads, smem, st>>>(a, counters);
  }
  IWPP_CUDA_TRY(cudaGetLastError());
  if (o.ev_end) IWPP_CUDA_TRY(cudaEventRecord((cudaEvent_t)o.ev_end, st));
  return IWPP_OK;
}

int run_tile_engine(void *J, const void *I, int W, int H, int dtype, int conn, TileQueue q,
                    unsigned long long *counters, const EngineOpts &o, cudaStream_t st) {
#define DISPATCH(T)                                                        \
  return conn == 8 ? launch_engine<T, 8>(J, I, W, H, q, counters, o, st) \
                   : launch_engine<T, 4>(J, I, W, H, q, counters, o, st)
  switch (dtype) {
    case IWPP_BIN:
      return conn == 8 ? launch_engine<uint8_t, 8>(J, I, W, H, q, counters, o, st, true)
                       : launch_engine<uint8_t, 4>(J, I, W, H, q, counters, o, st, true);
    case IWPP_U8:
      DISPATCH(uint8_t);
    case IWPP_U16:
      DISPATCH(uint16_t);
    case IWPP_I32:
      DISPATCH(int32_t);
    case IWPP_F32:  // f32 bit patterns, ordered inside the 32-bit register engine
      if (!f32_in_engine(o)) break;
      return conn == 8 ? launch_engine<int32_t, 8>(J, I, W, H, q, counters, o, st, false, true)
                       : launch_engine<int32_t, 4>(J, I, W, H, q, counters, o, st, false, true);
  }
#undef DISPATCH
  return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
}

}  // namespace recon
}  // namespace iwpp
