// recon_tiles.cuh -- tile engine interface (see recon_tiles.cu).
#pragma once
#include "iwpp_common.cuh"

namespace iwpp {
namespace recon {

// One warp owns one TS x TS tile at a time (plus a 1-pixel halo).
constexpr int TS = 32;                   // tile side
constexpr int TSB = 128;                 // the binary engine's tile side (the largest)
constexpr int PW = TS + 2;               // logical tile side with the halo
constexpr int PS = PW + 1;               // shared-memory row stride (odd: conflict-free)
constexpr int PN = PW * PW;              // logical cells
constexpr int PNS = PW * PS;             // shared-memory cells
constexpr int RQ = 2048;                 // per-warp pixel ring (>= PN: a full rescan fits)
constexpr int BITW = (PNS + 31) / 32;    // in-queue bitmap words
constexpr int kWarpsPerCta = 4;
constexpr int kCtaThreads = 32 * kWarpsPerCta;
constexpr int kCtaMinBlocks = 5;  // resident CTAs per SM (shared memory allows 5 for u8)
#ifndef IWPP_REG_MIN_BLOCKS
#define IWPP_REG_MIN_BLOCKS 5
#endif
#ifndef IWPP_REG32_MIN_BLOCKS
#define IWPP_REG32_MIN_BLOCKS 4
#endif
// register engines: registers are the limit (u8 / binary; 16/32-bit kinds)
constexpr int kRegCtaMinBlocks = IWPP_REG_MIN_BLOCKS;
constexpr int kReg32CtaMinBlocks = IWPP_REG32_MIN_BLOCKS;

// Per-phase clock counters (pop / load / sweep / ... ; CNT_PH_*) cost
// registers in the engines: compiled in only with -DIWPP_PHASES.
#ifdef IWPP_PHASES
constexpr bool kPhases = true;
#else
constexpr bool kPhases = false;
#endif
__device__ __forceinline__ long long pclock(bool l0) { return (kPhases && l0) ? clock64() : 0; }
static_assert(RQ >= PN && (RQ & (RQ - 1)) == 0, "ring must hold a full rescan");
static_assert(PNS < 65536, "queue entries are 16-bit");

// re-activations whose halo front is wider than this sweep before queueing
constexpr unsigned kHaloSweepThreshold = 16;

// device counters (workspace)
enum {
  CNT_TILES = 0, CNT_RERUNS, CNT_PUSHES, CNT_OVERFLOW, CNT_SEEDS, CNT_VIOL,
  CNT_STEPS,  // register engine: Jacobi steps summed over tile activations
  CNT_ROUNDS, // round engine: rounds of the last run
  // per-phase SM cycles summed over warps (lane 0's clock; diagnostics)
  CNT_PH_POP = 8, CNT_PH_LOAD, CNT_PH_SWEEP, CNT_PH_DETECT, CNT_PH_BFS, CNT_PH_STORE,
  CNT_LIMIT = 14,  // round engine: stopped at max_rounds with work left
  CNT_IDLE_POLLS = 15,  // register engine: ring polls that found their slot empty
  CNT_N = 16
};

struct TileQueue {
  unsigned *state;           // per-tile state bits (recon_tiles.cu: Q, R, V)
  unsigned long long *ring;  // (pos << 32) | tile
  unsigned mask;             // ring capacity - 1
  unsigned band = 0;         // initial queue order: 2x2 colour order within bands of this
                             // many tile rows (even; 0 = over the whole image).  (It sits in
                             // the padding after `mask`: a larger struct shifts the engines'
                             // kernel parameters and measurably changed their code.)
  unsigned *head, *tail, *pending;
  void *tmaps;               // 2 TMA descriptors (register engine), in device memory
};

struct EngineOpts {
  int max_blocks = 0;    // persistent grid cap in CTAs (0 = all resident)
  int qcap = 0;          // per-warp pixel-queue capacity (0 = RQ)
  int sweeps = 1;        // in-tile sweep passes on a tile's first visit
  int halo_thresh = -1;  // re-activation front that triggers sweeps (-1 = default)
  void *ev_begin = nullptr, *ev_end = nullptr;  // cudaEvent_t around the engine kernel
  int rows_mode = 0;     // 0: every tile, first visit; bit0 / bit1: only the top / bottom
                         // tile row, as re-visits (slab waves after a halo exchange)
  // Queue initialisation.  INIT_FULL resets the ring (clears every slot) and
  // queues every tile.  INIT_CONTINUE keeps the ring's ticket sequence of the
  // previous run on this workspace (no clearing: stale slots carry older
  // tags) and queues tile rows [sel_lo, sel_hi] as first visits; every other
  // tile must be idle (it is after any completed run).
  int init_mode = 0;
  int sel_lo = 0, sel_hi = -1;  // INIT_CONTINUE: tile-row range (-1 = last row)
  uint8_t *dirty = nullptr;     // optional: set to 1 for each tile row the run wrote
  bool keep_counters = false;   // accumulate into the device counters (no reset)
  int engine = 0;               // ENGINE_AUTO / ENGINE_SMEM / ENGINE_REG / ENGINE_ROUNDS
  int sweeps_set = 0;           // the caller fixed the in-tile sweep count
  int max_rounds = 0;           // round engine: > 0 caps the rounds (CNT_LIMIT)
  const void *src = nullptr;    // marker to copy into J first (the fused u8 engine
                                // copies it in its prologue)
};
// ENGINE_REG: the register engine on the tile queue; ENGINE_ROUNDS: the
// register engine in level-synchronous tile rounds (u8; AUTO picks it when
// it applies)
enum { ENGINE_AUTO = 0, ENGINE_SMEM = 1, ENGINE_REG = 2, ENGINE_ROUNDS = 3 };
enum { INIT_FULL = 0, INIT_CONTINUE = 1 };

size_t tile_queue_bytes(unsigned ntiles);
TileQueue carve_tile_queue(Carver &c, unsigned ntiles);
// f32 images can run on their float bits directly (the register engine
// orders them as it stages its boxes) under these options
bool f32_in_engine(const EngineOpts &o);
int run_tile_engine(void *J, const void *I, int W, int H, int dtype, int conn, TileQueue q,
                    unsigned long long *counters, const EngineOpts &o, cudaStream_t st);
// side of the square tiles the engine run_tile_engine picks for (dtype, o)
// works on: sel_lo / sel_hi and the dirty flags count rows of these tiles
int tile_side(int dtype, const EngineOpts &o);
// activation trace (development builds with -DIWPP_ATRACE; else IWPP_E_CONTRACT)
int atrace_control(void *buf, unsigned cap, unsigned *n_out);
// binary kind: J / I as bit planes (ceil(W/32) words per row) for the engine
size_t bin_plane_words(int64_t W, int64_t H);
// (src2 / bits2: a second plane packed by the same launch)
int bin_pack(const void *src, int W, int H, uint32_t *bits, cudaStream_t st,
             const void *src2 = nullptr, uint32_t *bits2 = nullptr);
int bin_unpack(const uint32_t *bits, int W, int H, void *dst, cudaStream_t st);

inline unsigned num_tiles(int64_t W, int64_t H) {
  return (unsigned)(((W + TS - 1) / TS) * ((H + TS - 1) / TS));
}

}  // namespace recon
}  // namespace iwpp
