// recon_tiles.cuh -- tile engine interface (see recon_tiles.cu).
#pragma once
#include "iwpp_common.cuh"

namespace iwpp {
namespace recon {

constexpr int TW = 64, TH = 64;         // tile interior
constexpr int PW = TW + 2, PH = TH + 2; // with a 1-pixel halo
constexpr int PN = PW * PH;
constexpr int QCAP = 4608;              // >= PN so a full rescan always fits
constexpr int kTileThreads = 256;
static_assert(TW == TH, "border ring indexing assumes square tiles");
static_assert(QCAP >= PN, "rescan must fit the block queue");

// device counters (workspace)
enum { CNT_TILES = 0, CNT_RERUNS, CNT_PUSHES, CNT_OVERFLOW, CNT_SEEDS, CNT_VIOL, CNT_N = 8 };

struct TileQueue {
  unsigned *state;          // per-tile state
  unsigned long long *ring; // (pos << 32) | tile
  unsigned mask;            // ring capacity - 1
  unsigned *head, *tail, *pending;
};

size_t tile_queue_bytes(unsigned ntiles);
TileQueue carve_tile_queue(Carver &c, unsigned ntiles);
int run_tile_engine(void *J, const void *I, int W, int H, int dtype, int conn, TileQueue q,
                    unsigned long long *counters, int max_blocks, int qcap, cudaStream_t st);

inline unsigned num_tiles(int64_t W, int64_t H) {
  return (unsigned)(((W + TW - 1) / TW) * ((H + TH - 1) / TH));
}

}  // namespace recon
}  // namespace iwpp
