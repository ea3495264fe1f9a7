// edt.cu -- level-synchronous wavefront EDT for sm_100a.
//
// Reference: edt.py:187-294 and the kernels K.309-433.  The reference pins
// ONE canonical schedule: two-phase rounds where every offer in
// round r uses the source its sender held at the start of round r, and a
// target adopts a candidate iff it is closer, or equally close with a
// smaller packed index (closer_source, K.320-336).  The end-of-round state is
// then the per-cell minimum of {start value, offers} under that total order,
// which is what this engine computes -- bit-identical to the reference.
//
// Design (B200):
//  * state: source per cell as a 32-bit (sy << 16 | sx) code.  Lexicographic
//    (y, x) order equals packed-index order, so the index tie-break is a
//    plain unsigned compare and no divisions are needed.  INF = 0xFFFFFFFF.
//  * double-buffered state (RD = start of round, WR = being built): one grid
//    barrier per round instead of two.  WR lags RD exactly on the current
//    frontier, which each frontier item re-syncs before offering.
//  * offers: read RD[q] (plain load); only an offer that beats the
//    round-start value does a CAS-min on WR[q] and claims q for the next
//    frontier through a per-cell round stamp (dedupe), pushed with
//    warp-aggregated reservations into the global frontier queue.
//  * one persistent cooperative kernel runs all rounds with a device-side
//    grid barrier (no host round trips); the frontier-size counters are
//    triple-buffered so no block can reset a counter another still reads.
//  * finalize fused: packed int64 vr and float32(sqrt(float64(d2)))
//    (edt.py:278-280 -- __dsqrt_rn then RN to float), INF count for
//    NoBackgroundError.

#include <stdio.h>
#include <stdlib.h>
#include "edt.cuh"

namespace iwpp {
namespace edt {

__device__ __forceinline__ long long sqd_yx(int qx, int qy, uint32_t s) {
  int sy = (int)(s >> 16), sx = (int)(s & 0xffffu);
  long long dx = qx - sx, dy = qy - sy;
  return dx * dx + dy * dy;
}

// K.320-336 closer_source on yx codes
__device__ __forceinline__ bool closer(int qx, int qy, uint32_t cand, uint32_t held) {
  if (held == INF32) return cand != INF32;
  if (cand == INF32) return false;
  long long dc = sqd_yx(qx, qy, cand), dh = sqd_yx(qx, qy, held);
  if (dc != dh) return dc < dh;
  return cand < held;
}

// WR[q] <- min(WR[q], cand) in the order at q
__device__ __forceinline__ void cas_min(uint32_t *WR, size_t q, int qx, int qy, uint32_t cand) {
  uint32_t old = __ldcg(WR + q);
  while (closer(qx, qy, cand, old)) {
    uint32_t prev = atomicCAS(WR + q, old, cand);
    if (prev == old) return;
    old = prev;
  }
}

// ---- init: fused assign (K.339-348) + contour seeds (K.351-373) -----------
template <int CONN>
__global__ void edt_init_kernel(const uint8_t *__restrict__ mask, int W, int H, EdtState s) {
  const unsigned FULL = 0xffffffffu;
  size_t n = (size_t)W * H;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n;
       base += stride) {
    size_t p = base + (threadIdx.x & 31u);
    bool push = false;
    uint32_t yx = 0;
    if (p < n) {
      int py = (int)(p / (unsigned)W), px = (int)(p - (size_t)py * W);
      yx = ((uint32_t)py << 16) | (uint32_t)px;
      bool bg = mask[p] == 0;
      uint32_t v = bg ? yx : INF32;
      s.buf[0][p] = v;
      s.buf[1][p] = v;
      s.stamp[p] = 0;
      if (bg) {
#pragma unroll
        for (int k = 0; k < Nbr<CONN>::N; k++) {
          int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
          if (qx >= 0 && qx < W && qy >= 0 && qy < H && mask[(size_t)qy * W + qx] != 0) push = true;
        }
      }
    }
    unsigned pos = warp_reserve(&s.cnt[0], push ? 1u : 0u, FULL);
    if (push) s.F[0][pos] = yx;
  }
}

// ---- import a user source map + seeds (edt_propagate) ----------------------
__global__ void edt_import_kernel(const int64_t *__restrict__ vr, int W, int H, EdtState s) {
  size_t n = (size_t)W * H;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    int64_t v = vr[p];
    uint32_t c;
    if (v < 0) {
      c = INF32;
    } else if (v >= (int64_t)n) {
      c = INF32;
      atomicAdd(&s.counters[EC_BAD], 1ull);
    } else {
      int sy = (int)(v / W), sx = (int)(v - (int64_t)sy * W);
      c = ((uint32_t)sy << 16) | (uint32_t)sx;
    }
    s.buf[0][p] = c;
    s.buf[1][p] = c;
    s.stamp[p] = 0;
  }
}

__global__ void edt_seed_kernel(const int64_t *__restrict__ seeds, int64_t n_seeds, int W, int H,
                                EdtState s) {
  const unsigned FULL = 0xffffffffu;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n_seeds;
       base += stride) {
    int64_t i = base + (threadIdx.x & 31u);
    bool push = false;
    uint32_t yx = 0;
    if (i < n_seeds) {
      int64_t p = seeds[i];
      if (p < 0 || p >= (int64_t)W * H) {
        atomicAdd(&s.counters[EC_BAD], 1ull);
      } else {
        int py = (int)(p / W), px = (int)(p - (int64_t)py * W);
        yx = ((uint32_t)py << 16) | (uint32_t)px;
        push = atomicExch(&s.stamp[p], SEED_STAMP) != SEED_STAMP;
      }
    }
    unsigned pos = warp_reserve(&s.cnt[0], push ? 1u : 0u, FULL);
    if (push) s.F[0][pos] = yx;
  }
}

// ---- the round engine ------------------------------------------------------
template <int CONN>
__global__ void __launch_bounds__(kRoundThreads) edt_rounds_kernel(int W, int H, EdtState s,
                                                                   long long max_rounds) {
  unsigned bar_g = grid_barrier_gen(&s.bar[kBarGen]);
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u;
  unsigned long long visits = 0;
  int r = 0;
  for (;; r++) {
    unsigned n = ld_acquire(&s.cnt[r % 3]);
    if (n == 0) break;
    if (max_rounds >= 0 && r >= max_rounds) {
      if (blockIdx.x == 0 && threadIdx.x == 0) s.counters[EC_LIMIT] = 1;
      break;
    }
    const uint32_t *RD = s.buf[r & 1];
    uint32_t *WR = s.buf[(r + 1) & 1];
    const uint32_t *cur = s.F[r & 1];
    uint32_t *nxt = s.F[(r + 1) & 1];
    unsigned *ncnt = &s.cnt[(r + 1) % 3];
    const uint32_t stamp_r = (uint32_t)r + 1u;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s.cnt[(r + 2) % 3] = 0;
      visits += n;
    }
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
      unsigned i = base + lane;
      unsigned mask = 0;
      int px = 0, py = 0;
      if (i < n) {
        uint32_t pyx = __ldcg(cur + i);
        py = (int)(pyx >> 16);
        px = (int)(pyx & 0xffffu);
        size_t p = (size_t)py * W + px;
        uint32_t src = __ldcg(RD + p);
        cas_min(WR, p, px, py, src);  // WR lags RD on the frontier
        if (src != INF32) {
#pragma unroll
          for (int k = 0; k < Nbr<CONN>::N; k++) {
            int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
            if (qx >= 0 && qx < W && qy >= 0 && qy < H) {
              size_t q = (size_t)qy * W + qx;
              uint32_t held = __ldcg(RD + q);
              if (closer(qx, qy, src, held)) {
                cas_min(WR, q, qx, qy, src);
                if (__ldcg(s.stamp + q) != stamp_r && atomicExch(s.stamp + q, stamp_r) != stamp_r)
                  mask |= 1u << k;
              }
            }
          }
        }
      }
      unsigned c = __popc(mask);
      unsigned pos = warp_reserve(ncnt, c, FULL);
      while (mask) {
        int k = __ffs(mask) - 1;
        mask &= mask - 1;
        int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
        nxt[pos++] = ((uint32_t)qy << 16) | (uint32_t)qx;
      }
    }
    grid_barrier(&s.bar[0], &s.bar[kBarGen], gridDim.x, bar_g);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s.counters[EC_ROUNDS] = (unsigned long long)r;
    s.counters[EC_VISITS] = visits;
    s.counters[EC_FINAL] = (unsigned long long)(r & 1);
  }
}

// ---- finalize (edt.py:272-281) --------------------------------------------

// finalize directly from an int64 source map (iwpp_edt_finalize)
__global__ void edt_finalize_vr_kernel(const int64_t *__restrict__ vr, int W, int H,
                                       float *__restrict__ dist, int64_t *__restrict__ d2out,
                                       unsigned long long *counters) {
  size_t n = (size_t)W * H;
  unsigned long long ninf = 0;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    int64_t s = vr[p];
    if (s < 0) {
      ninf++;
      if (dist) dist[p] = 0.f;
      if (d2out) d2out[p] = (int64_t)1 << 62;
      continue;
    }
    int64_t py = (int64_t)(p / (unsigned)W), px = (int64_t)p - py * W;
    int64_t sy = s / W, sx = s - sy * W;
    long long dx = px - sx, dy = py - sy, d2 = dx * dx + dy * dy;
    if (dist) dist[p] = __double2float_rn(__dsqrt_rn((double)d2));
    if (d2out) d2out[p] = d2;
  }
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 16);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 8);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 4);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 2);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 1);
  if ((threadIdx.x & 31) == 0 && ninf) atomicAdd(&counters[EC_NINF], ninf);
}

// Key layout: the two key buffers of a cell (round start / being built)
// either interleaved (16 B per cell: one sector holds both; the queue
// engine's resync and read then share a sector) or as two planes (a warp's
// neighbour-key reads -- the raster rounds' main traffic -- then use every
// byte of the sectors they fetch).  IWPP_KEY_PLANAR selects; one switch for
// every key kernel (init, import, rounds, finalize).
#ifndef IWPP_KEY_PLANAR
#define IWPP_KEY_PLANAR 1
#endif
__device__ __forceinline__ unsigned long long *kslot(unsigned long long *K, size_t p, int b, size_t n) {
#if IWPP_KEY_PLANAR
  return K + (size_t)b * n + p;
#else
  (void)n;
  return K + 2 * p + b;
#endif
}
__device__ __forceinline__ void kput2(unsigned long long *K, size_t p, size_t n, unsigned long long k) {
#if IWPP_KEY_PLANAR
  K[p] = k;
  K[n + p] = k;
#else
  (void)n;
  reinterpret_cast<ulonglong2 *>(K)[p] = make_ulonglong2(k, k);
#endif
}

// ===========================================================================
// Key engine (default whenever every d^2 fits 32 bits, i.e. up to ~46K^2).
//
// Each cell holds key = (d2(cell, src) << 32) | src_yx; the reference's total
// order (K.320-336: closer, then smaller packed index; INF loses) is then
// the plain unsigned order of keys (INF = all ones), so an offer is one
// 64-bit atomicMin -- no CAS loop.  Keys are double-buffered and
// interleaved per cell (16 B: the round-start key and the key being built
// share a sector).  Next-frontier dedupe needs no stamp array: q is pushed
// by the one offer whose atomicMin moves the building key from >= q's
// round-start key to < it (values only decrease), which is exactly one
// push per changed cell.
// ===========================================================================


template <int CONN>
__global__ void edt_init_key_kernel(const uint8_t *__restrict__ mask, int W, int H, EdtState s) {
  const unsigned FULL = 0xffffffffu;
  size_t n = (size_t)W * H;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t base = (size_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n;
       base += stride) {
    size_t p = base + (threadIdx.x & 31u);
    bool push = false;
    uint32_t yx = 0;
    if (p < n) {
      int py = (int)(p / (unsigned)W), px = (int)(p - (size_t)py * W);
      yx = ((uint32_t)py << 16) | (uint32_t)px;
      bool bg = mask[p] == 0;
      unsigned long long k = bg ? (unsigned long long)yx : KINF;  // d2 = 0 for itself
      kput2(s.keys, p, (size_t)W * H, k);
      if (bg) {
#pragma unroll
        for (int k8 = 0; k8 < Nbr<CONN>::N; k8++) {
          int qx = px + Nbr<CONN>::dx(k8), qy = py + Nbr<CONN>::dy(k8);
          if (qx >= 0 && qx < W && qy >= 0 && qy < H && mask[(size_t)qy * W + qx] != 0) push = true;
        }
      }
    }
    unsigned pos = warp_reserve(&s.cnt[0], push ? 1u : 0u, FULL);
    if (push) s.F[0][pos] = yx;
  }
}

// The same init, restructured for whole-slide sizes (the per-cell version
// spent 105 ms of a 64K^2 EDT: one division per cell and, above all, one
// global atomic per warp on the seed counter -- ~10^8 atomics on one
// address when 8% of the cells are contour seeds).  A warp takes a
// 128-pixel row segment (lane + 32 j, j < 4: every key store instruction
// writes 32 consecutive cells, 512 contiguous bytes), reads the three mask
// rows once (neighbours by shuffle, the two edge bytes by lanes 0 / 31) and
// stages its seeds in a per-warp shared-memory buffer that is flushed with
// one global atomic per ~384 seeds.
// ROUND0 (the raster engine's init): round 0 is computed here as well.  Its
// frontier is exactly the contour seeds, whose sources are themselves, so
// round 0 gives every foreground cell next to the background the best of its
// background neighbours -- (d2 = 1, then 2 for 8-conn; the smaller packed
// index on ties: up, left, right, down; up-left, up-right, down-left,
// down-right) -- and leaves everything else unchanged; its next frontier is
// those foreground cells.  Both key planes get the post-round-0 keys and the
// list goes to F[1] / cnt[1]: the rounds start at r = 1 (K.403-433 rounds and
// counts unchanged: round 0's frontier size is added to the visits).  The
// rounds' biggest frontier -- 8% of a nuclei slide -- never becomes a list.
constexpr int kInitWarps = 8, kInitBuf = 512;
constexpr unsigned kOff = 0x100u;  // a mask sample outside the image
template <int CONN, bool ROUND0 = false>
__global__ void __launch_bounds__(32 * kInitWarps) edt_init_key_rows_kernel(const uint8_t *__restrict__ mask,
                                                                            int W, int H, EdtState s) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  __shared__ uint32_t buf[kInitWarps][kInitBuf];
  unsigned nbuf = 0;  // warp-uniform
  unsigned long long nseed = 0;  // (ROUND0) round 0's frontier, lane 0's count
  const int li = ROUND0 ? 1 : 0;  // the list the rounds start from
  const long long segs_per_row = (W + 127) / 128;
  const long long nseg = segs_per_row * H;
  auto flush = [&]() {
    unsigned base = 0;
    if (lane == 0 && nbuf) base = atomicAdd(&s.cnt[li], nbuf);
    base = __shfl_sync(FULL, base, 0);
    for (unsigned i = lane; i < nbuf; i += 32) s.F[li][base + i] = buf[wib][i];
    __syncwarp();
    nbuf = 0;
  };
  for (long long g = (long long)blockIdx.x * kInitWarps + wib; g < nseg; g += (long long)gridDim.x * kInitWarps) {
    const int y = (int)(g / segs_per_row);
    const int x0 = (int)(g - (long long)y * segs_per_row) * 128;
    // rows y-1, y, y+1: 4 bytes per lane (x0 + lane + 32 j) + the edge bytes;
    // outside the image: 0 = background, never a foreground neighbour
    unsigned v[3][4], eL[3], eR[3];
#pragma unroll
    for (int rr = 0; rr < 3; rr++) {
      const int yy = y + rr - 1;
      const bool rin = yy >= 0 && yy < H;
      const uint8_t *row = mask + (size_t)(rin ? yy : 0) * W;
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int x = x0 + lane + 32 * j;
        v[rr][j] = (rin && x < W) ? (unsigned)__ldg(row + x) : kOff;
      }
      eL[rr] = (rin && lane == 0 && x0 > 0) ? (unsigned)__ldg(row + x0 - 1) : kOff;
      eR[rr] = (rin && lane == 31 && x0 + 128 < W) ? (unsigned)__ldg(row + x0 + 128) : kOff;
      eL[rr] = __shfl_sync(FULL, eL[rr], 0);
      eR[rr] = __shfl_sync(FULL, eR[rr], 31);
    }
    unsigned seeds = 0;  // bit j: pixel j of this lane is a contour seed
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int x = x0 + lane + 32 * j;
      unsigned l[3], r[3];
#pragma unroll
      for (int rr = 0; rr < 3; rr++) {
        const unsigned up = __shfl_up_sync(FULL, v[rr][j], 1), dn = __shfl_down_sync(FULL, v[rr][j], 1);
        const unsigned prevw = __shfl_sync(FULL, v[rr][j > 0 ? j - 1 : 0], 31);
        const unsigned nextw = __shfl_sync(FULL, v[rr][j < 3 ? j + 1 : 3], 0);
        l[rr] = lane > 0 ? up : (j > 0 ? prevw : eL[rr]);
        r[rr] = lane < 31 ? dn : (j < 3 ? nextw : eR[rr]);
      }
      if (x >= W) continue;
      const bool bg = v[1][j] == 0;
      // foreground = a nonzero sample inside the image (off-image: kOff)
      auto fg = [](unsigned a) { return (a & 0xffu) != 0u; };
      const bool near = CONN == 8 ? (fg(l[0]) || fg(v[0][j]) || fg(r[0]) || fg(l[1]) || fg(r[1]) ||
                                     fg(l[2]) || fg(v[2][j]) || fg(r[2]))
                                  : (fg(v[0][j]) || fg(l[1]) || fg(r[1]) || fg(v[2][j]));
      const uint32_t yx = ((uint32_t)y << 16) | (uint32_t)x;
      unsigned long long k = bg ? (unsigned long long)yx : KINF;
      if (ROUND0) {
        if (bg && near) nseed += 1;
        if (!bg) {  // round 0's offers from the background neighbours
          const uint32_t yu = (uint32_t)(y - 1) << 16, yc = (uint32_t)y << 16, yd = (uint32_t)(y + 1) << 16;
          if (v[0][j] == 0) k = (1ull << 32) | (yu | (uint32_t)x);
          else if (l[1] == 0) k = (1ull << 32) | (yc | (uint32_t)(x - 1));
          else if (r[1] == 0) k = (1ull << 32) | (yc | (uint32_t)(x + 1));
          else if (v[2][j] == 0) k = (1ull << 32) | (yd | (uint32_t)x);
          else if (CONN == 8) {
            if (l[0] == 0) k = (2ull << 32) | (yu | (uint32_t)(x - 1));
            else if (r[0] == 0) k = (2ull << 32) | (yu | (uint32_t)(x + 1));
            else if (l[2] == 0) k = (2ull << 32) | (yd | (uint32_t)(x - 1));
            else if (r[2] == 0) k = (2ull << 32) | (yd | (uint32_t)(x + 1));
          }
          if (k != KINF) seeds |= 1u << j;  // changed in round 0: round 1's frontier
        }
      } else if (bg && near) {
        seeds |= 1u << j;
      }
      kput2(s.keys, (size_t)y * W + x, (size_t)W * H, k);
    }
    // stage the seeds (warp-aggregated), flush before the buffer can overflow
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const bool p = (seeds >> j) & 1u;
      const unsigned bal = __ballot_sync(FULL, p);
      if (p) buf[wib][nbuf + __popc(bal & lanemask_lt())] = ((uint32_t)y << 16) | (uint32_t)(x0 + lane + 32 * j);
      nbuf += __popc(bal);
    }
    __syncwarp();
    if (nbuf > kInitBuf - 128) flush();
  }
  flush();
  if (ROUND0) {  // round 0's frontier size joins the visits (queued_total)
    for (int o = 16; o; o >>= 1) nseed += __shfl_xor_sync(FULL, nseed, o);
    if (lane == 0 && nseed) atomicAdd(&s.counters[EC_VISITS], nseed);
  }
}

// The same init with 4 consecutive cells per lane, for W % 128 == 0 (every
// segment full, rows 16-byte aligned) and planar keys: one 32-bit mask word
// per row and lane, the neighbours across lanes by one shuffle of a 4-bit
// mask per row, 16-byte key stores, and the next segment's words loaded
// before this one is processed.  Same keys, same seeds (listed in another
// order: the rounds' results do not depend on it).
__device__ __forceinline__ unsigned nz4(unsigned w) {  // bit b: byte b of w is nonzero
  // high bit of each byte = (low 7 bits nonzero) | top bit; then one multiply
  // gathers bits 0 / 8 / 16 / 24 into bits 28-31 (the cross terms land below)
  const unsigned m = (((w & 0x7f7f7f7fu) + 0x7f7f7f7fu) | w) & 0x80808080u;
  return ((m >> 7) * 0x10204080u) >> 28;
}
template <int CONN, bool ROUND0 = false>
__global__ void __launch_bounds__(32 * kInitWarps) edt_init_key_rows4_kernel(const uint8_t *__restrict__ mask,
                                                                             int W, int H, EdtState s) {
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
  __shared__ uint32_t buf[kInitWarps][kInitBuf];
  unsigned nbuf = 0;
  unsigned long long nseed = 0;
  const int li = ROUND0 ? 1 : 0;
  // segments as 32-bit indices (W / 128 * H < 2^24 here), row = g >> shift
  // when W / 128 is a power of two (64-bit division is ~60 instructions)
  const unsigned spr = (unsigned)W / 128u, nseg = spr * (unsigned)H;
  const int sh = (spr & (spr - 1u)) == 0u ? __ffs(spr) - 1 : -1;
  const size_t NN = (size_t)W * H;
  auto flush = [&]() {
    unsigned base = 0;
    if (lane == 0 && nbuf) base = atomicAdd(&s.cnt[li], nbuf);
    base = __shfl_sync(FULL, base, 0);
    for (unsigned i = lane; i < nbuf; i += 32) s.F[li][base + i] = buf[wib][i];
    __syncwarp();
    nbuf = 0;
  };
  // rows y-1, y, y+1 of segment g: this lane's word, and (lanes 0 / 31) the
  // byte just left / right of the segment; kOff outside the image
  auto seg_yx = [&](unsigned g, int &y, int &x0) {
    const unsigned yy = sh >= 0 ? g >> sh : g / spr;
    y = (int)yy;
    x0 = (int)(g - yy * spr) * 128;
  };
  auto load = [&](unsigned g, unsigned (&w)[3], unsigned (&e)[3]) {
    int y, x0;
    seg_yx(g, y, x0);
#pragma unroll
    for (int rr = 0; rr < 3; rr++) {
      const int yy = y + rr - 1;
      const bool rin = yy >= 0 && yy < H;
      const uint8_t *row = mask + (size_t)(rin ? yy : 0) * W + x0;
      w[rr] = rin ? __ldg(reinterpret_cast<const unsigned *>(row) + lane) : 0u;
      const int ex = lane == 0 ? -1 : 128;
      e[rr] = (rin && (lane == 0 || lane == 31) && x0 + ex >= 0 && x0 + ex < W) ? (unsigned)__ldg(row + ex) : kOff;
    }
  };
  const unsigned stride = gridDim.x * kInitWarps;
  unsigned g = blockIdx.x * kInitWarps + wib;
  unsigned nw[3], ne[3];
  if (g < nseg) load(g, nw, ne);
  for (; g < nseg; g += stride) {
    unsigned w[3] = {nw[0], nw[1], nw[2]}, e[3] = {ne[0], ne[1], ne[2]};
    if (g + stride < nseg) load(g + stride, nw, ne);
    int y, x0;
    seg_yx(g, y, x0);
    // 6-bit masks per row: bit 0 the cell left of my 4, bits 1-4 mine, bit 5
    // the one right of them (fg = a nonzero sample inside the image, bg = a
    // zero sample inside it; outside the image: neither)
    unsigned fg[3], bg[3];
#pragma unroll
    for (int rr = 0; rr < 3; rr++) {
      const int yy = y + rr - 1;
      const bool rin = yy >= 0 && yy < H;
      const unsigned f4 = rin ? nz4(w[rr]) : 0u, b4 = rin ? (~nz4(w[rr]) & 0xfu) : 0u;
      unsigned fl = (__shfl_up_sync(FULL, f4, 1) >> 3) & 1u, bl = (__shfl_up_sync(FULL, b4, 1) >> 3) & 1u;
      unsigned fr = __shfl_down_sync(FULL, f4, 1) & 1u, br = __shfl_down_sync(FULL, b4, 1) & 1u;
      if (lane == 0) fl = e[rr] != kOff && e[rr] != 0u, bl = e[rr] == 0u;
      if (lane == 31) fr = e[rr] != kOff && e[rr] != 0u, br = e[rr] == 0u;
      fg[rr] = fl | (f4 << 1) | (fr << 5);
      bg[rr] = bl | (b4 << 1) | (br << 5);
    }
    const size_t p = (size_t)y * W + x0 + 4 * lane;
    ulonglong2 *k0 = reinterpret_cast<ulonglong2 *>(s.keys + p), *k1 = reinterpret_cast<ulonglong2 *>(s.keys + NN + p);
    // the common case, warp-wide: no foreground near any of my cells (all
    // background, own source, no seed) or no background near any (all
    // foreground, INF, no offer, no seed)
    const bool far_bg = (fg[0] | fg[1] | fg[2]) == 0u, far_fg = (bg[0] | bg[1] | bg[2]) == 0u;
    if (__all_sync(FULL, far_bg || far_fg)) {
      const uint32_t yx = ((uint32_t)y << 16) | (uint32_t)(x0 + 4 * lane);
      const ulonglong2 a = far_bg ? make_ulonglong2(yx, yx + 1) : make_ulonglong2(KINF, KINF);
      const ulonglong2 b = far_bg ? make_ulonglong2(yx + 2, yx + 3) : make_ulonglong2(KINF, KINF);
      k0[0] = a, k0[1] = b, k1[0] = a, k1[1] = b;
      continue;
    }
    unsigned long long k[4];
    unsigned seeds = 0;
    const uint32_t yc = (uint32_t)y << 16;
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const int c = b + 1;
      const uint32_t x = (uint32_t)(x0 + 4 * (int)lane + b);
      const bool isbg = (bg[1] >> c) & 1u;
      const unsigned n3 = 7u << (c - 1);  // cells c-1, c, c+1
      const bool near = CONN == 8 ? ((fg[0] & n3) | (fg[1] & (5u << (c - 1))) | (fg[2] & n3)) != 0u
                                  : (((fg[0] >> c) | (fg[2] >> c)) & 1u) || (fg[1] & (5u << (c - 1))) != 0u;
      unsigned long long kk = isbg ? (unsigned long long)(yc | x) : KINF;
      if (ROUND0) {
        if (isbg && near) nseed += 1;
        if (!isbg) {
          // round 0's offers in the order that breaks their ties: up, left,
          // right, down; then up-left, up-right, down-left, down-right
          // (branch-free: the first background neighbour in that order)
          unsigned cand = ((bg[0] >> c) & 1u) | (((bg[1] >> (c - 1)) & 1u) << 1) |
                          (((bg[1] >> (c + 1)) & 1u) << 2) | (((bg[2] >> c) & 1u) << 3);
          if (CONN == 8)
            cand |= (((bg[0] >> (c - 1)) & 1u) << 4) | (((bg[0] >> (c + 1)) & 1u) << 5) |
                    (((bg[2] >> (c - 1)) & 1u) << 6) | (((bg[2] >> (c + 1)) & 1u) << 7);
          if (cand) {
            const unsigned i = (unsigned)__ffs(cand) - 1u;
            // 2-bit fields per candidate: dy + 1, dx + 1
            const unsigned dy = (0xA094u >> (2 * i)) & 3u, dx = (0x8861u >> (2 * i)) & 3u;
            const uint32_t src = (((uint32_t)(y + (int)dy - 1)) << 16) | (x + dx - 1u);
            kk = ((unsigned long long)(i < 4 ? 1u : 2u) << 32) | src;
            seeds |= 1u << b;
          }
        }
      } else if (isbg && near) {
        seeds |= 1u << b;
      }
      k[b] = kk;
    }
    k0[0] = make_ulonglong2(k[0], k[1]);
    k0[1] = make_ulonglong2(k[2], k[3]);
    k1[0] = make_ulonglong2(k[0], k[1]);
    k1[1] = make_ulonglong2(k[2], k[3]);
#pragma unroll
    for (int b = 0; b < 4; b++) {
      const bool q = (seeds >> b) & 1u;
      const unsigned bal = __ballot_sync(FULL, q);
      if (q) buf[wib][nbuf + __popc(bal & lanemask_lt())] = ((uint32_t)y << 16) | (uint32_t)(x0 + 4 * lane + b);
      nbuf += __popc(bal);
    }
    __syncwarp();
    if (nbuf > kInitBuf - 128) flush();
  }
  flush();
  if (ROUND0) {
    for (int o = 16; o; o >>= 1) nseed += __shfl_xor_sync(FULL, nseed, o);
    if (lane == 0 && nseed) atomicAdd(&s.counters[EC_VISITS], nseed);
  }
}

__global__ void edt_import_key_kernel(const int64_t *__restrict__ vr, int W, int H, EdtState s) {
  size_t n = (size_t)W * H;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    int64_t v = vr[p];
    unsigned long long k = KINF;
    if (v >= (int64_t)n) {
      atomicAdd(&s.counters[EC_BAD], 1ull);
    } else if (v >= 0) {
      int sy = (int)(v / W), sx = (int)(v - (int64_t)sy * W);
      int py = (int)(p / (unsigned)W), px = (int)(p - (size_t)py * W);
      bool ok;
      k = make_key_checked(px, py, ((uint32_t)sy << 16) | (uint32_t)sx, ok);
      if (!ok) {
        k = KINF;
        s.counters[EC_RANGE] = 1;
      }
    }
    kput2(s.keys, p, (size_t)W * H, k);
  }
}

// seeds as given (duplicates are harmless: they offer identical keys and
// the transition rule pushes each changed cell once)
__global__ void edt_seed_key_kernel(const int64_t *__restrict__ seeds, int64_t n_seeds, int W,
                                    int H, EdtState s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_seeds;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = seeds[i];
    if (p < 0 || p >= (int64_t)W * H) {
      atomicAdd(&s.counters[EC_BAD], 1ull);
      s.F[0][i] = 0;  // harmless stand-in (cell (0,0) offers its own key)
      continue;
    }
    int py = (int)(p / W), px = (int)(p - (int64_t)py * W);
    s.F[0][i] = ((uint32_t)py << 16) | (uint32_t)px;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) s.cnt[0] = (unsigned)n_seeds;
}

// QMODE selects how the next frontier is appended (the paper's queue study,
// PAPER.md:1563-1595, Table 1): QM_BQ = warp-aggregated reservations into a
// per-block shared-memory queue, spilled with one global atomic per block
// (the default; the paper's TQ + block queue); QM_PF = warp-aggregated
// reservations straight into the global queue (one atomic per warp, the
// paper's prefix-sum variant); QM_NAIVE = one global atomicAdd per pushed
// item (the paper's naive queue).
enum { QM_BQ = 0, QM_PF = 1, QM_NAIVE = 2 };

template <int CONN, bool CHECK, int QMODE = QM_BQ>
__global__ void __launch_bounds__(kRoundThreads) edt_rounds_key_kernel(int W, int H, EdtState s,
                                                                       long long max_rounds) {
  unsigned bar_g = grid_barrier_gen(&s.bar[kBarGen]);
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u;
  // BQ: the block's next-frontier items, spilled to the global queue (GBQ)
  // with one reservation per block per round
  __shared__ uint32_t bq[kEdtBq];
  __shared__ unsigned bq_n, bq_base;
  unsigned long long visits = 0;
  unsigned long long *K = s.keys;
  const size_t NN = (size_t)W * H;
  int r = 0;
  for (;; r++) {
    unsigned n = ld_acquire(&s.cnt[r % 3]);
    if (n == 0) break;
    if (max_rounds >= 0 && r >= max_rounds) {
      if (blockIdx.x == 0 && threadIdx.x == 0) s.counters[EC_LIMIT] = 1;
      break;
    }
    const int kr = r & 1, kw = kr ^ 1;  // round-start keys / keys being built
    const uint32_t *cur = s.F[r & 1];
    uint32_t *nxt = s.F[(r + 1) & 1];
    unsigned *ncnt = &s.cnt[(r + 1) % 3];
    if (threadIdx.x == 0) {
      bq_n = 0;
      if (blockIdx.x == 0) {
        s.cnt[(r + 2) % 3] = 0;
        visits += n;
      }
    }
    __syncthreads();
    const unsigned stride = gridDim.x * blockDim.x;
    for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
      unsigned i = base + lane;
      unsigned mask = 0;
      int px = 0, py = 0;
      if (i < n) {
        uint32_t pyx = __ldcg(cur + i);
        py = (int)(pyx >> 16);
        px = (int)(pyx & 0xffffu);
        size_t p = (size_t)py * W + px;
        unsigned long long kp = __ldcg(kslot(K, p, kr, NN));
        atomicMin(kslot(K, p, kw, NN), kp);  // the building key lags on the frontier
        if (kp != KINF) {
          const uint32_t src = (uint32_t)kp;
          unsigned long long rq[Nbr<CONN>::N], nk[Nbr<CONN>::N];
          unsigned cand = 0;
#pragma unroll
          for (int k = 0; k < Nbr<CONN>::N; k++) {  // loads first (independent)
            int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
            bool in = qx >= 0 && qx < W && qy >= 0 && qy < H;
            rq[k] = in ? __ldcg(kslot(K, (size_t)qy * W + qx, kr, NN)) : 0ull;
          }
#pragma unroll
          for (int k = 0; k < Nbr<CONN>::N; k++) {
            int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
            if (CHECK) {  // d2 beyond 32 bits: flag it (the host re-runs), never offer
              bool ok;
              nk[k] = make_key_checked(qx, qy, src, ok);
              if (!ok) {
                s.counters[EC_RANGE] = 1;
                continue;
              }
            } else {
              nk[k] = make_key(qx, qy, src);
            }
            if (nk[k] < rq[k]) cand |= 1u << k;  // beats q's round-start key
          }
          // the offers, issued back to back (predicated, no branches)
#pragma unroll
          for (int k = 0; k < Nbr<CONN>::N; k++) {
            int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
            unsigned on = (cand >> k) & 1u;
            unsigned long long old =
                gmem_atomic_min_if(kslot(K, (size_t)qy * W + qx, kw, NN), nk[k], on);
            if (on && old >= rq[k]) mask |= 1u << k;  // this offer made q change
          }
        }
      }
      unsigned c = __popc(mask);
      if (QMODE == QM_NAIVE) {
        while (mask) {
          int k = __ffs(mask) - 1;
          mask &= mask - 1;
          int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
          nxt[atomicAdd(ncnt, 1u)] = ((uint32_t)qy << 16) | (uint32_t)qx;
        }
        continue;
      }
      unsigned pos = QMODE == QM_PF ? warp_reserve(ncnt, c, FULL) : warp_reserve(&bq_n, c, FULL);
      while (mask) {
        int k = __ffs(mask) - 1;
        mask &= mask - 1;
        int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
        uint32_t item = ((uint32_t)qy << 16) | (uint32_t)qx;
        if (QMODE == QM_PF)
          nxt[pos] = item;
        else if (pos < kEdtBq)
          bq[pos] = item;
        else
          nxt[atomicAdd(ncnt, 1u)] = item;  // BQ full: spill directly
        pos++;
      }
    }
    __syncthreads();
    unsigned m = min(bq_n, (unsigned)kEdtBq);
    if (threadIdx.x == 0 && m) bq_base = atomicAdd(ncnt, m);
    __syncthreads();
    for (unsigned i = threadIdx.x; i < m; i += blockDim.x) nxt[bq_base + i] = bq[i];
    grid_barrier(&s.bar[0], &s.bar[kBarGen], gridDim.x, bar_g);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s.counters[EC_ROUNDS] = (unsigned long long)r;
    s.counters[EC_VISITS] = visits;
    s.counters[EC_FINAL] = (unsigned long long)(r & 1);
  }
}

// ---- raster-frontier key engine ---------------------------------------------
// rounds whose frontier is smaller than this run as queue rounds (below)
constexpr int kRtraceRounds = 32768;
__device__ __forceinline__ void rtrace_stamp(const EdtState &s, int r, int slot) {
  if (s.rtrace && blockIdx.x == 0 && threadIdx.x == 0 && r < kRtraceRounds) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    s.rtrace[4 * r + slot] = t;
  }
}
constexpr unsigned kRasterWpt = 4;  // bitmap words per thread per compaction pass (one uint4)
//
// The same two-phase rounds as edt_rounds_key_kernel, with no returned
// atomic on a round's critical path and the frontier in raster order:
//   phase 1: every frontier cell resyncs its building key (RED.MIN) and
//            offers make_key(q, src) to each neighbour whose round-start key
//            it beats: RED.MIN on q's building key and RED.OR of q's bit in
//            the next-frontier bitmap.  q changed iff some offer beat its
//            round-start key, so the bitmap is exactly the next frontier --
//            no dedupe, no per-item reservation.  Neighbour keys are read
//            through L1 (the round-start buffer is read-only within the
//            round; every barrier's acquire invalidates L1).
//   phase 2: the bitmap is compacted into the next frontier list: each CTA
//            scans a contiguous run of words (block prefix sum, one global
//            atomic per CTA) and clears them.  The list is raster-ordered
//            within each run, so neighbouring lanes offer to neighbouring
//            cells in the next round.
// Two grid barriers per round.
template <int CONN, bool CHECK>
__global__ void __launch_bounds__(kRoundThreads) edt_rounds_raster_kernel(int W, int H, EdtState s,
                                                                          long long max_rounds, int r0) {
  unsigned bar_g = grid_barrier_gen(&s.bar[kBarGen]);
  const unsigned FULL = 0xffffffffu;
  const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  __shared__ unsigned wsum[kRoundThreads / 32];
  __shared__ unsigned blk_base, bq_n;
  __shared__ uint32_t bq[kEdtBq];
  const int WW = (W + 31) >> 5;
  const unsigned nwords = (unsigned)WW * (unsigned)H;
  uint32_t *Fb = s.fbits[0];
  unsigned long long visits = 0;
  unsigned long long *K = s.keys;
  const size_t NN = (size_t)W * H;
  // this CTA's run of bitmap words (phase 2)
  const unsigned per = ((nwords + gridDim.x - 1) / gridDim.x + kRasterWpt - 1) / kRasterWpt * kRasterWpt;
  const unsigned w_lo = min(nwords, blockIdx.x * per), w_hi = min(nwords, w_lo + per);
  int r = r0;  // 1: round 0 ran in the init (edt_init_key_rows_kernel<CONN, true>)
  for (;; r++) {
    const unsigned n = ld_acquire(&s.cnt[r % 3]);
    if (n == 0) break;
    if (max_rounds >= 0 && r >= max_rounds) {
      if (blockIdx.x == 0 && threadIdx.x == 0) s.counters[EC_LIMIT] = 1;
      break;
    }
    const int kr = r & 1, kw = kr ^ 1;
    const uint32_t *cur = s.F[r & 1];
    uint32_t *nxt = s.F[(r + 1) & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      s.cnt[(r + 2) % 3] = 0;
      visits += n;
      if (s.rtrace && r < kRtraceRounds) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        s.rtrace[4 * r] = t;
        s.rtrace[4 * r + 1] = n;
      }
    }
    if (n < kRasterMinFrontier) {
      // a small frontier: the queue round (returned atomics, transition-rule
      // pushes into a shared-memory block queue) -- one barrier
      if (threadIdx.x == 0) bq_n = 0;
      __syncthreads();
      unsigned *ncnt = &s.cnt[(r + 1) % 3];
      const unsigned stride = gridDim.x * blockDim.x;
      const unsigned first = blockIdx.x * blockDim.x + threadIdx.x;
      uint32_t pyx_next = first < n ? __ldcg(cur + first) : 0u;  // one item ahead
      for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
        const unsigned i = base + lane;
        unsigned mask = 0;
        const uint32_t pyx = pyx_next;
        pyx_next = i + stride < n ? __ldcg(cur + i + stride) : 0u;
        const int py = (int)(pyx >> 16), px = (int)(pyx & 0xffffu);
        if (i < n) {
          const size_t p = (size_t)py * W + px;
          // the cell's key and its neighbours' round-start keys in flight together
          const unsigned long long kp = __ldcg(kslot(K, p, kr, NN));
          unsigned long long rq[Nbr<CONN>::N], nk[Nbr<CONN>::N];
#pragma unroll
          for (int k = 0; k < Nbr<CONN>::N; k++) {
            const int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
            const bool in = qx >= 0 && qx < W && qy >= 0 && qy < H;
            rq[k] = in ? __ldcg(kslot(K, (size_t)qy * W + qx, kr, NN)) : 0ull;
          }
          atomicMin(kslot(K, p, kw, NN), kp);
          if (kp != KINF) {
            const uint32_t src = (uint32_t)kp;
            unsigned cand = 0;
#pragma unroll
            for (int k = 0; k < Nbr<CONN>::N; k++) {
              const int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
              bool ok = true;
              if (CHECK) {
                nk[k] = make_key_checked(qx, qy, src, ok);
                if (!ok) s.counters[EC_RANGE] = 1;
              } else {
                nk[k] = make_key(qx, qy, src);
              }
              if (ok && nk[k] < rq[k]) cand |= 1u << k;
            }
#pragma unroll
            for (int k = 0; k < Nbr<CONN>::N; k++) {
              const int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
              const unsigned on = (cand >> k) & 1u;
              const unsigned long long old =
                  gmem_atomic_min_if(kslot(K, (size_t)qy * W + qx, kw, NN), nk[k], on);
              if (on && old >= rq[k]) mask |= 1u << k;
            }
          }
        }
        const unsigned c = __popc(mask);
        unsigned pos = warp_reserve(&bq_n, c, FULL);
        while (mask) {
          const int k = __ffs(mask) - 1;
          mask &= mask - 1;
          const int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
          const uint32_t item = ((uint32_t)qy << 16) | (uint32_t)qx;
          if (pos < kEdtBq)
            bq[pos] = item;
          else
            nxt[atomicAdd(ncnt, 1u)] = item;
          pos++;
        }
      }
      __syncthreads();
      const unsigned m = min(bq_n, (unsigned)kEdtBq);
      if (threadIdx.x == 0 && m) blk_base = atomicAdd(ncnt, m);
      __syncthreads();
      for (unsigned i = threadIdx.x; i < m; i += blockDim.x) nxt[blk_base + i] = bq[i];
      grid_barrier(&s.bar[0], &s.bar[kBarGen], gridDim.x, bar_g);
      continue;
    }
    // phase 1: offers
    const unsigned stride = gridDim.x * blockDim.x;
    const unsigned first = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t pyx_next = first < n ? __ldcg(cur + first) : 0u;  // the item, one step ahead
    for (unsigned base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
      const unsigned i = base + lane;
      const bool act = i < n;
      const uint32_t pyx = pyx_next;
      pyx_next = i + stride < n ? __ldcg(cur + i + stride) : 0u;
      const int py = (int)(pyx >> 16), px = (int)(pyx & 0xffffu);
      const size_t p = (size_t)py * W + px;
      // the cell's key and its neighbours' round-start keys, all in flight at once
      const unsigned long long kp = act ? *kslot(K, p, kr, NN) : KINF;
      unsigned long long rq[Nbr<CONN>::N];
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        const int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
        const bool in = act && qx >= 0 && qx < W && qy >= 0 && qy < H;
        rq[k] = in ? *kslot(K, (size_t)qy * W + qx, kr, NN) : 0ull;
      }
      if (act) atomicMin(kslot(K, p, kw, NN), kp);  // the building key lags on the frontier (RED)
      const uint32_t src = (uint32_t)kp;
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        const int qx = px + Nbr<CONN>::dx(k), qy = py + Nbr<CONN>::dy(k);
        unsigned long long nk;
        bool ok = true;
        if (CHECK) {
          nk = make_key_checked(qx, qy, src, ok);
          if (kp != KINF && !ok) s.counters[EC_RANGE] = 1;
        } else {
          nk = make_key(qx, qy, src);
        }
        const bool push = kp != KINF && ok && nk < rq[k];  // rq = 0 off the image / inactive
        if (push) atomicMin(kslot(K, (size_t)qy * W + qx, kw, NN), nk);
        const unsigned waddr = push ? (unsigned)qy * (unsigned)WW + ((unsigned)qx >> 5) : 0xffffffffu;
        const unsigned grp = __match_any_sync(FULL, waddr);
        const unsigned orb = __reduce_or_sync(grp, push ? (1u << (qx & 31)) : 0u);
        if (push && lane == (unsigned)(__ffs(grp) - 1)) atomicOr(Fb + waddr, orb);
      }
    }
    __syncthreads();
    rtrace_stamp(s, r, 3);
    grid_barrier(&s.bar[0], &s.bar[kBarGen], gridDim.x, bar_g);
    rtrace_stamp(s, r, 2);
    // phase 2: compact this CTA's words of the bitmap into the next list,
    // kRasterWpt words per thread per pass (one 16-byte load; one block
    // prefix sum and one global atomic per pass), clearing them
    for (unsigned wb = w_lo; wb < w_hi; wb += blockDim.x * kRasterWpt) {
      const unsigned wi = wb + threadIdx.x * kRasterWpt;
      unsigned w4[kRasterWpt];
      const bool full = wi + kRasterWpt <= w_hi;
      if (full) {
        const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(Fb + wi));
        w4[0] = v.x, w4[1] = v.y, w4[2] = v.z, w4[3] = v.w;
      } else {
#pragma unroll
        for (unsigned k = 0; k < kRasterWpt; k++) w4[k] = wi + k < w_hi ? __ldcg(Fb + wi + k) : 0u;
      }
      unsigned c = 0;
#pragma unroll
      for (unsigned k = 0; k < kRasterWpt; k++) c += __popc(w4[k]);
      unsigned incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(FULL, incl, o);
        if (lane >= (unsigned)o) incl += v;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned t = 0;
        for (int k = 0; k < kRoundThreads / 32; k++) {
          const unsigned v = wsum[k];
          wsum[k] = t;  // exclusive prefix over warps
          t += v;
        }
        blk_base = t ? atomicAdd(&s.cnt[(r + 1) % 3], t) : 0u;
      }
      __syncthreads();
      unsigned o = blk_base + wsum[warp] + incl - c;
      if (CONN == 8) {
        // 8-conn: the warp writes its items together, 32 consecutive list
        // entries per store -- item j goes to lane j % 32, which finds the
        // owning lane (the last with exclusive count <= j) by a binary
        // search over the lanes, then the word and the bit (__fns) in that
        // lane's words.  Same order as the per-thread walk below; coalesced
        // stores, no divergent per-bit loops.  Blob 4K^2 c8 5.59 -> 5.28 ms
        // (compaction 11.2 -> 8.3 us per raster round); the 4-conn kernel
        // measured 2-4% slower with it, so it keeps the walk.
        if (c) {
          if (full) {
            *reinterpret_cast<uint4 *>(Fb + wi) = make_uint4(0u, 0u, 0u, 0u);
          } else {
            for (unsigned k = 0; k < kRasterWpt; k++)
              if (w4[k]) Fb[wi + k] = 0u;
          }
        }
        const unsigned excl = incl - c;
        const unsigned wtot = __shfl_sync(FULL, incl, 31);
        const unsigned obase = blk_base + wsum[warp];
        const unsigned wbase = wb + warp * 32u * kRasterWpt;  // this warp's first word
        for (unsigned j0 = 0; j0 < wtot; j0 += 32) {
          const unsigned j = j0 + lane;
          unsigned lo = 0;
#pragma unroll
          for (unsigned step = 16; step; step >>= 1) {
            const unsigned e = __shfl_sync(FULL, excl, lo + step);
            if (e <= j) lo += step;
          }
          unsigned r = j - __shfl_sync(FULL, excl, lo);
          unsigned ow[kRasterWpt];
#pragma unroll
          for (unsigned k = 0; k < kRasterWpt; k++) ow[k] = __shfl_sync(FULL, w4[k], lo);
          unsigned kk = 0, word = ow[0];
          bool found = false;
#pragma unroll
          for (unsigned k = 0; k < kRasterWpt; k++) {
            const unsigned pc = __popc(ow[k]);
            if (!found) {
              if (r < pc) {
                kk = k;
                word = ow[k];
                found = true;
              } else {
                r -= pc;
              }
            }
          }
          if (j < wtot) {
            const unsigned bb = __fns(word, 0, (int)r + 1);
            const unsigned wi2 = wbase + lo * kRasterWpt + kk;
            const unsigned y = wi2 / (unsigned)WW, x0 = (wi2 - y * (unsigned)WW) * 32;
            nxt[obase + j] = (y << 16) | (x0 + bb);
          }
        }
      } else if (c) {
        if (full) {
          *reinterpret_cast<uint4 *>(Fb + wi) = make_uint4(0u, 0u, 0u, 0u);
        } else {
          for (unsigned k = 0; k < kRasterWpt; k++)
            if (w4[k]) Fb[wi + k] = 0u;
        }
#pragma unroll
        for (unsigned k = 0; k < kRasterWpt; k++) {
          unsigned w = w4[k];
          if (!w) continue;
          const unsigned y = (wi + k) / (unsigned)WW, x0 = (wi + k - y * (unsigned)WW) * 32;
          while (w) {
            const int bb = __ffs(w) - 1;
            w &= w - 1;
            nxt[o++] = (y << 16) | (x0 + bb);
          }
        }
      }
      __syncthreads();
    }
    grid_barrier(&s.bar[0], &s.bar[kBarGen], gridDim.x, bar_g);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // (r0 = 1 with nothing to do: there were no seeds, so no round 0 either)
    s.counters[EC_ROUNDS] = (unsigned long long)(r == r0 ? 0 : r);
    s.counters[EC_VISITS] += visits;  // (+ round 0's frontier, added by the init)
    s.counters[EC_FINAL] = (unsigned long long)(r & 1);
  }
}

__global__ void edt_finalize_key_kernel(EdtState s, int W, int H, int64_t *vr, float *dist,
                                        int64_t *d2) {
  const int fb = (int)s.counters[EC_FINAL];
  size_t n = (size_t)W * H;
  unsigned long long ninf = 0;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    unsigned long long k = __ldcg(kslot(s.keys, p, fb, n));
    if (k == KINF) {
      ninf++;
      if (vr) vr[p] = -1;
      if (dist) dist[p] = 0.f;
      if (d2) d2[p] = (int64_t)1 << 62;
      continue;
    }
    uint32_t src = (uint32_t)k;
    long long dd = (long long)(k >> 32);
    if (vr) vr[p] = (int64_t)(src >> 16) * W + (src & 0xffffu);
    if (dist) dist[p] = __double2float_rn(__dsqrt_rn((double)dd));
    if (d2) d2[p] = dd;
  }
  for (int o = 16; o; o >>= 1) ninf += __shfl_xor_sync(0xffffffffu, ninf, o);
  if ((threadIdx.x & 31) == 0 && ninf) atomicAdd(&s.counters[EC_NINF], ninf);
}

// ---- host side -------------------------------------------------------------

thread_local int g_engine_override = ENGINE_AUTO;  // per host thread: diagnostics only

// One layout for both engines: the key engine's 16 B/px key array doubles
// as the CAS engine's two source buffers + stamps (12 B/px), so a key run
// that overflows its range can re-run on the same workspace.
static EdtState carve_any(Carver &c, int64_t W, int64_t H, bool cas) {
  size_t n = (size_t)W * H;
  EdtState s;
  if (g_engine_override == ENGINE_CAS) cas = true;
  s.keymode = cas ? 0 : 1;
  s.keycheck = s.keymode && (!key_mode_ok(W, H) || g_engine_override == ENGINE_KEYCHECK);
  unsigned long long *keys = c.take<unsigned long long>(2 * n);
  s.keys = nullptr;
  s.buf[0] = s.buf[1] = s.stamp = nullptr;
  if (s.keymode) {
    s.keys = keys;
  } else {
    s.buf[0] = reinterpret_cast<uint32_t *>(keys);
    s.buf[1] = s.buf[0] + n;
    s.stamp = s.buf[1] + n;
  }
  s.F[0] = c.take<uint32_t>(n);
  s.F[1] = c.take<uint32_t>(n);
  // the frontier counters, the barrier's arrival count and its generation
  // (polled by every CTA) each get their own 256-byte line
  unsigned *ctl = c.take<unsigned>(256);
  s.cnt = ctl;        // [0..2]
  s.bar = ctl + 64;   // bar[0] = arrivals, bar[kBarGen] = generation
  s.acnt = ctl + 192;  // [192..194]
  s.wc = ctl + 200;    // [200..202]
  s.counters = c.take<unsigned long long>(EC_N);
  // block engine: two planes over the same 2n keys, frontier bitmaps, regions
  const bool force_queue = g_engine_override == ENGINE_QUEUE ||
                           g_engine_override == ENGINE_QUEUE_PF ||
                           g_engine_override == ENGINE_QUEUE_NAIVE ||
                           g_engine_override == ENGINE_RASTER;
  // the default is the raster-frontier engine (queue rounds for small
  // frontiers) at every size -- on B200 it beat the blocked engine on the
  // 64K^2 whole slide too (287 vs 319 ms); 4 forces the blocked engine
  s.block = s.keymode && !force_queue && g_engine_override == ENGINE_BLOCK;
  // 3 / 5 / 6 force the plain queue engine
  s.raster = s.keymode && !s.block && g_engine_override != ENGINE_QUEUE &&
             g_engine_override != ENGINE_QUEUE_PF && g_engine_override != ENGINE_QUEUE_NAIVE;
  s.plane[0] = keys;
  s.plane[1] = keys + n;
  const size_t words = (size_t)((W + 31) / 32) * H;
  s.fbits[0] = c.take<uint32_t>(words);
  s.fbits[1] = c.take<uint32_t>(words);
  const size_t nreg = (size_t)block_regions(W, H);
  s.rplane = c.take<unsigned>(nreg);
  s.fstamp[0] = c.take<unsigned>(nreg);
  s.fstamp[1] = c.take<unsigned>(nreg);
  s.astamp = c.take<unsigned>(nreg);
  s.rflag = c.take<unsigned>(nreg);
  for (int i = 0; i < 3; i++) s.alist[i] = c.take<unsigned>(nreg);
  s.diag = c.take<unsigned long long>(16);
  s.rtrace = nullptr;
  return s;
}

size_t state_bytes(int64_t W, int64_t H) {
  Carver c(nullptr);
  carve_any(c, W, H, false);
  return c.off + 256;
}

EdtState carve_state(Carver &c, int64_t W, int64_t H, bool cas) { return carve_any(c, W, H, cas); }

int read_counters(const EdtState &s, unsigned long long *c, cudaStream_t st) {
  IWPP_CUDA_TRY(cudaMemcpyAsync(c, s.counters, sizeof(unsigned long long) * EC_N,
                                cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  return IWPP_OK;
}

static int grid_for(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  size_t cap = (size_t)device_sm_count() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

int reset_control(const EdtState &s, cudaStream_t st) {
  IWPP_CUDA_TRY(cudaMemsetAsync(s.cnt, 0, sizeof(unsigned) * (64 + kBarGen + 1), st));
  IWPP_CUDA_TRY(cudaMemsetAsync(s.counters, 0, sizeof(unsigned long long) * EC_N, st));
  return IWPP_OK;
}

int launch_init(const uint8_t *mask, int W, int H, int conn, const EdtState &s, cudaStream_t st,
                int *r0) {
  if (r0) *r0 = 0;
  size_t n = (size_t)W * H;
  int g = grid_for(n, 256);
  if (s.keymode) {
    // row segments of 128 cells, 8 warps per CTA, 8 CTAs per SM
    const long long nseg = (long long)((W + 127) / 128) * H;
    long long gb = (nseg + kInitWarps - 1) / kInitWarps;
    const long long cap = (long long)device_sm_count() * 8;
    if (gb > cap) gb = cap;
    // the raster engine takes round 0 from the init (IWPP_EDT_ROUND0=0: off)
    static int round0_env = -1;
    if (round0_env < 0) round0_env = getenv("IWPP_EDT_ROUND0") ? atoi(getenv("IWPP_EDT_ROUND0")) : 1;
    const bool round0 = s.raster && round0_env && r0;
    if (round0) *r0 = 1;
    // 4 cells per lane when every segment is full (IWPP_EDT_INIT4=0: off)
    static int init4_env = -1;
    if (init4_env < 0) init4_env = getenv("IWPP_EDT_INIT4") ? atoi(getenv("IWPP_EDT_INIT4")) : 1;
    const bool four = init4_env && IWPP_KEY_PLANAR && W % 128 == 0 && ((uintptr_t)mask % 16) == 0;
    const dim3 gd((unsigned)gb), bd(32 * kInitWarps);
    if (four) {
      if (conn == 8)
        round0 ? edt_init_key_rows4_kernel<8, true><<<gd, bd, 0, st>>>(mask, W, H, s)
               : edt_init_key_rows4_kernel<8><<<gd, bd, 0, st>>>(mask, W, H, s);
      else
        round0 ? edt_init_key_rows4_kernel<4, true><<<gd, bd, 0, st>>>(mask, W, H, s)
               : edt_init_key_rows4_kernel<4><<<gd, bd, 0, st>>>(mask, W, H, s);
    } else if (conn == 8)
      round0 ? edt_init_key_rows_kernel<8, true><<<gd, bd, 0, st>>>(mask, W, H, s)
             : edt_init_key_rows_kernel<8><<<gd, bd, 0, st>>>(mask, W, H, s);
    else
      round0 ? edt_init_key_rows_kernel<4, true><<<gd, bd, 0, st>>>(mask, W, H, s)
             : edt_init_key_rows_kernel<4><<<gd, bd, 0, st>>>(mask, W, H, s);
  } else {
    if (conn == 8)
      edt_init_kernel<8><<<g, 256, 0, st>>>(mask, W, H, s);
    else
      edt_init_kernel<4><<<g, 256, 0, st>>>(mask, W, H, s);
  }
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int launch_import(const int64_t *vr, const int64_t *seeds, int64_t n_seeds, int W, int H,
                  const EdtState &s, cudaStream_t st) {
  size_t n = (size_t)W * H;
  if (s.keymode) {
    edt_import_key_kernel<<<grid_for(n, 256), 256, 0, st>>>(vr, W, H, s);
    IWPP_CUDA_TRY(cudaGetLastError());
    if (n_seeds > 0) {
      edt_seed_key_kernel<<<grid_for((size_t)n_seeds, 256), 256, 0, st>>>(seeds, n_seeds, W, H, s);
      IWPP_CUDA_TRY(cudaGetLastError());
    }
    return IWPP_OK;
  }
  edt_import_kernel<<<grid_for(n, 256), 256, 0, st>>>(vr, W, H, s);
  IWPP_CUDA_TRY(cudaGetLastError());
  if (n_seeds > 0) {
    edt_seed_kernel<<<grid_for((size_t)n_seeds, 256), 256, 0, st>>>(seeds, n_seeds, W, H, s);
    IWPP_CUDA_TRY(cudaGetLastError());
  }
  return IWPP_OK;
}

int launch_rounds(int W, int H, int conn, const EdtState &s, long long max_rounds,
                  cudaStream_t st, int r0) {
  const int qm = g_engine_override == ENGINE_QUEUE_PF ? QM_PF
                 : g_engine_override == ENGINE_QUEUE_NAIVE ? QM_NAIVE : QM_BQ;
  if (s.raster) {  // the raster-frontier engine
    void *rk = s.keycheck ? (conn == 8 ? (void *)edt_rounds_raster_kernel<8, true>
                                       : (void *)edt_rounds_raster_kernel<4, true>)
                          : (conn == 8 ? (void *)edt_rounds_raster_kernel<8, false>
                                       : (void *)edt_rounds_raster_kernel<4, false>);
    static int rblocks[4] = {0, 0, 0, 0};
    int &rb = rblocks[(conn == 8) + 2 * s.keycheck];
    if (rb == 0) {
      int per_sm = 0;
      IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rk, kRoundThreads, 0));
      if (per_sm < 1) per_sm = 1;
      if (per_sm > kRoundBlocksPerSm) per_sm = kRoundBlocksPerSm;
      rb = device_sm_count() * per_sm;
    }
    // the next-frontier bitmap starts empty
    IWPP_CUDA_TRY(cudaMemsetAsync(s.fbits[0], 0, sizeof(uint32_t) * ((W + 31) / 32) * (size_t)H, st));
    int w = W, h = H;
    EdtState ss = s;
    void *args[] = {&w, &h, &ss, &max_rounds, &r0};
    static unsigned long long *rtrace = nullptr;  // diagnostics: IWPP_EDT_RTRACE=1
    const char *tr = getenv("IWPP_EDT_RTRACE");
    if (tr && tr[0] == '1') {
      if (!rtrace) IWPP_CUDA_TRY(cudaMalloc(&rtrace, 4 * sizeof(unsigned long long) * kRtraceRounds));
      IWPP_CUDA_TRY(cudaMemsetAsync(rtrace, 0, 4 * sizeof(unsigned long long) * kRtraceRounds, st));
      ss.rtrace = rtrace;
    }
    IWPP_CUDA_TRY(cudaLaunchCooperativeKernel(rk, dim3(rb), dim3(kRoundThreads), args, 0, st));
    if (ss.rtrace) {
      static unsigned long long h[4 * kRtraceRounds];
      IWPP_CUDA_TRY(cudaMemcpyAsync(h, rtrace, sizeof h, cudaMemcpyDeviceToHost, st));
      IWPP_CUDA_TRY(cudaStreamSynchronize(st));
      int nr = 0;
      while (nr + 1 < kRtraceRounds && h[4 * (nr + 1)]) nr++;
      for (int i = 0; i < nr; i++) {
        const unsigned long long t0 = h[4 * i], t1 = h[4 * i + 4];
        const bool rs = h[4 * i + 2] != 0;  // a raster round: work / barrier / compaction
        fprintf(stderr, "[edt rtrace] round %d n %llu dt_us %.2f work_us %.2f bar_us %.2f comp_us %.2f\n",
                i, h[4 * i + 1], (t1 - t0) * 1e-3, rs ? (h[4 * i + 3] - t0) * 1e-3 : 0.0,
                rs ? (h[4 * i + 2] - h[4 * i + 3]) * 1e-3 : 0.0, rs ? (t1 - h[4 * i + 2]) * 1e-3 : 0.0);
      }
    }
    return IWPP_OK;
  }
  void *kern = s.keymode
                   ? (s.keycheck ? (conn == 8 ? (void *)edt_rounds_key_kernel<8, true>
                                              : (void *)edt_rounds_key_kernel<4, true>)
                                 : (qm == QM_PF ? (conn == 8 ? (void *)edt_rounds_key_kernel<8, false, QM_PF>
                                                             : (void *)edt_rounds_key_kernel<4, false, QM_PF>)
                                    : qm == QM_NAIVE
                                        ? (conn == 8 ? (void *)edt_rounds_key_kernel<8, false, QM_NAIVE>
                                                     : (void *)edt_rounds_key_kernel<4, false, QM_NAIVE>)
                                        : (conn == 8 ? (void *)edt_rounds_key_kernel<8, false>
                                                     : (void *)edt_rounds_key_kernel<4, false>)))
                   : (conn == 8 ? (void *)edt_rounds_kernel<8> : (void *)edt_rounds_kernel<4>);
  static int blocks_cache[16] = {0};
  int &blocks = blocks_cache[(conn == 8) + 2 * s.keymode + 4 * s.keycheck + 8 * (qm != QM_BQ)];
  if (blocks == 0) {
    int per_sm = 0;
    IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRoundThreads, 0));
    if (per_sm < 1) per_sm = 1;
    if (per_sm > kRoundBlocksPerSm) per_sm = kRoundBlocksPerSm;
    blocks = device_sm_count() * per_sm;
  }
  int w = W, h = H;
  EdtState ss = s;
  void *args[] = {&w, &h, &ss, &max_rounds};
  IWPP_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3(blocks), dim3(kRoundThreads), args, 0, st));
  return IWPP_OK;
}

int launch_finalize_vr(const int64_t *vr, int W, int H, float *dist, int64_t *d2,
                       unsigned long long *counters, cudaStream_t st) {
  size_t n = (size_t)W * H;
  edt_finalize_vr_kernel<<<grid_for(n, 256), 256, 0, st>>>(vr, W, H, dist, d2, counters);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

// The final state lives in buf[rounds & 1]; the rounds kernel records it in
// counters[EC_FINAL].  A tiny copy kernel selects it on the device so the
// whole pipeline stays asynchronous.
__global__ void edt_select_final_kernel(EdtState s, int W, int H, int64_t *vr, float *dist,
                                        int64_t *d2) {
  // launched with the same grid as finalize; reads the flag once per thread
  int fb = (int)s.counters[EC_FINAL];
  const uint32_t *st = s.buf[fb];
  size_t n = (size_t)W * H;
  unsigned long long ninf = 0;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    uint32_t c = st[p];
    if (c == INF32) {
      ninf++;
      if (vr) vr[p] = -1;
      if (dist) dist[p] = 0.f;
      if (d2) d2[p] = (int64_t)1 << 62;
      continue;
    }
    int py = (int)(p / (unsigned)W), px = (int)(p - (size_t)py * W);
    int sy = (int)(c >> 16), sx = (int)(c & 0xffffu);
    long long dx = px - sx, dy = py - sy, dd = dx * dx + dy * dy;
    if (vr) vr[p] = (int64_t)sy * W + sx;
    if (dist) dist[p] = __double2float_rn(__dsqrt_rn((double)dd));
    if (d2) d2[p] = dd;
  }
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 16);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 8);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 4);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 2);
  ninf += __shfl_xor_sync(0xffffffffu, ninf, 1);
  if ((threadIdx.x & 31) == 0 && ninf) atomicAdd(&s.counters[EC_NINF], ninf);
}

int launch_finalize_auto(const EdtState &s, int W, int H, int64_t *vr, float *dist, int64_t *d2,
                         cudaStream_t st) {
  if (s.block) return block_finalize(s, W, H, vr, dist, d2, st);
  size_t n = (size_t)W * H;
  if (s.keymode)
    edt_finalize_key_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, W, H, vr, dist, d2);
  else
    edt_select_final_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, W, H, vr, dist, d2);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

}  // namespace edt
}  // namespace iwpp
