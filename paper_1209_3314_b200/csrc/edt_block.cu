// edt_block.cu -- temporally blocked wavefront EDT (the default key engine).
//
// Same canonical schedule as the frontier engine in edt.cu (the reference's
// two-phase rounds, K.403-433, with the (d^2, packed index) total order of
// K.320-336): every offer of round r uses the source its sender held at the
// start of round r, a target keeps the minimum key, and the next frontier is
// the set of cells whose key changed.  What changes is how the rounds are
// scheduled on the machine.
//
// The image is cut into C x C regions (C = 32).  One pass = up to K = 8
// rounds: a CTA loads an active region plus a K-cell halo (48 x 48 keys)
// into shared memory, runs the rounds there, and writes back only the
// C x C centre.  A cell's value after j rounds depends only on cells within
// distance j (Chebyshev for 8-conn, less for 4-conn), so after K rounds the
// centre is exactly what the global round-synchronous schedule computes;
// the halo ring is recomputed redundantly by each neighbour.  Grid-wide
// synchronisation drops from once per round to once per K rounds, offers
// become shared-memory atomics, and global traffic is coalesced region
// tiles instead of per-item gathers.
//
// Global state, double-buffered per region so a region can be rewritten
// while its neighbours read it as halo in the same pass:
//   plane[2]  64-bit keys (d2 << 32 | src_yx), INF = all ones
//   rplane    per region: (pass << 1) | the plane holding its current keys
//             (a region written in pass P is read from the other plane
//             until P ends)
//   fbits[2]  frontier bitmaps; fstamp[b][region] = the pass whose start
//             fbits[b] describes for that region (stale bits are ignored)
//   alist     active regions: a region runs in pass P iff a frontier cell
//             lies within its centre or halo at the start of P
// Round/visit counters match the reference's RunStats: rounds = last round
// with a change + 2, visits = seeds + changed cells.

#include <cstdlib>

#include "edt.cuh"

namespace iwpp {
namespace edt {

constexpr int BC = kBlockC;
constexpr int BSH = kBlockShift;  // log2(BC)
constexpr int BK = kBlockK;
constexpr int BE = BC + 2 * BK;  // extended region side
constexpr int BN = BE * BE;      // extended region cells
constexpr int BT = kBlockThreads;
constexpr int BIT = (BN + BT - 1) / BT;
constexpr unsigned PW_INIT = 0xFFFFFFFEu;  // pass field never matches, plane 0
static_assert(BC == (1 << BSH) && BK <= BC, "region geometry");

constexpr int LW = 3;            // local bitmap words per extended row (96 bits >= 80)
constexpr int LBW = BE * LW;      // 240 local words
static_assert(BC == 64 && BK == 8 && BE <= 32 * LW, "local bitmap layout");

struct BlockSmem {
  unsigned long long key[BN];  // keys of centre + halo (the region's working state)
  uint32_t snap[BN];           // round-start sources of the frontier cells
  unsigned F[2][LBW];          // frontier bitmaps (current / next), 3 words per row
  uint16_t cl[BN];             // this round's candidates (cells next to the frontier)
  int plane9[9];
  int fvalid9[9];
  unsigned ncl, nfront[2];
  unsigned nchg[2];
  int bbox[4];  // centre frontier: min x, min y, max x, max y (global)
  unsigned ticket;
  unsigned long long dg[8];  // diagnostics (thread 0 only), flushed at kernel end
};

__device__ __forceinline__ unsigned cur_plane(unsigned pw, unsigned P) {
  return ((pw >> 1) == P) ? ((pw & 1u) ^ 1u) : (pw & 1u);
}

// valid-cell mask of local word (ly, i): inside the extended region and the image
__device__ __forceinline__ unsigned word_mask(int i, int gx0, int gy, int W, int H) {
  if (gy < 0 || gy >= H) return 0u;
  const int lo = max(0, -gx0), hi = min(min(32, BE - 32 * i), W - gx0);  // bits [lo, hi)
  if (hi <= lo) return 0u;
  const unsigned up = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  return up & (0xffffffffu << lo);
}

// One pass over region A: pull formulation of the two-phase round.  A
// candidate q (a cell next to a frontier cell) takes the minimum of its key
// and make_key(q, round-start source of p) over its frontier neighbours p;
// each candidate word is owned by one warp (lane = cell), so there are no
// atomics and the next frontier word is a ballot.
template <int CONN, bool CHECK>
__device__ void process_region(BlockSmem &S, const EdtState &s, int W, int H, unsigned A,
                               unsigned P, long long r0, int kp, unsigned long long &visits,
                               long long &lastchg) {
  unsigned long long *dg = S.dg;
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31;
  const int RX = (W + BC - 1) / BC, RY = (H + BC - 1) / BC;
  const int WW = (W + 31) >> 5;
  const int rx = (int)(A % (unsigned)RX), ry = (int)(A / (unsigned)RX);
  const int cx0 = rx * BC, cy0 = ry * BC, ex0 = cx0 - BK, ey0 = cy0 - BK;

  if (tid < 9) {
    int nrx = rx + tid % 3 - 1, nry = ry + tid / 3 - 1;
    int pl = 0, fv = 0;
    if (nrx >= 0 && nrx < RX && nry >= 0 && nry < RY) {
      unsigned B = (unsigned)(nry * RX + nrx);
      pl = (int)cur_plane(ld_relaxed(&s.rplane[B]), P);
      fv = __ldcg(&s.fstamp[P & 1][B]) == P;
    }
    S.plane9[tid] = pl;
    S.fvalid9[tid] = fv;
  }
  if (tid == 0) {
    S.nchg[0] = S.nchg[1] = 0;
    S.bbox[0] = S.bbox[1] = INT_MAX;
    S.bbox[2] = S.bbox[3] = INT_MIN;
  }
  for (int w = tid; w < LBW; w += BT) S.F[0][w] = 0;
  long long t0 = clock64();
  if (tid == 0) dg[0]++;
  __syncthreads();

  // frontier at the start of the pass (global bitmap words -> local words)
  bool any = false;
  {
    const int wx0 = (ex0 >= 0 ? ex0 : ex0 - 31) / 32;  // floor
    const int nwx = (ex0 + BE - 1) / 32 - wx0 + 1;
    for (int i = tid; i < BE * nwx; i += BT) {
      const int ly = i / nwx, wx = wx0 + i % nwx, gy = ey0 + ly;
      if (gy < 0 || gy >= H || wx < 0 || wx >= WW) continue;
      const int ri = ((gy >> BSH) - ry + 1) * 3 + ((wx >> (BSH - 5)) - rx + 1);
      if (!S.fvalid9[ri]) continue;
      unsigned w = __ldcg(&s.fbits[P & 1][(size_t)gy * WW + wx]);
      const int off = wx * 32 - ex0;  // local x of the word's bit 0
      const int lo = max(-off, 0), hi = min(BE - off, 32);
      if (hi <= lo) continue;
      w &= (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & (0xffffffffu << lo);
      if (!w) continue;
      any = true;
      if (off < 0) {
        atomicOr(&S.F[0][ly * LW], w >> (-off));
      } else {
        const int a = off >> 5, sh = off & 31;
        atomicOr(&S.F[0][ly * LW + a], w << sh);
        if (sh && a + 1 < LW) atomicOr(&S.F[0][ly * LW + a + 1], w >> (32 - sh));
      }
    }
  }
  if (!__syncthreads_or(any)) {
    if (tid == 0) dg[1]++;
    return;
  }

  // keys of centre + halo (round-start state of the pass): batches of
  // independent L2 loads, then shared-memory stores
#pragma unroll
  for (int h = 0; h < BIT; h += 7) {
    unsigned long long v[7];
#pragma unroll
    for (int t = 0; t < 7; t++) {
      const int c = tid + (h + t) * BT;
      v[t] = KINF;
      if (h + t < BIT && c < BN) {
        const int lx = c % BE, ly = c / BE, gx = ex0 + lx, gy = ey0 + ly;
        if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
          const int ri = ((gy >> BSH) - ry + 1) * 3 + ((gx >> BSH) - rx + 1);
          v[t] = __ldcg(&s.plane[S.plane9[ri]][(size_t)gy * W + gx]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < 7; t++) {
      const int c = tid + (h + t) * BT;
      if (h + t < BIT && c < BN) S.key[c] = v[t];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) dg[4] += t1 - t0;

  int cur = 0;
  bool anychg = false;
  for (int j = 0; j < kp; j++) {
    // phase A (thread per local word): snapshot the frontier's sources,
    // clear the next bitmap, dilate the frontier into the candidate words
    if (tid == 0) {
      S.ncl = 0;
      S.nfront[j & 1] = 0;
      S.nchg[j & 1] = 0;
    }
    __syncthreads();
    for (int w0 = 0; w0 < LBW; w0 += BT) {
      const int w = w0 + tid;
      unsigned D = 0;
      int cbase = 0;
      if (w < LBW) {
        const int ly = w / LW, i = w - ly * LW;
        unsigned f = S.F[cur][w];
        S.F[cur ^ 1][w] = 0;
        cbase = ly * BE + i * 32;
        while (f) {
          const int b = __ffs(f) - 1;
          f &= f - 1;
          S.snap[cbase + b] = (uint32_t)S.key[cbase + b];
        }
        auto row = [&](int r, int k) -> unsigned {
          return (r >= 0 && r < BE && k >= 0 && k < LW) ? S.F[cur][r * LW + k] : 0u;
        };
        if (CONN == 8) {
          const unsigned vm = row(ly - 1, i - 1) | row(ly, i - 1) | row(ly + 1, i - 1);
          const unsigned v0 = row(ly - 1, i) | row(ly, i) | row(ly + 1, i);
          const unsigned vp = row(ly - 1, i + 1) | row(ly, i + 1) | row(ly + 1, i + 1);
          D = v0 | (v0 << 1) | (vm >> 31) | (v0 >> 1) | (vp << 31);
        } else {
          const unsigned c0 = row(ly, i);
          D = row(ly - 1, i) | row(ly + 1, i) | (c0 << 1) | (row(ly, i - 1) >> 31) | (c0 >> 1) |
              (row(ly, i + 1) << 31);
        }
        D &= word_mask(i, ex0 + 32 * i, ey0 + ly, W, H);
      }
      // candidate cells -> list (one reservation per warp, exclusive scan of counts)
      const unsigned cnt = __popc(D);
      unsigned incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
      }
      const unsigned tot = __shfl_sync(FULL, incl, 31);
      unsigned base = 0;
      if (lane == 31 && tot) base = atomicAdd(&S.ncl, tot);
      base = __shfl_sync(FULL, base, 31);
      unsigned pos = base + incl - cnt;
      while (D) {
        const int b = __ffs(D) - 1;
        D &= D - 1;
        S.cl[pos++] = (uint16_t)(cbase + b);
      }
    }
    __syncthreads();
    // phase B (thread per candidate): pull the offers of the frontier neighbours
    const unsigned ncl = S.ncl;
    unsigned my_chg = 0, my_front = 0;
    int bx0 = INT_MAX, by0 = INT_MAX, bx1 = INT_MIN, by1 = INT_MIN;
    for (unsigned li = tid; li < ncl; li += BT) {
      const int q = S.cl[li];
      const int ly = q / BE, lx = q - ly * BE;
      const int qx = ex0 + lx, qy = ey0 + ly;
      const unsigned long long kq = S.key[q];
      unsigned long long best = kq;
#pragma unroll
      for (int k = 0; k < Nbr<CONN>::N; k++) {
        const int plx = lx + Nbr<CONN>::dx(k), ply = ly + Nbr<CONN>::dy(k);
        if (plx < 0 || plx >= BE || ply < 0 || ply >= BE) continue;
        if (!((S.F[cur][ply * LW + (plx >> 5)] >> (plx & 31)) & 1u)) continue;
        const uint32_t src = S.snap[ply * BE + plx];
        unsigned long long nk;
        if (CHECK) {
          bool okr;
          nk = make_key_checked(qx, qy, src, okr);
          if (!okr) {
            s.counters[EC_RANGE] = 1;
            continue;
          }
        } else {
          nk = make_key(qx, qy, src);
        }
        best = nk < best ? nk : best;
      }
      if (best < kq) {
        S.key[q] = best;
        atomicOr(&S.F[cur ^ 1][ly * LW + (lx >> 5)], 1u << (lx & 31));
        my_front++;
        if (lx >= BK && lx < BK + BC && ly >= BK && ly < BK + BC) {
          my_chg++;
          bx0 = min(bx0, qx);
          bx1 = max(bx1, qx);
          by0 = min(by0, qy);
          by1 = max(by1, qy);
        }
      }
    }
    for (int o = 16; o; o >>= 1) {
      my_chg += __shfl_xor_sync(FULL, my_chg, o);
      my_front += __shfl_xor_sync(FULL, my_front, o);
    }
    if (lane == 0 && my_chg) atomicAdd(&S.nchg[j & 1], my_chg);
    if (lane == 0 && my_front) atomicAdd(&S.nfront[j & 1], my_front);
    if (j == kp - 1 && bx0 != INT_MAX) {  // the centre's outgoing frontier box
      atomicMin(&S.bbox[0], bx0);
      atomicMin(&S.bbox[1], by0);
      atomicMax(&S.bbox[2], bx1);
      atomicMax(&S.bbox[3], by1);
    }
    __syncthreads();
    const unsigned nchg = S.nchg[j & 1];
    if (nchg) {  // uniform: read after the barrier by every thread
      lastchg = max(lastchg, r0 + j);
      anychg = true;
      if (tid == 0) visits += nchg;
    }
    if (tid == 0) {
      dg[2] += ncl;
      dg[3]++;
    }
    cur ^= 1;
    if (S.nfront[j & 1] == 0) break;
  }
  long long t2 = clock64();
  if (tid == 0) dg[5] += t2 - t1;

  // outgoing frontier: centre bits of the last round, in global words
  const bool has_front = S.bbox[0] != INT_MAX;
  if (anychg) {  // write the centre back to the other plane
    const unsigned out = (unsigned)S.plane9[4] ^ 1u;
    unsigned long long *G = s.plane[out];
    for (int c = tid; c < BC * BC; c += BT) {
      const int gx = cx0 + (c & (BC - 1)), gy = cy0 + (c >> BSH);
      if (gx < W && gy < H) G[(size_t)gy * W + gx] = S.key[(BK + (c >> BSH)) * BE + BK + (c & (BC - 1))];
    }
    if (tid == 0) s.rplane[A] = (P << 1) | out;
  }
  if (has_front) {
    uint32_t *F = s.fbits[(P + 1) & 1];
    for (int w = tid; w < BC * 2; w += BT) {
      const int r = w >> 1, k = w & 1, gy = cy0 + r, wx = (cx0 >> 5) + k;
      const unsigned *row = &S.F[cur][(BK + r) * LW];
      const unsigned bits = (row[k] >> BK) | (row[k + 1] << (32 - BK));
      if (gy < H && wx < WW) F[(size_t)gy * WW + wx] = bits;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s.fstamp[(P + 1) & 1][A] = P + 1;
    if (tid == 0) dg[7]++;
    if (tid < 9) {  // activate every region whose centre + halo holds the box
      const int nrx = rx + tid % 3 - 1, nry = ry + tid / 3 - 1;
      if (nrx >= 0 && nrx < RX && nry >= 0 && nry < RY) {
        const int bx0 = nrx * BC - BK, by0 = nry * BC - BK;
        if (S.bbox[2] >= bx0 && S.bbox[0] < bx0 + BE && S.bbox[3] >= by0 && S.bbox[1] < by0 + BE) {
          const unsigned B = (unsigned)(nry * RX + nrx);
          if (atomicExch(&s.astamp[B], P + 1) != P + 1) {
            const unsigned slot = atomicAdd(&s.acnt[(P + 1) % 3], 1u);
            s.alist[(P + 1) % 3][slot] = B;
          }
        }
      }
    }
  }
  if (tid == 0) dg[6] += clock64() - t2;
}

template <int CONN, bool CHECK>
__global__ void __launch_bounds__(BT, kBlockMinCtas)
    edt_block_kernel(int W, int H, EdtState s, long long max_rounds) {
  unsigned bar_g = grid_barrier_gen(&s.bar[kBarGen]);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BlockSmem &S = *reinterpret_cast<BlockSmem *>(smem_raw);
  const int tid = threadIdx.x;
  unsigned long long visits = 0;
  long long lastchg = -1;
  long long r0 = 0;
  if (tid < 8) S.dg[tid] = 0;
  for (unsigned P = 0;; P++) {
    const unsigned nact = ld_acquire(&s.acnt[P % 3]);
    if (nact == 0) break;
    int kp = BK;
    if (max_rounds >= 0) {
      const long long rem = max_rounds - r0;
      if (rem <= 0) {
        if (blockIdx.x == 0 && tid == 0) s.counters[EC_LIMIT] = 1;
        break;
      }
      if (rem < kp) kp = (int)rem;
    }
    if (blockIdx.x == 0 && tid == 0) {  // the lists of pass P + 2 (last read in P - 1)
      s.acnt[(P + 2) % 3] = 0;
      s.wc[(P + 2) % 3] = 0;
    }
    for (;;) {
      if (tid == 0) S.ticket = atomicAdd(&s.wc[P % 3], 1u);
      __syncthreads();
      const unsigned i = S.ticket;
      __syncthreads();
      if (i >= nact) break;
      process_region<CONN, CHECK>(S, s, W, H, __ldcg(&s.alist[P % 3][i]), P, r0, kp, visits,
                                  lastchg);
      __syncthreads();
    }
    grid_barrier(&s.bar[0], &s.bar[kBarGen], gridDim.x, bar_g);
    r0 += kp;
  }
  if (tid == 0 && visits) atomicAdd(&s.counters[EC_VISITS], visits);
  if (tid == 0)
    for (int i = 0; i < 8; i++) atomicAdd(&s.diag[i], S.dg[i]);
  if (tid == 0 && blockIdx.x == 0) atomicAdd(&s.diag[8], (unsigned long long)r0);
  if (tid == 0 && lastchg >= 0)
    atomicMax(&s.counters[EC_LASTCHG], (unsigned long long)(lastchg + 1));
}

// rounds = last round with a change + 2 (the following round finds an empty
// frontier); no seeds -> no rounds; an exceeded max_rounds -> max_rounds
__global__ void edt_block_finish_kernel(EdtState s, long long max_rounds) {
  unsigned long long seeds = s.counters[EC_FINAL];
  unsigned long long r = seeds ? s.counters[EC_LASTCHG] + 1 : 0;
  if (s.counters[EC_LIMIT]) r = (unsigned long long)max_rounds;
  s.counters[EC_ROUNDS] = r;
  s.counters[EC_VISITS] += seeds;  // frontier sizes summed over rounds
}

// ---- init -------------------------------------------------------------------

__global__ void edt_block_regions_kernel(EdtState s, int nreg) {
  for (int A = blockIdx.x * blockDim.x + threadIdx.x; A < nreg; A += gridDim.x * blockDim.x) {
    s.rplane[A] = PW_INIT;
    s.fstamp[0][A] = 0;
    s.fstamp[1][A] = 0xFFFFFFFFu;
    s.astamp[A] = 0xFFFFFFFFu;
    s.rflag[A] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x < 3) {
    s.acnt[threadIdx.x] = 0;
    s.wc[threadIdx.x] = 0;
  }
}

// keys (plane 0) + seed bits from the mask (K.339-373): one warp per 32-cell
// word, so every bitmap word is written whole (no atomics).
template <int CONN>
__global__ void edt_block_init_kernel(const uint8_t *__restrict__ mask, int W, int H, EdtState s) {
  const unsigned FULL = 0xffffffffu;
  const int WW = (W + 31) >> 5, RX = (W + BC - 1) / BC;
  const size_t nwords = (size_t)WW * H;
  const int lane = threadIdx.x & 31;
  unsigned long long seeds = 0;
  for (size_t wi = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < nwords;
       wi += ((size_t)gridDim.x * blockDim.x) >> 5) {
    const int y = (int)(wi / WW), x = (int)(wi - (size_t)y * WW) * 32 + lane;
    bool seed = false;
    if (x < W) {
      const size_t p = (size_t)y * W + x;
      const bool bg = mask[p] == 0;
      const uint32_t yx = ((uint32_t)y << 16) | (uint32_t)x;
      s.plane[0][p] = bg ? (unsigned long long)yx : KINF;
      if (bg) {
#pragma unroll
        for (int k = 0; k < Nbr<CONN>::N; k++) {
          int qx = x + Nbr<CONN>::dx(k), qy = y + Nbr<CONN>::dy(k);
          if (qx >= 0 && qx < W && qy >= 0 && qy < H && mask[(size_t)qy * W + qx] != 0) seed = true;
        }
      }
    }
    const unsigned bal = __ballot_sync(FULL, seed);
    if (lane == 0) {
      s.fbits[0][wi] = bal;
      if (bal) {
        seeds += __popc(bal);
        s.rflag[(y >> BSH) * RX + ((x - lane) >> BSH)] = 1;
      }
    }
  }
  if (lane == 0 && seeds) atomicAdd(&s.counters[EC_FINAL], seeds);
}

// edt_propagate: keys from a user source map (plane 0), seed bits as given
__global__ void edt_block_import_kernel(const int64_t *__restrict__ vr, int W, int H, EdtState s) {
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
    s.plane[0][p] = k;
  }
}

__global__ void edt_block_seed_kernel(const int64_t *__restrict__ seeds, int64_t n_seeds, int W,
                                      int H, EdtState s) {
  const int WW = (W + 31) >> 5, RX = (W + BC - 1) / BC;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_seeds;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = seeds[i];
    if (p < 0 || p >= (int64_t)W * H) {
      atomicAdd(&s.counters[EC_BAD], 1ull);
      continue;
    }
    if (s.plane[0][p] == KINF) continue;  // an unset source offers nothing (K.320-336)
    int y = (int)(p / W), x = (int)(p - (int64_t)y * W);
    unsigned b = 1u << (x & 31);
    if (!(atomicOr(&s.fbits[0][(size_t)y * WW + (x >> 5)], b) & b)) {
      atomicAdd(&s.counters[EC_FINAL], 1ull);
      s.rflag[(y >> BSH) * RX + (x >> BSH)] = 1;
    }
  }
}

// pass-0 activation: a region with seeds activates itself and its 8
// neighbours (their halos reach into it)
__global__ void edt_block_activate_kernel(EdtState s, int RX, int RY) {
  const int nreg = RX * RY;
  for (int A = blockIdx.x * blockDim.x + threadIdx.x; A < nreg; A += gridDim.x * blockDim.x) {
    if (!s.rflag[A]) continue;
    const int rx = A % RX, ry = A / RX;
    for (int d = 0; d < 9; d++) {
      const int nrx = rx + d % 3 - 1, nry = ry + d / 3 - 1;
      if (nrx < 0 || nrx >= RX || nry < 0 || nry >= RY) continue;
      const unsigned B = (unsigned)(nry * RX + nrx);
      if (atomicExch(&s.astamp[B], 0u) != 0u) s.alist[0][atomicAdd(&s.acnt[0], 1u)] = B;
    }
  }
}

// ---- finalize (edt.py:272-281) ------------------------------------------------

__global__ void edt_block_finalize_kernel(EdtState s, int W, int H, int64_t *vr, float *dist,
                                          int64_t *d2) {
  const int RX = (W + BC - 1) / BC;
  size_t n = (size_t)W * H;
  unsigned long long ninf = 0;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(p / (unsigned)W), x = (int)(p - (size_t)y * W);
    const unsigned pl = __ldg(&s.rplane[(y >> BSH) * RX + (x >> BSH)]) & 1u;
    const unsigned long long k = s.plane[pl][p];
    if (k == KINF) {
      ninf++;
      if (vr) vr[p] = -1;
      if (dist) dist[p] = 0.f;
      if (d2) d2[p] = (int64_t)1 << 62;
      continue;
    }
    const uint32_t src = (uint32_t)k;
    const long long dd = (long long)(k >> 32);
    if (vr) vr[p] = (int64_t)(src >> 16) * W + (src & 0xffffu);
    if (dist) dist[p] = __double2float_rn(__dsqrt_rn((double)dd));
    if (d2) d2[p] = dd;
  }
  for (int o = 16; o; o >>= 1) ninf += __shfl_xor_sync(0xffffffffu, ninf, o);
  if ((threadIdx.x & 31) == 0 && ninf) atomicAdd(&s.counters[EC_NINF], ninf);
}

// ---- host side ------------------------------------------------------------------

static int grid_cap(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  size_t cap = (size_t)device_sm_count() * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

int block_init(const uint8_t *mask, const int64_t *vr, const int64_t *seeds, int64_t n_seeds,
               int W, int H, int conn, const EdtState &s, cudaStream_t st) {
  const int RX = (W + BC - 1) / BC, RY = (H + BC - 1) / BC, nreg = RX * RY;
  IWPP_CUDA_TRY(cudaMemsetAsync(s.diag, 0, 16 * sizeof(unsigned long long), st));
  edt_block_regions_kernel<<<grid_cap((size_t)nreg, 256), 256, 0, st>>>(s, nreg);
  IWPP_CUDA_TRY(cudaGetLastError());
  if (mask) {
    const size_t threads = (size_t)((W + 31) / 32) * H * 32;
    if (conn == 8)
      edt_block_init_kernel<8><<<grid_cap(threads, 256), 256, 0, st>>>(mask, W, H, s);
    else
      edt_block_init_kernel<4><<<grid_cap(threads, 256), 256, 0, st>>>(mask, W, H, s);
  } else {
    const size_t words = (size_t)((W + 31) / 32) * H;
    IWPP_CUDA_TRY(cudaMemsetAsync(s.fbits[0], 0, words * sizeof(uint32_t), st));
    edt_block_import_kernel<<<grid_cap((size_t)W * H, 256), 256, 0, st>>>(vr, W, H, s);
    IWPP_CUDA_TRY(cudaGetLastError());
    if (n_seeds > 0)
      edt_block_seed_kernel<<<grid_cap((size_t)n_seeds, 256), 256, 0, st>>>(seeds, n_seeds, W, H, s);
  }
  IWPP_CUDA_TRY(cudaGetLastError());
  edt_block_activate_kernel<<<grid_cap((size_t)nreg, 256), 256, 0, st>>>(s, RX, RY);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int block_rounds(int W, int H, int conn, const EdtState &s, long long max_rounds,
                 cudaStream_t st) {
  void *kern = s.keycheck ? (conn == 8 ? (void *)edt_block_kernel<8, true>
                                       : (void *)edt_block_kernel<4, true>)
                          : (conn == 8 ? (void *)edt_block_kernel<8, false>
                                       : (void *)edt_block_kernel<4, false>);
  const int smem = (int)sizeof(BlockSmem);
  static int blocks_cache[4] = {0, 0, 0, 0};
  int &blocks = blocks_cache[(conn == 8) + 2 * s.keycheck];
  if (blocks == 0) {
    IWPP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    IWPP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BT, smem));
    if (per_sm < 1) per_sm = 1;
    blocks = device_sm_count() * per_sm;
  }
  int w = W, h = H;
  EdtState ss = s;
  void *args[] = {&w, &h, &ss, &max_rounds};
  int nb = blocks;
  if (const char *e = getenv("IWPP_EDT_BLOCKS")) {  // diagnostics: smaller persistent grid
    int v = atoi(e);
    if (v > 0 && v < nb) nb = v;
  }
  IWPP_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3(nb), dim3(BT), args, smem, st));
  edt_block_finish_kernel<<<1, 1, 0, st>>>(s, max_rounds);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int block_finalize(const EdtState &s, int W, int H, int64_t *vr, float *dist, int64_t *d2,
                   cudaStream_t st) {
  edt_block_finalize_kernel<<<grid_cap((size_t)W * H, 256), 256, 0, st>>>(s, W, H, vr, dist, d2);
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

}  // namespace edt
}  // namespace iwpp
