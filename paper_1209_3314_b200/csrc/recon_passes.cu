// recon_passes.cu -- the reference's individual scan passes, exactly:
//   raster pass            K.38-74   (recon.raster_pass)
//   anti-raster pass+seeds K.77-112  (recon.antiraster_pass / _antiraster_packed)
//   column sweeps fwd/bwd  K.142-190 (recon.parallel_sweeps, 8-conn diagonals)
// (the row sweeps, K.115-139, are row_sweep_kernel in recon_sweeps.cu).
//
// These passes are not on the reconstruction hot path -- the tile engine
// never needs them -- but callers of the reference's recon module use them
// directly, and their intermediate states are schedule-specific, so they
// are reproduced cell for cell.  Each pass is a chain of lines (rows for the
// raster passes, columns for the column sweeps) in which every line depends
// on the one before: one CTA walks the lines in order, and inside a line the
// Gauss-Seidel recurrence
//     v_e = min(I_e, max(a_e, v_{e-1})),   a_e = max(J_e, previous-line terms)
// is a chain of clamp functions clamp(., min(a_e, I_e), I_e), closed under
// composition, so the line is one block-wide scan (thread composite ->
// warp shuffle scan -> scan over the warp totals) instead of a serial walk.

#include <climits>

#include "iwpp_common.cuh"
#include "recon_sweeps.cuh"

namespace iwpp {
namespace recon {

enum { PASS_RASTER = 0, PASS_ANTIRASTER = 1, PASS_COLS_FWD = 2, PASS_COLS_BWD = 3 };
constexpr int kPassThreads = 1024;
constexpr int kPassE = 8;  // elements per thread per chunk
constexpr int kPassChunk = kPassThreads * kPassE;

__device__ __forceinline__ int pclamp(int v, int lo, int hi) { return min(hi, max(lo, v)); }

template <int MODE>
__device__ __forceinline__ void pass_pos(int line, int e, int W, int H, int &y, int &x) {
  if (MODE == PASS_RASTER) { y = line; x = e; }
  else if (MODE == PASS_ANTIRASTER) { y = H - 1 - line; x = W - 1 - e; }
  else if (MODE == PASS_COLS_FWD) { x = line; y = e; }
  else { x = line; y = H - 1 - e; }
}

// Block-wide exclusive scan of clamp composites (l, h) in thread order.
__device__ __forceinline__ void block_clamp_scan(int &l, int &h, int *sl, int *sh) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {  // inclusive: earlier functions first
    const int ol = __shfl_up_sync(FULL, l, o), oh = __shfl_up_sync(FULL, h, o);
    if (lane >= o) {
      const int nl = pclamp(ol, l, h), nh = pclamp(oh, l, h);
      l = nl;
      h = nh;
    }
  }
  if (lane == 31) { sl[warp] = l; sh[warp] = h; }
  __syncthreads();
  if (warp == 0) {  // scan the warp totals, exclusive
    int wl = sl[lane], wh = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ol = __shfl_up_sync(FULL, wl, o), oh = __shfl_up_sync(FULL, wh, o);
      if (lane >= o) {
        const int nl = pclamp(ol, wl, wh), nh = pclamp(oh, wl, wh);
        wl = nl;
        wh = nh;
      }
    }
    int el = __shfl_up_sync(FULL, wl, 1), eh = __shfl_up_sync(FULL, wh, 1);
    if (lane == 0) { el = INT_MIN; eh = INT_MAX; }
    sl[lane] = el;
    sh[lane] = eh;
  }
  __syncthreads();
  // my exclusive composite = (my warp's exclusive prefix) then (lanes before me)
  int el = __shfl_up_sync(FULL, l, 1), eh = __shfl_up_sync(FULL, h, 1);
  if (lane == 0) { el = INT_MIN; eh = INT_MAX; }
  const int pl = sl[warp], ph = sh[warp];
  l = pclamp(pl, el, eh);
  h = pclamp(ph, el, eh);
}

template <typename T, int MODE>
__global__ void __launch_bounds__(kPassThreads, 1)
    line_pass_kernel(T *__restrict__ J, const T *__restrict__ I, int W, int H, int conn8,
                     int64_t *__restrict__ seeds, unsigned long long *ctr) {
  __shared__ int sl[32], sh[32];
  __shared__ int s_carry;
  __shared__ unsigned s_cnt[32];
  __shared__ unsigned long long s_seed_base;
  __shared__ int s_out[kPassChunk];  // anti-raster seeds: this chunk's new values
  constexpr bool ROWS = MODE == PASS_RASTER || MODE == PASS_ANTIRASTER;
  const int L = ROWS ? W : H, NL = ROWS ? H : W;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned changed = 0;
  if (t == 0) s_seed_base = 0;
  for (int line = 0; line < NL; line++) {
    int carry = INT_MIN;
    for (int c0 = 0; c0 < L; c0 += kPassChunk) {
      int lo[kPassE], hi[kPassE], orig[kPassE];
#pragma unroll
      for (int i = 0; i < kPassE; i++) {
        const int e = c0 + t * kPassE + i;
        lo[i] = INT_MIN;
        hi[i] = INT_MAX;
        orig[i] = INT_MIN;
        if (e >= L) continue;
        int y, x;
        pass_pos<MODE>(line, e, W, H, y, x);
        const size_t p = (size_t)y * W + x;
        const int jv = (int)J[p], iv = (int)I[p];
        int a = jv;
        if (MODE == PASS_RASTER || MODE == PASS_ANTIRASTER) {
          // the half neighbourhood in the previous (already updated) row
          const int py = MODE == PASS_RASTER ? y - 1 : y + 1;
          if (py >= 0 && py < H) {
            const T *R = J + (size_t)py * W;
            a = max(a, (int)R[x]);
            if (conn8) {
              if (x > 0) a = max(a, (int)R[x - 1]);
              if (x + 1 < W) a = max(a, (int)R[x + 1]);
            }
          }
        } else if (conn8) {
          // column sweeps: the diagonal reads of the previous row, from the
          // column before (updated) and the column after (not yet visited)
          const int py = MODE == PASS_COLS_FWD ? y - 1 : y + 1;
          if (py >= 0 && py < H) {
            const T *R = J + (size_t)py * W;
            if (x > 0) a = max(a, (int)R[x - 1]);
            if (x + 1 < W) a = max(a, (int)R[x + 1]);
          }
        }
        lo[i] = min(a, iv);
        hi[i] = iv;
        orig[i] = jv;
      }
      // the first element of a column sweep keeps its value (K.160: y from y0 + 1)
      int l = INT_MIN, h = INT_MAX;
#pragma unroll
      for (int i = 0; i < kPassE; i++) {
        l = pclamp(l, lo[i], hi[i]);
        h = pclamp(h, lo[i], hi[i]);
      }
      block_clamp_scan(l, h, sl, sh);
      int v = pclamp(carry, l, h);
      int out[kPassE];
#pragma unroll
      for (int i = 0; i < kPassE; i++) {
        const int e = c0 + t * kPassE + i;
        v = (MODE >= PASS_COLS_FWD && e == 0) ? orig[i] : pclamp(v, lo[i], hi[i]);
        out[i] = v;
        if (e < L && v != orig[i]) {
          int y, x;
          pass_pos<MODE>(line, e, W, H, y, x);
          J[(size_t)y * W + x] = (T)v;
          changed = 1;
        }
      }
      // carry = the chunk's last value
      const int last = min(kPassChunk, L - c0) - 1;
      if (t == last / kPassE) {
#pragma unroll
        for (int i = 0; i < kPassE; i++)
          if (t * kPassE + i == last) s_carry = out[i];
      }
      if (MODE == PASS_ANTIRASTER && seeds) {
        // K.99-110: after its update a cell is a seed if one of the
        // neighbours the sweep has already visited -- E in this row, SE /
        // S / SW in the row below, all at their values from this pass -- is
        // below the cell's value and below its own mask.  Seeds in
        // anti-raster order (the order the sweep met them).
#pragma unroll
        for (int i = 0; i < kPassE; i++) s_out[t * kPassE + i] = out[i];
        __syncthreads();
        unsigned mine = 0;
        bool is_seed[kPassE];
#pragma unroll
        for (int i = 0; i < kPassE; i++) {
          const int e = c0 + t * kPassE + i;
          is_seed[i] = false;
          if (e >= L) continue;
          int y, x;
          pass_pos<MODE>(line, e, W, H, y, x);
          const int vp = out[i];
          bool s = false;
          if (x + 1 < W) {  // E: the previous element in scan order
            const int li = t * kPassE + i - 1;
            const int w = li >= 0 ? s_out[li] : carry;
            s = w < vp && w < (int)I[(size_t)y * W + x + 1];
          }
          if (y + 1 < H) {
            const T *R = J + (size_t)(y + 1) * W;
            const T *RI = I + (size_t)(y + 1) * W;
            // K.28-31 order: SE, S, SW
            const int xa = conn8 ? min(x + 1, W - 1) : x, xb = conn8 ? max(x - 1, 0) : x;
            for (int nx = xa; nx >= xb && !s; nx--) {
              const int w = (int)R[nx];
              s = w < vp && w < (int)RI[nx];
            }
          }
          is_seed[i] = s;
          mine += s;
        }
        // block exclusive prefix of the per-thread counts
        unsigned incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        if (lane == 31) s_cnt[warp] = incl;
        __syncthreads();
        unsigned wbase = 0, tot = 0;
        for (int k = 0; k < 32; k++) {
          const unsigned c = s_cnt[k];
          if (k < warp) wbase += c;
          tot += c;
        }
        unsigned long long pos = s_seed_base + wbase + incl - mine;
#pragma unroll
        for (int i = 0; i < kPassE; i++) {
          if (!is_seed[i]) continue;
          int y, x;
          pass_pos<MODE>(line, c0 + t * kPassE + i, W, H, y, x);
          seeds[pos++] = (int64_t)y * W + x;
        }
        __syncthreads();
        if (t == 0) s_seed_base += tot;
      }
      __syncthreads();
      carry = s_carry;
      __syncthreads();
    }
  }
  changed = __syncthreads_or(changed);
  if (t == 0) {
    ctr[0] = changed;
    ctr[1] = s_seed_base;
  }
}

template <typename T>
static int pass_impl(void *J, const void *I, int W, int H, int conn, int mode, int64_t *seeds,
                     unsigned long long *ctr, cudaStream_t st) {
  const int c8 = conn == 8;
  T *j = (T *)J;
  const T *i = (const T *)I;
  switch (mode) {
    case PASS_RASTER: line_pass_kernel<T, PASS_RASTER><<<1, kPassThreads, 0, st>>>(j, i, W, H, c8, nullptr, ctr); break;
    case PASS_ANTIRASTER: line_pass_kernel<T, PASS_ANTIRASTER><<<1, kPassThreads, 0, st>>>(j, i, W, H, c8, seeds, ctr); break;
    case PASS_COLS_FWD: line_pass_kernel<T, PASS_COLS_FWD><<<1, kPassThreads, 0, st>>>(j, i, W, H, c8, nullptr, ctr); break;
    case PASS_COLS_BWD: line_pass_kernel<T, PASS_COLS_BWD><<<1, kPassThreads, 0, st>>>(j, i, W, H, c8, nullptr, ctr); break;
    default: return set_error(IWPP_E_CONTRACT, "unknown pass %d", mode);
  }
  IWPP_CUDA_TRY(cudaGetLastError());
  return IWPP_OK;
}

int line_pass(void *J, const void *I, int W, int H, int dtype, int conn, int mode, int64_t *seeds,
              unsigned long long *ctr, cudaStream_t st) {
  switch (dtype) {
    case IWPP_U8:
    case IWPP_BIN: return pass_impl<uint8_t>(J, I, W, H, conn, mode, seeds, ctr, st);
    case IWPP_U16: return pass_impl<uint16_t>(J, I, W, H, conn, mode, seeds, ctr, st);
    case IWPP_I32: return pass_impl<int32_t>(J, I, W, H, conn, mode, seeds, ctr, st);
  }
  return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
}

}  // namespace recon
}  // namespace iwpp
