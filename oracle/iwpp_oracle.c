/*
 * iwpp_oracle.c -- CPU restatement of the reference ("gridwave") hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package may link,
 * load or call this file.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py use it, and there only as
 * the checker (or as the timed CPU baseline), never as the thing measured.
 *
 * Each function restates one numba kernel of the reference,
 * /root/reference/pkg/src/gridwave/_kernels.py (cited as K.<line>), or the
 * Python driver around it (recon.py / edt.py).  Loops, neighbor order,
 * bounds handling and the EDT total order follow the reference exactly so
 * the outputs are bit-identical.  Parity of this restatement is pinned by
 * tests/test_oracle.py against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py).
 *
 * dtype codes: 0 = u8 (also "binary"), 1 = u16, 2 = i32, 3 = f32.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IWPO_UNSET (-1LL)
#define IWPO_FAR (1LL << 62)

/* Full neighborhoods in raster order (K.22-25) and the raster half (K.28-31). */
static const long DX8[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
static const long DY8[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
static const long DX4[4] = {0, -1, 1, 0};
static const long DY4[4] = {-1, 0, 0, 1};
static const long RDX8[4] = {-1, 0, 1, -1};
static const long RDY8[4] = {-1, -1, -1, 0};
static const long RDX4[2] = {0, -1};
static const long RDY4[2] = {-1, 0};

/* ------------------------------------------------------------------------ */
/* reconstruction (templated over the element type by macro)                */

#define DEFINE_RECON(T, SUF)                                                   \
  /* K.38-64 recon_raster_pass */                                              \
  static int raster_pass_##SUF(T *J, const T *I, long W, int conn8, long x0,   \
                               long y0, long x1, long y1) {                    \
    int nk = conn8 ? 4 : 2, changed = 0;                                       \
    for (long y = y0; y < y1; y++)                                             \
      for (long x = x0; x < x1; x++) {                                         \
        T v = J[y * W + x];                                                    \
        for (int k = 0; k < nk; k++) {                                         \
          long nx = x + (conn8 ? RDX8[k] : RDX4[k]);                           \
          long ny = y + (conn8 ? RDY8[k] : RDY4[k]);                           \
          if (x0 <= nx && nx < x1 && y0 <= ny && ny < y1) {                    \
            T w = J[ny * W + nx];                                              \
            if (w > v) v = w;                                                  \
          }                                                                    \
        }                                                                      \
        T m = I[y * W + x];                                                    \
        if (v > m) v = m;                                                      \
        if (v != J[y * W + x]) { J[y * W + x] = v; changed = 1; }              \
      }                                                                        \
    return changed;                                                            \
  }                                                                            \
  /* K.67-112 recon_antiraster_pass (collect = seed emission, Alg.2 l.8) */    \
  static long antiraster_pass_##SUF(T *J, const T *I, long W, int conn8,       \
                                    long x0, long y0, long x1, long y1,        \
                                    int64_t *seeds, int collect,               \
                                    int *changed_out) {                        \
    int nk = conn8 ? 4 : 2, changed = 0;                                       \
    long n = 0;                                                                \
    for (long y = y1 - 1; y >= y0; y--)                                        \
      for (long x = x1 - 1; x >= x0; x--) {                                    \
        T v = J[y * W + x];                                                    \
        for (int k = 0; k < nk; k++) {                                         \
          long nx = x - (conn8 ? RDX8[k] : RDX4[k]);                           \
          long ny = y - (conn8 ? RDY8[k] : RDY4[k]);                           \
          if (x0 <= nx && nx < x1 && y0 <= ny && ny < y1) {                    \
            T w = J[ny * W + nx];                                              \
            if (w > v) v = w;                                                  \
          }                                                                    \
        }                                                                      \
        T m = I[y * W + x];                                                    \
        if (v > m) v = m;                                                      \
        if (v != J[y * W + x]) { J[y * W + x] = v; changed = 1; }              \
        if (collect) {                                                         \
          T vp = J[y * W + x];                                                 \
          for (int k = 0; k < nk; k++) {                                       \
            long nx = x - (conn8 ? RDX8[k] : RDX4[k]);                         \
            long ny = y - (conn8 ? RDY8[k] : RDY4[k]);                         \
            if (x0 <= nx && nx < x1 && y0 <= ny && ny < y1) {                  \
              T w = J[ny * W + nx];                                            \
              if (w < vp && w < I[ny * W + nx]) {                              \
                seeds[n++] = y * W + x;                                        \
                break;                                                         \
              }                                                                \
            }                                                                  \
          }                                                                    \
        }                                                                      \
      }                                                                        \
    if (changed_out) *changed_out = changed;                                   \
    return n;                                                                  \
  }                                                                            \
  /* K.193-217 recon_seed_scan: full-neighborhood active-pixel predicate */    \
  long iwpo_recon_seed_scan_##SUF(const T *J, const T *I, long W, int conn8,   \
                                  long x0, long y0, long x1, long y1,          \
                                  int64_t *out) {                              \
    int nk = conn8 ? 8 : 4;                                                    \
    long n = 0;                                                                \
    for (long y = y0; y < y1; y++)                                             \
      for (long x = x0; x < x1; x++) {                                         \
        T vp = J[y * W + x];                                                   \
        for (int k = 0; k < nk; k++) {                                         \
          long nx = x + (conn8 ? DX8[k] : DX4[k]);                             \
          long ny = y + (conn8 ? DY8[k] : DY4[k]);                             \
          if (x0 <= nx && nx < x1 && y0 <= ny && ny < y1) {                    \
            T w = J[ny * W + nx];                                              \
            if (w < vp && w < I[ny * W + nx]) { out[n++] = y * W + x; break; } \
          }                                                                    \
        }                                                                      \
      }                                                                        \
    return n;                                                                  \
  }                                                                            \
  /* K.220-270 recon_wavefront: FIFO to the fixed point inside bounds.     */  \
  /* Returns total insertions including seeds (or -1 on allocation error). */  \
  long iwpo_recon_wavefront_##SUF(T *J, const T *I, long W, int conn8,         \
                                  long x0, long y0, long x1, long y1,          \
                                  const int64_t *seeds, long n_seeds) {        \
    int nk = conn8 ? 8 : 4;                                                    \
    long cap = 4 * n_seeds + 1024;                                             \
    int64_t *buf = (int64_t *)malloc(sizeof(int64_t) * cap);                   \
    if (!buf) return -1;                                                       \
    memcpy(buf, seeds, sizeof(int64_t) * n_seeds);                             \
    long head = 0, tail = n_seeds, total = n_seeds;                            \
    while (head < tail) {                                                      \
      int64_t p = buf[head++];                                                 \
      long py = p / W, px = p % W;                                             \
      T vp = J[py * W + px];                                                   \
      for (int k = 0; k < nk; k++) {                                           \
        long nx = px + (conn8 ? DX8[k] : DX4[k]);                              \
        long ny = py + (conn8 ? DY8[k] : DY4[k]);                              \
        if (x0 <= nx && nx < x1 && y0 <= ny && ny < y1) {                      \
          T vq = J[ny * W + nx];                                               \
          T m = I[ny * W + nx];                                                \
          if (vq < vp && m != vq) {                                            \
            J[ny * W + nx] = vp < m ? vp : m;                                  \
            if (tail == cap) {                                                 \
              long live = tail - head;                                         \
              if (live * 2 < cap) {                                            \
                memmove(buf, buf + head, sizeof(int64_t) * live);              \
                head = 0; tail = live;                                         \
              } else {                                                         \
                int64_t *nb = (int64_t *)realloc(buf, sizeof(int64_t) * cap * 2); \
                if (!nb) { free(buf); return -1; }                             \
                buf = nb; cap *= 2;                                            \
              }                                                                \
            }                                                                  \
            buf[tail++] = ny * W + nx;                                         \
            total++;                                                           \
          }                                                                    \
        }                                                                      \
      }                                                                        \
    }                                                                          \
    free(buf);                                                                 \
    return total;                                                              \
  }                                                                            \
  /* recon.py:174-182 recon_fh: raster, antiraster+seeds, FIFO wavefront.  */  \
  /* stats[0]=seeds, stats[1]=queue insertions.  Returns 0, -1 on ENOMEM.  */  \
  long iwpo_recon_fh_##SUF(T *J, const T *I, long W, long H, int conn8,        \
                           int64_t *stats) {                                   \
    raster_pass_##SUF(J, I, W, conn8, 0, 0, W, H);                             \
    int64_t *seeds = (int64_t *)malloc(sizeof(int64_t) * (W * H > 0 ? W * H : 1)); \
    if (!seeds) return -1;                                                     \
    long n = antiraster_pass_##SUF(J, I, W, conn8, 0, 0, W, H, seeds, 1, 0);   \
    long tot = iwpo_recon_wavefront_##SUF(J, I, W, conn8, 0, 0, W, H, seeds, n); \
    free(seeds);                                                               \
    if (stats) { stats[0] = n; stats[1] = tot; }                               \
    return tot < 0 ? -1 : 0;                                                   \
  }                                                                            \
  /* recon.py:164-171 recon_sr: alternate sweeps until neither changes.    */  \
  long iwpo_recon_sr_##SUF(T *J, const T *I, long W, long H, int conn8) {      \
    long passes = 0;                                                           \
    for (;;) {                                                                 \
      int c1 = raster_pass_##SUF(J, I, W, conn8, 0, 0, W, H), c2 = 0;          \
      antiraster_pass_##SUF(J, I, W, conn8, 0, 0, W, H, 0, 0, &c2);            \
      passes++;                                                                \
      if (!(c1 || c2)) return passes;                                          \
    }                                                                          \
  }                                                                            \
  /* K.436-444 _recon_offer */                                                 \
  static inline long offer_##SUF(T *J, const T *I, long W, long px, long py,   \
                                 long qx, long qy, int64_t *out, long n) {     \
    T vq = J[qy * W + qx], vp = J[py * W + px];                                \
    if (vq < vp && I[qy * W + qx] != vq) {                                     \
      T iq = I[qy * W + qx];                                                   \
      J[qy * W + qx] = vp < iq ? vp : iq;                                      \
      out[n++] = qy * W + qx;                                                  \
    }                                                                          \
    return n;                                                                  \
  }                                                                            \
  /* K.460-490 recon_bp_sweep: every ordered pair straddling a tile cut.   */  \
  long iwpo_recon_bp_sweep_##SUF(T *J, const T *I, long W, long H, int conn8,  \
                                 long tw, long th, int64_t *out) {             \
    long n = 0;                                                                \
    for (long bx = tw; bx < W; bx += tw)                                       \
      for (long y = 0; y < H; y++) {                                           \
        n = offer_##SUF(J, I, W, bx - 1, y, bx, y, out, n);                    \
        n = offer_##SUF(J, I, W, bx, y, bx - 1, y, out, n);                    \
        if (conn8) {                                                           \
          if (y > 0) {                                                         \
            n = offer_##SUF(J, I, W, bx - 1, y, bx, y - 1, out, n);            \
            n = offer_##SUF(J, I, W, bx, y, bx - 1, y - 1, out, n);            \
          }                                                                    \
          if (y + 1 < H) {                                                     \
            n = offer_##SUF(J, I, W, bx - 1, y, bx, y + 1, out, n);            \
            n = offer_##SUF(J, I, W, bx, y, bx - 1, y + 1, out, n);            \
          }                                                                    \
        }                                                                      \
      }                                                                        \
    for (long by = th; by < H; by += th)                                       \
      for (long x = 0; x < W; x++) {                                           \
        n = offer_##SUF(J, I, W, x, by - 1, x, by, out, n);                    \
        n = offer_##SUF(J, I, W, x, by, x, by - 1, out, n);                    \
        if (conn8) {                                                           \
          if (x > 0 && x / tw == (x - 1) / tw) {                               \
            n = offer_##SUF(J, I, W, x, by - 1, x - 1, by, out, n);            \
            n = offer_##SUF(J, I, W, x, by, x - 1, by - 1, out, n);            \
          }                                                                    \
          if (x + 1 < W && x / tw == (x + 1) / tw) {                           \
            n = offer_##SUF(J, I, W, x, by - 1, x + 1, by, out, n);            \
            n = offer_##SUF(J, I, W, x, by, x + 1, by - 1, out, n);            \
          }                                                                    \
        }                                                                      \
      }                                                                        \
    return n;                                                                  \
  }

DEFINE_RECON(uint8_t, u8)
DEFINE_RECON(uint16_t, u16)
DEFINE_RECON(int32_t, i32)
DEFINE_RECON(float, f32)

/* The single passes of recon.py:134-161 and parallel_sweeps
 * (recon.py:275-305, one band): K.38-112 via the statics above, and the
 * axis sweeps K.115-190 restated here.  pass: 0 raster, 1 anti-raster (+
 * seeds), 2 rows forward, 3 columns forward, 4 rows backward, 5 columns
 * backward.  Returns the seed count (pass 1) and sets *changed. */
#define DEFINE_PASSES(T, SUF)                                                    /* K.115-126 recon_rows_forward */                                             static int rows_fwd_##SUF(T *J, const T *I, long W, long H) {                    int ch = 0;                                                                    for (long y = 0; y < H; y++)                                                     for (long x = 1; x < W; x++) {                                                   T v = J[y * W + x - 1];                                                        if (v > J[y * W + x]) {                                                          if (v > I[y * W + x]) v = I[y * W + x];                                        if (v > J[y * W + x]) { J[y * W + x] = v; ch = 1; }                          }                                                                            }                                                                            return ch;                                                                   }                                                                              /* K.129-139 recon_rows_backward */                                            static int rows_bwd_##SUF(T *J, const T *I, long W, long H) {                    int ch = 0;                                                                    for (long y = 0; y < H; y++)                                                     for (long x = W - 2; x >= 0; x--) {                                              T v = J[y * W + x + 1];                                                        if (v > J[y * W + x]) {                                                          if (v > I[y * W + x]) v = I[y * W + x];                                        if (v > J[y * W + x]) { J[y * W + x] = v; ch = 1; }                          }                                                                            }                                                                            return ch;                                                                   }                                                                              /* K.142-167 recon_cols_forward / K.170-190 recon_cols_backward (dir)     */   static int cols_##SUF(T *J, const T *I, long W, long H, int conn8, int dir) {    int ch = 0;                                                                    for (long x = 0; x < W; x++)                                                     for (long k = 1; k < H; k++) {                                                   long y = dir > 0 ? k : H - 1 - k, py = y - dir;                                T v = J[py * W + x];                                                           if (conn8) {                                                                     if (x - 1 >= 0 && J[py * W + x - 1] > v) v = J[py * W + x - 1];                if (x + 1 < W && J[py * W + x + 1] > v) v = J[py * W + x + 1];               }                                                                              if (v > J[y * W + x]) {                                                          if (v > I[y * W + x]) v = I[y * W + x];                                        if (v > J[y * W + x]) { J[y * W + x] = v; ch = 1; }                          }                                                                            }                                                                            return ch;                                                                   }                                                                              static long pass_##SUF(T *J, const T *I, long W, long H, int conn8,                                   int pass, int64_t *seeds, int *changed) {                 long n = 0;                                                                    switch (pass) {                                                                  case 0: *changed = raster_pass_##SUF(J, I, W, conn8, 0, 0, W, H); break;       case 1:                                                                          n = antiraster_pass_##SUF(J, I, W, conn8, 0, 0, W, H, seeds,                                             seeds != 0, changed);                                break;                                                                       case 2: *changed = rows_fwd_##SUF(J, I, W, H); break;                          case 3: *changed = cols_##SUF(J, I, W, H, conn8, 1); break;                    case 4: *changed = rows_bwd_##SUF(J, I, W, H); break;                          case 5: *changed = cols_##SUF(J, I, W, H, conn8, -1); break;                   default: return -2;                                                          }                                                                              return n;                                                                    }

DEFINE_PASSES(uint8_t, u8)
DEFINE_PASSES(uint16_t, u16)
DEFINE_PASSES(int32_t, i32)
DEFINE_PASSES(float, f32)

long iwpo_recon_pass(void *J, const void *I, int dtype, long W, long H, int conn8, int pass,
                     int64_t *seeds, int *changed) {
  switch (dtype) {
    case 0: return pass_u8((uint8_t *)J, (const uint8_t *)I, W, H, conn8, pass, seeds, changed);
    case 1: return pass_u16((uint16_t *)J, (const uint16_t *)I, W, H, conn8, pass, seeds, changed);
    case 2: return pass_i32((int32_t *)J, (const int32_t *)I, W, H, conn8, pass, seeds, changed);
    case 3: return pass_f32((float *)J, (const float *)I, W, H, conn8, pass, seeds, changed);
  }
  return -2;
}

/* dtype-dispatching front ends used by the Python wrapper */
long iwpo_recon_fh(void *J, const void *I, int dtype, long W, long H, int conn8,
                   int64_t *stats) {
  switch (dtype) {
    case 0: return iwpo_recon_fh_u8((uint8_t *)J, (const uint8_t *)I, W, H, conn8, stats);
    case 1: return iwpo_recon_fh_u16((uint16_t *)J, (const uint16_t *)I, W, H, conn8, stats);
    case 2: return iwpo_recon_fh_i32((int32_t *)J, (const int32_t *)I, W, H, conn8, stats);
    case 3: return iwpo_recon_fh_f32((float *)J, (const float *)I, W, H, conn8, stats);
  }
  return -2;
}

long iwpo_recon_sr(void *J, const void *I, int dtype, long W, long H, int conn8) {
  switch (dtype) {
    case 0: return iwpo_recon_sr_u8((uint8_t *)J, (const uint8_t *)I, W, H, conn8);
    case 1: return iwpo_recon_sr_u16((uint16_t *)J, (const uint16_t *)I, W, H, conn8);
    case 2: return iwpo_recon_sr_i32((int32_t *)J, (const int32_t *)I, W, H, conn8);
    case 3: return iwpo_recon_sr_f32((float *)J, (const float *)I, W, H, conn8);
  }
  return -2;
}

long iwpo_recon_seed_scan(const void *J, const void *I, int dtype, long W, long H,
                          int conn8, int64_t *out) {
  switch (dtype) {
    case 0: return iwpo_recon_seed_scan_u8((const uint8_t *)J, (const uint8_t *)I, W, conn8, 0, 0, W, H, out);
    case 1: return iwpo_recon_seed_scan_u16((const uint16_t *)J, (const uint16_t *)I, W, conn8, 0, 0, W, H, out);
    case 2: return iwpo_recon_seed_scan_i32((const int32_t *)J, (const int32_t *)I, W, conn8, 0, 0, W, H, out);
    case 3: return iwpo_recon_seed_scan_f32((const float *)J, (const float *)I, W, conn8, 0, 0, W, H, out);
  }
  return -2;
}

long iwpo_recon_wavefront(void *J, const void *I, int dtype, long W, int conn8,
                          long x0, long y0, long x1, long y1,
                          const int64_t *seeds, long n) {
  switch (dtype) {
    case 0: return iwpo_recon_wavefront_u8((uint8_t *)J, (const uint8_t *)I, W, conn8, x0, y0, x1, y1, seeds, n);
    case 1: return iwpo_recon_wavefront_u16((uint16_t *)J, (const uint16_t *)I, W, conn8, x0, y0, x1, y1, seeds, n);
    case 2: return iwpo_recon_wavefront_i32((int32_t *)J, (const int32_t *)I, W, conn8, x0, y0, x1, y1, seeds, n);
    case 3: return iwpo_recon_wavefront_f32((float *)J, (const float *)I, W, conn8, x0, y0, x1, y1, seeds, n);
  }
  return -2;
}

long iwpo_recon_bp_sweep(void *J, const void *I, int dtype, long W, long H,
                         int conn8, long tw, long th, int64_t *out) {
  switch (dtype) {
    case 0: return iwpo_recon_bp_sweep_u8((uint8_t *)J, (const uint8_t *)I, W, H, conn8, tw, th, out);
    case 1: return iwpo_recon_bp_sweep_u16((uint16_t *)J, (const uint16_t *)I, W, H, conn8, tw, th, out);
    case 2: return iwpo_recon_bp_sweep_i32((int32_t *)J, (const int32_t *)I, W, H, conn8, tw, th, out);
    case 3: return iwpo_recon_bp_sweep_f32((float *)J, (const float *)I, W, H, conn8, tw, th, out);
  }
  return -2;
}

/* ------------------------------------------------------------------------ */
/* distance transform                                                       */

/* K.309-317 sqdist */
static inline int64_t sqdist(long qx, long qy, int64_t src, long W) {
  if (src < 0) return IWPO_FAR;
  int64_t sy = src / W, sx = src % W;
  int64_t dx = qx - sx, dy = qy - sy;
  return dx * dx + dy * dy;
}

/* K.320-336 closer_source: (d^2, packed index) total order; UNSET loses. */
static inline int closer_source(long qx, long qy, int64_t cand, int64_t held, long W) {
  if (held < 0) return cand >= 0;
  if (cand < 0) return 0;
  int64_t dc = sqdist(qx, qy, cand, W), dh = sqdist(qx, qy, held, W);
  if (dc != dh) return dc < dh;
  return cand < held;
}

/* K.339-348 edt_assign */
void iwpo_edt_assign(const uint8_t *mask, long W, long H, int64_t *vr) {
  for (long y = 0; y < H; y++)
    for (long x = 0; x < W; x++)
      vr[y * W + x] = mask[y * W + x] == 0 ? y * W + x : IWPO_UNSET;
}

/* K.351-373 edt_contour_seeds (raster order) */
long iwpo_edt_contour_seeds(const uint8_t *mask, long W, long H, int conn8,
                            int64_t *out) {
  int nk = conn8 ? 8 : 4;
  long n = 0;
  for (long y = 0; y < H; y++)
    for (long x = 0; x < W; x++) {
      if (mask[y * W + x] != 0) continue;
      for (int k = 0; k < nk; k++) {
        long nx = x + (conn8 ? DX8[k] : DX4[k]);
        long ny = y + (conn8 ? DY8[k] : DY4[k]);
        if (0 <= nx && nx < W && 0 <= ny && ny < H && mask[ny * W + nx] != 0) {
          out[n++] = y * W + x;
          break;
        }
      }
    }
  return n;
}

/* K.403-433 edt_round_block over a window, one stream (start=0, stride=1). */
static long edt_round(int64_t *vr, long W, int conn8, long x0, long y0, long x1,
                      long y1, const int64_t *items, const int64_t *srcs, long n,
                      int64_t *out) {
  int nk = conn8 ? 8 : 4;
  long n_out = 0;
  for (long i = 0; i < n; i++) {
    int64_t p = items[i], src = srcs[i];
    if (src < 0) continue;
    long py = p / W, px = p % W;
    for (int k = 0; k < nk; k++) {
      long nx = px + (conn8 ? DX8[k] : DX4[k]);
      long ny = py + (conn8 ? DY8[k] : DY4[k]);
      if (x0 <= nx && nx < x1 && y0 <= ny && ny < y1) {
        if (closer_source(nx, ny, src, vr[ny * W + nx], W)) {
          vr[ny * W + nx] = src;
          out[n_out++] = ny * W + nx;
        }
      }
    }
  }
  return n_out;
}

/* edt.py:217-226 _run_rounds_single: the canonical two-phase round loop.
 * stats[0] = rounds, stats[1] = item visits (sum of round sizes).
 * max_rounds < 0 means unbounded; returns -3 when the cap is hit
 * (engine.py:311-317 semantics), -1 on allocation failure, else 0. */
long iwpo_edt_propagate(int64_t *vr, long W, long H, int conn8, const int64_t *seeds,
                        long n_seeds, long max_rounds, int64_t *stats) {
  int nk = conn8 ? 8 : 4;
  long cap = n_seeds > 0 ? n_seeds : 1;
  int64_t *items = (int64_t *)malloc(sizeof(int64_t) * cap);
  int64_t *srcs = (int64_t *)malloc(sizeof(int64_t) * cap);
  if (!items || !srcs) { free(items); free(srcs); return -1; }
  memcpy(items, seeds, sizeof(int64_t) * n_seeds);
  long n = n_seeds, rounds = 0, visits = 0;
  while (n > 0) {
    if (max_rounds >= 0 && rounds >= max_rounds) { free(items); free(srcs); return -3; }
    for (long i = 0; i < n; i++) srcs[i] = vr[items[i]]; /* gather: edt.py:136 */
    int64_t *out = (int64_t *)malloc(sizeof(int64_t) * (n * nk > 0 ? n * nk : 1));
    if (!out) { free(items); free(srcs); return -1; }
    long m = edt_round(vr, W, conn8, 0, 0, W, H, items, srcs, n, out);
    visits += n;
    rounds++;
    free(items);
    free(srcs);
    items = out;
    srcs = (int64_t *)malloc(sizeof(int64_t) * (m > 0 ? m : 1));
    if (!srcs) { free(items); return -1; }
    n = m;
  }
  free(items);
  free(srcs);
  if (stats) { stats[0] = rounds; stats[1] = visits; }
  return 0;
}

/* edt.py:272-281 finalize_distance_map (squared_distances edt.py:70-80):
 * dist = float32(sqrt(float64(d2))).  Returns the number of INF cells;
 * the caller raises NoBackgroundError when it is non-zero. */
long iwpo_edt_finalize(const int64_t *vr, long W, long H, float *dist, int64_t *d2out) {
  long n_inf = 0;
  for (long y = 0; y < H; y++)
    for (long x = 0; x < W; x++) {
      int64_t s = vr[y * W + x];
      if (s < 0) { n_inf++; if (d2out) d2out[y * W + x] = IWPO_FAR; continue; }
      int64_t d2 = sqdist(x, y, s, W);
      if (d2out) d2out[y * W + x] = d2;
      if (dist) dist[y * W + x] = (float)sqrt((double)d2);
    }
  return n_inf;
}

/* edt.py:284-294 edt: init, propagate, finalize.  Returns the INF count
 * (>0 means NoBackgroundError), -1 on allocation failure. */
long iwpo_edt(const uint8_t *mask, long W, long H, int conn8, int64_t *vr,
              float *dist, int64_t *stats) {
  iwpo_edt_assign(mask, W, H, vr);
  int64_t *seeds = (int64_t *)malloc(sizeof(int64_t) * (W * H > 0 ? W * H : 1));
  if (!seeds) return -1;
  long n = iwpo_edt_contour_seeds(mask, W, H, conn8, seeds);
  long rc = iwpo_edt_propagate(vr, W, H, conn8, seeds, n, -1, stats);
  free(seeds);
  if (rc < 0) return rc;
  return iwpo_edt_finalize(vr, W, H, dist, 0);
}

/* K.446-457 _edt_offer + K.493-522 edt_bp_sweep (wave-start snapshot vr0). */
static inline long edt_offer(int64_t *vr, const int64_t *vr0, long W, long px, long py,
                             long qx, long qy, int64_t *out, long n) {
  int64_t src = vr0[py * W + px];
  if (src >= 0 && closer_source(qx, qy, src, vr[qy * W + qx], W)) {
    vr[qy * W + qx] = src;
    out[n++] = qy * W + qx;
  }
  return n;
}

long iwpo_edt_bp_sweep(int64_t *vr, const int64_t *vr0, long W, long H, int conn8,
                       long tw, long th, int64_t *out) {
  long n = 0;
  for (long bx = tw; bx < W; bx += tw)
    for (long y = 0; y < H; y++) {
      n = edt_offer(vr, vr0, W, bx - 1, y, bx, y, out, n);
      n = edt_offer(vr, vr0, W, bx, y, bx - 1, y, out, n);
      if (conn8) {
        if (y > 0) {
          n = edt_offer(vr, vr0, W, bx - 1, y, bx, y - 1, out, n);
          n = edt_offer(vr, vr0, W, bx, y, bx - 1, y - 1, out, n);
        }
        if (y + 1 < H) {
          n = edt_offer(vr, vr0, W, bx - 1, y, bx, y + 1, out, n);
          n = edt_offer(vr, vr0, W, bx, y, bx - 1, y + 1, out, n);
        }
      }
    }
  for (long by = th; by < H; by += th)
    for (long x = 0; x < W; x++) {
      n = edt_offer(vr, vr0, W, x, by - 1, x, by, out, n);
      n = edt_offer(vr, vr0, W, x, by, x, by - 1, out, n);
      if (conn8) {
        if (x > 0 && x / tw == (x - 1) / tw) {
          n = edt_offer(vr, vr0, W, x, by - 1, x - 1, by, out, n);
          n = edt_offer(vr, vr0, W, x, by, x - 1, by - 1, out, n);
        }
        if (x + 1 < W && x / tw == (x + 1) / tw) {
          n = edt_offer(vr, vr0, W, x, by - 1, x + 1, by, out, n);
          n = edt_offer(vr, vr0, W, x, by, x + 1, by - 1, out, n);
        }
      }
    }
  return n;
}

/* Exact squared EDT by brute force (oracles.py:57-73), for small inputs. */
void iwpo_bruteforce_sqdist(const uint8_t *mask, long W, long H, int64_t *out) {
  for (long i = 0; i < W * H; i++) out[i] = IWPO_FAR;
  for (long s = 0; s < W * H; s++) {
    if (mask[s] != 0) continue;
    long sx = s % W, sy = s / W;
    for (long y = 0; y < H; y++)
      for (long x = 0; x < W; x++) {
        int64_t dx = x - sx, dy = y - sy, d = dx * dx + dy * dy;
        if (d < out[y * W + x]) out[y * W + x] = d;
      }
  }
}
