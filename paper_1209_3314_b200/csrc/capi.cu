// capi.cu -- extern "C" entry points of libiwpp_b200.so (include/iwpp_b200.h).

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "edt.cuh"
#include "iwpp_common.cuh"
#include "recon_sweeps.cuh"
#include "recon_tiles.cuh"

namespace iwpp {

static thread_local char g_err[512] = "";

int set_error(int status, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return status;
}

int set_cuda_error(cudaError_t e, const char *what, const char *file, int line) {
  return set_error(IWPP_E_CUDA, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                   cudaGetErrorString(e), what, file, line);
}

int device_sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 1;
  }
  return cache[dev];
}

static size_t elem_size(int dtype) {
  switch (dtype) {
    case IWPP_U8: return 1;
    case IWPP_U16: return 2;
    case IWPP_I32: return 4;
  }
  return 0;
}

static int check_dims(int64_t W, int64_t H) {
  if (W < 1 || H < 1) return set_error(IWPP_E_CONTRACT, "image dimensions must be >= 1");
  if (W > (1 << 30) || H > (1 << 30) || W * H > ((int64_t)1 << 36))
    return set_error(IWPP_E_CONTRACT, "image too large for one device (%lld x %lld)",
                     (long long)W, (long long)H);
  return IWPP_OK;
}

// recon workspace: tile queue + counters + column-sweep scratch
struct ReconWs {
  recon::TileQueue q;
  unsigned long long *counters;
  void *col_scratch;
};

static ReconWs carve_recon(Carver &c, int64_t W, int64_t H) {
  ReconWs w;
  w.q = recon::carve_tile_queue(c, recon::num_tiles(W, H));
  w.counters = c.take<unsigned long long>(recon::CNT_N);
  w.col_scratch = c.take<char>(recon::col_scratch_bytes(W, H));
  return w;
}

static size_t recon_ws_bytes(int64_t W, int64_t H) {
  Carver c(nullptr);
  carve_recon(c, W, H);
  return c.off + 256;
}

}  // namespace iwpp

using namespace iwpp;

extern "C" {

const char *iwpp_last_error(void) { return g_err; }
const char *iwpp_version(void) { return "iwpp_b200 0.1.0 (sm_100a)"; }

int iwpp_device_info(int device, int *sm_count, int *cc_major, int *cc_minor) {
  IWPP_CUDA_TRY(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  IWPP_CUDA_TRY(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  IWPP_CUDA_TRY(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return IWPP_OK;
}

// ---------------------------------------------------------------- recon

size_t iwpp_recon_workspace_bytes(int64_t W, int64_t H, int dtype, int conn) {
  (void)dtype;
  (void)conn;
  return recon_ws_bytes(W, H);
}

static int fill_recon_stats(const ReconWs &w, iwpp_stats *stats, cudaStream_t st) {
  unsigned long long c[recon::CNT_N];
  IWPP_CUDA_TRY(cudaMemcpyAsync(c, w.counters, sizeof c, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  memset(stats, 0, sizeof *stats);
  stats->executions = 1;
  stats->tiles_processed = (int64_t)c[recon::CNT_TILES];
  stats->tile_reruns = (int64_t)c[recon::CNT_RERUNS];
  stats->queued_total = (int64_t)c[recon::CNT_PUSHES] + (int64_t)c[recon::CNT_SEEDS];
  stats->overflow_count = (int64_t)c[recon::CNT_OVERFLOW];
  stats->seeds = (int64_t)c[recon::CNT_SEEDS];
  stats->contract_violations = (int64_t)c[recon::CNT_VIOL];
  return IWPP_OK;
}

int iwpp_recon(void *J, const void *I, int64_t W, int64_t H, int dtype, int conn,
               void *workspace, size_t workspace_bytes, const iwpp_recon_opts *opts,
               iwpp_stats *stats, void *stream) {
  int rc = check_dims(W, H);
  if (rc) return rc;
  if (conn != 4 && conn != 8)
    return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8, got %d", conn);
  if (!elem_size(dtype)) return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
  if (workspace_bytes < recon_ws_bytes(W, H))
    return set_error(IWPP_E_WORKSPACE, "workspace too small (%zu < %zu)", workspace_bytes,
                     recon_ws_bytes(W, H));
  cudaStream_t st = (cudaStream_t)stream;
  Carver c(workspace);
  ReconWs w = carve_recon(c, W, H);
  int sweeps = opts ? opts->sweeps : -1;
  if (sweeps < 0) sweeps = 0;  // auto: the tile engine alone (measured best on random inputs)
  for (int s = 0; s < sweeps; s++) {
    if ((rc = recon::sweep_rows(J, I, (int)W, (int)H, dtype, st))) return rc;
    if ((rc = recon::sweep_cols(J, I, (int)W, (int)H, dtype, w.col_scratch, st))) return rc;
  }
  recon::EngineOpts eo;
  if (opts) {
    eo.max_blocks = opts->max_blocks;
    eo.qcap = opts->queue_capacity;
    if (opts->tile_sweeps >= 0) eo.sweeps = opts->tile_sweeps;
    eo.halo_thresh = opts->halo_sweep_threshold;
    eo.ev_begin = opts->ev_begin;
    eo.ev_end = opts->ev_end;
    eo.rows_mode = opts->slab_rows & 3;
  }
  if ((rc = recon::run_tile_engine(J, I, (int)W, (int)H, dtype, conn, w.q, w.counters, eo, st)))
    return rc;
  if (opts && opts->check_contract) {
    if ((rc = recon::check_le(J, I, (size_t)W * H, dtype, &w.counters[recon::CNT_VIOL], st)))
      return rc;
  }
  if (stats) return fill_recon_stats(w, stats, st);
  return IWPP_OK;
}

size_t iwpp_recon_host_workspace_bytes(int64_t W, int64_t H, int dtype, int conn) {
  size_t img = align_up((size_t)W * H * elem_size(dtype), 256);
  return 2 * img + recon_ws_bytes(W, H) + 256;
}

int iwpp_recon_host(void *out, const void *marker, const void *mask, int64_t W, int64_t H,
                    int dtype, int conn, void *workspace, size_t workspace_bytes,
                    const iwpp_recon_opts *opts, iwpp_stats *stats, void *stream) {
  int rc = check_dims(W, H);
  if (rc) return rc;
  size_t es = elem_size(dtype);
  if (!es) return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
  if (workspace_bytes < iwpp_recon_host_workspace_bytes(W, H, dtype, conn))
    return set_error(IWPP_E_WORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  size_t nb = (size_t)W * H * es;
  Carver c(workspace);
  char *dJ = c.take<char>(nb);
  char *dI = c.take<char>(nb);
  char *rest = c.base + align_up(c.off, 256);
  size_t rest_bytes = workspace_bytes - align_up(c.off, 256);
  IWPP_CUDA_TRY(cudaMemcpyAsync(dJ, marker, nb, cudaMemcpyHostToDevice, st));
  IWPP_CUDA_TRY(cudaMemcpyAsync(dI, mask, nb, cudaMemcpyHostToDevice, st));
  // contract check (recon.py:60) fused into the same stream
  Carver c2(rest);
  ReconWs w = carve_recon(c2, W, H);
  IWPP_CUDA_TRY(cudaMemsetAsync(&w.counters[recon::CNT_VIOL], 0, sizeof(unsigned long long), st));
  if ((rc = recon::check_le(dJ, dI, (size_t)W * H, dtype, &w.counters[recon::CNT_VIOL], st))) return rc;
  unsigned long long viol = 0;
  IWPP_CUDA_TRY(cudaMemcpyAsync(&viol, &w.counters[recon::CNT_VIOL], sizeof viol,
                                cudaMemcpyDeviceToHost, st));
  iwpp_recon_opts o = opts ? *opts : iwpp_recon_opts{-1, 0, 0, 0, -1, -1, nullptr, nullptr, 0};
  o.check_contract = 0;
  if ((rc = iwpp_recon(dJ, dI, W, H, dtype, conn, rest, rest_bytes, &o, nullptr, stream))) return rc;
  IWPP_CUDA_TRY(cudaMemcpyAsync(out, dJ, nb, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  if (viol) return set_error(IWPP_E_CONTRACT, "marker exceeds mask somewhere (%llu cells)", viol);
  if (stats) return fill_recon_stats(w, stats, st);
  return IWPP_OK;
}

int iwpp_event_create(void **ev) {
  cudaEvent_t e;
  IWPP_CUDA_TRY(cudaEventCreate(&e));
  *ev = (void *)e;
  return IWPP_OK;
}
int iwpp_event_destroy(void *ev) {
  IWPP_CUDA_TRY(cudaEventDestroy((cudaEvent_t)ev));
  return IWPP_OK;
}
int iwpp_event_record(void *ev, void *stream) {
  IWPP_CUDA_TRY(cudaEventRecord((cudaEvent_t)ev, (cudaStream_t)stream));
  return IWPP_OK;
}
int iwpp_event_elapsed_ms(void *begin, void *end, float *ms) {
  IWPP_CUDA_TRY(cudaEventSynchronize((cudaEvent_t)end));
  IWPP_CUDA_TRY(cudaEventElapsedTime(ms, (cudaEvent_t)begin, (cudaEvent_t)end));
  return IWPP_OK;
}

int iwpp_recon_engine_counters(const void *workspace, int64_t W, int64_t H, uint64_t *out,
                               int n, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  Carver c((void *)workspace);
  ReconWs w = carve_recon(c, W, H);
  if (n > recon::CNT_N) n = recon::CNT_N;
  IWPP_CUDA_TRY(cudaMemcpyAsync(out, w.counters, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  return n;
}

int iwpp_check_le(const void *J, const void *I, int64_t n, int dtype, void *workspace,
                  int64_t *n_violations_host, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *ctr = (unsigned long long *)workspace;
  IWPP_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof *ctr, st));
  int rc = recon::check_le(J, I, (size_t)n, dtype, ctr, st);
  if (rc) return rc;
  unsigned long long v = 0;
  IWPP_CUDA_TRY(cudaMemcpyAsync(&v, ctr, sizeof v, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  *n_violations_host = (int64_t)v;
  return IWPP_OK;
}

int iwpp_recon_sweep_rows(void *J, const void *I, int64_t W, int64_t H, int dtype, void *stream) {
  int rc = check_dims(W, H);
  if (rc) return rc;
  return recon::sweep_rows(J, I, (int)W, (int)H, dtype, (cudaStream_t)stream);
}

int iwpp_recon_sweep_cols(void *J, const void *I, int64_t W, int64_t H, int dtype, void *workspace,
                          void *stream) {
  int rc = check_dims(W, H);
  if (rc) return rc;
  Carver c(workspace);
  ReconWs w = carve_recon(c, W, H);
  return recon::sweep_cols(J, I, (int)W, (int)H, dtype, w.col_scratch, (cudaStream_t)stream);
}

int iwpp_recon_seed_scan(const void *J, const void *I, int64_t W, int64_t H, int dtype, int conn,
                         int64_t *out, int64_t *n_host, void *workspace, void *stream) {
  int rc = check_dims(W, H);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *ctr = (unsigned long long *)workspace;
  IWPP_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof *ctr, st));
  if ((rc = recon::seed_scan(J, I, (int)W, (int)H, dtype, conn, out, ctr, st))) return rc;
  unsigned long long v = 0;
  IWPP_CUDA_TRY(cudaMemcpyAsync(&v, ctr, sizeof v, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  *n_host = (int64_t)v;
  return IWPP_OK;
}

// ---------------------------------------------------------------- EDT

size_t iwpp_edt_workspace_bytes(int64_t W, int64_t H, int conn) {
  (void)conn;
  return edt::state_bytes(W, H);
}

static int edt_check(int64_t W, int64_t H, int conn, size_t ws, size_t need) {
  int rc = check_dims(W, H);
  if (rc) return rc;
  if (!edt::size_supported(W, H))
    return set_error(IWPP_E_CONTRACT, "EDT on one device supports up to 65536 x 65535 (got %lld x %lld)",
                     (long long)W, (long long)H);
  if (conn != 4 && conn != 8)
    return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8, got %d", conn);
  if (ws < need) return set_error(IWPP_E_WORKSPACE, "workspace too small (%zu < %zu)", ws, need);
  return IWPP_OK;
}

static int edt_finish(const edt::EdtState &s, iwpp_stats *stats, bool need_inf, cudaStream_t st) {
  if (!stats && !need_inf) return IWPP_OK;
  unsigned long long c[edt::EC_N];
  IWPP_CUDA_TRY(cudaMemcpyAsync(c, s.counters, sizeof c, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  if (stats) {
    memset(stats, 0, sizeof *stats);
    stats->rounds = (int64_t)c[edt::EC_ROUNDS];
    stats->executions = 1;
    stats->queued_total = (int64_t)c[edt::EC_VISITS];
    stats->n_inf = (int64_t)c[edt::EC_NINF];
  }
  if (c[edt::EC_BAD]) return set_error(IWPP_E_CONTRACT, "source map / seeds hold out-of-range indices");
  if (c[edt::EC_LIMIT]) return set_error(IWPP_E_ENGINE_LIMIT, "no fixed point within max_rounds");
  if (need_inf && c[edt::EC_NINF])
    return set_error(IWPP_E_NO_BACKGROUND, "no background reachable: distance map undefined");
  return IWPP_OK;
}

int iwpp_edt(const uint8_t *mask, int64_t W, int64_t H, int conn, int64_t *vr, float *dist,
             void *workspace, size_t workspace_bytes, int64_t max_rounds, iwpp_stats *stats,
             void *stream) {
  int rc = edt_check(W, H, conn, workspace_bytes, edt::state_bytes(W, H));
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  Carver c(workspace);
  edt::EdtState s = edt::carve_state(c, W, H);
  if ((rc = edt::reset_control(s, st))) return rc;
  if ((rc = edt::launch_init(mask, (int)W, (int)H, conn, s, st))) return rc;
  if ((rc = edt::launch_rounds((int)W, (int)H, conn, s, (long long)max_rounds, st))) return rc;
  if ((rc = edt::launch_finalize_auto(s, (int)W, (int)H, vr, dist, nullptr, st))) return rc;
  return edt_finish(s, stats, true, st);
}

int iwpp_edt_propagate(int64_t *vr, int64_t W, int64_t H, int conn, const int64_t *seeds,
                       int64_t n_seeds, void *workspace, size_t workspace_bytes,
                       int64_t max_rounds, iwpp_stats *stats, void *stream) {
  int rc = edt_check(W, H, conn, workspace_bytes, edt::state_bytes(W, H));
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  Carver c(workspace);
  edt::EdtState s = edt::carve_state(c, W, H);
  if ((rc = edt::reset_control(s, st))) return rc;
  if ((rc = edt::launch_import(vr, seeds, n_seeds, (int)W, (int)H, s, st))) return rc;
  if ((rc = edt::launch_rounds((int)W, (int)H, conn, s, (long long)max_rounds, st))) return rc;
  if ((rc = edt::launch_finalize_auto(s, (int)W, (int)H, vr, nullptr, nullptr, st))) return rc;
  return edt_finish(s, stats, false, st);
}

int iwpp_edt_finalize(const int64_t *vr, int64_t W, int64_t H, float *dist, int64_t *d2,
                      void *workspace, void *stream) {
  int rc = check_dims(W, H);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *ctr = (unsigned long long *)workspace;  // EC_N counters
  IWPP_CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * edt::EC_N, st));
  if ((rc = edt::launch_finalize_vr(vr, (int)W, (int)H, dist, d2, ctr, st))) return rc;
  unsigned long long ninf = 0;
  IWPP_CUDA_TRY(cudaMemcpyAsync(&ninf, &ctr[edt::EC_NINF], sizeof ninf, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  if (ninf) return set_error(IWPP_E_NO_BACKGROUND, "no background reachable: distance map undefined");
  return IWPP_OK;
}

size_t iwpp_edt_host_workspace_bytes(int64_t W, int64_t H, int conn) {
  size_t n = (size_t)W * H;
  return align_up(n, 256) + align_up(n * 8, 256) + align_up(n * 4, 256) + edt::state_bytes(W, H) + 256;
}

int iwpp_edt_host(const uint8_t *mask, int64_t W, int64_t H, int conn, int64_t *vr, float *dist,
                  void *workspace, size_t workspace_bytes, int64_t max_rounds, iwpp_stats *stats,
                  void *stream) {
  int rc = edt_check(W, H, conn, workspace_bytes, iwpp_edt_host_workspace_bytes(W, H, conn));
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  size_t n = (size_t)W * H;
  Carver c(workspace);
  uint8_t *dm = c.take<uint8_t>(n);
  int64_t *dvr = c.take<int64_t>(n);
  float *dd = c.take<float>(n);
  edt::EdtState s = edt::carve_state(c, W, H);
  IWPP_CUDA_TRY(cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, st));
  if ((rc = edt::reset_control(s, st))) return rc;
  if ((rc = edt::launch_init(dm, (int)W, (int)H, conn, s, st))) return rc;
  if ((rc = edt::launch_rounds((int)W, (int)H, conn, s, (long long)max_rounds, st))) return rc;
  if ((rc = edt::launch_finalize_auto(s, (int)W, (int)H, dvr, dd, nullptr, st))) return rc;
  if (vr) IWPP_CUDA_TRY(cudaMemcpyAsync(vr, dvr, n * 8, cudaMemcpyDeviceToHost, st));
  if (dist) IWPP_CUDA_TRY(cudaMemcpyAsync(dist, dd, n * 4, cudaMemcpyDeviceToHost, st));
  return edt_finish(s, stats, true, st);
}

}  // extern "C"

// ---------------------------------------------------------------- EDT slabs

extern "C" {

size_t iwpp_edt_slab_workspace_bytes(int64_t W, int64_t h) { return edt::slab_bytes(W, h); }

int iwpp_edt_slab_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H,
                       int conn, int has_up, int has_down, void *workspace, uint64_t *out_up,
                       uint64_t *out_dn, void *stream) {
  int rc = check_dims(W, h);
  if (rc) return rc;
  if (W > 65536 || H > 65536 || y0 < 0 || y0 + h > H)
    return set_error(IWPP_E_CONTRACT, "bad slab geometry");
  if (conn != 4 && conn != 8) return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8");
  return edt::slab_init(mask_ext, W, h, y0, H, conn, has_up, has_down, workspace,
                        (unsigned long long *)out_up, (unsigned long long *)out_dn,
                        (cudaStream_t)stream);
}

int iwpp_edt_slab_round(void *workspace, int64_t W, int64_t h, int64_t y0, int conn, int64_t r,
                        const uint64_t *halo_up, const uint64_t *halo_dn, uint64_t *out_up,
                        uint64_t *out_dn, int64_t *n_next_host, void *stream) {
  return edt::slab_round(workspace, W, h, y0, conn, r, (const unsigned long long *)halo_up,
                         (const unsigned long long *)halo_dn, (unsigned long long *)out_up,
                         (unsigned long long *)out_dn, n_next_host, (cudaStream_t)stream);
}

int iwpp_edt_slab_finalize(void *workspace, int64_t W, int64_t h, int64_t y0, int64_t rounds,
                           int64_t *vr, float *dist, void *stream) {
  int64_t ninf = 0, range = 0;
  int rc = edt::slab_finalize(workspace, W, h, y0, rounds, vr, dist, &ninf, &range,
                              (cudaStream_t)stream);
  if (rc) return rc;
  if (range)
    return set_error(IWPP_E_OVERFLOW, "a squared distance exceeded the 32-bit key range");
  if (ninf) return set_error(IWPP_E_NO_BACKGROUND, "no background reachable: distance map undefined");
  return IWPP_OK;
}

}  // extern "C"
