// capi.cu -- extern "C" entry points of libiwpp_b200.so (include/iwpp_b200.h).

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <chrono>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "edt.cuh"
#include "iwpp_common.cuh"
#include "recon_sweeps.cuh"
#include "recon_tiles.cuh"

namespace iwpp {

static thread_local char g_err[512] = "";

// NVTX ranges around every public entry point (header-only NVTX 3: free
// unless a profiler is attached; `ncu --nvtx --nvtx-include "iwpp_recon/"`
// selects the engine launches of one call)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
constexpr int kMaxSlabs = 256;

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
    case IWPP_BIN: return 1;
    case IWPP_U16: return 2;
    case IWPP_I32: return 4;
    case IWPP_F32: return 4;
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
  (void)conn;
  size_t b = recon_ws_bytes(W, H);
  if (dtype == IWPP_F32) b += align_up((size_t)W * H * 4, 256) + 256;  // the mask as ordered ints
  if (dtype == IWPP_BIN) b += 2 * align_up(recon::bin_plane_words(W, H) * 4, 256) + 256;  // bit planes
  return b;
}

static int fill_recon_stats(const ReconWs &w, iwpp_stats *stats, cudaStream_t st) {
  unsigned long long c[recon::CNT_N];
  IWPP_CUDA_TRY(cudaMemcpyAsync(c, w.counters, sizeof c, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  memset(stats, 0, sizeof *stats);
  stats->executions = 1;
  stats->rounds = (int64_t)c[recon::CNT_ROUNDS];
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
  NvtxRange nvtx_range("iwpp_recon");
  int rc = check_dims(W, H);
  if (rc) return rc;
  if (conn != 4 && conn != 8)
    return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8, got %d", conn);
  if (!elem_size(dtype)) return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
  if (workspace_bytes < iwpp_recon_workspace_bytes(W, H, dtype, conn))
    return set_error(IWPP_E_WORKSPACE, "workspace too small (%zu < %zu)", workspace_bytes,
                     iwpp_recon_workspace_bytes(W, H, dtype, conn));
  cudaStream_t st = (cudaStream_t)stream;
  Carver c(workspace);
  ReconWs w = carve_recon(c, W, H);
  // a separate marker: the plain u8 path hands it to the engine (copied in
  // the fused kernel's prologue); everything else starts from a copy in J
  const void *msrc = opts && opts->marker != J ? opts->marker : nullptr;
  // (binary: the bit planes are packed straight from the marker)
  if (msrc && !((dtype == IWPP_U8 || dtype == IWPP_BIN) && (!opts || (opts->sweeps <= 0 && !opts->slab_rows)))) {
    IWPP_CUDA_TRY(cudaMemcpyAsync(J, msrc, (size_t)W * H * elem_size(dtype), cudaMemcpyDeviceToDevice, st));
    msrc = nullptr;
  }
  // f32: the 32-bit register engine orders the float bits as it stages its
  // boxes (no conversion passes); other engine choices run the int32 engine
  // on converted copies
  bool f32_fused = false;
  if (dtype == IWPP_F32) {
    recon::EngineOpts probe;
    if (opts) {
      probe.qcap = opts->queue_capacity;
      probe.sweeps_set = opts->tile_sweeps >= 0;
      probe.engine = opts->engine;
    }
    f32_fused = (!opts || (opts->sweeps <= 0 && !opts->slab_rows)) && recon::f32_in_engine(probe);
  }
  if (dtype == IWPP_F32 && !f32_fused) {  // int32 engine on order-preserving ints, then back
    const size_t n = (size_t)W * H;
    void *Io = c.take<int32_t>(n);
    if ((rc = recon::f32_to_ord(J, J, n, st))) return rc;
    if ((rc = recon::f32_to_ord(I, Io, n, st))) return rc;
    iwpp_recon_opts o{};
    if (opts) o = *opts;
    else o.sweeps = o.tile_sweeps = o.halo_sweep_threshold = -1;
    o.marker = nullptr;  // (copied above)
    rc = iwpp_recon(J, Io, W, H, IWPP_I32, conn, workspace, recon_ws_bytes(W, H), &o, stats, stream);
    int rc2 = recon::ord_to_f32(J, J, n, st);
    return rc ? rc : rc2;
  }
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
    if (opts->tile_sweeps >= 0) {
      eo.sweeps = opts->tile_sweeps;
      eo.sweeps_set = 1;
    }
    eo.engine = opts->engine;
    eo.halo_thresh = opts->halo_sweep_threshold;
    eo.ev_begin = opts->ev_begin;
    eo.ev_end = opts->ev_end;
    eo.rows_mode = opts->slab_rows & 3;
    eo.max_rounds = opts->max_rounds > 0 ? opts->max_rounds : 0;
  }
  eo.src = msrc;
  if (dtype == IWPP_BIN && recon::tile_side(IWPP_BIN, eo) != recon::TSB)
    dtype = IWPP_U8;  // a byte engine was asked for: 0 / 255 is ordinary grey data
  if (dtype == IWPP_BIN) {  // the bit-plane engine: pack, propagate, unpack
    const size_t nw = recon::bin_plane_words(W, H);
    uint32_t *Jb = c.take<uint32_t>(nw), *Ib = c.take<uint32_t>(nw);
    if ((rc = recon::bin_pack(msrc ? msrc : J, (int)W, (int)H, Jb, st, I, Ib))) return rc;
    eo.src = nullptr;  // (J is written whole by the unpack)
    if ((rc = recon::run_tile_engine(Jb, Ib, (int)W, (int)H, IWPP_BIN, conn, w.q, w.counters, eo, st)))
      return rc;
    if ((rc = recon::bin_unpack(Jb, (int)W, (int)H, J, st))) return rc;
  } else if ((rc = recon::run_tile_engine(J, I, (int)W, (int)H, dtype, conn, w.q, w.counters, eo,
                                          st))) {
    return rc;
  }
  if (opts && opts->check_contract) {
    if ((rc = recon::check_le(J, I, (size_t)W * H, dtype, &w.counters[recon::CNT_VIOL], st)))
      return rc;
  }
  if (eo.max_rounds > 0) {  // the round engine stopped with work left (engine.py:311-317)
    unsigned long long lim = 0;
    IWPP_CUDA_TRY(cudaMemcpyAsync(&lim, &w.counters[recon::CNT_LIMIT], sizeof lim,
                                  cudaMemcpyDeviceToHost, st));
    IWPP_CUDA_TRY(cudaStreamSynchronize(st));
    if (lim) return set_error(IWPP_E_ENGINE_LIMIT, "no fixed point within %d rounds", eo.max_rounds);
  }
  if (stats) return fill_recon_stats(w, stats, st);
  return IWPP_OK;
}

size_t iwpp_recon_host_workspace_bytes(int64_t W, int64_t H, int dtype, int conn) {
  (void)conn;
  size_t img = align_up((size_t)W * H * elem_size(dtype), 256);
  size_t nty = (size_t)((H + recon::TS - 1) / recon::TS);
  // the device call runs on the copies (f32 is converted in place first)
  const size_t inner = iwpp_recon_workspace_bytes(W, H, dtype == IWPP_F32 ? IWPP_I32 : dtype, conn);
  // + one violation counter of its own (the engine resets its counter block
  // at every pipelined run, so check_le must not count into CNT_VIOL there)
  return 2 * img + align_up(nty, 256) + 256 + inner + 512;
}

}  // extern "C"

namespace iwpp {

// Copy streams + events of the pipelined host path, one set per device
// (created on first use; host calls on one device are serialised).
struct HostPipe {
  std::mutex m;
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t start = nullptr, in[kMaxSlabs], ready[kMaxSlabs];
};

static int host_pipe(HostPipe *&hp) {
  static HostPipe pipes[64];
  int dev = 0;
  IWPP_CUDA_TRY(cudaGetDevice(&dev));
  hp = &pipes[dev & 63];
  return IWPP_OK;
}

static int host_pipe_init(HostPipe &p) {
  if (p.h2d) return IWPP_OK;
  IWPP_CUDA_TRY(cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking));
  IWPP_CUDA_TRY(cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking));
  IWPP_CUDA_TRY(cudaEventCreateWithFlags(&p.start, cudaEventDisableTiming));
  for (int i = 0; i < kMaxSlabs; i++) {
    IWPP_CUDA_TRY(cudaEventCreateWithFlags(&p.in[i], cudaEventDisableTiming));
    IWPP_CUDA_TRY(cudaEventCreateWithFlags(&p.ready[i], cudaEventDisableTiming));
  }
  return IWPP_OK;
}

// Slab row bounds for the pipelined host path: slabs of ~4 MB of each image
// (a multiple of the tile side, at least 8 tile rows), the last two tapered
// to 1/2 and 1/4 of that so the compute + copy-back after the final H2D is
// short.  `rows` > 0 forces uniform slabs of that height.  Returns false
// (no pipelining) when the image is too small for two slabs.
static bool host_slabs(int64_t W, int64_t H, size_t es, int64_t rows, std::vector<int64_t> &b) {
  const int64_t TS = recon::TSB;  // cuts on every engine's tile grid
  b.clear();
  bool taper = rows <= 0;
  if (rows <= 0) {
    double mb = 4.0;
    if (const char *e = getenv("IWPP_SLAB_MB")) mb = atof(e);  // diagnostics
    rows = (int64_t)(mb * (1 << 20) / ((double)W * es));
    if (rows < 8 * TS) rows = 8 * TS;
  }
  rows = (rows + TS - 1) / TS * TS;
  while ((H + rows - 1) / rows > kMaxSlabs - 2) rows *= 2;
  if (H < 2 * rows) return false;
  b.push_back(0);
  int64_t tail = 0;
  std::vector<int64_t> last;
  if (taper) {
    std::vector<int64_t> parts = {rows / 4, rows / 2};
    if (const char *e = getenv("IWPP_TAPER")) {  // diagnostics: divisors, smallest slab first
      parts.clear();
      for (const char *q = e; *q;) {
        int d = atoi(q);
        if (d > 0) parts.push_back(rows / d);
        while (*q && *q != ',') q++;
        if (*q == ',') q++;
      }
    }
    for (int64_t part : parts) {
      part = std::max<int64_t>(TS, part / TS * TS);
      if (H - tail - part >= rows) {
        last.push_back(part);
        tail += part;
      }
    }
  }
  for (int64_t y = rows; y + rows / 2 < H - tail; y += rows) b.push_back(y);
  int64_t y = H - tail;
  for (auto it = last.rbegin(); it != last.rend(); ++it) {
    b.push_back(y);
    y += *it;
  }
  b.push_back(H);
  return b.size() >= 3;
}

// Optional timeline of the pipelined host path (IWPP_TRACE=1 in the
// environment): a one-thread kernel on each stream stamps %globaltimer when
// the stream reaches it; printed to stderr at the end (diagnostics only).
// The host path's last transfer, when the output buffer is page-locked and
// mapped: the last slab's rows and every tile row a later run re-wrote
// (dirty), written straight into host memory by the SMs.  One kernel
// instead of a D2H copy, a host read of the dirty flags and the recopies.
// gridDim.x = tile rows, gridDim.y CTAs share one; 16-byte stores when rows
// allow.
__global__ void recopy_mapped_kernel(const char *__restrict__ dJ, char *out, const uint8_t *__restrict__ dirty,
                                     int64_t H, int64_t TS, size_t row_bytes, int64_t y_last) {
  const int64_t t = blockIdx.x, r0 = t * TS, r1 = r0 + TS < H ? r0 + TS : H;
  if (r1 <= y_last && !dirty[t]) return;
  const size_t off = (size_t)r0 * row_bytes, nb = (size_t)(r1 - r0) * row_bytes;
  const size_t tid = (size_t)blockIdx.y * blockDim.x + threadIdx.x, nt = (size_t)gridDim.y * blockDim.x;
  if (((uintptr_t)(dJ + off) | (uintptr_t)(out + off) | nb) % 16 == 0) {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(dJ + off);
    uint4 *d4 = reinterpret_cast<uint4 *>(out + off);
    for (size_t i = tid; i < nb / 16; i += nt) d4[i] = __ldcg(s4 + i);
  } else {
    for (size_t i = tid; i < nb; i += nt) out[off + i] = dJ[off + i];
  }
}

__global__ void trace_stamp_kernel(unsigned long long *slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *slot = t;
}

struct Trace {
  bool on = false;
  int n = 0;
  const char *what[256];
  int idx[256];
  unsigned long long *dev = nullptr;
  Trace() {
    const char *e = getenv("IWPP_TRACE");
    on = e && e[0] == '1' && cudaMalloc(&dev, 256 * sizeof(unsigned long long)) == cudaSuccess;
  }
  void mark(cudaStream_t s, const char *w, int i) {
    if (!on || n >= 256) return;
    what[n] = w;
    idx[n] = i;
    trace_stamp_kernel<<<1, 1, 0, s>>>(dev + n);
    n++;
  }
  ~Trace() {
    if (!on) return;
    unsigned long long t[256];
    cudaDeviceSynchronize();
    cudaMemcpy(t, dev, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost);
    for (int i = 0; i < n; i++)
      fprintf(stderr, "[iwpp trace] %8.3f ms  %s %d\n", (double)(t[i] - t[0]) * 1e-6, what[i], idx[i]);
    cudaFree(dev);
  }
};

// Pipelined e2e reconstruction (the reference-facing host call).
//
// The image streams in as horizontal slabs on a copy stream.  As soon as
// slab k lands, one engine run over rows [0, end of slab k) processes the
// slab's tiles and re-visits the tile row above its top cut: rows not yet
// landed lie outside that run's image, so every intermediate state lies
// between the marker and the true result, and each run carries raises across
// the cut and on to wherever they reach (the fixed point is unique,
// engine.py:9-18).  Once the cut below a slab has been crossed the slab is
// copied back speculatively on a second copy stream while later slabs are
// still arriving; every tile row a later run writes is flagged and copied
// again at the end.  Transfers in both directions overlap the
// compute, so the call costs ~ max(H2D, D2H) + one slab's compute.
static int recon_host_pipelined(char *out, const char *marker, const char *mask, int64_t W,
                                int64_t H, int dtype, int conn, const std::vector<int64_t> &bnd, char *dJ,
                                char *dI, uint8_t *dirty, unsigned long long *vctr, char *rest,
                                const iwpp_recon_opts *opts, iwpp_stats *stats,
                                cudaStream_t st) {
  HostPipe *hp;
  int rc = host_pipe(hp);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(hp->m);
  if ((rc = host_pipe_init(*hp))) return rc;
  const size_t es = elem_size(dtype), row_bytes = (size_t)W * es;
  const int S = (int)bnd.size() - 1;
  Carver c2(rest);
  ReconWs w = carve_recon(c2, W, H);
  recon::EngineOpts eo;
  if (opts) {
    eo.max_blocks = opts->max_blocks;
    eo.qcap = opts->queue_capacity;
    if (opts->tile_sweeps >= 0) {
      eo.sweeps = opts->tile_sweeps;
      eo.sweeps_set = 1;
    }
    eo.engine = opts->engine;
    eo.halo_thresh = opts->halo_sweep_threshold;
  }
  // the engine's tile rows: slab cuts (multiples of TSB) fall on them
  const int64_t TS = recon::tile_side(dtype, eo), nty = (H + TS - 1) / TS;
  // a page-locked, mapped output takes the last transfer from the SMs
  // (IWPP_E2E_MAPPED=0: copies only)
  char *out_dev = nullptr;
  {
    static int mapped_env = -1;
    if (mapped_env < 0) mapped_env = getenv("IWPP_E2E_MAPPED") ? atoi(getenv("IWPP_E2E_MAPPED")) : 1;
    cudaPointerAttributes pa;
    if (mapped_env && cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer)
      out_dev = static_cast<char *>(pa.devicePointer);
    (void)cudaGetLastError();
  }
  Trace tr;
  tr.mark(st, "start", 0);
  IWPP_CUDA_TRY(cudaEventRecord(hp->start, st));
  IWPP_CUDA_TRY(cudaStreamWaitEvent(hp->h2d, hp->start, 0));
  IWPP_CUDA_TRY(cudaStreamWaitEvent(hp->d2h, hp->start, 0));
  for (int k = 0; k < S; k++) {
    size_t off = (size_t)bnd[k] * row_bytes;
    size_t nb = (size_t)(bnd[k + 1] - bnd[k]) * row_bytes;
    IWPP_CUDA_TRY(cudaMemcpyAsync(dJ + off, marker + off, nb, cudaMemcpyHostToDevice, hp->h2d));
    IWPP_CUDA_TRY(cudaMemcpyAsync(dI + off, mask + off, nb, cudaMemcpyHostToDevice, hp->h2d));
    IWPP_CUDA_TRY(cudaEventRecord(hp->in[k], hp->h2d));
    tr.mark(hp->h2d, "h2d done", k);
  }
  IWPP_CUDA_TRY(cudaMemsetAsync(vctr, 0, sizeof(unsigned long long), st));
  IWPP_CUDA_TRY(cudaMemsetAsync(dirty, 0, (size_t)nty, st));
  auto copy_back = [&](int64_t r0, int64_t r1) -> int {  // rows [r0, r1) -> host (d2h)
    size_t off = (size_t)r0 * row_bytes;
    IWPP_CUDA_TRY(cudaMemcpyAsync(out + off, dJ + off, (size_t)(r1 - r0) * row_bytes,
                                  cudaMemcpyDeviceToHost, hp->d2h));
    return IWPP_OK;
  };
  for (int k = 0; k < S; k++) {
    const int64_t y0 = bnd[k], y1 = bnd[k + 1];
    size_t off = (size_t)y0 * row_bytes;
    IWPP_CUDA_TRY(cudaStreamWaitEvent(st, hp->in[k], 0));
    tr.mark(st, "compute begin", k);
    if ((rc = recon::check_le(dJ + off, dI + off, (size_t)(y1 - y0) * W, dtype, vctr, st)))
      return rc;
    // Rows [0, y1): the slab's tiles (first visits) plus the tile row above
    // the cut at y0 (re-visited with the slab's rows as its halo); a raise
    // may run on into any earlier slab, so tile rows written are flagged.
    // Rows below y1 have not landed: for this run they lie outside the image.
    recon::EngineOpts so = eo;
    so.init_mode = k == 0 ? recon::INIT_FULL : recon::INIT_CONTINUE;
    so.keep_counters = k > 0;
    so.sel_lo = k == 0 ? 0 : (int)(y0 / TS) - 1;
    so.sel_hi = -1;
    so.dirty = dirty;
    if ((rc = recon::run_tile_engine(dJ, dI, (int)W, (int)y1, dtype, conn, w.q, w.counters, so, st)))
      return rc;
    tr.mark(st, "engine done", k);
    // slab k as this run left it goes back now: clear its flags first, so
    // every tile row a later run rewrites (the row above the next cut, and
    // any raise that runs on upward) is flagged and copied again at the end
    // (a copy that races with such a run is superseded by that recopy).
    // Copying right after the slab's own run, not after the next one, takes
    // one run off the transfer tail.
    const int64_t p0 = y0, p1 = k == S - 1 ? H : y1;
    if (out_dev && k == S - 1) {
      // the last slab and the re-written rows, from the SMs, after every
      // earlier copy of those rows has landed (a stale copy must not
      // overwrite a recopy)
      IWPP_CUDA_TRY(cudaEventRecord(hp->ready[k], hp->d2h));
      IWPP_CUDA_TRY(cudaStreamWaitEvent(st, hp->ready[k], 0));
      {
        static int gy = 0;
        if (!gy) gy = getenv("IWPP_MAPPED_SPLIT") ? atoi(getenv("IWPP_MAPPED_SPLIT")) : 8;
        recopy_mapped_kernel<<<dim3((unsigned)nty, (unsigned)gy), 256, 0, st>>>(dJ, out_dev, dirty, H, TS,
                                                                                 row_bytes, y0);
      }
      IWPP_CUDA_TRY(cudaGetLastError());
      tr.mark(st, "mapped copy done", k);
      break;
    }
    IWPP_CUDA_TRY(cudaMemsetAsync(dirty + p0 / TS, 0, (size_t)((p1 + TS - 1) / TS - p0 / TS), st));
    IWPP_CUDA_TRY(cudaEventRecord(hp->ready[k], st));
    IWPP_CUDA_TRY(cudaStreamWaitEvent(hp->d2h, hp->ready[k], 0));
    if ((rc = copy_back(p0, p1))) return rc;
    tr.mark(hp->d2h, "d2h done", k);
  }
  unsigned long long viol = 0;
  if (out_dev) {
    IWPP_CUDA_TRY(cudaMemcpyAsync(&viol, vctr, sizeof viol, cudaMemcpyDeviceToHost, st));
    IWPP_CUDA_TRY(cudaStreamSynchronize(st));
    tr.mark(st, "done", 0);
    if (viol) return set_error(IWPP_E_CONTRACT, "marker exceeds mask somewhere (%llu cells)", viol);
    if (stats) return fill_recon_stats(w, stats, st);
    return IWPP_OK;
  }
  // tile rows written after their slab was copied: copy them again
  std::vector<uint8_t> flags((size_t)nty);
  IWPP_CUDA_TRY(cudaMemcpyAsync(flags.data(), dirty, (size_t)nty, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaMemcpyAsync(&viol, vctr, sizeof viol, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  tr.mark(st, "flags read", 0);
  for (int64_t t = 0; t < nty;) {
    if (!flags[t]) {
      t++;
      continue;
    }
    int64_t e = t;
    while (e < nty && flags[e]) e++;
    if ((rc = copy_back(t * TS, std::min<int64_t>(H, e * TS)))) return rc;
    t = e;
  }
  tr.mark(hp->d2h, "recopy done", 0);
  IWPP_CUDA_TRY(cudaStreamSynchronize(hp->d2h));
  if (viol) return set_error(IWPP_E_CONTRACT, "marker exceeds mask somewhere (%llu cells)", viol);
  if (stats) return fill_recon_stats(w, stats, st);
  return IWPP_OK;
}

}  // namespace iwpp

extern "C" {

int iwpp_recon_host(void *out, const void *marker, const void *mask, int64_t W, int64_t H,
                    int dtype, int conn, void *workspace, size_t workspace_bytes,
                    const iwpp_recon_opts *opts, iwpp_stats *stats, void *stream) {
  NvtxRange nvtx_range("iwpp_recon_host");
  int rc = check_dims(W, H);
  if (rc) return rc;
  size_t es = elem_size(dtype);
  if (!es) return set_error(IWPP_E_CONTRACT, "unsupported dtype %d", dtype);
  if (conn != 4 && conn != 8)
    return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8, got %d", conn);
  if (workspace_bytes < iwpp_recon_host_workspace_bytes(W, H, dtype, conn))
    return set_error(IWPP_E_WORKSPACE, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  size_t nb = (size_t)W * H * es;
  Carver c(workspace);
  char *dJ = c.take<char>(nb);
  char *dI = c.take<char>(nb);
  uint8_t *dirty = c.take<uint8_t>((size_t)((H + recon::TS - 1) / recon::TS));
  unsigned long long *vctr = c.take<unsigned long long>(1);
  char *rest = c.base + align_up(c.off, 256);
  size_t rest_bytes = workspace_bytes - align_up(c.off, 256);
  std::vector<int64_t> bnd;
  const bool pipelined =
      dtype != IWPP_F32 && dtype != IWPP_BIN &&
      !(opts && (opts->sweeps > 0 || opts->slab_rows || opts->pipeline_rows < 0)) &&
      host_slabs(W, H, es, opts ? opts->pipeline_rows : 0, bnd);
  if (pipelined)
    return recon_host_pipelined((char *)out, (const char *)marker, (const char *)mask, W, H, dtype,
                                conn, bnd, dJ, dI, dirty, vctr, rest, opts, stats, st);
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
  iwpp_recon_opts o{};
  if (opts) o = *opts;
  else o.sweeps = o.tile_sweeps = o.halo_sweep_threshold = -1;
  o.check_contract = 0;
  o.marker = nullptr;  // (the marker is the host buffer, uploaded into dJ)
  int edtype = dtype;
  if (dtype == IWPP_F32) {  // our own device copies: convert in place
    if ((rc = recon::f32_to_ord(dJ, dJ, (size_t)W * H, st))) return rc;
    if ((rc = recon::f32_to_ord(dI, dI, (size_t)W * H, st))) return rc;
    edtype = IWPP_I32;
  }
  if ((rc = iwpp_recon(dJ, dI, W, H, edtype, conn, rest, rest_bytes, &o, nullptr, stream))) return rc;
  if (dtype == IWPP_F32 && (rc = recon::ord_to_f32(dJ, dJ, (size_t)W * H, st))) return rc;
  (void)0;
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

int iwpp_debug_atrace(void *buf, uint32_t cap, uint32_t *n_out) {
  return recon::atrace_control(buf, cap, n_out);
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

int iwpp_recon_pass(void *J, const void *I, int64_t W, int64_t H, int dtype, int conn, int pass,
                    int64_t *seeds, int64_t *n_seeds_host, int *changed_host, void *workspace,
                    void *stream) {
  NvtxRange nvtx_range("iwpp_recon_pass");
  int rc = check_dims(W, H);
  if (rc) return rc;
  if (conn != 4 && conn != 8)
    return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8, got %d", conn);
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long *ctr = (unsigned long long *)workspace;
  IWPP_CUDA_TRY(cudaMemsetAsync(ctr, 0, 2 * sizeof *ctr, st));
  if (dtype == IWPP_F32) {  // the passes on order-preserving ints, converted in place
    const size_t n = (size_t)W * H;
    int32_t *Io = (int32_t *)((char *)workspace + 256);
    if ((rc = recon::f32_to_ord(J, J, n, st))) return rc;
    if ((rc = recon::f32_to_ord(I, Io, n, st))) return rc;
    rc = iwpp_recon_pass(J, Io, W, H, IWPP_I32, conn, pass, seeds, n_seeds_host, changed_host,
                         workspace, stream);
    const int rc2 = recon::ord_to_f32(J, J, n, st);
    return rc ? rc : rc2;
  }
  switch (pass) {
    case IWPP_PASS_RASTER:
      rc = recon::line_pass(J, I, (int)W, (int)H, dtype, conn, 0, nullptr, ctr, st);
      break;
    case IWPP_PASS_ANTIRASTER:
      rc = recon::line_pass(J, I, (int)W, (int)H, dtype, conn, 1, seeds, ctr, st);
      break;
    case IWPP_PASS_COLS_FWD:
      rc = recon::line_pass(J, I, (int)W, (int)H, dtype, conn, 2, nullptr, ctr, st);
      break;
    case IWPP_PASS_COLS_BWD:
      rc = recon::line_pass(J, I, (int)W, (int)H, dtype, conn, 3, nullptr, ctr, st);
      break;
    case IWPP_PASS_ROWS_FWD:
    case IWPP_PASS_ROWS_BWD:
      rc = recon::sweep_rows(J, I, (int)W, (int)H, dtype, st, pass == IWPP_PASS_ROWS_FWD ? 1 : 2,
                             ctr);
      break;
    default:
      return set_error(IWPP_E_CONTRACT, "unknown pass %d", pass);
  }
  if (rc) return rc;
  unsigned long long v[2] = {0, 0};
  IWPP_CUDA_TRY(cudaMemcpyAsync(v, ctr, sizeof v, cudaMemcpyDeviceToHost, st));
  IWPP_CUDA_TRY(cudaStreamSynchronize(st));
  if (changed_host) *changed_host = (int)v[0];
  if (n_seeds_host) *n_seeds_host = (int64_t)v[1];
  return IWPP_OK;
}

size_t iwpp_recon_pass_workspace_bytes(int64_t W, int64_t H, int dtype) {
  return 256 + (dtype == IWPP_F32 ? (size_t)W * H * 4 : 0);
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
    return set_error(IWPP_E_CONTRACT, "EDT on one device supports up to 65536 x 65536 (got %lld x %lld)",
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

}  // extern "C"

namespace iwpp {

// init (from a mask, or from a user source map + seeds) + all rounds.  On
// images whose squared distances may exceed 32 bits the key engine runs with
// range-checked offers; if any offer was out of range it re-runs on the CAS
// engine (same workspace).  `s` returns the state holding the result.
static int edt_solve(edt::EdtState &s, void *workspace, int64_t W, int64_t H, int conn,
                     const uint8_t *mask, const int64_t *vr_in, const int64_t *seeds,
                     int64_t n_seeds, int64_t max_rounds, cudaStream_t st) {
  int rc;
  for (int attempt = 0; attempt < 2; attempt++) {
    Carver c(workspace);
    s = edt::carve_state(c, W, H, attempt == 1);
    if (!s.keymode && !edt::cas_supported(W, H))  // (a forced CAS run at 65536^2)
      return set_error(IWPP_E_CONTRACT,
                       "the 32-bit-source engine has no free 'no source' code at %lld x %lld",
                       (long long)W, (long long)H);
    if ((rc = edt::reset_control(s, st))) return rc;
    int r0 = 0;  // 1: round 0 ran inside the init
    if (s.block)
      rc = edt::block_init(mask, vr_in, seeds, n_seeds, (int)W, (int)H, conn, s, st);
    else if (mask)
      rc = edt::launch_init(mask, (int)W, (int)H, conn, s, st, &r0);
    else
      rc = edt::launch_import(vr_in, seeds, n_seeds, (int)W, (int)H, s, st);
    if (rc) return rc;
    if (s.block)
      rc = edt::block_rounds((int)W, (int)H, conn, s, (long long)max_rounds, st);
    else
      rc = edt::launch_rounds((int)W, (int)H, conn, s, (long long)max_rounds, st, r0);
    if (rc) return rc;
    if (s.block && getenv("IWPP_TRACE") && getenv("IWPP_TRACE")[0] == '1') {
      unsigned long long d[16];
      cudaMemcpy(d, s.diag, sizeof d, cudaMemcpyDeviceToHost);
      fprintf(stderr,
              "[iwpp edt block] region-passes %llu (empty %llu, with frontier out %llu) items %llu "
              "local-rounds %llu rounds %llu | cycles/region-pass load %.0f rounds %.0f out %.0f\n",
              d[0], d[1], d[7], d[2], d[3], d[8], (double)d[4] / (d[0] - d[1] + 1e-9),
              (double)d[5] / (d[0] - d[1] + 1e-9), (double)d[6] / (d[0] - d[1] + 1e-9));
    }
    if (!s.keycheck) return IWPP_OK;
    unsigned long long c8[edt::EC_N];
    if ((rc = edt::read_counters(s, c8, st))) return rc;
    if (!c8[edt::EC_RANGE]) return IWPP_OK;
    if (!edt::cas_supported(W, H))
      return set_error(IWPP_E_OVERFLOW,
                       "a squared distance exceeds 32 bits and the %lld x %lld image leaves no "
                       "free source code for the CAS engine",
                       (long long)W, (long long)H);
  }
  return IWPP_OK;
}

}  // namespace iwpp

extern "C" {

int iwpp_edt_set_engine(int mode) {
  if (mode < edt::ENGINE_AUTO || mode > edt::ENGINE_RASTER)
    return set_error(IWPP_E_CONTRACT, "unknown EDT engine mode %d", mode);
  edt::g_engine_override = mode;
  return IWPP_OK;
}

int iwpp_edt(const uint8_t *mask, int64_t W, int64_t H, int conn, int64_t *vr, float *dist,
             void *workspace, size_t workspace_bytes, int64_t max_rounds, iwpp_stats *stats,
             void *stream) {
  NvtxRange nvtx_range("iwpp_edt");
  int rc = edt_check(W, H, conn, workspace_bytes, edt::state_bytes(W, H));
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  edt::EdtState s;
  if ((rc = edt_solve(s, workspace, W, H, conn, mask, nullptr, nullptr, 0, max_rounds, st)))
    return rc;
  if ((rc = edt::launch_finalize_auto(s, (int)W, (int)H, vr, dist, nullptr, st))) return rc;
  return edt_finish(s, stats, true, st);
}

int iwpp_edt_propagate(int64_t *vr, int64_t W, int64_t H, int conn, const int64_t *seeds,
                       int64_t n_seeds, void *workspace, size_t workspace_bytes,
                       int64_t max_rounds, iwpp_stats *stats, void *stream) {
  NvtxRange nvtx_range("iwpp_edt_propagate");
  int rc = edt_check(W, H, conn, workspace_bytes, edt::state_bytes(W, H));
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  edt::EdtState s;
  if ((rc = edt_solve(s, workspace, W, H, conn, nullptr, vr, seeds, n_seeds, max_rounds, st)))
    return rc;
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
  NvtxRange nvtx_range("iwpp_edt_host");
  int rc = edt_check(W, H, conn, workspace_bytes, iwpp_edt_host_workspace_bytes(W, H, conn));
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  size_t n = (size_t)W * H;
  Carver c(workspace);
  uint8_t *dm = c.take<uint8_t>(n);
  int64_t *dvr = c.take<int64_t>(n);
  float *dd = c.take<float>(n);
  char *rest = c.base + align_up(c.off, 256);
  IWPP_CUDA_TRY(cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, st));
  edt::EdtState s;
  if ((rc = edt_solve(s, rest, W, H, conn, dm, nullptr, nullptr, 0, max_rounds, st))) return rc;
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
  NvtxRange nvtx_range("iwpp_edt_slab_round");
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

size_t iwpp_edt_mg_workspace_bytes(int64_t W, int64_t h) { return edt::mg_slab_bytes(W, h); }
size_t iwpp_edt_mg_mailbox_bytes(int64_t W) { return edt::mg_mailbox_bytes(W); }

int iwpp_edt_mg_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H, int conn,
                     int has_up, int has_down, void *workspace, void *mailbox_up, void *mailbox_down,
                     void *stream) {
  int rc = check_dims(W, h);
  if (rc) return rc;
  if (W > 65536 || H > 65536 || y0 < 0 || y0 + h > H)
    return set_error(IWPP_E_CONTRACT, "bad slab geometry");
  if (conn != 4 && conn != 8) return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8");
  if ((has_up && !mailbox_up) || (has_down && !mailbox_down))
    return set_error(IWPP_E_CONTRACT, "a neighbour's mailbox is missing");
  return edt::mg_init(mask_ext, W, h, y0, H, conn, has_up, has_down, workspace, nullptr,
                      has_up ? mailbox_up : nullptr, has_down ? mailbox_down : nullptr,
                      (cudaStream_t)stream);
}

int iwpp_edt_mg_run(const iwpp_edt_mg_slab *slabs, int n_local, int conn, int64_t max_rounds,
                    int64_t *rounds, void *stream) {
  NvtxRange nvtx_range("iwpp_edt_mg_run");
  if (!slabs) return set_error(IWPP_E_CONTRACT, "no slabs");
  if (conn != 4 && conn != 8) return set_error(IWPP_E_CONTRACT, "connectivity must be 4 or 8");
  return edt::mg_run(slabs, n_local, conn, max_rounds, rounds, (cudaStream_t)stream);
}

}  // extern "C"
