/*
 * iwpp_b200.h -- C ABI of the B200-native IWPP library (libiwpp_b200.so).
 *
 * Drop-in boundary for the hot path of the reference package "gridwave"
 * (/root/reference/pkg/src/gridwave).  The reference has no C ABI: its
 * "native" layer is numba-JIT kernels called from Python
 * (_kernels.py, cited K.<line>).  Each entry point below replaces one
 * reference call (file:line given per function); the Python package
 * paper_1209_3314_b200 binds these with ctypes exactly where the
 * reference's operators call their kernels.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Image buffers are row-major (H, W),
 *    C-contiguous, DEVICE pointers unless the function name ends in _host.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  All work is enqueued on it; a function synchronizes the
 *    stream only when it must return a host-visible result (stats != NULL,
 *    *_host variants, error flags).
 *  - Scratch memory is caller-owned: query *_workspace_bytes(), allocate
 *    that many bytes of device memory (256-byte aligned), pass it in.
 *    The library never allocates device memory itself.
 *  - Return value: IWPP_OK (0) or a negative IWPP_E* status;
 *    iwpp_last_error() returns a thread-local message for the last failure.
 *    The Python layer maps statuses onto the reference's exceptions
 *    (errors.py:4-25): CONTRACT -> ContractViolation,
 *    NO_BACKGROUND -> NoBackgroundError, ENGINE_LIMIT -> EngineError.
 */
#ifndef IWPP_B200_H
#define IWPP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element kinds (grid.py:22-27 plus int32) */
enum iwpp_dtype {
  IWPP_U8 = 0,  /* "u8" and "binary" */
  IWPP_U16 = 1, /* "u16" */
  IWPP_I32 = 2, /* "i32" (not an Image2D kind in the reference; its kernels accept it) */
  IWPP_F32 = 3, /* "f32": runs the int32 engine on an order-preserving bit map of the
                   floats (-0.0 is taken as +0.0; NaN fails the marker <= mask contract) */
  IWPP_BIN = 4, /* "binary": u8 storage holding only 0 / 255 (grid.py binary); runs a
                   one-bit-per-pixel engine.  Other byte values are read as 255 */
};

enum iwpp_status {
  IWPP_OK = 0,
  IWPP_E_CONTRACT = -1,      /* precondition violated (marker > mask, bad dims/kind/conn) */
  IWPP_E_NO_BACKGROUND = -2, /* EDT finalize saw an unassigned cell (edt.py:275-276) */
  IWPP_E_ENGINE_LIMIT = -3,  /* max_rounds exceeded (engine.py:311-317) */
  IWPP_E_CUDA = -4,          /* CUDA runtime error */
  IWPP_E_WORKSPACE = -5,     /* workspace too small */
  IWPP_E_OVERFLOW = -6,      /* queue overflow not resolved by rescans */
};

/* Counters mirrored from RunStats (engine.py:46-59) plus device-engine
 * counters.  Filled only when a non-NULL pointer is passed (forces a sync). */
typedef struct iwpp_stats {
  int64_t rounds;          /* EDT: two-phase rounds; recon: tile rounds of the round engine
                              (engine 3), 0 for the asynchronous tile-queue engines */
  int64_t executions;      /* engine executions (overflow re-runs included) */
  int64_t overflow_count;  /* block-queue overflows resolved by an in-tile rescan */
  int64_t queued_total;    /* queue insertions (pixels) */
  int64_t seeds;           /* initial wavefront size (pixels) */
  int64_t tiles_processed; /* recon: tile activations (incl. re-runs) */
  int64_t tile_reruns;     /* recon: activations caused by a neighbour's border change */
  int64_t contract_violations; /* recon: cells with marker > mask seen by the engine */
  int64_t n_inf;           /* EDT: cells left without a source */
} iwpp_stats;

/* ---- library -------------------------------------------------------- */
const char *iwpp_last_error(void);
const char *iwpp_version(void);
/* Device properties the engines size themselves by (SM count etc.). */
int iwpp_device_info(int device, int *sm_count, int *cc_major, int *cc_minor);

/* ---- morphological reconstruction by dilation -----------------------
 * Replaces recon_fh / recon_sr / recon_qb / recon_parallel / recon_tiled
 * (recon.py:164-342): their common fixed point is unique, so every entry
 * routes to one device engine.  J (marker in, result out, in place) and I
 * (mask) are device buffers of `dtype`.  conn is 4 or 8.
 * The engine = row/column clamp-scan sweeps (K.115-190 semantics) +
 * persistent tile engine (in-tile seed detection K.193-217, warp-aggregated
 * shared-memory queue propagation K.220-270 semantics, global tile queue).
 */
typedef struct iwpp_recon_opts {
  int sweeps;        /* full-image row/col sweep pairs before the tile engine (-1 = auto) */
  int max_blocks;    /* persistent grid size cap (0 = auto) */
  int check_contract;/* 1: count cells with marker > mask (stats->contract_violations) */
  int queue_capacity;/* block-queue capacity (0 = default 4608); smaller values force the
                        overflow -> rescan path (QueueConfig.gbq_capacity, wqueue.py:58-60) */
  int tile_sweeps;   /* in-tile row/column sweep passes on a tile's first visit (-1 = auto) */
  int halo_sweep_threshold; /* re-visit: sweep when more halo pixels than this are active (-1 = auto) */
  void *ev_begin;    /* optional events (iwpp_event_create) recorded on the stream */
  void *ev_end;      /* right before / after the tile-engine kernel (roofline timing) */
  int slab_rows;     /* 0: normal run.  Multi-GPU slab waves: bit0 / bit1 = the first /
                        last image row is a halo row that changed; only the tile rows
                        holding or touching it are re-run (the rest of J must already be
                        at its fixed point) */
  int pipeline_rows; /* iwpp_recon_host only: slab height of the transfer/compute pipeline
                        (0 = auto, ~2 MB slabs; > 0 = this many rows, rounded up to the
                        32-row tile side; < 0 = off: copy in, compute, copy out) */
  int engine;        /* 0 = auto, 1 = shared-memory queue engine (every dtype), 2 = register
                        engine (u8/binary: Jacobi steps on packed bytes) on the tile queue,
                        3 = register engine in level-synchronous tile rounds (u8, rows
                        16-byte aligned; one grid barrier per round, no per-tile protocol;
                        else as 2).  Auto picks the register engine on the tile queue for
                        u8 unless queue_capacity or tile_sweeps is set */
  int max_rounds;    /* EngineConfig.max_rounds (engine.py:311-317): > 0 caps the rounds
                        of the tile-rounds engine (engine 3; auto picks it when set):
                        IWPP_E_ENGINE_LIMIT if the fixed point needs more.  0 / -1: no cap.
                        Other engines have no rounds and ignore it */
  const void *marker;/* optional device marker (nullptr: J already holds it).  When set, J is
                        output only: the u8 register engine copies the marker into J in its
                        own prologue (one pass less over HBM, one launch less); other paths
                        copy it first.  May equal J.  iwpp_recon_host ignores it */
} iwpp_recon_opts;

/* Timing helpers (events live in this library's CUDA runtime). */
int iwpp_event_create(void **ev);
int iwpp_event_destroy(void *ev);
int iwpp_event_record(void *ev, void *stream);
/* milliseconds between two recorded events (synchronizes on `end`) */
int iwpp_event_elapsed_ms(void *begin, void *end, float *ms);

size_t iwpp_recon_workspace_bytes(int64_t W, int64_t H, int dtype, int conn);
int iwpp_recon(void *J, const void *I, int64_t W, int64_t H, int dtype, int conn,
               void *workspace, size_t workspace_bytes, const iwpp_recon_opts *opts,
               iwpp_stats *stats, void *stream);

/* Host-buffer variant (the e2e path of the reference-facing call):
 * copies marker/mask host->device (into the workspace), runs iwpp_recon,
 * copies the result device->host into `out`, synchronizes.  Host buffers
 * may be pageable or pinned.  Returns IWPP_E_CONTRACT if marker > mask
 * anywhere (ReconInput.__post_init__, recon.py:60-61). */
size_t iwpp_recon_host_workspace_bytes(int64_t W, int64_t H, int dtype, int conn);
int iwpp_recon_host(void *out, const void *marker, const void *mask, int64_t W,
                    int64_t H, int dtype, int conn, void *workspace,
                    size_t workspace_bytes, const iwpp_recon_opts *opts,
                    iwpp_stats *stats, void *stream);

/* Diagnostics: copy the engine's device counters of the last iwpp_recon on
 * this workspace (tile activations, re-runs, pushes, overflows, seeds,
 * violations, then per-phase SM cycles: pop, load, sweep, detect, queue,
 * store).  Returns the number of counters written.  Syncs. */
int iwpp_recon_engine_counters(const void *workspace, int64_t W, int64_t H, uint64_t *out,
                               int n, void *stream);

/* Diagnostics (no reference counterpart): the register engine's activation
 * trace, compiled in only with -DIWPP_ATRACE (development builds; otherwise
 * returns IWPP_E_CONTRACT).  buf != NULL arms the trace with a device buffer
 * of cap 32-byte records (recon_tiles.cu ATraceRec) and resets the count;
 * n_out != NULL receives the number of records written so far.  Returns the
 * record size. */
int iwpp_debug_atrace(void *buf, uint32_t cap, uint32_t *n_out);

/* marker <= mask check (recon.py:60): *n_violations_host = count. Syncs. */
int iwpp_check_le(const void *J, const void *I, int64_t n, int dtype,
                  void *workspace, int64_t *n_violations_host, void *stream);

/* Individual stages (for the stage-level parity tests and the tiled /
 * multi-GPU drivers). */
/* Row sweeps forward+backward (K.115-139, exact clamp-composition scan). */
int iwpp_recon_sweep_rows(void *J, const void *I, int64_t W, int64_t H, int dtype,
                          void *stream);
/* Column sweeps forward+backward (K.142-190, vertical part exact; segment
 * composites + carry scan + apply).  workspace: iwpp_recon_workspace_bytes. */
int iwpp_recon_sweep_cols(void *J, const void *I, int64_t W, int64_t H, int dtype,
                          void *workspace, void *stream);
/* The reference's individual sequential passes, cell for cell (their
 * intermediate states are schedule-specific): recon.raster_pass
 * (recon.py:134-139 -> K.38-74), recon.antiraster_pass / _antiraster_packed
 * (recon.py:142-161 -> K.77-112; seeds = packed y*W+x in the order the
 * sweep met them, written to `seeds` (W*H capacity) when non-null) and the
 * four phases of recon.parallel_sweeps (recon.py:275-305 -> K.115-190,
 * single band).  In place on J; *changed_host = any cell changed.  Syncs.
 * workspace: iwpp_recon_pass_workspace_bytes. */
enum {
  IWPP_PASS_RASTER = 0, IWPP_PASS_ANTIRASTER = 1, IWPP_PASS_ROWS_FWD = 2, IWPP_PASS_COLS_FWD = 3,
  IWPP_PASS_ROWS_BWD = 4, IWPP_PASS_COLS_BWD = 5
};
size_t iwpp_recon_pass_workspace_bytes(int64_t W, int64_t H, int dtype);
int iwpp_recon_pass(void *J, const void *I, int64_t W, int64_t H, int dtype, int conn, int pass,
                    int64_t *seeds, int64_t *n_seeds_host, int *changed_host, void *workspace,
                    void *stream);
/* Full-neighbourhood seed scan (K.193-217): writes active pixels (packed
 * y*W+x, int64, raster order NOT guaranteed) to out; *n_host = count. */
int iwpp_recon_seed_scan(const void *J, const void *I, int64_t W, int64_t H,
                         int dtype, int conn, int64_t *out, int64_t *n_host,
                         void *workspace, void *stream);

/* ---- Euclidean distance transform ----------------------------------
 * Replaces edt() / edt_propagate() / finalize_distance_map()
 * (edt.py:248-294).  Level-synchronous two-phase rounds (K.403-433,
 * edt.py:217-226) with the (d^2, packed index) total order (K.320-336):
 * bit-identical to the reference's canonical schedule. */
size_t iwpp_edt_workspace_bytes(int64_t W, int64_t H, int conn);
/* mask: device u8 (0 = background).  vr: device int64 (H,W) out (packed
 * source, -1 = INF).  dist: device f32 (H,W) out, or NULL.
 * Returns IWPP_E_NO_BACKGROUND when some cell has no source (vr is still
 * written, dist is not meaningful). */
int iwpp_edt(const uint8_t *mask, int64_t W, int64_t H, int conn, int64_t *vr,
             float *dist, void *workspace, size_t workspace_bytes,
             int64_t max_rounds, iwpp_stats *stats, void *stream);
/* edt_propagate (edt.py:248-269): vr in/out (device int64), seeds device
 * int64 packed (duplicates allowed). */
int iwpp_edt_propagate(int64_t *vr, int64_t W, int64_t H, int conn,
                       const int64_t *seeds, int64_t n_seeds, void *workspace,
                       size_t workspace_bytes, int64_t max_rounds,
                       iwpp_stats *stats, void *stream);
/* Engine selection for tests/diagnostics (per host thread):
 * 0 = auto (64-bit keys on the raster-frontier engine; range-checked with a
 * CAS re-run when W, H exceed the 32-bit d^2 range), 1 = force the 32-bit-source CAS
 * engine, 2 = force range-checked keys, 3 = force the per-round
 * frontier-queue engine, 4 = force the blocked engine; 5 / 6 = the queue
 * engine with the paper's prefix-sum / naive global queue instead of the
 * block queue (PAPER.md:1563-1595 queue study), 7 = force the raster engine.
 * Results never depend on it. */
int iwpp_edt_set_engine(int mode);
/* finalize_distance_map (edt.py:272-281): dist = f32(sqrt(f64(d2))).
 * Returns IWPP_E_NO_BACKGROUND if any vr == -1.  d2 may be NULL. */
int iwpp_edt_finalize(const int64_t *vr, int64_t W, int64_t H, float *dist,
                      int64_t *d2, void *workspace, void *stream);
/* init_packed / edt_init (edt.py:187-202; K.edt_assign K.339-347,
 * K.edt_contour_seeds K.350-373): vr (device int64 (H,W), may be NULL) =
 * own packed index on background, -1 on foreground; seeds (device int64,
 * capacity W*H, may be NULL) = background cells with an in-bounds foreground
 * neighbour, in raster order; *n_seeds_host (may be NULL; syncs) = count. */
size_t iwpp_edt_init_workspace_bytes(int64_t W, int64_t H);
int iwpp_edt_init(const uint8_t *mask, int64_t W, int64_t H, int conn, int64_t *vr, int64_t *seeds,
                  int64_t *n_seeds_host, void *workspace, size_t workspace_bytes, void *stream);
/* edt_exact_bruteforce (edt.py:313-323, oracles.bruteforce_sqdist
 * oracles.py:57-73): exact squared distance to the nearest background cell
 * (separable exact transform, integer arithmetic: the brute-force minimum).
 * d2 (device int64, may be NULL: then the workspace holds it), dist (device
 * f32 = f32(sqrt(f64(d2))), may be NULL).  IWPP_E_NO_BACKGROUND if the mask
 * has no background (syncs). */
size_t iwpp_edt_exact_workspace_bytes(int64_t W, int64_t H);
int iwpp_edt_exact(const uint8_t *mask, int64_t W, int64_t H, int64_t *d2, float *dist,
                   void *workspace, size_t workspace_bytes, void *stream);
/* ---- EDT on one horizontal slab of a multi-GPU run ----
 * The rank owns rows [y0, y0+h) of an H-row image.  The synchronous rule
 * needs one exchange per round (tiles.py:10-15, edt_bp_sweep K.493-522):
 * each round takes the neighbours' boundary frontier rows (halo_up /
 * halo_dn: W uint64 sources, all-ones = none; NULL at the image edge) and
 * produces this slab's (out_up / out_dn).  Keys use global coordinates, so
 * the result equals the single-device EDT cell for cell.
 * mask_ext: (h + 2) x W device u8, rows 0 / h+1 = the neighbours' rows. */
size_t iwpp_edt_slab_workspace_bytes(int64_t W, int64_t h);
int iwpp_edt_slab_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H,
                       int conn, int has_up, int has_down, void *workspace,
                       uint64_t *out_up, uint64_t *out_dn, void *stream);
/* round r: *n_next_host = this slab's next frontier size (syncs) */
int iwpp_edt_slab_round(void *workspace, int64_t W, int64_t h, int64_t y0, int conn, int64_t r,
                        const uint64_t *halo_up, const uint64_t *halo_dn, uint64_t *out_up,
                        uint64_t *out_dn, int64_t *n_next_host, void *stream);
/* after `rounds` rounds: vr (h x W int64, global packed indices) and dist;
 * returns IWPP_E_NO_BACKGROUND if a cell has no source, IWPP_E_OVERFLOW if
 * a squared distance exceeded the 32-bit key range. */
int iwpp_edt_slab_finalize(void *workspace, int64_t W, int64_t h, int64_t y0, int64_t rounds,
                           int64_t *vr, float *dist, void *stream);

/* ---- multi-GPU EDT, device-resident rounds ------------------------------
 * Replaces the per-round host loop of the slab protocol (tiles.py:305-331,
 * edt_bp_sweep K.493-522: one boundary exchange per synchronous round) with
 * one persistent kernel per GPU.  Every rank owns a mailbox (size
 * iwpp_edt_mg_mailbox_bytes, in its own device memory, zeroed by its owner
 * before any rank calls iwpp_edt_mg_init); the neighbours write the
 * boundary frontier items into it and every rank adds its frontier counts,
 * with system-scope stores / atomics -- so mailbox[] must hold pointers
 * that are valid on the calling GPU: its own memory, or peer memory mapped
 * over NVLink (CUDA IPC / symmetric memory).  Several slabs of one GPU
 * (n_local > 1) run as CTA groups of one launch: the single-GPU form of the
 * same protocol.  The result is identical to iwpp_edt on the whole image. */
typedef struct iwpp_edt_mg_slab {
  void *workspace;    /* iwpp_edt_mg_workspace_bytes(W, h), set up by iwpp_edt_mg_init */
  int64_t W, h, y0, H;
  int has_up, has_down, rank, world;
  void *mailbox[16];  /* every rank's mailbox (rank order), valid on this GPU */
} iwpp_edt_mg_slab;
size_t iwpp_edt_mg_workspace_bytes(int64_t W, int64_t h);
size_t iwpp_edt_mg_mailbox_bytes(int64_t W);
/* slab init (as iwpp_edt_slab_init) + the initial boundary items into the
 * neighbours' mailboxes (NULL at the image edge) */
int iwpp_edt_mg_init(const uint8_t *mask_ext, int64_t W, int64_t h, int64_t y0, int64_t H, int conn,
                     int has_up, int has_down, void *workspace, void *mailbox_up, void *mailbox_down,
                     void *stream);
/* all rounds to the global fixed point; *rounds = rounds run (the same on
 * every rank).  IWPP_E_ENGINE_LIMIT past max_rounds (< 0: no cap).  Syncs.
 * The slabs are then finalized with iwpp_edt_slab_finalize(workspace, ...). */
int iwpp_edt_mg_run(const iwpp_edt_mg_slab *slabs, int n_local, int conn, int64_t max_rounds,
                    int64_t *rounds, void *stream);

/* Host-buffer variant: mask host -> device, edt, vr/dist device -> host. */
size_t iwpp_edt_host_workspace_bytes(int64_t W, int64_t H, int conn);
int iwpp_edt_host(const uint8_t *mask, int64_t W, int64_t H, int conn, int64_t *vr,
                  float *dist, void *workspace, size_t workspace_bytes,
                  int64_t max_rounds, iwpp_stats *stats, void *stream);

/* ---- image I/O on the device (reference: gridwave/imgio.py) ----
 * The Python readers put the file's raster in pinned host memory, copy it
 * to the device and decode it there. */
/* read_pgm (imgio.py:62-110): P5 raster -> samples.  bytes_per_sample 1
 * (maxval <= 255) or 2 (16-bit big-endian); binary = 1 maps nonzero -> 255
 * (maxval 1, imgio.py:108-109).  *max_sample_host (if not NULL; syncs) gets
 * the largest raw sample, for the "sample exceeds maxval" check
 * (imgio.py:105-106).  dst / raster 16-byte aligned; workspace >= 8 bytes. */
int iwpp_pgm_decode(void *dst, const void *raster, int64_t n, int bytes_per_sample, int binary,
                    void *workspace, int64_t *max_sample_host, void *stream);
/* write_pgm (imgio.py:113-130): samples -> P5 raster (u16 big-endian). */
int iwpp_pgm_encode(void *raster, const void *src, int64_t n, int bytes_per_sample, void *stream);
/* gen_marker (imgio.py:216-228): marker = max(mask - h, 0), dtype u8 / u16 /
 * i32 / f32 (f32: np.maximum semantics, NaN propagates). */
int iwpp_gen_marker(void *marker, const void *mask, int64_t n, int dtype, double h, void *stream);
/* the CLI's quantized EDT view (cli.py:98-101): min(rint(dist), 255) as u8 */
int iwpp_quantize_u8(uint8_t *out, const float *dist, int64_t n, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* IWPP_B200_H */
