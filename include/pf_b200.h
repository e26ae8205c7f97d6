/*
 * pf_b200.h -- C ABI of the B200-native particle-filter tracking step.
 *
 * Drop-in boundary for the reference's per-frame path (arXiv 2308.00763,
 * reference package `halfpf`).  The reference is pure Python; these are the
 * entry points its Python layer would bind through ctypes:
 *
 *   pf_create / pf_destroy   <- halfpf.filter.make_engine + init
 *                               (/root/reference/pkg/src/halfpf/filter.py:154-166,
 *                                181-193, 327-344; _validate_k :137-143)
 *   pf_run                   <- halfpf.filter.run (filter.py:591-662): whole
 *                               video, per-frame estimates -> trajectory
 *   pf_step                  <- one iteration of the frame loop
 *                               (filter.py:617-654) + estimate (:638)
 *   pf_stage_*               <- the six engine stage methods
 *                               (filter.py:195-255 wide, 346-567 binary16)
 *   pf_systematic_ancestors  <- systematic_ancestors (filter.py:583-588)
 *   pf_rng_normals           <- RngStream.normals / uniform (filter.py:71-82),
 *                               product LCG stream
 *
 * Plain C types only: pointers, sizes, int status codes.  No torch types.
 * A handle owns every device buffer; it is not thread-safe (one stream per
 * handle), separate handles may run concurrently.
 */
#ifndef PF_B200_H
#define PF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (reference exceptions: ValueError, DegeneracyError) */
#define PF_OK 0
#define PF_EINVAL 1          /* ValueError (bad K, parity, precision, shapes) */
#define PF_EDEGENERATE 2     /* DegeneracyError; frame index via pf_degenerate_frame */
#define PF_ECUDA 3           /* CUDA runtime failure (message in pf_last_error) */
#define PF_ENOMEM 4
#define PF_EIO 5             /* I/O or container parse failure (cli.py exit code 3) */

/* precisions (PrecisionMode, filter.py:49-60) */
#define PF_FP64 0
#define PF_FP32 1
#define PF_FP16 2            /* "fp16"        : binary16, scalar lanes          */
#define PF_FP16_PACKED 3     /* "fp16-packed" : binary16, half2 lanes (same values) */

/* ModelParams (model.py:27-49) */
typedef struct pf_params {
  double drift_x, std_x, drift_y, std_y;
  double bg_mean, fg_mean, likelihood_scale;
  int32_t disk_radius;
  double noise_std;
} pf_params;

typedef struct pf_config {
  int32_t precision;          /* PF_FP64 .. PF_FP16_PACKED */
  int64_t K;                  /* particles per track */
  int32_t width, height;      /* frame shape (W, H) */
  int32_t n_tracks;           /* independent filters run together (1 = single filter) */
  int32_t n_videos;           /* track i observes video (i % n_videos) */
  const uint64_t* seeds;      /* n_tracks run seeds (host) */
  pf_params params;
  const int32_t* offsets_xy;  /* n_offsets (dx, dy) pairs, template order (model.py:69-78) */
  int32_t n_offsets;
  int32_t tpb;                /* threads per block of the fused kernel: 32..1024, 0 = default 256 */
  int32_t device;
  double start_x, start_y;    /* start hint (filter.py:606-607) */
} pf_config;

typedef struct pf_handle pf_handle;

const char* pf_version(void);
const char* pf_global_error(void);

int pf_create(pf_handle** out, const pf_config* cfg);
int pf_destroy(pf_handle* h);
const char* pf_last_error(const pf_handle* h);

/* Re-initialise every track at (x0, y0), frame counter 0 (init, filter.py:181-193). */
int pf_reset(pf_handle* h, double x0, double y0);

/* Whole-video run (filter.py:591-662).  frames: [n_videos][n_frames][H][W] u8,
 * host memory (frames_on_device = 0) or device memory (1).  traj_out: host
 * [n_tracks][n_frames][2] f64.  Returns PF_EDEGENERATE on a collapsed weight
 * sum (frame via pf_degenerate_frame). */
int pf_run(pf_handle* h, const uint8_t* frames, int32_t n_frames, int32_t frames_on_device,
           double* traj_out);

/* One frame for every track: frame: [n_videos][H][W] u8; est_out host [n_tracks][2]. */
int pf_step(pf_handle* h, const uint8_t* frame, int32_t frame_on_device, double* est_out);

/* Stream-ordered variants (no host synchronisation).  `stream` is a
 * cudaStream_t of the handle's device (NULL = none): the run starts after the
 * work already queued on `stream` (e.g. the kernels producing device frames),
 * and work queued on `stream` afterwards sees traj_out / est_out, which may be
 * device, pinned host or pageable host memory (a pageable destination makes
 * the final copy blocking).  Frame buffers must stay valid until the run has
 * completed.  pf_sync waits for the handle's enqueued run and returns
 * PF_EDEGENERATE / timings exactly as pf_run would.  This is the stream-ordered
 * form of the frame loop of run() (filter.py:617-654). */
int pf_run_async(pf_handle* h, const uint8_t* frames, int32_t n_frames, int32_t frames_on_device, double* traj_out,
                 void* stream);
int pf_step_async(pf_handle* h, const uint8_t* frame, int32_t frame_on_device, double* est_out, void* stream);
int pf_sync(pf_handle* h);
/* Order the handle's next work after the work already queued on `stream` (a
 * cudaStream_t of the handle's device), without a host synchronisation: e.g.
 * before a synchronous pf_step on a device frame produced on `stream`. */
int pf_stream_wait(pf_handle* h, void* stream);

int pf_degenerate_frame(const pf_handle* h);

/* Debug/parity: the per-frame likelihood maps of F host frames (one video),
 * [F][H+2r][W+2r] in the mode dtype (fp16 as uint16 bits): entry (iy+r, ix+r)
 * is the reference likelihood of a particle at rint position (ix, iy),
 * filter.py:204-217 (wide) / 384-423 (binary16). */
int pf_likelihood_maps(pf_handle* h, const uint8_t* frames, int32_t n_frames, void* maps_out);

/* Device-event timings of the last pf_run/pf_step, milliseconds:
 * [0] total, [1] upload, [2] likelihood maps, [3] fused frame kernels,
 * [4] tile tables, [5] download. */
int pf_last_timings(const pf_handle* h, float* ms6);

/* Per-kernel event timing: when on, timings [3]/[4] of the next runs are the
 * summed durations of the fused frame kernels / tile-table kernels alone
 * (events between launches on the handle's stream). */
int pf_set_profiling(pf_handle* h, int32_t on);

/* ---------------------------------------------------------------------------
 * Input side of the step.
 *
 * pf_generate_video renders the reference's synthetic video model
 * (model.generate_video, model.py:123-157) on the device: frames_dev receives
 * [F][H][W] uint8, truth_host [F][2] (x, y) is the reference trajectory
 * (specular bounces, model.py:105-121).  Pixel noise comes from the
 * counter-based LCG ziggurat stream of `seed` (pixel (t, y, x) at stream
 * position (t*H + y)*W + x), so frames are a pure function of (seed, t, y, x);
 * oracle/video.py restates it.  Same model, not NumPy's PCG64 bytes.
 *
 * pf_pfvd_info / pf_read_pfvd ingest a PFVD container (model.py:274-297:
 * "PFVD", u32 frames, width, height, pixels) straight into device memory
 * through pinned double-buffered staging; fwh = {frames, width, height}.
 * Errors: PF_EIO with the reference's messages ("bad container magic at
 * offset 0", "truncated header at offset 4", "expected N pixel bytes at
 * offset 16, got M"), readable with pf_global_error(). */
int pf_generate_video(const pf_params* params, int32_t n_frames, int32_t width, int32_t height, double start_x,
                      double start_y, uint64_t seed, const int32_t* offsets_xy, int32_t n_offsets,
                      uint8_t* frames_dev, double* truth_host, int32_t device);
int pf_pfvd_info(const char* path, int32_t* fwh);
int pf_read_pfvd(const char* path, uint8_t* frames_dev, int64_t capacity, int32_t* fwh, int32_t device);

/* ---------------------------------------------------------------------------
 * Sharded filter (one track, particle range split over n_shards <= 8 GPUs or
 * handles).  Replaces, for a filter too large for one
 * device, the reference's single-process run() loop (filter.py:591-662): the
 * resampling CDF / normalisation become per-shard exact partial sums combined
 * by three small all-gathers per frame, and resampled ancestors on other
 * shards are read peer-to-peer (NVLink) through the peer buffers below.
 * Results are bit-identical to the same filter run by pf_create/pf_run.
 *
 * Tiles per shard = next power of two >= ceil(n_tiles / n_shards); shard r
 * holds global tiles [r * shard_tiles, ...) (pf_shard_info).  Per frame f,
 * on every shard's stream, in this order:
 *   pf_shard_fused(h, f)
 *   all-gather 8 B:   exchange[0] (send) -> exchange[1] (recv, [n_shards])
 *   pf_shard_tables(h)
 *   all-gather 32 B:  exchange[2] (send) -> exchange[3] (recv, [n_shards][4])
 *   pf_shard_finish(h, f)
 *   barrier (every shard's window records written before the next frame)
 * between pf_shard_begin (frames upload + likelihood maps) and pf_shard_end
 * (trajectory download, PF_EDEGENERATE check).  Shards in one process use
 * pf_shard_local_allgather(hs, S, 0 | 1 | 2) for the three exchanges. */
int pf_shard_create(pf_handle** out, const pf_config* cfg, int32_t n_shards, int32_t shard);
/* {shard_tiles, first global tile, local tiles, local particles} */
int pf_shard_info(const pf_handle* h, int64_t* out4);
/* device pointers a peer needs: X0, X1, C0, C1, tab_s, tab_O, tab_invM, win */
int pf_shard_buffers(pf_handle* h, void** out8);
/* the same eight buffers as cudaIpcMemHandle_t[8] (8 x 64 bytes) */
int pf_shard_ipc_export(pf_handle* h, void* out512);
/* peer buffers: raw device pointers (same process / already mapped) or IPC handles */
int pf_shard_set_peer(pf_handle* h, int32_t peer, void* const* ptrs8);
int pf_shard_open_peer(pf_handle* h, int32_t peer, const void* handles512);
/* exchange buffers (device): {max key u64 send, u64[n_shards] recv, i64[4] send, i64[n_shards][4] recv} */
int pf_shard_exchange(pf_handle* h, void** out4);
void* pf_shard_stream(pf_handle* h);
int pf_shard_begin(pf_handle* h, const uint8_t* frames, int32_t n_frames, int32_t frames_on_device);
int pf_shard_fused(pf_handle* h, int32_t frame);
int pf_shard_tables(pf_handle* h);
int pf_shard_finish(pf_handle* h, int32_t frame);
int pf_shard_end(pf_handle* h, int32_t n_frames, double* traj_out);
int pf_shard_local_allgather(pf_handle* const* handles, int32_t n_shards, int32_t which);

/* Timeline tracing (performance analysis): when on, thread 0 of every CTA of
 * track 0 stamps %globaltimer (ns) at fixed points of the next runs:
 * per frame f, (n_tiles + n_chunks) records of 8 uint64 -- fused tile b:
 * [0] entry [1] draws done [2] predecessor released [3] window ready
 * [4] particles done [5] exit; table chunk c: [0] entry [1] released
 * [2] tree done [3] estimate written (last CTA only).  Unset slots are 0.
 * pf_get_trace copies the first n uint64 of the last run's buffer. */
int pf_set_trace(pf_handle* h, int32_t on);
int pf_get_trace(pf_handle* h, uint64_t* out, int64_t n);

/* Kernel launches issued by the last pf_run/pf_step. */
int64_t pf_last_launches(const pf_handle* h);

/* Debug/parity: copy track `track` state to host.  xs, ys, cdf_local in the
 * mode dtype (fp16 as uint16 bit patterns); any pointer may be NULL. */
int pf_get_state(pf_handle* h, int32_t track, void* xs, void* ys, void* cdf_local);
/* Draw stream of the fused path: switch the handle (one unsharded track,
 * 128 or 256 threads per block) from the product LCG stream to the
 * reference's own stream, Generator(Philox(seed)) (filter.py:71-82, RngStream):
 * frame t consumes standard_normal((K, 2)) then random(), exactly as run()
 * does (filter.py:617-650), generated in parallel on the device
 * (pf_philox.cuh).  state11 = NumPy's Philox state after seeding: key[2],
 * counter[4], buffer[4], buffer_pos (np.random.Philox(seed).state).  pf_reset
 * rewinds the stream to this state; pf_set_state leaves it where it is.
 * Debug capture (pf_get_debug) and tracing are not available in this mode. */
int pf_set_rng_philox(pf_handle* h, const uint64_t* state11);

/* State injection (teacher forcing / snapshot restore): track `track`'s
 * positions become xs, ys (mode dtype, fp16 as uint16 patterns) as the
 * post-resample state entering frame `frame`.  The next frame of EVERY track
 * then runs with identity ancestors (the positions are already resampled)
 * and frame `frame`'s draws; the frames after it proceed normally.  The
 * reference's seam for the same thing is a stage_hook mutating ParticleSet
 * after "resample" (filter.py:617-654; pkg/tests/test_filter.py:391-393).
 * Not available on sharded handles. */
int pf_set_state(pf_handle* h, int32_t track, const void* xs, const void* ys, int64_t frame);
/* Last frame's ancestors (int64 [K]) and per-particle log-likelihoods (mode dtype). */
int pf_get_debug(pf_handle* h, int32_t track, int64_t* ancestors, void* loglik);

/* ---- reference-semantics stage engine (stage_hook / make_engine path) ----
 * State lives on the device; arrays cross the boundary in the mode dtype
 * (fp16 as uint16 patterns), ancestors as int64.  Draws are injected. */
typedef struct pf_stage pf_stage;
int pf_stage_create(pf_stage** out, int32_t precision, int64_t K, const pf_params* params,
                    const int32_t* offsets_xy, int32_t n_offsets, int32_t device);
int pf_stage_destroy(pf_stage* s);
const char* pf_stage_error(const pf_stage* s);
int pf_stage_init(pf_stage* s, double x0, double y0);
int pf_stage_propagate(pf_stage* s, const double* noise_Kx2);
int pf_stage_likelihood(pf_stage* s, const uint8_t* frame, int32_t width, int32_t height);
int pf_stage_max(pf_stage* s, double* m_out);
int pf_stage_weight(pf_stage* s, double m, double* total_out);
int pf_stage_normalize(pf_stage* s, double total);
int pf_stage_estimate(pf_stage* s, double* ex, double* ey);
int pf_stage_resample(pf_stage* s, double u);
/* field: 0 xs, 1 ys, 2 loglik, 3 weights, 4 cdf (mode dtype), 5 ancestors (int64) */
int pf_stage_get(pf_stage* s, int32_t field, void* out);
int pf_stage_set(pf_stage* s, int32_t field, const void* in);

/* systematic_ancestors(cdf, u) on the device (filter.py:583-588). */
int pf_systematic_ancestors(const double* cdf, int64_t K, double u, int64_t* anc_out, int32_t device);

/* LCG stream draws (product RNG), generated on the device: normals for
 * stream positions [pos, pos+n); uniforms (w >> 11) * 2^-53 likewise. */
int pf_rng_normals(uint64_t seed, uint64_t pos, int64_t n, double* out, int32_t device);
int pf_rng_uniforms(uint64_t seed, uint64_t pos, int64_t n, double* out, int32_t device);

/* NumPy-compatible reference stream (Generator(Philox(seed)), filter.py:71-82)
 * generated on the device.  state11 = NumPy's Philox state: key[2],
 * counter[4], buffer[4], buffer_pos.  The ziggurat's variable word
 * consumption is resolved in parallel (pf_philox.cuh: classify every word
 * position, speculate block entries, repair, scan, emit). */
typedef struct pf_philox pf_philox;
int pf_philox_create(pf_philox** out, const uint64_t* state11, int32_t device);
int pf_philox_destroy(pf_philox* p);
int pf_philox_normals(pf_philox* p, int64_t n, double* out);
int pf_philox_uniforms(pf_philox* p, int64_t n, double* out);
/* the same normals into device memory, stream-ordered on `stream` (no sync) */
int pf_philox_normals_device(pf_philox* p, int64_t n, double* out_dev, void* stream);

/* RN16(exp(x)) for all 65536 binary16 patterns (host-built table used by the
 * kernels; exposed so tests can pin it against halfnum.exp16 on CPU). */
int pf_exp16_table(uint16_t* out65536);
/* The device's exp16 as used by the fused FP16 kernel (fast path + table
 * fallback) for all 65536 inputs -- must equal pf_exp16_table on d <= 0. */
int pf_exp16_device(uint16_t* out65536, int32_t device);

#ifdef __cplusplus
}
#endif
#endif /* PF_B200_H */
