/*
 * cbessfm.h -- C ABI of the B200-native CB-ESSFM digital-backpropagation
 * hot path (libcbessfm.so, built from paper_2409_14489_b200/csrc).
 *
 * The reference (fiberdbp 0.1.0, /root/reference/pkg/src/fiberdbp) has no
 * FFI layer: its hot path is the pure-Python call
 *     run_dbp(w, cfg, coeffs, counter)              dbp.py:437-478
 * with the per-run engine state built in
 *     _BlockEngine.__init__                         dbp.py:318-369
 * and the per-block pipeline
 *     _BlockEngine._process_cb                      dbp.py:382-401
 *     _nlpr_fields                                  dbp.py:185-208.
 * This ABI is what a binding of that call needs (INTEGRATION.md shows the
 * ctypes stub a maintainer would add to dbp.py): the host builds the FP64
 * tables exactly as _BlockEngine.__init__ does, hands them to
 * cbessfm_plan_create (which uploads them once), and every run_dbp call
 * becomes one cbessfm_run over device buffers.
 *
 * Conventions: plain pointers and sizes only; no C++ exceptions cross the
 * ABI; every function returns a cbessfm_status and leaves a thread-local
 * message for cbessfm_last_error(). Complex data is interleaved (re, im).
 * A plan is immutable after creation and may be used concurrently on
 * distinct streams. All input/output memory is owned by the caller.
 */
#ifndef CBESSFM_H
#define CBESSFM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBESSFM_VERSION 3

typedef enum {
  CBESSFM_OK = 0,
  CBESSFM_ERR_INVALID = 1,     /* bad argument; Python raises ValueError   */
  CBESSFM_ERR_UNSUPPORTED = 2, /* valid for the reference, not for this
                                  build (e.g. non power-of-two N/N_sb);
                                  Python raises ValueError                 */
  CBESSFM_ERR_CUDA = 3         /* CUDA runtime error; RuntimeError         */
} cbessfm_status;

typedef enum { CBESSFM_C64 = 0, CBESSFM_C128 = 1 } cbessfm_dtype;

typedef struct cbessfm_plan cbessfm_plan;

/* Engine tables, built on the host in FP64 (replaces dbp.py:318-369).
 * All pointers are HOST pointers; the plan copies (and for C64 rounds)
 * them into device memory it owns. */
typedef struct {
  int32_t dtype;        /* cbessfm_dtype: arithmetic of the device path   */
  int32_t n_subbands;   /* N_sb = P (DbpConfig.n_subbands, dbp.py:56)    */
  int32_t block_size;   /* N = P * Q (DbpConfig.block_size, dbp.py:58)   */
  int32_t overlap;      /* N_ov (DbpConfig.overlap, dbp.py:59)           */
  int32_t n_steps;      /* N_st (DbpConfig.n_steps, dbp.py:55)           */
  int32_t n_phasors;    /* distinct dispersion tables (dbp.py:356-359)   */
  /* [n_phasors][P][Q] complex128: exp(j 2 pi^2 beta2 dz f_abs^2) / Q     */
  const double* phasors;
  /* [n_steps + 1]: table applied before step s (s < n_steps) and the
   * final one (s == n_steps), i.e. gvd_lengths + [final_gvd]            */
  const int32_t* phasor_index;
  /* [n_sets][P][Q/2 + 1] complex128 spectra S_h = rfft(centred taps c_h),
   * S_h for h >= 1 pre-multiplied by the 3/2 XPM weight (dbp.py:152-182);
   * may be NULL when n_steps == 0                                       */
  const double* mimo;
  /* [n_sets][n_steps]: step_scales / reference_power_w / Q (dbp.py:386,
   * :196)                                                                */
  const double* theta_scale;
  int32_t device;       /* CUDA device ordinal the plan lives on          */
  /* Coefficient sets (CoefficientSet, kernel.py:390-453) sharing this
   * geometry; waveform w of a launch uses set w % n_sets. 0 or 1: one set.
   * Several sets evaluate candidate coefficients on one waveform in one
   * launch (in_batch_stride 0), as optimize_coefficients' finite
   * differences do one run_dbp call at a time (optimize.py:129-167).     */
  int32_t n_sets;
} cbessfm_desc;

/* One launch over a block range of a batch of waveforms. Buffers are
 * DEVICE pointers of the plan's dtype, layout [batch][2][*] (x then y).
 * Input element j of a waveform holds sample (in_origin + j) mod n of the
 * circular sequence; output element j receives kept sample out_origin + j.
 * For whole waveforms both origins are 0; the shard planner uses them for
 * halo'd slices. */
typedef struct {
  const void* in;
  int64_t in_batch_stride; /* elements between waveforms                 */
  int64_t in_pol_stride;   /* elements between x and y                    */
  int64_t in_origin;
  void* out;
  int64_t out_batch_stride;
  int64_t out_pol_stride;
  int64_t out_origin;
  int64_t n;               /* samples per polarisation (circular period)  */
  int64_t batch;           /* waveforms                                   */
  int64_t block_begin;     /* global block range [begin, end) of the       */
  int64_t block_end;       /*   overlap-save schedule (dbp.py:471-477)     */
} cbessfm_io;

/* Host-buffer variant (the call a reference-side binding makes with the
 * waveform in host memory): in/out are HOST pointers, layout [batch][2][n]
 * contiguous, of the plan's dtype; page-locked memory is required for the
 * copies to overlap. The waveform is copied in `chunks` sample ranges and
 * every block range launches as soon as its input window has landed, while
 * finished kept samples are copied back (three-way overlap). */
typedef struct {
  const void* in;
  void* out;
  int64_t n;               /* samples per polarisation                    */
  int64_t batch;           /* waveforms                                   */
  int32_t chunks;          /* pipeline depth (<= 0: default 8)            */
} cbessfm_host_io;

/* The reference's own waveform layout (DualPolWaveform, signals.py:32-86):
 * x and y as separate HOST arrays of complex128, in any (pageable) memory,
 * results into separate HOST complex128 arrays. For a c64 plan the cast to
 * complex64 and back happens in the host copies. The copies run on a pool
 * of host threads owned by the plan and are pipelined with the chunked
 * H2D / kernel / D2H of cbessfm_run_host (page-locked staging kept by the
 * plan). Synchronous: returns once out_x / out_y hold the result, like
 * run_dbp (dbp.py:437-478). ABI 3. */
typedef struct {
  const double* in_x;      /* [n] complex128 (interleaved re, im)         */
  const double* in_y;
  double* out_x;           /* [n] complex128                              */
  double* out_y;
  int64_t n;               /* samples per polarisation                    */
  int32_t chunks;          /* pipeline depth (<= 0: default 8)            */
  int32_t host_threads;    /* copy threads (<= 0: min(8, hardware))       */
} cbessfm_dualpol_io;

typedef struct {
  int32_t threads_per_cta;
  int32_t cluster_size;
  int64_t smem_per_cta;
  int32_t max_active_clusters;
  int32_t q;               /* per-subband FFT size N' = N / N_sb          */
  char kernel[64];         /* the block kernel a device-resident launch   */
                           /* runs, e.g. "cbessfm_block_kernel<double,5,2048>" (ABI 3) */
} cbessfm_plan_info;

/* Version of this ABI (CBESSFM_VERSION). */
int32_t cbessfm_version(void);

/* Number of overlap-save blocks for n samples: ceil(n / (N - N_ov))
 * (dbp.py:471). Returns -1 on invalid arguments. Host-only. */
int64_t cbessfm_num_blocks(int64_t n, int32_t block_size, int32_t overlap);

/* Whether this build has a kernel for (dtype, P, Q). Host-only. */
int32_t cbessfm_supported(int32_t dtype, int32_t n_subbands, int32_t block_size);

/* Validate desc, upload the tables, configure the kernel. */
cbessfm_status cbessfm_plan_create(const cbessfm_desc* desc, cbessfm_plan** plan);

/* Launch configuration of a plan (threads, cluster, smem, occupancy). */
cbessfm_status cbessfm_plan_info_get(const cbessfm_plan* plan, cbessfm_plan_info* info);

/* Enqueue the fused block kernel on `stream` (a cudaStream_t, NULL for
 * the legacy default stream). Asynchronous; errors of the launch itself
 * are reported, kernel faults surface at the caller's next sync. */
cbessfm_status cbessfm_run(const cbessfm_plan* plan, const cbessfm_io* io, void* stream);

/* Enqueue H2D, the fused kernel and D2H on `stream` for host buffers;
 * returns once enqueued (synchronise `stream` before reading `out`). */
cbessfm_status cbessfm_run_host(const cbessfm_plan* plan, const cbessfm_host_io* io, void* stream);

/* One waveform in the reference's layout (cbessfm_dualpol_io), host in,
 * host out, synchronous; `stream` orders the device work. The entry the
 * drop-in run_dbp calls. The staging copies also check every input sample
 * (dbp.py:449 w.require_finite()): a NaN or infinity returns
 * CBESSFM_ERR_INVALID "waveform contains non-finite samples" (outputs
 * undefined). */
cbessfm_status cbessfm_run_dualpol(const cbessfm_plan* plan, const cbessfm_dualpol_io* io,
                                   void* stream);

/* The public nlpr_step helper (dbp.py:211-230) on the GPU: coupled-band
 * nonlinear phase rotation of P time-domain subband waveforms of n_prime
 * samples. in/out: DEVICE [2][P][n_prime] of `dtype`; mimo: HOST
 * [P][P][n_prime/2+1] complex128 (a MimoTransfer matrix, any structure);
 * theta_scale = step_power_scale / reference_power_w. Synchronous. */
cbessfm_status cbessfm_nlpr(int32_t dtype, int32_t n_subbands, int32_t n_prime, const void* in,
                            void* out, const double* mimo, double theta_scale, void* stream);

/* Replace the coefficient-set tables of a plan (same geometry, same n_sets):
 * mimo [n_sets][P][Q/2+1] and theta_scale [n_sets][n_steps], HOST, laid
 * out as in cbessfm_desc. n_sets must equal the plan's (CBESSFM_ERR_INVALID
 * otherwise: the host arrays are read for exactly that many sets). Ordered on `stream` and synchronous; an
 * optimiser re-evaluating candidate taps reuses one plan this way instead
 * of rebuilding it (the dispersion tables and twiddles do not change). */
cbessfm_status cbessfm_plan_update_sets(cbessfm_plan* plan, int32_t n_sets, const double* mimo,
                                        const double* theta_scale, void* stream);

/* Free the plan's device tables. */
cbessfm_status cbessfm_plan_destroy(cbessfm_plan* plan);

/* Debug: copy up to n slots of the last launch's profile into out: 256
 * phase timestamps (clock64) of CTA 0, then 3 per cluster c at 256 + 3c
 * (globaltimer ns at start and end, SM id). Only builds compiled with
 * -DCB_PHASE_PROFILE record them; other builds return 0. */
int32_t cbessfm_debug_phase_times(const cbessfm_plan* plan, int64_t* out, int32_t n);

/* Message of the last failing call on this thread ("" if none). */
const char* cbessfm_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CBESSFM_H */
