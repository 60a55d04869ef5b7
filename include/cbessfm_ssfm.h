/*
 * cbessfm_ssfm.h -- C ABI of the fine-step split-step Fourier propagator
 * in libcbessfm.so: the reference's ground-truth channel
 * and ideal backpropagation,
 *     propagate_link(w, link, sim)          channel.py:216-236
 *     backward_propagate(w, link, sim)      channel.py:239-256
 *     _run_spans(field, rate, link, steps)  channel.py:176-213
 * i.e. per span and per fine step dz of the span:
 *     spec *= half(dz); field = ifft(spec);
 *     field *= exp(-j sgn gamma Leff(dz) (|x|^2 + |y|^2));
 *     spec = fft(field); spec *= half(dz)
 * with the EDFA field gain (and seeded ASE) after every forward span, or the
 * gain removed before every backward span. The whole propagation is one
 * cooperative launch: four-step FFTs of length n = n1 * n2 with the
 * column passes (inverse FFT, nonlinear rotation, forward FFT) and the row
 * passes (forward FFT, dispersion halves, inverse FFT) fused, separated by
 * grid-wide barriers; the waveform stays L2-resident for n up to 2^21.
 *
 * Conventions as in cbessfm.h (status codes, cbessfm_last_error).
 */
#ifndef CBESSFM_SSFM_H
#define CBESSFM_SSFM_H

#include <stdint.h>

#include "cbessfm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t dtype;            /* cbessfm_dtype                                   */
  int64_t n;                /* samples per polarisation, power of two, 2..2^22 */
  int32_t batch;            /* waveforms                                       */
  int32_t n_spans;          /* spans to run                                    */
  int32_t steps_per_span;   /* fine steps per span (span_step_sizes)           */
  int32_t n_tables;         /* distinct step lengths                           */
  /* HOST [n_tables][n] complex128 in numpy fftfreq order: the half-step
   * operator _gvd_phasor(n, rate, sgn beta2, dz/2) * exp(-sgn alpha dz/4)
   * (channel.py:201-203), built by the caller in FP64                   */
  const double* half;
  const int32_t* step_table;/* HOST [steps_per_span]: table of each fine step  */
  /* HOST [steps_per_span]: -sgn * gamma * Leff(dz) (channel.py:204-205,
   * :210); the rotation angle is nl_coef * (|x|^2 + |y|^2)             */
  const double* nl_coef;
  int32_t backward;         /* 0: propagate_link, 1: backward_propagate         */
  double gain;              /* span field gain 10^(G_dB / 20) (channel.py:148)  */
  int32_t device;
} cbessfm_ssfm_desc;

/* Propagate `data` (DEVICE [batch][2][n] of the dtype, in place) through
 * n_spans spans. noise: DEVICE [n_spans][batch][2][n] ASE samples added
 * after each forward span's gain (edfa, channel.py:150-165), or NULL.
 * Synchronous with respect to the host for its own table upload; the
 * propagation itself is enqueued on `stream`. */
cbessfm_status cbessfm_ssfm_run(const cbessfm_ssfm_desc* desc, void* data, const void* noise,
                                void* stream);

/* The four-step geometry the run would use (n1 * n2 == n, tile sizes and
 * the cooperative grid), for tests and profiling. */
typedef struct {
  int32_t n1, n2, rows_per_tile, cols_per_tile, grid, threads;
  int64_t smem_bytes;
} cbessfm_ssfm_info;
cbessfm_status cbessfm_ssfm_info_get(int32_t dtype, int64_t n, int32_t batch, int32_t device,
                                     cbessfm_ssfm_info* info);

/* Message of the last failing cbessfm_ssfm_* call on this thread. */
const char* cbessfm_ssfm_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CBESSFM_SSFM_H */
