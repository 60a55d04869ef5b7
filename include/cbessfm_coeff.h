/*
 * cbessfm_coeff.h -- C ABI of the GPU coefficient builder
 * in libcbessfm.so: the weighted uniform-grid kernel transform behind the
 * reference's analytic coefficients,
 *     _coeff_grid_eval(geom, separation, memory, rate, p_ref, nodes)
 *                                                    kernel.py:274-303
 * with the step kernel K(mu, nu) of kernel.py:153-250 (closed form for
 * span-aligned symmetric steps, exact piecewise form otherwise).
 *
 * The reference materialises the nodes x nodes kernel matrix (and its
 * conjugate transpose) to take anti-diagonal sums, which is what runs it
 * out of host memory past ~1000 taps; here every anti-diagonal sum is one
 * CTA evaluating its kernel entries on the fly, so memory is O(nodes).
 *
 * Conventions as in cbessfm.h (status codes).
 */
#ifndef CBESSFM_COEFF_H
#define CBESSFM_COEFF_H

#include <stdint.h>

#include "cbessfm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t closed_form;   /* 1: kernel_closed_form (kernel.py:153-174)
                            0: _kernel_segments (kernel.py:227-250)       */
  double gamma_w_km;
  double alpha_np_km;    /* power attenuation, 1/km                       */
  double beat_scale;     /* 2 pi^2 beta2_s2_km (b = beat_scale nu (mu-nu),
                            kernel.py:148-150)                             */
  double span_km;        /* closed form: span length                      */
  int32_t num_spans;     /* closed form: identical spans in the step      */
  int32_t n_segments;    /* piecewise form: power-profile pieces          */
  const double* segments;/* HOST [n_segments][3]: z0, z1, g0 (kernel.py:108-129) */
} cbessfm_step_kernel;

/* c[m] = sum_{off} exp(2 pi j m (-off) / (n-1)) sum_i Kh[i, i+off] w_i w_{i+off}
 * for m = -memory..memory, Kh = (K + K^H)/2 on the grid mu (kernel.py:285-302,
 * before the reference_power_w / rate^2 scaling). mu, weights: HOST [num_nodes];
 * out: HOST [2 memory + 1] complex128 (interleaved). Synchronous. */
cbessfm_status cbessfm_coeff_grid(const cbessfm_step_kernel* kernel, int64_t num_nodes,
                                  const double* mu, const double* weights, int32_t memory,
                                  double* out, int32_t device);

/* K(mu_i, nu_i) for i < count (HOST arrays in/out, out complex128
 * interleaved): the step kernel itself, for validation. Synchronous. */
cbessfm_status cbessfm_step_kernel_eval(const cbessfm_step_kernel* kernel, int64_t count,
                                        const double* mu, const double* nu, double* out,
                                        int32_t device);

/* Message of the last failing cbessfm_coeff_* / step-kernel call. */
const char* cbessfm_coeff_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CBESSFM_COEFF_H */
