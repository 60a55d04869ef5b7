/*
 * cbessfm_peaks.h -- roofline denominators measured on the running GPU.
 *
 * MEASURED_PEAKS.json (driver-written) carries the HBM copy bandwidth and
 * the bf16 tensor peak only; the CB-ESSFM roofline (BASELINE.json
 * north_star) needs the FP32 / FP64 FMA lane rate, so the
 * benchmark measures it with these microkernels. Not part of the DBP path.
 */
#ifndef CBESSFM_PEAKS_H
#define CBESSFM_PEAKS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FMA lane operations per second (one fused multiply-add on one lane = 1)
 * sustained by a register-resident FMA loop over all SMs for about `ms`
 * milliseconds. kind: 0 = FP32 FFMA, 1 = FP32 packed FFMA2 (fma.rn.f32x2,
 * two lane-ops per instruction), 2 = FP64 DFMA. Returns < 0 on error. */
double cbessfm_fma_peak(int32_t kind, double ms);

#ifdef __cplusplus
}
#endif

#endif /* CBESSFM_PEAKS_H */
