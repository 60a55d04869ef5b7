/*
 * cbessfm_rx.h -- C ABI of the receiver chain at scale in
 * libcbessfm.so: per-channel soft symbols and SNR of a whole-band waveform,
 *     demux_channel(w, f_c, bw)                 signals.py:323-346
 *     matched_filter(w, wdm)                    signals.py:260-270
 *     resample(w, baud, allow_alias=True)       signals.py:290-320
 *     symbols_from_dbp_output(w, wdm)           metrics.py:131-140
 *     snr(rx, tx)                               metrics.py:54-105
 * The chain's transforms collapse in the frequency domain: one four-step
 * FFT of the whole band, then per channel a gather of its bins (brick-wall
 * demux, RRC matched filter, fold onto the symbol grid) written straight
 * into the transposed order of a symbol-length inverse four-step FFT.
 *
 * Conventions as in cbessfm.h (status codes).
 */
#ifndef CBESSFM_RX_H
#define CBESSFM_RX_H

#include <stdint.h>

#include "cbessfm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t dtype;              /* cbessfm_dtype of the waveform and symbols   */
  int64_t n;                  /* samples per polarisation (power of two)     */
  double sample_rate;         /* Hz                                          */
  int32_t n_channels;
  const double* channel_freq; /* HOST [n_channels], Hz from the band centre  */
  double bandwidth;           /* demux bandwidth, Hz (n_channels > 1 or rate
                                 above the channel's: brick wall)            */
  double baud;                /* symbol rate, Hz                             */
  double rolloff;             /* RRC roll-off                                */
  double launch_power_w;      /* per-channel launch power (amplitude undo)   */
  int32_t device;
} cbessfm_rx_desc;

/* Number of symbols per channel and polarisation the chain produces
 * (round(baud / (rate / n)), resample's grid), or -1 (cbessfm_rx_last_error). */
int64_t cbessfm_rx_symbol_count(const cbessfm_rx_desc* desc);

/* in: DEVICE [2][n] (x then y), not modified. out: DEVICE
 * [n_channels][2][n_sym] soft symbols. Synchronous. */
cbessfm_status cbessfm_rx_symbols(const cbessfm_rx_desc* desc, const void* in, void* out,
                                  void* stream);

/* SNR of rx against tx (both DEVICE [n_channels][2][n_sym] of dtype), with
 * the joint mean-phase removal of metrics.py:62-78. out: HOST
 * [n_channels][4] = pooled dB, x dB, y dB, removed phase (rad); the dB
 * figures are capped at 100 as the reference does. Synchronous. */
cbessfm_status cbessfm_rx_snr(int32_t dtype, int32_t n_channels, int64_t n_sym, const void* rx,
                              const void* tx, double* out, void* stream);

const char* cbessfm_rx_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CBESSFM_RX_H */
