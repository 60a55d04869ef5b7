// Receiver chain at scale: per-channel soft symbols of a
// whole-band waveform and their SNR (signals.py:260-346, metrics.py:54-140).
//
// The reference chains demux (FFT_n, bin slice, IFFT_m), matched filter
// (FFT_m, x RRC, IFFT_m) and the symbol-rate resample (FFT_m, fold onto
// the symbol grid, IFFT_L). The inner IFFT/FFT pairs cancel, so here the
// chain is: one four-step FFT of the band (csrc/cbessfm_fft4.cuh), a gather
// that builds every channel's symbol-grid spectrum
//   Y_c[t] = (L/m) sum_{s = t mod L, -m/2 <= s < m/2} (m/n) S[c_idx + s] g[s]
// (same scalings, same fold order as np.add.at) directly in the transposed
// order of the length-L inverse four-step, and that inverse (all channels
// in one batch) with the launch-amplitude division fused into its last
// pass. SNR: two reductions per channel (correlation, then signal and
// error energies after the joint phase removal).
#include <cuda_runtime.h>

#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/cbessfm_rx.h"
#include "cbessfm_fft4.cuh"

namespace cbessfm {
namespace rx {
using namespace ssfm;

template <typename R, int LG>
__global__ void __launch_bounds__(kThreads, 1024 / kThreads)
    col_kernel(const __grid_constant__ ssfm::Params<R> p, int inv_in, int fwd_out, int pre_div) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CB_POISON_SMEM(smem_raw);
  col_phase<R, Split<LG>::N1>(p, reinterpret_cast<Cx<R>*>(smem_raw), inv_in != 0, kNone, (R)0,
                              nullptr, pre_div != 0, fwd_out != 0);
}

template <typename R, int LG>
__global__ void __launch_bounds__(kThreads, 1024 / kThreads)
    row_kernel(const __grid_constant__ ssfm::Params<R> p, int fwd, int inv) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CB_POISON_SMEM(smem_raw);
  row_phase<R, Split<LG>::N2>(p, reinterpret_cast<Cx<R>*>(smem_raw), (const Cx<R>*)nullptr,
                              (const Cx<R>*)nullptr, fwd != 0, inv != 0);
}

template <typename R>
struct ColFor {
  template <int LG>
  struct At {
    static const void* get() { return (const void*)col_kernel<R, LG>; }
  };
};
template <typename R>
struct RowFor {
  template <int LG>
  struct At {
    static const void* get() { return (const void*)row_kernel<R, LG>; }
  };
};

struct Grid {
  int64_t n;       // length
  int n1, lg_n2;   // X[k] sits at (k mod n1) << lg_n2 | k / n1
};

template <typename R>
__global__ void gather_kernel(const Cx<R>* __restrict__ S, Grid gs, Cx<R>* __restrict__ Y,
                              Grid gl, const int64_t* __restrict__ cidx, int64_t m,
                              const double* __restrict__ g, R demux_scale, R fold_scale,
                              int n_ch) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t L = gl.n;
  if (idx >= (int64_t)n_ch * L) return;
  const int c = (int)(idx / L);
  const int64_t t = idx - (int64_t)c * L;
  const int64_t h = m / 2;
  const int64_t q_max = (t + h) / L;  // s = t - q L >= -m/2
  for (int pol = 0; pol < 2; ++pol) {
    const Cx<R>* Sp = S + pol * gs.n;
    Cx<R> acc = mk((R)0, (R)0);
    auto term = [&](int64_t s) {
      int64_t k = (cidx[c] + s) % gs.n;
      if (k < 0) k += gs.n;
      Cx<R> v = Sp[((k % gs.n1) << gs.lg_n2) + k / gs.n1];
      v = mk(v.x * demux_scale, v.y * demux_scale);            // signals.py:343
      const R gj = (R)g[s >= 0 ? s : s + m];                  // signals.py:268
      return mk(v.x * gj, v.y * gj);
    };
    // np.add.at order: unshifted bins ascending = s >= 0 first, then s < 0
    for (int64_t s = t; s < h; s += L) acc = acc + term(s);
    for (int64_t q = q_max; q >= 1; --q) acc = acc + term(t - q * L);
    acc = mk(acc.x * fold_scale, acc.y * fold_scale);          // signals.py:316
    Y[((int64_t)c * 2 + pol) * L + (((t % gl.n1) << gl.lg_n2) + t / gl.n1)] = acc;
  }
}

constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_reduce(double v, double* sh) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kRedThreads / 32; ++i) r += sh[i];
  __syncthreads();
  return r;
}

// pass 1: corr_c = sum rx conj(tx) over both polarisations (metrics.py:73)
template <typename R>
__global__ void corr_kernel(const Cx<R>* rx, const Cx<R>* tx, int64_t per_ch, double* out) {
  __shared__ double sh[kRedThreads / 32];
  const int c = blockIdx.y;
  double re = 0.0, im = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < per_ch;
       i += (int64_t)gridDim.x * kRedThreads) {
    const Cx<R> a = rx[c * per_ch + i], b = tx[c * per_ch + i];
    re += (double)a.x * b.x + (double)a.y * b.y;
    im += (double)a.y * b.x - (double)a.x * b.y;
  }
  re = block_reduce(re, sh);
  im = block_reduce(im, sh);
  if (threadIdx.x == 0) {
    atomicAdd(out + 2 * c, re);
    atomicAdd(out + 2 * c + 1, im);
  }
}

// pass 2: per polarisation sum |tx|^2 and sum |rx e^{-j phi} - tx|^2
// (metrics.py:78, :81-90)
template <typename R>
__global__ void energy_kernel(const Cx<R>* rx, const Cx<R>* tx, int64_t per_pol,
                              const double* phase, double* out) {
  __shared__ double sh[kRedThreads / 32];
  const int c = blockIdx.y, pol = blockIdx.z;
  double cs, sn;
  sincos(phase[c], &sn, &cs);
  const double rr = cs, ri = -sn;  // exp(-j phi)
  double sig = 0.0, noise = 0.0;
  const int64_t base = ((int64_t)c * 2 + pol) * per_pol;
  for (int64_t i = (int64_t)blockIdx.x * kRedThreads + threadIdx.x; i < per_pol;
       i += (int64_t)gridDim.x * kRedThreads) {
    const Cx<R> a = rx[base + i], b = tx[base + i];
    const double ar = (double)a.x * rr - (double)a.y * ri;
    const double ai = (double)a.x * ri + (double)a.y * rr;
    const double dr = ar - b.x, di = ai - b.y;
    sig += (double)b.x * b.x + (double)b.y * b.y;
    noise += dr * dr + di * di;
  }
  sig = block_reduce(sig, sh);
  noise = block_reduce(noise, sh);
  if (threadIdx.x == 0) {
    atomicAdd(out + 4 * c + 2 * pol, sig);
    atomicAdd(out + 4 * c + 2 * pol + 1, noise);
  }
}

thread_local std::string g_err;

cbessfm_status fail(cbessfm_status s, const std::string& m) {
  g_err = m;
  return s;
}

struct Plan {
  int64_t n, m, L;
  std::vector<int64_t> cidx;
  std::vector<double> g;
};

cbessfm_status plan(const cbessfm_rx_desc* d, Plan* pl, bool need_g = true) {
  if (!d) return fail(CBESSFM_ERR_INVALID, "null rx description");
  if (d->n < 2 || (d->n & (d->n - 1)))
    return fail(CBESSFM_ERR_UNSUPPORTED, "the GPU receiver needs a power-of-two length");
  if (d->n > (int64_t(1) << kMaxLog2N)) return fail(CBESSFM_ERR_UNSUPPORTED, "n above 2^22");
  if (d->n_channels < 1 || !d->channel_freq || !(d->sample_rate > 0) || !(d->baud > 0))
    return fail(CBESSFM_ERR_INVALID, "bad channel plan");
  const double df = d->sample_rate / (double)d->n;
  // demux_channel (signals.py:329-341)
  int64_t m = (int64_t)std::llround(d->bandwidth / df);
  m -= m % 2;
  if (m < 2 || m > d->n) return fail(CBESSFM_ERR_INVALID, "bandwidth out of range for this grid");
  pl->n = d->n;
  pl->m = m;
  pl->cidx.resize(d->n_channels);
  for (int c = 0; c < d->n_channels; ++c) {
    const int64_t ci = (int64_t)std::llround(d->channel_freq[c] / df);
    const int64_t lo = d->n / 2 + ci - m / 2;
    if (lo < 0 || lo + m > d->n)
      return fail(CBESSFM_ERR_INVALID, "channel band exceeds the sampled spectrum");
    pl->cidx[c] = ci;
  }
  // resample to the symbol rate (signals.py:296-300)
  const double rate_c = (double)m * df;
  const double lf = (double)m * d->baud / rate_c;
  const int64_t L = (int64_t)std::llround(lf);
  if (std::fabs(lf - (double)L) > 1e-6)
    return fail(CBESSFM_ERR_INVALID, "new_rate not representable on this block grid");
  if (L < 2 || (L & (L - 1)))
    return fail(CBESSFM_ERR_UNSUPPORTED, "the GPU receiver needs a power-of-two symbol count");
  pl->L = L;
  if (!need_g) return CBESSFM_OK;
  // sqrt(raised_cosine_spectrum(fftfreq(m, 1/rate_c))) (signals.py:186-201, :268)
  pl->g.resize(m);
  const double pass_edge = (1 - d->rolloff) * d->baud / 2, stop_edge = (1 + d->rolloff) * d->baud / 2;
  const double val = 1.0 / ((double)m * (1.0 / rate_c));  // np.fft.fftfreq scaling
  for (int64_t j = 0; j < m; ++j) {
    const int64_t s = j < (m + 1) / 2 ? j : j - m;
    const double f = std::fabs((double)s * val);
    double rc = 0.0;
    if (f <= pass_edge)
      rc = 1.0;
    else if (d->rolloff > 0 && f < stop_edge)
      rc = 0.5 * (1 + std::cos(M_PI / (d->rolloff * d->baud) * (f - pass_edge)));
    pl->g[j] = std::sqrt(rc);
  }
  return CBESSFM_OK;
}

cbessfm_status cuda_fail(cudaError_t e, const char* what) {
  return fail(CBESSFM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename R>
cudaError_t launch_transform(ssfm::Params<R>& p, const Geo& g, bool inverse, bool div, cudaStream_t st) {
  const int lg = __builtin_ctzll(p.n);
  const void* ck = dispatch_lg<ColFor<R>::template At>(lg);
  const void* rk = dispatch_lg<RowFor<R>::template At>(lg);
  if (!ck || !rk) return cudaErrorInvalidValue;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(ck, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem)) ||
      (e = cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem)))
    return e;
  const unsigned col_tiles = (unsigned)((int64_t)p.batch * g.n2 / g.cols);
  const unsigned row_tiles = (unsigned)((int64_t)p.batch * g.n1 / g.rows);
  int one = 1, zero = 0, dv = div ? 1 : 0;
  void* cfwd[] = {&p, &zero, &one, &zero};
  void* rfwd[] = {&p, &one, &zero};
  void* rinv[] = {&p, &zero, &one};
  void* cinv[] = {&p, &one, &zero, &dv};
  if (!inverse) {
    if ((e = cudaLaunchKernel(ck, dim3(col_tiles), dim3(kThreads), cfwd, g.smem, st))) return e;
    return cudaLaunchKernel(rk, dim3(row_tiles), dim3(kThreads), rfwd, g.smem, st);
  }
  if ((e = cudaLaunchKernel(rk, dim3(row_tiles), dim3(kThreads), rinv, g.smem, st))) return e;
  return cudaLaunchKernel(ck, dim3(col_tiles), dim3(kThreads), cinv, g.smem, st);
}

// Twiddle tables per transform geometry and device, built once and kept
// (a receiver is called per waveform with the same grid).
template <typename R>
struct CachedTables {
  Fft4Tables<R> t;
  ssfm::Params<R> p{};
};

template <typename R>
cudaError_t cached_params(int64_t n, const Geo& g, int device, cudaStream_t st,
                          ssfm::Params<R>* out) {
  static std::mutex mu;
  static std::map<std::tuple<int64_t, int, int, int, int>, std::unique_ptr<CachedTables<R>>> cache;
  const auto key = std::make_tuple(n, g.n1, g.rows, g.cols, device);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it == cache.end()) {
    auto entry = std::make_unique<CachedTables<R>>();
    cudaError_t e = entry->t.build(n, g, st, &entry->p);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    it = cache.emplace(key, std::move(entry)).first;
  }
  *out = it->second->p;
  return cudaSuccess;
}

// The matched-filter response on the channel grid, uploaded once per
// (grid, pulse, device).
cudaError_t cached_filter(const Plan& pl, const cbessfm_rx_desc* d, cudaStream_t st,
                          const void** out) {
  static std::mutex mu;
  static std::map<std::tuple<int64_t, double, double, double, double, int>, void*> cache;
  const auto key = std::make_tuple(pl.m, d->sample_rate / (double)d->n, d->baud, d->rolloff,
                                   (double)d->n, d->device);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it == cache.end()) {
    void* dg = nullptr;
    cudaError_t e = cudaMalloc(&dg, pl.g.size() * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(dg, pl.g.data(), pl.g.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    it = cache.emplace(key, dg).first;
  }
  *out = it->second;
  return cudaSuccess;
}

template <typename R>
cbessfm_status symbols(const cbessfm_rx_desc* d, const Plan& pl, const void* in, void* out,
                       cudaStream_t st) {
  using C = Cx<R>;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
  const Geo gs = geometry(pl.n, 1, sizeof(C), 2 * sms);
  const Geo gl = geometry(pl.L, d->n_channels, sizeof(C), 2 * sms);
  void *spec = nullptr, *dcidx = nullptr;
  const void* dg = nullptr;
  StreamFrees frees(st);
  cudaError_t e = cudaMallocAsync(&spec, 2 * pl.n * sizeof(C), st);
  frees.add(spec);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(spec, in, 2 * pl.n * sizeof(C), cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess) e = upload(pl.cidx, &dcidx, st);
  frees.add(dcidx);
  if (e == cudaSuccess) e = cached_filter(pl, d, st, &dg);
  if (e != cudaSuccess) return cuda_fail(e, "rx staging");
  ssfm::Params<R> ps{}, pls{};
  if ((e = cached_params<R>(pl.n, gs, d->device, st, &ps)) ||
      (e = cached_params<R>(pl.L, gl, d->device, st, &pls)))
    return cuda_fail(e, "rx twiddles");
  ps.data = reinterpret_cast<C*>(spec);
  ps.batch = 1;
  if ((e = launch_transform<R>(ps, gs, false, false, st))) return cuda_fail(e, "band FFT");
  const int64_t total = (int64_t)d->n_channels * pl.L;
  Grid g_s{pl.n, gs.n1, __builtin_ctz(gs.n2)}, g_l{pl.L, gl.n1, __builtin_ctz(gl.n2)};
  gather_kernel<R><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      reinterpret_cast<const C*>(spec), g_s, reinterpret_cast<C*>(out), g_l,
      reinterpret_cast<const int64_t*>(dcidx), pl.m, reinterpret_cast<const double*>(dg),
      (R)((double)pl.m / (double)pl.n), (R)((double)pl.L / (double)pl.m), d->n_channels);
  if ((e = cudaGetLastError())) return cuda_fail(e, "channel gather");
  pls.data = reinterpret_cast<C*>(out);
  pls.batch = d->n_channels;
  pls.gain = (R)std::sqrt(d->launch_power_w / 2);  // metrics.py:138-140
  if ((e = launch_transform<R>(pls, gl, true, true, st))) return cuda_fail(e, "symbol IFFT");
  if ((e = cudaStreamSynchronize(st))) return cuda_fail(e, "rx");
  return CBESSFM_OK;
}

}  // namespace rx
}  // namespace cbessfm

extern "C" {

int64_t cbessfm_rx_symbol_count(const cbessfm_rx_desc* d) {
  using namespace cbessfm::rx;
  g_err.clear();
  Plan pl;
  if (plan(d, &pl, false) != CBESSFM_OK) return -1;
  return pl.L;
}

cbessfm_status cbessfm_rx_symbols(const cbessfm_rx_desc* d, const void* in, void* out,
                                  void* stream) {
  using namespace cbessfm::rx;
  g_err.clear();
  Plan pl;
  if (cbessfm_status s = plan(d, &pl)) return s;
  if (!in || !out) return fail(CBESSFM_ERR_INVALID, "null buffers");
  if (d->dtype != CBESSFM_C64 && d->dtype != CBESSFM_C128) return fail(CBESSFM_ERR_INVALID, "bad dtype");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return d->dtype == CBESSFM_C64 ? symbols<float>(d, pl, in, out, st)
                                 : symbols<double>(d, pl, in, out, st);
}

cbessfm_status cbessfm_rx_snr(int32_t dtype, int32_t n_ch, int64_t n_sym, const void* rx,
                              const void* tx, double* out, void* stream) {
  using namespace cbessfm::rx;
  g_err.clear();
  if (n_ch < 1 || n_sym < 1 || !rx || !tx || !out) return fail(CBESSFM_ERR_INVALID, "bad arguments");
  if (dtype != CBESSFM_C64 && dtype != CBESSFM_C128) return fail(CBESSFM_ERR_INVALID, "bad dtype");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  double* acc = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync((void**)&acc, sizeof(double) * 7 * n_ch, st)) ||
      (e = cudaMemsetAsync(acc, 0, sizeof(double) * 7 * n_ch, st)))
    return cuda_fail(e, "snr alloc");
  double* corr = acc;                 // [n_ch][2]
  double* phase = acc + 2 * n_ch;     // [n_ch]
  double* energy = acc + 3 * n_ch;    // [n_ch][2 pol][sig, noise]
  const unsigned blocks = (unsigned)std::min<int64_t>(64, (2 * n_sym + kRedThreads - 1) / kRedThreads);
  std::vector<double> h(7 * n_ch);
  if (dtype == CBESSFM_C64)
    corr_kernel<float><<<dim3(blocks, n_ch), kRedThreads, 0, st>>>(
        (const cbessfm::Cx<float>*)rx, (const cbessfm::Cx<float>*)tx, 2 * n_sym, corr);
  else
    corr_kernel<double><<<dim3(blocks, n_ch), kRedThreads, 0, st>>>(
        (const cbessfm::Cx<double>*)rx, (const cbessfm::Cx<double>*)tx, 2 * n_sym, corr);
  if ((e = cudaMemcpyAsync(h.data(), corr, sizeof(double) * 2 * n_ch, cudaMemcpyDeviceToHost, st)) ||
      (e = cudaStreamSynchronize(st)))
    return cuda_fail(e, "snr correlation");
  std::vector<double> ph(n_ch);
  for (int c = 0; c < n_ch; ++c) {
    if (h[2 * c] == 0.0 && h[2 * c + 1] == 0.0) {
      cudaFreeAsync(acc, st);
      return fail(CBESSFM_ERR_INVALID, "zero cross-correlation; mean phase undefined");
    }
    ph[c] = std::atan2(h[2 * c + 1], h[2 * c]);  // np.angle (metrics.py:76)
  }
  if ((e = cudaMemcpyAsync(phase, ph.data(), sizeof(double) * n_ch, cudaMemcpyHostToDevice, st)))
    return cuda_fail(e, "snr phase");
  const unsigned b2 = (unsigned)std::min<int64_t>(64, (n_sym + kRedThreads - 1) / kRedThreads);
  if (dtype == CBESSFM_C64)
    energy_kernel<float><<<dim3(b2, n_ch, 2), kRedThreads, 0, st>>>(
        (const cbessfm::Cx<float>*)rx, (const cbessfm::Cx<float>*)tx, n_sym, phase, energy);
  else
    energy_kernel<double><<<dim3(b2, n_ch, 2), kRedThreads, 0, st>>>(
        (const cbessfm::Cx<double>*)rx, (const cbessfm::Cx<double>*)tx, n_sym, phase, energy);
  if ((e = cudaMemcpyAsync(h.data(), energy, sizeof(double) * 4 * n_ch, cudaMemcpyDeviceToHost, st)) ||
      (e = cudaStreamSynchronize(st)))
    return cuda_fail(e, "snr energies");
  cudaFreeAsync(acc, st);
  auto db = [](double sig, double noise) {  // _pool_snr_db (metrics.py:81-90)
    if (noise <= sig * 1e-30) return 100.0;
    return std::min(10 * std::log10(sig / noise), 100.0);
  };
  for (int c = 0; c < n_ch; ++c) {
    const double sx = h[4 * c], nx = h[4 * c + 1], sy = h[4 * c + 2], ny = h[4 * c + 3];
    if (sx + sy == 0.0) return fail(CBESSFM_ERR_INVALID, "tx symbols carry no energy");
    out[4 * c] = db(sx + sy, nx + ny);
    out[4 * c + 1] = db(sx, nx);
    out[4 * c + 2] = db(sy, ny);
    out[4 * c + 3] = ph[c];
  }
  return CBESSFM_OK;
}

const char* cbessfm_rx_last_error(void) { return cbessfm::rx::g_err.c_str(); }

}  // extern "C"
