// Fine-step split-step Fourier propagation: the
// reference's ground-truth channel propagate_link and its exact inverse
// backward_propagate (channel.py:176-256), the IDEAL_SSFM variant of
// run_dbp (dbp.py:451-454).
//
// The whole waveform (n up to 2^22 per polarisation) is transformed with a
// four-step FFT, n = n1 * n2, data kept in natural time order [n1][n2]:
//   forward:  column FFTs of length n1, twiddle W_n^(j2 k1), row FFTs of
//             length n2 -> spectrum X[k1 + n1 k2] stored at (k1, k2);
//   inverse:  the same passes undone in reverse order.
// A fine step (channel.py:206-212) touches the spectrum only between the
// row FFT and the row IFFT, and the time samples only between the column
// IFFT and the column FFT, so one step is two fused passes over HBM/L2:
//   row phase    : FFT_n2 -> x half(dz_prev) -> x half(dz) -> IFFT_n2
//   column phase : x conj(W) -> IFFT_n1 -> /n -> exp(-j phi |E|^2) ->
//                  FFT_n1 -> x W
// Every phase is a loop over tiles (rows or column strips, both
// polarisations of one waveform per tile) held in shared memory; the
// phases are separated by grid-wide barriers of one cooperative launch
// that runs every span and step. The half-step tables are permuted on the
// host into the (k1, k2) storage order so the row phase reads them
// coalesced; the four-step twiddles come from two small tables.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/cbessfm_ssfm.h"
#include "cbessfm_kernel.cuh"

namespace cbessfm {
namespace ssfm {
namespace cg = cooperative_groups;

#ifndef CB_SSFM_THREADS  // experiment knob (build.py --variant ... --define)
#define CB_SSFM_THREADS 1024
#endif
constexpr int kThreads = CB_SSFM_THREADS;
constexpr int kTileElems = 4096;  // complex elements per tile, both polarisations
constexpr int kMaxLog2N = 22;     // n1, n2 <= 2048

// Shared-memory layout of a tile: sequence m of length L starts at
// m * seq_stride(L) and element i sits at pad(i). One pad slot per 128 B
// row plus one per sequence keeps the Stockham stride-RAD writes and the
// column-strip transposes free of bank conflicts.
template <typename R>
__host__ __device__ constexpr int pad_shift() {
  return sizeof(R) == 8 ? 4 : 3;
}
template <typename R>
__device__ __forceinline__ int spad(int i) {
  return i + (i >> pad_shift<R>());
}
template <typename R>
__host__ __device__ constexpr int seq_stride(int L) {
  return L + (L >> pad_shift<R>()) + 1;
}

template <typename R>
struct Params {
  Cx<R>* data;             // [batch][2][n], in place
  int64_t n;
  int batch;
  int n1, n2;              // column length, row length
  int rows, cols;          // rows per row tile, columns per column tile
  int lg_n2, lg_rows, lg_cols;
  const Cx<R>* tw_hi;      // W_n^(h << lo_bits)
  const Cx<R>* tw_lo;      // W_n^l, l < 2^lo_bits
  int lo_bits;
  const Cx<R>* tw1;        // W_n1^m
  const Cx<R>* tw2;        // W_n2^m
  const Cx<R>* half;       // [n_tables][n1][n2]
  const int* step_table;   // [k]
  const R* nl_coef;        // [k]
  int k;                   // fine steps per span
  int n_spans;
  int backward;
  R gain;
  const Cx<R>* noise;      // [n_spans][batch][2][n] or null
};

// One Stockham pass of radix RAD and stride ns over M sequences of length L
// (sequence m at buf + m * seq_stride(L), padded): inputs j + r L/RAD, twiddled by
// W_(RAD ns)^(r k), k = j mod ns, outputs (j/ns) ns RAD + k + r ns.
// Reads all of the thread's butterflies before a barrier, then writes.
// L and ns are compile-time: every pass is specialised (no runtime shifts,
// the butterfly arrays stay in registers).
template <typename R, int RAD, bool INV, int L, int NS>
__device__ __forceinline__ void stockham_pass(Cx<R>* buf, int M, const Cx<R>* __restrict__ twL) {
  constexpr int LR = L / RAD, SL = seq_stride<R>(L), TSTEP = L / (RAD * NS);
  constexpr int KMAX = (kTileElems / RAD + kThreads - 1) / kThreads;
  const int nb = M * LR, tid = threadIdx.x;
  Cx<R> v[KMAX][RAD];
#pragma unroll
  for (int q = 0; q < KMAX; ++q) {
    const int u = tid + q * kThreads;
    if (u < nb) {
      const int m = u / LR, j = u % LR, kk = j % NS;
      const Cx<R>* b = buf + m * SL;
#pragma unroll
      for (int r = 0; r < RAD; ++r) v[q][r] = b[spad<R>(j + r * LR)];
      if (NS > 1) {
#pragma unroll
        for (int r = 1; r < RAD; ++r) {
          const Cx<R> w = ldg(twL + r * kk * TSTEP);
          v[q][r] = INV ? cmulc(v[q][r], w) : cmul(v[q][r], w);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < KMAX; ++q) {
    const int u = tid + q * kThreads;
    if (u < nb) {
      const int m = u / LR, j = u % LR, kk = j % NS;
      Cx<R>* b = buf + m * SL;
      const int o = (j / NS) * NS * RAD + kk;
      if (RAD == 2) {
        b[spad<R>(o)] = v[q][0] + v[q][1];
        b[spad<R>(o + NS)] = v[q][0] - v[q][1];
      } else {
        const Cx<R> t0 = v[q][0] + v[q][2], t1 = v[q][0] - v[q][2];
        const Cx<R> t2 = v[q][1] + v[q][3], d = v[q][1] - v[q][3];
        const Cx<R> t3 = INV ? mk(-d.y, d.x) : mk(d.y, -d.x);  // +-j (a1 - a3)
        b[spad<R>(o)] = t0 + t2;
        b[spad<R>(o + NS)] = t1 + t3;
        b[spad<R>(o + 2 * NS)] = t0 - t2;
        b[spad<R>(o + 3 * NS)] = t1 - t3;
      }
    }
  }
  __syncthreads();
}

template <typename R, bool INV, int L, int NS>
__device__ __forceinline__ void radix4_passes(Cx<R>* buf, int M, const Cx<R>* twL) {
  if constexpr (NS < L) {
    stockham_pass<R, 4, INV, L, NS>(buf, M, twL);
    radix4_passes<R, INV, L, NS * 4>(buf, M, twL);
  }
}

// Unnormalised DFT (INV: conjugate kernel) of M sequences of length L.
template <typename R, bool INV, int L>
__device__ __noinline__ void cta_fft_l(Cx<R>* buf, int M, const Cx<R>* __restrict__ twL) {
  constexpr int LG = __builtin_ctz(L);
  if constexpr (LG & 1) {
    stockham_pass<R, 2, INV, L, 1>(buf, M, twL);
    radix4_passes<R, INV, L, 2>(buf, M, twL);
  } else {
    radix4_passes<R, INV, L, 1>(buf, M, twL);
  }
}

template <typename R, bool INV>
__device__ __forceinline__ void cta_fft(Cx<R>* buf, int M, int L, const Cx<R>* twL) {
  switch (L) {
    case 2: cta_fft_l<R, INV, 2>(buf, M, twL); break;
    case 4: cta_fft_l<R, INV, 4>(buf, M, twL); break;
    case 8: cta_fft_l<R, INV, 8>(buf, M, twL); break;
    case 16: cta_fft_l<R, INV, 16>(buf, M, twL); break;
    case 32: cta_fft_l<R, INV, 32>(buf, M, twL); break;
    case 64: cta_fft_l<R, INV, 64>(buf, M, twL); break;
    case 128: cta_fft_l<R, INV, 128>(buf, M, twL); break;
    case 256: cta_fft_l<R, INV, 256>(buf, M, twL); break;
    case 512: cta_fft_l<R, INV, 512>(buf, M, twL); break;
    case 1024: cta_fft_l<R, INV, 1024>(buf, M, twL); break;
    case 2048: cta_fft_l<R, INV, 2048>(buf, M, twL); break;
    default: break;  // L == 1: identity
  }
}

template <typename R>
__device__ __forceinline__ Cx<R> tw_n(const Params<R>& p, int64_t e) {
  return cmul(ldg(p.tw_hi + (e >> p.lo_bits)), ldg(p.tw_lo + (e & ((1 << p.lo_bits) - 1))));
}

// Row phase: FFT_n2, the spectral half steps, IFFT_n2 (channel.py:206, :211).
template <typename R>
__device__ void row_phase(const Params<R>& p, Cx<R>* buf, const Cx<R>* ha, const Cx<R>* hb) {
  const int per_wave = p.n1 >> p.lg_rows;
  const int tile_len = p.rows << p.lg_n2;  // per polarisation
  const int SL = seq_stride<R>(p.n2);
  // element e of the tile: pol, row r, column c -> sequence pol*rows + r
  auto at = [&](int e) {
    return buf + (e >> p.lg_n2) * SL + spad<R>(e & (p.n2 - 1));
  };
  for (int t = blockIdx.x; t < p.batch * per_wave; t += gridDim.x) {
    const int b = t / per_wave;
    const int64_t r0 = (int64_t)(t % per_wave) << p.lg_rows;
    Cx<R>* base = p.data + (int64_t)b * 2 * p.n + (r0 << p.lg_n2);
    for (int e = threadIdx.x; e < 2 * tile_len; e += kThreads) {
      const int pol = e >= tile_len, i = e - pol * tile_len;
      *at(e) = base[pol * p.n + i];
    }
    __syncthreads();
    cta_fft<R, false>(buf, 2 * p.rows, p.n2, p.tw2);
    if (ha || hb) {
      const int64_t h0 = r0 << p.lg_n2;
      for (int e = threadIdx.x; e < 2 * tile_len; e += kThreads) {
        const int pol = e >= tile_len, i = e - pol * tile_len;
        Cx<R> v = *at(e);
        if (ha) v = cmul(v, ldg(ha + h0 + i));
        if (hb) v = cmul(v, ldg(hb + h0 + i));
        *at(e) = v;
      }
      __syncthreads();
    }
    cta_fft<R, true>(buf, 2 * p.rows, p.n2, p.tw2);
    for (int e = threadIdx.x; e < 2 * tile_len; e += kThreads) {
      const int pol = e >= tile_len, i = e - pol * tile_len;
      base[pol * p.n + i] = *at(e);
    }
    __syncthreads();
  }
}

enum Mid { kNone = 0, kNonlinear = 1, kSpanEnd = 2 };

// Column phase. inv_in: conj twiddle + IFFT_n1 + 1/n (completes the
// inverse transform); then the time-domain operation; fwd_out: FFT_n1 +
// twiddle (starts the next forward transform).
template <typename R>
__device__ void col_phase(const Params<R>& p, Cx<R>* buf, bool inv_in, int mid, R nl,
                          const Cx<R>* noise, bool pre_div, bool fwd_out) {
  const int per_wave = p.n2 >> p.lg_cols;
  const int seq = p.n1;                  // sequence length
  const int tile_len = p.cols * seq;     // per polarisation
  const int SL = seq_stride<R>(seq);
  const R inv_n = (R)1 / (R)p.n;         // exact: n is a power of two
  for (int t = blockIdx.x; t < p.batch * per_wave; t += gridDim.x) {
    const int b = t / per_wave;
    const int c0 = (t % per_wave) << p.lg_cols;
    Cx<R>* base = p.data + (int64_t)b * 2 * p.n + c0;
    // element e: pol, row k1, column c (fastest) -> sequence pol*cols + c
    for (int e = threadIdx.x; e < 2 * tile_len; e += kThreads) {
      const int pol = e >= tile_len, i = e - pol * tile_len;
      const int k1 = i >> p.lg_cols, c = i & (p.cols - 1);
      Cx<R> v = base[pol * p.n + ((int64_t)k1 << p.lg_n2) + c];
      if (inv_in) v = cmulc(v, tw_n(p, (int64_t)(c0 + c) * k1));
      buf[(pol * p.cols + c) * SL + spad<R>(k1)] = v;
    }
    __syncthreads();
    if (inv_in) cta_fft<R, true>(buf, 2 * p.cols, seq, p.tw1);
    for (int e = threadIdx.x; e < tile_len; e += kThreads) {
      const int c = e / seq, j1 = e & (seq - 1);
      Cx<R>* px = buf + c * SL + spad<R>(j1);
      Cx<R>* py = buf + (p.cols + c) * SL + spad<R>(j1);
      Cx<R> x = *px, y = *py;
      if (inv_in) {
        x = scale(x, inv_n);
        y = scale(y, inv_n);
      }
      if (mid == kNonlinear) {
        // exp(-j sgn gamma Leff (|x|^2 + |y|^2)), channel.py:209-210
        const R pw = (x.x * x.x + x.y * x.y) + (y.x * y.x + y.y * y.y);
        R s, co;
        sincos_acc<R>(nl * pw, &s, &co);
        const Cx<R> rot = mk(co, s);
        x = cmul(x, rot);
        y = cmul(y, rot);
      } else if (mid == kSpanEnd && !p.backward) {
        // edfa: field gain, then ASE (channel.py:148-165)
        x = scale(x, p.gain);
        y = scale(y, p.gain);
        if (noise) {
          const int64_t at = (int64_t)b * 2 * p.n + ((int64_t)j1 << p.lg_n2) + c0 + c;
          x = x + ldg(noise + at);
          y = y + ldg(noise + at + p.n);
        }
      }
      if (pre_div) {  // backward_propagate: field / g before each span (channel.py:252)
        x = mk(x.x / p.gain, x.y / p.gain);
        y = mk(y.x / p.gain, y.y / p.gain);
      }
      *px = x;
      *py = y;
    }
    __syncthreads();
    if (fwd_out) cta_fft<R, false>(buf, 2 * p.cols, seq, p.tw1);
    for (int e = threadIdx.x; e < 2 * tile_len; e += kThreads) {
      const int pol = e >= tile_len, i = e - pol * tile_len;
      const int k1 = i >> p.lg_cols, c = i & (p.cols - 1);
      Cx<R> v = buf[(pol * p.cols + c) * SL + spad<R>(k1)];
      if (fwd_out) v = cmul(v, tw_n(p, (int64_t)(c0 + c) * k1));
      base[pol * p.n + ((int64_t)k1 << p.lg_n2) + c] = v;
    }
    __syncthreads();
  }
}

template <typename R>
__global__ void __launch_bounds__(kThreads, 1024 / kThreads) ssfm_kernel(Params<R> p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<R>* buf = reinterpret_cast<Cx<R>*>(smem_raw);
  cg::grid_group grid = cg::this_grid();
  const size_t tab = (size_t)p.n;
  for (int span = 0; span < p.n_spans; ++span) {
    if (span == 0)  // spec = fft(field) (channel.py:206), after / g when backward
      col_phase<R>(p, buf, false, kNone, (R)0, nullptr, p.backward != 0, true);
    for (int s = 0; s < p.k; ++s) {
      grid.sync();
      const Cx<R>* ha = s ? p.half + tab * p.step_table[s - 1] : nullptr;
      row_phase<R>(p, buf, ha, p.half + tab * p.step_table[s]);
      grid.sync();
      col_phase<R>(p, buf, true, kNonlinear, p.nl_coef[s], nullptr, false, true);
    }
    grid.sync();
    row_phase<R>(p, buf, p.half + tab * p.step_table[p.k - 1], (const Cx<R>*)nullptr);
    grid.sync();
    const bool more = span + 1 < p.n_spans;
    const Cx<R>* nz = p.noise ? p.noise + (int64_t)span * p.batch * 2 * p.n : nullptr;
    col_phase<R>(p, buf, true, kSpanEnd, (R)0, nz, more && p.backward, more);
    if (more) grid.sync();
  }
}

thread_local std::string g_err;

cbessfm_status fail(cbessfm_status s, const std::string& m) {
  g_err = m;
  return s;
}

struct Geo {
  int n1, n2, rows, cols;
  size_t smem;
};

Geo geometry(int64_t n, int batch, size_t esz, int target_tiles) {
  int lg = 0;
  while ((int64_t(1) << lg) < n) ++lg;
  Geo g;
  g.n2 = 1 << ((lg + 1) / 2);
  g.n1 = (int)(n / g.n2);
  g.rows = 1;
  while (g.rows * 2 <= g.n1 && 2 * (g.rows * 2) * g.n2 <= kTileElems &&
         (int64_t)batch * g.n1 / (g.rows * 2) >= target_tiles)
    g.rows *= 2;
  g.cols = 1;
  while (g.cols * 2 <= g.n2 && 2 * (g.cols * 2) * g.n1 <= kTileElems &&
         ((int64_t)batch * g.n2 / (g.cols * 2) >= target_tiles || g.cols < 4))
    g.cols *= 2;
  const int ps = esz == 16 ? 4 : 3;
  auto stride = [&](int L) { return L + (L >> ps) + 1; };
  g.smem = esz * (size_t)std::max(2 * g.rows * stride(g.n2), 2 * g.cols * stride(g.n1));
  return g;
}

std::vector<long double> unit_ld(int64_t n, int64_t count, int64_t stride) {
  // W_n^(m stride) for m < count, cos/sin in long double
  std::vector<long double> t(2 * count);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int64_t m = 0; m < count; ++m) {
    const long double a = -2.0L * pi * (long double)((m * stride) % n) / (long double)n;
    t[2 * m] = cosl(a);
    t[2 * m + 1] = sinl(a);
  }
  return t;
}

template <typename R>
cudaError_t upload(const std::vector<R>& h, void** d, cudaStream_t st) {
  cudaError_t e = cudaMallocAsync(d, std::max<size_t>(h.size(), 2) * sizeof(R), st);
  if (e != cudaSuccess) return e;
  if (h.empty()) return cudaSuccess;
  return cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(R), cudaMemcpyHostToDevice, st);
}

template <typename R>
std::vector<R> to_r(const std::vector<long double>& v) {
  std::vector<R> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = (R)v[i];
  return o;
}

template <typename R>
cbessfm_status run(const cbessfm_ssfm_desc* d, void* data, const void* noise, cudaStream_t st) {
  const int64_t n = d->n;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
  const Geo g = geometry(n, d->batch, sizeof(Cx<R>), 2 * sms);
  auto kern = ssfm_kernel<R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)g.smem);
  if (e != cudaSuccess) return fail(CBESSFM_ERR_CUDA, cudaGetErrorString(e));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, g.smem);
  if (occ < 1) return fail(CBESSFM_ERR_CUDA, "ssfm kernel does not fit on an SM");
  const int64_t tiles = std::max<int64_t>((int64_t)d->batch * g.n1 / g.rows,
                                          (int64_t)d->batch * g.n2 / g.cols);
  const int grid = (int)std::min<int64_t>((int64_t)occ * sms, tiles);

  // host tables: four-step twiddles, per-length twiddles, permuted halves
  int lo_bits = 0;
  while ((int64_t(1) << (2 * lo_bits)) < n) ++lo_bits;
  const int64_t n_lo = int64_t(1) << lo_bits, n_hi = (n + n_lo - 1) / n_lo;
  const std::vector<R> hi = to_r<R>(unit_ld(n, n_hi, n_lo)), lo = to_r<R>(unit_ld(n, n_lo, 1));
  const std::vector<R> t1 = to_r<R>(unit_ld(g.n1, g.n1, 1)), t2 = to_r<R>(unit_ld(g.n2, g.n2, 1));
  std::vector<R> half(2 * (size_t)d->n_tables * n);
  for (int tb = 0; tb < d->n_tables; ++tb)
    for (int64_t k1 = 0; k1 < g.n1; ++k1)
      for (int64_t k2 = 0; k2 < g.n2; ++k2) {
        const size_t src = (size_t)tb * n + (size_t)(k1 + (int64_t)g.n1 * k2);
        const size_t dst = (size_t)tb * n + (size_t)(k1 * g.n2 + k2);
        half[2 * dst] = (R)d->half[2 * src];
        half[2 * dst + 1] = (R)d->half[2 * src + 1];
      }
  std::vector<int> steps(d->step_table, d->step_table + d->steps_per_span);
  std::vector<R> nl(d->steps_per_span);
  for (int s = 0; s < d->steps_per_span; ++s) nl[s] = (R)d->nl_coef[s];

  void *dhi = nullptr, *dlo = nullptr, *d1 = nullptr, *d2 = nullptr, *dh = nullptr, *ds = nullptr,
       *dn = nullptr;
  if ((e = upload(hi, &dhi, st)) != cudaSuccess || (e = upload(lo, &dlo, st)) != cudaSuccess ||
      (e = upload(t1, &d1, st)) != cudaSuccess || (e = upload(t2, &d2, st)) != cudaSuccess ||
      (e = upload(half, &dh, st)) != cudaSuccess || (e = upload(steps, &ds, st)) != cudaSuccess ||
      (e = upload(nl, &dn, st)) != cudaSuccess)
    return fail(CBESSFM_ERR_CUDA, std::string("ssfm table upload: ") + cudaGetErrorString(e));

  Params<R> p;
  p.data = reinterpret_cast<Cx<R>*>(data);
  p.n = n;
  p.batch = d->batch;
  p.n1 = g.n1;
  p.n2 = g.n2;
  p.rows = g.rows;
  p.cols = g.cols;
  p.lg_n2 = __builtin_ctz(g.n2);
  p.lg_rows = __builtin_ctz(g.rows);
  p.lg_cols = __builtin_ctz(g.cols);
  p.tw_hi = reinterpret_cast<const Cx<R>*>(dhi);
  p.tw_lo = reinterpret_cast<const Cx<R>*>(dlo);
  p.lo_bits = lo_bits;
  p.tw1 = reinterpret_cast<const Cx<R>*>(d1);
  p.tw2 = reinterpret_cast<const Cx<R>*>(d2);
  p.half = reinterpret_cast<const Cx<R>*>(dh);
  p.step_table = reinterpret_cast<const int*>(ds);
  p.nl_coef = reinterpret_cast<const R*>(dn);
  p.k = d->steps_per_span;
  p.n_spans = d->n_spans;
  p.backward = d->backward;
  p.gain = (R)d->gain;
  p.noise = reinterpret_cast<const Cx<R>*>(noise);
  void* args[] = {&p};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kThreads), args, g.smem, st);
  for (void* ptr : {dhi, dlo, d1, d2, dh, ds, dn}) cudaFreeAsync(ptr, st);
  // the host staging vectors are read by the async copies
  const cudaError_t s2 = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(CBESSFM_ERR_CUDA, std::string("ssfm launch: ") + cudaGetErrorString(e));
  if (s2 != cudaSuccess) return fail(CBESSFM_ERR_CUDA, std::string("ssfm: ") + cudaGetErrorString(s2));
  return CBESSFM_OK;
}

}  // namespace ssfm
}  // namespace cbessfm

extern "C" {

cbessfm_status cbessfm_ssfm_info_get(int32_t dtype, int64_t n, int32_t batch, int32_t device,
                                     cbessfm_ssfm_info* info) {
  using namespace cbessfm::ssfm;
  g_err.clear();
  if (!info || n < 2 || (n & (n - 1)) || batch < 1)
    return fail(CBESSFM_ERR_INVALID, "n must be a power of two >= 2, batch >= 1");
  if (n > (int64_t(1) << kMaxLog2N)) return fail(CBESSFM_ERR_UNSUPPORTED, "n above 2^22");
  int sms = 148;
  if (device >= 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const size_t esz = dtype == CBESSFM_C64 ? 8 : 16;
  const Geo g = geometry(n, batch, esz, 2 * sms);
  info->n1 = g.n1;
  info->n2 = g.n2;
  info->rows_per_tile = g.rows;
  info->cols_per_tile = g.cols;
  info->threads = kThreads;
  info->smem_bytes = (int64_t)g.smem;
  info->grid = 0;
  return CBESSFM_OK;
}

cbessfm_status cbessfm_ssfm_run(const cbessfm_ssfm_desc* d, void* data, const void* noise,
                                void* stream) {
  using namespace cbessfm::ssfm;
  g_err.clear();
  if (!d || !data) return fail(CBESSFM_ERR_INVALID, "null desc or data");
  if (d->dtype != CBESSFM_C64 && d->dtype != CBESSFM_C128)
    return fail(CBESSFM_ERR_INVALID, "bad dtype");
  if (d->n < 2 || (d->n & (d->n - 1)))
    return fail(CBESSFM_ERR_UNSUPPORTED, "the GPU propagator needs a power-of-two length");
  if (d->n > (int64_t(1) << kMaxLog2N)) return fail(CBESSFM_ERR_UNSUPPORTED, "n above 2^22");
  if (d->batch < 1 || d->n_spans < 0 || d->steps_per_span < 1 || d->n_tables < 1 || !d->half ||
      !d->step_table || !d->nl_coef)
    return fail(CBESSFM_ERR_INVALID, "bad propagation description");
  for (int s = 0; s < d->steps_per_span; ++s)
    if (d->step_table[s] < 0 || d->step_table[s] >= d->n_tables)
      return fail(CBESSFM_ERR_INVALID, "step table index out of range");
  if (noise && d->backward) return fail(CBESSFM_ERR_INVALID, "ASE only on forward spans");
  if (d->n_spans == 0) return CBESSFM_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return d->dtype == CBESSFM_C64 ? run<float>(d, data, noise, st) : run<double>(d, data, noise, st);
}

const char* cbessfm_ssfm_last_error(void) { return cbessfm::ssfm::g_err.c_str(); }

}  // extern "C"
