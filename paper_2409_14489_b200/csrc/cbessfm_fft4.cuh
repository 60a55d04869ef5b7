// Shared four-step FFT machinery of the whole-sequence transforms (the
// fine-step propagator, csrc/cbessfm_ssfm.cu, and the receiver chain,
// csrc/cbessfm_rx.cu): n = n1 * n2, data in natural order [n1][n2], column
// phases (length-n1 FFTs of column strips) and row phases (length-n2 FFTs
// of rows) over tiles held in padded shared memory; the spectrum X[k1 + n1
// k2] is left at (k1, k2).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "cbessfm_kernel.cuh"

namespace cbessfm {
namespace ssfm {

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

// Row phase: FFT_n2, the spectral half steps, IFFT_n2 (channel.py:206, :211);
// fwd / inv select the transforms (a plain four-step FFT or IFFT uses one).
template <typename R>
__device__ void row_phase(const Params<R>& p, Cx<R>* buf, const Cx<R>* ha, const Cx<R>* hb,
                          bool fwd = true, bool inv = true) {
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
    if (fwd) cta_fft<R, false>(buf, 2 * p.rows, p.n2, p.tw2);
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
    if (inv) cta_fft<R, true>(buf, 2 * p.rows, p.n2, p.tw2);
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


// ---------------------------------------------------------------- host side

struct Geo {
  int n1, n2, rows, cols;
  size_t smem;
};

inline Geo geometry(int64_t n, int batch, size_t esz, int target_tiles) {
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

inline std::vector<long double> unit_ld(int64_t n, int64_t count, int64_t stride) {
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


// Device twiddle tables of one four-step geometry. build() uploads them on
// `st` and fills the transform fields of p; the host staging vectors live
// here until release(), which the caller issues after synchronising.
template <typename R>
struct Fft4Tables {
  std::vector<R> hi, lo, t1, t2;
  void *dhi = nullptr, *dlo = nullptr, *d1 = nullptr, *d2 = nullptr;

  cudaError_t build(int64_t n, const Geo& g, cudaStream_t st, Params<R>* p) {
    int lo_bits = 0;
    while ((int64_t(1) << (2 * lo_bits)) < n) ++lo_bits;
    const int64_t n_lo = int64_t(1) << lo_bits, n_hi = (n + n_lo - 1) / n_lo;
    hi = to_r<R>(unit_ld(n, n_hi, n_lo));
    lo = to_r<R>(unit_ld(n, n_lo, 1));
    t1 = to_r<R>(unit_ld(g.n1, g.n1, 1));
    t2 = to_r<R>(unit_ld(g.n2, g.n2, 1));
    cudaError_t e;
    if ((e = upload(hi, &dhi, st)) != cudaSuccess || (e = upload(lo, &dlo, st)) != cudaSuccess ||
        (e = upload(t1, &d1, st)) != cudaSuccess || (e = upload(t2, &d2, st)) != cudaSuccess)
      return e;
    p->n = n;
    p->n1 = g.n1;
    p->n2 = g.n2;
    p->rows = g.rows;
    p->cols = g.cols;
    p->lg_n2 = __builtin_ctz(g.n2);
    p->lg_rows = __builtin_ctz(g.rows);
    p->lg_cols = __builtin_ctz(g.cols);
    p->tw_hi = reinterpret_cast<const Cx<R>*>(dhi);
    p->tw_lo = reinterpret_cast<const Cx<R>*>(dlo);
    p->lo_bits = lo_bits;
    p->tw1 = reinterpret_cast<const Cx<R>*>(d1);
    p->tw2 = reinterpret_cast<const Cx<R>*>(d2);
    return cudaSuccess;
  }
  void release(cudaStream_t st) {
    for (void* ptr : {dhi, dlo, d1, d2})
      if (ptr) cudaFreeAsync(ptr, st);
    dhi = dlo = d1 = d2 = nullptr;
  }
};

}  // namespace ssfm
}  // namespace cbessfm
