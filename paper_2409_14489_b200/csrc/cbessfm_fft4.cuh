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
#ifndef CB_SSFM_TILE      // experiment knob
#define CB_SSFM_TILE 4096
#endif
constexpr int kTileElems = CB_SSFM_TILE;  // complex elements per tile, both polarisations
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
  int buf_elems;           // elements of each of the two tile buffers
  const Cx<R>* twn;        // [n1][n2]: W_n^(j2 k1) at (k1, j2), laid out like the data
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

// One Stockham pass of radix RAD and stride NS over M sequences of length L
// (sequence m at m * seq_stride(L), padded), from src to dst: inputs
// j + r L/RAD, twiddled by W_(RAD NS)^(r k), k = j mod NS, outputs
// (j/NS) NS RAD + k + r NS. Ping-pong buffers: one barrier per pass and no
// value lives across it (a butterfly kept in registers over a barrier is
// what ptxas spills once the tile loop hoists its addressing).
template <typename R, int RAD, bool INV, int L, int NS>
__device__ __forceinline__ void stockham_pass(const Cx<R>* src, Cx<R>* dst, int M,
                                              const Cx<R>* __restrict__ twL, const int* zero) {
  constexpr int LR = L / RAD, SL = seq_stride<R>(L), TSTEP = L / (RAD * NS);
  // the shared zero read keeps ptxas from hoisting every pass's addressing
  // out of the tile loop
  const unsigned nb = M * LR;
  for (unsigned u = threadIdx.x + *(volatile const int*)zero; u < nb; u += kThreads) {
    const unsigned m = u / LR, j = u % LR, kk = j % NS;
    const Cx<R>* b = src + m * SL;
    Cx<R> v[RAD];
#pragma unroll
    for (int r = 0; r < RAD; ++r) v[r] = b[spad<R>(j + r * LR)];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < RAD; ++r) {
        const Cx<R> w = twL[r * kk * TSTEP];  // staged in shared memory
        v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
      }
    }
    dft_reg<R, RAD, INV>(v);  // in place, outputs in bit-reversed order
    Cx<R>* o = dst + m * SL;
    const int base = (j / NS) * NS * RAD + kk;
#pragma unroll
    for (int r = 0; r < RAD; ++r) o[spad<R>(base + r * NS)] = v[bitrev<RAD>(r)];
  }
  __syncthreads();
}

template <typename R, bool INV, int L, int NS, int PASS>
__device__ __forceinline__ void radix4_passes(Cx<R>* a, Cx<R>* b, int M, const Cx<R>* twL,
                                              const int* z) {
  if constexpr (NS < L) {
    if constexpr (PASS & 1)
      stockham_pass<R, 4, INV, L, NS>(b, a, M, twL, z);
    else
      stockham_pass<R, 4, INV, L, NS>(a, b, M, twL, z);
    radix4_passes<R, INV, L, NS * 4, PASS + 1>(a, b, M, twL, z);
  }
}

template <typename R, bool INV, int L, int NS, int PASS>
__device__ __forceinline__ void radix8_passes(Cx<R>* a, Cx<R>* b, int M, const Cx<R>* twL,
                                              const int* z) {
  if constexpr (NS < L) {
    if constexpr (PASS & 1)
      stockham_pass<R, 8, INV, L, NS>(b, a, M, twL, z);
    else
      stockham_pass<R, 8, INV, L, NS>(a, b, M, twL, z);
    radix8_passes<R, INV, L, NS * 8, PASS + 1>(a, b, M, twL, z);
  }
}

// FP32 tiles run radix-8 passes (8 complex values fit the 64-register
// budget), FP64 tiles radix-4 (radix-8 doubles would spill); the leftover
// factor of L leads.
template <typename R>
constexpr int tile_radix_log() {
  return sizeof(R) == 4 ? 3 : 2;
}

template <typename R, int L>
constexpr int fft_passes() {
  constexpr int B = tile_radix_log<R>(), LG = __builtin_ctz(L);
  return (LG % B != 0) + LG / B;
}

// Unnormalised DFT (INV: conjugate kernel) of M sequences of length L that
// start in buffer a; returns the buffer holding the result (a after an even
// number of passes, b after an odd one).
template <typename R, bool INV, int L>
__device__ __forceinline__ Cx<R>* cta_fft_l(Cx<R>* a, Cx<R>* b, int M,
                                            const Cx<R>* __restrict__ twL, const int* z) {
  constexpr int B = tile_radix_log<R>(), REM = __builtin_ctz(L) % B;
  if constexpr (REM != 0) stockham_pass<R, (1 << REM), INV, L, 1>(a, b, M, twL, z);
  constexpr int NS0 = REM ? (1 << REM) : 1, P0 = REM ? 1 : 0;
  if constexpr (B == 3)
    radix8_passes<R, INV, L, NS0, P0>(a, b, M, twL, z);
  else
    radix4_passes<R, INV, L, NS0, P0>(a, b, M, twL, z);
  return (fft_passes<R, L>() & 1) ? b : a;
}

// The four-step twiddle W_n^(j2 k1) of element (k1, j2): one coalesced
// load from a table with the data's layout.
template <typename R>
__device__ __forceinline__ Cx<R> tw_n(const Params<R>& p, int k1, int j2) {
  return ldg(p.twn + ((int64_t)k1 << p.lg_n2) + j2);
}

// twn[k1 n2 + j2] = exp(-2 pi i ((j2 k1) mod n) / n): sincospi of an exactly
// representable argument (n is a power of two), about 1 ulp.
template <typename R>
__global__ void fill_twn(Cx<R>* twn, int64_t n, int n2, int lg_n2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t k1 = i >> lg_n2, j2 = i & (n2 - 1);
  const int64_t e = (k1 * j2) & (n - 1);
  R s, c;
  if constexpr (sizeof(R) == 8)
    sincospi(-2.0 * (double)e / (double)n, &s, &c);
  else
    sincospif(-2.0f * (float)e / (float)n, &s, &c);
  twn[i] = mk(c, s);
}

// Row phase: FFT_n2, the spectral half steps, IFFT_n2 (channel.py:206, :211);
// fwd / inv select the transforms (a plain four-step FFT or IFFT uses one).
// N2 == p.n2 at compile time (kernels are instantiated per transform length).
template <typename R, int N2>
__device__ __noinline__ void row_phase(const Params<R>& p, Cx<R>* buf, const Cx<R>* ha, const Cx<R>* hb,
                          bool fwd = true, bool inv = true, bool staged = false) {
  __shared__ int s_zero;
  if (threadIdx.x == 0) s_zero = 0;
  __syncthreads();
  const int per_wave = p.n1 >> p.lg_rows;
  const int tile_len = p.rows << p.lg_n2;  // per polarisation
  const int SL = seq_stride<R>(p.n2);
  Cx<R>* const bufA = buf;
  Cx<R>* const bufB = buf + p.buf_elems;
  Cx<R>* cur = bufA;
  // the length-n2 twiddles live behind the tile buffers and the n1 ones
  // (staged here unless the caller staged both for the whole kernel)
  Cx<R>* const tws = buf + 2 * p.buf_elems + p.n1;
  if (!staged) {
    for (int i = threadIdx.x; i < N2; i += kThreads) tws[i] = ldg(p.tw2 + i);
    __syncthreads();
  }
  // element e of the tile: pol, row r, column c -> sequence pol*rows + r
  auto at = [&](int e) {
    return cur + (e >> p.lg_n2) * SL + spad<R>(e & (p.n2 - 1));
  };
  for (int t = blockIdx.x; t < p.batch * per_wave; t += gridDim.x) {
    const int b = t / per_wave;
    const int64_t r0 = (int64_t)(t % per_wave) << p.lg_rows;
    Cx<R>* base = p.data + (int64_t)b * 2 * p.n + (r0 << p.lg_n2);
    cur = bufA;
    for (int e = threadIdx.x + *(volatile int*)&s_zero; e < 2 * tile_len; e += kThreads) {
      const int pol = e >= tile_len, i = e - pol * tile_len;
      *at(e) = base[pol * p.n + i];
    }
    __syncthreads();
    if (fwd) cur = cta_fft_l<R, false, N2>(cur, cur == bufA ? bufB : bufA, 2 * p.rows, tws, &s_zero);
    if (ha || hb) {
      const int64_t h0 = r0 << p.lg_n2;
      for (int e = threadIdx.x + *(volatile int*)&s_zero; e < 2 * tile_len; e += kThreads) {
        const int pol = e >= tile_len, i = e - pol * tile_len;
        Cx<R> v = *at(e);
        if (ha) v = cmul(v, ldg(ha + h0 + i));
        if (hb) v = cmul(v, ldg(hb + h0 + i));
        *at(e) = v;
      }
      __syncthreads();
    }
    if (inv) cur = cta_fft_l<R, true, N2>(cur, cur == bufA ? bufB : bufA, 2 * p.rows, tws, &s_zero);
    for (int e = threadIdx.x + *(volatile int*)&s_zero; e < 2 * tile_len; e += kThreads) {
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
template <typename R, int N1>
__device__ __noinline__ void col_phase(const Params<R>& p, Cx<R>* buf, bool inv_in, int mid, R nl,
                          const Cx<R>* noise, bool pre_div, bool fwd_out,
                          bool staged = false) {
  __shared__ int s_zero;
  if (threadIdx.x == 0) s_zero = 0;
  __syncthreads();
  const int per_wave = p.n2 >> p.lg_cols;
  const int seq = p.n1;                  // sequence length
  const int tile_len = p.cols * seq;     // per polarisation
  const int SL = seq_stride<R>(seq);
  const R inv_n = (R)1 / (R)p.n;         // exact: n is a power of two
  Cx<R>* const bufA = buf;
  Cx<R>* const bufB = buf + p.buf_elems;
  Cx<R>* const tws = buf + 2 * p.buf_elems;  // length-n1 twiddles
  if (!staged) {
    for (int i = threadIdx.x; i < N1; i += kThreads) tws[i] = ldg(p.tw1 + i);
    __syncthreads();
  }
  for (int t = blockIdx.x; t < p.batch * per_wave; t += gridDim.x) {
    const int b = t / per_wave;
    const int c0 = (t % per_wave) << p.lg_cols;
    Cx<R>* cur = bufA;
    Cx<R>* base = p.data + (int64_t)b * 2 * p.n + c0;
    // element e: pol, row k1, column c (fastest) -> sequence pol*cols + c
    for (int e = threadIdx.x + *(volatile int*)&s_zero; e < 2 * tile_len; e += kThreads) {
      const int pol = e >= tile_len, i = e - pol * tile_len;
      const int k1 = i >> p.lg_cols, c = i & (p.cols - 1);
      Cx<R> v = base[pol * p.n + ((int64_t)k1 << p.lg_n2) + c];
      if (inv_in) v = cmulc(v, tw_n(p, k1, c0 + c));
      cur[(pol * p.cols + c) * SL + spad<R>(k1)] = v;
    }
    __syncthreads();
    if (inv_in) cur = cta_fft_l<R, true, N1>(cur, bufB, 2 * p.cols, tws, &s_zero);
    for (int e = threadIdx.x + *(volatile int*)&s_zero; e < tile_len; e += kThreads) {
      const int c = e / seq, j1 = e & (seq - 1);
      Cx<R>* px = cur + c * SL + spad<R>(j1);
      Cx<R>* py = cur + (p.cols + c) * SL + spad<R>(j1);
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
    if (fwd_out) cur = cta_fft_l<R, false, N1>(cur, cur == bufA ? bufB : bufA, 2 * p.cols, tws, &s_zero);
    for (int e = threadIdx.x + *(volatile int*)&s_zero; e < 2 * tile_len; e += kThreads) {
      const int pol = e >= tile_len, i = e - pol * tile_len;
      const int k1 = i >> p.lg_cols, c = i & (p.cols - 1);
      Cx<R> v = cur[(pol * p.cols + c) * SL + spad<R>(k1)];
      if (fwd_out) v = cmul(v, tw_n(p, k1, c0 + c));
      base[pol * p.n + ((int64_t)k1 << p.lg_n2) + c] = v;
    }
    __syncthreads();
  }
}


// ---------------------------------------------------------------- host side

struct Geo {
  int n1, n2, rows, cols;
  int buf_elems;  // elements per tile buffer (two buffers: Stockham ping-pong)
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
  g.buf_elems = std::max(2 * g.rows * stride(g.n2), 2 * g.cols * stride(g.n1));
  // two tile buffers (Stockham ping-pong) + the staged length-n1 and
  // length-n2 twiddles
  g.smem = esz * (2 * (size_t)g.buf_elems + (size_t)g.n1 + (size_t)g.n2);
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


// Stream-ordered frees of device buffers on scope exit (error paths too).
struct StreamFrees {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit StreamFrees(cudaStream_t s) : st(s) {}
  void add(void* p) {
    if (p) ptrs.push_back(p);
  }
  ~StreamFrees() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// Device twiddle tables of one four-step geometry. build() uploads them on
// `st` and fills the transform fields of p; the host staging vectors live
// here until release(), which the caller issues after synchronising.
template <typename R>
struct Fft4Tables {
  std::vector<R> t1, t2;
  void *dn = nullptr, *d1 = nullptr, *d2 = nullptr;

  cudaError_t build(int64_t n, const Geo& g, cudaStream_t st, Params<R>* p) {
    t1 = to_r<R>(unit_ld(g.n1, g.n1, 1));
    t2 = to_r<R>(unit_ld(g.n2, g.n2, 1));
    cudaError_t e;
    if ((e = cudaMallocAsync(&dn, n * sizeof(Cx<R>), st)) != cudaSuccess ||
        (e = upload(t1, &d1, st)) != cudaSuccess || (e = upload(t2, &d2, st)) != cudaSuccess)
      return e;
    fill_twn<R><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(reinterpret_cast<Cx<R>*>(dn), n,
                                                            g.n2, __builtin_ctz(g.n2));
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    p->n = n;
    p->n1 = g.n1;
    p->n2 = g.n2;
    p->rows = g.rows;
    p->cols = g.cols;
    p->lg_n2 = __builtin_ctz(g.n2);
    p->lg_rows = __builtin_ctz(g.rows);
    p->lg_cols = __builtin_ctz(g.cols);
    p->buf_elems = g.buf_elems;
    p->twn = reinterpret_cast<const Cx<R>*>(dn);
    p->tw1 = reinterpret_cast<const Cx<R>*>(d1);
    p->tw2 = reinterpret_cast<const Cx<R>*>(d2);
    return cudaSuccess;
  }
  void release(cudaStream_t st) {
    for (void* ptr : {dn, d1, d2})
      if (ptr) cudaFreeAsync(ptr, st);
    dn = d1 = d2 = nullptr;
  }
};

// Compile-time four-step split of n = 2^LG (same rule as geometry()).
template <int LG>
struct Split {
  static constexpr int N2 = 1 << ((LG + 1) / 2);
  static constexpr int N1 = 1 << (LG - (LG + 1) / 2);
};

// Kernel pointer for LG = 1..kMaxLog2N: F<LG>::get() per length.
template <template <int> class F, int LG = 1>
inline auto dispatch_lg(int lg) -> decltype(F<1>::get()) {
  if constexpr (LG > kMaxLog2N) {
    return nullptr;
  } else {
    if (lg == LG) return F<LG>::get();
    return dispatch_lg<F, LG + 1>(lg);
  }
}

}  // namespace ssfm
}  // namespace cbessfm
