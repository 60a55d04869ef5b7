// Wide-subband path of the CB-ESSFM block pipeline: N' = N/N_sb larger than
// the fused kernels hold in shared memory (c128 N' >= 8192, c64 N' >= 16384;
// the reference's own full-scale configuration, configs/fullscale.yaml:14-21,
// runs N = 16384 with N_sb in {1, 2, 4, 8}).
//
// Same algorithm and operation order as the fused block kernel
// (cbessfm_kernel.cuh), staged through a device workspace instead of one
// CTA's shared memory: every transform is a batched Stockham FFT whose
// passes (radix 16, leftover radix first) each read and write the chunk's
// rows once (L2-resident for a chunk of blocks), with the elementwise steps
// fused into the first / last pass where they touch natural-order samples:
//
//   window load ............. dbp.py:473-475          wide_window (polyphase rows)
//   outer FFT_N + demux ..... dbp.py:387-389          FFT_Q passes + wide_outer_fwd (radix P, 1/P, first phasor)
//   per step (dbp.py:394-398):
//     IFFT_Q, |x|^2+|y|^2 ... dbp.py:396, :193        passes, last one writes I
//     rfft(I) (half-length FFT of the packed reals)   passes over I viewed as complex
//     untangle, MIMO, twist . dbp.py:194-195          wide_mimo (fat-kernel formulas)
//     irfft ................. dbp.py:196               passes -> theta (packed reals)
//     rotation, FFT_Q ....... dbp.py:208, :398        passes, first one rotates
//     next phasor ........... dbp.py:395 / :399       last pass multiplies
//   merge + IFFT_N .......... dbp.py:400-401          wide_outer_inv (radix P) + IFFT_Q passes
//   keep .................... dbp.py:476-477          wide_store
//
// Twiddles of every length L in {Q, Q/2} and W_N, W_P come from the plan's
// W_N table (N = P * Q) with stride N / L.
#include <cuda_runtime.h>

#include <algorithm>

#include "cbessfm_kernel.cuh"

namespace cbessfm {
namespace wide {

constexpr int kThreads = 256;

enum Hook { kNoHook = 0, kRotate = 1, kPhasor = 2, kIntensity = 3 };

template <typename R>
struct PassArgs {
  const Cx<R>* src;
  Cx<R>* dst;
  int64_t rows;      // rows of length L (kIntensity: processed in (x, y) pairs)
  int L, NS;
  const Cx<R>* twN;  // W_N^m, m < N
  int tw_stride;     // N / L
  // hooks
  const R* theta;    // kRotate: packed reals, row q = row / 2, length L
  const R* tscale;   // kRotate: per-row-pair scale (theta_scale[set][st])
  const Cx<R>* phasor;  // kPhasor: [n_tab][P][L] tables, table ph_index[step + 1]
  const int* ph_index;
  int P;
  R* inten;          // kIntensity: row pair q -> I[q][L]
  int64_t rows_per_wave;  // row pairs (blocks x P) per waveform (set lookup)
  int64_t q0;             // global index of the chunk's first row pair
  int n_sets, n_steps, step;
};

// One Stockham pass of radix RAD and sub-transform size NS on rows of
// length L: inputs j + r L/RAD twiddled by W_(RAD NS)^(r k), k = j mod NS,
// outputs (j / NS) NS RAD + k + r NS (natural order after the last pass).
template <typename R, int RAD, bool INV, int HOOK>
__global__ void __launch_bounds__(kThreads) wide_pass(const PassArgs<R> a) {
  const int LR = a.L / RAD;
  const int64_t units = (HOOK == kIntensity ? a.rows / 2 : a.rows) * LR;
  for (int64_t u = (int64_t)blockIdx.x * kThreads + threadIdx.x; u < units;
       u += (int64_t)gridDim.x * kThreads) {
    const int64_t row0 = u / LR;
    const int j = (int)(u % LR), k = j % a.NS;
    const int base = (j / a.NS) * a.NS * RAD + k;
    constexpr int NR = HOOK == kIntensity ? 2 : 1;
    Cx<R> v[NR][RAD];
#pragma unroll
    for (int h = 0; h < NR; ++h) {
      const int64_t row = HOOK == kIntensity ? 2 * row0 + h : row0;
      const Cx<R>* s = a.src + row * a.L;
#pragma unroll
      for (int r = 0; r < RAD; ++r) {
        CB_CHECK(row >= 0 && row < a.rows && j + r * LR < a.L);
        v[h][r] = s[j + r * LR];
      }
      if constexpr (HOOK == kRotate) {
        // exp(-i theta) on the natural-order inputs (dbp.py:208), the same
        // sincos and product as the fused kernel's RotationHook
        const R* th = a.theta + (row >> 1) * (int64_t)a.L;
        const int64_t q = row >> 1;
        const int set = a.n_sets > 1 ? (int)(((a.q0 + q) / a.rows_per_wave) % a.n_sets) : 0;
        const R sc = a.tscale[(int64_t)set * a.n_steps + a.step];
#pragma unroll
        for (int r = 0; r < RAD; ++r) {
          R sn, cs;
          sincos_acc<R>(th[j + r * LR] * sc, &sn, &cs);
          v[h][r] = cmul(v[h][r], mk(cs, -sn));
        }
      }
      if (a.NS > 1) {
        const int e0 = k * (a.L / (a.NS * RAD));
#pragma unroll
        for (int r = 1; r < RAD; ++r) {
          const Cx<R> w = ldg(a.twN + (int64_t)(r * e0) * a.tw_stride);
          v[h][r] = INV ? cmulc(v[h][r], w) : cmul(v[h][r], w);
        }
      }
      dft_reg<R, RAD, INV>(v[h]);
      if constexpr (HOOK == kPhasor) {
        // next dispersion phasor on the natural-order bins (dbp.py:395, :399)
        const int i = (int)((row >> 1) % a.P);
        const Cx<R>* ph =
            a.phasor + ((int64_t)a.ph_index[a.step + 1] * a.P + i) * (int64_t)a.L;
#pragma unroll
        for (int r = 0; r < RAD; ++r)
          v[h][bitrev<RAD>(r)] = cmul(v[h][bitrev<RAD>(r)], ldg(ph + base + r * a.NS));
      }
      Cx<R>* d = a.dst + row * a.L;
#pragma unroll
      for (int r = 0; r < RAD; ++r) {
        CB_CHECK(base + r * a.NS < a.L);
        d[base + r * a.NS] = v[h][bitrev<RAD>(r)];
      }
    }
    if constexpr (HOOK == kIntensity) {
      // I = |x|^2 + |y|^2 of the time samples (dbp.py:193)
      R* I = a.inten + row0 * (int64_t)a.L;
#pragma unroll
      for (int r = 0; r < RAD; ++r) {
        const Cx<R> x = v[0][bitrev<RAD>(r)], y = v[1][bitrev<RAD>(r)];
        const R ox = x.x * x.x + x.y * x.y;
        const R oy = y.x * y.x + y.y * y.y;
        I[base + r * a.NS] = ox + oy;
      }
    }
  }
}

template <typename R>
struct StepArgs {
  Params<R> prm;
  int P, Q, N;
  int64_t c0, nc;  // chunk: flattened (waveform, block) indices [c0, c0 + nc)
};

// Circular window of block b, both polarisations, split into its P
// polyphase components (dbp.py:473-475): A[c][pol][r][t2] = u[(b keep -
// half + r + P t2) mod n] -- the outer FFT_N is P FFT_Q plus a radix-P stage,
// as in the fused kernels (N = P Q need not be a power of two).
template <typename R>
__global__ void __launch_bounds__(kThreads) wide_window(const StepArgs<R> s, Cx<R>* A) {
  const Params<R>& p = s.prm;
  const int64_t total = s.nc * 2 * s.N;
  for (int64_t u = (int64_t)blockIdx.x * kThreads + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * kThreads) {
    const int64_t c = u / (2 * s.N);
    const int pol = (int)((u / s.N) & 1);
    const int rem = (int)(u % s.N);
    const int t = rem / s.Q + s.P * (rem % s.Q);  // r + P t2
    const int64_t cid = s.c0 + c, wv = cid / p.nb, b = p.b0 + cid % p.nb;
    int64_t start = (b * p.keep - p.half) % p.n;
    if (start < 0) start += p.n;
    start -= p.in_origin;
    if (start < 0) start += p.n;
    int64_t idx = start + t;
    if (idx >= p.n) idx -= p.n;
    CB_CHECK(idx >= 0 && idx < p.n);
    A[u] = p.in[wv * p.in_bstride + pol * p.in_pstride + idx];
  }
}

// Position of global FFT_N bin g in the subband layout (fftshift / reshape /
// ifftshift of dbp.py:387-389), as bin_home in the fused kernels.
__device__ __forceinline__ void wide_bin_home(int g, int P, int Q, int& i, int& m) {
  const int N = P * Q;
  int sh = g + N / 2;
  if (sh >= N) sh -= N;
  i = sh / Q;
  m = (sh % Q + Q / 2) % Q;
}

// Radix-P stage of the outer FFT_N over the polyphase spectra Y_r[k2] (rows
// [c][pol][r]), x 1/P x first phasor, scattered to the subband rows
// S[c][i][pol][m] (dbp.py:387-389): the fused kernels' step 3, same order.
template <typename R, int P>
__global__ void __launch_bounds__(kThreads) wide_outer_fwd(const StepArgs<R> s, const Cx<R>* Y,
                                                           Cx<R>* S) {
  const Params<R>& p = s.prm;
  const int Q = s.Q, N = s.N;
  const int64_t total = s.nc * 2 * Q;
  const R invP = (R)1 / (R)P;
  const Cx<R>* ph0 = p.phasor + (int64_t)p.ph_index[0] * N;
  Cx<R> wP[P];
#pragma unroll
  for (int m = 0; m < P; ++m) wP[m] = ldg(p.twN + (int64_t)m * Q);
  for (int64_t u = (int64_t)blockIdx.x * kThreads + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * kThreads) {
    const int k2 = (int)(u % Q);
    const int64_t cp = u / Q;  // c * 2 + pol
    const int64_t c = cp >> 1;
    const int pol = (int)(cp & 1);
    Cx<R> bv[P];
#pragma unroll
    for (int r = 0; r < P; ++r) {
      Cx<R> v = Y[(cp * P + r) * (int64_t)Q + k2];
      if (r) v = cmul(v, ldg(p.twN + (int64_t)r * k2));
      bv[r] = v;
    }
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
      Cx<R> sm = bv[0];
#pragma unroll
      for (int r = 1; r < P; ++r) sm = sm + cmul(bv[r], wP[(r * k1) % P]);
      int i, m;
      wide_bin_home(Q * k1 + k2, P, Q, i, m);
      CB_CHECK(i >= 0 && i < P && m >= 0 && m < Q);
      const Cx<R> w = ldg(ph0 + (int64_t)i * Q + m);
      S[((c * P + i) * 2 + pol) * (int64_t)Q + m] = P > 1 ? cmul(scale(sm, invP), w) : cmul(sm, w);
    }
  }
}

// Merge (dbp.py:399-401): gather the P bins Q k1 + k2 from their subband
// rows, inverse radix-P stage and W_N^-(n1 k2), polyphase row n1 of the
// outer IFFT_N (the merge's x N_sb and the outer 1/N are in the final
// phasor's 1/Q): the fused kernels' step 5, same order.
template <typename R, int P>
__global__ void __launch_bounds__(kThreads) wide_outer_inv(const StepArgs<R> s, const Cx<R>* S,
                                                           Cx<R>* Y) {
  const Params<R>& p = s.prm;
  const int Q = s.Q;
  const int64_t total = s.nc * 2 * Q;
  Cx<R> wP[P];
#pragma unroll
  for (int m = 0; m < P; ++m) wP[m] = ldg(p.twN + (int64_t)m * Q);
  for (int64_t u = (int64_t)blockIdx.x * kThreads + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * kThreads) {
    const int k2 = (int)(u % Q);
    const int64_t cp = u / Q;
    const int64_t c = cp >> 1;
    const int pol = (int)(cp & 1);
    Cx<R> xv[P];
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
      int i, m;
      wide_bin_home(Q * k1 + k2, P, Q, i, m);
      xv[k1] = S[((c * P + i) * 2 + pol) * (int64_t)Q + m];
    }
#pragma unroll
    for (int n1 = 0; n1 < P; ++n1) {
      Cx<R> sm = xv[0];
#pragma unroll
      for (int k1 = 1; k1 < P; ++k1) sm = sm + cmulc(xv[k1], wP[(n1 * k1) % P]);
      if (n1) sm = cmulc(sm, ldg(p.twN + (int64_t)n1 * k2));
      Y[(cp * P + n1) * (int64_t)Q + k2] = sm;
    }
  }
}

// Keep proc[half : half + span] of every block (dbp.py:476-477); sample t
// of the block is polyphase row t mod P, position t / P.
template <typename R>
__global__ void __launch_bounds__(kThreads) wide_store(const StepArgs<R> s, const Cx<R>* Y) {
  const Params<R>& p = s.prm;
  const int64_t total = s.nc * 2 * p.keep;
  for (int64_t u = (int64_t)blockIdx.x * kThreads + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * kThreads) {
    const int64_t c = u / (2 * p.keep);
    const int pol = (int)((u / p.keep) & 1);
    const int64_t t = p.half + u % p.keep;
    const int64_t cid = s.c0 + c, wv = cid / p.nb, b = p.b0 + cid % p.nb;
    const int64_t span = min(p.keep, p.n - b * p.keep);
    if (t >= p.half + span) continue;
    const int64_t obase = b * p.keep - p.half - p.out_origin;
    CB_CHECK(obase + t >= 0 && (p.out_origin != 0 || obase + t < p.n));
    const int n1 = (int)(t % s.P);
    const int64_t t2 = t / s.P;
    p.out[wv * p.out_bstride + pol * p.out_pstride + obase + t] =
        Y[((c * 2 + pol) * s.P + n1) * (int64_t)s.Q + t2];
  }
}

// r2c untangle of every subband's half-length spectrum, MIMO (dbp.py:195)
// and c2r pre-twist for one bin pair (k, H - k) of one block: the
// one-block-per-CTA kernel's fused phase, same operations in the same order.
template <typename R, int P>
__global__ void __launch_bounds__(kThreads) wide_mimo(const StepArgs<R> s, const Cx<R>* Z,
                                                      Cx<R>* T) {
  const Params<R>& p = s.prm;
  const int H = s.Q / 2;
  const int64_t pairs = (int64_t)(H / 2 + 1);
  const int64_t total = s.nc * pairs;
  for (int64_t u = (int64_t)blockIdx.x * kThreads + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * kThreads) {
    const int64_t c = u / pairs;
    const int kp = (int)(u % pairs), kq = H - kp;
    const int64_t wv = (s.c0 + c) / p.nb;
    const int64_t cset = p.n_sets > 1 ? wv % p.n_sets : 0;
    const Cx<R>* mimo = p.mimo + cset * (int64_t)P * (H + 1);
    const Cx<R> wk = ldg(p.twN + (int64_t)kp * s.P);  // W_Q^kp
    Cx<R> ia[P], ib[P];
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const Cx<R>* Il = Z + (c * P + l) * (int64_t)H;
      if (kp == 0) {
        const Cx<R> z = Il[0];
        ia[l] = mk(z.x + z.y, (R)0);
        ib[l] = mk(z.x - z.y, (R)0);
      } else {
        const Cx<R> a = Il[kp];
        const Cx<R> bq = conj(Il[kq]);
        const Cx<R> e = scale(a + bq, (R)0.5);
        const Cx<R> dd = a - bq;
        const Cx<R> o = mk(dd.y * (R)0.5, -dd.x * (R)0.5);
        const Cx<R> wo = cmul(o, wk);
        ia[l] = e + wo;
        ib[l] = kp == kq ? ia[l] : conj(e - wo);
      }
    }
    Cx<R> ta[P], tb[P];
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int k = half ? kq : kp;
      const Cx<R>* iv = half ? ib : ia;
      Cx<R> sv[P];
#pragma unroll
      for (int l = 0; l < P; ++l) sv[l] = ldg(mimo + (int64_t)l * (H + 1) + k);
#pragma unroll
      for (int i = 0; i < P; ++i) {
        Cx<R> acc = mk((R)0, (R)0);
#pragma unroll
        for (int l = 0; l < P; ++l)
          acc = l >= i ? cmac(acc, sv[l - i], iv[l]) : cmacc(acc, sv[i - l], iv[l]);
        (half ? tb : ta)[i] = acc;
      }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
      Cx<R>* Ti = T + (c * P + i) * (int64_t)H;
      if (kp == 0) {
        Ti[0] = mk(ta[i].x + tb[i].x, ta[i].x - tb[i].x);
      } else {
        const Cx<R> a = ta[i];
        const Cx<R> cc = conj(tb[i]);
        const Cx<R> s2 = a + cc;
        const Cx<R> dd = cmulc(a - cc, wk);
        Ti[kp] = mk(s2.x - dd.y, s2.y + dd.x);
        if (kp != kq) {
          const Cx<R> a2 = conj(cc);
          const Cx<R> c2 = conj(a);
          const Cx<R> s3 = a2 + c2;
          const Cx<R> w2 = mk(-wk.x, wk.y);
          const Cx<R> d2 = cmulc(a2 - c2, w2);
          Ti[kq] = mk(s3.x - d2.y, s3.y + d2.x);
        }
      }
    }
  }
}

inline int grid_for(int64_t units) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((units + kThreads - 1) / kThreads, 148 * 16));
}

// Batched FFT of `rows` rows of length L (src -> result in *cur, ping-pong
// with *alt); the first pass may rotate, the last may apply a phasor or
// write the intensity.
template <typename R, bool INV>
cudaError_t fft_rows(PassArgs<R> a, Cx<R>** cur, Cx<R>** alt, int first_hook, int last_hook,
                     cudaStream_t st) {
  int lg = 0;
  while ((1 << lg) < a.L) ++lg;
  const int lead = lg % 4;  // leftover radix first, then radix 16
  int ns = 1;
  bool first = true;
  while (ns < a.L) {
    const int rad = (first && lead) ? (1 << lead) : 16;
    const bool last = ns * rad == a.L;
    const int hook = (first ? first_hook : kNoHook) | (last ? last_hook : kNoHook);
    a.src = *cur;
    a.dst = *alt;
    a.NS = ns;
    const int64_t units = (hook == kIntensity ? a.rows / 2 : a.rows) * (a.L / rad);
    const int grid = grid_for(units);
#define CB_WPASS(RD, HK) wide_pass<R, RD, INV, HK><<<grid, kThreads, 0, st>>>(a)
#define CB_WHOOK(RD)                                         \
  switch (hook) {                                            \
    case kRotate: CB_WPASS(RD, kRotate); break;              \
    case kPhasor: CB_WPASS(RD, kPhasor); break;              \
    case kIntensity: CB_WPASS(RD, kIntensity); break;        \
    default: CB_WPASS(RD, kNoHook); break;                   \
  }
    switch (rad) {
      case 2: CB_WHOOK(2) break;
      case 4: CB_WHOOK(4) break;
      case 8: CB_WHOOK(8) break;
      default: CB_WHOOK(16) break;
    }
#undef CB_WHOOK
#undef CB_WPASS
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    std::swap(*cur, *alt);
    ns *= rad;
    first = false;
  }
  return cudaSuccess;
}

template <typename R, int P>
cudaError_t mimo_launch(const StepArgs<R>& s, const Cx<R>* Z, Cx<R>* T, cudaStream_t st) {
  const int64_t units = s.nc * (s.Q / 4 + 1);
  wide_mimo<R, P><<<grid_for(units), kThreads, 0, st>>>(s, Z, T);
  return cudaGetLastError();
}

template <typename R>
cudaError_t mimo_dispatch(const StepArgs<R>& s, const Cx<R>* Z, Cx<R>* T, cudaStream_t st) {
  switch (s.P) {
    case 1: return mimo_launch<R, 1>(s, Z, T, st);
    case 2: return mimo_launch<R, 2>(s, Z, T, st);
    case 3: return mimo_launch<R, 3>(s, Z, T, st);
    case 4: return mimo_launch<R, 4>(s, Z, T, st);
    case 5: return mimo_launch<R, 5>(s, Z, T, st);
    case 6: return mimo_launch<R, 6>(s, Z, T, st);
    case 7: return mimo_launch<R, 7>(s, Z, T, st);
    case 8: return mimo_launch<R, 8>(s, Z, T, st);
    case 9: return mimo_launch<R, 9>(s, Z, T, st);
    default: return cudaErrorInvalidValue;
  }
}

template <typename R, int P>
cudaError_t outer_launch(const StepArgs<R>& s, const Cx<R>* a, Cx<R>* b, bool fwd, cudaStream_t st) {
  const int64_t units = s.nc * 2 * s.Q;
  if (fwd)
    wide_outer_fwd<R, P><<<grid_for(units), kThreads, 0, st>>>(s, a, b);
  else
    wide_outer_inv<R, P><<<grid_for(units), kThreads, 0, st>>>(s, a, b);
  return cudaGetLastError();
}

template <typename R>
cudaError_t outer_dispatch(const StepArgs<R>& s, const Cx<R>* a, Cx<R>* b, bool fwd,
                           cudaStream_t st) {
  switch (s.P) {
    case 1: return outer_launch<R, 1>(s, a, b, fwd, st);
    case 2: return outer_launch<R, 2>(s, a, b, fwd, st);
    case 3: return outer_launch<R, 3>(s, a, b, fwd, st);
    case 4: return outer_launch<R, 4>(s, a, b, fwd, st);
    case 5: return outer_launch<R, 5>(s, a, b, fwd, st);
    case 6: return outer_launch<R, 6>(s, a, b, fwd, st);
    case 7: return outer_launch<R, 7>(s, a, b, fwd, st);
    case 8: return outer_launch<R, 8>(s, a, b, fwd, st);
    case 9: return outer_launch<R, 9>(s, a, b, fwd, st);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------------
// Per-row kernels: one CTA holds one length-L row in shared memory (padded,
// one slot per 16) and runs every pass of the transform in place (load,
// barrier, store, barrier), so a step reads and writes the field once
// instead of once per pass. Rows that fit: L <= 8192 at c128, 16384 at c64.

template <typename R>
constexpr int smem_max_q() {
  return sizeof(R) == 8 ? 8192 : 16384;
}
template <int L>
constexpr int row_threads() {
  return L / 16 < 512 ? L / 16 : 512;
}
template <int L>
constexpr int row_padded() {
  return L + L / 16 + 1;
}

template <typename R, int L, int RAD, bool INV>
__device__ __forceinline__ void smem_pass(Cx<R>* F, int NS, const Cx<R>* __restrict__ twN,
                                          int tws) {
  constexpr int NT = row_threads<L>();
  constexpr int NB = L / RAD;
  static_assert(NB % NT == 0, "butterflies must tile the CTA");
  constexpr int PER = NB / NT;
  const int tstep = L / (NS * RAD);
  Cx<R> v[PER][RAD];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int j = (int)threadIdx.x + p * NT, k = j % NS;
#pragma unroll
    for (int r = 0; r < RAD; ++r) v[p][r] = F[pad(j + r * NB)];
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < RAD; ++r) {
        const Cx<R> w = ldg(twN + (int64_t)(r * k * tstep) * tws);
        v[p][r] = INV ? cmulc(v[p][r], w) : cmul(v[p][r], w);
      }
    }
    dft_reg<R, RAD, INV>(v[p]);
  }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int j = (int)threadIdx.x + p * NT, k = j % NS;
    const int d0 = (j / NS) * NS * RAD + k;
#pragma unroll
    for (int r = 0; r < RAD; ++r) F[pad(d0 + r * NS)] = v[p][bitrev<RAD>(r)];
  }
  __syncthreads();
}

// Unnormalised in-place FFT of the row in F (natural order in and out).
template <typename R, int L, bool INV>
__device__ __forceinline__ void row_fft(Cx<R>* F, const Cx<R>* twN, int tws) {
  constexpr int LG = __builtin_ctz(L), LEAD = LG % 4;
  int ns = 1;
  if constexpr (LEAD != 0) {
    smem_pass<R, L, (1 << LEAD), INV>(F, 1, twN, tws);
    ns = 1 << LEAD;
  }
  for (; ns < L; ns *= 16) smem_pass<R, L, 16, INV>(F, ns, twN, tws);
}

enum FieldMode { kFirstIfft = 0, kStep = 1, kLastStep = 2 };

// One field row (c, i, pol) per CTA: [rotation, FFT, next phasor,] [IFFT,
// intensity] -- dbp.py:208, :398, :395 / :399, :396, :193.
template <typename R, int L>
__global__ void __launch_bounds__(row_threads<L>()) wide_row_field(const StepArgs<R> s, Cx<R>* rows,
                                                                  const R* theta, R* Ix, R* Iy,
                                                                  int step, int mode) {
  constexpr int NT = row_threads<L>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<R>* F = reinterpret_cast<Cx<R>*>(smem_raw);
  const Params<R>& p = s.prm;
  const int64_t row = blockIdx.x;  // (c * P + i) * 2 + pol
  const int64_t q = row >> 1;      // (c, i)
  const int pol = (int)(row & 1), i = (int)(q % s.P);
  Cx<R>* g = rows + row * L;
  if (mode == kFirstIfft) {
    for (int t = threadIdx.x; t < L; t += NT) F[pad(t)] = g[t];
  } else {
    // rotation exp(-i theta) of the natural-order time samples
    const int64_t wv = (s.c0 + q / s.P) / p.nb;
    const int set = p.n_sets > 1 ? (int)(wv % p.n_sets) : 0;
    const R sc = p.theta_scale[(int64_t)set * p.n_steps + step];
    const R* th = theta + q * L;
    for (int t = threadIdx.x; t < L; t += NT) {
      R sn, cs;
      sincos_acc<R>(th[t] * sc, &sn, &cs);
      F[pad(t)] = cmul(g[t], mk(cs, -sn));
    }
  }
  __syncthreads();
  if (mode != kFirstIfft) {
    row_fft<R, L, false>(F, p.twN, s.P);
    const Cx<R>* ph = p.phasor + ((int64_t)p.ph_index[step + 1] * s.P + i) * (int64_t)L;
    for (int t = threadIdx.x; t < L; t += NT) F[pad(t)] = cmul(F[pad(t)], ldg(ph + t));
    __syncthreads();
  }
  if (mode == kLastStep) {
    for (int t = threadIdx.x; t < L; t += NT) g[t] = F[pad(t)];
    return;
  }
  row_fft<R, L, true>(F, p.twN, s.P);
  R* I = (pol ? Iy : Ix) + q * L;
  for (int t = threadIdx.x; t < L; t += NT) {
    const Cx<R> v = F[pad(t)];
    g[t] = v;
    I[t] = v.x * v.x + v.y * v.y;
  }
}

// Half-length FFT of the packed intensity z[t] = I[2t] + i I[2t+1],
// I = |x|^2 + |y|^2 (x first, as the reference sums), one (c, i) per CTA.
template <typename R, int L>
__global__ void __launch_bounds__(row_threads<L>()) wide_row_rfft(const StepArgs<R> s, const R* Ix,
                                                                 const R* Iy, Cx<R>* Z) {
  constexpr int NT = row_threads<L>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<R>* F = reinterpret_cast<Cx<R>*>(smem_raw);
  const int64_t q = blockIdx.x;
  const R* ix = Ix + q * 2 * L;
  const R* iy = Iy + q * 2 * L;
  for (int t = threadIdx.x; t < L; t += NT)
    F[pad(t)] = mk(ix[2 * t] + iy[2 * t], ix[2 * t + 1] + iy[2 * t + 1]);
  __syncthreads();
  row_fft<R, L, false>(F, s.prm.twN, 2 * s.P);
  Cx<R>* z = Z + q * L;
  for (int t = threadIdx.x; t < L; t += NT) z[t] = F[pad(t)];
}

// Inverse half-length FFT of the twisted theta_hat, in place (theta packed
// as reals, dbp.py:196).
template <typename R, int L>
__global__ void __launch_bounds__(row_threads<L>()) wide_row_irfft(const StepArgs<R> s, Cx<R>* T) {
  constexpr int NT = row_threads<L>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Cx<R>* F = reinterpret_cast<Cx<R>*>(smem_raw);
  Cx<R>* t_row = T + (int64_t)blockIdx.x * L;
  for (int t = threadIdx.x; t < L; t += NT) F[pad(t)] = t_row[t];
  __syncthreads();
  row_fft<R, L, true>(F, s.prm.twN, 2 * s.P);
  for (int t = threadIdx.x; t < L; t += NT) t_row[t] = F[pad(t)];
}

// The steps of one chunk with per-row kernels at subband length Q.
template <typename R, int Q>
cudaError_t smem_steps(const StepArgs<R>& s, Cx<R>* cur, R* Ix, R* Iy, Cx<R>* hA, Cx<R>* hB,
                       cudaStream_t st) {
  constexpr int H = Q / 2;
  const Params<R>& prm = s.prm;
  const int64_t frows = s.nc * s.P * 2, hrows = s.nc * s.P;
  const size_t fsm = sizeof(Cx<R>) * row_padded<Q>(), hsm = sizeof(Cx<R>) * row_padded<H>();
  cudaError_t e;
  auto kf = wide_row_field<R, Q>;
  auto kh = wide_row_rfft<R, H>;
  auto ki = wide_row_irfft<R, H>;
  if ((e = cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(kh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(ki, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm)) != cudaSuccess)
    return e;
  if (prm.n_steps > 0)
    kf<<<(unsigned)frows, row_threads<Q>(), fsm, st>>>(s, cur, nullptr, Ix, Iy, 0, kFirstIfft);
  for (int stp = 0; stp < prm.n_steps; ++stp) {
    kh<<<(unsigned)hrows, row_threads<H>(), hsm, st>>>(s, Ix, Iy, hA);
    if ((e = mimo_dispatch<R>(s, hA, hB, st)) != cudaSuccess) return e;
    ki<<<(unsigned)hrows, row_threads<H>(), hsm, st>>>(s, hB);
    kf<<<(unsigned)frows, row_threads<Q>(), fsm, st>>>(s, cur, reinterpret_cast<const R*>(hB), Ix,
                                                       Iy, stp,
                                                       stp + 1 < prm.n_steps ? kStep : kLastStep);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

// Bytes of device workspace per (waveform, block) of a chunk.
template <typename R>
size_t bytes_per_block(int N) {
  // two ping-pong field buffers [2][N], two half-length buffers (N reals,
  // i.e. N/2 complex, each)
  return sizeof(Cx<R>) * (size_t)(2 * 2 * N + 2 * (N / 2));
}

// Workspace a launch of nclusters (waveform, block) pairs uses: chunks of
// at most ~256 MB.
template <typename R>
size_t workspace_bytes(int N, int64_t nclusters) {
  const size_t per = bytes_per_block<R>(N);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nclusters, (int64_t)((256u << 20) / per)));
  return per * (size_t)chunk;
}

template <typename R>
cudaError_t run(const Params<R>& prm, int P, int Q, int64_t nclusters, cudaStream_t st, void* ws,
                size_t ws_bytes) {
  const int N = P * Q, H = Q / 2;
  const size_t per = bytes_per_block<R>(N);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nclusters, (int64_t)(ws_bytes / per)));
  cudaError_t e = cudaSuccess;
  Cx<R>* bufA = reinterpret_cast<Cx<R>*>(ws);
  Cx<R>* bufB = bufA + (size_t)chunk * 2 * N;
  Cx<R>* hA = bufB + (size_t)chunk * 2 * N;
  Cx<R>* hB = hA + (size_t)chunk * (N / 2);
  for (int64_t c0 = 0; c0 < nclusters && e == cudaSuccess; c0 += chunk) {
    StepArgs<R> s{prm, P, Q, N, c0, std::min<int64_t>(chunk, nclusters - c0)};
    const int64_t units = s.nc * 2 * N;
    PassArgs<R> pa{};
    pa.twN = prm.twN;
    pa.P = P;
    pa.n_sets = prm.n_sets;
    pa.n_steps = prm.n_steps;
    pa.rows_per_wave = prm.nb * P;
    pa.q0 = c0 * P;
    // ---- window (polyphase rows), FFT_Q of each, radix-P stage + demux
    //      (+ 1/P, first phasor)
    wide_window<R><<<grid_for(units), kThreads, 0, st>>>(s, bufA);
    Cx<R>* cur = bufA;
    Cx<R>* alt = bufB;
    pa.rows = s.nc * 2 * P;
    pa.L = Q;
    pa.tw_stride = P;
    if ((e = fft_rows<R, false>(pa, &cur, &alt, kNoHook, kNoHook, st)) != cudaSuccess) break;
    if ((e = outer_dispatch<R>(s, cur, alt, true, st)) != cudaSuccess) break;
    std::swap(cur, alt);  // cur: subband rows [c][i][pol][Q] (spectra)
    // ---- steps: per-row kernels where a row fits one CTA's shared memory
    if (Q == smem_max_q<R>()) {
      // intensity of x and y in the idle second field buffer
      R* Ix = reinterpret_cast<R*>(alt);
      R* Iy = Ix + (size_t)s.nc * N;
      // (the wide path starts above the fused kernels' N': 4096 c128, 8192 c64)
      e = smem_steps<R, smem_max_q<R>()>(s, cur, Ix, Iy, hA, hB, st);
    } else {
      for (int stp = 0; stp < prm.n_steps; ++stp) {
        pa.rows = s.nc * P * 2;
        pa.L = Q;
        pa.tw_stride = P;
        pa.inten = reinterpret_cast<R*>(hA);
        if ((e = fft_rows<R, true>(pa, &cur, &alt, kNoHook, kIntensity, st)) != cudaSuccess) break;
        // rfft of the intensity: half-length FFT of the packed reals
        PassArgs<R> ph = pa;
        ph.rows = s.nc * P;
        ph.L = H;
        ph.tw_stride = 2 * P;
        Cx<R>* hc = hA;
        Cx<R>* ha = hB;
        if ((e = fft_rows<R, false>(ph, &hc, &ha, kNoHook, kNoHook, st)) != cudaSuccess) break;
        if ((e = mimo_dispatch<R>(s, hc, ha, st)) != cudaSuccess) break;
        std::swap(hc, ha);  // hc: twisted theta_hat
        if ((e = fft_rows<R, true>(ph, &hc, &ha, kNoHook, kNoHook, st)) != cudaSuccess) break;
        // rotation fused into the first pass of the forward FFT, the next
        // phasor into its last
        pa.theta = reinterpret_cast<const R*>(hc);
        pa.tscale = prm.theta_scale;
        pa.step = stp;
        pa.phasor = prm.phasor;
        pa.ph_index = prm.ph_index;
        if ((e = fft_rows<R, false>(pa, &cur, &alt, kRotate, kPhasor, st)) != cudaSuccess) break;
      }
    }
    if (e != cudaSuccess) break;
    // ---- merge + inverse radix-P stage, IFFT_Q of each polyphase row, keep
    if ((e = outer_dispatch<R>(s, cur, alt, false, st)) != cudaSuccess) break;
    std::swap(cur, alt);
    pa.rows = s.nc * 2 * P;
    pa.L = Q;
    pa.tw_stride = P;
    if ((e = fft_rows<R, true>(pa, &cur, &alt, kNoHook, kNoHook, st)) != cudaSuccess) break;
    wide_store<R><<<grid_for(s.nc * 2 * prm.keep), kThreads, 0, st>>>(s, cur);
    e = cudaGetLastError();
  }
  return e;
}

}  // namespace wide

size_t wide_workspace_bytes(int real_bytes, int N, int64_t nclusters) {
  return real_bytes == 4 ? wide::workspace_bytes<float>(N, nclusters)
                         : wide::workspace_bytes<double>(N, nclusters);
}
cudaError_t wide_run_float(const Params<float>& prm, int P, int Q, int64_t nclusters,
                           cudaStream_t st, void* ws, size_t ws_bytes) {
  return wide::run<float>(prm, P, Q, nclusters, st, ws, ws_bytes);
}
cudaError_t wide_run_double(const Params<double>& prm, int P, int Q, int64_t nclusters,
                            cudaStream_t st, void* ws, size_t ws_bytes) {
  return wide::run<double>(prm, P, Q, nclusters, st, ws, ws_bytes);
}

}  // namespace cbessfm
