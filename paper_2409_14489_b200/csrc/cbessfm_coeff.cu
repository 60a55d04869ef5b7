// GPU coefficient builder: the anti-diagonal sums and the
// tap transform of the reference's _coeff_grid_eval (kernel.py:274-303),
// with the step kernel of kernel.py:139-250 evaluated on the fly.
//
//   S[off] = sum_i Kh[i, i+off] w_i w_(i+off),  Kh = (K + K^H) / 2
//   c[m]   = sum_off exp(2 pi j m (-off) / (n-1)) S[off],   |m| <= memory
//
// One CTA per anti-diagonal (2n-1 of them) evaluates its kernel entries
// K(mu_p, mu_q) and K(mu_q, mu_p) directly, so nothing of size n^2 is ever
// stored (the reference holds the n x n matrix and its conjugate
// transpose). Every expression follows the reference's evaluation order
// so the FP64 values agree to rounding.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/cbessfm_coeff.h"
#include "cbessfm_kernel.cuh"

namespace cbessfm {
namespace coeff {

using C = Cx<double>;
constexpr int kThreads = 256;
constexpr int kMaxSegments = 64;

struct KernelParams {
  int closed_form;
  double gamma, alpha, beat, span;
  int num_spans, n_seg;
  double seg[kMaxSegments][3];
};

__device__ __forceinline__ C cexp_(C z) {
  const double e = exp(z.x);
  double s, c;
  sincos(z.y, &s, &c);
  return mk(e * c, e * s);
}

// Smith's complex division (numpy's algorithm)
__device__ __forceinline__ C cdiv_(C a, C b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, den = b.x + b.y * r;
    return mk((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  const double r = b.x / b.y, den = b.y + b.x * r;
  return mk((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

__device__ __forceinline__ double sinc_np(double t) {  // np.sinc
  const double y = M_PI * (t == 0.0 ? 1.0e-20 : t);
  return sin(y) / y;
}

// sin(n x)/sin(x) with the removable singularities filled (kernel.py:132-138)
__device__ __forceinline__ double sin_ratio(double x, int n) {
  const double k = rint(x / M_PI);
  const double eps = __dsub_rn(x, __dmul_rn(k, M_PI));
  const long long kk = (long long)k;
  const double sign = ((kk * (long long)(n - 1)) % 2 == 0) ? 1.0 : -1.0;
  return sign * n * sinc_np(n * eps / M_PI) / sinc_np(eps / M_PI);
}

// K(mu, nu), kernel.py:148-250
__device__ C step_kernel(const KernelParams& k, double mu, double nu) {
  const double b = __dmul_rn(__dmul_rn(k.beat, nu), __dsub_rn(mu, nu));
  if (k.closed_form) {
    const double a = k.alpha / 2.0, lsp = k.span;
    const C w = mk(__dmul_rn(a, lsp), __dmul_rn(b, lsp));
    C sh;
    if (hypot(w.x, w.y) < 1e-6) {
      const C w2 = mk(w.x * w.x - w.y * w.y, 2.0 * w.x * w.y);
      sh = mk(1.0 + w2.x / 6.0, w2.y / 6.0);
    } else {
      const C s = mk(sinh(w.x) * cos(w.y), cosh(w.x) * sin(w.y));
      sh = cdiv_(s, w);
    }
    const double pre = __dmul_rn(__dmul_rn(k.gamma, exp(-a * lsp)), lsp);
    const double sr = sin_ratio(__dmul_rn(b, lsp), k.num_spans);
    return mk(pre * sh.x * sr, pre * sh.y * sr);
  }
  C total = mk(0.0, 0.0);
  for (int s = 0; s < k.n_seg; ++s) {
    const double z0 = k.seg[s][0], z1 = k.seg[s][1], g0 = k.seg[s][2];
    const double len = __dsub_rn(z1, z0);
    const C w = mk(__dmul_rn(k.alpha, len), __dmul_rn(2.0 * b, len));
    C core;
    if (hypot(w.x, w.y) < 1e-9) {
      core = mk(1.0 - w.x / 2.0, -w.y / 2.0);
    } else {
      const C e = cexp_(mk(-w.x, -w.y));
      core = cdiv_(mk(1.0 - e.x, -e.y), w);
    }
    const C ph = cexp_(mk(0.0, __dmul_rn(-2.0 * b, z0)));
    const C t = mk(__dmul_rn(__dmul_rn(g0, ph.x), len), __dmul_rn(__dmul_rn(g0, ph.y), len));
    total = total + cmul(t, core);
  }
  return mk(total.x * k.gamma, total.y * k.gamma);
}

__device__ __forceinline__ C block_sum(C v) {
  __shared__ double sx[kThreads / 32], sy[kThreads / 32];
  for (int o = 16; o; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sx[w] = v.x;
    sy[w] = v.y;
  }
  __syncthreads();
  C r = mk(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int i = 0; i < kThreads / 32; ++i) r = r + mk(sx[i], sy[i]);
  return r;
}

// S[k], off = k - (n-1): sum_i Kh[i, i+off] w_i w_(i+off) (kernel.py:289-297)
__global__ void __launch_bounds__(kThreads) diag_kernel(KernelParams kp, const double* __restrict__ mu,
                                                        const double* __restrict__ w, int64_t n,
                                                        C* __restrict__ diag) {
  const int64_t off = (int64_t)blockIdx.x - (n - 1);
  const int64_t i0 = off < 0 ? -off : 0, i1 = off < 0 ? n : n - off;
  C acc = mk(0.0, 0.0);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kThreads) {
    const int64_t p = i, q = i + off;
    const C kpq = step_kernel(kp, mu[p], mu[q]);
    const C kqp = step_kernel(kp, mu[q], mu[p]);
    const C kh = mk(0.5 * (kpq.x + kqp.x), 0.5 * (kpq.y - kqp.y));
    const double wp = w[p], wq = w[q];
    acc = acc + mk(__dmul_rn(__dmul_rn(kh.x, wp), wq), __dmul_rn(__dmul_rn(kh.y, wp), wq));
  }
  const C s = block_sum(acc);
  if (threadIdx.x == 0) diag[blockIdx.x] = s;
}

// c[m] = sum_k exp(2 pi j m (-d_k) / (n-1)) S[k], d_k = k - (n-1) (kernel.py:299-302)
__global__ void __launch_bounds__(kThreads) taps_kernel(const C* __restrict__ diag, int64_t n,
                                                        int memory, C* __restrict__ out) {
  const int64_t m = (int64_t)blockIdx.x - memory;
  const double two_pi = 2.0 * M_PI;
  C acc = mk(0.0, 0.0);
  for (int64_t k = threadIdx.x; k < 2 * n - 1; k += kThreads) {
    const int64_t o = m * (-(k - (n - 1)));
    const double ang = __ddiv_rn(__dmul_rn(two_pi, (double)o), (double)(n - 1));
    double s, c;
    sincos(ang, &s, &c);
    acc = acc + cmul(mk(c, s), diag[k]);
  }
  const C r = block_sum(acc);
  if (threadIdx.x == 0) out[blockIdx.x] = r;
}

__global__ void eval_kernel(KernelParams kp, const double* mu, const double* nu, int64_t count,
                            C* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = step_kernel(kp, mu[i], nu[i]);
}

thread_local std::string g_err;

cbessfm_status fail(cbessfm_status s, const std::string& m) {
  g_err = m;
  return s;
}

cbessfm_status to_params(const cbessfm_step_kernel* k, KernelParams* p) {
  if (!k) return fail(CBESSFM_ERR_INVALID, "null kernel description");
  if (!k->closed_form && (k->n_segments < 1 || k->n_segments > kMaxSegments || !k->segments))
    return fail(CBESSFM_ERR_INVALID, "piecewise kernel needs 1..64 segments");
  if (k->closed_form && k->num_spans < 1) return fail(CBESSFM_ERR_INVALID, "num_spans must be >= 1");
  *p = KernelParams{};
  p->closed_form = k->closed_form;
  p->gamma = k->gamma_w_km;
  p->alpha = k->alpha_np_km;
  p->beat = k->beat_scale;
  p->span = k->span_km;
  p->num_spans = k->num_spans;
  p->n_seg = k->closed_form ? 0 : k->n_segments;
  for (int s = 0; s < p->n_seg; ++s)
    for (int j = 0; j < 3; ++j) p->seg[s][j] = k->segments[3 * s + j];
  return CBESSFM_OK;
}

cbessfm_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return CBESSFM_OK;
  return fail(CBESSFM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace coeff
}  // namespace cbessfm

extern "C" {

cbessfm_status cbessfm_coeff_grid(const cbessfm_step_kernel* kernel, int64_t num_nodes,
                                  const double* mu, const double* weights, int32_t memory,
                                  double* out, int32_t device) {
  using namespace cbessfm::coeff;
  g_err.clear();
  KernelParams kp;
  if (cbessfm_status s = to_params(kernel, &kp)) return s;
  if (num_nodes < 3 || !mu || !weights || !out || memory < 0)
    return fail(CBESSFM_ERR_INVALID, "need num_nodes >= 3, grid, weights, output, memory >= 0");
  if (num_nodes > (int64_t(1) << 22)) return fail(CBESSFM_ERR_UNSUPPORTED, "num_nodes above 2^22");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_check(e, "cudaSetDevice");
  const int64_t n = num_nodes, nd = 2 * n - 1, nt = 2 * (int64_t)memory + 1;
  double *dmu = nullptr, *dw = nullptr;
  C *ddiag = nullptr, *dout = nullptr;
  cbessfm_status st = CBESSFM_OK;
  if ((st = cuda_check(cudaMalloc(&dmu, n * sizeof(double)), "alloc")) ||
      (st = cuda_check(cudaMalloc(&dw, n * sizeof(double)), "alloc")) ||
      (st = cuda_check(cudaMalloc(&ddiag, nd * sizeof(C)), "alloc")) ||
      (st = cuda_check(cudaMalloc(&dout, nt * sizeof(C)), "alloc")) ||
      (st = cuda_check(cudaMemcpy(dmu, mu, n * sizeof(double), cudaMemcpyHostToDevice), "h2d")) ||
      (st = cuda_check(cudaMemcpy(dw, weights, n * sizeof(double), cudaMemcpyHostToDevice), "h2d"))) {
  } else {
    diag_kernel<<<(unsigned)nd, kThreads>>>(kp, dmu, dw, n, ddiag);
    taps_kernel<<<(unsigned)nt, kThreads>>>(ddiag, n, memory, dout);
    if (!(st = cuda_check(cudaGetLastError(), "coefficient kernels")))
      st = cuda_check(cudaMemcpy(out, dout, nt * sizeof(C), cudaMemcpyDeviceToHost), "d2h");
  }
  cudaFree(dmu);
  cudaFree(dw);
  cudaFree(ddiag);
  cudaFree(dout);
  return st;
}

cbessfm_status cbessfm_step_kernel_eval(const cbessfm_step_kernel* kernel, int64_t count,
                                        const double* mu, const double* nu, double* out,
                                        int32_t device) {
  using namespace cbessfm::coeff;
  g_err.clear();
  KernelParams kp;
  if (cbessfm_status s = to_params(kernel, &kp)) return s;
  if (count < 0 || (count && (!mu || !nu || !out))) return fail(CBESSFM_ERR_INVALID, "bad arrays");
  if (!count) return CBESSFM_OK;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_check(e, "cudaSetDevice");
  double *dmu = nullptr, *dnu = nullptr;
  C* dout = nullptr;
  cbessfm_status st = CBESSFM_OK;
  if (!(st = cuda_check(cudaMalloc(&dmu, count * sizeof(double)), "alloc")) &&
      !(st = cuda_check(cudaMalloc(&dnu, count * sizeof(double)), "alloc")) &&
      !(st = cuda_check(cudaMalloc(&dout, count * sizeof(C)), "alloc")) &&
      !(st = cuda_check(cudaMemcpy(dmu, mu, count * sizeof(double), cudaMemcpyHostToDevice), "h2d")) &&
      !(st = cuda_check(cudaMemcpy(dnu, nu, count * sizeof(double), cudaMemcpyHostToDevice), "h2d"))) {
    eval_kernel<<<(unsigned)((count + 255) / 256), 256>>>(kp, dmu, dnu, count, dout);
    if (!(st = cuda_check(cudaGetLastError(), "kernel eval")))
      st = cuda_check(cudaMemcpy(out, dout, count * sizeof(C), cudaMemcpyDeviceToHost), "d2h");
  }
  cudaFree(dmu);
  cudaFree(dnu);
  cudaFree(dout);
  return st;
}

const char* cbessfm_coeff_last_error(void) { return cbessfm::coeff::g_err.c_str(); }

}  // extern "C"
