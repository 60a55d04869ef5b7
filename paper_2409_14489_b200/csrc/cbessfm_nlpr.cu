// Stand-alone coupled-band nonlinear phase rotation on subband waveforms:
// the public nlpr_step helper (dbp.py:211-230, formula dbp.py:185-208) on
// the GPU. Inside run_dbp the same rotation runs fused in the block kernel;
// this entry takes time-domain subband fields and a general MIMO matrix
// T[i][l][k] (a MimoTransfer need not be Toeplitz) and applies
//   theta_i = irfft(sum_l T[i,l] rfft(|x_l|^2 + |y_l|^2)) * scale,
//   (x_i, y_i) *= exp(-j theta_i).
// One cluster of P CTAs, CTA i owns subband i; spectra are exchanged over
// DSMEM. A helper, not a hot path: P is a runtime value.
#include <cooperative_groups.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/cbessfm.h"
#include "cbessfm_kernel.cuh"

namespace cbessfm {
namespace {

constexpr int kMaxSub = 16;

template <typename R, int Q>
__global__ void __launch_bounds__(Q / 8) nlpr_kernel(const Cx<R>* in, Cx<R>* out,
                                                     const Cx<R>* T, const Cx<R>* twQ,
                                                     const Cx<R>* twp, R theta_scale, int P) {
  constexpr int NT = Q / 8;
  constexpr int H = Q / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CB_POISON_SMEM(smem_raw);
  Cx<R>* IS = reinterpret_cast<Cx<R>*>(smem_raw);   // packed intensity -> I_hat
  Cx<R>* TS = IS + padded_len(H + 1);                // theta_hat -> theta
  __shared__ int s_zero;
  if (threadIdx.x == 0) s_zero = 0;
  const int i = (int)blockIdx.x;                     // subband = cluster rank
  const int tid = threadIdx.x;
  const Cx<R>* xi = in + (size_t)i * Q;
  const Cx<R>* yi = in + (size_t)(P + i) * Q;
  // intensity packed as z[t] = I[2t] + i I[2t+1]
  for (int t = tid; t < H; t += NT) {
    const Cx<R> a0 = xi[2 * t], a1 = xi[2 * t + 1], b0 = yi[2 * t], b1 = yi[2 * t + 1];
    IS[pad(t)] = mk(a0.x * a0.x + a0.y * a0.y + (b0.x * b0.x + b0.y * b0.y),
                    a1.x * a1.x + a1.y * a1.y + (b1.x * b1.x + b1.y * b1.y));
  }
  __syncthreads();
  fft1<R, Q, H, NT, false>(IS, twp, &s_zero);
  // r2c untangle in place (same algebra as the block kernel)
  for (int k = tid; k <= H / 2; k += NT) {
    if (k == 0) {
      const Cx<R> z = IS[pad(0)];
      IS[pad(0)] = mk(z.x + z.y, (R)0);
      IS[pad(H)] = mk(z.x - z.y, (R)0);
    } else {
      const Cx<R> a = IS[pad(k)];
      const Cx<R> bq = conj(IS[pad(H - k)]);
      const Cx<R> e = scale(a + bq, (R)0.5);
      const Cx<R> dd = a - bq;
      const Cx<R> o = mk(dd.y * (R)0.5, -dd.x * (R)0.5);
      const Cx<R> wo = cmul(o, ldg(twQ + k));
      IS[pad(k)] = e + wo;
      if (k != H - k) IS[pad(H - k)] = conj(e - wo);
    }
  }
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  // theta_hat_i[k] = sum_l T[i,l,k] I_hat_l[k]   (dbp.py:195)
  for (int k = tid; k <= H; k += NT) {
    Cx<R> acc = mk((R)0, (R)0);
    for (int l = 0; l < P; ++l) {
      const Cx<R>* rl = cluster.map_shared_rank(IS, l);
      acc = acc + cmul(ldg(T + ((size_t)i * P + l) * (H + 1) + k), rl[pad(k)]);
    }
    TS[pad(k)] = acc;
  }
  cluster.sync();  // every remote read of IS is done (no CTA exits early)
  // c2r twist (numpy irfft ignores Im of bins 0 and H) then IFFT_H
  for (int k = tid; k <= H / 2; k += NT) {
    if (k == 0) {
      const R x0 = TS[pad(0)].x, xh = TS[pad(H)].x;
      TS[pad(0)] = mk(x0 + xh, x0 - xh);
    } else {
      const Cx<R> a = TS[pad(k)];
      const Cx<R> c = conj(TS[pad(H - k)]);
      const Cx<R> wk = ldg(twQ + k);
      const Cx<R> s = a + c;
      const Cx<R> dd = cmulc(a - c, wk);
      TS[pad(k)] = mk(s.x - dd.y, s.y + dd.x);
      if (k != H - k) {
        const Cx<R> a2 = conj(c), c2 = conj(a);
        const Cx<R> s2 = a2 + c2;
        const Cx<R> w2 = mk(-wk.x, wk.y);
        const Cx<R> d2 = cmulc(a2 - c2, w2);
        TS[pad(H - k)] = mk(s2.x - d2.y, s2.y + d2.x);
      }
    }
  }
  __syncthreads();
  fft1<R, Q, H, NT, true>(TS, twp, &s_zero);
  // rotation exp(-j theta) of both polarisations (dbp.py:208)
  Cx<R>* xo = out + (size_t)i * Q;
  Cx<R>* yo = out + (size_t)(P + i) * Q;
  for (int t = tid; t < Q; t += NT) {
    const Cx<R> z = TS[pad(t >> 1)];
    R s, c;
    sincos_acc<R>(((t & 1) ? z.y : z.x) * theta_scale, &s, &c);
    const Cx<R> rot = mk(c, -s);
    xo[t] = cmul(xi[t], rot);
    yo[t] = cmul(yi[t], rot);
  }
}

thread_local std::string g_nlpr_err;

std::vector<double> unit_table(int64_t n) {
  std::vector<double> t(2 * n);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int64_t m = 0; m < n; ++m) {
    t[2 * m] = (double)cosl(-2.0L * pi * m / n);
    t[2 * m + 1] = (double)sinl(-2.0L * pi * m / n);
  }
  return t;
}

template <typename R, int Q>
cudaError_t run_q(const void* in, void* out, const double* T, int P, double theta_scale,
                  cudaStream_t st) {
  constexpr int H = Q / 2;
  // twiddles for the half-length FFT passes (kHalf schedule) and W_Q^k
  const std::vector<double> tq = unit_table(Q);
  std::vector<R> hp(2 * (size_t)twp_size(H, kHalf), (R)0);
  for (int ns = 1; ns < H; ns *= sched_radix(H, ns, kHalf)) {
    const int Rr = sched_radix(H, ns, kHalf);
    if (ns == 1) continue;
    for (int k = 0; k < ns; ++k)
      for (int r = 1; r < Rr; ++r) {
        const int64_t e = ((int64_t)r * k * (Q / (ns * Rr))) % Q;
        const size_t at = twp_offset(H, ns, kHalf) + tw_plane_index((int)sizeof(R), ns, k, r);
        hp[2 * at] = (R)tq[2 * e];
        hp[2 * at + 1] = (R)tq[2 * e + 1];
      }
  }
  std::vector<R> hq(2 * (size_t)Q), ht(2 * (size_t)P * P * (H + 1));
  for (size_t m = 0; m < hq.size(); ++m) hq[m] = (R)tq[m];
  for (size_t m = 0; m < ht.size(); ++m) ht[m] = (R)T[m];
  // stream-ordered scratch, released on every exit path (also when a later
  // allocation or upload fails)
  struct Frees {
    cudaStream_t st;
    void* p[3] = {nullptr, nullptr, nullptr};
    ~Frees() {
      for (void* q : p)
        if (q) cudaFreeAsync(q, st);
    }
  } fr{st};
  void *&dtq = fr.p[0], *&dtp = fr.p[1], *&dT = fr.p[2];
  cudaError_t e;
  if ((e = cudaMallocAsync(&dtq, hq.size() * sizeof(R), st)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&dtp, hp.size() * sizeof(R) + 16, st)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&dT, ht.size() * sizeof(R), st)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(dtq, hq.data(), hq.size() * sizeof(R), cudaMemcpyHostToDevice, st)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(dtp, hp.data(), hp.size() * sizeof(R), cudaMemcpyHostToDevice, st)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(dT, ht.data(), ht.size() * sizeof(R), cudaMemcpyHostToDevice, st)) !=
          cudaSuccess) {
    cudaStreamSynchronize(st);  // the host staging vectors may still be read
    return e;
  }
  auto kern = nlpr_kernel<R, Q>;
  const size_t smem = sizeof(Cx<R>) * 2 * (size_t)padded_len(H + 1);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (P > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P, 1, 1);
  cfg.blockDim = dim3(Q / 8, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, reinterpret_cast<const Cx<R>*>(in),
                         reinterpret_cast<Cx<R>*>(out), reinterpret_cast<const Cx<R>*>(dT),
                         reinterpret_cast<const Cx<R>*>(dtq), reinterpret_cast<const Cx<R>*>(dtp),
                         (R)(theta_scale / Q), P);
  // the host staging vectors are read by the async copies: wait for them
  // (the scratch is freed stream-ordered when `fr` goes out of scope)
  const cudaError_t s2 = cudaStreamSynchronize(st);
  return e != cudaSuccess ? e : s2;
}

template <typename R>
cudaError_t run_r(int q, const void* in, void* out, const double* T, int P, double ts,
                  cudaStream_t st) {
  switch (q) {
    case 256: return run_q<R, 256>(in, out, T, P, ts, st);
    case 512: return run_q<R, 512>(in, out, T, P, ts, st);
    case 1024: return run_q<R, 1024>(in, out, T, P, ts, st);
    case 2048: return run_q<R, 2048>(in, out, T, P, ts, st);
    case 4096: return run_q<R, 4096>(in, out, T, P, ts, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace
}  // namespace cbessfm

extern "C" cbessfm_status cbessfm_nlpr(int32_t dtype, int32_t n_subbands, int32_t n_prime,
                                       const void* in, void* out, const double* mimo,
                                       double theta_scale, void* stream) {
  using namespace cbessfm;
  if (dtype != CBESSFM_C64 && dtype != CBESSFM_C128) return CBESSFM_ERR_INVALID;
  if (n_subbands < 1 || n_subbands > kMaxSub || !in || !out || !mimo) return CBESSFM_ERR_INVALID;
  if (n_prime < 256 || n_prime > 4096 || (n_prime & (n_prime - 1))) return CBESSFM_ERR_UNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const cudaError_t e =
      dtype == CBESSFM_C64
          ? run_r<float>(n_prime, in, out, mimo, n_subbands, theta_scale, st)
          : run_r<double>(n_prime, in, out, mimo, n_subbands, theta_scale, st);
  return e == cudaSuccess ? CBESSFM_OK : CBESSFM_ERR_CUDA;
}
