// Standalone check of the shared-memory Stockham FFTs used by the fused
// kernel (two-polarisation fft2 with per-pass twiddle rows, and the
// half-length fft1), forward/inverse, float/double, against a long-double DFT.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2409_14489_b200/csrc/cbessfm_kernel.cuh"
using namespace cbessfm;

template <typename R, int Q, bool HALF, bool INV>
__global__ void __launch_bounds__(threads_for<R, Q>()) kfft(const Cx<R>* twp, Cx<R>* data) {
  constexpr int NT = threads_for<R, Q>();
  constexpr int L = HALF ? Q / 2 : Q;
  constexpr int NA = HALF ? 1 : 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int z;
  if (threadIdx.x == 0) z = 0;
  Cx<R>* buf = reinterpret_cast<Cx<R>*>(smem_raw);
  for (int a = 0; a < NA; ++a)
    for (int i = threadIdx.x; i < L; i += NT) buf[a * padded_len(L) + pad(i)] = data[a * L + i];
  __syncthreads();
  if constexpr (HALF)
    fft1<R, Q, L, NT, INV>(buf, twp + twp_base(Q, kHalf), &z);
  else if constexpr (INV)
    fft2<R, Q, NT, kTail, INV>(buf, twp + twp_base(Q, kTail), &z);
  else
    fft2<R, Q, NT, kHead, INV>(buf, twp + twp_base(Q, kHead), &z);
  for (int a = 0; a < NA; ++a)
    for (int i = threadIdx.x; i < L; i += NT) data[a * L + i] = buf[a * padded_len(L) + pad(i)];
}

template <typename R>
std::vector<Cx<R>> tables(int Q) {
  const long double pi = 3.141592653589793238462643383279502884L;
  std::vector<Cx<R>> out(twp_total(Q));
  auto fill = [&](int L, int sched) {
    for (int ns = 1; ns < L; ns *= sched_radix(L, ns, sched)) {
      const int Rr = sched_radix(L, ns, sched);
      if (ns == 1) continue;
      for (int k = 0; k < ns; ++k)
        for (int r = 0; r < Rr; ++r) {
          const long long e = (long long)r * k * (Q / (ns * Rr)) % Q;
          if (r == 0) continue;
          Cx<R>& o = out[twp_base(Q, sched) + twp_offset(L, ns, sched) +
                         tw_plane_index((int)sizeof(R), ns, k, r)];
          o.x = (R)cosl(-2 * pi * e / Q);
          o.y = (R)sinl(-2 * pi * e / Q);
        }
    }
  };
  fill(Q, kTail);
  fill(Q, kHead);
  fill(Q / 2, kHalf);
  return out;
}

template <typename R, int Q, bool HALF, bool INV>
double run() {
  constexpr int L = HALF ? Q / 2 : Q;
  constexpr int NA = HALF ? 1 : 2;
  const int n = NA * L;
  std::vector<Cx<R>> h(n);
  std::vector<long double> re(n), im(n);
  srand(1);
  for (int i = 0; i < n; ++i) {
    h[i].x = (R)(rand() / (double)RAND_MAX - 0.5);
    h[i].y = (R)(rand() / (double)RAND_MAX - 0.5);
    re[i] = h[i].x;
    im[i] = h[i].y;
  }
  const std::vector<Cx<R>> tw = tables<R>(Q);
  Cx<R>*dd, *dt;
  cudaMalloc(&dd, n * sizeof(Cx<R>));
  cudaMalloc(&dt, tw.size() * sizeof(Cx<R>));
  cudaMemcpy(dd, h.data(), n * sizeof(Cx<R>), cudaMemcpyHostToDevice);
  cudaMemcpy(dt, tw.data(), tw.size() * sizeof(Cx<R>), cudaMemcpyHostToDevice);
  const size_t smem = 2 * padded_len(Q) * sizeof(Cx<R>);
  cudaFuncSetAttribute(kfft<R, Q, HALF, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kfft<R, Q, HALF, INV><<<1, threads_for<R, Q>(), smem>>>(dt, dd);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  std::vector<Cx<R>> o(n);
  cudaMemcpy(o.data(), dd, n * sizeof(Cx<R>), cudaMemcpyDeviceToHost);
  const long double pi = 3.141592653589793238462643383279502884L;
  long double num = 0, den = 0;
  const long double sg = INV ? 1 : -1;
  for (int a = 0; a < NA; ++a)
    for (int k = 0; k < L; ++k) {
      long double sr = 0, si = 0;
      for (int t = 0; t < L; ++t) {
        const long double ang = sg * 2 * pi * (long double)((long long)k * t % L) / L;
        const long double c = cosl(ang), s = sinl(ang);
        sr += re[a * L + t] * c - im[a * L + t] * s;
        si += re[a * L + t] * s + im[a * L + t] * c;
      }
      const long double dr = o[a * L + k].x - sr, di = o[a * L + k].y - si;
      num += dr * dr + di * di;
      den += sr * sr + si * si;
    }
  cudaFree(dd);
  cudaFree(dt);
  return (double)sqrtl(num / den);
}

#define T(R, Q, HALF, INV) \
  printf("%-6s Q=%5d half=%d inv=%d relL2=%.3e\n", #R, Q, HALF, INV, run<R, Q, HALF, INV>());

int main() {
  T(float, 256, false, false) T(float, 256, true, false) T(float, 512, false, true)
  T(float, 512, true, true) T(float, 1024, false, false) T(float, 1024, true, true)
  T(float, 2048, false, false) T(float, 2048, false, true) T(float, 2048, true, false)
  T(float, 2048, true, true) T(float, 4096, false, true) T(float, 4096, true, false)
  T(float, 8192, false, false) T(float, 8192, true, true)
  T(double, 256, true, true) T(double, 512, false, false) T(double, 2048, false, true)
  T(double, 2048, true, false) T(double, 4096, false, false) T(double, 4096, true, true)
  return 0;
}
