// Standalone check of the shared-memory Stockham FFT used by the fused
// kernel: forward/inverse, float/double, NA = 1/2, against a long-double DFT.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2409_14489_b200/csrc/cbessfm_kernel.cuh"
using namespace cbessfm;

template <typename R, int Q, int L, int NA, bool INV>
__global__ void __launch_bounds__(threads_for<R, Q>()) kfft(const Cx<R>* tw, Cx<R>* data) {
  constexpr int NT = threads_for<R, Q>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int z;
  if (threadIdx.x == 0) z = 0;
  Cx<R>* buf = reinterpret_cast<Cx<R>*>(smem_raw);
  for (int a = 0; a < NA; ++a)
    for (int i = threadIdx.x; i < L; i += NT) buf[a * padded_len(L) + pad(i)] = data[a * L + i];
  __syncthreads();
  fft<R, Q, L, NA, NT, Cfg<R>::MAXRAD, INV>(buf, tw, &z);
  for (int a = 0; a < NA; ++a)
    for (int i = threadIdx.x; i < L; i += NT) data[a * L + i] = buf[a * padded_len(L) + pad(i)];
}

template <typename R, int Q, int L, int NA, bool INV>
double run() {
  const int n = NA * L;
  std::vector<Cx<R>> h(n), tw(Q);
  std::vector<long double> re(n), im(n);
  srand(1);
  for (int i = 0; i < n; ++i) {
    re[i] = rand() / (long double)RAND_MAX - 0.5L;
    im[i] = rand() / (long double)RAND_MAX - 0.5L;
    h[i].x = (R)re[i];
    h[i].y = (R)im[i];
    re[i] = h[i].x;
    im[i] = h[i].y;
  }
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int m = 0; m < Q; ++m) {
    tw[m].x = (R)cosl(-2 * pi * m / Q);
    tw[m].y = (R)sinl(-2 * pi * m / Q);
  }
  Cx<R>*dd, *dt;
  cudaMalloc(&dd, n * sizeof(Cx<R>));
  cudaMalloc(&dt, Q * sizeof(Cx<R>));
  cudaMemcpy(dd, h.data(), n * sizeof(Cx<R>), cudaMemcpyHostToDevice);
  cudaMemcpy(dt, tw.data(), Q * sizeof(Cx<R>), cudaMemcpyHostToDevice);
  const size_t smem = NA * padded_len(L) * sizeof(Cx<R>);
  cudaFuncSetAttribute(kfft<R, Q, L, NA, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kfft<R, Q, L, NA, INV><<<1, threads_for<R, Q>(), smem>>>(dt, dd);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  std::vector<Cx<R>> o(n);
  cudaMemcpy(o.data(), dd, n * sizeof(Cx<R>), cudaMemcpyDeviceToHost);
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

#define T(R, Q, L, NA, INV) \
  printf("%-6s Q=%5d L=%5d NA=%d inv=%d relL2=%.3e\n", #R, Q, L, NA, INV, run<R, Q, L, NA, INV>());

int main() {
  T(float, 512, 512, 2, false) T(float, 512, 256, 1, false) T(float, 2048, 2048, 2, false)
  T(float, 2048, 2048, 2, true) T(float, 2048, 1024, 1, false) T(float, 2048, 1024, 1, true)
  T(float, 4096, 4096, 2, false) T(float, 4096, 2048, 1, true) T(float, 1024, 1024, 2, false)
  T(float, 1024, 512, 1, false) T(float, 256, 256, 2, false) T(float, 256, 128, 1, false)
  T(double, 2048, 2048, 2, false) T(double, 2048, 1024, 1, true) T(double, 4096, 4096, 2, true)
  T(double, 4096, 2048, 1, false) T(double, 512, 512, 2, false) T(double, 256, 128, 1, true)
  return 0;
}
