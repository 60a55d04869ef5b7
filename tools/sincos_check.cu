// Accuracy of the kernel's FP32 sincos against FP64 over the range a
// nonlinear phase can take (and past the reduction threshold).
#include <cstdio>
#include <cmath>
#include "../paper_2409_14489_b200/csrc/cbessfm_kernel.cuh"
__global__ void k(const float* a, float* s, float* c, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cbessfm::sincos_acc<float>(a[i], s + i, c + i);
}
int main() {
  const int n = 1 << 22;
  float *a, *s, *c;
  cudaMallocManaged(&a, n * 4); cudaMallocManaged(&s, n * 4); cudaMallocManaged(&c, n * 4);
  const float lim[] = {1.0f, 10.0f, 1000.0f, 8192.0f, 1e5f};
  for (float L : lim) {
    for (int i = 0; i < n; ++i) a[i] = L * (2.0f * (i + 0.5f) / n - 1.0f);
    k<<<n / 256, 256>>>(a, s, c, n);
    cudaDeviceSynchronize();
    double es = 0, ec = 0;
    for (int i = 0; i < n; ++i) {
      es = fmax(es, fabs(s[i] - sin((double)a[i])));
      ec = fmax(ec, fabs(c[i] - cos((double)a[i])));
    }
    printf("|a|<=%g  max abs err sin %.3e cos %.3e (2^-24=%.3e)\n", L, es, ec, ldexp(1.0, -24));
  }
  return 0;
}
