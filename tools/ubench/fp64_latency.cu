// Dependent-issue latency of FP64 instructions on B200 (one warp, one chain),
// and throughput of one warp with 1..16 independent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, int KIND>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-7 + c;
  double x = a + threadIdx.x * 1e-9, y = b;
  const long long t0 = clock64();
  for (int i = 0; i < 256; ++i) {
#pragma unroll
    for (int q = 0; q < 16; ++q)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (KIND == 0) acc[c] = fma(acc[c], x, y);
        if (KIND == 1) acc[c] = acc[c] + x;
        if (KIND == 2) acc[c] = acc[c] * x;
      }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int CH, int KIND>
double run(double* out, long long* cyc) {
  k<CH, KIND><<<1, 32>>>(out, cyc, 0.999999, 1e-6);
  k<CH, KIND><<<1, 32>>>(out, cyc, 0.999999, 1e-6);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  return (double)h / (256.0 * 16 * CH);
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
  const char* n[3] = {"DFMA", "DADD", "DMUL"};
  printf("cycles per instruction, one warp, CH independent chains\n");
  printf("%s: CH=1 %.2f  CH=2 %.2f  CH=4 %.2f  CH=8 %.2f  CH=16 %.2f\n", n[0], run<1,0>(out,cyc), run<2,0>(out,cyc), run<4,0>(out,cyc), run<8,0>(out,cyc), run<16,0>(out,cyc));
  printf("%s: CH=1 %.2f  CH=2 %.2f  CH=4 %.2f  CH=8 %.2f  CH=16 %.2f\n", n[1], run<1,1>(out,cyc), run<2,1>(out,cyc), run<4,1>(out,cyc), run<8,1>(out,cyc), run<16,1>(out,cyc));
  printf("%s: CH=1 %.2f  CH=2 %.2f  CH=4 %.2f  CH=8 %.2f  CH=16 %.2f\n", n[2], run<1,2>(out,cyc), run<2,2>(out,cyc), run<4,2>(out,cyc), run<8,2>(out,cyc), run<16,2>(out,cyc));
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
}
