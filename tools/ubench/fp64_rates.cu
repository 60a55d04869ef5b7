// FP64 issue rates on a B200 SM by instruction and operand pattern
// (warp-instructions per clock per SM; the nominal rate is 2.0 = 64 lanes).
// 8 independent chains per thread, 256 threads per CTA, 2 / 4 / 8 CTAs per SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_rates fp64_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 256, CH = 8, INNER = 64;

// KIND 0: DFMA acc = acc*a + b (a, b loop constants: the peak tool's form)
// KIND 1: DFMA acc[c] = acc[c]*x[c] + y[c] (three distinct varying registers)
// KIND 2: DADD acc[c] = acc[c] + x[c]
// KIND 3: DMUL acc[c] = acc[c] * x[c]
// KIND 4: butterfly mix: DADD : DFMA : DMUL = 52 : 27 : 21, all operands varying
template <int KIND>
__global__ void __launch_bounds__(NT) k(double* out, int iters, double a, double b) {
  double acc[CH], x[CH], y[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    acc[c] = threadIdx.x * 1e-7 + c;
    x[c] = a + c * 1e-9 * threadIdx.x;
    y[c] = b + c * 1e-9;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < INNER; ++q)
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        if (KIND == 0) acc[c] = fma(acc[c], a, b);
        if (KIND == 1) acc[c] = fma(acc[c], x[c], y[c]);
        if (KIND == 2) acc[c] = acc[c] + x[c];
        if (KIND == 3) acc[c] = acc[c] * x[c];
        if (KIND == 4) {
          const int s = (q * CH + c) % 4;
          if (s == 0 || s == 2) acc[c] = acc[c] + x[(c + 1) % CH];
          if (s == 1) acc[c] = fma(acc[c], x[c], y[c]);
          if (s == 3) acc[c] = acc[c] * x[c];
        }
      }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int KIND>
double rate(int ctas_per_sm, int sms, int khz, double* out) {
  const int iters = 400;
  k<KIND><<<sms * ctas_per_sm, NT>>>(out, 4, 0.999999, 1e-6);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<KIND><<<sms * ctas_per_sm, NT>>>(out, iters, 0.999999, 1e-6);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double winst = (double)ctas_per_sm * (NT / 32) * CH * INNER * iters;  // per SM
  return winst / (ms * 1e-3 * khz * 1e3);
}

int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 64);
  const char* names[5] = {"DFMA acc*a+b (constants)", "DFMA three varying regs", "DADD two varying regs",
                          "DMUL two varying regs", "butterfly mix 52/27/21"};
  printf("FP64 warp-instructions per clock per SM (nominal 2.0), clock %d MHz\n", khz / 1000);
  for (int cps : {2, 4, 8}) {
    const double r[5] = {rate<0>(cps, sms, khz, out), rate<1>(cps, sms, khz, out), rate<2>(cps, sms, khz, out),
                         rate<3>(cps, sms, khz, out), rate<4>(cps, sms, khz, out)};
    for (int m = 0; m < 5; ++m) printf("  %d CTAs/SM  %-28s %.3f\n", cps, names[m], r[m]);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
