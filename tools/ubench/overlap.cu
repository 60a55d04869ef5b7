// Do FP64 arithmetic and shared-memory traffic overlap on a B200 SM?
// Each "pass" of a thread mimics one field pass of the c128 cluster kernel:
// 16 LDS.128, NF FP64 FMAs (8 independent chains), 16 STS.128.
//   mode 0: FP64 only            mode 1: shared memory only
//   mode 2: both, free-running warps (no barriers)
//   mode 3: both, __syncthreads between load / compute+store (the kernel's form)
//   mode 4: warp-specialised: even warps only FP64, odd warps only LDS/STS (2x each)
// 256 threads per CTA, 2 CTAs per SM (shared memory sized to force that).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o overlap overlap.cu
#include <cstdio>
#include <cuda_runtime.h>

// -DADDMIX: the FP64 work is two-operand DADDs (2 issue cycles each, like most of
// a butterfly) instead of three-operand DFMAs (3 cycles each here)
#ifdef ADDMIX
#define FPOP(a, m, b) ((a) + (b))
#else
#define FPOP(a, m, b) fma((a), (m), (b))
#endif
constexpr int NT = 256;
constexpr int NF = 200;

template <int MODE>
__global__ void __launch_bounds__(NT, 2) k(double2* out, int passes, double seed) {
  extern __shared__ __align__(16) double2 sm[];
  const int tid = threadIdx.x;
  double2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = make_double2(seed * (tid + r), seed * r);
  for (int i = tid; i < 4096; i += NT) sm[i] = make_double2(seed, i);
  __syncthreads();
  const bool fp = MODE == 0 || MODE == 2 || MODE == 3 || (MODE == 4 && ((tid >> 5) & 1) == 0);
  const bool ls = MODE == 1 || MODE == 2 || MODE == 3 || (MODE == 4 && ((tid >> 5) & 1) == 1);
  const int reps = MODE == 4 ? 2 : 1;
  for (int p = 0; p < passes; ++p) {
    if (ls) {
#pragma unroll
      for (int q = 0; q < reps; ++q)
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double2 t = sm[((tid + p + q) & 255) + 256 * r];
          v[r].x += t.x;
          v[r].y += t.y;
        }
    }
    if (fp) {
      // (accumulators and multipliers in registers of their own: operands
      // taken straight from the 4-aligned quads an LDS.128 fills collide on
      // the register banks and cost a third cycle per DFMA)
      double ax[8], ay[8], mx[8], my[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        ax[r] = v[r].x;
        ay[r] = v[r].y;
        mx[r] = v[r + 8].x + 1.0;
        my[r] = v[r + 8].y + 1.0;
      }
#pragma unroll
      for (int q = 0; q < reps; ++q)
#pragma unroll
        for (int f = 0; f < NF / 16; ++f)
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            ax[r] = FPOP(ax[r], my[r], ay[r]);
            ay[r] = FPOP(ay[r], mx[r], ax[r]);
          }
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        v[r].x = ax[r];
        v[r].y = ay[r];
      }
    }
    if (MODE == 3) __syncthreads();
    if (ls) {
#pragma unroll
      for (int q = 0; q < reps; ++q)
#pragma unroll
        for (int r = 0; r < 16; ++r) sm[((tid + p + q) & 255) + 256 * r] = v[r];
    }
    if (MODE == 3) __syncthreads();
  }
  double2 acc = make_double2(0, 0);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    acc.x += v[r].x;
    acc.y += v[r].y;
  }
  if (acc.x == 1.2345) out[blockIdx.x * NT + tid] = acc;
}

template <int MODE>
float run(int ctas, int passes, double2* out) {
  const size_t smem = 100 * 1024;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k<MODE>, NT, smem);
  if (MODE == 0 && passes == 2000) printf("  (occupancy query: %d CTAs per SM)\n", occ);
  k<MODE><<<ctas, NT, smem>>>(out, 10, 1e-9);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<ctas, NT, smem>>>(out, passes, 1e-9);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms = 0, khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
  double2* out;
  cudaMalloc(&out, sizeof(double2) * NT * sms * 2);
  const int passes = 2000;
  for (int per_sm = 1; per_sm <= 2; ++per_sm) {
    const int ctas = sms * per_sm;
    const float t[5] = {run<0>(ctas, passes, out), run<1>(ctas, passes, out), run<2>(ctas, passes, out),
                        run<3>(ctas, passes, out), run<4>(ctas, passes / 2, out) * 2};
    const char* names[5] = {"fp64 only", "smem only", "both, free-running", "both, barriers",
                            "warp-specialised"};
    printf("%d CTA(s) of %d threads per SM, %d passes, clock %d MHz\n", per_sm, NT, passes, khz / 1000);
    for (int m = 0; m < 5; ++m)
      printf("  %-22s %8.3f ms  %7.0f cycles per pass\n", names[m], t[m],
             t[m] * 1e-3 * khz * 1e3 / passes);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
