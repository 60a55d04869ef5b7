// Host-side launch helpers for the fused block kernel (cluster launch via
// cudaLaunchKernelEx, dynamic shared memory opt-in, non-portable clusters).
#pragma once

#include <cstdio>
#include <cstdlib>

#include "cbessfm_kernel.cuh"
#include "cbessfm_ip.cuh"

namespace cbessfm {

struct KernelInfo {
  int threads;
  int cluster;
  size_t smem;
  int max_active_clusters;
  char name[64];  // the kernel a launch of this shape runs
};

template <typename R>
constexpr const char* real_name() {
  return sizeof(R) == 4 ? "float" : "double";
}

template <typename R>
constexpr int max_q() {
  return sizeof(R) == 4 ? 8192 : 4096;
}

// One-block-per-CTA kernel (cbessfm_fat_kernel): one CTA of P * Q/16
// threads per overlap-save block, no cluster. Used where fat_ok() holds
// (see use_fat_kernel).
template <typename R, int P, int Q>
cudaError_t launch_fat(const Params<R>& prm, int64_t nblocks, cudaStream_t stream,
                       KernelInfo* info) {
  auto kern = cbessfm_fat_kernel<R, P, Q>;
  constexpr int NT = P * fat_group<Q>();
  constexpr size_t smem = fat_smem_bytes<R, P, Q>();
  static unsigned long long configured = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
  }
  if (info) {
    info->threads = NT;
    info->cluster = 1;
    info->smem = smem;
    snprintf(info->name, sizeof info->name, "cbessfm_fat_kernel<%s,%d,%d>", real_name<R>(), P, Q);
    int per_sm = 0, sms = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
    if (e != cudaSuccess) return e;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    info->max_active_clusters = per_sm * sms;
    if (nblocks == 0) return cudaSuccess;
  }
  const int64_t max_blocks = 0x7fffffff;
  Params<R> p = prm;
  for (int64_t c0 = 0; c0 < nblocks; c0 += max_blocks) {
    const int64_t nc = nblocks - c0 < max_blocks ? nblocks - c0 : max_blocks;
    p.cid0 = prm.cid0 + c0;
    kern<<<dim3((unsigned)nc), dim3(NT), smem, stream>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Kernel choice where both kernels apply (FP32, N' = 2048, P <= 5): the
// one-block-per-CTA kernel for device-resident launches (configs[1]
// waveforms: 0.386 / 0.741 / 1.43 / 2.81 / 5.55 ms for 1 / 2 / 4 / 8 / 16
// per launch vs 0.471 / 0.815 / 1.53 / 2.95 / 5.81 for the cluster kernel),
// the cluster kernel for the pipelined host path, whose chunks of a few
// blocks want the lower per-block latency of spreading a block over P SMs
// (end to end 2.74e9 vs 2.63e9 2D/s). CBESSFM_KERNEL=fat|cluster overrides.
inline bool use_fat_kernel(int64_t nblocks, int pref) {
  (void)nblocks;
  const char* env = getenv("CBESSFM_KERNEL");
  if (env && env[0] == 'c') return false;
  if (env && env[0] == 'f') return true;
  return pref != 1;
}

// Launch of a P-CTA-cluster block kernel (one cluster per overlap-save
// block): dynamic shared memory opt-in and sizing, non-portable clusters,
// occupancy query for `info`. KERN is cbessfm_block_kernel<R, P, Q> or
// cbessfm_ip_kernel<R, P> (same Params, threads, shared memory and TMEM).
template <typename R, int P, int Q, void (*KERN)(const Params<R>), bool PERSIST = false>
cudaError_t launch_cluster(const char* kname, const Params<R>& prm, int64_t nclusters,
                           cudaStream_t stream, KernelInfo* info) {
  auto kern = KERN;
  constexpr int NT = threads_for<R, Q>();
  size_t smem = smem_bytes<R, Q>(P);
  // function attributes are per device; set them once per device
  static unsigned long long configured = 0;
  static size_t smem_tm = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if constexpr (tm_on<R, Q>()) {
    // TMEM twiddles: every resident CTA holds 512 / min_blocks columns, so
    // no more than min_blocks CTAs of TMEM-using kernels may share an SM.
    // Claiming 1/min_blocks of the SM's shared memory (the fields use most
    // of it anyway) guarantees that for any mix of such kernels, and the
    // tcgen05.alloc in the kernel never waits.
    if (!smem_tm) {
      int per_sm = 0, reserved = 0;
      cudaFuncAttributes fa = {};
      cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
      cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
      cudaError_t e = cudaFuncGetAttributes(&fa, kern);
      if (e != cudaSuccess) return e;
      // (1 KB below the exact share: the occupancy calculator treats an
      // exactly full SM as one CTA short)
      const size_t need =
          (size_t)per_sm / min_blocks<R, Q>() - (size_t)reserved - fa.sharedSizeBytes - 1024;
      smem_tm = need > smem ? need : smem;
    }
    smem = smem_tm;
  }
  if (!(__atomic_load_n(&configured, __ATOMIC_ACQUIRE) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (P > 8) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    if constexpr (tm_on<R, Q>()) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
      if (e != cudaSuccess) return e;
    }
    __atomic_fetch_or(&configured, bit, __ATOMIC_RELEASE);
  }
  if (const char* env = getenv("CBESSFM_CARVEOUT")) {  // experiment hook
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(env));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = P > 1 ? 1 : 0;
  if (const char* env = getenv("CBESSFM_CLUSTER_POLICY")) {  // experiment hook: 1 spread, 2 load balancing
    if (P > 1 && atoi(env) > 0) {
      attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
      attr[1].val.clusterSchedulingPolicyPreference =
          atoi(env) == 1 ? cudaClusterSchedulingPolicySpread : cudaClusterSchedulingPolicyLoadBalancing;
      cfg.numAttrs = 2;
    }
  }
  if (info) {
    info->threads = NT;
    info->cluster = P;
    info->smem = smem;
    snprintf(info->name, sizeof info->name, "%s<%s,%d,%d>", kname, real_name<R>(), P, Q);
    cfg.gridDim = dim3(P, 1, 1);
    int nc = 0;
    if (P > 1) {
      cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, kern, &cfg);
      if (e != cudaSuccess) return e;
    } else {
      int per_sm = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem);
      if (e != cudaSuccess) return e;
      int sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      nc = per_sm * sms;
    }
    info->max_active_clusters = nc;
    if (nclusters == 0) return cudaSuccess;
  }
  Params<R> p = prm;
  if (PERSIST && p.work) {
    // persistent launch (cbessfm_block_kernel): twice as many clusters as
    // the register budget lets the SMs hold -- those beyond what the GPU
    // actually co-schedules start late, find the counter spent and exit --
    // each claiming blocks until all nclusters are done. CBESSFM_PERSIST=0
    // launches one cluster per block (A/B); CBESSFM_PERSIST=k > 0 sets the
    // grid to k clusters (tests: every block count takes the loop).
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t g = (int64_t)2 * sms * min_blocks<R, Q>() / P > 1
                    ? (int64_t)2 * sms * min_blocks<R, Q>() / P
                    : 1;
    const char* env = getenv("CBESSFM_PERSIST");
    if (env && atoi(env) > 0) g = atoi(env);
    if (nclusters > g && !(env && env[0] == '0')) {
      cudaError_t e = cudaMemsetAsync(p.work, 0, sizeof(unsigned long long), stream);
      if (e != cudaSuccess) return e;
      p.total = nclusters;
      cfg.gridDim = dim3((unsigned)(g * P), 1, 1);
      return cudaLaunchKernelEx(&cfg, kern, p);
    }
  }
  p.work = nullptr;
  // grid.x is limited to 2^31-1 CTAs: launch in chunks of whole clusters
  const int64_t max_clusters = (int64_t)(0x7fffffff / P);
  for (int64_t c0 = 0; c0 < nclusters; c0 += max_clusters) {
    const int64_t nc = nclusters - c0 < max_clusters ? nclusters - c0 : max_clusters;
    p.cid0 = prm.cid0 + c0;
    cfg.gridDim = dim3((unsigned)(nc * P), 1, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}


// In-place-pass kernel (cbessfm_ip.cuh, complex128, N' = 2048, P >= 2):
// selected with CBESSFM_KERNEL=ip. Same results as the cluster kernel within
// rounding (parity-tested), same persistent launch, prefetch and rotation
// table, but not faster: at equal features it went from 1.5 % ahead (367.2
// vs 372.9 ms on configs[4], one cluster per block, polynomial sincos) to
// 1.9 % behind once both had the persistent launch and the table (353.2 vs
// 346.7 ms; tools/gpu/r2_s4_ip2.sh, r2_s4_ipp.sh), so the Stockham cluster
// kernel stays the default.
template <typename R, int P, int Q>
constexpr bool ip_ok() {
  return sizeof(R) == 8 && Q == kIpQ && P >= 2;
}
inline bool use_ip_kernel() {
  const char* env = getenv("CBESSFM_KERNEL");
  return env && env[0] == 'i';
}

template <typename R, int P, int Q>
cudaError_t launch_one(const Params<R>& prm, int64_t nclusters, cudaStream_t stream,
                       KernelInfo* info) {
  if constexpr (fat_ok<R, P, Q>()) {
    if (use_fat_kernel(nclusters, prm.kernel_pref)) return launch_fat<R, P, Q>(prm, nclusters, stream, info);
  }
  if constexpr (ip_ok<R, P, Q>()) {
    if (use_ip_kernel() && prm.phasor_rev)
      return launch_cluster<R, P, Q, cbessfm_ip_kernel<R, P>, true>("cbessfm_ip_kernel", prm,
                                                                    nclusters, stream, info);
  }
  return launch_cluster<R, P, Q, cbessfm_block_kernel<R, P, Q>, true>("cbessfm_block_kernel", prm,
                                                                      nclusters, stream, info);
}

template <typename R, int P>
cudaError_t launch_q(const Params<R>& prm, int q, int64_t nclusters, cudaStream_t stream,
                     KernelInfo* info) {
  switch (q) {
    case 256: return launch_one<R, P, 256>(prm, nclusters, stream, info);
    case 512: return launch_one<R, P, 512>(prm, nclusters, stream, info);
    case 1024: return launch_one<R, P, 1024>(prm, nclusters, stream, info);
    case 2048: return launch_one<R, P, 2048>(prm, nclusters, stream, info);
    case 4096: return launch_one<R, P, 4096>(prm, nclusters, stream, info);
    case 8192:
      if constexpr (max_q<R>() >= 8192) return launch_one<R, P, 8192>(prm, nclusters, stream, info);
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

#define CB_DECLARE(T, P)                                                                 \
  cudaError_t launch_##T##_##P(const Params<T>& prm, int q, int64_t nclusters, cudaStream_t, \
                               KernelInfo* info);
#define CB_FOR_P(T) \
  CB_DECLARE(T, 1) CB_DECLARE(T, 2) CB_DECLARE(T, 3) CB_DECLARE(T, 4) CB_DECLARE(T, 5) \
  CB_DECLARE(T, 6) CB_DECLARE(T, 7) CB_DECLARE(T, 8) CB_DECLARE(T, 9)
CB_FOR_P(float)
CB_FOR_P(double)
#undef CB_FOR_P
#undef CB_DECLARE

}  // namespace cbessfm
