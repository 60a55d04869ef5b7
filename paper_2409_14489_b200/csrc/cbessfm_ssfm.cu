// Fine-step split-step Fourier propagation: the
// reference's ground-truth channel propagate_link and its exact inverse
// backward_propagate (channel.py:176-256), the IDEAL_SSFM variant of
// run_dbp (dbp.py:451-454).
//
// The whole waveform (n up to 2^22 per polarisation) is transformed with a
// four-step FFT, n = n1 * n2, data kept in natural time order [n1][n2]:
//   forward:  column FFTs of length n1, twiddle W_n^(j2 k1), row FFTs of
//             length n2 -> spectrum X[k1 + n1 k2] stored at (k1, k2);
//   inverse:  the same passes undone in reverse order.
// A fine step (channel.py:206-212) touches the spectrum only between the
// row FFT and the row IFFT, and the time samples only between the column
// IFFT and the column FFT, so one step is two fused passes over HBM/L2:
//   row phase    : FFT_n2 -> x half(dz_prev) -> x half(dz) -> IFFT_n2
//   column phase : x conj(W) -> IFFT_n1 -> /n -> exp(-j phi |E|^2) ->
//                  FFT_n1 -> x W
// Every phase is a loop over tiles (rows or column strips, both
// polarisations of one waveform per tile) held in shared memory; the
// phases are separated by grid-wide barriers of one cooperative launch
// that runs every span and step. The half-step tables are permuted on the
// host into the (k1, k2) storage order so the row phase reads them
// coalesced; the four-step twiddles come from two small tables.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/cbessfm_ssfm.h"
#include "cbessfm_fft4.cuh"

namespace cbessfm {
namespace ssfm {
namespace cg = cooperative_groups;

template <typename R, int LG>
__global__ void __launch_bounds__(kThreads, 1024 / kThreads) ssfm_kernel(const __grid_constant__ Params<R> p) {
  constexpr int N1 = Split<LG>::N1, N2 = Split<LG>::N2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CB_POISON_SMEM(smem_raw);
  Cx<R>* buf = reinterpret_cast<Cx<R>*>(smem_raw);
  cg::grid_group grid = cg::this_grid();
  {  // both per-length twiddle tables, staged once for every phase of the run
    Cx<R>* tw = buf + 2 * p.buf_elems;
    for (int i = threadIdx.x; i < N1; i += kThreads) tw[i] = ldg(p.tw1 + i);
    for (int i = threadIdx.x; i < N2; i += kThreads) tw[N1 + i] = ldg(p.tw2 + i);
    __syncthreads();
  }
  const size_t tab = (size_t)p.n;
  for (int span = 0; span < p.n_spans; ++span) {
    if (span == 0)  // spec = fft(field) (channel.py:206), after / g when backward
      col_phase<R, N1>(p, buf, false, kNone, (R)0, nullptr, p.backward != 0, true, true);
    for (int s = 0; s < p.k; ++s) {
      grid.sync();
      const Cx<R>* ha = s ? p.half + tab * p.step_table[s - 1] : nullptr;
      row_phase<R, N2>(p, buf, ha, p.half + tab * p.step_table[s], true, true, true);
      grid.sync();
      col_phase<R, N1>(p, buf, true, kNonlinear, p.nl_coef[s], nullptr, false, true, true);
    }
    grid.sync();
    row_phase<R, N2>(p, buf, p.half + tab * p.step_table[p.k - 1], (const Cx<R>*)nullptr, true,
                     true, true);
    grid.sync();
    const bool more = span + 1 < p.n_spans;
    const Cx<R>* nz = p.noise ? p.noise + (int64_t)span * p.batch * 2 * p.n : nullptr;
    col_phase<R, N1>(p, buf, true, kSpanEnd, (R)0, nz, more && p.backward, more, true);
    if (more) grid.sync();
  }
}

template <typename R>
struct KernelFor {
  template <int LG>
  struct At {
    static const void* get() { return (const void*)ssfm_kernel<R, LG>; }
  };
};

thread_local std::string g_err;

cbessfm_status fail(cbessfm_status s, const std::string& m) {
  g_err = m;
  return s;
}

template <typename R>
cbessfm_status run(const cbessfm_ssfm_desc* d, void* data, const void* noise, cudaStream_t st) {
  const int64_t n = d->n;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
  const Geo g = geometry(n, d->batch, sizeof(Cx<R>), 2 * sms);
  const void* kern = dispatch_lg<KernelFor<R>::template At>(__builtin_ctzll(n));
  if (!kern) return fail(CBESSFM_ERR_UNSUPPORTED, "no propagator kernel for this length");
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)g.smem);
  if (e != cudaSuccess) return fail(CBESSFM_ERR_CUDA, cudaGetErrorString(e));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, g.smem);
  if (occ < 1) return fail(CBESSFM_ERR_CUDA, "ssfm kernel does not fit on an SM");
  const int64_t tiles = std::max<int64_t>((int64_t)d->batch * g.n1 / g.rows,
                                          (int64_t)d->batch * g.n2 / g.cols);
  const int grid = (int)std::min<int64_t>((int64_t)occ * sms, tiles);

  // host tables: four-step twiddles (Fft4Tables), permuted halves
  Params<R> p;
  Fft4Tables<R> tw;
  StreamFrees frees(st);
  e = tw.build(n, g, st, &p);
  frees.add(tw.dn);
  frees.add(tw.d1);
  frees.add(tw.d2);
  if (e != cudaSuccess)
    return fail(CBESSFM_ERR_CUDA, std::string("ssfm twiddle upload: ") + cudaGetErrorString(e));
  std::vector<R> half(2 * (size_t)d->n_tables * n);
  for (int tb = 0; tb < d->n_tables; ++tb)
    for (int64_t k1 = 0; k1 < g.n1; ++k1)
      for (int64_t k2 = 0; k2 < g.n2; ++k2) {
        const size_t src = (size_t)tb * n + (size_t)(k1 + (int64_t)g.n1 * k2);
        const size_t dst = (size_t)tb * n + (size_t)(k1 * g.n2 + k2);
        half[2 * dst] = (R)d->half[2 * src];
        half[2 * dst + 1] = (R)d->half[2 * src + 1];
      }
  std::vector<int> steps(d->step_table, d->step_table + d->steps_per_span);
  std::vector<R> nl(d->steps_per_span);
  for (int s = 0; s < d->steps_per_span; ++s) nl[s] = (R)d->nl_coef[s];

  void *dh = nullptr, *ds = nullptr, *dn = nullptr;
  e = upload(half, &dh, st);
  if (e == cudaSuccess) e = upload(steps, &ds, st);
  if (e == cudaSuccess) e = upload(nl, &dn, st);
  frees.add(dh);
  frees.add(ds);
  frees.add(dn);
  if (e != cudaSuccess)
    return fail(CBESSFM_ERR_CUDA, std::string("ssfm table upload: ") + cudaGetErrorString(e));

  p.data = reinterpret_cast<Cx<R>*>(data);
  p.batch = d->batch;
  p.half = reinterpret_cast<const Cx<R>*>(dh);
  p.step_table = reinterpret_cast<const int*>(ds);
  p.nl_coef = reinterpret_cast<const R*>(dn);
  p.k = d->steps_per_span;
  p.n_spans = d->n_spans;
  p.backward = d->backward;
  p.gain = (R)d->gain;
  p.noise = reinterpret_cast<const Cx<R>*>(noise);
  void* args[] = {&p};
  e = cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kThreads), args, g.smem, st);
  // the StreamFrees guard releases the tables after the launch, in stream order
  // the host staging vectors are read by the async copies
  const cudaError_t s2 = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(CBESSFM_ERR_CUDA, std::string("ssfm launch: ") + cudaGetErrorString(e));
  if (s2 != cudaSuccess) return fail(CBESSFM_ERR_CUDA, std::string("ssfm: ") + cudaGetErrorString(s2));
  return CBESSFM_OK;
}

}  // namespace ssfm
}  // namespace cbessfm

extern "C" {

cbessfm_status cbessfm_ssfm_info_get(int32_t dtype, int64_t n, int32_t batch, int32_t device,
                                     cbessfm_ssfm_info* info) {
  using namespace cbessfm::ssfm;
  g_err.clear();
  if (!info || n < 2 || (n & (n - 1)) || batch < 1)
    return fail(CBESSFM_ERR_INVALID, "n must be a power of two >= 2, batch >= 1");
  if (n > (int64_t(1) << kMaxLog2N)) return fail(CBESSFM_ERR_UNSUPPORTED, "n above 2^22");
  int sms = 148;
  if (device >= 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const size_t esz = dtype == CBESSFM_C64 ? 8 : 16;
  const Geo g = geometry(n, batch, esz, 2 * sms);
  info->n1 = g.n1;
  info->n2 = g.n2;
  info->rows_per_tile = g.rows;
  info->cols_per_tile = g.cols;
  info->threads = kThreads;
  info->smem_bytes = (int64_t)g.smem;
  info->grid = 0;
  return CBESSFM_OK;
}

cbessfm_status cbessfm_ssfm_run(const cbessfm_ssfm_desc* d, void* data, const void* noise,
                                void* stream) {
  using namespace cbessfm::ssfm;
  g_err.clear();
  if (!d || !data) return fail(CBESSFM_ERR_INVALID, "null desc or data");
  if (d->dtype != CBESSFM_C64 && d->dtype != CBESSFM_C128)
    return fail(CBESSFM_ERR_INVALID, "bad dtype");
  if (d->n < 2 || (d->n & (d->n - 1)))
    return fail(CBESSFM_ERR_UNSUPPORTED, "the GPU propagator needs a power-of-two length");
  if (d->n > (int64_t(1) << kMaxLog2N)) return fail(CBESSFM_ERR_UNSUPPORTED, "n above 2^22");
  if (d->batch < 1 || d->n_spans < 0 || d->steps_per_span < 1 || d->n_tables < 1 || !d->half ||
      !d->step_table || !d->nl_coef)
    return fail(CBESSFM_ERR_INVALID, "bad propagation description");
  for (int s = 0; s < d->steps_per_span; ++s)
    if (d->step_table[s] < 0 || d->step_table[s] >= d->n_tables)
      return fail(CBESSFM_ERR_INVALID, "step table index out of range");
  if (noise && d->backward) return fail(CBESSFM_ERR_INVALID, "ASE only on forward spans");
  if (d->n_spans == 0) return CBESSFM_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return d->dtype == CBESSFM_C64 ? run<float>(d, data, noise, st) : run<double>(d, data, noise, st);
}

const char* cbessfm_ssfm_last_error(void) { return cbessfm::ssfm::g_err.c_str(); }

}  // extern "C"
