// C ABI of the CB-ESSFM hot path (include/cbessfm.h): plan creation
// (coefficient and filter upload), kernel dispatch over (dtype, P, Q), and
// error reporting. No torch types cross this boundary.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <tuple>
#include <new>
#include <string>
#include <vector>

#include "../../include/cbessfm.h"
#include "cbessfm_launch.cuh"

namespace cbessfm {
size_t wide_workspace_bytes(int real_bytes, int N, int64_t nclusters);
cudaError_t wide_run_float(const Params<float>& prm, int P, int Q, int64_t nclusters,
                           cudaStream_t st, void* ws, size_t ws_bytes);
cudaError_t wide_run_double(const Params<double>& prm, int P, int Q, int64_t nclusters,
                            cudaStream_t st, void* ws, size_t ws_bytes);
}  // namespace cbessfm

namespace {

thread_local std::string g_err;

cbessfm_status fail(cbessfm_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

cbessfm_status cuda_fail(cudaError_t e, const char* what) {
  return fail(CBESSFM_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

constexpr int kMaxP = 9;

// largest N' of the fused one-block kernels; wider subbands (up to
// kMaxWideQ) run the wide path (csrc/cbessfm_wide.cu)
int max_q(int dtype) { return dtype == CBESSFM_C64 ? 8192 : 4096; }
constexpr int kMaxWideQ = 65536;
bool is_wide(const cbessfm_plan* p);

// exp(-2 pi i m / n), m in [0, n), evaluated in long double and rounded once.
std::vector<double> twiddles(int64_t n) {
  std::vector<double> t(2 * n);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int64_t m = 0; m < n; ++m) {
    const long double a = -2.0L * pi * (long double)m / (long double)n;
    t[2 * m] = (double)cosl(a);
    t[2 * m + 1] = (double)sinl(a);
  }
  if (n % 4 == 0) {  // exact values on the axes
    const double c[4] = {1.0, 0.0, -1.0, 0.0}, sn[4] = {0.0, -1.0, 0.0, 1.0};
    for (int q = 0; q < 4; ++q) {
      t[2 * (q * n / 4)] = c[q];
      t[2 * (q * n / 4) + 1] = sn[q];
    }
  }
  return t;
}

// Per-pass twiddles of the length-Q and length-Q/2 Stockham FFTs in the
// layout cbessfm_kernel.cuh reads (twp_base / twp_offset / tw_plane_index):
// entry (k, r) of the pass with sub-transform size ns is W_Q^(r*k*Q/(ns*R)).
std::vector<double> pass_tables(int Q, const std::vector<double>& tq, int real_bytes) {
  using namespace cbessfm;
  std::vector<double> out(2 * (size_t)twp_total(Q), 0.0);
  auto fill = [&](int L, int sched) {
    const size_t base = twp_base(Q, sched);
    for (int ns = 1; ns < L; ns *= sched_radix(L, ns, sched)) {
      const int R = sched_radix(L, ns, sched);
      if (ns == 1) continue;
      const size_t off = base + twp_offset(L, ns, sched);
      for (int k = 0; k < ns; ++k)
        for (int r = 1; r < R; ++r) {
          const int64_t e = ((int64_t)r * k * (Q / (ns * R))) % Q;
          const size_t at = off + (size_t)tw_plane_index(real_bytes, ns, k, r);
          out[2 * at] = tq[2 * e];
          out[2 * at + 1] = tq[2 * e + 1];
        }
    }
  };
  fill(Q, kTail);
  fill(Q, kHead);
  fill(Q, kMid);
  fill(Q / 2, kHalf);
  fill(Q / 2, kHalf | kWide);  // one-block-per-CTA kernel
  return out;
}

}  // namespace

struct cbessfm_plan {
  int dtype, P, Q, N, overlap, n_steps, n_phasors, n_sets, device;
  void* phasor = nullptr;  // [n_phasors][P][Q]
  void* phasor_rev = nullptr;  // the same rows in cbessfm_ip_kernel's bin order (c128, Q = 2048)
  int* ph_index = nullptr; // [n_steps + 1]
  void* mimo = nullptr;    // [P][Q/2+1]
  void* theta = nullptr;   // [n_sets][n_steps]
  void* twQ = nullptr;     // [Q]
  void* twN = nullptr;     // [P*Q]
  void* twp = nullptr;     // per-pass twiddle rows
  void* rot_tab = nullptr; // complex128: exp(i k / kRotDen), k = -kRotTab/2 .. kRotTab/2 - 1
  long long* dbg = nullptr;  // phase clocks (CB_PHASE_PROFILE builds)
  // block counters of persistent cluster-kernel launches: each launch takes
  // the next slot of the ring (zeroed on its stream), so launches in flight
  // on different streams do not share one
  static constexpr int kWorkSlots = 64;
  unsigned long long* work = nullptr;
  mutable std::atomic<unsigned> work_next{0};
  // host-buffer pipeline (cbessfm_run_host): streams created on first use
  std::mutex host_mu;
  std::vector<cudaStream_t> host_streams;  // [0] copy in, [1] copy out, [2..] compute
  // device staging of cbessfm_run_host: a ring of slots reused across calls
  // (each waits for its previous user's D2H), so calls with several steps
  // in flight neither allocate per call nor pick up the stream-ordered
  // allocator's cross-stream reuse dependencies
  struct HostSlot {
    void* din = nullptr;
    void* dout = nullptr;
    size_t bytes = 0;
    cudaEvent_t done = nullptr;
  };
  static constexpr int kHostSlots = 4;
  HostSlot host_slots[kHostSlots];
  int host_next = 0;
  // cbessfm_run_dualpol: page-locked staging (in, out: [2][n] of the plan's
  // dtype) and the host copy threads, created on first use
  std::vector<cudaEvent_t> host_events;  // run_dualpol's D2H events, destroyed after sync
  void* pin_in = nullptr;
  void* pin_out = nullptr;
  size_t pin_bytes = 0;
  struct Pool* pool = nullptr;
  // wide-subband path workspace (csrc/cbessfm_wide.cu), kept across calls;
  // calls on different streams take turns (wide_done orders them)
  std::mutex wide_mu;
  void* wide_ws = nullptr;
  size_t wide_bytes = 0;
  cudaEvent_t wide_done = nullptr;
};

// Host worker threads for cbessfm_run_dualpol's staging copies (FIFO task
// queue; a call submits its chunk copies in pipeline order and waits on
// per-task completion flags).
struct Pool {
  std::vector<std::thread> workers;
  std::deque<std::function<void()>> q;
  std::mutex mu;
  std::condition_variable cv;
  bool stop = false;
  explicit Pool(int n) {
    for (int i = 0; i < n; ++i)
      workers.emplace_back([this] {
        for (;;) {
          std::function<void()> task;
          {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [this] { return stop || !q.empty(); });
            if (stop && q.empty()) return;
            task = std::move(q.front());
            q.pop_front();
          }
          task();
        }
      });
  }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu);
      q.push_back(std::move(f));
    }
    cv.notify_one();
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& t : workers) t.join();
  }
};

namespace {

constexpr int kDbgSlots = 256 + 3 * 4096;  // phase clocks + per-cluster timeline

// Round a complex double of (near-)unit modulus, scaled by an exact power of
// two, to a float pair. Among the +-1 ulp neighbours of the nearest pair we
// keep the one whose modulus is closest to the exact one: twiddles and
// dispersion phasors are applied to the same bins every step, so a
// modulus error would act as a per-bin gain that accumulates coherently
// over the steps (measured: 1.8e-5 rel L2 after 50 steps with plain
// rounding), while their phase errors cancel between FFT and IFFT.
void round_unit(double re, double im, float* ore, float* oim) {
  const double mod = std::sqrt(re * re + im * im);
  if (!(mod > 0) || !std::isfinite(mod)) {
    *ore = (float)re;
    *oim = (float)im;
    return;
  }
  const int e = std::ilogb(mod);  // unit-modulus form: scale by 2^-e exactly
  const double ur = std::ldexp(re, -e), ui = std::ldexp(im, -e);
  const double target = std::ldexp(mod, -e);
  const double t2 = target * target;
  const float fr = (float)ur, fi = (float)ui;
  float best_r = fr, best_i = fi;
  double best = 1e300;
  for (int a = -1; a <= 1; ++a) {
    float cr = fr;
    if (a < 0) cr = std::nextafter(fr, -INFINITY);
    if (a > 0) cr = std::nextafter(fr, INFINITY);
    for (int b = -1; b <= 1; ++b) {
      float ci = fi;
      if (b < 0) ci = std::nextafter(fi, -INFINITY);
      if (b > 0) ci = std::nextafter(fi, INFINITY);
      const double m2 = (double)cr * cr + (double)ci * ci;
      // phase error as the cross product (sin of the angle, ~1e-7 here)
      const double ang = std::fabs((double)ci * ur - (double)cr * ui) / target;
      const double score = std::fabs(m2 - t2) + 1e-3 * ang;
      if (score < best) {
        best = score;
        best_r = cr;
        best_i = ci;
      }
    }
  }
  *ore = std::ldexp(best_r, e);
  *oim = std::ldexp(best_i, e);
}

template <typename R>
cudaError_t upload_complex(const double* host, size_t count, void** dev, bool unit = false) {
  const size_t bytes = count * 2 * sizeof(R);
  cudaError_t e = cudaMalloc(dev, bytes ? bytes : sizeof(R) * 2);
  if (e != cudaSuccess) return e;
  if (!count) return cudaMemset(*dev, 0, sizeof(R) * 2);
  if (sizeof(R) == sizeof(double)) return cudaMemcpy(*dev, host, bytes, cudaMemcpyHostToDevice);
  std::vector<float> tmp(2 * count);
  for (size_t i = 0; i < count; ++i) {
    if (unit)
      round_unit(host[2 * i], host[2 * i + 1], &tmp[2 * i], &tmp[2 * i + 1]);
    else {
      tmp[2 * i] = (float)host[2 * i];
      tmp[2 * i + 1] = (float)host[2 * i + 1];
    }
  }
  return cudaMemcpy(*dev, tmp.data(), bytes, cudaMemcpyHostToDevice);
}

template <typename R>
cudaError_t upload_real(const double* host, size_t count, void** dev) {
  const size_t bytes = count * sizeof(R);
  cudaError_t e = cudaMalloc(dev, bytes ? bytes : sizeof(R));
  if (e != cudaSuccess || !count) return e;
  if (sizeof(R) == sizeof(double)) return cudaMemcpy(*dev, host, bytes, cudaMemcpyHostToDevice);
  std::vector<float> tmp(count);
  for (size_t i = 0; i < count; ++i) tmp[i] = (float)host[i];
  return cudaMemcpy(*dev, tmp.data(), bytes, cudaMemcpyHostToDevice);
}

// Overwrite the coefficient-set tables (MIMO spectra, theta scales) of an
// existing plan in place; same rounding as upload_complex / upload_real.
template <typename R>
cudaError_t rewrite_sets(cbessfm_plan* p, const double* mimo, const double* theta,
                         cudaStream_t st) {
  const size_t H1 = (size_t)p->Q / 2 + 1;
  const size_t nm = (size_t)p->n_sets * p->P * H1, nt = (size_t)p->n_sets * p->n_steps;
  std::vector<R> m(2 * nm), t(nt);
  for (size_t i = 0; i < 2 * nm; ++i) m[i] = (R)mimo[i];
  for (size_t i = 0; i < nt; ++i) t[i] = (R)theta[i];
  cudaError_t e = cudaMemcpyAsync(p->mimo, m.data(), m.size() * sizeof(R), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && nt)
    e = cudaMemcpyAsync(p->theta, t.data(), t.size() * sizeof(R), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the staging vectors die here
  return e;
}

template <typename R>
cbessfm_status upload_all(cbessfm_plan* p, const cbessfm_desc* d) {
  const size_t PQ = (size_t)p->P * p->Q;
  const size_t H1 = (size_t)p->Q / 2 + 1;
  cudaError_t e;
  if ((e = upload_complex<R>(d->phasors, (size_t)p->n_phasors * PQ, &p->phasor, true)) != cudaSuccess)
    return cuda_fail(e, "upload phasors");
  if (sizeof(R) == 8 && p->Q == cbessfm::kIpQ && p->P >= 2) {
    // permuted copy for the in-place-pass kernel: row (tab, subband), entry
    // ip_rev_index(s, m0, m1) = natural bin s + 16 m0 + 128 m1
    std::vector<double> rev(2 * (size_t)p->n_phasors * PQ);
    for (size_t row = 0; row < (size_t)p->n_phasors * p->P; ++row)
      for (int k = 0; k < p->Q; ++k) {
        const size_t dst = row * p->Q + cbessfm::ip_rev_index(k & 15, (k >> 4) & 7, k >> 7);
        rev[2 * dst] = d->phasors[2 * (row * p->Q + k)];
        rev[2 * dst + 1] = d->phasors[2 * (row * p->Q + k) + 1];
      }
    if ((e = upload_complex<R>(rev.data(), (size_t)p->n_phasors * PQ, &p->phasor_rev, true)) !=
        cudaSuccess)
      return cuda_fail(e, "upload permuted phasors");
  }
  if ((e = cudaMalloc((void**)&p->ph_index, sizeof(int) * (p->n_steps + 1))) != cudaSuccess)
    return cuda_fail(e, "alloc phasor index");
  if ((e = cudaMemcpy(p->ph_index, d->phasor_index, sizeof(int) * (p->n_steps + 1),
                      cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "upload phasor index");
  std::vector<double> zeros;
  const double* mimo = d->mimo;
  if (!mimo) {
    zeros.assign(2 * (size_t)p->n_sets * p->P * H1, 0.0);
    mimo = zeros.data();
  }
  if ((e = upload_complex<R>(mimo, (size_t)p->n_sets * p->P * H1, &p->mimo)) != cudaSuccess)
    return cuda_fail(e, "upload MIMO spectra");
  if ((e = upload_real<R>(d->theta_scale, (size_t)p->n_sets * p->n_steps, &p->theta)) !=
      cudaSuccess)
    return cuda_fail(e, "upload theta scales");
  const std::vector<double> tq = twiddles(p->Q), tn = twiddles((int64_t)p->P * p->Q);
  if ((e = upload_complex<R>(tq.data(), (size_t)p->Q, &p->twQ, true)) != cudaSuccess)
    return cuda_fail(e, "upload twiddles");
  if ((e = upload_complex<R>(tn.data(), PQ, &p->twN, true)) != cudaSuccess)
    return cuda_fail(e, "upload outer twiddles");
  // per-pass rows of the fused kernels (the wide path reads W_N only)
  const std::vector<double> tp =
      p->Q <= max_q(p->dtype) ? pass_tables(p->Q, tq, (int)sizeof(R)) : std::vector<double>(2, 0.0);
  if ((e = upload_complex<R>(tp.data(), tp.size() / 2, &p->twp, true)) != cudaSuccess)
    return cuda_fail(e, "upload pass twiddles");
  if (sizeof(R) == sizeof(double)) {
    // rotation table of the complex128 cluster kernel (RotationTabHook)
    std::vector<double> rt(2 * (size_t)cbessfm::kRotTab);
    for (int i = 0; i < cbessfm::kRotTab; ++i) {
      const double a = (double)(i - cbessfm::kRotTab / 2) / cbessfm::kRotDen;
      rt[2 * i] = std::cos(a);
      rt[2 * i + 1] = std::sin(a);
    }
    if ((e = upload_complex<R>(rt.data(), (size_t)cbessfm::kRotTab, &p->rot_tab)) != cudaSuccess)
      return cuda_fail(e, "upload rotation table");
  }
  if ((e = cudaMalloc((void**)&p->work, sizeof(unsigned long long) * cbessfm_plan::kWorkSlots)) !=
      cudaSuccess)
    return cuda_fail(e, "alloc block counters");
#ifdef CB_PHASE_PROFILE
  if ((e = cudaMalloc((void**)&p->dbg, kDbgSlots * sizeof(long long))) != cudaSuccess)
    return cuda_fail(e, "alloc phase clocks");
  cudaMemset(p->dbg, 0, kDbgSlots * sizeof(long long));
#endif
  return CBESSFM_OK;
}

bool is_wide(const cbessfm_plan* p) { return p->Q > max_q(p->dtype); }

void free_plan(cbessfm_plan* p) {
  if (!p) return;
  for (auto& sl : p->host_slots) {
    if (sl.done) cudaEventSynchronize(sl.done);
    cudaFree(sl.din);
    cudaFree(sl.dout);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  for (cudaStream_t st : p->host_streams) cudaStreamDestroy(st);
  if (p->wide_done) {
    cudaEventSynchronize(p->wide_done);
    cudaEventDestroy(p->wide_done);
  }
  cudaFree(p->wide_ws);
  delete p->pool;
  if (p->pin_in) cudaFreeHost(p->pin_in);
  if (p->pin_out) cudaFreeHost(p->pin_out);
  cudaFree(p->phasor);
  cudaFree(p->phasor_rev);
  cudaFree(p->ph_index);
  cudaFree(p->mimo);
  cudaFree(p->theta);
  cudaFree(p->twQ);
  cudaFree(p->twN);
  cudaFree(p->twp);
  cudaFree(p->rot_tab);
  cudaFree(p->dbg);
  cudaFree(p->work);
  delete p;
}

template <typename R>
cudaError_t dispatch(int P, const cbessfm::Params<R>& prm, int q, int64_t nclusters,
                     cudaStream_t st, cbessfm::KernelInfo* info);

#define CB_CASE(T, P) \
  case P: return cbessfm::launch_##T##_##P(prm, q, nclusters, st, info);
template <>
cudaError_t dispatch<float>(int P, const cbessfm::Params<float>& prm, int q, int64_t nclusters,
                            cudaStream_t st, cbessfm::KernelInfo* info) {
  switch (P) {
    CB_CASE(float, 1) CB_CASE(float, 2) CB_CASE(float, 3) CB_CASE(float, 4) CB_CASE(float, 5)
    CB_CASE(float, 6) CB_CASE(float, 7) CB_CASE(float, 8) CB_CASE(float, 9)
    default: return cudaErrorInvalidValue;
  }
}
template <>
cudaError_t dispatch<double>(int P, const cbessfm::Params<double>& prm, int q, int64_t nclusters,
                             cudaStream_t st, cbessfm::KernelInfo* info) {
  switch (P) {
    CB_CASE(double, 1) CB_CASE(double, 2) CB_CASE(double, 3) CB_CASE(double, 4)
    CB_CASE(double, 5) CB_CASE(double, 6) CB_CASE(double, 7) CB_CASE(double, 8)
    CB_CASE(double, 9)
    default: return cudaErrorInvalidValue;
  }
}
#undef CB_CASE

// Every entry point that touches a plan runs on the plan's device and
// restores the caller's current device on return (a process may drive
// several GPUs from one thread).
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// set while cbessfm_run_host issues its pipelined chunk launches
thread_local int g_kernel_pref = 0;

template <typename R>
cbessfm::Params<R> make_params(const cbessfm_plan* p, const cbessfm_io* io) {
  using C = cbessfm::Cx<R>;
  cbessfm::Params<R> prm;
  prm.kernel_pref = g_kernel_pref;
  prm.in = reinterpret_cast<const C*>(io->in);
  prm.out = reinterpret_cast<C*>(io->out);
  prm.in_bstride = io->in_batch_stride;
  prm.in_pstride = io->in_pol_stride;
  prm.in_origin = io->in_origin;
  prm.out_bstride = io->out_batch_stride;
  prm.out_pstride = io->out_pol_stride;
  prm.out_origin = io->out_origin;
  prm.n = io->n;
  prm.b0 = io->block_begin;
  prm.nb = io->block_end - io->block_begin;
  prm.keep = p->N - p->overlap;
  prm.half = p->overlap / 2;
  prm.phasor = reinterpret_cast<const C*>(p->phasor);
  prm.phasor_rev = reinterpret_cast<const C*>(p->phasor_rev);
  prm.ph_index = p->ph_index;
  prm.mimo = reinterpret_cast<const C*>(p->mimo);
  prm.theta_scale = reinterpret_cast<const R*>(p->theta);
  prm.twQ = reinterpret_cast<const C*>(p->twQ);
  prm.twN = reinterpret_cast<const C*>(p->twN);
  prm.twp = reinterpret_cast<const C*>(p->twp);
  prm.rot_tab = reinterpret_cast<const C*>(p->rot_tab);
  prm.n_steps = p->n_steps;
  prm.n_sets = p->n_sets;
  prm.cid0 = 0;
  prm.work = p->work ? p->work + p->work_next.fetch_add(1) % cbessfm_plan::kWorkSlots : nullptr;
  prm.total = 0;
  prm.dbg = p->dbg;
  return prm;
}

}  // namespace

extern "C" {

int32_t cbessfm_version(void) { return CBESSFM_VERSION; }

int64_t cbessfm_num_blocks(int64_t n, int32_t block_size, int32_t overlap) {
  if (n <= 0 || block_size <= 0 || overlap < 0 || overlap >= block_size) return -1;
  const int64_t keep = block_size - overlap;
  return (n + keep - 1) / keep;
}

int32_t cbessfm_supported(int32_t dtype, int32_t n_subbands, int32_t block_size) {
  if (dtype != CBESSFM_C64 && dtype != CBESSFM_C128) return 0;
  if (n_subbands < 1 || n_subbands > kMaxP || block_size % n_subbands) return 0;
  const int q = block_size / n_subbands;
  return is_pow2(q) && q >= 256 && q <= kMaxWideQ;
}

cbessfm_status cbessfm_plan_create(const cbessfm_desc* d, cbessfm_plan** out) {
  g_err.clear();
  if (!d || !out) return fail(CBESSFM_ERR_INVALID, "null descriptor or output pointer");
  *out = nullptr;
  if (d->dtype != CBESSFM_C64 && d->dtype != CBESSFM_C128)
    return fail(CBESSFM_ERR_INVALID, "dtype must be CBESSFM_C64 or CBESSFM_C128");
  if (d->n_subbands < 1) return fail(CBESSFM_ERR_INVALID, "n_subbands must be >= 1");
  if (d->block_size <= d->overlap || d->overlap < 0)
    return fail(CBESSFM_ERR_INVALID, "need block_size > overlap >= 0");
  if (d->block_size % d->n_subbands)
    return fail(CBESSFM_ERR_INVALID, "block_size must divide into n_subbands");
  if (d->overlap % (2 * d->n_subbands))
    return fail(CBESSFM_ERR_INVALID, "overlap must be a multiple of 2*n_subbands");
  if (d->n_steps < 0) return fail(CBESSFM_ERR_INVALID, "n_steps must be >= 0");
  if (d->n_sets < 0) return fail(CBESSFM_ERR_INVALID, "n_sets must be >= 0");
  if (d->n_phasors < 1 || !d->phasors || !d->phasor_index)
    return fail(CBESSFM_ERR_INVALID, "phasor tables missing");
  if (d->n_steps > 0 && !d->theta_scale)
    return fail(CBESSFM_ERR_INVALID, "theta scales missing");
  for (int s = 0; s <= d->n_steps; ++s)
    if (d->phasor_index[s] < 0 || d->phasor_index[s] >= d->n_phasors)
      return fail(CBESSFM_ERR_INVALID, "phasor index out of range");
  if (!cbessfm_supported(d->dtype, d->n_subbands, d->block_size)) {
    char buf[256];
    snprintf(buf, sizeof buf,
             "unsupported shape for the sm_100a kernel: n_subbands=%d (1..%d), "
             "N'=block_size/n_subbands=%d (power of two in [256, %d])",
             d->n_subbands, kMaxP, d->block_size / d->n_subbands, kMaxWideQ);
    return fail(CBESSFM_ERR_UNSUPPORTED, buf);
  }
  cbessfm_plan* p = new (std::nothrow) cbessfm_plan;
  if (!p) return fail(CBESSFM_ERR_INVALID, "out of host memory");
  p->dtype = d->dtype;
  p->P = d->n_subbands;
  p->Q = d->block_size / d->n_subbands;
  p->N = d->block_size;
  p->overlap = d->overlap;
  p->n_steps = d->n_steps;
  p->n_phasors = d->n_phasors;
  p->n_sets = d->n_sets > 1 ? d->n_sets : 1;
  p->device = d->device;
  DeviceGuard dg(d->device);
  if (dg.err != cudaSuccess) {
    delete p;
    return cuda_fail(dg.err, "cudaSetDevice");
  }
  const cbessfm_status st =
      p->dtype == CBESSFM_C64 ? upload_all<float>(p, d) : upload_all<double>(p, d);
  if (st != CBESSFM_OK) {
    free_plan(p);
    return st;
  }
  *out = p;
  return CBESSFM_OK;
}

cbessfm_status cbessfm_plan_info_get(const cbessfm_plan* p, cbessfm_plan_info* info) {
  g_err.clear();
  if (!p || !info) return fail(CBESSFM_ERR_INVALID, "null plan or info");
  DeviceGuard dg(p->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  cbessfm::KernelInfo ki{};
  cudaError_t e;
  if (is_wide(p)) {
    info->threads_per_cta = 256;
    info->cluster_size = 1;
    info->smem_per_cta = 0;
    info->max_active_clusters = 0;
    info->q = p->Q;
    snprintf(info->kernel, sizeof info->kernel, "%s",
             "cbessfm_wide (Stockham passes, device workspace)");
    return CBESSFM_OK;
  }
  if (p->dtype == CBESSFM_C64) {
    cbessfm::Params<float> prm{};
    e = dispatch<float>(p->P, prm, p->Q, 0, nullptr, &ki);
  } else {
    cbessfm::Params<double> prm{};
    prm.phasor_rev = reinterpret_cast<const cbessfm::Cx<double>*>(p->phasor_rev);
    e = dispatch<double>(p->P, prm, p->Q, 0, nullptr, &ki);
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel occupancy query");
  info->threads_per_cta = ki.threads;
  info->cluster_size = ki.cluster;
  info->smem_per_cta = (int64_t)ki.smem;
  info->max_active_clusters = ki.max_active_clusters;
  info->q = p->Q;
  snprintf(info->kernel, sizeof info->kernel, "%s", ki.name);
  return CBESSFM_OK;
}

cbessfm_status cbessfm_run(const cbessfm_plan* p, const cbessfm_io* io, void* stream) {
  g_err.clear();
  if (!p || !io) return fail(CBESSFM_ERR_INVALID, "null plan or io");
  if (!io->in || !io->out) return fail(CBESSFM_ERR_INVALID, "null input or output buffer");
  if (io->n < p->N) return fail(CBESSFM_ERR_INVALID, "block_size exceeds the sequence length");
  if (io->batch < 0) return fail(CBESSFM_ERR_INVALID, "negative batch");
  const int64_t nblk = cbessfm_num_blocks(io->n, p->N, p->overlap);
  if (io->block_begin < 0 || io->block_end > nblk || io->block_begin > io->block_end)
    return fail(CBESSFM_ERR_INVALID, "block range outside [0, n_blocks]");
  if (io->in_origin < 0 || io->in_origin >= io->n || io->out_origin < 0)
    return fail(CBESSFM_ERR_INVALID, "origins out of range");
  const int64_t nclusters = io->batch * (io->block_end - io->block_begin);
  if (nclusters == 0) return CBESSFM_OK;
  DeviceGuard dg(p->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (is_wide(p)) {
    cbessfm_plan* wp = const_cast<cbessfm_plan*>(p);  // only the workspace is touched
    std::lock_guard<std::mutex> lk(wp->wide_mu);
    const size_t need =
        cbessfm::wide_workspace_bytes(p->dtype == CBESSFM_C64 ? 4 : 8, p->N, nclusters);
    if (!wp->wide_done &&
        (e = cudaEventCreateWithFlags(&wp->wide_done, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "event create");
    if (wp->wide_bytes < need) {
      cudaEventSynchronize(wp->wide_done);  // its last user has finished
      cudaFree(wp->wide_ws);
      wp->wide_ws = nullptr;
      wp->wide_bytes = 0;
      if ((e = cudaMalloc(&wp->wide_ws, need)) != cudaSuccess) return cuda_fail(e, "wide workspace");
      wp->wide_bytes = need;
    }
    cudaStreamWaitEvent(st, wp->wide_done, 0);
    if (p->dtype == CBESSFM_C64)
      e = cbessfm::wide_run_float(make_params<float>(p, io), p->P, p->Q, nclusters, st,
                                  wp->wide_ws, wp->wide_bytes);
    else
      e = cbessfm::wide_run_double(make_params<double>(p, io), p->P, p->Q, nclusters, st,
                                   wp->wide_ws, wp->wide_bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cbessfm wide-path launch");
    if ((e = cudaEventRecord(wp->wide_done, st)) != cudaSuccess) return cuda_fail(e, "event record");
    return CBESSFM_OK;
  }
  if (p->dtype == CBESSFM_C64)
    e = dispatch<float>(p->P, make_params<float>(p, io), p->Q, nclusters, st, nullptr);
  else
    e = dispatch<double>(p->P, make_params<double>(p, io), p->Q, nclusters, st, nullptr);
  if (e != cudaSuccess) return cuda_fail(e, "cbessfm kernel launch");
  return CBESSFM_OK;
}

}  // extern "C"

namespace {

// The pipelined host-buffer schedule shared by cbessfm_run_host and
// cbessfm_run_dualpol: `in` / `out` page-locked [batch][2][n] of the plan's
// dtype. before_h2d(a, b) runs on the calling thread before samples [a, b)
// of every row are copied in (run_dualpol waits there for its staging
// copies); after_d2h(o0, o1, ev) after the D2H of kept samples [o0, o1) has
// been enqueued, ev completing with it. Caller holds p->host_mu.
cbessfm_status host_pipeline(cbessfm_plan* p, const void* in, void* out, int64_t n,
                             int64_t batch, int chunks_req, cudaStream_t st,
                             const std::function<void(int64_t, int64_t)>& before_h2d,
                             const std::function<void(int64_t, int64_t, cudaEvent_t)>& after_d2h) {
  const int64_t keep = p->N - p->overlap, half = p->overlap / 2;
  const int64_t nb = cbessfm_num_blocks(n, p->N, p->overlap);
  const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(chunks_req > 0 ? chunks_req : 8, nb));
  const size_t esz = p->dtype == CBESSFM_C64 ? 8 : 16;
  const size_t rowb = (size_t)n * esz, rows = (size_t)batch * 2;
  cudaError_t e;
  while ((int)p->host_streams.size() < 2 + chunks) {
    cudaStream_t s2;
    if ((e = cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "stream create");
    p->host_streams.push_back(s2);
  }
  cudaStream_t s_in = p->host_streams[0], s_out = p->host_streams[1];
  cbessfm_plan::HostSlot& slot = p->host_slots[p->host_next];
  p->host_next = (p->host_next + 1) % cbessfm_plan::kHostSlots;
  if (!slot.done) {
    if ((e = cudaEventCreateWithFlags(&slot.done, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "event create");
  } else {
    cudaStreamWaitEvent(st, slot.done, 0);  // its previous call's D2H has finished
  }
  if (slot.bytes < rows * rowb) {
    // grow the slot (rare: first call or a longer waveform). Plain
    // cudaMalloc/cudaFree: the slot outlives the call, and the device's
    // default stream-ordered pool is left alone
    if (slot.done) cudaEventSynchronize(slot.done);
    cudaFree(slot.din);
    cudaFree(slot.dout);
    slot.din = slot.dout = nullptr;
    slot.bytes = 0;
    if ((e = cudaMalloc(&slot.din, rows * rowb)) != cudaSuccess) return cuda_fail(e, "alloc in");
    if ((e = cudaMalloc(&slot.dout, rows * rowb)) != cudaSuccess) {
      cudaFree(slot.din);
      slot.din = nullptr;
      return cuda_fail(e, "alloc out");
    }
    slot.bytes = rows * rowb;
  }
  void *din = slot.din, *dout = slot.dout;
  std::vector<cudaEvent_t> evs;
  auto event = [&](cudaStream_t s2) {
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, s2);
    evs.push_back(ev);
    return ev;
  };
  cudaEvent_t ev0 = event(st);
  for (int i = 0; i < 2 + chunks; ++i) cudaStreamWaitEvent(p->host_streams[i], ev0, 0);
  // column ranges [a, b) of every (waveform, polarisation) row in one call
  auto h2d = [&](int64_t a, int64_t b) {
    if (before_h2d) before_h2d(a, b);
    return cudaMemcpy2DAsync((char*)din + a * esz, rowb, (const char*)in + a * esz, rowb,
                             (size_t)(b - a) * esz, rows, cudaMemcpyHostToDevice, s_in);
  };
  auto d2h = [&](int64_t a, int64_t b) {
    const cudaError_t r = cudaMemcpy2DAsync((char*)out + a * esz, rowb, (const char*)dout + a * esz,
                                            rowb, (size_t)(b - a) * esz, rows,
                                            cudaMemcpyDeviceToHost, s_out);
    if (r == cudaSuccess && after_d2h) after_d2h(a, b, event(s_out));
    return r;
  };
  // wrap piece first, then `chunks` sample ranges; blocks whose windows end
  // inside the copied prefix run as soon as it lands, the last chunk takes
  // the remaining blocks
  auto enqueue = [&]() -> cbessfm_status {
    const int64_t wrap = half > 0 ? n - half : n;
    if (half > 0 && (e = h2d(wrap, n)) != cudaSuccess) return cuda_fail(e, "h2d");
    int64_t b_prev = 0, lo = 0;
    for (int c = 1; c <= chunks; ++c) {
      const int64_t hi = c == chunks ? n : (n * c) / chunks;
      int64_t b1 = c == chunks ? nb : (hi + half - p->N >= 0 ? (hi + half - p->N) / keep + 1 : 0);
      b1 = std::max(b_prev, std::min(b1, nb));
      if (std::min(hi, wrap) > lo && (e = h2d(lo, std::min(hi, wrap))) != cudaSuccess)
        return cuda_fail(e, "h2d");
      cudaEvent_t ev_in = event(s_in);
      if (b1 > b_prev) {
        cudaStream_t sk = p->host_streams[1 + c];
        cudaStreamWaitEvent(sk, ev_in, 0);
        cbessfm_io dio{din, 2 * n, n, 0, dout, 2 * n, n, 0, n, batch, b_prev, b1};
        const cbessfm_status r = cbessfm_run(p, &dio, sk);
        if (r != CBESSFM_OK) return r;
        cudaEvent_t ev_k = event(sk);
        cudaStreamWaitEvent(s_out, ev_k, 0);
        const int64_t o0 = b_prev * keep, o1 = std::min(b1 * keep, n);
        if ((e = d2h(o0, o1)) != cudaSuccess) return cuda_fail(e, "d2h");
      }
      b_prev = b1;
      lo = hi;
    }
    return CBESSFM_OK;
  };
  g_kernel_pref = 1;  // chunks of several steps in flight: cluster kernel
  const cbessfm_status status = enqueue();
  g_kernel_pref = 0;
  // join every pipeline stream into the caller's stream (also after an
  // error); the staging slot is reusable once that point is reached
  for (int i = 0; i < 2 + chunks; ++i) cudaStreamWaitEvent(st, event(p->host_streams[i]), 0);
  cudaEventRecord(slot.done, st);  // the slot is free once this call completes
  if (!after_d2h)
    for (cudaEvent_t ev : evs) cudaEventDestroy(ev);  // released once complete
  else
    for (cudaEvent_t ev : evs) p->host_events.push_back(ev);  // the caller syncs first
  if (status != CBESSFM_OK) return status;
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "cbessfm_run_host");
  return CBESSFM_OK;
}

// c128 -> plan dtype copy of samples [a, b) of one polarisation row
// Staging copy of samples [a, b) of one polarisation into the page-locked
// row (cast to float for c64). Returns false if any component is NaN or
// infinite: the copy reads every sample anyway, so the reference's
// require_finite check (dbp.py:449) rides along at no extra memory pass.
bool stage_in(const cbessfm_plan* p, const double* src, void* row, int64_t a, int64_t b) {
  constexpr uint64_t kExp = 0x7ff0000000000000ull;
  uint64_t bad = 0;
  if (p->dtype == CBESSFM_C128) {
    const uint64_t* s = reinterpret_cast<const uint64_t*>(src);
    uint64_t* d = reinterpret_cast<uint64_t*>(row);
    for (int64_t i = 2 * a; i < 2 * b; ++i) {
      const uint64_t v = s[i];
      d[i] = v;
      bad |= (uint64_t)((v & kExp) == kExp);
    }
  } else {
    const uint64_t* s = reinterpret_cast<const uint64_t*>(src);
    float* d = (float*)row;
    for (int64_t i = 2 * a; i < 2 * b; ++i) {
      d[i] = (float)src[i];
      bad |= (uint64_t)((s[i] & kExp) == kExp);
    }
  }
  return bad == 0;
}
void stage_out(const cbessfm_plan* p, const void* row, double* dst, int64_t a, int64_t b) {
  if (p->dtype == CBESSFM_C128) {
    memcpy(dst + 2 * a, (const double*)row + 2 * a, (size_t)(b - a) * 16);
  } else {
    const float* s = (const float*)row;
    for (int64_t i = 2 * a; i < 2 * b; ++i) dst[i] = (double)s[i];
  }
}

}  // namespace

extern "C" {

cbessfm_status cbessfm_run_host(const cbessfm_plan* cp, const cbessfm_host_io* io, void* stream) {
  g_err.clear();
  if (!cp || !io) return fail(CBESSFM_ERR_INVALID, "null plan or io");
  if (!io->in || !io->out) return fail(CBESSFM_ERR_INVALID, "null input or output buffer");
  if (io->n < cp->N) return fail(CBESSFM_ERR_INVALID, "block_size exceeds the sequence length");
  if (io->batch <= 0) return fail(CBESSFM_ERR_INVALID, "batch must be positive");
  cbessfm_plan* p = const_cast<cbessfm_plan*>(cp);  // only the stream pool is touched
  std::lock_guard<std::mutex> lock(p->host_mu);
  DeviceGuard dg(p->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  return host_pipeline(p, io->in, io->out, io->n, io->batch, io->chunks,
                       reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr);
}

cbessfm_status cbessfm_run_dualpol(const cbessfm_plan* cp, const cbessfm_dualpol_io* io,
                                   void* stream) {
  g_err.clear();
  if (!cp || !io) return fail(CBESSFM_ERR_INVALID, "null plan or io");
  if (!io->in_x || !io->in_y || !io->out_x || !io->out_y)
    return fail(CBESSFM_ERR_INVALID, "null input or output buffer");
  if (io->n < cp->N) return fail(CBESSFM_ERR_INVALID, "block_size exceeds the sequence length");
  cbessfm_plan* p = const_cast<cbessfm_plan*>(cp);
  std::lock_guard<std::mutex> lock(p->host_mu);
  DeviceGuard dg(p->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  const int64_t n = io->n;
  const size_t esz = p->dtype == CBESSFM_C64 ? 8 : 16;
  const size_t bytes = 2 * (size_t)n * esz;
  cudaError_t e;
  if (p->pin_bytes < bytes) {
    if (p->pin_in) cudaFreeHost(p->pin_in);
    if (p->pin_out) cudaFreeHost(p->pin_out);
    p->pin_in = p->pin_out = nullptr;
    p->pin_bytes = 0;
    if ((e = cudaHostAlloc(&p->pin_in, bytes, cudaHostAllocPortable)) != cudaSuccess)
      return cuda_fail(e, "pinned staging");
    if ((e = cudaHostAlloc(&p->pin_out, bytes, cudaHostAllocPortable)) != cudaSuccess)
      return cuda_fail(e, "pinned staging");
    p->pin_bytes = bytes;
  }
  if (!p->pool) {
    const int hw = (int)std::thread::hardware_concurrency();
    int nt = io->host_threads > 0 ? io->host_threads : std::min(8, std::max(1, hw));
    p->pool = new Pool(nt);
  }
  char* rin = (char*)p->pin_in;
  char* rout = (char*)p->pin_out;
  const size_t rowb = (size_t)n * esz;
  // staging copies in pieces, the wrap piece (the tail block 0 reads) first,
  // then ascending; before each H2D the pipeline waits for its pieces
  const int64_t half = p->overlap / 2;
  const int64_t piece = std::max<int64_t>(4096, (n + 63) / 64);
  std::vector<std::pair<int64_t, int64_t>> ranges;
  const int64_t wrap = half > 0 ? n - half : n;
  if (half > 0) ranges.push_back({wrap, n});
  for (int64_t a = 0; a < wrap; a += piece) ranges.push_back({a, std::min(wrap, a + piece)});
  std::vector<std::atomic<int>> done(ranges.size());
  for (auto& d : done) d.store(0);
  std::atomic<int> nonfinite{0};
  std::mutex wmu;
  std::condition_variable wcv;
  for (size_t t = 0; t < ranges.size(); ++t) {
    p->pool->submit([&, t] {
      const bool okx = stage_in(p, io->in_x, rin, ranges[t].first, ranges[t].second);
      const bool oky = stage_in(p, io->in_y, rin + rowb, ranges[t].first, ranges[t].second);
      if (!(okx && oky)) nonfinite.store(1);
      {
        std::lock_guard<std::mutex> lk(wmu);
        done[t].store(1);
      }
      wcv.notify_all();
    });
  }
  auto before_h2d = [&](int64_t a, int64_t b) {
    std::unique_lock<std::mutex> lk(wmu);
    wcv.wait(lk, [&] {
      for (size_t t = 0; t < ranges.size(); ++t)
        if (ranges[t].first < b && ranges[t].second > a && !done[t].load()) return false;
      return true;
    });
  };
  std::vector<std::tuple<int64_t, int64_t, cudaEvent_t>> outs;
  auto after_d2h = [&](int64_t a, int64_t b, cudaEvent_t ev) { outs.emplace_back(a, b, ev); };
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const cbessfm_status status =
      host_pipeline(p, rin, rout, n, 1, io->chunks, st, before_h2d, after_d2h);
  // drain the copy-in tasks even on error (they reference this frame)
  before_h2d(0, n);
  if (status != CBESSFM_OK) {
    cudaStreamSynchronize(st);
    for (cudaEvent_t ev : p->host_events) cudaEventDestroy(ev);
    p->host_events.clear();
    return status;
  }
  // copy the kept samples out as their D2H pieces complete
  e = cudaSuccess;
  std::atomic<int> pending{0};
  for (auto& o : outs) {
    const int64_t a = std::get<0>(o), b = std::get<1>(o);
    if ((e = cudaEventSynchronize(std::get<2>(o))) != cudaSuccess) break;
    for (int64_t x0 = a; x0 < b; x0 += piece) {
      const int64_t x1 = std::min(b, x0 + piece);
      pending.fetch_add(1);
      p->pool->submit([&, x0, x1] {
        stage_out(p, rout, io->out_x, x0, x1);
        stage_out(p, rout + rowb, io->out_y, x0, x1);
        {
          std::lock_guard<std::mutex> lk(wmu);
          pending.fetch_sub(1);
        }
        wcv.notify_all();
      });
    }
  }
  {
    std::unique_lock<std::mutex> lk(wmu);
    wcv.wait(lk, [&] { return pending.load() == 0; });
  }
  const cudaError_t e2 = cudaStreamSynchronize(st);
  for (cudaEvent_t ev : p->host_events) cudaEventDestroy(ev);
  p->host_events.clear();
  if (e != cudaSuccess) return cuda_fail(e, "cbessfm_run_dualpol d2h");
  if (e2 != cudaSuccess) return cuda_fail(e2, "cbessfm_run_dualpol");
  if (nonfinite.load())  // the outputs are left undefined, as after any error
    return fail(CBESSFM_ERR_INVALID, "waveform contains non-finite samples");
  return CBESSFM_OK;
}

cbessfm_status cbessfm_plan_update_sets(cbessfm_plan* p, int32_t n_sets, const double* mimo,
                                        const double* theta_scale, void* stream) {
  g_err.clear();
  if (!p || !mimo || (p->n_steps > 0 && !theta_scale))
    return fail(CBESSFM_ERR_INVALID, "null plan or tables");
  if (p->n_steps == 0) return fail(CBESSFM_ERR_INVALID, "plan has no nonlinear steps");
  if (n_sets != p->n_sets) {
    char buf[128];
    snprintf(buf, sizeof buf, "plan holds %d coefficient sets, %d given", p->n_sets, (int)n_sets);
    return fail(CBESSFM_ERR_INVALID, buf);
  }
  DeviceGuard dg(p->device);
  if (dg.err != cudaSuccess) return cuda_fail(dg.err, "cudaSetDevice");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const cudaError_t e = p->dtype == CBESSFM_C64 ? rewrite_sets<float>(p, mimo, theta_scale, st)
                                                : rewrite_sets<double>(p, mimo, theta_scale, st);
  return e == cudaSuccess ? CBESSFM_OK : cuda_fail(e, "update coefficient sets");
}

cbessfm_status cbessfm_plan_destroy(cbessfm_plan* p) {
  g_err.clear();
  if (!p) return CBESSFM_OK;
  DeviceGuard dg(p->device);
  free_plan(p);
  return CBESSFM_OK;
}

const char* cbessfm_last_error(void) { return g_err.c_str(); }

int32_t cbessfm_debug_phase_times(const cbessfm_plan* p, int64_t* out, int32_t n) {
  if (!p || !out || !p->dbg) return 0;
  if (n > kDbgSlots) n = kDbgSlots;
  DeviceGuard dg(p->device);
  return cudaMemcpy(out, p->dbg, sizeof(long long) * n, cudaMemcpyDeviceToHost) == cudaSuccess
             ? n
             : -1;
}

}  // extern "C"
