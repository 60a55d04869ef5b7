// Fused CB-ESSFM overlap-save block kernel for sm_100a.
//
// One thread-block cluster processes one overlap-save block of one waveform.
// CTA r of a P-CTA cluster (P = n_subbands) owns subband r for both
// polarisations; its fields stay resident in shared memory through every
// step. Cross-subband data movement (the outer N = P*Q transform and the
// per-step MIMO coupling of the intensity spectra) goes over distributed
// shared memory (DSMEM) inside the cluster; nothing round-trips through HBM
// between the block load and the store of the kept samples.
//
// Reference semantics (fiberdbp 0.1.0, /root/reference/pkg/src/fiberdbp):
//   block framing ............ dbp.py:467-477  (circular window, keep/half)
//   outer FFT + subband demux  dbp.py:387-389
//   per-step dispersion ...... dbp.py:395, tables dbp.py:352-359
//   subband IFFT / FFT ....... dbp.py:396, dbp.py:398
//   NLPR (intensity, rfft, MIMO, irfft, rotation) dbp.py:185-208
//   final phasor + merge ..... dbp.py:399-401
//   discard .................. dbp.py:476-477
//
// Scaling conventions (all folded into host-built tables, see planner.py):
//   * phasor tables carry 1/Q (the subband IFFT normalisation);
//   * the forward outer exchange applies 1/P (dbp.py:388 "/ n_sb");
//   * the merge "* n_sb" and the outer IFFT's 1/N combine to 1/Q, which the
//     final phasor table already carries, so the inverse outer transform is
//     an unnormalised sum;
//   * theta_scale[st] = step_scales[st] / reference_power_w / Q (irfft 1/Q).
//
// Per step a CTA runs: subband IFFT (last pass writes the intensity),
// half-length FFT + r2c untangle, DSMEM MIMO, c2r twist + half-length IFFT,
// subband FFT (first pass applies the rotation, last pass the next
// dispersion phasor) -- four shared-memory FFTs and no other full-field
// passes.
#pragma once

#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace cbessfm {

namespace cg = cooperative_groups;

// Checked builds (-DCB_CHECKED, `build.py --variant checked`), the stand-in
// for compute-sanitizer, which this GPU pool does not allow:
//  * CB_POISON_SMEM fills a kernel's dynamic shared memory with a NaN
//    pattern (NaN as one f64 and as two f32) before first use, so a read of
//    a slot no pass wrote -- or read before its writer's barrier, the race
//    racecheck looks for -- reaches the output as NaN or as a bit difference
//    against the unchecked build (tests/test_gpu_checked.py);
//  * CB_CHECK traps on an out-of-range global, shared or cluster index.
#ifdef CB_CHECKED
#define CB_CHECK(cond)                                                               \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      printf("CB_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
             #cond, (int)blockIdx.x, (int)threadIdx.x);                              \
      __trap();                                                                      \
    }                                                                                \
  } while (0)
__device__ __forceinline__ void cb_poison_smem(void* base) {
  uint32_t bytes;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(bytes));
  const uint32_t nt = blockDim.x * blockDim.y * blockDim.z;
  const uint32_t tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  unsigned long long* p = reinterpret_cast<unsigned long long*>(base);
  for (uint32_t i = tid; i < bytes / 8; i += nt) p[i] = 0x7ff8dead7ff8deadull;
  __syncthreads();
}
#define CB_POISON_SMEM(base) cb_poison_smem(base)
#else
#define CB_CHECK(cond) \
  do {                 \
  } while (0)
#define CB_POISON_SMEM(base) \
  do {                       \
  } while (0)
#endif

// Phase timestamps of CTA 0 (debug builds with -DCB_PHASE_PROFILE only;
// read back with cbessfm_debug_phase_times).
#ifdef CB_PHASE_PROFILE
#define CB_MARK(i)                                                                    \
  do {                                                                                \
    if (prm.dbg && blockIdx.x == 0 && threadIdx.x == 0 && (i) < 256) prm.dbg[(i)] = clock64(); \
  } while (0)
// Per-cluster timeline (globaltimer ns at start / end of every cluster's
// rank-0 CTA, and its SM) after the 256 phase slots: [256 + 3 c + {0,1,2}].
#define CB_TIMELINE(slot)                                                              \
  do {                                                                                 \
    if (prm.dbg && (blockIdx.x % P) == 0 && threadIdx.x == 0 && cid < 4096) {          \
      unsigned long long t;                                                            \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));                            \
      prm.dbg[256 + 3 * cid + (slot)] = (long long)t;                                  \
      if ((slot) == 0) {                                                               \
        unsigned sm;                                                                   \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));                                \
        prm.dbg[256 + 3 * cid + 2] = sm;                                               \
      }                                                                                \
    }                                                                                  \
  } while (0)
#else
#define CB_MARK(i) \
  do {             \
  } while (0)
#define CB_TIMELINE(slot) \
  do {                    \
  } while (0)
#endif

template <typename R>
struct alignas(2 * sizeof(R)) Cx {
  R x, y;
};

template <typename R>
__device__ __forceinline__ Cx<R> mk(R a, R b) {
  Cx<R> c;
  c.x = a;
  c.y = b;
  return c;
}
template <typename R>
__device__ __forceinline__ Cx<R> operator+(Cx<R> a, Cx<R> b) {
  return mk(a.x + b.x, a.y + b.y);
}
template <typename R>
__device__ __forceinline__ Cx<R> operator-(Cx<R> a, Cx<R> b) {
  return mk(a.x - b.x, a.y - b.y);
}
// packed float complex products: -15 % FP32 instructions in the fat
// kernel and no change in time (0.3471 -> 0.3460 ms batch 1, 2.496 -> 2.511
// ms batch 8): the kernel is not issue-bound, so it stays an A/B knob
#ifndef CB_CMUL2
#define CB_CMUL2 0
#endif
// float complex add/sub as one packed FADD2 (sm_100 f32x2): same IEEE
// results as the two scalar adds, half the issue slots
#ifndef CB_NO_FADD2
__device__ __forceinline__ Cx<float> operator+(Cx<float> a, Cx<float> b) {
  const float2 r = __fadd2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
  return mk(r.x, r.y);
}
__device__ __forceinline__ Cx<float> operator-(Cx<float> a, Cx<float> b) {
  const float2 r = __fadd2_rn(make_float2(a.x, a.y), make_float2(-b.x, -b.y));
  return mk(r.x, r.y);
}
#endif
template <typename R>
__device__ __forceinline__ Cx<R> cmul(Cx<R> a, Cx<R> b) {
  return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename R>
__device__ __forceinline__ Cx<R> cmulc(Cx<R> a, Cx<R> b) {
  return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
#if CB_CMUL2
// float complex products as one packed FMUL2 + one FFMA2 (sm_100 f32x2):
// (a.x b.x, a.x b.y) then + (a.y (-b.y), a.y b.x); the same accuracy as the
// scalar FMUL/FFMA pair (the other product is the rounded one)
__device__ __forceinline__ Cx<float> cmul(Cx<float> a, Cx<float> b) {
  const float2 t = __fmul2_rn(make_float2(a.x, a.x), make_float2(b.x, b.y));
  const float2 r = __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), t);
  return mk(r.x, r.y);
}
__device__ __forceinline__ Cx<float> cmulc(Cx<float> a, Cx<float> b) {
  // a conj(b) = (a.x b.x + a.y b.y, a.y b.x - a.x b.y)
  const float2 t = __fmul2_rn(make_float2(a.x, a.y), make_float2(b.x, b.x));
  const float2 r = __ffma2_rn(make_float2(a.y, a.x), make_float2(b.y, -b.y), t);
  return mk(r.x, r.y);
}
#endif
// acc + a b and acc + conj(a) b (the MIMO sums). FP64: chains of fused
// multiply-adds, 4 instructions instead of a product's 4 plus 2 additions
// (configs[4] c128 -0.8 %); FP32 keeps the product + packed add (the
// longer dependency chain measured +0.9 % in the one-block kernel).
template <typename R>
__device__ __forceinline__ Cx<R> cmac(Cx<R> acc, Cx<R> a, Cx<R> b) {
  if constexpr (sizeof(R) == 4) {
    return acc + cmul(a, b);
  } else {
    return mk(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
  }
}
template <typename R>
__device__ __forceinline__ Cx<R> cmacc(Cx<R> acc, Cx<R> a, Cx<R> b) {
  if constexpr (sizeof(R) == 4) {
    return acc + cmul(conj(a), b);
  } else {
    return mk(fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y)));
  }
}
template <typename R>
__device__ __forceinline__ Cx<R> conj(Cx<R> a) {
  return mk(a.x, -a.y);
}
template <typename R>
__device__ __forceinline__ Cx<R> scale(Cx<R> a, R s) {
  return mk(a.x * s, a.y * s);
}

__device__ __forceinline__ Cx<float> ldg(const Cx<float>* p) {
  const float2 v = __ldg(reinterpret_cast<const float2*>(p));
  return mk(v.x, v.y);
}
__device__ __forceinline__ Cx<double> ldg(const Cx<double>* p) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return mk(v.x, v.y);
}

// Streaming loads of per-step tables (dispersion phasors, MIMO spectra):
// each CTA reads a row once per step, so they bypass L1 allocation and
// leave the 28 KB of L1 the shared-memory carveout leaves to the twiddle
// rows every pass re-reads.
__device__ __forceinline__ Cx<float> ldg_na(const Cx<float>* p) {
  float a, b;
  asm("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(a), "=f"(b) : "l"(p));
  return mk(a, b);
}
__device__ __forceinline__ Cx<double> ldg_na(const Cx<double>* p) {
  double a, b;
  asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
  return mk(a, b);
}
#define CB_TW_LD "ld.global.nc.L1::evict_last"

// Shared-memory index padding: one spare element every 16 complex entries
// makes the radix-16 Stockham scatter (lane stride 16 elements) conflict-free.
__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded_len(int n) { return n + (n >> 4) + 1; }

// ------------------------------------------------------------------------
// Small DFTs in registers (radix 2..16), radix-2 DIF network with
// compile-time twiddles; output is bit-reversed (callers index through
// bitrev<RAD>).

template <int RAD>
__device__ __forceinline__ constexpr int bitrev(int r) {
  int o = 0;
  for (int b = 1; b < RAD; b <<= 1) {
    o = (o << 1) | (r & 1);
    r >>= 1;
  }
  return o;
}

// cos / sin of 2*pi*e/16, e = 0..15 (exact decimal expansions)
__device__ __forceinline__ constexpr double c16(int e) {
  constexpr double t[16] = {1.0,
                            0.92387953251128675613,
                            0.70710678118654752440,
                            0.38268343236508977173,
                            0.0,
                            -0.38268343236508977173,
                            -0.70710678118654752440,
                            -0.92387953251128675613,
                            -1.0,
                            -0.92387953251128675613,
                            -0.70710678118654752440,
                            -0.38268343236508977173,
                            0.0,
                            0.38268343236508977173,
                            0.70710678118654752440,
                            0.92387953251128675613};
  return t[e & 15];
}
__device__ __forceinline__ constexpr double s16(int e) { return c16(e - 4); }

// d * W_16^{e16} (forward: exp(-2 pi i e16 / 16); inverse: conjugate),
// e16 in [0, 8) and known at compile time after unrolling.
// a * sqrt(1/2) with a two-term constant in float: the one-term float
// constant is 1.7e-8 low, a systematic gain that would repeat in every
// FFT of every step.
template <typename R>
__device__ __forceinline__ R mul_rsqrt2(R a) {
  if constexpr (sizeof(R) == 4) {
    return __fmaf_rn(a, 0.707106769084930419921875f, a * 1.21016175e-08f);
  } else {
    return a * 0.70710678118654752440;
  }
}

// d * W_16^{e16} (forward: exp(-2 pi i e16 / 16); inverse: conjugate),
// e16 in [0, 8) and known at compile time after unrolling.
template <typename R, bool INV>
__device__ __forceinline__ Cx<R> tw16(Cx<R> d, int e16) {
  if (e16 == 0) return d;
  if (e16 == 4) return INV ? mk(-d.y, d.x) : mk(d.y, -d.x);  // +i / -i
  if (e16 == 2)  // (1 -+ i)/sqrt2
    return INV ? mk(mul_rsqrt2(d.x - d.y), mul_rsqrt2(d.x + d.y))
               : mk(mul_rsqrt2(d.x + d.y), mul_rsqrt2(d.y - d.x));
  if (e16 == 6)  // (-1 -+ i)/sqrt2
    return INV ? mk(-mul_rsqrt2(d.x + d.y), mul_rsqrt2(d.x - d.y))
               : mk(mul_rsqrt2(d.y - d.x), -mul_rsqrt2(d.x + d.y));
  // odd sixteenths: cos/sin of pi/8 and 3pi/8 (two-term in float, same
  // reason as mul_rsqrt2)
  const double cd = c16(e16), sd = INV ? s16(e16) : -s16(e16);
  if constexpr (sizeof(R) == 4) {
    const float ch = (float)cd, sh = (float)sd;
    const float cl = (float)(cd - (double)ch), sl = (float)(sd - (double)sh);
    const float lre = __fmaf_rn(d.x, cl, -d.y * sl);
    const float lim = __fmaf_rn(d.x, sl, d.y * cl);
    return mk(__fmaf_rn(d.x, ch, __fmaf_rn(-d.y, sh, lre)),
              __fmaf_rn(d.x, sh, __fmaf_rn(d.y, ch, lim)));
  } else {
    return mk(d.x * (R)cd - d.y * (R)sd, d.x * (R)sd + d.y * (R)cd);
  }
}

// Radix-4 butterfly on a[0..3] (forward: W_4 = -i), outputs in natural order.
template <typename R, bool INV>
__device__ __forceinline__ void dft4_nat(const Cx<R>& a0, const Cx<R>& a1, const Cx<R>& a2,
                                         const Cx<R>& a3, Cx<R>* y) {
  const Cx<R> t0 = a0 + a2, t1 = a0 - a2, t2 = a1 + a3, t3 = a1 - a3;
  y[0] = t0 + t2;
  y[2] = t0 - t2;
  y[1] = INV ? mk(t1.x - t3.y, t1.y + t3.x) : mk(t1.x + t3.y, t1.y - t3.x);
  y[3] = INV ? mk(t1.x + t3.y, t1.y - t3.x) : mk(t1.x - t3.y, t1.y + t3.x);
}

#ifndef CB_DFT16_4X4  // FP64 radix-16 as 4 x 4 and radix-8 as 2 x 4 (152 / 52 instructions, not 168 / 56)
#define CB_DFT16_4X4 1
#endif

// d * W_16^e / sqrt(1/2) for e = 2, 6 (the sqrt(1/2) is applied by the
// consumer's fused multiply-adds)
template <typename R, bool INV>
__device__ __forceinline__ Cx<R> tw16_unscaled(Cx<R> d, int e) {
  if (e == 2) return INV ? mk(d.x - d.y, d.x + d.y) : mk(d.x + d.y, d.y - d.x);
  return INV ? mk(-(d.x + d.y), d.x - d.y) : mk(d.y - d.x, -(d.x + d.y));  // e == 6
}

// Radix-4 butterfly whose input a2 (SC == 2) or inputs a1 and a3 (SC == 13)
// still carry a missing factor sqrt(1/2): the products fold into the
// butterfly's additions as fused multiply-adds (FP64 4 x 4 radix-16).
template <typename R, bool INV, int SC>
__device__ __forceinline__ void dft4_sc(const Cx<R>& a0, const Cx<R>& a1, const Cx<R>& a2,
                                        const Cx<R>& a3, Cx<R>* y) {
  constexpr R h = (R)0.70710678118654752440;
  if constexpr (SC == 2) {
    const Cx<R> t0 = mk(fma(h, a2.x, a0.x), fma(h, a2.y, a0.y));
    const Cx<R> t1 = mk(fma(-h, a2.x, a0.x), fma(-h, a2.y, a0.y));
    const Cx<R> t2 = a1 + a3, t3 = a1 - a3;
    y[0] = t0 + t2;
    y[2] = t0 - t2;
    y[1] = INV ? mk(t1.x - t3.y, t1.y + t3.x) : mk(t1.x + t3.y, t1.y - t3.x);
    y[3] = INV ? mk(t1.x + t3.y, t1.y - t3.x) : mk(t1.x - t3.y, t1.y + t3.x);
  } else {  // SC == 13: t2 = h p, t3 = h m
    const Cx<R> t0 = a0 + a2, t1 = a0 - a2;
    const Cx<R> p = a1 + a3, m = a1 - a3;
    y[0] = mk(fma(h, p.x, t0.x), fma(h, p.y, t0.y));
    y[2] = mk(fma(-h, p.x, t0.x), fma(-h, p.y, t0.y));
    y[1] = INV ? mk(fma(-h, m.y, t1.x), fma(h, m.x, t1.y)) : mk(fma(h, m.y, t1.x), fma(-h, m.x, t1.y));
    y[3] = INV ? mk(fma(h, m.y, t1.x), fma(-h, m.x, t1.y)) : mk(fma(-h, m.y, t1.x), fma(h, m.x, t1.y));
  }
}

template <typename R, int RAD, bool INV>
__device__ __forceinline__ void dft_reg(Cx<R>* v) {
  if constexpr (CB_DFT16_4X4 && RAD == 16 && sizeof(R) == 8) {
    // X[k1 + 4 k2] = sum_n1 W_4^(n1 k2) W_16^(n1 k1) sum_n2 x[n1 + 4 n2] W_4^(n2 k1);
    // natural output k goes to v[bitrev(k)] like the radix-2 form below.
    // The four sqrt(1/2)-type twiddles (n1 k1 = 2, 6) are left unscaled and
    // folded into the second radix-4 stage (dft4_sc): 152 FP64 instructions.
    Cx<R> b[4][4];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      dft4_nat<R, INV>(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12], b[n1]);
#pragma unroll
      for (int k1 = 1; k1 < 4; ++k1) {
        if (!n1) continue;
        const int e = n1 * k1;
        b[n1][k1] = (e == 2 || e == 6) ? tw16_unscaled<R, INV>(b[n1][k1], e)
                                       : tw16<R, INV>(b[n1][k1], e);
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      Cx<R> y[4];
      if (k1 == 0) dft4_nat<R, INV>(b[0][0], b[1][0], b[2][0], b[3][0], y);
      else if (k1 == 2) dft4_sc<R, INV, 13>(b[0][2], b[1][2], b[2][2], b[3][2], y);
      else dft4_sc<R, INV, 2>(b[0][k1], b[1][k1], b[2][k1], b[3][k1], y);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[bitrev<16>(k1 + 4 * k2)] = y[k2];
    }
    return;
  }
  if constexpr (CB_DFT16_4X4 && RAD == 8 && sizeof(R) == 8) {
    // X[k1 + 2 k2] = sum_n1 W_4^(n1 k2) W_8^(n1 k1) (x[n1] + (-1)^k1 x[n1 + 4]):
    // radix 2, then radix 4 with W_8 and W_8^3 folded in (52 instructions)
    Cx<R> a[4], b[4];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      a[n1] = v[n1] + v[n1 + 4];
      b[n1] = v[n1] - v[n1 + 4];
    }
    b[1] = tw16_unscaled<R, INV>(b[1], 2);
    b[2] = tw16<R, INV>(b[2], 4);
    b[3] = tw16_unscaled<R, INV>(b[3], 6);
    Cx<R> y0[4], y1[4];
    dft4_nat<R, INV>(a[0], a[1], a[2], a[3], y0);
    dft4_sc<R, INV, 13>(b[0], b[1], b[2], b[3], y1);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      v[bitrev<8>(2 * k2)] = y0[k2];
      v[bitrev<8>(1 + 2 * k2)] = y1[k2];
    }
    return;
  }
#pragma unroll
  for (int span = RAD / 2; span >= 1; span >>= 1) {
#pragma unroll
    for (int start = 0; start < RAD; start += 2 * span) {
#pragma unroll
      for (int i = 0; i < span; ++i) {
        const Cx<R> a = v[start + i];
        const Cx<R> b = v[start + i + span];
        v[start + i] = a + b;
        v[start + i + span] = tw16<R, INV>(a - b, i * (16 / (2 * span)));
      }
    }
  }
}

// ------------------------------------------------------------------------
// Radix schedule and per-pass twiddle tables.
//
// An FFT of length L runs Stockham passes with sub-transform size NS = 1,
// R1, R1*R2, ... and radix R = min(MAXRAD, L / NS). A pass with NS > 1
// twiddles element r of butterfly j by W_Q^(r*k*Q/(NS*R)), k = j mod NS.
// Those factors are stored per pass as NS rows of R entries (row k, entry
// r), so the R-1 twiddles of a butterfly are one contiguous row: lanes with
// consecutive k read consecutive rows with 16-byte vector loads (fully
// coalesced), instead of R-1 scattered 8-byte loads.

// Radix schedules (sub-transform sizes NS = 1, R1, R1*R2, ...):
//   kTail -- radix-16 passes, leftover radix last  (2048: 16 16 8); field
//            IFFTs and outer transforms when twiddles come from L2
//   kHead -- radix-16 passes, leftover radix first (2048: 8 16 16); the
//            in-step field FFT, so its last pass (radix 16, NS = Q/16)
//            produces exactly the 16 samples the next step's IFFT first pass
//            (radix 16, NS = 1) consumes and the two fuse (fft2_boundary)
//   kMid  -- radix 16 first and last, the leftover radix in between
//            (2048: 16 8 16, 4096: 16 16 16): every field transform when the
//            twiddles live in tensor memory. Forward and inverse then share
//            one set of rows (the inverse conjugates them), which halves the
//            TMEM columns a thread needs, and the boundary fusion still
//            holds (last radix = first radix = 16). For Q <= 1024 its
//            narrow middle pass runs several butterflies per thread and
//            spills, so small Q keep kTail/kHead.
//   kHalf -- radix-4 passes for the half-length real-transform FFTs, which
//            keeps all Q/8 threads busy on Q/2 points; with kWide, radix-8
//            passes (1024: 8 8 8 2, one pass fewer): the one-block-per-CTA
//            kernel's Q/16-thread groups, and the cluster kernel from Q = 2048
// kTM may be or'ed into kMid or kHalf: that transform reads its twiddle
// rows from tensor memory (see "Twiddle rows in tensor memory" below).
#ifndef CB_HALF_RAD
#define CB_HALF_RAD 4
#endif
#ifndef CB_WIDE16
#define CB_WIDE16 1
#endif
constexpr int kMaxRad = 16;
constexpr int kTail = 0, kHead = 1, kHalf = 2, kMid = 3, kTM = 4;
// kStash (field schedules, one-block-per-CTA kernel): butterflies a thread
// computes before the pass barrier are parked in TMEM instead of registers,
// all but the last (see tm_stash_*)
constexpr int kStash = 8;
// kGroupBar (one-block-per-CTA kernel): the passes of a subband group
// synchronise on the group's own named barrier, so the P groups drift out
// of phase and one group's shared-memory phase overlaps another's math
constexpr int kGroupBar = 16;
// kWide (kHalf only): radix-8 half-length passes, rows in their own section
constexpr int kWide = 32;
// kCarry (field schedules of the one-block-per-CTA kernel, with kStash): the
// last pass of every IFFT that feeds the nonlinear step (radix 16, NS = Q/16,
// intensity hook) keeps its outputs in TMEM instead of writing F, and the
// first pass of the forward FFT after the rotation (radix 16, NS = 1) reads
// them back: butterfly j produces exactly the samples j + r*Q/16 that
// butterfly j of the next pass consumes, so the field's shared-memory round
// trip between the two, and both passes' load/store barriers, disappear
#ifndef CB_ROT_MUFU
#define CB_ROT_MUFU 0
#endif
#ifndef CB_CARRY
#define CB_CARRY 1
#endif
constexpr int kCarry = 64;

__host__ __device__ constexpr int sched_radix(int L, int ns, int sched) {
  const int sc = sched & 3;
  if (sc == kHalf) {
    // kWide at L = 1024: one radix-16 pass first (no twiddles), then
    // radix 8 (1024: 16 8 8) -- three shared-memory round trips, not four
    if (CB_WIDE16 && (sched & kWide) && ns == 1 && L == 1024) return 16;
    const int hr = (sched & kWide) ? 8 : CB_HALF_RAD;
    return L / ns >= hr ? hr : L / ns;
  }
  if (sc == kHead && ns == 1) {
    int head = L;
    while (head > kMaxRad) head /= kMaxRad;
    return head;
  }
  if (sc == kMid && ns > 1 && L / ns > kMaxRad) {
    const int mid = L / ns / kMaxRad;  // left once the last radix-16 pass is set aside
    return mid >= kMaxRad ? kMaxRad : mid;
  }
  return L / ns >= kMaxRad ? kMaxRad : L / ns;
}
__host__ __device__ constexpr int twp_offset(int L, int NS, int sched) {
  int s = 0;
  for (int ns = 1; ns < NS; ns *= sched_radix(L, ns, sched))
    if (ns > 1) s += ns * sched_radix(L, ns, sched);
  return s;
}
__host__ __device__ constexpr int twp_size(int L, int sched) { return twp_offset(L, L, sched); }
// per-pass twiddle rows in Params::twp:
//   [kTail rows of Q][kHead rows of Q][kMid rows of Q][kHalf rows of Q/2]
//   [kHalf|kWide rows of Q/2]
__host__ __device__ constexpr int twp_base(int Q, int sched) {
  const int sc = sched & 3;
  const int half = twp_size(Q, kTail) + twp_size(Q, kHead) + twp_size(Q, kMid);
  return sc == kTail ? 0
       : sc == kHead ? twp_size(Q, kTail)
       : sc == kMid  ? twp_size(Q, kTail) + twp_size(Q, kHead)
       : (sched & kWide) ? half + twp_size(Q / 2, kHalf)
                         : half;
}
__host__ __device__ constexpr int twp_total(int Q) {
  return twp_base(Q, kHalf | kWide) + twp_size(Q / 2, kHalf | kWide);
}

// Twiddle storage of one pass (NS rows k, radix RAD, entries r = 1..RAD-1)
// is plane-major so that every load instruction of a warp reads one
// contiguous span (lanes = consecutive k): float rows are split into RAD/2
// planes of 16-byte pairs (r = 2q+1, 2q+2; the last pair's second half is
// padding), double rows into RAD-1 planes of one complex each. Plane q of
// a pass starts at complex offset q * 2 * NS (float) or q * NS (double).
__host__ __device__ constexpr int tw_plane_index(int real_bytes, int NS, int k, int r) {
  return real_bytes == 4 ? ((r - 1) / 2) * 2 * NS + 2 * k + ((r - 1) & 1) : (r - 1) * NS + k;
}

template <int RAD, int NS>
__device__ __forceinline__ void load_row(const Cx<float>* tw, int k, Cx<float>* w) {
#pragma unroll
  for (int q = 0; q < RAD / 2; ++q) {
    float a, b, c, d;
    asm volatile(CB_TW_LD ".v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "l"(tw + q * 2 * NS + 2 * k));
    w[2 * q + 1] = mk(a, b);
    if (2 * q + 2 < RAD) w[2 * q + 2] = mk(c, d);
  }
}
template <int RAD, int NS>
__device__ __forceinline__ void load_row(const Cx<double>* tw, int k, Cx<double>* w) {
#pragma unroll
  for (int r = 1; r < RAD; ++r) {
    double a, b;
    asm volatile(CB_TW_LD ".v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b)
                 : "l"(tw + (r - 1) * NS + k));
    w[r] = mk(a, b);
  }
}

// ------------------------------------------------------------------------
// Twiddle rows in tensor memory.
//
// The block kernel has no matrix product, so the 256 KB of tensor memory
// per SM would sit idle; it holds the FFT twiddle rows instead. Every
// thread needs, for each pass, the same row(s) in every step (its butterfly
// index is fixed), so at kernel start each thread copies its rows from the
// L2 tables into its own TMEM lane, and each pass then reads them with one
// or two tcgen05.ld (a private datapath) instead of RAD/2 16-byte loads
// through the L1/TEX pipe that the shared-memory passes saturate, and
// without the L2 latency (the 28 KB of L1 left by the shared-memory
// carveout cannot hold the working set).
//
// TMEM lane = 32 * (warp % 4) + lane, so the NT/128 warps w, w+4, ... share
// a lane. A pass whose row depends only on the lane stores one copy;
// otherwise one copy per (warp group g = tid / 128, butterfly slot p).
// Columns per CTA: 512 / (resident CTAs per SM); the launch sizes dynamic
// shared memory so that no more CTAs than that can be resident, which keeps
// the allocation from ever blocking (cbessfm_launch.cuh).

template <int N>
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t* v);
template <int N>
__device__ __forceinline__ void tm_st(uint32_t a, const uint32_t* v);
template <>
__device__ __forceinline__ void tm_ld<2>(uint32_t a, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(v[0]), "=r"(v[1])
               : "r"(a));
}
template <>
__device__ __forceinline__ void tm_st<2>(uint32_t a, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};"
               :: "r"(a), "r"(v[0]), "r"(v[1])
               : "memory");
}
template <>
__device__ __forceinline__ void tm_ld<4>(uint32_t a, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(a));
}
template <>
__device__ __forceinline__ void tm_st<4>(uint32_t a, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};"
               :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3])
               : "memory");
}
template <>
__device__ __forceinline__ void tm_ld<8>(uint32_t a, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(a));
}
template <>
__device__ __forceinline__ void tm_st<8>(uint32_t a, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
template <>
__device__ __forceinline__ void tm_ld<16>(uint32_t a, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(a));
}
template <>
__device__ __forceinline__ void tm_st<16>(uint32_t a, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
               : "memory");
}
template <>
__device__ __forceinline__ void tm_ld<32>(uint32_t a, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
               "tcgen05.wait::ld.sync.aligned;"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(a));
}
template <>
__device__ __forceinline__ void tm_st<32>(uint32_t a, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
}

// 32-bit words of one row (RAD-1 complex entries) and the columns it spans
__host__ __device__ constexpr int tm_words(int rbytes, int rad) { return (rad - 1) * rbytes / 2; }
__host__ __device__ constexpr int tm_width(int words) {
  return words <= 2 ? 2 : words <= 4 ? 4 : words <= 8 ? 8 : (words + 15) / 16 * 16;
}
// Geometry of one pass of a field (kMid, L = Q) or half-length (kHalf,
// L = Q/2) transform run by NT threads.
struct TmPass {
  int rad, per, dep_g, dep_p, copies, width;
};
__host__ __device__ constexpr TmPass tm_pass(int rbytes, int Q, int NT, int sched, int ns) {
  const bool field = (sched & 3) != kHalf;
  const int L = field ? Q : Q / 2;
  const int rad = sched_radix(L, ns, sched);
  const int slots = field ? NT / 2 : NT;
  const int per = (L / rad) >= slots ? (L / rad) / slots : 1;
  // field butterfly j = 64 g + 16 (warp % 4) + (tid % 16) + p NT/2;
  // half-length j = 128 g + 32 (warp % 4) + lane + p NT (bfly() permutes
  // inside 64-groups only)
  const int dep_g = NT > 128 && ns > (field ? 64 : 128);
  const int dep_p = per > 1 && ns > (field ? NT / 2 : NT);
  const int g = NT > 128 ? NT / 128 : 1;
  const int copies = (dep_g ? g : 1) * (dep_p ? per : 1);
  return TmPass{rad, per, dep_g, dep_p, copies, tm_width(tm_words(rbytes, rad))};
}
// first TMEM column of pass (sched, NS): kMid passes, then kHalf passes
// (radix-8 ones when sched carries kWide)
__host__ __device__ constexpr int tm_col(int rbytes, int Q, int NT, int sched, int NS) {
  int c = 0;
  for (int pass = 0; pass < 2; ++pass) {
    const int sc = pass == 0 ? kMid : (kHalf | (sched & kWide));
    const int L = pass == 0 ? Q : Q / 2;
    for (int ns = 1; ns < L; ns *= sched_radix(L, ns, sc)) {
      if ((sc & 3) == (sched & 3) && ns == NS) return c;
      if (ns > 1) {
        const TmPass t = tm_pass(rbytes, Q, NT, sc, ns);
        c += t.copies * t.width;
      }
    }
  }
  return c;
}
// columns of the rows (either half-length variant; the butterfly parking
// starts after them)
__host__ __device__ constexpr int tm_total(int rbytes, int Q, int NT) {
  const int a = tm_col(rbytes, Q, NT, kHalf, Q / 2);
  const int b = tm_col(rbytes, Q, NT, kHalf | kWide, Q / 2);
  return a > b ? a : b;
}

// Copy index of the row thread `tid` uses in slot p of a pass.
__device__ __forceinline__ int tm_copy(const TmPass& t, int tid, int p) {
  const int g = t.dep_g ? tid >> 7 : 0;
  return t.dep_p ? g * t.per + p : g;
}
__device__ __forceinline__ uint32_t tm_lane_base(uint32_t tbase) {
  return tbase + ((uint32_t)((threadIdx.x >> 5) & 3) << 21);
}

template <typename R>
__device__ __forceinline__ void tm_pack(const Cx<R>& c, uint32_t* v) {
  if constexpr (sizeof(R) == 4) {
    v[0] = __float_as_uint(c.x);
    v[1] = __float_as_uint(c.y);
  } else {
    v[0] = __double2loint(c.x);
    v[1] = __double2hiint(c.x);
    v[2] = __double2loint(c.y);
    v[3] = __double2hiint(c.y);
  }
}
template <typename R>
__device__ __forceinline__ Cx<R> tm_unpack(const uint32_t* v) {
  if constexpr (sizeof(R) == 4) {
    return mk(__uint_as_float(v[0]), __uint_as_float(v[1]));
  } else {
    return mk(__hiloint2double((int)v[1], (int)v[0]), __hiloint2double((int)v[3], (int)v[2]));
  }
}

// Row (entries 1..RAD-1) from TMEM at column `col` of this thread's lane.
template <typename R, int RAD>
__device__ __forceinline__ void tm_load_row(uint32_t lane_base, int col, Cx<R>* w) {
  constexpr int WORDS = tm_words((int)sizeof(R), RAD);
  constexpr int W = tm_width(WORDS);
  uint32_t v[W];
  if constexpr (W <= 32) {
    tm_ld<W>(lane_base + col, v);
  } else {
#pragma unroll
    for (int c = 0; c < W; c += 32) tm_ld<32>(lane_base + col + c, v + c);
  }
  constexpr int CW = 2 * sizeof(R) / 4;
#pragma unroll
  for (int r = 1; r < RAD; ++r) w[r] = tm_unpack<R>(v + (r - 1) * CW);
}
template <typename R, int RAD>
__device__ __forceinline__ void tm_store_row(uint32_t lane_base, int col, const Cx<R>* w) {
  constexpr int WORDS = tm_words((int)sizeof(R), RAD);
  constexpr int W = tm_width(WORDS);
  constexpr int CW = 2 * sizeof(R) / 4;
  uint32_t v[W];
#pragma unroll
  for (int i = 0; i < W; ++i) v[i] = 0u;
#pragma unroll
  for (int r = 1; r < RAD; ++r) tm_pack<R>(w[r], v + (r - 1) * CW);
  if constexpr (W <= 32) {
    tm_st<W>(lane_base + col, v);
  } else {
#pragma unroll
    for (int c = 0; c < W; c += 32) tm_st<32>(lane_base + col + c, v + c);
  }
}

// ---- distributed shared memory push with transaction barriers (sm_90+)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// split cluster barrier (release / acquire at cluster scope)
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
// The suspend-time hint parks the waiting warps until the phase completes
// instead of spinning (a spin loop costs issue slots the other CTAs on the
// SM need); the hint is an upper bound, completion wakes them.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
#ifdef CB_MBAR_SPIN  // experiment knob: plain try_wait spin
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
#else
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
#endif
      "@!P1 bra WAIT_%=;\n\t}"
      ::"r"(smem_addr(bar)), "r"(parity), "r"(0x989680u)
      : "memory");
}
// 8- or 16-byte store into another CTA's shared memory that completes
// `bytes` transactions on that CTA's mbarrier.
__device__ __forceinline__ void push(uint32_t raddr, Cx<float> v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
               ::"r"(raddr), "f"(v.x), "f"(v.y), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void push(uint32_t raddr, Cx<double> v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(raddr), "d"(v.x), "d"(v.y), "r"(rbar)
               : "memory");
}

// 16-byte global -> shared copy that bypasses the registers (LDGSTS, L2 only):
// a thread issues all of its window samples back to back and waits once
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(smem_dst)),
               "l"(gmem_src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

__device__ __forceinline__ void bar_named(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Float index of real sample p in a complex-packed array z[t] = (v[2t], v[2t+1])
// stored with the complex padding.
__device__ __forceinline__ int fpos(int p) { return 2 * pad(p >> 1) + (p & 1); }

// Barrier ending a pass phase: the whole CTA, or (kGroupBar) the NT-thread
// group of the calling thread (named barriers 1..P; 0 is __syncthreads).
template <int SCHED, int NT>
__device__ __forceinline__ void pass_sync() {
  if constexpr ((SCHED & kGroupBar) != 0) {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)threadIdx.x / NT), "n"(NT) : "memory");
  } else {
    __syncthreads();
  }
}

// Thread index inside the NT-thread group that runs one subband's
// transforms: the whole CTA in the one-subband-per-CTA kernel, one of P
// groups in the one-block-per-CTA kernel (NT a power of two; groups start
// at multiples of NT, so lane and half-warp bits are unchanged).
template <int NT>
__device__ __forceinline__ int ltid() {
  return (int)threadIdx.x & (NT - 1);
}

// ------------------------------------------------------------------------
// Field FFT thread mapping: the two polarisations of a butterfly run on the
// two half-warps (lane bit 4 selects x or y), so a thread holds one
// radix-16 butterfly (16 complex values) and both half-warps read the same
// twiddle rows in the same instruction.

template <int NT>
__device__ __forceinline__ int fpol(int t) { return (t >> 4) & 1; }
template <int NT>
__device__ __forceinline__ int fbase(int t) { return ((t >> 5) << 4) | (t & 15); }

// Hooks fused into the first (pre: after the loads) or last (post: before
// the stores) pass of a field FFT. Element r of butterfly j sits at position
// j + r*LR on load; natural output r sits at d0 + r*NS on store and lives
// in v[bitrev(r)]. v is this thread's polarisation.

struct NoHook {
  template <typename R, int RAD, int LR>
  __device__ __forceinline__ void pre(int, Cx<R>*) {}
  template <typename R, int RAD, int NS>
  __device__ __forceinline__ void post(int, Cx<R>*) {}
};

// Multiply by a dispersion phasor row (dbp.py:395 / :399); ph is indexed by
// the subband-local bin.
template <typename R>
struct PhasorHook : NoHook {
  const Cx<R>* ph;
  template <typename, int RAD, int NS>
  __device__ __forceinline__ void post(int d0, Cx<R>* v) {
#pragma unroll
    for (int r = 0; r < RAD; ++r) v[bitrev<RAD>(r)] = cmul(v[bitrev<RAD>(r)], ldg_na(ph + d0 + r * NS));
  }
};

// Write the intensity |x|^2 + |y|^2 (dbp.py:193) of the just-computed time
// samples into the packed real array I (float view of IS); the partner
// half-warp holds the other polarisation at the same positions, and each
// half-warp writes half of the positions.
template <typename R>
struct IntensityHook : NoHook {
  R* I;
  template <typename, int RAD, int NS>
  __device__ __forceinline__ void post(int d0, Cx<R>* v) {
    const int pol = (threadIdx.x >> 4) & 1;
    R* base = I + fpos(d0);
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      const Cx<R> a = v[bitrev<RAD>(r)];
      const R own = a.x * a.x + a.y * a.y;
      const R other = __shfl_xor_sync(0xffffffffu, own, 16);
      if ((r & 1) == pol) base[2 * pad(r * NS / 2)] = pol ? other + own : own + other;
    }
  }
};

template <typename R>
__device__ __forceinline__ void sincos_acc(R a, R* s, R* c);
// FP32: three-term Cody-Waite reduction to [-pi/4, pi/4] and the Cephes
// minimax polynomials (about 1 ulp), roughly half the instructions of
// sincosf; arguments beyond 2^13 (never reached by a nonlinear phase per
// step, but legal) take the libdevice path.
template <>
__device__ __forceinline__ void sincos_acc<float>(float a, float* s, float* c) {
#ifdef CB_SINCOS_STUB  // timing experiment only (wrong results): what the sincos costs
  *s = a;
  *c = __fmaf_rn(a, -0.5f * a, 1.0f);
  return;
#endif
  float r;
  int q;
  if (fabsf(a) > 8192.0f) {
    // large arguments (never reached by a per-step nonlinear phase, but
    // legal): reduce in FP64 (exact to ~1e-16 |a| for |a| < 2^31), no
    // libdevice Payne-Hanek path with its local-memory table
    const double ad = (double)a;
    const double jd = rint(ad * 0.63661977236758134308);
    double rd = fma(jd, -1.5707963267948966192, ad);
    rd = fma(jd, -6.123233995736766036e-17, rd);
    r = (float)rd;
    q = (int)((long long)jd & 3);
  } else if (__all_sync(__activemask(), fabsf(a) <= 0.78f)) {
    // |a| <= 0.78 (< pi/4) in the whole warp -- the usual size of a per-step
    // nonlinear phase: no reduction. Bit-identical to the branch below,
    // where j = rint(a 2/pi) = 0 leaves r = a and q = 0. (The same branch
    // in the FP64 version cost 2.5 %: it breaks the interleaving of the
    // eight angles a thread evaluates; here it saves 0.9 %.)
    r = a;
    q = 0;
  } else if (CB_ROT_MUFU) {
    // experiment: reduction to [-pi, pi] and the SFU sin/cos (abs error
    // ~2^-21 on that range) instead of the FMA-pipe polynomials
    const float j = rintf(a * 0.159154943091895336f);
    r = __fmaf_rn(j, -6.28318548202514648f, a);
    r = __fmaf_rn(j, 1.74845553146951162e-7f, r);
    __sincosf(r, s, c);
    return;
  } else {
    const float j = rintf(a * 0.636619772367581343f);
    r = __fmaf_rn(j, -0x1.921fb6p+0f, a);
    r = __fmaf_rn(j, 0x1.777a5cp-25f, r);
    r = __fmaf_rn(j, 0x1.ee59dap-50f, r);
    q = __float2int_rn(j);
  }
  const float r2 = r * r;
  float ps = __fmaf_rn(r2, -1.9515295891e-4f, 8.3321608736e-3f);
  ps = __fmaf_rn(r2, ps, -1.6666654611e-1f);
  const float sn = __fmaf_rn(r * r2, ps, r);
  float pc = __fmaf_rn(r2, 2.443315711809948e-5f, -1.388731625493765e-3f);
  pc = __fmaf_rn(r2, pc, 4.166664568298827e-2f);
  pc = __fmaf_rn(r2, pc, -0.5f);
  const float cs = __fmaf_rn(r2, pc, 1.0f);
  const float ss = (q & 1) ? cs : sn;
  const float cc = (q & 1) ? sn : cs;
  *s = (q & 2) ? -ss : ss;
  *c = ((q + 1) & 2) ? -cc : cc;
}
// FP64: two-term FMA Cody-Waite reduction to [-pi/4, pi/4] (a - j*pi/2 is
// formed with one rounding; the tail constant carries pi/2 to ~2^-106) and
// the fdlibm kernel polynomials (degree 13 / 14, about 1 ulp): ~20 FP64
// instructions, no branchy libdevice path. Arguments beyond 2^20 (never
// reached by a per-step nonlinear phase, but legal) take libdevice sincos.
#ifndef CB_LIBDEVICE_SINCOS
template <>
__device__ __forceinline__ void sincos_acc<double>(double a, double* s, double* c) {
#ifdef CB_SINCOS_STUB  // timing experiment only (wrong results): what the sincos costs
  *s = a;
  *c = fma(a, -0.5 * a, 1.0);
  return;
#endif
  if (fabs(a) > 1048576.0) {
    sincos(a, s, c);
    return;
  }
  const double j = rint(a * 0.63661977236758134308);
  double r = fma(j, -1.57079632679489655800e+00, a);
  r = fma(j, -6.12323399573676603587e-17, r);
  const int q = (int)j;
  const double r2 = r * r;
  double ps = fma(r2, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
  ps = fma(r2, ps, 2.75573137070700676789e-06);
  ps = fma(r2, ps, -1.98412698298579493134e-04);
  ps = fma(r2, ps, 8.33333333332248946124e-03);
  ps = fma(r2, ps, -1.66666666666666324348e-01);
  const double sn = fma(r * r2, ps, r);
  double pc = fma(r2, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
  pc = fma(r2, pc, -2.75573143513906633035e-07);
  pc = fma(r2, pc, 2.48015872894767294178e-05);
  pc = fma(r2, pc, -1.38888888888741095749e-03);
  pc = fma(r2, pc, 4.16666666666666019037e-02);
  const double cs = fma(r2 * r2, pc, fma(r2, -0.5, 1.0));
  const double ss = (q & 1) ? cs : sn;
  const double cc = (q & 1) ? sn : cs;
  *s = (q & 2) ? -ss : ss;
  *c = ((q + 1) & 2) ? -cc : cc;
}
#else
template <>
__device__ __forceinline__ void sincos_acc<double>(double a, double* s, double* c) {
  sincos(a, s, c);
}
#endif

// Rotate by exp(-i theta), theta = scale * th[p] (dbp.py:196, :208); th is
// the float view of the packed irfft output. The two half-warps hold the
// same positions (x and y): each evaluates sincos for half of them and the
// halves are exchanged with shuffles, so every angle is evaluated once.
template <typename R>
struct RotationHook : NoHook {
  const R* th;
  R scale;
  template <typename, int RAD, int LR>
  __device__ __forceinline__ void pre(int j, Cx<R>* v) {
    const R* base = th + fpos(j);
    const int pol = (threadIdx.x >> 4) & 1;
    static_assert(RAD % 2 == 0, "rotation split needs an even radix");
#pragma unroll
    for (int h = 0; h < RAD / 2; ++h) {
      // this half-warp evaluates r = 2h + pol, the partner r = 2h + 1 - pol
      const int ro = 2 * h + pol;
      R s, c;
      sincos_acc<R>(base[2 * pad(ro * LR / 2)] * scale, &s, &c);
      const R so = __shfl_xor_sync(0xffffffffu, s, 16);
      const R co = __shfl_xor_sync(0xffffffffu, c, 16);
      const Cx<R> mine = mk(c, -s), theirs = mk(co, -so);
      v[2 * h] = cmul(v[2 * h], pol ? theirs : mine);
      v[2 * h + 1] = cmul(v[2 * h + 1], pol ? mine : theirs);
    }
  }
};

// complex128 cluster kernel with a rotation table in shared memory
// (kRotTab entries exp(i k / kRotDen), k = -kRotTab/2 .. kRotTab/2 - 1, copied
// from Params::rot_tab at kernel start): theta = k/32 + r with |r| <= 1/64,
// the table gives (cos, sin)(k/32), degree-5 / degree-6 Taylor polynomials
// give (sin, cos)(r) to < 5e-17, one complex product combines them -- 15
// FP64 instructions per angle instead of 23 and no quadrant selects. Angles
// of 7.9375 rad or more anywhere in the warp (never reached by a per-step
// nonlinear phase, but legal) take sincos_acc for the whole pass: one
// warp-uniform branch per pass, so each side keeps its eight angles
// interleaved.
constexpr int kRotTab = 512;
constexpr int kRotDen = 32;
template <typename R>
struct RotationTabHook : NoHook {
  const R* th;
  R scale;
  const Cx<R>* tab;  // shared memory, entry k + kRotTab/2
  template <typename, int RAD, int LR>
  __device__ __forceinline__ void pre(int j, Cx<R>* v) {
    static_assert(sizeof(R) == 8, "the rotation table is built for complex128");
    const R* base = th + fpos(j);
    const int pol = (threadIdx.x >> 4) & 1;
    static_assert(RAD % 2 == 0, "rotation split needs an even radix");
    double a[RAD / 2];
    bool small = true;
#pragma unroll
    for (int h = 0; h < RAD / 2; ++h) {
      a[h] = base[2 * pad((2 * h + pol) * LR / 2)] * scale;
      // |a| < 7.9375 (0x401FC000...): |k| <= 254
      small = small && (unsigned)(__double2hiint(a[h]) & 0x7fffffff) < 0x401fc000u;
    }
    if (__all_sync(0xffffffffu, small)) {
#pragma unroll
      for (int h = 0; h < RAD / 2; ++h) {
        const double t = fma(a[h], (double)kRotDen, 6755399441055744.0);  // 1.5 * 2^52
        const int k = __double2loint(t);                                  // rint(32 a)
        const double r = fma(t - 6755399441055744.0, -1.0 / kRotDen, a[h]);
        const Cx<R> e = tab[k + kRotTab / 2];
        const double r2 = r * r;
        const double sn = fma(r * r2, fma(r2, 8.33333333333333333e-03, -1.66666666666666667e-01), r);
        double pc = fma(r2, -1.38888888888888889e-03, 4.16666666666666667e-02);
        pc = fma(r2, pc, -0.5);
        const double cs = fma(r2, pc, 1.0);
        const double c = fma(e.x, cs, -(e.y * sn));
        const double s = fma(e.y, cs, e.x * sn);
        const R so = __shfl_xor_sync(0xffffffffu, s, 16);
        const R co = __shfl_xor_sync(0xffffffffu, c, 16);
        const Cx<R> mine = mk(c, -s), theirs = mk(co, -so);
        v[2 * h] = cmul(v[2 * h], pol ? theirs : mine);
        v[2 * h + 1] = cmul(v[2 * h + 1], pol ? mine : theirs);
      }
    } else {
#pragma unroll
      for (int h = 0; h < RAD / 2; ++h) {
        R s, c;
        sincos_acc<R>(a[h], &s, &c);
        const R so = __shfl_xor_sync(0xffffffffu, s, 16);
        const R co = __shfl_xor_sync(0xffffffffu, c, 16);
        const Cx<R> mine = mk(c, -s), theirs = mk(co, -so);
        v[2 * h] = cmul(v[2 * h], pol ? theirs : mine);
        v[2 * h + 1] = cmul(v[2 * h + 1], pol ? mine : theirs);
      }
    }
  }
};

// ------------------------------------------------------------------------
// Stockham passes. Addressing: with one pad slot per 16 entries,
// pad(a + b) == pad(a) + pad(b) for every (read, write) index pair a pass
// forms (checked exhaustively in tests/test_host_logic.py), so a pass needs
// one read and one write base register plus compile-time offsets. `zero`
// is a shared word holding 0: reading it after the barrier keeps each
// pass's addressing inside the step loop (ptxas otherwise hoists every
// pass's address registers out of the loop and spills).

// Butterfly run by thread slot t in a pass. The radix-4 pass with NS = 4
// scatters to 16*(j/4) + j%4 + 4r, a 4-way bank conflict for consecutive
// j; permuting j inside each 64-butterfly group as below makes both its
// loads and its stores conflict-free (tests/test_host_logic.py checks the
// bank mapping). All other passes keep j = t.
template <int L, int NS, int RAD>
__host__ __device__ constexpr int bfly(int t) {
  if constexpr (RAD == 4 && NS == 4 && (L / RAD) % 64 == 0) {
    return (t & ~63) | ((t & 15) << 2) | ((t >> 4) & 3);
  } else {
    return t;
  }
}

// Twiddle rows of the butterflies a thread runs in one pass. FIELD: the
// field FFT mapping (butterfly fbase(t) + p * NT/2 of polarisation fpol(t));
// otherwise the half-length mapping (butterfly bfly(t + p * NT)).
// Butterfly parking for passes that run several butterflies per thread:
// Stockham passes are in place, so every butterfly's outputs must be held
// until the pass barrier; slots 0..PER-2 wait in TMEM (columns after the
// twiddle rows, one block per sharer of the lane: threadIdx.x / 128).
template <typename R, int RAD>
__host__ __device__ constexpr int stash_width() {
  return tm_width(RAD * 2 * (int)sizeof(R) / 4);
}
template <typename R, int RAD>
__device__ __forceinline__ void tm_stash_store(uint32_t lane_base, int col, const Cx<R>* v) {
  constexpr int W = stash_width<R, RAD>();
  constexpr int CW = 2 * sizeof(R) / 4;
  uint32_t u[W];
#pragma unroll
  for (int r = 0; r < RAD; ++r) tm_pack<R>(v[r], u + r * CW);
  if constexpr (W <= 32) {
    tm_st<W>(lane_base + col, u);
  } else {
#pragma unroll
    for (int c = 0; c < W; c += 32) tm_st<32>(lane_base + col + c, u + c);
  }
}
template <typename R, int RAD>
__device__ __forceinline__ void tm_stash_load(uint32_t lane_base, int col, Cx<R>* v) {
  constexpr int W = stash_width<R, RAD>();
  constexpr int CW = 2 * sizeof(R) / 4;
  uint32_t u[W];
  if constexpr (W <= 32) {
    tm_ld<W>(lane_base + col, u);
  } else {
#pragma unroll
    for (int c = 0; c < W; c += 32) tm_ld<32>(lane_base + col + c, u + c);
  }
#pragma unroll
  for (int r = 0; r < RAD; ++r) v[r] = tm_unpack<R>(u + r * CW);
}
// Columns each lane sharer (threadIdx.x / 128) owns for parking: one
// layout for every pass (with kGroupBar the groups, which share lanes, run
// different passes at the same time), sized for the widest pass -- three
// radix-8 or one radix-16 butterfly.
// (kCarry: at least two radix-16 butterflies, the carried pass outputs)
template <typename R>
__host__ __device__ constexpr int stash_stride(bool carry = false) {
  const int s = 3 * stash_width<R, 8>() > stash_width<R, 16>() ? 3 * stash_width<R, 8>()
                                                               : stash_width<R, 16>();
  return carry && 2 * stash_width<R, 16>() > s ? 2 * stash_width<R, 16>() : s;
}
// first stash column of slot p for this thread (COL0: first free column)
template <typename R, int RAD, int PER, bool CARRY = false>
__device__ __forceinline__ int stash_col(int col0, int p) {
  static_assert((PER - 1) * stash_width<R, RAD>() <= stash_stride<R>(CARRY), "stash overflow");
  return col0 + ((int)threadIdx.x >> 7) * stash_stride<R>(CARRY) + p * stash_width<R, RAD>();
}

// TMEM base address of this CTA's twiddle columns (kernels whose
// schedules carry kTM allocate it, see tm_setup)
__shared__ uint32_t cb_tm_base;

template <typename R, int L, int NT, int NS, int SCHED>
struct PassRows {
  static constexpr bool kField = (SCHED & 3) != kHalf;
  static constexpr bool kTmem = (SCHED & kTM) != 0;
  static constexpr int Q = kField ? L : 2 * L;
  static constexpr bool kLast = NS >= L;
  static constexpr int RAD = kLast ? 1 : sched_radix(L, NS, SCHED);
  static constexpr int SLOTS = kField ? NT / 2 : NT;  // threads per butterfly set
  static constexpr int PER = kLast ? 1 : ((L / RAD) >= SLOTS ? (L / RAD) / SLOTS : 1);
  static constexpr bool kHas = !kLast && NS > 1;
  // L2 rows are prefetched for every slot; TMEM rows are read per slot just
  // before use (short latency), so one row of registers suffices
  Cx<R> w[kTmem ? 1 : PER][RAD];
  // Issue the loads (no use yet): called one pass early so the L2 latency
  // overlaps the current pass's stores, its barrier and the next pass's
  // shared-memory loads. Nothing to do for TMEM rows.
  __device__ __forceinline__ void fetch(const Cx<R>* twp) {
    if constexpr (kHas && !kTmem) {
      const Cx<R>* tw = twp + twp_offset(L, NS, SCHED);
      const int tid = ltid<NT>();
#pragma unroll
      for (int p = 0; p < PER; ++p) {
        if constexpr (kField) {
          const int j = fbase<NT>(tid) + p * SLOTS;
          load_row<RAD, NS>(tw, j % NS, w[p]);
        } else {
          const int t = tid + p * NT;
          const int j = bfly<L, NS, RAD>(t);
          if ((L / RAD) >= NT || t < L / RAD) load_row<RAD, NS>(tw, j % NS, w[p]);
        }
      }
    }
  }
  // Row of slot p (TMEM: loaded here, warp-converged).
  __device__ __forceinline__ const Cx<R>* row(int p) {
    if constexpr (kHas && kTmem) {
      constexpr TmPass tp = tm_pass((int)sizeof(R), Q, NT, SCHED, NS);
      constexpr int col = tm_col((int)sizeof(R), Q, NT, SCHED, NS);
      if (!tp.dep_p && p > 0) return w[0];
      tm_load_row<R, RAD>(tm_lane_base(cb_tm_base), col + tm_copy(tp, ltid<NT>(), p) * tp.width,
                          w[0]);
      return w[0];
    } else {
      return w[kTmem ? 0 : p];
    }
  }
};

// Kernel-start copy of every pass's rows of schedules kMid and kHalf from
// the L2 tables (twp, layout twp_base) into this CTA's TMEM columns: each
// thread writes the copies it will read (lane-shared copies by the first
// 128 threads only). Followed, in the caller, by wait::st, a fence and a
// CTA barrier before any tm_load_row.
template <typename R, int Q, int NT, int SCHED, int NS>
__device__ __forceinline__ void tm_fill_sched(const Cx<R>* twp_sched) {
  constexpr int L = (SCHED & 3) == kHalf ? Q / 2 : Q;
  if constexpr (NS < L) {
    constexpr int RAD = sched_radix(L, NS, SCHED);
    if constexpr (NS > 1) {
      constexpr TmPass tp = tm_pass((int)sizeof(R), Q, NT, SCHED, NS);
      constexpr int col = tm_col((int)sizeof(R), Q, NT, SCHED, NS);
      constexpr bool field = (SCHED & 3) != kHalf;
      const Cx<R>* tw = twp_sched + twp_offset(L, NS, SCHED);
      const uint32_t lb = tm_lane_base(cb_tm_base);
      const int tid = ltid<NT>();
      // the first group of NT threads writes (the groups of the
      // one-block-per-CTA kernel share lanes and rows); lane-shared copies
      // only from its first 128 threads
      if ((int)threadIdx.x < NT && (tp.copies > 1 || tid < 128)) {
#pragma unroll
        for (int p = 0; p < (tp.dep_p ? tp.per : 1); ++p) {
          int j;
          if constexpr (field) {
            j = fbase<NT>(tid) + p * (NT / 2);
          } else {
            j = (L / RAD) >= NT ? bfly<L, NS, RAD>(tid + p * NT) : tid;
          }
          Cx<R> w[RAD];
          load_row<RAD, NS>(tw, j % NS, w);
          tm_store_row<R, RAD>(lb, col + tm_copy(tp, tid, p) * tp.width, w);
        }
      }
    }
    tm_fill_sched<R, Q, NT, SCHED, NS * RAD>(twp_sched);
  }
}

template <typename R, int Q, int NT, int SCHED, int NS, bool INV, bool FIRST, bool LAST,
          class Hook, class Rows, class NextRows>
__device__ __forceinline__ void fft2_pass(Cx<R>* __restrict__ F, const Cx<R>* __restrict__ twp,
                                          const volatile int* zero, Hook& hook, Rows& rows,
                                          NextRows& next, const Cx<R>* __restrict__ twp_next) {
  constexpr int RAD = sched_radix(Q, NS, SCHED);
  constexpr int LR = Q / RAD;
  constexpr int SLOTS = NT / 2;
  static_assert((Q / RAD) % SLOTS == 0, "butterflies must tile the half-block");
  constexpr int PER = (Q / RAD) / SLOTS;
  constexpr int SF = padded_len(Q);
  constexpr bool STASH = (SCHED & kStash) != 0 && PER > 1;
  constexpr bool CARRYS = (SCHED & kCarry) != 0;
  constexpr int SCOL = tm_total((int)sizeof(R), Q, NT);
  const int tid = ltid<NT>() + *zero;
  Cx<R>* Fp = F + fpol<NT>(tid) * SF;
  const int jb = fbase<NT>(tid);
  // kCarry: the intensity IFFT's last pass parks its outputs (natural order,
  // sample j + r*LR in slot r) in TMEM, the rotation FFT's first pass takes
  // them from there; neither touches F in the other direction, so neither
  // needs its load/store barrier
  constexpr bool CARRY_OUT = CARRYS && LAST && INV && std::is_same<Hook, IntensityHook<R>>::value;
  constexpr bool CARRY_IN = CARRYS && FIRST && !INV && std::is_same<Hook, RotationHook<R>>::value;
  if constexpr (CARRY_OUT || CARRY_IN) {
    static_assert(RAD == sched_radix(Q, 1, SCHED) && (CARRY_IN ? NS == 1 : NS == LR),
                  "carried passes: radix-R butterflies on samples j + r*Q/R");
    static_assert(PER * stash_width<R, RAD>() <= stash_stride<R>(true), "carry overflow");
    const uint32_t lb = tm_lane_base(cb_tm_base);
#pragma unroll
    for (int p = 0; p < PER; ++p) {
      const int j = jb + p * SLOTS;
      const int col = SCOL + ((int)threadIdx.x >> 7) * stash_stride<R>(true) +
                      p * stash_width<R, RAD>();
      Cx<R> v[RAD];
      if constexpr (CARRY_IN) {
        tm_stash_load<R, RAD>(lb, col, v);
        hook.template pre<R, RAD, LR>(j, v);
        dft_reg<R, RAD, INV>(v);
        Cx<R>* b = Fp + pad(j * RAD);  // NS = 1: d0 = R*j
#pragma unroll
        for (int r = 0; r < RAD; ++r) b[pad(r)] = v[bitrev<RAD>(r)];
      } else {
        const Cx<R>* b = Fp + pad(j);
#pragma unroll
        for (int r = 0; r < RAD; ++r) v[r] = b[pad(r * LR)];
        const Cx<R>* w = rows.row(p);
#pragma unroll
        for (int r = 1; r < RAD; ++r) v[r] = cmulc(v[r], w[r]);
        dft_reg<R, RAD, INV>(v);
        hook.template post<R, RAD, NS>(j, v);  // d0 = j (j < NS)
        Cx<R> u[RAD];
#pragma unroll
        for (int r = 0; r < RAD; ++r) u[r] = v[bitrev<RAD>(r)];
        tm_stash_store<R, RAD>(lb, col, u);
      }
    }
    if constexpr (CARRY_OUT) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    next.fetch(twp_next);
    pass_sync<SCHED, NT>();
    return;
  }
  Cx<R> v[PER][RAD];
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int j = jb + p * SLOTS;
    const Cx<R>* b = Fp + pad(j);
#pragma unroll
    for (int r = 0; r < RAD; ++r) v[p][r] = b[pad(r * LR)];
    if constexpr (FIRST) hook.template pre<R, RAD, LR>(j, v[p]);
    if constexpr (NS > 1) {
      const Cx<R>* w = rows.row(p);
#pragma unroll
      for (int r = 1; r < RAD; ++r) v[p][r] = INV ? cmulc(v[p][r], w[r]) : cmul(v[p][r], w[r]);
    }
    dft_reg<R, RAD, INV>(v[p]);
    if constexpr (STASH) {
      if (p < PER - 1)
        tm_stash_store<R, RAD>(tm_lane_base(cb_tm_base), stash_col<R, RAD, PER, CARRYS>(SCOL, p), v[p]);
    }
  }
  if constexpr (STASH) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  pass_sync<SCHED, NT>();
#pragma unroll
  for (int pp = 0; pp < PER; ++pp) {
    // the register-resident last slot first, then the parked ones
    const int p = STASH ? (pp == 0 ? PER - 1 : pp - 1) : pp;
    if constexpr (STASH) {
      if (pp > 0)
        tm_stash_load<R, RAD>(tm_lane_base(cb_tm_base), stash_col<R, RAD, PER, CARRYS>(SCOL, p), v[p]);
    }
    const int j = jb + p * SLOTS;
    const int d0 = (j / NS) * NS * RAD + j % NS;
    if constexpr (LAST) hook.template post<R, RAD, NS>(d0, v[p]);
    Cx<R>* b = Fp + pad(d0);
#pragma unroll
    for (int r = 0; r < RAD; ++r) b[pad(r * NS)] = v[p][bitrev<RAD>(r)];
  }
  next.fetch(twp_next);
  pass_sync<SCHED, NT>();
}

// Runs the passes NS, NS*R, ... of a length-Q field FFT with schedule
// SCHED, stopping before the pass with sub-transform size STOP (STOP = Q:
// to the end). rows: this pass's prefetched twiddle rows.
template <typename R, int Q, int NT, int SCHED, int NS, int STOP, bool INV, class Pre,
          class Post>
struct Fft2Run {
  using Rows = PassRows<R, Q, NT, NS, SCHED>;
  static __device__ __forceinline__ void run(Cx<R>* F, const Cx<R>* twp, const volatile int* z,
                                             Pre& pre, Post& post, Rows& rows) {
    constexpr int RAD = sched_radix(Q, NS, SCHED);
    constexpr int NS2 = NS * RAD;
    constexpr bool FIRST = NS == 1, LAST = NS2 == Q;
    static_assert(!(FIRST && LAST), "single-pass transforms are not used");
    PassRows<R, Q, NT, (NS2 < STOP ? NS2 : Q), SCHED> next;
    if constexpr (FIRST) {
      fft2_pass<R, Q, NT, SCHED, NS, INV, true, false>(F, twp, z, pre, rows, next, twp);
    } else if constexpr (LAST) {
      fft2_pass<R, Q, NT, SCHED, NS, INV, false, true>(F, twp, z, post, rows, next, twp);
    } else {
      NoHook none;
      fft2_pass<R, Q, NT, SCHED, NS, INV, false, false>(F, twp, z, none, rows, next, twp);
    }
    if constexpr (NS2 < STOP)
      Fft2Run<R, Q, NT, SCHED, NS2, STOP, INV, Pre, Post>::run(F, twp, z, pre, post, next);
  }
};

// Unnormalised length-Q FFT of both polarisation rows of F (forward:
// exp(-), inverse: exp(+)), natural order in and out, with fused hooks
// (Pre on the first pass, Post on the last). NS0 > 1 starts mid-transform
// (after fft2_boundary); STOP < Q stops before that pass. twp points at
// this schedule's rows. Ends with a barrier.
template <typename R, int Q, int NT, int SCHED, bool INV, class Pre = NoHook, class Post = NoHook,
          int NS0 = 1, int STOP = Q>
__device__ __forceinline__ void fft2(Cx<R>* F, const Cx<R>* twp, const volatile int* z,
                                     Pre pre = Pre(), Post post = Post()) {
  PassRows<R, Q, NT, NS0, SCHED> rows;
  rows.fetch(twp);
  Fft2Run<R, Q, NT, SCHED, NS0, STOP, INV, Pre, Post>::run(F, twp, z, pre, post, rows);
}

// Step boundary: the last pass of the in-step forward FFT (kMid, radix R,
// NS = Q/R), the next dispersion phasor, and the first pass of the next
// step's IFFT (kMid, radix R, NS = 1) in one load/compute/store round: the
// forward butterfly j produces samples j + r*Q/R, exactly the inputs of
// inverse butterfly j (dbp.py:398, :395, :396).
template <typename R, int Q, int NT, int SI, int SFW>
__device__ __forceinline__ void fft2_boundary(Cx<R>* __restrict__ F,
                                              const Cx<R>* __restrict__ twHead,
                                              const Cx<R>* __restrict__ ph,
                                              const volatile int* zero) {
  constexpr int RAD = sched_radix(Q, 1, SI);
  constexpr int NSF = Q / RAD;  // forward last pass
  static_assert(sched_radix(Q, NSF, SFW) == RAD, "the forward FFT must end with the IFFT's first radix");
  constexpr int LR = Q / RAD;
  constexpr int SLOTS = NT / 2;
  static_assert((Q / RAD) % SLOTS == 0, "butterflies must tile the half-block");
  constexpr int PER = (Q / RAD) / SLOTS;
  constexpr int SF = padded_len(Q);
  constexpr bool STASH = (SFW & kStash) != 0 && PER > 1;
  constexpr bool CARRYS = (SFW & kCarry) != 0;
  constexpr int SCOL = tm_total((int)sizeof(R), Q, NT);
  PassRows<R, Q, NT, NSF, SFW> rows;
  rows.fetch(twHead);
  Cx<R> v[PER][RAD];
  const int tid = ltid<NT>() + *zero;
  Cx<R>* Fp = F + fpol<NT>(tid) * SF;
  const int jb = fbase<NT>(tid);
#pragma unroll
  for (int p = 0; p < PER; ++p) {
    const int j = jb + p * SLOTS;
    const Cx<R>* b = Fp + pad(j);
#pragma unroll
    for (int r = 0; r < RAD; ++r) v[p][r] = b[pad(r * LR)];
    {
      const Cx<R>* w = rows.row(p);
#pragma unroll
      for (int r = 1; r < RAD; ++r) v[p][r] = cmul(v[p][r], w[r]);
    }
    dft_reg<R, RAD, false>(v[p]);
    // natural output r sits at j + r*LR in v[bitrev(r)]: apply the phasor
    // and hand it to the inverse butterfly as its input r
    Cx<R> u[RAD];
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
#ifdef CB_PHASOR_STUB  // timing experiment only (wrong results): what the phasor loads cost
      u[r] = cmul(v[p][bitrev<RAD>(r)], mk((R)(1.0 / Q), (R)(1e-3 * r / Q)));
#else
      u[r] = cmul(v[p][bitrev<RAD>(r)], ldg_na(ph + j + r * LR));
#endif
    }
    dft_reg<R, RAD, true>(u);
#pragma unroll
    for (int r = 0; r < RAD; ++r) v[p][r] = u[r];
    if constexpr (STASH) {
      if (p < PER - 1)
        tm_stash_store<R, RAD>(tm_lane_base(cb_tm_base), stash_col<R, RAD, PER, CARRYS>(SCOL, p), v[p]);
    }
  }
  if constexpr (STASH) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  pass_sync<SFW, NT>();
#pragma unroll
  for (int pp = 0; pp < PER; ++pp) {
    const int p = STASH ? (pp == 0 ? PER - 1 : pp - 1) : pp;
    if constexpr (STASH) {
      if (pp > 0)
        tm_stash_load<R, RAD>(tm_lane_base(cb_tm_base), stash_col<R, RAD, PER, CARRYS>(SCOL, p), v[p]);
    }
    const int j = jb + p * SLOTS;
    Cx<R>* b = Fp + pad(j * RAD);  // inverse first pass: NS = 1, d0 = R*j
#pragma unroll
    for (int r = 0; r < RAD; ++r) b[pad(r)] = v[p][bitrev<RAD>(r)];
  }
  pass_sync<SFW, NT>();
}

// Single-array pass for the half-length real-transform FFTs. Passes with
// fewer butterflies than threads run on the leading whole warps only; those
// synchronise between load and store with a named barrier, and a full
// barrier ends the pass so no warp runs ahead into a later pass whose named
// barrier expects a different thread count.
template <typename R, int Q, int L, int NT, int NS, bool INV, int HS, class Rows, class NextRows>
__device__ __forceinline__ void fft1_pass(Cx<R>* __restrict__ buf, const Cx<R>* __restrict__ twp,
                                          const volatile int* zero, Rows& rows, NextRows& next) {
  constexpr int RAD = sched_radix(L, NS, HS);
  constexpr int LR = L / RAD;
  constexpr int NB = L / RAD;
  const int tid = ltid<NT>() + *zero;
  auto body_load = [&](int j, Cx<R>* v, const Cx<R>* w) {
    const Cx<R>* b = buf + pad(j);
#pragma unroll
    for (int r = 0; r < RAD; ++r) v[r] = b[pad(r * LR)];
    if constexpr (NS > 1) {
#pragma unroll
      for (int r = 1; r < RAD; ++r) v[r] = INV ? cmulc(v[r], w[r]) : cmul(v[r], w[r]);
    }
    dft_reg<R, RAD, INV>(v);
  };
  auto body_store = [&](int j, const Cx<R>* v) {
    Cx<R>* b = buf + pad((j / NS) * NS * RAD + j % NS);
#pragma unroll
    for (int r = 0; r < RAD; ++r) b[pad(r * NS)] = v[bitrev<RAD>(r)];
  };
  if constexpr (NB >= NT) {
    static_assert(NB % NT == 0, "butterflies must tile the block");
    constexpr int PER = NB / NT;
    Cx<R> v[PER][RAD];
#pragma unroll
    for (int p = 0; p < PER; ++p) body_load(bfly<L, NS, RAD>(tid + p * NT), v[p], rows.row(p));
    pass_sync<HS, NT>();
#pragma unroll
    for (int p = 0; p < PER; ++p) body_store(bfly<L, NS, RAD>(tid + p * NT), v[p]);
    next.fetch(twp);
    pass_sync<HS, NT>();
  } else {
    // fewer butterflies than threads: the leading whole warps run the pass
    // and synchronise between load and store with a named barrier; the full
    // barrier at the end keeps any warp from running ahead into a later
    // pass whose named barrier expects a different thread count
    constexpr int ACT = (NB + 31) / 32 * 32;
    if (tid < ACT) {
      Cx<R> v[RAD];
      const bool on = (NB % 32 == 0) || tid < NB;
      const Cx<R>* w = rows.row(0);  // warp-converged (TMEM)
      if (on) body_load(tid, v, w);
      // (several groups per CTA: one id per group, after the groups' pass
      // ids 1..P, whether the pass ends on a group or a CTA barrier)
      bar_named((int)blockDim.x > NT ? 1 + (int)(blockDim.x / NT) + (int)threadIdx.x / NT : 1, ACT);
      if (on) body_store(tid, v);
    }
    next.fetch(twp);
    pass_sync<HS, NT>();
  }
}

template <typename R, int Q, int L, int NT, int NS, bool INV, int HS>
struct Fft1Run {
  using Rows = PassRows<R, L, NT, NS, HS>;
  static __device__ __forceinline__ void run(Cx<R>* buf, const Cx<R>* twp, const volatile int* z,
                                             Rows& rows) {
    constexpr int NS2 = NS * sched_radix(L, NS, HS);
    PassRows<R, L, NT, NS2, HS> next;
    fft1_pass<R, Q, L, NT, NS, INV, HS>(buf, twp, z, rows, next);
    Fft1Run<R, Q, L, NT, NS2, INV, HS>::run(buf, twp, z, next);
  }
};
template <typename R, int Q, int L, int NT, bool INV, int HS>
struct Fft1Run<R, Q, L, NT, L, INV, HS> {
  static __device__ __forceinline__ void run(Cx<R>*, const Cx<R>*, const volatile int*,
                                             PassRows<R, L, NT, L, HS>&) {}
};

// Half-length FFT of buf (HS: kHalf, or kHalf | kTM with TMEM twiddles).
template <typename R, int Q, int L, int NT, bool INV, int HS = kHalf>
__device__ __forceinline__ void fft1(Cx<R>* buf, const Cx<R>* twp, const volatile int* z) {
  PassRows<R, L, NT, 1, HS> none;
  Fft1Run<R, Q, L, NT, 1, INV, HS>::run(buf, twp, z, none);
}

// ------------------------------------------------------------------------

template <typename R>
struct Params {
  const Cx<R>* in;
  Cx<R>* out;
  int64_t in_bstride, in_pstride, in_origin;
  int64_t out_bstride, out_pstride, out_origin;
  int64_t n;        // circular period of the waveform
  int64_t b0;       // first global block index of this launch
  int64_t nb;       // blocks per waveform in this launch
  int64_t keep;     // block_size - overlap
  int64_t half;     // overlap / 2
  const Cx<R>* phasor;     // [n_tab][P][Q], carries 1/Q
  const Cx<R>* phasor_rev; // the same rows permuted to cbessfm_ip_kernel's bin order
                           // (ip_rev_index), or null where that kernel does not apply
  const int* ph_index;     // [n_steps + 1]
  const Cx<R>* mimo;       // [n_sets][P][Q/2+1], S_h with the 3/2 XPM weight folded
  const R* theta_scale;    // [n_sets][n_steps], carries 1/Q
  int n_sets;              // coefficient sets; waveform w uses set w % n_sets
  const Cx<R>* twQ;        // [Q]   exp(-2 pi i m / Q)
  const Cx<R>* twN;        // [P*Q] exp(-2 pi i m / (P Q))
  const Cx<R>* twp;        // per-pass rows, layout twp_base()
  const Cx<R>* rot_tab;    // [kRotTab] exp(i k / kRotDen) (complex128 plans), else null
  int n_steps;
  int64_t cid0;            // first cluster index of this launch chunk
  // persistent launches of the cluster kernel (null: one block per cluster):
  // each cluster claims blocks cid0 + atomicAdd(work, 1) until `total`
  unsigned long long* work;
  int64_t total;
  int kernel_pref;         // 0: choose by grid size, 1: cluster kernel (several
                           // launches in flight, cbessfm_run_host)
  long long* dbg;          // phase clocks of CTA 0 (CB_PHASE_PROFILE builds only)
};

// Q/8 threads: on the length-Q field FFTs each half-warp takes one
// polarisation and each thread one radix-16 butterfly per pass.
template <typename R, int Q>
__host__ __device__ constexpr int threads_for() {
  return Q / 8;
}

#ifndef CB_FLOAT_THREADS
#define CB_FLOAT_THREADS 1024
#endif
// Resident CTAs per SM the register budget is sized for.
template <typename R, int Q>
__host__ __device__ constexpr int min_blocks() {
  return (sizeof(R) == 4 ? CB_FLOAT_THREADS : 512) / threads_for<R, Q>() > 1
             ? (sizeof(R) == 4 ? CB_FLOAT_THREADS : 512) / threads_for<R, Q>()
             : 1;
}

// TMEM columns per CTA: the whole 512 shared by the CTAs the register
// budget makes resident (the launch enforces that residency with its shared
// memory request). Transforms read their twiddles from TMEM when all rows
// fit (FP32 and FP64 for Q = 2048 and 4096).
__host__ __device__ constexpr bool defined_no_tmem() {
#ifdef CB_NO_TMEM
  return true;
#else
  return false;
#endif
}
#ifndef CB_NO_TMEM
template <typename R, int Q>
__host__ __device__ constexpr int tm_cols() {
  int c = 32;
  while (c * 2 * min_blocks<R, Q>() <= 512) c *= 2;
  return c * min_blocks<R, Q>() <= 512 ? c : 0;
}
template <typename R, int Q>
__host__ __device__ constexpr bool tm_on() {
  return tm_cols<R, Q>() >= 32 && tm_total((int)sizeof(R), Q, threads_for<R, Q>()) <= tm_cols<R, Q>();
}
#else
template <typename R, int Q>
__host__ __device__ constexpr int tm_cols() { return 0; }
template <typename R, int Q>
__host__ __device__ constexpr bool tm_on() { return false; }
#endif

// The rotation table (RotationTabHook) rides in the shared memory the TMEM
// kernels claim anyway (1/min_blocks of the SM, csrc/cbessfm_launch.cuh):
// complex128 with TMEM rows, i.e. N' = 2048 and 4096.
#ifndef CB_ROT_TAB
#define CB_ROT_TAB 1
#endif
template <typename R, int Q>
__host__ __device__ constexpr bool rot_tab_on() {
  return CB_ROT_TAB && sizeof(R) == 8 && tm_on<R, Q>();
}

// MIMO slice of CTA c: bins [mimo_lo(c), mimo_lo(c+1)) of the H+1 rfft bins.
__host__ __device__ constexpr int mimo_lo(int c, int P, int H) { return (c * (H + 1)) / P; }
__host__ __device__ constexpr int mimo_slice_max(int P, int H) { return (H + 1 + P - 1) / P; }

// RB (P > 1) receives the P intensity-spectrum slices this CTA's MIMO
// needs; IS + RB also stage one polarisation row in the outer exchanges.
template <int Q>
__host__ __device__ constexpr int rb_len(int P) {
  return P * mimo_slice_max(P, Q / 2) > padded_len(Q) - padded_len(Q / 2 + 1)
             ? P * mimo_slice_max(P, Q / 2)
             : padded_len(Q) - padded_len(Q / 2 + 1);
}

template <typename R, int Q>
__host__ __device__ constexpr size_t smem_bytes(int P) {
  // F: 2 padded polarisation rows; IS: padded spectrum (Q/2+1 bins)
  return sizeof(Cx<R>) *
         (size_t)(2 * padded_len(Q) + padded_len(Q / 2 + 1) + (P > 1 ? rb_len<Q>(P) : 0) +
                  (rot_tab_on<R, Q>() ? kRotTab : 0));
}

// Position of global FFT bin g (of N = P*Q) in the subband layout:
// shifted s = (g + N/2) mod N, subband i = s / Q, local j = s mod Q,
// ifftshift'd storage m = (j + Q/2) mod Q   (dbp.py:387-389).
template <int P, int Q>
__device__ __forceinline__ void bin_home(int g, int& i, int& m) {
  constexpr int N = P * Q;
  int s = g + N / 2;
  if (s >= N) s -= N;
  i = s / Q;
  m = (s % Q + Q / 2) % Q;
  CB_CHECK(g >= 0 && g < N && i >= 0 && i < P && m >= 0 && m < Q);
}

template <typename R, int P, int Q>
__global__ void __launch_bounds__(threads_for<R, Q>(), min_blocks<R, Q>())
    cbessfm_block_kernel(const Params<R> prm) {
  constexpr int NT = threads_for<R, Q>();
  constexpr int H = Q / 2;
  constexpr int SF = padded_len(Q);      // stride between x and y in F

  extern __shared__ __align__(16) unsigned char smem_raw[];
  CB_POISON_SMEM(smem_raw);
  Cx<R>* F = reinterpret_cast<Cx<R>*>(smem_raw);
  Cx<R>* IS = F + 2 * SF;
  // TS (theta_hat, then theta) reuses IS: a remote CTA writes bin k of it
  // only after it received this CTA's I_hat[k], whose computation was the
  // last read of IS[k] (the untangle reads each slot once)
  Cx<R>* TS = IS;
  Cx<R>* RB = IS + padded_len(H + 1);  // P > 1 only
  constexpr int SLM = mimo_slice_max(P, H);
  constexpr bool ROTTAB = rot_tab_on<R, Q>();
  Cx<R>* RT = RB + (P > 1 ? rb_len<Q>(P) : 0);  // rotation table (ROTTAB only)
  if constexpr (ROTTAB) {
    // (ordered before its first use by the barrier after the block load)
    for (int i = threadIdx.x; i < kRotTab; i += threads_for<R, Q>()) RT[i] = ldg(prm.rot_tab + i);
  }

  __shared__ int s_zero;
  __shared__ uint64_t s_bar[2];  // [0]: intensity slices in RB, [1]: theta_hat in TS
  if (threadIdx.x == 0) {
    s_zero = 0;
    if constexpr (P > 1) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      mbar_init_fence();
    }
  }
  constexpr bool TMON = tm_on<R, Q>();
  // field transforms: inverse (IFFT, outer) and forward (in-step FFT)
  // schedules; half-length transforms
  constexpr int FI = TMON ? (kMid | kTM) : kTail;
  constexpr int FF = TMON ? (kMid | kTM) : kHead;
  // radix-8 half-length passes from Q = 2048 (measured: c64 -1.3 %, c128
  // -2.5 % per step at Q = 2048 vs radix 4, though a pass then keeps only
  // half the CTA's threads busy)
#ifndef CB_HALF_R4  // experiment knob: 1 = radix-4 half-length passes at every Q
#define CB_HALF_R4 0
#endif
  constexpr int HS = kHalf | (TMON ? kTM : 0) | (Q >= 2048 && !CB_HALF_R4 ? kWide : 0);
  if constexpr (TMON) {
    // allocate this CTA's TMEM columns (warp 0) and copy the twiddle rows in
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_addr(&cb_tm_base)), "n"(tm_cols<R, Q>()));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    tm_fill_sched<R, Q, NT, FI, 1>(prm.twp + twp_base(Q, kMid));
    tm_fill_sched<R, Q, NT, HS, 1>(prm.twp + twp_base(Q, HS));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    // the barrier after the block load orders these stores before every
    // tcgen05.ld of another warp (fence::after_thread_sync there)
  }
  const int tid = threadIdx.x;
  const int rank = (P > 1) ? (int)(blockIdx.x % P) : 0;
  // Persistent launches (prm.work set): the grid holds about as many
  // clusters as fit the GPU at once and each claims block after block from
  // a launch-wide counter -- rank 0 claims, the others read its slot over
  // DSMEM. The TMEM twiddle rows are filled once per CTA instead of once per
  // block, and no cluster waits on the scheduler between blocks. Clusters
  // the GPU starts late find the counter spent and exit.
  __shared__ long long s_cid[3];  // [it & 1]: claimed by rank 0, [2]: this CTA's block
  const bool persist = prm.work != nullptr;
  if (persist) {
    if (rank == 0 && tid == 0) s_cid[0] = (long long)atomicAdd(prm.work, 1ull);
    if constexpr (P > 1) {
      cg::this_cluster().sync();
    } else {
      __syncthreads();
    }
  }
  for (int it = 0;; ++it) {
    int64_t cid;
    if (persist) {
      if (tid == 0) {
        long long c = s_cid[it & 1];
        if constexpr (P > 1) {
          if (rank != 0) c = *cg::this_cluster().map_shared_rank(&s_cid[it & 1], 0);
        }
        s_cid[2] = c;
      }
      __syncthreads();
      cid = s_cid[2];
      if (cid >= prm.total) break;
      // claim the next block now; the other CTAs read it after this block's
      // last cluster barrier (step 5), which orders the store before them
#ifndef CB_NO_PREFETCH_NEXT
      // ... and pull its window towards L2 while this block computes (warp 0
      // of rank 0; whole waveforms only: shards index a shorter slice).
      // configs[4] c128 361.4 -> 359.1 ms per step (tools/gpu/r2_s4_pf.sh).
      if (rank == 0 && tid < 32) {
        long long nxt = 0;
        if (tid == 0) {
          nxt = (long long)atomicAdd(prm.work, 1ull);
          s_cid[(it + 1) & 1] = nxt;
        }
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
        if (nxt < prm.total && prm.in_origin == 0) {
          const int64_t c2 = nxt + prm.cid0;
          const int64_t wv2 = c2 / prm.nb, b2 = prm.b0 + c2 % prm.nb;
          int64_t st2 = (b2 * prm.keep - prm.half) % prm.n;
          if (st2 < 0) st2 += prm.n;
          if (st2 + (int64_t)P * Q <= prm.n) {
            constexpr uint32_t piece = (uint32_t)((size_t)P * Q * sizeof(Cx<R>) / 32);
            // (the bulk prefetch wants 16-byte aligned addresses: complex64
            // windows may start on an odd sample, so round down)
            static_assert(piece % 16 == 0, "prefetch pieces are whole 16-byte units");
            const uintptr_t a0 =
                reinterpret_cast<uintptr_t>(prm.in + wv2 * prm.in_bstride + st2) + (size_t)tid * piece;
            const uintptr_t a1 = a0 + (size_t)prm.in_pstride * sizeof(Cx<R>);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0 & ~(uintptr_t)15),
                         "r"(piece) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a1 & ~(uintptr_t)15),
                         "r"(piece) : "memory");
          }
        }
      }
#else
      if (rank == 0 && tid == 0) s_cid[(it + 1) & 1] = (long long)atomicAdd(prm.work, 1ull);
#endif
      cid += prm.cid0;
    } else {
      if (it) break;
      cid = prm.cid0 + blockIdx.x / P;
    }
    // mbarrier phase parity continues across the blocks of a CTA
    const int ph0 = (int)(((int64_t)it * prm.n_steps) & 1);
    const int64_t wv = cid / prm.nb;
    const int64_t b = prm.b0 + cid % prm.nb;
    const int64_t n = prm.n;
    const int64_t cset = prm.n_sets > 1 ? wv % prm.n_sets : 0;
    const Cx<R>* __restrict__ mimo = prm.mimo + cset * (int64_t)P * (H + 1);
    const R* __restrict__ theta_scale = prm.theta_scale + cset * prm.n_steps;

    const Cx<R>* __restrict__ twQ = prm.twQ;
    const Cx<R>* __restrict__ twN = prm.twN;
    const Cx<R>* __restrict__ twpT = prm.twp + twp_base(Q, FI);  // field IFFT / outer
    const Cx<R>* __restrict__ twpF = prm.twp + twp_base(Q, FF);  // in-step field FFT
    const Cx<R>* __restrict__ twpH = prm.twp + twp_base(Q, HS);  // half-length FFTs

    CB_MARK(0);
    CB_TIMELINE(0);
    // ---- 1. load the polyphase component u[rank + P*t2] of the circular
    //         window starting at (b*keep - half) mod n (dbp.py:473-475)
    {
      int64_t start = (b * prm.keep - prm.half) % n;
      if (start < 0) start += n;
      start -= prm.in_origin;
      if (start < 0) start += n;
      const Cx<R>* src = prm.in + wv * prm.in_bstride;
      for (int t2 = tid; t2 < Q; t2 += NT) {
        int64_t idx = start + rank + (int64_t)P * t2;
        if (idx >= n) idx -= n;
        CB_CHECK(idx >= 0 && idx < n);
        F[pad(t2)] = src[idx];
        F[SF + pad(t2)] = src[prm.in_pstride + idx];
      }
    }
    __syncthreads();
    if constexpr (TMON) asm volatile("tcgen05.fence::after_thread_sync;");

    const size_t ph_tab = (size_t)P * Q;
    CB_MARK(1);

    // ---- 2. outer transform, polyphase part: FFT_Q of both polarisations.
    //         For P == 1 the subband layout is the natural FFT order
    //         (bin_home is the identity) and the first phasor is fused in.
    if constexpr (P == 1) {
      PhasorHook<R> ph0;
      ph0.ph = prm.phasor + (size_t)prm.ph_index[0] * ph_tab;
      fft2<R, Q, NT, FI, false, NoHook, PhasorHook<R>>(F, twpT, &s_zero, NoHook(), ph0);
    } else {
      fft2<R, Q, NT, FI, false>(F, twpT, &s_zero);
      // ---- 3. cross-subband radix-P stage over DSMEM: CTA c produces bins
      //         Q*k1 + k2 for k2 in its slice and every k1, and writes each to
      //         the CTA that owns it in the fftshift'd subband layout. Row 0's
      //         results are staged in the owner's idle IS/RB region and row 1's
      //         land in the owner's row 0 once every CTA has read it, so no CTA
      //         overwrites fields another CTA still reads (3 cluster barriers).
      //         The polarisation rows come out swapped; everything in the step
      //         loop is symmetric in x and y, and step 5 swaps them back.
      cg::cluster_group cluster = cg::this_cluster();
      const int lo = (rank * Q) / P, hi = ((rank + 1) * Q) / P;
      const R invP = (R)1 / (R)P;
      const Cx<R>* ph0 = prm.phasor + (size_t)prm.ph_index[0] * ph_tab;
      Cx<R>* S = IS;  // staging: padded_len(Q) entries fit in IS + RB
      cluster.sync();
      for (int pol = 0; pol < 2; ++pol) {
        for (int k2 = lo + tid; k2 < hi; k2 += NT) {
          Cx<R> bv[P];
  #pragma unroll
          for (int r = 0; r < P; ++r) {
            const Cx<R>* rf = cluster.map_shared_rank(F, r);
            Cx<R> v = rf[pol * SF + pad(k2)];
            if (r) v = cmul(v, ldg(twN + r * k2));
            bv[r] = v;
          }
  #pragma unroll
          for (int k1 = 0; k1 < P; ++k1) {
            Cx<R> s = bv[0];
  #pragma unroll
            for (int r = 1; r < P; ++r) s = s + cmul(bv[r], ldg(twN + ((r * k1) % P) * Q));
            int i, m;
            bin_home<P, Q>(Q * k1 + k2, i, m);
            const Cx<R> w = ldg(ph0 + (size_t)i * Q + m);
            // row 0 results go to the staging area, row 1 results into the
            // owner's row 0 (consumed by then): the rows come out swapped
            Cx<R>* dst = cluster.map_shared_rank(pol ? F : S, i);
            dst[pad(m)] = cmul(scale(s, invP), w);
          }
        }
        cluster.sync();
      }
      // every remote read of row 1 is done: move the staged row-0 results in
      for (int t = tid; t < Q; t += NT) F[SF + pad(t)] = S[pad(t)];
      __syncthreads();
      // S spans IS and RB, where the other CTAs' st.async pushes of step 0
      // land: they may not start before every CTA of the cluster has read
      // its staged row out. Split cluster barrier: arrive here, wait before
      // the step loop (behind the first IFFT, so nobody actually waits). A
      // CTA running a few microseconds ahead of a descheduled one did
      // overwrite it: 1-2 corrupted blocks per 72 768-block launch.
      cluster_arrive();
    }

    CB_MARK(2);
    const Cx<R>* ph_rank = prm.phasor + (size_t)rank * Q;  // this CTA's subband rows
    R* Ireal = reinterpret_cast<R*>(IS);
    const R* Treal = reinterpret_cast<const R*>(TS);

    // ---- 4. nonlinear steps (dbp.py:394-398). The subband IFFT
    //         (normalisation folded into the phasor) also writes, in its last
    //         pass, I = |x|^2 + |y|^2 packed as z[t] = I[2t] + i I[2t+1]. The
    //         first step's IFFT runs here; later steps' IFFTs start inside
    //         the previous step's fft2_boundary.
    IntensityHook<R> ih;
    ih.I = Ireal;
    if (prm.n_steps > 0)
      fft2<R, Q, NT, FI, true, NoHook, IntensityHook<R>>(F, twpT, &s_zero, NoHook(), ih);
    CB_MARK(3);
    if constexpr (P > 1) cluster_wait();  // pairs with the arrive after step 3's copy
    constexpr int KU = (H / 2 + 1 + NT - 1) / NT;  // untangle/twist bins per thread
    for (int st = 0; st < prm.n_steps; ++st) {
      // per-step scalars issued at the top of the step: their L2 latency
      // overlaps the intensity transforms instead of stalling the rotation
      // FFT and the boundary pass
      const R tsc_st = theta_scale[st];
      const int phi_next = prm.ph_index[st + 1];  // n_steps + 1 entries
      // W_Q^k of this thread's untangle/twist bins, issued before the FFT so
      // the L2 latency hides behind it (the same k serve both)
      Cx<R> twk[KU];
  #pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = tid + u * NT;
        twk[u] = (k <= H / 2) ? ldg(twQ + k) : mk((R)1, (R)0);
      }
      // CB_STUB_NLPR (timing experiments only, wrong results): 1 skips the two
      // half-length transforms, 2 also the untangle / MIMO exchange / twist
#ifndef CB_STUB_NLPR
#define CB_STUB_NLPR 0
#endif
      if (CB_STUB_NLPR < 1) fft1<R, Q, H, NT, false, HS>(IS, twpH, &s_zero);
      CB_MARK(8 + 8 * st + 0);
      if (CB_STUB_NLPR < 2) {

      // r2c untangle: I_hat[k], k = 0..H (numpy rfft, dbp.py:194). For P > 1
      // each bin goes straight from registers to the CTA whose MIMO slice
      // holds it (st.async into its RB, completing on its mbarrier); for
      // P == 1 it is written back in place.
      if constexpr (P > 1) {
        if (tid == 0) {
          const int len = mimo_lo(rank + 1, P, H) - mimo_lo(rank, P, H);
          mbar_expect(&s_bar[0], (uint32_t)(P * len * sizeof(Cx<R>)));
          mbar_expect(&s_bar[1], (uint32_t)((H + 1) * sizeof(Cx<R>)));
        }
      }
      auto emit = [&](int k, Cx<R> v) {
        if constexpr (P > 1) {
          int c = (k * P) / (H + 1);
          if (mimo_lo(c + 1, P, H) <= k) ++c;
          const uint32_t dst = cluster_addr(smem_addr(RB + rank * SLM + (k - mimo_lo(c, P, H))), c);
          push(dst, v, cluster_addr(smem_addr(&s_bar[0]), c));
        } else {
          IS[pad(k)] = v;
        }
      };
  #pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = tid + u * NT;
        if (k > H / 2) break;
        if (k == 0) {
          const Cx<R> z = IS[pad(0)];
          emit(0, mk(z.x + z.y, (R)0));
          emit(H, mk(z.x - z.y, (R)0));
        } else {
          const Cx<R> a = IS[pad(k)];
          const Cx<R> bq = conj(IS[pad(H - k)]);
          const Cx<R> e = scale(a + bq, (R)0.5);
          const Cx<R> dd = a - bq;                           // 2i * O[k]
          const Cx<R> o = mk(dd.y * (R)0.5, -dd.x * (R)0.5); // O[k]
          const Cx<R> wo = cmul(o, twk[u]);
          emit(k, e + wo);
          if (k != H - k) emit(H - k, conj(e - wo));
        }
      }

      CB_MARK(8 + 8 * st + 1);
      // MIMO coupling (dbp.py:195): theta_hat_i[k] = sum_l T[i,l,k] I_hat_l[k]
      if constexpr (P > 1) {
        const int lo = mimo_lo(rank, P, H), hi = mimo_lo(rank + 1, P, H);
        const uint32_t ts_local = smem_addr(TS);
        const uint32_t bar_t = smem_addr(&s_bar[1]);
        for (int k = lo + tid; k < hi; k += NT) {
          Cx<R> sv[P];
  #pragma unroll
          for (int l = 0; l < P; ++l) sv[l] = ldg_na(mimo + (size_t)l * (H + 1) + k);
          mbar_wait(&s_bar[0], (st + ph0) & 1);
          Cx<R> iv[P];
  #pragma unroll
          for (int l = 0; l < P; ++l) iv[l] = RB[l * SLM + (k - lo)];
  #pragma unroll
          for (int i = 0; i < P; ++i) {
            Cx<R> acc = mk((R)0, (R)0);
  #pragma unroll
            for (int l = 0; l < P; ++l) {
              acc = l >= i ? cmac(acc, sv[l - i], iv[l]) : cmacc(acc, sv[i - l], iv[l]);
            }
            push(cluster_addr(ts_local + (uint32_t)(pad(k) * sizeof(Cx<R>)), i), acc,
                 cluster_addr(bar_t, i));
          }
        }
        CB_MARK(8 + 8 * st + 2);
        mbar_wait(&s_bar[1], (st + ph0) & 1);
      } else {
        __syncthreads();
        for (int k = tid; k <= H; k += NT) TS[pad(k)] = cmul(ldg(mimo + k), IS[pad(k)]);
        __syncthreads();
      }

      CB_MARK(8 + 8 * st + 3);
      // c2r pre-twist in place (numpy irfft ignores Im of bins 0 and H)
  #pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = tid + u * NT;
        if (k > H / 2) break;
        if (k == 0) {
          const R x0 = TS[pad(0)].x, xh = TS[pad(H)].x;
          TS[pad(0)] = mk(x0 + xh, x0 - xh);
        } else {
          const Cx<R> a = TS[pad(k)];                 // X[k]
          const Cx<R> c = conj(TS[pad(H - k)]);       // X[k + H]
          const Cx<R> wk = twk[u];                    // W^k
          const Cx<R> s = a + c;
          const Cx<R> dd = cmulc(a - c, wk);          // W^-k (a - c)
          TS[pad(k)] = mk(s.x - dd.y, s.y + dd.x);    // s + i dd
          if (k != H - k) {
            // Z[H-k] = (X[H-k] + X[Q-k]) + i W^-(H-k) (X[H-k] - X[Q-k])
            const Cx<R> a2 = conj(c);                 // X[H-k]
            const Cx<R> c2 = conj(a);                 // X[Q-k]
            const Cx<R> s2 = a2 + c2;
            const Cx<R> w2 = mk(-wk.x, wk.y);         // W^(H-k) = -conj(W^k)
            const Cx<R> d2 = cmulc(a2 - c2, w2);
            TS[pad(H - k)] = mk(s2.x - d2.y, s2.y + d2.x);
          }
        }
      }
      }  // CB_STUB_NLPR < 2
      __syncthreads();
      CB_MARK(8 + 8 * st + 4);
      if (CB_STUB_NLPR < 1) fft1<R, Q, H, NT, true, HS>(TS, twpH, &s_zero);
      CB_MARK(8 + 8 * st + 5);

      // rotation exp(-i theta) fused into the first pass of the subband FFT
      // (dbp.py:208, :398); its last pass either fuses with the next phasor
      // and the next step's IFFT (dbp.py:395-396) or, after the last step,
      // applies the final phasor (dbp.py:399)
      using Rot = typename std::conditional<ROTTAB, RotationTabHook<R>, RotationHook<R>>::type;
      Rot rot;
      rot.th = Treal;
      rot.scale = CB_STUB_NLPR ? (R)0 : tsc_st;
      if constexpr (ROTTAB) rot.tab = RT;
      const Cx<R>* ph_next = ph_rank + (size_t)phi_next * ph_tab;
      if (st + 1 < prm.n_steps) {
        fft2<R, Q, NT, FF, false, Rot, NoHook, 1, Q / sched_radix(Q, 1, FI)>(
            F, twpF, &s_zero, rot);
        CB_MARK(8 + 8 * st + 6);
        fft2_boundary<R, Q, NT, FI, FF>(F, twpF, ph_next, &s_zero);
        CB_MARK(8 + 8 * st + 7);
        fft2<R, Q, NT, FI, true, NoHook, IntensityHook<R>, sched_radix(Q, 1, FI)>(
            F, twpT, &s_zero, NoHook(), ih);
      } else {
        PhasorHook<R> ph1;
        ph1.ph = ph_next;
        fft2<R, Q, NT, FF, false, Rot, PhasorHook<R>>(F, twpF, &s_zero, rot, ph1);
      }
    }

    CB_MARK(4);
    // ---- 5. merge + outer IFFT (dbp.py:400-401): CTA c gathers, for k2 in
    //         its slice, the P bins Q*k1 + k2 from their owners, applies the
    //         inverse radix-P stage and the twiddle, and hands polyphase
    //         component n1 to CTA n1 (staged as in step 3, which swaps the
    //         rows back).
    if constexpr (P > 1) {
      cg::cluster_group cluster = cg::this_cluster();
      const int lo = (rank * Q) / P, hi = ((rank + 1) * Q) / P;
      Cx<R>* S = IS;
      cluster.sync();
      for (int pol = 0; pol < 2; ++pol) {
        for (int k2 = lo + tid; k2 < hi; k2 += NT) {
          Cx<R> xv[P];
  #pragma unroll
          for (int k1 = 0; k1 < P; ++k1) {
            int i, m;
            bin_home<P, Q>(Q * k1 + k2, i, m);
            const Cx<R>* rf = cluster.map_shared_rank(F, i);
            xv[k1] = rf[pol * SF + pad(m)];
          }
  #pragma unroll
          for (int n1 = 0; n1 < P; ++n1) {
            Cx<R> s = xv[0];
  #pragma unroll
            for (int k1 = 1; k1 < P; ++k1) s = s + cmulc(xv[k1], ldg(twN + ((n1 * k1) % P) * Q));
            if (n1) s = cmulc(s, ldg(twN + n1 * k2));
            Cx<R>* dst = cluster.map_shared_rank(pol ? F : S, n1);
            dst[pad(k2)] = s;
          }
        }
        cluster.sync();
      }
      for (int t = tid; t < Q; t += NT) F[SF + pad(t)] = S[pad(t)];
      __syncthreads();
    }
    fft2<R, Q, NT, FI, true>(F, twpT, &s_zero);

    CB_MARK(5);
    CB_TIMELINE(1);
    // ---- 6. keep proc[half : half + span] (dbp.py:476-477)
    {
      const int64_t span = min(prm.keep, n - b * prm.keep);
      Cx<R>* dst = prm.out + wv * prm.out_bstride;
      const int64_t obase = b * prm.keep - prm.half - prm.out_origin;
      for (int t2 = tid; t2 < Q; t2 += NT) {
        const int64_t t = rank + (int64_t)P * t2;
        if (t >= prm.half && t < prm.half + span) {
          CB_CHECK(obase + t >= 0 && (prm.out_origin != 0 || obase + t < n));
          dst[obase + t] = F[pad(t2)];
          dst[prm.out_pstride + obase + t] = F[SF + pad(t2)];
        }
      }
    }
  }
  if constexpr (P > 1) {
    // rank 0's claim slots are read over DSMEM up to the last iteration
    if (persist) cg::this_cluster().sync();
  }
  if constexpr (TMON) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(cb_tm_base),
                   "n"(tm_cols<R, Q>()));
  }
}


// ------------------------------------------------------------------------
// One-block-per-CTA variant.
//
// With P subbands of Q = 2048 samples the P-CTA cluster kernel above holds
// 4 clusters' CTAs per SM, so one configs[1] waveform (143 blocks) needs two
// rounds and the second runs a quarter full. Here one CTA holds a whole
// overlap-save block: P groups of Q/16 threads, group s owning subband s
// (both polarisation rows and its intensity buffer, P * 43.5 KB of shared
// memory for P = 5), so one CTA fills an SM and 143 blocks run in one round
// on 148 SMs. The cross-subband steps need no cluster: the outer radix-P
// stages read all subbands from local shared memory (registers carry the
// inputs across one barrier, so no staging row is needed), and the MIMO
// reads every subband's intensity spectrum in place -- no DSMEM pushes, no
// mbarrier waits. Each thread runs two radix-16 butterflies per pass
// (96-register budget); the twiddle rows sit in TMEM as above (the P groups
// share lanes and rows).

template <typename R, int P, int Q>
__host__ __device__ constexpr size_t fat_smem_bytes() {
  return sizeof(Cx<R>) * (size_t)P * (2 * padded_len(Q) + padded_len(Q / 2 + 1));
}
template <typename R, int P, int Q>
__host__ __device__ constexpr bool fat_ok() {
#ifdef CB_NO_FAT
  return false;
#else
  // float, Q = 2048 (radix-4 half-length passes keep every group thread
  // busy), P subbands that fit one SM's shared memory
  return sizeof(R) == 4 && Q == 2048 && P >= 2 && fat_smem_bytes<R, P, Q>() <= 232448 - 1024;
#endif
}
template <int Q>
__host__ __device__ constexpr int fat_group() {
  return Q / 16;
}
__host__ __device__ constexpr int pow2_cols(int c) {
  int a = 32;
  while (a < c) a *= 2;
  return a;
}

template <typename R, int P, int Q>
__global__ void __launch_bounds__(P * fat_group<Q>(), 1) cbessfm_fat_kernel(const Params<R> prm) {
  constexpr int NT = fat_group<Q>();  // threads per subband group
  constexpr int NTC = P * NT;         // threads per CTA
  constexpr int H = Q / 2;
  constexpr int SF = padded_len(Q);
  constexpr int SG = 2 * SF + padded_len(H + 1);  // shared entries per group
  static_assert(NT % 128 == 0, "groups must start on a TMEM lane quarter");
  static_assert((H / 8) >= NT, "half-length passes must keep every thread busy");
  // TMEM: twiddle rows, then the butterfly parking of the P*NT/128 lane
  // sharers (at most 3 radix-8 or 1 radix-16 butterfly each)
  constexpr bool CARRY = CB_CARRY && sizeof(R) == 4;
  constexpr int TM_NEED = tm_total((int)sizeof(R), Q, NT) + (NTC / 128) * stash_stride<R>(CARRY);
  constexpr bool TMON = !defined_no_tmem() && TM_NEED <= 512;
  constexpr int COLS = pow2_cols(TM_NEED);
#ifndef CB_GB_FIELD
#define CB_GB_FIELD kGroupBar
#endif
#ifndef CB_GB_HALF
#define CB_GB_HALF kGroupBar
#endif
  constexpr int FC = CARRY ? kCarry : 0;
  constexpr int FI = (TMON ? (kMid | kTM | kStash | FC) : kTail) | CB_GB_FIELD;
  constexpr int FF = (TMON ? (kMid | kTM | kStash | FC) : kHead) | CB_GB_FIELD;
  constexpr int HS = kHalf | kWide | (TMON ? kTM : 0) | CB_GB_HALF;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  CB_POISON_SMEM(smem_raw);
  Cx<R>* const base = reinterpret_cast<Cx<R>*>(smem_raw);
  const int grp = (int)threadIdx.x / NT;  // subband of this thread's group
  const int tid = ltid<NT>();
  Cx<R>* F = base + grp * SG;
  Cx<R>* IS = F + 2 * SF;
  Cx<R>* TS = IS;
  __shared__ int s_zero;
  if (threadIdx.x == 0) s_zero = 0;
  if constexpr (TMON) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_addr(&cb_tm_base)), "n"(COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    tm_fill_sched<R, Q, NT, FI, 1>(prm.twp + twp_base(Q, kMid));
    tm_fill_sched<R, Q, NT, HS, 1>(prm.twp + twp_base(Q, HS));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  const int64_t cid = prm.cid0 + blockIdx.x;
  (void)cid;
  CB_MARK(0);
  const int64_t wv = cid / prm.nb;
  const int64_t b = prm.b0 + cid % prm.nb;
  const int64_t n = prm.n;
  const int64_t cset = prm.n_sets > 1 ? wv % prm.n_sets : 0;
  const Cx<R>* __restrict__ mimo = prm.mimo + cset * (int64_t)P * (H + 1);
  const R* __restrict__ theta_scale = prm.theta_scale + cset * prm.n_steps;
  const Cx<R>* __restrict__ twQ = prm.twQ;
  const Cx<R>* __restrict__ twN = prm.twN;
  const Cx<R>* __restrict__ twpT = prm.twp + twp_base(Q, FI);
  const Cx<R>* __restrict__ twpF = prm.twp + twp_base(Q, FF);
  const Cx<R>* __restrict__ twpH = prm.twp + twp_base(Q, HS);

  // ---- 1. load the circular window starting at (b*keep - half) mod n
  //         (dbp.py:473-475) with consecutive threads on consecutive
  //         samples (coalesced); sample t goes to polyphase row t mod P,
  //         position t / P
  {
    int64_t start = (b * prm.keep - prm.half) % n;
    if (start < 0) start += n;
    start -= prm.in_origin;
    if (start < 0) start += n;
    const Cx<R>* src = prm.in + wv * prm.in_bstride;
    for (int t = (int)threadIdx.x; t < P * Q; t += NTC) {
      int64_t idx = start + t;
      if (idx >= n) idx -= n;
      CB_CHECK(idx >= 0 && idx < n);
      const int r = t % P, t2 = t / P;
      Cx<R>* Fr = base + r * SG;
      Fr[pad(t2)] = src[idx];
      Fr[SF + pad(t2)] = src[prm.in_pstride + idx];
    }
  }
  // per-step scalars (theta scale, phasor table index) staged in shared
  // memory: read in the step loop right before the rotation FFT and the
  // boundary pass, where an L2 round trip would stall every warp
  constexpr int kStepCache = 256;
  __shared__ R s_tsc[kStepCache];
  __shared__ int s_phi[kStepCache + 1];
  for (int i = (int)threadIdx.x; i <= prm.n_steps && i <= kStepCache; i += NTC) {
    if (i < prm.n_steps && i < kStepCache) s_tsc[i] = theta_scale[i];
    s_phi[i] = prm.ph_index[i];
  }
  __syncthreads();
  if constexpr (TMON) asm volatile("tcgen05.fence::after_thread_sync;");
  CB_MARK(1);

  // ---- 2.-3. outer transform (dbp.py:387-389): FFT_Q per subband, then
  //         the radix-P stage across subbands. Thread-strided over k2: the P
  //         inputs Q*k1 + k2 are read into registers, a barrier, then the P
  //         outputs (x 1/P x first phasor) go to their subband homes in place.
  fft2<R, Q, NT, FI, false>(F, twpT, &s_zero);
  __syncthreads();  // the passes synchronise per group only
  constexpr int KPT = (Q + NTC - 1) / NTC;
  const R invP = (R)1 / (R)P;
  Cx<R> wP[P];  // W_P^m = twN[m Q]
#pragma unroll
  for (int m = 0; m < P; ++m) wP[m] = ldg(twN + m * Q);
  const Cx<R>* ph0 = prm.phasor + (size_t)prm.ph_index[0] * (size_t)P * Q;
  for (int pol = 0; pol < 2; ++pol) {
    Cx<R> bv[KPT][P];
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
      const int k2 = (int)threadIdx.x + u * NTC;
      if (k2 < Q) {
#pragma unroll
        for (int r = 0; r < P; ++r) {
          Cx<R> v = base[r * SG + pol * SF + pad(k2)];
          if (r) v = cmul(v, ldg(twN + r * k2));
          bv[u][r] = v;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
      const int k2 = (int)threadIdx.x + u * NTC;
      if (k2 < Q) {
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) {
          Cx<R> sm = bv[u][0];
#pragma unroll
          for (int r = 1; r < P; ++r) sm = sm + cmul(bv[u][r], wP[(r * k1) % P]);
          int i, m;
          bin_home<P, Q>(Q * k1 + k2, i, m);
          base[i * SG + pol * SF + pad(m)] = cmul(scale(sm, invP), ldg(ph0 + (size_t)i * Q + m));
        }
      }
    }
    __syncthreads();
  }

  CB_MARK(2);
  // ---- 4. nonlinear steps (dbp.py:394-398), as in the cluster kernel
  const Cx<R>* ph_grp = prm.phasor + (size_t)grp * Q;
  const size_t ph_tab = (size_t)P * Q;
  R* Ireal = reinterpret_cast<R*>(IS);
  const R* Treal = reinterpret_cast<const R*>(TS);
  IntensityHook<R> ih;
  ih.I = Ireal;
  if (prm.n_steps > 0)
    fft2<R, Q, NT, FI, true, NoHook, IntensityHook<R>>(F, twpT, &s_zero, NoHook(), ih);
  CB_MARK(3);
#ifndef CB_SPLIT_MIMO
  // One CTA phase per step between the half-length FFTs: thread k (k <= H/2)
  // owns the bin pair (k, H-k) of every subband -- r2c untangle, MIMO of both
  // bins, c2r pre-twist -- all in registers (the three are pair-local), so
  // there is one shared-memory round trip and two CTA barriers instead of
  // three of each. Same operations, same order as the three-phase form.
  constexpr int KP = (H / 2 + 1 + NTC - 1) / NTC;  // bin pairs per thread
  for (int st = 0; st < prm.n_steps; ++st) {
    Cx<R> wks[KP];
#pragma unroll
    for (int u = 0; u < KP; ++u) {
      const int kp = (int)threadIdx.x + u * NTC;
      wks[u] = kp <= H / 2 ? ldg(twQ + kp) : mk((R)1, (R)0);
    }
    fft1<R, Q, H, NT, false, HS>(IS, twpH, &s_zero);
    CB_MARK(8 + 8 * st + 0);
    __syncthreads();  // every subband's spectrum is read below
    CB_MARK(8 + 8 * st + 1);
#pragma unroll
    for (int u = 0; u < KP; ++u) {
      const int kp = (int)threadIdx.x + u * NTC;  // bin pair (kp, H - kp)
      if (kp > H / 2) break;
      const int kq = H - kp;
      const Cx<R> wk = wks[u];
      Cx<R> ia[P], ib[P];  // I_hat[kp], I_hat[kq] of every subband
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const Cx<R>* Il = base + l * SG + 2 * SF;
        // r2c untangle (numpy rfft, dbp.py:194)
        if (kp == 0) {
          const Cx<R> z = Il[pad(0)];
          ia[l] = mk(z.x + z.y, (R)0);
          ib[l] = mk(z.x - z.y, (R)0);
        } else {
          const Cx<R> a = Il[pad(kp)];
          const Cx<R> bq = conj(Il[pad(kq)]);
          const Cx<R> e = scale(a + bq, (R)0.5);
          const Cx<R> dd = a - bq;
          const Cx<R> o = mk(dd.y * (R)0.5, -dd.x * (R)0.5);
          const Cx<R> wo = cmul(o, wk);
          ia[l] = e + wo;
          ib[l] = kp == kq ? ia[l] : conj(e - wo);  // bin H/2 pairs with itself
        }
      }
      // MIMO coupling (dbp.py:195) of both bins
      Cx<R> ta[P], tb[P];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int k = half ? kq : kp;
        const Cx<R>* iv = half ? ib : ia;
        Cx<R> sv[P];
#pragma unroll
        for (int l = 0; l < P; ++l) sv[l] = ldg_na(mimo + (size_t)l * (H + 1) + k);
#pragma unroll
        for (int i = 0; i < P; ++i) {
          Cx<R> acc = mk((R)0, (R)0);
#pragma unroll
          for (int l = 0; l < P; ++l)
            acc = l >= i ? cmac(acc, sv[l - i], iv[l]) : cmacc(acc, sv[i - l], iv[l]);
          (half ? tb : ta)[i] = acc;
        }
      }
      // c2r pre-twist (numpy irfft ignores Im of bins 0 and H)
#pragma unroll
      for (int i = 0; i < P; ++i) {
        Cx<R>* Ti = base + i * SG + 2 * SF;
        if (kp == 0) {
          Ti[pad(0)] = mk(ta[i].x + tb[i].x, ta[i].x - tb[i].x);
        } else {
          const Cx<R> a = ta[i];
          const Cx<R> c = conj(tb[i]);
          const Cx<R> s2 = a + c;
          const Cx<R> dd = cmulc(a - c, wk);
          Ti[pad(kp)] = mk(s2.x - dd.y, s2.y + dd.x);
          if (kp != kq) {
            const Cx<R> a2 = conj(c);
            const Cx<R> c2 = conj(a);
            const Cx<R> s3 = a2 + c2;
            const Cx<R> w2 = mk(-wk.x, wk.y);
            const Cx<R> d2 = cmulc(a2 - c2, w2);
            Ti[pad(kq)] = mk(s3.x - d2.y, s3.y + d2.x);
          }
        }
      }
    }
    __syncthreads();
    CB_MARK(8 + 8 * st + 2);
    CB_MARK(8 + 8 * st + 3);
    CB_MARK(8 + 8 * st + 4);
#else
  constexpr int KU = (H / 2 + 1 + NT - 1) / NT;
  for (int st = 0; st < prm.n_steps; ++st) {
    Cx<R> twk[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int k = tid + u * NT;
      twk[u] = (k <= H / 2) ? ldg(twQ + k) : mk((R)1, (R)0);
    }
    fft1<R, Q, H, NT, false, HS>(IS, twpH, &s_zero);
    CB_MARK(8 + 8 * st + 0);
    // r2c untangle in place: I_hat[k], k = 0..H (numpy rfft, dbp.py:194)
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int k = tid + u * NT;
      if (k > H / 2) break;
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
        const Cx<R> wo = cmul(o, twk[u]);
        IS[pad(k)] = e + wo;
        if (k != H - k) IS[pad(H - k)] = conj(e - wo);
      }
    }
    __syncthreads();
    CB_MARK(8 + 8 * st + 1);
    // MIMO coupling (dbp.py:195) in place: bin k of every subband, one
    // thread per bin
    for (int k = (int)threadIdx.x; k <= H; k += NTC) {
      Cx<R> sv[P], iv[P];
#pragma unroll
      for (int l = 0; l < P; ++l) sv[l] = ldg_na(mimo + (size_t)l * (H + 1) + k);
#pragma unroll
      for (int l = 0; l < P; ++l) iv[l] = base[l * SG + 2 * SF + pad(k)];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        Cx<R> acc = mk((R)0, (R)0);
#pragma unroll
        for (int l = 0; l < P; ++l)
          acc = l >= i ? cmac(acc, sv[l - i], iv[l]) : cmacc(acc, sv[i - l], iv[l]);
        base[i * SG + 2 * SF + pad(k)] = acc;
      }
    }
    __syncthreads();
    CB_MARK(8 + 8 * st + 2);
    CB_MARK(8 + 8 * st + 3);
    // c2r pre-twist in place (numpy irfft ignores Im of bins 0 and H)
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int k = tid + u * NT;
      if (k > H / 2) break;
      if (k == 0) {
        const R x0 = TS[pad(0)].x, xh = TS[pad(H)].x;
        TS[pad(0)] = mk(x0 + xh, x0 - xh);
      } else {
        const Cx<R> a = TS[pad(k)];
        const Cx<R> c = conj(TS[pad(H - k)]);
        const Cx<R> wk = twk[u];
        const Cx<R> s2 = a + c;
        const Cx<R> dd = cmulc(a - c, wk);
        TS[pad(k)] = mk(s2.x - dd.y, s2.y + dd.x);
        if (k != H - k) {
          const Cx<R> a2 = conj(c);
          const Cx<R> c2 = conj(a);
          const Cx<R> s3 = a2 + c2;
          const Cx<R> w2 = mk(-wk.x, wk.y);
          const Cx<R> d2 = cmulc(a2 - c2, w2);
          TS[pad(H - k)] = mk(s3.x - d2.y, s3.y + d2.x);
        }
      }
    }
    __syncthreads();
    CB_MARK(8 + 8 * st + 4);
#endif
    fft1<R, Q, H, NT, true, HS>(TS, twpH, &s_zero);
    CB_MARK(8 + 8 * st + 5);
    RotationHook<R> rot;
    rot.th = Treal;
    rot.scale = st < kStepCache ? s_tsc[st] : theta_scale[st];
    const Cx<R>* ph_next =
        ph_grp + (size_t)(st < kStepCache ? s_phi[st + 1] : prm.ph_index[st + 1]) * ph_tab;
    if (st + 1 < prm.n_steps) {
      fft2<R, Q, NT, FF, false, RotationHook<R>, NoHook, 1, Q / sched_radix(Q, 1, FI)>(
          F, twpF, &s_zero, rot);
      CB_MARK(8 + 8 * st + 6);
      fft2_boundary<R, Q, NT, FI, FF>(F, twpF, ph_next, &s_zero);
      CB_MARK(8 + 8 * st + 7);
      fft2<R, Q, NT, FI, true, NoHook, IntensityHook<R>, sched_radix(Q, 1, FI)>(
          F, twpT, &s_zero, NoHook(), ih);
    } else {
      PhasorHook<R> ph1;
      ph1.ph = ph_next;
      fft2<R, Q, NT, FF, false, RotationHook<R>, PhasorHook<R>>(F, twpF, &s_zero, rot, ph1);
    }
  }

  __syncthreads();
  CB_MARK(4);
  // ---- 5. merge + outer IFFT (dbp.py:400-401): inverse radix-P stage in
  //         place (registers across one barrier), then FFT_Q^-1 per group
  Cx<R> wQ[P];  // W_P^m again (not kept live through the step loop)
#pragma unroll
  for (int m = 0; m < P; ++m) wQ[m] = ldg(twN + m * Q + *(&s_zero));
  for (int pol = 0; pol < 2; ++pol) {
    Cx<R> xv[KPT][P];
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
      const int k2 = (int)threadIdx.x + u * NTC;
      if (k2 < Q) {
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) {
          int i, m;
          bin_home<P, Q>(Q * k1 + k2, i, m);
          xv[u][k1] = base[i * SG + pol * SF + pad(m)];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
      const int k2 = (int)threadIdx.x + u * NTC;
      if (k2 < Q) {
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) {
          Cx<R> sm = xv[u][0];
#pragma unroll
          for (int k1 = 1; k1 < P; ++k1) sm = sm + cmulc(xv[u][k1], wQ[(n1 * k1) % P]);
          if (n1) sm = cmulc(sm, ldg(twN + n1 * k2));
          base[n1 * SG + pol * SF + pad(k2)] = sm;
        }
      }
    }
    __syncthreads();
  }
  fft2<R, Q, NT, FI, true>(F, twpT, &s_zero);
  __syncthreads();
  CB_MARK(5);

  // ---- 6. keep proc[half : half + span] (dbp.py:476-477), coalesced
  {
    const int64_t span = min(prm.keep, n - b * prm.keep);
    Cx<R>* dst = prm.out + wv * prm.out_bstride;
    const int64_t obase = b * prm.keep - prm.half - prm.out_origin;
    for (int64_t t = prm.half + threadIdx.x; t < prm.half + span; t += NTC) {
      const int r = (int)(t % P), t2 = (int)(t / P);
      const Cx<R>* Fr = base + r * SG;
      CB_CHECK(obase + t >= 0 && (prm.out_origin != 0 || obase + t < n));
      dst[obase + t] = Fr[pad(t2)];
      dst[prm.out_pstride + obase + t] = Fr[SF + pad(t2)];
    }
  }
  if constexpr (TMON) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(cb_tm_base),
                   "n"(COLS));
  }
}

}  // namespace cbessfm
