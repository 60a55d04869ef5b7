// In-place field transforms and the block kernel built on them
// (cbessfm_ip_kernel: complex128, N' = 2048, 2 <= P <= 9).
//
// The cluster kernel's field FFTs are Stockham passes: every pass reads the
// whole row, waits at a CTA barrier (the pass is out of order, so nobody may
// store before everybody has loaded), writes it back and waits again -- ten
// CTA barriers per step for the five field passes, each stalling all eight
// warps of the CTA. Here the subband-domain samples are kept in a
// digit-reversed order instead, which makes every pass in place (a thread
// writes exactly the positions it read) and, for two of the three passes,
// local to one warp:
//
//   time sample n = j + 128 r                (j < 128, r < 16)
//   bin k = s + 16 (m0 + 8 m1)               (s < 16, m0 < 8, m1 < 16)
//   the bin is stored at position 128 s + 16 m0 + m1   ("pos(k)")
//
//   forward (time natural -> bins at pos(k)), decimation in frequency:
//     G : y[j + 128 s]     = W_2048^{js} sum_r x[j + 128 r] W_16^{rs}
//     L1: z[j0 + 16 m0]    = W_128^{j0 m0} sum_j1 y_s[j0 + 16 j1] W_8^{j1 m0}
//     L2: X at m1 + 16 m0  = sum_j0 z[j0 + 16 m0] W_16^{j0 m1}
//   inverse: the same passes in reverse order with conjugate factors
//   (decimation in time, bins at pos(k) -> natural time order).
//
// G mixes the 16 regions [128 s, 128 s + 128) of a row; L1 and L2 stay
// inside one region. A warp owns four regions of one polarisation for the
// L passes, so they synchronise with __syncwarp only; the CTA waits at a
// barrier after G and before G' (and for the NLPR exchange, as before). The
// in-step FFT's last pass L2 and the next IFFT's first pass L2' run the same
// 16 samples, fused with the dispersion phasor in registers (boundary pass).
// Per step: five field round trips as before, but 3 CTA barriers for the
// field transforms instead of 10, and the warp-local passes of different
// warps overlap freely.
//
// The twiddle rows are exactly the kMid rows the cluster kernel keeps in
// TMEM: G uses the radix-16 pass's W_2048^{j s} (butterfly j = fbase(tid)),
// L1 the radix-8 pass's W_128^{j0 m0} (j0 = lane % 16). Time-domain hooks
// (intensity, rotation) see the natural positions j + 128 r they see in the
// cluster kernel. The phasor rows are read from a copy permuted to pos()
// order (Params::phasor_rev) so each boundary-pass load of a warp is one
// contiguous 512-byte span. The outer transforms (prologue FFT_Q, epilogue
// IFFT_Q) keep the Stockham fft2; only the radix-P stages map bins through
// pos().
#pragma once

namespace cbessfm {

constexpr int kIpQ = 2048;

// position of subband-local bin k (natural storage index) in the
// digit-reversed layout, and its padded shared-memory index
__host__ __device__ constexpr int ip_pos(int k) {
  return 128 * (k & 15) + 16 * ((k >> 4) & 7) + (k >> 7);
}
__host__ __device__ constexpr int ip_ppos(int k) {
  return 136 * (k & 15) + 17 * ((k >> 4) & 7) + (k >> 7);
}
// index of bin (s, m0, m1) in the permuted phasor rows: for fixed m1 the
// 32 lanes of a boundary-pass warp (4 regions x 8 m0) read 32 consecutive
// entries
__host__ __device__ constexpr int ip_rev_index(int s, int m0, int m1) {
  return (((s >> 2) * 16 + m1) * 4 + (s & 3)) * 8 + m0;
}

// ---- G: the stride-128 radix-16 pass (mixes all regions of a row).
// Forward: pre-hook on the natural inputs, DFT_16, twiddle the outputs.
// Inverse: twiddle the inputs, IDFT_16, post-hook on the natural outputs.
template <typename R, bool INV, class Hook, class Rows>
__device__ __forceinline__ void ip_global(Cx<R>* __restrict__ F, const volatile int* zero,
                                          Hook& hook, Rows& rows) {
  constexpr int SF = padded_len(kIpQ);
  const int tid = (int)threadIdx.x + *zero;
  Cx<R>* Fp = F + fpol<256>(tid) * SF;
  const int j = fbase<256>(tid);
  Cx<R>* b = Fp + pad(j);
  Cx<R> v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = b[pad(r * 128)];
  if constexpr (!INV) {
    hook.template pre<R, 16, 128>(j, v);
    dft_reg<R, 16, false>(v);
    const Cx<R>* w = rows.row(0);
#pragma unroll
    for (int s = 1; s < 16; ++s) v[bitrev<16>(s)] = cmul(v[bitrev<16>(s)], w[s]);
#pragma unroll
    for (int s = 0; s < 16; ++s) b[pad(s * 128)] = v[bitrev<16>(s)];
  } else {
    const Cx<R>* w = rows.row(0);
#pragma unroll
    for (int s = 1; s < 16; ++s) v[s] = cmulc(v[s], w[s]);
    dft_reg<R, 16, true>(v);
    hook.template post<R, 16, 128>(j, v);
#pragma unroll
    for (int r = 0; r < 16; ++r) b[pad(r * 128)] = v[bitrev<16>(r)];
  }
}

// Regions of this warp for the L passes: polarisation warp / 4, regions
// s = 4 (warp % 4) + i, i < 4.
__device__ __forceinline__ int ip_region_pol(int warp) { return warp >> 2; }
__device__ __forceinline__ int ip_region0(int warp) { return 4 * (warp & 3); }

// ---- L1: radix 8 over j1 inside a region (stride 16), twiddle W_128^{j0 m0}.
// Lane l runs butterfly j0 = l % 16 of regions 2 (l / 16) + p, p < 2.
template <typename R, bool INV, class Rows>
__device__ __forceinline__ void ip_l1(Cx<R>* __restrict__ F, const volatile int* zero,
                                      Rows& rows) {
  constexpr int SF = padded_len(kIpQ);
  const int tid = (int)threadIdx.x + *zero;
  const int warp = tid >> 5, lane = tid & 31;
  const int j0 = lane & 15;
  Cx<R>* base = F + ip_region_pol(warp) * SF + j0 +
                136 * (ip_region0(warp) + 2 * (lane >> 4));
  const Cx<R>* w = rows.row(0);
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    Cx<R>* b = base + 136 * p;
    Cx<R> v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = b[17 * i];
    if constexpr (!INV) {
      dft_reg<R, 8, false>(v);
#pragma unroll
      for (int m = 1; m < 8; ++m) v[bitrev<8>(m)] = cmul(v[bitrev<8>(m)], w[m]);
    } else {
#pragma unroll
      for (int m = 1; m < 8; ++m) v[m] = cmulc(v[m], w[m]);
      dft_reg<R, 8, true>(v);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) b[17 * i] = v[bitrev<8>(i)];
  }
}

// ---- L2 (+ L2'): radix 16 over the 16 contiguous samples of (region, m0).
// Lane l runs region 4 (warp % 4) + l / 8, m0 = l % 8.
//   MODE 0: IDFT only (the first IFFT after the prologue: bins -> z')
//   MODE 1: DFT, x phasor, IDFT (step boundary: L2, phasor, next L2')
//   MODE 2: DFT, x phasor (last step: bins stay at pos() for the epilogue)
template <typename R, int MODE>
__device__ __forceinline__ void ip_l2(Cx<R>* __restrict__ F, const volatile int* zero,
                                      const Cx<R>* __restrict__ ph_rev) {
  constexpr int SF = padded_len(kIpQ);
  const int tid = (int)threadIdx.x + *zero;
  const int warp = tid >> 5, lane = tid & 31;
  const int s = ip_region0(warp) + (lane >> 3), m0 = lane & 7;
  Cx<R>* b = F + ip_region_pol(warp) * SF + 136 * s + 17 * m0;
  Cx<R> v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = b[i];
  if constexpr (MODE != 0) {
    dft_reg<R, 16, false>(v);
    // bin m1 lives in v[bitrev(m1)]; the phasor of (s, m0, m1)
    const Cx<R>* ph = ph_rev + ip_rev_index(s, m0, 0);
    Cx<R> u[16];
#pragma unroll
    for (int m1 = 0; m1 < 16; ++m1) u[m1] = cmul(v[bitrev<16>(m1)], ldg_na(ph + 32 * m1));
    if constexpr (MODE == 2) {
#pragma unroll
      for (int m1 = 0; m1 < 16; ++m1) b[m1] = u[m1];
      return;
    }
#pragma unroll
    for (int m1 = 0; m1 < 16; ++m1) v[m1] = u[m1];
  }
  dft_reg<R, 16, true>(v);
#pragma unroll
  for (int i = 0; i < 16; ++i) b[i] = v[bitrev<16>(i)];
}

template <typename R, int P>
__global__ void __launch_bounds__(256, 2) cbessfm_ip_kernel(const Params<R> prm) {
  constexpr int Q = kIpQ;
  constexpr int NT = 256;
  static_assert(threads_for<R, Q>() == NT && P >= 2, "ip kernel: Q = 2048, P >= 2");
  static_assert(tm_on<R, Q>(), "ip kernel: twiddle rows in TMEM");
  constexpr int H = Q / 2;
  constexpr int SF = padded_len(Q);

  extern __shared__ __align__(16) unsigned char smem_raw[];
  CB_POISON_SMEM(smem_raw);
  Cx<R>* F = reinterpret_cast<Cx<R>*>(smem_raw);
  Cx<R>* IS = F + 2 * SF;
  Cx<R>* TS = IS;  // as in cbessfm_block_kernel
  Cx<R>* RB = IS + padded_len(H + 1);
  constexpr int SLM = mimo_slice_max(P, H);
  constexpr bool ROTTAB = rot_tab_on<R, Q>();
  Cx<R>* RT = RB + rb_len<Q>(P);  // rotation table (RotationTabHook)
  if constexpr (ROTTAB) {
    for (int i = threadIdx.x; i < kRotTab; i += NT) RT[i] = ldg(prm.rot_tab + i);
  }

  __shared__ int s_zero;
  __shared__ uint64_t s_bar[2];
  if (threadIdx.x == 0) {
    s_zero = 0;
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init_fence();
  }
  constexpr int FI = kMid | kTM;
  constexpr int HS = kHalf | kTM | kWide;
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

  const int tid = threadIdx.x;
  const int rank = (int)(blockIdx.x % P);
  // persistent launches: as in cbessfm_block_kernel (rank 0 claims blocks from
  // the launch-wide counter, the next one at the top of the current block, and
  // pulls its window towards L2; mbarrier phase parity continues across blocks)
  __shared__ long long s_cid[3];
  const bool persist = prm.work != nullptr;
  if (persist) {
    if (rank == 0 && tid == 0) s_cid[0] = (long long)atomicAdd(prm.work, 1ull);
    cg::this_cluster().sync();
  }
  for (int it = 0;; ++it) {
  int64_t cid;
  if (persist) {
    if (tid == 0) {
      long long c = s_cid[it & 1];
      if (rank != 0) c = *cg::this_cluster().map_shared_rank(&s_cid[it & 1], 0);
      s_cid[2] = c;
    }
    __syncthreads();
    cid = s_cid[2];
    if (cid >= prm.total) break;
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
    cid += prm.cid0;
  } else {
    if (it) break;
    cid = prm.cid0 + blockIdx.x / P;
  }
  const int ph0 = (int)(((int64_t)it * prm.n_steps) & 1);
  CB_MARK(0);
  CB_TIMELINE(0);
  const int64_t wv = cid / prm.nb;
  const int64_t b = prm.b0 + cid % prm.nb;
  const int64_t n = prm.n;
  const int64_t cset = prm.n_sets > 1 ? wv % prm.n_sets : 0;
  const Cx<R>* __restrict__ mimo = prm.mimo + cset * (int64_t)P * (H + 1);
  const R* __restrict__ theta_scale = prm.theta_scale + cset * prm.n_steps;
  const Cx<R>* __restrict__ twQ = prm.twQ;
  const Cx<R>* __restrict__ twN = prm.twN;
  const Cx<R>* __restrict__ twpT = prm.twp + twp_base(Q, FI);
  const Cx<R>* __restrict__ twpH = prm.twp + twp_base(Q, HS);

  // ---- 1. polyphase component u[rank + P*t2] of the circular window
  //         starting at (b*keep - half) mod n (dbp.py:473-475)
  {
    int64_t start = (b * prm.keep - prm.half) % n;
    if (start < 0) start += n;
    start -= prm.in_origin;
    if (start < 0) start += n;
    const Cx<R>* src = prm.in + wv * prm.in_bstride;
    // all 2 x Q/NT samples of a thread in flight at once (cp.async): the
    // load is latency-bound (stride-P gather), not bandwidth-bound
#pragma unroll
    for (int t2 = tid; t2 < Q; t2 += NT) {
      int64_t idx = start + rank + (int64_t)P * t2;
      if (idx >= n) idx -= n;
      CB_CHECK(idx >= 0 && idx < n);
      cp_async16(&F[pad(t2)], src + idx);
      cp_async16(&F[SF + pad(t2)], src + prm.in_pstride + idx);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  CB_MARK(1);

  const size_t ph_tab = (size_t)P * Q;
  // ---- 2.-3. FFT_Q of both polarisations (Stockham, natural order), then
  //         the cross-subband radix-P stage over DSMEM (dbp.py:387-389),
  //         first phasor and 1/P fused, bins written to pos() of the owner
  cg::cluster_group cluster = cg::this_cluster();
  {
    fft2<R, Q, NT, FI, false>(F, twpT, &s_zero);
    const int lo = (rank * Q) / P, hi = ((rank + 1) * Q) / P;
    const R invP = (R)1 / (R)P;
    const Cx<R>* ph0 = prm.phasor + (size_t)prm.ph_index[0] * ph_tab;
    Cx<R>* S = IS;
    cluster.sync();
    // W_P^e, e < P (the radix-P DFT's constants), once per thread
    Cx<R> wp[P];
#pragma unroll
    for (int e = 0; e < P; ++e) wp[e] = ldg(twN + e * Q);
    for (int pol = 0; pol < 2; ++pol) {
      for (int k2 = lo + tid; k2 < hi; k2 += NT) {
        // independent loads first: the P remote bins, their twiddles and
        // the P destination phasors
        Cx<R> bv[P], tw[P], w[P];
#pragma unroll
        for (int r = 0; r < P; ++r) {
          const Cx<R>* rf = cluster.map_shared_rank(F, r);
          bv[r] = rf[pol * SF + pad(k2)];
          tw[r] = r ? ldg(twN + r * k2) : mk((R)1, (R)0);
          int i, m;
          bin_home<P, Q>(Q * r + k2, i, m);
          w[r] = ldg(ph0 + (size_t)i * Q + m);
        }
#pragma unroll
        for (int r = 1; r < P; ++r) bv[r] = cmul(bv[r], tw[r]);
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) {
          Cx<R> s = bv[0];
#pragma unroll
          for (int r = 1; r < P; ++r) s = s + cmul(bv[r], wp[(r * k1) % P]);
          int i, m;
          bin_home<P, Q>(Q * k1 + k2, i, m);
          Cx<R>* dst = cluster.map_shared_rank(pol ? F : S, i);
          dst[ip_ppos(m)] = cmul(scale(s, invP), w[k1]);
        }
      }
      cluster.sync();
    }
    // the staged row-0 results (pos() layout, same padding) move in
    for (int t = tid; t < Q; t += NT) F[SF + pad(t)] = S[pad(t)];
    __syncthreads();
    // as in cbessfm_block_kernel: no step-0 push may land in IS / RB (which
    // S spans) before every CTA has read its staged row out
    cluster_arrive();
  }
  CB_MARK(2);

  const Cx<R>* phr_rank = prm.phasor_rev + (size_t)rank * Q;  // this subband's permuted rows
  R* Ireal = reinterpret_cast<R*>(IS);
  const R* Treal = reinterpret_cast<const R*>(TS);
  PassRows<R, Q, NT, 128, FI> rowsG;
  PassRows<R, Q, NT, 16, FI> rowsL;

  // ---- 4. steps. First IFFT: L2' (bins at pos() -> z'), L1', G' with the
  //         intensity hook (time samples in natural order)
  IntensityHook<R> ih;
  ih.I = Ireal;
  if (prm.n_steps > 0) {
    ip_l2<R, 0>(F, &s_zero, nullptr);
    __syncwarp();
    ip_l1<R, true>(F, &s_zero, rowsL);
    __syncthreads();
    ip_global<R, true>(F, &s_zero, ih, rowsG);
    __syncthreads();
  }
  CB_MARK(3);
  cluster_wait();
  constexpr int KU = (H / 2 + 1 + NT - 1) / NT;
  for (int st = 0; st < prm.n_steps; ++st) {
    const R tsc_st = theta_scale[st];
    const int phi_next = prm.ph_index[st + 1];
    Cx<R> twk[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const int k = tid + u * NT;
      twk[u] = (k <= H / 2) ? ldg(twQ + k) : mk((R)1, (R)0);
    }
    fft1<R, Q, H, NT, false, HS>(IS, twpH, &s_zero);
    CB_MARK(8 + 8 * st + 0);

    // r2c untangle (dbp.py:194), bins pushed to their MIMO owners
#ifndef CB_EXP_NOXCHG
    if (tid == 0) {
#else
    if (false) {
#endif
      const int len = mimo_lo(rank + 1, P, H) - mimo_lo(rank, P, H);
      mbar_expect(&s_bar[0], (uint32_t)(P * len * sizeof(Cx<R>)));
      mbar_expect(&s_bar[1], (uint32_t)((H + 1) * sizeof(Cx<R>)));
    }
    auto emit = [&](int k, Cx<R> v) {
#ifdef CB_EXP_NOXCHG  // experiment: no cluster exchange (wrong results, timing only)
      IS[pad(k)] = v;
      return;
#endif
      int c = (k * P) / (H + 1);
      if (mimo_lo(c + 1, P, H) <= k) ++c;
      const uint32_t dst = cluster_addr(smem_addr(RB + rank * SLM + (k - mimo_lo(c, P, H))), c);
      push(dst, v, cluster_addr(smem_addr(&s_bar[0]), c));
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
        const Cx<R> dd = a - bq;
        const Cx<R> o = mk(dd.y * (R)0.5, -dd.x * (R)0.5);
        const Cx<R> wo = cmul(o, twk[u]);
        emit(k, e + wo);
        if (k != H - k) emit(H - k, conj(e - wo));
      }
    }

    CB_MARK(8 + 8 * st + 1);
    // MIMO coupling (dbp.py:195) on this CTA's bin slice
#ifdef CB_EXP_NOXCHG
    __syncthreads();
    for (int k = tid; k <= H; k += NT) {
      Cx<R> acc = mk((R)0, (R)0);
#pragma unroll
      for (int l = 0; l < P; ++l) acc = acc + cmul(ldg_na(mimo + (size_t)l * (H + 1) + (k + l) % (H + 1)), IS[pad(k)]);
      TS[pad(k)] = acc;
    }
    __syncthreads();
    if (false)
#endif
    {
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
          for (int l = 0; l < P; ++l)
            acc = l >= i ? cmac(acc, sv[l - i], iv[l]) : cmacc(acc, sv[i - l], iv[l]);
          push(cluster_addr(ts_local + (uint32_t)(pad(k) * sizeof(Cx<R>)), i), acc,
               cluster_addr(bar_t, i));
        }
      }
      CB_MARK(8 + 8 * st + 2);
      mbar_wait(&s_bar[1], (st + ph0) & 1);
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
        const Cx<R> a = TS[pad(k)];
        const Cx<R> c = conj(TS[pad(H - k)]);
        const Cx<R> wk = twk[u];
        const Cx<R> s = a + c;
        const Cx<R> dd = cmulc(a - c, wk);
        TS[pad(k)] = mk(s.x - dd.y, s.y + dd.x);
        if (k != H - k) {
          const Cx<R> a2 = conj(c);
          const Cx<R> c2 = conj(a);
          const Cx<R> s2 = a2 + c2;
          const Cx<R> w2 = mk(-wk.x, wk.y);
          const Cx<R> d2 = cmulc(a2 - c2, w2);
          TS[pad(H - k)] = mk(s2.x - d2.y, s2.y + d2.x);
        }
      }
    }
    __syncthreads();
    CB_MARK(8 + 8 * st + 4);
    fft1<R, Q, H, NT, true, HS>(TS, twpH, &s_zero);
    CB_MARK(8 + 8 * st + 5);

    // rotation exp(-i theta) fused into G (dbp.py:208, :398), then the
    // warp-local passes; the boundary pass applies the next phasor and
    // starts the next IFFT (dbp.py:395-396), or the final phasor (:399)
    typename std::conditional<ROTTAB, RotationTabHook<R>, RotationHook<R>>::type rot;
    rot.th = Treal;
    rot.scale = tsc_st;
    if constexpr (ROTTAB) rot.tab = RT;
    ip_global<R, false>(F, &s_zero, rot, rowsG);
    __syncthreads();
    ip_l1<R, false>(F, &s_zero, rowsL);
    __syncwarp();
    const Cx<R>* phr_next = phr_rank + (size_t)phi_next * ph_tab;
    CB_MARK(8 + 8 * st + 6);
    if (st + 1 < prm.n_steps) {
      ip_l2<R, 1>(F, &s_zero, phr_next);
      __syncwarp();
      ip_l1<R, true>(F, &s_zero, rowsL);
      __syncthreads();
      CB_MARK(8 + 8 * st + 7);
      ip_global<R, true>(F, &s_zero, ih, rowsG);
      __syncthreads();
    } else {
      ip_l2<R, 2>(F, &s_zero, phr_next);
      __syncthreads();
    }
  }

  CB_MARK(4);
  // ---- 5. merge + outer IFFT (dbp.py:400-401): bins read from their
  //         owners at pos(), the inverse radix-P stage writes natural order
  {
    const int lo = (rank * Q) / P, hi = ((rank + 1) * Q) / P;
    Cx<R>* S = IS;
    cluster.sync();
    Cx<R> wp[P];
#pragma unroll
    for (int e = 0; e < P; ++e) wp[e] = ldg(twN + e * Q);
    for (int pol = 0; pol < 2; ++pol) {
      for (int k2 = lo + tid; k2 < hi; k2 += NT) {
        Cx<R> xv[P], tw[P];
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) {
          int i, m;
          bin_home<P, Q>(Q * k1 + k2, i, m);
          const Cx<R>* rf = cluster.map_shared_rank(F, i);
          xv[k1] = rf[pol * SF + ip_ppos(m)];
          tw[k1] = k1 ? ldg(twN + k1 * k2) : mk((R)1, (R)0);
        }
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) {
          Cx<R> s = xv[0];
#pragma unroll
          for (int k1 = 1; k1 < P; ++k1) s = s + cmulc(xv[k1], wp[(n1 * k1) % P]);
          if (n1) s = cmulc(s, tw[n1]);
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
  }  // blocks of this cluster
  // rank 0's claim slots are read over DSMEM up to the last iteration
  if (persist) cg::this_cluster().sync();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(cb_tm_base),
                 "n"(tm_cols<R, Q>()));
}

}  // namespace cbessfm
