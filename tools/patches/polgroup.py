"""One-off source patch (kept for the record): kPolGroup field-pass mapping
for the cluster kernel. Applied once to csrc/cbessfm_kernel.cuh."""
import sys

p = sys.argv[1] if len(sys.argv) > 1 else 'paper_2409_14489_b200/csrc/cbessfm_kernel.cuh'
s = open(p).read()


def rep(old, new, cnt=1):
    global s
    assert s.count(old) == cnt, (old[:70], s.count(old))
    s = s.replace(old, new)


rep("""constexpr int kCarry = 64;""", """constexpr int kCarry = 64;
// kPolGroup (field schedules of the cluster kernel): the two polarisation
// rows run on two thread groups (threads [0, NT/2) x, [NT/2, NT) y) instead
// of the two half-warps, and each group's passes synchronise on the group's
// own named barrier (2 + group), so one polarisation's shared-memory phase
// can overlap the other's arithmetic; the intensity and the rotation then
// meet through shared memory (IntensityHook / RotationHook <R, true>)
constexpr int kPolGroup = 128;
#ifndef CB_POLGROUP
#define CB_POLGROUP 1
#endif""")
rep("""template <int NT>
__device__ __forceinline__ int fpol(int t) { return (t >> 4) & 1; }
template <int NT>
__device__ __forceinline__ int fbase(int t) { return ((t >> 5) << 4) | (t & 15); }""",
    """template <int NT, int SCHED = 0>
__device__ __forceinline__ int fpol(int t) {
  return (SCHED & kPolGroup) ? (t >= NT / 2) : ((t >> 4) & 1);
}
template <int NT, int SCHED = 0>
__device__ __forceinline__ int fbase(int t) {
  return (SCHED & kPolGroup) ? (t & (NT / 2 - 1)) : (((t >> 5) << 4) | (t & 15));
}
// named barriers of the kPolGroup protocol (0: CTA, 1: half-length passes,
// 2-3: the two groups' field passes)
constexpr int kBarIntensity = 4;  // x arrives after writing |x|^2, y syncs before adding |y|^2
constexpr int kBarTheta = 5;      // y arrives after reading theta, x syncs before rewriting I""")
rep("""template <int SCHED, int NT>
__device__ __forceinline__ void pass_sync() {
  if constexpr ((SCHED & kGroupBar) != 0) {""", """template <int SCHED, int NT>
__device__ __forceinline__ void pass_sync() {
  if constexpr ((SCHED & kPolGroup) != 0) {
    asm volatile("bar.sync %0, %1;" ::"r"(2 + ((int)threadIdx.x >= NT / 2)), "n"(NT / 2) : "memory");
  } else if constexpr ((SCHED & kGroupBar) != 0) {""")
rep("""template <typename R>
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
};""", """template <typename R, bool PG = false>
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
// kPolGroup form: the x thread and the y thread of a position are in
// different groups. x writes |x|^2 (after y's reads of the previous theta
// in the same slots, kBarTheta) and arrives on kBarIntensity; y waits there
// and adds |y|^2: I = |x|^2 + |y|^2, the same sum as above.
template <typename R>
struct IntensityHook<R, true> : NoHook {
  R* I;
  int nt;            // threads of the CTA (both groups)
  bool wait_theta;   // a rotation pass read theta from these slots before
  template <typename, int RAD, int NS>
  __device__ __forceinline__ void post(int d0, Cx<R>* v) {
    const bool ypol = (int)threadIdx.x >= nt / 2;
    R* base = I + fpos(d0);
    if (!ypol) {
      if (wait_theta) bar_named(kBarTheta, nt);
#pragma unroll
      for (int r = 0; r < RAD; ++r) {
        const Cx<R> a = v[bitrev<RAD>(r)];
        base[fpos(r * NS)] = a.x * a.x + a.y * a.y;
      }
      asm volatile("bar.arrive %0, %1;" ::"r"(kBarIntensity), "r"(nt) : "memory");
    } else {
      bar_named(kBarIntensity, nt);
#pragma unroll
      for (int r = 0; r < RAD; ++r) {
        const Cx<R> a = v[bitrev<RAD>(r)];
        R* q = base + fpos(r * NS);
        *q = *q + (a.x * a.x + a.y * a.y);
      }
    }
  }
};""")
rep("""template <typename R>
struct RotationHook : NoHook {
  const R* th;
  R scale;""", """template <typename R, bool PG = false>
struct RotationHook : NoHook {
  const R* th;
  R scale;""")
rep("""      v[2 * h] = cmul(v[2 * h], pol ? theirs : mine);
      v[2 * h + 1] = cmul(v[2 * h + 1], pol ? mine : theirs);
    }
  }
};""", """      v[2 * h] = cmul(v[2 * h], pol ? theirs : mine);
      v[2 * h + 1] = cmul(v[2 * h + 1], pol ? mine : theirs);
    }
  }
};
// kPolGroup form: each thread evaluates its own 16 angles (the partner
// polarisation is in the other group); y arrives on kBarTheta once its
// reads are done, unless no intensity pass follows (last step).
template <typename R>
struct RotationHook<R, true> : NoHook {
  const R* th;
  R scale;
  int nt;
  bool arrive;
  template <typename, int RAD, int LR>
  __device__ __forceinline__ void pre(int j, Cx<R>* v) {
    const R* base = th + fpos(j);
    R a[RAD];
#pragma unroll
    for (int r = 0; r < RAD; ++r) a[r] = base[fpos(r * LR)];
#pragma unroll
    for (int r = 0; r < RAD; ++r) {
      R sn, cs;
      sincos_acc<R>(a[r] * scale, &sn, &cs);
      v[r] = cmul(v[r], mk(cs, -sn));
    }
    // after the loaded angles have been consumed
    if (arrive && (int)threadIdx.x >= nt / 2)
      asm volatile("bar.arrive %0, %1;" ::"r"(kBarTheta), "r"(nt) : "memory");
  }
};""")
# fft2_pass (SCHED) and fft2_boundary (SFW)
i = s.index("  Cx<R>* Fp = F + fpol<NT>(tid) * SF;\n  const int jb = fbase<NT>(tid);")
s = s[:i] + "  Cx<R>* Fp = F + fpol<NT, SCHED>(tid) * SF;\n  const int jb = fbase<NT, SCHED>(tid);" + \
    s[i + len("  Cx<R>* Fp = F + fpol<NT>(tid) * SF;\n  const int jb = fbase<NT>(tid);"):]
rep("  Cx<R>* Fp = F + fpol<NT>(tid) * SF;\n  const int jb = fbase<NT>(tid);",
    "  Cx<R>* Fp = F + fpol<NT, SFW>(tid) * SF;\n  const int jb = fbase<NT, SFW>(tid);")
rep("""          const int j = fbase<NT>(tid) + p * SLOTS;""", """          const int j = fbase<NT, SCHED>(tid) + p * SLOTS;""")
rep("""            j = fbase<NT>(tid) + p * (NT / 2);""", """            j = fbase<NT, SCHED>(tid) + p * (NT / 2);""")
open(p, 'w').write(s)
print("patched")
