"""One-off source patch: kRegCarry (field butterfly carried in registers
across the nonlinear step) for the cluster kernel."""
p = 'paper_2409_14489_b200/csrc/cbessfm_kernel.cuh'
s = open(p).read()


def rep(old, new, cnt=1, first=False):
    global s
    n = s.count(old)
    assert (n >= 1 if first else n == cnt), (old[:70], n)
    s = s.replace(old, new, 1 if first else -1)


rep("""constexpr int kCarry = 64;""", """constexpr int kCarry = 64;
// kRegCarry (cluster kernel): the same carry in registers -- the carried
// butterfly stays live across the nonlinear step in the hooks' carry array
// (the TMEM columns are taken by the twiddle rows there)
constexpr int kRegCarry = 256;
#ifndef CB_REG_CARRY
#define CB_REG_CARRY 1
#endif""")
rep("""template <typename R>
struct IntensityHook : NoHook {
  R* I;""", """template <typename R>
struct IntensityHook : NoHook {
  R* I;
  Cx<R>* carry = nullptr;  // kRegCarry: where the carried butterfly goes""")
rep("""template <typename R>
struct RotationHook : NoHook {
  const R* th;
  R scale;""", """template <typename R>
struct RotationHook : NoHook {
  const R* th;
  R scale;
  Cx<R>* carry = nullptr;  // kRegCarry: the butterfly carried from the IFFT""")
rep("""  constexpr bool CARRY_OUT = CARRYS && LAST && INV && std::is_same<Hook, IntensityHook<R>>::value;
  constexpr bool CARRY_IN = CARRYS && FIRST && !INV && std::is_same<Hook, RotationHook<R>>::value;
  if constexpr (CARRY_OUT || CARRY_IN) {""", """  constexpr bool RCARRY = (SCHED & kRegCarry) != 0;
  constexpr bool CARRY_OUT =
      (CARRYS || RCARRY) && LAST && INV && std::is_same<Hook, IntensityHook<R>>::value;
  constexpr bool CARRY_IN =
      (CARRYS || RCARRY) && FIRST && !INV && std::is_same<Hook, RotationHook<R>>::value;
  if constexpr (RCARRY && (CARRY_OUT || CARRY_IN)) {
    static_assert(PER == 1 && RAD == sched_radix(Q, 1, SCHED) && (CARRY_IN ? NS == 1 : NS == LR),
                  "register carry: one radix-R butterfly on samples j + r*Q/R per thread");
    const int j = jb;
    Cx<R> v[RAD];
    if constexpr (CARRY_IN) {
#pragma unroll
      for (int r = 0; r < RAD; ++r) v[r] = hook.carry[r];
      hook.template pre<R, RAD, LR>(j, v);
      dft_reg<R, RAD, INV>(v);
      Cx<R>* b = Fp + pad(j * RAD);  // NS = 1: d0 = R*j
#pragma unroll
      for (int r = 0; r < RAD; ++r) b[pad(r)] = v[bitrev<RAD>(r)];
    } else {
      const Cx<R>* b = Fp + pad(j);
#pragma unroll
      for (int r = 0; r < RAD; ++r) v[r] = b[pad(r * LR)];
      const Cx<R>* w = rows.row(0);
#pragma unroll
      for (int r = 1; r < RAD; ++r) v[r] = cmulc(v[r], w[r]);
      dft_reg<R, RAD, INV>(v);
      hook.template post<R, RAD, NS>(j, v);  // d0 = j (j < NS)
#pragma unroll
      for (int r = 0; r < RAD; ++r) hook.carry[r] = v[bitrev<RAD>(r)];
    }
    next.fetch(twp_next);
    pass_sync<SCHED, NT>();
    return;
  } else if constexpr (CARRY_OUT || CARRY_IN) {""")
rep("""  constexpr bool TMON = tm_on<R, Q>();
  // field transforms: inverse (IFFT, outer) and forward (in-step FFT)
  // schedules; half-length transforms
  constexpr int FI = TMON ? (kMid | kTM) : kTail;
  constexpr int FF = TMON ? (kMid | kTM) : kHead;""", """  constexpr bool TMON = tm_on<R, Q>();
  // kRegCarry: FP64 at N' = 2048 / 4096 (one radix-16 butterfly per thread)
  constexpr int FC = (CB_REG_CARRY && TMON && sizeof(R) == 8) ? kRegCarry : 0;
  // field transforms: inverse (IFFT, outer) and forward (in-step FFT)
  // schedules; half-length transforms
  constexpr int FI = TMON ? (kMid | kTM | FC) : kTail;
  constexpr int FF = TMON ? (kMid | kTM | FC) : kHead;""")
rep("""  IntensityHook<R> ih;
  ih.I = Ireal;
  if (prm.n_steps > 0)
    fft2<R, Q, NT, FI, true, NoHook, IntensityHook<R>>(F, twpT, &s_zero, NoHook(), ih);
  CB_MARK(3);""", """  // the field butterfly carried across the nonlinear step (kRegCarry)
  Cx<R> carry[kMaxRad];
  IntensityHook<R> ih;
  ih.I = Ireal;
  ih.carry = carry;
  if (prm.n_steps > 0)
    fft2<R, Q, NT, FI, true, NoHook, IntensityHook<R>>(F, twpT, &s_zero, NoHook(), ih);
  CB_MARK(3);""", first=True)
rep("""    RotationHook<R> rot;
    rot.th = Treal;
    rot.scale = tsc_st;""", """    RotationHook<R> rot;
    rot.th = Treal;
    rot.scale = tsc_st;
    rot.carry = carry;""", first=True)
open(p, 'w').write(s)
print("patched")
