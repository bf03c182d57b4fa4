// sk_fused.cu — the fused dense executor: one HBM sweep applies many gates.
//
// GPU analogue of the reference's gate-by-gate loop `dense_reference`
// (validate.py:83-111), which makes one full NumPy pass per gate.  A program
// (planned on the host by paper_2304_14969_b200/fusion.py) is a list of
// sweeps.  A sweep streams the state through shared memory in tiles of 2^T
// amplitudes: the tile's T "tile bits" are the gate targets of the sweep plus
// the lowest contiguous bits (so every warp load/store covers >= 256
// contiguous bytes); all other index bits are fixed per tile (blockIdx).
//
// Inside a tile the sweep runs a sequence of stages.  In a stage each thread
// holds 2^NR amplitudes in registers, spanning the stage's NR register bits,
// and applies that stage's ops on them.  Between stages the tile is
// exchanged through (XOR-swizzled) shared memory; stage 0 loads from HBM and
// the last stage stores back: one read and one write per amplitude per sweep.
// Element addresses are walked in Gray-code order, so each element costs one
// 64-bit add (HBM) or one XOR (shared memory; the swizzle is GF(2)-linear).
//
// ABI ops (sk_op) are lowered per stage, on the host, into kernel ops whose
// register-bit predicates are precomputed element masks:
//   K_MAT    generic 2x2 on a register slot (K_MATR: real coefficients)
//   K_BFLY   H-like 2x2: y0 = c0 (a0 + a1), y1 = c1 (a0 - a1), optionally
//            with a per-thread phase tau folded into c1 (QFT's H(j)·RAMP(j))
//   K_PHASE  a[e] *= c for e in the element mask, c = c1 if a thread-side
//            bit is set else c0 (DIAG gates; RAMP's register part)
//   K_TPHASE a[e] *= tau (RAMP's thread part)
// tau = exp(2 pi i frac(F * turn / 2^64)), F a bit field of the thread's
// index, `turn` the RAMP scale in 64-bit fixed-point turns: exact modular
// arithmetic, then one MUFU sin/cos (fp32) or sincospi (fp64) per thread.
#include <cuda.h>  // CUtensorMap (types only; the encoder comes via cudaGetDriverEntryPoint)
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "sk_internal.cuh"

namespace sk {

constexpr int kMaxS = SK_MAX_STAGES;
constexpr int kMaxR = SK_MAX_REG_BITS;
constexpr int kMaxRuns = 16;

enum KKind : int { K_MAT = 0, K_MATR = 1, K_PHASE = 2, K_TPHASE = 3, K_BFLY = 4, K_QFTS = 5 };
enum KFlag : unsigned { F_TPRED = 1, F_QMASK = 2, F_C0REAL = 4, F_FOLD = 8, F_TABLE = 16, F_C0ONE = 32,
                        F_ENTRY = 64, F_END = 128, F_SCALE = 256 };

struct Run {  // bits [src, src+w) of a counter go to bits [dst, dst+w)
  uint8_t src, dst, w, pad;
};

struct DStage {
  int op_begin, op_end;
  int ng, nl;
  Run grun[kMaxRuns];       // thread index bits -> global index bits
  Run lrun[kMaxRuns];       // thread index bits -> tile-local index bits
  uint64_t reg_goff[kMaxR]; // byte offset of register slot p in HBM
  uint32_t reg_soff[kMaxR]; // swizzled byte offset of register slot p in shared memory
};

struct DSweep {
  int ntile;
  int nstages;
  int nr;        // register bits per stage (4 for c64; 3 or 4 for c128)
  int lean;      // every kernel op has a fast-path opcode (k_sweep<..., LEAN>)
  int qft_only;  // every kernel op is a K_QFTS chunk: use the specialised kernel
  int nb;
  Run brun[kMaxRuns];  // tile index (blockIdx) bits -> non-tile global bits
  DStage st[kMaxS];
};

struct alignas(16) KHdr {
  int16_t kind;
  int8_t slot;
  int8_t pat;
  uint16_t emask;
  uint8_t lo, nbits;
  uint32_t flags;
  uint32_t opc;  // fast-path opcode for k_sweep's dispatch (OPC_*), 0 = interpret via apply_kop
};

// fast paths of the generic interpreter: the unpredicated dense 2x2 (every
// U3 of a random circuit), the same behind a thread-side control, and the
// controlled-X register swap; everything else goes through apply_kop
enum KOpc : uint32_t {
  OPC_GENERIC = 0,
  OPC_MAT = 1,     // + P: dense 2x2 on slot P, unpredicated
  OPC_MATRP = 5,   // + P: 2x2 with a real first column = real rotation after a phase on a1 (split 1q gates)
  OPC_MATR = 9,    // + P: real 2x2 on slot P, unpredicated
  OPC_MATT = 13,   // + P: dense 2x2 behind a thread-side predicate
  OPC_MATQ = 17,   // + 2 (4P + Q) + V: dense 2x2 on slot P where register slot Q == V
  OPC_SWAPM = 49,  // + P: X on slot P for the pairs in the element mask, thread predicate
  OPC_YSWAPM = 53, // + P: Y likewise (swap with +-i: bit moves and sign flips)
  OPC_SIGNM = 57,  // by -1 (CZ-type couplers) on the elements in the mask: sign-bit flips
  OPC_DIAG1 = 58,  // + 2P + V: phase on the elements whose slot P == V, unpredicated
  OPC_PHASE = 66,  // any other K_PHASE: a selected multiplier per element
  OPC_END = 67
};

template <typename R>
struct alignas(16) KOp {
  KHdr h;
  uint64_t tmask, tval;  // predicate on the thread-constant index part (F_TPRED)
  uint64_t qmask;        // K_PHASE: c1 when (gthr & qmask) != 0 (F_QMASK)
  uint64_t turn;         // phase scale in 2^-64 turns
  uint64_t fmask;        // phase field mask (applied after >> lo)
  uint64_t pad2;
  R m[8];                // K_MAT: 2x2; K_PHASE: c0 = m[0..1], c1 = m[2..3]; K_BFLY: c0 = m[0..1], c1 = m[4..5]
  R mr[8];               // m rotated by i per complex entry, (-im, re): packed-FMA operand pairs
  R tw[16];              // K_BFLY (F_TABLE): extra row-1 twiddle per pair k (8 complex)
};

// swizzle of the tile-local index (element units): fold the high bits into
// the low SB bits; linear over GF(2), so swz(a ^ b) = swz(a) ^ swz(b)
template <int SB>
__host__ __device__ __forceinline__ uint32_t swz(uint32_t l) {
  uint32_t h = l >> SB;
  uint32_t f = h ^ (h >> SB) ^ (h >> (2 * SB)) ^ (h >> (3 * SB));
  return l ^ (f & ((1u << SB) - 1));
}

__host__ __device__ constexpr int ctz_c(int k) {
  int b = 0;
  while (!((k >> b) & 1)) ++b;
  return b;
}

__device__ __forceinline__ uint64_t deposit(uint64_t x, const Run* r, int n) {
  uint64_t o = 0;
  for (int i = 0; i < n; ++i) o |= ((x >> r[i].src) & ((1ull << r[i].w) - 1)) << r[i].dst;
  return o;
}

template <typename R>
__device__ __forceinline__ vec2_t<R> thread_phase(uint64_t turn, uint64_t gthr, int lo, uint64_t fmask) {
  const uint64_t f = (gthr >> lo) & fmask;
  const uint64_t t = f * turn;  // exact: frac(F * s / 2) in 2^-64 turns
  if (sizeof(R) == 4) {
    const float ang = (float)(int32_t)(uint32_t)(t >> 32) * 1.4629180792671596e-09f;  // 2 pi / 2^32, in [-pi, pi)
    float fs, fc;
    __sincosf(ang, &fs, &fc);
    return mk<R>((R)fc, (R)fs);
  } else {
    const double x = (double)(int64_t)t * 1.0842021724855044e-19;  // 2 / 2^64: half-turns in [-1, 1)
    double ds, dc;
    sincospi(x, &ds, &dc);
    return mk<R>((R)dc, (R)ds);
  }
}

template <int NR, int P>
struct PairMask {
  static constexpr uint32_t value() {
    uint32_t f = 0;
    for (int e = 0; e < (1 << NR); ++e)
      if (!((e >> P) & 1)) f |= 1u << e;
    return f;
  }
};

// y = m0 * a0 + m1 * a1 with r = m rotated by i: one paired multiply and
// three paired FMAs (scalar-broadcast operands are free modifiers)
template <typename R>
__device__ __forceinline__ vec2_t<R> cmac2(vec2_t<R> a0, vec2_t<R> a1, vec2_t<R> m0, vec2_t<R> r0, vec2_t<R> m1,
                                           vec2_t<R> r1) {
  if constexpr (sizeof(R) == 4) {
    float2 t = __fmul2_rn(make_float2(a0.x, a0.x), m0);
    t = __ffma2_rn(make_float2(a0.y, a0.y), r0, t);
    t = __ffma2_rn(make_float2(a1.x, a1.x), m1, t);
    return __ffma2_rn(make_float2(a1.y, a1.y), r1, t);
  } else {
    return mk<R>(a0.x * m0.x + a0.y * r0.x + a1.x * m1.x + a1.y * r1.x,
                 a0.x * m0.y + a0.y * r0.y + a1.x * m1.y + a1.y * r1.y);
  }
}

// c[0..7] = m00, r00, m01, r01, m10, r10, m11, r11
template <typename R, int NR, int P>
__device__ __forceinline__ void mat_slot(vec2_t<R> (&a)[1 << NR], const vec2_t<R> (&c)[8], uint32_t emask) {
  const bool full = emask == PairMask<NR, P>::value();
#pragma unroll
  for (int e = 0; e < (1 << NR); ++e) {
    if ((e >> P) & 1) continue;
    if (!full && !((emask >> e) & 1u)) continue;
    const int e1 = e | (1 << P);
    const vec2_t<R> y0 = cmac2<R>(a[e], a[e1], c[0], c[1], c[2], c[3]);
    const vec2_t<R> y1 = cmac2<R>(a[e], a[e1], c[4], c[5], c[6], c[7]);
    a[e] = y0;
    a[e1] = y1;
  }
}

template <typename R, int NR, int P>
__device__ __forceinline__ void matr_slot(vec2_t<R> (&a)[1 << NR], R m00, R m01, R m10, R m11, uint32_t emask) {
  const bool full = emask == PairMask<NR, P>::value();
#pragma unroll
  for (int e = 0; e < (1 << NR); ++e) {
    if ((e >> P) & 1) continue;
    if (!full && !((emask >> e) & 1u)) continue;
    const int e1 = e | (1 << P);
    const vec2_t<R> x0 = a[e], x1 = a[e1];
    if constexpr (sizeof(R) == 4) {
      a[e] = __ffma2_rn(x1, make_float2(m01, m01), __fmul2_rn(x0, make_float2(m00, m00)));
      a[e1] = __ffma2_rn(x1, make_float2(m11, m11), __fmul2_rn(x0, make_float2(m10, m10)));
    } else {
      a[e] = mk<R>(m00 * x0.x + m01 * x1.x, m00 * x0.y + m01 * x1.y);
      a[e1] = mk<R>(m10 * x0.x + m11 * x1.x, m10 * x0.y + m11 * x1.y);
    }
  }
}

template <typename R, int NR, int P>
__device__ __forceinline__ void bfly_slot(vec2_t<R> (&a)[1 << NR], vec2_t<R> c0, const vec2_t<R>* w, unsigned flags) {
  // pair k of slot P: e = k with a zero inserted at bit P, e1 = e | 2^P
  using PK_ = PK<R>;
#pragma unroll
  for (int e = 0, k = 0; e < (1 << NR); ++e) {
    if ((e >> P) & 1) continue;
    const int e1 = e | (1 << P);
    const vec2_t<R> s = PK_::add(a[e], a[e1]);
    const vec2_t<R> d = PK_::sub(a[e], a[e1]);
    if (flags & F_C0ONE)
      a[e] = s;
    else if (flags & F_C0REAL)
      a[e] = PK_::scale(s, c0.x);
    else
      a[e] = PK_::mul(c0, s);
    a[e1] = PK_::mul(w[k], d);
    ++k;
  }
}

// element patterns: all elements, one register-bit condition, or two
template <int NR, int P, int VP, int Q, int VQ>
__device__ __forceinline__ constexpr bool pat_hit(int e) {
  return (P < 0 || ((e >> P) & 1) == VP) && (Q < 0 || ((e >> Q) & 1) == VQ);
}

template <typename R, int NR, int P, int VP, int Q, int VQ>
__device__ __forceinline__ void phase_pat(vec2_t<R> (&a)[1 << NR], vec2_t<R> c) {
  if constexpr (P < NR && Q < NR) {
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e)
      if (pat_hit<NR, P, VP, Q, VQ>(e)) a[e] = PK<R>::mul(a[e], c);
  }
}

// pattern codes (host pattern_of agrees): 0 = all; 1 + 2P + VP = one
// condition; 9 + 4*pair(P<Q) + 2VP + VQ = two conditions
#define SK_PAT_PAIR(P, Q, IDX)                                             \
  case 9 + 4 * IDX + 0: phase_pat<R, NR, P, 0, Q, 0>(a, c); return true; \
  case 9 + 4 * IDX + 1: phase_pat<R, NR, P, 0, Q, 1>(a, c); return true; \
  case 9 + 4 * IDX + 2: phase_pat<R, NR, P, 1, Q, 0>(a, c); return true; \
  case 9 + 4 * IDX + 3: phase_pat<R, NR, P, 1, Q, 1>(a, c); return true;

template <typename R, int NR>
__device__ __forceinline__ bool phase_dispatch(int pat, vec2_t<R> (&a)[1 << NR], vec2_t<R> c) {
  switch (pat) {
    case 0: phase_pat<R, NR, -1, 0, -1, 0>(a, c); return true;
    case 1: phase_pat<R, NR, 0, 0, -1, 0>(a, c); return true;
    case 2: phase_pat<R, NR, 0, 1, -1, 0>(a, c); return true;
    case 3: phase_pat<R, NR, 1, 0, -1, 0>(a, c); return true;
    case 4: phase_pat<R, NR, 1, 1, -1, 0>(a, c); return true;
    case 5: phase_pat<R, NR, 2, 0, -1, 0>(a, c); return true;
    case 6: phase_pat<R, NR, 2, 1, -1, 0>(a, c); return true;
    case 7: phase_pat<R, NR, 3, 0, -1, 0>(a, c); return true;
    case 8: phase_pat<R, NR, 3, 1, -1, 0>(a, c); return true;
    SK_PAT_PAIR(0, 1, 0)
    SK_PAT_PAIR(0, 2, 1)
    SK_PAT_PAIR(0, 3, 2)
    SK_PAT_PAIR(1, 2, 3)
    SK_PAT_PAIR(1, 3, 4)
    SK_PAT_PAIR(2, 3, 5)
    default: return false;
  }
}
#undef SK_PAT_PAIR

#define SK_SLOT_SWITCH(slot, CALL)                  \
  switch (slot) {                                   \
    case 0: CALL(0); break;                         \
    case 1: if (NR > 1) CALL((NR > 1 ? 1 : 0)); break; \
    case 2: if (NR > 2) CALL((NR > 2 ? 2 : 0)); break; \
    case 3: if (NR > 3) CALL((NR > 3 ? 3 : 0)); break; \
    default: break;                                 \
  }

// ---------------------------------------------------------------------------
// QFT window chunk in FFT form (K_QFTS).  For a window of QFT layers
// j = w_hi..w_lo (each H(j) followed by its CP fan from all lower bits), a
// chunk of L consecutive layer bits held in register slots TOP-L+1..TOP:
//  * entry (not the first chunk): per-element phase
//      exp(i pi [Th_all * sum_{i in chunk} e_i 2^i + Th_new * Lv])
//    Th_all = sum_{j in earlier chunks} b_j 2^-j (their CPs onto this chunk),
//    Th_new = the same over the previous chunk only (its deferred below-window
//    phase), Lv = index bits below the window; in 2^-64-turn fixed point
//    Th = brev64(bits) exactly;
//  * L butterflies y0 = a0 + a1, y1 = (a0 - a1) exp(i pi sum_{p<P} e_p 2^(p-P))
//    with compile-time internal twiddles (the 1/sqrt2 per layer is deferred);
//  * end (last chunk, w_lo > 0): phase exp(i pi Lv sum_{i in chunk} e_i 2^-i)
//    (the chunk's deferred below-window phase); the window's (1/sqrt2)^K
//    scale rides on the last chunk's first phase.
// All deferred factors are diagonal in bits no later butterfly of the window
// touches, so moving them is exact (checked against the oracle by
// tests/test_kernel_lowering.py and tests/test_executor_gpu.py).
// ---------------------------------------------------------------------------
template <typename R>
__device__ __forceinline__ vec2_t<R> turn_phase(uint64_t t) {
  if (sizeof(R) == 4) {
    const float ang = (float)(int32_t)(uint32_t)(t >> 32) * 1.4629180792671596e-09f;
    float fs, fc;
    __sincosf(ang, &fs, &fc);
    return mk<R>((R)fc, (R)fs);
  } else {
    double ds, dc;
    sincospi((double)(int64_t)t * 1.0842021724855044e-19, &ds, &dc);
    return mk<R>((R)dc, (R)ds);
  }
}

// multiply by exp(i pi K / 8), K compile-time
template <typename R, int K>
__device__ __forceinline__ vec2_t<R> mul_pi8(vec2_t<R> x) {
  constexpr R c1 = (R)0.92387953251128674, s1 = (R)0.38268343236508978, h = (R)0.70710678118654752;
  if constexpr (K == 0) return x;
  else if constexpr (K == 4) return mk<R>(-x.y, x.x);
  else if constexpr (K == 2) return mk<R>(h * (x.x - x.y), h * (x.x + x.y));
  else if constexpr (K == 6) return mk<R>(-h * (x.x + x.y), h * (x.x - x.y));
  else {
    constexpr R cr = K == 1 ? c1 : K == 3 ? s1 : K == 5 ? -s1 : -c1;
    constexpr R ci = K == 1 ? s1 : K == 3 ? c1 : K == 5 ? c1 : s1;
    return mk<R>(cr * x.x - ci * x.y, cr * x.y + ci * x.x);
  }
}

template <int NR, int L, int TOP, int P, int E>
__host__ __device__ constexpr int qft_k8() {  // internal twiddle of pair base E at layer slot P, units of pi/8
  int k = 0;
  for (int p = TOP - L + 1; p < P; ++p)
    if ((E >> p) & 1) k += 1 << (3 - (P - p));
  return k;
}

template <typename R, int NR, int L, int TOP, int P, int E>
__device__ __forceinline__ void qft_pair(vec2_t<R> (&a)[1 << NR]) {
  if constexpr (E < (1 << NR)) {
    if constexpr (!((E >> P) & 1)) {
      constexpr int E1 = E | (1 << P);
      const vec2_t<R> s = mk<R>(a[E].x + a[E1].x, a[E].y + a[E1].y);
      const vec2_t<R> d = mk<R>(a[E].x - a[E1].x, a[E].y - a[E1].y);
      a[E] = s;
      a[E1] = mul_pi8<R, qft_k8<NR, L, TOP, P, E>()>(d);
    }
    qft_pair<R, NR, L, TOP, P, E + 1>(a);
  }
}

template <typename R, int NR, int L, int TOP, int P>
__device__ __forceinline__ void qft_layers(vec2_t<R> (&a)[1 << NR]) {
  if constexpr (P >= TOP - L + 1 && P >= 0) {
    qft_pair<R, NR, L, TOP, P, 0>(a);
    qft_layers<R, NR, L, TOP, P - 1>(a);
  }
}

// a[e] *= phase(base + sum_{layer slots p} e_p u_p) * scale, walked in Gray
// order (one complex multiply per element and per layer-bit flip)
template <typename R, int NR, int L, int TOP>
__device__ __forceinline__ void qft_phase(vec2_t<R> (&a)[1 << NR], uint64_t base, const uint64_t (&ut)[NR], R scale) {
  vec2_t<R> u[NR];
#pragma unroll
  for (int p = 0; p < NR; ++p)
    if (p >= TOP - L + 1 && p <= TOP) u[p] = turn_phase<R>(ut[p]);
  vec2_t<R> w = turn_phase<R>(base);
  w = mk<R>(w.x * scale, w.y * scale);
  a[0] = cmul<R>(a[0], w);
#pragma unroll
  for (int k = 1; k < (1 << NR); ++k) {
    const int b = ctz_c(k);
    const int e = k ^ (k >> 1);
    if (b >= TOP - L + 1 && b <= TOP) {
      if ((e >> b) & 1)
        w = cmul<R>(w, u[b]);
      else
        w = mk<R>(w.x * u[b].x + w.y * u[b].y, w.y * u[b].x - w.x * u[b].y);
    }
    a[e] = cmul<R>(a[e], w);
  }
}

template <typename R, int NR, int L, int TOP>
__device__ __forceinline__ void qft_chunk(const KOp<R>* __restrict__ op, const KHdr& h, vec2_t<R> (&a)[1 << NR],
                                          uint64_t gthr) {
  if constexpr (L >= 1 && L <= NR && TOP < NR && TOP - L + 1 >= 0) {
    const unsigned fl = h.flags;
    const R scale = op->m[0];
    bool scaled = !(fl & F_SCALE);
    const uint64_t lv = gthr & op->qmask;
    if (fl & F_ENTRY) {
      const uint64_t th_all = __brevll(gthr & op->tmask), th_new = __brevll(gthr & op->tval);
      uint64_t ut[NR];
#pragma unroll
      for (int p = 0; p < NR; ++p) ut[p] = th_all << ((h.lo + p - (TOP - L + 1)) & 63);
      const bool here = !scaled && !(fl & F_END);
      qft_phase<R, NR, L, TOP>(a, th_new * lv, ut, here ? scale : (R)1);
      scaled = scaled || here;
    }
    qft_layers<R, NR, L, TOP, TOP>(a);
    if (fl & F_END) {
      uint64_t ut[NR];
#pragma unroll
      for (int p = 0; p < NR; ++p) ut[p] = lv << ((63 - (h.lo + p - (TOP - L + 1))) & 63);
      qft_phase<R, NR, L, TOP>(a, 0, ut, scaled ? (R)1 : scale);
      scaled = true;
    }
    if (!scaled) {
#pragma unroll
      for (int e = 0; e < (1 << NR); ++e) a[e] = mk<R>(a[e].x * scale, a[e].y * scale);
    }
  }
}

template <typename R, int NR>
__device__ __forceinline__ void qft_dispatch(const KOp<R>* __restrict__ op, const KHdr& h, vec2_t<R> (&a)[1 << NR],
                                             uint64_t gthr) {
  switch (h.nbits * 8 + h.slot) {
#define SK_Q(L, TOP) \
  case L * 8 + TOP: qft_chunk<R, NR, L, TOP>(op, h, a, gthr); break;
    SK_Q(1, 0) SK_Q(1, 1) SK_Q(1, 2) SK_Q(1, 3)
    SK_Q(2, 1) SK_Q(2, 2) SK_Q(2, 3)
    SK_Q(3, 2) SK_Q(3, 3)
    SK_Q(4, 3)
#undef SK_Q
    default: break;
  }
}

template <typename R, int NR>
__device__ __forceinline__ void apply_kop(const KOp<R>* __restrict__ op, vec2_t<R> (&a)[1 << NR], uint64_t gthr) {
  const uint4 raw = *reinterpret_cast<const uint4*>(&op->h);
  KHdr h;
  memcpy(&h, &raw, sizeof(h));
  if (h.kind == K_QFTS) {
    qft_dispatch<R, NR>(op, h, a, gthr);
    return;
  }
  if ((h.flags & F_TPRED) && (gthr & op->tmask) != op->tval) return;
  const uint32_t emask = h.emask;
  const int kind = h.kind;
  if (kind == K_BFLY) {
    const vec2_t<R> c0 = mk<R>(op->m[0], op->m[1]);
    vec2_t<R> c1 = mk<R>(op->m[4], op->m[5]);
    if (h.flags & F_FOLD) c1 = PK<R>::mul(c1, thread_phase<R>(op->turn, gthr, h.lo, op->fmask));
    vec2_t<R> w[1 << (NR - 1)];
    if (h.flags & F_TABLE) {
#pragma unroll
      for (int k = 0; k < (1 << (NR - 1)); ++k) w[k] = PK<R>::mul(c1, mk<R>(op->tw[2 * k], op->tw[2 * k + 1]));
    } else {
#pragma unroll
      for (int k = 0; k < (1 << (NR - 1)); ++k) w[k] = c1;
    }
    const unsigned fl = h.flags;
#define SK_BF(P) bfly_slot<R, NR, P>(a, c0, w, fl)
    SK_SLOT_SWITCH(h.slot, SK_BF)
#undef SK_BF
  } else if (kind == K_PHASE || kind == K_TPHASE) {
    vec2_t<R> c;
    if (kind == K_PHASE)
      c = ((h.flags & F_QMASK) && (gthr & op->qmask)) ? mk<R>(op->m[2], op->m[3]) : mk<R>(op->m[0], op->m[1]);
    else
      c = thread_phase<R>(op->turn, gthr, h.lo, op->fmask);
    if (!phase_dispatch<R, NR>(h.pat, a, c)) {
#pragma unroll
      for (int e = 0; e < (1 << NR); ++e)
        if ((emask >> e) & 1u) a[e] = PK<R>::mul(a[e], c);
    }
  } else if (kind == K_MATR) {
    const R m00 = op->m[0], m01 = op->m[2], m10 = op->m[4], m11 = op->m[6];
#define SK_MR(P) matr_slot<R, NR, P>(a, m00, m01, m10, m11, emask)
    SK_SLOT_SWITCH(h.slot, SK_MR)
#undef SK_MR
  } else {  // K_MAT
    vec2_t<R> c[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      c[2 * i] = mk<R>(op->m[2 * i], op->m[2 * i + 1]);
      c[2 * i + 1] = mk<R>(op->mr[2 * i], op->mr[2 * i + 1]);
    }
    if (h.flags & F_FOLD) {
      const vec2_t<R> tau = thread_phase<R>(op->turn, gthr, h.lo, op->fmask);
      c[4] = PK<R>::mul(c[4], tau);
      c[6] = PK<R>::mul(c[6], tau);
      c[5] = mk<R>(-c[4].y, c[4].x);
      c[7] = mk<R>(-c[6].y, c[6].x);
    }
#define SK_M(P) mat_slot<R, NR, P>(a, c, emask)
    SK_SLOT_SWITCH(h.slot, SK_M)
#undef SK_M
  }
}

// unpredicated dense 2x2 on slot P from c[0..7] = m00 r00 m01 r01 m10 r10 m11 r11
// (r = m rotated by i): 8 (fp32) paired ops per element pair
template <typename R, int NR, int P>
__device__ __forceinline__ void mat_full_c(vec2_t<R> (&a)[1 << NR], const vec2_t<R> (&c)[8]) {
#pragma unroll
  for (int e = 0; e < (1 << NR); ++e) {
    if ((e >> P) & 1) continue;
    const int e1 = e | (1 << P);
    const vec2_t<R> y0 = cmac2<R>(a[e], a[e1], c[0], c[1], c[2], c[3]);
    const vec2_t<R> y1 = cmac2<R>(a[e], a[e1], c[4], c[5], c[6], c[7]);
    a[e] = y0;
    a[e1] = y1;
  }
}

// dense 2x2 on slot P restricted to the pairs whose register slot Q == V
template <typename R, int NR, int P, int Q, int V>
__device__ __forceinline__ void mat_q_c(vec2_t<R> (&a)[1 << NR], const vec2_t<R> (&c)[8]) {
  if constexpr (P < NR && Q < NR && P != Q) {
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e) {
      if (((e >> P) & 1) || ((e >> Q) & 1) != V) continue;
      const int e1 = e | (1 << P);
      const vec2_t<R> y0 = cmac2<R>(a[e], a[e1], c[0], c[1], c[2], c[3]);
      const vec2_t<R> y1 = cmac2<R>(a[e], a[e1], c[4], c[5], c[6], c[7]);
      a[e] = y0;
      a[e1] = y1;
    }
  }
}

__device__ __forceinline__ void swap_bits(float& a, float& b, uint64_t m) {
  const uint32_t x = __float_as_uint(a), y = __float_as_uint(b), t = (x ^ y) & (uint32_t)m;
  a = __uint_as_float(x ^ t);
  b = __uint_as_float(y ^ t);
}
__device__ __forceinline__ void swap_bits(double& a, double& b, uint64_t m) {
  const uint64_t x = (uint64_t)__double_as_longlong(a), y = (uint64_t)__double_as_longlong(b), t = (x ^ y) & m;
  a = __longlong_as_double((long long)(x ^ t));
  b = __longlong_as_double((long long)(y ^ t));
}

template <typename R>
struct SignBit;
template <>
struct SignBit<float> {
  static constexpr uint64_t value = 0x80000000ull;
};
template <>
struct SignBit<double> {
  static constexpr uint64_t value = 0x8000000000000000ull;
};

__device__ __forceinline__ float flip_bits(float x, uint64_t m) { return __uint_as_float(__float_as_uint(x) ^ (uint32_t)m); }
__device__ __forceinline__ double flip_bits(double x, uint64_t m) {
  return __longlong_as_double(__double_as_longlong(x) ^ (long long)m);
}


// real 2x2 on slot P: y0 = m00 a0 + m01 a1, y1 = m10 a0 + m11 a1 (2 paired
// instructions per output in fp32, half the dense 2x2)
template <typename R, int NR, int P>
__device__ __forceinline__ void matr_full_c(vec2_t<R> (&a)[1 << NR], const vec2_t<R> (&c)[8]) {
  matr_slot<R, NR, P>(a, c[0].x, c[2].x, c[4].x, c[6].x, PairMask<NR, P>::value());
}

// A LEAN sweep's ops travel in the kernel's parameter space (LSweep, up to
// kLeanOps ops): warp-uniform constant-bank operands, so coefficients are
// LDCU loads into uniform registers read directly by FFMA2/FMUL2 — no vector
// registers, no LSU traffic and a short dispatch chain per op.
template <typename R>
struct alignas(16) LOp {
  KHdr h;
  uint64_t tmask, tval;  // thread-side predicate
  uint64_t qmask, pad;   // K_PHASE: c1 when (gthr & qmask) != 0
  R m[8];                // 2x2 (or phase c0 = m[0..1], c1 = m[2..3])
  R mr[8];               // m rotated by i per entry
};
constexpr int kLeanOps = 128;

template <typename R>
struct LSweep {
  DSweep d;  // op_begin / op_end index op[]
  LOp<R> op[kLeanOps];
};

template <typename R>
__device__ __forceinline__ void coefs_of(const LOp<R>& op, vec2_t<R> (&c)[8]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    c[2 * i] = mk<R>(op.m[2 * i], op.m[2 * i + 1]);
    c[2 * i + 1] = mk<R>(op.mr[2 * i], op.mr[2 * i + 1]);
  }
}

// thread-predicated 2x2: the identity where the predicate fails (selects, no
// divergent exit: the op loop stays warp-uniform so its indices and
// coefficients live in uniform registers)
template <typename R>
__device__ __forceinline__ void coefs_if(const LOp<R>& op, vec2_t<R> (&c)[8], bool p) {
  coefs_of<R>(op, c);
  const R one = 1, zero = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool diag = i == 0 || i == 1 || i == 6 || i == 7;  // m00, r00, m11, r11
    const bool rot = i & 1;                                   // identity r = (0, 1)
    const R ix = diag && !rot ? one : zero, iy = diag && rot ? one : zero;
    c[i] = mk<R>(p ? c[i].x : ix, p ? c[i].y : iy);
  }
}

// [[c, -s w], [s, c w]] on slot P (c, s real, |w| = 1; split_1q's gates):
// t = w a1 (w and its rotation wr = (-w.y, w.x) as packed operands), then
// y0 = c a0 - s t, y1 = s a0 + c t: 6 paired instructions per pair, not 8
template <typename R, int NR, int P>
__device__ __forceinline__ void matrp_slot(vec2_t<R> (&a)[1 << NR], R c, R s, vec2_t<R> w, vec2_t<R> wr) {
  if constexpr (P < NR) {
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e) {
      if ((e >> P) & 1) continue;
      const int e1 = e | (1 << P);
      const vec2_t<R> x0 = a[e], x1 = a[e1];
      if constexpr (sizeof(R) == 4) {
        const float2 t = __ffma2_rn(make_float2(x1.y, x1.y), wr, __fmul2_rn(make_float2(x1.x, x1.x), w));
        a[e] = __ffma2_rn(t, make_float2(-s, -s), __fmul2_rn(x0, make_float2(c, c)));
        a[e1] = __ffma2_rn(t, make_float2(c, c), __fmul2_rn(x0, make_float2(s, s)));
      } else {
        const vec2_t<R> t = mk<R>(x1.x * w.x - x1.y * w.y, x1.x * w.y + x1.y * w.x);
        a[e] = mk<R>(c * x0.x - s * t.x, c * x0.y - s * t.y);
        a[e1] = mk<R>(s * x0.x + c * t.x, s * x0.y + c * t.y);
      }
    }
  }
}

template <typename R, int NR, int P, int V>
__device__ __forceinline__ void phase_slot(vec2_t<R> (&a)[1 << NR], vec2_t<R> c) {
  if constexpr (P < NR) {
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e)
      if (((e >> P) & 1) == V) a[e] = PK<R>::mul(a[e], c);
  }
}

// compile-time dispatch of a warp-uniform index by binary search: nested
// two-way branches stay uniform (BRA.U), where a large switch becomes a
// jump table whose indirect branch pushes the whole op loop (index,
// coefficients) out of the uniform datapath
template <int LO, int HI, typename F>
__device__ __forceinline__ void sel(int i, F&& f) {
  if constexpr (HI - LO == 1) {
    f(std::integral_constant<int, LO>{});
  } else {
    constexpr int MID = (LO + HI) / 2;
    if (i < MID)
      sel<LO, MID>(i, f);
    else
      sel<MID, HI>(i, f);
  }
}

// masked forms (one code path per slot instead of one per register-control
// pattern: less hot code): the pairs / elements to touch are the bits of a
// runtime mask em (already zero when the thread predicate fails)
template <typename R, int NR, int P>
__device__ __forceinline__ void swap_mask(vec2_t<R> (&a)[1 << NR], uint32_t em) {
  if constexpr (P < NR) {
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e) {
      if ((e >> P) & 1) continue;
      const uint64_t m = 0ull - (uint64_t)((em >> e) & 1u);
      swap_bits(a[e].x, a[e | (1 << P)].x, m);
      swap_bits(a[e].y, a[e | (1 << P)].y, m);
    }
  }
}

template <typename R, int NR, int P>
__device__ __forceinline__ void yswap_mask(vec2_t<R> (&a)[1 << NR], uint32_t em) {
  if constexpr (P < NR) {
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e) {
      if ((e >> P) & 1) continue;
      const int e1 = e | (1 << P);
      const uint64_t m = 0ull - (uint64_t)((em >> e) & 1u), sb = m & SignBit<R>::value;
      R a0x = a[e].x, a0y = a[e].y, a1x = a[e1].x, a1y = a[e1].y;
      swap_bits(a0x, a1y, m);
      swap_bits(a0y, a1x, m);
      a[e] = mk<R>(a0x, flip_bits(a0y, sb));
      a[e1] = mk<R>(flip_bits(a1x, sb), a1y);
    }
  }
}

template <typename R, int NR>
__device__ __forceinline__ void sign_mask(vec2_t<R> (&a)[1 << NR], uint32_t em) {
#pragma unroll
  for (int e = 0; e < (1 << NR); ++e) {
    const uint64_t sb = (0ull - (uint64_t)((em >> e) & 1u)) & SignBit<R>::value;
    a[e] = mk<R>(flip_bits(a[e].x, sb), flip_bits(a[e].y, sb));
  }
}

// LEAN dispatch: one uniform branch tree per op (opcode class, then the
// slot); thread predicates are masks and selects, never exits.  H tiles per
// thread (a[h], their index parts gthr[h]): one dispatch and one set of
// (uniform) coefficients serve H independent element groups.
template <typename R, int NR, int H>
__device__ __forceinline__ void lean_op(const LOp<R>& op, uint32_t opc, vec2_t<R> (&a)[H][1 << NR],
                                        const uint64_t (&gthr)[H]) {
  const int o = (int)opc;
  if (o < OPC_MATR) {
    if (o < OPC_MATRP) {  // dense 2x2
      vec2_t<R> c[8];
      coefs_of<R>(op, c);
      sel<0, 4>(o - OPC_MAT, [&](auto k) {
        constexpr int P = decltype(k)::value;
#pragma unroll
        for (int h = 0; h < H; ++h)
          if constexpr (P < NR) mat_full_c<R, NR, P>(a[h], c);
      });
    } else {  // real first column: m = c, s; mr = w, wr
      const R c = op.m[0], sn = op.m[4];
      const vec2_t<R> w = mk<R>(op.mr[0], op.mr[1]), wr = mk<R>(op.mr[2], op.mr[3]);
      sel<0, 4>(o - OPC_MATRP, [&](auto k) {
#pragma unroll
        for (int h = 0; h < H; ++h) matrp_slot<R, NR, decltype(k)::value>(a[h], c, sn, w, wr);
      });
    }
    return;
  }
  if (o >= OPC_SWAPM && o < OPC_DIAG1) {  // masked X / Y / sign couplers
    uint32_t em[H];
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const bool p = (gthr[h] & op.tmask) == op.tval && (op.qmask == 0 || (gthr[h] & op.qmask) != 0);
      em[h] = p ? op.h.emask : 0u;
    }
    if (o == OPC_SIGNM) {
#pragma unroll
      for (int h = 0; h < H; ++h) sign_mask<R, NR>(a[h], em[h]);
    } else if (o >= OPC_YSWAPM) {
      sel<0, 4>(o - OPC_YSWAPM, [&](auto k) {
#pragma unroll
        for (int h = 0; h < H; ++h) yswap_mask<R, NR, decltype(k)::value>(a[h], em[h]);
      });
    } else {
      sel<0, 4>(o - OPC_SWAPM, [&](auto k) {
#pragma unroll
        for (int h = 0; h < H; ++h) swap_mask<R, NR, decltype(k)::value>(a[h], em[h]);
      });
    }
    return;
  }
  if (o < OPC_MATT) {  // real 2x2
    vec2_t<R> c[8];
    coefs_of<R>(op, c);
    sel<0, 4>(o - OPC_MATR, [&](auto k) {
      constexpr int P = decltype(k)::value;
#pragma unroll
      for (int h = 0; h < H; ++h)
        if constexpr (P < NR) matr_full_c<R, NR, P>(a[h], c);
    });
    return;
  }
  if (o < OPC_MATQ) {  // dense 2x2 behind a thread predicate (identity where it fails)
#pragma unroll
    for (int h = 0; h < H; ++h) {
      vec2_t<R> c[8];
      coefs_if<R>(op, c, (gthr[h] & op.tmask) == op.tval);
      sel<0, 4>(o - OPC_MATT, [&](auto k) {
        constexpr int P = decltype(k)::value;
        if constexpr (P < NR) mat_full_c<R, NR, P>(a[h], c);
      });
    }
    return;
  }
  if (o < OPC_SWAPM) {  // dense 2x2 on the pairs with slot Q == V
#pragma unroll
    for (int h = 0; h < H; ++h) {
      vec2_t<R> c[8];
      coefs_if<R>(op, c, (gthr[h] & op.tmask) == op.tval);
      sel<0, 32>(o - OPC_MATQ, [&](auto k) {
        constexpr int K = decltype(k)::value;
        mat_q_c<R, NR, K / 8, (K / 2) % 4, K % 2>(a[h], c);
      });
    }
    return;
  }
  if (o < OPC_PHASE) {  // phase on one slot value
    const vec2_t<R> c = mk<R>(op.m[0], op.m[1]);
    sel<0, 8>(o - OPC_DIAG1, [&](auto k) {
      constexpr int K = decltype(k)::value;
#pragma unroll
      for (int h = 0; h < H; ++h) phase_slot<R, NR, K / 2, K % 2>(a[h], c);
    });
    return;
  }
  // OPC_PHASE: a selected multiplier per element
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const vec2_t<R> c = (gthr[h] & op.qmask) ? mk<R>(op.m[2], op.m[3]) : mk<R>(op.m[0], op.m[1]);
    const uint32_t em = (gthr[h] & op.tmask) == op.tval ? op.h.emask : 0u;
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e) {
      const bool hit = (em >> e) & 1u;
      a[h][e] = PK<R>::mul(a[h][e], mk<R>(hit ? c.x : (R)1, hit ? c.y : (R)0));
    }
  }
}

// Generic fused sweep (random circuits, mixed gate streams): NS compile-time
// stages with per-thread index parts from the host-built table `thr`
// (uint4 per stage and thread: global bits lo/hi, swizzled shared offset),
// ops interpreted from `ops` with warp-uniform loads and packed arithmetic.
__device__ __forceinline__ const DSweep& dsweep_of(const DSweep& s) { return s; }
template <typename R>
__device__ __forceinline__ const DSweep& dsweep_of(const LSweep<R>& s) { return s.d; }

template <typename R, bool LEAN>
using SweepArg = std::conditional_t<LEAN, LSweep<R>, DSweep>;

// H = 2 (LEAN fp32): each CTA runs tiles 2b and 2b + 1 together, each thread
// holding its 16 amplitudes of both, so every op dispatch and coefficient
// load serves twice the arithmetic
template <typename R, int NR, int NS, bool LEAN, int H>
__device__ __forceinline__ void sweep_body(vec2_t<R>* __restrict__ amps, const SweepArg<R, LEAN>& arg,
                                           const KOp<R>* __restrict__ ops, const uint4* __restrict__ thr) {
  using V = vec2_t<R>;
  const DSweep& sw = dsweep_of(arg);
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int NE = 1 << NR;
  const uint32_t tid = threadIdx.x;
  const int nthreads = blockDim.x;
  const size_t tile_bytes = ((size_t)nthreads << NR) * sizeof(V);
  uint64_t base[H];
#pragma unroll
  for (int h = 0; h < H; ++h) base[h] = deposit((uint64_t)blockIdx.x * H + h, sw.brun, sw.nb);

  V a[H][NE];
#pragma unroll 1
  for (int s = 0; s < NS; ++s) {  // not unrolled: one copy of the op loop (its uniform index) per kernel
    const DStage& st = sw.st[s];
    const uint4 t = __ldg(thr + s * nthreads + tid);
    uint64_t gthr[H];
#pragma unroll
    for (int h = 0; h < H; ++h) gthr[h] = base[h] | ((uint64_t)t.y << 32 | t.x);
    if (s == 0) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const char* p = reinterpret_cast<const char*>(amps + gthr[h]);
#pragma unroll
        for (int k = 0; k < NE; ++k) {
          const int e = k ^ (k >> 1);
          if (k) {
            const int b = ctz_c(k);
            p = ((e >> b) & 1) ? p + st.reg_goff[b] : p - st.reg_goff[b];
          }
          a[h][e] = *reinterpret_cast<const V*>(p);
        }
      }
    } else {
      __syncthreads();
#pragma unroll
      for (int h = 0; h < H; ++h) {
        uint32_t so = t.z;
#pragma unroll
        for (int k = 0; k < NE; ++k) {
          const int e = k ^ (k >> 1);
          if (k) so ^= st.reg_soff[ctz_c(k)];
          a[h][e] = *reinterpret_cast<const V*>(smraw + h * tile_bytes + so);
        }
      }
    }
    if constexpr (LEAN) {  // every op of the sweep has a fast path: no interpreter in the loop
      for (int o = st.op_begin; o < st.op_end; ++o) lean_op<R, NR, H>(arg.op[o], arg.op[o].h.opc, a, gthr);
    } else {
      // sweeps with ops outside the fast-path set are interpreted op by op
      // (inlining the fast-path table here too multiplied nvcc time)
#pragma unroll
      for (int h = 0; h < H; ++h)
        for (int o = st.op_begin; o < st.op_end; ++o) apply_kop<R, NR>(ops + o, a[h], gthr[h]);
    }
    if (s == NS - 1) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        char* p = reinterpret_cast<char*>(amps + gthr[h]);
#pragma unroll
        for (int k = 0; k < NE; ++k) {
          const int e = k ^ (k >> 1);
          if (k) {
            const int b = ctz_c(k);
            p = ((e >> b) & 1) ? p + st.reg_goff[b] : p - st.reg_goff[b];
          }
          *reinterpret_cast<V*>(p) = a[h][e];
        }
      }
    } else {
      if (s > 0) __syncthreads();
#pragma unroll
      for (int h = 0; h < H; ++h) {
        uint32_t so = t.z;
#pragma unroll
        for (int k = 0; k < NE; ++k) {
          const int e = k ^ (k >> 1);
          if (k) so ^= st.reg_soff[ctz_c(k)];
          *reinterpret_cast<V*>(smraw + h * tile_bytes + so) = a[h][e];
        }
      }
    }
  }
}

template <typename R, int NR, int NS, bool LEAN, int H = 1>
__global__ void k_sweep(vec2_t<R>* __restrict__ amps, const __grid_constant__ SweepArg<R, LEAN> arg,
                        const KOp<R>* __restrict__ ops, const uint4* __restrict__ thr) {
  sweep_body<R, NR, NS, LEAN, H>(amps, arg, ops, thr);
}

#ifndef SK_SWEEP1_MINB
#define SK_SWEEP1_MINB 6
#endif
// one-tile LEAN kernel for 128-thread tiles with a register budget for
// SK_SWEEP1_MINB resident CTAs (0: use k_sweep, no bound).  c128 random
// 30x20: 472 ms at 6 (80 registers) vs 497 unbounded (96) and 511 at 7
// (72 registers, spills); A/B alternated on one box.
template <typename R, int NR, int NS>
__global__ void __launch_bounds__(128, (SK_SWEEP1_MINB > 0 ? SK_SWEEP1_MINB : 1)) k_sweep1(vec2_t<R>* __restrict__ amps,
                                                             const __grid_constant__ LSweep<R> arg,
                                                             const KOp<R>* __restrict__ ops,
                                                             const uint4* __restrict__ thr) {
  sweep_body<R, NR, NS, true, 1>(amps, arg, ops, thr);
}

#ifndef SK_SWEEP2_MINB
#define SK_SWEEP2_MINB 4
#endif
// the two-tile fp32 kernel for 128-thread tiles (T = NR + 7), with a
// register budget for SK_SWEEP2_MINB resident CTAs.  c64 random 30x20:
// 179.5 ms at 4 (128 registers) vs 192.4 unbounded (same register count:
// the bound changes the schedule) and 210.7 at 5 (96 registers, spills).
template <typename R, int NR, int NS>
__global__ void __launch_bounds__(128, SK_SWEEP2_MINB) k_sweep2(vec2_t<R>* __restrict__ amps,
                                                             const __grid_constant__ LSweep<R> arg,
                                                             const KOp<R>* __restrict__ ops,
                                                             const uint4* __restrict__ thr) {
  sweep_body<R, NR, NS, true, 2>(amps, arg, ops, thr);
}

// ---------------------------------------------------------------------------
// k_qft: the QFT-window sweep with every chunk parameter in the (constant-
// bank) kernel argument instead of an op stream, and packed arithmetic
// (PK<R>: FADD2/FMUL2/FFMA2 for fp32).  Same math as qft_chunk above — the
// host builds its QSweep from the same lowered K_QFTS ops
// (qsweep_from), so tests/test_kernel_lowering.py's emulation covers both.
// Per amplitude and 4-layer chunk: 4 paired adds for the butterflies, ~1.25
// paired multiply pairs for the compile-time internal twiddles, and 4 paired
// ops per Gray-walked entry / end phase.
// ---------------------------------------------------------------------------
constexpr int kQRuns = 4;

struct QStage {
  int code;  // L * 8 + TOP of the stage's chunk; 0 = no chunk (store stage)
  uint32_t flags;
  int lo, pad;
  uint64_t tmask, tval, qmask;
  double scale;
  uint64_t reg_goff[kMaxR];
  uint32_t reg_soff[kMaxR];
};

// Per-thread index parts are precomputed on the host (thr table, one uint4
// per stage and thread: global index bits lo/hi, swizzled shared-memory
// byte offset): one L1-resident 16-byte load per thread and stage instead of
// a bit-deposit.
struct QSweep {
  int ntile, nstages, nb, nthreads;
  int tma;           // last stage stores the tile with one TMA bulk-tensor copy (see k_qft)
  int pshift;        // phase index = (address index << pshift) | pconst (a shard whose low
  uint64_t pconst;   // pshift QFT qubits are rank constants; 0 / 0 otherwise)
  int tile0;         // first tile of this launch (sk_program_run_tiles; 0 = the whole sweep from tile 0)
  int pad5;
  Run brun[kQRuns];
  const uint4* thr;  // [nstages][nthreads]
  QStage st[kMaxS];
};

__device__ __forceinline__ uint64_t deposit_q(uint64_t x, const Run* r, int n) {
  uint64_t o = 0;
#pragma unroll
  for (int i = 0; i < kQRuns; ++i)
    if (i < n) o |= ((x >> r[i].src) & ((1ull << r[i].w) - 1)) << r[i].dst;
  return o;
}

// cos(pi K / 16) for K = 0..15 (sin(pi K / 16) = cos16(8 - K) for K <= 8)
__host__ __device__ constexpr double cos16(int K) {
  return K == 0 ? 1.0 : K == 1 ? 0.98078528040323044 : K == 2 ? 0.92387953251128674 : K == 3 ? 0.83146961230254524
       : K == 4 ? 0.70710678118654752 : K == 5 ? 0.55557023301960218 : K == 6 ? 0.38268343236508978
       : K == 7 ? 0.19509032201612826 : K == 8 ? 0.0 : -cos16(16 - K);
}
__host__ __device__ constexpr double sin16(int K) { return K <= 8 ? cos16(8 - K) : cos16(K - 8); }

template <typename R, int K>
__device__ __forceinline__ vec2_t<R> pk_pi16(vec2_t<R> x) {  // x * exp(i pi K / 16), 0 <= K < 16 compile-time
  if constexpr (K == 0) return x;
  else if constexpr (K == 8) return mk<R>(-x.y, x.x);
  else return PK<R>::mul(x, mk<R>((R)cos16(K), (R)sin16(K)));
}

template <int NR, int L, int TOP, int P, int E>
__host__ __device__ constexpr int qft_k16() {  // internal twiddle of pair base E at layer slot P, units of pi/16
  int k = 0;
  for (int p = TOP - L + 1; p < P; ++p)
    if ((E >> p) & 1) k += 1 << (4 - (P - p));
  return k;
}

template <typename R, int NR, int L, int TOP, int P, int E>
__device__ __forceinline__ void pk_pair(vec2_t<R> (&a)[1 << NR]) {
  if constexpr (E < (1 << NR)) {
    if constexpr (!((E >> P) & 1)) {
      constexpr int E1 = E | (1 << P);
      const vec2_t<R> s = PK<R>::add(a[E], a[E1]);
      const vec2_t<R> d = PK<R>::sub(a[E], a[E1]);
      a[E] = s;
      a[E1] = pk_pi16<R, qft_k16<NR, L, TOP, P, E>()>(d);
    }
    pk_pair<R, NR, L, TOP, P, E + 1>(a);
  }
}

template <typename R, int NR, int L, int TOP, int P>
__device__ __forceinline__ void pk_layers(vec2_t<R> (&a)[1 << NR]) {
  if constexpr (P >= TOP - L + 1 && P >= 0) {
    pk_pair<R, NR, L, TOP, P, 0>(a);
    pk_layers<R, NR, L, TOP, P - 1>(a);
  }
}

// a[e] *= phase(base + sum_{chunk slots p} e_p u_p) * scale, Gray-walked:
// per element one paired multiply to step the phase and one to apply it.
// The slot phases are successive doublings of one angle (DIR = +1: ut[p+1] =
// 2 ut[p], the entry phase; DIR = -1: ut[p-1] = 2 ut[p], the end phase), so in
// fp64 one sincospi plus complex squarings replaces L of them (the sincospi
// calls were a third of the c128 sweep's FP64 pipe work); fp32 keeps one MUFU
// sincos per slot.
template <typename R, int NR, int L, int TOP, int DIR, bool ZERO_BASE>
__device__ __forceinline__ void pk_phase(vec2_t<R> (&a)[1 << NR], uint64_t base, const uint64_t (&ut)[NR], R scale) {
  using P = PK<R>;
  constexpr int B0 = TOP - L + 1;
  vec2_t<R> u[NR], uc[NR];
  if constexpr (sizeof(R) == 8) {
    constexpr int first = DIR > 0 ? B0 : TOP;
    u[first] = turn_phase<R>(ut[first]);
#pragma unroll
    for (int i = 1; i < L; ++i) {
      const int p = DIR > 0 ? B0 + i : TOP - i, q = DIR > 0 ? p - 1 : p + 1;
      const vec2_t<R> v = u[q];
      u[p] = mk<R>(v.x * v.x - v.y * v.y, 2.0 * v.x * v.y);
    }
#pragma unroll
    for (int p = B0; p <= TOP; ++p) uc[p] = P::conj(u[p]);
  } else {
#pragma unroll
    for (int p = 0; p < NR; ++p)
      if (p >= B0 && p <= TOP) {
        u[p] = turn_phase<R>(ut[p]);
        uc[p] = P::conj(u[p]);
      }
  }
  vec2_t<R> w = ZERO_BASE ? mk<R>(scale, (R)0) : P::scale(turn_phase<R>(base), scale);
  a[0] = P::mul(a[0], w);
#pragma unroll
  for (int k = 1; k < (1 << NR); ++k) {
    const int b = ctz_c(k);
    const int e = k ^ (k >> 1);
    if (b >= B0 && b <= TOP) w = P::mul(w, ((e >> b) & 1) ? u[b] : uc[b]);
    a[e] = P::mul(a[e], w);
  }
}

template <typename R, int NR, int L, int TOP>
__device__ __forceinline__ void pk_chunk(const QStage& st, vec2_t<R> (&a)[1 << NR], uint64_t gthr) {
  if constexpr (L >= 1 && L <= NR && TOP < NR && TOP - L + 1 >= 0) {
    constexpr int B0 = TOP - L + 1;
    const unsigned fl = st.flags;
    const R scale = (R)st.scale;
    bool scaled = !(fl & F_SCALE);
    const uint64_t lv = gthr & st.qmask;
    if (fl & F_ENTRY) {
      const uint64_t th_all = __brevll(gthr & st.tmask), th_new = __brevll(gthr & st.tval);
      uint64_t ut[NR];
#pragma unroll
      for (int p = 0; p < NR; ++p) ut[p] = (p >= B0 && p <= TOP) ? th_all << ((st.lo + p - B0) & 63) : 0;
      const bool here = !scaled && !(fl & F_END);
      pk_phase<R, NR, L, TOP, +1, false>(a, th_new * lv, ut, here ? scale : (R)1);
      scaled = scaled || here;
    }
    pk_layers<R, NR, L, TOP, TOP>(a);
    if (fl & F_END) {
      uint64_t ut[NR];
#pragma unroll
      for (int p = 0; p < NR; ++p) ut[p] = (p >= B0 && p <= TOP) ? lv << ((63 - (st.lo + p - B0)) & 63) : 0;
      pk_phase<R, NR, L, TOP, -1, true>(a, 0, ut, scaled ? (R)1 : scale);
      scaled = true;
    }
    if (!scaled) {
#pragma unroll
      for (int e = 0; e < (1 << NR); ++e) a[e] = PK<R>::scale(a[e], scale);
    }
  }
}

// 16 fp32 amplitudes per thread fit 64 registers (512 threads x 2 CTAs);
// 32 fp32 or 16 fp64 amplitudes get 128 (tiles of <= 256 threads)
template <typename R, int NR>
constexpr int qft_max_threads() { return (sizeof(R) == 4 && NR <= 4) ? 512 : (sizeof(R) == 8 && NR == 4) ? 128 : 256; }
// c128 with 16 amplitudes per thread: 128-thread tiles, 4 resident per SM at
// <= 128 registers (5 per SM would need <= 102 registers: 1-3 KB of spills)
template <typename R, int NR>
constexpr int qft_min_blocks() { return (sizeof(R) == 8 && NR == 4) ? 4 : 2; }

template <typename R, int NR, int NS>
__global__ void __launch_bounds__(qft_max_threads<R, NR>(), (qft_min_blocks<R, NR>())) k_qft(vec2_t<R>* __restrict__ amps, const __grid_constant__ QSweep sw,
                                                                    const __grid_constant__ CUtensorMap tmap) {
  using V = vec2_t<R>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  constexpr int NE = 1 << NR;
  const uint32_t tid = threadIdx.x;
  const uint64_t base = deposit_q(blockIdx.x + (uint64_t)sw.tile0, sw.brun, sw.nb);

  V a[NE];
#pragma unroll
  for (int s = 0; s < NS; ++s) {  // compile-time stages: every st.* is a constant-bank operand
    const QStage& st = sw.st[s];
    const uint4 t = __ldg(sw.thr + s * sw.nthreads + tid);
    const uint64_t gthr = base | ((uint64_t)t.y << 32 | t.x);
    if (s == 0) {
      const char* p = reinterpret_cast<const char*>(amps + gthr);
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const int e = k ^ (k >> 1);
        if (k) {
          const int b = ctz_c(k);
          p = ((e >> b) & 1) ? p + st.reg_goff[b] : p - st.reg_goff[b];
        }
        a[e] = *reinterpret_cast<const V*>(p);
      }
    } else {
      __syncthreads();
      uint32_t so = t.z;
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const int e = k ^ (k >> 1);
        if (k) so ^= st.reg_soff[ctz_c(k)];
        a[e] = *reinterpret_cast<const V*>(smraw + so);
      }
    }
    switch (st.code) {
#define SK_QC(L, TOP) \
  case L * 8 + TOP: pk_chunk<R, NR, L, TOP>(st, a, (gthr << sw.pshift) | sw.pconst); break;
      SK_QC(1, 0) SK_QC(1, 1) SK_QC(1, 2) SK_QC(1, 3) SK_QC(1, 4)
      SK_QC(2, 1) SK_QC(2, 2) SK_QC(2, 3) SK_QC(2, 4)
      SK_QC(3, 2) SK_QC(3, 3) SK_QC(3, 4)
      SK_QC(4, 3) SK_QC(4, 4)
      SK_QC(5, 4)
#undef SK_QC
      default: break;
    }
    if (s == NS - 1) {
      bool done = false;
      if constexpr (NR == 4) {
        if (sw.tma) {
          // The tile is the contiguous index range [base, base + 2^T) and the
          // registers hold index bits 0..3: each thread owns one (c64) or two
          // (c128) 128-byte rows (t.w = its tile-local index).  Rows go to shared memory in the
          // TMA 128B-swizzle layout (16-byte chunk j of row r at chunk j ^ (r & 7):
          // 8 consecutive rows cover all 32 banks), then one thread stores the
          // whole tile with a single bulk-tensor copy.  Replaces the extra
          // shared-memory round trip that would re-map lanes onto the low bits.
          __syncthreads();  // every lane has finished reading this stage's shared-memory input
          if constexpr (sizeof(V) == 8) {  // c64: one 128-byte row = 16 amplitudes = this thread's registers
            const uint32_t row = t.w >> 4;
            unsigned char* rp = smraw + row * 128u;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(rp + ((j ^ (row & 7)) << 4)) =
                  make_float4(a[2 * j].x, a[2 * j].y, a[2 * j + 1].x, a[2 * j + 1].y);
          } else {  // c128: two rows of 8 amplitudes, one 16-byte chunk each
            // Rows 2i and 2i+1 of thread i: with every thread writing the same
            // register at once, the 8 threads of a 16-byte-store phase would
            // cover only 4 distinct (row & 7) values (8 wavefronts instead of
            // 4).  Threads whose even row repeats within the phase write their
            // odd row first, so each phase hits all 8 chunk slots.
            const uint32_t rb = t.w >> 3;
            const uint32_t flip = ((rb >> 3) & 1u) << 3;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              const uint32_t e = (uint32_t)k ^ flip;
              const V v = flip ? a[k ^ 8] : a[k];
              const uint32_t row = rb + (e >> 3);
              *reinterpret_cast<V*>(smraw + row * 128u + (((e & 7u) ^ (row & 7u)) << 4)) = v;
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
          if (tid == 0) {
            const uint32_t sm = (uint32_t)__cvta_generic_to_shared(smraw);
            const int32_t y = (int32_t)(base >> (sizeof(V) == 8 ? 4 : 3));
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tmap), "r"(0),
                "r"(y), "r"(sm)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          done = true;
        }
      }
      if (!done) {
        char* p = reinterpret_cast<char*>(amps + gthr);
#pragma unroll
        for (int k = 0; k < NE; ++k) {
          const int e = k ^ (k >> 1);
          if (k) {
            const int b = ctz_c(k);
            p = ((e >> b) & 1) ? p + st.reg_goff[b] : p - st.reg_goff[b];
          }
          *reinterpret_cast<V*>(p) = a[e];
        }
      }
    } else {
      if (s > 0) __syncthreads();
      uint32_t so = t.z;
#pragma unroll
      for (int k = 0; k < NE; ++k) {
        const int e = k ^ (k >> 1);
        if (k) so ^= st.reg_soff[ctz_c(k)];
        *reinterpret_cast<V*>(smraw + so) = a[e];
      }
    }
  }
}
constexpr int kQftMaxStages = 6;

// register bits per stage: 16 fp32 amplitudes (32 regs) or 8 fp64 (32 regs)
constexpr int kNR32 = 4;
constexpr int kNR64 = 3;
constexpr int kMaxTile32 = 13;  // 64 KiB of shared memory per tile, 512 threads
constexpr int kMaxTile64 = 12;

// ---------------------------------------------------------------------------
// host side: geometry (bit runs) and lowering of ABI ops into kernel ops
// ---------------------------------------------------------------------------
// runs mapping consecutive counter bits 0..k-1 to the ascending positions `dst`
static int make_runs(const std::vector<int>& dst, Run* out) {
  int n = 0;
  for (size_t i = 0; i < dst.size(); ++i) {
    if (n > 0 && out[n - 1].dst + out[n - 1].w == dst[i] && out[n - 1].src + out[n - 1].w == (int)i) {
      out[n - 1].w++;
    } else {
      if (n >= kMaxRuns) return -1;
      out[n].src = (uint8_t)i;
      out[n].dst = (uint8_t)dst[i];
      out[n].w = 1;
      out[n].pad = 0;
      ++n;
    }
  }
  return n;
}

static uint64_t turn_of(double s) {
  // exp(i pi s F) = exp(2 pi i F s/2): s/2 in 2^-64 turns, exact for |s| >~ 2^-11
  int e = 0;
  const double m = std::frexp(0.5 * s, &e);  // 0.5 s = m 2^e, |m| in [0.5, 1)
  const int64_t M = (int64_t)std::ldexp(m, 53);
  const int sh = e + 64 - 53;
  if (sh >= 64) return 0;
  if (sh >= 0) return (uint64_t)M << sh;
  if (sh <= -63) return (uint64_t)(M < 0 ? -1 : 0);
  return (uint64_t)(M >> -sh);
}

struct HostKOp {
  int kind = K_PHASE, slot = -1, pat = -1;
  uint32_t emask = 0, flags = 0;
  int lo = 0, nbits = 0;
  uint64_t tmask = 0, tval = 0, qmask = 0, turn = 0, fmask = 0;
  double m[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double tw[16] = {1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1, 0};
  int nr = 4;  // register bits of the sweep it belongs to (pattern codes depend on it)
};

struct StageCtx {
  int NR;
  int slot_of[64];
  uint64_t regmask;
  uint64_t reg_off[kMaxR];
};

static uint32_t reg_pred_mask(const StageCtx& c, uint64_t cmask, uint64_t cval) {
  uint32_t em = 0;
  for (int e = 0; e < (1 << c.NR); ++e) {
    bool ok = true;
    for (int p = 0; p < c.NR; ++p) {
      const uint64_t bit = c.reg_off[p];
      if (cmask & bit) ok = ok && (((cval & bit) != 0) == (((e >> p) & 1) != 0));
    }
    if (ok) em |= 1u << e;
  }
  return em;
}

static uint32_t slot_mask(int NR, int p, int val) {
  uint32_t em = 0;
  for (int e = 0; e < (1 << NR); ++e)
    if (((e >> p) & 1) == val) em |= 1u << e;
  return em;
}

static bool is_one(double re, double im) { return re == 1.0 && im == 0.0; }

static int pattern_of(int NR, uint32_t emask) {
  const uint32_t all = (1u << (1 << NR)) - 1;
  if (emask == all) return 0;
  for (int p = 0; p < NR; ++p)
    for (int v = 0; v < 2; ++v)
      if (emask == slot_mask(NR, p, v)) return 1 + 2 * p + v;
  int idx = 0;
  for (int p = 0; p < 4; ++p)
    for (int q = p + 1; q < 4; ++q, ++idx) {
      if (q >= NR) continue;
      for (int vp = 0; vp < 2; ++vp)
        for (int vq = 0; vq < 2; ++vq)
          if (emask == (slot_mask(NR, p, vp) & slot_mask(NR, q, vq))) return 9 + 4 * idx + 2 * vp + vq;
    }
  return -1;
}

static void set_pred(HostKOp& k, uint64_t tmask, uint64_t tval) {
  k.tmask = tmask;
  k.tval = tval;
  if (tmask) k.flags |= F_TPRED;
}

// appends the kernel ops of ABI op `o` for one stage
static int lower_op(const StageCtx& c, const sk_op& op, int o, int width, std::vector<HostKOp>& out,
                    double* scale) {
  if (op.ctrl_val & ~op.ctrl_mask) return set_error(SK_EVALUE, "op %d: ctrl_val outside ctrl_mask", o);
  if (width < 64 && (op.ctrl_mask >> width)) return set_error(SK_EVALUE, "op %d: control beyond width %d", o, width);
  const uint64_t tmask = op.ctrl_mask & ~c.regmask, tval = op.ctrl_val & ~c.regmask;
  const uint32_t rpred = reg_pred_mask(c, op.ctrl_mask, op.ctrl_val);
  if (op.kind == SK_OP_MAT) {
    if (op.qubit < 0 || op.qubit >= width || c.slot_of[op.qubit] < 0)
      return set_error(SK_EVALUE, "op %d: MAT target %d is not a register bit of its stage", o, op.qubit);
    if ((op.ctrl_mask >> op.qubit) & 1ull) return set_error(SK_EVALUE, "op %d: target %d is a control", o, op.qubit);
    HostKOp k;
    const int p = c.slot_of[op.qubit];
    bool real = true;
    for (int i = 1; i < 8; i += 2) real = real && op.m[i] == 0.0;
    k.kind = real ? K_MATR : K_MAT;
    k.slot = p;
    k.emask = rpred & slot_mask(c.NR, p, 0);
    set_pred(k, tmask, tval);
    for (int i = 0; i < 8; ++i) k.m[i] = op.m[i];
    const bool bfly = op.m[0] == op.m[2] && op.m[1] == op.m[3] && op.m[4] == -op.m[6] && op.m[5] == -op.m[7];
    if (bfly && k.emask == slot_mask(c.NR, p, 0)) {  // H-like: y0 = c0 (a0 + a1), y1 = c1 (a0 - a1)
      k.kind = K_BFLY;
      k.m[2] = k.m[3] = k.m[6] = k.m[7] = 0;
      if (op.m[1] == 0.0) k.flags |= F_C0REAL;
      const double c0r = op.m[0], c0i = op.m[1], den = c0r * c0r + c0i * c0i;
      if (tmask == 0 && den > 0 && scale != nullptr) {
        // an unpredicated butterfly is c0 * [[1, 1], [c1/c0, -c1/c0]]: defer the scalar c0
        const double qr = (op.m[4] * c0r + op.m[5] * c0i) / den, qi = (op.m[5] * c0r - op.m[4] * c0i) / den;
        const double sr = scale[0] * c0r - scale[1] * c0i, si = scale[0] * c0i + scale[1] * c0r;
        scale[0] = sr;
        scale[1] = si;
        k.m[0] = 1;
        k.m[1] = 0;
        k.m[4] = qr;
        k.m[5] = qi;
        k.flags |= F_C0ONE;
      }
    }
    if (k.emask) out.push_back(k);
    return SK_OK;
  }
  if (op.kind == SK_OP_DIAG) {
    if (op.qubit < 0 || op.qubit >= width) return set_error(SK_EVALUE, "op %d: DIAG qubit %d out of range", o, op.qubit);
    if ((op.ctrl_mask >> op.qubit) & 1ull) return set_error(SK_EVALUE, "op %d: qubit %d is a control", o, op.qubit);
    const int p = c.slot_of[op.qubit];
    if (p >= 0) {
      for (int v = 0; v < 2; ++v) {
        const double re = op.m[v ? 6 : 0], im = op.m[v ? 7 : 1];
        if (is_one(re, im)) continue;
        HostKOp k;
        k.kind = K_PHASE;
        k.emask = rpred & slot_mask(c.NR, p, v);
        set_pred(k, tmask, tval);
        k.m[0] = k.m[2] = re;
        k.m[1] = k.m[3] = im;
        if (k.emask) out.push_back(k);
      }
    } else {
      if (is_one(op.m[0], op.m[1]) && is_one(op.m[6], op.m[7])) return SK_OK;
      HostKOp k;
      k.kind = K_PHASE;
      k.emask = rpred;
      set_pred(k, tmask, tval);
      k.qmask = 1ull << op.qubit;
      k.flags |= F_QMASK;
      k.m[0] = op.m[0];
      k.m[1] = op.m[1];
      k.m[2] = op.m[6];
      k.m[3] = op.m[7];
      if (k.emask) out.push_back(k);
    }
    return SK_OK;
  }
  if (op.kind == SK_OP_RAMP) {
    if (op.qubit < 0 || op.nbits < 1 || op.nbits > 62 || op.qubit + op.nbits > width)
      return set_error(SK_EVALUE, "op %d: bad RAMP field at bit %d", o, op.qubit);
    const uint64_t field = ((1ull << op.nbits) - 1) << op.qubit;
    if (op.ctrl_mask & field) return set_error(SK_EVALUE, "op %d: RAMP field overlaps its controls", o);
    const double s = op.m[0];
    const uint64_t turn = turn_of(s);
    // thread part: one per-thread phase (register bits are zero in gthr)
    bool fold = false;
    if (!out.empty() && tmask == 0) {  // fold into a preceding unpredicated MAT/BFLY on the control slot
      HostKOp& prev = out.back();
      if ((prev.kind == K_MAT || prev.kind == K_MATR || prev.kind == K_BFLY) && prev.tmask == 0 &&
          !(prev.flags & F_FOLD) && prev.emask == slot_mask(c.NR, prev.slot, 0) &&
          rpred == slot_mask(c.NR, prev.slot, 1)) {
        if (prev.kind == K_MATR) prev.kind = K_MAT;
        prev.flags |= F_FOLD;
        prev.lo = op.qubit;
        prev.nbits = op.nbits;
        prev.fmask = (1ull << op.nbits) - 1;
        prev.turn = turn;
        fold = true;
      }
    }
    const bool table = fold && out.back().kind == K_BFLY;
    const int jslot = fold ? out.back().slot : -1;
    if (!fold && rpred) {
      HostKOp t;
      t.kind = K_TPHASE;
      t.emask = rpred;
      set_pred(t, tmask, tval);
      t.lo = op.qubit;
      t.nbits = op.nbits;
      t.fmask = (1ull << op.nbits) - 1;
      t.turn = turn;
      out.push_back(t);
    }
    // register part: constant phases on elements whose field register bit is set
    for (int p = 0; p < c.NR; ++p) {
      const uint64_t bit = c.reg_off[p];
      if (!(bit & field)) continue;
      const int q = __builtin_ctzll(bit);
      double x = s * (double)(1ull << (q - op.qubit));
      x -= 2.0 * std::floor(0.5 * x);
      if (x == 0.0) continue;
      const double wr = std::cos(M_PI * x), wi = std::sin(M_PI * x);
      if (table) {  // multiply into the butterfly's row-1 twiddle of every pair whose e1 has bit p
        HostKOp& bf = out.back();
        for (int k = 0; k < (1 << (c.NR - 1)); ++k) {
          const int e1 = (int)(insert0((uint64_t)k, jslot) | (1u << jslot));
          if (!((e1 >> p) & 1)) continue;
          const double r = bf.tw[2 * k] * wr - bf.tw[2 * k + 1] * wi, i = bf.tw[2 * k] * wi + bf.tw[2 * k + 1] * wr;
          bf.tw[2 * k] = r;
          bf.tw[2 * k + 1] = i;
        }
        bf.flags |= F_TABLE;
        continue;
      }
      HostKOp k;
      k.kind = K_PHASE;
      k.emask = rpred & slot_mask(c.NR, p, 1);
      set_pred(k, tmask, tval);
      k.m[0] = k.m[2] = wr;
      k.m[1] = k.m[3] = wi;
      if (k.emask) out.push_back(k);
    }
    return SK_OK;
  }
  if (op.kind == SK_OP_QFT) {
    const int c_lo = op.qubit, L = op.nbits, c_hi = c_lo + L - 1;
    const int w_lo = (int)op.m[0], w_hi = (int)op.m[1], prev_hi = (int)op.m[2];
    if (L < 1 || L > c.NR || c_lo < w_lo || c_hi > w_hi || w_lo < 0 || w_hi >= width || w_hi - w_lo > 62)
      return set_error(SK_EVALUE, "op %d: bad QFT chunk [%d, %d]", o, c_lo, c_hi);
    const int s0 = c.slot_of[c_lo];
    for (int b = c_lo; b <= c_hi; ++b)
      if (s0 < 0 || c.slot_of[b] != s0 + (b - c_lo))
        return set_error(SK_EVALUE, "op %d: QFT chunk bit %d not in consecutive register slots", o, b);
    const bool entry = c_hi < w_hi, end = c_lo == w_lo && w_lo > 0;
    if (entry && (prev_hi <= c_hi || prev_hi > w_hi)) return set_error(SK_EVALUE, "op %d: bad previous chunk", o);
    for (int p = 0; p < c.NR; ++p) {
      const int q = __builtin_ctzll(c.reg_off[p]);
      if (entry && q > c_hi && q <= w_hi)
        return set_error(SK_EVALUE, "op %d: earlier window bit %d held in a register", o, q);
      if ((entry || end) && q < w_lo) return set_error(SK_EVALUE, "op %d: below-window bit %d in a register", o, q);
    }
    auto range = [](int lo, int hi) -> uint64_t {
      return hi < lo ? 0ull : (((hi - lo + 1) >= 64 ? ~0ull : ((1ull << (hi - lo + 1)) - 1)) << lo);
    };
    HostKOp k;
    k.kind = K_QFTS;
    k.slot = s0 + L - 1;
    k.lo = c_lo;
    k.nbits = L;
    k.flags = (entry ? F_ENTRY : 0u) | (end ? F_END : 0u) | (c_lo == w_lo ? F_SCALE : 0u);
    k.tmask = range(c_hi + 1, w_hi);
    k.tval = entry ? range(c_hi + 1, prev_hi) : 0;
    k.qmask = range(0, w_lo - 1);
    k.m[0] = std::pow(0.5, 0.5 * (w_hi - w_lo + 1));
    out.push_back(k);
    return SK_OK;
  }
  return set_error(SK_EVALUE, "op %d: unknown kind %d", o, op.kind);
}

static uint32_t opcode_of(const HostKOp& k) {
  if (k.nr > 4) return OPC_GENERIC;
  if (k.kind == K_PHASE && k.pat >= 0 && !(k.flags & ~(uint32_t)(F_TPRED | F_QMASK))) {
    // by -1 (CZ-type couplers): sign flips instead of complex multiplies
    const bool q = (k.flags & F_QMASK) != 0;
    if (k.m[2] == -1 && k.m[3] == 0 && k.m[1] == 0 && k.m[0] == (q ? 1 : -1)) return OPC_SIGNM;
    if (k.flags == 0 && k.pat >= 1 && k.pat <= 8) return OPC_DIAG1 + (k.pat - 1);  // one slot condition
    return OPC_PHASE;
  }
  if (k.slot < 0 || k.slot >= k.nr || (k.flags & ~(uint32_t)F_TPRED)) return OPC_GENERIC;
  const bool swap = k.kind == K_MATR && k.m[0] == 0 && k.m[2] == 1 && k.m[4] == 1 && k.m[6] == 0;
  const bool ymat = k.kind == K_MAT && k.m[0] == 0 && k.m[1] == 0 && k.m[2] == 0 && k.m[3] == -1 && k.m[4] == 0 &&
                    k.m[5] == 1 && k.m[6] == 0 && k.m[7] == 0;
  if (k.kind == K_MATR && !swap && k.tmask == 0 && k.emask == slot_mask(k.nr, k.slot, 0)) return OPC_MATR + k.slot;
  if (k.kind == K_MAT && k.m[1] == 0 && k.m[5] == 0 && k.m[0] >= 0 && k.m[4] >= 0 && k.tmask == 0 &&
      k.emask == slot_mask(k.nr, k.slot, 0) && !(k.flags & ~(uint32_t)F_TPRED) && (k.m[0] > 0 || k.m[4] > 0)) {
    // [[c, -s w], [s, c w]] (see lean_param) only when the matrix has exactly that form
    const double c = k.m[0], sn = k.m[4];
    const double wx = c >= sn ? k.m[6] / c : -k.m[2] / sn, wy = c >= sn ? k.m[7] / c : -k.m[3] / sn;
    const double e = std::fabs(k.m[2] + sn * wx) + std::fabs(k.m[3] + sn * wy) + std::fabs(k.m[6] - c * wx) +
                     std::fabs(k.m[7] - c * wy) + std::fabs(wx * wx + wy * wy - 1.0);
    if (e < 1e-13) return OPC_MATRP + k.slot;
  }
  if (k.kind != K_MAT && !swap) return OPC_GENERIC;
  const bool tp = (k.flags & F_TPRED) != 0;
  const uint32_t full = slot_mask(k.nr, k.slot, 0);
  if ((swap || ymat) && (k.emask & ~full) == 0) return (swap ? OPC_SWAPM : OPC_YSWAPM) + k.slot;  // any register controls
  if (k.emask == full) return (tp ? OPC_MATT : OPC_MAT) + k.slot;
  for (int q = 0; q < k.nr; ++q)  // one register-side control
    for (int v = 0; v < 2; ++v)
      if (q != k.slot && k.emask == (full & slot_mask(k.nr, q, v))) return OPC_MATQ + 2 * (4 * k.slot + q) + v;
  return OPC_GENERIC;
}

template <typename R>
static void pack_kops(std::vector<HostKOp>& h, std::vector<unsigned char>& buf) {
  buf.assign(sizeof(KOp<R>) * h.size(), 0);
  KOp<R>* k = reinterpret_cast<KOp<R>*>(buf.data());
  for (size_t i = 0; i < h.size(); ++i) {
    if (h[i].kind == K_PHASE || h[i].kind == K_TPHASE) h[i].pat = pattern_of(h[i].nr, h[i].emask);
    KOp<R> x{};
    x.h.kind = (int16_t)h[i].kind;
    x.h.slot = (int8_t)h[i].slot;
    x.h.pat = (int8_t)h[i].pat;
    x.h.emask = (uint16_t)h[i].emask;
    x.h.lo = (uint8_t)h[i].lo;
    x.h.nbits = (uint8_t)h[i].nbits;
    x.h.flags = h[i].flags;
    x.h.opc = opcode_of(h[i]);
    x.tmask = h[i].tmask;
    x.tval = h[i].tval;
    x.qmask = h[i].qmask;
    x.turn = h[i].turn;
    x.fmask = h[i].fmask;
    for (int j = 0; j < 8; ++j) x.m[j] = (R)h[i].m[j];
    for (int j = 0; j < 4; ++j) {
      x.mr[2 * j] = (R)-h[i].m[2 * j + 1];
      x.mr[2 * j + 1] = (R)h[i].m[2 * j];
    }
    for (int j = 0; j < 16; ++j) x.tw[j] = (R)h[i].tw[j];
    k[i] = x;
  }
}

// the LEAN kernel's parameter block of one sweep: its DSweep with op indices
// rebased onto the sweep's own ops, copied out of the packed KOp array
template <typename R>
static void lean_param(const DSweep& d, const std::vector<unsigned char>& buf, std::vector<unsigned char>& out) {
  out.clear();
  if (!d.lean || d.nstages < 1) return;
  const int first = d.st[0].op_begin, last = d.st[d.nstages - 1].op_end;
  if (last - first > kLeanOps) return;  // too many ops for the parameter space: generic kernel
  static_assert(sizeof(LSweep<R>) + 3 * sizeof(void*) <= 32764, "LSweep exceeds the kernel parameter space");
  out.assign(sizeof(LSweep<R>), 0);
  LSweep<R>* ls = reinterpret_cast<LSweep<R>*>(out.data());
  ls->d = d;
  static const int noops = [] {  // SK_SWEEP_NOOPS=1: data movement only (cost split, A/B timing)
    const char* e = std::getenv("SK_SWEEP_NOOPS");
    return e ? std::atoi(e) : 0;
  }();
  for (int s = 0; s < d.nstages; ++s) {
    ls->d.st[s].op_begin -= first;
    ls->d.st[s].op_end = noops ? ls->d.st[s].op_begin : ls->d.st[s].op_end - first;
  }
  const KOp<R>* k = reinterpret_cast<const KOp<R>*>(buf.data());
  for (int o = first; o < last; ++o) {
    LOp<R>& x = ls->op[o - first];
    x.h = k[o].h;
    x.tmask = k[o].tmask;
    x.tval = k[o].tval;
    x.qmask = k[o].qmask;
    for (int j = 0; j < 8; ++j) {
      x.m[j] = k[o].m[j];
      x.mr[j] = k[o].mr[j];
    }
    if (x.h.opc >= OPC_MATRP && x.h.opc < OPC_MATRP + 4) {  // m = (c, s) at m[0], m[4]; mr = w, (-w.y, w.x)
      const double c = (double)k[o].m[0], sn = (double)k[o].m[4];
      double wx, wy;
      if (c >= sn) {
        wx = (double)k[o].m[6] / c;
        wy = (double)k[o].m[7] / c;
      } else {
        wx = -(double)k[o].m[2] / sn;
        wy = -(double)k[o].m[3] / sn;
      }
      x.mr[0] = (R)wx;
      x.mr[1] = (R)wy;
      x.mr[2] = (R)-wy;
      x.mr[3] = (R)wx;
    }
  }
}

static uint64_t deposit_h(uint64_t x, const Run* r, int n) {
  uint64_t o = 0;
  for (int i = 0; i < n; ++i) o |= ((x >> r[i].src) & ((1ull << r[i].w) - 1)) << r[i].dst;
  return o;
}

// QFT-window sweep of an (n-G)-qubit shard whose index is the top of an
// n-qubit QFT register with the low G qubits fixed to `value` (the rank's
// bits): every phase-space mask and bit position moves up by G, and the
// bottom window's deferred below-window phase (the CP fans from the G
// constant qubits) switches on.
static QSweep phase_shifted(const QSweep& q, int G, uint64_t value) {
  QSweep o = q;
  o.pshift = G;
  o.pconst = value;
  const uint64_t low = G >= 64 ? ~0ull : ((1ull << G) - 1);
  for (int s = 0; s < o.nstages; ++s) {
    QStage& st = o.st[s];
    if (!st.code) continue;
    st.tmask <<= G;
    st.tval <<= G;
    st.qmask = (st.qmask << G) | low;
    st.lo += G;
    if ((st.flags & F_SCALE) && G > 0) st.flags |= F_END;
  }
  return o;
}

// per-thread index table of a sweep: [stage][thread] = {global bits lo, hi,
// swizzled shared-memory byte offset, 0}
static void append_thr(const DSweep& d, size_t esz, std::vector<uint4>& thr) {
  const int nthreads = 1 << (d.ntile - d.nr);
  for (int s = 0; s < d.nstages; ++s) {
    const DStage& a = d.st[s];
    for (int t = 0; t < nthreads; ++t) {
      const uint64_t g = deposit_h((uint64_t)t, a.grun, a.ng);
      const uint32_t l = (uint32_t)deposit_h((uint64_t)t, a.lrun, a.nl);
      const uint32_t so = (esz == 8 ? swz<4>(l) : swz<3>(l)) * (uint32_t)esz;
      thr.push_back(make_uint4((uint32_t)g, (uint32_t)(g >> 32), so, l));
    }
  }
}

// QSweep for k_qft from a lowered QFT-only sweep (at most one K_QFTS op per
// stage); false = run it through the generic k_sweep
static bool qft_tma_enabled() {  // SK_QFT_TMA=0 keeps the shared-memory store stage (A/B timing)
  static const int v = [] {
    const char* e = std::getenv("SK_QFT_TMA");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

static bool qsweep_from(const DSweep& d, const std::vector<HostKOp>& kops, size_t esz, QSweep* q) {
  *q = QSweep{};
  if (!d.qft_only || d.nb > kQRuns || d.nstages > kQftMaxStages) return false;
  q->ntile = d.ntile;
  q->nstages = d.nstages;
  q->nb = d.nb;
  q->nthreads = 1 << (d.ntile - d.nr);
  // TMA store of the tile (c64, 4 register bits): the tile is the contiguous
  // low bits [0, T) (no tile bits above: brun starts at bit T), the last stage
  // is an op-less lane re-map and the stage before it holds index bits 0..3
  // in slots 0..3; the re-map stage is then replaced by the bulk store.
  const int row_bits = esz == 8 ? 4 : 3;  // log2 amplitudes per 128-byte row
  if (d.nr == 4 && d.ntile - row_bits <= 8 && d.nstages >= 2 && qft_tma_enabled()) {
    const DStage& last = d.st[d.nstages - 1];
    const DStage& prev = d.st[d.nstages - 2];
    bool ok = last.op_end == last.op_begin && (d.nb == 0 || d.brun[0].dst == d.ntile);
    for (int p = 0; p < 4; ++p) ok = ok && prev.reg_goff[p] == ((uint64_t)esz << p);
    if (ok) {
      q->tma = 1;
      q->nstages = d.nstages - 1;
    }
  }
  for (int i = 0; i < d.nb; ++i) q->brun[i] = d.brun[i];
  for (int s = 0; s < q->nstages; ++s) {
    const DStage& a = d.st[s];
    QStage& b = q->st[s];
    if (a.op_end - a.op_begin > 1) return false;
    for (int p = 0; p < kMaxR; ++p) {
      b.reg_goff[p] = a.reg_goff[p];
      b.reg_soff[p] = a.reg_soff[p];
    }
    b.code = 0;
    if (a.op_end > a.op_begin) {
      const HostKOp& k = kops[a.op_begin];
      if (k.kind != K_QFTS) return false;
      b.code = k.nbits * 8 + k.slot;
      b.flags = k.flags;
      b.lo = k.lo;
      b.tmask = k.tmask;
      b.tval = k.tval;
      b.qmask = k.qmask;
      b.scale = k.m[0];
    }
  }
  return true;
}

}  // namespace sk

struct sk_program {
  int width = 0;
  int dtype = SK_C128;
  int device = 0;
  int nr = 0;
  std::vector<sk::DSweep> sweeps;
  std::vector<sk::QSweep> qsweeps;  // per sweep: k_qft arguments (valid when qft_ok[i])
  std::vector<char> qft_ok;
  std::vector<size_t> thr_off;  // per sweep: offset of its per-thread table in d_thr (uint4 units)
  void* d_thr = nullptr;  // per-thread index tables
  int pshift = 0;         // sk_program_set_phase_index
  uint64_t pconst = 0;
  void* d_ops = nullptr;
  int nkops = 0;
  std::vector<std::vector<unsigned char>> lean;  // per sweep: LSweep<R> bytes (empty: not a LEAN sweep)
};

using namespace sk;

// SK_LEAN_KERNEL=0 keeps the interpreter in every generic sweep (A/B timing)
static bool use_lean_kernel() {
  static const int v = [] {
    const char* e = std::getenv("SK_LEAN_KERNEL");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

// SK_QFT_KERNEL=0 runs QFT windows through the generic k_sweep (A/B timing)
static bool use_qft_kernel() {
  static const int v = [] {
    const char* e = std::getenv("SK_QFT_KERNEL");
    return e ? std::atoi(e) : 1;
  }();
  return v != 0;
}

// 2-D tensor map over a state viewed as 128-byte rows (16 c64 or 8 c128
// amplitudes): box = one tile of 2^T amplitudes, 128-byte swizzle
static int tile_store_map(CUtensorMap* m, void* d, int width, int T, int row_bits) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)f;
  }();
  if (!enc) return set_error(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {16, (cuuint64_t)1 << (width - row_bits)};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {16, (cuuint32_t)1 << (T - row_bits)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, d, dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SK_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return SK_OK;
}

template <typename R, int NR>
static int launch_one(sk_state* s, const sk_program* p, int i, DevCtx* c, int64_t tb = 0, int64_t te = -1) {
  static bool attr_set[64] = {false};
  if (!attr_set[s->device]) {
#define SK_ATTR(K) SK_CUDA(cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024))
    if constexpr (NR <= 4 && !(sizeof(R) == 8 && NR == 4)) {
#ifndef SK_DEV_SWEEP_ONLY
      SK_ATTR((k_sweep<R, NR, 1, false>)); SK_ATTR((k_sweep<R, NR, 2, false>)); SK_ATTR((k_sweep<R, NR, 3, false>));
      SK_ATTR((k_sweep<R, NR, 4, false>)); SK_ATTR((k_sweep<R, NR, 5, false>)); SK_ATTR((k_sweep<R, NR, 6, false>));
      SK_ATTR((k_sweep<R, NR, 7, false>)); SK_ATTR((k_sweep<R, NR, 8, false>));
#endif
      SK_ATTR((k_sweep<R, NR, 1, true>)); SK_ATTR((k_sweep<R, NR, 2, true>)); SK_ATTR((k_sweep<R, NR, 3, true>));
      SK_ATTR((k_sweep<R, NR, 4, true>)); SK_ATTR((k_sweep<R, NR, 5, true>)); SK_ATTR((k_sweep<R, NR, 6, true>));
      SK_ATTR((k_sweep<R, NR, 7, true>)); SK_ATTR((k_sweep<R, NR, 8, true>));
      if constexpr (sizeof(R) == 4) {
#define SK_ATTR2(NS_) SK_CUDA(cudaFuncSetAttribute(k_sweep2<R, NR, NS_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024));
        SK_ATTR2(1) SK_ATTR2(2) SK_ATTR2(3) SK_ATTR2(4) SK_ATTR2(5) SK_ATTR2(6) SK_ATTR2(7) SK_ATTR2(8)
#undef SK_ATTR2
      }
    }
#ifndef SK_DEV_SWEEP_ONLY
    SK_ATTR((k_qft<R, NR, 1>)); SK_ATTR((k_qft<R, NR, 2>)); SK_ATTR((k_qft<R, NR, 3>));
    SK_ATTR((k_qft<R, NR, 4>)); SK_ATTR((k_qft<R, NR, 5>)); SK_ATTR((k_qft<R, NR, 6>));
#endif
#undef SK_ATTR
    attr_set[s->device] = true;
  }
  const DSweep& d = p->sweeps[i];
  const int T = d.ntile;
  const uint64_t all_tiles = 1ull << (s->width - T);
  if (te < 0) te = (int64_t)all_tiles;
  if (tb < 0 || te > (int64_t)all_tiles || tb >= te)
    return set_error(SK_EVALUE, "tile range [%lld, %lld) outside sweep %d's %llu tiles", (long long)tb, (long long)te, i,
                     (unsigned long long)all_tiles);
  const uint64_t tiles = (uint64_t)(te - tb);
  const unsigned threads = 1u << (T - NR);
  const size_t smem = ((size_t)1 << T) * sizeof(vec2_t<R>);
  if (all_tiles > 0x7fffffffull) return set_error(SK_EVALUE, "too many tiles (%d bits outside the tile)", s->width - T);
  vec2_t<R>* d_amps = (vec2_t<R>*)s->d;
  // 5-bit c64 and 4-bit c128 sweeps exist only as QFT windows: SK_QFT_KERNEL=0 cannot route them elsewhere
  constexpr bool qft_only = NR > 4 || (sizeof(R) == 8 && NR == 4);
#ifndef SK_DEV_SWEEP_ONLY
  if (p->qft_ok[i] && threads <= (unsigned)qft_max_threads<R, NR>() && (qft_only || use_qft_kernel())) {
    QSweep q = p->pshift ? phase_shifted(p->qsweeps[i], p->pshift, p->pconst) : p->qsweeps[i];
    q.tile0 = (int)tb;
    CUtensorMap tmap{};
    if (q.tma) SK_TRY(tile_store_map(&tmap, s->d, s->width, T, sizeof(vec2_t<R>) == 8 ? 4 : 3));
    switch (q.nstages) {
#define SK_QS(NS_) \
  case NS_: k_qft<R, NR, NS_><<<(unsigned)tiles, threads, smem, c->stream>>>(d_amps, q, tmap); break;
      SK_QS(1) SK_QS(2) SK_QS(3) SK_QS(4) SK_QS(5) SK_QS(6)
#undef SK_QS
      default: return set_error(SK_EVALUE, "sweep %d: %d stages", i, q.nstages);
    }
  } else
#endif
  if (tb != 0 || te != (int64_t)all_tiles) {
    return set_error(SK_EVALUE, "sweep %d: tile ranges need the QFT-window kernel", i);
  } else if constexpr (NR > 4 || (sizeof(R) == 8 && NR == 4)) {  // 4-bit c128 / 5-bit c64: QFT windows only
    return set_error(SK_EVALUE, "sweep %d: %d register bits need the QFT-window kernel", i, NR);
  } else if (p->pshift) {
    return set_error(SK_EVALUE, "sweep %d: a phase-index offset needs the QFT-window kernel", i);
  } else {
    const KOp<R>* ops = (const KOp<R>*)p->d_ops;
    const uint4* thr = (const uint4*)p->d_thr + p->thr_off[i];
    const bool lean = !p->lean[i].empty() && use_lean_kernel();
    // fp32 LEAN sweeps: two tiles per CTA (SK_SWEEP_H=1 runs one, A/B timing)
    static const int hpair = [] {
      const char* e = std::getenv("SK_SWEEP_H");
      return e ? std::atoi(e) : 2;
    }();
    const bool two = lean && sizeof(R) == 4 && hpair == 2 && tiles >= 2 && tiles % 2 == 0 && threads == 128;
    const LSweep<R>* ls = lean ? reinterpret_cast<const LSweep<R>*>(p->lean[i].data()) : nullptr;
    switch (d.nstages * 2 + (lean ? 1 : 0)) {
#ifdef SK_DEV_SWEEP_ONLY
#define SK_GENERIC_SWEEP(NS_) return set_error(SK_EVALUE, "development build: LEAN sweeps only");
#else
#define SK_GENERIC_SWEEP(NS_) \
  k_sweep<R, NR, NS_, false><<<(unsigned)tiles, threads, smem, c->stream>>>(d_amps, d, ops, thr); break;
#endif
#define SK_GS(NS_)                                                                                          \
  case 2 * NS_: SK_GENERIC_SWEEP(NS_)                                                                       \
  case 2 * NS_ + 1:                                                                                     \
    if (two) {                                                                                           \
      if constexpr (sizeof(R) == 4)                                                                      \
        k_sweep2<R, NR, NS_><<<(unsigned)(tiles / 2), threads, 2 * smem, c->stream>>>(d_amps, *ls, ops, thr); \
    } else if (SK_SWEEP1_MINB > 0 && threads == 128) {                                                   \
      k_sweep1<R, NR, NS_><<<(unsigned)tiles, threads, smem, c->stream>>>(d_amps, *ls, ops, thr);         \
    } else {                                                                                             \
      k_sweep<R, NR, NS_, true><<<(unsigned)tiles, threads, smem, c->stream>>>(d_amps, *ls, ops, thr);   \
    }                                                                                                    \
    break;
      SK_GS(1) SK_GS(2) SK_GS(3) SK_GS(4) SK_GS(5) SK_GS(6) SK_GS(7) SK_GS(8)
#undef SK_GS
#undef SK_GENERIC_SWEEP
      default: return set_error(SK_EVALUE, "sweep %d: %d stages", i, d.nstages);
    }
  }
  SK_CHECK_LAUNCH();
  return SK_OK;
}

static int launch_sweeps(sk_state* s, const sk_program* p, int first, int count, DevCtx* c, int64_t tb = 0,
                         int64_t te = -1) {
  for (int i = first; i < first + count; ++i) {
    const int nr = p->sweeps[i].nr;
#ifdef SK_DEV_SWEEP_ONLY  // fast development build: generic LEAN sweeps only (c64 4-bit, c128 3-bit)
    if (s->dtype == SK_C64 && nr == 4) {
      SK_TRY((launch_one<float, 4>(s, p, i, c, tb, te)));
    } else if (s->dtype == SK_C128 && nr == 3) {
      SK_TRY((launch_one<double, 3>(s, p, i, c, tb, te)));
    } else {
      return set_error(SK_EVALUE, "development build: generic sweeps only");
    }
    continue;
#endif
    if (s->dtype == SK_C64 && nr == 5) {
      SK_TRY((launch_one<float, 5>(s, p, i, c, tb, te)));
    } else if (s->dtype == SK_C64) {
      SK_TRY((launch_one<float, 4>(s, p, i, c, tb, te)));
    } else if (nr == 4) {
      SK_TRY((launch_one<double, 4>(s, p, i, c, tb, te)));
    } else {
      SK_TRY((launch_one<double, 3>(s, p, i, c, tb, te)));
    }
  }
  return SK_OK;
}

static int lower_program(int width, int dtype, const sk_sweep* sweeps, int nsweeps, const sk_op* ops, int nops,
                         std::vector<DSweep>& dsw, std::vector<HostKOp>& kops) {
  if (dtype != SK_C64 && dtype != SK_C128) return set_error(SK_EVALUE, "bad dtype %d", dtype);
  const int NR0 = dtype == SK_C64 ? kNR32 : kNR64;
  const uint32_t esz = dtype == SK_C64 ? 8 : 16;
  if (width < NR0 || width > 40) return set_error(SK_EVALUE, "fused program needs %d <= width <= 40", NR0);
  if (nsweeps < 0 || nops < 0) return set_error(SK_EVALUE, "negative counts");
  std::vector<int> op_seen(nops, 0);
  for (int si = 0; si < nsweeps; ++si) {
    const sk_sweep& sw = sweeps[si];
    if (sw.nstages < 1 || sw.nstages > kMaxS) return set_error(SK_EVALUE, "sweep %d: bad stage count %d", si, sw.nstages);
    DSweep d{};
    const int NR = sw.nreg ? sw.nreg : NR0;
    if (!(NR == 4 || (dtype == SK_C128 && NR == 3) || (dtype == SK_C64 && NR == 5)))
      return set_error(SK_EVALUE, "sweep %d: %d register bits not supported for this dtype", si, NR);
    if (NR == 5 || (dtype == SK_C128 && NR == 4))  // these register sets exist only in the QFT-window kernel
      for (int s = 0; s < sw.nstages; ++s)
        for (int o = sw.op_begin[s]; o < sw.op_begin[s + 1]; ++o)
          if (o >= 0 && o < nops && ops[o].kind != SK_OP_QFT)
            return set_error(SK_EVALUE, "sweep %d: %d register bits are only supported for QFT-window ops", si, NR);
    d.nr = NR;
    const int maxT = dtype == SK_C64 ? kMaxTile32 : kMaxTile64;
    const int T = sw.ntile;
    if (T < NR || T > maxT || T > width) return set_error(SK_EVALUE, "sweep %d: bad tile bit count %d", si, T);
    int local_of[64];
    for (int b = 0; b < 64; ++b) local_of[b] = -1;
    uint64_t tilemask = 0;
    for (int i = 0; i < T; ++i) {
      const int b = sw.tile_bits[i];
      if (b < 0 || b >= width || (i > 0 && b <= sw.tile_bits[i - 1]))
        return set_error(SK_EVALUE, "sweep %d: tile bits must be ascending and < width (bit %d)", si, b);
      local_of[b] = i;
      tilemask |= 1ull << b;
    }
    d.ntile = T;
    std::vector<int> nontile;
    for (int b = 0; b < width; ++b)
      if (!((tilemask >> b) & 1ull)) nontile.push_back(b);
    d.nb = make_runs(nontile, d.brun);
    if (d.nb < 0) return set_error(SK_EVALUE, "sweep %d: non-tile bits too fragmented", si);
    if (sw.nstages < 1 || sw.nstages > kMaxS) return set_error(SK_EVALUE, "sweep %d: bad stage count %d", si, sw.nstages);
    d.nstages = sw.nstages;
    double scale[2] = {1.0, 0.0};
    for (int s = 0; s < sw.nstages; ++s) {
      DStage& st = d.st[s];
      StageCtx c{};
      c.NR = NR;
      c.regmask = 0;
      for (int b = 0; b < 64; ++b) c.slot_of[b] = -1;
      for (int p = 0; p < NR; ++p) {
        const int q = sw.reg_bits[s][p];
        if (q < 0 || q >= width || local_of[q] < 0 || ((c.regmask >> q) & 1ull))
          return set_error(SK_EVALUE, "sweep %d: register bit %d not a distinct tile bit", si, q);
        c.regmask |= 1ull << q;
        c.slot_of[q] = p;
        c.reg_off[p] = 1ull << q;
        st.reg_goff[p] = (uint64_t)esz << q;
        st.reg_soff[p] = (esz == 8 ? swz<4>(1u << local_of[q]) : swz<3>(1u << local_of[q])) * esz;
      }
      std::vector<int> gdst, ldst;
      for (int i = 0; i < T; ++i) {
        const int b = sw.tile_bits[i];
        if ((c.regmask >> b) & 1ull) continue;
        gdst.push_back(b);
        ldst.push_back(i);
      }
      st.ng = make_runs(gdst, st.grun);
      st.nl = make_runs(ldst, st.lrun);
      if (st.ng < 0 || st.nl < 0) return set_error(SK_EVALUE, "sweep %d: thread bits too fragmented", si);
      const int ob = sw.op_begin[s], oe = sw.op_begin[s + 1];
      if (ob < 0 || oe < ob || oe > nops) return set_error(SK_EVALUE, "sweep %d: bad op range in stage %d", si, s);
      st.op_begin = (int)kops.size();
      for (int o = ob; o < oe; ++o) {
        if (op_seen[o]) return set_error(SK_EVALUE, "op %d used by two stages (sweep %d)", o, si);
        op_seen[o] = 1;
        const size_t first = kops.size();
      SK_TRY(lower_op(c, ops[o], o, width, kops, scale));
      for (size_t k = first; k < kops.size(); ++k) kops[k].nr = NR;
      }
      if (s == sw.nstages - 1 && !(scale[0] == 1.0 && scale[1] == 0.0)) {  // deferred butterfly scalars
        HostKOp k;
        k.kind = K_PHASE;
        k.nr = NR;
        k.emask = (uint32_t)((1ull << (1 << NR)) - 1);
        k.m[0] = k.m[2] = scale[0];
        k.m[1] = k.m[3] = scale[1];
        kops.push_back(k);
      }
      st.op_end = (int)kops.size();
    }
    d.qft_only = 1;
    for (int s2 = 0; s2 < d.nstages; ++s2)
      for (int o2 = d.st[s2].op_begin; o2 < d.st[s2].op_end; ++o2)
        if (kops[o2].kind != K_QFTS) d.qft_only = 0;
    dsw.push_back(d);
  }
  return SK_OK;
}

extern "C" {

int sk_program_reg_bits(int dtype, int* nreg) {
  if (dtype != SK_C64 && dtype != SK_C128) return set_error(SK_EVALUE, "bad dtype %d", dtype);
  *nreg = dtype == SK_C64 ? kNR32 : kNR64;
  return SK_OK;
}

int sk_program_create(int width, int dtype, int device, const sk_sweep* sweeps, int nsweeps, const sk_op* ops,
                      int nops, sk_program** out) {
  std::vector<HostKOp> kops;
  std::vector<DSweep> dsw;
  SK_TRY(lower_program(width, dtype, sweeps, nsweeps, ops, nops, dsw, kops));
  const int NR = dtype == SK_C64 ? kNR32 : kNR64;
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  std::vector<unsigned char> buf;
  if (dtype == SK_C64)
    pack_kops<float>(kops, buf);
  else
    pack_kops<double>(kops, buf);
  for (auto& d : dsw) {  // pack_kops resolved the phase patterns the opcodes depend on
    d.lean = d.nr <= 4;
    for (int st = 0; st < d.nstages; ++st)
      for (int o = d.st[st].op_begin; o < d.st[st].op_end; ++o)
        if (opcode_of(kops[o]) == OPC_GENERIC) d.lean = 0;
  }
  sk_program* prog = new sk_program();
  prog->width = width;
  prog->dtype = dtype;
  prog->device = device;
  prog->nr = NR;
  prog->qsweeps.resize(dsw.size());
  prog->qft_ok.resize(dsw.size());
  std::vector<uint4> thr;
  prog->thr_off.assign(dsw.size(), 0);
  for (size_t i = 0; i < dsw.size(); ++i) {
    prog->thr_off[i] = thr.size();
    append_thr(dsw[i], dtype == SK_C64 ? 8 : 16, thr);
    prog->qft_ok[i] = qsweep_from(dsw[i], kops, dtype == SK_C64 ? 8 : 16, &prog->qsweeps[i]);
  }
  if (!thr.empty()) {
    cudaError_t e = cudaMalloc(&prog->d_thr, thr.size() * sizeof(uint4));
    if (e == cudaSuccess) e = cudaMemcpy(prog->d_thr, thr.data(), thr.size() * sizeof(uint4), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (prog->d_thr) cudaFree(prog->d_thr);
      delete prog;
      return set_error(SK_ECUDA, "program upload: %s", cudaGetErrorString(e));
    }
    for (size_t i = 0; i < dsw.size(); ++i) prog->qsweeps[i].thr = (const uint4*)prog->d_thr + prog->thr_off[i];
  }
  prog->lean.resize(dsw.size());
  for (size_t i = 0; i < dsw.size(); ++i) {
    if (dtype == SK_C64)
      lean_param<float>(dsw[i], buf, prog->lean[i]);
    else
      lean_param<double>(dsw[i], buf, prog->lean[i]);
  }
  prog->sweeps = std::move(dsw);
  prog->nkops = (int)kops.size();
  if (!buf.empty()) {
    cudaError_t e = cudaMalloc(&prog->d_ops, buf.size());
    if (e == cudaSuccess) e = cudaMemcpy(prog->d_ops, buf.data(), buf.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (prog->d_ops) cudaFree(prog->d_ops);
      if (prog->d_thr) cudaFree(prog->d_thr);
      delete prog;
      return set_error(SK_ECUDA, "program upload: %s", cudaGetErrorString(e));
    }
  }
  *out = prog;
  return SK_OK;
}

int sk_program_lower(int width, int dtype, const sk_sweep* sweeps, int nsweeps, const sk_op* ops, int nops,
                     int64_t* ints, double* reals, int cap, int* count, int* stage_ops) {
  std::vector<HostKOp> kops;
  std::vector<DSweep> dsw;
  SK_TRY(lower_program(width, dtype, sweeps, nsweeps, ops, nops, dsw, kops));
  for (auto& k : kops)
    if (k.kind == K_PHASE || k.kind == K_TPHASE) k.pat = pattern_of(k.nr, k.emask);
  *count = (int)kops.size();
  if ((int)kops.size() > cap) return set_error(SK_EVALUE, "need room for %d kernel ops", (int)kops.size());
  for (size_t i = 0; i < kops.size(); ++i) {
    const HostKOp& k = kops[i];
    int64_t* x = ints + 12 * i;
    x[0] = k.kind; x[1] = k.slot; x[2] = k.pat; x[3] = k.emask; x[4] = k.flags; x[5] = k.lo; x[6] = k.nbits;
    x[7] = (int64_t)k.tmask; x[8] = (int64_t)k.tval; x[9] = (int64_t)k.qmask; x[10] = (int64_t)k.turn;
    x[11] = (int64_t)k.fmask;
    for (int j = 0; j < 8; ++j) reals[24 * i + j] = k.m[j];
    for (int j = 0; j < 16; ++j) reals[24 * i + 8 + j] = k.tw[j];
  }
  for (int si = 0; si < nsweeps; ++si)
    for (int st = 0; st <= SK_MAX_STAGES; ++st)
      stage_ops[si * (SK_MAX_STAGES + 1) + st] =
          st < dsw[si].nstages ? dsw[si].st[st].op_begin : (st == dsw[si].nstages ? dsw[si].st[st - 1].op_end : -1);
  return SK_OK;
}

int sk_program_destroy(sk_program* p) {
  if (!p) return SK_OK;
  if (p->d_ops || p->d_thr) {
    DevCtx* c;
    SK_TRY(ctx_get(p->device, &c));
    SK_CUDA(cudaStreamSynchronize(c->stream));
    if (p->d_ops) SK_CUDA(cudaFree(p->d_ops));
    if (p->d_thr) SK_CUDA(cudaFree(p->d_thr));
  }
  delete p;
  return SK_OK;
}

int sk_program_set_phase_index(sk_program* p, int shift, uint64_t value) {
  if (!p) return set_error(SK_EVALUE, "null program");
  if (shift < 0 || shift > 24 || (shift < 64 && (value >> shift)))
    return set_error(SK_EVALUE, "bad phase index offset (shift %d, value %llu)", shift, (unsigned long long)value);
  for (size_t i = 0; i < p->sweeps.size(); ++i)
    if (shift && !p->qft_ok[i]) return set_error(SK_EVALUE, "sweep %zu is not a QFT-window sweep", i);
  p->pshift = shift;
  p->pconst = value;
  return SK_OK;
}

int sk_program_nsweeps(const sk_program* p, int* n) {
  if (!p) return set_error(SK_EVALUE, "null program");
  *n = (int)p->sweeps.size();
  return SK_OK;
}

int sk_program_run(sk_state* s, const sk_program* p, int first, int count) {
  if (!s || !p) return set_error(SK_EVALUE, "null state or program");
  if (s->width != p->width || s->dtype != p->dtype || s->device != p->device)
    return set_error(SK_EVALUE, "program planned for width %d dtype %d, state has width %d dtype %d", p->width,
                     p->dtype, s->width, s->dtype);
  const int ns = (int)p->sweeps.size();
  if (count < 0) count = ns - first;
  if (first < 0 || first + count > ns) return set_error(SK_EVALUE, "sweep range [%d, %d) outside program", first, first + count);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  return launch_sweeps(s, p, first, count, c);
}

int sk_program_run_tiles(sk_state* s, const sk_program* p, int sweep, int64_t tile_begin, int64_t tile_end) {
  if (!s || !p) return set_error(SK_EVALUE, "null state or program");
  if (s->width != p->width || s->dtype != p->dtype || s->device != p->device)
    return set_error(SK_EVALUE, "program planned for width %d dtype %d, state has width %d dtype %d", p->width,
                     p->dtype, s->width, s->dtype);
  if (sweep < 0 || sweep >= (int)p->sweeps.size()) return set_error(SK_EVALUE, "sweep %d outside program", sweep);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  return launch_sweeps(s, p, sweep, 1, c, tile_begin, tile_end);
}

int sk_program_sweep_tiles(const sk_program* p, int sweep, int* tile_bits, int64_t* tiles) {
  if (!p) return set_error(SK_EVALUE, "null program");
  if (sweep < 0 || sweep >= (int)p->sweeps.size()) return set_error(SK_EVALUE, "sweep %d outside program", sweep);
  const DSweep& d = p->sweeps[sweep];
  *tile_bits = d.ntile;
  *tiles = int64_t(1) << (p->width - d.ntile);
  // contiguous tiles (the tile is index bits [0, T)): tile t covers [t 2^T, (t+1) 2^T)
  if (!(d.nb == 0 || (d.nb == 1 && d.brun[0].dst == d.ntile))) *tile_bits = -*tile_bits;
  return SK_OK;
}

}  // extern "C"
