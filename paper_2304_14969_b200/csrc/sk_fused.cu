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
// and applies that stage's ops on them:
//   MAT  — 2x2 on a register bit, predicated on arbitrary control bits
//          (controls outside the tile are a per-tile predicate),
//   DIAG — diag(d0, d1) on ANY qubit (diagonal gates need no pairing),
//   RAMP — per-element phase exp(i*pi*s*F(idx)), F a bit field of the
//          index: the fan-in of a run of controlled phases onto one target
//          (the QFT's CP(pi/2^k) chain collapses to one RAMP per target).
// Between stages the tile is exchanged through (XOR-swizzled) shared memory.
// Stage 0 loads from HBM, the last stage stores back: one read and one
// write of every amplitude per sweep.
#include <vector>

#include "sk_internal.cuh"

namespace sk {

constexpr int kMaxT = SK_MAX_TILE_BITS;
constexpr int kMaxS = SK_MAX_STAGES;
constexpr int kMaxR = SK_MAX_REG_BITS;

struct DStage {
  int op_begin, op_end;
  uint64_t thr_off[kMaxT];  // global index offset contributed by thread-index bit i
  uint32_t thr_loc[kMaxT];  // tile-local offset of thread-index bit i
  uint64_t reg_off[kMaxR];  // global offset of register slot p
  uint32_t reg_loc[kMaxR];  // tile-local offset of register slot p
};

struct DSweep {
  int ntile;
  int nstages;
  int tile_bits[kMaxT];
  DStage st[kMaxS];
};

struct DOp {
  int kind;
  int slot;              // MAT: target slot; DIAG: qubit slot or -1
  uint32_t rmask, rval;  // control predicate on register slots
  uint64_t tmask, tval;  // control predicate on the thread-constant index part
  uint64_t qmask;        // DIAG: qubit mask when not a register bit
  int lo, nbits;         // RAMP field
  double s;              // RAMP scale
  double m[8];
  double w[2 * kMaxR];   // RAMP: exp(i*pi*s*F(reg_off[p]))
};

// swizzle of the tile-local index: fold the high bits into the low SB bits so
// every stage's warp access pattern is bank-conflict free for contiguous
// register-bit runs (SB = 4 for 8-byte, 3 for 16-byte elements)
template <int SB>
__device__ __forceinline__ uint32_t swz(uint32_t l) {
  uint32_t h = l >> SB;
  uint32_t f = h ^ (h >> SB) ^ (h >> (2 * SB)) ^ (h >> (3 * SB));
  return l ^ (f & ((1u << SB) - 1));
}

template <typename R>
__device__ __forceinline__ void sincospi_r(double x, R* s, R* c);
template <>
__device__ __forceinline__ void sincospi_r<float>(double x, float* s, float* c) {
  sincospif((float)x, s, c);
}
template <>
__device__ __forceinline__ void sincospi_r<double>(double x, double* s, double* c) {
  sincospi(x, s, c);
}

template <typename R, int NR, int P>
__device__ __forceinline__ void mat_slot(vec2_t<R> (&a)[1 << NR], const Mat2<R>& m, uint32_t rmask, uint32_t rval) {
#pragma unroll
  for (int e = 0; e < (1 << NR); ++e) {
    if ((e >> P) & 1) continue;
    if ((e & rmask) != rval) continue;
    const int e1 = e | (1 << P);
    vec2_t<R> y0 = cmad2<R>(m.m00, a[e], m.m01, a[e1]);
    vec2_t<R> y1 = cmad2<R>(m.m10, a[e], m.m11, a[e1]);
    a[e] = y0;
    a[e1] = y1;
  }
}

template <typename R, int NR>
__device__ __forceinline__ void apply_op(const DOp* __restrict__ op, vec2_t<R> (&a)[1 << NR], uint64_t gthr) {
  const int kind = op->kind;
  const uint64_t tmask = op->tmask, tval = op->tval;
  if ((gthr & tmask) != tval) return;  // control outside the registers not satisfied
  const uint32_t rmask = op->rmask, rval = op->rval;
  if (kind == SK_OP_MAT) {
    Mat2<R> m;
    m.m00 = mk<R>((R)op->m[0], (R)op->m[1]);
    m.m01 = mk<R>((R)op->m[2], (R)op->m[3]);
    m.m10 = mk<R>((R)op->m[4], (R)op->m[5]);
    m.m11 = mk<R>((R)op->m[6], (R)op->m[7]);
    switch (op->slot) {
      case 0: mat_slot<R, NR, 0>(a, m, rmask, rval); break;
      case 1: if (NR > 1) mat_slot<R, NR, (NR > 1 ? 1 : 0)>(a, m, rmask, rval); break;
      case 2: if (NR > 2) mat_slot<R, NR, (NR > 2 ? 2 : 0)>(a, m, rmask, rval); break;
      case 3: if (NR > 3) mat_slot<R, NR, (NR > 3 ? 3 : 0)>(a, m, rmask, rval); break;
      default: break;
    }
  } else if (kind == SK_OP_DIAG) {
    const vec2_t<R> d0 = mk<R>((R)op->m[0], (R)op->m[1]);
    const vec2_t<R> d1 = mk<R>((R)op->m[6], (R)op->m[7]);
    const int slot = op->slot;
    const bool tbit = (gthr & op->qmask) != 0;
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e) {
      if ((e & rmask) != rval) continue;
      const bool b = slot >= 0 ? ((e >> slot) & 1) : tbit;
      a[e] = cmul<R>(a[e], b ? d1 : d0);
    }
  } else {  // SK_OP_RAMP
    const uint64_t fmask = op->nbits >= 64 ? ~0ull : ((1ull << op->nbits) - 1);
    const uint64_t f = (gthr >> op->lo) & fmask;
    double x = op->s * (double)f;
    x -= 2.0 * floor(0.5 * x);
    R sn, cs;
    sincospi_r<R>(x, &sn, &cs);
    const vec2_t<R> base = mk<R>(cs, sn);
    vec2_t<R> w[NR];
#pragma unroll
    for (int p = 0; p < NR; ++p) w[p] = mk<R>((R)op->w[2 * p], (R)op->w[2 * p + 1]);
#pragma unroll
    for (int e = 0; e < (1 << NR); ++e) {
      if ((e & rmask) != rval) continue;
      vec2_t<R> ph = base;
#pragma unroll
      for (int p = 0; p < NR; ++p)
        if ((e >> p) & 1) ph = cmul<R>(ph, w[p]);
      a[e] = cmul<R>(a[e], ph);
    }
  }
}

template <typename R, int NR>
__global__ void __launch_bounds__(512, 2) k_sweep(vec2_t<R>* __restrict__ amps, const __grid_constant__ DSweep sw,
                                                  const DOp* __restrict__ ops) {
  extern __shared__ __align__(16) unsigned char smraw[];
  vec2_t<R>* sm = reinterpret_cast<vec2_t<R>*>(smraw);
  constexpr int NE = 1 << NR;
  constexpr int SB = sizeof(vec2_t<R>) == 8 ? 4 : 3;
  const int T = sw.ntile;
  const int TB = T - NR;
  const uint32_t tid = threadIdx.x;

  // tile base: deposit blockIdx into the non-tile bits
  uint64_t base = blockIdx.x;
  for (int i = 0; i < T; ++i) base = insert0(base, sw.tile_bits[i]);

  vec2_t<R> a[NE];
  const int ns = sw.nstages;
  for (int s = 0; s < ns; ++s) {
    const DStage& st = sw.st[s];
    uint64_t gthr = base;
    uint32_t lthr = 0;
    for (int i = 0; i < TB; ++i) {
      if ((tid >> i) & 1u) {
        gthr += st.thr_off[i];
        lthr += st.thr_loc[i];
      }
    }
    if (s == 0) {
      const vec2_t<R>* src = amps + gthr;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        uint64_t o = 0;
#pragma unroll
        for (int p = 0; p < NR; ++p)
          if ((e >> p) & 1) o += st.reg_off[p];
        a[e] = src[o];
      }
    } else {
      __syncthreads();
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        uint32_t l = lthr;
#pragma unroll
        for (int p = 0; p < NR; ++p)
          if ((e >> p) & 1) l += st.reg_loc[p];
        a[e] = sm[swz<SB>(l)];
      }
    }
    for (int o = st.op_begin; o < st.op_end; ++o) apply_op<R, NR>(ops + o, a, gthr);
    if (s == ns - 1) {
      vec2_t<R>* dst = amps + gthr;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        uint64_t o = 0;
#pragma unroll
        for (int p = 0; p < NR; ++p)
          if ((e >> p) & 1) o += st.reg_off[p];
        dst[o] = a[e];
      }
    } else {
      if (s > 0) __syncthreads();
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        uint32_t l = lthr;
#pragma unroll
        for (int p = 0; p < NR; ++p)
          if ((e >> p) & 1) l += st.reg_loc[p];
        sm[swz<SB>(l)] = a[e];
      }
    }
  }
}

// register bits per stage: 16 fp32 amplitudes (32 regs) or 8 fp64 (32 regs)
constexpr int kNR32 = 4;
constexpr int kNR64 = 3;
constexpr int kMaxTile32 = 13;  // 64 KiB of shared memory per tile, 512 threads
constexpr int kMaxTile64 = 12;

}  // namespace sk

struct sk_program {
  int width = 0;
  int dtype = SK_C128;
  int device = 0;
  int nr = 0;
  std::vector<sk::DSweep> sweeps;
  sk::DOp* d_ops = nullptr;
  int nops = 0;
};

using namespace sk;

template <typename R, int NR>
static int launch_sweeps(sk_state* s, const sk_program* p, int first, int count, DevCtx* c) {
  static bool attr_set[64] = {false};
  if (!attr_set[s->device]) {
    SK_CUDA(cudaFuncSetAttribute(k_sweep<R, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    attr_set[s->device] = true;
  }
  for (int i = first; i < first + count; ++i) {
    const DSweep& d = p->sweeps[i];
    const int T = d.ntile;
    const uint64_t tiles = 1ull << (s->width - T);
    const unsigned threads = 1u << (T - NR);
    const size_t smem = ((size_t)1 << T) * sizeof(vec2_t<R>);
    if (tiles > 0x7fffffffull) return set_error(SK_EVALUE, "too many tiles (%d bits outside the tile)", s->width - T);
    k_sweep<R, NR><<<(unsigned)tiles, threads, smem, c->stream>>>((vec2_t<R>*)s->d, d, p->d_ops);
    SK_CHECK_LAUNCH();
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
  if (dtype != SK_C64 && dtype != SK_C128) return set_error(SK_EVALUE, "bad dtype %d", dtype);
  const int NR = dtype == SK_C64 ? kNR32 : kNR64;
  const int maxT = dtype == SK_C64 ? kMaxTile32 : kMaxTile64;
  if (width < NR || width > 40) return set_error(SK_EVALUE, "fused program needs %d <= width <= 40", NR);
  if (nsweeps < 0 || nops < 0) return set_error(SK_EVALUE, "negative counts");
  std::vector<DOp> dops(nops);
  std::vector<int> op_seen(nops, 0);
  sk_program* prog = new sk_program();
  prog->width = width;
  prog->dtype = dtype;
  prog->device = device;
  prog->nr = NR;
  auto fail = [&](int code, const char* msg, int a, int b) {
    delete prog;
    return set_error(code, msg, a, b);
  };
  for (int si = 0; si < nsweeps; ++si) {
    const sk_sweep& sw = sweeps[si];
    DSweep d{};
    const int T = sw.ntile;
    if (T < NR || T > maxT || T > width) return fail(SK_EVALUE, "sweep %d: bad tile bit count %d", si, T);
    int local_of[64];
    for (int b = 0; b < 64; ++b) local_of[b] = -1;
    for (int i = 0; i < T; ++i) {
      const int b = sw.tile_bits[i];
      if (b < 0 || b >= width || (i > 0 && b <= sw.tile_bits[i - 1]))
        return fail(SK_EVALUE, "sweep %d: tile bits must be ascending and < width (bit %d)", si, b);
      local_of[b] = i;
      d.tile_bits[i] = b;
    }
    d.ntile = T;
    if (sw.nstages < 1 || sw.nstages > kMaxS) return fail(SK_EVALUE, "sweep %d: bad stage count %d", si, sw.nstages);
    d.nstages = sw.nstages;
    for (int s = 0; s < sw.nstages; ++s) {
      DStage& st = d.st[s];
      uint64_t regmask = 0;
      int slot_of[64];
      for (int b = 0; b < 64; ++b) slot_of[b] = -1;
      for (int p = 0; p < NR; ++p) {
        const int q = sw.reg_bits[s][p];
        if (q < 0 || q >= width || local_of[q] < 0 || ((regmask >> q) & 1ull))
          return fail(SK_EVALUE, "sweep %d: register bit %d not a distinct tile bit", si, q);
        regmask |= 1ull << q;
        slot_of[q] = p;
        st.reg_off[p] = 1ull << q;
        st.reg_loc[p] = 1u << local_of[q];
      }
      int ti = 0;
      for (int i = 0; i < T; ++i) {
        const int b = sw.tile_bits[i];
        if ((regmask >> b) & 1ull) continue;
        st.thr_off[ti] = 1ull << b;
        st.thr_loc[ti] = 1u << i;
        ++ti;
      }
      const int ob = sw.op_begin[s], oe = sw.op_begin[s + 1];
      if (ob < 0 || oe < ob || oe > nops) return fail(SK_EVALUE, "sweep %d: bad op range in stage %d", si, s);
      st.op_begin = ob;
      st.op_end = oe;
      for (int o = ob; o < oe; ++o) {
        if (op_seen[o]) return fail(SK_EVALUE, "op %d used by two stages (sweep %d)", o, si);
        op_seen[o] = 1;
        const sk_op& op = ops[o];
        DOp& x = dops[o];
        x.kind = op.kind;
        if (op.ctrl_val & ~op.ctrl_mask) return fail(SK_EVALUE, "op %d: ctrl_val outside ctrl_mask (sweep %d)", o, si);
        if (width < 64 && (op.ctrl_mask >> width)) return fail(SK_EVALUE, "op %d: control beyond width %d", o, width);
        x.tmask = op.ctrl_mask & ~regmask;
        x.tval = op.ctrl_val & ~regmask;
        x.rmask = 0;
        x.rval = 0;
        for (int p = 0; p < NR; ++p) {
          const int q = sw.reg_bits[s][p];
          if ((op.ctrl_mask >> q) & 1ull) {
            x.rmask |= 1u << p;
            if ((op.ctrl_val >> q) & 1ull) x.rval |= 1u << p;
          }
        }
        for (int k = 0; k < 8; ++k) x.m[k] = op.m[k];
        if (op.kind == SK_OP_MAT) {
          if (op.qubit < 0 || op.qubit >= width || slot_of[op.qubit] < 0)
            return fail(SK_EVALUE, "op %d: MAT target %d is not a register bit of its stage", o, op.qubit);
          if ((op.ctrl_mask >> op.qubit) & 1ull) return fail(SK_EVALUE, "op %d: target %d is a control", o, op.qubit);
          x.slot = slot_of[op.qubit];
        } else if (op.kind == SK_OP_DIAG) {
          if (op.qubit < 0 || op.qubit >= width) return fail(SK_EVALUE, "op %d: DIAG qubit %d out of range", o, op.qubit);
          if ((op.ctrl_mask >> op.qubit) & 1ull) return fail(SK_EVALUE, "op %d: qubit %d is a control", o, op.qubit);
          x.slot = slot_of[op.qubit];
          x.qmask = x.slot >= 0 ? 0 : (1ull << op.qubit);
        } else if (op.kind == SK_OP_RAMP) {
          if (op.qubit < 0 || op.nbits < 1 || op.qubit + op.nbits > width)
            return fail(SK_EVALUE, "op %d: bad RAMP field at bit %d", o, op.qubit);
          x.slot = -1;
          x.lo = op.qubit;
          x.nbits = op.nbits;
          x.s = op.m[0];
          const uint64_t fmask = (1ull << op.nbits) - 1;
          for (int p = 0; p < NR; ++p) {
            const uint64_t f = (st.reg_off[p] >> op.qubit) & fmask;
            double xx = op.m[0] * (double)f;
            xx -= 2.0 * std::floor(0.5 * xx);
            x.w[2 * p] = std::cos(M_PI * xx);
            x.w[2 * p + 1] = std::sin(M_PI * xx);
          }
        } else {
          return fail(SK_EVALUE, "op %d: unknown kind %d", o, op.kind);
        }
      }
    }
    prog->sweeps.push_back(d);
  }
  DevCtx* c;
  int rc = ctx_get(device, &c);
  if (rc != SK_OK) {
    delete prog;
    return rc;
  }
  prog->nops = nops;
  if (nops > 0) {
    cudaError_t e = cudaMalloc(&prog->d_ops, sizeof(DOp) * nops);
    if (e == cudaSuccess) e = cudaMemcpy(prog->d_ops, dops.data(), sizeof(DOp) * nops, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (prog->d_ops) cudaFree(prog->d_ops);
      delete prog;
      return set_error(SK_ECUDA, "program upload: %s", cudaGetErrorString(e));
    }
  }
  *out = prog;
  return SK_OK;
}

int sk_program_destroy(sk_program* p) {
  if (!p) return SK_OK;
  if (p->d_ops) {
    DevCtx* c;
    SK_TRY(ctx_get(p->device, &c));
    SK_CUDA(cudaStreamSynchronize(c->stream));
    SK_CUDA(cudaFree(p->d_ops));
  }
  delete p;
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
  if (s->dtype == SK_C64) return launch_sweeps<float, kNR32>(s, p, first, count, c);
  return launch_sweeps<double, kNR64>(s, p, first, count, c);
}

}  // extern "C"
