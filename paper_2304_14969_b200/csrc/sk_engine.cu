// sk_engine.cu — native hybrid-engine runtime: the factorised simulator
// that feeds the device ket.
//
// The reference's HybridState (pkg/src/shardsim/engine.py) keeps the global
// state as a tensor product of shards and decides, after every committed
// coupler, whether to split off or Schmidt-round each operand qubit.  Its
// Python control flow costs ~0.1 ms per gate and its per-coupler decisions
// each need the operands' Bloch sums.  Here the whole commit stream runs in
// C++ next to the kernels:
//   * gates arrive as one packed array per circuit (no per-gate FFI crossing);
//   * 1q buffers, the pending controlled-op queues and every rewrite are
//     host-side 2x2 algebra (std::complex<double>), in the reference's order;
//   * the decision inputs (Bloch sums of the committed coupler's operands,
//     fused with the gate itself in one pass) come back through mapped pinned
//     memory — the device writes them, the host reads a sequence word — with no
//     cudaMemcpy / stream synchronisation per coupler;
//   * width-1 shards carry their Bloch sums in a host cache filled by the
//     kernels that last wrote them (control elimination, engine.py:407-436,
//     reads them without a device round trip);
//   * SDRP rounding is one fused rotate-project-compact pass whose P0 is
//     analytic in the sums already in hand (engine.py:464-488).
// Decisions are bit-for-bit those of the reference engine's rules
// (engine.py:276-512, 525-535, 575-594, 669-711), which tests/test_engine_gpu.py
// and tests/test_scale_gpu.py pin against the reference's own records.
//
// Stabilizer (tableau) shards are not modelled: qubits start as width-1
// dense shards, as in the reference with OptFlags(stabilizer_hybrid=False).
#include <algorithm>
#include <cmath>
#include <complex>
#include <deque>
#include <memory>
#include <unordered_set>
#include <vector>

#include "sk_internal.cuh"
#include "sk_ops.cuh"
#include "sk_tableau.h"

namespace {

using cd = std::complex<double>;

struct M2 {
  cd a[4];  // row-major m00 m01 m10 m11
};

M2 m_from8(const double* p) {
  M2 m;
  for (int i = 0; i < 4; ++i) m.a[i] = cd(p[2 * i], p[2 * i + 1]);
  return m;
}

void m_to8(const M2& m, double* p) {
  for (int i = 0; i < 4; ++i) {
    p[2 * i] = m.a[i].real();
    p[2 * i + 1] = m.a[i].imag();
  }
}

M2 mmul(const M2& x, const M2& y) {  // x @ y
  M2 r;
  r.a[0] = x.a[0] * y.a[0] + x.a[1] * y.a[2];
  r.a[1] = x.a[0] * y.a[1] + x.a[1] * y.a[3];
  r.a[2] = x.a[2] * y.a[0] + x.a[3] * y.a[2];
  r.a[3] = x.a[2] * y.a[1] + x.a[3] * y.a[3];
  return r;
}

M2 mdag(const M2& x) {
  M2 r;
  r.a[0] = std::conj(x.a[0]);
  r.a[1] = std::conj(x.a[2]);
  r.a[2] = std::conj(x.a[1]);
  r.a[3] = std::conj(x.a[3]);
  return r;
}

const M2 kI = {{cd(1, 0), cd(0, 0), cd(0, 0), cd(1, 0)}};
const M2 kPauli[3] = {{{cd(0, 0), cd(1, 0), cd(1, 0), cd(0, 0)}},     // X
                      {{cd(0, 0), cd(0, -1), cd(0, 1), cd(0, 0)}},    // Y
                      {{cd(1, 0), cd(0, 0), cd(0, 0), cd(-1, 0)}}};   // Z

constexpr double kStructTol = 1e-14;  // engine.py _is_diag / _is_antidiag

bool is_diag(const M2& m) { return std::abs(m.a[1]) < kStructTol && std::abs(m.a[2]) < kStructTol; }
bool is_antidiag(const M2& m) { return std::abs(m.a[0]) < kStructTol && std::abs(m.a[3]) < kStructTol; }

double max_abs_diff(const M2& x, const M2& y) {
  double d = 0;
  for (int i = 0; i < 4; ++i) d = std::max(d, std::abs(x.a[i] - y.a[i]));
  return d;
}

bool is_identity(const M2& m) { return max_abs_diff(m, kI) < 1e-12; }  // engine.py:313-314

// zero the structurally dead entries of a (near) diagonal / antidiagonal
// matrix; false otherwise (engine.py:132-143)
bool snap(const M2& m, M2* out) {
  if (is_diag(m)) {
    *out = m;
    out->a[1] = out->a[2] = 0.0;
    return true;
  }
  if (is_antidiag(m)) {
    *out = m;
    out->a[0] = out->a[3] = 0.0;
    return true;
  }
  return false;
}

// ket.py:57-59 unitarity check of every committed matrix
bool unitary(const M2& m) { return max_abs_diff(mmul(mdag(m), m), kI) <= 1e-10; }

// Bloch-sphere rotation of a 2x2 unitary (engine.py:146-152)
void so3(const M2& u, double r[3][3]) {
  const M2 ud = mdag(u);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      M2 t = mmul(mmul(mmul(kPauli[i], u), kPauli[j]), ud);
      r[i][j] = 0.5 * (t.a[0] + t.a[3]).real();
    }
}

// m = phase * Pauli within 1e-12 (engine.py:155-161); returns 0/1/2 or -1
int as_pauli(const M2& m, cd* phase) {
  for (int p = 0; p < 3; ++p) {
    M2 t = mmul(kPauli[p], m);
    cd tr = (t.a[0] + t.a[3]) / 2.0;
    if (std::abs(std::abs(tr) - 1.0) < 1e-12) {
      double d = 0;
      for (int i = 0; i < 4; ++i) d = std::max(d, std::abs(m.a[i] - tr * kPauli[p].a[i]));
      if (d < 1e-12) {
        *phase = tr;
        return p;
      }
    }
  }
  return -1;
}

struct Bloch {
  double rx, ry, rz;
  double length() const { return std::sqrt(rx * rx + ry * ry + rz * rz); }
};

Bloch bloch_from_sums(const double s[4]) { return {2.0 * s[0], 2.0 * s[1], s[2] - s[3]}; }  // ket.py:204-210

double epsilon(const Bloch& r) { return (1.0 - std::min(r.length(), 1.0)) / 2.0; }  // ket.py:37-39

// unit Bloch vector -> pure single-qubit state along it (ket.py:42-54)
void bloch_to_state(const Bloch& r, cd phi[2]) {
  const double norm = r.length();
  const double nz = r.rz / norm;
  const double c = std::sqrt(std::max(0.0, (1.0 + nz) / 2.0));
  const double s = std::sqrt(std::max(0.0, (1.0 - nz) / 2.0));
  if (s < 1e-15) {
    phi[0] = 1.0;
    phi[1] = 0.0;
    return;
  }
  const double a = std::atan2(r.ry / norm, r.rx / norm);
  phi[0] = c;
  phi[1] = s * std::exp(cd(0, 1) * a);
}

struct Qubit;

// Bloch sums of a width-1 shard: none, known on the host, or being
// published by the kernel that wrote the shard into a mapped ring slot
enum SumsKind { kSumsNone = 0, kSumsHost = 1, kSumsSlot = 2 };

struct SumsTicket {
  int kind = kSumsNone;
  int slot = 0;
  unsigned long long seq = 0;
  double v[4] = {0, 0, 0, 0};
};

struct Shard {
  sk_state* st = nullptr;                 // dense shards (a distributed shard: this rank's slab)
  std::unique_ptr<sktab::Tableau> tab;    // stabilizer shards (engine.py Shard kind "stab")
  std::vector<Qubit*> qubits;  // position -> qubit
  SumsTicket sums;             // width-1 shards only
  int G = 0;                   // distributed over 2^G ranks: positions [w-G, w) are the rank bits
  int width() const { return (int)qubits.size(); }
  int wl() const { return width() - G; }  // local positions [0, wl) = bits of this rank's slab
  bool stab() const { return (bool)tab; }
};

constexpr int kRingSlots = 4096;
constexpr int kSlotDoubles = 8;  // 4 sums, the sequence word, padding

struct PendingOp {  // a buffered controlled phase / inversion (engine.py:_CtrlOp)
  int64_t seq;
  std::vector<Qubit*> controls;
  std::vector<int> polarity;
  Qubit* target;
  M2 m;
  std::vector<Qubit*> qubits() const {
    std::vector<Qubit*> q = controls;
    q.push_back(target);
    return q;
  }
};

struct Qubit {
  Shard* shard = nullptr;
  int pos = 0;
  bool has_u = false;
  M2 u;
  std::deque<PendingOp*> pending;
};

}  // namespace

// ---------------------------------------------------------------------------
// engine kernels.  Every element operation and reduction is the shared one
// of sk_ops.cuh, so results are bit-identical to the separate ket kernels
// (k_apply_1q, k_kron, k_ctrl_bloch, k_round, k_set_single) they fuse.
// ---------------------------------------------------------------------------
namespace sk {

constexpr int kEThreads = 256;
// widths whose one-control gate k_ctrl_bloch reduces in a single block
// (2^(w-2) quads <= 256 threads x 2): the fused coupler kernel keeps its
// summation order
constexpr int kFusedMaxW = 11;

template <typename R>
__device__ __forceinline__ Mat2<R> dmat(const double* m) {
  Mat2<R> r;
  r.m00 = mk<R>((R)m[0], (R)m[1]);
  r.m01 = mk<R>((R)m[2], (R)m[3]);
  r.m10 = mk<R>((R)m[4], (R)m[5]);
  r.m11 = mk<R>((R)m[6], (R)m[7]);
  return r;
}

struct CouplerArgs {
  void* pre_ptr[2];  // committed 1q buffers (engine.py:376 -> :305-322), in order
  int pre_w[2], pre_q[2], pre_diag[2];
  double pre_m[2][8];
  int npre;
  const void* lo;    // merge (engine.py:224-243): out = kron(hi, lo); lo == nullptr: no merge
  const void* hi;
  int wa, wb;
  void* out;         // the state the gate acts on
  int c, pol, t, w;
  double m[8];
};

// A committed one-control coupler on a small shard, one block: the operands'
// 1q buffers, the Kronecker merge, the gate and both operands' Bloch sums
// (engine.py:367-394) in one launch.
template <typename R>
__global__ void __launch_bounds__(kEThreads) k_e_coupler(const __grid_constant__ CouplerArgs A, RedOut ro) {
  const int tid = threadIdx.x;
  for (int i = 0; i < A.npre; ++i) {
    vec2_t<R>* a = (vec2_t<R>*)A.pre_ptr[i];
    const Mat2<R> m = dmat<R>(A.pre_m[i]);
    const int64_t np = int64_t(1) << (A.pre_w[i] - 1);
    const uint64_t bit = 1ull << A.pre_q[i];
    for (int64_t k = tid; k < np; k += kEThreads) apply_1q_pair<R>(a, insert0(k, A.pre_q[i]), bit, m, A.pre_diag[i]);
    __syncthreads();
  }
  vec2_t<R>* s = (vec2_t<R>*)A.out;
  if (A.lo) {
    const vec2_t<R>* lo = (const vec2_t<R>*)A.lo;
    const vec2_t<R>* hi = (const vec2_t<R>*)A.hi;
    const int64_t n = int64_t(1) << (A.wa + A.wb);
    const uint64_t mask = (1ull << A.wa) - 1;
    for (int64_t i = tid; i < n; i += kEThreads) s[i] = cmul<R>(hi[(uint64_t)i >> A.wa], lo[(uint64_t)i & mask]);
    __syncthreads();
  }
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const Mat2<R> m = dmat<R>(A.m);
  const uint64_t C = 1ull << A.c, T = 1ull << A.t;
  const int lo_b = A.c < A.t ? A.c : A.t, hi_b = A.c < A.t ? A.t : A.c;
  const int64_t nq = int64_t(1) << (A.w - 2);
  for (int64_t k = tid; k < nq; k += kEThreads) ctrl_bloch_quad<R>(s, insert0(insert0(k, lo_b), hi_b), C, T, A.pol, m, v);
  block_reduce_finish<8>(v, ro);
}

// kron_compose (ket.py:239-241) into a caller-provided buffer
template <typename R>
__global__ void __launch_bounds__(kEThreads) k_e_kron(const vec2_t<R>* __restrict__ lo, const vec2_t<R>* __restrict__ hi,
                                                     vec2_t<R>* __restrict__ out, int64_t n, int wa) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t mask = (1ull << wa) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = cmul<R>(hi[(uint64_t)i >> wa], lo[(uint64_t)i & mask]);
}

// the same with a narrow high factor: lo read once, 2^wb products written
template <typename R>
__global__ void __launch_bounds__(kEThreads) k_e_kron_narrow(const vec2_t<R>* __restrict__ lo,
                                                            const vec2_t<R>* __restrict__ hi, vec2_t<R>* __restrict__ out,
                                                            int64_t nlo, int wa, int nhi) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlo; i += stride) {
    const vec2_t<R> x = lo[i];
    for (int j = 0; j < nhi; ++j) out[((uint64_t)j << wa) | (uint64_t)i] = cmul<R>(__ldg(hi + j), x);
  }
}

// this rank's slab of a product that becomes distributed: out[i] = prod[base + i]
template <typename R>
__global__ void __launch_bounds__(kEThreads) k_e_kron_slice(const vec2_t<R>* __restrict__ lo,
                                                           const vec2_t<R>* __restrict__ hi, vec2_t<R>* __restrict__ out,
                                                           int64_t n, int wa, uint64_t base) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t mask = (1ull << wa) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t j = base + (uint64_t)i;
    out[i] = cmul<R>(hi[j >> wa], lo[j & mask]);
  }
}

// SDRP rounding split (engine.py:464-488) in one launch: the remainder
// rest[k] = (u00 a0[k] + u01 a1[k]) / sqrt(P0) and the new width-1 shard phi
// with its published Bloch sums
template <typename R>
__global__ void __launch_bounds__(kEThreads) k_e_round_split(const vec2_t<R>* __restrict__ a, vec2_t<R>* __restrict__ out,
                                                            int64_t nout, int q, vec2_t<R> u00, vec2_t<R> u01, R scale,
                                                            vec2_t<R>* single, double p0r, double p0i, double p1r,
                                                            double p1i, double* out4, unsigned long long* flag,
                                                            unsigned long long seq) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nout; k += stride) {
    uint64_t i0 = insert0(k, q);
    vec2_t<R> y = cmad2<R>(u00, a[i0], u01, a[i0 | bit]);
    out[k] = mk<R>(y.x * scale, y.y * scale);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) publish_single<R>(single, p0r, p0i, p1r, p1i, out4, flag, seq);
}

}  // namespace sk

using namespace sk;

constexpr int kPoolMaxW = 18;   // cache freed shard buffers up to 4 MiB (c128)
static const float kOneF[2] = {1.0f, 0.0f};
constexpr size_t kPoolPerW = 32;

struct sk_engine {
  int n = 0;
  sk_engine_config cfg{};
  std::vector<std::unique_ptr<Qubit>> own;
  std::vector<Qubit*> handles;  // label -> qubit
  std::unordered_set<Shard*> shards;
  std::vector<double> eps;
  int64_t dense_total = 0, peak = 0;
  int64_t stats[SK_ENGINE_NSTATS] = {0};
  int64_t seq = 0;
  int64_t needed = 0;  // last budget failure
  sk_uniform_fn ufn = nullptr;
  void* uctx = nullptr;
  sk_bit_fn bfn = nullptr;  // rng.integers(0, 2): tableau measurements (tableau.py:214)
  void* bctx = nullptr;
  // distributed largest shard: SPMD over `world` ranks, every
  // rank runs this engine on the same circuit; a dense shard wider than
  // local_max is split over the ranks by its top log2(world) positions and its
  // reductions are summed over ranks, so all ranks take the same decisions
  int world = 1, rank = 0, Gw = 0, local_max = 64;
  sk_allreduce_fn f_allreduce = nullptr;
  sk_sendrecv_fn f_sendrecv = nullptr;
  sk_allgather_fn f_allgather = nullptr;
  void* dctx = nullptr;
  double* h_ring = nullptr;  // mapped pinned ring of sums slots
  double* d_ring = nullptr;
  int ring_next = 0;
  unsigned long long ring_seq = 0;
  std::vector<void*> pool[kPoolMaxW + 1];  // freed shard buffers by width (stream-ordered reuse)
  DevCtx* ctx = nullptr;

  ~sk_engine() {
    std::unordered_set<PendingOp*> ops;
    for (auto& q : own)
      for (auto* op : q->pending) ops.insert(op);
    for (auto* op : ops) delete op;
    for (auto* s : shards) {
      sk_destroy(s->st);
      delete s;
    }
    DevCtx* c;
    if (ctx_get(cfg.device, &c) == SK_OK) {
      for (auto& v : pool)
        for (void* p : v) cudaFreeAsync(p, c->stream);
      if (h_ring) cudaStreamSynchronize(c->stream);  // kernels may still publish
    }
    if (h_ring) cudaFreeHost(h_ring);
  }

  // shard buffers: engine-side cache of freed device buffers per width, so
  // the merge / split churn of small shards never reaches the driver
  int alloc_state(int w, sk_state** out) {
    if (w <= kPoolMaxW && !pool[w].empty()) {
      sk_state* s = new sk_state();
      s->width = w;
      s->dtype = cfg.dtype;
      s->device = cfg.device;
      s->n = int64_t(1) << w;
      s->elem = elem_size(cfg.dtype);
      s->d = pool[w].back();
      pool[w].pop_back();
      *out = s;
    } else {
      SK_TRY(state_alloc(w, cfg.dtype, cfg.device, out));
    }
    stats[SK_ENGINE_STAT_ALLOCS]++;
    return SK_OK;
  }

  void free_state(sk_state* s) {
    if (!s) return;
    if (s->owned && s->d && s->width <= kPoolMaxW && pool[s->width].size() < kPoolPerW) {
      pool[s->width].push_back(s->d);
      delete s;
      return;
    }
    sk_destroy(s);
  }

  unsigned long long ring_ticket(double** dslot, int* slot) {
    *slot = ring_next;
    ring_next = (ring_next + 1) % kRingSlots;
    *dslot = d_ring + (size_t)*slot * kSlotDoubles;
    return ++ring_seq;
  }

  int init_ring() {
    DevCtx* c;
    SK_TRY(ctx_get(cfg.device, &c));
    ctx = c;
    SK_CUDA(cudaHostAlloc(&h_ring, sizeof(double) * kRingSlots * kSlotDoubles, cudaHostAllocMapped));
    SK_CUDA(cudaHostGetDevicePointer((void**)&d_ring, h_ring, 0));
    memset(h_ring, 0, sizeof(double) * kRingSlots * kSlotDoubles);
    return SK_OK;
  }

  // ---- budget (engine.py:202-214) -----------------------------------------
  int charge(int64_t amount, int64_t transient = 0) {
    const int64_t need = dense_total + amount + transient;
    if (need > cfg.mem_budget) {
      needed = need;
      return set_error(SK_EBUDGET, "needs %lld dense amplitudes, budget is %lld", (long long)need,
                       (long long)cfg.mem_budget);
    }
    dense_total += amount;
    peak = std::max(peak, need);
    return SK_OK;
  }

  int release(int64_t amount) {
    dense_total -= amount;
    if (dense_total < 0) return set_error(SK_EVALUE, "dense amplitude accounting went negative");
    return SK_OK;
  }

  // ---- shards ------------------------------------------------------------------
  Shard* new_shard(sk_state* st) {
    Shard* s = new Shard();
    s->st = st;
    shards.insert(s);
    return s;
  }

  void drop_shard(Shard* s) {
    shards.erase(s);
    free_state(s->st);
    delete s;
  }

  // a width-1 device shard holding amps; its kernel publishes the shard's
  // Bloch sums (from the stored precision, as a reduction would) to a ring slot
  int make_single(const cd amps[2], sk_state** out, SumsTicket* t) {
    const double h[4] = {amps[0].real(), amps[0].imag(), amps[1].real(), amps[1].imag()};
    const int slot = ring_next;
    ring_next = (ring_next + 1) % kRingSlots;
    const unsigned long long seq = ++ring_seq;
    double* d = d_ring + (size_t)slot * kSlotDoubles;
    SK_TRY(create_single_with_sums(cfg.dtype, cfg.device, h, d, (unsigned long long*)(d + 4), seq, out));
    t->kind = kSumsSlot;
    t->slot = slot;
    t->seq = seq;
    stats[SK_ENGINE_STAT_ALLOCS]++;
    return SK_OK;
  }

  int fresh_single(Qubit* q, int bit) {  // engine.py:187-200
    if (cfg.stabilizer_hybrid) {  // a width-1 tableau, no dense amplitudes
      Shard* s = new Shard();
      shards.insert(s);
      s->tab.reset(new sktab::Tableau(1));
      if (bit) s->tab->px(0);
      s->qubits = {q};
      q->shard = s;
      q->pos = 0;
      return SK_OK;
    }
    SK_TRY(charge(2));
    cd a[2] = {bit ? 0.0 : 1.0, bit ? 1.0 : 0.0};
    sk_state* st;
    double h[4] = {a[0].real(), a[0].imag(), a[1].real(), a[1].imag()};
    SK_TRY(sk_create_from(1, cfg.dtype, cfg.device, h, &st));
    stats[SK_ENGINE_STAT_ALLOCS]++;
    Shard* s = new_shard(st);
    s->qubits = {q};
    s->sums.kind = kSumsHost;  // basis states: the sums are exact
    s->sums.v[0] = s->sums.v[1] = 0.0;
    s->sums.v[2] = bit ? 0.0 : 1.0;
    s->sums.v[3] = bit ? 1.0 : 0.0;
    q->shard = s;
    q->pos = 0;
    return SK_OK;
  }

  // exact dense ket of a tableau: replay its log on |0..0> with the device
  // kernels (tableau.py:258-282)
  int replay(const sktab::Tableau& t, sk_state** out) {
    sk_state* st;
    SK_TRY(alloc_state(t.w, &st));
    const size_t bytes = (size_t)st->n * st->elem;
    SK_CUDA(cudaMemsetAsync(st->d, 0, bytes, ctx->stream));
    const double one[2] = {1.0, 0.0};
    SK_CUDA(cudaMemcpyAsync(st->d, cfg.dtype == SK_C64 ? (const void*)&kOneF : (const void*)one,
                            cfg.dtype == SK_C64 ? 8 : 16, cudaMemcpyHostToDevice, ctx->stream));
    const double s2 = 1.0 / std::sqrt(2.0);
    const cd e = std::exp(cd(0, 1) * (M_PI / 2));
    const double H[8] = {s2, 0, s2, 0, s2, 0, -s2, 0};
    const double S[8] = {1, 0, 0, 0, 0, 0, e.real(), e.imag()};
    const double X[8] = {0, 0, 1, 0, 1, 0, 0, 0};
    const double Y[8] = {0, 0, 0, -1, 0, 1, 0, 0};
    const double Z[8] = {1, 0, 0, 0, 0, 0, -1, 0};
    int rc = SK_OK;
    for (const auto& en : t.log) {
      switch (en.op) {
        case sktab::L_H: rc = sk_apply_1q(st, en.a, H); break;
        case sktab::L_S: rc = sk_apply_1q(st, en.a, S); break;
        case sktab::L_X: rc = sk_apply_1q(st, en.a, X); break;
        case sktab::L_Y: rc = sk_apply_1q(st, en.a, Y); break;
        case sktab::L_Z: rc = sk_apply_1q(st, en.a, Z); break;
        case sktab::L_SWAP: rc = sk_swap_qubits(st, en.a, en.b); break;
        case sktab::L_CX: rc = sk_apply_controlled(st, 1ull << en.a, 1ull << en.a, en.b, X); break;
        case sktab::L_M: {
          double prob;
          rc = sk_project(st, en.a, en.b, &prob);
          break;
        }
        case sktab::L_GPHASE: rc = sk_scale(st, en.phase.real(), en.phase.imag()); break;
      }
      if (rc != SK_OK) {
        free_state(st);
        return rc;
      }
    }
    *out = st;
    return SK_OK;
  }

  int to_dense(Shard* s) {  // engine.py:216-222
    if (!s->stab()) return SK_OK;
    SK_TRY(charge(int64_t(1) << s->width()));
    sk_state* st;
    if (s->width() == 1 && s->tab->log.empty()) {  // an untouched qubit: |0>, sums exact
      double h[4] = {1.0, 0.0, 0.0, 0.0};
      SK_TRY(sk_create_from(1, cfg.dtype, cfg.device, h, &st));
      stats[SK_ENGINE_STAT_ALLOCS]++;
      s->tab.reset();
      s->st = st;
      s->sums.kind = kSumsHost;
      s->sums.v[0] = s->sums.v[1] = s->sums.v[3] = 0.0;
      s->sums.v[2] = 1.0;
      return SK_OK;
    }
    SK_TRY(replay(*s->tab, &st));
    s->tab.reset();
    s->st = st;
    s->sums.kind = kSumsNone;
    return SK_OK;
  }

  // ---- distributed shard (row f2) -------------------------------------------------
  int sync_stream() {
    SK_CUDA(cudaStreamSynchronize(ctx->stream));
    return SK_OK;
  }

  int allreduce(double* x, int n) {  // sum over ranks (every rank gets the same doubles)
    if (world == 1) return SK_OK;
    if (f_allreduce(dctx, x, n) != 0) return set_error(SK_ECUDA, "distributed all-reduce failed");
    return SK_OK;
  }

  // bring the qubit at global position pos into the slab: swap its rank bit
  // with the top local bit (first moving a non-busy local qubit there);
  // partners exchange the half slab whose top bit disagrees with their rank bit
  int localize(Shard* s, int pos, const std::vector<int>& busy) {
    const int wl = s->wl();
    if (pos < wl) return SK_OK;
    int v = -1;
    for (int p = wl - 1; p >= 0 && v < 0; --p)
      if (std::find(busy.begin(), busy.end(), p) == busy.end()) v = p;
    if (v < 0) return set_error(SK_EVALUE, "distributed shard: no free local qubit to swap with");
    if (v != wl - 1) {  // a local bit swap puts the victim on top (one slab pass)
      SK_TRY(sk_swap_qubits(s->st, v, wl - 1));
      std::swap(s->qubits[v], s->qubits[wl - 1]);
      s->qubits[v]->pos = v;
      s->qubits[wl - 1]->pos = wl - 1;
    }
    const int g = pos - wl;
    const int rb = (rank >> g) & 1, partner = rank ^ (1 << g);
    const size_t half = ((size_t)1 << (wl - 1)) * s->st->elem;
    unsigned char* mine = (unsigned char*)s->st->d + (size_t)(1 - rb) * half;
    void* tmp = nullptr;
    SK_CUDA(cudaMallocAsync(&tmp, half, ctx->stream));
    SK_TRY(sync_stream());
    const int rc = f_sendrecv(dctx, partner, (uint64_t)mine, (uint64_t)tmp, (int64_t)half);
    if (rc != 0) {
      cudaFreeAsync(tmp, ctx->stream);
      return set_error(SK_ECUDA, "distributed exchange with rank %d failed", partner);
    }
    SK_CUDA(cudaMemcpyAsync(mine, tmp, half, cudaMemcpyDeviceToDevice, ctx->stream));
    SK_CUDA(cudaFreeAsync(tmp, ctx->stream));
    std::swap(s->qubits[wl - 1], s->qubits[pos]);
    s->qubits[wl - 1]->pos = wl - 1;
    s->qubits[pos]->pos = pos;
    stats[SK_ENGINE_STAT_EXCHANGES]++;
    return SK_OK;
  }

  // a distributed shard narrow enough for one device again (or any, for a
  // read-out): all-gather the slabs
  int undistribute(Shard* s, bool force = false) {
    if (!s->G || (s->width() > local_max && !force)) return SK_OK;
    sk_state* full;
    SK_TRY(alloc_state(s->width(), &full));
    const size_t bytes = (size_t)s->st->n * s->st->elem;
    SK_TRY(sync_stream());
    if (f_allgather(dctx, (uint64_t)s->st->d, (uint64_t)full->d, (int64_t)bytes) != 0)
      return set_error(SK_ECUDA, "distributed all-gather failed");
    free_state(s->st);
    s->st = full;
    s->G = 0;
    return SK_OK;
  }

  int dist_product(Shard* a, Shard* b, Shard** out) {  // a (wider) x b wider than local_max: split it
    const int wa = a->width(), wb = b->width(), w = wa + wb, wl = w - Gw;
    if (wl < 2) return set_error(SK_EVALUE, "distributed shard of %d qubits over %d ranks is too narrow", w, world);
    SK_TRY(charge(int64_t(1) << w));
    sk_state* st;
    SK_TRY(alloc_state(wl, &st));
    const int64_t n = int64_t(1) << wl;
    const int g = grid_for(n, kEThreads, 2, ctx->num_sms);
    const uint64_t base = (uint64_t)rank << wl;
    if (cfg.dtype == SK_C64)
      k_e_kron_slice<float><<<g, kEThreads, 0, ctx->stream>>>((const float2*)a->st->d, (const float2*)b->st->d,
                                                               (float2*)st->d, n, wa, base);
    else
      k_e_kron_slice<double><<<g, kEThreads, 0, ctx->stream>>>((const double2*)a->st->d, (const double2*)b->st->d,
                                                                (double2*)st->d, n, wa, base);
    SK_CHECK_LAUNCH();
    SK_TRY(merged_shard(a, b, st, out));
    (*out)->G = Gw;  // positions [wl, w): the top Gw positions are the rank bits
    stats[SK_ENGINE_STAT_DIST_SHARDS]++;
    return SK_OK;
  }

  int dist_kron(Shard* d, Shard* r, Shard** out) {  // distributed d x replicated r: each slab grows locally
    if (r->G) return set_error(SK_EVALUE, "merging two distributed shards is not supported");
    const int wl = d->wl(), wr = r->width(), w = d->width() + wr;
    SK_TRY(charge(int64_t(1) << w));
    sk_state* st;
    SK_TRY(alloc_state(wl + wr, &st));
    const int64_t n = int64_t(1) << (wl + wr);
    const int g = grid_for(n, kEThreads, 2, ctx->num_sms);
    if (cfg.dtype == SK_C64)
      k_e_kron<float><<<g, kEThreads, 0, ctx->stream>>>((const float2*)d->st->d, (const float2*)r->st->d,
                                                         (float2*)st->d, n, wl);
    else
      k_e_kron<double><<<g, kEThreads, 0, ctx->stream>>>((const double2*)d->st->d, (const double2*)r->st->d,
                                                          (double2*)st->d, n, wl);
    SK_CHECK_LAUNCH();
    stats[SK_ENGINE_STAT_MERGES]++;
    stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << w;
    SK_TRY(release((int64_t(1) << d->width()) + (int64_t(1) << wr)));
    Shard* m = new_shard(st);
    // positions: d's local, r's (new local bits above them), d's rank bits on top
    m->qubits.assign(d->qubits.begin(), d->qubits.begin() + wl);
    m->qubits.insert(m->qubits.end(), r->qubits.begin(), r->qubits.end());
    m->qubits.insert(m->qubits.end(), d->qubits.begin() + wl, d->qubits.end());
    m->G = d->G;
    for (int i = 0; i < m->width(); ++i) {
      m->qubits[i]->shard = m;
      m->qubits[i]->pos = i;
    }
    drop_shard(d);
    drop_shard(r);
    *out = m;
    return SK_OK;
  }

  int merge_pair(Shard* a, Shard* b, Shard** out, bool stab_ok = false) {  // engine.py:224-243
    if (a->width() < b->width()) std::swap(a, b);  // the wider keeps its positions
    if (stab_ok && a->stab() && b->stab()) {
      stats[SK_ENGINE_STAT_MERGES]++;
      Shard* m = new Shard();
      shards.insert(m);
      m->tab.reset(new sktab::Tableau(sktab::merge(*a->tab, *b->tab)));
      m->qubits = a->qubits;
      m->qubits.insert(m->qubits.end(), b->qubits.begin(), b->qubits.end());
      for (int i = 0; i < m->width(); ++i) {
        m->qubits[i]->shard = m;
        m->qubits[i]->pos = i;
      }
      shards.erase(a);
      shards.erase(b);
      delete a;
      delete b;
      *out = m;
      return SK_OK;
    }
    SK_TRY(to_dense(a));
    SK_TRY(to_dense(b));
    const int wa = a->width(), wb = b->width();
    if (a->G || b->G) return a->G ? dist_kron(a, b, out) : dist_kron(b, a, out);
    if (world > 1 && wa + wb > local_max) return dist_product(a, b, out);
    SK_TRY(charge(int64_t(1) << (wa + wb)));
    sk_state* st;
    SK_TRY(alloc_state(wa + wb, &st));
    const int64_t n = int64_t(1) << (wa + wb);
    if (wb <= 4 && wa >= 10) {
      const int64_t nlo = int64_t(1) << wa;
      const int g = grid_for(nlo, kEThreads, 2, ctx->num_sms);
      if (cfg.dtype == SK_C64)
        k_e_kron_narrow<float><<<g, kEThreads, 0, ctx->stream>>>((const float2*)a->st->d, (const float2*)b->st->d,
                                                                  (float2*)st->d, nlo, wa, 1 << wb);
      else
        k_e_kron_narrow<double><<<g, kEThreads, 0, ctx->stream>>>((const double2*)a->st->d, (const double2*)b->st->d,
                                                                   (double2*)st->d, nlo, wa, 1 << wb);
      SK_CHECK_LAUNCH();
      return merged_shard(a, b, st, out);
    }
    const int g = grid_for(n, kEThreads, 2, ctx->num_sms);
    if (cfg.dtype == SK_C64)
      k_e_kron<float><<<g, kEThreads, 0, ctx->stream>>>((const float2*)a->st->d, (const float2*)b->st->d,
                                                         (float2*)st->d, n, wa);
    else
      k_e_kron<double><<<g, kEThreads, 0, ctx->stream>>>((const double2*)a->st->d, (const double2*)b->st->d,
                                                          (double2*)st->d, n, wa);
    SK_CHECK_LAUNCH();
    SK_TRY(merged_shard(a, b, st, out));
    return SK_OK;
  }

  // bookkeeping of a merge whose product is already (being) written to st
  int merged_shard(Shard* a, Shard* b, sk_state* st, Shard** out) {
    const int wa = a->width(), wb = b->width();
    stats[SK_ENGINE_STAT_MERGES]++;
    stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << (wa + wb);
    SK_TRY(release((int64_t(1) << wa) + (int64_t(1) << wb)));
    Shard* m = new_shard(st);
    m->qubits = a->qubits;
    m->qubits.insert(m->qubits.end(), b->qubits.begin(), b->qubits.end());
    for (int i = 0; i < m->width(); ++i) {
      m->qubits[i]->shard = m;
      m->qubits[i]->pos = i;
    }
    drop_shard(a);
    drop_shard(b);
    *out = m;
    return SK_OK;
  }

  int merge_for(const std::vector<Qubit*>& qs, Shard** out, bool stab_ok = false) {  // engine.py:245-255
    std::vector<Shard*> list;
    for (Qubit* q : qs)
      if (std::find(list.begin(), list.end(), q->shard) == list.end()) list.push_back(q->shard);
    Shard* m = list[0];
    for (size_t i = 1; i < list.size(); ++i) SK_TRY(merge_pair(m, list[i], &m, stab_ok));
    if (!stab_ok) SK_TRY(to_dense(m));
    *out = m;
    return SK_OK;
  }

  // replace shard by (rest, new width-1 shard {single}) (engine.py:257-270)
  int split(Shard* shard, int pos, sk_state* single, const SumsTicket& single_sums, sk_state* rest) {
    Qubit* q = shard->qubits[pos];
    const int64_t old = int64_t(1) << shard->width();
    stats[SK_ENGINE_STAT_SPLITS]++;
    Shard* s1 = new_shard(single);
    s1->qubits = {q};
    s1->sums = single_sums;
    q->shard = s1;
    q->pos = 0;
    shard->qubits.erase(shard->qubits.begin() + pos);
    for (int i = 0; i < shard->width(); ++i) shard->qubits[i]->pos = i;
    free_state(shard->st);
    shard->st = rest;
    shard->sums.kind = kSumsNone;
    dense_total += (2 + (int64_t(1) << shard->width())) - old;  // global widths (a distributed rest is a slab)
    return undistribute(shard);
  }

  // Bloch sums of q in its shard: width-1 shards carry them (host values or
  // a ring slot their kernel published); else one device reduction returned
  // through mapped memory
  int sums_of(Qubit* q, double out[4]) {
    Shard* s = q->shard;
    if (s->width() == 1 && s->sums.kind == kSumsSlot) {
      volatile double* slot = h_ring + (size_t)s->sums.slot * kSlotDoubles;
      volatile unsigned long long* flag = (volatile unsigned long long*)(slot + 4);
      if (*flag <= s->sums.seq) {  // not overwritten by a newer publication: wait for ours
        SK_TRY(wait_mapped(cfg.device, flag, s->sums.seq));
        for (int k = 0; k < 4; ++k) s->sums.v[k] = slot[k];
        s->sums.kind = *flag == s->sums.seq ? kSumsHost : kSumsNone;
      } else {
        s->sums.kind = kSumsNone;
      }
    }
    if (s->width() == 1 && s->sums.kind == kSumsHost) {
      std::copy(s->sums.v, s->sums.v + 4, out);
      return SK_OK;
    }
    if (s->G) {  // a distributed shard: local reduction on every rank, summed over ranks
      SK_TRY(localize(s, q->pos, {}));
      SK_TRY(sk_bloch_sums(s->st, q->pos, out));
      return allreduce(out, 4);
    }
    SK_TRY(sk_bloch_sums(s->st, q->pos, out));
    if (s->width() == 1) {
      s->sums.kind = kSumsHost;
      std::copy(out, out + 4, s->sums.v);
    }
    return SK_OK;
  }

  // ---- 1q buffers (engine.py:276-322) ----------------------------------------
  int absorb_1q(Qubit* q, const M2& m) {
    if (!q->pending.empty() && !commute_past(q, m)) SK_TRY(flush_pending(q));
    q->u = q->has_u ? mmul(m, q->u) : m;
    q->has_u = true;
    return SK_OK;
  }

  bool commute_past(Qubit* q, const M2& m) {  // all or nothing (engine.py:281-303)
    struct Plan {
      PendingOp* op;
      int action;  // 0 matrix, 1 keep, 2 flip
      M2 conj;
    };
    std::vector<Plan> plans;
    const bool d = is_diag(m), ad = !d && is_antidiag(m);
    for (PendingOp* op : q->pending) {
      if (op->target == q) {
        M2 c;
        if (!snap(mmul(mmul(m, op->m), mdag(m)), &c)) return false;
        plans.push_back({op, 0, c});
      } else if (d) {
        plans.push_back({op, 1, M2()});
      } else if (ad) {
        plans.push_back({op, 2, M2()});
      } else {
        return false;
      }
    }
    for (auto& p : plans) {
      if (p.action == 0) {
        p.op->m = p.conj;
      } else if (p.action == 2) {
        auto it = std::find(p.op->controls.begin(), p.op->controls.end(), q);
        p.op->polarity[it - p.op->controls.begin()] ^= 1;
      }
    }
    return true;
  }

  int commit_1q(Qubit* q) {  // engine.py:305-322
    if (!q->has_u) return SK_OK;
    const M2 m = q->u;
    q->has_u = false;
    if (is_identity(m)) return SK_OK;
    Shard* s = q->shard;
    if (s->stab()) {  // a Clifford buffer commits into the tableau, anything else converts it
      std::string word;
      cd phase;
      if (sktab::match_clifford_1q(m.a, &word, &phase)) {
        s->tab->apply_word(word, q->pos);
        s->tab->append_phase(phase);
        return SK_OK;
      }
      SK_TRY(to_dense(s));
    }
    if (!unitary(m)) return set_error(SK_EVALUE, "matrix is not unitary within 1e-10");
    double m8[8];
    m_to8(m, m8);
    if (s->G) SK_TRY(localize(s, q->pos, {}));
    SK_TRY(sk_apply_1q(s->st, q->pos, m8));
    stats[SK_ENGINE_STAT_KERNELS]++;
    stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << s->width();
    s->sums.kind = kSumsNone;
    return SK_OK;
  }

  // ---- buffered controlled ops (engine.py:328-365) ------------------------------
  int buffer_ctrl(const std::vector<Qubit*>& chs, const std::vector<int>& pol, Qubit* target, const M2& m) {
    PendingOp* tail = target->pending.empty() ? nullptr : target->pending.back();
    if (tail && tail->target == target && tail->controls == chs && tail->polarity == pol) {
      bool all_tail = true;
      for (Qubit* x : tail->qubits())
        if (x->pending.empty() || x->pending.back() != tail) all_tail = false;
      if (all_tail) {
        M2 fused;
        if (!snap(mmul(m, tail->m), &fused))
          return set_error(SK_EVALUE, "fused controlled op left the buffered class");
        if (is_identity(fused)) {
          for (Qubit* x : tail->qubits()) x->pending.erase(std::find(x->pending.begin(), x->pending.end(), tail));
          delete tail;
        } else {
          tail->m = fused;
        }
        return SK_OK;
      }
    }
    PendingOp* op = new PendingOp{++seq, chs, pol, target, m};
    for (Qubit* x : op->qubits()) x->pending.push_back(op);
    return SK_OK;
  }

  int flush_pending(Qubit* q) {
    while (!q->pending.empty()) SK_TRY(commit_chain(q->pending.front()));
    return SK_OK;
  }

  int commit_chain(PendingOp* op) {
    const std::vector<Qubit*> qs = op->qubits();
    for (Qubit* x : qs)
      while (!x->pending.empty() && x->pending.front() != op) SK_TRY(commit_chain(x->pending.front()));
    for (Qubit* x : qs) {
      if (x->pending.empty() || x->pending.front() != op)
        return set_error(SK_EVALUE, "pending op queues lost chronological order");
      x->pending.pop_front();
    }
    std::vector<Qubit*> c = op->controls;
    std::vector<int> p = op->polarity;
    Qubit* t = op->target;
    const M2 m = op->m;
    delete op;
    return commit_ctrl(c, p, t, m);
  }

  // flush operand buffers, merge, run the kernel, then try to factor or
  // round each operand (engine.py:367-394); with one control the kernel
  // also returns both operands' Bloch sums (one pass instead of three)
  int commit_ctrl(const std::vector<Qubit*>& controls, const std::vector<int>& pol, Qubit* target, const M2& m) {
    std::vector<Qubit*> qs = controls;
    qs.push_back(target);
    double out8[8];
    bool fused = false;
    bool any_stab = false;
    for (Qubit* q : qs) any_stab = any_stab || q->shard->stab();
    if (any_stab) {
      // The fused path below serves tableau operands whose own 1q buffer is
      // non-Clifford (every qubit of the random-circuit workloads): the
      // reference's commit_1q converts exactly those shards, in operand order
      // (engine.py:318-321), before the merge — so convert them here the same
      // way.  Anything else (a tableau coupler, or a conversion the merge would
      // order by width) takes the general path.
      bool fast = controls.size() == 1 && !stab_coupler_ok(controls, target, m);
      for (Qubit* q : qs) {
        std::string word;
        cd phase;
        if (q->shard->stab() && !(q->has_u && !is_identity(q->u) && !sktab::match_clifford_1q(q->u.a, &word, &phase)))
          fast = false;
      }
      if (!fast) return commit_ctrl_stab(controls, pol, target, m);
      for (Qubit* q : qs) SK_TRY(to_dense(q->shard));
    }
    if (controls.size() == 1) SK_TRY(coupler_small(controls[0], pol[0], target, m, out8, &fused));
    if (!fused) {
      for (Qubit* q : qs) SK_TRY(commit_1q(q));
      Shard* s;
      SK_TRY(merge_for(qs, &s));
      if (!unitary(m)) return set_error(SK_EVALUE, "matrix is not unitary within 1e-10");
      double m8[8];
      m_to8(m, m8);
      if (s->G) {  // every operand into this rank's slab (rank-bit operands are swapped in)
        for (Qubit* q : qs) {
          std::vector<int> busy;
          for (Qubit* o : qs)
            if (o != q && o->pos < s->wl()) busy.push_back(o->pos);
          SK_TRY(localize(s, q->pos, busy));
        }
      }
      if (controls.size() == 1) {
        SK_TRY(sk_apply_controlled_bloch(s->st, controls[0]->pos, pol[0], target->pos, m8, out8));
        if (s->G) SK_TRY(allreduce(out8, 8));
        stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << (s->width() - 1);
      } else {
        uint64_t mask = 0, val = 0;
        for (size_t i = 0; i < controls.size(); ++i) {
          mask |= 1ull << controls[i]->pos;
          if (pol[i]) val |= 1ull << controls[i]->pos;
        }
        SK_TRY(sk_apply_controlled(s->st, mask, val, target->pos, m8));
        stats[SK_ENGINE_STAT_WRITES] += 2 * (int64_t(1) << (s->width() - 1 - (int)controls.size()));
      }
      s->sums.kind = kSumsNone;
      stats[SK_ENGINE_STAT_KERNELS]++;
    }
    const double* pre = controls.size() == 1 ? out8 : nullptr;
    for (size_t i = 0; i < qs.size(); ++i) {
      bool changed = false;
      SK_TRY(try_factor(qs[i], pre ? pre + 4 * i : nullptr, &changed));
      if (changed) pre = nullptr;  // later operands see a new state: recompute their sums
    }
    return SK_OK;
  }

  // engine.py:371-379, 396-403: the coupler can stay in the tableau (a
  // single-control Pauli or identity on tableau operands whose 1q buffers are Clifford)
  bool stab_coupler_ok(const std::vector<Qubit*>& controls, Qubit* target, const M2& m) const {
    if (!cfg.stabilizer_hybrid || controls.size() != 1) return false;
    bool ok = max_abs_diff(m, kI) < 1e-12;
    for (int p = 0; p < 3 && !ok; ++p) ok = max_abs_diff(m, kPauli[p]) < 1e-12;
    if (!ok) return false;
    for (Qubit* q : {controls[0], target}) {
      std::string word;
      cd phase;
      if (!q->shard->stab() || (q->has_u && !sktab::match_clifford_1q(q->u.a, &word, &phase))) return false;
    }
    return true;
  }

  // engine.py:367-394 with tableau operands: the coupler stays in the tableau
  // when it is a single-control Pauli (or identity) and every operand is a
  // tableau qubit whose 1q buffer is Clifford (engine.py:371-379, 396-403)
  int commit_ctrl_stab(const std::vector<Qubit*>& controls, const std::vector<int>& pol, Qubit* target, const M2& m) {
    std::vector<Qubit*> qs = controls;
    qs.push_back(target);
    int pauli = -1;
    const bool stab_ok = stab_coupler_ok(controls, target, m);
    for (Qubit* q : qs) SK_TRY(commit_1q(q));
    Shard* s;
    SK_TRY(merge_for(qs, &s, stab_ok));
    if (s->stab()) {
      cd ph;
      pauli = as_pauli(m, &ph);  // engine.py:382 drops the phase (it is 1 here)
      if (pauli >= 0) s->tab->ctrl_pauli(controls[0]->pos, pol[0], target->pos, pauli);
    } else {
      if (!unitary(m)) return set_error(SK_EVALUE, "matrix is not unitary within 1e-10");
      double m8[8];
      m_to8(m, m8);
      uint64_t mask = 0, val = 0;
      for (size_t i = 0; i < controls.size(); ++i) {
        mask |= 1ull << controls[i]->pos;
        if (pol[i]) val |= 1ull << controls[i]->pos;
      }
      SK_TRY(sk_apply_controlled(s->st, mask, val, target->pos, m8));
      stats[SK_ENGINE_STAT_WRITES] += 2 * (int64_t(1) << (s->width() - 1 - (int)controls.size()));
      s->sums.kind = kSumsNone;
      stats[SK_ENGINE_STAT_KERNELS]++;
    }
    for (Qubit* q : qs) {
      bool changed;
      SK_TRY(try_factor(q, nullptr, &changed));
    }
    return SK_OK;
  }

  // The one-control coupler on shards whose merged width is small, as ONE
  // launch (k_e_coupler): commit the operands' 1q buffers (engine.py:376),
  // merge (engine.py:377, :224-243), apply the gate and return both operands'
  // Bloch sums.  Bookkeeping and budget checks run in the reference's order;
  // *fused = false leaves everything to the general path.
  int coupler_small(Qubit* c, int pol, Qubit* t, const M2& m, double out8[8], bool* fused) {
    *fused = false;
    Shard *sa = c->shard, *sb = t->shard;
    const bool merge = sa != sb;
    const int w = merge ? sa->width() + sb->width() : sa->width();
    if (w > kFusedMaxW) return SK_OK;
    if (world > 1 && (sa->G || sb->G || w > local_max)) return SK_OK;  // distributed: the general path
    CouplerArgs A{};
    for (Qubit* q : {c, t}) {  // commit_1q of each operand (engine.py:305-322)
      if (!q->has_u) continue;
      const M2 u = q->u;
      q->has_u = false;
      if (is_identity(u)) continue;
      if (!unitary(u)) return set_error(SK_EVALUE, "matrix is not unitary within 1e-10");
      const int i = A.npre++;
      A.pre_ptr[i] = q->shard->st->d;
      A.pre_w[i] = q->shard->width();
      A.pre_q[i] = q->pos;
      m_to8(u, A.pre_m[i]);
      A.pre_diag[i] = (A.pre_m[i][2] == 0.0 && A.pre_m[i][3] == 0.0 && A.pre_m[i][4] == 0.0 && A.pre_m[i][5] == 0.0);
      stats[SK_ENGINE_STAT_KERNELS]++;
      stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << q->shard->width();
      q->shard->sums.kind = kSumsNone;
    }
    Shard *lo = sa, *hi = sb;
    sk_state* st = sa->st;
    if (merge) {
      if (lo->width() < hi->width()) std::swap(lo, hi);
      int rc = charge(int64_t(1) << w);
      if (rc != SK_OK) {  // the reference committed the buffers before its budget check
        for (int i = 0; i < A.npre; ++i) {
          sk_state tmp;
          tmp.d = A.pre_ptr[i];
          tmp.width = A.pre_w[i];
          tmp.dtype = cfg.dtype;
          tmp.device = cfg.device;
          tmp.n = int64_t(1) << A.pre_w[i];
          tmp.elem = elem_size(cfg.dtype);
          SK_TRY(sk_apply_1q(&tmp, A.pre_q[i], A.pre_m[i]));
        }
        return rc;
      }
      SK_TRY(alloc_state(w, &st));
      A.lo = lo->st->d;
      A.hi = hi->st->d;
      A.wa = lo->width();
      A.wb = hi->width();
    }
    if (!unitary(m)) return set_error(SK_EVALUE, "matrix is not unitary within 1e-10");
    A.out = st->d;
    A.w = w;
    A.pol = pol;
    m_to8(m, A.m);
    if (merge) {  // positions in the merged shard: the wider keeps its own
      A.c = c->shard == lo ? c->pos : lo->width() + c->pos;
      A.t = t->shard == lo ? t->pos : lo->width() + t->pos;
    } else {
      A.c = c->pos;
      A.t = t->pos;
    }
    std::lock_guard<std::mutex> lk(ctx->red_mu);
    const RedOut ro = red_out(ctx);
    if (cfg.dtype == SK_C64)
      k_e_coupler<float><<<1, kEThreads, 0, ctx->stream>>>(A, ro);
    else
      k_e_coupler<double><<<1, kEThreads, 0, ctx->stream>>>(A, ro);
    SK_CHECK_LAUNCH();
    Shard* s = sa;
    if (merge) SK_TRY(merged_shard(lo, hi, st, &s));
    stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << (w - 1);
    stats[SK_ENGINE_STAT_KERNELS]++;
    s->sums.kind = kSumsNone;
    SK_TRY(red_wait(ctx, ro, out8, 8));
    *fused = true;
    return SK_OK;
  }

  // ---- control elimination (engine.py:407-436) -----------------------------------
  int z_eigenstate(Qubit* q, int* z) {
    *z = -1;
    if (!q->pending.empty()) return SK_OK;
    const double tol = cfg.separability_tol;
    double r0[3];
    if (q->shard->stab()) {  // engine.py:418-423
      int basis, sign;
      if (!q->shard->tab->deterministic_eigen(q->pos, &basis, &sign)) return SK_OK;
      r0[0] = basis == 0 ? sign : 0.0;
      r0[1] = basis == 1 ? sign : 0.0;
      r0[2] = basis == 2 ? sign : 0.0;
    } else {
      if (q->shard->width() > 1) return SK_OK;  // entangled-shard scan not worth the pass
      double sums[4];
      SK_TRY(sums_of(q, sums));
      const Bloch b = bloch_from_sums(sums);
      if (epsilon(b) > tol) return SK_OK;
      r0[0] = b.rx, r0[1] = b.ry, r0[2] = b.rz;
    }
    if (q->has_u) {
      double R[3][3];
      so3(q->u, R);
      double r[3];
      for (int i = 0; i < 3; ++i) r[i] = R[i][0] * r0[0] + R[i][1] * r0[1] + R[i][2] * r0[2];
      std::copy(r, r + 3, r0);
    }
    if (r0[2] >= 1.0 - 2 * tol - 1e-12) *z = 0;
    else if (r0[2] <= -1.0 + 2 * tol + 1e-12) *z = 1;
    return SK_OK;
  }

  // ---- factorisation and Schmidt rounding (engine.py:442-512) ----------------------
  int try_decompose(Shard* shard, int pos, const double sums[4], bool* done) {
    // ket.py:243-267 with phi analytic in the sums: <dominant|a0>, <dominant|a1>
    *done = false;
    const cd cross(sums[0], sums[1]);
    const double n0 = sums[2], n1 = sums[3];
    int half;
    double ndom;
    cd phi[2];
    if (n0 >= 0.5) {
      half = 0, ndom = n0, phi[0] = n0, phi[1] = cross;
    } else {
      half = 1, ndom = n1, phi[0] = std::conj(cross), phi[1] = n1;
    }
    const double pn = std::sqrt(std::norm(phi[0]) + std::norm(phi[1]));
    phi[0] /= pn;
    phi[1] /= pn;
    sk_state* rest;
    SK_TRY(sk_compact(shard->st, pos, half, 1.0 / std::sqrt(ndom), 0.0, &rest));
    stats[SK_ENGINE_STAT_ALLOCS]++;
    sk_state* single;
    SumsTicket ss;
    SK_TRY(make_single(phi, &single, &ss));
    SK_TRY(split(shard, pos, single, ss, rest));
    *done = true;
    return SK_OK;
  }

  // returns the recorded eps (or -1 when none / degenerate); *rounded tells
  // whether the state changed
  int round_qubit(Shard* shard, int pos, const Bloch& r, double eps, const double sums[4], bool* rounded) {
    *rounded = false;
    M2 u = kI;
    cd phi[2] = {1.0, 0.0};
    if (r.length() >= 1e-12) {  // maximally mixed: identity rotation
      bloch_to_state(r, phi);
      u.a[0] = std::conj(phi[0]);
      u.a[1] = std::conj(phi[1]);
      u.a[2] = -phi[1];
      u.a[3] = phi[0];
    }
    const cd cross(sums[0], sums[1]);
    const double p0 = std::norm(u.a[0]) * sums[2] + std::norm(u.a[1]) * sums[3] +
                      2.0 * (std::conj(u.a[0]) * u.a[1] * cross).real();
    if (p0 < 1e-12) return SK_OK;  // numerically degenerate: leave the state alone (engine.py:477-480)
    const int w = shard->wl();  // the slab (a distributed shard rounds a local qubit on every rank)
    sk_state *rest, *single;
    SK_TRY(alloc_state(w - 1, &rest));
    SK_TRY(alloc_state(1, &single));
    SumsTicket ss;
    double* dslot;
    ss.kind = kSumsSlot;
    ss.seq = ring_ticket(&dslot, &ss.slot);
    const int64_t nout = int64_t(1) << (w - 1);
    const int g = grid_for(nout, kEThreads, 2, ctx->num_sms);
    const double scale = 1.0 / std::sqrt(p0);
    unsigned long long* dflag = (unsigned long long*)(dslot + 4);
    if (cfg.dtype == SK_C64)
      k_e_round_split<float><<<g, kEThreads, 0, ctx->stream>>>(
          (const float2*)shard->st->d, (float2*)rest->d, nout, pos, mk<float>((float)u.a[0].real(), (float)u.a[0].imag()),
          mk<float>((float)u.a[1].real(), (float)u.a[1].imag()), (float)scale, (float2*)single->d, phi[0].real(),
          phi[0].imag(), phi[1].real(), phi[1].imag(), dslot, dflag, ss.seq);
    else
      k_e_round_split<double><<<g, kEThreads, 0, ctx->stream>>>(
          (const double2*)shard->st->d, (double2*)rest->d, nout, pos, mk<double>(u.a[0].real(), u.a[0].imag()),
          mk<double>(u.a[1].real(), u.a[1].imag()), scale, (double2*)single->d, phi[0].real(), phi[0].imag(),
          phi[1].real(), phi[1].imag(), dslot, dflag, ss.seq);
    SK_CHECK_LAUNCH();
    stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << shard->width();
    SK_TRY(split(shard, pos, single, ss, rest));
    if (eps > cfg.separability_tol) eps_push(eps);
    *rounded = true;
    return SK_OK;
  }

  void eps_push(double e) { eps.push_back(e); }

  int try_factor(Qubit* q, const double* given, bool* changed) {
    *changed = false;
    Shard* shard = q->shard;
    if (shard->stab()) {  // engine.py:444-450: only p = 1 rounds a tableau (a forced measurement)
      int basis, sign;
      if (cfg.sdrp >= 1.0 - 1e-12 && shard->width() > 1 && !shard->tab->deterministic_eigen(q->pos, &basis, &sign)) {
        shard->tab->measure(q->pos, 0, [] { return 0; });
        eps_push(0.5);
      }
      return SK_OK;
    }
    if (shard->width() < 2) return SK_OK;
    double sums[4];
    if (given)
      std::copy(given, given + 4, sums);
    else
      SK_TRY(sums_of(q, sums));
    const Bloch r = bloch_from_sums(sums);
    const double e = epsilon(r);
    if (e <= cfg.separability_tol) return try_decompose(shard, q->pos, sums, changed);
    if (cfg.sdrp > 0.0 && e <= cfg.sdrp / 2.0) return round_qubit(shard, q->pos, r, e, sums, changed);
    return SK_OK;
  }

  // ---- gate dispatch (engine.py:514-573) ----------------------------------------
  int apply_ctrl_gate(std::vector<Qubit*> chs, std::vector<int> pol, Qubit* target, const M2& m) {
    if (cfg.control_elimination) {
      std::vector<Qubit*> kc;
      std::vector<int> kp;
      for (size_t i = 0; i < chs.size(); ++i) {
        int z;
        SK_TRY(z_eigenstate(chs[i], &z));
        if (z < 0) {
          kc.push_back(chs[i]);
          kp.push_back(pol[i]);
        } else if (z == pol[i]) {
          stats[SK_ENGINE_STAT_ELIMINATED]++;
        } else {
          return SK_OK;  // this control can never fire
        }
      }
      chs.swap(kc);
      pol.swap(kp);
    }
    if (chs.empty()) return absorb_1q(target, m);
    M2 snapped;
    if (cfg.hx_commutation && snap(m, &snapped)) return buffer_ctrl(chs, pol, target, snapped);
    for (Qubit* c : chs) SK_TRY(flush_pending(c));
    SK_TRY(flush_pending(target));
    return commit_ctrl(chs, pol, target, m);
  }

  int tab_measure(Shard* s, int pos, int* outcome) {  // tableau.py:195-221 with the caller's rng
    if (!bfn) return set_error(SK_EVALUE, "tableau measurement needs the engine rng (sk_engine_set_rng_bits)");
    *outcome = s->tab->measure(pos, -1, [this] { return bfn(bctx); });
    return SK_OK;
  }

  int measure_qubit(int label, int* outcome) {  // engine.py:575-594
    Qubit* h = handles[label];
    SK_TRY(flush_pending(h));
    SK_TRY(commit_1q(h));
    Shard* s = h->shard;
    if (s->stab()) {  // engine.py:580-581
      SK_TRY(tab_measure(s, h->pos, outcome));
      return SK_OK;
    }
    double sums[4];
    SK_TRY(sums_of(h, sums));
    const double p1 = sums[3];
    if (!ufn) return set_error(SK_EVALUE, "circuit contains measurements but the engine has no rng");
    const int out = ufn(uctx) < p1 ? 1 : 0;
    *outcome = out;
    if (s->width() > 1) {
      const double prob = out ? p1 : sums[2];
      if (prob <= 1e-12)
        return set_error(SK_EVALUE, "outcome %d on qubit %d has probability %.3e", out, label, prob);
      sk_state* rest;
      SK_TRY(sk_compact(s->st, h->pos, out, 1.0 / std::sqrt(prob), 0.0, &rest));
      stats[SK_ENGINE_STAT_ALLOCS]++;
      stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << s->width();
      const cd basis[2] = {out ? 0.0 : 1.0, out ? 1.0 : 0.0};
      sk_state* single;
      SumsTicket ss;
      SK_TRY(make_single(basis, &single, &ss));
      SK_TRY(split(s, h->pos, single, ss, rest));
    } else {
      double prob;
      SK_TRY(sk_project(s->st, h->pos, out, &prob));
      stats[SK_ENGINE_STAT_WRITES] += 2;
      s->sums.kind = kSumsNone;
    }
    return SK_OK;
  }

  int apply_gate(int kind, const int32_t* tg, const int32_t* cs, const int32_t* ps, int nc, const double* m8) {
    for (int i = 0; i < (kind == SK_GATE_SWAP ? 2 : 1); ++i)
      if (tg[i] < 0 || tg[i] >= n) return set_error(SK_EINDEX, "qubit %d out of range for %d-qubit simulator", tg[i], n);
    for (int i = 0; i < nc; ++i)
      if (cs[i] < 0 || cs[i] >= n) return set_error(SK_EINDEX, "qubit %d out of range for %d-qubit simulator", cs[i], n);
    if (kind == SK_GATE_MEASURE) {
      int o;
      return measure_qubit(tg[0], &o);
    }
    if (kind == SK_GATE_SWAP) {
      const int a = tg[0], b = tg[1];
      if (cfg.label_swap) {
        std::swap(handles[a], handles[b]);
        stats[SK_ENGINE_STAT_LABEL_SWAPS]++;
        return SK_OK;
      }
      const M2& X = kPauli[0];
      SK_TRY(apply_ctrl_gate({handles[a]}, {1}, handles[b], X));
      SK_TRY(apply_ctrl_gate({handles[b]}, {1}, handles[a], X));
      return apply_ctrl_gate({handles[a]}, {1}, handles[b], X);
    }
    const M2 m = m_from8(m8);
    if (nc == 0) return absorb_1q(handles[tg[0]], m);
    std::vector<Qubit*> chs(nc);
    std::vector<int> pol(nc);
    for (int i = 0; i < nc; ++i) {
      chs[i] = handles[cs[i]];
      pol[i] = ps[i];
    }
    return apply_ctrl_gate(chs, pol, handles[tg[0]], m);
  }

  // ---- flushes (engine.py:669-711) -------------------------------------------------
  int flush_all() {
    std::vector<PendingOp*> ops;
    std::unordered_set<PendingOp*> seen;
    for (Qubit* h : handles)
      for (PendingOp* op : h->pending)
        if (seen.insert(op).second) ops.push_back(op);
    std::sort(ops.begin(), ops.end(), [](PendingOp* a, PendingOp* b) { return a->seq < b->seq; });
    // an op may be committed (and freed) by an earlier op's chain: test
    // liveness through the queues before touching it
    for (size_t i = 0; i < ops.size(); ++i) {
      PendingOp* op = ops[i];
      bool live = false;
      for (Qubit* h : handles)
        if (std::find(h->pending.begin(), h->pending.end(), op) != h->pending.end()) {
          live = true;
          break;
        }
      if (!live) continue;
      if (std::find(op->target->pending.begin(), op->target->pending.end(), op) != op->target->pending.end())
        SK_TRY(commit_chain(op));
    }
    if (cfg.pauli_coalescing) SK_TRY(coalesced_flush());
    for (Qubit* h : handles) SK_TRY(commit_1q(h));
    return SK_OK;
  }

  int coalesced_flush() {
    std::unordered_set<Shard*> seen;
    for (Qubit* h : handles) {
      Shard* s = h->shard;
      if (!seen.insert(s).second || s->stab()) continue;
      if (s->G) {  // the layer's qubits into this rank's slab first
        std::vector<Qubit*> paulis;
        for (Qubit* qb : s->qubits) {
          cd ph;
          if (qb->has_u && as_pauli(qb->u, &ph) >= 0) paulis.push_back(qb);
        }
        for (Qubit* qb : paulis) {
          std::vector<int> busy;
          for (Qubit* o : paulis)
            if (o != qb && o->pos < s->wl()) busy.push_back(o->pos);
          SK_TRY(localize(s, qb->pos, busy));
        }
      }
      uint64_t flip = 0, sign = 0;
      int y = 0, count = 0, first_pos = -1, first_p = -1;
      cd scale = 1.0;
      for (Qubit* qb : s->qubits) {
        if (!qb->has_u) continue;
        cd ph;
        const int p = as_pauli(qb->u, &ph);
        if (p < 0) continue;
        if (count == 0) first_pos = qb->pos, first_p = p;
        ++count;
        if (p == 0) flip |= 1ull << qb->pos;
        if (p == 1) flip |= 1ull << qb->pos, sign |= 1ull << qb->pos, ++y;
        if (p == 2) sign |= 1ull << qb->pos;
        scale *= ph;
        qb->has_u = false;
      }
      if (count >= 2) {
        const cd iy = std::pow(cd(0, 1), y % 4);  // ket.py:188-190: i^#Y belongs to the layer
        const cd exact_iy = (y % 4 == 0) ? cd(1, 0) : (y % 4 == 1) ? cd(0, 1) : (y % 4 == 2) ? cd(-1, 0) : cd(0, -1);
        (void)iy;
        SK_TRY(sk_apply_pauli_layer(s->st, flip, sign, exact_iy.real(), exact_iy.imag()));
        stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << s->width();
        if (std::abs(scale - 1.0) > 1e-15) SK_TRY(sk_scale(s->st, scale.real(), scale.imag()));
        stats[SK_ENGINE_STAT_KERNELS]++;
        s->sums.kind = kSumsNone;
      } else if (count == 1) {
        M2 m = kPauli[first_p];
        for (auto& v : m.a) v *= scale;
        double m8[8];
        m_to8(m, m8);
        SK_TRY(sk_apply_1q(s->st, first_pos, m8));
        stats[SK_ENGINE_STAT_WRITES] += int64_t(1) << s->width();
        stats[SK_ENGINE_STAT_KERNELS]++;
        s->sums.kind = kSumsNone;
      }
    }
    return SK_OK;
  }

  int sdrp_round(int label, double p, double* eps_out) {  // engine.py:490-512
    *eps_out = -1.0;
    Qubit* h = handles[label];
    SK_TRY(flush_pending(h));
    SK_TRY(commit_1q(h));
    Shard* s = h->shard;
    if (s->stab() || s->width() < 2) return set_error(SK_EVALUE, "sdrp_round needs a dense shard of width >= 2");
    double sums[4];
    SK_TRY(sums_of(h, sums));
    const Bloch r = bloch_from_sums(sums);
    const double e = epsilon(r);
    bool changed;
    if (e <= cfg.separability_tol) return try_decompose(s, h->pos, sums, &changed);
    if (e > p / 2.0) return SK_OK;
    const size_t before = eps.size();
    SK_TRY(round_qubit(s, h->pos, r, e, sums, &changed));
    if (eps.size() > before) *eps_out = eps.back();
    return SK_OK;
  }
};

namespace {

int check_engine(const sk_engine* e) {
  if (!e) return set_error(SK_EVALUE, "null engine");
  return SK_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int sk_engine_create(int n, const sk_engine_config* cfg, sk_engine** out) {
  if (n < 1) return set_error(SK_EVALUE, "simulator needs at least 1 qubit");
  if (!cfg) return set_error(SK_EVALUE, "null config");
  if (!(cfg->sdrp >= 0.0 && cfg->sdrp <= 1.0)) return set_error(SK_EVALUE, "sdrp must be in [0, 1]");
  if (cfg->mem_budget < 2) return set_error(SK_EVALUE, "mem_budget must be >= 2");
  if (cfg->dtype != SK_C64 && cfg->dtype != SK_C128) return set_error(SK_EVALUE, "bad dtype %d", cfg->dtype);
  if (cfg->stabilizer_hybrid && n > 64) return set_error(SK_EVALUE, "tableau shards hold at most 64 qubits");
  auto e = std::make_unique<sk_engine>();
  e->n = n;
  e->cfg = *cfg;
  e->own.reserve(n);
  SK_TRY(e->init_ring());
  for (int i = 0; i < n; ++i) {
    e->own.emplace_back(new Qubit());
    e->handles.push_back(e->own.back().get());
    int rc = e->fresh_single(e->own.back().get(), 0);
    if (rc != SK_OK) {
      if (rc == SK_EBUDGET) return rc;
      return rc;
    }
  }
  *out = e.release();
  return SK_OK;
}

int sk_engine_destroy(sk_engine* e) {
  delete e;
  return SK_OK;
}

int sk_engine_set_rng(sk_engine* e, sk_uniform_fn fn, void* ctx) {
  SK_TRY(check_engine(e));
  e->ufn = fn;
  e->uctx = ctx;
  return SK_OK;
}

int sk_engine_apply(sk_engine* e, int ngates, const int32_t* kind, const int32_t* targets, const int32_t* ctrl_off,
                    const int32_t* ctrls, const int32_t* pols, const double* mats, int* done) {
  SK_TRY(check_engine(e));
  *done = 0;
  for (int g = 0; g < ngates; ++g) {
    const int nc = ctrl_off[g + 1] - ctrl_off[g];
    SK_TRY(e->apply_gate(kind[g], targets + 2 * g, ctrls + ctrl_off[g], pols + ctrl_off[g], nc, mats + 8 * g));
    *done = g + 1;
  }
  return SK_OK;
}

int sk_engine_measure(sk_engine* e, int label, int* outcome) {
  SK_TRY(check_engine(e));
  if (label < 0 || label >= e->n) return set_error(SK_EINDEX, "qubit %d out of range", label);
  return e->measure_qubit(label, outcome);
}

int sk_engine_flush_all(sk_engine* e) {
  SK_TRY(check_engine(e));
  return e->flush_all();
}

int sk_engine_flush_qubit(sk_engine* e, int label) {
  SK_TRY(check_engine(e));
  if (label < 0 || label >= e->n) return set_error(SK_EINDEX, "qubit %d out of range", label);
  SK_TRY(e->flush_pending(e->handles[label]));
  return e->commit_1q(e->handles[label]);
}

int sk_engine_sdrp_round(sk_engine* e, int label, double p, double* eps_out) {
  SK_TRY(check_engine(e));
  if (label < 0 || label >= e->n) return set_error(SK_EINDEX, "qubit %d out of range", label);
  return e->sdrp_round(label, p, eps_out);
}

int sk_engine_stats(const sk_engine* e, int64_t out[SK_ENGINE_NSTATS]) {
  SK_TRY(check_engine(e));
  for (int i = 0; i < SK_ENGINE_NSTATS; ++i) out[i] = e->stats[i];
  out[SK_ENGINE_STAT_DENSE_TOTAL] = e->dense_total;
  out[SK_ENGINE_STAT_PEAK] = e->peak;
  out[SK_ENGINE_STAT_NEPS] = (int64_t)e->eps.size();
  out[SK_ENGINE_STAT_NEEDED] = e->needed;
  return SK_OK;
}

int sk_engine_eps(const sk_engine* e, double* out, int64_t cap) {
  SK_TRY(check_engine(e));
  const int64_t k = std::min<int64_t>(cap, (int64_t)e->eps.size());
  std::copy(e->eps.begin(), e->eps.begin() + k, out);
  return SK_OK;
}

int sk_engine_set_distributed(sk_engine* e, int world, int rank, int local_max_width, sk_allreduce_fn allreduce,
                              sk_sendrecv_fn sendrecv, sk_allgather_fn allgather, void* ctx) {
  SK_TRY(check_engine(e));
  int G = 0;
  while ((1 << G) < world) ++G;
  if (world < 1 || (1 << G) != world) return set_error(SK_EVALUE, "world size must be a power of two, got %d", world);
  if (rank < 0 || rank >= world) return set_error(SK_EVALUE, "rank %d outside world %d", rank, world);
  if (world > 1 && (!allreduce || !sendrecv || !allgather)) return set_error(SK_EVALUE, "missing collective callbacks");
  if (local_max_width < G + 2) return set_error(SK_EVALUE, "local_max_width must be >= log2(world) + 2");
  for (Shard* sh : e->shards)
    if (sh->G) return set_error(SK_EVALUE, "set the distribution before any shard is distributed");
  e->world = world;
  e->rank = rank;
  e->Gw = G;
  e->local_max = local_max_width;
  e->f_allreduce = allreduce;
  e->f_sendrecv = sendrecv;
  e->f_allgather = allgather;
  e->dctx = ctx;
  return SK_OK;
}

int sk_engine_set_rng_bits(sk_engine* e, sk_bit_fn fn, void* ctx) {
  SK_TRY(check_engine(e));
  e->bfn = fn;
  e->bctx = ctx;
  return SK_OK;
}

int sk_engine_shards(sk_engine* e, int cap, sk_state** states, int* widths, int* labels, int* owned, int* nshards) {
  SK_TRY(check_engine(e));
  for (Shard* sh : std::vector<Shard*>(e->shards.begin(), e->shards.end())) SK_TRY(e->undistribute(sh, true));
  // shards in order of their lowest label (engine.py _shards_in_label_order);
  // labels[] lists each shard's qubits by position, shard after shard; a
  // tableau shard is handed out as a fresh dense ket (owned[i] = 1, the
  // caller destroys it; engine.py:712-717: wider than 28 qubits is a budget error)
  std::vector<int> lab(e->own.size());
  for (int l = 0; l < e->n; ++l)
    for (size_t i = 0; i < e->own.size(); ++i)
      if (e->own[i].get() == e->handles[l]) lab[i] = l;
  std::vector<Shard*> order;
  for (int l = 0; l < e->n; ++l) {
    Shard* s = e->handles[l]->shard;
    if (std::find(order.begin(), order.end(), s) == order.end()) order.push_back(s);
  }
  if ((int)order.size() > cap) return set_error(SK_EVALUE, "need room for %d shards", (int)order.size());
  int k = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    owned[i] = 0;
    if (order[i]->stab()) {
      if (order[i]->width() > 28) {
        e->needed = int64_t(1) << order[i]->width();
        for (size_t j = 0; j < i; ++j)
          if (owned[j]) sk_destroy(states[j]);
        return set_error(SK_EBUDGET, "needs %lld dense amplitudes", (long long)e->needed);
      }
      sk_state* st;
      SK_TRY(e->replay(*order[i]->tab, &st));
      states[i] = st;
      owned[i] = 1;
    } else {
      states[i] = order[i]->st;
    }
    widths[i] = order[i]->width();
    for (const Qubit* q : order[i]->qubits) {
      for (size_t j = 0; j < e->own.size(); ++j)
        if (e->own[j].get() == q) labels[k] = lab[j];
      ++k;
    }
  }
  *nshards = (int)order.size();
  return SK_OK;
}

int sk_engine_load_state(sk_engine* e, const sk_state* s) {  // engine.py:768-784
  SK_TRY(check_engine(e));
  if (!s || s->width != e->n) return set_error(SK_EVALUE, "state width must equal simulator width %d", e->n);
  std::unordered_set<PendingOp*> ops;
  for (Qubit* h : e->handles) {
    for (PendingOp* op : h->pending) ops.insert(op);
    h->pending.clear();
    h->has_u = false;
  }
  for (PendingOp* op : ops) delete op;
  int64_t total = 0;
  for (Shard* sh : e->shards)
    if (!sh->stab()) total += int64_t(1) << sh->width();  // engine.py:774-777: only dense amplitudes are charged
  SK_TRY(e->release(total));
  SK_TRY(e->charge(int64_t(1) << s->width));
  sk_state* copy;
  if (s->dtype == e->cfg.dtype) {
    SK_TRY(sk_copy(s, &copy));
  } else {
    std::vector<double> host(2 * s->n);
    SK_TRY(sk_download(s, host.data(), s->n));
    SK_TRY(sk_create_from(s->width, e->cfg.dtype, e->cfg.device, host.data(), &copy));
  }
  e->stats[SK_ENGINE_STAT_ALLOCS]++;
  std::vector<Shard*> old(e->shards.begin(), e->shards.end());
  for (Shard* sh : old) e->drop_shard(sh);
  Shard* sh = e->new_shard(copy);
  sh->qubits = e->handles;
  for (int l = 0; l < e->n; ++l) {
    e->handles[l]->shard = sh;
    e->handles[l]->pos = l;
  }
  return SK_OK;
}

int sk_engine_measure_all(sk_engine* e, uint8_t* bits) {  // engine.py:596-626
  SK_TRY(check_engine(e));
  SK_TRY(e->flush_all());
  for (Shard* sh : std::vector<Shard*>(e->shards.begin(), e->shards.end())) SK_TRY(e->undistribute(sh, true));
  std::vector<Shard*> order;
  for (int l = 0; l < e->n; ++l) {
    Shard* s = e->handles[l]->shard;
    if (std::find(order.begin(), order.end(), s) == order.end()) order.push_back(s);
  }
  std::vector<int> outcome_of(e->own.size());
  auto idx_of = [e](const Qubit* q) {
    for (size_t j = 0; j < e->own.size(); ++j)
      if (e->own[j].get() == q) return (int)j;
    return -1;
  };
  for (Shard* s : order) {
    if (s->stab()) {  // the tableau collapses in place
      for (int pos = 0; pos < s->width(); ++pos) {
        int o;
        SK_TRY(e->tab_measure(s, pos, &o));
        outcome_of[idx_of(s->qubits[pos])] = o;
      }
      continue;
    }
    if (!e->ufn) return set_error(SK_EVALUE, "measure_all needs the engine rng");
    const double u = e->ufn(e->uctx);  // == rng.choice(size, p=|a|^2): one uniform
    int64_t idx;
    SK_TRY(sk_sample(s->st, &u, 1, &idx));
    std::vector<Qubit*> members = s->qubits;
    SK_TRY(e->release(int64_t(1) << s->width()));  // before charging the singles
    e->drop_shard(s);
    for (int pos = 0; pos < (int)members.size(); ++pos) {
      const int bit = (int)((idx >> pos) & 1);
      outcome_of[idx_of(members[pos])] = bit;
      SK_TRY(e->fresh_single(members[pos], bit));
    }
  }
  for (int l = 0; l < e->n; ++l) bits[l] = (uint8_t)outcome_of[idx_of(e->handles[l])];
  return SK_OK;
}

int sk_engine_sample(sk_engine* e, int64_t shots, uint8_t* bits) {  // engine.py:628-657, bits[shot * n + label]
  SK_TRY(check_engine(e));
  if (shots < 0) return set_error(SK_EVALUE, "negative shot count");
  SK_TRY(e->flush_all());
  for (Shard* sh : std::vector<Shard*>(e->shards.begin(), e->shards.end())) SK_TRY(e->undistribute(sh, true));
  std::vector<Shard*> order;
  for (int l = 0; l < e->n; ++l) {
    Shard* s = e->handles[l]->shard;
    if (std::find(order.begin(), order.end(), s) == order.end()) order.push_back(s);
  }
  std::vector<int> label_of(e->own.size(), -1);
  for (int l = 0; l < e->n; ++l)
    for (size_t j = 0; j < e->own.size(); ++j)
      if (e->own[j].get() == e->handles[l]) label_of[j] = l;
  auto lab = [&](const Qubit* q) {
    for (size_t j = 0; j < e->own.size(); ++j)
      if (e->own[j].get() == q) return label_of[j];
    return -1;
  };
  for (Shard* s : order) {
    if (s->stab()) {  // a fresh tableau copy per shot, every qubit measured in order
      for (int64_t k = 0; k < shots; ++k) {
        sktab::Tableau t = *s->tab;
        for (int pos = 0; pos < s->width(); ++pos) {
          if (!e->bfn) return set_error(SK_EVALUE, "tableau sampling needs the engine rng");
          bits[k * e->n + lab(s->qubits[pos])] = (uint8_t)t.measure(pos, -1, [e] { return e->bfn(e->bctx); });
        }
      }
      continue;
    }
    if (!e->ufn) return set_error(SK_EVALUE, "sampling needs the engine rng");
    std::vector<double> u(shots);
    for (auto& v : u) v = e->ufn(e->uctx);  // rng.choice(size=shots): shots uniforms in order
    std::vector<int64_t> idx(shots);
    SK_TRY(sk_sample(s->st, u.data(), shots, idx.data()));
    for (int pos = 0; pos < s->width(); ++pos) {
      const int l = lab(s->qubits[pos]);
      for (int64_t k = 0; k < shots; ++k) bits[k * e->n + l] = (uint8_t)((idx[k] >> pos) & 1);
    }
  }
  return SK_OK;
}

}  // extern "C"
