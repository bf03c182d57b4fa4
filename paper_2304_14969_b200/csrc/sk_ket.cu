// sk_ket.cu — per-gate kernels, reductions, splits and composition of the
// dense ket engine, plus the C-ABI entry points that wrap them.
//
// Every kernel is a coalesced grid-stride stream over the 2^w amplitudes
// (or the 2^(w-1) bit-q pairs) with several independent pairs in flight per
// thread; reductions accumulate in fp64 with a warp-shuffle -> block ->
// last-block pass whose order is fixed, so results are deterministic.
// Reference semantics are cited per kernel (paths relative to
// /root/reference/pkg/src/shardsim).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <vector>

#include "sk_internal.cuh"
#include "sk_ops.cuh"

namespace sk {

// ---------------------------------------------------------------------------
// error state
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// ---------------------------------------------------------------------------
// device contexts
// ---------------------------------------------------------------------------
static std::mutex g_ctx_mu;
static DevCtx g_ctx[64];

int ctx_get(int device, DevCtx** out) {
  if (device < 0 || device >= 64) return set_error(SK_EVALUE, "bad device %d", device);
  DevCtx& c = g_ctx[device];
  if (!c.init) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (!c.init) {
      int count = 0;
      if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return set_error(SK_ECUDA, "no CUDA device available (libshardcu has no CPU path)");
      }
      if (device >= count) return set_error(SK_EVALUE, "device %d >= device count %d", device, count);
      SK_CUDA(cudaSetDevice(device));
      c.device = device;
      SK_CUDA(cudaStreamCreateWithFlags(&c.own_stream, cudaStreamNonBlocking));
      c.stream = c.own_stream;
      SK_CUDA(cudaMalloc(&c.d_partials, sizeof(double) * kRedMaxBlocks * kRedMaxK));
      SK_CUDA(cudaHostAlloc(&c.h_map, sizeof(double) * (kRedMaxK + 1), cudaHostAllocMapped));
      SK_CUDA(cudaHostGetDevicePointer((void**)&c.d_map, c.h_map, 0));
      memset(c.h_map, 0, sizeof(double) * (kRedMaxK + 1));
      SK_CUDA(cudaMalloc(&c.d_counter, sizeof(unsigned int)));
      SK_CUDA(cudaMemset(c.d_counter, 0, sizeof(unsigned int)));
      SK_CUDA(cudaMallocHost(&c.h_result, sizeof(double) * kRedMaxK));
      SK_CUDA(cudaDeviceGetAttribute(&c.num_sms, cudaDevAttrMultiProcessorCount, device));
      // keep freed state buffers pooled: engine merges/splits allocate often
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
      c.init = true;
    }
  }
  SK_CUDA(cudaSetDevice(device));
  *out = &c;
  return SK_OK;
}

constexpr int kSmallAmps = 16;

int state_alloc(int width, int dtype, int device, sk_state** out) {
  if (width < 1) return set_error(SK_EVALUE, "shard width must be >= 1");
  if (width > 40) return set_error(SK_EVALUE, "width %d exceeds 40", width);
  if (dtype != SK_C64 && dtype != SK_C128) return set_error(SK_EVALUE, "bad dtype %d", dtype);
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  sk_state* s = new sk_state();
  s->width = width;
  s->dtype = dtype;
  s->device = device;
  s->n = (int64_t)1 << width;
  s->elem = elem_size(dtype);
  const size_t bytes = (size_t)s->n * s->elem;
  // no cudaMemGetInfo guess (the pool may hold reusable memory): the
  // allocation itself is the check, and a failure maps to SK_ENOMEM
  cudaError_t e = cudaMallocAsync(&s->d, bytes, c->stream);
  if (e == cudaErrorMemoryAllocation) {
    // the pool keeps freed buffers (release threshold raised in ctx_get); on a
    // miss, hand them back to the device once and retry before reporting OOM
    cudaGetLastError();
    cudaMemPool_t pool;
    if (cudaStreamSynchronize(c->stream) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess)
      cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(&s->d, bytes, c->stream);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete s;
    return set_error(e == cudaErrorMemoryAllocation ? SK_ENOMEM : SK_ECUDA, "cudaMallocAsync(%zu) for width %d: %s",
                     bytes, width, cudaGetErrorString(e));
  }
  *out = s;
  return SK_OK;
}

template <typename R>
__global__ void k_set_single(vec2_t<R>* d, double ar, double ai, double br, double bi, double* out4,
                             unsigned long long* flag, unsigned long long seq);

int create_single_with_sums(int dtype, int device, const double amps[4], double* d_out4,
                            unsigned long long* d_flag, unsigned long long seq, sk_state** out) {
  sk_state* s;
  SK_TRY(state_alloc(1, dtype, device, &s));
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  if (dtype == SK_C64)
    k_set_single<float><<<1, 1, 0, c->stream>>>((float2*)s->d, amps[0], amps[1], amps[2], amps[3], d_out4, d_flag,
                                                seq);
  else
    k_set_single<double><<<1, 1, 0, c->stream>>>((double2*)s->d, amps[0], amps[1], amps[2], amps[3], d_out4, d_flag,
                                                  seq);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    sk_destroy(s);
    return set_error(SK_ECUDA, "k_set_single: %s", cudaGetErrorString(e));
  }
  *out = s;
  return SK_OK;
}

int wait_mapped(int device, volatile unsigned long long* hflag, unsigned long long seq) {
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  for (long it = 1; *hflag < seq; ++it) {  // sequence words only grow
    if ((it & 4095) == 0) {
      cudaError_t e = cudaStreamQuery(c->stream);
      if (e == cudaSuccess) {
        if (*hflag >= seq) break;
        return set_error(SK_ECUDA, "mapped result %llu never published", seq);
      }
      if (e != cudaErrorNotReady) return set_error(SK_ECUDA, "stream: %s", cudaGetErrorString(e));
      if (it > (1l << 22)) SK_CUDA(cudaStreamSynchronize(c->stream));
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  return SK_OK;
}

// tiny shards (the engine's width-1 qubits, engine.py:187-200) travel as a
// kernel argument: no staging copy and no host wait
struct SmallAmps {
  double v[2 * kSmallAmps];
};

template <typename R>
__global__ void k_set_small(vec2_t<R>* d, int n, const __grid_constant__ SmallAmps a) {
  const int i = threadIdx.x;
  if (i < n) d[i] = mk<R>((R)a.v[2 * i], (R)a.v[2 * i + 1]);
}

RedOut red_out(DevCtx* c) {
  RedOut ro;
  ro.partials = c->d_partials;
  ro.counter = c->d_counter;
  ro.result = c->d_map;
  ro.flag = (unsigned long long*)(c->d_map + kRedMaxK);
  ro.seq = ++c->seq;
  return ro;
}

int red_wait(DevCtx* c, const RedOut& ro, double* out, int k) {
  SK_CHECK_LAUNCH();
  SK_TRY(wait_mapped(c->device, (volatile unsigned long long*)(c->h_map + kRedMaxK), ro.seq));
  for (int i = 0; i < k; ++i) out[i] = ((volatile double*)c->h_map)[i];
  return SK_OK;
}

template <int K>
static int reduce_fetch(DevCtx* c, const RedOut& ro, double* out) {
  return red_wait(c, ro, out, K);
}

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

// a width-1 shard from two host amplitudes, plus its Bloch sums (as k_bloch
// would reduce them from the stored precision) published to mapped host
// memory with a sequence word: the hybrid engine's control elimination
// (engine.py:407-436) then reads them without a device round trip
template <typename R>
__global__ void k_set_single(vec2_t<R>* d, double ar, double ai, double br, double bi, double* out4,
                             unsigned long long* flag, unsigned long long seq) {
  publish_single<R>(d, ar, ai, br, bi, out4, flag, seq);
}

// bloch_vector (ket.py:204-210): sum conj(a0)*a1, sum |a0|^2, sum |a1|^2
template <typename R>
__global__ void __launch_bounds__(kThreads) k_bloch(const vec2_t<R>* __restrict__ a, int64_t npairs, int q,
                                                   RedOut ro) {
  constexpr int U = kUnroll;  // (8 fp32 pairs per iteration measured slower: 0.72 vs 0.52 ms at w = 28)
  double v[4] = {0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  if constexpr (sizeof(R) == 4) {
    if (npairs >= (int64_t(1) << 12)) {
      // c64, large: two neighbouring pairs per 16-byte load (pairs 2k, 2k+1
      // share a float4 in each half; for q = 0 a pair is itself one float4),
      // so each thread keeps twice the bytes in flight per load instruction
      const float4* a4 = reinterpret_cast<const float4*>(a);
      const int64_t nq = npairs >> 1;
      for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < nq; k0 += U * stride) {
        float4 x0[U], x1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = k0 + u * stride;
          if (k < nq) {
            if (q == 0) {
              x0[u] = a4[2 * k];
              x1[u] = a4[2 * k + 1];
            } else {
              const uint64_t i0 = insert0(2 * k, q);
              x0[u] = a4[i0 >> 1];
              x1[u] = a4[(i0 | bit) >> 1];
            }
          } else {
            x0[u] = make_float4(0, 0, 0, 0);
            x1[u] = make_float4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (q == 0) {  // x0 = (a0, a1) of pair 2k, x1 = pair 2k+1
            bloch_acc(v, x0[u].x, x0[u].y, x0[u].z, x0[u].w);
            bloch_acc(v, x1[u].x, x1[u].y, x1[u].z, x1[u].w);
          } else {  // x0 = a0 of pairs 2k, 2k+1; x1 = their a1
            bloch_acc(v, x0[u].x, x0[u].y, x1[u].x, x1[u].y);
            bloch_acc(v, x0[u].z, x0[u].w, x1[u].z, x1[u].w);
          }
        }
      }
      block_reduce_finish<4>(v, ro);
      return;
    }
  }
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < npairs; k0 += U * stride) {
    vec2_t<R> x0[U], x1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t k = k0 + u * stride;
      if (k < npairs) {
        uint64_t i0 = insert0(k, q);
        x0[u] = a[i0];
        x1[u] = a[i0 | bit];
      } else {
        x0[u] = mk<R>(0, 0);
        x1[u] = mk<R>(0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) bloch_acc(v, x0[u].x, x0[u].y, x1[u].x, x1[u].y);
  }
  block_reduce_finish<4>(v, ro);
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_norm2(const vec2_t<R>* __restrict__ a, int64_t n, RedOut ro) {
  double v[1] = {0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += kUnroll * stride) {
    vec2_t<R> x[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t i = i0 + u * stride;
      x[u] = i < n ? a[i] : mk<R>(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) v[0] += (double)x[u].x * x[u].x + (double)x[u].y * x[u].y;
  }
  block_reduce_finish<1>(v, ro);
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_vdot(const vec2_t<R>* __restrict__ a, const vec2_t<R>* __restrict__ b,
                                                  int64_t n, RedOut ro) {
  double v[2] = {0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += kUnroll * stride) {
    vec2_t<R> x[kUnroll], y[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t i = i0 + u * stride;
      x[u] = i < n ? a[i] : mk<R>(0, 0);
      y[u] = i < n ? b[i] : mk<R>(0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      double ar = x[u].x, ai = x[u].y, br = y[u].x, bi = y[u].y;
      v[0] += ar * br + ai * bi;
      v[1] += ar * bi - ai * br;
    }
  }
  block_reduce_finish<2>(v, ro);
}

// ---------------------------------------------------------------------------
// gate kernels
// ---------------------------------------------------------------------------
// DenseKet._apply_1q_unchecked (ket.py:133-144)
template <typename R>
__global__ void __launch_bounds__(kThreads) k_apply_1q(vec2_t<R>* __restrict__ a, int64_t npairs, int q, Mat2<R> m,
                                                      int diag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < npairs; k0 += kUnroll * stride) {
    vec2_t<R> x0[kUnroll], x1[kUnroll];
    uint64_t i0[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t k = k0 + u * stride;
      i0[u] = insert0(k, q);
      if (k < npairs) {
        x0[u] = a[i0[u]];
        x1[u] = a[i0[u] | bit];
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t k = k0 + u * stride;
      if (k < npairs) {
        vec2_t<R> y0, y1;
        if (diag) {
          y0 = cmul<R>(m.m00, x0[u]);
          y1 = cmul<R>(m.m11, x1[u]);
        } else {
          y0 = cmad2<R>(m.m00, x0[u], m.m01, x1[u]);
          y1 = cmad2<R>(m.m10, x0[u], m.m11, x1[u]);
        }
        a[i0[u]] = y0;
        a[i0[u] | bit] = y1;
      }
    }
  }
}

struct CtrlSpec {
  int npos;
  int pos[24];  // sorted positions of controls and target
  uint64_t cval;
};

__device__ __forceinline__ uint64_t insert_zeros(uint64_t k, const CtrlSpec& cs) {
  for (int j = 0; j < cs.npos; ++j) k = insert0(k, cs.pos[j]);
  return k | cs.cval;
}

// DenseKet.apply_controlled (ket.py:146-164) on the control-matching subspace
template <typename R>
__global__ void __launch_bounds__(kThreads) k_apply_ctrl(vec2_t<R>* __restrict__ a, int64_t nitems, CtrlSpec cs,
                                                        int target, Mat2<R> m, int diag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << target;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < nitems; k0 += kUnroll * stride) {
    vec2_t<R> x0[kUnroll], x1[kUnroll];
    uint64_t i0[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t k = k0 + u * stride;
      i0[u] = insert_zeros(k, cs);
      if (k < nitems) {
        x0[u] = a[i0[u]];
        x1[u] = a[i0[u] | bit];
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      int64_t k = k0 + u * stride;
      if (k < nitems) {
        vec2_t<R> y0, y1;
        if (diag) {
          y0 = cmul<R>(m.m00, x0[u]);
          y1 = cmul<R>(m.m11, x1[u]);
        } else {
          y0 = cmad2<R>(m.m00, x0[u], m.m01, x1[u]);
          y1 = cmad2<R>(m.m10, x0[u], m.m11, x1[u]);
        }
        a[i0[u]] = y0;
        a[i0[u] | bit] = y1;
      }
    }
  }
}

// One-control gate fused with the Bloch sums of control and target
// (engine.py:389-394 runs apply_controlled then bloch_vector twice).
template <typename R>
__global__ void __launch_bounds__(kThreads, (sizeof(R) == 8 ? 3 : 4)) k_ctrl_bloch(vec2_t<R>* __restrict__ a, int64_t nquads, int c, int pol,
                                                        int t, Mat2<R> m, RedOut ro) {
  double v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t C = 1ull << c, T = 1ull << t;
  const int lo = c < t ? c : t, hi = c < t ? t : c;
  // c128: two quads per iteration, both loaded before either is written (8
  // loads in flight per thread; measured 0.83 -> 0.80 ms at w = 27); the sums
  // still accumulate quad by quad in k order.  c64 keeps one quad (faster).
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; sizeof(R) == 8 && k + stride < nquads; k += 2 * stride) {
    const uint64_t b0 = insert0(insert0(k, lo), hi), b1 = insert0(insert0(k + stride, lo), hi);
    vec2_t<R> x0[2][2], x1[2][2];
    ctrl_bloch_load<R>(a, b0, C, T, x0);
    ctrl_bloch_load<R>(a, b1, C, T, x1);
    ctrl_bloch_apply<R>(a, b0, C, T, pol, m, x0, v);
    ctrl_bloch_apply<R>(a, b1, C, T, pol, m, x1, v);
  }
  for (; k < nquads; k += stride) ctrl_bloch_quad<R>(a, insert0(insert0(k, lo), hi), C, T, pol, m, v);
  block_reduce_finish<8>(v, ro);
}

// apply_pauli_layer (ket.py:166-202), in place (the reference gathers out of
// place; pairing j with j^flip makes each pair one thread's job)
template <typename R>
__global__ void __launch_bounds__(kThreads) k_pauli(vec2_t<R>* __restrict__ a, int64_t nitems, int fbit, uint64_t flip,
                                                   uint64_t sign, vec2_t<R> scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (sizeof(R) == 8 && flip != 0) {  // c128: two pairs per iteration, loaded before either is written
    for (; k0 + stride < nitems; k0 += 2 * stride) {
      const uint64_t j0 = insert0(k0, fbit), j1 = insert0(k0 + stride, fbit);
      const vec2_t<R> x0 = a[j0], y0 = a[j0 ^ flip], x1 = a[j1], y1 = a[j1 ^ flip];
      const vec2_t<R> nscale = mk<R>(-scale.x, -scale.y);
      a[j0 ^ flip] = cmul<R>(x0, (__popcll(j0 & sign) & 1) ? nscale : scale);
      a[j0] = cmul<R>(y0, (__popcll((j0 ^ flip) & sign) & 1) ? nscale : scale);
      a[j1 ^ flip] = cmul<R>(x1, (__popcll(j1 & sign) & 1) ? nscale : scale);
      a[j1] = cmul<R>(y1, (__popcll((j1 ^ flip) & sign) & 1) ? nscale : scale);
    }
  }
  for (int64_t k = k0; k < nitems; k += stride) {
    if (flip == 0) {
      vec2_t<R> x = a[k];
      vec2_t<R> f = (__popcll(k & sign) & 1) ? mk<R>(-scale.x, -scale.y) : scale;
      a[k] = cmul<R>(x, f);
    } else {
      uint64_t j = insert0(k, fbit);
      uint64_t j2 = j ^ flip;
      vec2_t<R> xj = a[j], xj2 = a[j2];
      vec2_t<R> fj = (__popcll(j & sign) & 1) ? mk<R>(-scale.x, -scale.y) : scale;
      vec2_t<R> fj2 = (__popcll(j2 & sign) & 1) ? mk<R>(-scale.x, -scale.y) : scale;
      a[j2] = cmul<R>(xj, fj);
      a[j] = cmul<R>(xj2, fj2);
    }
  }
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_scale(vec2_t<R>* __restrict__ a, int64_t n, vec2_t<R> z) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = cmul<R>(a[i], z);
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_swap(vec2_t<R>* __restrict__ a, int64_t nitems, int lo, int hi) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nitems; k += stride) {
    uint64_t b = insert0(insert0(k, lo), hi);
    uint64_t i1 = b | (1ull << lo), i2 = b | (1ull << hi);
    vec2_t<R> x = a[i1];
    a[i1] = a[i2];
    a[i2] = x;
  }
}

// project_and_renormalize (ket.py:212-226) after the probability check
template <typename R>
__global__ void __launch_bounds__(kThreads) k_project(vec2_t<R>* __restrict__ a, int64_t npairs, int q, int outcome,
                                                     R scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < npairs; k += stride) {
    uint64_t i0 = insert0(k, q);
    uint64_t keep = outcome ? (i0 | bit) : i0, drop = outcome ? i0 : (i0 | bit);
    vec2_t<R> x = a[keep];
    a[keep] = mk<R>(x.x * scale, x.y * scale);
    a[drop] = mk<R>(0, 0);
  }
}

// remove_qubit / try_decompose remainder / measurement split: compaction
template <typename R>
__global__ void __launch_bounds__(kThreads) k_compact(const vec2_t<R>* __restrict__ a, vec2_t<R>* __restrict__ out,
                                                     int64_t nout, int q, int half, vec2_t<R> z) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t hb = half ? (1ull << q) : 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nout; k += stride)
    out[k] = cmul<R>(a[insert0(k, q) | hb], z);
}

// fused SDRP rotate-project-compact (engine.py:464-488)
template <typename R>
__global__ void __launch_bounds__(kThreads) k_round(const vec2_t<R>* __restrict__ a, vec2_t<R>* __restrict__ out,
                                                   int64_t nout, int q, vec2_t<R> u00, vec2_t<R> u01, R scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t bit = 1ull << q;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nout; k += stride) {
    uint64_t i0 = insert0(k, q);
    vec2_t<R> y = cmad2<R>(u00, a[i0], u01, a[i0 | bit]);
    out[k] = mk<R>(y.x * scale, y.y * scale);
  }
}

// kron_compose (ket.py:239-241)
template <typename R>
__global__ void __launch_bounds__(kThreads) k_kron(const vec2_t<R>* __restrict__ lo, const vec2_t<R>* __restrict__ hi,
                                                  vec2_t<R>* __restrict__ out, int64_t n, int wa) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint64_t mask = (1ull << wa) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = cmul<R>(hi[(uint64_t)i >> wa], lo[(uint64_t)i & mask]);
}

// kron_compose with a narrow high factor (<= 16 amplitudes): each thread reads
// lo[i] once and writes all 2^wb products (the generic form re-reads the whole
// low factor 2^wb times once it exceeds L2); same elementwise arithmetic
template <typename R>
__global__ void __launch_bounds__(kThreads) k_kron_narrow(const vec2_t<R>* __restrict__ lo,
                                                         const vec2_t<R>* __restrict__ hi, vec2_t<R>* __restrict__ out,
                                                         int64_t nlo, int wa, int nhi) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nlo; i += stride) {
    const vec2_t<R> x = lo[i];
    for (int j = 0; j < nhi; ++j) out[((uint64_t)j << wa) | (uint64_t)i] = cmul<R>(__ldg(hi + j), x);
  }
}

struct PermSpec {
  int w;
  int order[40];
};

// permute_qubits (ket.py:284-292): new qubit k is old qubit order[k]
template <typename R>
__global__ void __launch_bounds__(kThreads) k_permute(const vec2_t<R>* __restrict__ a, vec2_t<R>* __restrict__ out,
                                                     int64_t n, PermSpec ps) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t old = 0;
    for (int k = 0; k < ps.w; ++k) old |= (((uint64_t)i >> k) & 1ull) << ps.order[k];
    out[i] = a[old];
  }
}

// permute_qubits as a tiled transpose.  The tile is the set of output bits
// {0..K-1} (output-contiguous) united with the output positions of input bits
// {0..K-1} (input-contiguous), at most 2K bits: the block reads it with input
// low bits fastest (coalesced), parks it in shared memory and writes it with
// output low bits fastest (coalesced).  Both tile-index maps are linear over
// GF(2), so per-thread parts are combined with XOR.
template <int SB>
__device__ __forceinline__ uint32_t swz(uint32_t l) {  // fold the high bits into the low SB (GF(2)-linear)
  uint32_t h = l >> SB;
  uint32_t f = h ^ (h >> SB) ^ (h >> (2 * SB)) ^ (h >> (3 * SB));
  return l ^ (f & ((1u << SB) - 1));
}

constexpr int kPermK = 5;
constexpr int kPermMaxT = 2 * kPermK + 1;  // tile bits: 10 (c128, 4 elements per thread) or 11 (c64, 8)

struct PermTile {
  int w, nrest;
  uint64_t in_of_bit[kPermMaxT];   // bit t of the input-ordered tile index -> input index bit (1 << pos)
  uint32_t rm[kPermMaxT];          // bit t of the input-ordered tile index -> output-ordered tile bit
  uint64_t out_of_bit[kPermMaxT];  // bit t of the output-ordered tile index -> output index bit
  uint8_t rest_out[40];            // block index bit j -> output bit position
  uint8_t rest_in[40];             // block index bit j -> input bit position
};

constexpr int kPermThreads = 256;

// tile = 2^(8 + EB) elements: EB = 2 (c128) or 3 (c64), i.e. 64 bytes per
// thread either way
template <typename R>
constexpr int perm_eb() { return sizeof(R) == 4 ? 3 : 2; }

template <typename R>
__global__ void __launch_bounds__(kPermThreads) k_permute_tiled(const vec2_t<R>* __restrict__ a,
                                                               vec2_t<R>* __restrict__ out,
                                                               const __grid_constant__ PermTile pt) {
  using V = vec2_t<R>;
  constexpr int EB = perm_eb<R>(), E = 1 << EB;
  __shared__ V sm[kPermThreads * E];
  constexpr int SB = sizeof(V) == 8 ? 4 : 3;  // elements per 128-byte row: the swizzle fold width
  // block base: lane j deposits block-index bit j, a warp OR-reduction combines them
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  uint64_t bin = 0, bout = 0;
  for (int j = lane; j < pt.nrest; j += 32) {
    const uint64_t bit = (blockIdx.x >> j) & 1u;
    bin |= bit << pt.rest_in[j];
    bout |= bit << pt.rest_out[j];
  }
  bin = ((uint64_t)__reduce_or_sync(0xffffffffu, (uint32_t)(bin >> 32)) << 32) |
        __reduce_or_sync(0xffffffffu, (uint32_t)bin);
  bout = ((uint64_t)__reduce_or_sync(0xffffffffu, (uint32_t)(bout >> 32)) << 32) |
         __reduce_or_sync(0xffffffffu, (uint32_t)bout);
  uint64_t in_t = bin, out_t = bout;  // the thread's part (tile bits 0..7), linear over GF(2)
  uint32_t mo_t = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if ((tid >> t) & 1u) {
      in_t |= pt.in_of_bit[t];
      mo_t |= pt.rm[t];
      out_t |= pt.out_of_bit[t];
    }
  V r[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {  // input order: each warp reads 32 consecutive input amplitudes
    uint64_t in = in_t;
#pragma unroll
    for (int b = 0; b < EB; ++b)
      if ((e >> b) & 1) in |= pt.in_of_bit[8 + b];
    r[e] = a[in];
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    uint32_t mo = mo_t;
#pragma unroll
    for (int b = 0; b < EB; ++b)
      if ((e >> b) & 1) mo ^= pt.rm[8 + b];
    sm[swz<SB>(mo)] = r[e];
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) {  // output order: each warp writes 32 consecutive output amplitudes
    const uint32_t m = tid | ((uint32_t)e << 8);
    uint64_t o = out_t;
#pragma unroll
    for (int b = 0; b < EB; ++b)
      if ((e >> b) & 1) o |= pt.out_of_bit[8 + b];
    out[o] = sm[swz<SB>(m)];
  }
}

template <typename R>
__global__ void k_set_basis0(vec2_t<R>* a) {
  a[0] = mk<R>(1, 0);
}

// float <-> double conversion for uploads/downloads of c64 states
__global__ void k_d2f(const double2* __restrict__ src, float2* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = make_float2((float)src[i].x, (float)src[i].y);
}
__global__ void k_f2d(const float2* __restrict__ src, double2* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = make_double2((double)src[i].x, (double)src[i].y);
}

// ---- sampling: per-chunk sums then per-sample in-chunk warp scan ----------
constexpr int kChunkBits = 10;

template <typename R>
__global__ void __launch_bounds__(kThreads) k_chunk_sums(const vec2_t<R>* __restrict__ a, int64_t nchunks,
                                                        int chunk, double* __restrict__ sums) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t ch = warp; ch < nchunks; ch += nwarps) {
    double acc = 0;
    const vec2_t<R>* p = a + ch * chunk;
    for (int i = lane; i < chunk; i += 32) {
      vec2_t<R> x = p[i];
      acc += (double)x.x * x.x + (double)x.y * x.y;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, off);
    if (lane == 0) sums[ch] = acc;
  }
}

template <typename R>
__global__ void __launch_bounds__(kThreads) k_sample_resolve(const vec2_t<R>* __restrict__ a, int chunk,
                                                            const int64_t* __restrict__ chunk_of,
                                                            const double* __restrict__ resid, int64_t k,
                                                            int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s = warp; s < k; s += nwarps) {
    const int64_t ch = chunk_of[s];
    const double r = resid[s];
    const vec2_t<R>* p = a + ch * chunk;
    double run = 0;
    int64_t found = -1, last_nz = -1;
    for (int base = 0; base < chunk && found < 0; base += 32) {
      double w = 0.0;
      if (base + lane < chunk) {
        vec2_t<R> x = p[base + lane];
        w = (double)x.x * x.x + (double)x.y * x.y;
      }
      double incl = w;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        double y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
      }
      unsigned hit = __ballot_sync(0xffffffffu, run + incl > r && w > 0);
      unsigned nz = __ballot_sync(0xffffffffu, w > 0);
      if (nz) last_nz = base + 31 - __clz(nz);
      if (hit) found = base + __ffs(hit) - 1;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (found < 0) found = last_nz >= 0 ? last_nz : chunk - 1;  // rounding at the chunk end
    if (lane == 0) out[s] = ch * chunk + found;
  }
}

// ---------------------------------------------------------------------------
// dispatch helpers
// ---------------------------------------------------------------------------
template <typename F>
static int dispatch(const sk_state* s, F&& f) {
  if (s->dtype == SK_C64) return f(float());
  return f(double());
}

static int check_state(const sk_state* s) {
  if (!s) return set_error(SK_EVALUE, "null state");
  return SK_OK;
}

static int check_qubit(const sk_state* s, int q) {
  if (q < 0 || q >= s->width) return set_error(SK_EINDEX, "qubit %d out of range for width %d", q, s->width);
  return SK_OK;
}

// pageable complex128 host <-> device state transfers (sk_io.cu)
int staged_upload(DevCtx* c, sk_state* s, const double* host, int64_t n);
int staged_download(DevCtx* c, const sk_state* s, double* host, int64_t n);
constexpr int64_t kStagedMin = int64_t(1) << 18;

}  // namespace sk

using namespace sk;

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* sk_last_error(void) { return g_err.c_str(); }
int sk_version(void) { return 1; }

int sk_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int sk_set_stream(int device, uint64_t stream) {
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  c->stream = stream == SK_OWN_STREAM ? c->own_stream : (cudaStream_t)stream;
  return SK_OK;
}

int sk_get_stream(int device, uint64_t* stream) {
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  *stream = (uint64_t)c->stream;
  return SK_OK;
}

int sk_synchronize(int device) {
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  SK_CUDA(cudaStreamSynchronize(c->stream));
  return SK_OK;
}

int sk_mem_info(int device, uint64_t* free_bytes, uint64_t* total_bytes) {
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  size_t f = 0, t = 0;
  SK_CUDA(cudaMemGetInfo(&f, &t));
  *free_bytes = f;
  *total_bytes = t;
  return SK_OK;
}

int sk_create(int width, int dtype, int device, sk_state** out) {
  sk_state* s;
  SK_TRY(state_alloc(width, dtype, device, &s));
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  SK_CUDA(cudaMemsetAsync(s->d, 0, (size_t)s->n * s->elem, c->stream));
  if (dtype == SK_C64)
    k_set_basis0<float><<<1, 1, 0, c->stream>>>((float2*)s->d);
  else
    k_set_basis0<double><<<1, 1, 0, c->stream>>>((double2*)s->d);
  SK_CHECK_LAUNCH();
  *out = s;
  return SK_OK;
}

int sk_destroy(sk_state* s) {
  if (!s) return SK_OK;
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  if (s->d && s->owned) SK_CUDA(cudaFreeAsync(s->d, c->stream));
  delete s;
  return SK_OK;
}

int sk_wrap(int width, int dtype, int device, uint64_t ptr, sk_state** out) {
  if (width < 1 || width > 40) return set_error(SK_EVALUE, "bad width %d", width);
  if (dtype != SK_C64 && dtype != SK_C128) return set_error(SK_EVALUE, "bad dtype %d", dtype);
  if (!ptr || (ptr & 15)) return set_error(SK_EVALUE, "wrapped buffer must be non-null and 16-byte aligned");
  DevCtx* c;
  SK_TRY(ctx_get(device, &c));
  sk_state* s = new sk_state();
  s->d = (void*)ptr;
  s->width = width;
  s->dtype = dtype;
  s->device = device;
  s->n = (int64_t)1 << width;
  s->elem = elem_size(dtype);
  s->owned = false;
  *out = s;
  return SK_OK;
}

int sk_rebind(sk_state* s, uint64_t ptr) {
  SK_TRY(check_state(s));
  if (s->owned) return set_error(SK_EVALUE, "only sk_wrap views can be rebound");
  if (!ptr || (ptr & 15)) return set_error(SK_EVALUE, "wrapped buffer must be non-null and 16-byte aligned");
  s->d = (void*)ptr;
  return SK_OK;
}

int sk_width(const sk_state* s, int* width) {
  SK_TRY(check_state(s));
  *width = s->width;
  return SK_OK;
}

int sk_dtype(const sk_state* s, int* dtype) {
  SK_TRY(check_state(s));
  *dtype = s->dtype;
  return SK_OK;
}

int sk_device_ptr(const sk_state* s, uint64_t* ptr) {
  SK_TRY(check_state(s));
  *ptr = (uint64_t)s->d;
  return SK_OK;
}

int sk_upload(sk_state* s, const double* host, int64_t n) {
  SK_TRY(check_state(s));
  if (n != s->n) return set_error(SK_EVALUE, "need %lld amplitudes, got %lld", (long long)s->n, (long long)n);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  if (n >= kStagedMin) return staged_upload(c, s, host, n);  // sk_io.cu: pinned chunks, parallel host pass
  if (s->dtype == SK_C128) {
    SK_CUDA(cudaMemcpyAsync(s->d, host, (size_t)n * 16, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(cudaStreamSynchronize(c->stream));
    return SK_OK;
  }
  // c64: stage through a bounded device buffer and narrow on the device
  const int64_t chunk = std::min<int64_t>(n, int64_t(1) << 24);
  double2* stage = nullptr;
  SK_CUDA(cudaMallocAsync(&stage, (size_t)chunk * 16, c->stream));
  for (int64_t off = 0; off < n; off += chunk) {
    int64_t m = std::min(chunk, n - off);
    SK_CUDA(cudaMemcpyAsync(stage, host + 2 * off, (size_t)m * 16, cudaMemcpyHostToDevice, c->stream));
    k_d2f<<<grid_for(m, kThreads, 4, c->num_sms), kThreads, 0, c->stream>>>(stage, (float2*)s->d + off, m);
    SK_CHECK_LAUNCH();
  }
  SK_CUDA(cudaFreeAsync(stage, c->stream));
  SK_CUDA(cudaStreamSynchronize(c->stream));
  return SK_OK;
}

int sk_download(const sk_state* s, double* host, int64_t n) {
  SK_TRY(check_state(s));
  if (n != s->n) return set_error(SK_EVALUE, "need %lld amplitudes, got %lld", (long long)s->n, (long long)n);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  if (n >= kStagedMin) {
    SK_CUDA(cudaStreamSynchronize(c->stream));  // the state's pending kernels
    return staged_download(c, s, host, n);
  }
  if (s->dtype == SK_C128) {
    SK_CUDA(cudaMemcpyAsync(host, s->d, (size_t)n * 16, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(cudaStreamSynchronize(c->stream));
    return SK_OK;
  }
  const int64_t chunk = std::min<int64_t>(n, int64_t(1) << 24);
  double2* stage = nullptr;
  SK_CUDA(cudaMallocAsync(&stage, (size_t)chunk * 16, c->stream));
  for (int64_t off = 0; off < n; off += chunk) {
    int64_t m = std::min(chunk, n - off);
    k_f2d<<<grid_for(m, kThreads, 4, c->num_sms), kThreads, 0, c->stream>>>((const float2*)s->d + off, stage, m);
    SK_CHECK_LAUNCH();
    SK_CUDA(cudaMemcpyAsync(host + 2 * off, stage, (size_t)m * 16, cudaMemcpyDeviceToHost, c->stream));
  }
  SK_CUDA(cudaFreeAsync(stage, c->stream));
  SK_CUDA(cudaStreamSynchronize(c->stream));
  return SK_OK;
}

int sk_upload_native(sk_state* s, const void* host, int64_t n) {
  SK_TRY(check_state(s));
  if (n != s->n) return set_error(SK_EVALUE, "need %lld amplitudes, got %lld", (long long)s->n, (long long)n);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  SK_CUDA(cudaMemcpyAsync(s->d, host, (size_t)n * s->elem, cudaMemcpyHostToDevice, c->stream));
  return SK_OK;
}

int sk_download_native(const sk_state* s, void* host, int64_t n) {
  SK_TRY(check_state(s));
  if (n != s->n) return set_error(SK_EVALUE, "need %lld amplitudes, got %lld", (long long)s->n, (long long)n);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  SK_CUDA(cudaMemcpyAsync(host, s->d, (size_t)n * s->elem, cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(cudaStreamSynchronize(c->stream));
  return SK_OK;
}

int sk_download_native_async(const sk_state* s, void* host, int64_t n) {
  SK_TRY(check_state(s));
  if (n != s->n) return set_error(SK_EVALUE, "need %lld amplitudes, got %lld", (long long)s->n, (long long)n);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  SK_CUDA(cudaMemcpyAsync(host, s->d, (size_t)n * s->elem, cudaMemcpyDeviceToHost, c->stream));
  return SK_OK;
}

int sk_copy_from_device(sk_state* s, uint64_t src, int64_t n) {
  SK_TRY(check_state(s));
  if (n != s->n) return set_error(SK_EVALUE, "need %lld amplitudes, got %lld", (long long)s->n, (long long)n);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  SK_CUDA(cudaMemcpyAsync(s->d, (const void*)src, (size_t)n * s->elem, cudaMemcpyDeviceToDevice, c->stream));
  return SK_OK;
}

int sk_copy_to_device(const sk_state* s, uint64_t dst, int64_t n) {
  SK_TRY(check_state(s));
  if (n != s->n) return set_error(SK_EVALUE, "need %lld amplitudes, got %lld", (long long)s->n, (long long)n);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  SK_CUDA(cudaMemcpyAsync((void*)dst, s->d, (size_t)n * s->elem, cudaMemcpyDeviceToDevice, c->stream));
  return SK_OK;
}

int sk_create_from(int width, int dtype, int device, const double* host, sk_state** out) {
  sk_state* s;
  SK_TRY(state_alloc(width, dtype, device, &s));
  if (s->n <= kSmallAmps) {
    sk::SmallAmps a{};
    for (int64_t i = 0; i < 2 * s->n; ++i) a.v[i] = host[i];
    DevCtx* c;
    SK_TRY(ctx_get(device, &c));
    if (dtype == SK_C64)
      sk::k_set_small<float><<<1, kSmallAmps, 0, c->stream>>>((float2*)s->d, (int)s->n, a);
    else
      sk::k_set_small<double><<<1, kSmallAmps, 0, c->stream>>>((double2*)s->d, (int)s->n, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      sk_destroy(s);
      return set_error(SK_ECUDA, "k_set_small: %s", cudaGetErrorString(e));
    }
    *out = s;
    return SK_OK;
  }
  int rc = sk_upload(s, host, s->n);
  if (rc != SK_OK) {
    std::string keep = g_err;
    sk_destroy(s);
    g_err = keep;
    return rc;
  }
  *out = s;
  return SK_OK;
}

int sk_copy(const sk_state* src, sk_state** out) {
  SK_TRY(check_state(src));
  sk_state* s;
  SK_TRY(state_alloc(src->width, src->dtype, src->device, &s));
  DevCtx* c;
  SK_TRY(ctx_get(src->device, &c));
  SK_CUDA(cudaMemcpyAsync(s->d, src->d, (size_t)s->n * s->elem, cudaMemcpyDeviceToDevice, c->stream));
  *out = s;
  return SK_OK;
}

int sk_apply_1q(sk_state* s, int q, const double m[8]) {
  SK_TRY(check_state(s));
  SK_TRY(check_qubit(s, q));
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int diag = (m[2] == 0.0 && m[3] == 0.0 && m[4] == 0.0 && m[5] == 0.0);  // ket.py:136
  const int64_t np_ = s->n / 2;
  const int g = grid_for(np_, kThreads, kUnroll, c->num_sms);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_apply_1q<R><<<g, kThreads, 0, c->stream>>>((vec2_t<R>*)s->d, np_, q, mat_from<R>(m), diag);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
}

int sk_apply_controlled(sk_state* s, uint64_t ctrl_mask, uint64_t ctrl_val, int target, const double m[8]) {
  SK_TRY(check_state(s));
  SK_TRY(check_qubit(s, target));
  if ((ctrl_mask >> target) & 1ull) return set_error(SK_EVALUE, "target %d is also a control", target);
  if (s->width < 64 && (ctrl_mask >> s->width)) return set_error(SK_EINDEX, "control out of range for width %d", s->width);
  if (ctrl_val & ~ctrl_mask) return set_error(SK_EVALUE, "ctrl_val has bits outside ctrl_mask");
  CtrlSpec cs{};
  cs.npos = 0;
  for (int b = 0; b < 64; ++b)
    if (((ctrl_mask >> b) & 1ull) || b == target) {
      if (cs.npos >= 24) return set_error(SK_EVALUE, "too many controls");
      cs.pos[cs.npos++] = b;
    }
  cs.cval = ctrl_val;
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int diag = (m[2] == 0.0 && m[3] == 0.0 && m[4] == 0.0 && m[5] == 0.0);  // ket.py:153
  const int64_t items = s->n >> cs.npos;
  const int g = grid_for(items, kThreads, kUnroll, c->num_sms);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_apply_ctrl<R><<<g, kThreads, 0, c->stream>>>((vec2_t<R>*)s->d, items, cs, target, mat_from<R>(m), diag);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
}

int sk_apply_controlled_bloch(sk_state* s, int control, int polarity, int target, const double m[8],
                              double out8[8]) {
  SK_TRY(check_state(s));
  SK_TRY(check_qubit(s, control));
  SK_TRY(check_qubit(s, target));
  if (control == target) return set_error(SK_EVALUE, "overlapping qubit indices (%d, %d)", control, target);
  if (polarity != 0 && polarity != 1) return set_error(SK_EVALUE, "polarity must be 0 or 1");
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int64_t nq = s->n / 4;
  const int g = grid_for(nq, kThreads, 2, c->num_sms);
  std::lock_guard<std::mutex> lk(c->red_mu);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    const RedOut ro = red_out(c);
    k_ctrl_bloch<R><<<g, kThreads, 0, c->stream>>>((vec2_t<R>*)s->d, nq, control, polarity, target, mat_from<R>(m),
                                                   ro);
    return reduce_fetch<8>(c, ro, out8);
  });
}

int sk_apply_pauli_layer(sk_state* s, uint64_t flip, uint64_t sign, double sre, double sim) {
  SK_TRY(check_state(s));
  if (s->width < 64 && ((flip | sign) >> s->width)) return set_error(SK_EINDEX, "pauli qubit out of range");
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  int fbit = flip ? __builtin_ctzll(flip) : 0;
  const int64_t items = flip ? s->n / 2 : s->n;
  const int g = grid_for(items, kThreads, 2, c->num_sms);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_pauli<R><<<g, kThreads, 0, c->stream>>>((vec2_t<R>*)s->d, items, fbit, flip, sign, mk<R>((R)sre, (R)sim));
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
}

int sk_scale(sk_state* s, double re, double im) {
  SK_TRY(check_state(s));
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int g = grid_for(s->n, kThreads, 2, c->num_sms);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_scale<R><<<g, kThreads, 0, c->stream>>>((vec2_t<R>*)s->d, s->n, mk<R>((R)re, (R)im));
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
}

int sk_swap_qubits(sk_state* s, int a, int b) {
  SK_TRY(check_state(s));
  SK_TRY(check_qubit(s, a));
  SK_TRY(check_qubit(s, b));
  if (a == b) return SK_OK;
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int lo = std::min(a, b), hi = std::max(a, b);
  const int64_t items = s->n / 4;
  const int g = grid_for(items, kThreads, 2, c->num_sms);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_swap<R><<<g, kThreads, 0, c->stream>>>((vec2_t<R>*)s->d, items, lo, hi);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
}

int sk_bloch_sums(const sk_state* s, int q, double out4[4]) {
  SK_TRY(check_state(s));
  SK_TRY(check_qubit(s, q));
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int64_t np_ = s->n / 2;
  const int g = grid_for(np_, kThreads, kUnroll, c->num_sms);
  std::lock_guard<std::mutex> lk(c->red_mu);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    const RedOut ro = red_out(c);
    k_bloch<R><<<g, kThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, np_, q, ro);
    return reduce_fetch<4>(c, ro, out4);
  });
}

int sk_norm2(const sk_state* s, double* out) {
  SK_TRY(check_state(s));
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int g = grid_for(s->n, kThreads, kUnroll, c->num_sms);
  std::lock_guard<std::mutex> lk(c->red_mu);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    const RedOut ro = red_out(c);
    k_norm2<R><<<g, kThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, s->n, ro);
    return reduce_fetch<1>(c, ro, out);
  });
}

int sk_vdot(const sk_state* a, const sk_state* b, double out2[2]) {
  SK_TRY(check_state(a));
  SK_TRY(check_state(b));
  if (a->width != b->width) return set_error(SK_EVALUE, "width mismatch: %d vs %d", a->width, b->width);
  if (a->dtype != b->dtype) return set_error(SK_EVALUE, "dtype mismatch");
  if (a->device != b->device) return set_error(SK_EVALUE, "device mismatch");
  DevCtx* c;
  SK_TRY(ctx_get(a->device, &c));
  const int g = grid_for(a->n, kThreads, kUnroll, c->num_sms);
  std::lock_guard<std::mutex> lk(c->red_mu);
  return dispatch(a, [&](auto r) {
    using R = decltype(r);
    const RedOut ro = red_out(c);
    k_vdot<R><<<g, kThreads, 0, c->stream>>>((const vec2_t<R>*)a->d, (const vec2_t<R>*)b->d, a->n, ro);
    return reduce_fetch<2>(c, ro, out2);
  });
}

int sk_amplitude(const sk_state* s, int64_t index, double out2[2]) {
  SK_TRY(check_state(s));
  if (index < 0 || index >= s->n) return set_error(SK_EINDEX, "index %lld out of range", (long long)index);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  if (s->dtype == SK_C128) {
    SK_CUDA(cudaMemcpyAsync(c->h_result, (const double2*)s->d + index, 16, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(cudaStreamSynchronize(c->stream));
    out2[0] = c->h_result[0];
    out2[1] = c->h_result[1];
  } else {
    SK_CUDA(cudaMemcpyAsync(c->h_result, (const float2*)s->d + index, 8, cudaMemcpyDeviceToHost, c->stream));
    SK_CUDA(cudaStreamSynchronize(c->stream));
    float f[2];
    memcpy(f, c->h_result, 8);
    out2[0] = f[0];
    out2[1] = f[1];
  }
  return SK_OK;
}

int sk_project(sk_state* s, int q, int outcome, double* prob) {
  SK_TRY(check_state(s));
  if (outcome != 0 && outcome != 1) return set_error(SK_EVALUE, "outcome must be 0 or 1, got %d", outcome);
  double sums[4];
  SK_TRY(sk_bloch_sums(s, q, sums));
  const double p = outcome ? sums[3] : sums[2];
  *prob = p;
  if (p <= 1e-12) return set_error(SK_EVALUE, "outcome %d on qubit %d has probability %.3e", outcome, q, p);
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const double scale = 1.0 / std::sqrt(p);
  const int64_t np_ = s->n / 2;
  const int g = grid_for(np_, kThreads, 2, c->num_sms);
  return dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_project<R><<<g, kThreads, 0, c->stream>>>((vec2_t<R>*)s->d, np_, q, outcome, (R)scale);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
}

int sk_compact(const sk_state* s, int q, int half, double re, double im, sk_state** out) {
  SK_TRY(check_state(s));
  SK_TRY(check_qubit(s, q));
  if (s->width < 2) return set_error(SK_EVALUE, "cannot remove the last qubit of a shard");
  if (half != 0 && half != 1) return set_error(SK_EVALUE, "half must be 0 or 1");
  sk_state* o;
  SK_TRY(state_alloc(s->width - 1, s->dtype, s->device, &o));
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int g = grid_for(o->n, kThreads, 2, c->num_sms);
  int rc = dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_compact<R><<<g, kThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, (vec2_t<R>*)o->d, o->n, q, half,
                                                mk<R>((R)re, (R)im));
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
  if (rc != SK_OK) {
    sk_destroy(o);
    return rc;
  }
  *out = o;
  return SK_OK;
}

int sk_round_compact(const sk_state* s, int q, const double u0[4], double scale, sk_state** out) {
  SK_TRY(check_state(s));
  SK_TRY(check_qubit(s, q));
  if (s->width < 2) return set_error(SK_EVALUE, "cannot round the last qubit of a shard");
  sk_state* o;
  SK_TRY(state_alloc(s->width - 1, s->dtype, s->device, &o));
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int g = grid_for(o->n, kThreads, 2, c->num_sms);
  int rc = dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_round<R><<<g, kThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, (vec2_t<R>*)o->d, o->n, q,
                                              mk<R>((R)u0[0], (R)u0[1]), mk<R>((R)u0[2], (R)u0[3]), (R)scale);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
  if (rc != SK_OK) {
    sk_destroy(o);
    return rc;
  }
  *out = o;
  return SK_OK;
}

int sk_kron(const sk_state* lo, const sk_state* hi, sk_state** out) {
  SK_TRY(check_state(lo));
  SK_TRY(check_state(hi));
  if (lo->dtype != hi->dtype || lo->device != hi->device) return set_error(SK_EVALUE, "kron operands differ in dtype/device");
  sk_state* o;
  SK_TRY(state_alloc(lo->width + hi->width, lo->dtype, lo->device, &o));
  DevCtx* c;
  SK_TRY(ctx_get(lo->device, &c));
  const int g = grid_for(o->n, kThreads, 2, c->num_sms);
  int rc = dispatch(lo, [&](auto r) {
    using R = decltype(r);
    if (hi->width <= 4 && lo->width >= 10)
      k_kron_narrow<R><<<grid_for(lo->n, kThreads, 2, c->num_sms), kThreads, 0, c->stream>>>(
          (const vec2_t<R>*)lo->d, (const vec2_t<R>*)hi->d, (vec2_t<R>*)o->d, lo->n, lo->width, (int)hi->n);
    else
      k_kron<R><<<g, kThreads, 0, c->stream>>>((const vec2_t<R>*)lo->d, (const vec2_t<R>*)hi->d, (vec2_t<R>*)o->d, o->n,
                                             lo->width);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
  if (rc != SK_OK) {
    sk_destroy(o);
    return rc;
  }
  *out = o;
  return SK_OK;
}

int sk_permute(const sk_state* s, const int* order, sk_state** out) {
  SK_TRY(check_state(s));
  PermSpec ps{};
  ps.w = s->width;
  uint64_t seen = 0;
  for (int k = 0; k < s->width; ++k) {
    if (order[k] < 0 || order[k] >= s->width || ((seen >> order[k]) & 1ull))
      return set_error(SK_EVALUE, "order must be a permutation of 0..%d", s->width - 1);
    seen |= 1ull << order[k];
    ps.order[k] = order[k];
  }
  sk_state* o;
  SK_TRY(state_alloc(s->width, s->dtype, s->device, &o));
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int w = s->width;
  int rc;
  const int TB = 8 + (s->dtype == SK_C64 ? 3 : 2);  // tile bits (perm_eb)
  if (w >= TB + 2) {  // tiled transpose (small states: the per-element gather below)
    PermTile pt{};
    pt.w = w;
    int inv[64];
    for (int k = 0; k < w; ++k) inv[order[k]] = k;
    bool in_tile[64] = {false};
    int T = 0;
    auto add = [&](int k) {
      if (!in_tile[k]) in_tile[k] = true, ++T;
    };
    for (int k = 0; k < kPermK; ++k) {
      add(k);        // output low bits
      add(inv[k]);   // output positions of the input low bits
    }
    for (int k = 0; k < w && T < TB; ++k) add(k);  // pad the tile to 2^TB elements
    std::vector<int> tout, tin;  // tile bits by output position / by input position
    for (int k = 0; k < w; ++k)
      if (in_tile[k]) tout.push_back(k);
    for (int k : tout) tin.push_back(order[k]);
    std::sort(tin.begin(), tin.end());
    for (int t = 0; t < TB; ++t) {
      pt.out_of_bit[t] = 1ull << tout[t];
      pt.in_of_bit[t] = 1ull << tin[t];
      const int ob = inv[tin[t]];  // output position of this input bit
      pt.rm[t] = 1u << (int)(std::find(tout.begin(), tout.end(), ob) - tout.begin());
    }
    for (int k = 0; k < w; ++k)
      if (!in_tile[k]) {
        pt.rest_out[pt.nrest] = (uint8_t)k;
        pt.rest_in[pt.nrest] = (uint8_t)order[k];
        ++pt.nrest;
      }
    const uint64_t blocks = 1ull << (w - TB);
    rc = dispatch(s, [&](auto r) {
      using R = decltype(r);
      k_permute_tiled<R><<<(unsigned)blocks, kPermThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, (vec2_t<R>*)o->d,
                                                                          pt);
      SK_CHECK_LAUNCH();
      return SK_OK;
    });
  } else {
    const int g = grid_for(o->n, kThreads, 2, c->num_sms);
    rc = dispatch(s, [&](auto r) {
      using R = decltype(r);
      k_permute<R><<<g, kThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, (vec2_t<R>*)o->d, o->n, ps);
      SK_CHECK_LAUNCH();
      return SK_OK;
    });
  }
  if (rc != SK_OK) {
    sk_destroy(o);
    return rc;
  }
  *out = o;
  return SK_OK;
}

int sk_sample(const sk_state* s, const double* uniforms, int64_t k, int64_t* out_idx) {
  SK_TRY(check_state(s));
  if (k < 0) return set_error(SK_EVALUE, "negative sample count");
  if (k == 0) return SK_OK;
  DevCtx* c;
  SK_TRY(ctx_get(s->device, &c));
  const int chunk = (int)std::min<int64_t>(s->n, int64_t(1) << kChunkBits);
  const int64_t nchunks = s->n / chunk;
  double* d_sums = nullptr;
  SK_CUDA(cudaMallocAsync(&d_sums, sizeof(double) * nchunks, c->stream));
  const int g1 = grid_for(nchunks * 32, kThreads, 1, c->num_sms, 16);
  int rc = dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_chunk_sums<R><<<g1, kThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, nchunks, chunk, d_sums);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
  if (rc != SK_OK) return rc;
  std::vector<double> sums(nchunks), prefix(nchunks);
  SK_CUDA(cudaMemcpyAsync(sums.data(), d_sums, sizeof(double) * nchunks, cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(cudaStreamSynchronize(c->stream));
  double run = 0;
  for (int64_t i = 0; i < nchunks; ++i) {
    run += sums[i];
    prefix[i] = run;
  }
  const double total = run;
  if (!(total > 0)) {
    cudaFreeAsync(d_sums, c->stream);
    return set_error(SK_EVALUE, "probabilities sum to %g", total);
  }
  std::vector<int64_t> chunk_of(k);
  std::vector<double> resid(k);
  for (int64_t i = 0; i < k; ++i) {
    const double target = uniforms[i] * total;
    int64_t ch = std::upper_bound(prefix.begin(), prefix.end(), target) - prefix.begin();
    if (ch >= nchunks) ch = nchunks - 1;
    while (ch > 0 && sums[ch] == 0.0) --ch;  // rounding past the last nonzero chunk
    chunk_of[i] = ch;
    resid[i] = target - (ch ? prefix[ch - 1] : 0.0);
  }
  int64_t* d_chunk = nullptr;
  double* d_resid = nullptr;
  int64_t* d_out = nullptr;
  SK_CUDA(cudaMallocAsync(&d_chunk, sizeof(int64_t) * k, c->stream));
  SK_CUDA(cudaMallocAsync(&d_resid, sizeof(double) * k, c->stream));
  SK_CUDA(cudaMallocAsync(&d_out, sizeof(int64_t) * k, c->stream));
  SK_CUDA(cudaMemcpyAsync(d_chunk, chunk_of.data(), sizeof(int64_t) * k, cudaMemcpyHostToDevice, c->stream));
  SK_CUDA(cudaMemcpyAsync(d_resid, resid.data(), sizeof(double) * k, cudaMemcpyHostToDevice, c->stream));
  const int g2 = grid_for(k * 32, kThreads, 1, c->num_sms, 16);
  rc = dispatch(s, [&](auto r) {
    using R = decltype(r);
    k_sample_resolve<R><<<g2, kThreads, 0, c->stream>>>((const vec2_t<R>*)s->d, chunk, d_chunk, d_resid, k, d_out);
    SK_CHECK_LAUNCH();
    return SK_OK;
  });
  if (rc != SK_OK) return rc;
  SK_CUDA(cudaMemcpyAsync(out_idx, d_out, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, c->stream));
  SK_CUDA(cudaFreeAsync(d_sums, c->stream));
  SK_CUDA(cudaFreeAsync(d_chunk, c->stream));
  SK_CUDA(cudaFreeAsync(d_resid, c->stream));
  SK_CUDA(cudaFreeAsync(d_out, c->stream));
  SK_CUDA(cudaStreamSynchronize(c->stream));
  return SK_OK;
}

}  // extern "C"
