// sk_internal.cuh — shared internals of libshardcu (state struct, per-device
// context, error plumbing, complex helpers).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>

#include "../../include/shardcu.h"

namespace sk {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
int set_error(int code, const char* fmt, ...);

#define SK_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      if (e_ == cudaErrorMemoryAllocation) {                                       \
        cudaGetLastError();                                                        \
        return ::sk::set_error(SK_ENOMEM, "%s: %s", #call, cudaGetErrorString(e_)); \
      }                                                                            \
      return ::sk::set_error(SK_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));   \
    }                                                                              \
  } while (0)

#define SK_CHECK_LAUNCH() SK_CUDA(cudaGetLastError())

#define SK_TRY(expr)          \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != SK_OK) return rc_; \
  } while (0)

// ---------------------------------------------------------------------------
// per-device context: stream, reduction scratch, pinned scalar buffer
// ---------------------------------------------------------------------------
constexpr int kRedMaxBlocks = 1184;  // 148 SMs x 8
constexpr int kRedMaxK = 8;

// Reductions hand their fp64 results to the host through mapped pinned
// memory: the last block writes the K sums straight into host memory, then
// (after __threadfence_system) a sequence number; the host spins on that
// number instead of a cudaMemcpyAsync + cudaStreamSynchronize round trip.
struct RedOut {
  double* partials;
  unsigned* counter;
  double* result;               // device alias of the mapped host slot
  unsigned long long* flag;     // device alias of the mapped sequence word
  unsigned long long seq;
};

struct DevCtx {
  bool init = false;
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  double* d_partials = nullptr;  // [kRedMaxBlocks * kRedMaxK]
  unsigned int* d_counter = nullptr;
  double* h_result = nullptr;    // pinned [kRedMaxK] (point reads)
  double* h_map = nullptr;       // mapped pinned: [kRedMaxK] results + 1 sequence word
  double* d_map = nullptr;       // its device alias
  unsigned long long seq = 0;
  std::mutex red_mu;             // one reduction scratch per device: reductions are serialised
  int num_sms = 148;
};

// launch argument for the next reduction on c (caller holds c->red_mu)
RedOut red_out(DevCtx* c);
// wait for that reduction's results (spins on the mapped sequence word)
int red_wait(DevCtx* c, const RedOut& ro, double* out, int k);

int ctx_get(int device, DevCtx** out);  // initialises lazily, sets current device

}  // namespace sk

struct sk_state {
  void* d = nullptr;
  int width = 0;
  int dtype = SK_C128;
  int device = 0;
  int64_t n = 0;  // 2^width amplitudes
  size_t elem = 16;
  bool owned = true;  // false for sk_wrap views over caller memory
};

namespace sk {

int state_alloc(int width, int dtype, int device, sk_state** out);
// width-1 state from host amplitudes (re0, im0, re1, im1) whose Bloch sums the
// kernel publishes to mapped memory (d_out4, then *d_flag = seq)
int create_single_with_sums(int dtype, int device, const double amps[4], double* d_out4,
                            unsigned long long* d_flag, unsigned long long seq, sk_state** out);
// spin until a kernel publishes `seq` into the mapped word hflag (stream errors surface)
int wait_mapped(int device, volatile unsigned long long* hflag, unsigned long long seq);
inline size_t elem_size(int dtype) { return dtype == SK_C64 ? 8 : 16; }

// ---------------------------------------------------------------------------
// complex helpers (device)
// ---------------------------------------------------------------------------
template <typename R> struct V2;
template <> struct V2<float> { using T = float2; };
template <> struct V2<double> { using T = double2; };

template <typename R>
using vec2_t = typename V2<R>::T;

template <typename R>
__host__ __device__ __forceinline__ vec2_t<R> mk(R x, R y) {
  vec2_t<R> v;
  v.x = x;
  v.y = y;
  return v;
}

template <typename R>
__device__ __forceinline__ vec2_t<R> cmul(vec2_t<R> a, vec2_t<R> b) {
  return mk<R>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// m0*a + m1*b
template <typename R>
__device__ __forceinline__ vec2_t<R> cmad2(vec2_t<R> m0, vec2_t<R> a, vec2_t<R> m1, vec2_t<R> b) {
  R x = m0.x * a.x - m0.y * a.y + m1.x * b.x - m1.y * b.y;
  R y = m0.x * a.y + m0.y * a.x + m1.x * b.y + m1.y * b.x;
  return mk<R>(x, y);
}

// Packed complex arithmetic.  For float2 every op is one or two sm_100
// paired-fp32 instructions (FADD2 / FMUL2 / FFMA2; the swizzles and the
// one-lane negation of the product term are free operand modifiers), so a
// complex multiply is 2 issue slots instead of 4 and an add 1 instead of 2.
// double2 falls back to scalar fp64.
template <typename R>
struct PK;

template <>
struct PK<float> {
  using V = float2;
  static __device__ __forceinline__ V add(V a, V b) { return __fadd2_rn(a, b); }
  static __device__ __forceinline__ V sub(V a, V b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
  // (a.x b.x - a.y b.y, a.x b.y + a.y b.x) = a.x * b + (-(a.y b.y), a.y b.x)
  static __device__ __forceinline__ V mul(V a, V b) {
    const V s = __fmul2_rn(make_float2(a.y, a.y), make_float2(b.y, b.x));
    return __ffma2_rn(make_float2(a.x, a.x), b, make_float2(-s.x, s.y));
  }
  static __device__ __forceinline__ V scale(V a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
  static __device__ __forceinline__ V conj(V a) { return make_float2(a.x, -a.y); }
};

template <>
struct PK<double> {
  using V = double2;
  static __device__ __forceinline__ V add(V a, V b) { return make_double2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ V sub(V a, V b) { return make_double2(a.x - b.x, a.y - b.y); }
  static __device__ __forceinline__ V mul(V a, V b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  static __device__ __forceinline__ V scale(V a, double s) { return make_double2(a.x * s, a.y * s); }
  static __device__ __forceinline__ V conj(V a) { return make_double2(a.x, -a.y); }
};

// 2x2 complex matrix in the precision of the state
template <typename R>
struct Mat2 {
  vec2_t<R> m00, m01, m10, m11;
};

template <typename R>
inline Mat2<R> mat_from(const double m[8]) {
  Mat2<R> r;
  r.m00 = mk<R>((R)m[0], (R)m[1]);
  r.m01 = mk<R>((R)m[2], (R)m[3]);
  r.m10 = mk<R>((R)m[4], (R)m[5]);
  r.m11 = mk<R>((R)m[6], (R)m[7]);
  return r;
}

// insert a zero bit at position b
__host__ __device__ __forceinline__ uint64_t insert0(uint64_t x, int b) {
  uint64_t lo = x & ((1ull << b) - 1);
  return ((x >> b) << (b + 1)) | lo;
}

inline int grid_for(int64_t items, int threads, int per_thread, int num_sms, int max_per_sm = 8) {
  int64_t want = (items + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread);
  int64_t cap = (int64_t)num_sms * max_per_sm;
  if (want < 1) want = 1;
  if (want > cap) want = cap;
  return (int)want;
}

}  // namespace sk
