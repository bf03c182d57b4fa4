// sk_ops.cuh — device building blocks shared by the ket kernels (sk_ket.cu)
// and the engine's fused kernels (sk_engine.cu).  Sharing them keeps the
// fused paths bit-identical to the separate kernels they replace: the same
// element arithmetic, and for reductions the same per-thread accumulation
// and the same warp -> block -> last-block combine.
#pragma once

#include "sk_internal.cuh"

namespace sk {

// one (a0, a1) pair's contribution to the Bloch sums; shared by k_bloch and
// k_set_single so a width-1 shard's cached sums are bit-identical to a reduction
__device__ __forceinline__ void bloch_acc(double (&v)[4], double ar, double ai, double br, double bi) {
  v[0] += ar * br + ai * bi;  // Re conj(a)*b
  v[1] += ar * bi - ai * br;  // Im conj(a)*b
  v[2] += ar * ar + ai * ai;
  v[3] += br * br + bi * bi;
}

// Write a width-1 shard's two amplitudes and publish its Bloch sums — as
// k_bloch would reduce them from the stored precision — to mapped host
// memory, then the sequence word (one thread).
template <typename R>
__device__ __forceinline__ void publish_single(vec2_t<R>* d, double ar, double ai, double br, double bi, double* out4,
                                               unsigned long long* flag, unsigned long long seq) {
  const vec2_t<R> a = mk<R>((R)ar, (R)ai), b = mk<R>((R)br, (R)bi);
  d[0] = a;
  d[1] = b;
  double v[4] = {0, 0, 0, 0};
  bloch_acc(v, a.x, a.y, b.x, b.y);
  for (int k = 0; k < 4; ++k) out4[k] = v[k];
  __threadfence_system();
  *(volatile unsigned long long*)flag = seq;
}

template <typename R>
__device__ __forceinline__ void ctrl_bloch_load(const vec2_t<R>* __restrict__ a, uint64_t b, uint64_t C, uint64_t T,
                                                vec2_t<R> (&x)[2][2]) {  // x[cbit][tbit]
  x[0][0] = a[b];
  x[0][1] = a[b | T];
  x[1][0] = a[b | C];
  x[1][1] = a[b | C | T];
}

template <typename R>
__device__ __forceinline__ void ctrl_bloch_apply(vec2_t<R>* __restrict__ a, uint64_t b, uint64_t C, uint64_t T, int pol,
                                                 const Mat2<R>& m, vec2_t<R> (&x)[2][2], double (&v)[8]) {
  vec2_t<R> y0 = cmad2<R>(m.m00, x[pol][0], m.m01, x[pol][1]);
  vec2_t<R> y1 = cmad2<R>(m.m10, x[pol][0], m.m11, x[pol][1]);
  x[pol][0] = y0;
  x[pol][1] = y1;
  uint64_t ib = pol ? (b | C) : b;
  a[ib] = y0;
  a[ib | T] = y1;
#pragma unroll
  for (int cb = 0; cb < 2; ++cb) {  // target sums over both control halves
    double ar = x[cb][0].x, ai = x[cb][0].y, br = x[cb][1].x, bi = x[cb][1].y;
    v[4] += ar * br + ai * bi;
    v[5] += ar * bi - ai * br;
    v[6] += ar * ar + ai * ai;
    v[7] += br * br + bi * bi;
  }
#pragma unroll
  for (int tb = 0; tb < 2; ++tb) {  // control sums over both target halves
    double ar = x[0][tb].x, ai = x[0][tb].y, br = x[1][tb].x, bi = x[1][tb].y;
    v[0] += ar * br + ai * bi;
    v[1] += ar * bi - ai * br;
    v[2] += ar * ar + ai * ai;
    v[3] += br * br + bi * bi;
  }
}

// One (c, t) quad of a one-control gate, with the Bloch sums of control
// (v[0..3]) and target (v[4..7]) accumulated from the post-gate amplitudes
// (engine.py:389-394 runs apply_controlled then bloch_vector twice).
template <typename R>
__device__ __forceinline__ void ctrl_bloch_quad(vec2_t<R>* __restrict__ a, uint64_t b, uint64_t C, uint64_t T, int pol,
                                                const Mat2<R>& m, double (&v)[8]) {
  vec2_t<R> x[2][2];
  ctrl_bloch_load<R>(a, b, C, T, x);
  ctrl_bloch_apply<R>(a, b, C, T, pol, m, x, v);
}

// DenseKet._apply_1q_unchecked element pair (ket.py:133-144)
template <typename R>
__device__ __forceinline__ void apply_1q_pair(vec2_t<R>* __restrict__ a, uint64_t i0, uint64_t bit, const Mat2<R>& m,
                                              int diag) {
  const vec2_t<R> x0 = a[i0], x1 = a[i0 | bit];
  vec2_t<R> y0, y1;
  if (diag) {
    y0 = cmul<R>(m.m00, x0);
    y1 = cmul<R>(m.m11, x1);
  } else {
    y0 = cmad2<R>(m.m00, x0, m.m01, x1);
    y1 = cmad2<R>(m.m10, x0, m.m11, x1);
  }
  a[i0] = y0;
  a[i0 | bit] = y1;
}

// ---------------------------------------------------------------------------
// reductions: K fp64 sums per launch, deterministic last-block combine
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ void block_reduce_finish(double (&v)[K], const RedOut& ro) {
  double* partials = ro.partials;
  unsigned* counter = ro.counter;
  double* result = ro.result;
  __shared__ double sh[32][K];
  __shared__ bool last;
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sh[warp][k] = v[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = lane < nw ? sh[lane][k] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
      if (lane == 0) partials[blockIdx.x * K + k] = x;
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] += ((volatile double*)partials)[b * K + k];
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_down_sync(0xffffffffu, acc[k], off);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) sh[warp][k] = acc[k];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double x = lane < nw ? sh[lane][k] : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) x += __shfl_down_sync(0xffffffffu, x, off);
      if (lane == 0) result[k] = x;
    }
    if (lane == 0) {
      *counter = 0;
      __threadfence_system();  // the K results reach host memory before the sequence word
      *(volatile unsigned long long*)ro.flag = ro.seq;
    }
  }
}

}  // namespace sk
