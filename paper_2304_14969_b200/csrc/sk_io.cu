// sk_io.cu — host <-> device transfers of whole states for the drop-in's
// `.amps` getter/setter and constructors (ket.py:73-91), whose host side is
// a pageable complex128 NumPy array.
//
// A pageable cudaMemcpy goes through the driver's own small staging buffer
// one piece at a time, with the host copy and the DMA serialised (~5-8 GB/s
// measured for 2 GiB).  Here a per-device pair of pinned 32 MiB chunks is
// filled / drained by several host threads while the copy engine moves the
// other chunk, so host memory bandwidth and PCIe overlap.  For c64 states the
// narrowing (complex128 -> complex64) / widening happens in that same host
// pass, so only native-width bytes cross PCIe.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "sk_internal.cuh"

namespace sk {

namespace {

constexpr size_t kChunk = size_t(32) << 20;

struct Staging {
  bool init = false;
  unsigned char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

Staging g_stage[64];
std::mutex g_stage_mu;

int staging_get(DevCtx* c, Staging** out) {
  Staging& s = g_stage[c->device];
  if (!s.init) {
    for (int b = 0; b < 2; ++b) {
      SK_CUDA(cudaHostAlloc((void**)&s.buf[b], kChunk, cudaHostAllocDefault));
      SK_CUDA(cudaEventCreateWithFlags(&s.ev[b], cudaEventDisableTiming));
    }
    s.init = true;
  }
  *out = &s;
  return SK_OK;
}

enum Mode { kCopy = 0, kNarrow = 1, kWiden = 2 };  // bytes / double->float / float->double

// dst[0..n) <- src[0..n) in `mode` units (bytes, doubles, floats), split over host threads
void par_transform(void* dst, const void* src, size_t n, Mode mode) {
  const size_t unit_bytes = mode == kCopy ? 1 : (mode == kNarrow ? 8 : 4);
  const size_t total = n * unit_bytes;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const int T = total >= (size_t(4) << 20) ? (int)std::min(8u, hw) : 1;
  auto work = [&](size_t lo, size_t hi) {
    if (mode == kCopy) {
      std::memcpy((char*)dst + lo, (const char*)src + lo, hi - lo);
    } else if (mode == kNarrow) {
      const double* s = (const double*)src;
      float* d = (float*)dst;
      for (size_t i = lo; i < hi; ++i) d[i] = (float)s[i];
    } else {
      const float* s = (const float*)src;
      double* d = (double*)dst;
      for (size_t i = lo; i < hi; ++i) d[i] = (double)s[i];
    }
  };
  if (T == 1) {
    work(0, n);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    const size_t lo = std::min(n, per * t), hi = std::min(n, per * (t + 1));
    if (lo < hi) th.emplace_back(work, lo, hi);
  }
  for (auto& x : th) x.join();
}

}  // namespace

// host (complex128, pageable) -> device state of n amplitudes in its native width
int staged_upload(DevCtx* c, sk_state* s, const double* host, int64_t n) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Staging* st;
  SK_TRY(staging_get(c, &st));
  const size_t esz = s->elem;
  const size_t per = kChunk / esz;  // amplitudes per chunk
  int k = 0;
  for (int64_t off = 0; off < n; off += (int64_t)per, ++k) {
    const size_t m = (size_t)std::min<int64_t>((int64_t)per, n - off);
    const int b = k & 1;
    if (k >= 2) SK_CUDA(cudaEventSynchronize(st->ev[b]));  // chunk k-2's DMA has drained buffer b
    if (esz == 16)
      par_transform(st->buf[b], host + 2 * off, m * 16, kCopy);
    else
      par_transform(st->buf[b], host + 2 * off, 2 * m, kNarrow);
    SK_CUDA(cudaMemcpyAsync((unsigned char*)s->d + off * esz, st->buf[b], m * esz, cudaMemcpyHostToDevice, c->stream));
    SK_CUDA(cudaEventRecord(st->ev[b], c->stream));
  }
  SK_CUDA(cudaStreamSynchronize(c->stream));
  return SK_OK;
}

// device state -> host (complex128, pageable)
int staged_download(DevCtx* c, const sk_state* s, double* host, int64_t n) {
  std::lock_guard<std::mutex> lk(g_stage_mu);
  Staging* st;
  SK_TRY(staging_get(c, &st));
  const size_t esz = s->elem;
  const int64_t per = (int64_t)(kChunk / esz);
  const int64_t nchunks = (n + per - 1) / per;
  auto enqueue = [&](int64_t k) -> int {
    const int64_t off = k * per;
    const size_t m = (size_t)std::min(per, n - off);
    SK_CUDA(cudaMemcpyAsync(st->buf[k & 1], (const unsigned char*)s->d + off * esz, m * esz, cudaMemcpyDeviceToHost,
                            c->stream));
    SK_CUDA(cudaEventRecord(st->ev[k & 1], c->stream));
    return SK_OK;
  };
  for (int64_t k = 0; k < std::min<int64_t>(2, nchunks); ++k) SK_TRY(enqueue(k));
  for (int64_t k = 0; k < nchunks; ++k) {
    const int64_t off = k * per;
    const size_t m = (size_t)std::min(per, n - off);
    SK_CUDA(cudaEventSynchronize(st->ev[k & 1]));
    if (esz == 16)
      par_transform(host + 2 * off, st->buf[k & 1], m * 16, kCopy);
    else
      par_transform(host + 2 * off, st->buf[k & 1], 2 * m, kWiden);
    if (k + 2 < nchunks) SK_TRY(enqueue(k + 2));
  }
  return SK_OK;
}

}  // namespace sk
