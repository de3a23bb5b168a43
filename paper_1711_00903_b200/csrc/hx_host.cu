// Host-memory runtime of the drop-in path: the reference's users hand
// apply_operator plain (pageable) numpy arrays (operators.py:306-331), which
// the copy engines cannot DMA at full rate.  hx_apply_host_staged streams
// such arrays through a small ring of page-locked staging slots: host worker
// threads copy chunk c+1 of q into a pinned slot while chunk c is on PCIe,
// its kernel runs and chunk c-1 drains back, so the host copies overlap the
// whole device pipeline instead of bracketing it.  Also here: the
// non-finite pre-checks (host scan and device kernel) that let
// apply_operator(..., out=) leave a caller's buffer untouched on bad input,
// as the reference's up-front np.isfinite scan does (operators.py:317-318).
#include <emmintrin.h>

#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {


namespace {

// Fixed pool of host worker threads for parallel memcpy / scans.  run(n, f)
// calls f(0..n-1) spread over the workers and the calling thread and returns
// when all have finished.  One job at a time (callers serialise on `job_mu`).
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  int size() const { return int(workers_.size()) + 1; }

  void run(int parts, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> job(job_mu_);
    if (parts <= 1 || workers_.empty()) {
      for (int i = 0; i < parts; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      parts_ = parts;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == parts_; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    int n = int(std::thread::hardware_concurrency());
    if (const char* e = std::getenv("HX_HOST_THREADS")) n = std::atoi(e);
    if (n < 1) n = 1;
    if (n > 32) n = 32;
    for (int i = 0; i + 1 < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void work() {
    int finished = 0;
    for (int i = next_.fetch_add(1); i < parts_; i = next_.fetch_add(1)) {
      (*fn_)(i);
      ++finished;
    }
    if (finished) {
      std::lock_guard<std::mutex> lk(mu_);
      done_ += finished;
      if (done_ == parts_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (!fn_) continue;
      }
      work();
    }
  }

  std::vector<std::thread> workers_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int parts_ = 0, done_ = 0;
  std::atomic<int> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// Streaming copy: non-temporal 16-byte stores, so the destination lines are
// not read for ownership first -- 2 instead of 3 bytes of host memory
// traffic per byte copied, which matters because the PCIe DMA of the same
// pipeline shares that bandwidth (tools/memcpy_probe.c on the GPU box: 82 vs
// 53 GB/s with 8-16 threads).
void stream_copy(char* d, const char* s, size_t n) {
  const size_t head = std::min(n, size_t((16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15));
  std::memcpy(d, s, head);
  d += head;
  s += head;
  n -= head;
  size_t i = 0;
  for (; i + 64 <= n; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(d + i + 48), e);
  }
  std::memcpy(d + i, s + i, n - i);
  _mm_sfence();  // the streaming stores are visible before the DMA that reads them
}

// dst[0, bytes) = src[0, bytes) with the pool; pieces of >= 1 MiB, 4 KiB aligned
void parallel_copy(void* dst, const void* src, size_t bytes) {
  HostPool& pool = HostPool::get();
  constexpr size_t kMin = size_t(1) << 20;
  int parts = int(std::min<size_t>(size_t(pool.size()), (bytes + kMin - 1) / kMin));
  if (parts < 1) parts = 1;
  const size_t piece = ((bytes + parts - 1) / parts + 4095) & ~size_t(4095);
  pool.run(parts, [&](int i) {
    const size_t lo = size_t(i) * piece;
    if (lo >= bytes) return;
    const size_t n = std::min(piece, bytes - lo);
    stream_copy(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, n);
  });
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

__global__ void finite_kernel(const double* __restrict__ x, int64_t n, int* flag) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  unsigned acc = 0x7ff00000u;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    acc = min(acc, ~static_cast<unsigned>(__double2hiint(__ldcs(x + i))) & 0x7ff00000u);
  if (__any_sync(0xffffffffu, acc == 0u) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace

cudaError_t launch_check_finite(const double* x, int64_t n, int* flag, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int64_t want = (n + 255) / 256;
  const unsigned grid = unsigned(min64(want, int64_t(sm_count()) * 8));
  finite_kernel<<<grid, 256, 0, s>>>(x, n, flag);
  return cudaGetLastError();
}

}  // namespace hx

using namespace hx;

extern "C" {

int hx_check_finite(const double* x, int64_t n, int* flag, void* stream) {
  if (n < 0 || !flag || (n > 0 && !x)) return HX_EINVAL;
  return cuda_status(launch_check_finite(x, n, flag, static_cast<cudaStream_t>(stream)));
}

int hx_host_all_finite(const double* x, int64_t n) {
  if (n <= 0 || !x) return 1;
  HostPool& pool = HostPool::get();
  constexpr int64_t kMin = int64_t(1) << 17;  // doubles per piece (1 MiB)
  const int parts = int(std::max<int64_t>(1, std::min<int64_t>(pool.size(), n / kMin)));
  const int64_t piece = (n + parts - 1) / parts;
  std::atomic<int> bad{0};
  pool.run(parts, [&](int i) {
    const int64_t lo = i * piece, hi = std::min(n, lo + piece);
    uint64_t acc = 0x7ff0000000000000ull;
    for (int64_t j = lo; j < hi; ++j) {
      uint64_t b;
      std::memcpy(&b, x + j, 8);
      acc = std::min<uint64_t>(acc, ~b & 0x7ff0000000000000ull);
    }
    if (acc == 0) bad.store(1);
  });
  return bad.load() ? 0 : 1;
}

int64_t hx_apply_host_staging_bytes(const hx_plan* P, int64_t chunk_el) {
  if (!P || chunk_el <= 0) return -1;
  const int64_t n3 = int64_t(P->n) * P->n * P->n;
  return hx_host_slots * 2 /*q,out*/ * chunk_el * n3 * int64_t(sizeof(double));
}

int hx_apply_host_staged(const hx_plan* Pc, const double* q_host, const double* factors,
                         double* out_host, int64_t n_el, int64_t chunk_el, void* work,
                         void* staging, int* flag, void* stream) {
  if (!Pc || n_el < 0 || chunk_el <= 0) return HX_EINVAL;
  if (n_el == 0) return HX_OK;
  if (!q_host || !factors || !out_host || !work || !staging) return HX_EINVAL;
  hx_plan* P = const_cast<hx_plan*>(Pc);
  std::lock_guard<std::mutex> lock(P->pipe_mu);
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  cudaError_t err = pipe_setup(P);
  if (err != cudaSuccess) return cuda_status(err);
  const int64_t n3 = int64_t(P->n) * P->n * P->n;
  const int64_t last = (n_el * n3 - 1);
  // page-locked buffers go straight to the copy engines; pageable ones
  // through the pinned ring
  const bool stage_q = !(is_pinned(q_host) && is_pinned(q_host + last));
  const bool stage_o = !(is_pinned(out_host) && is_pinned(out_host + last));
  constexpr int S = hx_host_slots;
  double *wq[S], *wo[S], *hq[S], *ho[S];
  double* base = static_cast<double*>(work);
  double* hb = static_cast<double*>(staging);
  for (int i = 0; i < S; ++i) {
    wq[i] = base + int64_t(i) * chunk_el * n3;
    wo[i] = base + int64_t(S + i) * chunk_el * n3;
    hq[i] = hb + int64_t(i) * chunk_el * n3;
    ho[i] = hb + int64_t(S + i) * chunk_el * n3;
  }
  cudaStream_t s_in = P->pipe[0], s_k = P->pipe[1], s_out = P->pipe[2];
  cudaEvent_t* e_in = P->ev[0];
  cudaEvent_t* e_k = P->ev[1];
  cudaEvent_t* e_out = P->ev[2];
  cudaEvent_t start;
  if ((err = cudaEventCreateWithFlags(&start, cudaEventDisableTiming)) != cudaSuccess)
    return cuda_status(err);
  cudaEventRecord(start, caller);
  cudaStreamWaitEvent(s_in, start, 0);
  cudaStreamWaitEvent(s_k, start, 0);
  cudaStreamWaitEvent(s_out, start, 0);
  cudaStreamWaitEvent(s_in, P->pipe_last, 0);  // the plan's previous pipeline call
  cudaStreamWaitEvent(s_k, P->pipe_last, 0);
  // the host copies below touch q_host / out_host directly: they too come
  // after the work queued on `stream` before the call
  if (stage_q || stage_o) err = cudaEventSynchronize(start);
  cudaEventDestroy(start);
  if (err != cudaSuccess) return cuda_status(err);
  const std::vector<int64_t> sched = chunk_schedule(n_el, chunk_el);
  const int64_t nchunks = int64_t(sched.size());
  std::vector<int64_t> first(nchunks + 1, 0);
  for (int64_t c = 0; c < nchunks; ++c) first[c + 1] = first[c] + sched[c];
  int64_t drained = 0;  // chunks whose output is in out_host
  // copy finished chunks [drained, upto) out of the pinned ring; without
  // `block` only as far as the D2H copies have already completed
  auto drain = [&](int64_t upto, bool block) -> cudaError_t {
    for (; drained < upto; ++drained) {
      const int slot = int(drained % S);
      cudaError_t e = block ? cudaEventSynchronize(e_out[slot]) : cudaEventQuery(e_out[slot]);
      if (e == cudaErrorNotReady) return cudaSuccess;
      if (e != cudaSuccess) return e;
      if (stage_o)
        parallel_copy(out_host + first[drained] * n3, ho[slot],
                      size_t(sched[drained] * n3) * sizeof(double));
    }
    return cudaSuccess;
  };
  for (int64_t c = 0; c < nchunks && err == cudaSuccess; ++c) {
    const int slot = int(c % S);
    const int64_t ne = sched[c], e0 = first[c];
    const size_t bytes = size_t(ne * n3) * sizeof(double);
    // chunk c - S must have left the slot's pinned buffers: its H2D has read
    // hq[slot], its output has been copied out of ho[slot]
    if (c >= S) {
      if (stage_o && (err = drain(c - S + 1, true)) != cudaSuccess) break;
      if (stage_q && (err = cudaEventSynchronize(e_in[slot])) != cudaSuccess) break;
    }
    const double* src = q_host + e0 * n3;
    if (stage_q) {
      parallel_copy(hq[slot], src, bytes);
      src = hq[slot];
    }
    if (c >= S) cudaStreamWaitEvent(s_in, e_k[slot], 0);  // kernel c-S done with wq[slot]
    cudaMemcpyAsync(wq[slot], src, bytes, cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(e_in[slot], s_in);
    cudaStreamWaitEvent(s_k, e_in[slot], 0);
    if (c >= S) cudaStreamWaitEvent(s_k, e_out[slot], 0);  // D2H c-S done with wo[slot]
    if ((err = launch_apply(*P, wq[slot], factors + e0 * P->elem_stride, wo[slot], ne, flag,
                            s_k)) != cudaSuccess)
      break;
    cudaEventRecord(e_k[slot], s_k);
    cudaStreamWaitEvent(s_out, e_k[slot], 0);
    cudaMemcpyAsync(stage_o ? ho[slot] : out_host + e0 * n3, wo[slot], bytes,
                    cudaMemcpyDeviceToHost, s_out);
    cudaEventRecord(e_out[slot], s_out);
    // copy out whatever has already come back while the device works on
    if (stage_o && (err = drain(c, false)) != cudaSuccess) break;
  }
  if (err != cudaSuccess) {
    cudaStreamSynchronize(s_in);
    cudaStreamSynchronize(s_k);
    cudaStreamSynchronize(s_out);
    return cuda_status(err);
  }
  P->pipe_cont = false;  // slot sequence restarted: HX_HOST_OVERLAP calls drain first
  cudaEventRecord(P->pipe_last, s_out);
  if ((err = drain(nchunks, true)) != cudaSuccess) return cuda_status(err);
  cudaStreamWaitEvent(caller, P->pipe_last, 0);
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
