// C ABI entry points (include/hexbench_b200.h).  Thin: validate, dispatch to
// the per-operator launchers, translate CUDA errors into HX_ECUDA.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {

// SM count of the current device (cached per device ordinal)
int sm_count() {
  static std::atomic<int> cache[kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  const bool cached = dev >= 0 && dev < kMaxDevices;
  int count = cached ? cache[dev].load(std::memory_order_relaxed) : 0;
  if (count > 0) return count;
  if (cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      count <= 0)
    count = 1;
  if (cached) cache[dev].store(count, std::memory_order_relaxed);
  return count;
}

static int kernel_shape(int bp, int degree, int* epb, int* nt, int* smem) {
#define HX_SHAPE(BP, N)                                                  \
  if (bp == BP && degree == N) {                                        \
    *epb = Cfg<BP, N>::EPB;                                             \
    *nt = Cfg<BP, N>::NT;                                               \
    *smem = smem_doubles<BP, N>() * int(sizeof(double));                \
    return HX_OK;                                                       \
  }
#define HX_SHAPES(BP)                                                                        \
  HX_SHAPE(BP, 1) HX_SHAPE(BP, 2) HX_SHAPE(BP, 3) HX_SHAPE(BP, 4) HX_SHAPE(BP, 5)            \
  HX_SHAPE(BP, 6) HX_SHAPE(BP, 7) HX_SHAPE(BP, 8) HX_SHAPE(BP, 9) HX_SHAPE(BP, 10)           \
  HX_SHAPE(BP, 11) HX_SHAPE(BP, 12) HX_SHAPE(BP, 13) HX_SHAPE(BP, 14) HX_SHAPE(BP, 15)
  HX_SHAPES(kBP1)
  HX_SHAPES(kBP35)
  HX_SHAPES(kBP3)
#undef HX_SHAPES
#undef HX_SHAPE
  return HX_EINVAL;
}

cudaError_t launch_apply(const hx_plan& P, const double* q, const double* fac, double* out,
                         int64_t n_el, int* flag, cudaStream_t s, double* energy, bool pdl,
                         const DirArgs* dir) {
  if (n_el == 0) return cudaSuccess;
  switch (P.bp) {
    case HX_BP1:
      return launch_bp1(P, q, fac, out, n_el, flag, energy, s, pdl, dir);
    case HX_BP35:
      return launch_bp35(P, q, fac, out, n_el, flag, energy, s, pdl, dir);
    default:
      return launch_bp3(P, q, fac, out, n_el, flag, energy, s, pdl, dir);
  }
}

// The kernels apply the 1-D matrices in even/odd folded form, which is exact
// only for centro-symmetric (sign +1: I, I^T) or centro-antisymmetric (sign
// -1: D, D~) matrices -- true of the reference's (reference_ops.py:42-44).
// Anything else is rejected rather than silently mis-applied.
static bool centro_ok(const double* M, int R, int C, double sign) {
  double scale = 0.0;
  for (int a = 0; a < R * C; ++a) {
    if (!std::isfinite(M[a])) return false;
    scale = std::fmax(scale, std::fabs(M[a]));
  }
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < C; ++b)
      if (std::fabs(M[a * C + b] - sign * M[(R - 1 - a) * C + (C - 1 - b)]) > 1e-12 * scale)
        return false;
  return true;
}

static thread_local char g_last_cuda[256];

int cuda_status(cudaError_t err) {
  if (err == cudaSuccess) return HX_OK;
  std::snprintf(g_last_cuda, sizeof(g_last_cuda), "CUDA error: %s",
                cudaGetErrorString(err));
  return HX_ECUDA;
}

}  // namespace hx

using namespace hx;

namespace hx {
// Device-path applies (hx_apply, hx_apply_range, hx_apply_energy) launch as
// programmatic dependent launches (hx_common.cuh): back-to-back applies on a
// stream overlap one kernel's retiring CTAs with the next one's start.
#ifndef HX_APPLY_PDL
#define HX_APPLY_PDL 1
#endif
constexpr bool kApplyPdl = HX_APPLY_PDL != 0;
// NVTX range names per operator ("hx_apply BP1.0", ...)
static const char* range_name(const hx_plan& P, const char* what) {
  static const char* names[3][4] = {
      {"hx_apply BP1.0", "hx_apply_host BP1.0", "hx_apply_baseline BP1.0", "hx_apply_energy BP1.0"},
      {"hx_apply BP3.5", "hx_apply_host BP3.5", "hx_apply_baseline BP3.5", "hx_apply_energy BP3.5"},
      {"hx_apply BP3.0", "hx_apply_host BP3.0", "hx_apply_baseline BP3.0", "hx_apply_energy BP3.0"}};
  const int b = P.bp == HX_BP1 ? 0 : P.bp == HX_BP35 ? 1 : 2;
  const int w = what[0] == 'a' ? 0 : what[0] == 'h' ? 1 : what[0] == 'b' ? 2 : 3;
  return names[b][w];
}
}  // namespace hx

extern "C" {

int hx_plan_create(int bp, int degree, double lam, const double* interp, const double* diff,
                   const double* nodes, const double* weights, hx_plan** out) {
  if (!out) return HX_EINVAL;
  *out = nullptr;
  if (bp != HX_BP1 && bp != HX_BP35 && bp != HX_BP3) return HX_EINVAL;
  if (degree < 1 || degree > 15) return HX_EINVAL;
  if (!(lam >= 0.0)) return HX_EINVAL;  // also rejects NaN
  if (!nodes || !weights) return HX_EINVAL;
  if (bp != HX_BP35 && !interp) return HX_EINVAL;
  if (bp != HX_BP1 && !diff) return HX_EINVAL;
  {
    const int n = degree + 1, m = degree + 2, q = bp == HX_BP35 ? n : m;
    if (interp && bp != HX_BP35 && !centro_ok(interp, m, n, 1.0)) return HX_EINVAL;
    if (diff && bp != HX_BP1 && !centro_ok(diff, q, q, -1.0)) return HX_EINVAL;
  }
  hx_plan* P = new (std::nothrow) hx_plan();
  if (!P) return HX_ENOMEM;
  P->bp = bp;
  P->degree = degree;
  P->n = degree + 1;
  P->m = degree + 2;
  P->q = bp == HX_BP35 ? P->n : P->m;
  P->lam = lam;
  if (interp) std::memcpy(P->interp, interp, sizeof(double) * P->m * P->n);
  if (diff) std::memcpy(P->diff, diff, sizeof(double) * P->q * P->q);
  std::memcpy(P->nodes, nodes, sizeof(double) * P->q);
  std::memcpy(P->weights, weights, sizeof(double) * P->q);
  const int64_t q3 = int64_t(P->q) * P->q * P->q;
  P->n_slots = bp == HX_BP1 ? 1 : 7;
  P->slot_stride = (q3 + 1) & ~int64_t(1);  // keep every slot 16-byte aligned
  P->elem_stride = P->n_slots * P->slot_stride;
  P->pipe_ready = false;
  *out = P;
  return HX_OK;
}

void hx_plan_destroy(hx_plan* P) {
  if (!P) return;
  if (P->pipe_ready) {
    int cur = 0;
    const bool moved = cudaGetDevice(&cur) == cudaSuccess && cur != P->pipe_dev;
    if (moved) cudaSetDevice(P->pipe_dev);
    for (int i = 0; i < 3; ++i) {
      cudaStreamDestroy(P->pipe[i]);
      for (int j = 0; j < hx_host_slots; ++j) cudaEventDestroy(P->ev[i][j]);
    }
    cudaEventDestroy(P->pipe_last);
    if (moved) cudaSetDevice(cur);
  }
  delete P;
}

int hx_plan_factor_layout(const hx_plan* P, int* n_slots, int64_t* slot_stride,
                          int64_t* element_stride) {
  if (!P) return HX_EINVAL;
  if (n_slots) *n_slots = P->n_slots;
  if (slot_stride) *slot_stride = P->slot_stride;
  if (element_stride) *element_stride = P->elem_stride;
  return HX_OK;
}

int hx_plan_kernel_shape(const hx_plan* P, int* epb, int* threads, int* smem_bytes) {
  if (!P || !epb || !threads || !smem_bytes) return HX_EINVAL;
  return kernel_shape(P->bp, P->degree, epb, threads, smem_bytes);
}

int hx_geometric_factors(const hx_plan* P, const double* vertices, int64_t n_el, int all_slots,
                         double* factors, int* flag, void* stream) {
  if (!P || n_el < 0) return HX_EINVAL;
  if (n_el > 0 && (!vertices || !factors)) return HX_EINVAL;
  hx::NvtxRange range("hx_geometric_factors");
  return cuda_status(launch_geometry(*P, vertices, n_el, all_slots, factors, flag,
                                     static_cast<cudaStream_t>(stream)));
}

int hx_repack_factors(const hx_plan* P, const double* src, int64_t n_el, double* dst,
                      int to_packed, void* stream) {
  hx::NvtxRange range("hx_repack_factors");
  if (!P || n_el < 0) return HX_EINVAL;
  if (n_el > 0 && (!src || !dst)) return HX_EINVAL;
  return cuda_status(launch_repack(*P, src, n_el, dst, to_packed,
                                   static_cast<cudaStream_t>(stream)));
}

int hx_apply(const hx_plan* P, const double* q, const double* factors, double* out,
             int64_t n_el, int* flag, void* stream) {
  if (!P || n_el < 0) return HX_EINVAL;
  if (n_el > 0 && (!q || !factors || !out)) return HX_EINVAL;
  // doubles must be naturally aligned (16-byte alignment is not required)
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(factors) |
       reinterpret_cast<uintptr_t>(out)) & 7)
    return HX_EINVAL;
  hx::NvtxRange range(hx::range_name(*P, "apply"));
  return cuda_status(launch_apply(*P, q, factors, out, n_el, flag, static_cast<cudaStream_t>(stream),
                                  nullptr, kApplyPdl));
}

int hx_apply_range(const hx_plan* P, const double* q, const double* factors, double* out,
                   int64_t e_begin, int64_t e_end, int* flag, void* stream) {
  if (!P || e_begin < 0 || e_end < e_begin) return HX_EINVAL;
  const int64_t n3 = int64_t(P->n) * P->n * P->n;
  if (e_end == e_begin) return HX_OK;
  if (!q || !factors || !out) return HX_EINVAL;
  return hx_apply(P, q + e_begin * n3, factors + e_begin * P->elem_stride, out + e_begin * n3,
                  e_end - e_begin, flag, stream);
}

int64_t hx_apply_baseline_workspace(const hx_plan* P, int64_t n_el) {
  if (!P || n_el < 0) return -1;
  return baseline_workspace_doubles(*P, n_el) * int64_t(sizeof(double));
}

int hx_apply_baseline(const hx_plan* P, const double* q, const double* factors, double* out,
                      int64_t n_el, void* work, int* flag, void* stream) {
  if (!P || n_el < 0) return HX_EINVAL;
  if (n_el > 0 && (!q || !factors || !out || !work)) return HX_EINVAL;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(factors) |
       reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(work)) & 7)
    return HX_EINVAL;
  hx::NvtxRange range(hx::range_name(*P, "baseline"));
  return cuda_status(launch_baseline(*P, q, factors, out, n_el, static_cast<double*>(work), flag,
                                     static_cast<cudaStream_t>(stream)));
}

int hx_interp_elements(int degree, const double* interp, int project, const double* src,
                       double* dst, int64_t n_el, int* flag, void* stream) {
  hx::NvtxRange range("hx_interp_elements");
  if (degree < 1 || degree > 15 || n_el < 0 || !interp) return HX_EINVAL;
  if (project != 0 && project != 1) return HX_EINVAL;
  if (n_el == 0) return HX_OK;
  if (!src || !dst) return HX_EINVAL;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 7) return HX_EINVAL;
  for (int a = 0; a < (degree + 2) * (degree + 1); ++a)
    if (!std::isfinite(interp[a])) return HX_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (centro_ok(interp, degree + 2, degree + 1, 1.0))
    return cuda_status(launch_interp(degree, interp, project, src, dst, n_el, flag, s));
  // any other (N+2) x (N+1) matrix: the dense passes (the reference's
  // contract_dim accepts every 2-D matrix)
  const int nsrc = project ? degree + 2 : degree + 1;
  cudaError_t err = flag ? launch_check_finite(src, n_el * nsrc * nsrc * nsrc, flag, s)
                         : cudaSuccess;
  if (err == cudaSuccess) err = launch_interp_dense(degree, interp, project, src, dst, n_el, s);
  return cuda_status(err);
}

int64_t hx_apply_host_workspace(const hx_plan* P, int64_t chunk_el) {
  if (!P || chunk_el <= 0) return -1;
  const int64_t n3 = int64_t(P->n) * P->n * P->n;
  return hx_host_slots * 2 /*q,out*/ * chunk_el * n3 * int64_t(sizeof(double));
}

}  // extern "C"

namespace hx {

// Chunk sizes of the host pipeline: ramp up from chunk_el/8 by doubling,
// full chunks in the middle, ramp down at the end.  The pipeline's fill (the
// first H2D runs alone) and drain (the last D2H runs alone) then cost a small
// chunk each instead of a full one.  Falls back to uniform chunks when the
// problem is too small for the ramps.
std::vector<int64_t> chunk_schedule(int64_t n_el, int64_t chunk_el) {
  std::vector<int64_t> head;
  int64_t ramp = 0;
  for (int64_t c = std::max<int64_t>(1, chunk_el / 8); c < chunk_el; c *= 2) {
    head.push_back(c);
    ramp += c;
  }
  std::vector<int64_t> out;
  if (head.empty() || n_el <= 2 * ramp + chunk_el) {
    for (int64_t e = 0; e < n_el; e += chunk_el) out.push_back(std::min(chunk_el, n_el - e));
    return out;
  }
  out = head;
  const int64_t mid = n_el - 2 * ramp;
  const int64_t k = (mid + chunk_el - 1) / chunk_el;
  for (int64_t i = 0; i < k; ++i) out.push_back(mid / k + (i < mid % k ? 1 : 0));
  out.insert(out.end(), head.rbegin(), head.rend());
  return out;
}

// (Re)create the host pipeline's streams and events on the current device.
cudaError_t pipe_setup(hx_plan* P) {
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (P->pipe_ready && P->pipe_dev == dev) return cudaSuccess;
  if (P->pipe_ready) {  // the caller moved to another device: rebuild there
    int cur = dev;
    cudaSetDevice(P->pipe_dev);
    for (int i = 0; i < 3; ++i) {
      cudaStreamSynchronize(P->pipe[i]);
      cudaStreamDestroy(P->pipe[i]);
      for (int j = 0; j < hx_host_slots; ++j) cudaEventDestroy(P->ev[i][j]);
    }
    cudaEventDestroy(P->pipe_last);
    cudaSetDevice(cur);
    P->pipe_ready = false;
  }
  for (int i = 0; i < 3; ++i) {
    if ((err = cudaStreamCreateWithFlags(&P->pipe[i], cudaStreamNonBlocking)) != cudaSuccess)
      return err;
    for (int j = 0; j < hx_host_slots; ++j)
      if ((err = cudaEventCreateWithFlags(&P->ev[i][j], cudaEventDisableTiming)) != cudaSuccess)
        return err;
  }
  if ((err = cudaEventCreateWithFlags(&P->pipe_last, cudaEventDisableTiming)) != cudaSuccess)
    return err;
  // nothing recorded yet: waiting on it is a no-op
  P->pipe_dev = dev;
  P->pipe_ready = true;
  P->pipe_cont = false;  // fresh slot events: the next overlapped call starts a new sequence
  return cudaSuccess;
}

}  // namespace hx

extern "C" {

int hx_apply_host(const hx_plan* Pc, const double* q_host, const double* factors,
                  double* out_host, int64_t n_el, int64_t chunk_el, void* work, int* flag,
                  void* stream) {
  return hx_apply_host_ex(Pc, q_host, factors, out_host, n_el, chunk_el, work, flag, 0u,
                          stream);
}

int hx_apply_host_ex(const hx_plan* Pc, const double* q_host, const double* factors,
                     double* out_host, int64_t n_el, int64_t chunk_el, void* work, int* flag,
                     unsigned flags, void* stream) {
  if (!Pc || n_el < 0 || chunk_el <= 0 || (flags & ~HX_HOST_OVERLAP)) return HX_EINVAL;
  if (n_el == 0) return HX_OK;
  if (!q_host || !factors || !out_host || !work) return HX_EINVAL;
  hx_plan* P = const_cast<hx_plan*>(Pc);  // lazily owned pipeline resources
  hx::NvtxRange range(hx::range_name(*P, "host"));
  std::lock_guard<std::mutex> lock(P->pipe_mu);
  cudaStream_t caller = static_cast<cudaStream_t>(stream);
  cudaError_t err = pipe_setup(P);
  if (err != cudaSuccess) return cuda_status(err);
  const int64_t n3 = int64_t(P->n) * P->n * P->n;
  constexpr int S = hx_host_slots;
  double* wq[S];
  double* wo[S];
  double* base = static_cast<double*>(work);
  for (int i = 0; i < S; ++i) {
    wq[i] = base + int64_t(i) * chunk_el * n3;
    wo[i] = base + int64_t(S + i) * chunk_el * n3;
  }
  cudaStream_t s_in = P->pipe[0], s_k = P->pipe[1], s_out = P->pipe[2];
  cudaEvent_t* e_in = P->ev[0];
  cudaEvent_t* e_k = P->ev[1];
  cudaEvent_t* e_out = P->ev[2];
  const bool overlap = (flags & HX_HOST_OVERLAP) != 0;
  if (!overlap) {
    // Stream-ordered like every other entry point: all three pipeline
    // streams start after what the caller queued before this call -- the
    // work that produces q_host (e.g. an earlier call's D2H into it),
    // earlier users of `work`, factor generation.
    cudaEvent_t start;
    if ((err = cudaEventCreateWithFlags(&start, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_status(err);
    cudaEventRecord(start, caller);
    cudaStreamWaitEvent(s_in, start, 0);
    cudaStreamWaitEvent(s_k, start, 0);
    cudaStreamWaitEvent(s_out, start, 0);
    cudaEventDestroy(start);  // released once recorded work completes
  }
  // After the plan's previous host-pipeline call, whatever stream it came
  // from (the pipeline streams and slot events are shared): a full drain,
  // or -- HX_HOST_OVERLAP with the same workspace and chunking -- per slot,
  // continuing the previous call's slot sequence.
  const bool cont = overlap && P->pipe_cont && P->pipe_work == work && P->pipe_chunk == chunk_el;
  const int64_t seq = cont ? P->pipe_seq : 0;
  if (!cont) {
    cudaStreamWaitEvent(s_in, P->pipe_last, 0);
    cudaStreamWaitEvent(s_k, P->pipe_last, 0);
  }
  std::vector<int64_t> sched;
  if (overlap) {  // uniform chunks: back-to-back calls keep the pipe full
    for (int64_t e = 0; e < n_el; e += chunk_el) sched.push_back(std::min(chunk_el, n_el - e));
  } else {
    sched = chunk_schedule(n_el, chunk_el);
  }
  const int64_t nchunks = int64_t(sched.size());
  int64_t e0 = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t g = seq + c;  // position in the slot sequence
    const int slot = int(g % S);
    const int64_t ne = sched[c];
    const size_t bytes = size_t(ne * n3) * sizeof(double);
    if (g >= S) cudaStreamWaitEvent(s_in, e_k[slot], 0);  // kernel g-S done reading wq[slot]
    cudaMemcpyAsync(wq[slot], q_host + e0 * n3, bytes, cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(e_in[slot], s_in);
    cudaStreamWaitEvent(s_k, e_in[slot], 0);
    if (g >= S) cudaStreamWaitEvent(s_k, e_out[slot], 0);  // D2H g-S done with wo[slot]
    if ((err = launch_apply(*P, wq[slot], factors + e0 * P->elem_stride, wo[slot], ne, flag, s_k)) !=
        cudaSuccess) {
      // copies into / out of the caller's host buffers may still be in
      // flight: finish them before handing the buffers back
      cudaStreamSynchronize(s_in);
      cudaStreamSynchronize(s_k);
      cudaStreamSynchronize(s_out);
      P->pipe_cont = false;
      return cuda_status(err);
    }
    cudaEventRecord(e_k[slot], s_k);
    cudaStreamWaitEvent(s_out, e_k[slot], 0);
    cudaMemcpyAsync(out_host + e0 * n3, wo[slot], bytes, cudaMemcpyDeviceToHost, s_out);
    cudaEventRecord(e_out[slot], s_out);
    e0 += ne;
  }
  // D2H is in order on one stream, and it runs after every H2D and kernel
  // of the call: its last chunk done means the whole pipeline is
  cudaEventRecord(P->pipe_last, s_out);
  cudaStreamWaitEvent(caller, P->pipe_last, 0);
  P->pipe_seq = seq + nchunks;
  P->pipe_work = work;
  P->pipe_chunk = chunk_el;
  P->pipe_cont = overlap;
  return cuda_status(cudaGetLastError());
}

int64_t hx_energy_partials(void) { return int64_t(32) * sm_count(); }

int hx_apply_energy(const hx_plan* P, const double* q, const double* factors, double* out,
                    int64_t n_el, double* partials, int64_t n_partials, double* energy,
                    int* flag, void* stream) {
  if (!P || n_el < 0 || !partials || !energy) return HX_EINVAL;
  if (n_el > 0 && (!q || !factors || !out)) return HX_EINVAL;
  if (n_partials < hx_energy_partials()) return HX_EINVAL;
  hx::NvtxRange range(hx::range_name(*P, "energy"));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t err = cudaMemsetAsync(partials, 0, sizeof(double) * n_partials, s);
  if (err == cudaSuccess) err = launch_apply(*P, q, factors, out, n_el, flag, s, partials, kApplyPdl);
  if (err == cudaSuccess) err = launch_sum(partials, int(n_partials), energy, s);
  return cuda_status(err);
}

int hx_apply_energy_dir(const hx_plan* P, double* p, const double* r, const double* rr_new,
                        const double* rr_old, const double* factors, double* out, int64_t n_el,
                        double* partials, int64_t n_partials, double* energy, int* flag,
                        void* stream) {
  if (!P || n_el < 0 || !partials || !energy || !rr_new || !rr_old) return HX_EINVAL;
  if (n_el > 0 && (!p || !r || !factors || !out || p == r || out == p || out == r))
    return HX_EINVAL;
  if (n_partials < hx_energy_partials()) return HX_EINVAL;
  hx::NvtxRange range(hx::range_name(*P, "energy"));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const DirArgs dir{p, r, rr_new, rr_old};
  cudaError_t err = cudaMemsetAsync(partials, 0, sizeof(double) * n_partials, s);
  if (err == cudaSuccess)
    err = launch_apply(*P, p, factors, out, n_el, flag, s, partials, kApplyPdl, &dir);
  if (err == cudaSuccess) err = launch_sum(partials, int(n_partials), energy, s);
  return cuda_status(err);
}

int hx_dot(const double* u, const double* v, int64_t n, double* partials, int64_t n_partials,
           double* result, void* stream) {
  hx::NvtxRange range("hx_dot");
  if (n < 0 || !partials || !result || (n > 0 && (!u || !v))) return HX_EINVAL;
  if (n_partials < hx_energy_partials()) return HX_EINVAL;
  return cuda_status(launch_dot(u, v, n, partials, result, static_cast<cudaStream_t>(stream)));
}

int hx_cg_update(double* x, const double* p, double* r, const double* ap, int64_t n,
                 const double* rr, const double* pap, double* partials, int64_t n_partials,
                 double* rr_new, void* stream) {
  hx::NvtxRange range("hx_cg_update");
  if (n < 0 || !rr || !pap || !partials || !rr_new) return HX_EINVAL;
  if (n > 0 && (!x || !p || !r || !ap)) return HX_EINVAL;
  if (n_partials < hx_energy_partials()) return HX_EINVAL;
  return cuda_status(launch_cg_update(x, p, r, ap, n, rr, pap, partials, rr_new,
                                      static_cast<cudaStream_t>(stream)));
}

int hx_cg_direction(double* p, const double* r, int64_t n, const double* rr_new,
                    const double* rr_old, void* stream) {
  hx::NvtxRange range("hx_cg_direction");
  if (n < 0 || !rr_new || !rr_old || (n > 0 && (!p || !r))) return HX_EINVAL;
  return cuda_status(launch_cg_direction(p, r, n, rr_new, rr_old,
                                         static_cast<cudaStream_t>(stream)));
}

static bool dss_args_ok(int side, int degree, int64_t e_begin, int64_t e_end) {
  // side <= 1600 keeps element indices below 2^32 (32-bit index math)
  return side >= 1 && side <= 1600 && degree >= 1 && degree <= 15 && e_begin >= 0 &&
         e_begin <= e_end && e_end <= int64_t(side) * side * side;
}

int hx_dss(const double* in, double* out, int side, int degree, int mask, int64_t e_begin,
           int64_t e_end, int64_t in_base, void* stream) {
  hx::NvtxRange range("hx_dss");
  if (!dss_args_ok(side, degree, e_begin, e_end) || in_base < 0 || in_base > e_begin)
    return HX_EINVAL;
  if (e_end == e_begin) return HX_OK;
  if (!in || !out || in == out) return HX_EINVAL;
  return cuda_status(launch_dss(in, out, side, degree, mask != 0, e_begin, e_end, in_base,
                                static_cast<cudaStream_t>(stream)));
}

int hx_dot_dss(const double* u, const double* v, int side, int degree, int64_t e_begin,
               int64_t e_end, double* partials, int64_t n_partials, double* result,
               void* stream) {
  hx::NvtxRange range("hx_dot_dss");
  if (!dss_args_ok(side, degree, e_begin, e_end) || !partials || !result) return HX_EINVAL;
  if (e_end > e_begin && (!u || !v)) return HX_EINVAL;
  if (n_partials < hx_energy_partials()) return HX_EINVAL;
  return cuda_status(launch_dot_dss(u, v, side, degree, e_begin, e_end, partials, result,
                                    static_cast<cudaStream_t>(stream)));
}

int hx_dss_inplace(double* u, int side, int degree, int64_t buf_begin, int64_t buf_end,
                   void* stream) {
  hx::NvtxRange range("hx_dss_inplace");
  if (!dss_args_ok(side, degree, buf_begin, buf_end)) return HX_EINVAL;
  if (buf_end > buf_begin && !u) return HX_EINVAL;
  return cuda_status(launch_dss_inplace(u, side, degree, buf_begin, buf_end,
                                        static_cast<cudaStream_t>(stream)));
}

int hx_cg_update_assembled(double* x, const double* p, double* r, double* ap, int side,
                           int degree, int mask, int64_t e_begin, int64_t e_end, int64_t ap_base,
                           int64_t ap_end, const double* rr, const double* pap, double* partials,
                           int64_t n_partials, double* rr_new, void* stream) {
  hx::NvtxRange range("hx_cg_update_assembled");
  if (!dss_args_ok(side, degree, e_begin, e_end) || ap_base < 0 || ap_base > e_begin ||
      ap_end < e_end || ap_end > int64_t(side) * side * side)
    return HX_EINVAL;
  if (!rr || !pap || !partials || !rr_new) return HX_EINVAL;
  if (e_end > e_begin && (!x || !p || !r || !ap)) return HX_EINVAL;
  if (n_partials < hx_energy_partials()) return HX_EINVAL;
  return cuda_status(launch_cg_update_assembled(x, p, r, ap, side, degree, mask != 0, e_begin,
                                                e_end, ap_base, ap_end, rr, pap, partials,
                                                rr_new, static_cast<cudaStream_t>(stream)));
}

int hx_measure_smem_bandwidth(double* bytes_per_s, void* stream) {
  if (!bytes_per_s) return HX_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* sink = nullptr;
  cudaError_t err = cudaMalloc(&sink, sizeof(double) * 4096);
  if (err != cudaSuccess) return cuda_status(err);
  const int iters = 4096;
  float ms = 0.f;
  err = launch_smem_probe(sink, iters, &ms, s);
  cudaFree(sink);
  if (err != cudaSuccess) return cuda_status(err);
  const double bytes = double(sm_count()) * 2 * 512 * double(iters) * 8 * 4 * sizeof(double);
  *bytes_per_s = bytes / (ms * 1e-3);
  return HX_OK;
}

const char* hx_strerror(int status) {
  switch (status) {
    case HX_OK:
      return "success";
    case HX_EINVAL:
      return "invalid argument";
    case HX_ENONFINITE:
      return "field vector contains non-finite values";
    case HX_EDEGENERATE:
      return "non-positive Jacobian determinant";
    case HX_ECUDA:
      return g_last_cuda[0] ? g_last_cuda : "CUDA error";
    case HX_ENOMEM:
      return "out of host memory";
    default:
      return "unknown status";
  }
}

int hx_device_ok(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major == 10 && minor == 0;
}

}  // extern "C"
