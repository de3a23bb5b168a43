// Shared device helpers for the BP1.0 / BP3.5 / BP3.0 element kernels.
//
// Every 1-D operator the matvecs apply is (anti-)centro-symmetric:
//   I  (GLL->GL)        I[a][b]  =  I[R-1-a][C-1-b]     (reference_ops.py:42-44)
//   D, D~ (collocation)  D[a][b]  = -D[R-1-a][C-1-b]
// and so are their transposes.  `Fold` stores such an R x C matrix as its
// even/odd halves; `fold_apply` applies it to one line held in registers with
// about half the multiply-adds of the dense product.  The coefficients live in
// the kernel's __grid_constant__ parameter block, i.e. the constant bank, and
// every lane of a warp reads the same entry at the same time, so they are
// free uniform DFMA operands: no registers and no shared memory are spent on
// the 1-D matrices.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler injects

// tuning builds substitute an alternative generated table
#ifdef HX_LAYOUTS_FILE
#include HX_LAYOUTS_FILE
#else
#include "hx_layouts.h"
#endif

namespace hx {

enum { kBP1 = 10, kBP35 = 35, kBP3 = 30, kINTERP = 11 };  // kINTERP: hx_interp.cu shapes

template <int R, int C>
struct Fold {
  static constexpr int HI = C / 2, HO = R / 2;
  static constexpr bool MID_IN = C & 1, MID_OUT = R & 1;
  static constexpr int RO = (R + 1) / 2;  // output rows incl. the middle one
  // e[a][b] = (M[a][b] + M[a][C-1-b]) / 2 for b < HI; e[a][HI] = M[a][HI] (odd C)
  double e[RO][HI + (MID_IN ? 1 : 0)];
  // o[a][b] = (M[a][b] - M[a][C-1-b]) / 2
  double o[RO][HI > 0 ? HI : 1];
};

// y = M x for a folded (SIGN=+1 centro-symmetric, SIGN=-1 anti) matrix.
template <int R, int C, int SIGN>
__device__ __forceinline__ void fold_apply(const Fold<R, C>& F, const double (&x)[C],
                                           double (&y)[R]) {
  constexpr int HI = C / 2, HO = R / 2;
  constexpr bool MID_IN = C & 1, MID_OUT = R & 1;
  double xe[HI], xo[HI];
#pragma unroll
  for (int b = 0; b < HI; ++b) {
    xe[b] = x[b] + x[C - 1 - b];
    xo[b] = x[b] - x[C - 1 - b];
  }
#pragma unroll
  for (int a = 0; a < HO; ++a) {
    double ye = F.e[a][0] * xe[0];
    double yo = F.o[a][0] * xo[0];
#pragma unroll
    for (int b = 1; b < HI; ++b) {
      ye = fma(F.e[a][b], xe[b], ye);
      yo = fma(F.o[a][b], xo[b], yo);
    }
    if constexpr (MID_IN) ye = fma(F.e[a][HI], x[HI], ye);
    y[a] = ye + yo;
    y[R - 1 - a] = (SIGN > 0) ? ye - yo : yo - ye;
  }
  if constexpr (MID_OUT) {
    if constexpr (SIGN > 0) {
      double ye = F.e[HO][0] * xe[0];
#pragma unroll
      for (int b = 1; b < HI; ++b) ye = fma(F.e[HO][b], xe[b], ye);
      if constexpr (MID_IN) ye = fma(F.e[HO][HI], x[HI], ye);
      y[HO] = ye;
    } else {
      double yo = F.o[HO][0] * xo[0];
#pragma unroll
      for (int b = 1; b < HI; ++b) yo = fma(F.o[HO][b], xo[b], yo);
      y[HO] = yo;
    }
  }
}

// Host: fill a Fold from a dense row-major R x C matrix.
template <int R, int C>
inline void fill_fold(Fold<R, C>& F, const double* M) {
  constexpr int HI = C / 2;
  for (int a = 0; a < Fold<R, C>::RO; ++a) {
    for (int b = 0; b < HI; ++b) {
      const double lo = M[a * C + b], hi = M[a * C + (C - 1 - b)];
      F.e[a][b] = 0.5 * (lo + hi);
      F.o[a][b] = 0.5 * (lo - hi);
    }
    if (C & 1) F.e[a][HI] = M[a * C + HI];
  }
}

// Host: transpose a dense row-major R x C matrix into C x R.
inline void transpose(const double* M, int R, int C, double* T) {
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < C; ++b) T[b * R + a] = M[a * C + b];
}

// Fire-and-forget DRAM->L2 prefetch of a byte range (TMA bulk engine).  The
// range is shrunk to 16-byte granularity so it never leaves the allocation.
__device__ __forceinline__ void prefetch_l2(const void* ptr, size_t bytes) {
  uintptr_t lo = (reinterpret_cast<uintptr_t>(ptr) + 15) & ~uintptr_t(15);
  uintptr_t hi = (reinterpret_cast<uintptr_t>(ptr) + bytes) & ~uintptr_t(15);
  constexpr uintptr_t kChunk = 1u << 20;
  for (; lo < hi; lo += kChunk) {
    uintptr_t n = hi - lo < kChunk ? hi - lo : kChunk;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((unsigned)n)
                 : "memory");
  }
}

// ---- bulk-copy (TMA engine, non-tensor) staging with an mbarrier ----------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Arm the barrier's current phase with this thread's arrival and `bytes` of
// expected bulk-copy transactions.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "HX_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HX_WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Generic-proxy accesses to shared memory made before this (and ordered by a
// barrier) are ordered before later async-proxy (bulk copy) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// HBM -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-byte
// aligned) completing as transactions on `bar`.  The source is streamed once:
// L2 evict-first so it does not displace data still to be read.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Host-side NVTX range over one C-ABI call (SURVEY.md §5 tracing): visible in
// nsys / ncu timelines, ~free when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

int sm_count();

// Per-device one-time launch setup of kernel `K`: the dynamic shared-memory
// opt-in (a function attribute, which lives in each device's context) and
// the resident-CTA count the persistent grids are sized by.  Cached per
// (kernel, device ordinal), so one process can drive several GPUs; the
// setup is idempotent, so two threads racing on a first launch are harmless.
constexpr int kMaxDevices = 64;

template <auto K>
inline cudaError_t resident_blocks(int threads, int smem, int* blocks) {
  static std::atomic<int> cache[kMaxDevices];  // 0: not set up on that device yet
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  if (dev >= 0 && dev < kMaxDevices) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) {
      *blocks = c;
      return cudaSuccess;
    }
  }
  if (smem > 48 * 1024) {
    err = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
  }
  int b = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, K, threads, smem);
  if (err != cudaSuccess) return err;
  if (b < 1) b = 1;
  if (dev >= 0 && dev < kMaxDevices) cache[dev].store(b, std::memory_order_relaxed);
  *blocks = b;
  return cudaSuccess;
}

// CG search-direction update fused into a matvec's first load
// (hx_apply_energy_dir): the kernel reads p_old and r where it would read q,
// forms p = r + beta p_old with beta = rr_new / rr_old -- hx_cg_direction's
// formula, bit for bit -- stores p back and applies the operator to it, so
// the direction update costs no pass of its own (DirArgs: hx_plan.h).
// Load one line of q, or (DIR) form and store the line of p = r + beta p_old.
template <bool DIR, int L, int STRIDE, class Dir>
__device__ __forceinline__ void load_line(const double* q, const Dir& d, double beta,
                                          int64_t off, double (&x)[L]) {
  if constexpr (DIR) {
    // all loads before any store: the stores may alias the loads as far as
    // the compiler knows, and interleaving them would serialise the line's
    // 2L loads into L dependent round trips
    const double* __restrict__ pp = d.p + off;
    const double* __restrict__ rp = d.r + off;
    double pv[L];
#pragma unroll
    for (int t = 0; t < L; ++t) {
      pv[t] = pp[t * STRIDE];
      x[t] = rp[t * STRIDE];
    }
#pragma unroll
    for (int t = 0; t < L; ++t) x[t] = fma(beta, pv[t], x[t]);
#pragma unroll
    for (int t = 0; t < L; ++t) d.p[off + int64_t(t) * STRIDE] = x[t];
  } else {
#pragma unroll
    for (int t = 0; t < L; ++t) x[t] = q[off + int64_t(t) * STRIDE];
  }
}

// Programmatic dependent launch (PDL).  A persistent element kernel launched
// with cudaLaunchAttributeProgrammaticStreamSerialization may start while
// the previous kernel of the stream is still retiring its last CTAs: it only
// issues L2 prefetch hints before pdl_wait(), which returns once the
// previous grid has completed and its memory is visible, so every load of
// q / factors and every store of out keeps plain stream order.
// pdl_allow_dependents() lets the next such launch do the same with ours.
// Both are no-ops for a plain launch.
__device__ __forceinline__ void pdl_allow_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <auto K, class Prm>
inline cudaError_t launch_kernel(unsigned grid, int threads, int smem, cudaStream_t s, bool pdl,
                                 const Prm& prm) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, K, prm);
}

// Persistent grid for `ntiles` tiles of kernel K on the current device.
template <auto K>
inline cudaError_t persistent_grid(int threads, int smem, int64_t ntiles, unsigned* grid) {
  int b = 0;
  cudaError_t err = resident_blocks<K>(threads, smem, &b);
  if (err != cudaSuccess) return err;
  *grid = unsigned(min64(ntiles, int64_t(b) * sm_count()));
  return cudaSuccess;
}

__device__ __forceinline__ bool nonfinite(double v) {
  // exponent all ones <=> inf or nan
  return (__double_as_longlong(v) & 0x7ff0000000000000ll) == 0x7ff0000000000000ll;
}

// Any inf / nan in a loaded line, on the integer pipe: (~hi & EXP) is 0 iff
// the exponent bits of the high word are all ones; one LOP3 + IMNMX per value
// instead of an FP64-pipe DSETP (the FP64 pipe is the busier one).
template <int L>
__device__ __forceinline__ bool any_nonfinite(const double (&x)[L]) {
  unsigned acc = 0x7ff00000u;
#pragma unroll
  for (int t = 0; t < L; ++t)
    acc = min(acc, ~static_cast<unsigned>(__double2hiint(x[t])) & 0x7ff00000u);
  return acc == 0u;
}

// Load the j-line (k, i) = divmod(line, n) of one element's (n, n, n) field:
// q[k][0..n-1][i] -- 8n-byte runs across the lanes of a warp.
template <int n>
__device__ __forceinline__ void load_jline(const double* qe, int line, double (&x)[n]) {
  const double* src = qe + (line / n) * n * n + line % n;
#pragma unroll
  for (int t = 0; t < n; ++t) x[t] = src[t * n];
}

// Load the k-line (j, i) = divmod(line, n): q[0..n-1][j][i], coalesced over
// consecutive lines.
template <int n>
__device__ __forceinline__ void load_kline(const double* qe, int line, double (&x)[n]) {
  const double* src = qe + line;
#pragma unroll
  for (int t = 0; t < n; ++t) x[t] = src[t * n * n];
}

// Streaming store: the output is never re-read by the kernel, keep the
// prefetched inputs resident in L2 instead.
__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }

// Run f(line) for this thread's lines of a stage with TOT lines on NT threads
// (line = tid, tid + NT, ...); a single guarded call when NT >= TOT.
template <int TOT, int NT, class F>
__device__ __forceinline__ void for_lines(int tid, F&& f) {
#pragma unroll
  for (int it = 0; it < (TOT + NT - 1) / NT; ++it) {
    const int g = tid + it * NT;
    if (g < TOT) f(g);
  }
}

// Coordinates (first, second) of line `ln` of a stage whose lines form an
// (A x B) grid: row-major (second fastest across lanes) or, with FIRST_FAST,
// first fastest.  The generated ORD flags pick the order per stage so that
// the lanes of a half-warp hit distinct shared-memory banks.
template <int A, int B, bool FIRST_FAST>
__device__ __forceinline__ void line_coords(int ln, int& first, int& second) {
  if constexpr (FIRST_FAST) {
    first = ln % A;
    second = ln / A;
  } else {
    first = ln / B;
    second = ln % B;
  }
}

// (k, a) of i-line `ln` over an (n x m) grid of lines in the lane order ORD
// picked by tools/gen_layouts.py: 0 a fastest; 2 k fastest; 4 k-paired (k
// pairs outermost, then a, then the k parity fastest; an odd last slice is
// enumerated alone) -- paired with k-paired layouts (Lay::sq) this keeps both
// the i-lines and the (k, i) j-lines of a tensor free of bank conflicts.
template <int n, int m, int ORD>
__device__ __forceinline__ void iline_coords(int ln, int& k, int& a) {
  if constexpr (ORD == 2) {
    k = ln % n;
    a = ln / n;
  } else if constexpr (ORD == 4) {
    constexpr int FULL = (n / 2) * 2 * m;
    if (FULL == n * m || ln < FULL) {
      const int kh = ln / (2 * m), r = ln % (2 * m);
      k = 2 * kh + (r & 1);
      a = r >> 1;
    } else {
      k = n - 1;
      a = ln - FULL;
    }
  } else {
    k = ln / m;
    a = ln % m;
  }
}

// Sum of one double per thread over the CTA (result valid in thread 0).
// `scratch` is shared memory of at least NT/32 doubles that no thread is
// still reading.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (NT + 31) / 32; ++w) s += scratch[w];
  return s;
}

// Shared memory per CTA in doubles: the per-element tensor buffers, plus for
// the TMA q-staged BP1.0 shape the staged q tile and 2 doubles (16 bytes,
// keeps the staging 16-byte aligned) holding its mbarrier.
template <int BP, int N>
constexpr int smem_doubles() {
  using C = Cfg<BP, N>;
  int s = 0;
  for (int b = 0; b < int(sizeof(C::EBUF) / sizeof(int)); ++b) s += C::EBUF[b];
  s *= C::EPB;
  if (C::QS > 0) s += 2 + C::EPB * (N + 1) * C::QS;
  return s;
}

}  // namespace hx
