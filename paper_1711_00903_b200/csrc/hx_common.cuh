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
#include <cstdint>
#include <cuda_runtime.h>

// tuning builds substitute an alternative generated table
#ifdef HX_LAYOUTS_FILE
#include HX_LAYOUTS_FILE
#else
#include "hx_layouts.h"
#endif

namespace hx {

enum { kBP1 = 10, kBP35 = 35, kBP3 = 30 };

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

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ bool nonfinite(double v) {
  // exponent all ones <=> inf or nan
  return (__double_as_longlong(v) & 0x7ff0000000000000ll) == 0x7ff0000000000000ll;
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

template <int BP, int N>
constexpr int smem_doubles() {
  using C = Cfg<BP, N>;
  int s = 0;
  for (int b = 0; b < int(sizeof(C::EBUF) / sizeof(int)); ++b) s += C::EBUF[b];
  return s * C::EPB;
}

}  // namespace hx
