// Element helpers on device (reference operators.py:352-364):
//
//   interpolate_to_gl(q_e, I) = I_k ( I_r ( I_s q_e ) )   (n,n,n) -> (m,m,m)
//   project_to_gll(t_e, I)    = I^T applied along the same three axes
//
// batched over elements.  Same building blocks as the BP1.0 kernel (BP1.0 is
// exactly project(GwJ * interpolate(q)), these are its two halves without the
// pointwise scale), in the (s, r, t) stage order that ends / starts with
// coalesced k-lines on the GL side (Cfg<kINTERP, N>: X is (n,m,n), Y is
// (n,m,m)).  Stage order:
//
//   interpolate  S1 j-lines (k,i)  src -> I_s -> X ; S2 i-lines (k,a) X -> I_r -> Y ;
//                S3 k-lines (a,c)  Y -> I_t -> dst (HBM, coalesced)
//   project      S1 k-lines (a,c)  src (HBM, coalesced) -> I_t^T -> Y ;
//                S2 i-lines (k,a)  Y -> I_r^T -> X ; S3 j-lines (k,i) X -> I_s^T -> dst
//
// The reference contracts axis 1, 2, 0 in both directions; the projection
// here contracts 0, 2, 1 (adjoint order), a floating-point reassociation only.
#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {

template <int N>
struct InterpParams {
  Fold<N + 2, N + 1> I;   // GLL -> GL
  Fold<N + 1, N + 2> It;  // GL -> GLL (transpose)
  const double* src;
  double* dst;
  int64_t n_el;
  int* flag;
};

template <int N, bool PROJECT>
__global__ void __launch_bounds__(Cfg<kINTERP, N>::NT)
    interp_kernel(const __grid_constant__ InterpParams<N> p) {
  using C = Cfg<kINTERP, N>;
  constexpr int n = N + 1, m = N + 2, n2 = n * n, n3 = n2 * n, m2 = m * m, m3 = m2 * m;
  constexpr int EPB = C::EPB, NT = C::NT;
  constexpr Lay LX = C::L[0], LY = C::L[1];
  constexpr int EX = C::EBUF[0], EY = C::EBUF[1];
  // lane order of the i-line stages (S2, S4), see iline_coords; the j-line
  // stages (S1, S5) touch HBM and keep i fastest
  constexpr int IORD = C::ORD;
  constexpr bool JKF = false;
  extern __shared__ double smem[];
  double* const X = smem;
  double* const Y = X + EPB * EX;
  const int tid = threadIdx.x;
  const int64_t ntiles = (p.n_el + EPB - 1) / EPB;
  constexpr int SRC = PROJECT ? m3 : n3, DST = PROJECT ? n3 : m3;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t e0 = tile * EPB;
    const int ne = int(min64(EPB, p.n_el - e0));
    if constexpr (!PROJECT) {
      for_lines<EPB * n2, NT>(tid, [&](int g) {
        const int el = g / n2, ln = g % n2;
        if (el >= ne) return;
        int k, i;
        line_coords<n, n, JKF>(ln, k, i);
        const double* src = p.src + (e0 + el) * SRC + k * n2 + i;
        double x[n], y[m];
#pragma unroll
        for (int t = 0; t < n; ++t) x[t] = src[t * n];
        const bool bad = any_nonfinite(x);
        if (bad && p.flag) atomicOr(p.flag, 1);
        fold_apply<m, n, 1>(p.I, x, y);
        double* dst = X + el * EX + LX.kofs(k) + i;
#pragma unroll
        for (int t = 0; t < m; ++t) dst[t * LX.s1] = y[t];
      });
      __syncthreads();
      for_lines<EPB * n * m, NT>(tid, [&](int g) {
        const int el = g / (n * m), ln = g % (n * m);
        if (el >= ne) return;
        int k, a;
        iline_coords<n, m, IORD>(ln, k, a);
        const double* src = X + el * EX + LX.kofs(k) + a * LX.s1;
        double x[n], y[m];
#pragma unroll
        for (int t = 0; t < n; ++t) x[t] = src[t];
        fold_apply<m, n, 1>(p.I, x, y);
        double* dst = Y + el * EY + LY.kofs(k) + a * LY.s1;
#pragma unroll
        for (int t = 0; t < m; ++t) dst[t] = y[t];
      });
      __syncthreads();
      for_lines<EPB * m2, NT>(tid, [&](int g) {
        const int el = g / m2, ln = g % m2;
        if (el >= ne) return;
        const int a = ln / m, c = ln % m;
        const double* line = Y + el * EY + a * LY.s1 + c;
        double x[n], y[m];
#pragma unroll
        for (int t = 0; t < n; ++t) x[t] = line[LY.kofs(t)];
        fold_apply<m, n, 1>(p.I, x, y);
        double* dst = p.dst + (e0 + el) * DST + ln;
#pragma unroll
        for (int t = 0; t < m; ++t) st_stream(dst + t * m2, y[t]);
      });
    } else {
      for_lines<EPB * m2, NT>(tid, [&](int g) {
        const int el = g / m2, ln = g % m2;
        if (el >= ne) return;
        const int a = ln / m, c = ln % m;
        const double* src = p.src + (e0 + el) * SRC + ln;
        double x[m], y[n];
#pragma unroll
        for (int t = 0; t < m; ++t) x[t] = src[t * m2];
        const bool bad = any_nonfinite(x);
        if (bad && p.flag) atomicOr(p.flag, 1);
        fold_apply<n, m, 1>(p.It, x, y);
        double* line = Y + el * EY + a * LY.s1 + c;
#pragma unroll
        for (int t = 0; t < n; ++t) line[LY.kofs(t)] = y[t];
      });
      __syncthreads();
      for_lines<EPB * n * m, NT>(tid, [&](int g) {
        const int el = g / (n * m), ln = g % (n * m);
        if (el >= ne) return;
        int k, a;
        iline_coords<n, m, IORD>(ln, k, a);
        const double* src = Y + el * EY + LY.kofs(k) + a * LY.s1;
        double x[m], y[n];
#pragma unroll
        for (int t = 0; t < m; ++t) x[t] = src[t];
        fold_apply<n, m, 1>(p.It, x, y);
        double* dst = X + el * EX + LX.kofs(k) + a * LX.s1;
#pragma unroll
        for (int t = 0; t < n; ++t) dst[t] = y[t];
      });
      __syncthreads();
      for_lines<EPB * n2, NT>(tid, [&](int g) {
        const int el = g / n2, ln = g % n2;
        if (el >= ne) return;
        int k, i;
        line_coords<n, n, JKF>(ln, k, i);
        const double* src = X + el * EX + LX.kofs(k) + i;
        double x[m], y[n];
#pragma unroll
        for (int t = 0; t < m; ++t) x[t] = src[t * LX.s1];
        fold_apply<n, m, 1>(p.It, x, y);
        double* dst = p.dst + (e0 + el) * DST + k * n2 + i;
#pragma unroll
        for (int t = 0; t < n; ++t) st_stream(dst + t * n, y[t]);
      });
    }
    __syncthreads();  // X / Y are rewritten by the next tile
  }
}

template <int N, bool PROJECT>
static cudaError_t launch_interp_t(const InterpParams<N>& prm, cudaStream_t s) {
  using C = Cfg<kINTERP, N>;
  constexpr int smem = (C::EBUF[0] + C::EBUF[1]) * C::EPB * int(sizeof(double));
  const int64_t ntiles = (prm.n_el + C::EPB - 1) / C::EPB;
  unsigned grid = 0;
  const cudaError_t err = persistent_grid<interp_kernel<N, PROJECT>>(C::NT, smem, ntiles, &grid);
  if (err != cudaSuccess) return err;
  interp_kernel<N, PROJECT><<<grid, C::NT, smem, s>>>(prm);
  return cudaGetLastError();
}

template <int N>
static cudaError_t launch_interp_n(const double* interp, int project, const double* src,
                                   double* dst, int64_t n_el, int* flag, cudaStream_t s) {
  constexpr int n = N + 1, m = N + 2;
  InterpParams<N> prm;
  double it[n * m];
  fill_fold(prm.I, interp);
  transpose(interp, m, n, it);
  fill_fold(prm.It, it);
  prm.src = src;
  prm.dst = dst;
  prm.n_el = n_el;
  prm.flag = flag;
  return project ? launch_interp_t<N, true>(prm, s) : launch_interp_t<N, false>(prm, s);
}

cudaError_t launch_interp(int degree, const double* interp, int project, const double* src,
                          double* dst, int64_t n_el, int* flag, cudaStream_t s) {
  switch (degree) {
#define HX_CASE(N) \
  case N:          \
    return launch_interp_n<N>(interp, project, src, dst, n_el, flag, s);
    HX_CASE(1) HX_CASE(2) HX_CASE(3) HX_CASE(4) HX_CASE(5) HX_CASE(6) HX_CASE(7) HX_CASE(8)
    HX_CASE(9) HX_CASE(10) HX_CASE(11) HX_CASE(12) HX_CASE(13) HX_CASE(14) HX_CASE(15)
#undef HX_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace hx
