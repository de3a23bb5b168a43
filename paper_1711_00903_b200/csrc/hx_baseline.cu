// Unfused "baseline" path: the paper's Kernel-1 structure on B200 (PAPER.md:518,
// "two additional global memory variables for storing intermediate results
// ... in all the loops, it reads from and writes to global memory") and the
// access pattern the reference's `variant="baseline"` counters charge
// (operators.py:170-200: every contraction pass reads and writes global
// memory).  Each 1-D contraction pass and each pointwise step is its own
// launch with its intermediate in HBM, in the reference's exact pass order
// (operators.py:208-268), so the fused kernels' speed-up over it is the
// paper's K1 -> K8/K10 story measured on this GPU.
//
//   BP1.0 (7 launches): I_s, I_r, I_t, * GwJ, I_s^T, I_r^T, I_t^T
//   BP3.5 (7):          D_r, D_s, D_t, chain rule (+ lam GwJ q), D_r^T, D_s^T, D_t^T (+=)
//   BP3.0 (13):         I x3, D~ x3, chain rule, D~^T x3 (+=), I^T x3
//
// Not a hot path: exercised by tests and bench.py's baseline report only.
#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {

constexpr int kBaseThreads = 256;

template <int R, int C>
struct LineOp {
  double M[R][C];  // row-major operator, out[a] = sum_b M[a][b] in[b]
};

// One thread per 1-D line of an (E, d0, d1, d2) tensor along axis `ax`
// (0 = k, 1 = j, 2 = i); the output has extent R along that axis.  ACC adds
// into the output instead of overwriting it.
template <int R, int C, bool ACC>
__global__ void __launch_bounds__(kBaseThreads)
    line_kernel(const __grid_constant__ LineOp<R, C> op, const double* __restrict__ in,
                double* __restrict__ out, int64_t n_el, int d0, int d1, int d2, int ax) {
  const int din[3] = {d0, d1, d2};
  int dout[3] = {d0, d1, d2};
  dout[ax] = R;
  const int lines_per_el = din[0] * din[1] * din[2] / din[ax];
  const int64_t total = n_el * lines_per_el;
  // strides of the contracted axis and of the two free axes, in and out
  const int sin2 = 1, sin1 = din[2], sin0 = din[1] * din[2];
  const int sout2 = 1, sout1 = dout[2], sout0 = dout[1] * dout[2];
  const int in_el = din[0] * din[1] * din[2], out_el = dout[0] * dout[1] * dout[2];
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = g / lines_per_el;
    const int l = int(g - e * lines_per_el);
    int ib, ob, is, os;  // base offsets and strides along the contracted axis
    if (ax == 0) {
      const int j = l / din[2], i = l % din[2];
      ib = j * sin1 + i * sin2; ob = j * sout1 + i * sout2; is = sin0; os = sout0;
    } else if (ax == 1) {
      const int k = l / din[2], i = l % din[2];
      ib = k * sin0 + i * sin2; ob = k * sout0 + i * sout2; is = sin1; os = sout1;
    } else {
      const int k = l / din[1], j = l % din[1];
      ib = k * sin0 + j * sin1; ob = k * sout0 + j * sout1; is = sin2; os = sout2;
    }
    const double* src = in + e * in_el + ib;
    double* dst = out + e * out_el + ob;
    double x[C];
#pragma unroll
    for (int b = 0; b < C; ++b) x[b] = src[b * is];
#pragma unroll
    for (int a = 0; a < R; ++a) {
      double y = 0.0;
#pragma unroll
      for (int b = 0; b < C; ++b) y = fma(op.M[a][b], x[b], y);
      dst[a * os] = ACC ? dst[a * os] + y : y;
    }
  }
}

// t[e][p] *= GwJ[e][p]  (operators.py:277); BP1.0's packed GwJ slot, which is
// i-major (hx_bp1.cu S3): point p = (k, j, i) of the (m, m, m) tensor at
// bp1_gwj_index(k, j, i, m, cfast)
__global__ void __launch_bounds__(kBaseThreads)
    scale_kernel(double* __restrict__ t, const double* __restrict__ fac, int64_t n_el, int m,
                 int64_t estride, int cfast, int* flag) {
  const int P = m * m * m;
  const int64_t total = n_el * P;
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = g / P;
    const int p = int(g - e * P);
    const int k = p / (m * m), j = (p / m) % m, i = p % m;
    const double v = t[g];
    if (flag && nonfinite(v)) atomicOr(flag, 1);  // non-finite q propagates into I q
    t[g] = fac[e * estride + bp1_gwj_index(k, j, i, m, cfast)] * v;
  }
}

// Chain rule in place (operators.py:252-255) and out = lam GwJ extra (:258)
__global__ void __launch_bounds__(kBaseThreads)
    chain_kernel(double* __restrict__ qr, double* __restrict__ qs, double* __restrict__ qt,
                 const double* extra, double* out,  // may alias (BP3.0 works in place)
                 const double* __restrict__ fac, int64_t n_el, int P, int64_t estride,
                 int64_t sstride, double lam, int* flag) {
  const int64_t total = n_el * P;
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = g / P;
    const int p = int(g - e * P);
    const double* f = fac + e * estride + p;
    const double grr = f[0], grs = f[sstride], grt = f[2 * sstride], gss = f[3 * sstride];
    const double gst = f[4 * sstride], gtt = f[5 * sstride], gwj = f[6 * sstride];
    const double a = qr[g], b = qs[g], c = qt[g];
    qr[g] = grr * a + grs * b + grt * c;
    qs[g] = grs * a + gss * b + gst * c;
    qt[g] = grt * a + gst * b + gtt * c;
    const double x = extra[g];
    if (flag && nonfinite(x)) atomicOr(flag, 1);
    out[g] = lam * gwj * x;
  }
}

static int base_blocks(int64_t work) {
  const int64_t want = (work + kBaseThreads - 1) / kBaseThreads;
  const int64_t cap = int64_t(sm_count()) * 16;
  return int(want < 1 ? 1 : (want < cap ? want : cap));
}

template <int R, int C>
static cudaError_t line(const double* M, bool transpose, const double* in, double* out,
                        int64_t n_el, int d0, int d1, int d2, int ax, bool acc,
                        cudaStream_t s) {
  LineOp<R, C> op;
  for (int a = 0; a < R; ++a)
    for (int b = 0; b < C; ++b) op.M[a][b] = transpose ? M[b * R + a] : M[a * C + b];
  const int d[3] = {d0, d1, d2};
  const int64_t lines = n_el * (int64_t(d0) * d1 * d2 / d[ax]);
  const int nb = base_blocks(lines);
  if (acc)
    line_kernel<R, C, true><<<nb, kBaseThreads, 0, s>>>(op, in, out, n_el, d0, d1, d2, ax);
  else
    line_kernel<R, C, false><<<nb, kBaseThreads, 0, s>>>(op, in, out, n_el, d0, d1, d2, ax);
  return cudaGetLastError();
}

#define HX_TRY(x)                              \
  do {                                         \
    cudaError_t e_ = (x);                      \
    if (e_ != cudaSuccess) return e_;          \
  } while (0)

// Interpolation passes (operators.py:208-219): axis 1, 2, 0; n^3 -> m^3.
template <int n, int m>
static cudaError_t interp3(const double* I, const double* q, double* t1, double* t2,
                           double* t3, int64_t E, cudaStream_t s) {
  HX_TRY((line<m, n>(I, false, q, t1, E, n, n, n, 1, false, s)));   // (n, m, n)
  HX_TRY((line<m, n>(I, false, t1, t2, E, n, m, n, 2, false, s)));  // (n, m, m)
  return line<m, n>(I, false, t2, t3, E, n, m, m, 0, false, s);     // (m, m, m)
}

// Projection passes (operators.py:222-232): I^T along axis 1, 2, 0; m^3 -> n^3.
template <int n, int m>
static cudaError_t project3(const double* I, const double* t, double* u1, double* u2,
                            double* out, int64_t E, cudaStream_t s) {
  HX_TRY((line<n, m>(I, true, t, u1, E, m, m, m, 1, false, s)));   // (m, n, m)
  HX_TRY((line<n, m>(I, true, u1, u2, E, m, n, m, 2, false, s)));  // (m, n, n)
  return line<n, m>(I, true, u2, out, E, m, n, n, 0, false, s);    // (n, n, n)
}

// Derivative chain + combine (operators.py:235-268) on a (p, p, p) tensor u:
// out = lam GwJ u + D^T_r rqr + D^T_s rqs + D^T_t rqt, summed in that order.
template <int p>
static cudaError_t diff_chain(const hx_plan& P, const double* u, double* qr, double* qs,
                              double* qt, double* out, const double* fac, int64_t E,
                              int* flag, cudaStream_t s) {
  HX_TRY((line<p, p>(P.diff, false, u, qr, E, p, p, p, 2, false, s)));
  HX_TRY((line<p, p>(P.diff, false, u, qs, E, p, p, p, 1, false, s)));
  HX_TRY((line<p, p>(P.diff, false, u, qt, E, p, p, p, 0, false, s)));
  chain_kernel<<<base_blocks(E * p * p * p), kBaseThreads, 0, s>>>(
      qr, qs, qt, u, out, fac, E, p * p * p, P.elem_stride, P.slot_stride, P.lam, flag);
  HX_TRY(cudaGetLastError());
  HX_TRY((line<p, p>(P.diff, true, qr, out, E, p, p, p, 2, true, s)));
  HX_TRY((line<p, p>(P.diff, true, qs, out, E, p, p, p, 1, true, s)));
  return line<p, p>(P.diff, true, qt, out, E, p, p, p, 0, true, s);
}

template <int N>
static cudaError_t baseline_n(const hx_plan& P, const double* q, const double* fac, double* out,
                              int64_t E, double* w, int* flag, cudaStream_t s) {
  constexpr int n = N + 1, m = N + 2, m3 = m * m * m;
  double* w0 = w;                 // workspace: 4 tensors of E * m^3 doubles
  double* w1 = w0 + E * m3;
  double* w2 = w1 + E * m3;
  double* w3 = w2 + E * m3;
  if (P.bp == HX_BP1) {
    HX_TRY((interp3<n, m>(P.interp, q, w0, w1, w2, E, s)));
    scale_kernel<<<base_blocks(E * m3), kBaseThreads, 0, s>>>(w2, fac, E, m, P.elem_stride,
                                                              int(bp1_gwj_cfast(P.degree)),
                                                              flag);
    HX_TRY(cudaGetLastError());
    return project3<n, m>(P.interp, w2, w0, w1, out, E, s);
  }
  if (P.bp == HX_BP35) return diff_chain<n>(P, q, w0, w1, w2, out, fac, E, flag, s);
  HX_TRY((interp3<n, m>(P.interp, q, w0, w1, w3, E, s)));               // t in w3
  HX_TRY((diff_chain<m>(P, w3, w0, w1, w2, w3, fac, E, flag, s)));        // a in w3
  return project3<n, m>(P.interp, w3, w0, w1, out, E, s);
}

// Dense (unfolded) element interpolation / projection for 1-D matrices the
// folded kernels cannot take (not centro-symmetric): the reference's
// contract_dim passes (operators.py:352-364) as line passes, intermediates in
// stream-ordered scratch.  Not a hot path.
template <int N>
static cudaError_t interp_dense_n(const double* I, int project, const double* src, double* dst,
                                  int64_t E, cudaStream_t s) {
  constexpr int n = N + 1, m = N + 2;
  const int64_t a = project ? m * n * m : n * m * n, b = project ? m * n * n : n * m * m;
  double* w = nullptr;
  HX_TRY(cudaMallocAsync(reinterpret_cast<void**>(&w), sizeof(double) * (a + b) * E, s));
  const cudaError_t err = project ? project3<n, m>(I, src, w, w + a * E, dst, E, s)
                                  : interp3<n, m>(I, src, w, w + a * E, dst, E, s);
  const cudaError_t fr = cudaFreeAsync(w, s);
  return err != cudaSuccess ? err : fr;
}

cudaError_t launch_interp_dense(int degree, const double* interp, int project, const double* src,
                                double* dst, int64_t n_el, cudaStream_t s) {
  if (n_el == 0) return cudaSuccess;
  switch (degree) {
#define HX_CASE(N) \
  case N:          \
    return interp_dense_n<N>(interp, project, src, dst, n_el, s);
    HX_CASE(1) HX_CASE(2) HX_CASE(3) HX_CASE(4) HX_CASE(5) HX_CASE(6) HX_CASE(7) HX_CASE(8)
    HX_CASE(9) HX_CASE(10) HX_CASE(11) HX_CASE(12) HX_CASE(13) HX_CASE(14) HX_CASE(15)
#undef HX_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

int64_t baseline_workspace_doubles(const hx_plan& P, int64_t n_el) {
  return 4 * n_el * int64_t(P.m) * P.m * P.m;
}

cudaError_t launch_baseline(const hx_plan& P, const double* q, const double* fac, double* out,
                            int64_t n_el, double* work, int* flag, cudaStream_t s) {
  if (n_el == 0) return cudaSuccess;
  switch (P.degree) {
#define HX_CASE(N) \
  case N:          \
    return baseline_n<N>(P, q, fac, out, n_el, work, flag, s);
    HX_CASE(1) HX_CASE(2) HX_CASE(3) HX_CASE(4) HX_CASE(5) HX_CASE(6) HX_CASE(7) HX_CASE(8)
    HX_CASE(9) HX_CASE(10) HX_CASE(11) HX_CASE(12) HX_CASE(13) HX_CASE(14) HX_CASE(15)
#undef HX_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace hx
