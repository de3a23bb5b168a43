// BP1.0 -- mass matvec with de-aliased Gauss quadrature (reference
// operators.py:274-281):  out = I^T ( GwJ * I q ),  I: GLL(n) -> GL(m).
//
// Persistent CTAs over tiles of EPB elements; a thread owns one 1-D line per
// stage (or walks over several when the CTA is smaller than the tile's line
// count); per-element tensors in padded shared memory (hx_layouts.h X, Y):
//
//   S1 j-lines (k,i)  n^2 : q (HBM, 8n-byte runs) -> I_s -> X[k][a][i]
//   S2 i-lines (k,a)  n*m : X -> I_r -> Y[k][a][c]
//   S3 k-lines (a,c)  m^2 : Y -> I_t -> * GwJ (HBM, coalesced) -> I_t^T -> Y (in place)
//   S4 i-lines (k,a)  n*m : Y -> I_r^T -> X[k][a][i]
//   S5 j-lines (k,i)  n^2 : X -> I_s^T -> out (HBM)
//
// The k-direction interpolation, the GwJ scaling and the k-direction
// projection are fused in registers in S3, so the GL-point tensor never
// leaves the thread that owns its k-line.  The contraction order differs from
// the reference's (j, i, k) only by floating-point reassociation.
//
// Cfg::ORD picks the lane order of the shared-memory-only i-line stages S2/S4
// jointly with the strides (tools/gen_layouts.py): at N=7 the k-paired order
// with k-paired X/Y layouts makes every stage bank-conflict free (r10:
// 173.6 -> 185.3 GDOF/s).  Cfg::QS > 0 would stage q through shared memory
// with the bulk-copy engine (measured slower, off: profiles/tuning).
#include "hx_common.cuh"
#include "hx_plan.h"

// HX_MINB_BP1 overrides Cfg<>::MINB (resident CTAs per SM for the register
// budget) in tuning builds only.
#ifdef HX_MINB_BP1
#define HX_MINB_BP1_OF(N) HX_MINB_BP1
#else
#define HX_MINB_BP1_OF(N) Cfg<kBP1, N>::MINB
#endif

namespace hx {

template <int N>
struct BP1Params {
  Fold<N + 2, N + 1> I;   // GLL -> GL interpolation (centro-symmetric)
  Fold<N + 1, N + 2> It;  // its transpose (projection)
  const double* q;
  const double* gwj;
  double* out;
  int64_t n_el;
  int64_t fac_estride;
  int* flag;
  double* energy;  // per-CTA partials of <q, A q> (ENERGY instantiation only)
};

template <int N, bool ENERGY, bool STAGE>
__global__ void __launch_bounds__(Cfg<kBP1, N>::NT, HX_MINB_BP1_OF(N))
    bp1_kernel(const __grid_constant__ BP1Params<N> p) {
  using C = Cfg<kBP1, N>;
  constexpr int n = N + 1, m = N + 2, n2 = n * n, n3 = n2 * n, m2 = m * m;
  constexpr int EPB = C::EPB, NT = C::NT;
  constexpr Lay LX = C::L[0], LY = C::L[1];
  constexpr int EX = C::EBUF[0], EY = C::EBUF[1];
  // lane order of the i-line stages (S2, S4), see iline_coords; the j-line
  // stages (S1, S5) touch HBM and keep i fastest
  constexpr int IORD = C::ORD;
  constexpr bool JKF = false;
  // a thread owns one line per stage when NT covers the tile's lines, else
  // it walks over several (small CTAs: cheap barriers, many CTAs per SM)
  constexpr bool ONE_C = EPB * m2 <= NT;
  // W_LATE: S3's GwJ is loaded after S1, so its L2 latency hides behind the
  // S1->S2 barrier and S2 instead of S1's q loads queueing behind it.  Faster
  // at N = 7, 10, 13, 14 (tune26: N=7 config 1 with L2 warm 18.4 -> 16.4 us,
  // E=32768 +1.5 %), slower at N = 1-4 and 9, where it costs registers.
  constexpr bool W_LATE = N == 7 || N == 10 || N == 13 || N == 14;
  // QS > 0: the q tile is staged in shared memory by the bulk-copy engine
  // one tile ahead (k-slabs of n*n doubles at stride QS), so S1 never waits
  // on HBM; the q L2 prefetch is then not needed.
  constexpr int QS = C::QS;
  constexpr bool QST = STAGE && QS > 0;
  extern __shared__ double smem[];
  uint64_t* const qbar = reinterpret_cast<uint64_t*>(smem);
  double* const QT = smem + (QST ? 2 : 0);
  double* const X = QT + (QST ? EPB * n * QS : 0);
  double* const Y = X + EPB * EX;

  const int tid = threadIdx.x;
  const int64_t ntiles = (p.n_el + EPB - 1) / EPB;
  const int64_t fs = p.fac_estride;

  // warp 0 stages tile `t`'s q: lane 0 arms the barrier with the byte count,
  // then the lanes issue one k-slab copy each
  auto stage_q = [&](int64_t t) {
    if constexpr (QST) {
      const int64_t f0 = t * EPB;
      const int nn = int(min64(EPB, p.n_el - f0));
      const int lane = tid & 31;
      if (lane == 0) mbar_arrive_expect_tx(qbar, unsigned(nn * n3 * sizeof(double)));
      __syncwarp();
      const uint64_t pol = l2_evict_first_policy();
      for (int s = lane; s < nn * n; s += 32)
        bulk_g2s(QT + s * QS, p.q + f0 * n3 + int64_t(s) * n2, n2 * sizeof(double), qbar, pol);
    }
  };
  if constexpr (QST) {
    if (tid == 0) mbar_init(qbar, 1);
    __syncthreads();
    if (tid < 32 && blockIdx.x < ntiles) stage_q(blockIdx.x);
  }
  unsigned qphase = 0;

  if (tid == 0 && blockIdx.x < ntiles) {
    const int64_t e0 = int64_t(blockIdx.x) * EPB;
    const int64_t ne = min64(EPB, p.n_el - e0);
    if constexpr (!QST) prefetch_l2(p.q + e0 * n3, ne * n3 * sizeof(double));
    prefetch_l2(p.gwj + e0 * fs, ne * fs * sizeof(double));
  }

  double en = 0.0;  // this thread's share of <q, A q> (ENERGY)
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t e0 = tile * EPB;
    const int ne = int(min64(EPB, p.n_el - e0));
    if (tid == 0) {
      const int64_t nt = tile + gridDim.x;
      if (nt < ntiles) {
        const int64_t f0 = nt * EPB;
        const int64_t nn = min64(EPB, p.n_el - f0);
        if constexpr (!QST) prefetch_l2(p.q + f0 * n3, nn * n3 * sizeof(double));
        prefetch_l2(p.gwj + f0 * fs, nn * fs * sizeof(double));
      }
    }
    // GwJ of this thread's S3 k-line (one-line-per-thread shapes), issued
    // before S1 or, where that measured faster (W_LATE), after it
    double w[m];
    auto load_w = [&]() {
      const int el_c = tid / m2, ln_c = tid % m2;
      if (el_c < ne) {
        const double* g = p.gwj + (e0 + el_c) * fs + ln_c;
#pragma unroll
        for (int c = 0; c < m; ++c) w[c] = g[c * m2];
      }
    };
    if constexpr (ONE_C && !W_LATE) load_w();
    // ---- S1: j-lines (k, i): interpolate along s
    if constexpr (QST) {
      mbar_wait(qbar, qphase);
      qphase ^= 1u;
    }
    for_lines<EPB * n2, NT>(tid, [&](int g) {
      const int el = g / n2, ln = g % n2;
      if (el >= ne) return;
      int k, i;
      line_coords<n, n, JKF>(ln, k, i);
#ifdef HX_EXP_COAL
      // EXPERIMENT (wrong numerics): k-line addressing, coalesced 256 B per warp
      const double* src = p.q + (e0 + el) * n3 + ln;
      double x[n], y[m];
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = src[t * n2];
#else
      const double* src = QST ? QT + (el * n + k) * QS + i : p.q + (e0 + el) * n3 + k * n2 + i;
      double x[n], y[m];
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = src[t * n];
#endif
      const bool bad = any_nonfinite(x);
      if (bad && p.flag) atomicOr(p.flag, 1);
      fold_apply<m, n, 1>(p.I, x, y);
      double* dst = X + el * EX + LX.kofs(k) + i;
#pragma unroll
      for (int t = 0; t < m; ++t) dst[t * LX.s1] = y[t];
    });
    if constexpr (ONE_C && W_LATE) load_w();
    __syncthreads();
    if constexpr (QST) {
      // the staged q has been consumed: fetch the next tile's into it
      if (tid < 32 && tile + gridDim.x < ntiles) {
        fence_proxy_async_smem();
        stage_q(tile + gridDim.x);
      }
    }
    // ---- S2: i-lines (k, a): interpolate along r
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
    // ---- S3: k-lines (a, c): interpolate along t, scale, project along t
    for_lines<EPB * m2, NT>(tid, [&](int g) {
      const int el = g / m2, ln = g % m2;
      if (el >= ne) return;
      const int a = ln / m, c = ln % m;
      double wl[m];
      if constexpr (ONE_C) {
#pragma unroll
        for (int t = 0; t < m; ++t) wl[t] = w[t];
      } else {
        const double* gp = p.gwj + (e0 + el) * fs + ln;
#pragma unroll
        for (int t = 0; t < m; ++t) wl[t] = gp[t * m2];
      }
      double* line = Y + el * EY + a * LY.s1 + c;
      double x[n], y[m];
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = line[LY.kofs(t)];
      fold_apply<m, n, 1>(p.I, x, y);
#pragma unroll
      for (int t = 0; t < m; ++t) {
        const double wy = y[t] * wl[t];
        if constexpr (ENERGY) en += wy * y[t];  // <q, A q> = sum GwJ (I q)^2
        y[t] = wy;
      }
      fold_apply<n, m, 1>(p.It, y, x);
#pragma unroll
      for (int t = 0; t < n; ++t) line[LY.kofs(t)] = x[t];
    });
    __syncthreads();
    // ---- S4: i-lines (k, a): project along r
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
    // ---- S5: j-lines (k, i): project along s and store
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
#ifdef HX_EXP_COAL
      double* dst = p.out + (e0 + el) * n3 + ln;
#pragma unroll
      for (int t = 0; t < n; ++t) st_stream(dst + t * n2, y[t]);
#else
      double* dst = p.out + (e0 + el) * n3 + k * n2 + i;
#pragma unroll
      for (int t = 0; t < n; ++t) st_stream(dst + t * n, y[t]);
#endif
    });
    __syncthreads();  // X is rewritten by the next tile's S1
  }
  if constexpr (ENERGY) {
    const double sum = block_sum<C::NT>(en, X);
    if (tid == 0) p.energy[blockIdx.x] = sum;
  }
}

template <int N, bool E, bool STAGE, class Prm>
static cudaError_t launch_t(const Prm& prm, int64_t n_el, cudaStream_t s) {
  using C = Cfg<kBP1, N>;
  constexpr int smem = smem_doubles<kBP1, N>() * int(sizeof(double));
  const int64_t ntiles = (n_el + C::EPB - 1) / C::EPB;
  unsigned grid = 0;
  const cudaError_t err = persistent_grid<bp1_kernel<N, E, STAGE>>(C::NT, smem, ntiles, &grid);
  if (err != cudaSuccess) return err;
  bp1_kernel<N, E, STAGE><<<grid, C::NT, smem, s>>>(prm);
  return cudaGetLastError();
}

// The staged shape needs 16-byte aligned q (the bulk engine's rule); a q
// view that is only 8-byte aligned takes the unstaged instantiation.
template <int N, bool E, class Prm>
static cudaError_t launch_s(const Prm& prm, int64_t n_el, cudaStream_t s) {
  if constexpr (Cfg<kBP1, N>::QS > 0) {
    if ((reinterpret_cast<uintptr_t>(prm.q) & 15) == 0) return launch_t<N, E, true>(prm, n_el, s);
  }
  return launch_t<N, E, false>(prm, n_el, s);
}

template <int N>
static cudaError_t launch_n(const hx_plan& P, const double* q, const double* fac, double* out,
                            int64_t n_el, int* flag, double* energy, cudaStream_t s) {
  using C = Cfg<kBP1, N>;
  constexpr int n = N + 1, m = N + 2;
  constexpr int smem = smem_doubles<kBP1, N>() * int(sizeof(double));
  BP1Params<N> prm;
  double it[n * m];
  fill_fold(prm.I, P.interp);
  transpose(P.interp, m, n, it);
  fill_fold(prm.It, it);
  prm.q = q;
  prm.gwj = fac;
  prm.out = out;
  prm.n_el = n_el;
  prm.fac_estride = P.elem_stride;
  prm.flag = flag;
  prm.energy = energy;
  return energy ? launch_s<N, true>(prm, n_el, s) : launch_s<N, false>(prm, n_el, s);
}

cudaError_t launch_bp1(const hx_plan& P, const double* q, const double* fac, double* out,
                       int64_t n_el, int* flag, double* energy, cudaStream_t s) {
  switch (P.degree) {
#define HX_CASE(N) \
  case N:          \
    return launch_n<N>(P, q, fac, out, n_el, flag, energy, s);
    HX_CASE(1) HX_CASE(2) HX_CASE(3) HX_CASE(4) HX_CASE(5) HX_CASE(6) HX_CASE(7) HX_CASE(8)
    HX_CASE(9) HX_CASE(10) HX_CASE(11) HX_CASE(12) HX_CASE(13) HX_CASE(14) HX_CASE(15)
#undef HX_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace hx
