// BP1.0 -- mass matvec with de-aliased Gauss quadrature (reference
// operators.py:274-281):  out = I^T ( GwJ * I q ),  I: GLL(n) -> GL(m).
//
// Persistent CTAs over tiles of EPB elements; a thread owns one 1-D line per
// stage (or walks over several when the CTA is smaller than the tile's line
// count); per-element tensors in padded shared memory (hx_layouts.h X, Y).
// The t (k) direction goes first and last, so the two stages that touch HBM
// move k-lines: lanes own consecutive (j, i) points and every warp access to
// q / out is one contiguous 256-byte run (2 L1 wavefronts instead of the 4
// of (k, i) j-lines; profiles/r2_02: +3.5 % at E=32768 from that alone):
//
//   S1 k-lines (j,i)  n^2 : q (HBM, coalesced) -> I_t -> X[c][j][i]
//   S2 j-lines (c,i)  m*n : X -> I_s -> Y[c][b][i]
//   S3 i-lines (c,b)  m^2 : Y -> I_r -> * GwJ (HBM, coalesced) -> I_r^T -> Y (in place)
//   S4 j-lines (c,i)  m*n : Y -> I_s^T -> X[c][j][i]
//   S5 k-lines (j,i)  n^2 : X -> I_t^T -> out (HBM, coalesced, streaming)
//
// The r-direction interpolation, the GwJ scaling and the r-direction
// projection are fused in registers in S3, so the GL-point tensor never
// leaves the thread that owns its i-line.  S3's lanes own consecutive (c, b)
// lines, so BP1.0's packed GwJ slot is stored i-major -- GwJ[a][c][b], point
// (k=c, j=b, i=a) -- which makes each S3 load one contiguous run over the
// warp (hx_geom.cu writes, hx_repack / hx_baseline read that order).  The
// contraction order differs from the reference's (j, i, k) only by
// floating-point reassociation.
//
// Cfg::ORD picks the lane order of the shared-memory-only j-line stages
// S2/S4 jointly with the strides (tools/gen_layouts.py): 0 i fastest, 2 c
// fastest, 4 c-paired (c pairs outermost, then i, then the c parity) with
// c-paired X/Y layouts.  At N=7 c fastest with X = (73, 8), Y = (153, 17)
// makes every stage conflict-free: the address of line L is a multiple of L
// mod 16 in each access pattern (ncu r2_04: 0.86 M excess of 11.3 M
// shared wavefronts, from 3.3 M with the c-paired order).
#include "hx_common.cuh"
#include "hx_plan.h"

// HX_MINB_BP1 overrides Cfg<>::MINB (resident CTAs per SM for the register
// budget) in tuning builds only.
#ifdef HX_MINB_BP1
#define HX_MINB_BP1_OF(N) HX_MINB_BP1
#else
#define HX_MINB_BP1_OF(N) Cfg<kBP1, N>::MINB
#endif

// Diagnostic builds only (numerically wrong, timing only): HX_EXP_NOQ reads
// q, HX_EXP_NOW reads GwJ, from the first 8 elements (L2-resident), so the
// kernel runs without that HBM stream.
#ifdef HX_EXP_NOQ
#define HX_QEL(e) ((e) & 7)
#else
#define HX_QEL(e) (e)
#endif
#ifdef HX_EXP_NOW
#define HX_WEL(e) ((e) & 7)
#else
#define HX_WEL(e) (e)
#endif

namespace hx {

template <int N>
struct BP1Params {
  Fold<N + 2, N + 1> I;   // GLL -> GL interpolation (centro-symmetric)
  Fold<N + 1, N + 2> It;  // its transpose (projection)
  const double* q;
  const double* gwj;  // packed, i-major per element: gwj[e * fac_estride + a * m^2 + c * m + b]
                      // (+ b * m + c with ORD bit 8: bp1_gwj_index)
  double* out;
  int64_t n_el;
  int64_t fac_estride;
  int* flag;
  double* energy;  // per-CTA partials of <q, A q> (ENERGY instantiation only)
  DirArgs dir;     // DIR instantiation: q = r + beta p_old formed in S1 (hx_common.cuh)
};

template <int N, bool ENERGY, bool DIR = false>
__global__ void __launch_bounds__(Cfg<kBP1, N>::NT, HX_MINB_BP1_OF(N))
    bp1_kernel(const __grid_constant__ BP1Params<N> p) {
  using C = Cfg<kBP1, N>;
  constexpr int n = N + 1, m = N + 2, n2 = n * n, n3 = n2 * n, m2 = m * m;
  constexpr int EPB = C::EPB, NT = C::NT;
  constexpr Lay LX = C::L[0], LY = C::L[1];
  constexpr int EX = C::EBUF[0], EY = C::EBUF[1];
  constexpr int JORD = C::ORD & 7;  // lane order of the j-line stages S2, S4
  // ORD bit 8: S3's lines run c-fastest, and the packed GwJ slot is stored
  // (i, j, k) -- gwj[a][b][c] -- so the S3 loads stay one contiguous run
  constexpr bool kCFast = (C::ORD & 8) != 0;
  // a thread owns one line per stage when NT covers the tile's lines, else
  // it walks over several (small CTAs: cheap barriers, many CTAs per SM)
  constexpr bool ONE_C = EPB * m2 <= NT;
  // W_LATE: S3's GwJ is loaded after S1, so its L2 latency hides behind the
  // S1->S2 barrier and S2 instead of S1's q loads queueing behind it
  // (tune26, measured on the former stage order at N = 7, 10, 13, 14).
  constexpr bool W_LATE = N == 7 || N == 10 || N == 13 || N == 14;
  extern __shared__ double smem[];
  double* const X = smem;
  double* const Y = X + EPB * EX;

  const int tid = threadIdx.x;
  const int64_t ntiles = (p.n_el + EPB - 1) / EPB;
  const int64_t fs = p.fac_estride;

  if (tid == 0 && blockIdx.x < ntiles) {
    const int64_t e0 = int64_t(blockIdx.x) * EPB;
    const int64_t ne = min64(EPB, p.n_el - e0);
    prefetch_l2(p.q + HX_QEL(e0) * n3, ne * n3 * sizeof(double));
    if (DIR) prefetch_l2(p.dir.r + e0 * n3, ne * n3 * sizeof(double));
    prefetch_l2(p.gwj + HX_WEL(e0) * fs, ne * fs * sizeof(double));
    // ... and the second tile's: with back-to-back (PDL) launches this runs
    // under the previous apply's tail (r2_40: +0.4 % at E=32768)
    const int64_t e1 = e0 + int64_t(gridDim.x) * EPB;
    if (e1 < p.n_el) {
      prefetch_l2(p.q + HX_QEL(e1) * n3, min64(EPB, p.n_el - e1) * n3 * sizeof(double));
      if (DIR) prefetch_l2(p.dir.r + e1 * n3, min64(EPB, p.n_el - e1) * n3 * sizeof(double));
      prefetch_l2(p.gwj + HX_WEL(e1) * fs, min64(EPB, p.n_el - e1) * fs * sizeof(double));
    }
  }

  // PDL (hx_common.cuh): only L2 prefetch hints above this point
  pdl_allow_dependents();
  pdl_wait();
  double beta = 0.0;
  if constexpr (DIR) beta = p.dir.rr_new[0] / p.dir.rr_old[0];

  double en = 0.0;  // this thread's share of <q, A q> (ENERGY)
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t e0 = tile * EPB;
    const int ne = int(min64(EPB, p.n_el - e0));
    // the next tile's inputs into L2 while this one computes (prefetching
    // after S1 instead measured the same at E=32768: profiles/r2_05)
    if (tid == 0) {
      const int64_t nt = tile + gridDim.x;
      if (nt < ntiles) {
        const int64_t f0 = nt * EPB;
        const int64_t nn = min64(EPB, p.n_el - f0);
        prefetch_l2(p.q + HX_QEL(f0) * n3, nn * n3 * sizeof(double));
        if (DIR) prefetch_l2(p.dir.r + f0 * n3, nn * n3 * sizeof(double));
        prefetch_l2(p.gwj + HX_WEL(f0) * fs, nn * fs * sizeof(double));
      }
    }
    // GwJ of this thread's S3 i-line (one-line-per-thread shapes), issued
    // before S1 or, where that measured faster (W_LATE), after it
    double w[m];
    auto load_w = [&]() {
      const int el_c = tid / m2, ln_c = tid % m2;
      if (el_c < ne) {
        const double* g = p.gwj + HX_WEL(e0 + el_c) * fs + ln_c;
#pragma unroll
        for (int a = 0; a < m; ++a) w[a] = g[a * m2];
      }
    };
    if constexpr (ONE_C && !W_LATE) load_w();
    // ---- S1: k-lines (j, i): interpolate along t
    for_lines<EPB * n2, NT>(tid, [&](int g) {
      const int el = g / n2, ln = g % n2;
      if (el >= ne) return;
      const int j = ln / n, i = ln % n;
      double x[n], y[m];
      load_line<DIR, n, n2>(p.q, p.dir, beta, HX_QEL(e0 + el) * n3 + ln, x);
      const bool bad = any_nonfinite(x);
      if (bad && p.flag) atomicOr(p.flag, 1);
      fold_apply<m, n, 1>(p.I, x, y);
      double* dst = X + el * EX + j * LX.s1 + i;
#pragma unroll
      for (int c = 0; c < m; ++c) dst[LX.kofs(c)] = y[c];
    });
    if constexpr (ONE_C && W_LATE) load_w();
    __syncthreads();
    // ---- S2: j-lines (c, i): interpolate along s
    for_lines<EPB * m * n, NT>(tid, [&](int g) {
      const int el = g / (m * n), ln = g % (m * n);
      if (el >= ne) return;
      int c, i;
      iline_coords<m, n, JORD>(ln, c, i);
      const double* src = X + el * EX + LX.kofs(c) + i;
      double x[n], y[m];
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = src[t * LX.s1];
      fold_apply<m, n, 1>(p.I, x, y);
      double* dst = Y + el * EY + LY.kofs(c) + i;
#pragma unroll
      for (int b = 0; b < m; ++b) dst[b * LY.s1] = y[b];
    });
    __syncthreads();
    // ---- S3: i-lines (c, b): interpolate along r, scale, project along r
    for_lines<EPB * m2, NT>(tid, [&](int g) {
      const int el = g / m2, ln = g % m2;
      if (el >= ne) return;
      const int c = kCFast ? ln % m : ln / m, b = kCFast ? ln / m : ln % m;
      double wl[m];
      if constexpr (ONE_C) {
#pragma unroll
        for (int a = 0; a < m; ++a) wl[a] = w[a];
      } else {
        const double* gp = p.gwj + HX_WEL(e0 + el) * fs + ln;
#pragma unroll
        for (int a = 0; a < m; ++a) wl[a] = gp[a * m2];
      }
      double* line = Y + el * EY + LY.kofs(c) + b * LY.s1;
      double x[n], y[m];
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = line[t];
      fold_apply<m, n, 1>(p.I, x, y);
#pragma unroll
      for (int a = 0; a < m; ++a) {
        const double wy = y[a] * wl[a];
        if constexpr (ENERGY) en += wy * y[a];  // <q, A q> = sum GwJ (I q)^2
        y[a] = wy;
      }
      fold_apply<n, m, 1>(p.It, y, x);
#pragma unroll
      for (int t = 0; t < n; ++t) line[t] = x[t];
    });
    __syncthreads();
    // ---- S4: j-lines (c, i): project along s
    for_lines<EPB * m * n, NT>(tid, [&](int g) {
      const int el = g / (m * n), ln = g % (m * n);
      if (el >= ne) return;
      int c, i;
      iline_coords<m, n, JORD>(ln, c, i);
      const double* src = Y + el * EY + LY.kofs(c) + i;
      double x[m], y[n];
#pragma unroll
      for (int t = 0; t < m; ++t) x[t] = src[t * LY.s1];
      fold_apply<n, m, 1>(p.It, x, y);
      double* dst = X + el * EX + LX.kofs(c) + i;
#pragma unroll
      for (int j = 0; j < n; ++j) dst[j * LX.s1] = y[j];
    });
    __syncthreads();
    // ---- S5: k-lines (j, i): project along t and store
    for_lines<EPB * n2, NT>(tid, [&](int g) {
      const int el = g / n2, ln = g % n2;
      if (el >= ne) return;
      const int j = ln / n, i = ln % n;
      const double* src = X + el * EX + j * LX.s1 + i;
      double x[m], y[n];
#pragma unroll
      for (int t = 0; t < m; ++t) x[t] = src[LX.kofs(t)];
      fold_apply<n, m, 1>(p.It, x, y);
      double* dst = p.out + (e0 + el) * n3 + ln;
#pragma unroll
      for (int k = 0; k < n; ++k) {
#ifdef HX_EXP_NOSTORE
        if (y[k] == 1.2345e300)  // never true: keeps the work, drops the HBM writes
#endif
          st_stream(dst + k * n2, y[k]);
      }
    });
    __syncthreads();  // X is rewritten by the next tile's S1
  }
  if constexpr (ENERGY) {
    const double sum = block_sum<C::NT>(en, X);
    if (tid == 0) p.energy[blockIdx.x] = sum;
  }
}

template <int N, bool E, bool D = false, class Prm>
static cudaError_t launch_t(const Prm& prm, int64_t n_el, cudaStream_t s, bool pdl) {
  using C = Cfg<kBP1, N>;
  constexpr int smem = smem_doubles<kBP1, N>() * int(sizeof(double));
  const int64_t ntiles = (n_el + C::EPB - 1) / C::EPB;
  unsigned grid = 0;
  const cudaError_t err = persistent_grid<bp1_kernel<N, E, D>>(C::NT, smem, ntiles, &grid);
  if (err != cudaSuccess) return err;
  return launch_kernel<bp1_kernel<N, E, D>>(grid, C::NT, smem, s, pdl, prm);
}

template <int N>
static cudaError_t launch_n(const hx_plan& P, const double* q, const double* fac, double* out,
                            int64_t n_el, int* flag, double* energy, cudaStream_t s, bool pdl,
                            const DirArgs* dir) {
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
  if (dir) {  // the CG direction form exists only with the energy epilogue (hx_apply_energy_dir)
    if (!energy) return cudaErrorInvalidValue;
    prm.q = dir->p;
    prm.dir = *dir;
    return launch_t<N, true, true>(prm, n_el, s, pdl);
  }
  prm.dir = DirArgs{};
  return energy ? launch_t<N, true>(prm, n_el, s, pdl) : launch_t<N, false>(prm, n_el, s, pdl);
}

bool bp1_gwj_cfast(int degree) {
  switch (degree) {
#define HX_CASE(N) \
  case N:          \
    return (Cfg<kBP1, N>::ORD & 8) != 0;
    HX_CASE(1) HX_CASE(2) HX_CASE(3) HX_CASE(4) HX_CASE(5) HX_CASE(6) HX_CASE(7) HX_CASE(8)
    HX_CASE(9) HX_CASE(10) HX_CASE(11) HX_CASE(12) HX_CASE(13) HX_CASE(14) HX_CASE(15)
#undef HX_CASE
    default:
      return false;
  }
}

cudaError_t launch_bp1(const hx_plan& P, const double* q, const double* fac, double* out,
                       int64_t n_el, int* flag, double* energy, cudaStream_t s, bool pdl,
                       const DirArgs* dir) {
  switch (P.degree) {
#define HX_CASE(N) \
  case N:          \
    return launch_n<N>(P, q, fac, out, n_el, flag, energy, s, pdl, dir);
    HX_CASE(1) HX_CASE(2) HX_CASE(3) HX_CASE(4) HX_CASE(5) HX_CASE(6) HX_CASE(7) HX_CASE(8)
    HX_CASE(9) HX_CASE(10) HX_CASE(11) HX_CASE(12) HX_CASE(13) HX_CASE(14) HX_CASE(15)
#undef HX_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace hx
