// BP3.5 -- collocated stiffness matvec on the GLL points (reference
// operators.py:282-286 -> _diff_chain_combine, operators.py:235-268):
//
//   out = lam * GwJ * q + sum_d D_d^T ( sum_d' G_dd' * D_d' q )
//
// One CTA processes a tile of EPB consecutive elements per iteration of a
// persistent loop.  Each thread owns one 1-D line of an element; the
// per-element tensors live in padded shared memory (strides from
// hx_layouts.h) and change orientation between stages:
//
//   S1 k-lines (j,i): q from HBM (coalesced over (j,i)), qt = D_t q (regs), q -> A
//   S2 i-lines (k,j): qr = D_r A -> B        j-lines (k,i): qs = D_s A -> C
//   S3 k-lines (j,i): G (HBM, coalesced) chain rule; rqr -> B, rqs -> C,
//                     acc = lam GwJ q + D_t^T rqt (regs)
//   S4 i-lines: B <- D_r^T B                 j-lines: C <- D_s^T C
//   S5 k-lines (j,i): out = acc + B + C (HBM, coalesced)
//
// Cfg::ORD (tools/gen_layouts.py BP35_ORD degrees): S2 / S4 enumerate their
// (k, r) lines k-fastest (2) or k-paired (4, with k-paired layouts) instead
// of r-fastest; the k-line stages touch HBM and keep (j, i) i-fastest lanes.
//
// The only HBM traffic is q, the 7 factor slots and out (Table 1: 9 n^3
// doubles per element).  Inputs are pulled into L2 ahead of use with bulk
// prefetches (schedule below), so the loads in S1/S3 hit L2.
#include "hx_common.cuh"
#include "hx_plan.h"

#ifndef HX_PF_BP35
#define HX_PF_BP35 1  // stage at which a tile's factors are prefetched into L2
#endif
// HX_MINB_BP35 overrides Cfg<>::MINB (resident CTAs per SM for the register
// budget) in tuning builds only.
#ifdef HX_MINB_BP35
#define HX_MINB_BP35_OF(N) HX_MINB_BP35
#else
#define HX_MINB_BP35_OF(N) Cfg<kBP35, N>::MINB
#endif

namespace hx {

template <int N>
struct BP35Params {
  Fold<N + 1, N + 1> D;   // derivative D (anti-centro-symmetric)
  Fold<N + 1, N + 1> Dt;  // its transpose
  const double* q;
  const double* fac;
  double* out;
  int64_t n_el;
  int64_t fac_estride;  // doubles per element in the packed factor array
  int64_t fac_sstride;  // doubles per slot
  double lam;
  int* flag;
  double* energy;  // per-CTA partials of <q, A q> (ENERGY instantiation only)
  DirArgs dir;     // DIR instantiation: q = r + beta p_old formed in S1 (hx_common.cuh)
};

template <int N, bool ENERGY, bool DIR = false>
__global__ void __launch_bounds__(Cfg<kBP35, N>::NT, HX_MINB_BP35_OF(N))
    bp35_kernel(const __grid_constant__ BP35Params<N> p) {
  using C = Cfg<kBP35, N>;
  constexpr int n = N + 1, n2 = n * n, n3 = n2 * n;
  constexpr int EPB = C::EPB;
  constexpr Lay LA = C::L[0], LB = C::L[1], LC = C::L[2];
  constexpr int EA = C::EBUF[0], EB = C::EBUF[1], EC = C::EBUF[2];
  extern __shared__ double smem[];
  double* const A = smem;
  double* const B = A + EPB * EA;
  double* const Cs = B + EPB * EB;

  const int tid = threadIdx.x;
  const int el = tid / n2;  // element of the tile this thread serves
  const int ln = tid % n2;  // its line within the element (same count every stage)
  const int64_t ntiles = (p.n_el + EPB - 1) / EPB;
  const int64_t ss = p.fac_sstride;

  // L2 prefetch schedule.  The lead time must cover DRAM latency but stay
  // short: prefetched-but-unconsumed bytes across all CTAs must fit in L2
  // with room to spare, or lines are evicted and fetched twice.  So a
  // tile's factors are requested when the tile starts (consumed in S3) and
  // the next tile's q when S3 starts (consumed in the next S1).
  if (tid == 0 && blockIdx.x < ntiles) {
    const int64_t e0 = int64_t(blockIdx.x) * EPB;
    const int64_t ne = min64(EPB, p.n_el - e0);
    prefetch_l2(p.q + e0 * n3, ne * n3 * sizeof(double));
    if (DIR) prefetch_l2(p.dir.r + e0 * n3, ne * n3 * sizeof(double));
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
    if (HX_PF_BP35 == 1 && tid == 0)
      prefetch_l2(p.fac + e0 * p.fac_estride, ne * p.fac_estride * sizeof(double));
    const bool act = el < ne;
    const int64_t e = e0 + el;
    double* const Ae = A + el * EA;
    double* const Be = B + el * EB;
    double* const Ce = Cs + el * EC;

    // kLean (Cfg::ACCS, high degrees): nothing stays in registers across a
    // barrier -- S3 re-reads q from its own k-line of A (nobody else reads
    // A after S2), takes D_t q there, and parks the accumulator in the same
    // line for S5 -- instead of carrying q, D_t q (S1 -> S3) and the
    // accumulator (S3 -> S5) through S2 / S4's two-line register peaks.
    constexpr bool kLean = C::ACCS != 0;
    double qv[kLean ? 1 : n], qt[kLean ? 1 : n], acc[kLean ? 1 : n];
    // ---- S1: k-lines over (j, i)
    if (act) {
      const int j = ln / n, i = ln % n;
      double qk[n];
      load_line<DIR, n, n2>(p.q, p.dir, beta, e * n3 + j * n + i, qk);
      const bool bad = any_nonfinite(qk);
      if (bad && p.flag) atomicOr(p.flag, 1);
      if constexpr (!kLean) {
#pragma unroll
        for (int k = 0; k < n; ++k) qv[k] = qk[k];
        fold_apply<n, n, -1>(p.D, qv, qt);
      }
      double* a = Ae + j * LA.s1 + i;
#pragma unroll
      for (int k = 0; k < n; ++k) a[LA.kofs(k)] = qk[k];
    }
    __syncthreads();
    // ---- S2: r- and s-derivatives
    if (HX_PF_BP35 == 2 && tid == 0)
      prefetch_l2(p.fac + e0 * p.fac_estride, ne * p.fac_estride * sizeof(double));
    if (act) {
      int k, r;  // Cfg::ORD: lane order over (k, r) (hx_common.cuh iline_coords)
      iline_coords<n, n, (C::ORD & 6)>(ln, k, r);
      double x[n], y[n];
      const double* a = Ae + LA.kofs(k) + r * LA.s1;  // i-line (k, j=r)
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = a[t];
      fold_apply<n, n, -1>(p.D, x, y);
      double* b = Be + LB.kofs(k) + r * LB.s1;
#pragma unroll
      for (int t = 0; t < n; ++t) b[t] = y[t];
      a = Ae + LA.kofs(k) + r;  // j-line (k, i=r)
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = a[t * LA.s1];
      fold_apply<n, n, -1>(p.D, x, y);
      double* c = Ce + LC.kofs(k) + r;
#pragma unroll
      for (int t = 0; t < n; ++t) c[t * LC.s1] = y[t];
    }
    __syncthreads();
    // ---- S3: metric chain rule on k-lines
    if (tid == 0) {
      const int64_t nt = tile + gridDim.x;
      if (nt < ntiles) {
        const int64_t f0 = nt * EPB;
        prefetch_l2(p.q + f0 * n3, min64(EPB, p.n_el - f0) * n3 * sizeof(double));
        if (DIR) prefetch_l2(p.dir.r + f0 * n3, min64(EPB, p.n_el - f0) * n3 * sizeof(double));
      }
    }
    if (act) {
      const int j = ln / n, i = ln % n;
      double* b = Be + j * LB.s1 + i;
      double* c = Ce + j * LC.s1 + i;
      const double* g = p.fac + e * p.fac_estride + j * n + i;
      double* a = Ae + j * LA.s1 + i;  // this thread's own k-line of q
      double rqt[n], qtl[n];
      if constexpr (kLean) {
        double x[n];
#pragma unroll
        for (int k = 0; k < n; ++k) x[k] = a[LA.kofs(k)];
        fold_apply<n, n, -1>(p.D, x, qtl);
      }
#pragma unroll
      for (int k = 0; k < n; ++k) {
        const double* gk = g + k * n2;
        const double grr = gk[0], grs = gk[ss], grt = gk[2 * ss];
        const double gss = gk[3 * ss], gst = gk[4 * ss], gtt = gk[5 * ss];
        const double gwj = gk[6 * ss];
        const double qk = kLean ? a[LA.kofs(k)] : qv[k];
        const double qr = b[LB.kofs(k)], qs = c[LC.kofs(k)], qtk = kLean ? qtl[k] : qt[k];
        const double rqr = grr * qr + grs * qs + grt * qtk;
        const double rqs = grs * qr + gss * qs + gst * qtk;
        b[LB.kofs(k)] = rqr;
        c[LC.kofs(k)] = rqs;
        rqt[k] = grt * qr + gst * qs + gtt * qtk;
        const double lq = p.lam * gwj * qk;
        // <q, A q> = sum over points of grad q . G grad q + lam GwJ q^2
        if constexpr (ENERGY) en += qr * rqr + qs * rqs + qtk * rqt[k] + qk * lq;
        if constexpr (kLean)
          a[LA.kofs(k)] = lq;
        else
          qv[k] = lq;
      }
      if constexpr (kLean) {
        double ac[n];
        fold_apply<n, n, -1>(p.Dt, rqt, ac);
#pragma unroll
        for (int k = 0; k < n; ++k) a[LA.kofs(k)] += ac[k];
      } else {
        fold_apply<n, n, -1>(p.Dt, rqt, acc);
#pragma unroll
        for (int k = 0; k < n; ++k) acc[k] += qv[k];
      }
    }
    __syncthreads();
    // ---- S4: transposed r- and s-derivatives, in place
    if (act) {
      int k, r;
      iline_coords<n, n, (C::ORD & 6)>(ln, k, r);
      double x[n], y[n];
      double* b = Be + LB.kofs(k) + r * LB.s1;
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = b[t];
      fold_apply<n, n, -1>(p.Dt, x, y);
#pragma unroll
      for (int t = 0; t < n; ++t) b[t] = y[t];
      double* c = Ce + LC.kofs(k) + r;
#pragma unroll
      for (int t = 0; t < n; ++t) x[t] = c[t * LC.s1];
      fold_apply<n, n, -1>(p.Dt, x, y);
#pragma unroll
      for (int t = 0; t < n; ++t) c[t * LC.s1] = y[t];
    }
    __syncthreads();
    // ---- S5: combine and store
    if (act) {
      const int j = ln / n, i = ln % n;
      const double* b = Be + j * LB.s1 + i;
      const double* c = Ce + j * LC.s1 + i;
      double* dst = p.out + e * n3 + j * n + i;
      const double* a = Ae + j * LA.s1 + i;
#pragma unroll
      for (int k = 0; k < n; ++k)
        st_stream(dst + k * n2, (kLean ? a[LA.kofs(k)] : acc[k]) + b[LB.kofs(k)] + c[LC.kofs(k)]);
    }
    // A is rewritten by the next tile's S1 only after it has passed this
    // tile's S3/S4 barriers (with kLean, S5 reads only the thread's own
    // k-line of A, which the same thread rewrites in the next S1); B and C
    // only after the next S1 barrier.
  }
  if constexpr (ENERGY) {
    const double sum = block_sum<C::NT>(en, A);  // A is idle after the last S3
    if (tid == 0) p.energy[blockIdx.x] = sum;
  }
}

template <int N, bool E, bool D = false, class Prm>
static cudaError_t launch_t(const Prm& prm, int64_t n_el, cudaStream_t s, bool pdl) {
  using C = Cfg<kBP35, N>;
  constexpr int smem = smem_doubles<kBP35, N>() * int(sizeof(double));
  const int64_t ntiles = (n_el + C::EPB - 1) / C::EPB;
  unsigned grid = 0;
  const cudaError_t err = persistent_grid<bp35_kernel<N, E, D>>(C::NT, smem, ntiles, &grid);
  if (err != cudaSuccess) return err;
  return launch_kernel<bp35_kernel<N, E, D>>(grid, C::NT, smem, s, pdl, prm);
}

template <int N>
static cudaError_t launch_n(const hx_plan& P, const double* q, const double* fac, double* out,
                            int64_t n_el, int* flag, double* energy, cudaStream_t s, bool pdl,
                            const DirArgs* dir) {
  BP35Params<N> prm;
  constexpr int n = N + 1;
  double dt[n * n];
  fill_fold(prm.D, P.diff);
  transpose(P.diff, n, n, dt);
  fill_fold(prm.Dt, dt);
  prm.q = q;
  prm.fac = fac;
  prm.out = out;
  prm.n_el = n_el;
  prm.fac_estride = P.elem_stride;
  prm.fac_sstride = P.slot_stride;
  prm.lam = P.lam;
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

cudaError_t launch_bp35(const hx_plan& P, const double* q, const double* fac, double* out,
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
