// Gather-scatter (direct stiffness summation, Q Q^T) on the structured cube
// mesh, and the assembled-CG vector kernels built on it (SURVEY.md §8f rank 2:
// the matvec's real caller is a CG Poisson solve; the reference
// keeps vectors element-local and has no assembly).
//
// Mesh: build_cube_mesh(side, extent) (reference mesh.py:44-56) orders
// elements e = (cx * side + cy) * side + cz and maps the reference axes
// r, s, t to x, y, z, so local node (k, j, i) of element (cx, cy, cz) is the
// global node (cx N + i, cy N + j, cz N + k).  A node on an element face,
// edge or corner has 2, 4 or 8 element-local copies.
//
// dss(u)[copy] = sum of u over every copy of the same global node.  The sum
// runs over the copies in one canonical order (x, then y, then z neighbours,
// each ascending), so all copies receive bit-identical values and the result
// is deterministic -- no atomics.  With `mask`, nodes on the cube boundary are
// zeroed (homogeneous Dirichlet conditions).
//
// Element ranges (multi-GPU): a rank owns elements [e_begin, e_end) of the
// cube; its own vectors start at e_begin, while the vector that is gathered
// (the one dss sums) starts at element `base` <= e_begin and must also hold
// every element sharing a node with the range -- at most side^2 + side + 1
// elements either side, filled by a halo exchange (cg.AssembledShard).
//
// Assembled CG keeps every vector in element-local storage as its continuous
// representative u_L = Q u_G.  Then
//   <p_G, A_G p_G> = <p_L, A_L p_L>                 (fused into the matvec)
//   A_G p_G        -> mask dss(A_L p_L)             (face passes in place on A p)
//   <r_G, r_G>     = sum_L r_L^2 / multiplicity      (fused into the update)
#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {

constexpr int kDssThreads = 256;

// Copies of one local node along one axis: element offsets (in that axis'
// element coordinate) and local indices, ascending by element.
struct AxisCopies {
  int cnt;
  int d[2], l[2];
};

__device__ __forceinline__ AxisCopies axis_copies(int c, int i, int side, int N) {
  AxisCopies a;
  if (i == 0 && c > 0) {
    a.cnt = 2; a.d[0] = -1; a.l[0] = N; a.d[1] = 0; a.l[1] = 0;
  } else if (i == N && c < side - 1) {
    a.cnt = 2; a.d[0] = 0; a.l[0] = N; a.d[1] = 1; a.l[1] = 0;
  } else {
    a.cnt = 1; a.d[0] = 0; a.l[0] = i; a.d[1] = 0; a.l[1] = i;
  }
  return a;
}

struct DssRange {
  int side;
  int64_t e_begin, e_end;  // elements processed (own vectors start at e_begin)
  int64_t base;            // first element of the gathered vector
};

// One element-local node: its element (and that element's cube coordinates,
// computed once per element by the caller) and its (k, j, i).
struct NodeRef {
  int64_t e;
  int cx, cy, cz, k, j, i;
};

template <int N>
__device__ __forceinline__ bool on_boundary(const NodeRef& r, int side) {
  const int G = side * N;
  const int gx = r.cx * N + r.i, gy = r.cy * N + r.j, gz = r.cz * N + r.k;
  return gx == 0 || gx == G || gy == 0 || gy == G || gz == 0 || gz == G;
}

// 1 / (number of element-local copies of node r): 1, 1/2, 1/4 or 1/8, so
// scaling by it is exact (same bits as dividing by the count)
template <int N>
__device__ __forceinline__ double inv_mult(const NodeRef& r, int side) {
  const int c = axis_copies(r.cx, r.i, side, N).cnt + axis_copies(r.cy, r.j, side, N).cnt +
                axis_copies(r.cz, r.k, side, N).cnt - 3;  // log2 of the count
  return c == 0 ? 1.0 : c == 1 ? 0.5 : c == 2 ? 0.25 : 0.125;
}

// sum over the copies of node r, in the canonical order (x outer, z inner,
// each ascending); bounded loops with predicates, no dynamic trip counts
template <int N>
__device__ __forceinline__ double gather_sum(const double* __restrict__ u, const NodeRef& r,
                                             int side, int64_t base) {
  constexpr int n = N + 1, n3 = n * n * n;
  const AxisCopies ax = axis_copies(r.cx, r.i, side, N);
  const AxisCopies ay = axis_copies(r.cy, r.j, side, N);
  const AxisCopies az = axis_copies(r.cz, r.k, side, N);
  const int64_t s = side;
  double sum = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    if (a >= ax.cnt) break;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (b >= ay.cnt) break;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (c >= az.cnt) break;
        const int64_t e = r.e + ax.d[a] * s * s + ay.d[b] * s + az.d[c];
        sum += u[(e - base) * n3 + (az.l[c] * n + ay.l[b]) * n + ax.l[a]];
      }
    }
  }
  return sum;
}

// Loop over every element-local node of the range: CTAs stride over
// elements (cube coordinates computed once per element), threads over the
// n^3 local nodes (constant-divisor index math), so consecutive threads touch
// consecutive addresses.  f(NodeRef, index into the range's own vectors).
template <int N, class F>
__device__ __forceinline__ void for_nodes(const DssRange& g, F&& f) {
  constexpr int n = N + 1, n3 = n * n * n;
  const int64_t side = g.side;
  for (int64_t e = g.e_begin + blockIdx.x; e < g.e_end; e += gridDim.x) {
    NodeRef r;
    r.e = e;
    // element indices fit 32 bits (side <= 1600): 32-bit divisions are
    // several times cheaper than 64-bit ones
    const uint32_t e32 = uint32_t(e), s32 = uint32_t(side);
    const uint32_t exy = e32 / s32;
    r.cz = int(e32 - exy * s32);
    r.cx = int(exy / s32);
    r.cy = int(exy - uint32_t(r.cx) * s32);
    const int64_t own = (e - g.e_begin) * n3;
    for (int l = threadIdx.x; l < n3; l += blockDim.x) {
      r.i = l % n;
      r.j = (l / n) % n;
      r.k = l / (n * n);
      f(r, own + l);
    }
  }
}

template <int N>
__global__ void __launch_bounds__(kDssThreads)
    dss_kernel(const double* __restrict__ in, double* __restrict__ out, DssRange g, int mask) {
  for_nodes<N>(g, [&](const NodeRef& r, int64_t idx) {
    out[idx] = (mask && on_boundary<N>(r, g.side)) ? 0.0 : gather_sum<N>(in, r, g.side, g.base);
  });
}

// partials of sum u v / multiplicity (the global inner product of continuous
// representatives)
template <int N>
__global__ void __launch_bounds__(kDssThreads)
    dot_dss_kernel(const double* __restrict__ u, const double* __restrict__ v, DssRange g,
                   double* __restrict__ part) {
  __shared__ double scratch[kDssThreads / 32];
  double s = 0.0;
  for_nodes<N>(g, [&](const NodeRef& r, int64_t idx) {
    s = fma(u[idx], v[idx] * inv_mult<N>(r, g.side), s);
  });
  s = block_sum<kDssThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// ---- separable in-place gather-scatter ------------------------------------
// Q Q^T on the cube mesh is a Kronecker product of 1-D gather-scatters, so it
// can be applied as three passes, one per axis: each pass replaces both
// copies of every node on an interior element face normal to that axis by
// (lower-element copy + upper-element copy).  After the x, y and z passes
// every copy of a node holds the same bits (addition is commutative and the
// operands of each pair are the same on both sides), and each pass only
// touches face nodes -- far cheaper than gathering up to 8 copies per node.
// A buffer holding elements [lo, hi) gets the correct result for every node
// whose copies all lie in the buffer (a rank's own nodes, given its halo).
template <int N, int AX>
__global__ void __launch_bounds__(kDssThreads)
    dss_pass_kernel(double* __restrict__ u, int side, int64_t lo, int64_t hi) {
  constexpr int n = N + 1, n2 = n * n, n3 = n2 * n;
  const int64_t s = side;
  const int64_t estride = AX == 0 ? s * s : (AX == 1 ? s : 1);  // x: cx, y: cy, z: cz
  const int64_t total = (hi - lo) * n2;
  const uint32_t s32 = uint32_t(side);
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = lo + g / n2;
    const int f = int(g % n2);
    const uint32_t e32 = uint32_t(e);  // side <= 1600: element indices fit 32 bits
    const int c = AX == 0 ? int(e32 / (s32 * s32))
                          : (AX == 1 ? int((e32 / s32) % s32) : int(e32 % s32));
    const int64_t nb = e - estride;  // lower neighbour along the axis
    if (c == 0 || nb < lo) continue;
    // face node f of the element's lower face (local index 0 along AX) and
    // the matching node on the neighbour's upper face (local index N)
    int lo_off, hi_off;
    if constexpr (AX == 0) {          // i = 0 / N, f = (k, j)
      lo_off = f * n;                 // (k * n + j) * n + 0
      hi_off = f * n + N;
    } else if constexpr (AX == 1) {   // j = 0 / N, f = (k, i)
      const int k = f / n, i = f % n;
      lo_off = k * n2 + i;
      hi_off = k * n2 + N * n + i;
    } else {                          // k = 0 / N, f = (j, i)
      lo_off = f;
      hi_off = N * n2 + f;
    }
    double* a = u + (nb - lo) * n3 + hi_off;  // lower element's copy
    double* b = u + (e - lo) * n3 + lo_off;   // upper element's copy
    const double sum = *a + *b;
    *a = sum;
    *b = sum;
  }
}

// Assembled-CG update.  w (= A_L p, halo-padded, elements from g.base on)
// has been assembled in place by the three face passes; then
//   alpha = rr / pAp;  x += alpha p;  r -= alpha mask w;  partials of
//   sum r^2 / multiplicity.
// >= 6 CTAs of 256 threads per SM (<= 40 registers, no spills): this kernel
// lives on memory parallelism (r15 ncu: 60 registers halved the resident
// warps and made it 1.5x slower than the element-local update).  Folding the
// strided x pass into it as a neighbour gather measured slower still (r16).
template <int N>
__global__ void __launch_bounds__(kDssThreads, 6)
    cg_update_assembled_kernel(double* __restrict__ x, const double* __restrict__ p,
                               double* __restrict__ r, const double* __restrict__ w, DssRange g,
                               int mask, const double* __restrict__ rr,
                               const double* __restrict__ pap, double* __restrict__ part) {
  // written out instead of through for_nodes: inside the lambda the
  // compiler lost __restrict__ and serialised each node's loads behind the
  // previous node's stores (r17: 179 us vs 118 us for the plain update)
  constexpr int n = N + 1, n3 = n * n * n;
  constexpr int IT = (n3 + kDssThreads - 1) / kDssThreads;
  constexpr int CH = IT < 2 ? IT : 2;  // nodes per thread with loads in flight together
  __shared__ double scratch[kDssThreads / 32];
  const double alpha = rr[0] / pap[0];
  const double* __restrict__ wown = w + (g.e_begin - g.base) * n3;
  const uint32_t s32 = uint32_t(g.side);
  double s = 0.0;
  for (int64_t e = g.e_begin + blockIdx.x; e < g.e_end; e += gridDim.x) {
    const uint32_t e32 = uint32_t(e), exy = e32 / s32;
    NodeRef nr;
    nr.e = e;
    nr.cz = int(e32 - exy * s32);
    nr.cx = int(exy / s32);
    nr.cy = int(exy - uint32_t(nr.cx) * s32);
    const int64_t own = (e - g.e_begin) * n3;
    for (int i0 = 0; i0 < IT; i0 += CH) {
      double pv[CH], xv[CH], rv[CH], wv[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) {  // the chunk's loads first
        const int l = threadIdx.x + (i0 + c) * kDssThreads;
        if (l < n3) {
          pv[c] = p[own + l];
          xv[c] = x[own + l];
          rv[c] = r[own + l];
          wv[c] = wown[own + l];
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int l = threadIdx.x + (i0 + c) * kDssThreads;
        if (l < n3) {
          nr.i = l % n;
          nr.j = (l / n) % n;
          nr.k = l / (n * n);
          const double wm = (mask && on_boundary<N>(nr, g.side)) ? 0.0 : wv[c];
          x[own + l] = fma(alpha, pv[c], xv[c]);
          const double ri = fma(-alpha, wm, rv[c]);
          r[own + l] = ri;
          s = fma(ri, ri * inv_mult<N>(nr, g.side), s);
        }
      }
    }
  }
  s = block_sum<kDssThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

static int dss_blocks(const DssRange& g) {
  const int64_t n_el = g.e_end - g.e_begin;
  const int64_t cap = int64_t(sm_count()) * 8;
  return int(n_el < 1 ? 1 : (n_el < cap ? n_el : cap));
}

#define HX_DSS_DISPATCH(CALL)                                                   \
  switch (degree) {                                                            \
    case 1: CALL(1); case 2: CALL(2); case 3: CALL(3); case 4: CALL(4);        \
    case 5: CALL(5); case 6: CALL(6); case 7: CALL(7); case 8: CALL(8);        \
    case 9: CALL(9); case 10: CALL(10); case 11: CALL(11); case 12: CALL(12);  \
    case 13: CALL(13); case 14: CALL(14); case 15: CALL(15);                   \
    default: return cudaErrorInvalidValue;                                     \
  }

static DssRange range(int side, int64_t e_begin, int64_t e_end, int64_t base) {
  DssRange g;
  g.side = side;
  g.e_begin = e_begin;
  g.e_end = e_end;
  g.base = base;
  return g;
}

cudaError_t launch_dss(const double* in, double* out, int side, int degree, int mask,
                       int64_t e_begin, int64_t e_end, int64_t base, cudaStream_t s) {
  const DssRange g = range(side, e_begin, e_end, base);
  const int nb = dss_blocks(g);
#define HX_CALL(N)                                              \
  dss_kernel<N><<<nb, kDssThreads, 0, s>>>(in, out, g, mask);  \
  return cudaGetLastError();
  HX_DSS_DISPATCH(HX_CALL)
#undef HX_CALL
}

cudaError_t launch_dot_dss(const double* u, const double* v, int side, int degree,
                           int64_t e_begin, int64_t e_end, double* part, double* result,
                           cudaStream_t s) {
  const DssRange g = range(side, e_begin, e_end, e_begin);
  const int nb = dss_blocks(g);
  cudaError_t err;
#define HX_CALL(N)                                                 \
  dot_dss_kernel<N><<<nb, kDssThreads, 0, s>>>(u, v, g, part);    \
  if ((err = cudaGetLastError()) != cudaSuccess) return err;      \
  return launch_sum(part, nb, result, s);
  HX_DSS_DISPATCH(HX_CALL)
#undef HX_CALL
}

cudaError_t launch_dss_inplace(double* u, int side, int degree, int64_t lo, int64_t hi,
                               cudaStream_t s) {
  if (hi <= lo) return cudaSuccess;
  const int64_t work = (hi - lo) * int64_t(degree + 1) * (degree + 1);
  const int64_t want = (work + kDssThreads - 1) / kDssThreads;
  const int nb = int(want < int64_t(sm_count()) * 16 ? want : int64_t(sm_count()) * 16);
  cudaError_t err;
#define HX_CALL(N)                                                                \
  dss_pass_kernel<N, 0><<<nb, kDssThreads, 0, s>>>(u, side, lo, hi);             \
  if ((err = cudaGetLastError()) != cudaSuccess) return err;                     \
  dss_pass_kernel<N, 1><<<nb, kDssThreads, 0, s>>>(u, side, lo, hi);             \
  if ((err = cudaGetLastError()) != cudaSuccess) return err;                     \
  dss_pass_kernel<N, 2><<<nb, kDssThreads, 0, s>>>(u, side, lo, hi);             \
  return cudaGetLastError();
  HX_DSS_DISPATCH(HX_CALL)
#undef HX_CALL
}

cudaError_t launch_cg_update_assembled(double* x, const double* p, double* r, double* ap,
                                       int side, int degree, int mask, int64_t e_begin,
                                       int64_t e_end, int64_t ap_base, int64_t ap_end,
                                       const double* rr, const double* pap, double* part,
                                       double* rr_new, cudaStream_t s) {
  const DssRange g = range(side, e_begin, e_end, ap_base);
  const int nb = dss_blocks(g);
  const int64_t work = (ap_end - ap_base) * int64_t(degree + 1) * (degree + 1);
  const int64_t want = (work + kDssThreads - 1) / kDssThreads;
  const int np = int(want < 1 ? 1 : (want < int64_t(sm_count()) * 16 ? want
                                                                     : int64_t(sm_count()) * 16));
  cudaError_t err;
#define HX_CALL(N)                                                                           \
  dss_pass_kernel<N, 0><<<np, kDssThreads, 0, s>>>(ap, side, ap_base, ap_end);               \
  if ((err = cudaGetLastError()) != cudaSuccess) return err;                                \
  dss_pass_kernel<N, 1><<<np, kDssThreads, 0, s>>>(ap, side, ap_base, ap_end);               \
  if ((err = cudaGetLastError()) != cudaSuccess) return err;                                \
  dss_pass_kernel<N, 2><<<np, kDssThreads, 0, s>>>(ap, side, ap_base, ap_end);               \
  if ((err = cudaGetLastError()) != cudaSuccess) return err;                                \
  cg_update_assembled_kernel<N><<<nb, kDssThreads, 0, s>>>(x, p, r, ap, g, mask, rr, pap,    \
                                                           part);                           \
  if ((err = cudaGetLastError()) != cudaSuccess) return err;                                \
  return launch_sum(part, nb, rr_new, s);
  HX_DSS_DISPATCH(HX_CALL)
#undef HX_CALL
}

}  // namespace hx
