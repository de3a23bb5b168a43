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
// Assembled CG keeps every vector in element-local storage as its continuous
// representative u_L = Q u_G.  Then
//   <p_G, A_G p_G> = <p_L, A_L p_L>                 (fused into the matvec)
//   A_G p_G        -> mask dss(A_L p_L)             (fused into the update)
//   <r_G, r_G>     = sum_L r_L^2 / multiplicity      (fused into the update)
#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {

constexpr int kDssThreads = 256;

struct DssGeom {
  int side, n;        // elements per cube side, GLL points per axis (N + 1)
  int64_t n3, ndof;   // n^3, side^3 n^3
  int mask;           // zero boundary nodes
};

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

struct NodeRef {
  int64_t e;
  int k, j, i, cx, cy, cz;
};

__device__ __forceinline__ NodeRef decompose(int64_t idx, const DssGeom& g) {
  NodeRef r;
  r.e = idx / g.n3;
  const int loc = int(idx - r.e * g.n3);
  r.i = loc % g.n;
  r.j = (loc / g.n) % g.n;
  r.k = loc / (g.n * g.n);
  const int64_t s = g.side;
  r.cz = int(r.e % s);
  r.cy = int((r.e / s) % s);
  r.cx = int(r.e / (s * s));
  return r;
}

__device__ __forceinline__ bool on_boundary(const NodeRef& r, const DssGeom& g) {
  const int N = g.n - 1, G = g.side * N;
  const int gx = r.cx * N + r.i, gy = r.cy * N + r.j, gz = r.cz * N + r.k;
  return gx == 0 || gx == G || gy == 0 || gy == G || gz == 0 || gz == G;
}

// number of element-local copies of node r
__device__ __forceinline__ int node_mult(const NodeRef& r, const DssGeom& g) {
  const int N = g.n - 1;
  return axis_copies(r.cx, r.i, g.side, N).cnt * axis_copies(r.cy, r.j, g.side, N).cnt *
         axis_copies(r.cz, r.k, g.side, N).cnt;
}

// sum over the copies of node r, in the canonical order
__device__ __forceinline__ double gather_sum(const double* __restrict__ u, const NodeRef& r,
                                             const DssGeom& g) {
  const int N = g.n - 1;
  const AxisCopies ax = axis_copies(r.cx, r.i, g.side, N);
  const AxisCopies ay = axis_copies(r.cy, r.j, g.side, N);
  const AxisCopies az = axis_copies(r.cz, r.k, g.side, N);
  const int64_t s = g.side;
  double sum = 0.0;
  for (int a = 0; a < ax.cnt; ++a)
    for (int b = 0; b < ay.cnt; ++b)
      for (int c = 0; c < az.cnt; ++c) {
        const int64_t e = r.e + ax.d[a] * s * s + ay.d[b] * s + az.d[c];
        sum += u[e * g.n3 + (int64_t(az.l[c]) * g.n + ay.l[b]) * g.n + ax.l[a]];
      }
  return sum;
}

__global__ void __launch_bounds__(kDssThreads)
    dss_kernel(const double* __restrict__ in, double* __restrict__ out, DssGeom g) {
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < g.ndof;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const NodeRef r = decompose(idx, g);
    out[idx] = (g.mask && on_boundary(r, g)) ? 0.0 : gather_sum(in, r, g);
  }
}

// partials of sum u v / multiplicity (the global inner product of continuous
// representatives)
__global__ void __launch_bounds__(kDssThreads)
    dot_dss_kernel(const double* __restrict__ u, const double* __restrict__ v, DssGeom g,
                   double* __restrict__ part) {
  __shared__ double scratch[kDssThreads / 32];
  double s = 0.0;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < g.ndof;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const NodeRef r = decompose(idx, g);
    s = fma(u[idx], v[idx] / double(node_mult(r, g)), s);
  }
  s = block_sum<kDssThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// alpha = rr / pAp;  x += alpha p;  r -= alpha mask dss(ap);  partials of
// sum r^2 / multiplicity.  The assembled A p is never written to memory.
__global__ void __launch_bounds__(kDssThreads)
    cg_update_dss_kernel(double* __restrict__ x, const double* __restrict__ p,
                         double* __restrict__ r, const double* __restrict__ ap, DssGeom g,
                         const double* __restrict__ rr, const double* __restrict__ pap,
                         double* __restrict__ part) {
  __shared__ double scratch[kDssThreads / 32];
  const double alpha = rr[0] / pap[0];
  double s = 0.0;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < g.ndof;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const NodeRef nr = decompose(idx, g);
    const double w = (g.mask && on_boundary(nr, g)) ? 0.0 : gather_sum(ap, nr, g);
    x[idx] = fma(alpha, p[idx], x[idx]);
    const double ri = fma(-alpha, w, r[idx]);
    r[idx] = ri;
    s = fma(ri, ri / double(node_mult(nr, g)), s);
  }
  s = block_sum<kDssThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

static int dss_blocks(int64_t n) {
  const int64_t want = (n + kDssThreads - 1) / kDssThreads;
  const int64_t cap = int64_t(sm_count()) * 8;
  return int(want < cap ? (want > 0 ? want : 1) : cap);
}

static DssGeom geom(int side, int degree, int mask) {
  DssGeom g;
  g.side = side;
  g.n = degree + 1;
  g.n3 = int64_t(g.n) * g.n * g.n;
  g.ndof = int64_t(side) * side * side * g.n3;
  g.mask = mask;
  return g;
}

cudaError_t launch_dss(const double* in, double* out, int side, int degree, int mask,
                       cudaStream_t s) {
  const DssGeom g = geom(side, degree, mask);
  dss_kernel<<<dss_blocks(g.ndof), kDssThreads, 0, s>>>(in, out, g);
  return cudaGetLastError();
}

cudaError_t launch_dot_dss(const double* u, const double* v, int side, int degree,
                           double* part, double* result, cudaStream_t s) {
  const DssGeom g = geom(side, degree, 0);
  const int nb = dss_blocks(g.ndof);
  dot_dss_kernel<<<nb, kDssThreads, 0, s>>>(u, v, g, part);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  return launch_sum(part, nb, result, s);
}

cudaError_t launch_cg_update_dss(double* x, const double* p, double* r, const double* ap,
                                 int side, int degree, int mask, const double* rr,
                                 const double* pap, double* part, double* rr_new,
                                 cudaStream_t s) {
  const DssGeom g = geom(side, degree, mask);
  const int nb = dss_blocks(g.ndof);
  cg_update_dss_kernel<<<nb, kDssThreads, 0, s>>>(x, p, r, ap, g, rr, pap, part);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  return launch_sum(part, nb, rr_new, s);
}

}  // namespace hx
