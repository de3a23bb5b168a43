// Conjugate-gradient building blocks around the element matvecs (SURVEY.md
// §8f rank 2: the matvec's real caller).  The operator stays
// element-local; CG needs three reductions per iteration, which are computed
// without extra passes over the vectors wherever possible:
//
//   <p, A p>   fused into the matvec kernel (ENERGY instantiation): evaluated
//              from the quadrature-point quantities the kernel already holds
//              (grad p . G grad p + lam GwJ p^2, or GwJ (I p)^2 for BP1.0);
//   <r, r>     fused into the x/r update kernel;
//   scalars    alpha, beta are read from device memory by the next kernel,
//              so an iteration never synchronises with the host.
//
// Every reduction is two-level and fixed-order (per-CTA partials, then one
// CTA sums them in index order), so a solve is bitwise reproducible.  Across
// GPUs the per-rank scalars are all-reduced (NCCL) between kernels.
#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {

constexpr int kVecThreads = 256;

int vec_blocks(int64_t n) {
  const int64_t want = (n + kVecThreads - 1) / kVecThreads;
  const int64_t cap = int64_t(sm_count()) * 8;
  return int(want < cap ? (want > 0 ? want : 1) : cap);
}

__global__ void __launch_bounds__(1024) sum_kernel(const double* __restrict__ part, int n,
                                                  double* __restrict__ out) {
  __shared__ double buf[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) s += part[i];
  buf[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) buf[threadIdx.x] += buf[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = buf[0];
}

cudaError_t launch_sum(const double* part, int n, double* out, cudaStream_t s) {
  sum_kernel<<<1, 1024, 0, s>>>(part, n, out);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(kVecThreads)
    dot_kernel(const double* __restrict__ u, const double* __restrict__ v, int64_t n,
               double* __restrict__ part) {
  __shared__ double scratch[kVecThreads / 32];
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    s = fma(u[i], v[i], s);
  s = block_sum<kVecThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// alpha = rr / pAp;  x += alpha p;  r -= alpha Ap;  partials of <r, r>
__global__ void __launch_bounds__(kVecThreads)
    cg_update_kernel(double* __restrict__ x, const double* __restrict__ p,
                     double* __restrict__ r, const double* __restrict__ ap, int64_t n,
                     const double* __restrict__ rr, const double* __restrict__ pap,
                     double* __restrict__ part) {
  __shared__ double scratch[kVecThreads / 32];
  const double alpha = rr[0] / pap[0];
  double s = 0.0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, ap[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum<kVecThreads>(s, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// beta = rr_new / rr_old;  p = r + beta p
__global__ void __launch_bounds__(kVecThreads)
    cg_direction_kernel(double* __restrict__ p, const double* __restrict__ r, int64_t n,
                        const double* __restrict__ rr_new, const double* __restrict__ rr_old) {
  const double beta = rr_new[0] / rr_old[0];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = fma(beta, p[i], r[i]);
}

cudaError_t launch_dot(const double* u, const double* v, int64_t n, double* part,
                       double* result, cudaStream_t s) {
  const int g = vec_blocks(n);
  dot_kernel<<<g, kVecThreads, 0, s>>>(u, v, n, part);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  return launch_sum(part, g, result, s);
}

cudaError_t launch_cg_update(double* x, const double* p, double* r, const double* ap, int64_t n,
                             const double* rr, const double* pap, double* part, double* rr_new,
                             cudaStream_t s) {
  const int g = vec_blocks(n);
  cg_update_kernel<<<g, kVecThreads, 0, s>>>(x, p, r, ap, n, rr, pap, part);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  return launch_sum(part, g, rr_new, s);
}

cudaError_t launch_cg_direction(double* p, const double* r, int64_t n, const double* rr_new,
                                const double* rr_old, cudaStream_t s) {
  cg_direction_kernel<<<vec_blocks(n), kVecThreads, 0, s>>>(p, r, n, rr_new, rr_old);
  return cudaGetLastError();
}

}  // namespace hx
