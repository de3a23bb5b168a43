// Device-side setup: geometric factors (reference mesh.py:101-139), layout
// repacking, and the shared-memory bandwidth probe used by the harness.
#include "hx_common.cuh"
#include "hx_plan.h"

namespace hx {

struct GeomParams {
  double nodes[kMaxQ];
  double weights[kMaxQ];
  const double* verts;  // (E, 8, 3)
  double* fac;          // packed: E x (nslot x sstride)
  int64_t n_el;
  int64_t estride, sstride;
  int q;         // points per axis
  int gwj_only;  // 1: write only GwJ into slot 0
  int gwj_cfast; // BP1.0 GwJ slot order (bp1_gwj_index)
  int* flag;
};

// One thread per (element, point).  A = sum_c x_c (x) grad phi_c, then
// G = det(A) A^-1 A^-T = adj(A) adj(A)^T / det(A), GwJ = det(A), all scaled
// by w_i w_j w_k.  Same corner ordering as reference mesh.py:9.
__global__ void geometry_kernel(const __grid_constant__ GeomParams p) {
  const int q = p.q, q3 = q * q * q;
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= p.n_el * q3) return;
  const int64_t e = gid / q3;
  const int pt = int(gid % q3);
  const int kk = pt / (q * q), jj = (pt / q) % q, ii = pt % q;
  const double r = p.nodes[ii], s = p.nodes[jj], t = p.nodes[kk];
  const double* v = p.verts + e * 24;
  double a[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double rc = (c & 4) ? 1.0 : -1.0, sc = (c & 2) ? 1.0 : -1.0,
                 tc = (c & 1) ? 1.0 : -1.0;
    const double dr = rc * (1 + s * sc) * (1 + t * tc) / 8.0;
    const double ds = (1 + r * rc) * sc * (1 + t * tc) / 8.0;
    const double dt = (1 + r * rc) * (1 + s * sc) * tc / 8.0;
#pragma unroll
    for (int x = 0; x < 3; ++x) {
      const double xc = v[c * 3 + x];
      a[x][0] += xc * dr;
      a[x][1] += xc * ds;
      a[x][2] += xc * dt;
    }
  }
  // adjugate (transpose of the cofactor matrix): inv = adj / det
  double adj[3][3];
  adj[0][0] = a[1][1] * a[2][2] - a[1][2] * a[2][1];
  adj[0][1] = a[0][2] * a[2][1] - a[0][1] * a[2][2];
  adj[0][2] = a[0][1] * a[1][2] - a[0][2] * a[1][1];
  adj[1][0] = a[1][2] * a[2][0] - a[1][0] * a[2][2];
  adj[1][1] = a[0][0] * a[2][2] - a[0][2] * a[2][0];
  adj[1][2] = a[0][2] * a[1][0] - a[0][0] * a[1][2];
  adj[2][0] = a[1][0] * a[2][1] - a[1][1] * a[2][0];
  adj[2][1] = a[0][1] * a[2][0] - a[0][0] * a[2][1];
  adj[2][2] = a[0][0] * a[1][1] - a[0][1] * a[1][0];
  const double det = a[0][0] * adj[0][0] + a[0][1] * adj[1][0] + a[0][2] * adj[2][0];
  if (!(det > 1e-14) && p.flag) atomicOr(p.flag, 2);
  const double w3 = p.weights[ii] * p.weights[jj] * p.weights[kk];
  if (p.gwj_only) {
    // BP1.0's packed slot is i-major (hx_bp1.cu S3): bp1_gwj_index
    p.fac[e * p.estride + bp1_gwj_index(kk, jj, ii, q, p.gwj_cfast)] = w3 * det;
    return;
  }
  double* dst = p.fac + e * p.estride + pt;
  const double sc = w3 / det;
  auto g = [&](int x, int y) {
    return sc * (adj[x][0] * adj[y][0] + adj[x][1] * adj[y][1] + adj[x][2] * adj[y][2]);
  };
  dst[0 * p.sstride] = g(0, 0);
  dst[1 * p.sstride] = g(0, 1);
  dst[2 * p.sstride] = g(0, 2);
  dst[3 * p.sstride] = g(1, 1);
  dst[4 * p.sstride] = g(1, 2);
  dst[5 * p.sstride] = g(2, 2);
  dst[6 * p.sstride] = w3 * det;
}

cudaError_t launch_geometry(const hx_plan& P, const double* verts, int64_t n_el, int all_slots,
                            double* fac, int* flag, cudaStream_t s) {
  if (n_el == 0) return cudaSuccess;
  GeomParams g;
  for (int i = 0; i < P.q; ++i) {
    g.nodes[i] = P.nodes[i];
    g.weights[i] = P.weights[i];
  }
  g.verts = verts;
  g.fac = fac;
  g.n_el = n_el;
  g.q = P.q;
  g.sstride = P.slot_stride;
  const bool gwj_only = !all_slots && P.n_slots == 1;
  g.gwj_only = gwj_only;
  g.gwj_cfast = gwj_only && bp1_gwj_cfast(P.degree);
  g.estride = all_slots ? 7 * P.slot_stride : P.elem_stride;
  g.flag = flag;
  const int64_t total = n_el * int64_t(P.q) * P.q * P.q;
  const int threads = 256;
  geometry_kernel<<<unsigned((total + threads - 1) / threads), threads, 0, s>>>(g);
  return cudaGetLastError();
}

// Reference layout (E, 7, q^3) <-> packed layout (E, nslot, sstride).
__global__ void repack_kernel(const double* __restrict__ src, double* __restrict__ dst,
                              int64_t n_el, int q, int nslot, int first_slot, int64_t sstride,
                              int to_packed, int imajor) {
  const int q3 = q * q * q;
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per = int64_t(nslot) * q3;
  if (gid >= n_el * per) return;
  const int64_t e = gid / per;
  const int rem = int(gid % per);
  const int sl = rem / q3, pt = rem % q3;
  const int64_t ref = (e * 7 + first_slot + sl) * q3 + pt;
  // BP1.0's single packed slot is i-major (hx_bp1.cu S3): bp1_gwj_index,
  // imajor = 1 + cfast
  int ppt = pt;
  if (imajor) {
    const int kk = pt / (q * q), jj = (pt / q) % q, ii = pt % q;
    ppt = bp1_gwj_index(kk, jj, ii, q, imajor == 2);
  }
  const int64_t pk = (e * nslot + sl) * sstride + ppt;
  if (to_packed)
    dst[pk] = src[ref];
  else
    dst[ref] = src[pk];
}

cudaError_t launch_repack(const hx_plan& P, const double* src, int64_t n_el, double* dst,
                          int to_packed, cudaStream_t s) {
  if (n_el == 0) return cudaSuccess;
  const int q3 = P.q * P.q * P.q;
  // ref -> packed keeps the plan's slots; packed -> ref expects all 7 slots
  const int nslot = to_packed ? P.n_slots : 7;
  const int first = (to_packed && P.n_slots == 1) ? 6 : 0;
  const int64_t total = n_el * int64_t(nslot) * q3;
  const int threads = 256;
  const int imajor = (to_packed && P.n_slots == 1) ? 1 + int(bp1_gwj_cfast(P.degree)) : 0;
  repack_kernel<<<unsigned((total + threads - 1) / threads), threads, 0, s>>>(
      src, dst, n_el, P.q, nslot, first, P.slot_stride, to_packed, imajor);
  return cudaGetLastError();
}

// Shared-memory bandwidth probe: every warp streams conflict-free 64-bit
// loads (32 consecutive doubles per warp request) from a 32 KB smem tile.
// The loads are volatile PTX so the compiler cannot merge repeated
// addresses, and the sum is written out so they cannot be elided.
__device__ __forceinline__ double lds_volatile(const double* p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];"
               : "=d"(v)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

__global__ void __launch_bounds__(512) smem_probe_kernel(double* sink, int iters) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i * 1e-9;
  __syncthreads();
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  const int lane = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int base = ((it * 8 + u) * 128) & 4095;
      acc0 += lds_volatile(buf + ((base + lane) & 4095));
      acc1 += lds_volatile(buf + ((base + lane + 1024) & 4095));
      acc2 += lds_volatile(buf + ((base + lane + 2048) & 4095));
      acc3 += lds_volatile(buf + ((base + lane + 3072) & 4095));
    }
  }
  if (acc0 + acc1 + acc2 + acc3 == 42.0) sink[blockIdx.x] = acc0;
}

cudaError_t launch_smem_probe(double* sink, int iters, float* ms, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sm_count() * 2;
  smem_probe_kernel<<<blocks, 512, 0, s>>>(sink, iters);  // warm-up
  cudaEventRecord(a, s);
  smem_probe_kernel<<<blocks, 512, 0, s>>>(sink, iters);
  cudaEventRecord(b, s);
  cudaError_t err = cudaEventSynchronize(b);
  if (err == cudaSuccess) err = cudaEventElapsedTime(ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (err != cudaSuccess) return err;
  return cudaGetLastError();
}

}  // namespace hx
