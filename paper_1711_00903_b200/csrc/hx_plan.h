// Host-side plan object behind the C ABI (include/hexbench_b200.h).
#pragma once

#include <cstdint>
#include <mutex>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/hexbench_b200.h"

namespace hx {

constexpr int kMaxQ = 17;  // N <= 15 -> at most N+2 points per axis

}  // namespace hx

// device buffer slots of the host pipeline (hx_apply_host): H2D, kernel and
// D2H of up to this many chunks are in flight at once
constexpr int hx_host_slots = 3;

struct hx_plan {
  int bp;       // HX_BP1 / HX_BP35 / HX_BP3
  int degree;   // N
  int n, m;     // GLL points (N+1) and GL points (N+2) per axis
  int q;        // quadrature points per axis of the factor rule (m, or n for BP3.5)
  double lam;
  double interp[hx::kMaxQ * hx::kMaxQ];  // m x n, row-major (BP1, BP3)
  double diff[hx::kMaxQ * hx::kMaxQ];    // q x q, row-major (BP3.5, BP3)
  double nodes[hx::kMaxQ];               // factor rule nodes / weights
  double weights[hx::kMaxQ];
  int n_slots;            // factor slots kept on device (1 for BP1, 7 otherwise)
  int64_t slot_stride;    // doubles per slot (q^3 rounded up to even)
  int64_t elem_stride;    // doubles per element (n_slots * slot_stride)
  // lazily created resources for the host-buffer (end-to-end) path, on
  // device `pipe_dev`; `pipe_mu` serialises hx_apply_host calls on one plan
  // (they share these streams and events), everything else about a plan is
  // immutable after create
  cudaStream_t pipe[3];
  cudaEvent_t ev[3][hx_host_slots];
  cudaEvent_t pipe_last;  // end of the plan's latest host-pipeline call
  // HX_HOST_OVERLAP continuation state: slot sequence, workspace and chunk
  // of the previous call (continued only when unchanged)
  int64_t pipe_seq = 0;
  const void* pipe_work = nullptr;
  int64_t pipe_chunk = 0;
  bool pipe_cont = false;
  bool pipe_ready;
  int pipe_dev = -1;
  std::mutex pipe_mu;
};

namespace hx {

// CG direction fused into the matvec's first load (hx_common.cuh load_line):
// the kernel forms p = r + (rr_new / rr_old) p, stores it and applies A to it
struct DirArgs {
  double* p;
  const double* r;
  const double* rr_new;
  const double* rr_old;
};

// the fused kernel of the plan's operator (energy: per-CTA <q, A q> partials)
// (pdl: as a programmatic dependent launch, hx_common.cuh launch_kernel)
// (dir: q is ignored and the operator applies to the updated direction)
cudaError_t launch_apply(const hx_plan& P, const double* q, const double* fac, double* out,
                         int64_t n_el, int* flag, cudaStream_t s, double* energy = nullptr,
                         bool pdl = false, const DirArgs* dir = nullptr);
// host pipeline helpers (hx_capi.cu): chunk sizes, lazily built streams
std::vector<int64_t> chunk_schedule(int64_t n_el, int64_t chunk_el);
cudaError_t pipe_setup(hx_plan* P);
int cuda_status(cudaError_t err);

// BP1.0's packed GwJ slot order for a degree: point (k, j, i) of the
// (m, m, m) GL tensor lives at i*m^2 + k*m + j, or -- when the degree's S3
// runs c-fastest (Cfg ORD bit 8, hx_bp1.cu) -- at i*m^2 + j*m + k
bool bp1_gwj_cfast(int degree);
__host__ __device__ inline int bp1_gwj_index(int k, int j, int i, int m, bool cfast) {
  return cfast ? (i * m + j) * m + k : (i * m + k) * m + j;
}

// launch the fused element kernel for elements [0, n_el) of device arrays
cudaError_t launch_bp1(const hx_plan& P, const double* q, const double* fac, double* out,
                       int64_t n_el, int* flag, double* energy, cudaStream_t s, bool pdl,
                       const DirArgs* dir);
cudaError_t launch_bp35(const hx_plan& P, const double* q, const double* fac, double* out,
                        int64_t n_el, int* flag, double* energy, cudaStream_t s, bool pdl,
                        const DirArgs* dir);
cudaError_t launch_bp3(const hx_plan& P, const double* q, const double* fac, double* out,
                       int64_t n_el, int* flag, double* energy, cudaStream_t s, bool pdl,
                       const DirArgs* dir);
cudaError_t launch_baseline(const hx_plan& P, const double* q, const double* fac, double* out,
                            int64_t n_el, double* work, int* flag, cudaStream_t s);
int64_t baseline_workspace_doubles(const hx_plan& P, int64_t n_el);
cudaError_t launch_interp(int degree, const double* interp, int project, const double* src,
                          double* dst, int64_t n_el, int* flag, cudaStream_t s);
cudaError_t launch_interp_dense(int degree, const double* interp, int project, const double* src,
                                double* dst, int64_t n_el, cudaStream_t s);
cudaError_t launch_check_finite(const double* x, int64_t n, int* flag, cudaStream_t s);
cudaError_t launch_geometry(const hx_plan& P, const double* verts, int64_t n_el, int all_slots,
                            double* fac, int* flag, cudaStream_t s);
cudaError_t launch_repack(const hx_plan& P, const double* src, int64_t n_el, double* dst,
                          int to_packed, cudaStream_t s);
cudaError_t launch_smem_probe(double* sink, int iters, float* ms, cudaStream_t s);
cudaError_t launch_sum(const double* part, int n, double* out, cudaStream_t s);
cudaError_t launch_dot(const double* u, const double* v, int64_t n, double* part,
                       double* result, cudaStream_t s);
cudaError_t launch_cg_update(double* x, const double* p, double* r, const double* ap, int64_t n,
                             const double* rr, const double* pap, double* part, double* rr_new,
                             cudaStream_t s);
cudaError_t launch_cg_direction(double* p, const double* r, int64_t n, const double* rr_new,
                                const double* rr_old, cudaStream_t s);

cudaError_t launch_dss(const double* in, double* out, int side, int degree, int mask,
                       int64_t e_begin, int64_t e_end, int64_t base, cudaStream_t s);
cudaError_t launch_dot_dss(const double* u, const double* v, int side, int degree,
                           int64_t e_begin, int64_t e_end, double* part, double* result,
                           cudaStream_t s);

cudaError_t launch_dss_inplace(double* u, int side, int degree, int64_t lo, int64_t hi,
                               cudaStream_t s);
cudaError_t launch_cg_update_assembled(double* x, const double* p, double* r, double* ap,
                                       int side, int degree, int mask, int64_t e_begin,
                                       int64_t e_end, int64_t ap_base, int64_t ap_end,
                                       const double* rr, const double* pap, double* part,
                                       double* rr_new, cudaStream_t s);

int sm_count();

}  // namespace hx
