/* A plain C caller of the C ABI, built and run by
 * tests/test_gpu_capi_c.py on the GPU box: no Python, no torch -- the
 * library, the CUDA runtime and this file only.
 *
 * One element = the reference cube [0, 2]^3 of build_cube_mesh(1, 2.0)
 * (reference mesh.py:44-56, corners in itertools.product((-1, 1), repeat=3)
 * order), BP3.5 at N = 2 with lam = 1: the constant field's action integrates
 * to the volume (the reference's criterion 10, test_acceptance.py:227-240),
 * A q = A (2 q) / 2 (linearity), and an inf in q raises the non-finite flag.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "hexbench_b200.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int s_ = (x);                                                             \
    if (s_ != HX_OK) {                                                        \
      fprintf(stderr, "%s failed: %s\n", #x, hx_strerror(s_));                \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  if (!hx_device_ok()) {
    fprintf(stderr, "not an sm_100 device\n");
    return 2;
  }
  /* GLL rule with 3 points and its collocation derivative matrix (N = 2) */
  const double nodes[3] = {-1.0, 0.0, 1.0};
  const double weights[3] = {1.0 / 3.0, 4.0 / 3.0, 1.0 / 3.0};
  const double diff[9] = {-1.5, 2.0, -0.5, -0.5, 0.0, 0.5, 0.5, -2.0, 1.5};
  double verts[8 * 3];
  int c = 0;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int d = 0; d < 2; ++d) {
        verts[3 * c + 0] = 2.0 * a;
        verts[3 * c + 1] = 2.0 * b;
        verts[3 * c + 2] = 2.0 * d;
        ++c;
      }
  hx_plan* plan = NULL;
  CHECK(hx_plan_create(HX_BP35, 2, 1.0, NULL, diff, nodes, weights, &plan));
  int64_t est = 0;
  CHECK(hx_plan_factor_layout(plan, NULL, NULL, &est));

  double *d_verts, *d_fac, *d_q, *d_out;
  int* d_flag;
  cudaMalloc((void**)&d_verts, sizeof(verts));
  cudaMalloc((void**)&d_fac, sizeof(double) * est);
  cudaMalloc((void**)&d_q, sizeof(double) * 27);
  cudaMalloc((void**)&d_out, sizeof(double) * 27);
  cudaMalloc((void**)&d_flag, sizeof(int));
  cudaMemcpy(d_verts, verts, sizeof(verts), cudaMemcpyHostToDevice);
  cudaMemset(d_flag, 0, sizeof(int));
  CHECK(hx_geometric_factors(plan, d_verts, 1, 0, d_fac, d_flag, NULL));

  double q[27], out[27], out2[27];
  for (int i = 0; i < 27; ++i) q[i] = 1.0;
  cudaMemcpy(d_q, q, sizeof(q), cudaMemcpyHostToDevice);
  CHECK(hx_apply(plan, d_q, d_fac, d_out, 1, d_flag, NULL));
  cudaMemcpy(out, d_out, sizeof(out), cudaMemcpyDeviceToHost);
  double total = 0.0;
  for (int i = 0; i < 27; ++i) total += out[i];
  int flag = -1;
  cudaMemcpy(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost);
  printf("sum(A 1) = %.15f (volume 8), flag %d\n", total, flag);
  if (fabs(total - 8.0) > 1e-12 || flag != 0) return 3;

  /* linearity on a non-constant field, through the host-buffer pipeline */
  for (int i = 0; i < 27; ++i) q[i] = sin(0.3 * i) + 0.1 * i;
  CHECK(hx_apply_range(plan, d_q, d_fac, d_out, 0, 0, d_flag, NULL)); /* empty range */
  void* work;
  cudaMalloc(&work, (size_t)hx_apply_host_workspace(plan, 1));
  CHECK(hx_apply_host(plan, q, d_fac, out, 1, 1, work, d_flag, NULL));
  for (int i = 0; i < 27; ++i) q[i] *= 2.0;
  CHECK(hx_apply_host(plan, q, d_fac, out2, 1, 1, work, d_flag, NULL));
  cudaDeviceSynchronize();
  double worst = 0.0;
  for (int i = 0; i < 27; ++i) {
    const double e = fabs(out2[i] - 2.0 * out[i]);
    if (e > worst) worst = e;
  }
  printf("linearity defect %.3e\n", worst);
  if (worst > 1e-13) return 4;

  /* a non-finite input is flagged, as the reference raises ValueError */
  q[5] = INFINITY;
  cudaMemcpy(d_q, q, sizeof(q), cudaMemcpyHostToDevice);
  CHECK(hx_apply(plan, d_q, d_fac, d_out, 1, d_flag, NULL));
  cudaMemcpy(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost);
  printf("flag after inf: %d\n", flag);
  if (!(flag & HX_FLAG_NONFINITE)) return 5;

  cudaFree(work);
  cudaFree(d_verts);
  cudaFree(d_fac);
  cudaFree(d_q);
  cudaFree(d_out);
  cudaFree(d_flag);
  hx_plan_destroy(plan);
  printf("c_abi_example: ok\n");
  return 0;
}
