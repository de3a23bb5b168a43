/*
 * hexbench_b200 -- C ABI of the B200-native BP1.0 / BP3.5 / BP3.0 element matvecs.
 *
 * The reference (`hexbench`, /root/reference/pkg) is pure Python and has no
 * FFI; these entry points are what its operator layer binds to when the
 * per-element numpy loop is replaced by sm_100a kernels.  Each function cites
 * the reference interface it stands in for.  Plain pointers and sizes only:
 * device buffers belong to the caller (PyTorch tensors in the Python layer),
 * the plan owns only its copy of the 1-D matrices.
 *
 * Conventions
 *   - fields q / out: element-major (n_el, (N+1)^3) float64, point order
 *     (k, j, i) with i fastest -- identical to FieldVector.data
 *     (reference operators.py:67-79).
 *   - factors: packed device layout, per element `n_slots` slots of
 *     `slot_stride` doubles (see hx_plan_factor_layout).  Slot order is the
 *     reference's FACTOR_NAMES (mesh.py:12); BP1.0 keeps only GwJ, stored
 *     i-major: point (k, j, i) at i*q^2 + k*q + j (every other slot is in the
 *     reference point order, k*q^2 + j*q + i).
 *   - every call that takes a `stream` is asynchronous on that cudaStream_t
 *     (NULL = legacy default stream) and never synchronises the device.
 *   - status: 0 on success, otherwise an HX_E* code; hx_strerror explains it.
 *   - threads: a plan is immutable after hx_plan_create, so calls on one plan
 *     from several host threads / streams are safe for distinct outputs; the
 *     host-buffer pipeline's lazily created streams are the one shared
 *     resource and hx_apply_host serialises its enqueue per plan.
 */
#ifndef HEXBENCH_B200_H
#define HEXBENCH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HX_OK = 0,
  HX_EINVAL = 1,       /* bad argument: maps to ValueError */
  HX_ENONFINITE = 2,   /* q holds inf/nan: ValueError (operators.py:317-318) */
  HX_EDEGENERATE = 3,  /* non-positive Jacobian: DegenerateGeometryError (mesh.py:128-129) */
  HX_ECUDA = 4,        /* CUDA runtime failure: RuntimeError */
  HX_ENOMEM = 5        /* host allocation failed */
};

/* benchmark ids (reference operators.py:30-33: "BP1.0", "BP3.5", "BP3.0") */
enum { HX_BP1 = 10, HX_BP35 = 35, HX_BP3 = 30 };

/* flag bits the kernels OR into *status_flag */
enum { HX_FLAG_NONFINITE = 1, HX_FLAG_DEGENERATE = 2 };

typedef struct hx_plan hx_plan;

/* Replaces the matrix / rule selection of make_operator (operators.py:118-143).
 *   interp : (N+2) x (N+1) row-major I            (BP1.0, BP3.0; NULL for BP3.5)
 *   diff   : q x q row-major D (q=N+1) or D~ (q=N+2) (BP3.5, BP3.0; NULL for BP1.0)
 *   nodes, weights : the q-point rule the factors live on (GL N+2 for BP1.0/3.0,
 *                    GLL N+1 for BP3.5)
 * Validation mirrors operators.py:120-129 (unknown bp, lam < 0, degree 1..15).
 * Touches no device state.                                                  */
int hx_plan_create(int bp, int degree, double lam, const double* interp, const double* diff,
                   const double* nodes, const double* weights, hx_plan** out);

/* Releases the plan (and any streams/events hx_apply_host created). */
void hx_plan_destroy(hx_plan* plan);

/* Packed factor layout of the plan: slots per element, doubles per slot and
 * doubles per element (= n_slots * slot_stride).                            */
int hx_plan_factor_layout(const hx_plan* plan, int* n_slots, int64_t* slot_stride,
                          int64_t* element_stride);

/* Replaces geometric_factors (mesh.py:101-139) for the plan's rule, on device.
 *   vertices : device (n_el, 8, 3) float64 corner coordinates (HexMesh.vertices)
 *   all_slots: 0 -> the plan's packed layout; 1 -> all 7 slots with the same
 *              slot_stride (used to materialise the reference array)
 *   status_flag: device int; HX_FLAG_DEGENERATE is OR-ed in if det <= 1e-14  */
int hx_geometric_factors(const hx_plan* plan, const double* vertices, int64_t n_el,
                         int all_slots, double* factors, int* status_flag, void* stream);

/* Converts between the reference factor layout (n_el, 7, q^3) and the packed
 * layout, device to device.  to_packed = 1: ref -> packed, 0: packed(7 slots)
 * -> ref.                                                                    */
int hx_repack_factors(const hx_plan* plan, const double* src, int64_t n_el, double* dst,
                      int to_packed, void* stream);

/* Replaces apply_operator / apply_bp1 / apply_bp35 / apply_bp3
 * (operators.py:306-349) on device-resident data: out = A q for elements
 * [0, n_el).  One fused kernel launch; no allocation, no synchronisation.
 * status_flag (device int, may be NULL) receives HX_FLAG_NONFINITE if any q
 * entry is inf/nan (the reference's np.isfinite scan, fused into the load).
 * The kernel is a programmatic dependent launch: it may start while the
 * previous kernel on `stream` retires, but issues nothing except L2 prefetch
 * hints before that kernel has completed -- plain stream order for every
 * read of q / factors and write of out (hx_apply_range, hx_apply_energy and
 * hx_apply_energy_dir likewise).                                            */
int hx_apply(const hx_plan* plan, const double* q, const double* factors, double* out,
             int64_t n_el, int* status_flag, void* stream);

/* hx_apply on the element range [e_begin, e_end) of full-size arrays (q, out:
 * n_el * (degree+1)^3 doubles from element 0; factors from element 0): the
 * range form of SURVEY.md §8b's boundary, what a rank of the element
 * partition calls (operators.py:324-331 chunks the same way).              */
int hx_apply_range(const hx_plan* plan, const double* q, const double* factors, double* out,
                   int64_t e_begin, int64_t e_end, int* status_flag, void* stream);

/* End-to-end variant on HOST q / out (page-locked for full overlap): chunks of
 * up to `chunk_el` elements (ramped up and down at the ends) are copied in,
 * applied and copied back on a three-stream pipeline with three buffer slots,
 * so PCIe transfers in both directions overlap each other and the kernel.
 * Stream-ordered like hx_apply: the pipeline starts after everything queued
 * on `stream` before the call (so q_host may be produced by earlier work on
 * `stream`, e.g. a previous call's D2H), and `stream` is made to wait for the
 * whole pipeline.  `work` is a device buffer of at least
 * hx_apply_host_workspace(plan, chunk_el) bytes, used under the same stream
 * order.  The pipeline streams live on the device current at the call (they
 * are rebuilt if a plan moves to another device).  On an error return no copy
 * into or out of the host buffers is still in flight.                        */
int64_t hx_apply_host_workspace(const hx_plan* plan, int64_t chunk_el);
int hx_apply_host(const hx_plan* plan, const double* q_host, const double* factors,
                  double* out_host, int64_t n_el, int64_t chunk_el, void* work,
                  int* status_flag, void* stream);

/* hx_apply_host with flags.  HX_HOST_OVERLAP opts into back-to-back
 * pipelining for streaming callers: the call does NOT wait for work queued on
 * `stream` before it; it follows only this plan's previous host-pipeline call
 * and continues its buffer-slot sequence (when `work` and `chunk_el` are
 * unchanged), so its H2D copies and kernels run under the previous call's D2H
 * tail, and its chunks are uniform (no ramp).  The caller guarantees that
 * q_host already holds its final contents, that nothing else reads or writes
 * q_host / out_host until `stream` reaches the end of the call, and that
 * `work` is used by no other plan or stream.  `stream` still waits for the
 * whole pipeline.  flags = 0 is exactly hx_apply_host.                      */
#define HX_HOST_OVERLAP 1u
int hx_apply_host_ex(const hx_plan* plan, const double* q_host, const double* factors,
                     double* out_host, int64_t n_el, int64_t chunk_el, void* work,
                     int* status_flag, unsigned flags, void* stream);

/* Drop-in host path for the arrays the reference's users pass to
 * apply_operator (operators.py:306-331): q_host / out_host may be PAGEABLE
 * (plain numpy memory).  Pageable buffers stream through `staging`, a
 * page-locked host buffer of hx_apply_host_staging_bytes(plan, chunk_el)
 * bytes: host worker threads copy chunk c+1 of q into a pinned slot while
 * chunk c is on PCIe / in the kernel, and copy finished chunks of out back
 * while later ones run; page-locked q_host / out_host skip their staging.
 * Same device pipeline and `work` buffer as hx_apply_host, same stream order;
 * HOST-SYNCHRONOUS: returns once out_host holds the result (or on error,
 * with no copy touching the host buffers still in flight).  Worker threads:
 * hardware concurrency, or HX_HOST_THREADS.                                  */
int64_t hx_apply_host_staging_bytes(const hx_plan* plan, int64_t chunk_el);
int hx_apply_host_staged(const hx_plan* plan, const double* q_host, const double* factors,
                         double* out_host, int64_t n_el, int64_t chunk_el, void* work,
                         void* staging, int* status_flag, void* stream);

/* The reference's up-front non-finite scan (operators.py:317-318), for
 * callers that must not have an output buffer touched on bad input (the
 * applies themselves fuse the same test into their loads):
 *   hx_check_finite   : device x[0, n); ORs HX_FLAG_NONFINITE into the device
 *                       int *status_flag (asynchronous on `stream`)
 *   hx_host_all_finite: host x[0, n) scanned by the host worker threads;
 *                       returns 1 if every entry is finite, else 0           */
int hx_check_finite(const double* x, int64_t n, int* status_flag, void* stream);
int hx_host_all_finite(const double* x, int64_t n);

/* Unfused "baseline" apply: the paper's Kernel-1 structure and
 * the reference's variant="baseline" access pattern (operators.py:170-200):
 * one launch per 1-D contraction pass / pointwise step, intermediates in HBM,
 * in the reference's pass order (operators.py:208-268).  Same result as
 * hx_apply up to rounding; exists to measure the fused kernels against.
 * `work` is a device buffer of hx_apply_baseline_workspace(plan, n_el) bytes. */
int64_t hx_apply_baseline_workspace(const hx_plan* plan, int64_t n_el);
int hx_apply_baseline(const hx_plan* plan, const double* q, const double* factors, double* out,
                      int64_t n_el, void* work, int* status_flag, void* stream);

/* Element helpers, batched: replace interpolate_to_gl / project_to_gll
 * (operators.py:352-364), which act on one (n,n,n) / (m,m,m) element tensor.
 * `interp` is the HOST m x n row-major GLL->GL matrix (reference_ops.py:39-44,
 * m = degree+2, n = degree+1); `src`/`dst` are device arrays of n_el element
 * tensors, (k,j,i) point order:
 *   project = 0: dst (n_el, m^3) = I (x) I (x) I  src (n_el, n^3)
 *   project = 1: dst (n_el, n^3) = I^T (x) I^T (x) I^T  src (n_el, m^3)
 * status_flag as in hx_apply (non-finite src).  Asynchronous on `stream`.
 * Centro-symmetric matrices (every GLL->GL interpolation matrix) take the
 * folded fused kernel; any other finite matrix takes unfused dense passes
 * with stream-ordered scratch (cudaMallocAsync), like the reference's
 * contract_dim, which accepts any 2-D matrix.                                */
int hx_interp_elements(int degree, const double* interp, int project, const double* src,
                       double* dst, int64_t n_el, int* status_flag, void* stream);

/* apply + <q, A q>: as hx_apply, and *energy (device double) receives
 * <q, A q>, evaluated inside the kernel from its quadrature-point values
 * (grad q . G grad q + lam GwJ q^2; GwJ (I q)^2 for BP1.0) -- no extra pass
 * over q or out.  `partials` is device scratch of n_partials >=
 * hx_energy_partials() doubles.  New: the reference has no solver; this
 * serves the CG driver.                       */
int64_t hx_energy_partials(void);
int hx_apply_energy(const hx_plan* plan, const double* q, const double* factors, double* out,
                    int64_t n_el, double* partials, int64_t n_partials, double* energy,
                    int* status_flag, void* stream);

/* CG direction update fused into the next matvec: p = r + (*rr_new / *rr_old) p
 * (hx_cg_direction's formula, bit for bit), then hx_apply_energy of the new p
 * -- out = A p, *energy = <p, A p> -- in one kernel that reads p_old and r
 * where it would read q and stores p back, so the direction update needs no
 * pass of its own.  p, r and out must be distinct element-local arrays of
 * n_el * (N+1)^3 doubles.  New: serves the CG driver.       */
int hx_apply_energy_dir(const hx_plan* plan, double* p, const double* r, const double* rr_new,
                        const double* rr_old, const double* factors, double* out, int64_t n_el,
                        double* partials, int64_t n_partials, double* energy, int* status_flag,
                        void* stream);

/* CG vector kernels on device arrays of n doubles; scalars are device
 * pointers so an iteration never synchronises with the host.
 *   hx_dot:          *result = <u, v>
 *   hx_cg_update:    alpha = *rr / *pap; x += alpha p; r -= alpha ap; *rr_new = <r, r>
 *   hx_cg_direction: p = r + (*rr_new / *rr_old) p
 * Reductions are fixed-order (bitwise reproducible).                        */
int hx_dot(const double* u, const double* v, int64_t n, double* partials, int64_t n_partials,
           double* result, void* stream);
int hx_cg_update(double* x, const double* p, double* r, const double* ap, int64_t n,
                 const double* rr, const double* pap, double* partials, int64_t n_partials,
                 double* rr_new, void* stream);
int hx_cg_direction(double* p, const double* r, int64_t n, const double* rr_new,
                    const double* rr_old, void* stream);

/* Assembly on the structured cube mesh of build_cube_mesh(side, extent)
 * (mesh.py:44-56; element e = (cx*side + cy)*side + cz, local (k,j,i) is
 * global node (cx N + i, cy N + j, cz N + k)).  New: the reference has no
 * assembly; this serves the assembled CG solve.
 * side <= 1600.  Each call processes the elements [e_begin, e_end) (a rank's shard; 0 and
 * side^3 on one GPU).  Own vectors (out, u, v, x, p, r) hold exactly those
 * elements; the GATHERED vector (in, ap) holds elements from `*_base` on and
 * must include every element that shares a node with the range (at most
 * side^2 + side + 1 elements beyond either end: the halo).
 *   hx_dss:           out = mask . Q Q^T in  (sum over the copies of each
 *                     global node, canonical order: bitwise deterministic;
 *                     mask_boundary zeroes the cube-boundary nodes)
 *   hx_dot_dss:       *result = sum u v / multiplicity over the range
 *                     (= <u_G, v_G> for continuous representatives, summed
 *                     over ranks)
 * The per-iteration assembled update is hx_cg_update_assembled (below).     */
int hx_dss(const double* in, double* out, int side, int degree, int mask_boundary,
           int64_t e_begin, int64_t e_end, int64_t in_base, void* stream);
int hx_dot_dss(const double* u, const double* v, int side, int degree, int64_t e_begin,
               int64_t e_end, double* partials, int64_t n_partials, double* result,
               void* stream);

/* Separable in-place gather-scatter: u (a buffer holding elements
 * [buf_begin, buf_end)) <- Q Q^T u as three per-axis face passes (each copy of
 * a face node becomes lower-element copy + upper-element copy).  Exact for
 * every node whose copies all lie in the buffer (a rank's own elements, given
 * its halo); bitwise deterministic and continuous, but summed in pass order,
 * not hx_dss's gather order.  No masking.
 *   hx_cg_update_assembled: the assembled-CG update -- ap (= A_L p for the
 *   elements [ap_base, ap_end): own range plus exchanged halo; used as
 *   scratch and overwritten) is assembled in place (the three face passes),
 *   then as hx_cg_update with
 *   r -= alpha mask (Q Q^T ap) and the multiplicity-weighted <r, r>.     */
int hx_dss_inplace(double* u, int side, int degree, int64_t buf_begin, int64_t buf_end,
                   void* stream);
int hx_cg_update_assembled(double* x, const double* p, double* r, double* ap, int side,
                           int degree, int mask_boundary, int64_t e_begin, int64_t e_end,
                           int64_t ap_base, int64_t ap_end, const double* rr, const double* pap,
                           double* partials, int64_t n_partials, double* rr_new, void* stream);

/* Elements each CTA processes per tile, threads per CTA and dynamic shared
 * memory bytes of the plan's kernel (for reports and tests).                */
int hx_plan_kernel_shape(const hx_plan* plan, int* elements_per_tile, int* threads,
                         int* smem_bytes);

/* Shared-memory bandwidth probe (harness calibration replacing the B_sh
 * ansatz, perf.py:155-160): fills *bytes_per_s with the measured aggregate
 * LDS bandwidth of the current device.  Synchronises `stream`.              */
int hx_measure_smem_bandwidth(double* bytes_per_s, void* stream);

const char* hx_strerror(int status);

/* 1 if the library was built for (and the current device is) sm_100. */
int hx_device_ok(void);

#ifdef __cplusplus
}
#endif

#endif /* HEXBENCH_B200_H */
