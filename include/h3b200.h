/*
 * h3b200 -- C ABI of the B200-native Hermite half-step (libh3b200.so).
 *
 * Drop-in boundary for the reference's grid kernels
 * (reference: pkg/src/hermite3d/gridkernels.py).  The reference binds these
 * through numba; the entry points below take exactly the arguments the
 * reference passes from pipeline.half_step (pipeline.py:247-266) --
 * src/dst DOF fields in the reference's rank-6 layout
 * [m3][m2][m1][n3][n2][n1] (C order, field.py:80-93), the interpolation matrix
 * h_mat (s x s), the derivative factors fac1..3 (s), the Horner stage factors
 * cfac (q) and the gather offset off -- plus what a device needs: a CUDA
 * stream, a slab range along x3, and a device flag for the fused
 * finiteness check (pipeline.py:210-215).
 *
 * Conventions
 *   - src/dst/coeff and every d_* pointer are DEVICE pointers; h_mat, fac*,
 *     cfac are HOST arrays (tiny, copied into kernel parameters per call).
 *   - All calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and reentrant.  The only process-wide state is a small
 *     constant-memory ring holding the DFMA kernels' operators; it is
 *     mutex-protected and a slot is rewritten only after every kernel that
 *     used it has completed (stream events), so concurrent calls on different
 *     streams with different operators are safe.
 *   - Return 0 on success, a positive cudaError_t on a CUDA error, or a
 *     negative H3_ERR_* code for invalid arguments.  No C++ exception crosses
 *     the ABI.
 *   - Cells [z_begin, z_end) along x3 are processed.  With periodic_z != 0
 *     node planes wrap modulo M3 (single-GPU field).  With periodic_z == 0 the
 *     planes -1 and M3 are read from memory directly before / after the field
 *     (ghost planes filled by the slab halo exchange).
 *   - d_first_bad (may be NULL) receives atomicMin of the linear node index
 *     (m3*M2 + m2)*M1 + m1 of every destination node holding a non-finite
 *     value; initialise it to H3_NO_BAD_NODE.  d_guard (may be NULL): when it
 *     holds anything other than H3_NO_BAD_NODE the call does no work (the
 *     reference never runs a half step after an unstable one).
 */
#ifndef H3B200_H
#define H3B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define H3_NO_BAD_NODE 0xFFFFFFFFFFFFFFFFull

/* kernel variants */
#define H3_VARIANT_AUTO 0      /* separable when q >= 3(2N+1) (exact), else literal   */
#define H3_VARIANT_LITERAL 1   /* bit-identical to the reference (no FMA, same order)  */
#define H3_VARIANT_SEPARABLE 2 /* node-factorised exact evolution, HBM-bound fast path */

/* negative status codes */
#define H3_ERR_ARG -1     /* null pointer, bad size, bad offset or slab range   */
#define H3_ERR_ORDER -2   /* order_n outside [0, h3_max_order()]                */
#define H3_ERR_STAGES -3  /* q < 1, literal with q > h3_max_stages(), or separable with q < 3(2N+1) */
#define H3_ERR_VARIANT -4 /* variant not available for this precision/kernel    */

/* Replaces gridkernels.fused_pass(src, dst, h_mat, fac1, fac2, fac3, cfac, tiles, off)
 * (reference gridkernels.py:121-139; called from pipeline.py:251).  `tiles` has
 * no device analogue (results never depend on tiling, pipeline.py:11-14). */
int h3_fused_pass(const double* src, double* dst, int64_t M1, int64_t M2, int64_t M3,
                  int order_n, const double* h_mat, const double* fac1, const double* fac2,
                  const double* fac3, const double* cfac, int q, int off, int64_t z_begin,
                  int64_t z_end, int periodic_z, int variant, void* stream,
                  unsigned long long* d_first_bad, const unsigned long long* d_guard);

/* precision="single" (field.py:30): literal variant only. */
int h3_fused_pass_f32(const float* src, float* dst, int64_t M1, int64_t M2, int64_t M3,
                      int order_n, const float* h_mat, const float* fac1, const float* fac2,
                      const float* fac3, const float* cfac, int q, int off, int64_t z_begin,
                      int64_t z_end, int periodic_z, int variant, void* stream,
                      unsigned long long* d_first_bad, const unsigned long long* d_guard);

/* Fused half step of an x3 slab [z_begin, z_end) of an M3-plane field whose ghost planes -1 and M3
 * are NOT stored next to it: ghost_lo / ghost_hi point at those planes wherever they live -- in
 * the multi-GPU solver, the neighbour rank's boundary plane mapped through CUDA IPC, read in
 * place over NVLink by the kernel's TMA plane loads (no separate halo copy).  Separable variant,
 * N = 3 and 5 (H3_ERR_VARIANT otherwise).  Synchronising the neighbours (the plane must be final
 * before it is read and not rewritten while it is read) is the caller's job.  Same per-cell
 * contract as fused_pass (reference gridkernels.py:121-139, gather offsets :42-55); the reference
 * has no multi-process path, this is the slab form SURVEY 8(b)/(e) asks for
 * ("h3_fused_half_step_dist or a separate halo call"). */
int h3_fused_pass_halo(const double* src, double* dst, int64_t M1, int64_t M2, int64_t M3,
                       int order_n, const double* h_mat, const double* fac1, const double* fac2,
                       const double* fac3, const double* cfac, int q, int off, int64_t z_begin,
                       int64_t z_end, const double* ghost_lo, const double* ghost_hi, int variant,
                       void* stream, unsigned long long* d_first_bad,
                       const unsigned long long* d_guard);

/* CUDA IPC helpers for the halo mapping: export the 64-byte handle of the allocation containing
 * `ptr` and ptr's byte offset in it; open / close a peer allocation. */
int h3_ipc_export(const void* ptr, unsigned char* handle64, int64_t* offset);
int h3_ipc_open(const unsigned char* handle64, void** base_out);
int h3_ipc_close(void* base);

/* Replaces gridkernels.recon_pass(src, coeff, h_mat, tiles, off) (gridkernels.py:142-160;
 * pipeline.py:262).  coeff holds only the cells [z_begin, z_end) (slab chunk):
 * coeff[(c3 - z_begin)][c2][c1][s][s][s].  variant LITERAL = reference summation
 * order without FMA (bit-identical); SEPARABLE/AUTO = the same tensor computed
 * node-factorised (FP64 tensor cores at N = 3, 5; constant-operand DFMA otherwise). */
int h3_recon_pass(const double* src, double* coeff, int64_t M1, int64_t M2, int64_t M3,
                  int order_n, const double* h_mat, int off, int64_t z_begin, int64_t z_end,
                  int periodic_z, int variant, void* stream, const unsigned long long* d_guard);
int h3_recon_pass_f32(const float* src, float* coeff, int64_t M1, int64_t M2, int64_t M3,
                      int order_n, const float* h_mat, int off, int64_t z_begin, int64_t z_end,
                      int periodic_z, int variant, void* stream, const unsigned long long* d_guard);

/* Replaces gridkernels.evolve_pass(coeff, dst, fac1, fac2, fac3, cfac, tiles)
 * (gridkernels.py:163-182; pipeline.py:265).  coeff is chunk-relative as above;
 * dst nodes of cells [z_begin, z_end) are written. */
int h3_evolve_pass(const double* coeff, double* dst, int64_t M1, int64_t M2, int64_t M3,
                   int order_n, const double* fac1, const double* fac2, const double* fac3,
                   const double* cfac, int q, int64_t z_begin, int64_t z_end, int variant,
                   void* stream, unsigned long long* d_first_bad, const unsigned long long* d_guard);
int h3_evolve_pass_f32(const float* coeff, float* dst, int64_t M1, int64_t M2, int64_t M3,
                       int order_n, const float* fac1, const float* fac2, const float* fac3,
                       const float* cfac, int q, int64_t z_begin, int64_t z_end, int variant,
                       void* stream, unsigned long long* d_first_bad,
                       const unsigned long long* d_guard);

/* Host helper: the separable operators the fast path uses, derived from the
 * reference's own arguments (delta = cfac[0], 1/h_k = fac_k[0]) in extended
 * precision and rounded once.  A_out: [3][n][2n] (A_k = S_k[0:n,:] H),
 * S_out: [3][n][2n] (S_k[m][j] = C(j,m) (delta/h_k)^(j-m)).  Either may be NULL. */
int h3_separable_operators(int order_n, const double* h_mat, const double* fac1,
                           const double* fac2, const double* fac3, const double* cfac, int q,
                           double* A_out, double* S_out);

/* Device initial data (reference problems.py:150-175): dst[m3][m2][m1][j3][j2][j1] =
 * sum_t t3[t][m3][j3] * t2[t][m2][j2] * t1[t][m1][j1]; t_k are DEVICE tables
 * [nterms][M_k][n] of per-axis scaled derivatives (problems.py:47-54). */
int h3_init_separable(double* dst, int64_t M1, int64_t M2, int64_t M3, int order_n, int nterms,
                      const double* t1, const double* t2, const double* t3, void* stream);

/* Device error norms (reference problems.py:202-213): d_out[0] = max |u - exact|,
 * d_out[1] = sum (u - exact)^2 over node values, exact = sum_t e3[t][m3] e2[t][m2] e1[t][m1]
 * (DEVICE tables [nterms][M_k]).  d_partials: scratch of 2*n_partials doubles. */
int h3_error_norms(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                   int nterms, const double* e1, const double* e2, const double* e3,
                   double* d_partials, int64_t n_partials, double* d_out, void* stream);

/* Standalone finiteness scan (reference pipeline.py:210-215). */
int h3_check_finite(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                    unsigned long long* d_first_bad, void* stream);

/* ---- per-cell API (reference kernels.py:73-191, the numpy per-cell API) -------------------
 * A batch of `batch` cells, each an (n3, n2, n1) tensor stored contiguously [n3][n2][n1];
 * every pointer is DEVICE memory of the precision `single` selects (1: float, 0: double).
 * The arithmetic is the reference's numpy arithmetic (separate multiplies and adds, same
 * order, same typed zeros), so results are bit-identical to it.  fac_k: per-axis factors
 * (i+1)*(1/h_k) rounded to the precision, length n_k (last entry unused), as
 * kernels.py:90-96 forms them. */

/* One sweep of reconstruct_cell (kernels.py:80-86) = operators.apply_along_axis(H, u, axis)
 * (operators.py:127-151): out = sum_k mat[i][k] x[k] along `axis` (1 = x1 = last index),
 * accumulated from zero in ascending k; mat is [len][len] of that axis. */
int h3_cell_apply_axis(const void* in, void* out, int64_t batch, int n3, int n2, int n1,
                       const void* mat, int axis, int single, void* stream);

/* advect_time_derivative (kernels.py:99-108). */
int h3_cell_advect(const void* w, void* out, int64_t batch, int n3, int n2, int n1,
                   const void* fac1, const void* fac2, const void* fac3, int single, void* stream);

/* taylor_evolve_horner (kernels.py:111-128): q stages, cstage[k-1] = step / k in the
 * precision; `tmp` is scratch of the same size as `out`. */
int h3_cell_horner(const void* b, void* out, void* tmp, int64_t batch, int n3, int n2, int n1,
                   const void* fac1, const void* fac2, const void* fac3, const void* cstage,
                   int q, int single, void* stream);

/* space_time_tensor (kernels.py:131-142): st[cell][j][...], j = 0..q, cstage[j] = dt/(j+1). */
int h3_cell_space_time(const void* b, void* st, int64_t batch, int n3, int n2, int n1,
                       const void* fac1, const void* fac2, const void* fac3, const void* cstage,
                       int q, int single, void* stream);

/* The sum of taylor_evolve_recursion (kernels.py:157-164): out = st[0] + st[1] t_1 + ...,
 * accumulated in ascending j; tpow[j-1] = tau^j (repeated products, rounded once). */
int h3_cell_time_sum(const void* st, void* out, int64_t batch, int64_t size, const void* tpow,
                     int q, int single, void* stream);

/* verify_space_time_identity (kernels.py:167-191): *d_worst (a double's bits, atomically
 * max-reduced; initialise to 0) = max over j, entries of |coef[j] st[j+1] - L st[j]|
 * (j < q) and |L st[q]|, coef[j] = (j+1)/dt in the precision. */
int h3_cell_identity_residual(const void* st, int64_t batch, int n3, int n2, int n1,
                              const void* fac1, const void* fac2, const void* fac3,
                              const void* coef, int q, unsigned long long* d_worst, int single,
                              void* stream);

const char* h3_version(void);
const char* h3_error_string(int status);
int h3_max_order(void);
int h3_max_stages(void);

#ifdef __cplusplus
}
#endif
#endif /* H3B200_H */
