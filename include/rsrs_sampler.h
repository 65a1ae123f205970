/*
 * rsrs_sampler.h -- HARNESS operator for the RSRS benchmarks and tests (not
 * part of the factorization path): an on-the-fly GPU kernel matvec
 *     Y = A X,   A_ij = delta_ij + weight * k(|x_i - x_j|)   (i != j), A_ii = 1
 * (PAPER.md:119-126 eq. kernel_eval; the black box of PAPER.md:53-61), used to
 * draw Y = A Omega and Z = A^* Psi and to form residuals.  Timed separately
 * from rsrs_factor (BASELINE.json north_star).
 *
 *   kind    0: 2D log kernel  k(r) = log r        (configs c1, c2)
 *           1: 3D Laplace     k(r) = 1 / r        (configs c3, c5; weight = 1/N)
 *   pts     DEVICE, N x 3 row-major doubles (2D points with z = 0), in the same
 *           row order as X and Y (normally tree order)
 *   X, Y    DEVICE, N x ldx / N x ldy row-major doubles; ncol columns used
 *   adjoint 1 computes A^* X (identical for the symmetric real kernels)
 *   stream  cudaStream_t (NULL = legacy default stream); asynchronous
 * Returns 0 on success, 1 invalid argument, 4 CUDA error (message in
 * rsrs_sampler_last_error()).
 */
#ifndef RSRS_SAMPLER_H_
#define RSRS_SAMPLER_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

int rsrs_sample_matvec(int kind, const double* pts, int64_t N, double weight, const void* X, int64_t ldx,
                       void* Y, int64_t ldy, int64_t ncol, int adjoint, void* stream);

/* Complex 2D Helmholtz operator (config c4):
 *     A_ij = delta_ij + weight * (i/4) H0^(1)(kappa |x_i - x_j|)   (i != j), A_ii = 1
 * (complex symmetric: A^* = conj(A)).  X, Y are DEVICE complex128 arrays
 * (interleaved {re, im} doubles), N x ldx / N x ldy complex elements, ncol
 * columns used; adjoint 1 computes A^* X.  Same return codes. */
int rsrs_sample_matvec_c128(const double* pts, int64_t N, double weight, double kappa, const void* X,
                            int64_t ldx, void* Y, int64_t ldy, int64_t ncol, int adjoint, void* stream);
/* Rows [row0, row0 + nrows) of Y = A X (or A^* X) for any kind (0 log2d, 1
 * lap3d real; 2 helm2d complex128 with kappa): Y holds nrows rows (ldy), X all N
 * rows.  Used by each rank of a multi-GPU run to draw its own sample rows. */
int rsrs_sample_matvec_rows(int kind, const double* pts, int64_t N, int64_t row0, int64_t nrows, double weight,
                            double kappa, const void* X, int64_t ldx, void* Y, int64_t ldy, int64_t ncol,
                            int adjoint, void* stream);
const char* rsrs_sampler_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
