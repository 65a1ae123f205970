// Device-side common definitions for the RSRS sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#define RSRS_DI __device__ __forceinline__

namespace rsrs {

typedef long long i64;

// FP64 tensor-core MMA (DMMA) m8n8k4, row.col: one A element per lane
// (row = lane>>2, col = lane&3), one B element per lane (k = lane&3,
// n = lane>>2), two accumulators per lane (row = lane>>2, cols 2*(lane&3)+{0,1}).
RSRS_DI void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// 16-byte async copy global -> shared with zero fill beyond src_bytes (0, 8 or 16).
RSRS_DI void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
RSRS_DI void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
RSRS_DI void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Scalar arithmetic shared by the real (double) and complex128 (double2 =
// {re, im}) instantiations of the per-box kernels.
RSRS_DI double s_zero(double) { return 0.0; }
RSRS_DI double2 s_zero(double2) { return make_double2(0.0, 0.0); }
RSRS_DI double s_one(double) { return 1.0; }
RSRS_DI double2 s_one(double2) { return make_double2(1.0, 0.0); }
RSRS_DI double s_add(double a, double b) { return a + b; }
RSRS_DI double2 s_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
RSRS_DI double s_sub(double a, double b) { return a - b; }
RSRS_DI double2 s_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
RSRS_DI double s_neg(double a) { return -a; }
RSRS_DI double2 s_neg(double2 a) { return make_double2(-a.x, -a.y); }
RSRS_DI double s_mul(double a, double b) { return a * b; }
RSRS_DI double2 s_mul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
RSRS_DI double s_conj(double a) { return a; }
RSRS_DI double2 s_conj(double2 a) { return make_double2(a.x, -a.y); }
// a * conj(b)
RSRS_DI double s_mulc(double a, double b) { return a * b; }
RSRS_DI double2 s_mulc(double2 a, double2 b) { return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }
RSRS_DI double s_scale(double a, double t) { return a * t; }
RSRS_DI double2 s_scale(double2 a, double t) { return make_double2(a.x * t, a.y * t); }
RSRS_DI double s_real(double a) { return a; }
RSRS_DI double s_real(double2 a) { return a.x; }
RSRS_DI double s_abs(double a) { return fabs(a); }
RSRS_DI double s_abs(double2 a) { return hypot(a.x, a.y); }
RSRS_DI double s_div(double a, double b) { return a / b; }
RSRS_DI double2 s_div(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  const double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}
template <bool C> struct ScalarOf { typedef double T; };
template <> struct ScalarOf<true> { typedef double2 T; };

// Per-box record of one (level, colour) batch.  Static fields are written by
// the host planner; r, self_pos (near-list build) and k, nr, nc, status (ID)
// by the device.
struct BoxDev {
  int nb;                     // |I_b| (active rows of the box, static)
  int rmax;                   // upper bound of |near| (every row of the neighbours)
  int ldr, ldn;               // even leading dims >= rmax, >= nb
  int row0;                   // first store row of b (its rows are contiguous)
  int level, box;             // for error messages
  int nnbr;                   // neighbour boxes (self included)
  i64 off_nbr;                // ints in the level's record array: nnbr x {boxdev index or -1, row0, count, box}
  i64 off_aug;                // doubles: Omega side [C (rmax x ldr); u (nb x ldr)], Psi side follows
  i64 off_yz;                 // doubles: [Y'' Z''] (nb x 2 nld)
  i64 off_h;                  // doubles: H (nb x ldn)
  i64 off_xy, off_xz;         // doubles: X_Y, X_Z (nb x ldr each)
  i64 off_xrc, off_xcr;       // doubles: X_rc (nb x ldr), X_cr (rmax x ldn)
  i64 off_linv;               // doubles: inverse diagonal blocks of the two Cholesky factors
  i64 off_rows;               // ints: near rows (capacity rmax) then b rows (nb)
  i64 off_skelrow, off_redrow, off_crow, off_cpos;  // ints: nb, nb, rmax, rmax
  i64 f_T, f_GL, f_GU, f_Xrr, f_Xinv;  // doubles in the level factor pool (lds ldn / ldr)
  i64 f_red, f_skel, f_c;              // ints (tree positions) in the level index pool
  int r, self_pos;                     // dynamic: |near| and position of b inside near
  int k, nr, nc, status;               // dynamic: ID results
  int ncp;                             // dynamic: leading entries of c outside unprocessed neighbours
  int kpull;                           // dynamic: inner dimension of the pulled L/U update (sum of n_r)
  i64 off_nflag;                       // ints: per near position, 1 = row of an unprocessed neighbour
  i64 off_prow;                        // ints: store rows of the pulled Y_r / Z_r (capacity rmax)
  i64 off_pull;                        // scalars: pulled update operands A_Y, A_Z (nb x ldr each)
  i64 off_est;                         // scalars: coupling estimator, Omega^_r and Psi^_r (nb x nld each)
  double est_y, est_z;                 // dynamic: estimates of |A~(r, f)|_F and |A~(f, r)|_F
};

// status codes in BoxDev::status (0 = ok)
enum { ST_OK = 0, ST_SAMPLES = 1, ST_SINGULAR_GRAM = 2, ST_SINGULAR_XRR = 3, ST_TOO_BIG = 4 };

// C = alpha * A_rows B_rows^T (m x n), K columns; rows gathered by index lists.
// Tiles entirely above the diagonal of the leading sym_rows x sym_rows block
// are skipped (symmetric Gram; only the lower triangle is consumed).
struct NTDesc {
  const double* A;
  const int* rowA;  // nullptr: contiguous rows
  i64 lda;
  const double* B;
  const int* rowB;
  i64 ldb;
  double* C;
  i64 ldc;
  int m, n, K, sym_rows;
  double alpha, beta;
  const int* pm;  // optional device size overrides
  const int* pn;
  const int* psym;
};

// D[rowD(i), j] = beta * Cin[rowC(i), j] + alpha * sum_k opA(i, k) B[rowB(k), j]
// opA(i, k) = transA ? A[k*lda + i] : A[i*lda + k]
struct NNDesc {
  const double* A;
  i64 lda;
  int transA, pad;
  const double* B;
  const int* rowB;
  i64 ldb;
  double* D;
  const int* rowD;
  i64 ldd;
  const double* Cin;  // nullptr: Cin = D (in place, rowC = rowD)
  const int* rowC;
  i64 ldc;
  int m, n, K, pad2;
  double alpha, beta;
  const int* pm;  // optional device size overrides
  const int* pn;
  const int* pK;
};

// augmented Cholesky of [C; B]: C = rows [0, r) (r = *pr), B = rows
// [uoff, uoff + mextra); see dense.cuh
struct CholDesc {
  double* A;
  i64 lda;
  const int* pr;
  int mextra, uoff;
  int* status;
  double* linv;  // workspace: one 64 x 64 inverse diagonal block per panel
};

}  // namespace rsrs
