// Per-box GEMM / Cholesky descriptors of a level, built on the device from the
// box records (one thread per box) -- the host used to build and upload ~2 KB of
// descriptors per box per level (40 MB at the sphere's leaf level), which left
// the GPU idle.  Same contents and order as the launch code expects:
//   Gram   [Omega Gram, Psi Gram]* (omitted with the level's Gram blocks), [Y cross, Z cross]
//   Chol   [Omega side, Psi side]     proj [Y, Z]     H [H_Y, H_Z]
//   E/F    [Y, Z, Omega, Psi]         G [G_U, G_L]    L/U [Y, Z]
// with every Z / Psi entry dropped by the symmetric shortcut.
#pragma once
#include "common.cuh"

namespace rsrs {

struct DescParams {
  double *Y, *Z, *Om, *Ps;       // current store
  i64 ld, nld;
  int p, SC, sym, blocks, nbox, pull;   // pull: L/U updates of not-yet-eliminated rows are pulled
  double* dws;                   // level workspace
  double* fpool;                 // level factor pool
  int* diws;                     // level int workspace
  BoxDev* boxes;
  NTDesc* gram;
  NTDesc* h;
  NNDesc* proj;
  NNDesc* ef;
  NNDesc* g;
  NNDesc* upd;
  NNDesc* pullD;                 // [Y, Z] per box (pull mode)
  CholDesc* chol;
  int tri;                       // triangular form (f4): g[2q] = M_U = C^-1 X_rc, g[2q+1] empty,
  NNDesc* g2;                    //   g2[q] = G_L = M_U^T C^-1 (a second launch: it reads M_U)
};

__global__ void make_desc_kernel(const DescParams P) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= P.nbox) return;
  BoxDev* dx = P.boxes + q;
  const BoxDev x = *dx;
  const int SC = P.SC, p = P.p;
  const int ns = P.sym ? 1 : 2;
  const i64 ld = P.ld, nld = P.nld;
  const int nb = x.nb, rm = x.rmax;
  const i64 ldr = x.ldr, ldn = x.ldn;
  const int* near = P.diws + x.off_rows;
  const int* brows = near + rm;
  double* augO = P.dws + SC * x.off_aug;
  double* augP = augO + SC * (i64)(rm + nb) * ldr;
  // ---- Gram + cross
  {
    NTDesc* o = P.gram + (i64)q * (P.blocks ? 1 : 2) * ns;
    if (!P.blocks) {
      NTDesc a{};
      a.A = P.Om; a.rowA = near; a.lda = ld; a.B = P.Om; a.rowB = near; a.ldb = ld;
      a.C = augO; a.ldc = ldr; a.m = rm; a.n = rm; a.K = p; a.sym_rows = rm; a.alpha = 1.0;
      a.pm = &dx->r; a.pn = &dx->r; a.psym = &dx->r;
      *o++ = a;
      if (!P.sym) {
        a.A = P.Ps; a.B = P.Ps; a.C = augP;
        *o++ = a;
      }
    }
    NTDesc bq{};
    bq.A = P.Y; bq.rowA = brows; bq.lda = ld; bq.B = P.Om; bq.rowB = near; bq.ldb = ld;
    bq.C = augO + SC * (i64)rm * ldr; bq.ldc = ldr; bq.m = nb; bq.n = rm; bq.K = p; bq.sym_rows = 0;
    bq.alpha = 1.0; bq.pn = &dx->r;
    *o++ = bq;
    if (!P.sym) {
      bq.A = P.Z; bq.B = P.Ps; bq.C = augP + SC * (i64)rm * ldr;
      *o++ = bq;
    }
  }
  // ---- Cholesky
  {
    const i64 nlv = (i64)((rm + 63) / 64) * 64 * 64;
    CholDesc* o = P.chol + (i64)q * ns;
    o[0] = CholDesc{augO, ldr, &dx->r, nb, rm, &dx->status, P.dws + SC * x.off_linv};
    if (!P.sym) o[1] = CholDesc{augP, ldr, &dx->r, nb, rm, &dx->status, P.dws + SC * (x.off_linv + nlv)};
  }
  double* yz = P.dws + SC * x.off_yz;
  // ---- projection
  {
    NNDesc* o = P.proj + (i64)q * ns;
    NNDesc pr{};
    pr.A = augO + SC * (i64)rm * ldr; pr.lda = ldr; pr.transA = 0;
    pr.B = P.Om; pr.rowB = near; pr.ldb = ld;
    pr.D = yz; pr.rowD = nullptr; pr.ldd = 2 * nld;
    pr.Cin = P.Y + SC * (i64)x.row0 * ld; pr.rowC = nullptr; pr.ldc = ld;
    pr.m = nb; pr.n = p; pr.K = rm; pr.alpha = -1.0; pr.beta = 1.0; pr.pK = &dx->r;
    o[0] = pr;
    if (!P.sym) {
      pr.A = augP + SC * (i64)rm * ldr; pr.B = P.Ps; pr.D = yz + SC * nld; pr.Cin = P.Z + SC * (i64)x.row0 * ld;
      o[1] = pr;
    }
  }
  // ---- H
  {
    NTDesc* o = P.h + (i64)q * ns;
    NTDesc h{};
    h.A = yz; h.rowA = nullptr; h.lda = 2 * nld; h.B = yz; h.rowB = nullptr; h.ldb = 2 * nld;
    h.C = P.dws + SC * x.off_h; h.ldc = ldn; h.m = nb; h.n = nb; h.K = p; h.sym_rows = 0;
    h.alpha = 1.0;
    o[0] = h;
    if (!P.sym) {
      h.A = yz + SC * nld; h.B = yz + SC * nld; h.C = P.dws + SC * (x.off_h + (i64)nb * ldn);
      o[1] = h;
    }
  }
  const int* skelrow = P.diws + x.off_skelrow;
  const int* redrow = P.diws + x.off_redrow;
  double* Tm = P.fpool + SC * x.f_T;
  // ---- E/F
  {
    NNDesc* o = P.ef + (i64)q * 2 * ns;
    NNDesc e{};
    e.A = Tm; e.lda = ldn; e.transA = 0; e.B = P.Y; e.rowB = skelrow; e.ldb = ld;
    e.D = P.Y; e.rowD = redrow; e.ldd = ld; e.Cin = nullptr;
    e.m = nb; e.n = p; e.K = nb; e.alpha = -1.0; e.beta = 1.0; e.pm = &dx->nr; e.pK = &dx->k;
    *o++ = e;
    if (!P.sym) {
      e.B = P.Z; e.D = P.Z;
      *o++ = e;
    }
    NNDesc fo{};
    fo.A = Tm; fo.lda = ldn; fo.transA = 1; fo.B = P.Om; fo.rowB = redrow; fo.ldb = ld;
    fo.D = P.Om; fo.rowD = skelrow; fo.ldd = ld; fo.Cin = nullptr;
    fo.m = nb; fo.n = p; fo.K = nb; fo.alpha = 1.0; fo.beta = 1.0; fo.pm = &dx->k; fo.pK = &dx->nr;
    *o++ = fo;
    if (!P.sym) {
      fo.B = P.Ps; fo.D = P.Ps;
      *o++ = fo;
    }
  }
  // ---- G_U, G_L
  {
    NNDesc* o = P.g + (i64)q * 2;
    NNDesc gu{};
    gu.A = P.fpool + SC * x.f_Xinv; gu.lda = ldn; gu.B = P.dws + SC * x.off_xrc; gu.rowB = nullptr; gu.ldb = ldr;
    gu.D = P.fpool + SC * x.f_GU; gu.ldd = ldr; gu.Cin = nullptr; gu.m = nb; gu.n = rm; gu.K = nb;
    gu.alpha = 1.0; gu.beta = 0.0; gu.pm = &dx->nr; gu.pn = &dx->nc; gu.pK = &dx->nr;
    o[0] = gu;
    NNDesc gl{};
    gl.A = P.dws + SC * x.off_xcr; gl.lda = ldn; gl.B = P.fpool + SC * x.f_Xinv; gl.rowB = nullptr; gl.ldb = ldn;
    gl.D = P.fpool + SC * x.f_GL; gl.ldd = ldn; gl.Cin = nullptr; gl.m = rm; gl.n = nb; gl.K = nb;
    gl.alpha = 1.0; gl.beta = 0.0; gl.pm = &dx->nc; gl.pn = &dx->nr; gl.pK = &dx->nr;
    if (P.tri) {
      // f_Xinv holds C^-1, so gu computes M_U = C^-1 X_rc (stored in f_GU for the solve);
      // G_L = X_cr X_rr^-1 = M_U^T C^-1 (real symmetric: X_cr = X_rc^T) for the L/U updates
      NNDesc g2{};
      g2.A = P.fpool + SC * x.f_GU; g2.lda = ldr; g2.transA = 1;
      g2.B = P.fpool + SC * x.f_Xinv; g2.rowB = nullptr; g2.ldb = ldn;
      g2.D = P.fpool + SC * x.f_GL; g2.ldd = ldn; g2.Cin = nullptr; g2.m = rm; g2.n = nb; g2.K = nb;
      g2.alpha = 1.0; g2.beta = 0.0; g2.pm = &dx->nc; g2.pn = &dx->nr; g2.pK = &dx->nr;
      P.g2[q] = g2;
      gl = NNDesc{};          // empty (m = 0)
    }
    o[1] = gl;
  }
  // ---- L/U updates
  {
    NNDesc* o = P.upd + (i64)q * ns;
    const int* crow = P.diws + x.off_crow;
    NNDesc u{};
    u.A = P.fpool + SC * x.f_GL; u.lda = ldn; u.transA = 0; u.B = P.Y; u.rowB = redrow; u.ldb = ld;
    u.D = P.Y; u.rowD = crow; u.ldd = ld; u.Cin = nullptr; u.m = rm; u.n = p; u.K = nb;
    u.alpha = -1.0; u.beta = 1.0; u.pm = P.pull ? &dx->ncp : &dx->nc; u.pK = &dx->nr;
    o[0] = u;
    if (!P.sym) {
      NNDesc uz = u;
      uz.A = P.fpool + SC * x.f_GU; uz.lda = ldr; uz.transA = 1; uz.B = P.Z; uz.D = P.Z;
      o[1] = uz;
    }
  }
  // ---- pulled L/U update into the box's own rows (pull_assemble_kernel gathers A and the rows)
  if (P.pull) {
    NNDesc* o = P.pullD + (i64)q * ns;
    double* AY = P.dws + SC * x.off_pull;
    NNDesc v{};
    v.A = AY; v.lda = ldr; v.transA = 0; v.B = P.Y; v.rowB = P.diws + x.off_prow; v.ldb = ld;
    v.D = P.Y + SC * (i64)x.row0 * ld; v.rowD = nullptr; v.ldd = ld; v.Cin = nullptr;
    v.m = nb; v.n = p; v.K = rm; v.alpha = -1.0; v.beta = 1.0; v.pK = &dx->kpull;
    o[0] = v;
    if (!P.sym) {
      v.A = AY + SC * (i64)nb * ldr; v.B = P.Z; v.D = P.Z + SC * (i64)x.row0 * ld;
      o[1] = v;
    }
  }
}

// Coupling estimator: after the box's elimination,
//   Omega^_r = Omega_r + G_U Omega_c,  Psi^_r = Psi_r + G_L^* Psi_c   (the U / L^-* updates of
//   the red rows, skipped by the sweep because eliminated rows are dead)
//   R_Y = Y_r (I - Omega^_r^dagger Omega^_r) = A~(r, f) Omega^_f null(Omega^_r),  same for Z
// through the same Gram / Cholesky / projection kernels as the nullification.
struct EstParams {
  double *Y, *Z, *Om, *Ps;
  i64 ld, nld;
  int p, SC, sym, nbox;
  double* dws;
  double* fpool;
  int* diws;
  BoxDev* boxes;
  NNDesc* form;      // [Omega^, Psi^] per box
  NTDesc* gram;      // [Omega^ Gram, Psi^ Gram, Y_r cross, Z_r cross]
  CholDesc* chol;    // [Omega side, Psi side]
  NNDesc* proj;      // [R_Y, R_Z]
};

__global__ void make_est_desc_kernel(const EstParams P) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= P.nbox) return;
  BoxDev* dx = P.boxes + q;
  const BoxDev x = *dx;
  const int SC = P.SC, p = P.p;
  const int ns = P.sym ? 1 : 2;
  const i64 ld = P.ld, nld = P.nld, ldr = x.ldr, ldn = x.ldn;
  const int nb = x.nb, rm = x.rmax;
  const int* redrow = P.diws + x.off_redrow;
  const int* crow = P.diws + x.off_crow;
  double* est = P.dws + SC * x.off_est;                 // [Omega^_r ; Psi^_r], nb x nld each
  double* augO = P.dws + SC * x.off_aug;
  double* augP = augO + SC * (i64)(rm + nb) * ldr;
  double* yz = P.dws + SC * x.off_yz;                   // [R_Y | R_Z], ld 2 nld
  for (int side = 0; side < ns; ++side) {
    double* eh = est + SC * (i64)side * nb * nld;
    double* aug = side ? augP : augO;
    NNDesc f{};
    f.A = side ? P.fpool + SC * x.f_GL : P.fpool + SC * x.f_GU;
    f.lda = side ? ldn : ldr;
    f.transA = side;                                    // G_L^* for Psi
    f.B = side ? P.Ps : P.Om; f.rowB = crow; f.ldb = ld;
    f.D = eh; f.rowD = nullptr; f.ldd = nld;
    f.Cin = side ? P.Ps : P.Om; f.rowC = redrow; f.ldc = ld;
    f.m = nb; f.n = p; f.K = rm; f.alpha = 1.0; f.beta = 1.0; f.pm = &dx->nr; f.pK = &dx->nc;
    P.form[(i64)q * ns + side] = f;
    NTDesc a{};
    a.A = eh; a.rowA = nullptr; a.lda = nld; a.B = eh; a.rowB = nullptr; a.ldb = nld;
    a.C = aug; a.ldc = ldr; a.m = nb; a.n = nb; a.K = p; a.sym_rows = nb; a.alpha = 1.0;
    a.pm = &dx->nr; a.pn = &dx->nr; a.psym = &dx->nr;
    P.gram[(i64)q * 2 * ns + side] = a;
    NTDesc c{};
    c.A = side ? P.Z : P.Y; c.rowA = redrow; c.lda = ld; c.B = eh; c.rowB = nullptr; c.ldb = nld;
    c.C = aug + SC * (i64)rm * ldr; c.ldc = ldr; c.m = nb; c.n = nb; c.K = p; c.sym_rows = 0; c.alpha = 1.0;
    c.pm = &dx->nr; c.pn = &dx->nr;
    P.gram[(i64)q * 2 * ns + ns + side] = c;
    P.chol[(i64)q * ns + side] =
        CholDesc{aug, ldr, &dx->nr, nb, rm, &dx->status, P.dws + SC * (x.off_linv + side * (i64)((rm + 63) / 64) * 64 * 64)};
    NNDesc pr{};
    pr.A = aug + SC * (i64)rm * ldr; pr.lda = ldr; pr.transA = 0;
    pr.B = eh; pr.rowB = nullptr; pr.ldb = nld;
    pr.D = yz + SC * (i64)side * nld; pr.rowD = nullptr; pr.ldd = 2 * nld;
    pr.Cin = side ? P.Z : P.Y; pr.rowC = redrow; pr.ldc = ld;
    pr.m = nb; pr.n = p; pr.K = nb; pr.alpha = -1.0; pr.beta = 1.0; pr.pm = &dx->nr; pr.pK = &dx->nr;
    P.proj[(i64)q * ns + side] = pr;
  }
}

// est = |R|_F / sqrt(p - n_r) per side (one CTA per box)
template <bool C>
__global__ void __launch_bounds__(256) est_norm_kernel(BoxDev* __restrict__ boxes, const double* __restrict__ wsd,
                                                       i64 nld, int p, int sides) {
  typedef typename ScalarOf<C>::T S;
  BoxDev& b = boxes[blockIdx.x];
  const int nr = b.nr;
  __shared__ double red[2][256];
  const S* R = reinterpret_cast<const S*>(wsd) + b.off_yz;
  for (int side = 0; side < sides; ++side) {
    double acc = 0.0;
    if (b.status == ST_OK)
      for (int idx = threadIdx.x; idx < nr * p; idx += 256) {
        const S v = R[(i64)(idx / p) * 2 * nld + (i64)side * nld + idx % p];
        const double a = s_abs(v);
        acc += a * a;
      }
    red[side][threadIdx.x] = acc;
  }
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int side = 0; side < sides; ++side) red[side][threadIdx.x] += red[side][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double w = (double)(p - nr);
    b.est_y = (nr > 0 && w > 0) ? sqrt(red[0][0] / w) : 0.0;
    b.est_z = sides > 1 ? ((nr > 0 && w > 0) ? sqrt(red[1][0] / w) : 0.0) : b.est_y;
  }
}

}  // namespace rsrs
