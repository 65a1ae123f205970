/*
 * rsrs.h -- C ABI of the B200-native RSRS (randomized strong recursive
 * skeletonization) hot path, arXiv 2311.01451 (Yesypenko & Martinsson).
 *
 * The library builds an invertible factorization K ~= A of an N x N
 * rank-structured operator A that is known only through the samples
 *     Y = A Omega,   Z = A^* Psi,   Omega, Psi ~ N(0, I)  (N x p)
 * (PAPER.md:53-61, 128-131 eq. rand_sample_setting; 1180-1183 section 5),
 * then applies K^-1 (solve) or K (apply).  All compute runs in the library's
 * own sm_100a CUDA kernels; there is no CPU fallback: without a CUDA device
 * every compute entry point returns RSRS_ERR_CUDA.
 *
 * Conventions shared by all entry points
 *   - Every call returns rsrs_status; a human-readable message for the last
 *     failure on the calling thread is returned by rsrs_last_error().
 *     No C++ exception crosses this boundary.
 *   - Handles (rsrs_tree, rsrs_factorization) are created by the library and freed
 *     with the matching *_destroy; a factor keeps a reference to nothing the
 *     caller owns (it copies what it needs from the tree).
 *   - Real data (RSRS_F64) are IEEE doubles; complex data (RSRS_C128) are
 *     interleaved {re, im} double pairs.  Matrices are ROW-MAJOR: element
 *     (i, j) of an n x m matrix with leading dimension ld is at [i*ld + j]
 *     (complex: at element index, i.e. byte offset 16*(i*ld + j)).
 *   - "tree order": rows permuted so that each box's points are contiguous;
 *     row t of a tree-ordered array holds original point perm[t]
 *     (rsrs_tree_perm).
 */
#ifndef RSRS_H_
#define RSRS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RSRS_OK = 0,
  RSRS_ERR_INVALID = 1,   /* bad argument (null pointer, size, dtype, ld < p, ...) */
  RSRS_ERR_SAMPLES = 2,   /* too few samples: p - r < k + l for some box (message names level/box/deficit) */
  RSRS_ERR_SINGULAR = 3,  /* X_rr, the near-field Gram or the top block is numerically singular */
  RSRS_ERR_CUDA = 4,      /* CUDA runtime failure or no device */
  RSRS_ERR_NCCL = 5,      /* reserved for the multi-GPU path */
  RSRS_ERR_NOMEM = 6,     /* device or host allocation failed */
  RSRS_ERR_STATE = 7      /* call not valid in the handle's state (e.g. unsupported nranks) */
} rsrs_status;

typedef enum { RSRS_F64 = 0, RSRS_C128 = 1 } rsrs_dtype;

typedef struct rsrs_tree_s* rsrs_tree;
typedef struct rsrs_factor_s* rsrs_factorization;

/* Options of rsrs_factor. */
typedef struct {
  double eps;          /* user tolerance epsilon ("atol at the leaf level") */
  double level_growth; /* g: atol(l) = id_scale * eps * g^(L - l) ("successively relaxed") */
  double id_scale;     /* c_id (default 1.0) */
  int oversample;      /* l: require p - r >= k + l (default 10) */
  int top_level;       /* last compressed level ("typically on level 2") */
  int rank;            /* this process's rank (0 .. nranks-1) */
  int nranks;          /* number of ranks (one process per GPU); 1 = single GPU */
  void* nccl_comm;     /* ncclComm_t from rsrs_comm_init when nranks > 1, else NULL */
  void* stream;        /* cudaStream_t the factorization runs on (NULL = legacy default stream) */
  int profile;         /* 1: time every kernel class with CUDA events on `stream` (rsrs_factor_profile) */
  int gather_level;    /* multi-GPU: boxes on levels <= gather_level are gathered on rank 0 (-1: auto,
                          the largest level with <= 16 * nranks boxes; always >= top_level - 1) */
  int symmetric;       /* symmetric shortcuts (not in the paper, which always draws two
                          independent sketches).  Only the Y / Omega side of the sweep
                          runs; Z and Psi are ignored (may be NULL).
                          RSRS_F64, symmetric = 1 (or 2): A real symmetric, Psi = Omega hence Z = Y;
                            H = 2 Y''Y''^T, X_rr symmetrised so that G_L = G_U^T.
                          RSRS_C128, symmetric = 2: A complex symmetric (A = A^T, e.g. the Helmholtz
                            operator of config c4), Psi = conj(Omega) hence Z = A^* Psi = conj(Y); every
                            Z-side quantity is the conjugate of its Y-side one: H = 2 Re(Y''Y''^*) (so T
                            is real), X_cr = X_Y^T, X_rr := (X_rr + X_rr^T)/2 so that G_L = G_U^T.
                          RSRS_C128 with symmetric = 1 (Hermitian) is rejected (RSRS_ERR_INVALID). */
  int direct_gram;     /* 1: compute every near-field Gram directly (r x r x p per box) instead of
                          assembling it from the level-wide box-pair blocks (single rank) */
  int push_updates;    /* 1: apply every L/U sample update when its box is eliminated (push, as the
                          multi-GPU ranks do) instead of pulling the updates of a box's rows when the
                          box comes up (single rank) */
  int estimate_coupling; /* 1: after each box's elimination, estimate |A~(r, f)|_F and |A~(f, r)|_F by
                          block nullification of its redundant sample rows (PAPER.md:1232-1235,
                          SURVEY 8(f) f1); read them with rsrs_factor_coupling */
  double noise_factor; /* theta > 0: noise-aware tolerance (reading R17) instead of
                          the fixed schedule: the estimator runs on every box, nu(l) = median over the boxes
                          eliminated on level l of max(est_Y, est_Z) / sqrt(|r_b|), and
                          atol(L) = id_scale * eps, atol(l-1) = max(atol(l), theta * nu(l)); level_growth is
                          ignored.  0 (default): atol(l) = id_scale * eps * level_growth^(L-l).
                          Single rank only (RSRS_ERR_INVALID with nranks > 1). */
  int triangular;      /* 1: triangular output form of the Remark PAPER.md:577-611 for a
                          real symmetric positive definite A (needs RSRS_F64 and opts.symmetric):
                          X_rr (symmetrised) = C C^T by Cholesky, stored C, C^-1 and M_U = C^-1 X_rc
                          instead of X_rr, G_L, G_U; K = V_1..V_n A~ W_n..W_1 with V = E [C 0; M_U^T I],
                          W = [C^T M_U; 0 I] F and identity blocks in the middle.  RSRS_ERR_SINGULAR if
                          some X_rr is not positive definite. */
} rsrs_opts;

/* Statistics of a factorization (Table 1). */
typedef struct {
  int64_t N, p;
  int L, top_level, nlevels_compressed;
  int64_t nsteps;            /* boxes eliminated (steps with |I_r| > 0) */
  int64_t top_size;          /* |S| */
  int64_t max_rank;          /* max k over boxes */
  int64_t memory_scalars;    /* M: stored scalars of T, G_L, G_U, X_rr, A_SS */
  double factor_ms;          /* device time of the last rsrs_factor (CUDA events) */
  double flops_model;        /* flops of THIS BUILD's formulation (CholeskyQR nullification, level-wide
                                Gram blocks, Gram-pivoted ID, explicit X_rr^-1),
                                real-equivalent, from the recorded (n_b, r, k) of every box; the
                                per-class split is rsrs_factor_profile */
  double bytes_model;        /* algorithmic HBM bytes of the sweep (same formulation) */
  int64_t launches;          /* kernels launched by the last rsrs_factor */
  int64_t solve_launches;    /* kernels one rsrs_solve / rsrs_apply call launches */
  double flops_survey;       /* flops of the method by SURVEY 8(d)'s standard dense forms (Householder QR
                                of the near field, projection, truncated CPQR, extraction, LU, sample
                                updates), real-equivalent, same (n_b, r, k) */
} rsrs_stats;

/* ---------------------------------------------------------------------------
 * rsrs_build_tree -- uniform 2^d-tree (section 4.1; neighbours
 * = boxes sharing an edge or corner, Fig. 1 caption PAPER.md:182-184).
 *   pts       host, N x d row-major doubles (d in 1..3); not retained.
 *   leaf_max  m: depth L = smallest L with max leaf occupancy <= m.
 *   root_lo   host, d doubles, lower corner of the root cube (NULL: bounding cube).
 *   root_side side of the root cube (ignored when root_lo == NULL).
 *   nranks    number of Morton ranges to plan (1 in this build).
 *   out       receives the handle.
 * Errors: RSRS_ERR_INVALID (N < 1, d out of range, leaf_max < 1, depth > 20).
 * Host-only integer work; safe without a GPU.
 * ------------------------------------------------------------------------- */
rsrs_status rsrs_build_tree(const double* pts, int64_t N, int d, int leaf_max,
                            const double* root_lo, double root_side, int nranks,
                            rsrs_tree* out);

/* Depth L, dimension d and N of a tree. Any out pointer may be NULL. */
rsrs_status rsrs_tree_info(rsrs_tree t, int* L, int* d, int64_t* N);

/* perm[t] = original index of the point at tree position t (host, N int64). */
rsrs_status rsrs_tree_perm(rsrs_tree t, int64_t* perm);

/* Sizes of level `level` (0..L): number of nonempty boxes and total
 * neighbour-list length. */
rsrs_status rsrs_tree_level_size(rsrs_tree t, int level, int64_t* nboxes, int64_t* nnbr);

/* Level arrays (host buffers sized from rsrs_tree_level_size; any may be NULL):
 *   keys[nboxes]      Morton keys, ascending (bit b of coordinate i -> bit b*d+i)
 *   start[nboxes+1]   tree-position ranges of the boxes' points
 *   parent[nboxes]    index of the parent box on level-1 (-1 on level 0)
 *   colour[nboxes]    sum_i (c_i mod 3) 3^i  (boxes of one colour are >= 3 apart)
 *   nbr_off[nboxes+1], nbr[nnbr]  neighbour CSR (self included, Morton order) */
rsrs_status rsrs_tree_level(rsrs_tree t, int level, uint64_t* keys, int64_t* start,
                            int32_t* parent, int32_t* colour, int32_t* nbr_off, int32_t* nbr);

/* Leaf-level sample-count bound max_b(r_b) + kmax_guess + oversample rounded up
 * to a multiple of 32 ("p = (3m + k)", generalised; coarse levels
 * are checked during the factorization). */
rsrs_status rsrs_plan_samples(rsrs_tree t, int kmax_guess, int oversample, int64_t* p_min);

void rsrs_tree_destroy(rsrs_tree t);

/* ---------------------------------------------------------------------------
 * rsrs_factor -- the level-by-level compress-and-eliminate sweep
 * (section 5; per box: nullification 1195-1200,
 * ID 613-666, extraction 1213-1218, elimination 934-955, sample updates
 * 1205-1212 / 1219-1227 in the consistency-forced orientation, R1).
 *   t                tree (only read; may be destroyed after the call returns)
 *   dt               RSRS_F64 or RSRS_C128
 *   p                number of samples (columns used of each array)
 *   Y, Z, Omega, Psi DEVICE pointers, N x ld row-major, TREE order.  BORROWED
 *                    AND OVERWRITTEN: the sweep updates them in place; their
 *                    contents are unspecified on return.
 *                    Or (single rank, pulled L/U updates) PINNED HOST pointers,
 *                    all four (cudaHostAlloc / cudaHostRegister; pageable memory is
 *                    RSRS_ERR_INVALID): the library allocates the device store,
 *                    copies Omega / Psi on `stream` and streams the Y / Z rows of
 *                    each leaf colour batch on a copy stream one batch ahead of the
 *                    sweep (zero-copy reads), so the transfer overlaps the compute;
 *                    host inputs are only read.
 *   ld               leading dimension (>= p, even)
 *   opts             options (NULL: defaults eps=1e-6, g=1, c_id=1, l=10, top_level=2)
 *   out              receives the factorization handle
 * Synchronous: returns after the device work completes so that device-side
 * errors can be reported.  Errors: RSRS_ERR_INVALID, RSRS_ERR_SAMPLES,
 * RSRS_ERR_SINGULAR, RSRS_ERR_CUDA, RSRS_ERR_NOMEM, RSRS_ERR_STATE.
 * ------------------------------------------------------------------------- */
rsrs_status rsrs_factor(rsrs_tree t, rsrs_dtype dt, int64_t p, void* Y, void* Z,
                        void* Omega, void* Psi, int64_t ld, const rsrs_opts* opts,
                        rsrs_factorization* out);

/* ---------------------------------------------------------------------------
 * rsrs_solve -- B <- K^-1 B, K = V_1..V_n A~_diag W_n..W_1 (PAPER.md:1130-1143,
 * 958-960; elim inverse = sign toggle 572-575).
 *   B     DEVICE (or pinned HOST: staged through a device buffer on stream s),
 *         N x ldb row-major in ORIGINAL point order, nrhs columns used
 *         (ldb >= nrhs); overwritten with the solution.
 *   s     cudaStream_t (NULL = legacy default stream); stream-ordered, asynchronous.
 * Errors: RSRS_ERR_INVALID (bad arguments), RSRS_ERR_CUDA.
 * rsrs_apply -- X <- K X with the same layout.
 * ------------------------------------------------------------------------- */
rsrs_status rsrs_solve(rsrs_factorization f, void* B, int64_t ldb, int64_t nrhs, void* s);
rsrs_status rsrs_apply(rsrs_factorization f, void* X, int64_t ldx, int64_t nrhs, void* s);

/* Kernel classes of the sweep, for rsrs_factor_profile. */
#define RSRS_NUM_KERNEL_CLASSES 12

/* Per-kernel-class record of the last rsrs_factor: class name, summed device
 * time (ms; only when opts.profile == 1, else 0), algorithmic FLOPs and HBM
 * bytes of all its launches and the launch count.
 * cls in [0, RSRS_NUM_KERNEL_CLASSES). */
rsrs_status rsrs_factor_profile(rsrs_factorization f, int cls, const char** name, double* ms,
                                double* flops, double* bytes, int64_t* launches);

/* Statistics of the factorization (host struct). */
rsrs_status rsrs_factor_stats(rsrs_factorization f, rsrs_stats* st);

/* Per-box ranks of a level (host, int32 per box of that level in Morton order):
 * k = skeleton count, or -1 for an empty box; cap = capacity of k[]. */
rsrs_status rsrs_factor_ranks(rsrs_factorization f, int level, int32_t* k, int64_t cap);

/* Coupling estimates of a level (opts.estimate_coupling): est[2 b] ~ |A~(r_b, f)|_F,
 * est[2 b + 1] ~ |A~(f, r_b)|_F after box b's elimination ("estimate the
 * extent to which A~_{r,f} and A~_{f,r} deviate from desired compression tolerance", f = all
 * indices but r_b), -1 for boxes with nothing eliminated; cap >= 2 * nboxes.
 * RSRS_ERR_STATE if the factorization ran without the estimator. */
rsrs_status rsrs_factor_coupling(rsrs_factorization f, int level, double* est, int64_t cap);

/* ID tolerance atol(level) the factorization used on a compressed level (0 otherwise):
 * the fixed schedule or the noise-aware one (rsrs_opts.noise_factor). */
rsrs_status rsrs_factor_atol(rsrs_factorization f, int level, double* atol);

/* Final skeleton set S (tree positions, host int64, ascending) and its size. */
rsrs_status rsrs_factor_top(rsrs_factorization f, int64_t* S, int64_t cap, int64_t* size);

void rsrs_factor_destroy(rsrs_factorization f);

/* ---------------------------------------------------------------------------
 * Multi-GPU (BASELINE.json north_star): one process per GPU.
 * Leaves are split into nranks Morton-contiguous ranges of about equal work
 * (rsrs_tree_partition); rank q owns the boxes whose first point lies in its
 * range, and boxes on levels <= gather_level belong to rank 0 (the coarse
 * levels and the top block A~_SS run there).  Per (level, colour) the sweep
 * fetches the active Y, Z, Omega, Psi rows of foreign neighbour boxes, updates
 * the foreign Y/Z rows in place and returns them (one writer per row: boxes of
 * one colour have disjoint near sets, R10); skeleton rows move to the
 * owner of their parent between levels.  Transport: NCCL point-to-point and
 * all-reduce on the communicator passed in rsrs_opts.nccl_comm.
 *
 * With nranks > 1, rsrs_factor takes THIS RANK's rows: Y, Z, Omega, Psi hold
 * tree positions [first[rank], first[rank+1]) (N_loc x ld).  rsrs_solve /
 * rsrs_apply take the FULL right-hand side, replicated on every rank, and leave
 * the full result on every rank (touched rows merged by an all-reduce after each
 * colour batch).  Every rank must make the same calls.
 * ------------------------------------------------------------------------- */

/* Partition of the leaves for nranks ranks: first[nranks + 1] tree positions
 * (host int64), and the gather level actually used (gather_level < 0: auto). */
rsrs_status rsrs_tree_partition(rsrs_tree t, int nranks, int gather_level, int top_level, int64_t* first,
                                int* gather_out);

/* Owner rank of every box of `level` (host int32[nboxes]). */
rsrs_status rsrs_dist_owner(rsrs_tree t, int nranks, int gather_level, int top_level, int level, int32_t* owner);

/* Host views of the exchange plans (what rsrs_factor executes), for tests and
 * tooling.  Records of 4 int32 {kind (0 send, 1 recv), peer, box, rows}, in the
 * order the rows travel; cap = record capacity of out, *len = records needed.
 *   halo plan of (level, colour) on `rank`: nb[box] = active rows of every box of
 *     the level, cnt[box] = rows a neighbour sees (skeletons once processed);
 *   move plan of `level` -> level-1 on `rank`: k[box] = skeleton count. */
rsrs_status rsrs_dist_halo_plan(rsrs_tree t, int nranks, int gather_level, int top_level, int level, int colour,
                                const int32_t* nb, const int32_t* cnt, int rank, int32_t* out, int64_t cap,
                                int64_t* len);
rsrs_status rsrs_dist_move_plan(rsrs_tree t, int nranks, int gather_level, int top_level, int level,
                                const int32_t* k, int rank, int32_t* out, int64_t cap, int64_t* len);

/* NCCL communicator: rank 0 calls rsrs_comm_unique_id (128 bytes, host), the
 * caller broadcasts it (e.g. over torch.distributed), every rank calls
 * rsrs_comm_init.  NCCL is loaded at run time (libnccl.so.2); RSRS_ERR_NCCL if absent. */
rsrs_status rsrs_comm_unique_id(void* id128);
rsrs_status rsrs_comm_init(int nranks, int rank, const void* id128, void** comm);
void rsrs_comm_destroy(void* comm);
/* Transport self-test (all ranks call it): all-reduces and a ring exchange. */
rsrs_status rsrs_comm_selftest(void* comm, int nranks, int rank);

/* Single-GPU emulation of a G-rank run (validation of the multi-GPU path on one
 * device): G host threads, one per rank, each with its own stream, exchanging
 * through device-to-device copies; no kernel waits on another.  Y, Z, Omega, Psi
 * are the FULL tree-ordered arrays (N x ld; overwritten); out receives G handles
 * (rank order).  rsrs_solve_emulated / rsrs_apply_emulated run the distributed
 * sweep over the G handles on the full B (original order, overwritten). */
rsrs_status rsrs_factor_emulated(rsrs_tree t, rsrs_dtype dt, int64_t p, int G, void* Y, void* Z, void* Omega,
                                 void* Psi, int64_t ld, const rsrs_opts* opts, rsrs_factorization* out);
rsrs_status rsrs_solve_emulated(rsrs_factorization* fs, int G, void* B, int64_t ldb, int64_t nrhs);
rsrs_status rsrs_apply_emulated(rsrs_factorization* fs, int G, void* X, int64_t ldx, int64_t nrhs);

/* Device memory of the library: rsrs_factor draws its workspace and the factor
 * storage from a process-wide arena of cudaMalloc'ed chunks that is kept between
 * calls (growing a stream-ordered pool on every call cost 0.1-3 s on B200).
 * rsrs_memory_info reports the bytes reserved from the driver and in use
 * (either pointer may be NULL); rsrs_release_memory synchronises the device and
 * returns every idle chunk to the driver. */
rsrs_status rsrs_memory_info(int64_t* reserved, int64_t* in_use);
void rsrs_release_memory(void);

/* Message of the last failed call on this thread ("" if none). */
const char* rsrs_last_error(void);

/* Library version string. */
const char* rsrs_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RSRS_H_ */
