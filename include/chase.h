/*
 * chase.h -- C-ABI of the B200-native ChASE hot path (arXiv 2309.15595):
 * the 2D-distributed Chebyshev polynomial filter and the condition-driven CholeskyQR family.
 *
 * Citations: P:NNN = /root/reference/PAPER.md line, S:NNN = SPEC.md line; "Alg.k l.m" = line m
 * of Algorithm k as printed.  Readings of silent/garbled passages are numbered #1..#33 in
 * DESIGN.md ("Readings").
 *
 * Conventions shared by every entry point
 *  - Matrices are column-major (BLAS convention).  Element type is double (CHASE_R64) or
 *    interleaved complex double {re, im} (CHASE_C128, = cuDoubleComplex = torch.complex128).
 *  - Device pointers are CUDA device memory owned by the caller (PyTorch allocates it).
 *    Host pointers are read or written only during the call.
 *  - All device work is enqueued on the handle's CUDA stream; calls return after enqueue
 *    unless stated otherwise.
 *  - The handle is not thread-safe; one handle per process/GPU.
 *  - Collective calls (chase_filter, chase_cholqr) must be made by every rank of the grid with
 *    identical scalar arguments (SPMD); otherwise the result is undefined or a hang.  With
 *    CHASE_SPMD_CHECK=1 in the environment (or a -DCHASE_DEBUG build) they first compare a hash
 *    of those arguments over the world communicator and return CHASE_EINVAL on every rank when
 *    they differ (two tiny AllReduces and one stream synchronisation per call).
 *  - Argument errors are reported synchronously, before any device work, and leave all
 *    buffers untouched.
 */
#ifndef CHASE_H_
#define CHASE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CHASE_OK = 0,
  CHASE_EINVAL = 1,   /* bad size / leading dimension / pointer / non-finite scalar          */
  CHASE_EDEGREE = 2,  /* a degree odd, < 2, or degrees not non-decreasing      */
  CHASE_EBOUNDS = 3,  /* e <= 0, or mu_1 inside the damped interval ((mu_1-c)/e > -1)         */
  CHASE_ECHOL = 4,    /* Cholesky failed even on the shifted path; *info = pivot      */
  CHASE_ECUDA = 5,    /* CUDA runtime / driver failure                                        */
  CHASE_ENCCL = 6,    /* NCCL failure                                                         */
  CHASE_ENOMEM = 7,   /* workspace missing or too small                                       */
  CHASE_ESTATE = 8,   /* call sequence error (e.g. no workspace set)                          */
  CHASE_ENOCONV = 9   /* chase_solve: not converged within max_iter (partial results)          */
} chase_status_t;

typedef enum { CHASE_R64 = 1, CHASE_C128 = 2 } chase_dtype_t;

/* QR variants of Alg.4.  CHOL1 = CholeskyQR (cholDegree 1), CHOL2 = CholeskyQR2,
 * SHIFTED = one shifted pass (POTRF(G + sI)) followed by CholeskyQR2 (reading #13),
 * HOUSEHOLDER = the HHQR fallback of Alg.4 l.9 / the HHQR mode of P:448. */
typedef enum {
  CHASE_QR_CHOL1 = 1,
  CHASE_QR_CHOL2 = 2,
  CHASE_QR_SHIFTED = 3,
  CHASE_QR_HOUSEHOLDER = 4
} chase_qr_variant_t;

/* Spectral bounds of Alg.1 l.2: mu_1 ~ lambda_min, mu_ne ~ lambda_{nev+nex},
 * b_sup >= lambda_max.  The filter uses mu_1 for the scaling point (reading #2); c and e are
 * passed separately and are authoritative. */
typedef struct {
  double mu_1, mu_ne, b_sup;
} chase_bounds_t;

/* Per-call statistics.  matvecs = sum_j d_j; steps = max degree D; qr_variant = the
 * Alg.4 branch actually executed; qr_passes = Gram/POTRF/TRSM rounds executed;
 * shift = the s = 11(mn + n(n+1)) u ||X||_F^2 of Alg.4 l.6 added to the Gram diagonal by
 * the shifted pass (0 when no shifted pass ran), as computed on the device (norm = Re tr G,
 * reading #12). */
typedef struct {
  int64_t matvecs;
  int32_t steps;
  int32_t qr_variant;
  int32_t qr_passes;
  int32_t reserved;
  double shift;
} chase_stats_t;

/* Bookkeeping record of one filter step s (1-based in the paper, index s-1 here):
 * k = #{j : d_j >= s} active columns, off = ncols - k first active column,
 * comm = 0 for an odd step (H^H-side: result in B-layout, AllReduce over the column
 * communicator) and 1 for an even step (result in C-layout, AllReduce over the row
 * communicator), elems = complex/real elements in this rank's AllReduce message
 * (n_c*k for odd, n_r*k for even); the AllReduce is skipped when that communicator has a
 * single member (p == 1 for odd steps, q == 1 for even steps).
 * use_beta = 1 when this rank adds beta_s * V_{s-2} before the AllReduce (the first rank of
 * the reducing communicator, never at s = 1; reading #7); [band_lo, band_hi) = local output
 * rows to which this rank applies the -c I shift (its share of the diagonal; reading #6). */
typedef struct {
  int32_t k;
  int32_t off;
  int32_t comm;
  int32_t use_beta;
  int64_t elems;
  int32_t band_lo;
  int32_t band_hi;
} chase_step_record_t;

typedef struct chase_handle_s* chase_handle_t;

/* ---------------------------------------------------------------------------------------
 * Setup (Alg.2 "Require": 2D grid with rcomm/ccomm; one GPU per rank).
 * ------------------------------------------------------------------------------------- */

/* Rank 0 calls this and distributes the 128 opaque bytes to every rank (the Python layer uses
 * torch.distributed.broadcast).  Wraps ncclGetUniqueId.  Errors: CHASE_EINVAL (null id),
 * CHASE_ENCCL. */
chase_status_t chase_get_unique_id(uint8_t id[128]);

/* Create a handle for rank (myrow, mycol) of a p x q grid holding block (myrow, mycol) of the
 * N x N Hermitian/symmetric matrix under the block distribution of P:113 with the remainder
 * rule of S:102 (the first N mod p grid rows get one extra row; same for columns).
 * n_max = the largest number of vector columns later passed (nev+nex).
 * id = the unique id from chase_get_unique_id (ignored, may be NULL, when p*q == 1).
 * device = CUDA ordinal; cuda_stream = cudaStream_t to enqueue on (NULL = legacy default).
 * World rank = myrow*q + mycol; the row communicator (rcomm) joins the q ranks of grid row
 * myrow, the column communicator (ccomm) the p ranks of grid column mycol.
 * Errors: CHASE_EINVAL (N < 1, n_max < 1 or > N, bad grid coordinates), CHASE_ECUDA,
 * CHASE_ENCCL, CHASE_ENOMEM. */
chase_status_t chase_create(chase_handle_t* h, chase_dtype_t dt, int64_t N, int64_t n_max, int p,
                            int q, int myrow, int mycol, const uint8_t id[128], int device,
                            void* cuda_stream);

/* Block-cyclic distribution ("either a block distribution or a block-cyclic
 * distribution"; C is distributed over each column communicator with the same block
 * size): grid row k owns the global rows g with (g / nb) mod p == k, in increasing order, and
 * likewise grid column k the global columns with (g / nb) mod q == k.  A_local holds
 * A[rows, cols] of those index sets, V the rows of the same row set.  The -cI shift is applied
 * through per-row maps of the diagonal (the band of chase_step_record_t is reported as
 * [-1, -1)).  nb == 0 is the block distribution of chase_create.  Errors as chase_create, plus
 * CHASE_EINVAL when nb < 0 or a grid row/column would own no block (N < nb * max(p, q)). */
chase_status_t chase_create_cyclic(chase_handle_t* h, chase_dtype_t dt, int64_t N, int64_t n_max,
                                   int p, int q, int myrow, int mycol, int64_t nb,
                                   const uint8_t id[128], int device, void* cuda_stream);

/* Virtual grid (tests and diagnostics): a handle for rank (myrow, mycol) of a
 * p x q grid -- block (nb == 0) or block-cyclic -- whose ranks ALL live in this process on the
 * same device, so the 2D distribution (bands of -cI, beta roles, C/B-layout alternation of P:149)
 * and the fused multi-member reduction protocol run on one GPU.  No NCCL communicator is created:
 * every filter step whose communicator has more than one member must run through the fused
 * peer-memory path (chase_set_fused_workspace with peer_bases[r] = the region of virtual rank r,
 * all on this device, and chase_set_fused_mode with an SM budget so the persistent kernels of
 * all ranks are co-resident); each rank's chase_filter must be issued from its own host thread
 * on its own stream (the call waits for its peers).  chase_filter without a fused workspace and
 * every other collective call (chase_cholqr / chase_hhqr with p > 1, chase_residuals,
 * chase_rayleigh_ritz, chase_solve) return CHASE_ESTATE on a virtual grid with p*q > 1.
 * Errors as chase_create_cyclic. */
chase_status_t chase_create_virtual(chase_handle_t* h, chase_dtype_t dt, int64_t N, int64_t n_max,
                                    int p, int q, int myrow, int mycol, int64_t nb, int device,
                                    void* cuda_stream);

/* Global indices of this rank's local rows (n_r entries) and columns (n_c entries), host
 * arrays; either may be NULL.  For the block distribution these are r0.. and c0.. */
chase_status_t chase_local_indices(chase_handle_t h, int64_t* rows, int64_t* cols);

/* Pure host function: the global indices grid row/column k of P owns under block-cyclic
 * distribution with block nb (idx may be NULL to query *count only). */
chase_status_t chase_cyclic_indices(int64_t N, int P, int k, int64_t nb, int64_t* idx,
                                    int64_t* count);

/* Change the stream later calls enqueue on. */
chase_status_t chase_set_stream(chase_handle_t h, void* cuda_stream);

/* Local block geometry of this rank: A_local is n_r x n_c, rows r0.., columns c0.. of A
 * (r0 = c0 = -1 under the block-cyclic distribution; see chase_local_indices). */
chase_status_t chase_local_dims(chase_handle_t h, int64_t* n_r, int64_t* n_c, int64_t* r0,
                                int64_t* c0);

/* Pure host function: the same geometry for any (N, p, q, i, j) without a handle. */
chase_status_t chase_block_dims(int64_t N, int p, int q, int i, int j, int64_t* n_r,
                                int64_t* n_c, int64_t* r0, int64_t* c0);

/* Bytes of device workspace the handle needs: the B-layout block n_c x n_max, the
 * n_max x n_max Gram matrix (Alg.3 l.3), an n_r x n_max TRSM output block, the inverted
 * 64 x 64 diagonal blocks of R, and small scalars -- the same order as the memory model
 * Eq.(2), P:216-223 (N^2/(pq) is the caller's A_local). */
chase_status_t chase_workspace_size(chase_handle_t h, size_t* bytes);

/* Hand the handle `bytes` of caller-owned device memory (>= chase_workspace_size, 256-byte
 * aligned).  The memory must stay valid until chase_destroy or the next set_workspace.
 * Errors: CHASE_EINVAL (null / misaligned), CHASE_ENOMEM (too small). */
chase_status_t chase_set_workspace(chase_handle_t h, void* dptr, size_t bytes);

/* ---------------------------------------------------------------------------------------
 * Fused compute+collective filter steps (complex or real double, p*q > 1).  With a symmetric
 * peer-mapped region set, every filter step whose communicator has more than one member runs as
 * ONE persistent kernel (zgemm_fused.cuh / dgemm_fused.cuh): the tensor-core HEMM publishes each partial output tile into its own
 * region, the tile's owner (tile mod m) sums the m partial tiles in fixed member order over
 * NVLink and stores the result into every member's region (P:149's AllReduce, done tile by tile
 * inside the GEMM, deterministic and replica-identical).  When the step's tiles leave the
 * persistent grid's last round partly idle, its last tiles run instead as split-K copies whose
 * partials every member pushes to every member and sums locally in the same fixed order
 * (fused_tail.cuh; same bits on every member).  Without it, steps call ncclAllReduce.
 *
 * chase_fused_workspace_size: bytes of the symmetric region (identical on every rank).
 * chase_set_fused_workspace: local = this rank's region (device, 256-byte aligned, >= size);
 *   peer_bases[r] = the address at which world rank r's region is mapped in this process
 *   (peer_bases[my world rank] == local); world = p*q.  Zeroes the region's control words; the
 *   caller must barrier all ranks after every rank returned and before the next chase_filter.
 *   local == NULL switches back to NCCL.  Errors: CHASE_EINVAL (bad pointers,
 *   p or q > 8), CHASE_ECUDA.  A peer that never arrives makes chase_filter return CHASE_ECUDA
 *   after a bounded wait (~10 s) instead of hanging. */
chase_status_t chase_fused_workspace_size(chase_handle_t h, size_t* bytes);
chase_status_t chase_set_fused_workspace(chase_handle_t h, void* local, const uint64_t* peer_bases,
                                         int world);

/* Options of the fused path (host only).  mode 0 (default): the fused kernel runs for the steps
 * whose communicator has more than one member; mode 1: every filter step runs it, single-member
 * communicators (and 1 x 1 grids, world = 1, peer_bases[0] = local) included -- the protocol
 * with itself, so the fused kernels can be exercised and measured on one GPU.
 * sm_budget > 0 caps the persistent grid of a fused launch at that many CTAs (one per SM; e.g.
 * #SMs / (p q) on a virtual grid); 0 = all SMs.  Errors: CHASE_EINVAL. */
chase_status_t chase_set_fused_mode(chase_handle_t h, int32_t mode, int32_t sm_budget);

/* ---------------------------------------------------------------------------------------
 * Chebyshev filter -- Eq.(1), Alg.1 l.4, Alg.2 l.12, with the
 * damped scalars of S:362 (reading #1):
 *   sigma_1 = e/(mu_1 - c);  V_1 = (sigma_1/e)(A - cI)V_0;
 *   sigma_s = 1/(2/sigma_1 - sigma_{s-1});
 *   V_s = 2(sigma_s/e)(A - cI)V_{s-1} - sigma_{s-1} sigma_s V_{s-2}   (s = 2..D)
 * Column j of V is replaced by V_{d_j}[:, j] = p_{d_j}(A) v_j with
 * p_d(lambda) = T_d((lambda - c)/e) / T_d((mu_1 - c)/e).
 * Odd steps compute A^H C into the B-layout workspace and all-reduce over ccomm; even steps
 * compute A B back into V (C-layout) and all-reduce over rcomm, so no redistribution is
 * needed and even degrees leave the result in V.  The -cI shift is applied by the
 * rank whose block contains the diagonal rows (reading #6); the beta term is added by the
 * first rank of the reducing communicator (reading #7).  A_local is never modified.
 *
 *  A_local  device, const: A[r0:r0+n_r, c0:c0+n_c], leading dimension lda >= n_r.
 *  V        device, in/out: rows [r0, r0+n_r) of the N x ncols block (C-layout), ldv >= n_r.
 *           Must be identical on all q ranks of a grid row on input; it is identical
 *           on output.  lda and ldv times the element size must be multiples of 16 bytes
 *           (TMA row pitch; i.e. even for CHASE_R64), pointers 16-byte aligned.
 *  ncols    1..n_max (Alg.2 filters C[:, locked+1:]).
 *  degrees  host, ncols int32: even, >= 2, non-decreasing (sorted, Alg.1 l.12 P:103).
 *  c, e     centre and half-width of the damped interval [mu_ne, b_sup] (Alg.2 l.3).
 *  bounds   host: mu_1 sets the scaling point; mu_ne, b_sup informational (reading #2).
 *  stats    host, nullable: matvecs and steps.
 * Errors: CHASE_EINVAL, CHASE_EDEGREE, CHASE_EBOUNDS, CHASE_ESTATE (no workspace; or a fused
 * handle after a peer timeout, until chase_set_fused_workspace is called again on every rank),
 * CHASE_ECUDA, CHASE_ENCCL.  Returns after enqueue -- except with a fused workspace set, where
 * the call copies V into and out of the symmetric region and synchronises the stream once at the
 * end to read the peer-timeout flag (a timeout returns CHASE_ECUDA). */
chase_status_t chase_filter(chase_handle_t h, const void* A_local, int64_t lda, void* V,
                            int64_t ldv, int64_t ncols, const int32_t* degrees, double c,
                            double e, const chase_bounds_t* bounds, chase_stats_t* stats);

/* Diagnostics (tests): this rank's partial of ONE filter step, without the reduction -- the
 * summand that rank (myrow, mycol) contributes to the AllReduce of P:149:
 *   odd != 0: Y (n_c x k) = alpha (A_local^H X - c band(X)) + [use_beta] beta Y,  X n_r x k
 *   odd == 0: Y (n_r x k) = alpha (A_local X - c band(X)) + [use_beta] beta Y,    X n_c x k
 * band(X) = the rows of X on this rank's share of the diagonal (reading #6; block-cyclic: the
 * per-row maps), exactly as chase_filter applies it; the same kernels as chase_filter's local
 * steps.  X and Y device, column-major, must not overlap; ldx/ldy >= their row counts, 16-byte
 * pitch for X.  Works on real and virtual handles.  Errors: CHASE_EINVAL, CHASE_ESTATE,
 * CHASE_ECUDA.  Returns after enqueue. */
chase_status_t chase_filter_step(chase_handle_t h, const void* A_local, int64_t lda, const void* X,
                                 int64_t ldx, void* Y, int64_t ldy, int64_t k, int32_t odd,
                                 double alpha, double beta, double c, int32_t use_beta);

/* The per-step record of the last chase_filter call on this handle (the schedule that was
 * actually launched).  rec: host array of max_steps entries; *nsteps = D. */
chase_status_t chase_filter_record(chase_handle_t h, int32_t max_steps, chase_step_record_t* rec,
                                   int32_t* nsteps, int64_t* matvecs);

/* Pure host function: the schedule chase_filter would run for rank (myrow, mycol). */
chase_status_t chase_filter_schedule(int64_t N, int p, int q, int myrow, int mycol, int64_t ncols,
                                     const int32_t* degrees, int32_t max_steps,
                                     chase_step_record_t* rec, int32_t* nsteps,
                                     int64_t* matvecs);

/* ---------------------------------------------------------------------------------------
 * 1D-CAQR -- Alg.4 over the column communicator, Alg.2 l.14.
 * Variant: cond_est > 1e8 -> shifted CholeskyQR2; cond_est < 20 -> CholeskyQR; else
 * CholeskyQR2 (ties -> CholeskyQR2, reading #9).  Each pass (Alg.3): G = V^H V (local Gram,
 * then AllReduce SUM over ccomm), [shifted pass: norm = ||V||_F^2 = Re tr(G) (reading #12),
 * s = 11(N*ncols + ncols(ncols+1)) u norm, u = 2^-53, G += sI], G = R^H R (POTRF, R upper
 * with positive real diagonal), V = V R^{-1} (TRSM).  If the first POTRF of CholeskyQR or
 * CholeskyQR2 fails (V untouched) the call escalates to the shifted path (reading #14).  If
 * the shifted POTRF fails, the call reverts to Householder QR (Alg.4 l.8-9), and
 * so does any later POTRF failure, on the V of the last successful pass (reading #33); with
 * chase_set_qr_mode(h, 1) every call runs Householder QR (the HHQR mode of P:448).
 *
 *  V        device, in/out: the C-layout block as for chase_filter, ldv >= n_r (16-byte
 *           pitch as for chase_filter).
 *  ncols    1..n_max columns to orthonormalise (all given columns; reading #16).
 *  cond_est >= 1, e.g. from chase_cond_est (Alg.5).
 *  stats    host, nullable: qr_variant (executed branch, CHASE_QR_HOUSEHOLDER when the
 *           fallback ran) and qr_passes (successful Cholesky passes).
 *  info     host, nullable: 0, or the 1-based failing pivot of the last failed POTRF.
 * Synchronises the stream once per POTRF (4-byte info read).
 * Errors: CHASE_EINVAL (bad sizes, cond_est < 1 or NaN), CHASE_ESTATE, CHASE_ECUDA,
 * CHASE_ENCCL.  (CHASE_ECHOL is no longer returned: Householder QR always succeeds.) */
chase_status_t chase_cholqr(chase_handle_t h, void* V, int64_t ldv, int64_t ncols, double cond_est,
                            chase_stats_t* stats, int32_t* info);

/* ---------------------------------------------------------------------------------------
 * Householder QR -- Alg.4 l.9 "X <- ScaLAPACK-HHQR(X, comm)" on the GPU:
 * blocked Householder QR of the C-layout block over the rows of the column communicator
 * (xGEQRF order, 128-wide panels -- the paper's ScaLAPACK run used a 32-column block, P:448,
 * reading #33d; reflectors of
 * LAPACK xLARFG; compact-WY trailing updates on the tensor-core GEMMs; AllReduce over ccomm
 * per column and per panel), then the thin Q (xUNGQR order), written back into V with column
 * j scaled by sign(R_jj) so diag(R) is non-negative (reading #33).  Never fails on rank
 * deficiency (H_j = I for a zero column).  Collective over the grid (identical ncols).
 *  V, ldv, ncols as for chase_cholqr.  Uses the W workspace for Q.
 * Errors: CHASE_EINVAL, CHASE_ESTATE, CHASE_ECUDA, CHASE_ENCCL. */
chase_status_t chase_hhqr(chase_handle_t h, void* V, int64_t ldv, int64_t ncols);

/* QR mode of chase_cholqr (and hence chase_solve): 0 = Alg.4 dispatch (default), 1 = Householder
 * QR in every call (the "ChASE with HHQR" configuration of P:448, Table 3).  Host only.
 * Errors: CHASE_EINVAL (mode not 0/1). */
chase_status_t chase_set_qr_mode(chase_handle_t h, int32_t mode);

/* ---------------------------------------------------------------------------------------
 * The full ChASE iteration -- Alg.2 for the nev lowest eigenpairs:
 * Lanczos bounds (Alg.1 l.2: 4 runs x 25 steps, b_sup = max theta + beta_k, mu_1 = min theta,
 * mu_ne from the Ritz-value density), then repeat {bounds update (l.6-7), degreeOpt (l.9, when
 * opt), Filter (l.12), CondEst (l.13), 1D-CAQR (l.14), C/C2 copies (l.15), Rayleigh-Ritz
 * (l.16-22), residuals (l.23-28), locking (l.29-30)} until nev pairs are locked.  Block
 * distribution only.  Collective; identical arguments on every rank.
 *  V        device, in/out, C-layout n_r x (nev+nex): initial vectors (init_random == 0: the
 *           caller's approximate eigenvectors) or filled with counter-based seeded
 *           Gaussians keyed by global row (init_random != 0); on return the first nev columns
 *           are the eigenvectors (ascending).
 *  tol      residual tolerance on ||H v - lambda v|| / max(|mu_1|, |b_sup|) (1e-10).
 *  deg      initial degree (even: 20), deg_max cap (even: 36); opt: degreeOpt on.
 *  lambda, resid  host out, nev+nex values (first nev: the locked eigenpairs).
 * Returns CHASE_OK when nev pairs converged, CHASE_ENOCONV after max_iter (partial results),
 * or the error of a failing step. */
typedef struct {
  int64_t matvecs;      /* filter + Rayleigh-Ritz + residual + Lanczos single-vector products */
  int32_t iterations;
  int32_t locked;
  int32_t reserved;
  double b_sup, mu_1, mu_ne;   /* Lanczos bounds of the first iteration / last update */
} chase_solve_stats_t;
chase_status_t chase_solve(chase_handle_t h, const void* A_local, int64_t lda, void* V, int64_t ldv,
                           int64_t nev, int64_t nex, double tol, int32_t deg, int32_t deg_max,
                           int32_t max_iter, int32_t opt, uint64_t seed, int32_t init_random,
                           double* lambda, double* resid, chase_solve_stats_t* stats);

/* ---------------------------------------------------------------------------------------
 * Rayleigh-Ritz -- Alg.2 l.16-22 on the orthonormal
 * C-layout block V (ncols columns, e.g. the chase_cholqr output):
 *   B2 <- Bcast(C2, ccomm); B <- H C (odd-step HEMM), AllReduce(ccomm);
 *   A <- B2^H B, AllReduce(rcomm);  Lambda, Y <- HEEVD(A)  (own GPU eigensolver: Householder
 *   tridiagonalisation, Cuppen divide and conquer with Gu-Eisenstat eigenvectors, blocked
 *   back-transformation; redundant and bit-identical on every rank; CHASE_RR_JACOBI=1 selects the
 *   parallel block-Jacobi solver instead);  V <- V Y.
 *  ritz    host out: the ncols Ritz values, ascending (V's columns in the same order).
 *  sweeps  host out, nullable: divide-and-conquer merge levels + 1 (Jacobi: sweeps used,
 *          convergence off(A) <= 1e-14 ||A||_F).
 * Uses the B-layout, Gram and eigensolver workspace.  Synchronises the stream once per merge
 * level (host deflation decisions) or once per Jacobi sweep.
 * Errors: CHASE_EINVAL, CHASE_ESTATE, CHASE_ECUDA, CHASE_ENCCL, CHASE_ENOCONV (the Jacobi
 * solver did not reach its off-norm test within 40 sweeps; the results are written anyway). */
chase_status_t chase_rayleigh_ritz(chase_handle_t h, const void* A_local, int64_t lda, void* V,
                                   int64_t ldv, int64_t ncols, double* ritz, int32_t* sweeps);

/* ---------------------------------------------------------------------------------------
 * Residuals -- Alg.2 l.23-28: resid[j] = ||H v_j - ritz[j] v_j||_2
 * for the ncols columns of V (Ritz vectors, C-layout):
 *   B2 <- Bcast(C, ccomm) (rows [c0, c0+n_c) of V, from the owning rank(s) of the column
 *   communicator), B <- H C with "B - ritzv B2" fused into the HEMM epilogue of the first rank of
 *   the column communicator, AllReduce(SUM, ccomm), squared column norms of the local rows,
 *   AllReduce(SUM, rcomm), sqrt.
 *  A_local, lda  as for chase_filter (read only).
 *  V, ldv        device, read only: C-layout block, ncols columns (1..n_max).
 *  ritz          host, ncols Ritz values (finite).
 *  resid         host out, ncols residual norms (identical on every rank).
 * Uses the B-layout workspace (its content is overwritten).  Synchronises the stream once.
 * Errors: CHASE_EINVAL, CHASE_ESTATE, CHASE_ECUDA, CHASE_ENCCL. */
chase_status_t chase_residuals(chase_handle_t h, const void* A_local, int64_t lda, const void* V,
                               int64_t ldv, int64_t ncols, const double* ritz, double* resid);

/* Alg.5, host, pure: t' = (ritz[0]-c)/e, t = (ritz[locked]-c)/e,
 * |rho| = max(|t - sqrt(t^2-1)|, |t + sqrt(t^2-1)|) (complex sqrt: 1 when |t| <= 1),
 * d = degrees[locked], d_M = max(degrees[locked..n-1]); returns |rho|^d |rho'|^(d_M - d).
 * ritz: host array of n Ritz values (ascending); degrees: host, n entries.
 * Returns NaN on invalid input (n < 1, locked outside [0, n), e <= 0). */
double chase_cond_est(const double* ritz, int64_t n, double c, double e, const int32_t* degrees,
                      int64_t locked);

/* Alg.4 l.6, host, pure: s = 11 (m n + n (n + 1)) u norm, u = 2^-53. */
double chase_shift_value(int64_t m, int64_t n, double norm);

/* ---------------------------------------------------------------------------------------
 * Measurement support (bench.py): when enabled, CUDA events bracket every launch on the
 * handle's stream; chase_profile_read synchronises, returns per-category device time (ms)
 * and kernel-launch counts since the last read, and resets.  Categories (arrays of 8):
 *   0 HEMM odd steps (A^H C -> B)   1 HEMM even steps (A B -> C)   2 AllReduce (NCCL calls)
 *   3 Gram   4 POTRF   5 TRSM   6 other kernels   7 Householder QR (whole call; launches
 *   counted there, its GEMMs included) */
chase_status_t chase_profile_enable(chase_handle_t h, int enable);
chase_status_t chase_profile_read(chase_handle_t h, double ms[8], int64_t launches[8]);

chase_status_t chase_destroy(chase_handle_t h);
const char* chase_status_string(chase_status_t s);

#ifdef __cplusplus
}
#endif
#endif /* CHASE_H_ */
