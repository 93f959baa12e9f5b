/*
 * include/eig.h — C ABI of the B200-native two-stage Hermitian generalized
 * eigensolver hot path (arXiv 1207.1773, /root/reference/PAPER.md = "P:Lnn").
 *
 * Library: paper_1207_1773_b200/libeigb200.so (CUDA, sm_100a).
 *
 * Conventions (all entry points):
 *   - complex128 = two little-endian binary64 (re, im), interleaved.
 *   - Matrices are column-major with a leading dimension ld >= rows.
 *   - Hermitian inputs: only the lower triangle is read; imag(diag) ignored.
 *   - Pointers are CUDA device pointers unless the entry point says "host".
 *     The caller owns every pointer it passes; the library owns its workspace
 *     (allocated on first use, grown on demand, freed by eig_finalize).
 *   - Work is enqueued on the handle's stream (eig_config.stream, or the
 *     legacy default stream if NULL).  Entry points are asynchronous unless
 *     they say "synchronous"; errors detected on the host are returned
 *     immediately, launch errors are returned as EIG_ERR_CUDA.
 *   - Return codes (LAPACK info style, reading R11):
 *       0                success
 *       -i               argument i (1-based, counting the handle as 1) illegal
 *       EIG_ERR_CUDA     a CUDA call failed (eig_last_cuda_error() has it)
 *       EIG_ERR_NOMEM    device allocation failed
 *       EIG_ERR_STATE    bad handle / not initialised
 *       EIG_ERR_NOTIMPL  entry point not available in this build
 *       EIG_ERR_NCCL     an NCCL call failed (collective handles)
 *   - One handle per host thread; many handles may coexist (kernel attributes
 *     are set per handle, i.e. per device).
 *   - Multi-GPU ("data on the GPUs is distributed", the
 *     back-transform's column independence S:L469): one process per GPU.  Rank
 *     0 calls eig_get_unique_id, ships the 128 bytes to the other ranks (e.g.
 *     torch.distributed), and every rank calls eig_init with
 *     {rank, nranks, nccl_id}.  eig_solve_gen and eig_hotpath are then
 *     COLLECTIVE (all ranks call them with the same n / range arguments):
 *     rank 0 runs the unsharded stages, the factors go out by NCCL broadcast
 *     (lower triangles only) on a communication stream overlapped with rank
 *     0's later stages, and rank r back-transforms the eigenvector columns
 *     eig_column_slice(m, r, nranks).
 */
#ifndef EIG_B200_H
#define EIG_B200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIG_ERR_CUDA    (-1001)
#define EIG_ERR_NCCL    (-1002)
#define EIG_ERR_NOMEM   (-1003)
#define EIG_ERR_STATE   (-1004)
#define EIG_ERR_NOTIMPL (-1005)

/* eig_solve_gen ranges (reading R12: "fraction" = the lowest ceil(f n)) */
#define EIG_RANGE_ALL      0
#define EIG_RANGE_FRACTION 1
#define EIG_RANGE_INDEX    2

/* eig_config.flags */
#define EIG_GATHER_Z     1u  /* collective eig_solve_gen: rank 0's Z receives all m columns      */
#define EIG_USE_3M       2u  /* complex GEMMs (he2hb updates, Q1, triangular solves, hegst) as
                                three real DMMA products (3M, Gauss) instead of four: 0.75 of
                                the tensor-pipe work; nominal flops stay 8 per complex MAC.
                                (The nb = 64, g = 32 Q2 wavefront is 3M by default
                                independently of these flags; environment EIG_Q2_3M=0
                                selects its four-product form.)                          */
#define EIG_NO_3M        4u  /* force the four-product form (overrides EIG_USE_3M / EIG_3M)   */
#define EIG_DIST_HE2HB   8u  /* collective eig_solve_gen: he2hb distributed over all ranks (1D
                                block-cyclic columns, NEXT-4) instead of on rank 0; every rank
                                then already holds V1 / T1 (no V1 broadcast)                  */

/* eig_hotpath flags */
#define EIG_HOST_BUFFERS 1u  /* pointers are host memory: copy in, run, copy E out (synchronous) */
#define EIG_SKIP_HE2HB   2u  /* back-transform only (A already holds he2hb output + T1)        */
#define EIG_SKIP_BT      4u  /* he2hb only                                                      */

typedef struct eig_ctx *eig_handle;

typedef struct {
  int device;        /* CUDA ordinal for this process                              */
  int nb;            /* band half-width = he2hb panel width; 0 -> 64.  eig_init
                        accepts 1..64 (he2hb, hb2st, Q1, trsm work for all); the
                        grouped Q2 back-transform (eig_apply_q2, eig_hotpath,
                        eig_solve_gen) needs an even nb >= 4 and returns
                        EIG_ERR_NOTIMPL otherwise                                   */
  int q2_group;      /* sweeps per grouped Q2 block (g); 0 -> min(32, 4*floor((nb+1)/4))
                        (0 for nb <= 2: no Q2).  Explicit values must satisfy
                        4 <= g <= 32, g % 4 == 0, g <= nb + 1 (else eig_init
                        returns -2).  nb = 64 with g = 32 selects the wavefront
                        kernel (3M form, blocks released by per-block completion
                        counters); other shapes the generic grouped kernel       */
  void *stream;      /* cudaStream_t to order with; NULL = legacy default stream    */
  int rank, nranks;  /* this process's rank and the number of ranks (GPUs); nranks
                        <= 1 with nccl_id == NULL: single GPU (non-collective)     */
  const void *nccl_id; /* host pointer to the 128-byte id from eig_get_unique_id() on
                        rank 0 (same bytes on every rank); non-NULL makes the
                        handle collective (nranks == 1 allowed: the collective
                        code path on one GPU).  eig_init is then collective too.   */
  int64_t n_max;     /* > 0: largest n this handle will see (calls with n > n_max
                        return EIG_ERR_STATE; collective receive buffers are
                        allocated at init); 0: grow lazily                        */
  unsigned flags;    /* EIG_GATHER_Z | EIG_USE_3M | EIG_NO_3M | EIG_DIST_HE2HB.  Neither 3M flag: the
                        environment EIG_3M=0/1 decides, else 3M is on (default)    */
} eig_config;

/* Per-call statistics (device seconds from CUDA events on this rank's
 * streams; nominal flops, 8 per complex multiply-add). */
enum {
  EIG_ST_POTRF = 0, EIG_ST_HEGST, EIG_ST_HE2HB, EIG_ST_HB2ST, EIG_ST_STEDC,
  EIG_ST_WAIT,     /* BT start minus call start (collective: waiting for rank 0 + factors) */
  EIG_ST_Q2, EIG_ST_Q1, EIG_ST_TRSM,
  EIG_ST_BT,       /* back-transform on this rank: complexify + Q2 + Q1 + L^-H = t_BT   */
  EIG_ST_GATHER,   /* EIG_GATHER_Z column gather                                        */
  EIG_ST_TOTAL,    /* whole call                                                        */
  EIG_NSTAGES
};
struct eig_stats {
  double seconds[EIG_NSTAGES];
  double flops[EIG_NSTAGES];
  int64_t m;                 /* selected eigenvectors (all ranks)                      */
  int64_t col_lo, col_hi;    /* this rank's columns [col_lo, col_hi) of the m          */
  int64_t bytes_comm;        /* NCCL payload bytes this rank sent + received            */
  int rank, nranks;
};

/* 128-byte NCCL unique id into id128 (host memory); call on rank 0 only.
 * Host-only (no device needed).  Returns 0 or EIG_ERR_NCCL. */
int eig_get_unique_id(void *id128);
/* Columns [lo, hi) of m that rank r of nranks owns in the collective calls:
 * lo = floor(r m / nranks), hi = floor((r+1) m / nranks).  Host-only.
 * Returns 0, or -1..-3 for an illegal m / rank / nranks. */
int eig_column_slice(int64_t m, int rank, int nranks, int64_t *lo, int64_t *hi);
/* eig_solve_gen's selection (reading R12) without solving: (range, fraction,
 * il, iu) for order n -> 1-based il..iu and m = iu - il + 1.  Host-only.
 * Returns 0 or -i with eig_solve_gen's argument numbering (2, 7..10). */
int eig_resolve_range(int64_t n, int range, double fraction, int64_t il_in, int64_t iu_in, int64_t *il,
                      int64_t *iu, int64_t *m);

/* Create a handle.  cfg may be NULL (defaults).  Returns 0 or an error;
 * the configuration is validated before any device call (-2: bad nb,
 * q2_group, rank / nranks, or nranks > 1 without nccl_id). */
int eig_init(eig_handle *h, const eig_config *cfg);
/* Destroy a handle and free its workspace (synchronises its stream). */
int eig_finalize(eig_handle h);
/* Static text for a return code. */
const char *eig_strerror(int code);
/* Text of the last CUDA error seen by this handle ("" if none). */
const char *eig_last_cuda_error(eig_handle h);
/* Kernel launches issued by this handle since creation (for bench accounting). */
int64_t eig_launch_count(eig_handle h);
/* Synchronise the handle's stream. */
int eig_sync(eig_handle h);

/* Number of he2hb panels K for order n and width nb (reading R3):
 * K = #{i = 0, nb, 2nb, ... : i + nb < n}. */
int64_t eig_num_panels(int64_t n, int nb);
/* Number of Q2 reflector slots (V2 layout below) for order n, width nb. */
int64_t eig_v2_slots(int64_t n, int nb);

/* ------------------------------------------------------------------ a1..a5
 * Reduction to band form, he2hb (Fig. 1; readings R1, R3, R6).
 *   A   [in/out] n x n complex128, lda >= n.  In: Hermitian, lower triangle.
 *       Out: lower band (0 <= r-c <= nb) = Band = Q1^H A Q1; below the band,
 *       in column k*nb+j, the tail of reflector v_{k,j} whose unit head sits
 *       at row (k+1)*nb+j.  The strict upper triangle is not referenced.
 *   tau [out] K*nb complex128: tau of reflector (k, j) at k*nb+j (0 if absent).
 *   T   [out] K*nb*nb complex128: T_k (nb x nb, column-major, upper
 *       triangular) with H_{k,0}...H_{k,nb-1} = I - V_k T_k V_k^H.
 * Uses nb from the handle's config. */
int eig_he2hb(eig_handle h, int64_t n, void *A, int64_t lda, void *tau, void *T);

/* ------------------------------------------------------------------ NEXT-4
 * The same reduction computed by the 1D block-cyclic DISTRIBUTED algorithm
 * (§6; csrc/he2hb_dist.cu) with `nranks` virtual ranks on this GPU:
 * rank r owns the full columns of the nb-wide blocks b = r mod nranks, the
 * panel runs on its owner, V / T / tau are broadcast, W = A22 V is the sum of
 * the ranks' partial products (allreduce), each rank updates its own columns.
 * The collectives are device copies and a fixed-order sum here; over NCCL in
 * the collective path.  Arguments and output layout as eig_he2hb (A
 * Hermitian, lower read; overwritten with band + V1).  Synchronous.
 * Library-internal scratch: nranks * n * (n / nranks + 6 nb) + n^2 complex128. */
int eig_he2hb_sim(eig_handle h, int64_t n, int nranks, void *A, int64_t lda, void *tau, void *T);

/* ------------------------------------------------------------------ a7
 * E <- Q1 E: E is n x m (lde >= n), A/T as produced by eig_he2hb. */
int eig_apply_q1(eig_handle h, int64_t n, const void *A, int64_t lda, const void *T, void *E, int64_t lde,
                 int64_t m);

/* ------------------------------------------------------------------ a6
 * Q2 reflector (V2) layout (reading R5): slot (j, i) for sweep i = 0..n-2 and
 * step j with i + 1 + j*nb <= n-1 is at index off_j + i,
 * off_j = sum_{j' < j} (n - 1 - j'*nb).  It acts on rows
 * i+1+j*nb .. min(i+(j+1)*nb, n-1); V2[slot*nb + r] = v[r] (v[0] = 1,
 * zero padded to nb), tau2[slot] = tau.  H = I - tau v v^H.
 * Q2 = product over sweeps i ascending, steps j ascending of H_{i,j}.
 *
 * E <- Q2 E:  Z [in] n x m real binary64 (ldz >= n) if Z != NULL, in which
 * case E is first set to complex(Z) (the complexification of a6);
 * E [in/out] n x m complex128 (lde >= n).  V2: slots*nb complex128,
 * tau2: slots complex128. */
int eig_apply_q2(eig_handle h, int64_t n, const void *V2, const void *tau2, const double *Z, int64_t ldz, void *E,
                 int64_t lde, int64_t m);

/* ------------------------------------------------------------------ NEXT-1
 * Band -> real symmetric tridiagonal by column-wise bulge chasing (P:L93,
 * reading R5), on the device.  A: he2hb output (only the lower band
 * 0 <= r-c <= nb is read; not modified).  d[n], e[n-1]: real diagonal and
 * sub-diagonal (e_i = beta of sweep i, LAPACK zlarfg convention, so T is
 * real without a phase diagonal).  V2 [slots*nb], tau2 [slots]: the chase
 * reflectors in the V2 layout below, so that Band = Q2 T Q2^H.  Uses nb of
 * the handle; library workspace holds a (2nb+2) x n band copy.  The chase
 * runs position-stationary (each nb-row position's diagonal and bulge blocks
 * resident in one CTA's shared memory for all sweeps) while ceil(J/2) CTAs,
 * J = (n-2)/nb + 1, fit on the device at once (n <= ~18900 at nb = 64 on a
 * 148-SM B200), else sweep per CTA; same reflectors and outputs either way
 * (up to rounding); environment EIG_HB2ST_SYS=0 forces the latter. */
int eig_hb2st(eig_handle h, int64_t n, const void *A, int64_t lda, double *d, double *e, void *V2, void *tau2);

/* ------------------------------------------------------------------ NEXT-2
 * Real symmetric tridiagonal eigensolver by divide and conquer:
 * d[n] diagonal, e[n-1] sub-diagonal (device, not modified).  w[n] receives
 * all eigenvalues ascending; Z (n x (iu-il+1), ldz >= n, real binary64)
 * the orthonormal eigenvectors of eigenvalues il..iu (1-based); only those
 * are formed at the last merge.  Library workspace ~5 n^2 doubles. */
int eig_stedc(eig_handle h, int64_t n, const double *d, const double *e, int64_t il, int64_t iu, double *w, double *Z,
              int64_t ldz);

/* ------------------------------------------------------------------ a8
 * E <- L^-H E (Algorithm 1 step 4): L n x n lower triangular
 * (non-unit; only the lower triangle read), E n x m. */
int eig_trsm_lh(eig_handle h, int64_t n, const void *L, int64_t ldl, void *E, int64_t lde, int64_t m);

/* ------------------------------------------------------------------ a1..a9
 * One pass of the whole hot path:
 *   he2hb(A) -> E = complex(Z) -> E = Q2 E -> E = Q1 E -> E = L^-H E
 * on the m selected eigenvector columns (a9: the caller passes the m columns
 * of the tridiagonal eigenvectors it wants, il..iu).
 *   A    n x n (lda), Hermitian lower; destroyed (he2hb output).
 * Collective handle: rank 0 passes A, V2, tau2, L (device); the other ranks
 * pass NULL for them (they receive V2, tau2 and the lower triangle of L while
 * rank 0 runs he2hb, then the lower triangle of A (V1) and T1) and tau1/T1
 * may be NULL on every rank; every rank passes ITS OWN column slice Z (n x m,
 * m = its width) and E.  EIG_HOST_BUFFERS is not available collectively
 * (EIG_ERR_NOTIMPL).  Per-stage times: eig_last_stats.
 *   tau1 K*nb, T1 K*nb*nb complex128: he2hb outputs (device).  With
 *        EIG_HOST_BUFFERS they are host pointers and may be NULL (then they
 *        stay in library workspace); if non-NULL they receive tau1 / T1.
 *        With EIG_SKIP_HE2HB, T1 is an INPUT (the T factors of the he2hb
 *        output held in A) and must not be NULL when K > 0 (else -6).
 *   V2, tau2  Q2 reflectors (layout above).
 *   L    n x n lower (ldl).   Z n x m real (ldz).   E n x m complex128 (lde) out.
 * flags: EIG_HOST_BUFFERS -> A, V2, tau2, L, Z, E are HOST pointers (pinned
 * recommended); the call copies the lower triangle of A to the device,
 * copies V2, tau2, Z and the lower triangle of L on a transfer stream while
 * he2hb runs, copies each final 256-row block of E back while the triangular
 * solve works on the blocks above it, and returns synchronously; the host A
 * is not modified in that mode.  EIG_SKIP_HE2HB / EIG_SKIP_BT select a part. */
int eig_hotpath(eig_handle h, int64_t n, void *A, int64_t lda, void *tau1, void *T1, const void *V2,
                const void *tau2, const void *L, int64_t ldl, const double *Z, int64_t ldz, void *E, int64_t lde,
                int64_t m, unsigned flags);

/* Statistics of the last eig_hotpath / eig_solve_gen call on this handle
 * (synchronises the handle's stream).  out: host. */
int eig_last_stats(eig_handle h, struct eig_stats *out);

/* ------------------------------------------------------------------ expert
 * Complex GEMM on the FP64 DMMA tile engine (exposed for parity tests):
 *   C = alpha op(A) op(B) + beta C, op in {'N','C'} (C = conjugate transpose);
 *   herm_a != 0: A is Hermitian with only its lower triangle stored (opa 'N');
 *   lower_c != 0: only the lower triangle of C (M == N) is written, imag(diag)=0.
 * alpha, beta real. */
int eig_zgemm(eig_handle h, char opa, char opb, int64_t M, int64_t N, int64_t K, double alpha, const void *A,
              int64_t lda, const void *B, int64_t ldb, double beta, void *C, int64_t ldc, int herm_a, int lower_c);

/* Debug: cycles spent by CTA 0 of apply_q2 in its phases [0..4] (load, A,
 * B, C, commit) and of panel_qr [8..13] (barrier, reduce, beta, update,
 * partials, tail) and of hb2st [16..21] (wait, reflector, a, b, c, flag),
 * accumulated since eig_init; needs EIG_Q2_PROFILE set in the environment at
 * eig_init (else EIG_ERR_NOTIMPL).  out16: host array of 32. */
int eig_debug_q2_profile(eig_handle h, unsigned long long *out16);

/* ------------------------------------------------------------------ NEXT-3
 * Cholesky B = L L^H (Algorithm 1 step 1), blocked, in place: the
 * lower triangle of B (n x n, ldb) is replaced by L (strict upper not
 * referenced).  Synchronous.  Returns 0, or n + j if the leading minor of
 * order j is not positive definite (LAPACK zhegv INFO convention, R11). */
int eig_potrf(eig_handle h, int64_t n, void *B, int64_t ldb);

/* Standard form A' = L^-1 A L^-H (Algorithm 1 step 2): A (lower
 * read) is overwritten by A' (full Hermitian storage, imag(diag) = 0);
 * L lower from eig_potrf.  Library workspace: n^2 complex128. */
int eig_hegst(eig_handle h, int64_t n, void *A, int64_t lda, const void *L, int64_t ldl);

/* ------------------------------------------------------------------ Algorithm 1
 * Generalized solver A x = lambda B x (Algorithm 1, with the
 * two-stage Algorithm 2, and the D&C tridiagonal solver, §4.3):
 * potrf -> hegst -> he2hb -> hb2st -> stedc (last merge restricted to il..iu)
 * -> Z = L^-H Q1 Q2 Z'.
 *   A   [in/destroyed] n x n (lda), Hermitian, lower read.
 *   B   [in/out] n x n (ldb), HPD, lower read; overwritten by L.
 *   range EIG_RANGE_ALL | EIG_RANGE_FRACTION (0 < fraction <= 1: il = 1,
 *       iu = ceil(fraction n)) | EIG_RANGE_INDEX (1 <= il <= iu <= n).
 *   w   [out, device] n binary64: all eigenvalues ascending.
 *   Z   [out, device] n x m complex128 (ldz >= n), m = iu - il + 1, the
 *       B-orthonormal eigenvectors of eigenvalues il..iu.
 *   m_out [out, host, nullable] m.
 *   stats [out, host, nullable] per-stage seconds and flops of this call.
 * Synchronous.  Returns 0, -i (illegal argument i), n + j (B not PD), or a
 * library error code.
 * Collective handle (all ranks call with the same n, range, fraction, il,
 * iu): rank 0 passes A and B; the others may pass NULL (lda, ldb ignored).
 * Every rank's w receives all n eigenvalues.  Rank r's Z (n x (hi-lo), ldz)
 * receives the columns [lo, hi) = eig_column_slice(m, r, nranks) of the m
 * selected eigenvectors; with EIG_GATHER_Z rank 0's Z is n x m and receives
 * all of them (the other ranks' Z may then be NULL).  Rank 0 runs potrf,
 * hegst, he2hb, hb2st and stedc; L, A's lower part (V1) and T1 are broadcast
 * during hb2st, V2/tau2 during stedc, and the tridiagonal eigenvectors are
 * scattered by column slice; errors on rank 0 are returned on every rank. */
int eig_solve_gen(eig_handle h, int64_t n, void *A, int64_t lda, void *B, int64_t ldb, int range, double fraction,
                  int64_t il, int64_t iu, double *w, void *Z, int64_t ldz, int64_t *m_out, struct eig_stats *stats);

#ifdef __cplusplus
}
#endif
#endif
