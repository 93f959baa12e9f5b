// kernels.h — host-side launchers of the sm_100a kernels (internal to libeigb200).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace eig {

struct Ctx;  // defined in abi.cu

// ------------------------------------------------------------- zgemm engine
enum Op { OP_N = 0, OP_C = 1 };

struct Zgemm {
  int opa = OP_N, opb = OP_N;
  int herm_a = 0;   // A Hermitian, lower stored (opa must be N)
  int lower_c = 0;  // 1: only lower triangle of C (M == N, lower tiles only), imag(diag) = 0
                    // 2: rectangular grid, writes only entries with row0 + gm >= gn, imag(diag) = 0
  int64_t row0 = 0;  // lower modes: matrix row of C row 0
  int64_t M = 0, N = 0, K = 0;
  const double2 *A = nullptr;
  int64_t lda = 0;
  const double2 *B = nullptr;
  int64_t ldb = 0;
  double2 *C = nullptr;
  int64_t ldc = 0;
  double alpha = 1.0, beta = 0.0;
  int splitk = 0;   // 0 = choose automatically, 1 = none, >1 = forced
  // > 0: choose the split-K factor as if N were split_n, so the result does
  // not depend on N (column-sliced calls are bitwise equal to the unsliced one:
  // the back-transform's per-rank column slices)
  int64_t split_n = 0;
  // 3M (Gauss) product: 0 = the handle's setting (EIG_USE_3M), 1 = on, -1 = off
  int m3 = 0;
  // in-place right products (C aliases A): every CTA must cover all N <= 64
  // columns, so the 64-column engine variants are required
  bool whole_n = false;
};

// N used by the back-transform GEMMs for their split-K choice (columns of E
// are the sharded dimension)
constexpr int64_t kBtSplitN = 1024;
// 3M products with K <= kShortK take the short-K engine
// variant (64 x 32 tiles, two CTAs per SM); see zgemm.cu
constexpr int64_t kShortK = 256;
// ... and so do products with N <= kNarrowN (the he2hb hemm W = A22 V, N = nb):
// twice the tiles of the 64-column variant (EIG_ZGEMM_NARROW overrides)
constexpr int64_t kNarrowN = 64;
// 1: plain long-K 3M products take the 128 x 64-tile variant (EIG_ZGEMM_V4 overrides)
constexpr int kZgemmV4 = 1;

// Enqueue C = alpha op(A) op(B) + beta C on ctx's stream.  Returns 0 or error.
int zgemm(Ctx &ctx, const Zgemm &g);

// ------------------------------------------------------------- he2hb pieces
// Panel QR + T factor (cooperative).  Panel P = A[r0:n, c0:c0+nb] (pn rows),
// writes V (explicit, pn x nb, ldv) into vout (and vout2 if non-null),
// tau[nb], T (nb x nb, ld nb).
int panel_qr(Ctx &ctx, double2 *P, int64_t lda, int64_t pn, int nb, double2 *tau, double2 *T, double2 *vout,
             double2 *vout2, int64_t ldv, cudaStream_t stream);

// Copy the reflectors of panel k from the he2hb layout into an explicit
// unit-lower s x nb matrix (ld ldv).
int extract_v(Ctx &ctx, const double2 *P, int64_t lda, int64_t pn, int nb, double2 *V, int64_t ldv);

// Inverse of the diagonal blocks of a lower triangular L: Linv[b] (bs x bs).
int trinv_blocks(Ctx &ctx, int64_t n, int bs, const double2 *L, int64_t ldl, double2 *Linv);

// E = complex(Z)
int complexify(Ctx &ctx, int64_t n, int64_t m, const double *Z, int64_t ldz, double2 *E, int64_t lde);

// Zero the imaginary part of the diagonal of A (n x n).
int real_diag(Ctx &ctx, int64_t n, double2 *A, int64_t lda);

// Device bulge chase (NEXT-1): band from he2hb output A -> d, e and V2/tau2.
int hb2st(Ctx &ctx, int64_t n, int nb, const double2 *A, int64_t lda, double *d, double *e, double2 *V2,
          double2 *tau2, const int64_t *d_off);

// ------------------------------------------------------------- real grouped GEMM
struct DgemmProb {
  int64_t M, N, K;
  const double *A;
  int64_t lda;
  const double *B;
  int64_t ldb;
  double *C;
  int64_t ldc;
};
// C_p = A_p B_p for each problem of the device array d_probs; max_tiles =
// max over p of dgemm_tiles(M_p, N_p).
int dgemm_group(Ctx &ctx, const DgemmProb *d_probs, int nprob, int max_tiles);
int dgemm_tiles(int64_t M, int64_t N);

// ------------------------------------------------------------- stedc (NEXT-2)
// Divide and conquer for the real symmetric tridiagonal (d, e): all
// eigenvalues ascending into w[n]; eigenvectors of indices il..iu (1-based)
// into Z (n x (iu-il+1), ldz).  d, e are device arrays (not modified).
int stedc(Ctx &ctx, int64_t n, const double *d, const double *e, int64_t il, int64_t iu, double *w, double *Z,
          int64_t ldz);

// ------------------------------------------------------------- front end (NEXT-3)
int potrf_lower(Ctx &ctx, int64_t n, double2 *B, int64_t ldb, int64_t *d_info);
int herm_full(Ctx &ctx, int64_t n, double2 *A, int64_t lda);
int conj_transpose(Ctx &ctx, int64_t n, const double2 *X, int64_t ldx, double2 *Y, int64_t ldy);

// ------------------------------------------------------------- Q2
struct Q2Plan {
  int64_t n = 0;
  int nb = 0, g = 0;
  int64_t ngroups = 0;
  int64_t nblocks = 0;
  int64_t *d_group_first_block = nullptr;  // [ngroups+1] device
  int64_t *d_off = nullptr;                // [J] device slot offsets per step j
  int64_t J = 0;
};
// Fill the V2 slot offsets off[0..J) and (if first != nullptr) the per-group
// first-block table first[0..ngroups] on ctx's stream.
int plan_tables(Ctx &ctx, int64_t n, int nb, int g, int64_t ngroups, int64_t J, int64_t *first, int64_t *off);
int q2_tfactors(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *tau2, double2 *T2);
int q2_apply(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *T2, double2 *E, int64_t lde, int64_t m);
// column-owning-warp variant (nb = 64, g = 32); returns 1 if the shape is not handled
int q2w_apply(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *T2, double2 *E, int64_t lde, int64_t m);

}  // namespace eig
