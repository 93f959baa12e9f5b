// stages.h — stage drivers of libeigb200 (internal), shared by the
// single-GPU entry points (abi.cu) and the collective ones (comm.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ctx.h"

namespace eig {

// K = #{i = 0, nb, 2nb, ... : i + nb < n} he2hb panels (reading R3)
int64_t num_panels(int64_t n, int nb);
// Q2 reflector slots of the V2 layout (include/eig.h)
int64_t v2_slots(int64_t n, int nb);

// a1..a5: A (lower) -> band + V1 in place, tau[K nb], T[K nb nb]
int he2hb_run(Ctx &c, int64_t n, double2 *A, int64_t lda, double2 *tau, double2 *T);
// a6: E <- Q2 E (grouped blocks)
int apply_q2_run(Ctx &c, int64_t n, const double2 *V2, const double2 *tau2, double2 *E, int64_t lde, int64_t m);
// a7: E <- Q1 E
int apply_q1_run(Ctx &c, int64_t n, const double2 *A, int64_t lda, const double2 *T, double2 *E, int64_t lde,
                 int64_t m);
// a8: E <- L^-H E; hostE (pinned, ld ldh) optional: final row blocks copied back on c.xfer
int trsm_lh_run(Ctx &c, int64_t n, const double2 *L, int64_t ldl, double2 *E, int64_t lde, int64_t m,
                double2 *hostE = nullptr, int64_t ldh = 0);
// Algorithm 1 step 2: A <- L^-1 A L^-H
int hegst_run(Ctx &c, int64_t n, double2 *A, int64_t lda, const double2 *L, int64_t ldl);

// Algorithm 1 step 1 (synchronous: returns the LAPACK info, 0 or n + j)
int potrf_run(Ctx &c, int64_t n, double2 *B, int64_t ldb);
// NEXT-1 bulge chase (offset tables built on the stream)
int hb2st_run(Ctx &c, int64_t n, const double2 *A, int64_t lda, double *d, double *e, double2 *V2, double2 *tau2);
// a6..a8 on m columns: E = L^-H Q1 Q2 complex(Zr) (Zr == nullptr: E already
// holds the columns to transform), recording the BT / Q2 / Q1 / trsm statistics
int bt_run(Ctx &c, int64_t n, const double *Zr, int64_t ldzr, const double2 *V2, const double2 *tau2,
           const double2 *A, int64_t lda, const double2 *T1, const double2 *L, int64_t ldl, double2 *E, int64_t lde,
           int64_t m, double2 *hostE = nullptr, int64_t ldh = 0);

// NEXT-4 (he2hb_dist.cu): the 1D block-cyclic distributed reduction computed by
// P virtual ranks on this GPU (arithmetic check), result in the he2hb layout
int he2hb_sim(Ctx &c, int64_t n, int P, double2 *A, int64_t lda, double2 *tau, double2 *T);
// ... and over NCCL for this rank of the handle's communicator (collective)
int64_t dist_ncols(int64_t n, int rank, int P, int nb);
size_t he2hb_dist_work(int64_t n, int nb, int P, int rank);
int dist_scatter(Ctx &c, int64_t n, const double2 *A, int64_t lda, double2 *Aloc, double2 *pack);
int he2hb_dist_nccl(Ctx &c, int64_t n, double2 *Aloc, double2 *V1, double2 *tau, double2 *T, double2 *work,
                    double2 *A0, int64_t lda0);

// ------------------------------------------------------------- collective (comm.cu)
int comm_unique_id(void *id128);
int comm_init(Ctx &c, const void *id128);   // ncclCommInitRank (collective over the ranks)
int comm_reserve(Ctx &c, int64_t n_max);    // receive buffers for n <= n_max
void comm_destroy(Ctx &c);
int coll_hotpath(Ctx &c, int64_t n, double2 *A, int64_t lda, double2 *tau1, double2 *T1, const double2 *V2,
                 const double2 *tau2, const double2 *L, int64_t ldl, const double *Z, int64_t ldz, double2 *E,
                 int64_t lde, int64_t m, unsigned flags);
int coll_solve_gen(Ctx &c, int64_t n, double2 *A, int64_t lda, double2 *B, int64_t ldb, int64_t il, int64_t iu,
                   double *w, double2 *Z, int64_t ldz);

}  // namespace eig
