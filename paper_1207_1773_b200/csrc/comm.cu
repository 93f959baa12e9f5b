// comm.cu — collective (multi-GPU) entry points of libeigb200 over NCCL.
//
// the back-transform E = L^-H Q1 Q2 Z acts on the eigenvector
// columns independently, so with P GPUs (one process each) rank r
// owns the contiguous columns [floor(r m / P), floor((r+1) m / P)) and the
// only exchange is the distribution of the read-only factors from rank 0,
// which runs the unsharded stages ("the data on the GPUs is
// distributed"; he2hb stays on one GPU, DESIGN.md §8 gives the numbers).
//
// Data movement (all on the handle's communication stream `cstream`, ordered
// against the compute stream with events, so it overlaps rank 0's compute):
//   - Hermitian / triangular factors travel as packed LOWER triangles (half
//     the bytes of the dense matrix): L (from B), and A after he2hb (band +
//     the V1 reflectors below it); T1 is K nb^2, V2/tau2 the bulge-chase
//     reflectors, w the eigenvalues: ncclBroadcast from rank 0.
//   - eig_solve_gen: L / V1 / T1 go out during hb2st, V2 / tau2 during stedc,
//     the tridiagonal eigenvectors are SCATTERED by column slice (grouped
//     ncclSend / ncclRecv; a slice of a column-major n x m matrix is
//     contiguous), and with EIG_GATHER_Z the E slices are gathered to rank 0.
//   - eig_hotpath: V2 / tau2 and L go out while rank 0 runs he2hb, then V1 and
//     T1.
// Every rank then runs the single-GPU back-transform (bt_run) on its slice.
// Errors detected on rank 0 (potrf info, stedc) are broadcast so that every
// rank returns the same code.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"
#include "stages.h"

namespace eig {
namespace {

// packed lower triangle, column-major: column j holds rows j..n-1 at j n - j (j - 1) / 2
__host__ __device__ __forceinline__ int64_t packed_off(int64_t n, int64_t j) { return j * n - j * (j - 1) / 2; }

__global__ void pack_lower_kernel(int64_t n, const double2 *M, int64_t ld, double2 *P) {
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    double2 *dst = P + packed_off(n, j) - j;
    const double2 *src = M + j * ld;
    for (int64_t i = j + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

__global__ void unpack_lower_kernel(int64_t n, const double2 *P, double2 *M, int64_t ld) {
  for (int64_t j = blockIdx.x; j < n; j += gridDim.x) {
    const double2 *src = P + packed_off(n, j) - j;
    double2 *dst = M + j * ld;
    for (int64_t i = j + threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
  }
}

int nccl_check(Ctx &c, ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return 0;
  c.last_err = std::string(what) + ": " + ncclGetErrorString(r);
  return EIG_ERR_NCCL;
}

ncclComm_t comm_of(Ctx &c) { return (ncclComm_t)c.nccl; }

int bcast(Ctx &c, void *buf, size_t bytes, const char *what) {
  if (bytes == 0) return 0;
  c.st.bytes_comm += (int64_t)bytes;
  return nccl_check(c, ncclBroadcast(buf, buf, bytes / sizeof(double), ncclDouble, 0, comm_of(c), c.cstream), what);
}

// Lower triangle of the n x n matrix M (ld) from rank 0 to every rank: rank 0
// packs M into `pk`, broadcasts it, the others unpack into their M.  All on
// the communication stream.
int bcast_lower(Ctx &c, double2 *M, int64_t n, int64_t ld, double2 *pk, const char *what) {
  const int grid = (int)std::min<int64_t>(n, 4LL * c.num_sms);
  if (c.rank == 0) {
    pack_lower_kernel<<<grid, 256, 0, c.cstream>>>(n, M, ld, pk);
    EIG_TRY(c.launched("pack_lower_kernel"));
  }
  EIG_TRY(bcast(c, pk, (size_t)packed_off(n, n) * sizeof(double2), what));
  if (c.rank != 0) {
    unpack_lower_kernel<<<grid, 256, 0, c.cstream>>>(n, pk, M, ld);
    EIG_TRY(c.launched("unpack_lower_kernel"));
  }
  return 0;
}

// `to` waits for everything enqueued on `from` so far
int order(Ctx &c, cudaStream_t from, cudaStream_t to, cudaEvent_t ev, const char *what) {
  EIG_TRY(c.check(cudaEventRecord(ev, from), what));
  return c.check(cudaStreamWaitEvent(to, ev, 0), what);
}

// Broadcast a status word of rank 0 (0 = continue) and return it on every rank
// (synchronous: every rank needs it before enqueueing more work).
int bcast_status(Ctx &c, int64_t status_on_root, int64_t *out) {
  int64_t *d = (int64_t *)c.ws(WS_C_STATUS, 64);
  if (!d) return EIG_ERR_NOMEM;
  static thread_local int64_t h;
  h = status_on_root;
  if (c.rank == 0)
    EIG_TRY(c.check(cudaMemcpyAsync(d, &h, sizeof(int64_t), cudaMemcpyHostToDevice, c.cstream), "status"));
  EIG_TRY(nccl_check(c, ncclBroadcast(d, d, 1, ncclInt64, 0, comm_of(c), c.cstream), "status broadcast"));
  EIG_TRY(c.check(cudaMemcpyAsync(&h, d, sizeof(int64_t), cudaMemcpyDeviceToHost, c.cstream), "status"));
  EIG_TRY(c.check(cudaStreamSynchronize(c.cstream), "status sync"));
  *out = h;
  return 0;
}

struct Recv {   // per-rank receive buffers of the factors (rank 0 uses its own)
  double2 *A = nullptr, *L = nullptr, *pk = nullptr, *T1 = nullptr, *tau1 = nullptr, *V2 = nullptr, *tau2 = nullptr;
};

int recv_buffers(Ctx &c, int64_t n, Recv &r) {
  const int nb = c.nb;
  const int64_t K = num_panels(n, nb), slots = v2_slots(n, nb);
  r.pk = (double2 *)c.ws(WS_C_PACK, (size_t)std::max<int64_t>(packed_off(n, n), 1) * sizeof(double2));
  r.T1 = (double2 *)c.ws(WS_C_T1, (size_t)std::max<int64_t>(K, 1) * nb * nb * sizeof(double2));
  r.tau1 = (double2 *)c.ws(WS_C_TAU1, (size_t)std::max<int64_t>(K, 1) * nb * sizeof(double2));
  if (!r.pk || !r.T1 || !r.tau1) return EIG_ERR_NOMEM;
  if (c.rank != 0) {
    r.A = (double2 *)c.ws(WS_C_A, (size_t)n * n * sizeof(double2));
    r.L = (double2 *)c.ws(WS_C_L, (size_t)n * n * sizeof(double2));
    r.V2 = (double2 *)c.ws(WS_C_V2, (size_t)std::max<int64_t>(slots, 1) * nb * sizeof(double2));
    r.tau2 = (double2 *)c.ws(WS_C_TAU2, (size_t)std::max<int64_t>(slots, 1) * sizeof(double2));
    if (!r.A || !r.L || !r.V2 || !r.tau2) return EIG_ERR_NOMEM;
  }
  return 0;
}

}  // namespace

int comm_unique_id(void *id128) {
  if (!id128) return -1;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return EIG_ERR_NCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof(id));
  return 0;
}

int comm_init(Ctx &c, const void *id128) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm = nullptr;
  EIG_TRY(nccl_check(c, ncclCommInitRank(&comm, c.nranks, id, c.rank), "ncclCommInitRank"));
  c.nccl = comm;
  EIG_TRY(c.check(cudaStreamCreateWithFlags(&c.cstream, cudaStreamNonBlocking), "comm stream"));
  for (int i = 0; i < 4; i++)
    EIG_TRY(c.check(cudaEventCreateWithFlags(&c.ev_c[i], cudaEventDisableTiming), "comm event"));
  return 0;
}

int comm_reserve(Ctx &c, int64_t n_max) {
  Recv r;
  return recv_buffers(c, n_max, r);
}

void comm_destroy(Ctx &c) {
  if (c.cstream) {
    cudaStreamSynchronize(c.cstream);
    cudaStreamDestroy(c.cstream);
    c.cstream = nullptr;
  }
  for (int i = 0; i < 4; i++)
    if (c.ev_c[i]) {
      cudaEventDestroy(c.ev_c[i]);
      c.ev_c[i] = nullptr;
    }
  if (c.nccl) {
    ncclCommDestroy(comm_of(c));
    c.nccl = nullptr;
  }
}

// Collective eig_hotpath (see include/eig.h): he2hb on rank 0, the factors
// broadcast, every rank back-transforms its own column slice.
int coll_hotpath(Ctx &c, int64_t n, double2 *A, int64_t lda, double2 *tau1, double2 *T1, const double2 *V2,
                 const double2 *tau2, const double2 *L, int64_t ldl, const double *Z, int64_t ldz, double2 *E,
                 int64_t lde, int64_t m, unsigned flags) {
  const bool root = c.rank == 0;
  const int nb = c.nb;
  const int64_t K = num_panels(n, nb), slots = v2_slots(n, nb);
  const bool do_bt = !(flags & EIG_SKIP_BT);
  if (root && (!A || lda < n)) return !A ? -3 : -4;
  if (root && do_bt && (!V2 || !tau2 || !L || ldl < n)) return !V2 ? -7 : (!tau2 ? -8 : (!L ? -9 : -11));
  if (root && (flags & EIG_SKIP_HE2HB) && K > 0 && !T1) return -6;
  Recv r;
  EIG_TRY(recv_buffers(c, n, r));
  double2 *dA = root ? A : r.A, *dL = root ? const_cast<double2 *>(L) : r.L;
  double2 *dV2 = root ? const_cast<double2 *>(V2) : r.V2, *dtau2 = root ? const_cast<double2 *>(tau2) : r.tau2;
  double2 *dT1 = (root && T1) ? T1 : r.T1, *dtau1 = (root && tau1) ? tau1 : r.tau1;
  const int64_t dlda = root ? lda : n, dldl = root ? ldl : n;
  c.stat_reset();
  c.st.m = m;   // this rank's slice width (the caller slices)
  c.st.col_hi = m;
  EIG_TRY(c.stat_begin(EIG_ST_TOTAL));
  if ((c.flags & EIG_DIST_HE2HB) && !(flags & EIG_SKIP_HE2HB)) {
    // NEXT-4: he2hb distributed over the ranks (he2hb_dist.cu); every rank
    // ends with V1 (in dA) and T1, so only V2 / tau2 / L travel afterwards.
    // All NCCL work in program order (one communicator, no concurrent streams).
    const int P = c.nranks;
    const int64_t nloc = dist_ncols(n, c.rank, P, nb);
    double2 *Aloc = (double2 *)c.ws(WS_C_ALOC, (size_t)n * std::max<int64_t>(nloc, 1) * sizeof(double2));
    double2 *work = (double2 *)c.ws(WS_C_DWORK, he2hb_dist_work(n, nb, P, c.rank) * sizeof(double2));
    double2 *pack = (root && dlda != n) ? (double2 *)c.ws(WS_C_E, (size_t)n * n * sizeof(double2)) : nullptr;
    if (!Aloc || !work || (root && dlda != n && !pack)) return EIG_ERR_NOMEM;
    EIG_TRY(c.stat_begin(EIG_ST_HE2HB));
    if (root) {
      EIG_TRY(real_diag(c, n, dA, dlda));
      EIG_TRY(herm_full(c, n, dA, dlda));
    }
    EIG_TRY(dist_scatter(c, n, dA, dlda, Aloc, pack));
    EIG_TRY(he2hb_dist_nccl(c, n, Aloc, dA, dtau1, dT1, work, root ? dA : nullptr, dlda));
    EIG_TRY(c.stat_end(EIG_ST_HE2HB));
    c.st.flops[EIG_ST_HE2HB] = 16.0 / 3.0 * (double)n * n * n / P;
    if (do_bt) {
      EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[0], "comm fork"));
      EIG_TRY(bcast(c, dV2, (size_t)slots * nb * sizeof(double2), "bcast V2"));
      EIG_TRY(bcast(c, dtau2, (size_t)slots * sizeof(double2), "bcast tau2"));
      EIG_TRY(bcast_lower(c, dL, n, dldl, r.pk, "bcast L"));
      EIG_TRY(order(c, c.cstream, c.stream, c.ev_c[2], "factors in"));
      EIG_TRY(bt_run(c, n, Z, ldz, dV2, dtau2, dA, dlda, dT1, dL, dldl, E, lde, m));
    }
    EIG_TRY(c.stat_end(EIG_ST_TOTAL));
    return c.check(cudaStreamSynchronize(c.stream), "sync");
  }
  // the communication stream starts after the inputs already queued on the compute stream
  EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[0], "comm fork"));
  if (do_bt) {   // inputs of the back-transform: available now, overlap he2hb on rank 0
    EIG_TRY(bcast(c, dV2, (size_t)slots * nb * sizeof(double2), "bcast V2"));
    EIG_TRY(bcast(c, dtau2, (size_t)slots * sizeof(double2), "bcast tau2"));
    EIG_TRY(bcast_lower(c, dL, n, dldl, r.pk, "bcast L"));
  }
  if (root && !(flags & EIG_SKIP_HE2HB)) {
    EIG_TRY(c.stat_begin(EIG_ST_HE2HB));
    EIG_TRY(he2hb_run(c, n, dA, dlda, dtau1, dT1));
    EIG_TRY(c.stat_end(EIG_ST_HE2HB));
    c.st.flops[EIG_ST_HE2HB] = 16.0 / 3.0 * (double)n * n * n;
  }
  if (do_bt) {
    EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[1], "he2hb done"));
    EIG_TRY(bcast_lower(c, dA, n, dlda, r.pk, "bcast A (V1)"));
    EIG_TRY(bcast(c, dT1, (size_t)K * nb * nb * sizeof(double2), "bcast T1"));
    EIG_TRY(order(c, c.cstream, c.stream, c.ev_c[2], "factors in"));
    EIG_TRY(bt_run(c, n, Z, ldz, dV2, dtau2, dA, dlda, dT1, dL, dldl, E, lde, m));
  }
  EIG_TRY(order(c, c.cstream, c.stream, c.ev_c[3], "comm join"));
  EIG_TRY(c.stat_end(EIG_ST_TOTAL));
  return c.check(cudaStreamSynchronize(c.stream), "sync");
}

// Collective eig_solve_gen (see include/eig.h).
int coll_solve_gen(Ctx &c, int64_t n, double2 *A, int64_t lda, double2 *B, int64_t ldb, int64_t il, int64_t iu,
                   double *w, double2 *Z, int64_t ldz) {
  const bool root = c.rank == 0;
  const bool gather = (c.flags & EIG_GATHER_Z) != 0;
  const int nb = c.nb, P = c.nranks;
  const int64_t m = iu - il + 1;
  int64_t lo = 0, hi = 0;
  EIG_TRY(eig_column_slice(m, c.rank, P, &lo, &hi));
  const int64_t mr = hi - lo;
  if (root && (!A || lda < std::max<int64_t>(1, n))) return !A ? -3 : -4;
  if (root && (!B || ldb < std::max<int64_t>(1, n))) return !B ? -5 : -6;
  if (!w && n > 0) return -11;
  if (ldz < std::max<int64_t>(1, n)) return -13;
  if (!Z && !(gather && !root) && mr > 0) return -12;
  if (n == 0) return 0;
  const int64_t K = num_panels(n, nb), slots = v2_slots(n, nb);
  const double dn = (double)n;
  Recv r;
  EIG_TRY(recv_buffers(c, n, r));
  double2 *dA = root ? A : r.A, *dL = root ? B : r.L;
  const int64_t dlda = root ? lda : n, dldl = root ? ldb : n;
  double2 *V2 = (double2 *)c.ws(WS_SG_V2, (size_t)std::max<int64_t>(slots, 1) * nb * sizeof(double2));
  double2 *tau2 = (double2 *)c.ws(WS_SG_TAU2, (size_t)std::max<int64_t>(slots, 1) * sizeof(double2));
  // tridiagonal eigenvectors: all m columns on rank 0, this rank's slice elsewhere
  double *Zr = (double *)c.ws(WS_SG_Z, (size_t)n * std::max<int64_t>(root ? m : mr, 1) * sizeof(double));
  double *dd = (double *)c.ws(WS_SG_D, (size_t)n * sizeof(double));
  double *de = (double *)c.ws(WS_SG_E, (size_t)n * sizeof(double));
  if (!V2 || !tau2 || !Zr || !dd || !de) return EIG_ERR_NOMEM;
  c.stat_reset();
  c.st.m = m;
  c.st.col_lo = lo;
  c.st.col_hi = hi;
  EIG_TRY(c.stat_begin(EIG_ST_TOTAL));
  // ---- step 1 on rank 0; its info is every rank's result
  int64_t info = 0;
  if (root) {
    EIG_TRY(c.stat_begin(EIG_ST_POTRF));
    info = potrf_run(c, n, B, ldb);
    if (info < 0) return (int)info;
    EIG_TRY(c.stat_end(EIG_ST_POTRF));
    c.st.flops[EIG_ST_POTRF] = 4.0 / 3.0 * dn * dn * dn;
  }
  EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[0], "comm fork"));
  EIG_TRY(bcast_status(c, info, &info));
  if (info) return (int)info;
  const bool dist = (c.flags & EIG_DIST_HE2HB) != 0;
  if (root) {
    EIG_TRY(c.stat_begin(EIG_ST_HEGST));
    EIG_TRY(hegst_run(c, n, dA, dlda, dL, dldl));
    EIG_TRY(c.stat_end(EIG_ST_HEGST));
    c.st.flops[EIG_ST_HEGST] = 4.0 * dn * dn * dn;
  }
  if (!dist) {
    // ---- step 3a on rank 0; L, V1, T1 broadcast while it chases the bulges
    if (root) {
      EIG_TRY(c.stat_begin(EIG_ST_HE2HB));
      EIG_TRY(he2hb_run(c, n, dA, dlda, r.tau1, r.T1));
      EIG_TRY(c.stat_end(EIG_ST_HE2HB));
      c.st.flops[EIG_ST_HE2HB] = 16.0 / 3.0 * dn * dn * dn;
    }
    EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[1], "he2hb done"));
    EIG_TRY(bcast_lower(c, dL, n, dldl, r.pk, "bcast L"));
    EIG_TRY(bcast_lower(c, dA, n, dlda, r.pk, "bcast A (V1)"));
    EIG_TRY(bcast(c, r.T1, (size_t)K * nb * nb * sizeof(double2), "bcast T1"));
  } else {
    // ---- NEXT-4: step 3a distributed over all ranks (1D block-cyclic
    // columns, he2hb_dist.cu).  Every rank ends with all of V1 (in dA) and
    // T1; rank 0 also gets the band for the bulge chase.  All NCCL work of
    // this phase is on the compute stream (one communicator, one order).
    if (root) EIG_TRY(herm_full(c, n, dA, dlda));
    const int64_t nloc = dist_ncols(n, c.rank, P, nb);
    double2 *Aloc = (double2 *)c.ws(WS_C_ALOC, (size_t)n * std::max<int64_t>(nloc, 1) * sizeof(double2));
    double2 *work = (double2 *)c.ws(WS_C_DWORK, he2hb_dist_work(n, nb, P, c.rank) * sizeof(double2));
    double2 *pack = (root && dlda != n) ? (double2 *)c.ws(WS_C_E, (size_t)n * n * sizeof(double2)) : nullptr;
    if (!Aloc || !work || (root && dlda != n && !pack)) return EIG_ERR_NOMEM;
    EIG_TRY(c.stat_begin(EIG_ST_HE2HB));
    EIG_TRY(dist_scatter(c, n, dA, dlda, Aloc, pack));
    EIG_TRY(he2hb_dist_nccl(c, n, Aloc, dA, r.tau1, r.T1, work, root ? dA : nullptr, dlda));
    EIG_TRY(c.stat_end(EIG_ST_HE2HB));
    c.st.flops[EIG_ST_HE2HB] = 16.0 / 3.0 * dn * dn * dn / P;
    EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[1], "he2hb done"));
    EIG_TRY(bcast_lower(c, dL, n, dldl, r.pk, "bcast L"));
  }
  // ---- bulge chase on rank 0; V2 / tau2 broadcast during stedc
  if (root) {
    EIG_TRY(c.stat_begin(EIG_ST_HB2ST));
    EIG_TRY(hb2st_run(c, n, dA, dlda, dd, de, V2, tau2));
    EIG_TRY(c.stat_end(EIG_ST_HB2ST));
  }
  EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[2], "hb2st done"));
  EIG_TRY(bcast(c, V2, (size_t)slots * nb * sizeof(double2), "bcast V2"));
  EIG_TRY(bcast(c, tau2, (size_t)slots * sizeof(double2), "bcast tau2"));
  int64_t st_rc = 0;
  if (root) {
    EIG_TRY(c.stat_begin(EIG_ST_STEDC));
    st_rc = stedc(c, n, dd, de, il, iu, w, Zr, n);   // an error here is every rank's result (below)
    if (!st_rc) EIG_TRY(c.stat_end(EIG_ST_STEDC));
  }
  EIG_TRY(order(c, c.stream, c.cstream, c.ev_c[3], "stedc done"));
  EIG_TRY(bcast_status(c, st_rc, &st_rc));
  if (st_rc) return (int)st_rc;
  // ---- eigenvalues to everyone, eigenvector columns scattered by slice
  EIG_TRY(bcast(c, w, (size_t)n * sizeof(double), "bcast w"));
  EIG_TRY(nccl_check(c, ncclGroupStart(), "group"));
  for (int q = 0; q < P; q++) {
    int64_t qlo = 0, qhi = 0;
    eig_column_slice(m, q, P, &qlo, &qhi);
    const size_t cnt = (size_t)(qhi - qlo) * n;
    if (cnt == 0) continue;
    if (root && q != 0) {
      EIG_TRY(nccl_check(c, ncclSend(Zr + qlo * n, cnt, ncclDouble, q, comm_of(c), c.cstream), "scatter send"));
      c.st.bytes_comm += (int64_t)(cnt * sizeof(double));
    } else if (!root && q == c.rank) {
      EIG_TRY(nccl_check(c, ncclRecv(Zr, cnt, ncclDouble, 0, comm_of(c), c.cstream), "scatter recv"));
      c.st.bytes_comm += (int64_t)(cnt * sizeof(double));
    }
  }
  EIG_TRY(nccl_check(c, ncclGroupEnd(), "group"));
  EIG_TRY(order(c, c.cstream, c.stream, c.ev_c[0], "factors in"));
  // ---- back-transform of this rank's columns
  const double *Zmine = Zr + (root ? lo * n : 0);
  double2 *Emine;
  int64_t lde;
  if (Z && (!gather || !root)) {
    Emine = Z;
    lde = ldz;
  } else if (Z) {   // rank 0 gathering: its own slice goes straight into place
    Emine = Z + lo * ldz;
    lde = ldz;
  } else {
    Emine = (double2 *)c.ws(WS_C_E, (size_t)n * std::max<int64_t>(mr, 1) * sizeof(double2));
    if (!Emine) return EIG_ERR_NOMEM;
    lde = n;
  }
  EIG_TRY(bt_run(c, n, Zmine, n, V2, tau2, dA, dlda, r.T1, dL, dldl, Emine, lde, mr));
  // ---- optional gather of the E slices to rank 0
  if (gather && P > 1) {
    EIG_TRY(c.stat_begin(EIG_ST_GATHER));
    // senders need contiguous slices (ld n)
    double2 *Esend = Emine;
    if (!root && lde != n && mr > 0) {
      Esend = (double2 *)c.ws(WS_C_E, (size_t)n * mr * sizeof(double2));
      if (!Esend) return EIG_ERR_NOMEM;
      EIG_TRY(c.check(cudaMemcpy2DAsync(Esend, n * sizeof(double2), Emine, lde * sizeof(double2),
                                        n * sizeof(double2), mr, cudaMemcpyDeviceToDevice, c.stream), "pack E"));
    }
    double2 *Rtmp = nullptr;
    if (root && ldz != n) {
      Rtmp = (double2 *)c.ws(WS_C_E, (size_t)n * std::max<int64_t>(m, 1) * sizeof(double2));
      if (!Rtmp) return EIG_ERR_NOMEM;
    }
    EIG_TRY(nccl_check(c, ncclGroupStart(), "group"));
    for (int q = 1; q < P; q++) {
      int64_t qlo = 0, qhi = 0;
      eig_column_slice(m, q, P, &qlo, &qhi);
      const size_t cnt = (size_t)(qhi - qlo) * n * 2;   // doubles
      if (cnt == 0) continue;
      if (root) {
        double2 *dst = Rtmp ? Rtmp + qlo * n : Z + qlo * ldz;
        EIG_TRY(nccl_check(c, ncclRecv(dst, cnt, ncclDouble, q, comm_of(c), c.stream), "gather recv"));
        c.st.bytes_comm += (int64_t)(cnt * sizeof(double));
      } else if (q == c.rank) {
        EIG_TRY(nccl_check(c, ncclSend(Esend, cnt, ncclDouble, 0, comm_of(c), c.stream), "gather send"));
        c.st.bytes_comm += (int64_t)(cnt * sizeof(double));
      }
    }
    EIG_TRY(nccl_check(c, ncclGroupEnd(), "group"));
    if (Rtmp) {
      int64_t qlo = 0, qhi = 0;
      eig_column_slice(m, 1, P, &qlo, &qhi);
      EIG_TRY(c.check(cudaMemcpy2DAsync(Z + qlo * ldz, ldz * sizeof(double2), Rtmp + qlo * n, n * sizeof(double2),
                                        n * sizeof(double2), m - qlo, cudaMemcpyDeviceToDevice, c.stream),
                      "unpack gathered E"));
    }
    EIG_TRY(c.stat_end(EIG_ST_GATHER));
  }
  EIG_TRY(c.stat_end(EIG_ST_TOTAL));
  return c.check(cudaStreamSynchronize(c.stream), "sync");
}

}  // namespace eig
