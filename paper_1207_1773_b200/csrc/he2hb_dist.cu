// he2hb_dist.cu — NEXT-4: reduction to band form with the columns of the
// Hermitian matrix distributed 1D block-cyclically over P ranks (§6:
// "The data on the GPUs is distributed in a 1D block cyclic way"; the
// trigger and the projection are in DESIGN.md §8).
//
// Rank r owns the FULL columns (both triangles) of the nb-wide column blocks
// b with b mod P == r, stored in order in a local n x nloc array (ld n).
// Step k (panel = block k, owner o = k mod P, trailing rows/cols r0 = (k+1) nb):
//   owner:  panel QR + T of A[r0:, block k]                (panel_qr_kernel, a1-a2)
//   bcast:  V_k (s x nb), T_k, tau_k from o                (every rank keeps them: V1, T1 for the BT)
//   all:    W_r = A[r0:, J_r] V_k[J_r]                     (J_r = r's trailing columns, one zgemm)
//   allreduce W = sum_r W_r                                 (a3: W = A22 V)
//   all:    W <- W T, M = T^H V^H W, X = W - 1/2 V M        (a4, replicated)
//   all:    A[r0:, J_r] -= V X[J_r]^H + X V[J_r]^H          (a5 on the owned full columns)
// Every rank therefore does 24 s^2 nb / P flops per step instead of the
// single-GPU 16 s^2 nb (full columns instead of the lower triangle).
//
// The collectives go through `DistOps`: NCCL on the handle's communicator
// for real ranks, or, for P "virtual" ranks on ONE GPU (eig_he2hb_sim, the
// arithmetic check), device copies and a fixed-order sum over the ranks'
// buffers.  Both run the same per-rank local code below.
#include <nccl.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"
#include "stages.h"

namespace eig {
namespace {

// global column of local column lc of rank r (1D block-cyclic, block nb)
__host__ __device__ __forceinline__ int64_t gcol_of(int64_t lc, int r, int P, int nb) {
  return ((lc / nb) * P + r) * nb + lc % nb;
}
// local columns of rank r
int64_t ncols_of(int64_t n, int r, int P, int nb) {
  const int64_t NB = (n + nb - 1) / nb;
  int64_t c = 0;
  for (int64_t b = r; b < NB; b += P) c += std::min<int64_t>(nb, n - b * nb);
  return c;
}
// first local column of rank r whose global column is >= g0 (g0 a block start)
int64_t first_local_ge(int64_t g0, int r, int P, int nb) {
  const int64_t b0 = g0 / nb;
  int64_t b = b0 + ((r - b0 % P) % P + P) % P;   // smallest owned block >= b0
  return (b / P) * nb;
}

// Mg[lr, :] = M[gcol(lc0 + lr) - r0, :]  (rows of an s x w matrix, ld ldm,
// for the trailing local columns of rank r), Mg ld ldg
__global__ void gather_rows_kernel(int64_t nl, int64_t lc0, int r, int P, int nb, int64_t r0, int w,
                                   const double2 *M, int64_t ldm, double2 *Mg, int64_t ldg) {
  const int64_t total = nl * w;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lr = e % nl;
    const int col = (int)(e / nl);
    Mg[lr + col * ldg] = M[(gcol_of(lc0 + lr, r, P, nb) - r0) + col * ldm];
  }
}

// local <-> global full columns (block-cyclic), for the virtual-rank check
__global__ void cyclic_copy_kernel(int64_t n, int r, int P, int nb, int64_t nl, double2 *G, int64_t ldg,
                                   double2 *Lc, bool to_local) {
  const int64_t total = n * nl;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e % n, lc = e / n;
    double2 *g = G + row + gcol_of(lc, r, P, nb) * ldg;
    if (to_local) Lc[e] = *g;
    else *g = Lc[e];
  }
}

// V_k tails into the he2hb layout of the (n x n, ld) V1 holder: column k nb + j,
// rows (k+1) nb + j + 1 .. n-1  <-  V[j+1.., j]
__global__ void place_v_kernel(int64_t s, int nb, const double2 *V, int64_t ldv, double2 *A, int64_t lda) {
  const int64_t total = s * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % s;
    const int j = (int)(e / s);
    if (i > j) A[i + j * lda] = V[i + j * ldv];
  }
}

// out = sum_q in[q] (fixed order q = 0..P-1)
__global__ void sum_ranks_kernel(int64_t count, int P, double2 *const *in, double2 *out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = in[0][e];
    for (int q = 1; q < P; q++) acc = cadd(acc, in[q][e]);
    out[e] = acc;
  }
}

int grid_for(Ctx &c, int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 8LL * c.num_sms)); }

}  // namespace

// Per-rank state of the distributed reduction.
struct DistRank {
  int r;                 // global rank id
  double2 *Aloc;         // n x nloc, ld n (full columns of the owned blocks)
  int64_t nloc;
  double2 *V1;           // n x n, ld n: V1 tails in the he2hb layout (receives every panel's V)
  double2 *tau, *T;      // K nb, K nb nb
  double2 *Vb, *Wb, *Xb, *Gb, *Sm;   // work: V (2 buffers of s x nb), W / X (s x nb), gathered rows, small
  double2 *Wpart;        // this rank's partial W
};

// The collectives of the distributed reduction.  For real ranks `ranks` has
// one entry (this process); for virtual ranks all P live on this GPU.
struct DistOps {
  Ctx *c;
  bool virt;
  int P;
  std::vector<DistRank> *ranks;
  double2 **d_ptrs;      // virtual: device array of P pointers (sum_ranks_kernel)
  // every rank's buf <- owner's buf (count complex)
  int bcast(std::vector<double2 *> bufs, size_t count, int owner) {
    if (count == 0) return 0;
    if (virt) {
      for (int q = 0; q < P; q++)
        if (q != owner)
          EIG_TRY(c->check(cudaMemcpyAsync(bufs[q], bufs[owner], count * sizeof(double2), cudaMemcpyDeviceToDevice,
                                           c->stream), "virtual bcast"));
      return 0;
    }
    c->st.bytes_comm += (int64_t)(count * sizeof(double2));
    if (ncclBroadcast(bufs[0], bufs[0], count * 2, ncclDouble, owner, (ncclComm_t)c->nccl, c->stream) != ncclSuccess) {
      c->last_err = "ncclBroadcast (he2hb_dist)";
      return EIG_ERR_NCCL;
    }
    return 0;
  }
  // every rank's out <- sum of every rank's in
  int allreduce(std::vector<double2 *> in, std::vector<double2 *> out, size_t count) {
    if (count == 0) return 0;
    if (virt) {
      EIG_TRY(c->check(cudaMemcpyAsync(d_ptrs, in.data(), P * sizeof(double2 *), cudaMemcpyHostToDevice, c->stream),
                       "virtual allreduce ptrs"));
      sum_ranks_kernel<<<grid_for(*c, (int64_t)count), 256, 0, c->stream>>>((int64_t)count, P, d_ptrs, out[0]);
      EIG_TRY(c->launched("sum_ranks_kernel"));
      for (int q = 1; q < P; q++)
        EIG_TRY(c->check(cudaMemcpyAsync(out[q], out[0], count * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream),
                         "virtual allreduce copy"));
      return 0;
    }
    c->st.bytes_comm += (int64_t)(count * sizeof(double2));
    if (ncclAllReduce(in[0], out[0], count * 2, ncclDouble, ncclSum, (ncclComm_t)c->nccl, c->stream) != ncclSuccess) {
      c->last_err = "ncclAllReduce (he2hb_dist)";
      return EIG_ERR_NCCL;
    }
    return 0;
  }
};

// The distributed reduction over the ranks in `ops.ranks` (see the header).
int he2hb_dist_run(Ctx &c, int64_t n, DistOps &ops) {
  const int nb = c.nb, P = ops.P;
  const int64_t K = num_panels(n, nb);
  std::vector<DistRank> &R = *ops.ranks;
  const int nv = (int)R.size();
  auto bufs = [&](auto f) {
    std::vector<double2 *> v(nv);
    for (int q = 0; q < nv; q++) v[q] = f(R[q]);
    return v;
  };
  auto local_of = [&](int owner) -> int {   // index in R of global rank `owner`, or -1
    for (int q = 0; q < nv; q++)
      if (R[q].r == owner) return q;
    return -1;
  };
  const int64_t s0 = n - nb;
  auto vbuf = [&](DistRank &d, int64_t k) { return d.Vb + (k & 1) * s0 * nb; };   // V_k, double-buffered
  // panel 0 on its owner
  if (K > 0) {
    const int qo = local_of(0);
    if (qo >= 0)
      EIG_TRY(panel_qr(c, R[qo].Aloc + nb, n, n - nb, nb, R[qo].tau, R[qo].T, vbuf(R[qo], 0), nullptr, n - nb,
                       c.stream));
  }
  for (int64_t k = 0; k < K; k++) {
    const int64_t r0 = (k + 1) * nb, s = n - r0;
    const int owner = (int)(k % P);
    const int nref = (int)std::min<int64_t>(nb, s);
    // a1-a2 ran on the owner: panel 0 above, panel k > 0 on the side stream during step k-1 (look-ahead)
    if (k > 0 && local_of(owner) >= 0) EIG_TRY(c.check(cudaStreamWaitEvent(c.stream, c.ev_join, 0), "panel join"));
    // V_k, T_k, tau_k to every rank (the BT needs them all: V1 and T1 stay replicated)
    EIG_TRY(ops.bcast(bufs([&](DistRank &d) { return vbuf(d, k); }), (size_t)s * nb, owner));
    EIG_TRY(ops.bcast(bufs([&](DistRank &d) { return d.T + k * nb * nb; }), (size_t)nb * nb, owner));
    EIG_TRY(ops.bcast(bufs([&](DistRank &d) { return d.tau + k * nb; }), (size_t)nb, owner));
    for (auto &d : R) {
      place_v_kernel<<<grid_for(c, s * nref), 256, 0, c.stream>>>(s, nref, vbuf(d, k), s, d.V1 + r0 + k * nb * n, n);
      EIG_TRY(c.launched("place_v_kernel"));
    }
    // a3: W_r = A[r0:, J_r] V[J_r]
    std::vector<int64_t> lc0(nv), nl(nv);
    for (int q = 0; q < nv; q++) {
      DistRank &d = R[q];
      lc0[q] = std::min<int64_t>(d.nloc, first_local_ge(r0, d.r, P, nb));
      nl[q] = d.nloc - lc0[q];
      if (nl[q] > 0) {
        gather_rows_kernel<<<grid_for(c, nl[q] * nb), 256, 0, c.stream>>>(nl[q], lc0[q], d.r, P, nb, r0, nb, vbuf(d, k), s,
                                                                           d.Gb, nl[q]);
        EIG_TRY(c.launched("gather_rows_kernel"));
        Zgemm g;
        g.M = s; g.N = nb; g.K = nl[q]; g.A = d.Aloc + r0 + lc0[q] * n; g.lda = n; g.B = d.Gb; g.ldb = nl[q];
        g.C = d.Wpart; g.ldc = s;
        EIG_TRY(zgemm(c, g));
      } else {
        EIG_TRY(c.check(cudaMemsetAsync(d.Wpart, 0, (size_t)s * nb * sizeof(double2), c.stream), "W = 0"));
      }
    }
    EIG_TRY(ops.allreduce(bufs([](DistRank &d) { return d.Wpart; }), bufs([](DistRank &d) { return d.Wb; }),
                          (size_t)s * nb));
    // a4 (replicated): X = W T - 1/2 V (T^H V^H W T)
    for (auto &d : R) {
      const double2 *Tk = d.T + k * nb * nb;
      Zgemm g;
      g.M = s; g.N = nb; g.K = nb; g.A = d.Wb; g.lda = s; g.B = Tk; g.ldb = nb; g.C = d.Xb; g.ldc = s;
      EIG_TRY(zgemm(c, g));   // X = W T
      g = Zgemm();
      g.opa = OP_C; g.M = nb; g.N = nb; g.K = s; g.A = vbuf(d, k); g.lda = s; g.B = d.Xb; g.ldb = s; g.C = d.Sm; g.ldc = nb;
      EIG_TRY(zgemm(c, g));   // V^H (W T)
      g = Zgemm();
      g.opa = OP_C; g.M = nb; g.N = nb; g.K = nb; g.A = Tk; g.lda = nb; g.B = d.Sm; g.ldb = nb; g.C = d.Sm + nb * nb;
      g.ldc = nb;
      EIG_TRY(zgemm(c, g));   // M = T^H V^H W T
      g = Zgemm();
      g.M = s; g.N = nb; g.K = nb; g.A = vbuf(d, k); g.lda = s; g.B = d.Sm + nb * nb; g.ldb = nb; g.C = d.Xb; g.ldc = s;
      g.alpha = -0.5; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));   // X = W T - 1/2 V M
    }
    // a5: owned full columns  A[r0:, J_r] -= [V X] [X_g V_g]^H
    for (int q = 0; q < nv; q++) {
      DistRank &d = R[q];
      if (nl[q] <= 0) continue;
      double2 *XV = d.Gb;   // [X_g | V_g]  (nl x 2nb)
      gather_rows_kernel<<<grid_for(c, nl[q] * nb), 256, 0, c.stream>>>(nl[q], lc0[q], d.r, P, nb, r0, nb, d.Xb, s,
                                                                         XV, nl[q]);
      EIG_TRY(c.launched("gather_rows_kernel"));
      gather_rows_kernel<<<grid_for(c, nl[q] * nb), 256, 0, c.stream>>>(nl[q], lc0[q], d.r, P, nb, r0, nb, vbuf(d, k), s,
                                                                         XV + nl[q] * nb, nl[q]);
      EIG_TRY(c.launched("gather_rows_kernel"));
      // [V | X] side by side: V in Vb, X in Xb (both ld s) -> two K = nb products
      auto update = [&](int64_t c0, int64_t cn) -> int {   // local trailing columns lc0 + c0 .. + cn
        if (cn <= 0) return 0;
        Zgemm g;
        g.opb = OP_C; g.M = s; g.N = cn; g.K = nb; g.A = vbuf(d, k); g.lda = s; g.B = XV + c0; g.ldb = nl[q];
        g.C = d.Aloc + r0 + (lc0[q] + c0) * n; g.ldc = n; g.alpha = -1.0; g.beta = 1.0;
        EIG_TRY(zgemm(c, g));   // -= V X_g^H
        g.A = d.Xb; g.B = XV + nl[q] * nb + c0;
        return zgemm(c, g);     // -= X V_g^H
      };
      const bool next_mine = (k + 1 < K) && (int)((k + 1) % P) == d.r;
      if (next_mine) {
        // look-ahead (Fig. 1 "(a) can be overlapped with (c)"): block k+1 is this
        // rank's first trailing block; update it, run panel k+1 on the side
        // stream, and update the remaining columns meanwhile
        EIG_TRY(update(0, nb));
        EIG_TRY(c.check(cudaEventRecord(c.ev_fork, c.stream), "fork"));
        EIG_TRY(c.check(cudaStreamWaitEvent(c.side, c.ev_fork, 0), "fork wait"));
        const int64_t r1 = r0 + nb;
        EIG_TRY(panel_qr(c, d.Aloc + r1 + lc0[q] * n, n, n - r1, nb, d.tau + (k + 1) * nb, d.T + (k + 1) * nb * nb,
                         vbuf(d, k + 1), nullptr, n - r1, c.side));
        EIG_TRY(c.check(cudaEventRecord(c.ev_join, c.side), "join"));
        EIG_TRY(update(nb, nl[q] - nb));
      } else {
        EIG_TRY(update(0, nl[q]));
      }
    }
  }
  return 0;
}

// ------------------------------------------------------------------ virtual ranks (one GPU)
// he2hb of the Hermitian A (n x n, lda, lower read) computed by the
// distributed algorithm with P virtual ranks on this GPU; the result is
// assembled into A in the single-GPU he2hb layout (band + V1), plus tau, T.
int he2hb_sim(Ctx &c, int64_t n, int P, double2 *A, int64_t lda, double2 *tau, double2 *T) {
  const int nb = c.nb;
  const int64_t K = num_panels(n, nb);
  EIG_TRY(real_diag(c, n, A, lda));
  if (K == 0) return 0;
  EIG_TRY(herm_full(c, n, A, lda));
  std::vector<double2 *> allocs;
  auto dalloc = [&](size_t elems) -> double2 * {
    double2 *p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(elems, 1) * sizeof(double2)) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    allocs.push_back(p);
    return p;
  };
  std::vector<DistRank> R(P);
  double2 **d_ptrs = nullptr;
  int rc = c.check(cudaMalloc(&d_ptrs, P * sizeof(double2 *)), "ptrs");
  const int64_t s0 = n - nb;
  for (int q = 0; q < P && !rc; q++) {
    DistRank &d = R[q];
    d.r = q;
    d.nloc = ncols_of(n, q, P, nb);
    d.Aloc = dalloc((size_t)n * d.nloc);
    d.V1 = (q == 0) ? A : nullptr;   // rank 0 writes V1 straight into A; the others into scratch
    if (q != 0) d.V1 = dalloc((size_t)n * n);
    d.tau = (q == 0) ? tau : dalloc((size_t)K * nb);
    d.T = (q == 0) ? T : dalloc((size_t)K * nb * nb);
    d.Vb = dalloc((size_t)2 * s0 * nb);
    d.Wb = dalloc((size_t)s0 * nb);
    d.Xb = dalloc((size_t)s0 * nb);
    d.Wpart = dalloc((size_t)s0 * nb);
    d.Gb = dalloc((size_t)n * 2 * nb);
    d.Sm = dalloc((size_t)2 * nb * nb);
    if (!d.Aloc || !d.V1 || !d.tau || !d.T || !d.Vb || !d.Wb || !d.Xb || !d.Wpart || !d.Gb || !d.Sm) rc = EIG_ERR_NOMEM;
    if (!rc && d.nloc > 0) {
      cyclic_copy_kernel<<<grid_for(c, n * d.nloc), 256, 0, c.stream>>>(n, q, P, nb, d.nloc, A, lda, d.Aloc, true);
      rc = c.launched("cyclic_copy_kernel");
    }
  }
  if (!rc) {
    DistOps ops{&c, true, P, &R, d_ptrs};
    rc = he2hb_dist_run(c, n, ops);
  }
  // assemble: band (rows c..c+nb of column c) from the owners' columns; V1 already in A
  for (int q = 0; q < P && !rc; q++) {
    DistRank &d = R[q];
    if (d.nloc <= 0) continue;
    // copy whole owned columns into a scratch n x n, then take the band rows into A
    double2 *full = dalloc((size_t)n * n);
    if (!full) { rc = EIG_ERR_NOMEM; break; }
    cyclic_copy_kernel<<<grid_for(c, n * d.nloc), 256, 0, c.stream>>>(n, q, P, nb, d.nloc, full, n, d.Aloc, false);
    rc = c.launched("cyclic_copy_kernel");
    if (rc) break;
    for (int64_t lc = 0; lc < d.nloc && !rc; lc += nb) {
      const int64_t g0 = gcol_of(lc, q, P, nb);
      const int64_t w = std::min<int64_t>(nb, n - g0);
      // rows g0 .. min(n, g0 + w + nb) of the block's columns (covers the band 0 <= r - c <= nb)
      const int64_t rows = std::min<int64_t>(n, g0 + w + nb) - g0;
      rc = c.check(cudaMemcpy2DAsync(A + g0 + g0 * lda, lda * sizeof(double2), full + g0 + g0 * n, n * sizeof(double2),
                                     rows * sizeof(double2), w, cudaMemcpyDeviceToDevice, c.stream), "band");
    }
  }
  // the band rows below the diagonal block of each column hold R (in the
  // panel columns) and nothing else; rows beyond c + nb are V1 (placed above)
  if (!rc) rc = c.check(cudaStreamSynchronize(c.stream), "sync");
  for (double2 *p : allocs) cudaFree(p);
  if (d_ptrs) cudaFree(d_ptrs);
  if (!rc) rc = real_diag(c, n, A, lda);
  return rc;
}

// ------------------------------------------------------------------ real ranks (NCCL)
namespace {

// band rows [g0, g0 + w + nb) of the w columns of every owned block, packed
// block after block as (2 nb) x w column-major slabs (rows past n zero)
__global__ void band_pack_kernel(int64_t n, int r, int P, int nb, int64_t nloc, const double2 *Aloc, double2 *out,
                                 bool unpack, double2 *A, int64_t lda) {
  const int64_t nblk = (nloc + nb - 1) / nb;
  const int64_t total = nblk * 2 * nb * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lb = e / (2 * nb * nb);
    const int64_t rem = e % (2 * nb * nb);
    const int j = (int)(rem / (2 * nb)), i = (int)(rem % (2 * nb));
    const int64_t lc = lb * nb + j;
    if (lc >= nloc) continue;
    const int64_t gc = gcol_of(lc, r, P, nb);
    const int64_t g0 = gc - j, row = g0 + i;
    if (!unpack) {
      out[e] = row < n ? Aloc[row + lc * n] : czero();
    } else if (row < n && row >= gc) {   // lower part only (band, then R / V heads of the panel)
      A[row + gc * lda] = out[e];
    }
  }
}

}  // namespace

// Rank 0 holds the full Hermitian A (n x n, lda); every rank receives the
// full columns of its blocks into Aloc (n x nloc, ld n).  Grouped
// send/recv, one message per block.
int dist_scatter(Ctx &c, int64_t n, const double2 *A, int64_t lda, double2 *Aloc, double2 *pack) {
  const int nb = c.nb, P = c.nranks, r = c.rank;
  const int64_t NB = (n + nb - 1) / nb;
  ncclComm_t comm = (ncclComm_t)c.nccl;
  if (r == 0) {   // own blocks: local copies
    for (int64_t b = 0; b < NB; b += P) {
      const int64_t w = std::min<int64_t>(nb, n - b * nb);
      EIG_TRY(c.check(cudaMemcpy2DAsync(Aloc + (b / P) * nb * n, n * sizeof(double2), A + b * nb * lda,
                                        lda * sizeof(double2), n * sizeof(double2), w, cudaMemcpyDeviceToDevice,
                                        c.stream), "scatter own"));
    }
    if (lda != n) {   // contiguous send copies of the other ranks' blocks
      for (int64_t b = 0; b < NB; b++)
        if (b % P)
          EIG_TRY(c.check(cudaMemcpy2DAsync(pack + b * nb * n, n * sizeof(double2), A + b * nb * lda,
                                            lda * sizeof(double2), n * sizeof(double2),
                                            std::min<int64_t>(nb, n - b * nb), cudaMemcpyDeviceToDevice, c.stream),
                          "scatter pack"));
    }
  }
  if (P == 1) return 0;
  if (ncclGroupStart() != ncclSuccess) return EIG_ERR_NCCL;
  for (int64_t b = 0; b < NB; b++) {
    const int q = (int)(b % P);
    if (q == 0) continue;
    const size_t cnt = (size_t)n * std::min<int64_t>(nb, n - b * nb) * 2;
    if (r == 0) {
      const double2 *src = (lda == n) ? A + b * nb * lda : pack + b * nb * n;
      if (ncclSend(src, cnt, ncclDouble, q, comm, c.stream) != ncclSuccess) return EIG_ERR_NCCL;
      c.st.bytes_comm += (int64_t)(cnt * sizeof(double));
    } else if (q == r) {
      if (ncclRecv(Aloc + (b / P) * nb * n, cnt, ncclDouble, 0, comm, c.stream) != ncclSuccess) return EIG_ERR_NCCL;
      c.st.bytes_comm += (int64_t)(cnt * sizeof(double));
    }
  }
  if (ncclGroupEnd() != ncclSuccess) return EIG_ERR_NCCL;
  return 0;
}

// The distributed reduction for this rank (NCCL collectives).  Aloc: this
// rank's columns; V1: n x n (ld n) receiving every panel's reflector tails in
// the he2hb layout; tau, T: K nb and K nb^2 (every rank gets all of them).
// Afterwards the band of every block is gathered into rank 0's A (lower, lda).
int he2hb_dist_nccl(Ctx &c, int64_t n, double2 *Aloc, double2 *V1, double2 *tau, double2 *T, double2 *work,
                    double2 *A0, int64_t lda0) {
  const int nb = c.nb, P = c.nranks;
  const int64_t s0 = std::max<int64_t>(n - nb, 1);
  std::vector<DistRank> R(1);
  DistRank &d = R[0];
  d.r = c.rank;
  d.nloc = ncols_of(n, c.rank, P, nb);
  d.Aloc = Aloc;
  d.V1 = V1;
  d.tau = tau;
  d.T = T;
  d.Vb = work;
  d.Wb = d.Vb + 2 * s0 * nb;
  d.Xb = d.Wb + s0 * nb;
  d.Wpart = d.Xb + s0 * nb;
  d.Gb = d.Wpart + s0 * nb;
  d.Sm = d.Gb + (size_t)n * 2 * nb;
  double2 *bandbuf = d.Sm + 2 * nb * nb;   // (NB_loc) x 2nb x nb per rank, P of them on rank 0
  DistOps ops{&c, false, P, &R, nullptr};
  EIG_TRY(he2hb_dist_run(c, n, ops));
  // band gather: every rank packs its blocks' band slabs, rank 0 receives and unpacks
  const int64_t NB = (n + nb - 1) / nb, maxblk = (NB + P - 1) / P;
  const size_t slab = (size_t)maxblk * 2 * nb * nb;
  if (c.rank != 0 || P == 1) {
    band_pack_kernel<<<grid_for(c, (int64_t)slab), 256, 0, c.stream>>>(n, c.rank, P, nb, d.nloc, Aloc, bandbuf,
                                                                      false, nullptr, 0);
    EIG_TRY(c.launched("band_pack_kernel"));
  }
  if (P > 1) {
    ncclComm_t comm = (ncclComm_t)c.nccl;
    if (ncclGroupStart() != ncclSuccess) return EIG_ERR_NCCL;
    for (int q = 1; q < P; q++) {
      if (c.rank == 0) {
        if (ncclRecv(bandbuf + (size_t)q * slab, slab * 2, ncclDouble, q, comm, c.stream) != ncclSuccess)
          return EIG_ERR_NCCL;
      } else if (c.rank == q) {
        if (ncclSend(bandbuf, slab * 2, ncclDouble, 0, comm, c.stream) != ncclSuccess) return EIG_ERR_NCCL;
      }
      c.st.bytes_comm += (int64_t)(slab * sizeof(double2));
    }
    if (ncclGroupEnd() != ncclSuccess) return EIG_ERR_NCCL;
  }
  if (c.rank == 0) {
    for (int q = 0; q < P; q++) {
      const int64_t nl = ncols_of(n, q, P, nb);
      if (nl <= 0) continue;
      double2 *src = bandbuf + (size_t)q * slab;
      if (q == 0 && P > 1) {   // rank 0's own slabs straight from its columns
        band_pack_kernel<<<grid_for(c, (int64_t)slab), 256, 0, c.stream>>>(n, 0, P, nb, nl, Aloc, src, false,
                                                                          nullptr, 0);
        EIG_TRY(c.launched("band_pack_kernel"));
      }
      band_pack_kernel<<<grid_for(c, (int64_t)slab), 256, 0, c.stream>>>(n, q, P, nb, nl, nullptr, src, true, A0,
                                                                        lda0);
      EIG_TRY(c.launched("band_pack_kernel"));
    }
  }
  return 0;
}

// workspace of he2hb_dist_nccl (complex elements)
size_t he2hb_dist_work(int64_t n, int nb, int P, int rank) {
  const int64_t s0 = std::max<int64_t>(n - nb, 1);
  const int64_t NB = (n + nb - 1) / nb, maxblk = (NB + P - 1) / P;
  const size_t slab = (size_t)maxblk * 2 * nb * nb;
  return (size_t)5 * s0 * nb + (size_t)n * 2 * nb + 2 * nb * nb + slab * (rank == 0 ? P : 1);
}
int64_t dist_ncols(int64_t n, int rank, int P, int nb) { return ncols_of(n, rank, P, nb); }

}  // namespace eig
