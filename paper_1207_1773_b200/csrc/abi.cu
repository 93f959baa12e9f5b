// abi.cu — C ABI (include/eig.h) and the stage drivers of libeigb200.
//
// he2hb driver (Fig. 1; readings R3, R6), Q1 / Q2 / trsm
// back-transform drivers, the whole hot-path pass, and the
// handle / workspace management.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/eig.h"
#include "ctx.h"
#include "kernels.h"
#include "stages.h"

namespace eig {

void *Ctx::ws(int id, size_t need) {
  if (need == 0) need = 16;
  if (buf[id] && bytes[id] >= need) return buf[id];
  if (buf[id]) {
    cudaFree(buf[id]);  // synchronising: no in-flight kernel can still use it
    buf[id] = nullptr;
    bytes[id] = 0;
  }
  size_t alloc = need + need / 8;
  if (cudaMalloc(&buf[id], alloc) != cudaSuccess) {
    cudaGetLastError();
    if (cudaMalloc(&buf[id], need) != cudaSuccess) {
      cudaGetLastError();
      buf[id] = nullptr;
      last_err = "cudaMalloc failed";
      return nullptr;
    }
    alloc = need;
  }
  bytes[id] = alloc;
  return buf[id];
}

int Ctx::check(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return 0;
  last_err = std::string(what) + ": " + cudaGetErrorString(e);
  return EIG_ERR_CUDA;
}

int64_t num_panels(int64_t n, int nb) {
  if (n <= nb) return 0;
  return (n - nb - 1) / nb + 1;
}

int64_t v2_slots(int64_t n, int nb) {
  int64_t tot = 0;
  for (int64_t j = 0; 1 + j * nb <= n - 1; j++) tot += n - 1 - j * nb;
  return tot;
}

// ------------------------------------------------------------------ he2hb
// Step k (panel i = k nb, trailing A22 = A[r0:, r0:], r0 = i + nb, s = n - r0):
//   a1+a2  panel QR + T of A[r0:, i:i+nb]          (panel_qr, cooperative)
//   a3     W = A22 V T                              (Hermitian-A GEMM, split-K)
//   a4     M = T^H (V^H W),  X = W - 1/2 V M
//   a5     A22 -= V X^H + X V^H (lower)
// Look-ahead (Fig. 1: "(a) can be overlapped with (c)"): a5 is split
// into (i) the next panel's nb columns and (ii) the rest; panel k+1 runs on a
// high-priority side stream right after (i), concurrently with (ii).  The
// [V | X | V] workspace is double-buffered by step parity.
int he2hb_run(Ctx &c, int64_t n, double2 *A, int64_t lda, double2 *tau, double2 *T) {
  const int nb = c.nb;
  const int64_t K = num_panels(n, nb);
  EIG_TRY(real_diag(c, n, A, lda));
  if (K == 0) return 0;
  const int64_t ldw = n - nb;
  const size_t vxv_elems = (size_t)ldw * 3 * nb;
  double2 *VXV = (double2 *)c.ws(WS_VXV, 2 * vxv_elems * sizeof(double2));
  double2 *Wb = (double2 *)c.ws(WS_W, (size_t)ldw * nb * sizeof(double2));
  double2 *Sm = (double2 *)c.ws(WS_SMALL, (size_t)2 * nb * nb * sizeof(double2));
  if (!VXV || !Wb || !Sm) return EIG_ERR_NOMEM;
  auto buf = [&](int64_t k) { return VXV + (k & 1) * vxv_elems; };
  {
    double2 *b0 = buf(0);
    EIG_TRY(panel_qr(c, A + nb, lda, n - nb, nb, tau, T, b0, b0 + 2 * ldw * nb, ldw, c.stream));
  }
  for (int64_t k = 0; k < K; k++) {
    const int64_t i = k * nb, r0 = i + nb, s = n - r0;
    double2 *A22 = A + r0 + r0 * lda;
    double2 *Tk = T + k * nb * nb;
    double2 *V = buf(k), *X = buf(k) + ldw * nb;
    if (k > 0) EIG_TRY(c.check(cudaStreamWaitEvent(c.stream, c.ev_join, 0), "wait panel"));
    Zgemm g;
    // a3: W = A22 V T
    g = Zgemm();
    g.herm_a = 1; g.M = s; g.N = nb; g.K = s; g.A = A22; g.lda = lda; g.B = V; g.ldb = ldw; g.C = Wb; g.ldc = ldw;
    EIG_TRY(zgemm(c, g));
    g = Zgemm();
    g.M = s; g.N = nb; g.K = nb; g.A = Wb; g.lda = ldw; g.B = Tk; g.ldb = nb; g.C = X; g.ldc = ldw;
    EIG_TRY(zgemm(c, g));
    // a4: M = T^H (V^H W);  X = W - 1/2 V M
    g = Zgemm();
    g.opa = OP_C; g.M = nb; g.N = nb; g.K = s; g.A = V; g.lda = ldw; g.B = X; g.ldb = ldw; g.C = Sm; g.ldc = nb;
    EIG_TRY(zgemm(c, g));
    g = Zgemm();
    g.opa = OP_C; g.M = nb; g.N = nb; g.K = nb; g.A = Tk; g.lda = nb; g.B = Sm; g.ldb = nb; g.C = Sm + nb * nb;
    g.ldc = nb;
    EIG_TRY(zgemm(c, g));
    g = Zgemm();
    g.M = s; g.N = nb; g.K = nb; g.A = V; g.lda = ldw; g.B = Sm + nb * nb; g.ldb = nb; g.C = X; g.ldc = ldw;
    g.alpha = -0.5; g.beta = 1.0;
    EIG_TRY(zgemm(c, g));
    // a5: A22 -= [V X] [X V]^H   (lower triangle)
    if (k + 1 < K) {
      // (i) the next panel's columns (rectangular s x nb, lower part)
      g = Zgemm();
      g.opb = OP_C; g.lower_c = 2; g.M = s; g.N = nb; g.K = 2 * nb; g.A = V; g.lda = ldw; g.B = X; g.ldb = ldw;
      g.C = A22; g.ldc = lda; g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
      // panel k+1 on the side stream, concurrent with (ii)
      EIG_TRY(c.check(cudaEventRecord(c.ev_fork, c.stream), "fork"));
      EIG_TRY(c.check(cudaStreamWaitEvent(c.side, c.ev_fork, 0), "fork wait"));
      double2 *bn = buf(k + 1);
      EIG_TRY(panel_qr(c, A + r0 + nb + r0 * lda, lda, s - nb, nb, tau + (k + 1) * nb, T + (k + 1) * nb * nb, bn,
                       bn + 2 * ldw * nb, ldw, c.side));
      EIG_TRY(c.check(cudaEventRecord(c.ev_join, c.side), "join"));
      // (ii) the remaining trailing lower triangle
      g = Zgemm();
      g.opb = OP_C; g.lower_c = 1; g.M = s - nb; g.N = s - nb; g.K = 2 * nb; g.A = V + nb; g.lda = ldw;
      g.B = X + nb; g.ldb = ldw; g.C = A22 + nb + nb * lda; g.ldc = lda; g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
    } else {
      g = Zgemm();
      g.opb = OP_C; g.lower_c = 1; g.M = s; g.N = s; g.K = 2 * nb; g.A = V; g.lda = ldw; g.B = X; g.ldb = ldw;
      g.C = A22; g.ldc = lda; g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
    }
  }
  return 0;
}

// ------------------------------------------------------------------ Q1
// E <- Q1 E with Q1 = Q^(0) ... Q^(K-1), Q^(k) = I - V_k T_k V_k^H.
// Panels are aggregated ga at a time (last group first):
//   Q^(k0)...Q^(k0+ga-1) = I - V T V^H,  V = [V_k0 ... V_k0+ga-1] (unit lower
//   trapezoidal from row (k0+1)nb),  T = [[T_a, -T_a (V_a^H V_b) T_b], [0, T_b]]
// merged pairwise from the per-panel T_k with the Gram matrix V^H V, so each
// pass over E is three GEMMs with K = ga*nb instead of nb.
// The preparation of a group (explicit V, Gram matrix, merged T) runs on the
// side stream one group ahead of the three big GEMMs on the main stream
// (double-buffered by group parity), so only the GEMMs are on the critical path.
int apply_q1_run(Ctx &c, int64_t n, const double2 *A, int64_t lda, const double2 *T, double2 *E, int64_t lde,
                        int64_t m) {
  const int nb = c.nb;
  const int64_t K = num_panels(n, nb);
  if (K == 0 || m <= 0) return 0;
  // panels aggregated per pass over E (K of the two big GEMMs); EIG_Q1_KW tunes it
  static const int kw_env = [] {
    const char *e = getenv("EIG_Q1_KW");
    return e ? atoi(e) : 256;
  }();
  const int ga_max = std::max(1, kw_env / nb);
  const int kw = ga_max * nb;                       // aggregated width
  const int64_t ldv = n - nb;
  double2 *Vb0 = (double2 *)c.ws(WS_V, (size_t)4 * ldv * kw * sizeof(double2));   // V and V T, per parity
  double2 *Y = (double2 *)c.ws(WS_Y, (size_t)kw * m * sizeof(double2));
  double2 *Tg0 = (double2 *)c.ws(WS_TAGG, (size_t)6 * kw * kw * sizeof(double2));
  if (!Vb0 || !Y || !Tg0) return EIG_ERR_NOMEM;
  const int64_t ngroups = (K + ga_max - 1) / ga_max;
  auto Vbuf = [&](int par) { return Vb0 + (size_t)par * ldv * kw; };
  auto VTbuf = [&](int par) { return Vb0 + (size_t)(2 + par) * ldv * kw; };
  auto Tbuf = [&](int par) { return Tg0 + (size_t)par * 3 * kw * kw; };
  // preparation of group gi into buffer par, on the side stream
  auto prep = [&](int64_t gi, int par) -> int {
    const int64_t k0 = gi * ga_max;
    const int ga = (int)std::min<int64_t>(ga_max, K - k0);
    const int w = ga * nb;
    const int64_t r0 = (k0 + 1) * nb, s = n - r0;
    double2 *Vb = Vbuf(par), *Tg = Tbuf(par);
    double2 *Gm = Tg + (size_t)kw * kw, *Tmp = Gm + (size_t)kw * kw;
    EIG_TRY(c.check(cudaStreamWaitEvent(c.side, c.ev_q1[2 + par], 0), "q1 buffer free"));
    const cudaStream_t keep = c.stream;
    c.stream = c.side;
    int rc = extract_v(c, A + r0 + k0 * nb * lda, lda, s, w, Vb, ldv);
    if (!rc && ga > 1) {
      // aggregated T: diagonal blocks T_k, off-diagonal blocks merged pairwise
      rc = c.check(cudaMemsetAsync(Tg, 0, (size_t)w * w * sizeof(double2), c.stream), "memset T");
      for (int p = 0; p < ga && !rc; p++)
        rc = c.check(cudaMemcpy2DAsync(Tg + (size_t)p * nb * w + p * nb, w * sizeof(double2), T + (k0 + p) * nb * nb,
                                       nb * sizeof(double2), nb * sizeof(double2), nb, cudaMemcpyDeviceToDevice,
                                       c.stream), "copy T");
      Zgemm g;   // Gram = V^H V
      g.opa = OP_C; g.M = w; g.N = w; g.K = s; g.A = Vb; g.lda = ldv; g.B = Vb; g.ldb = ldv; g.C = Gm; g.ldc = w;
      if (!rc) rc = zgemm(c, g);
      for (int span = nb; span < w && !rc; span *= 2)
        for (int p0 = 0; p0 + span < w && !rc; p0 += 2 * span) {
          const int p1 = p0 + span, p2 = std::min(w, p1 + span);
          // Tmp = T[p0:p1, p0:p1] G[p0:p1, p1:p2];  T[p0:p1, p1:p2] = -Tmp T[p1:p2, p1:p2]
          g = Zgemm();
          g.M = span; g.N = p2 - p1; g.K = span; g.A = Tg + (size_t)p0 * w + p0; g.lda = w;
          g.B = Gm + (size_t)p1 * w + p0; g.ldb = w; g.C = Tmp; g.ldc = w;
          rc = zgemm(c, g);
          if (rc) break;
          g = Zgemm();
          g.M = span; g.N = p2 - p1; g.K = p2 - p1; g.A = Tmp; g.lda = w; g.B = Tg + (size_t)p1 * w + p1; g.ldb = w;
          g.C = Tg + (size_t)p1 * w + p0; g.ldc = w; g.alpha = -1.0;
          rc = zgemm(c, g);
        }
    }
    if (!rc) {   // V T (so that the main stream's update is one GEMM: E -= (V T) (V^H E))
      Zgemm g;
      g.M = s; g.N = w; g.K = w; g.A = Vb; g.lda = ldv; g.B = ga > 1 ? Tg : T + k0 * nb * nb; g.ldb = ga > 1 ? w : nb;
      g.C = VTbuf(par); g.ldc = ldv;
      rc = zgemm(c, g);
    }
    c.stream = keep;
    if (rc) return rc;
    return c.check(cudaEventRecord(c.ev_q1[par], c.side), "q1 prep done");
  };
  // the side stream starts after everything already queued (he2hb's A and T)
  EIG_TRY(c.check(cudaEventRecord(c.ev_fork, c.stream), "q1 fork"));
  EIG_TRY(c.check(cudaStreamWaitEvent(c.side, c.ev_fork, 0), "q1 fork wait"));
  EIG_TRY(prep(ngroups - 1, (int)((ngroups - 1) & 1)));
  for (int64_t gi = ngroups - 1; gi >= 0; gi--) {
    const int par = (int)(gi & 1);
    if (gi > 0) EIG_TRY(prep(gi - 1, par ^ 1));   // overlaps this group's GEMMs
    const int64_t k0 = gi * ga_max;
    const int ga = (int)std::min<int64_t>(ga_max, K - k0);
    const int w = ga * nb;
    const int64_t r0 = (k0 + 1) * nb, s = n - r0;
    const double2 *Vb = Vbuf(par);
    EIG_TRY(c.check(cudaStreamWaitEvent(c.stream, c.ev_q1[par], 0), "q1 prep wait"));
    Zgemm g;   // Y = V^H E
    g.opa = OP_C; g.M = w; g.N = m; g.K = s; g.A = Vb; g.lda = ldv; g.B = E + r0; g.ldb = lde; g.C = Y; g.ldc = w;
    g.split_n = kBtSplitN;
    EIG_TRY(zgemm(c, g));
    g = Zgemm();   // E -= (V T) Y
    g.M = s; g.N = m; g.K = w; g.A = VTbuf(par); g.lda = ldv; g.B = Y; g.ldb = w; g.C = E + r0; g.ldc = lde;
    g.alpha = -1.0; g.beta = 1.0; g.split_n = kBtSplitN;
    EIG_TRY(zgemm(c, g));
    EIG_TRY(c.check(cudaEventRecord(c.ev_q1[2 + par], c.stream), "q1 gemms done"));
  }
  return 0;
}

// ------------------------------------------------------------------ trsm
// E <- L^-H E, left-looking and two-level: outer 256-row blocks take
// the bulk of the flops in one GEMM each (M = 256, K = n - I1), the 256 x 256
// diagonal block is solved with 64-row steps using precomputed inverses of
// the 64 x 64 diagonal blocks of L.
// hostE (optional, pinned host, leading dimension ldh): every 256-row block of E
// is copied back on the transfer stream as soon as it is final (bottom block
// first), overlapping the copy with the remaining blocks.
int trsm_lh_run(Ctx &c, int64_t n, const double2 *L, int64_t ldl, double2 *E, int64_t lde, int64_t m,
                double2 *hostE, int64_t ldh) {
  if (n <= 0 || m <= 0) return 0;
  const int bs = 64, BS = 256;
  const int64_t nblk = (n + bs - 1) / bs;
  double2 *Linv = (double2 *)c.ws(WS_LINV, (size_t)nblk * bs * bs * sizeof(double2));
  if (!Linv) return EIG_ERR_NOMEM;
  EIG_TRY(trinv_blocks(c, n, bs, L, ldl, Linv));
  for (int64_t I = (n + BS - 1) / BS - 1; I >= 0; I--) {
    const int64_t I0 = I * BS, I1 = std::min<int64_t>(n, I0 + BS);
    Zgemm g;
    if (I1 < n) {
      g.opa = OP_C; g.M = I1 - I0; g.N = m; g.K = n - I1; g.A = L + I1 + I0 * ldl; g.lda = ldl; g.B = E + I1;
      g.ldb = lde; g.C = E + I0; g.ldc = lde; g.alpha = -1.0; g.beta = 1.0; g.split_n = kBtSplitN;
      EIG_TRY(zgemm(c, g));
    }
    for (int64_t i0 = I0 + ((I1 - I0 - 1) / bs) * bs; i0 >= I0; i0 -= bs) {
      const int64_t i1 = std::min<int64_t>(I1, i0 + bs), bi = i1 - i0;
      if (i1 < I1) {
        g = Zgemm();
        g.opa = OP_C; g.M = bi; g.N = m; g.K = I1 - i1; g.A = L + i1 + i0 * ldl; g.lda = ldl; g.B = E + i1;
        g.ldb = lde; g.C = E + i0; g.ldc = lde; g.alpha = -1.0; g.beta = 1.0; g.split_n = kBtSplitN;
        EIG_TRY(zgemm(c, g));
      }
      // in place: one 64-row M tile per column tile, no split-K -> every CTA reads
      // its whole K range before its epilogue writes
      g = Zgemm();
      g.opa = OP_C; g.M = bi; g.N = m; g.K = bi; g.A = Linv + (i0 / bs) * bs * bs; g.lda = bs; g.B = E + i0;
      g.ldb = lde; g.C = E + i0; g.ldc = lde; g.alpha = 1.0; g.beta = 0.0; g.splitk = 1;
      EIG_TRY(zgemm(c, g));
    }
    if (hostE) {   // rows I0..I1-1 are final
      EIG_TRY(c.check(cudaEventRecord(c.ev_blk, c.stream), "blk event"));
      EIG_TRY(c.check(cudaStreamWaitEvent(c.xfer, c.ev_blk, 0), "blk wait"));
      EIG_TRY(c.check(cudaMemcpy2DAsync(hostE + I0, ldh * sizeof(double2), E + I0, lde * sizeof(double2),
                                        (I1 - I0) * sizeof(double2), m, cudaMemcpyDeviceToHost, c.xfer),
                      "D2H E block"));
    }
  }
  return 0;
}

// E <- L^-1 E (forward substitution, left, lower, no transpose), two-level like trsm_lh.
static int trsm_ln_run(Ctx &c, int64_t n, const double2 *L, int64_t ldl, double2 *E, int64_t lde, int64_t m) {
  if (n <= 0 || m <= 0) return 0;
  const int bs = 64, BS = 256;
  const int64_t nblk = (n + bs - 1) / bs;
  double2 *Linv = (double2 *)c.ws(WS_LINV, (size_t)nblk * bs * bs * sizeof(double2));
  if (!Linv) return EIG_ERR_NOMEM;
  EIG_TRY(trinv_blocks(c, n, bs, L, ldl, Linv));
  for (int64_t I0 = 0; I0 < n; I0 += BS) {
    const int64_t I1 = std::min<int64_t>(n, I0 + BS);
    Zgemm g;
    if (I0 > 0) {
      g.M = I1 - I0; g.N = m; g.K = I0; g.A = L + I0; g.lda = ldl; g.B = E; g.ldb = lde; g.C = E + I0; g.ldc = lde;
      g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
    }
    for (int64_t i0 = I0; i0 < I1; i0 += bs) {
      const int64_t i1 = std::min<int64_t>(I1, i0 + bs), bi = i1 - i0;
      if (i0 > I0) {
        g = Zgemm();
        g.M = bi; g.N = m; g.K = i0 - I0; g.A = L + i0 + I0 * ldl; g.lda = ldl; g.B = E + I0; g.ldb = lde;
        g.C = E + i0; g.ldc = lde; g.alpha = -1.0; g.beta = 1.0;
        EIG_TRY(zgemm(c, g));
      }
      g = Zgemm();   // in place: single 64-row M tile, no split-K
      g.M = bi; g.N = m; g.K = bi; g.A = Linv + (i0 / bs) * bs * bs; g.lda = bs; g.B = E + i0; g.ldb = lde;
      g.C = E + i0; g.ldc = lde; g.splitk = 1;
      EIG_TRY(zgemm(c, g));
    }
  }
  return 0;
}

// Z = X L^-H on the lower trapezoid only (rows >= the column block): column
// block J of Z needs, besides X's own lower part, only Z's columns left of J
// on the same rows, i.e. lower entries again.  Left-looking over 256-column
// blocks, 64-column steps with the precomputed inverses of L's 64 x 64
// diagonal blocks; in place (X's strictly upper blocks are never touched).
static int trsm_rlh_lower(Ctx &c, int64_t n, const double2 *L, int64_t ldl, double2 *X, int64_t ldx) {
  if (n <= 0) return 0;
  const int bs = 64, BS = 256;
  const int64_t nblk = (n + bs - 1) / bs;
  double2 *Linv = (double2 *)c.ws(WS_LINV, (size_t)nblk * bs * bs * sizeof(double2));
  if (!Linv) return EIG_ERR_NOMEM;
  EIG_TRY(trinv_blocks(c, n, bs, L, ldl, Linv));
  for (int64_t J0 = 0; J0 < n; J0 += BS) {
    const int64_t J1 = std::min<int64_t>(n, J0 + BS);
    Zgemm g;
    if (J0 > 0) {   // X[J0:, J0:J1] -= Z[J0:, 0:J0] L[J0:J1, 0:J0]^H
      g.opb = OP_C; g.M = n - J0; g.N = J1 - J0; g.K = J0; g.A = X + J0; g.lda = ldx; g.B = L + J0; g.ldb = ldl;
      g.C = X + J0 + J0 * ldx; g.ldc = ldx; g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
    }
    for (int64_t j0 = J0; j0 < J1; j0 += bs) {
      const int64_t j1 = std::min<int64_t>(J1, j0 + bs), bj = j1 - j0;
      if (j0 > J0) {   // X[j0:, j0:j1] -= Z[j0:, J0:j0] L[j0:j1, J0:j0]^H
        g = Zgemm();
        g.opb = OP_C; g.M = n - j0; g.N = bj; g.K = j0 - J0; g.A = X + j0 + J0 * ldx; g.lda = ldx;
        g.B = L + j0 + J0 * ldl; g.ldb = ldl; g.C = X + j0 + j0 * ldx; g.ldc = ldx; g.alpha = -1.0; g.beta = 1.0;
        EIG_TRY(zgemm(c, g));
      }
      // in place: Z[j0:, j0:j1] = X[j0:, j0:j1] Linv_jj^H (one 64-col N tile, no split-K)
      g = Zgemm();
      g.opb = OP_C; g.M = n - j0; g.N = bj; g.K = bj; g.A = X + j0 + j0 * ldx; g.lda = ldx;
      g.B = Linv + (j0 / bs) * bs * bs; g.ldb = bs; g.C = X + j0 + j0 * ldx; g.ldc = ldx; g.splitk = 1;
      g.whole_n = true;
      EIG_TRY(zgemm(c, g));
    }
  }
  return 0;
}

// A' = L^-1 A L^-H (A' Hermitian), Algorithm 1 step 2: X = L^-1 A in
// full, then only the lower trapezoid of X L^-H (a third of the first solve's
// flops).
int hegst_run(Ctx &c, int64_t n, double2 *A, int64_t lda, const double2 *L, int64_t ldl) {
  if (n <= 0) return 0;
  EIG_TRY(herm_full(c, n, A, lda));
  EIG_TRY(trsm_ln_run(c, n, L, ldl, A, lda, n));        // X = L^-1 A
  EIG_TRY(trsm_rlh_lower(c, n, L, ldl, A, lda));        // A' = X L^-H (lower)
  return real_diag(c, n, A, lda);
}

// ------------------------------------------------------------------ Q2
// Plan tables of the grouped Q2 blocks (reading R7), built on the device on
// c.stream and cached in the handle for (n, nb, g).
static int q2_plan(Ctx &c, int64_t n, Q2Plan &p) {
  if (c.q2_n == n && c.q2_plan_nb == c.nb && c.q2_plan_g == c.q2g && c.q2_plan.d_group_first_block == c.buf[WS_Q2PLAN]) {
    p = c.q2_plan;
    return 0;
  }
  const int nb = c.nb, g = c.q2g;
  p.n = n;
  p.nb = nb;
  p.g = g;
  p.ngroups = (n - 1 + g - 1) / g;
  int64_t tot = 0;
  for (int64_t gi = 0; gi < p.ngroups; gi++) {
    const int64_t i0 = gi * g;
    tot += (i0 > n - 2) ? 0 : (n - 2 - i0) / nb + 1;
  }
  p.nblocks = tot;
  p.J = (n >= 2) ? (n - 2) / nb + 1 : 0;   // steps j with 1 + j nb <= n - 1
  int64_t *d = (int64_t *)c.ws(WS_Q2PLAN, (p.ngroups + 1 + p.J + 1) * sizeof(int64_t));
  if (!d) return EIG_ERR_NOMEM;
  p.d_group_first_block = d;
  p.d_off = d + p.ngroups + 1;
  EIG_TRY(plan_tables(c, n, nb, g, p.ngroups, p.J, p.d_group_first_block, p.d_off));
  c.q2_n = n;
  c.q2_plan_nb = nb;
  c.q2_plan_g = g;
  c.q2_plan = p;
  return 0;
}

int apply_q2_run(Ctx &c, int64_t n, const double2 *V2, const double2 *tau2, double2 *E, int64_t lde,
                        int64_t m) {
  if (n <= 1 || m <= 0) return 0;
  if (c.q2g < 4) return EIG_ERR_NOTIMPL;  // nb < 3: no grouped blocks
  Q2Plan p;
  EIG_TRY(q2_plan(c, n, p));
  double2 *T2 = (double2 *)c.ws(WS_T2, (size_t)p.nblocks * p.g * p.g * sizeof(double2));
  if (!T2) return EIG_ERR_NOMEM;
  EIG_TRY(q2_tfactors(c, p, V2, tau2, T2));
  return q2_apply(c, p, V2, T2, E, lde, m);
}

}  // namespace eig

using namespace eig;

struct eig_ctx {
  Ctx c;
};

static int valid(eig_handle h) { return (h != nullptr) ? 0 : EIG_ERR_STATE; }

extern "C" {

int eig_init(eig_handle *h, const eig_config *cfg) {
  if (!h) return -1;
  *h = nullptr;
  // validate the whole configuration before any device call
  if (cfg) {
    if (cfg->nb < 0 || cfg->nb > 64) return -2;
    if (cfg->nranks > 1 && !cfg->nccl_id) return -2;
    if (cfg->nranks < 0 || (cfg->nranks > 0 && (cfg->rank < 0 || cfg->rank >= cfg->nranks))) return -2;
    if (cfg->nranks <= 0 && cfg->rank != 0) return -2;
    if (cfg->n_max < 0) return -2;
  }
  eig_ctx *x = new (std::nothrow) eig_ctx();
  if (!x) return EIG_ERR_NOMEM;
  if (cfg) {
    x->c.device = cfg->device;
    x->c.stream = (cudaStream_t)cfg->stream;
    if (cfg->nb) x->c.nb = cfg->nb;
    if (cfg->q2_group) x->c.q2g = cfg->q2_group;
    x->c.rank = cfg->rank;
    x->c.nranks = std::max(1, cfg->nranks);
    x->c.coll = cfg->nccl_id != nullptr;
    x->c.n_max = cfg->n_max;
    x->c.flags = cfg->flags;
  }
  {   // 3M complex GEMMs: flag, else environment EIG_3M (0 / 1), else on
    const char *e = getenv("EIG_3M");
    x->c.use_3m = (x->c.flags & EIG_USE_3M) ? true : ((x->c.flags & EIG_NO_3M) ? false : (e ? atoi(e) > 0 : true));
  }
  if (x->c.nb < 1 || x->c.nb > 64) { delete x; return -2; }
  if (!cfg || !cfg->q2_group) x->c.q2g = std::min(32, ((x->c.nb + 1) / 4) * 4);  // g <= nb + 1, multiple of 4
  if (x->c.q2g != 0 && (x->c.q2g < 4 || x->c.q2g > 32 || x->c.q2g % 4 || x->c.q2g - 1 > x->c.nb)) {
    delete x;
    return -2;
  }
  int rc = x->c.check(cudaSetDevice(x->c.device), "cudaSetDevice");
  if (rc) { delete x; return rc; }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->c.device);
  if (sms > 0) x->c.num_sms = sms;
  int lo_prio = 0, hi_prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
  rc = x->c.check(cudaStreamCreateWithPriority(&x->c.side, cudaStreamNonBlocking, hi_prio), "side stream");
  if (!rc) rc = x->c.check(cudaEventCreateWithFlags(&x->c.ev_fork, cudaEventDisableTiming), "event");
  if (!rc) rc = x->c.check(cudaEventCreateWithFlags(&x->c.ev_join, cudaEventDisableTiming), "event");
  if (!rc) rc = x->c.check(cudaStreamCreateWithFlags(&x->c.xfer, cudaStreamNonBlocking), "xfer stream");
  if (!rc) rc = x->c.check(cudaEventCreateWithFlags(&x->c.ev_xfer, cudaEventDisableTiming), "event");
  if (!rc) rc = x->c.check(cudaEventCreateWithFlags(&x->c.ev_blk, cudaEventDisableTiming), "event");
  for (int i = 0; i < 4 && !rc; i++)
    rc = x->c.check(cudaEventCreateWithFlags(&x->c.ev_q1[i], cudaEventDisableTiming), "event");
  for (int i = 0; i < EIG_NSTAGES && !rc; i++) {
    rc = x->c.check(cudaEventCreate(&x->c.st_beg[i]), "event");
    if (!rc) rc = x->c.check(cudaEventCreate(&x->c.st_end[i]), "event");
  }
  if (rc) { eig_finalize(x); return rc; }
  if (x->c.coll) {
    rc = comm_init(x->c, cfg->nccl_id);
    if (rc) { eig_finalize(x); return rc; }
  }
  void *bar = x->c.ws(WS_BARRIER, 64);
  if (!bar) { eig_finalize(x); return EIG_ERR_NOMEM; }
  rc = x->c.check(cudaMemset(bar, 0, 64), "barrier init");
  if (rc) { eig_finalize(x); return rc; }
  if (x->c.coll && x->c.n_max > 0) {
    rc = comm_reserve(x->c, x->c.n_max);
    if (rc) { eig_finalize(x); return rc; }
  }
  if (getenv("EIG_Q2_PROFILE")) {
    x->c.q2_prof = (unsigned long long *)x->c.ws(WS_Q2PROF, 256);
    if (x->c.q2_prof) cudaMemset(x->c.q2_prof, 0, 256);
  }
  *h = x;
  return 0;
}

int eig_debug_q2_profile(eig_handle h, unsigned long long *out16) {
  if (!h) return EIG_ERR_STATE;
  if (!h->c.q2_prof) return EIG_ERR_NOTIMPL;
  return h->c.check(cudaMemcpy(out16, h->c.q2_prof, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "prof");
}

int eig_finalize(eig_handle h) {
  if (!h) return EIG_ERR_STATE;
  cudaSetDevice(h->c.device);
  cudaStreamSynchronize(h->c.stream);
  comm_destroy(h->c);
  for (int i = 0; i < EIG_NSTAGES; i++) {
    if (h->c.st_beg[i]) cudaEventDestroy(h->c.st_beg[i]);
    if (h->c.st_end[i]) cudaEventDestroy(h->c.st_end[i]);
  }
  if (h->c.side) { cudaStreamSynchronize(h->c.side); cudaStreamDestroy(h->c.side); }
  if (h->c.ev_fork) cudaEventDestroy(h->c.ev_fork);
  if (h->c.ev_join) cudaEventDestroy(h->c.ev_join);
  if (h->c.xfer) { cudaStreamSynchronize(h->c.xfer); cudaStreamDestroy(h->c.xfer); }
  if (h->c.ev_xfer) cudaEventDestroy(h->c.ev_xfer);
  if (h->c.ev_blk) cudaEventDestroy(h->c.ev_blk);
  for (int i = 0; i < 4; i++)
    if (h->c.ev_q1[i]) cudaEventDestroy(h->c.ev_q1[i]);
  for (int i = 0; i < WS_COUNT; i++) {
    if (h->c.buf[i]) cudaFree(h->c.buf[i]);
  }
  delete h;
  return 0;
}

const char *eig_strerror(int code) {
  switch (code) {
    case 0: return "success";
    case EIG_ERR_CUDA: return "CUDA error";
    case EIG_ERR_NCCL: return "NCCL error";
    case EIG_ERR_NOMEM: return "device allocation failed";
    case EIG_ERR_STATE: return "bad handle or state";
    case EIG_ERR_NOTIMPL: return "not implemented in this build";
    default: return code < 0 ? "illegal argument" : "matrix B not positive definite / stage failure";
  }
}

const char *eig_last_cuda_error(eig_handle h) { return h ? h->c.last_err.c_str() : "no handle"; }
int64_t eig_launch_count(eig_handle h) { return h ? h->c.launches : -1; }
int eig_sync(eig_handle h) {
  if (!h) return EIG_ERR_STATE;
  return h->c.check(cudaStreamSynchronize(h->c.stream), "cudaStreamSynchronize");
}
int64_t eig_num_panels(int64_t n, int nb) { return num_panels(n, nb); }
int64_t eig_v2_slots(int64_t n, int nb) { return v2_slots(n, nb); }

int eig_he2hb(eig_handle h, int64_t n, void *A, int64_t lda, void *tau, void *T) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (!A && n > 0) return -3;
  if (lda < std::max<int64_t>(1, n)) return -4;
  if (num_panels(n, h->c.nb) > 0 && (!tau || !T)) return !tau ? -5 : -6;
  cudaSetDevice(h->c.device);
  return he2hb_run(h->c, n, (double2 *)A, lda, (double2 *)tau, (double2 *)T);
}

int eig_he2hb_sim(eig_handle h, int64_t n, int nranks, void *A, int64_t lda, void *tau, void *T) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (nranks < 1) return -3;
  if (!A && n > 0) return -4;
  if (lda < std::max<int64_t>(1, n)) return -5;
  if (num_panels(n, h->c.nb) > 0 && (!tau || !T)) return !tau ? -6 : -7;
  cudaSetDevice(h->c.device);
  return he2hb_sim(h->c, n, nranks, (double2 *)A, lda, (double2 *)tau, (double2 *)T);
}

int eig_apply_q1(eig_handle h, int64_t n, const void *A, int64_t lda, const void *T, void *E, int64_t lde, int64_t m) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (lda < std::max<int64_t>(1, n)) return -4;
  if (lde < std::max<int64_t>(1, n)) return -7;
  if (m < 0) return -8;
  cudaSetDevice(h->c.device);
  return apply_q1_run(h->c, n, (const double2 *)A, lda, (const double2 *)T, (double2 *)E, lde, m);
}

int eig_apply_q2(eig_handle h, int64_t n, const void *V2, const void *tau2, const double *Z, int64_t ldz, void *E,
                 int64_t lde, int64_t m) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (Z && ldz < std::max<int64_t>(1, n)) return -6;
  if (lde < std::max<int64_t>(1, n)) return -8;
  if (m < 0) return -9;
  cudaSetDevice(h->c.device);
  if (Z) EIG_TRY(complexify(h->c, n, m, Z, ldz, (double2 *)E, lde));
  return apply_q2_run(h->c, n, (const double2 *)V2, (const double2 *)tau2, (double2 *)E, lde, m);
}

int eig_trsm_lh(eig_handle h, int64_t n, const void *L, int64_t ldl, void *E, int64_t lde, int64_t m) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (ldl < std::max<int64_t>(1, n)) return -4;
  if (lde < std::max<int64_t>(1, n)) return -6;
  if (m < 0) return -7;
  cudaSetDevice(h->c.device);
  return trsm_lh_run(h->c, n, (const double2 *)L, ldl, (double2 *)E, lde, m);
}

int eig_hb2st(eig_handle h, int64_t n, const void *A, int64_t lda, double *d, double *e, void *V2, void *tau2) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (lda < std::max<int64_t>(1, n)) return -4;
  cudaSetDevice(h->c.device);
  return hb2st_run(h->c, n, (const double2 *)A, lda, d, e, (double2 *)V2, (double2 *)tau2);
}

}  // extern "C"

namespace eig {
int hb2st_run(Ctx &c, int64_t n, const double2 *A, int64_t lda, double *d, double *e, double2 *V2, double2 *tau2) {
  if (n <= 1) {
    if (n == 1) EIG_TRY(c.check(cudaMemcpy2DAsync(d, sizeof(double), A, sizeof(double2), sizeof(double), 1,
                                                  cudaMemcpyDeviceToDevice, c.stream), "d"));
    return 0;
  }
  const int64_t J = (n - 2) / c.nb + 1;   // steps j with 1 + j nb <= n - 1
  int64_t *d_off = (int64_t *)c.ws(WS_HBOFF, J * sizeof(int64_t));
  if (!d_off) return EIG_ERR_NOMEM;
  EIG_TRY(plan_tables(c, n, c.nb, 1, 0, J, nullptr, d_off));   // V2 slot offsets, on the stream
  return hb2st(c, n, c.nb, A, lda, d, e, V2, tau2, d_off);
}
}  // namespace eig

extern "C" {

int eig_stedc(eig_handle h, int64_t n, const double *d, const double *e, int64_t il, int64_t iu, double *w, double *Z,
              int64_t ldz) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (n > 0 && (il < 1 || iu > n || il > iu)) return -5;
  if (ldz < std::max<int64_t>(1, n)) return -9;
  cudaSetDevice(h->c.device);
  return stedc(h->c, n, d, e, il, iu, w, Z, ldz);
}

int eig_zgemm(eig_handle h, char opa, char opb, int64_t M, int64_t N, int64_t K, double alpha, const void *A,
              int64_t lda, const void *B, int64_t ldb, double beta, void *C, int64_t ldc, int herm_a, int lower_c) {
  EIG_TRY(valid(h));
  Zgemm g;
  if (opa != 'N' && opa != 'C') return -2;
  if (opb != 'N' && opb != 'C') return -3;
  if (M < 0) return -4;
  if (N < 0) return -5;
  if (K < 0) return -6;
  g.opa = (opa == 'C') ? OP_C : OP_N;
  g.opb = (opb == 'C') ? OP_C : OP_N;
  g.M = M; g.N = N; g.K = K; g.alpha = alpha; g.beta = beta;
  g.A = (const double2 *)A; g.lda = lda; g.B = (const double2 *)B; g.ldb = ldb; g.C = (double2 *)C; g.ldc = ldc;
  g.herm_a = herm_a; g.lower_c = lower_c;
  cudaSetDevice(h->c.device);
  return zgemm(h->c, g);
}

int eig_hotpath(eig_handle h, int64_t n, void *A, int64_t lda, void *tau1, void *T1, const void *V2,
                const void *tau2, const void *L, int64_t ldl, const double *Z, int64_t ldz, void *E, int64_t lde,
                int64_t m, unsigned flags) {
  EIG_TRY(valid(h));
  Ctx &c = h->c;
  if (n < 1) return -2;
  if (c.coll) {
    if (flags & EIG_HOST_BUFFERS) return EIG_ERR_NOTIMPL;
    if (ldz < n) return -13;
    if (lde < n) return -15;
    if (m < 0 || m > n) return -16;
    if (c.n_max > 0 && n > c.n_max) return EIG_ERR_STATE;
    cudaSetDevice(c.device);
    return coll_hotpath(c, n, (double2 *)A, lda, (double2 *)tau1, (double2 *)T1, (const double2 *)V2,
                        (const double2 *)tau2, (const double2 *)L, ldl, Z, ldz, (double2 *)E, lde, m, flags);
  }
  if (lda < n) return -4;
  if (ldl < n) return -11;
  if (ldz < n) return -13;
  if (lde < n) return -15;
  if (m < 0 || m > n) return -16;
  if (c.n_max > 0 && n > c.n_max) return EIG_ERR_STATE;
  cudaSetDevice(c.device);
  c.stat_reset();
  c.st.m = m;
  c.st.col_hi = m;
  EIG_TRY(c.stat_begin(EIG_ST_TOTAL));
  const int nb = c.nb;
  const int64_t K = num_panels(n, nb), slots = v2_slots(n, nb);
  const bool host = flags & EIG_HOST_BUFFERS;
  double2 *dA = (double2 *)A, *dT1 = (double2 *)T1, *dtau1 = (double2 *)tau1, *dE = (double2 *)E;
  const double2 *dV2 = (const double2 *)V2, *dtau2 = (const double2 *)tau2, *dL = (const double2 *)L;
  const double *dZ = Z;
  int64_t dlda = lda, dldl = ldl, dldz = ldz, dlde = lde;
  if (host) {
    // device staging in library workspace, packed leading dimensions
    dA = (double2 *)c.ws(WS_HOST_A, (size_t)n * n * sizeof(double2));
    double2 *v2 = (double2 *)c.ws(WS_HOST_V2, (size_t)std::max<int64_t>(slots, 1) * nb * sizeof(double2));
    double2 *t2 = (double2 *)c.ws(WS_HOST_TAU2, (size_t)std::max<int64_t>(slots, 1) * sizeof(double2));
    double2 *l = (double2 *)c.ws(WS_HOST_L, (size_t)n * n * sizeof(double2));
    double *z = (double *)c.ws(WS_HOST_Z, (size_t)n * std::max<int64_t>(m, 1) * sizeof(double));
    dE = (double2 *)c.ws(WS_HOST_E, (size_t)n * std::max<int64_t>(m, 1) * sizeof(double2));
    dtau1 = (double2 *)c.ws(WS_HOST_TAU1, (size_t)std::max<int64_t>(K, 1) * nb * sizeof(double2));
    dT1 = (double2 *)c.ws(WS_HOST_T1, (size_t)std::max<int64_t>(K, 1) * nb * nb * sizeof(double2));
    if (!dA || !v2 || !t2 || !l || !z || !dE || !dtau1 || !dT1) return EIG_ERR_NOMEM;
    if ((flags & EIG_SKIP_HE2HB) && !(flags & EIG_SKIP_BT) && K > 0) {
      // back-transform only: the caller's he2hb T factors are an input
      if (!T1) return -6;
      EIG_TRY(c.check(cudaMemcpyAsync(dT1, T1, (size_t)K * nb * nb * sizeof(double2), cudaMemcpyHostToDevice,
                                      c.stream), "H2D T1"));
    }
    // only the lower triangle of A is referenced: upload it in 256-column blocks
    for (int64_t j0 = 0; j0 < n; j0 += 256) {
      const int64_t w = std::min<int64_t>(256, n - j0);
      EIG_TRY(c.check(cudaMemcpy2DAsync(dA + j0 + j0 * n, n * sizeof(double2), (const double2 *)A + j0 + j0 * lda,
                                        lda * sizeof(double2), (n - j0) * sizeof(double2), w, cudaMemcpyHostToDevice,
                                        c.stream), "H2D A"));
    }
    if (!(flags & EIG_SKIP_BT)) {
      // the back-transform inputs travel on the transfer stream while he2hb runs
      EIG_TRY(c.check(cudaEventRecord(c.ev_xfer, c.stream), "xfer fork"));
      EIG_TRY(c.check(cudaStreamWaitEvent(c.xfer, c.ev_xfer, 0), "xfer fork wait"));
      EIG_TRY(c.check(cudaMemcpyAsync(v2, V2, (size_t)slots * nb * sizeof(double2), cudaMemcpyHostToDevice, c.xfer),
                      "H2D V2"));
      EIG_TRY(c.check(cudaMemcpyAsync(t2, tau2, (size_t)slots * sizeof(double2), cudaMemcpyHostToDevice, c.xfer),
                      "H2D tau2"));
      if (m > 0)
        EIG_TRY(c.check(cudaMemcpy2DAsync(z, n * sizeof(double), Z, ldz * sizeof(double), n * sizeof(double), m,
                                          cudaMemcpyHostToDevice, c.xfer), "H2D Z"));
      for (int64_t j0 = 0; j0 < n; j0 += 256) {   // lower triangle of L only
        const int64_t w = std::min<int64_t>(256, n - j0);
        EIG_TRY(c.check(cudaMemcpy2DAsync(l + j0 + j0 * n, n * sizeof(double2), (const double2 *)L + j0 + j0 * ldl,
                                          ldl * sizeof(double2), (n - j0) * sizeof(double2), w,
                                          cudaMemcpyHostToDevice, c.xfer), "H2D L"));
      }
      EIG_TRY(c.check(cudaEventRecord(c.ev_xfer, c.xfer), "xfer join"));
    }
    dV2 = v2; dtau2 = t2; dL = l; dZ = z;
    dlda = n; dldl = n; dldz = n; dlde = n;
  }
  if (!(flags & EIG_SKIP_HE2HB)) {
    EIG_TRY(c.stat_begin(EIG_ST_HE2HB));
    EIG_TRY(he2hb_run(c, n, dA, dlda, dtau1, dT1));
    EIG_TRY(c.stat_end(EIG_ST_HE2HB));
    c.st.flops[EIG_ST_HE2HB] = 16.0 / 3.0 * (double)n * n * n;
  } else if (!host && !(flags & EIG_SKIP_BT) && K > 0 && !T1) {
    return -6;
  }
  if (host && !(flags & EIG_SKIP_BT)) EIG_TRY(c.check(cudaStreamWaitEvent(c.stream, c.ev_xfer, 0), "xfer join wait"));
  if (!(flags & EIG_SKIP_BT) && m > 0) {
    // a6 complexify + Q2, a7 Q1, a8 L^-H; with host buffers each final row
    // block of E is copied back on the transfer stream while the blocks above
    // it are solved
    EIG_TRY(bt_run(c, n, dZ, dldz, dV2, dtau2, dA, dlda, dT1, dL, dldl, dE, dlde, m,
                   (host && E) ? (double2 *)E : nullptr, lde));
  }
  EIG_TRY(c.stat_end(EIG_ST_TOTAL));
  if (host) {
    // he2hb's tau / T factors to the caller's host buffers if given (queued
    // after the back-transform, which only reads them)
    if (!(flags & EIG_SKIP_HE2HB) && K > 0) {
      if (tau1)
        EIG_TRY(c.check(cudaMemcpyAsync(tau1, dtau1, (size_t)K * nb * sizeof(double2), cudaMemcpyDeviceToHost,
                                        c.stream), "D2H tau1"));
      if (T1)
        EIG_TRY(c.check(cudaMemcpyAsync(T1, dT1, (size_t)K * nb * nb * sizeof(double2), cudaMemcpyDeviceToHost,
                                        c.stream), "D2H T1"));
    }
    EIG_TRY(c.check(cudaStreamSynchronize(c.stream), "sync"));
    EIG_TRY(c.check(cudaStreamSynchronize(c.xfer), "sync xfer"));
  }
  return 0;
}

int eig_potrf(eig_handle h, int64_t n, void *B, int64_t ldb) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (ldb < std::max<int64_t>(1, n)) return -4;
  cudaSetDevice(h->c.device);
  return potrf_run(h->c, n, (double2 *)B, ldb);
}

}  // extern "C"

namespace eig {
// Cholesky with LAPACK info (synchronous: the info word is read back)
int potrf_run(Ctx &c, int64_t n, double2 *B, int64_t ldb) {
  int64_t *d_info = (int64_t *)c.ws(WS_INFO, 64);
  if (!d_info) return EIG_ERR_NOMEM;
  EIG_TRY(c.check(cudaMemsetAsync(d_info, 0, sizeof(int64_t), c.stream), "info"));
  EIG_TRY(potrf_lower(c, n, B, ldb, d_info));
  int64_t info = 0;
  EIG_TRY(c.check(cudaMemcpyAsync(&info, d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream), "info"));
  EIG_TRY(c.check(cudaStreamSynchronize(c.stream), "sync"));
  return (int)info;
}

// E = L^-H Q1 Q2 complex(Zr) on m columns (a6..a8), with stage statistics
int bt_run(Ctx &c, int64_t n, const double *Zr, int64_t ldzr, const double2 *V2, const double2 *tau2,
           const double2 *A, int64_t lda, const double2 *T1, const double2 *L, int64_t ldl, double2 *E, int64_t lde,
           int64_t m, double2 *hostE, int64_t ldh) {
  const double dn = (double)n, dm = (double)m;
  EIG_TRY(c.stat_begin(EIG_ST_BT));
  if (m > 0) {
    if (Zr) EIG_TRY(complexify(c, n, m, Zr, ldzr, E, lde));
    EIG_TRY(c.stat_begin(EIG_ST_Q2));
    if (c.q2g >= 4) EIG_TRY(apply_q2_run(c, n, V2, tau2, E, lde, m));
    else if (n > 1) return EIG_ERR_NOTIMPL;
    EIG_TRY(c.stat_end(EIG_ST_Q2));
    EIG_TRY(c.stat_begin(EIG_ST_Q1));
    EIG_TRY(apply_q1_run(c, n, A, lda, T1, E, lde, m));
    EIG_TRY(c.stat_end(EIG_ST_Q1));
    EIG_TRY(c.stat_begin(EIG_ST_TRSM));
    EIG_TRY(trsm_lh_run(c, n, L, ldl, E, lde, m, hostE, ldh));
    EIG_TRY(c.stat_end(EIG_ST_TRSM));
  }
  EIG_TRY(c.stat_end(EIG_ST_BT));
  c.st.flops[EIG_ST_Q2] = 8.0 * dn * dn * dm;
  c.st.flops[EIG_ST_Q1] = 8.0 * dn * dn * dm;
  c.st.flops[EIG_ST_TRSM] = 4.0 * dn * dn * dm;
  c.st.flops[EIG_ST_BT] = 20.0 * dn * dn * dm;
  return 0;
}
}  // namespace eig

extern "C" {

int eig_hegst(eig_handle h, int64_t n, void *A, int64_t lda, const void *L, int64_t ldl) {
  EIG_TRY(valid(h));
  if (n < 0) return -2;
  if (lda < std::max<int64_t>(1, n)) return -4;
  if (ldl < std::max<int64_t>(1, n)) return -6;
  cudaSetDevice(h->c.device);
  return hegst_run(h->c, n, (double2 *)A, lda, (const double2 *)L, ldl);
}

int eig_resolve_range(int64_t n, int range, double fraction, int64_t il_in, int64_t iu_in, int64_t *il, int64_t *iu,
                      int64_t *m) {
  if (n < 0) return -2;
  int64_t lo = il_in, hi = iu_in;
  if (range == EIG_RANGE_ALL) {
    lo = 1;
    hi = n;
  } else if (range == EIG_RANGE_FRACTION) {
    if (!(fraction > 0.0 && fraction <= 1.0)) return -8;
    lo = 1;
    hi = (int64_t)std::ceil(fraction * (double)n);
    hi = std::max<int64_t>(1, std::min<int64_t>(n, hi));
  } else if (range == EIG_RANGE_INDEX) {
    if (lo < 1 || lo > std::max<int64_t>(1, n)) return -9;
    if (hi < lo || hi > n) return -10;
  } else {
    return -7;
  }
  if (n == 0) {
    lo = 1;
    hi = 0;
  }
  if (il) *il = lo;
  if (iu) *iu = hi;
  if (m) *m = hi - lo + 1;
  return 0;
}

int eig_column_slice(int64_t m, int rank, int nranks, int64_t *lo, int64_t *hi) {
  if (m < 0) return -1;
  if (nranks < 1) return -3;
  if (rank < 0 || rank >= nranks) return -2;
  if (lo) *lo = (m * rank) / nranks;
  if (hi) *hi = (m * (rank + 1)) / nranks;
  return 0;
}

int eig_get_unique_id(void *id128) { return comm_unique_id(id128); }

int eig_last_stats(eig_handle h, struct eig_stats *out) {
  EIG_TRY(valid(h));
  if (!out) return -2;
  Ctx &c = h->c;
  cudaSetDevice(c.device);
  EIG_TRY(c.check(cudaStreamSynchronize(c.stream), "sync"));
  eig_stats st = c.st;
  for (int k = 0; k < EIG_NSTAGES; k++) {
    st.seconds[k] = 0.0;
    if (!c.st_on[k]) continue;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c.st_beg[k], c.st_end[k]) == cudaSuccess) st.seconds[k] = ms * 1e-3;
    else cudaGetLastError();
  }
  if (c.st_on[EIG_ST_TOTAL] && c.st_on[EIG_ST_BT]) {   // waiting time before this rank's back-transform
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c.st_beg[EIG_ST_TOTAL], c.st_beg[EIG_ST_BT]) == cudaSuccess)
      st.seconds[EIG_ST_WAIT] = ms * 1e-3;
    else
      cudaGetLastError();
  }
  *out = st;
  return 0;
}

int eig_solve_gen(eig_handle h, int64_t n, void *A, int64_t lda, void *B, int64_t ldb, int range, double fraction,
                  int64_t il, int64_t iu, double *w, void *Z, int64_t ldz, int64_t *m_out, struct eig_stats *stats) {
  EIG_TRY(valid(h));
  Ctx &c = h->c;
  if (n < 0) return -2;
  int64_t m = 0;
  EIG_TRY(eig_resolve_range(n, range, fraction, il, iu, &il, &iu, &m));
  if (c.n_max > 0 && n > c.n_max) return EIG_ERR_STATE;
  cudaSetDevice(c.device);
  if (c.coll) {
    const int rc = coll_solve_gen(c, n, (double2 *)A, lda, (double2 *)B, ldb, il, iu, w, (double2 *)Z, ldz);
    if (!rc && m_out) *m_out = m;
    if (!rc && stats) EIG_TRY(eig_last_stats(h, stats));
    return rc;
  }
  if (lda < std::max<int64_t>(1, n)) return -4;
  if (ldb < std::max<int64_t>(1, n)) return -6;
  if (ldz < std::max<int64_t>(1, n)) return -13;
  c.stat_reset();
  c.st.m = m;
  c.st.col_lo = 0;
  c.st.col_hi = m;
  if (n == 0) {
    if (m_out) *m_out = 0;
    if (stats) *stats = c.st;
    return 0;
  }
  const int nb = c.nb;
  const double dn = (double)n;
  EIG_TRY(c.stat_begin(EIG_ST_TOTAL));
  // step 1: B = L L^H
  EIG_TRY(c.stat_begin(EIG_ST_POTRF));
  const int rc = potrf_run(c, n, (double2 *)B, ldb);
  if (rc) return rc;
  EIG_TRY(c.stat_end(EIG_ST_POTRF));
  double2 *dA = (double2 *)A, *dL = (double2 *)B;
  // step 2: A' = L^-1 A L^-H
  EIG_TRY(c.stat_begin(EIG_ST_HEGST));
  EIG_TRY(hegst_run(c, n, dA, lda, dL, ldb));
  EIG_TRY(c.stat_end(EIG_ST_HEGST));
  // step 3: two-stage standard eigensolver
  const int64_t K = num_panels(n, nb), slots = v2_slots(n, nb);
  double2 *tau1 = (double2 *)c.ws(WS_SG_TAU1, (size_t)std::max<int64_t>(K, 1) * nb * sizeof(double2));
  double2 *T1 = (double2 *)c.ws(WS_SG_T1, (size_t)std::max<int64_t>(K, 1) * nb * nb * sizeof(double2));
  double *dd = (double *)c.ws(WS_SG_D, (size_t)n * sizeof(double));
  double *de = (double *)c.ws(WS_SG_E, (size_t)n * sizeof(double));
  double2 *V2 = (double2 *)c.ws(WS_SG_V2, (size_t)std::max<int64_t>(slots, 1) * nb * sizeof(double2));
  double2 *tau2 = (double2 *)c.ws(WS_SG_TAU2, (size_t)std::max<int64_t>(slots, 1) * sizeof(double2));
  double *Zr = (double *)c.ws(WS_SG_Z, (size_t)n * m * sizeof(double));
  if (!tau1 || !T1 || !dd || !de || !V2 || !tau2 || !Zr) return EIG_ERR_NOMEM;
  EIG_TRY(c.stat_begin(EIG_ST_HE2HB));
  EIG_TRY(he2hb_run(c, n, dA, lda, tau1, T1));
  EIG_TRY(c.stat_end(EIG_ST_HE2HB));
  EIG_TRY(c.stat_begin(EIG_ST_HB2ST));
  EIG_TRY(hb2st_run(c, n, dA, lda, dd, de, V2, tau2));
  EIG_TRY(c.stat_end(EIG_ST_HB2ST));
  EIG_TRY(c.stat_begin(EIG_ST_STEDC));
  EIG_TRY(stedc(c, n, dd, de, il, iu, w, Zr, n));
  EIG_TRY(c.stat_end(EIG_ST_STEDC));
  // step 3 back-transform and step 4: Z = L^-H Q1 Q2 complex(Zr)
  EIG_TRY(bt_run(c, n, Zr, n, V2, tau2, dA, lda, T1, dL, ldb, (double2 *)Z, ldz, m));
  EIG_TRY(c.stat_end(EIG_ST_TOTAL));
  c.st.flops[EIG_ST_POTRF] = 4.0 / 3.0 * dn * dn * dn;
  c.st.flops[EIG_ST_HEGST] = 4.0 * dn * dn * dn;
  c.st.flops[EIG_ST_HE2HB] = 16.0 / 3.0 * dn * dn * dn;
  if (m_out) *m_out = m;
  EIG_TRY(c.check(cudaStreamSynchronize(c.stream), "sync"));
  if (stats) EIG_TRY(eig_last_stats(h, stats));
  return 0;
}

}  // extern "C"
