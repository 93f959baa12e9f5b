// panel.cu — he2hb panel QR (a1) and T factor (a2) as ONE cooperative kernel.
//
// Panel P = A[(k+1)nb : n, k nb : (k+1)nb] (pn x nb).  zgeqr2 with the LAPACK
// zlarfg convention (reading R1): for column j,
//   beta = -sign(Re alpha) ||(alpha, x)||,  tau = (beta - alpha)/beta,
//   v = (1, x / (alpha - beta)),  P[j:, l] -= conj(tau) v (v^H P[j:, l]),  l > j.
// Then T (zlarft forward/columnwise): T_jj = tau_j,
//   T[0:j, j] = -tau_j T[0:j,0:j] (V[:,0:j]^H v_j).
// Paper: Fig. 1 (a) "panel", P:L97 (run on the CPU there); P:L41 (the
// memory-bound panel work the two-stage method isolates).
//
// B200 design: the panel rows are split over G CTAs (one per SM) and stay in
// shared memory for the whole factorisation; each column costs ONE grid
// barrier: every CTA publishes (||x_local||^2, conj(P[:,j])^H P[:,l] partial
// dots, row j) and every CTA reduces all records in a fixed order (so the
// result is deterministic), computes beta/tau/v locally and updates its rows.
// Because v = (a_j - beta e_j)/(alpha - beta), v^H P[:,l] follows from the raw
// dots a_j^H P[:,l] without a second reduction.
//
// Scaling (reading R1: LAPACK zlarfg's dznrm2 / dlapy3 / safmin rescale keep
// the reflector well defined near both ends of the binary64 range): after the
// load, one extra exchange gives every CTA U_l = the binary exponent of
// max |P[:, l]| over the whole panel, and the resident panel is multiplied by
// D = diag(2^-U_l).  Householder QR is equivariant under column scaling
// (QR(P D) = Q (R D)), so V, tau and T are unchanged and R comes out times D:
// the write-back multiplies the R part (rows <= l) of column l by 2^U_l.  All
// factors are exact powers of two, so for inputs away from the range ends the
// result is bitwise the unscaled one; at the ends the dots and norms (entries
// now <= ~2 sqrt(pn) in magnitude) neither overflow nor underflow.  (A column
// that shrinks by > 2^500 relative to its panel-load maximum during the
// factorisation would still underflow; LAPACK's per-column dznrm2 would not.)
#include <algorithm>
#include <cstdlib>


#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int PT = 512;
constexpr int NQ = PT / 64;   // row parts (64 columns x NQ parts of the rows)

struct PanelArgs {
  double2 *P;
  int64_t lda;
  int64_t pn;
  int nb, nref, R, R0, G;   // CTA 0 owns R0 = R - nb rows, the others R (CTA 0 keeps T in the rest)
  double2 *tau, *T, *vout, *vout2;
  int64_t ldv;
  double2 *rec;                  // [2][G][recw]: s_l (l != j), sumsq at l = j, then row j
  unsigned long long *cnt;       // monotonic arrival counter (never reset)
  unsigned long long epoch0;     // counter value when this launch starts
  unsigned long long *prof;      // optional: CTA 0 phase cycles [8..13]
};

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// One column step costs one exchange: every CTA publishes, for the next pivot
// column a_j (rows below j that it owns), s_l = sum conj(a_j[r]) P[r, l] for
// all l != j, sum |a_j[r]|^2 (in slot j) and, if it owns row j, row j itself;
// then it increments a monotonic counter.  After all G arrivals every CTA
// reduces the records in a fixed order (deterministic) and derives
//   beta, tau, v = (1, a_j / (alpha - beta)),
//   w_l = v^H P[:, l] = P[j, l] + conj(scale) s_l              (l > j),
//   y_i = V[:, i]^H v  = conj(V[j, i]) + scale conj(s_i)       (i < j),
// so the trailing-column update and the T column
//   T[0:j, j] = -tau_j T[0:j, 0:j] y   (zlarft, forward/columnwise)
// need no second reduction.
// Warp PT/32 (the messenger) writes the exchange records to global memory and
// releases the arrival; the PT compute threads hand it each record through a
// shared-memory slot (bar.arrive) and synchronise among themselves with a
// named barrier, so no compute barrier waits for the records' global stores
// or for the release (a CTA barrier right after global stores and a release
// costs ~1 us; see the bulge chase).
__device__ __forceinline__ void pbar() { asm volatile("bar.sync 1, %0;" ::"n"(PT) : "memory"); }
__device__ __forceinline__ void pmsg_arrive() { asm volatile("bar.arrive 2, %0;" ::"n"(PT + 32) : "memory"); }
__device__ __forceinline__ void pmsg_sync() { asm volatile("bar.sync 2, %0;" ::"n"(PT + 32) : "memory"); }

__global__ void __launch_bounds__(PT + 32, 1) panel_qr_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int nb = a.nb, R = a.R, G = a.G;
  const int LR = R | 1;   // odd column stride of the resident rows: conflict-free column-parallel access
  const int recw = 2 * nb;
  double2 *sTau = sm;               // [nb]
  double2 *sRow = sTau + nb;        // [nb]   row j (owner's record)
  double2 *sS = sRow + nb;          // [nb]   conj(tau) w_l for the column updates
  double2 *sW = sS + nb;            // [nb]   w_l / y_i
  double2 *sY = sW + nb;            // [nb]   y_i (T column)
  double2 *sPart = sY + nb;         // [NQ][64]
  double2 *sP = sPart + NQ * 64;    // [nb][R], column l at sP + l*R
  // CTA 0: T (nb x nb, column stride R) in the unused tail rows R0..R-1 of sP
  double2 *sT = sP + a.R0;
  __shared__ double2 s_tau, s_scale;
  __shared__ double s_beta;
  __shared__ double sColUp[64];   // 2^U_l: column l's scale (R part written back times this)

  const int tid = threadIdx.x;
  const int g = blockIdx.x;
  __shared__ double2 sRec[2][128];   // the next record, by column parity (messenger input)
  if (tid >= PT) {   // ================= messenger: one record per column, in order
    const int lane = tid - PT;
    for (int c = 0; c < a.nref; c++) {
      pmsg_sync();
      double2 *out = a.rec + ((int64_t)(c & 1) * G + g) * recw;
      for (int e = lane; e < recw; e += 32) __stcg(&out[e], sRec[c & 1][e]);
      __syncwarp();   // orders the lanes' stores before lane 0's (cumulative) release
      if (lane == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.cnt) : "memory");
    }
    return;
  }
  const int64_t row0 = g == 0 ? 0 : (int64_t)a.R0 + (int64_t)(g - 1) * R;
  const int64_t left = a.pn - row0;
  const int cap = g == 0 ? a.R0 : R;
  const int rows = left <= 0 ? 0 : (left < cap ? (int)left : cap);
  const int cl = tid & 63, rq = tid >> 6;          // column / row-quarter of this thread
  const int R4 = (rows + NQ - 1) / NQ;
  const int rlo = min(rows, rq * R4), rhi = min(rows, (rq + 1) * R4);

  for (int l = 0; l < nb; l++)
    for (int r = tid; r < R; r += PT) sP[l * LR + r] = (r < rows) ? a.P[(row0 + r) + (int64_t)l * a.lda] : czero();
  if (g == 0)
    for (int e = tid; e < nb * nb; e += PT) sT[(e % nb) + (e / nb) * LR] = czero();
  pbar();
  // column magnitude keys of this CTA's rows (thread cl, rows rlo..rhi)
  {
    unsigned k = 0;
    if (cl < nb)
      for (int r = rlo; r < rhi; r++) k = max(k, mag_key2(sP[cl * LR + r]));
    reinterpret_cast<unsigned *>(sPart)[rq * 64 + cl] = k;
  }
  pbar();
  // exchange round 0 (records of parity 1: the column-1 records are written
  // only after every CTA has published column 0, i.e. has read these keys)
  {
    double2 *out = a.rec + ((int64_t)G + g) * recw;
    if (tid < nb) {
      unsigned k = 0;
#pragma unroll
      for (int q = 0; q < NQ; q++) k = max(k, reinterpret_cast<const unsigned *>(sPart)[q * 64 + tid]);
      __stcg(&out[tid], make_double2(__longlong_as_double((long long)k), 0.0));
    }
    pbar();
    if (tid == 0) {
      asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.cnt) : "memory");
      const unsigned long long target = a.epoch0 + (unsigned long long)G;
      while (ld_acquire_u64(a.cnt) < target) {
      }
    }
    pbar();
    {   // every thread takes CTAs q = rq, rq + NQ, ... of column cl (loads batched 4 at a time)
      unsigned k = 0;
      if (cl < nb)
        for (int q0 = rq; q0 < G; q0 += 4 * NQ) {
          unsigned kk[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int q = q0 + u * NQ;
            kk[u] = q < G ? (unsigned)__double_as_longlong(__ldcg((const double *)(a.rec + ((int64_t)G + q) * recw + cl)))
                          : 0u;
          }
          k = max(k, max(max(kk[0], kk[1]), max(kk[2], kk[3])));
        }
      reinterpret_cast<unsigned *>(sPart)[NQ * 64 + rq * 64 + cl] = k;   // second half of sPart
    }
    pbar();
    if (tid < nb) {
      unsigned k = 0;
#pragma unroll
      for (int q = 0; q < NQ; q++) k = max(k, reinterpret_cast<const unsigned *>(sPart)[NQ * 64 + q * 64 + tid]);
      const int U = exp_of_key(k);   // kExpZero: zero column, scale 1
      sColUp[tid] = U == kExpZero ? 1.0 : pow2i(U);
      sW[tid] = make_double2(U == kExpZero ? 1.0 : pow2i(-U), 0.0);   // 2^-U_l (sW is free until column 0)
    }
    pbar();
    for (int l = 0; l < nb; l++) {
      const double f = sW[l].x;
      for (int r = tid; r < rows; r += PT) sP[l * LR + r] = cscale(f, sP[l * LR + r]);
    }
  }
  pbar();

  const bool prof = a.prof != nullptr && g == 0 && tid == 0;
  long long tm = prof ? clock64() : 0, tacc[6] = {0, 0, 0, 0, 0, 0};
  auto mark = [&](int k) {
    if (prof) {
      const long long now = clock64();
      tacc[k] += now - tm;
      tm = now;
    }
  };

  // publish the record for pivot column jn and arrive.  With look-ahead, only
  // column jn has been updated by the previous reflector (column jp = jn-1,
  // holding v); columns l > jn are stale and their dots are corrected with
  //   s_l = s_l(stale) - conj(tau) w_l (a^H v)   and   P[jn,l] -= conj(tau) v[jn] w_l.
  auto publish = [&](int jn, bool corr, double2 ctau) {
    double2 acc = czero();
    if (cl < nb) {
      const double2 *aj = sP + jn * LR, *pl = sP + cl * LR;
      for (int r = rlo; r < rhi; r++) {
        if (row0 + r <= jn) continue;
        const double2 x = aj[r];
        if (cl == jn) acc.x += x.x * x.x + x.y * x.y;
        else acc = cadd(acc, cmulc(x, pl[r]));
      }
    }
    sPart[rq * 64 + cl] = acc;
    pbar();
    double2 *out = sRec[jn & 1];
    if (tid < nb) {
      double2 t = sPart[tid];
#pragma unroll
      for (int q = 1; q < NQ; q++) t = cadd(t, sPart[q * 64 + tid]);
      if (corr && tid > jn) {
        const int jp = jn - 1;
        double2 c1 = sPart[jp];
#pragma unroll
        for (int q = 1; q < NQ; q++) c1 = cadd(c1, sPart[q * 64 + jp]);
        t = csub(t, cmul(ctau, cmul(sW[tid], c1)));
      }
      out[tid] = t;
    }
    if (jn >= row0 && jn < row0 + rows)
      for (int l = tid; l < nb; l += PT) {
        double2 pv = sP[l * LR + (jn - row0)];
        if (corr && l > jn) pv = csub(pv, cmul(ctau, cmul(sP[(jn - 1) * LR + (jn - row0)], sW[l])));
        out[nb + l] = pv;
      }
    pmsg_arrive();   // the messenger stores the record and releases the arrival
    pbar();          // keeps the bulk update below from overwriting row jn before it is recorded
  };
  // record q (CTA q) of the exchange for column j
  auto rec_of = [&](int q, int j) -> const double2 * { return a.rec + ((int64_t)(j & 1) * G + q) * recw; };

  if (a.nref > 0) publish(0, false, czero());
  mark(4);
  for (int j = 0; j < a.nref; j++) {
    if (tid == 0) {   // round 0 was the scaling exchange
      const unsigned long long target = a.epoch0 + (unsigned long long)G * (j + 2);
      while (ld_acquire_u64(a.cnt) < target) {
      }
    }
    pbar();
    mark(0);
    {
      // s_l for l >= j (every CTA: norm, w_l); s_i for i < j only feed T (CTA 0)
      double2 acc = czero();
      // the loads of a batch are issued together (one L2 round trip per 4
      // records instead of one per record); the sum keeps the order q = rq,
      // rq + NQ, ... so the result is unchanged
      if (cl < nb && (cl >= j || g == 0))
        for (int q0 = rq; q0 < G; q0 += 4 * NQ) {
          double2 v[4];
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int q = q0 + u * NQ;
            v[u] = q < G ? __ldcg(rec_of(q, j) + cl) : czero();
          }
#pragma unroll
          for (int u = 0; u < 4; u++)
            if (q0 + u * NQ < G) acc = cadd(acc, v[u]);
        }
      sPart[rq * 64 + cl] = acc;
      const int owner = j < a.R0 ? 0 : 1 + (j - a.R0) / R;
      if (tid < nb) sRow[tid] = __ldcg(rec_of(owner, j) + nb + tid);
    }
    pbar();
    // thread l < nb keeps the reduced s_l in a register; thread j (which holds
    // ||x||^2 and has row j) forms beta / tau / scale: one CTA barrier fewer
    double2 sl = czero();
    if (tid < nb) {
      sl = sPart[tid];
#pragma unroll
      for (int q = 1; q < NQ; q++) sl = cadd(sl, sPart[q * 64 + tid]);
      sPart[tid] = sl;   // every thread forms w_{j+1} from it below
    }
    mark(1);
    if (tid == j) {   // zlarfg (reading R1); alpha and x are in column j's units (|.| <~ 2 sqrt(pn))
      const double2 alpha = sRow[j];
      const double xnorm2 = sl.x;
      double2 tau, scale;
      double beta;
      if (xnorm2 == 0.0 && alpha.y == 0.0) {
        tau = czero();
        beta = alpha.x;
        scale = czero();
      } else {
        beta = -copysign(sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2), alpha.x);
        tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
        const double2 d = make_double2(alpha.x - beta, alpha.y);   // 1 / (alpha - beta)
        const double dd = d.x * d.x + d.y * d.y;
        scale = make_double2(d.x / dd, -d.y / dd);
      }
      s_tau = tau;
      s_scale = scale;
      s_beta = beta;
      sTau[j] = tau;
    }
    pbar();
    mark(2);
    const double2 tau = s_tau, scale = s_scale;
    const double2 ctau = cconj(tau);
    if (tid < nb) {
      if (tid > j) {
        sW[tid] = cadd(sRow[tid], cmulc(scale, sl));                  // w_l = v^H P[:,l]
        sS[tid] = cmul(cconj(tau), sW[tid]);                          // conj(tau) w_l
      }
      else if (tid < j) sY[tid] = cadd(cconj(sRow[tid]), cmul(scale, cconj(sl)));  // y_i = V_i^H v
    }
    // scale column j into v and, with look-ahead, apply H_j to the next pivot
    // column in the same pass (same rows per thread: no barrier between)
    const double2 *vj = sP + j * LR;
    const bool la = (j + 1 < a.nref);
    const double2 cw = la ? cmul(ctau, cadd(sRow[j + 1], cmulc(scale, sPart[j + 1]))) : czero();
    double2 *pn1 = sP + (j + 1) * LR;
    for (int r = tid; r < rows; r += PT) {
      const int64_t grow = row0 + r;
      if (grow < j) continue;
      double2 v;
      if (grow > j) {
        v = cmul(sP[j * LR + r], scale);
        sP[j * LR + r] = v;
      } else {
        sP[j * LR + r] = make_double2(s_beta, 0.0);
        v = make_double2(1.0, 0.0);
      }
      if (la) pn1[r] = csub(pn1[r], cmul(v, cw));
    }
    pbar();
    if (la) {
      mark(3);
      publish(j + 1, true, ctau);
      mark(4);
    }
    // bulk update of the remaining trailing columns (overlaps the other CTAs'
    // exchange).  One work item = one row x up to 16 columns: v[r] is loaded
    // once per item and a warp touches 32 consecutive rows of a column
    // (conflict-free); the loop is bound by shared-memory bandwidth
    {
      const int lo = la ? j + 2 : j + 1;
      const int c = nb - lo;
      if (c > 0) {
        constexpr int CH = 16;
        const int nch = (c + CH - 1) / CH;
        const int rstart = (int)max((int64_t)0, (int64_t)j - row0);   // rows at or below j
        const int nr = max(0, rows - rstart);
        for (int it = tid; it < nr * nch; it += PT) {
          const int ch = it / nr, r = rstart + (it - ch * nr);
          const double2 v = (row0 + r == j) ? make_double2(1.0, 0.0) : vj[r];
          const int l0 = lo + ch * CH, l1 = min(nb, l0 + CH);
          for (int l = l0; l < l1; l++) {
            double2 *pl = sP + l * LR;
            pl[r] = csub(pl[r], cmul(v, sS[l]));
          }
        }
      }
    }
    if (g == 0) {
      // T column j: T[0:j, j] = -tau_j T[0:j, 0:j] y   (4 threads per row, shared memory)
      const int i = tid >> 2, part = tid & 3;
      double2 acc = czero();
      if (i < j)
        for (int l = i + part; l < j; l += 4) acc = cadd(acc, cmul(sT[i + l * LR], sY[l]));
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
      if (i < j && part == 0)
        sT[i + j * LR] = make_double2(-(tau.x * acc.x - tau.y * acc.y), -(tau.x * acc.y + tau.y * acc.x));
      if (tid == 0) sT[j + j * LR] = tau;
    }
    pbar();
    mark(5);
  }

  // write back the factored rows (R part times 2^U_l) and the explicit unit-lower V
  for (int l = 0; l < nb; l++) {
    const double up = sColUp[l];
    for (int r = tid; r < rows; r += PT) {
      const int64_t grow = row0 + r;
      const double2 p = sP[l * LR + r];
      a.P[grow + (int64_t)l * a.lda] = grow <= l ? cscale(up, p) : p;
      const double2 v = (grow > l) ? p : (grow == l ? make_double2(1.0, 0.0) : czero());
      a.vout[grow + (int64_t)l * a.ldv] = v;
      if (a.vout2) a.vout2[grow + (int64_t)l * a.ldv] = v;
    }
  }
  if (g == 0) {
    for (int l = tid; l < nb; l += PT) a.tau[l] = (l < a.nref) ? sTau[l] : czero();
    for (int e = tid; e < nb * nb; e += PT) a.T[e] = sT[(e % nb) + (e / nb) * LR];
  }
  if (prof)
    for (int k = 0; k < 6; k++) atomicAdd(&a.prof[8 + k], (unsigned long long)tacc[k]);
}

// Explicit unit-lower V (s x nb) from the he2hb storage of one panel.
__global__ void extract_v_kernel(const double2 *P, int64_t lda, int64_t pn, int nb, double2 *V, int64_t ldv) {
  const int64_t total = pn * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % pn;
    const int l = (int)(e / pn);
    double2 v;
    if (r > l) v = P[r + l * lda];
    else v = (r == l) ? make_double2(1.0, 0.0) : czero();
    V[r + l * ldv] = v;
  }
}

__global__ void real_diag_kernel(int64_t n, double2 *A, int64_t lda) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    A[i + i * lda].y = 0.0;
}

}  // namespace

int panel_qr(Ctx &ctx, double2 *P, int64_t lda, int64_t pn, int nb, double2 *tau, double2 *T, double2 *vout,
             double2 *vout2, int64_t ldv, cudaStream_t stream) {
  if (pn <= 0) return 0;
  if (nb > 64) return EIG_ERR_NOTIMPL;
  const int nref = (int)std::min<int64_t>(pn, nb);
  // CTAs: one per nb rows, capped at 32 (fewer records to exchange per
  // column, and the SMs left free run the concurrent trailing update), but at
  // least as many as hold the panel rows in shared memory; EIG_PANEL_CTAS
  // replaces the cap (tuning; he2hb n = 10^4: cap 8 / 16 / 24 / 32 / 48 / 148
  // -> 283 / 277 / 273 / 269 / 273 / 281 ms)
  static const int gmax_env = [] {
    const char *e = getenv("EIG_PANEL_CTAS");
    return e ? atoi(e) : 0;
  }();
  const int recw = 2 * nb;
  const int words = 220 * 1024 / (int)sizeof(double2);
  const int64_t rows_nb = (pn + nb - 1) / nb;
  const int gmax = gmax_env > 0 ? std::min(gmax_env, ctx.num_sms) : std::min(32, ctx.num_sms);
  int G = (int)std::min<int64_t>(gmax, rows_nb);
  G = std::max(G, 1);
  const int rmax = (words - 5 * nb - NQ * 64) / nb - 1;   // rows that fit on chip (odd stride)
  G = std::max<int64_t>(G, (pn + nb + rmax - 1) / rmax);
  int R = (int)((pn + nb + G - 1) / G);   // CTA 0 holds R - nb rows
  R = std::max(R, nb);
  G = (int)((pn + nb + R - 1) / R);
  const size_t smem = ((size_t)5 * nb + NQ * 64 + (size_t)nb * (R | 1)) * sizeof(double2);
  if (smem > 220 * 1024) return EIG_ERR_NOTIMPL;  // panel too tall for on-chip residency (n > ~20000 at nb=64)
  PanelArgs a;
  a.P = P;
  a.lda = lda;
  a.pn = pn;
  a.nb = nb;
  a.nref = nref;
  a.R = R;
  a.R0 = R - nb;
  a.G = G;
  a.tau = tau;
  a.T = T;
  a.vout = vout;
  a.vout2 = vout2;
  a.ldv = ldv;
  a.rec = (double2 *)ctx.ws(WS_PANEL_REC, (size_t)2 * G * recw * sizeof(double2));
  a.cnt = (unsigned long long *)ctx.buf[WS_BARRIER];
  a.epoch0 = ctx.bar_epoch;
  a.prof = ctx.q2_prof;
  if (!a.rec || !a.cnt) return EIG_ERR_NOMEM;
  EIG_TRY(ctx.smem_attr((const void *)panel_qr_kernel, 220 * 1024, "panel attr"));
  void *args[] = {&a};
  EIG_TRY(ctx.check(cudaLaunchCooperativeKernel((void *)panel_qr_kernel, dim3(G), dim3(PT + 32), args, smem, stream),
                    "panel_qr_kernel launch"));
  ctx.bar_epoch += (unsigned long long)G * (nref + 1);   // arrivals this launch performs (scaling round + columns)
  return ctx.launched("panel_qr_kernel");
}

int extract_v(Ctx &ctx, const double2 *P, int64_t lda, int64_t pn, int nb, double2 *V, int64_t ldv) {
  if (pn <= 0) return 0;
  const int64_t total = pn * nb;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4LL * ctx.num_sms);
  extract_v_kernel<<<blocks, 256, 0, ctx.stream>>>(P, lda, pn, nb, V, ldv);
  return ctx.launched("extract_v_kernel");
}

int real_diag(Ctx &ctx, int64_t n, double2 *A, int64_t lda) {
  if (n <= 0) return 0;
  real_diag_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, ctx.stream>>>(n, A, lda);
  return ctx.launched("real_diag_kernel");
}

}  // namespace eig
