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
// Panels short enough for one thread-block cluster (CL = true: at most
// EIG_PANEL_CLUSTER CTAs; opt-in) keep the records in each CTA's own shared
// memory and exchange them through distributed shared memory; the split
// barrier.cluster arrive (after publishing) / wait (before reducing) replaces
// the L2 counter.  These are the late panels, whose latency the shrinking
// trailing update no longer hides.
// Because v = (a_j - beta e_j)/(alpha - beta), v^H P[:,l] follows from the raw
// dots a_j^H P[:,l] without a second reduction.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

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
template <bool CL>
__global__ void __launch_bounds__(PT, 1) panel_qr_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int nb = a.nb, R = a.R, G = a.G;
  const int LR = R | 1;   // odd column stride of the resident rows: conflict-free column-parallel access
  const int recw = 2 * nb;
  double2 *sTau = sm;               // [nb]
  double2 *sRow = sTau + nb;        // [nb]   row j (owner's record)
  double2 *sS = sRow + nb;          // [nb]   conj(tau) w_l for the column updates
  double2 *sW = sS + nb;            // [nb]   w_l / y_i
  double2 *sY = sW + nb;            // [nb]   y_i (T column)
  double2 *sPart = sY + nb;         // [4][64]
  double2 *sRec = sPart + NQ * 64;  // CL: [2][recw] this CTA's records
  double2 *sP = sRec + (CL ? 2 * recw : 0);   // [nb][R], column l at sP + l*R
  // CTA 0: T (nb x nb, column stride R) in the unused tail rows R0..R-1 of sP
  double2 *sT = sP + a.R0;
  __shared__ double2 s_tau, s_scale;
  __shared__ double s_beta;

  const int tid = threadIdx.x;
  const int g = blockIdx.x;
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
  __syncthreads();

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
    __syncthreads();
    double2 *out = CL ? sRec + (jn & 1) * recw : a.rec + ((int64_t)(jn & 1) * G + g) * recw;
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
      if (CL) out[tid] = t;
      else __stcg(&out[tid], t);
    }
    if (jn >= row0 && jn < row0 + rows)
      for (int l = tid; l < nb; l += PT) {
        double2 pv = sP[l * LR + (jn - row0)];
        if (corr && l > jn) pv = csub(pv, cmul(ctau, cmul(sP[(jn - 1) * LR + (jn - row0)], sW[l])));
        if (CL) out[nb + l] = pv;
        else __stcg(&out[nb + l], pv);
      }
    // the barrier orders every thread's record stores before thread 0's
    // release increment (fence cumulativity): one release instead of a
    // membar in every thread; it also keeps the bulk update below from
    // overwriting row jn before it is recorded
    __syncthreads();
    if (CL) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    else if (tid == 0) asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.cnt) : "memory");
  };
  // record q (CTA q) of the exchange for column j
  auto rec_of = [&](int q, int j) -> const double2 * {
    if (CL) return cooperative_groups::this_cluster().map_shared_rank(sRec + (j & 1) * recw, q);
    return a.rec + ((int64_t)(j & 1) * G + q) * recw;
  };

  if (a.nref > 0) publish(0, false, czero());
  mark(4);
  for (int j = 0; j < a.nref; j++) {
    if (CL) {
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      if (tid == 0) {
        const unsigned long long target = a.epoch0 + (unsigned long long)G * (j + 1);
        while (ld_acquire_u64(a.cnt) < target) {
        }
      }
      __syncthreads();
    }
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
            v[u] = q < G ? (CL ? rec_of(q, j)[cl] : __ldcg(rec_of(q, j) + cl)) : czero();
          }
#pragma unroll
          for (int u = 0; u < 4; u++)
            if (q0 + u * NQ < G) acc = cadd(acc, v[u]);
        }
      sPart[rq * 64 + cl] = acc;
      const int owner = j < a.R0 ? 0 : 1 + (j - a.R0) / R;
      if (tid < nb) sRow[tid] = CL ? rec_of(owner, j)[nb + tid] : __ldcg(rec_of(owner, j) + nb + tid);
    }
    __syncthreads();
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
    if (tid == j) {
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
    __syncthreads();
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
    __syncthreads();
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
    __syncthreads();
    mark(5);
  }

  // write back the factored rows and the explicit unit-lower V
  for (int l = 0; l < nb; l++)
    for (int r = tid; r < rows; r += PT) {
      const int64_t grow = row0 + r;
      const double2 p = sP[l * LR + r];
      a.P[grow + (int64_t)l * a.lda] = p;
      const double2 v = (grow > l) ? p : (grow == l ? make_double2(1.0, 0.0) : czero());
      a.vout[grow + (int64_t)l * a.ldv] = v;
      if (a.vout2) a.vout2[grow + (int64_t)l * a.ldv] = v;
    }
  if (g == 0) {
    for (int l = tid; l < nb; l += PT) a.tau[l] = (l < a.nref) ? sTau[l] : czero();
    for (int e = tid; e < nb * nb; e += PT) a.T[e] = sT[(e % nb) + (e / nb) * LR];
  }
  if (prof)
    for (int k = 0; k < 6; k++) atomicAdd(&a.prof[8 + k], (unsigned long long)tacc[k]);
  if (CL) {
    // no CTA leaves while another may still read its records
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
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
  // cluster path (opt-in): panels whose rows fit in at most EIG_PANEL_CLUSTER
  // CTAs (<= 8 portable, up to 16 non-portable; default 0 = off).  Measured
  // he2hb n = 2000 / 10^4: off 15.5 / 241.3 ms, 4: 15.9 / 241.7, 8: 16.5 /
  // 242.3, 16: 15.2 / 242.8 -- the ~7 us per column is not the exchange.
  static const int clmax = [] {
    const char *e = getenv("EIG_PANEL_CLUSTER");
    return std::min(16, std::max(0, e ? atoi(e) : 0));
  }();
  const int recw = 2 * nb;
  const int words = 220 * 1024 / (int)sizeof(double2);
  const int64_t rows_nb = (pn + nb - 1) / nb;
  {
    const int rmax_cl = (words - 5 * nb - NQ * 64 - 2 * recw) / nb - 1;
    const int64_t gmin = (pn + nb + rmax_cl - 1) / rmax_cl;
    if (gmin <= clmax) {
      int G = (int)std::max<int64_t>(gmin, std::min<int64_t>(clmax, rows_nb));
      int R = (int)std::max<int64_t>((pn + nb + G - 1) / G, nb);
      G = (int)((pn + nb + R - 1) / R);
      PanelArgs a{P, lda, pn, nb, nref, R, R - nb, G, tau, T, vout, vout2, ldv, nullptr, nullptr, 0, ctx.q2_prof};
      const size_t smem = ((size_t)5 * nb + NQ * 64 + 2 * recw + (size_t)nb * (R | 1)) * sizeof(double2);
      static bool attr_cl = false;
      if (!attr_cl) {
        EIG_TRY(ctx.check(cudaFuncSetAttribute(panel_qr_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               220 * 1024), "panel attr"));
        EIG_TRY(ctx.check(cudaFuncSetAttribute(panel_qr_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                          "panel cluster attr"));
        attr_cl = true;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G);
      cfg.blockDim = dim3(PT);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = G;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      EIG_TRY(ctx.check(cudaLaunchKernelEx(&cfg, panel_qr_kernel<true>, a), "panel_qr_kernel<cluster> launch"));
      return ctx.launched("panel_qr_kernel");
    }
  }
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
  static bool attr = false;
  if (!attr) {
    EIG_TRY(ctx.check(cudaFuncSetAttribute(panel_qr_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           220 * 1024), "panel attr"));
    attr = true;
  }
  void *args[] = {&a};
  EIG_TRY(ctx.check(cudaLaunchCooperativeKernel((void *)panel_qr_kernel<false>, dim3(G), dim3(PT), args, smem, stream),
                    "panel_qr_kernel launch"));
  ctx.bar_epoch += (unsigned long long)G * nref;   // arrivals this launch performs
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
