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
#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int PT = 256;

struct PanelArgs {
  double2 *P;
  int64_t lda;
  int64_t pn;
  int nb, nref, R, G;
  double2 *tau, *T, *vout, *vout2;
  int64_t ldv;
  double2 *rec;    // [2][G][recw]
  double2 *gram;   // [G][nb*nb] partials, then [nb*nb] final
  unsigned *bar;   // [0] count, [1] generation
};

__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(PT, 1) panel_qr_kernel(PanelArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  const int nb = a.nb, R = a.R, G = a.G;
  const int recw = 1 + 2 * nb;
  double2 *sTau = sm;               // [nb]
  double2 *sRed = sTau + nb;        // [recw]
  double2 *sW = sRed + recw;        // [nb]
  double2 *sP = sW + nb;            // [nb][max(R, 2nb)], column l at sP + l*R
  __shared__ double2 s_tau, s_scale, s_alpha;
  __shared__ double s_beta;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = blockIdx.x;
  const int64_t row0 = (int64_t)g * R;
  const int64_t left = a.pn - row0;
  const int rows = left <= 0 ? 0 : (left < R ? (int)left : R);

  for (int e = tid; e < R * nb; e += PT) {
    const int r = e % R, l = e / R;
    sP[l * R + r] = (r < rows) ? a.P[(row0 + r) + (int64_t)l * a.lda] : czero();
  }
  __syncthreads();

  auto partials = [&](int j) {
    double2 *out = a.rec + ((int64_t)(j & 1) * G + g) * recw;
    for (int t = warp; t < nb - j; t += PT / 32) {
      double2 acc = czero();
      if (t == 0) {
        for (int r = lane; r < rows; r += 32)
          if (row0 + r > j) {
            const double2 v = sP[j * R + r];
            acc.x += v.x * v.x + v.y * v.y;
          }
      } else {
        const int l = j + t;
        for (int r = lane; r < rows; r += 32)
          if (row0 + r >= j) acc = cadd(acc, cmulc(sP[j * R + r], sP[l * R + r]));
      }
      acc = warp_sum2(acc);
      if (lane == 0) __stcg(&out[t == 0 ? 0 : 1 + j + t], acc);
    }
    if (j >= row0 && j < row0 + rows)
      for (int l = j + tid; l < nb; l += PT) __stcg(&out[1 + nb + l], sP[l * R + (j - row0)]);
  };

  if (a.nref > 0) partials(0);
  for (int j = 0; j < a.nref; j++) {
    grid_barrier(a.bar, G);
    const double2 *recs = a.rec + (int64_t)(j & 1) * G * recw;
    // reduce: warp per entry, lanes over CTAs, fixed order
    for (int t = warp; t < nb - j; t += PT / 32) {
      const int idx = (t == 0) ? 0 : 1 + j + t;
      double2 s = czero();
      for (int q = lane; q < G; q += 32) s = cadd(s, __ldcg(&recs[(int64_t)q * recw + idx]));
      s = warp_sum2(s);
      if (lane == 0) sRed[idx] = s;
    }
    const int owner = j / R;
    for (int l = j + tid; l < nb; l += PT) sRed[1 + nb + l] = __ldcg(&recs[(int64_t)owner * recw + 1 + nb + l]);
    __syncthreads();
    if (tid == 0) {
      const double2 alpha = sRed[1 + nb + j];
      const double xnorm2 = sRed[0].x;
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
      s_alpha = alpha;
      sTau[j] = tau;
    }
    __syncthreads();
    const double2 tau = s_tau, scale = s_scale, alpha = s_alpha;
    const double beta = s_beta;
    for (int l = j + 1 + tid; l < nb; l += PT) {
      const double2 pj = sRed[1 + nb + l];
      const double2 d = csub(sRed[1 + l], cmulc(alpha, pj));   // dot_l - conj(alpha) P[j,l]
      sW[l] = cadd(pj, cmulc(scale, d));                       // v^H P[:, l]
    }
    for (int r = tid; r < rows; r += PT) {
      const int64_t grow = row0 + r;
      if (grow > j) sP[j * R + r] = cmul(sP[j * R + r], scale);
      else if (grow == j) sP[j * R + r] = make_double2(beta, 0.0);
    }
    __syncthreads();
    const int ncols = nb - j - 1;
    const double2 ctau = cconj(tau);
    for (int e = tid; e < rows * ncols; e += PT) {
      const int r = e % rows, l = j + 1 + e / rows;
      const int64_t grow = row0 + r;
      if (grow < j) continue;
      const double2 v = (grow == j) ? make_double2(1.0, 0.0) : sP[j * R + r];
      sP[l * R + r] = csub(sP[l * R + r], cmul(ctau, cmul(v, sW[l])));
    }
    __syncthreads();
    if (j + 1 < a.nref) partials(j + 1);
  }

  // write back the factored rows and the explicit unit-lower V
  for (int e = tid; e < rows * nb; e += PT) {
    const int r = e % rows, l = e / rows;
    const int64_t grow = row0 + r;
    const double2 p = sP[l * R + r];
    a.P[grow + (int64_t)l * a.lda] = p;
    const double2 v = (grow > l) ? p : (grow == l ? make_double2(1.0, 0.0) : czero());
    a.vout[grow + (int64_t)l * a.ldv] = v;
    if (a.vout2) a.vout2[grow + (int64_t)l * a.ldv] = v;
  }
  // Gram partials G[x][y] = sum_r conj(V[r,x]) V[r,y], x < y
  {
    double2 *out = a.gram + (int64_t)g * nb * nb;
    for (int pidx = tid; pidx < nb * nb; pidx += PT) {
      const int x = pidx % nb, y = pidx / nb;
      double2 s = czero();
      if (x < y) {
        for (int r = 0; r < rows; r++) {
          const int64_t grow = row0 + r;
          if (grow < y) continue;
          const double2 vy = (grow == y) ? make_double2(1.0, 0.0) : sP[y * R + r];
          const double2 vx = sP[x * R + r];   // grow >= y > x: strictly below the diagonal
          s = cadd(s, cmulc(vx, vy));
        }
      }
      __stcg(&out[pidx], s);
    }
  }
  grid_barrier(a.bar, G);
  {
    double2 *fin = a.gram + (int64_t)G * nb * nb;
    const int per = (nb * nb + G - 1) / G;
    for (int pidx = g * per + tid; pidx < min(nb * nb, (g + 1) * per); pidx += PT) {
      double2 s = czero();
      for (int q = 0; q < G; q++) s = cadd(s, __ldcg(&a.gram[(int64_t)q * nb * nb + pidx]));
      __stcg(&fin[pidx], s);
    }
  }
  grid_barrier(a.bar, G);
  if (g == 0) {
    double2 *sG = sP;                // reuse: [nb][nb]
    double2 *sT = sP + nb * nb;      // [nb][nb]
    const double2 *fin = a.gram + (int64_t)G * nb * nb;
    for (int pidx = tid; pidx < nb * nb; pidx += PT) {
      sG[pidx] = __ldcg(&fin[pidx]);
      sT[pidx] = czero();
    }
    __syncthreads();
    for (int j = 0; j < a.nref; j++) {
      const double2 tj = sTau[j];
      if (tid < j) {
        const int i = tid;
        double2 s = czero();
        for (int l = i; l < j; l++) s = cadd(s, cmul(sT[i + l * nb], sG[l + j * nb]));
        sT[i + j * nb] = make_double2(-(tj.x * s.x - tj.y * s.y), -(tj.x * s.y + tj.y * s.x));
      }
      if (tid == 0) sT[j + j * nb] = tj;
      __syncthreads();
    }
    for (int pidx = tid; pidx < nb * nb; pidx += PT) a.T[pidx] = sT[pidx];
    for (int l = tid; l < nb; l += PT) a.tau[l] = (l < a.nref) ? sTau[l] : czero();
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
             double2 *vout2, int64_t ldv) {
  if (pn <= 0) return 0;
  const int nref = (int)std::min<int64_t>(pn, nb);
  int G = (int)std::min<int64_t>(ctx.num_sms, (pn + nb - 1) / nb);
  G = std::max(G, 1);
  int R = (int)((pn + G - 1) / G);
  R = std::max(R, nb);
  G = (int)((pn + R - 1) / R);
  const int recw = 1 + 2 * nb;
  const size_t smem = ((size_t)nb * std::max(R, 2 * nb) + recw + 2 * nb) * sizeof(double2);
  if (smem > 220 * 1024) return EIG_ERR_NOTIMPL;  // panel too tall for on-chip residency (n > ~24000)
  PanelArgs a;
  a.P = P;
  a.lda = lda;
  a.pn = pn;
  a.nb = nb;
  a.nref = nref;
  a.R = R;
  a.G = G;
  a.tau = tau;
  a.T = T;
  a.vout = vout;
  a.vout2 = vout2;
  a.ldv = ldv;
  a.rec = (double2 *)ctx.ws(WS_PANEL_REC, (size_t)2 * G * recw * sizeof(double2));
  a.gram = (double2 *)ctx.ws(WS_PANEL_GRAM, (size_t)(G + 1) * nb * nb * sizeof(double2));
  a.bar = (unsigned *)ctx.buf[WS_BARRIER];
  if (!a.rec || !a.gram || !a.bar) return EIG_ERR_NOMEM;
  static bool attr = false;
  if (!attr) {
    EIG_TRY(ctx.check(cudaFuncSetAttribute(panel_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024),
                      "panel attr"));
    attr = true;
  }
  void *args[] = {&a};
  EIG_TRY(ctx.check(cudaLaunchCooperativeKernel((void *)panel_qr_kernel, dim3(G), dim3(PT), args, smem, ctx.stream),
                    "panel_qr_kernel launch"));
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
