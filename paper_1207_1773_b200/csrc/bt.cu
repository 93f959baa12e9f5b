// bt.cu — back-transform kernels: grouped Q2 blocks (a6), complexify (a6),
// diagonal-block inverses for the blocked L^-H solve (a8).
//
// Q2 (reading R7): the bulge-chase reflectors H_{i,j} are applied in
// blocks of g consecutive sweeps i0..i0+g-1 at a fixed step j; block (i0, j)
// is the forward product H_{i0,j} ... H_{i0+g-1,j} = I - V T V^H, where V is
// a parallelogram of (nb+g-1) x g (reflector t occupies block rows t..t+nb-1).
// Groups are applied last to first, and inside a group the steps j ascending.
//
// apply_q2_kernel: one CTA per column slab of E (bn = 64 columns).  The CTA
// walks all blocks in that order with a sliding row window of nb+g-1 rows in
// shared memory (each E row is loaded and stored once per group), and per
// block runs three DMMA contractions from shared memory:
//   Y = V^H E_win (g x bn), Y = T Y, E_win -= V Y,
// skipping the DMMA fragments that fall in the zero corners of the
// parallelogram and below the diagonal of T.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int QT = 256;       // threads
constexpr int QBN = 64;       // columns per slab
constexpr int QMAXG = 32;     // max group size
constexpr int QMAXNB = 64;

struct Q2Args {
  int64_t n, m, lde;
  int nb, g, W, LDE, LDY, LDT;
  int64_t ngroups;
  const int64_t *first;  // [ngroups+1]
  const int64_t *off;    // [J]
  const double2 *V2;
  const double2 *T2;
  double2 *E;
};

__device__ __forceinline__ int64_t q2_steps(int64_t n, int nb, int64_t i0) {
  // number of steps j with i0 + 1 + j*nb <= n-1
  return (i0 > n - 2) ? 0 : (n - 2 - i0) / nb + 1;
}

__global__ void __launch_bounds__(QT, 1) apply_q2_kernel(Q2Args a) {
  extern __shared__ __align__(16) double2 sm[];
  const int nb = a.nb, g = a.g, W = a.W, LDE = a.LDE, LDY = a.LDY, LDT = a.LDT;
  double2 *sV = sm;                    // [g][nb]
  double2 *sT = sV + g * nb;           // [g][LDT] column-major T[x][y] at y*LDT + x
  double2 *sE = sT + g * LDT;          // [QBN][LDE]
  double2 *sY = sE + QBN * LDE;        // [QBN][LDY]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 1, wn = warp >> 1;  // 2 x 4 warps
  const LaneEmb le(lane);
  const int64_t c0 = (int64_t)blockIdx.x * QBN;
  const int ncols = (int)imin64(QBN, a.m - c0);
  const int Wp = (W + 1) & ~1;   // rows padded to even (k-steps of 2 complex rows)

  for (int64_t gi = a.ngroups - 1; gi >= 0; gi--) {
    const int64_t i0 = gi * g;
    const int64_t J = q2_steps(a.n, nb, i0);
    for (int64_t j = 0; j < J; j++) {
      const int64_t rs = i0 + 1 + j * nb;
      const int64_t blk = a.first[gi] + j;
      // ---- load V (g slots), T, and the window rows
      {
        const int64_t last_i = a.n - 2 - j * nb;                 // last sweep with a slot at step j
        const int64_t nvalid = imax64(0, imin64(g, last_i - i0 + 1));
        const double2 *src = a.V2 + (a.off[j] + i0) * nb;
        for (int e = tid; e < g * nb; e += QT) {
          const bool ok = (e / nb) < nvalid;
          cp_async16(&sV[e], ok ? src + e : a.V2, ok);
        }
        const double2 *tsrc = a.T2 + blk * g * g;
        for (int e = tid; e < g * g; e += QT) {
          const int x = e % g, y = e / g;
          cp_async16(&sT[y * LDT + x], tsrc + e, true);
        }
        const int rfirst = (j == 0) ? 0 : g - 1;
        const int nload = Wp - rfirst;
        for (int e = tid; e < QBN * nload; e += QT) {
          const int q = rfirst + e % nload, c = e / nload;
          const int64_t row = rs + q;
          const bool ok = (q < W) && (row < a.n) && (c < ncols);
          cp_async16(&sE[c * LDE + q], ok ? a.E + row + (c0 + c) * a.lde : a.E, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
      }
      // ---- phase A: Y = V^H E_win   (2g real rows x QBN)
      {
        double acc[4][2][2];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int jj = 0; jj < 2; jj++) acc[i][jj][0] = acc[i][jj][1] = 0.0;
        const double *e = reinterpret_cast<const double *>(sE);
        const double *v = reinterpret_cast<const double *>(sV);
        const int mf0 = wm * 4;                 // 4 m-frags of 4 reflectors each
        const int nmf = g / 4;                  // m-frags that exist
        for (int ks = 0; ks < Wp / 2; ks++) {
          const int q = ks * 2 + ((lane & 3) >> 1);
          double bf[2];
#pragma unroll
          for (int jj = 0; jj < 2; jj++) {
            const int nn = (wn * 2 + jj) * 8 + (lane >> 2);
            bf[jj] = e[(nn * LDE + q) * 2 + le.b_comp];
          }
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int mf = mf0 + i;
            if (mf >= nmf) continue;
            const int t0 = mf * 4;
            if (ks * 2 + 1 < t0 || ks * 2 > t0 + 3 + nb - 1) continue;  // zero corner
            const int t = t0 + (lane >> 3);
            const int d = q - t;
            double av = 0.0;
            if (d >= 0 && d < nb) av = xsign(v[(t * nb + d) * 2 + le.a_comp], le.a_neg_conj);
#pragma unroll
            for (int jj = 0; jj < 2; jj++) dmma(acc[i][jj], av, bf[jj]);
          }
        }
        // store Y into sY[n][t]
        const int rp = (lane >> 2) & 1;
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int jj = 0; jj < 2; jj++) {
            const double send = rp ? acc[i][jj][0] : acc[i][jj][1];
            const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
            const int mf = mf0 + i;
            if (mf >= nmf) continue;
            const double2 val = rp ? make_double2(recv, acc[i][jj][1]) : make_double2(acc[i][jj][0], recv);
            const int t = mf * 4 + (lane >> 3);
            const int nn = (wn * 2 + jj) * 8 + (lane & 3) * 2 + rp;
            sY[nn * LDY + t] = val;
          }
      }
      __syncthreads();
      // ---- phase B: Y = T Y
      {
        double acc[4][2][2];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int jj = 0; jj < 2; jj++) acc[i][jj][0] = acc[i][jj][1] = 0.0;
        const double *y = reinterpret_cast<const double *>(sY);
        const double *t = reinterpret_cast<const double *>(sT);
        const int mf0 = wm * 4, nmf = g / 4;
        for (int ks = 0; ks < g / 2; ks++) {
          const int kb = ks * 2 + ((lane & 3) >> 1);
          double bf[2];
#pragma unroll
          for (int jj = 0; jj < 2; jj++) {
            const int nn = (wn * 2 + jj) * 8 + (lane >> 2);
            bf[jj] = y[(nn * LDY + kb) * 2 + le.b_comp];
          }
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int mf = mf0 + i;
            if (mf >= nmf) continue;
            if (ks * 2 + 1 < mf * 4) continue;   // T upper triangular
            const int ra = mf * 4 + (lane >> 3);
            const double av = xsign(t[(kb * LDT + ra) * 2 + le.a_comp], le.a_neg);
#pragma unroll
            for (int jj = 0; jj < 2; jj++) dmma(acc[i][jj], av, bf[jj]);
          }
        }
        __syncthreads();   // all reads of sY done
        const int rp = (lane >> 2) & 1;
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int jj = 0; jj < 2; jj++) {
            const double send = rp ? acc[i][jj][0] : acc[i][jj][1];
            const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
            const int mf = mf0 + i;
            if (mf >= nmf) continue;
            const double2 val = rp ? make_double2(recv, acc[i][jj][1]) : make_double2(acc[i][jj][0], recv);
            const int ta = mf * 4 + (lane >> 3);
            const int nn = (wn * 2 + jj) * 8 + (lane & 3) * 2 + rp;
            sY[nn * LDY + ta] = val;
          }
      }
      __syncthreads();
      // ---- phase C: E_win -= V Y   (2W real rows x QBN)
      {
        constexpr int MFC = 12;   // m-frags per warp (covers 2 x 12 x 4 = 96 complex rows)
        double acc[MFC][2][2];
#pragma unroll
        for (int i = 0; i < MFC; i++)
#pragma unroll
          for (int jj = 0; jj < 2; jj++) acc[i][jj][0] = acc[i][jj][1] = 0.0;
        const double *y = reinterpret_cast<const double *>(sY);
        const double *v = reinterpret_cast<const double *>(sV);
        const int nmf = (W + 3) / 4;
        for (int ks = 0; ks < g / 2; ks++) {
          const int kt = ks * 2 + ((lane & 3) >> 1);   // reflector index (k)
          double bf[2];
#pragma unroll
          for (int jj = 0; jj < 2; jj++) {
            const int nn = (wn * 2 + jj) * 8 + (lane >> 2);
            bf[jj] = y[(nn * LDY + kt) * 2 + le.b_comp];
          }
#pragma unroll
          for (int i = 0; i < MFC; i++) {
            const int mf = wm * MFC + i;
            if (mf >= nmf) continue;
            const int q0 = mf * 4;
            // nonzero t in [q0 - nb + 1, q0 + 3]
            if (ks * 2 > q0 + 3 || ks * 2 + 1 < q0 - nb + 1) continue;
            const int q = q0 + (lane >> 3);
            const int d = q - kt;
            double av = 0.0;
            if (d >= 0 && d < nb) av = xsign(v[(kt * nb + d) * 2 + le.a_comp], le.a_neg);
#pragma unroll
            for (int jj = 0; jj < 2; jj++) dmma(acc[i][jj], av, bf[jj]);
          }
        }
        const int rp = (lane >> 2) & 1;
#pragma unroll
        for (int i = 0; i < MFC; i++)
#pragma unroll
          for (int jj = 0; jj < 2; jj++) {
            const double send = rp ? acc[i][jj][0] : acc[i][jj][1];
            const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
            const int mf = wm * MFC + i;
            if (mf >= nmf) continue;
            const double2 val = rp ? make_double2(recv, acc[i][jj][1]) : make_double2(acc[i][jj][0], recv);
            const int q = mf * 4 + (lane >> 3);
            const int nn = (wn * 2 + jj) * 8 + (lane & 3) * 2 + rp;
            if (q < W) {
              double2 &ev = sE[nn * LDE + q];
              ev.x -= val.x;
              ev.y -= val.y;
            }
          }
      }
      __syncthreads();
      // ---- store the rows leaving the window; shift the overlap up
      {
        const bool lastj = (j == J - 1);
        const int nstore = lastj ? W : nb;
        for (int e = tid; e < QBN * nstore; e += QT) {
          const int q = e % nstore, c = e / nstore;
          const int64_t row = rs + q;
          if (row < a.n && c < ncols) a.E[row + (c0 + c) * a.lde] = sE[c * LDE + q];
        }
        if (!lastj) {
          __syncthreads();
          for (int e = tid; e < QBN * (g - 1); e += QT) {
            const int q = e % (g - 1), c = e / (g - 1);
            sE[c * LDE + q] = sE[c * LDE + nb + q];
          }
        }
        __threadfence();
        __syncthreads();
      }
    }
  }
}

// T factor per Q2 block: T upper g x g with H_{i0}...H_{i0+g-1} = I - V T V^H.
__global__ void q2_tfactor_kernel(int64_t n, int nb, int g, int64_t ngroups, const int64_t *first, const int64_t *off,
                                  const double2 *V2, const double2 *tau2, double2 *T2) {
  extern __shared__ __align__(16) double2 sm[];
  double2 *sV = sm;                // [g][nb]
  double2 *sG = sV + g * nb;       // [g][g]  G[x][y] at y*g + x
  double2 *sT = sG + g * g;        // [g][g]
  double2 *sTau = sT + g * g;      // [g]
  const int64_t blk = blockIdx.x;
  // find group: first[gi] <= blk < first[gi+1]
  int64_t lo = 0, hi = ngroups - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (first[mid] <= blk) lo = mid; else hi = mid - 1;
  }
  const int64_t gi = lo, j = blk - first[gi], i0 = gi * g;
  const int64_t last_i = n - 2 - j * nb;
  const int64_t nvalid = imax64(0, imin64(g, last_i - i0 + 1));
  const int tid = threadIdx.x;
  for (int e = tid; e < g * nb; e += blockDim.x) {
    const int t = e / nb;
    sV[e] = (t < nvalid) ? V2[(off[j] + i0) * nb + e] : czero();
  }
  for (int t = tid; t < g; t += blockDim.x) sTau[t] = (t < nvalid) ? tau2[off[j] + i0 + t] : czero();
  __syncthreads();
  for (int p = tid; p < g * g; p += blockDim.x) {
    const int x = p % g, y = p / g;
    double2 s = czero();
    if (x < y) {
      // rows q in [y, x+nb-1]: v_x[q-x], v_y[q-y]
      for (int q = y; q <= x + nb - 1; q++) s = cadd(s, cmulc(sV[x * nb + (q - x)], sV[y * nb + (q - y)]));
    }
    sG[p] = s;
    sT[p] = czero();
  }
  __syncthreads();
  for (int jj = 0; jj < g; jj++) {
    const double2 tj = sTau[jj];
    if (tid < jj) {
      const int i = tid;
      double2 s = czero();
      for (int l = i; l < jj; l++) s = cadd(s, cmul(sT[i + l * g], sG[l + jj * g]));
      sT[i + jj * g] = make_double2(-(tj.x * s.x - tj.y * s.y), -(tj.x * s.y + tj.y * s.x));
    }
    if (tid == 0) sT[jj + jj * g] = tj;
    __syncthreads();
  }
  for (int p = tid; p < g * g; p += blockDim.x) T2[blk * g * g + p] = sT[p];
}

__global__ void complexify_kernel(int64_t n, int64_t m, const double *Z, int64_t ldz, double2 *E, int64_t lde) {
  const int64_t total = n * m;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % n, c = e / n;
    E[r + c * lde] = make_double2(Z[r + c * ldz], 0.0);
  }
}

// Inverse of each bs x bs diagonal block of lower-triangular L (one CTA per block,
// one thread per column of the inverse: forward substitution on e_c).
__global__ void trinv_kernel(int64_t n, int bs, const double2 *L, int64_t ldl, double2 *Linv) {
  extern __shared__ __align__(16) double2 sm[];
  double2 *sL = sm;          // [bs][bs] column-major
  double2 *sX = sL + bs * bs;
  const int64_t b0 = (int64_t)blockIdx.x * bs;
  const int b = (int)imin64(bs, n - b0);
  for (int e = threadIdx.x; e < bs * bs; e += blockDim.x) {
    const int r = e % bs, c = e / bs;
    sL[e] = (r < b && c < b && r >= c) ? L[(b0 + r) + (b0 + c) * ldl] : (r == c ? make_double2(1.0, 0.0) : czero());
  }
  __syncthreads();
  const int c = threadIdx.x;
  if (c < bs) {
    for (int r = 0; r < bs; r++) {
      double2 s = (r == c) ? make_double2(1.0, 0.0) : czero();
      if (r >= c) {
        for (int k = c; k < r; k++) s = csub(s, cmul(sL[r + k * bs], sX[k + c * bs]));
        const double2 d = sL[r + r * bs];
        const double dd = d.x * d.x + d.y * d.y;
        s = make_double2((s.x * d.x + s.y * d.y) / dd, (s.y * d.x - s.x * d.y) / dd);
      } else {
        s = czero();
      }
      sX[r + c * bs] = s;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < bs * bs; e += blockDim.x) Linv[(int64_t)blockIdx.x * bs * bs + e] = sX[e];
}

}  // namespace

int q2_tfactors(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *tau2, double2 *T2) {
  if (p.nblocks <= 0) return 0;
  const size_t smem = ((size_t)p.g * p.nb + 2 * p.g * p.g + p.g) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    EIG_TRY(ctx.check(cudaFuncSetAttribute(q2_tfactor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024),
                      "q2t attr"));
    attr = true;
  }
  q2_tfactor_kernel<<<(unsigned)p.nblocks, 128, smem, ctx.stream>>>(p.n, p.nb, p.g, p.ngroups, p.d_group_first_block,
                                                                    p.d_off, V2, tau2, T2);
  return ctx.launched("q2_tfactor_kernel");
}

int q2_apply(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *T2, double2 *E, int64_t lde, int64_t m) {
  if (p.nblocks <= 0 || m <= 0) return 0;
  if (p.g > QMAXG || p.nb > QMAXNB || p.g % 4 != 0 || p.g < 4 || p.nb < p.g - 1) return -1;
  Q2Args a;
  a.n = p.n;
  a.m = m;
  a.lde = lde;
  a.nb = p.nb;
  a.g = p.g;
  a.W = p.nb + p.g - 1;
  const int Wp = (a.W + 1) & ~1;
  a.LDE = Wp;
  while (a.LDE % 8 != 2) a.LDE++;
  a.LDY = p.g + 2;
  a.LDT = p.g + 4;
  a.ngroups = p.ngroups;
  a.first = p.d_group_first_block;
  a.off = p.d_off;
  a.V2 = V2;
  a.T2 = T2;
  a.E = E;
  const size_t smem = ((size_t)p.g * p.nb + (size_t)p.g * a.LDT + (size_t)QBN * a.LDE + (size_t)QBN * a.LDY) *
                      sizeof(double2);
  static bool attr = false;
  if (!attr) {
    EIG_TRY(ctx.check(cudaFuncSetAttribute(apply_q2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024),
                      "q2 attr"));
    attr = true;
  }
  const unsigned slabs = (unsigned)((m + QBN - 1) / QBN);
  apply_q2_kernel<<<slabs, QT, smem, ctx.stream>>>(a);
  return ctx.launched("apply_q2_kernel");
}

int complexify(Ctx &ctx, int64_t n, int64_t m, const double *Z, int64_t ldz, double2 *E, int64_t lde) {
  if (n <= 0 || m <= 0) return 0;
  const int64_t total = n * m;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * ctx.num_sms);
  complexify_kernel<<<blocks, 256, 0, ctx.stream>>>(n, m, Z, ldz, E, lde);
  return ctx.launched("complexify_kernel");
}

int trinv_blocks(Ctx &ctx, int64_t n, int bs, const double2 *L, int64_t ldl, double2 *Linv) {
  if (n <= 0) return 0;
  const int64_t nblk = (n + bs - 1) / bs;
  const size_t smem = (size_t)2 * bs * bs * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    EIG_TRY(ctx.check(cudaFuncSetAttribute(trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024),
                      "trinv attr"));
    attr = true;
  }
  trinv_kernel<<<(unsigned)nblk, std::max(bs, 32), smem, ctx.stream>>>(n, bs, L, ldl, Linv);
  return ctx.launched("trinv_kernel");
}

}  // namespace eig
