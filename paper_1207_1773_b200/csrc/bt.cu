// bt.cu — back-transform kernels: grouped Q2 blocks (a6), complexify (a6),
// diagonal-block inverses for the blocked L^-H solve (a8).
//
// Q2 (reading R7): T factor of each grouped block (the application
// kernel is in q2.cu).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

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

// Plan tables on the device (no host staging, no synchronisation):
//   off[j] = sum_{j' < j} (n - 1 - j' nb) = j (n - 1) - nb j (j - 1) / 2   (V2 slot offsets)
//   first[gi] = number of Q2 blocks in the groups before gi (group gi = sweeps gi*g ..)
__global__ void plan_tables_kernel(int64_t n, int nb, int g, int64_t ngroups, int64_t J, int64_t *first,
                                   int64_t *off) {
  for (int64_t j = threadIdx.x; j < J; j += blockDim.x) off[j] = j * (n - 1) - (int64_t)nb * j * (j - 1) / 2;
  if (first && threadIdx.x == 0) {
    int64_t tot = 0;
    for (int64_t gi = 0; gi < ngroups; gi++) {
      first[gi] = tot;
      const int64_t i0 = gi * g;
      tot += (i0 > n - 2) ? 0 : (n - 2 - i0) / nb + 1;
    }
    first[ngroups] = tot;
  }
}

}  // namespace

int plan_tables(Ctx &ctx, int64_t n, int nb, int g, int64_t ngroups, int64_t J, int64_t *first, int64_t *off) {
  if (J <= 0 && !first) return 0;
  plan_tables_kernel<<<1, 256, 0, ctx.stream>>>(n, nb, g, ngroups, J, first, off);
  return ctx.launched("plan_tables_kernel");
}

int q2_tfactors(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *tau2, double2 *T2) {
  if (p.nblocks <= 0) return 0;
  const size_t smem = ((size_t)p.g * p.nb + 2 * p.g * p.g + p.g) * sizeof(double2);
  EIG_TRY(ctx.smem_attr((const void *)q2_tfactor_kernel, 100 * 1024, "q2t attr"));
  q2_tfactor_kernel<<<(unsigned)p.nblocks, 128, smem, ctx.stream>>>(p.n, p.nb, p.g, p.ngroups, p.d_group_first_block,
                                                                    p.d_off, V2, tau2, T2);
  return ctx.launched("q2_tfactor_kernel");
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
  EIG_TRY(ctx.smem_attr((const void *)trinv_kernel, 140 * 1024, "trinv attr"));
  trinv_kernel<<<(unsigned)nblk, std::max(bs, 32), smem, ctx.stream>>>(n, bs, L, ldl, Linv);
  return ctx.launched("trinv_kernel");
}

}  // namespace eig
