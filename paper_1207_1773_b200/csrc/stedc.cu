// stedc.cu — tridiagonal divide and conquer on the device (NEXT-2).
//
// Paper §4.3: split T recursively, then merge
//   T = diag(T1, T2) + rho v v^T
//     = diag(Z1, Z2) (diag(L1, L2) + rho u u^T) diag(Z1, Z2)^T,
// solve the rank-one modified problem (the paper does this on the CPU, here
// on the device), and update the eigenvectors with a matrix product
// ("the GPU updates the eigenvectors with a matrix-matrix
// multiplication").  At the last merge only the requested eigenvectors are
// formed.  Gu-Eisenstat recomputation of u keeps the eigenvectors
// orthogonal; deflation follows the classical small-|u_i| and close-pole
// (Givens) criteria.
//
// Device layout: the tree nodes of one height are disjoint index ranges, so
// every per-node array is a length-n array indexed by global position; the
// eigenvector blocks live on the block diagonal of n x n buffers (ping-pong
// between heights).  Leaves (<= 32) are solved by one warp each with cyclic
// Jacobi; merges use one CTA for the sort/deflation scan, thread-per-root
// bisection on the secular equation, thread-per-entry Gu-Eisenstat products,
// and a grouped real DGEMM on the DMMA pipe for Z_old Q.
#include <algorithm>
#include <cfloat>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int LEAF = 32;
constexpr int PT = 256;
constexpr int KSMEM = 12288;   // merge sizes whose (D, z) fit in shared memory for the deflation scan

struct Node {
  int64_t lo, mid, hi;
};
// per-node counters: [0] K' (non-deflated), [1] KD (deflated), [2] NR (rotations),
// [3] Kneed, [4] K1 / [5] K3 / [6] K2 non-deflated columns of child 1 only, mixed, child 2 only
constexpr int NCNT = 8;

struct DcBufs {
  int64_t n;
  const double *d, *e;
  double *w;          // eigenvalues (children on input, merged on output)
  double *Zold, *Znew, *Q, *Zg, *Zt;   // n x n, ld n
  double *Ds, *zs;    // sorted poles / normalized u (global positions)
  int *perm;          // local column of each sorted position
  double *Dn, *zn;    // non-deflated poles, z
  int *cn;            // their local columns
  double *Dd;         // deflated values
  int *cd;            // their local columns
  int *rc0, *rc1;     // Givens rotations (local columns)
  double *rcc, *rcs;
  int *org;           // secular root origin (non-deflated index)
  double *tau;        // root offset from its origin pole
  double *zh;         // Gu-Eisenstat z-hat
  int *qcol;          // root j -> compact needed column (or -1)
  int64_t *fpos;      // final position of root j (at lo + j)
  double *DdS;        // deflated values sorted ascending
  int *cdS;           // and their local columns
  int64_t *fposd;     // final position of sorted deflated t (at lo + t)
  int *cnt;           // per node: NCNT counters (see Node)
  int *cpos;          // non-deflated column i -> its position in type order [child 1 | mixed | child 2]
  double *rho;        // per node: rho * |u|^2
  const Node *nodes;
  int64_t il, iu;     // selection (only for the root node)
  double *Zout;       // root output (n x m), ld ldz
  int64_t ldz;
};

// ------------------------------------------------------------------ leaves
// One warp per leaf: cyclic Jacobi on the (modified) leaf tridiagonal.
__global__ void dc_leaf_kernel(DcBufs b, const int64_t *leaf_lo, const int64_t *leaf_hi, int nleaves) {
  __shared__ double sS[2][LEAF][LEAF + 1];
  __shared__ double sV[2][LEAF][LEAF + 1];
  __shared__ int sP[2][LEAF];
  const int lw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int leaf = blockIdx.x * 2 + lw;
  if (leaf >= nleaves) return;
  const int64_t lo = leaf_lo[leaf], hi = leaf_hi[leaf], n = b.n;
  const int k = (int)(hi - lo);
  double(*S)[LEAF + 1] = sS[lw];
  double(*V)[LEAF + 1] = sV[lw];
  for (int c = 0; c < k; c++) {
    if (lane < k) {
      S[lane][c] = 0.0;
      V[lane][c] = (lane == c) ? 1.0 : 0.0;
    }
  }
  __syncwarp();
  if (lane < k) {
    const int64_t g = lo + lane;
    double dg = b.d[g];
    if (lane == 0 && lo > 0) dg -= fabs(b.e[lo - 1]);        // split adjustments (Cuppen)
    if (lane == k - 1 && hi < n) dg -= fabs(b.e[hi - 1]);
    S[lane][lane] = dg;
    if (lane + 1 < k) {
      S[lane + 1][lane] = b.e[g];
      S[lane][lane + 1] = b.e[g];
    }
  }
  __syncwarp();
  for (int sweep = 0; sweep < 30; sweep++) {
    double off = 0.0, tot = 0.0;
    for (int c = 0; c < k; c++)
      if (lane < k) {
        const double x = S[lane][c] * S[lane][c];
        tot += x;
        if (lane != c) off += x;
      }
    off = warp_sum(off);
    tot = warp_sum(tot);
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < k - 1; p++)
      for (int q = p + 1; q < k; q++) {
        const double apq = S[p][q];
        if (apq == 0.0) continue;
        const double th = (S[q][q] - S[p][p]) / (2.0 * apq);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
        const double c = 1.0 / sqrt(1.0 + t * t), s = t * c;
        __syncwarp();
        if (lane < k) {   // columns
          const double xp = S[lane][p], xq = S[lane][q];
          S[lane][p] = c * xp - s * xq;
          S[lane][q] = s * xp + c * xq;
          const double vp = V[lane][p], vq = V[lane][q];
          V[lane][p] = c * vp - s * vq;
          V[lane][q] = s * vp + c * vq;
        }
        __syncwarp();
        if (lane < k) {   // rows
          const double xp = S[p][lane], xq = S[q][lane];
          S[p][lane] = c * xp - s * xq;
          S[q][lane] = s * xp + c * xq;
        }
        __syncwarp();
        if (lane == 0) {
          S[p][q] = 0.0;
          S[q][p] = 0.0;
        }
        __syncwarp();
      }
  }
  // sort ascending (stable) by rank
  if (lane < k) {
    const double x = S[lane][lane];
    int r = 0;
    for (int c = 0; c < k; c++) {
      const double y = S[c][c];
      if (y < x || (y == x && c < lane)) r++;
    }
    sP[lw][r] = lane;
    b.w[lo + r] = x;
  }
  __syncwarp();
  for (int c = 0; c < k; c++)
    if (lane < k) b.Zold[(lo + lane) + (lo + c) * n] = V[lane][sP[lw][c]];
}

// ------------------------------------------------------------------ merge: sort + deflation
__device__ double block_sum(double v, double *red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

__device__ double block_max(double v, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
  }
  __syncthreads();
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(PT) dc_prep_kernel(DcBufs b) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[32];
  __shared__ int s_cnt[3];
  const Node nd = b.nodes[blockIdx.x];
  const int64_t n = b.n, lo = nd.lo, mid = nd.mid, hi = nd.hi;
  const int k1 = (int)(mid - lo), k2 = (int)(hi - mid), k = (int)(hi - lo);
  const double beta = b.e[mid - 1];
  const double rho = fabs(beta), sg = beta >= 0.0 ? 1.0 : -1.0;
  const int tid = threadIdx.x;
  // merge the two sorted child spectra; u = (last row of Z1, sg * first row of Z2)
  for (int a = tid; a < k1; a += PT) {
    const double v = b.w[lo + a];
    int l = 0, h = k2;   // # child-2 values < v
    while (l < h) {
      const int m = (l + h) >> 1;
      if (b.w[mid + m] < v) l = m + 1; else h = m;
    }
    const int64_t r = lo + a + l;
    b.Ds[r] = v;
    b.zs[r] = b.Zold[(mid - 1) + (lo + a) * n];
    b.perm[r] = a;
  }
  for (int c = tid; c < k2; c += PT) {
    const double v = b.w[mid + c];
    int l = 0, h = k1;   // # child-1 values <= v
    while (l < h) {
      const int m = (l + h) >> 1;
      if (b.w[lo + m] <= v) l = m + 1; else h = m;
    }
    const int64_t r = lo + c + l;
    b.Ds[r] = v;
    b.zs[r] = sg * b.Zold[mid + (mid + c) * n];
    b.perm[r] = k1 + c;
  }
  __syncthreads();
  double s2 = 0.0, dm = 0.0;
  for (int i = tid; i < k; i += PT) {
    const double z = b.zs[lo + i];
    s2 += z * z;
    dm = fmax(dm, fabs(b.Ds[lo + i]));
  }
  const double nrm2 = block_sum(s2, red);
  const double dmax = block_max(dm, red);
  const double rho2 = rho * nrm2;
  const double inv = nrm2 > 0.0 ? 1.0 / sqrt(nrm2) : 0.0;
  const bool use_smem = k <= KSMEM;
  double *D = use_smem ? sm : b.Ds + lo;
  double *z = use_smem ? sm + k : b.zs + lo;
  for (int i = tid; i < k; i += PT) {
    const double zi = b.zs[lo + i] * inv;
    b.zs[lo + i] = zi;
    if (use_smem) {
      D[i] = b.Ds[lo + i];
      z[i] = zi;
    }
  }
  __syncthreads();
  if (tid == 0) {
    const double tol = 8.0 * DBL_EPSILON * fmax(dmax, rho2);
    int K = 0, KD = 0, NR = 0, pj = -1;
    // column types (LAPACK dlaed2 ctot): 1 = rows of child 1 only, 2 = child 2
    // only, 3 = mixed by a rotation; tpj is the type of the pending column pj
    int tpj = 0;
    auto type0 = [&](int j) { return b.perm[lo + j] < k1 ? 1 : 2; };
    for (int j = 0; j < k; j++) {
      const double zj = z[j];
      if (rho2 * fabs(zj) <= tol) {
        b.Dd[lo + KD] = D[j];
        b.cd[lo + KD] = b.perm[lo + j];
        KD++;
        continue;
      }
      if (pj < 0) {
        pj = j;
        tpj = type0(j);
        continue;
      }
      double s = z[pj], c = zj;
      const double t = D[j] - D[pj];
      const double ta = hypot(c, s);
      c /= ta;
      s = -s / ta;
      if (fabs(t * c * s) <= tol) {
        // close poles: rotate columns (pj, j) so that z[pj] = 0, deflate pj
        z[j] = ta;
        z[pj] = 0.0;
        b.rc0[lo + NR] = b.perm[lo + pj];
        b.rc1[lo + NR] = b.perm[lo + j];
        b.rcc[lo + NR] = c;
        b.rcs[lo + NR] = s;
        NR++;
        const double td = D[pj] * c * c + D[j] * s * s;
        D[j] = D[pj] * s * s + D[j] * c * c;
        D[pj] = td;
        b.Dd[lo + KD] = D[pj];
        b.cd[lo + KD] = b.perm[lo + pj];
        KD++;
        pj = j;
        tpj |= type0(j);
      } else {
        b.Dn[lo + K] = D[pj];
        b.zn[lo + K] = z[pj];
        b.cn[lo + K] = b.perm[lo + pj];
        b.cpos[lo + K] = tpj;
        K++;
        pj = j;
        tpj = type0(j);
      }
    }
    if (pj >= 0) {
      b.Dn[lo + K] = D[pj];
      b.zn[lo + K] = z[pj];
      b.cn[lo + K] = b.perm[lo + pj];
      b.cpos[lo + K] = tpj;
      K++;
    }
    // type order [child 1 | mixed | child 2]: the merge GEMM then skips the
    // zero blocks of diag(Z1, Z2)
    int K1 = 0, K3 = 0, K2 = 0;
    for (int i = 0; i < K; i++) {
      const int t = b.cpos[lo + i];
      K1 += t == 1;
      K3 += t == 3;
      K2 += t == 2;
    }
    int p1 = 0, p3 = K1, p2 = K1 + K3;
    for (int i = 0; i < K; i++) {
      const int t = b.cpos[lo + i];
      b.cpos[lo + i] = t == 1 ? p1++ : (t == 3 ? p3++ : p2++);
    }
    b.cnt[blockIdx.x * NCNT + 4] = K1;
    b.cnt[blockIdx.x * NCNT + 5] = K3;
    b.cnt[blockIdx.x * NCNT + 6] = K2;
    s_cnt[0] = K;
    s_cnt[1] = KD;
    s_cnt[2] = NR;
    b.cnt[blockIdx.x * NCNT + 0] = K;
    b.cnt[blockIdx.x * NCNT + 1] = KD;
    b.cnt[blockIdx.x * NCNT + 2] = NR;
    b.rho[blockIdx.x] = rho2;
  }
  __syncthreads();
  // Givens rotations on the (full-height) columns of the node's eigenvector block
  const int NR = s_cnt[2];
  for (int r = tid; r < k; r += PT) {
    double *zr = b.Zold + (lo + r);
    for (int t = 0; t < NR; t++) {
      const int64_t c0 = lo + b.rc0[lo + t], c1 = lo + b.rc1[lo + t];
      const double c = b.rcc[lo + t], s = b.rcs[lo + t];
      const double x = zr[c0 * n], y = zr[c1 * n];
      zr[c0 * n] = c * x + s * y;
      zr[c1 * n] = c * y - s * x;
    }
  }
}

// ------------------------------------------------------------------ secular equation
// f(lambda) = 1 + rho sum_i z_i^2 / (D_i - lambda), increasing between poles;
// root j is stored as (origin pole, offset tau) for accurate gaps.
// One warp per root: every lane sums a strided share of the K terms and the
// shares are combined with a fixed butterfly (deterministic), so the O(K^2)
// bisection runs on all SMs instead of K threads.
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_allprod(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v *= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void dc_secular_kernel(DcBufs b) {
  const Node nd = b.nodes[blockIdx.y];
  const int K = b.cnt[blockIdx.y * NCNT + 0];
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= K) return;   // warp-uniform
  const int64_t lo = nd.lo;
  const double *D = b.Dn + lo, *z = b.zn + lo;
  const double rho = b.rho[blockIdx.y];
  int og;
  double tl, th;
  if (j < K - 1) {
    const double half = 0.5 * (D[j + 1] - D[j]);
    double f = 0.0;
    for (int i = lane; i < K; i += 32) f += rho * z[i] * z[i] / ((D[i] - D[j]) - half);
    f = 1.0 + warp_allsum(f);
    if (f >= 0.0) {
      og = j;
      tl = 0.0;
      th = half;
    } else {
      og = j + 1;
      tl = -half;
      th = 0.0;
    }
  } else {
    double sq = 0.0;
    for (int i = lane; i < K; i += 32) sq += z[i] * z[i];
    sq = warp_allsum(sq);
    og = K - 1;
    tl = 0.0;
    th = rho * sq;
  }
  const double Do = D[og];
  for (int it = 0; it < 200; it++) {
    const double tm = 0.5 * (tl + th);
    if (tm <= tl || tm >= th) break;
    double f = 0.0;
    for (int i = lane; i < K; i += 32) f += rho * z[i] * z[i] / ((D[i] - Do) - tm);
    f = 1.0 + warp_allsum(f);
    if (f > 0.0) th = tm; else tl = tm;
  }
  if (lane == 0) {
    b.org[lo + j] = og;
    b.tau[lo + j] = 0.5 * (tl + th);
  }
}

// Gu-Eisenstat: zh_i^2 = ((lambda_i - D_i)/rho) prod_{j != i} (lambda_j - D_i)/(D_j - D_i)
// (one warp per i, strided partial products combined with a fixed butterfly)
__global__ void dc_zhat_kernel(DcBufs b) {
  const Node nd = b.nodes[blockIdx.y];
  const int K = b.cnt[blockIdx.y * NCNT + 0];
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= K) return;   // warp-uniform
  const int64_t lo = nd.lo;
  const double *D = b.Dn + lo;
  const double rho = b.rho[blockIdx.y];
  const double Di = D[i];
  auto lam_minus_Di = [&](int j) { return (D[b.org[lo + j]] - Di) + b.tau[lo + j]; };
  double p = 1.0;
  for (int j = lane; j < K; j += 32)
    if (j != i) p *= lam_minus_Di(j) / (D[j] - Di);
  p = warp_allprod(p) * (lam_minus_Di(i) / rho);
  if (lane == 0) {
    const double zi = b.zn[lo + i];
    b.zh[lo + i] = copysign(sqrt(fabs(p)), zi);
  }
}

// Final order of the node's k eigenpairs: roots (ascending) merged with the
// sorted deflated values; w receives the merged spectrum; qcol numbers the
// roots whose final position is selected.
__global__ void __launch_bounds__(PT) dc_order_kernel(DcBufs b, int root_node) {
  extern __shared__ __align__(16) double sm[];
  const Node nd = b.nodes[blockIdx.x];
  const int64_t lo = nd.lo;
  const int K = b.cnt[blockIdx.x * NCNT + 0], KD = b.cnt[blockIdx.x * NCNT + 1];
  const int tid = threadIdx.x;
  const bool root = (int)blockIdx.x == root_node;
  double *DdS = b.DdS + lo;
  int *cdS = b.cdS + lo;
  // rank the deflated values (ties by index) and scatter into sorted order
  for (int t = tid; t < KD; t += PT) {
    const double x = b.Dd[lo + t];
    int r = 0;
    for (int u = 0; u < KD; u++) {
      const double y = b.Dd[lo + u];
      if (y < x || (y == x && u < t)) r++;
    }
    DdS[r] = x;
    cdS[r] = b.cd[lo + t];
  }
  __syncthreads();
  // roots: lambda_j = D[org] + tau
  for (int j = tid; j < K; j += PT) {
    const double lam = b.Dn[lo + b.org[lo + j]] + b.tau[lo + j];
    int l = 0, h = KD;   // # deflated < lam
    while (l < h) {
      const int m = (l + h) >> 1;
      if (DdS[m] < lam) l = m + 1; else h = m;
    }
    const int64_t pos = j + l;
    b.w[lo + pos] = lam;
    b.fpos[lo + j] = pos;
  }
  // deflated
  for (int t = tid; t < KD; t += PT) {
    const double x = DdS[t];
    int l = 0, h = K;    // # roots <= x
    while (l < h) {
      const int m = (l + h) >> 1;
      const double lam = b.Dn[lo + b.org[lo + m]] + b.tau[lo + m];
      if (lam <= x) l = m + 1; else h = m;
    }
    const int64_t pos = t + l;
    b.w[lo + pos] = x;
    b.fposd[lo + t] = pos;
  }
  __syncthreads();
  // needed roots -> compact Q columns (ascending root order)
  if (tid == 0) {
    int q = 0;
    for (int j = 0; j < K; j++) {
      const int64_t pos = b.fpos[lo + j];
      const bool need = !root || (pos >= b.il - 1 && pos <= b.iu - 1);
      b.qcol[lo + j] = need ? q++ : -1;
    }
    b.cnt[blockIdx.x * NCNT + 3] = q;
  }
}

// Q column for root j (one block per needed root): q_i = zh_i / (D_i - lambda_j), normalized.
__global__ void __launch_bounds__(PT) dc_qbuild_kernel(DcBufs b) {
  __shared__ double red[32];
  const Node nd = b.nodes[blockIdx.y];
  const int64_t lo = nd.lo, n = b.n;
  const int K = b.cnt[blockIdx.y * NCNT + 0];
  const int j = blockIdx.x;
  if (j >= K) return;
  const int qc = b.qcol[lo + j];
  if (qc < 0) return;
  const double *D = b.Dn + lo;
  const double Do = D[b.org[lo + j]], tj = b.tau[lo + j];
  double *q = b.Q + lo + (lo + qc) * n;
  double s2 = 0.0;
  for (int i = threadIdx.x; i < K; i += PT) {
    const double v = b.zh[lo + i] / ((D[i] - Do) - tj);
    q[b.cpos[lo + i]] = v;   // row in type order (matches the gathered columns)
    s2 += v * v;
  }
  const double inv = 1.0 / sqrt(block_sum(s2, red));
  for (int i = threadIdx.x; i < K; i += PT) q[i] *= inv;
}

// Zg[:, i] = Zold[lo:hi, lo + cn_i]  (non-deflated columns, gathered)
__global__ void dc_gather_kernel(DcBufs b) {
  const Node nd = b.nodes[blockIdx.y];
  const int64_t lo = nd.lo, n = b.n;
  const int k = (int)(nd.hi - nd.lo);
  const int K = b.cnt[blockIdx.y * NCNT + 0];
  const int64_t total = (int64_t)k * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % k), i = (int)(e / k);
    b.Zg[(lo + r) + (lo + b.cpos[lo + i]) * n] = b.Zold[(lo + r) + (lo + b.cn[lo + i]) * n];
  }
}

// Scatter: roots from Zt (GEMM output, compact needed columns), deflated
// columns from Zold, into Znew (or the root output) at their final positions.
__global__ void dc_scatter_kernel(DcBufs b, int root_node) {
  const int node = blockIdx.y;
  const Node nd = b.nodes[node];
  const int64_t lo = nd.lo, n = b.n;
  const int k = (int)(nd.hi - nd.lo);
  const int K = b.cnt[node * NCNT + 0], KD = b.cnt[node * NCNT + 1];
  const bool root = node == root_node;
  const int64_t total = (int64_t)k * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % k), src = (int)(e / k);   // src < K: root; else deflated (sorted index src - K)
    int64_t pos;
    double v;
    if (src < K) {
      const int qc = b.qcol[lo + src];
      if (qc < 0) continue;
      pos = b.fpos[lo + src];
      v = b.Zt[(lo + r) + (lo + qc) * n];
    } else {
      const int t = src - K;
      if (t >= KD) continue;
      pos = b.fposd[lo + t];
      if (root && (pos < b.il - 1 || pos > b.iu - 1)) continue;
      v = b.Zold[(lo + r) + (lo + b.cdS[lo + t]) * n];
    }
    if (root) b.Zout[(lo + r) + (pos - (b.il - 1)) * b.ldz] = v;
    else b.Znew[(lo + r) + (lo + pos) * n] = v;
  }
}

// Zold[lo:hi, lo:hi] = Znew[lo:hi, lo:hi] for every node of the level (the
// tree is not balanced, so a block must stay in Zold until its parent merges).
__global__ void dc_copyback_kernel(DcBufs b) {
  const Node nd = b.nodes[blockIdx.y];
  const int64_t lo = nd.lo, n = b.n;
  const int k = (int)(nd.hi - nd.lo);
  const int64_t total = (int64_t)k * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e % k), col = (int)(e / k);
    b.Zold[(lo + r) + (lo + col) * n] = b.Znew[(lo + r) + (lo + col) * n];
  }
}

}  // namespace

int stedc(Ctx &c, int64_t n, const double *d, const double *e, int64_t il, int64_t iu, double *w, double *Z,
          int64_t ldz) {
  if (n <= 0) return 0;
  if (il < 1 || iu > n || il > iu) return -5;
  // ---- tree (host): leaves <= LEAF, merges grouped by height
  std::vector<int64_t> leaf_lo, leaf_hi;
  std::vector<std::vector<Node>> levels;
  struct Rec {
    static int build(int64_t lo, int64_t hi, std::vector<int64_t> &llo, std::vector<int64_t> &lhi,
                     std::vector<std::vector<Node>> &lv) {
      if (hi - lo <= LEAF) {
        llo.push_back(lo);
        lhi.push_back(hi);
        return 0;
      }
      const int64_t mid = lo + (hi - lo) / 2;
      const int h = std::max(build(lo, mid, llo, lhi, lv), build(mid, hi, llo, lhi, lv)) + 1;
      if ((int)lv.size() <= h) lv.resize(h + 1);
      lv[h].push_back(Node{lo, mid, hi});
      return h;
    }
  };
  const int H = Rec::build(0, n, leaf_lo, leaf_hi, levels);
  // ---- workspace
  const size_t nn = (size_t)n * n;
  const size_t nd = (size_t)n;
  size_t bytes = 5 * nn * sizeof(double) + 9 * nd * sizeof(double) + 10 * nd * sizeof(int64_t) +
                 (size_t)(leaf_lo.size() * 2) * sizeof(int64_t) + 32 * 256;   // + alignment of each take
  char *wsp = (char *)c.ws(WS_DC, bytes);
  if (!wsp) return EIG_ERR_NOMEM;
  auto take = [&](size_t b) {
    char *p = wsp;
    wsp += (b + 255) & ~(size_t)255;
    return p;
  };
  DcBufs b;
  b.n = n;
  b.d = d;
  b.e = e;
  b.w = w;
  b.Zold = (double *)take(nn * 8);
  b.Znew = (double *)take(nn * 8);
  b.Q = (double *)take(nn * 8);
  b.Zg = (double *)take(nn * 8);
  b.Zt = (double *)take(nn * 8);
  b.Ds = (double *)take(nd * 8);
  b.zs = (double *)take(nd * 8);
  b.Dn = (double *)take(nd * 8);
  b.zn = (double *)take(nd * 8);
  b.Dd = (double *)take(nd * 8);
  b.rcc = (double *)take(nd * 8);
  b.rcs = (double *)take(nd * 8);
  b.tau = (double *)take(nd * 8);
  b.zh = (double *)take(nd * 8);
  b.DdS = (double *)take(nd * 8);
  b.perm = (int *)take(nd * 4);
  b.cn = (int *)take(nd * 4);
  b.cd = (int *)take(nd * 4);
  b.rc0 = (int *)take(nd * 4);
  b.rc1 = (int *)take(nd * 4);
  b.org = (int *)take(nd * 4);
  b.qcol = (int *)take(nd * 4);
  b.cdS = (int *)take(nd * 4);
  b.cpos = (int *)take(nd * 4);
  b.fpos = (int64_t *)take(nd * 8);
  b.fposd = (int64_t *)take(nd * 8);
  int64_t *d_llo = (int64_t *)take(leaf_lo.size() * 8), *d_lhi = (int64_t *)take(leaf_lo.size() * 8);
  b.il = il;
  b.iu = iu;
  b.Zout = Z;
  b.ldz = ldz;
  // per-level node arrays / counters (small, separate buffer)
  size_t maxnodes = 1;
  for (auto &lv : levels) maxnodes = std::max(maxnodes, lv.size());
  char *small = (char *)c.ws(WS_DC_SMALL, maxnodes * (sizeof(Node) + NCNT * sizeof(int) + sizeof(double) +
                                                       2 * sizeof(DgemmProb)) + 4096);
  if (!small) return EIG_ERR_NOMEM;
  Node *d_nodes = (Node *)small;
  int *d_cnt = (int *)(small + ((maxnodes * sizeof(Node) + 255) & ~(size_t)255));
  double *d_rho = (double *)((char *)d_cnt + ((maxnodes * NCNT * sizeof(int) + 255) & ~(size_t)255));
  DgemmProb *d_probs = (DgemmProb *)((char *)d_rho + ((maxnodes * sizeof(double) + 255) & ~(size_t)255));
  b.cnt = d_cnt;
  b.rho = d_rho;
  b.nodes = d_nodes;
  // ---- leaves
  EIG_TRY(c.check(cudaMemsetAsync(b.Zold, 0, nn * 8, c.stream), "zero Z"));
  EIG_TRY(c.check(cudaMemcpyAsync(d_llo, leaf_lo.data(), leaf_lo.size() * 8, cudaMemcpyHostToDevice, c.stream), "leaves"));
  EIG_TRY(c.check(cudaMemcpyAsync(d_lhi, leaf_hi.data(), leaf_hi.size() * 8, cudaMemcpyHostToDevice, c.stream), "leaves"));
  const int nleaves = (int)leaf_lo.size();
  dc_leaf_kernel<<<(nleaves + 1) / 2, 64, 0, c.stream>>>(b, d_llo, d_lhi, nleaves);
  EIG_TRY(c.launched("dc_leaf_kernel"));
  if (H == 0) {
    // a single leaf: copy the selected columns
    EIG_TRY(c.check(cudaMemcpy2DAsync(Z, ldz * 8, b.Zold + (il - 1) * n, n * 8, n * 8, iu - il + 1,
                                      cudaMemcpyDeviceToDevice, c.stream), "leaf out"));
    return c.check(cudaStreamSynchronize(c.stream), "sync");   // host vectors go out of scope
  }
  EIG_TRY(c.smem_attr((const void *)dc_prep_kernel, 2 * KSMEM * 8, "dc attr"));
  std::vector<int> cnt;
  std::vector<DgemmProb> probs;
  for (int h = 1; h <= H; h++) {
    const std::vector<Node> &lv = levels[h];
    const int nn_ = (int)lv.size();
    const bool top = (h == H);
    int64_t kmax = 0;
    for (auto &x : lv) kmax = std::max(kmax, x.hi - x.lo);
    EIG_TRY(c.check(cudaMemcpyAsync(d_nodes, lv.data(), nn_ * sizeof(Node), cudaMemcpyHostToDevice, c.stream),
                    "nodes"));
    const size_t psm = 2 * (size_t)std::min<int64_t>(kmax, KSMEM) * 8;
    dc_prep_kernel<<<nn_, PT, psm, c.stream>>>(b);
    EIG_TRY(c.launched("dc_prep_kernel"));
    cnt.resize(NCNT * nn_);
    EIG_TRY(c.check(cudaMemcpyAsync(cnt.data(), d_cnt, NCNT * nn_ * sizeof(int), cudaMemcpyDeviceToHost, c.stream), "cnt"));
    EIG_TRY(c.check(cudaStreamSynchronize(c.stream), "sync cnt"));
    int Kmax = 0;
    for (int i = 0; i < nn_; i++) Kmax = std::max(Kmax, cnt[NCNT * i]);
    if (Kmax > 0) {
      dc_secular_kernel<<<dim3((Kmax + 7) / 8, nn_), 256, 0, c.stream>>>(b);   // 8 roots (warps) per CTA
      EIG_TRY(c.launched("dc_secular_kernel"));
      dc_zhat_kernel<<<dim3((Kmax + 7) / 8, nn_), 256, 0, c.stream>>>(b);
      EIG_TRY(c.launched("dc_zhat_kernel"));
    }
    dc_order_kernel<<<nn_, PT, 0, c.stream>>>(b, top ? 0 : -1);
    EIG_TRY(c.launched("dc_order_kernel"));
    EIG_TRY(c.check(cudaMemcpyAsync(cnt.data(), d_cnt, NCNT * nn_ * sizeof(int), cudaMemcpyDeviceToHost, c.stream), "cnt"));
    EIG_TRY(c.check(cudaStreamSynchronize(c.stream), "sync cnt"));
    if (Kmax > 0) {
      dc_qbuild_kernel<<<dim3(Kmax, nn_), PT, 0, c.stream>>>(b);
      EIG_TRY(c.launched("dc_qbuild_kernel"));
      dc_gather_kernel<<<dim3(std::max<int64_t>(1, std::min<int64_t>(4096, kmax * Kmax / 256 + 1)), nn_), 256, 0,
                         c.stream>>>(b);
      EIG_TRY(c.launched("dc_gather_kernel"));
      probs.clear();
      int max_tiles = 0;
      for (int i = 0; i < nn_; i++) {
        const int K = cnt[NCNT * i], Kn = cnt[NCNT * i + 3];
        const int K1 = cnt[NCNT * i + 4], K3 = cnt[NCNT * i + 5];
        const int64_t lo = lv[i].lo, mid = lv[i].mid, hi = lv[i].hi;
        if (K == 0 || Kn == 0) continue;
        // rows of child 1: columns [child 1 | mixed]; rows of child 2: [mixed | child 2]
        DgemmProb pr;
        pr.M = mid - lo;
        pr.N = Kn;
        pr.K = K1 + K3;
        pr.A = b.Zg + lo + lo * n;
        pr.lda = n;
        pr.B = b.Q + lo + lo * n;
        pr.ldb = n;
        pr.C = b.Zt + lo + lo * n;
        pr.ldc = n;
        probs.push_back(pr);
        max_tiles = std::max(max_tiles, dgemm_tiles(pr.M, Kn));
        pr.M = hi - mid;
        pr.K = K - K1;
        pr.A = b.Zg + mid + (lo + K1) * n;
        pr.B = b.Q + (lo + K1) + lo * n;
        pr.C = b.Zt + mid + lo * n;
        probs.push_back(pr);
        max_tiles = std::max(max_tiles, dgemm_tiles(pr.M, Kn));
      }
      if (!probs.empty()) {
        EIG_TRY(c.check(cudaMemcpyAsync(d_probs, probs.data(), probs.size() * sizeof(DgemmProb), cudaMemcpyHostToDevice,
                                        c.stream), "probs"));
        EIG_TRY(dgemm_group(c, d_probs, (int)probs.size(), max_tiles));
      }
    }
    dc_scatter_kernel<<<dim3(std::max<int64_t>(1, std::min<int64_t>(4096, kmax * kmax / 256 + 1)), nn_), 256, 0,
                        c.stream>>>(b, top ? 0 : -1);
    EIG_TRY(c.launched("dc_scatter_kernel"));
    if (!top) {
      dc_copyback_kernel<<<dim3(std::max<int64_t>(1, std::min<int64_t>(4096, kmax * kmax / 256 + 1)), nn_), 256, 0,
                           c.stream>>>(b);
      EIG_TRY(c.launched("dc_copyback_kernel"));
    }
    EIG_TRY(c.check(cudaStreamSynchronize(c.stream), "sync level"));   // host arrays reused next level
  }
  return 0;
}

}  // namespace eig
