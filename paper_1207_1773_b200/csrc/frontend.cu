// frontend.cu — NEXT-3 front end: Cholesky B = L L^H (Algorithm 1 step 1,
// P:L66) and the standard-form transform A' = L^-1 A L^-H (step 2),
// plus the forward triangular solve they need.
//
// potrf: blocked right-looking, 64-column panels: the diagonal block is
// factored (and inverted) by one CTA in shared memory, the panel below it is
// L21 = A21 L11^-H (one DMMA GEMM with the inverse), the trailing matrix gets
// the Hermitian rank-64 update on the lower triangle.
// hegst: A' = L^-1 (L^-1 A)^H, which is Hermitian, computed as two blocked
// forward solves with n right-hand sides (GEMM-rich and fully parallel; twice
// the flops of LAPACK's zhegst but no sequential trailing solves).
#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int FB = 64;

// Factor the b x b Hermitian diagonal block (lower) in place and write its
// inverse (lower, zeros above) to Linv (ld 64).  info (1-based global pivot
// index, + n) is set on the first non-positive pivot.
__global__ void __launch_bounds__(256) potrf_diag_kernel(double2 *A11, int64_t lda, int b, double2 *Linv,
                                                         int64_t gofs, int64_t n, int64_t *info) {
  extern __shared__ __align__(16) double2 fsm[];
  double2 *L = fsm;                  // [64][65]
  double2 *X = fsm + 64 * 65;        // [64][65]
  __shared__ double s_piv;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  for (int e = tid; e < b * b; e += 256) {
    const int r = e % b, c = e / b;
    L[r + c * 65] = (r >= c) ? A11[r + c * lda] : czero();
  }
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int j = 0; j < b; j++) {
    if (tid == 0) {
      const double d = L[j + j * 65].x;
      if (!(d > 0.0) || !isfinite(d)) {
        if (!s_bad) {
          s_bad = 1;
          atomicCAS(reinterpret_cast<unsigned long long *>(info), 0ull, (unsigned long long)(n + gofs + j + 1));
        }
        s_piv = 1.0;
      } else {
        s_piv = sqrt(d);
      }
      L[j + j * 65] = make_double2(s_piv, 0.0);
    }
    __syncthreads();
    const double inv = 1.0 / s_piv;
    for (int i = j + 1 + tid; i < b; i += 256) L[i + j * 65] = cscale(inv, L[i + j * 65]);
    __syncthreads();
    const int m = b - j - 1;
    for (int e = tid; e < m * m; e += 256) {
      const int i = j + 1 + e % m, k = j + 1 + e / m;
      if (i >= k) L[i + k * 65] = csub(L[i + k * 65], cmul(L[i + j * 65], cconj(L[k + j * 65])));
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += 256) {
    const int r = e % b, c = e / b;
    if (r >= c) A11[r + c * lda] = L[r + c * 65];
  }
  // inverse: column c by forward substitution, four lanes per column (each
  // sums every fourth term; two xor-shuffles combine them)
  {
    const int c = tid >> 2, part = tid & 3;
    for (int r = 0; r < 64; r++) {
      double2 acc = czero();
      if (c < b && r < b && r > c)
        for (int k = c + part; k < r; k += 4) acc = cadd(acc, cmul(L[r + k * 65], X[k + c * 65]));
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
      if (part == 0 && c < b && r < b) {
        double2 v = czero();
        if (r >= c) {
          const double2 s = (r == c) ? make_double2(1.0 - acc.x, -acc.y) : make_double2(-acc.x, -acc.y);
          const double d = L[r + r * 65].x;   // diagonal is real positive
          v = make_double2(s.x / d, s.y / d);
        }
        X[r + c * 65] = v;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < FB * FB; e += 256) {
    const int r = e % FB, c = e / FB;
    Linv[r + c * FB] = (r < b && c < b) ? X[r + c * 65] : czero();
  }
}

// Full Hermitian from the lower triangle (imag(diag) = 0): upper <- conj(lower)^T.
__global__ void herm_full_kernel(int64_t n, double2 *A, int64_t lda) {
  const int64_t total = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % n, c = e / n;
    if (r < c) A[r + c * lda] = cconj(A[c + r * lda]);
    else if (r == c) A[r + c * lda].y = 0.0;
  }
}

// Y = X^H (n x n, tiled transpose through shared memory)
__global__ void conj_transpose_kernel(int64_t n, const double2 *X, int64_t ldx, double2 *Y, int64_t ldy) {
  __shared__ double2 t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < n && c < n) t[k][threadIdx.x] = X[r + c * ldx];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = c0 + threadIdx.x, c = r0 + k;   // Y[r, c] = conj(X[c, r])
    if (r < n && c < n) Y[r + c * ldy] = cconj(t[threadIdx.x][k]);
  }
}

}  // namespace

// Look-ahead (like he2hb's): the trailing update of step k is split
// into (i) the next block column and (ii) the rest; the next diagonal block
// and its panel L21 are factored on the high-priority side stream right
// after (i), concurrently with (ii).
int potrf_lower(Ctx &c, int64_t n, double2 *B, int64_t ldb, int64_t *d_info) {
  double2 *Linv = (double2 *)c.ws(WS_FRONT, (size_t)FB * FB * sizeof(double2));
  if (!Linv) return EIG_ERR_NOMEM;
  const size_t smem = (size_t)2 * 64 * 65 * sizeof(double2);
  EIG_TRY(c.smem_attr((const void *)potrf_diag_kernel, (int)smem, "potrf attr"));
  // diagonal block at k (size b) and, below it, L21 = A21 L11^-H (s rows), on `st`
  auto factor_block = [&](int64_t k, cudaStream_t st) -> int {
    const int b = (int)std::min<int64_t>(FB, n - k);
    double2 *A11 = B + k + k * ldb;
    potrf_diag_kernel<<<1, 256, smem, st>>>(A11, ldb, b, Linv, k, n, d_info);
    EIG_TRY(c.launched("potrf_diag_kernel"));
    const int64_t s = n - k - b;
    if (s <= 0) return 0;
    Zgemm g;   // in place: one 64-col N tile, no split-K
    g.opb = OP_C; g.M = s; g.N = b; g.K = b; g.A = A11 + b; g.lda = ldb; g.B = Linv; g.ldb = FB; g.C = A11 + b;
    g.ldc = ldb; g.splitk = 1; g.whole_n = true;
    const cudaStream_t keep = c.stream;
    c.stream = st;
    const int rc = zgemm(c, g);
    c.stream = keep;
    return rc;
  };
  // outer blocks of PB = 128 columns (two 64-column diagonal factorisations
  // each), so the trailing update has K = 128
  constexpr int PB = 2 * FB;
  auto factor_outer = [&](int64_t k, cudaStream_t st) -> int {
    const int b = (int)std::min<int64_t>(PB, n - k);
    EIG_TRY(factor_block(k, st));
    if (b <= FB) return 0;
    // second sub-column (rows >= k + FB) -= L21a L21a[0:b-FB]^H, then its factorisation
    Zgemm g;
    g.opb = OP_C; g.lower_c = 2; g.M = n - k - FB; g.N = b - FB; g.K = FB; g.A = B + (k + FB) + k * ldb; g.lda = ldb;
    g.B = B + (k + FB) + k * ldb; g.ldb = ldb; g.C = B + (k + FB) + (k + FB) * ldb; g.ldc = ldb;
    g.alpha = -1.0; g.beta = 1.0;
    const cudaStream_t keep = c.stream;
    c.stream = st;
    const int rc = zgemm(c, g);
    c.stream = keep;
    EIG_TRY(rc);
    return factor_block(k + FB, st);
  };
  EIG_TRY(factor_outer(0, c.stream));
  for (int64_t k = 0; k < n; k += PB) {
    const int b = (int)std::min<int64_t>(PB, n - k);
    const int64_t s = n - k - b;
    if (s <= 0) break;
    if (k > 0) EIG_TRY(c.check(cudaStreamWaitEvent(c.stream, c.ev_join, 0), "potrf join"));
    double2 *A11 = B + k + k * ldb, *L21 = A11 + b, *A22 = A11 + b + b * ldb;
    const int b2 = (int)std::min<int64_t>(PB, s);
    Zgemm g;
    if (s > b2) {
      // (i) the next block column: A22[:, 0:b2] -= L21 L21[0:b2]^H (rows >= cols)
      g.opb = OP_C; g.lower_c = 2; g.M = s; g.N = b2; g.K = b; g.A = L21; g.lda = ldb; g.B = L21; g.ldb = ldb;
      g.C = A22; g.ldc = ldb; g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
      EIG_TRY(c.check(cudaEventRecord(c.ev_fork, c.stream), "potrf fork"));
      EIG_TRY(c.check(cudaStreamWaitEvent(c.side, c.ev_fork, 0), "potrf fork wait"));
      EIG_TRY(factor_outer(k + b, c.side));
      EIG_TRY(c.check(cudaEventRecord(c.ev_join, c.side), "potrf join rec"));
      // (ii) the rest of the trailing lower triangle
      g = Zgemm();
      g.opb = OP_C; g.lower_c = 1; g.M = s - b2; g.N = s - b2; g.K = b; g.A = L21 + b2; g.lda = ldb; g.B = L21 + b2;
      g.ldb = ldb; g.C = A22 + b2 + b2 * ldb; g.ldc = ldb; g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
    } else {
      // last block: the whole (b2 x b2) update, then its factorisation, in order
      g.opb = OP_C; g.lower_c = 1; g.M = s; g.N = s; g.K = b; g.A = L21; g.lda = ldb; g.B = L21; g.ldb = ldb;
      g.C = A22; g.ldc = ldb; g.alpha = -1.0; g.beta = 1.0;
      EIG_TRY(zgemm(c, g));
      EIG_TRY(factor_outer(k + b, c.stream));
      break;
    }
  }
  return 0;
}

int herm_full(Ctx &c, int64_t n, double2 *A, int64_t lda) {
  const int64_t total = n * n;
  herm_full_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 16LL * c.num_sms), 256, 0, c.stream>>>(n, A, lda);
  return c.launched("herm_full_kernel");
}

int conj_transpose(Ctx &c, int64_t n, const double2 *X, int64_t ldx, double2 *Y, int64_t ldy) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  conj_transpose_kernel<<<grid, dim3(32, 8), 0, c.stream>>>(n, X, ldx, Y, ldy);
  return c.launched("conj_transpose_kernel");
}

}  // namespace eig
