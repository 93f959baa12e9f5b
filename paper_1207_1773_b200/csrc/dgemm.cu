// dgemm.cu — real FP64 grouped GEMM on the DMMA pipe (sm_100a), used by the
// divide-and-conquer merges (Z = Z_old Q, "(GPU) = Z Lambda Z^T").
//
// C_p = A_p B_p (op N, column-major) for a group of problems p (one grid.y
// slice per problem).  Block tile 128 x 64, K tile 32, 3-stage cp.async,
// 8 warps as 4 x 2, warp tile 32 x 32 = 4 x 4 DMMA.8x8x4.
#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int BM = 128, BN = 64, BK = 32, STAGES = 3, THREADS = 256;
constexpr int LDA_S = BM + 8;   // sA[k][m] (m contiguous), 8*LDA_S == 64 mod 128
constexpr int LDB_S = BK + 4;   // sB[n][k] (k contiguous), 8*LDB_S == 32 mod 128
constexpr int SA = BK * LDA_S, SB = BN * LDB_S, STAGE = SA + SB;
constexpr size_t SMEM = (size_t)STAGES * STAGE * sizeof(double);

__global__ void __launch_bounds__(THREADS, 2) dgemm_group_kernel(const DgemmProb *probs) {
  extern __shared__ __align__(16) double dsm[];
  const DgemmProb p = probs[blockIdx.y];
  const int tiles_m = (int)((p.M + BM - 1) / BM), tiles_n = (int)((p.N + BN - 1) / BN);
  if ((int)blockIdx.x >= tiles_m * tiles_n) return;
  const int tm = blockIdx.x % tiles_m, tn = blockIdx.x / tiles_m;
  const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int nk = (int)((p.K + BK - 1) / BK);

  auto load = [&](int st, int64_t k0) {
    double *sA = dsm + st * STAGE, *sB = sA + SA;
    // A tile 128 x 32: 16-byte chunks of 2 doubles along m
#pragma unroll
    for (int r = 0; r < (BM * BK / 2) / THREADS; r++) {
      const int i = tid + r * THREADS;
      const int m2 = i % (BM / 2), k = i / (BM / 2);
      const int64_t gm = m0 + 2 * m2, gk = k0 + k;
      const bool ok = gk < p.K && gm + 1 < p.M && ((reinterpret_cast<uintptr_t>(p.A + gm + gk * p.lda) & 15) == 0);
      if (ok) {
        cp_async16(&sA[k * LDA_S + 2 * m2], p.A + gm + gk * p.lda, true);
      } else {
        sA[k * LDA_S + 2 * m2] = (gk < p.K && gm < p.M) ? p.A[gm + gk * p.lda] : 0.0;
        sA[k * LDA_S + 2 * m2 + 1] = (gk < p.K && gm + 1 < p.M) ? p.A[gm + 1 + gk * p.lda] : 0.0;
      }
    }
    // B tile 32 x 64: chunks of 2 doubles along k
#pragma unroll
    for (int r = 0; r < (BN * BK / 2) / THREADS; r++) {
      const int i = tid + r * THREADS;
      const int k2 = i % (BK / 2), n = i / (BK / 2);
      const int64_t gk = k0 + 2 * k2, gn = n0 + n;
      const bool ok = gn < p.N && gk + 1 < p.K && ((reinterpret_cast<uintptr_t>(p.B + gk + gn * p.ldb) & 15) == 0);
      if (ok) {
        cp_async16(&sB[n * LDB_S + 2 * k2], p.B + gk + gn * p.ldb, true);
      } else {
        sB[n * LDB_S + 2 * k2] = (gn < p.N && gk < p.K) ? p.B[gk + gn * p.ldb] : 0.0;
        sB[n * LDB_S + 2 * k2 + 1] = (gn < p.N && gk + 1 < p.K) ? p.B[gk + 1 + gn * p.ldb] : 0.0;
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < nk) load(s, (int64_t)s * BK);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load(nxt % STAGES, (int64_t)nxt * BK);
      cp_async_commit();
    }
    const double *a = dsm + (kt % STAGES) * STAGE, *b = a + SA;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ks++) {
      const int kk = ks * 4 + (lane & 3);
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; i++) af[i] = a[kk * LDA_S + wm * 32 + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; j++) bf[j] = b[(wn * 32 + j * 8 + (lane >> 2)) * LDB_S + kk];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int64_t gm = m0 + wm * 32 + i * 8 + (lane >> 2);
      const int64_t gn = n0 + wn * 32 + j * 8 + (lane & 3) * 2;
      if (gm < p.M) {
        if (gn < p.N) p.C[gm + gn * p.ldc] = acc[i][j][0];
        if (gn + 1 < p.N) p.C[gm + (gn + 1) * p.ldc] = acc[i][j][1];
      }
    }
}

}  // namespace

int dgemm_group(Ctx &ctx, const DgemmProb *d_probs, int nprob, int max_tiles) {
  if (nprob <= 0 || max_tiles <= 0) return 0;
  EIG_TRY(ctx.smem_attr((const void *)dgemm_group_kernel, (int)SMEM, "dgemm attr"));
  dgemm_group_kernel<<<dim3(max_tiles, nprob), THREADS, SMEM, ctx.stream>>>(d_probs);
  return ctx.launched("dgemm_group_kernel");
}

int dgemm_tiles(int64_t M, int64_t N) { return (int)(((M + BM - 1) / BM) * ((N + BN - 1) / BN)); }

}  // namespace eig
