// zgemm.cu — complex-FP64 tile engine on the DMMA pipe (sm_100a).
//
// C = alpha op(A) op(B) + beta C via the real embedding described in
// common.cuh.  Block tile 64 x 64 complex (128 real rows x 64 cols of C~),
// K tile 16 complex, 3-stage cp.async pipeline, 8 warps as 4 (M) x 2 (N),
// warp tile 32 real rows x 32 cols = 4 x 4 DMMA.8x8x4 accumulators.
// Modes: Hermitian-lower A (hemm, a3), lower-triangular C (her2k, a5),
// split-K with a deterministic reduction (skinny products, a4/a7/a8).
// Used by he2hb (Fig. 1 (c) P:L97), Q1 and trsm.
//
// M3 = true: the 3M (Gauss) product instead of the real embedding.  With
// planes a = ar + i ai, b = br + i bi and the sums as = ar + ai, bs = br + bi,
//   P1 = sum ar br,  P2 = sum ai bi,  P3 = sum as bs,
//   Re c = P1 - P2,  Im c = P3 - P1 - P2,
// three real DMMA products per complex product instead of four (0.75 of the
// DMMA work; nominal flops stay 8 per complex multiply-add, the pipe does 6).
// The planes are formed in registers from one 16-byte shared-memory load per
// complex operand element (conjugation flips ai / bi), warp tile 16 x 32
// complex = 2 x 4 DMMA tiles per plane.  Normwise error bound of the same
// order as the 4-real-product form (Higham, "Stability of a method for
// multiplying complex matrices with three real matrix multiplications");
// only the imaginary part's componentwise bound is weaker.  The path's
// gates (parity 1e-11, residual / B-orthogonality 1e-14) are unchanged.
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int BM = 64, THREADS = 256;   // (variant 4: BM 128, see Lay)
// Engine variants V: 0 = real embedding (4 real products; BN 64, BK 16, two
// 120-register CTAs per SM); 1 = 3M, long K (BN 64, BK 32, warp tile 16 x 32,
// one 208-register CTA per SM); 2 = 3M, short K (BN 32, BK 16, warp tile
// 16 x 16, two CTAs per SM, so one CTA's prologue / epilogue overlaps the
// other's main loop — the he2hb rank-2k update and the K = 256 Q1 update).
// Shared-memory layouts (complex elements).  4M: 8-byte fragment loads;
// 3M: 16-byte complex loads, eight lanes per phase (row g = lane>>2 in {0,1},
// k t = lane&3), so the k-major strides are 2 mod 8 and the k-contiguous ones
// 4 mod 8 (eight distinct 16-byte bank groups per phase).
template <int V>
struct Lay {
  static constexpr bool M3 = V >= 1;
  // variant 4 = 3M, 128 x 64 tiles, 32 x 32 warp tiles (8 DADDs per 48 DMMAs
  // instead of 6 per 24), BK 16, one CTA per SM; plain products only
  static constexpr int BMV = V == 4 ? 128 : 64;
  // variant 5 = variant 2's 64 x 32 tiles with 4 warps of 32 x 16 (6 DADDs per
  // 24 DMMAs instead of 4 per 12), 128 threads, two CTAs per SM
  static constexpr int WMR = (V == 4 || V == 5) ? 32 : 16;   // 3M warp tile height (complex rows)
  static constexpr int WARPS_M = BMV / WMR;
  static constexpr int BN = (V == 2 || V == 5) ? 32 : 64;
  static constexpr int WN = (V == 2 || V == 5) ? 16 : 32;   // 3M warp tile width (complex columns)
  static constexpr int MINB = (V == 1 || V == 4) ? 1 : 2;   // resident CTAs per SM
  static constexpr int NT = V == 5 ? 128 : THREADS;         // threads per CTA
  // K tile (complex): variant 1 runs one CTA per SM, so it takes twice the K
  // per pipeline stage (half the CTA barriers per flop)
  static constexpr int BK = V == 1 ? 32 : 16;
  static constexpr int STAGES = 3;
  static constexpr int LDA_S = M3 ? BMV + 2 : BMV + 4;  // sA[k][m]: k-major, m contiguous
  static constexpr int LDB_S = M3 ? BK + 4 : BK + 2;  // sB[n][k]: n-major, k contiguous
  static constexpr int LDAK = M3 ? BK + 4 : BK + 2;   // op(A) = A^H: sA[m][k], k contiguous
  static constexpr int LDBN = M3 ? BN + 2 : BN + 4;   // op(B) = B^H: sB[k][n], n contiguous
  static constexpr int SA_ELEMS = (BK * LDA_S > BMV * LDAK) ? BK * LDA_S : BMV * LDAK;
  static constexpr int SB_ELEMS = (BN * LDB_S > BK * LDBN) ? BN * LDB_S : BK * LDBN;
  static constexpr int STAGE_ELEMS = SA_ELEMS + SB_ELEMS;
  static constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_ELEMS * sizeof(double2);
};

struct Params {
  int64_t M, N, K;
  const double2 *A;
  int64_t lda;
  const double2 *B;
  int64_t ldb;
  double2 *C;
  int64_t ldc;
  double alpha, beta;
  double2 *part;   // split-K partials [split][M*N] (ld M), or nullptr
  int64_t row0;    // lower modes: C row gm is matrix row row0 + gm (column gn is column gn)
  int64_t kchunk;  // K per split (multiple of BK)
  int tiles_m;
};

template <int OPA, int OPB, bool HERM, int LOWER, int V>
__global__ void __launch_bounds__(Lay<V>::NT, Lay<V>::MINB) zgemm_kernel(Params p) {
  using LY = Lay<V>;
  constexpr int THREADS = LY::NT;   // (shadows the file-scope 256)
  constexpr int BM = LY::BMV;   // (shadows the file-scope 64)
  constexpr bool M3 = LY::M3;
  constexpr int BN = LY::BN, M3_WN = LY::WN;
  constexpr int BK = LY::BK, STAGES = LY::STAGES;
  constexpr int LDA_S = LY::LDA_S, LDB_S = LY::LDB_S, LDAK = LY::LDAK, LDBN = LY::LDBN;
  constexpr int SA_ELEMS = LY::SA_ELEMS, STAGE_ELEMS = LY::STAGE_ELEMS;
  extern __shared__ __align__(16) double2 smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;

  int tm, tn;
  if (LOWER == 1) {
    // tile row I holds q (I + 1) column tiles (q = BM / BN): rows before it
    // hold q I (I + 1) / 2 tiles
    constexpr int q = BM / BN;
    const int64_t x = blockIdx.x;
    int64_t I = (int64_t)((sqrt(8.0 * (double)x / q + 1.0) - 1.0) * 0.5);
    while (q * (I + 1) * (I + 2) / 2 <= x) I++;
    while (q * I * (I + 1) / 2 > x) I--;
    tm = (int)I;
    tn = (int)(x - q * I * (I + 1) / 2);
  } else {
    tm = blockIdx.x % p.tiles_m;
    tn = blockIdx.x / p.tiles_m;
  }
  const int64_t m0 = (int64_t)tm * BM, n0 = (int64_t)tn * BN;
  const int64_t kbeg = (int64_t)blockIdx.y * p.kchunk;
  const int64_t kend = min(p.K, kbeg + p.kchunk);
  const int nk = (int)((kend - kbeg + BK - 1) / BK);

  auto load = [&](int stage, int64_t k0) {
    double2 *sA = smem + stage * STAGE_ELEMS;
    double2 *sB = sA + SA_ELEMS;
    int mode;  // 0: A[m,k]; 1: A[k,m] (conj applied at fragment time); 2: Hermitian diagonal-crossing
    if (HERM)
      mode = (k0 + BK - 1 <= m0) ? 0 : ((k0 >= m0 + BM) ? 1 : 2);
    else
      mode = (OPA == OP_C) ? 1 : 0;
#pragma unroll
    for (int r = 0; r < (BM * BK) / THREADS; r++) {
      const int i = tid + r * THREADS;
      int m, k;
      if (mode == 1) {
        k = i % BK;
        m = i / BK;
      } else {
        m = i % BM;
        k = i / BM;
      }
      const int64_t gm = m0 + m, gk = k0 + k;
      const bool valid = gm < p.M && gk < kend;
      const double2 *src;
      if (mode == 0)
        src = p.A + gm + gk * p.lda;
      else if (mode == 1)
        src = p.A + gk + gm * p.lda;
      else
        src = (gm >= gk) ? p.A + gm + gk * p.lda : p.A + gk + gm * p.lda;
      if (mode == 1)   // A^H tile (op C, or the Hermitian upper part): k contiguous
        cp_async16(&sA[m * LDAK + k], valid ? src : p.A, valid);
      else
        cp_async16(&sA[k * LDA_S + m], valid ? src : p.A, valid);
    }
#pragma unroll
    for (int r = 0; r < (BN * BK) / THREADS; r++) {
      const int i = tid + r * THREADS;
      int n, k;
      const double2 *src;
      if (OPB == OP_N) {
        k = i % BK;
        n = i / BK;
      } else {
        n = i % BN;
        k = i / BN;
      }
      const int64_t gn = n0 + n, gk = k0 + k;
      const bool valid = gn < p.N && gk < kend;
      src = (OPB == OP_N) ? p.B + gk + gn * p.ldb : p.B + gn + gk * p.ldb;
      if (OPB == OP_C)
        cp_async16(&sB[k * LDBN + n], valid ? src : p.B, valid);
      else
        cp_async16(&sB[n * LDB_S + k], valid ? src : p.B, valid);
    }
  };

#pragma unroll
  for (int s0 = 0; s0 < STAGES - 1; s0++) {
    if (s0 < nk) load(s0, kbeg + (int64_t)s0 * BK);
    cp_async_commit();
  }
  // C += alpha A B with alpha = +-1: start the accumulators from C (its loads
  // overlap the pipeline prologue instead of trailing the main loop) and fold
  // the sign of alpha into the A fragments.
  const bool fuse_c = (p.part == nullptr) && p.beta == 1.0 && (p.alpha == 1.0 || p.alpha == -1.0);
  const unsigned aflip = (fuse_c && p.alpha == -1.0) ? 0x80000000u : 0u;

  // per k-tile: is op(A) conjugated, and is the A tile stored [m][k] (KM)
  auto tile_mode = [&](int kt, int st, bool &conjA) {
    conjA = (OPA == OP_C);
    if (HERM) {
      const int64_t k0 = kbeg + (int64_t)kt * BK;
      if (k0 >= m0 + BM) {
        conjA = true;
      } else if (k0 + BK - 1 <= m0) {
        conjA = false;
      } else {
        conjA = false;
        double2 *sA = smem + st * STAGE_ELEMS;
        for (int i = tid; i < BM * BK; i += THREADS) {
          const int m = i % BM, k = i / BM;
          const int64_t gm = m0 + m, gk = k0 + k;
          double2 v = sA[k * LDA_S + m];
          if (gm < gk) v.y = -v.y;
          else if (gm == gk) v.y = 0.0;
          sA[k * LDA_S + m] = v;
        }
        __syncthreads();
      }
    }
  };

  if constexpr (M3) {
    // ------------------------------------------------------------ 3M path
    // warp tile WMR complex rows (wm) x M3_WN complex cols (wn): MI x NJ tiles per plane
    const int g8 = lane >> 2, t4 = lane & 3;
    constexpr int NJ = M3_WN / 8, MI = LY::WMR / 8;
    const int wm3 = warp % LY::WARPS_M, wn3 = warp / LY::WARPS_M;
    double acc[3][MI][NJ][2];
#pragma unroll
    for (int q = 0; q < 3; q++)
#pragma unroll
      for (int i = 0; i < MI; i++)
#pragma unroll
        for (int j = 0; j < NJ; j++) acc[q][i][j][0] = acc[q][i][j][1] = 0.0;
    // alpha = -1 (fused): accumulate from -C and negate at the end (exact), so
    // the A planes need no sign flips
    const double cs = aflip ? -1.0 : 1.0;
    if (fuse_c) {   // P1 = Re C, P2 = 0, P3 = Re C + Im C  (times cs)
#pragma unroll
      for (int i = 0; i < MI; i++)
#pragma unroll
        for (int j = 0; j < NJ; j++)
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const int64_t gm = m0 + wm3 * LY::WMR + i * 8 + g8, gn = n0 + wn3 * M3_WN + j * 8 + 2 * t4 + h;
            const double2 c = (gm < p.M && gn < p.N) ? p.C[gm + gn * p.ldc] : czero();
            acc[0][i][j][h] = cs * c.x;
            acc[2][i][j][h] = cs * (c.x + c.y);
          }
    }
    for (int kt = 0; kt < nk; kt++) {
      const int st = kt % STAGES;
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nxt = kt + STAGES - 1;
        if (nxt < nk) load(nxt % STAGES, kbeg + (int64_t)nxt * BK);
        cp_async_commit();
      }
      bool conjA;
      tile_mode(kt, st, conjA);
      const double2 *a2 = smem + st * STAGE_ELEMS;
      const double2 *b2 = a2 + SA_ELEMS;
      auto compute = [&](auto km) {
        constexpr bool KM = decltype(km)::value;   // A tile stored [m][k]
#pragma unroll
        for (int ks = 0; ks < BK / 4; ks++) {
          const int kk = ks * 4 + t4;
          double ar[MI], ai[MI], as[MI], br[NJ], bi[NJ], bs[NJ];
#pragma unroll
          for (int i = 0; i < MI; i++) {
            const int mm = wm3 * LY::WMR + i * 8 + g8;
            const double2 v = KM ? a2[mm * LDAK + kk] : a2[kk * LDA_S + mm];
            ar[i] = v.x;
            ai[i] = conjA ? -v.y : v.y;
            as[i] = ar[i] + ai[i];
          }
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int nn = wn3 * M3_WN + j * 8 + g8;
            const double2 v = OPB == OP_C ? b2[kk * LDBN + nn] : b2[nn * LDB_S + kk];
            br[j] = v.x;
            bi[j] = OPB == OP_C ? -v.y : v.y;
            bs[j] = br[j] + bi[j];
          }
          // plane-major order: consecutive DMMAs share their A operand
#pragma unroll
          for (int i = 0; i < MI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) dmma(acc[0][i][j], ar[i], br[j]);
#pragma unroll
          for (int i = 0; i < MI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) dmma(acc[1][i][j], ai[i], bi[j]);
#pragma unroll
          for (int i = 0; i < MI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) dmma(acc[2][i][j], as[i], bs[j]);
        }
      };
      if (HERM) {
        if (conjA) compute(std::true_type{});
        else compute(std::false_type{});
      } else {
        compute(std::integral_constant<bool, OPA == OP_C>{});
      }
    }
    cp_async_wait<0>();
    // epilogue: lane holds complex (row g8, cols 2 t4 + h) of every tile
#pragma unroll
    for (int i = 0; i < MI; i++)
#pragma unroll
      for (int j = 0; j < NJ; j++)
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t gm = m0 + wm3 * LY::WMR + i * 8 + g8, gn = n0 + wn3 * M3_WN + j * 8 + 2 * t4 + h;
          if (gm >= p.M || gn >= p.N) continue;
          const double p1 = acc[0][i][j][h], p2 = acc[1][i][j][h], p3 = acc[2][i][j][h];
          const double2 v = make_double2(cs * (p1 - p2), cs * (p3 - p1 - p2));
          if (p.part) {
            p.part[(int64_t)blockIdx.y * p.M * p.N + gm + gn * p.M] = v;
          } else {
            if (LOWER && p.row0 + gm < gn) continue;
            double2 *cp = p.C + gm + gn * p.ldc;
            double2 out = fuse_c ? v : make_double2(p.alpha * v.x, p.alpha * v.y);
            if (!fuse_c && p.beta != 0.0) {
              const double2 c = *cp;
              out.x += p.beta * c.x;
              out.y += p.beta * c.y;
            }
            if (LOWER && p.row0 + gm == gn) out.y = 0.0;
            *cp = out;
          }
        }
    return;
  } else {
  // ------------------------------------------------------------ 4M (real embedding) path
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  const LaneEmb le(lane);
  if (fuse_c) {
    const int rpc = (lane >> 2) & 1;
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int64_t gm = m0 + wm * 16 + i * 4 + (lane >> 3);
        const int64_t gn = n0 + wn * 32 + j * 8 + (lane & 3) * 2;
        const double *cb = reinterpret_cast<const double *>(p.C);
        acc[i][j][0] = (gm < p.M && gn < p.N) ? cb[(gm + gn * p.ldc) * 2 + rpc] : 0.0;
        acc[i][j][1] = (gm < p.M && gn + 1 < p.N) ? cb[(gm + (gn + 1) * p.ldc) * 2 + rpc] : 0.0;
      }
  }

  for (int kt = 0; kt < nk; kt++) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load(nxt % STAGES, kbeg + (int64_t)nxt * BK);
      cp_async_commit();
    }
    const int st = kt % STAGES;
    bool conjA;
    tile_mode(kt, st, conjA);
    const double *a = reinterpret_cast<const double *>(smem + st * STAGE_ELEMS);
    const double *b = reinterpret_cast<const double *>(smem + st * STAGE_ELEMS + SA_ELEMS);
    const unsigned anm = (conjA ? le.a_neg_conj : le.a_neg) ^ aflip;
    const unsigned bnm = (OPB == OP_C) ? le.b_neg_conj : 0u;
    // the A^H layout is chosen per k-tile (uniform branch: two specialised loops)
    auto compute = [&](auto km) {
      constexpr bool KM = decltype(km)::value;   // A tile stored [m][k]
#pragma unroll
      for (int ks = 0; ks < BK / 2; ks++) {
        const int kk = ks * 2 + ((lane & 3) >> 1);
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; i++) {
          const int mm = wm * 16 + i * 4 + (lane >> 3);
          af[i] = xsign(KM ? a[(mm * LDAK + kk) * 2 + le.a_comp] : a[(kk * LDA_S + mm) * 2 + le.a_comp], anm);
        }
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const int nn = wn * 32 + j * 8 + (lane >> 2);
          bf[j] = xsign(OPB == OP_C ? b[(kk * LDBN + nn) * 2 + le.b_comp] : b[(nn * LDB_S + kk) * 2 + le.b_comp], bnm);
        }
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
          for (int j = 0; j < 4; j++) dmma(acc[i][j], af[i], bf[j]);
      }
    };
    if (HERM) {
      if (conjA) compute(std::true_type{});
      else compute(std::false_type{});
    } else {
      compute(std::integral_constant<bool, OPA == OP_C>{});
    }
  }
  cp_async_wait<0>();

  // epilogue: pair lanes (lane, lane^4) hold (Re, Im) rows of the same complex row
  const int rp = (lane >> 2) & 1;
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const double send = rp ? acc[i][j][0] : acc[i][j][1];
      const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
      const double2 v = rp ? make_double2(recv, acc[i][j][1]) : make_double2(acc[i][j][0], recv);
      const int64_t gm = m0 + wm * 16 + i * 4 + (lane >> 3);
      const int64_t gn = n0 + wn * 32 + j * 8 + (lane & 3) * 2 + rp;
      if (gm < p.M && gn < p.N) {
        if (p.part) {
          p.part[(int64_t)blockIdx.y * p.M * p.N + gm + gn * p.M] = v;
        } else {
          if (LOWER && p.row0 + gm < gn) continue;
          double2 *cp = p.C + gm + gn * p.ldc;
          double2 out = fuse_c ? v : make_double2(p.alpha * v.x, p.alpha * v.y);
          if (!fuse_c && p.beta != 0.0) {
            const double2 c = *cp;
            out.x += p.beta * c.x;
            out.y += p.beta * c.y;
          }
          if (LOWER && p.row0 + gm == gn) out.y = 0.0;
          *cp = out;
        }
      }
    }
  }
}

// C = alpha * sum_z part[z] + beta * C  (fixed summation order -> deterministic)
__global__ void splitk_reduce_kernel(int64_t M, int64_t N, int split, const double2 *__restrict__ part, double2 *C,
                                     int64_t ldc, double alpha, double beta, int lower, int64_t row0) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gm = e % M, gn = e / M;
    if (lower && row0 + gm < gn) continue;
    double2 s = part[e];
    for (int z = 1; z < split; z++) {
      const double2 t = part[(int64_t)z * total + e];
      s.x += t.x;
      s.y += t.y;
    }
    double2 out = make_double2(alpha * s.x, alpha * s.y);
    double2 *cp = C + gm + gn * ldc;
    if (beta != 0.0) {
      const double2 c = *cp;
      out.x += beta * c.x;
      out.y += beta * c.y;
    }
    if (lower && row0 + gm == gn) out.y = 0.0;
    *cp = out;
  }
}

template <int OPA, int OPB, bool HERM, int LOWER, int V>
int launch_v(Ctx &ctx, const Params &p, dim3 grid) {
  constexpr size_t sm = Lay<V>::SMEM_BYTES;
  EIG_TRY(ctx.smem_attr((const void *)zgemm_kernel<OPA, OPB, HERM, LOWER, V>, (int)sm, "zgemm attr"));
  zgemm_kernel<OPA, OPB, HERM, LOWER, V><<<grid, Lay<V>::NT, sm, ctx.stream>>>(p);
  return ctx.launched("zgemm_kernel");
}
template <int OPA, int OPB, bool HERM, int LOWER>
int launch_t(Ctx &ctx, const Params &p, dim3 grid, int v) {
  if (v == 4) {
    if constexpr (LOWER == 0 && !HERM) return launch_v<OPA, OPB, HERM, LOWER, 4>(ctx, p, grid);
    return -2;
  }
  if (v == 5) return launch_v<OPA, OPB, HERM, LOWER, 5>(ctx, p, grid);
  if (v == 2) return launch_v<OPA, OPB, HERM, LOWER, 2>(ctx, p, grid);
  if (v == 1) return launch_v<OPA, OPB, HERM, LOWER, 1>(ctx, p, grid);
  return launch_v<OPA, OPB, HERM, LOWER, 0>(ctx, p, grid);
}

}  // namespace

int zgemm(Ctx &ctx, const Zgemm &g) {
  if (g.M <= 0 || g.N <= 0) return 0;
  if (g.K <= 0 && g.beta == 1.0) return 0;  // K = 0 otherwise runs the epilogue only: C = beta C
  if (g.herm_a && (g.opa != OP_N || g.M != g.K)) return -2;
  if (g.lower_c == 1 && g.M != g.N) return -2;

  const bool m3 = g.m3 > 0 || (g.m3 == 0 && ctx.use_3m);
  // 3M short-K variant (2 CTAs/SM) where the K loop is too short to hide a
  // CTA's prologue and epilogue; EIG_ZGEMM_SHORTK=<K> moves the threshold
  // (0 disables it)
  static const int64_t shortk = [] {
    const char *e = getenv("EIG_ZGEMM_SHORTK");
    return e ? (int64_t)atoll(e) : (int64_t)kShortK;
  }();
  static const int64_t narrow = [] {
    const char *e = getenv("EIG_ZGEMM_NARROW");
    return e ? (int64_t)atoll(e) : (int64_t)kNarrowN;
  }();
  if (g.whole_n && g.N > Lay<0>::BN) return -2;
  // variant 4 (128 x 64 tiles) for plain long-K products when EIG_ZGEMM_V4=1
  static const int v4_env = [] {
    const char *e = getenv("EIG_ZGEMM_V4");
    return e ? atoi(e) : kZgemmV4;
  }();
  // (with split_n set the choice must not depend on N: column slices stay bitwise)
  const bool narrow_n = g.split_n <= 0 && g.N <= narrow;
  int v = !m3 ? 0 : ((g.K <= shortk || narrow_n) && !g.whole_n ? 2 : 1);
  if (v == 1 && v4_env && g.lower_c == 0 && !g.herm_a && !g.whole_n) v = 4;
  // tall plain products with 128 < K <= 256 (Q1's E -= (V T) Y): the 128 x 64
  // tiles beat the two-CTA 64 x 32 ones once M fills the machine
  if (v == 2 && v4_env && g.K > 128 && g.M >= 2048 && g.lower_c == 0 && !g.herm_a && !g.whole_n) v = 4;
  static const int v5_env = [] {
    const char *e = getenv("EIG_ZGEMM_V5");
    return e ? atoi(e) : 0;
  }();
  if (v == 2 && v5_env) v = 5;
  const int BMv = v == 4 ? Lay<4>::BMV : BM;
  const int BN = (v == 2 || v == 5) ? Lay<2>::BN : Lay<0>::BN;
  const int64_t q = BM / BN;
  const int tiles_m = (int)((g.M + BMv - 1) / BMv), tiles_n = (int)((g.N + BN - 1) / BN);
  const int64_t tiles = g.lower_c == 1 ? q * tiles_m * (tiles_m + 1) / 2 : (int64_t)tiles_m * tiles_n;
  // the split model sees N = split_n when set (N-independent split, see kernels.h)
  const int64_t Nm = g.split_n > 0 ? g.split_n : g.N;
  const int64_t tiles_model =
      g.split_n > 0 ? (int64_t)tiles_m * ((g.split_n + BN - 1) / BN) : tiles;
  const int BK = v == 1 ? Lay<1>::BK : Lay<0>::BK;
  const int64_t ktiles = std::max<int64_t>(1, (g.K + BK - 1) / BK);
  int split = g.splitk;
  if (split <= 0) {
    // pick the split that minimises (waves of resident CTAs) x (k-tiles per CTA + fixed per-CTA cost),
    // plus the partial-sum traffic of the reduction (in k-tile units)
    const int64_t cap = (v == 1 || v == 4 ? 1LL : 2LL) * ctx.num_sms;   // resident CTAs (variant 1: one 208-register CTA per SM)
    const int64_t maxs = std::max<int64_t>(1, std::min<int64_t>(64, ktiles / 4));
    double best = 1e300;
    split = 1;
    for (int64_t sp = 1; sp <= maxs; sp++) {
      const int64_t kt = (ktiles + sp - 1) / sp;
      const int64_t waves = (tiles_model * sp + cap - 1) / cap;
      const double red = sp > 1 ? 0.02 * (double)sp * (double)g.M * (double)Nm / (double)(cap * BMv * BN) * 8.0 : 0.0;
      const double t = (double)waves * (double)(kt + 3) + red;
      if (t < best * 0.98) {
        best = t;
        split = (int)sp;
      }
    }
  }
  int64_t kt_per = (ktiles + split - 1) / split;
  split = (int)((ktiles + kt_per - 1) / kt_per);

  Params p;
  p.M = g.M;
  p.N = g.N;
  p.K = std::max<int64_t>(g.K, 0);
  p.A = g.A;
  p.lda = g.lda;
  p.B = g.B;
  p.ldb = g.ldb;
  p.C = g.C;
  p.ldc = g.ldc;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.kchunk = kt_per * BK;
  p.tiles_m = tiles_m;
  p.part = nullptr;
  p.row0 = g.row0;
  if (split > 1) {
    p.part = (double2 *)ctx.ws(ctx.stream == ctx.side ? WS_PART_SIDE : WS_PART,
                               (size_t)split * g.M * g.N * sizeof(double2));
    if (!p.part) return EIG_ERR_NOMEM;
  }
  dim3 grid((unsigned)tiles, (unsigned)split);
  int rc;
  if (g.herm_a)
    rc = launch_t<OP_N, OP_N, true, 0>(ctx, p, grid, v);
  else if (g.lower_c == 1) {
    if (g.opa == OP_N && g.opb == OP_C) rc = launch_t<OP_N, OP_C, false, 1>(ctx, p, grid, v);
    else if (g.opa == OP_N && g.opb == OP_N) rc = launch_t<OP_N, OP_N, false, 1>(ctx, p, grid, v);
    else return -2;
  } else if (g.lower_c == 2) {
    if (g.opa == OP_N && g.opb == OP_C) rc = launch_t<OP_N, OP_C, false, 2>(ctx, p, grid, v);
    else return -2;
  } else if (g.opa == OP_N && g.opb == OP_N)
    rc = launch_t<OP_N, OP_N, false, 0>(ctx, p, grid, v);
  else if (g.opa == OP_C && g.opb == OP_N)
    rc = launch_t<OP_C, OP_N, false, 0>(ctx, p, grid, v);
  else if (g.opa == OP_N && g.opb == OP_C)
    rc = launch_t<OP_N, OP_C, false, 0>(ctx, p, grid, v);
  else
    rc = launch_t<OP_C, OP_C, false, 0>(ctx, p, grid, v);
  if (rc) return rc;
  if (split > 1) {
    const int64_t total = g.M * g.N;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8LL * ctx.num_sms);
    splitk_reduce_kernel<<<blocks, 256, 0, ctx.stream>>>(g.M, g.N, split, p.part, g.C, g.ldc, g.alpha, g.beta,
                                                          g.lower_c, g.row0);
    EIG_TRY(ctx.launched("splitk_reduce_kernel"));
  }
  return 0;
}

}  // namespace eig
