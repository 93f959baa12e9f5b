// q2.cu — E <- Q2 E, the bulge-chase half of the back-transform (a6).
//
// Paper: P:L93 ("since the tridiagonalisation is performed in two steps, the
// backtransformation requires two steps too"); grouping per DESIGN.md R7:
// block (i0, j) = H_{i0,j} ... H_{i0+g-1,j} = I - V T V^H, V a parallelogram
// (W = nb+g-1 rows x g cols, reflector t on block rows t..t+nb-1); groups of
// sweeps applied last to first, steps j ascending inside a group.
//
// B200 design (one persistent CTA per SM, 8 warps):
//  * the CTA owns a balanced, contiguous range of 8-column fragments of E and
//    sweeps all blocks for it in slabs of <= 9 fragments (72 columns);
//  * per block: V is expanded in shared memory into a dense zero-padded
//    parallelogram Vd[q][t] (the zero pattern never changes, so only the
//    g*nb live entries are rewritten by cp.async), T is copied, and only the
//    nb new rows of the sliding E window are loaded (each E row is read and
//    written once per group);
//  * three DMMA contractions from shared memory:
//      A: Y  = V^H E_win   warp w owns reflectors 4w..4w+3 and walks exactly
//                           the nb/2+2 k-steps where they are nonzero;
//      B: Y  = T Y         warp w walks k >= 4w (T upper triangular);
//      C: E -= V Y         warp w owns row groups w, w+8, w+16 and skips the
//                           k-steps outside the parallelogram;
//    all fragment loads are plain LDS.64 (no per-element bounds logic).
#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int QT = 256;
constexpr int NFMAX = 9;           // 8-column fragments per slab
constexpr int QBN = NFMAX * 8;     // 72 columns
constexpr int LDV = 36;            // Vd row stride (complex), == 4 mod 8
constexpr int LDT = 36;            // T column stride
constexpr int WPMAX = 96;          // padded window rows (nb + g - 1 <= 95)
constexpr int LDE = 98;            // E window column stride (complex), == 2 mod 8
constexpr int LDY = 34;            // Y column stride, == 2 mod 8

struct Q2Args {
  int64_t n, m, lde;
  int nb, g, W, Wp;
  int64_t ngroups;
  const int64_t *first;  // [ngroups+1]
  const int64_t *off;    // [J]
  const double2 *V2;
  const double2 *T2;
  double2 *E;
  int nfr_total;         // ceil(m / 8)
};

struct Smem {
  double2 *Vd, *T, *E, *Y;
};

__device__ __forceinline__ int64_t q2_steps(int64_t n, int nb, int64_t i0) {
  return (i0 > n - 2) ? 0 : (n - 2 - i0) / nb + 1;
}

// pair lanes (lane, lane^4) hold (Re, Im) rows of one complex row of a DMMA C fragment
__device__ __forceinline__ double2 c_pair(const double (&c)[2], int rp) {
  const double send = rp ? c[0] : c[1];
  const double recv = __shfl_xor_sync(0xffffffffu, send, 4);
  return rp ? make_double2(recv, c[1]) : make_double2(c[0], recv);
}

template <int NF>
__device__ void q2_slab(const Q2Args &a, const Smem &s, int64_t c0, int ncols) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const LaneEmb le(lane);
  const int rp = (lane >> 2) & 1;
  const int nb = a.nb, g = a.g, W = a.W, Wp = a.Wp;
  const int wu = __shfl_sync(0xffffffffu, warp, 0);   // provably warp-uniform copy of the warp id
  const double *vd = reinterpret_cast<const double *>(s.Vd);
  const double *se = reinterpret_cast<const double *>(s.E);
  const double *sy = reinterpret_cast<const double *>(s.Y);
  const double *st = reinterpret_cast<const double *>(s.T);
  const int nmfA = g / 4;            // reflector groups of 4
  const int nmfC = Wp / 4;           // row groups of 4

  for (int64_t gi = a.ngroups - 1; gi >= 0; gi--) {
    const int64_t i0 = gi * g;
    const int64_t J = q2_steps(a.n, nb, i0);
    for (int64_t j = 0; j < J; j++) {
      const int64_t rs = i0 + 1 + j * nb;
      const int64_t blk = a.first[gi] + j;
      // ---------------- loads: live V entries, T, new window rows
      {
        const int64_t last_i = a.n - 2 - j * nb;
        const int64_t nvalid = imax64(0, imin64(g, last_i - i0 + 1));
        const double2 *src = a.V2 + (a.off[j] + i0) * nb;
        for (int e = tid; e < g * nb; e += QT) {
          const int t = e / nb, sidx = e - t * nb;
          const bool ok = t < nvalid;
          cp_async16(&s.Vd[(t + sidx) * LDV + t], ok ? src + e : a.V2, ok);
        }
        const double2 *tsrc = a.T2 + blk * g * g;
        for (int e = tid; e < g * g; e += QT) {
          const int x = e % g, y = e / g;
          cp_async16(&s.T[y * LDT + x], tsrc + e, true);
        }
        const int rfirst = (j == 0) ? 0 : g - 1;
        const int nload = Wp - rfirst;
        for (int e = tid; e < NF * 8 * nload; e += QT) {
          const int q = rfirst + e % nload, c = e / nload;
          const int64_t row = rs + q;
          const bool ok = (q < W) && (row < a.n) && (c < ncols);
          cp_async16(&s.E[c * LDE + q], ok ? a.E + row + (c0 + c) * a.lde : a.E, ok);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
      }
      // ---------------- phase A: Y = V^H E_win
      if (warp < nmfA) {
        double acc[NF][2];
#pragma unroll
        for (int jj = 0; jj < NF; jj++) acc[jj][0] = acc[jj][1] = 0.0;
        const int t = wu * 4 + (lane >> 3);
        const int ks0 = wu * 2, nks = nb / 2 + 2;
        const int kq = (lane & 3) >> 1;
        for (int ks = ks0; ks < ks0 + nks; ks++) {
          const int q = ks * 2 + kq;
          const double av = xsign(vd[(q * LDV + t) * 2 + le.a_comp], le.a_neg_conj);
#pragma unroll
          for (int jj = 0; jj < NF; jj++) {
            const int nn = jj * 8 + (lane >> 2);
            dmma(acc[jj], av, se[(nn * LDE + q) * 2 + le.b_comp]);
          }
        }
#pragma unroll
        for (int jj = 0; jj < NF; jj++) {
          const double2 v = c_pair(acc[jj], rp);
          const int nn = jj * 8 + (lane & 3) * 2 + rp;
          s.Y[nn * LDY + t] = v;
        }
      }
      __syncthreads();
      // ---------------- phase B: Y = T Y   (T upper triangular)
      {
        double acc[NF][2];
#pragma unroll
        for (int jj = 0; jj < NF; jj++) acc[jj][0] = acc[jj][1] = 0.0;
        const bool act = warp < nmfA;
        if (act) {
          const int ra = warp * 4 + (lane >> 3);
          const int kq = (lane & 3) >> 1;
          for (int ks = wu * 2; ks < g / 2; ks++) {
            const int kb = ks * 2 + kq;
            const double av = st[(kb * LDT + ra) * 2 + le.a_comp];
            const double avs = xsign(av, le.a_neg);
#pragma unroll
            for (int jj = 0; jj < NF; jj++) {
              const int nn = jj * 8 + (lane >> 2);
              dmma(acc[jj], avs, sy[(nn * LDY + kb) * 2 + le.b_comp]);
            }
          }
        }
        __syncthreads();
        if (act) {
          const int ra = warp * 4 + (lane >> 3);
#pragma unroll
          for (int jj = 0; jj < NF; jj++) {
            const double2 v = c_pair(acc[jj], rp);
            const int nn = jj * 8 + (lane & 3) * 2 + rp;
            s.Y[nn * LDY + ra] = v;
          }
        }
      }
      __syncthreads();
      // ---------------- phase C: E_win -= V Y
      {
        const int kq = (lane & 3) >> 1;
#pragma unroll 1
        for (int i = 0; i < 3; i++) {
          const int mf = wu + 8 * i;
          if (mf >= nmfC) break;
          const int q0 = mf * 4;
          const int klo = max(0, q0 - nb + 1) >> 1, khi = min(g - 1, q0 + 3) >> 1;   // inclusive k-steps
          double acc[NF][2];
#pragma unroll
          for (int jj = 0; jj < NF; jj++) acc[jj][0] = acc[jj][1] = 0.0;
          const int q = q0 + (lane >> 3);
          for (int ks = klo; ks <= khi; ks++) {
            const int kt = ks * 2 + kq;
            const double av = xsign(vd[(q * LDV + kt) * 2 + le.a_comp], le.a_neg);
#pragma unroll
            for (int jj = 0; jj < NF; jj++) {
              const int nn = jj * 8 + (lane >> 2);
              dmma(acc[jj], av, sy[(nn * LDY + kt) * 2 + le.b_comp]);
            }
          }
          const int qo = q0 + (lane >> 3);
#pragma unroll
          for (int jj = 0; jj < NF; jj++) {
            const double2 v = c_pair(acc[jj], rp);
            const int nn = jj * 8 + (lane & 3) * 2 + rp;
            if (qo < W) {
              double2 &ev = s.E[nn * LDE + qo];
              ev.x -= v.x;
              ev.y -= v.y;
            }
          }
        }
      }
      __syncthreads();
      // ---------------- store rows leaving the window, shift the overlap
      {
        const bool lastj = (j == J - 1);
        const int nstore = lastj ? W : nb;
        for (int e = tid; e < NF * 8 * nstore; e += QT) {
          const int q = e % nstore, c = e / nstore;
          const int64_t row = rs + q;
          if (row < a.n && c < ncols) a.E[row + (c0 + c) * a.lde] = s.E[c * LDE + q];
        }
        if (!lastj) {
          __syncthreads();
          for (int e = tid; e < NF * 8 * (g - 1); e += QT) {
            const int q = e % (g - 1), c = e / (g - 1);
            s.E[c * LDE + q] = s.E[c * LDE + nb + q];
          }
        } else {
          __threadfence();   // the next group re-reads these rows through L2
        }
        __syncthreads();
      }
    }
  }
}

__global__ void __launch_bounds__(QT, 1) apply_q2_kernel(Q2Args a) {
  extern __shared__ __align__(16) double2 sm[];
  Smem s;
  s.Vd = sm;
  s.T = s.Vd + WPMAX * LDV;
  s.E = s.T + 32 * LDT;
  s.Y = s.E + QBN * LDE;
  // the parallelogram's zeros never change: clear Vd once
  for (int e = threadIdx.x; e < WPMAX * LDV; e += QT) s.Vd[e] = czero();
  __syncthreads();
  // balanced contiguous range of 8-column fragments for this CTA
  const int F = a.nfr_total, G = gridDim.x;
  const int f0 = (int)((int64_t)F * blockIdx.x / G), f1 = (int)((int64_t)F * (blockIdx.x + 1) / G);
  const int nslab = (f1 - f0 + NFMAX - 1) / NFMAX;
  for (int sl = 0; sl < nslab; sl++) {
    const int fa = f0 + (int)((int64_t)(f1 - f0) * sl / nslab), fb = f0 + (int)((int64_t)(f1 - f0) * (sl + 1) / nslab);
    const int nf = fb - fa;
    const int64_t c0 = (int64_t)fa * 8;
    const int ncols = (int)imin64((int64_t)nf * 8, a.m - c0);
    switch (nf) {
      case 1: q2_slab<1>(a, s, c0, ncols); break;
      case 2: q2_slab<2>(a, s, c0, ncols); break;
      case 3: q2_slab<3>(a, s, c0, ncols); break;
      case 4: q2_slab<4>(a, s, c0, ncols); break;
      case 5: q2_slab<5>(a, s, c0, ncols); break;
      case 6: q2_slab<6>(a, s, c0, ncols); break;
      case 7: q2_slab<7>(a, s, c0, ncols); break;
      case 8: q2_slab<8>(a, s, c0, ncols); break;
      case 9: q2_slab<9>(a, s, c0, ncols); break;
      default: break;
    }
  }
}

}  // namespace

int q2_apply(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *T2, double2 *E, int64_t lde, int64_t m) {
  if (p.nblocks <= 0 || m <= 0) return 0;
  if (p.g > 32 || p.nb > 64 || p.g % 4 != 0 || p.g < 4 || p.nb < p.g - 1 || (p.nb % 2)) return EIG_ERR_NOTIMPL;
  Q2Args a;
  a.n = p.n;
  a.m = m;
  a.lde = lde;
  a.nb = p.nb;
  a.g = p.g;
  a.W = p.nb + p.g - 1;
  a.Wp = (a.W + 3) & ~3;   // multiple of 4 rows (phase C row groups); <= 96
  a.ngroups = p.ngroups;
  a.first = p.d_group_first_block;
  a.off = p.d_off;
  a.V2 = V2;
  a.T2 = T2;
  a.E = E;
  a.nfr_total = (int)((m + 7) / 8);
  const size_t smem = ((size_t)WPMAX * LDV + 32 * LDT + (size_t)QBN * LDE + (size_t)QBN * LDY) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    EIG_TRY(ctx.check(cudaFuncSetAttribute(apply_q2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "q2 attr"));
    attr = true;
  }
  const int grid = std::min(ctx.num_sms, a.nfr_total);
  apply_q2_kernel<<<grid, QT, smem, ctx.stream>>>(a);
  return ctx.launched("apply_q2_kernel");
}

}  // namespace eig
