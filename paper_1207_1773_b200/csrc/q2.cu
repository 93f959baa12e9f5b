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
#include <cstdlib>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int NH = 2;                // column parts
constexpr int QT = 256 * NH;         // 8 reflector/row groups x NH column parts

// fragments of part h when NF fragments are split over NH parts
__host__ __device__ constexpr int nf_part(int NF, int h) { return (NF + NH - 1 - h) / NH; }
__host__ __device__ constexpr int nf_lo(int NF, int h) { return h == 0 ? 0 : nf_lo(NF, h - 1) + nf_part(NF, h - 1); }
__host__ __device__ constexpr int nf_c(int NF, int h) { return nf_part(NF, h) > 0 ? nf_part(NF, h) : 1; }
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
  unsigned long long *prof;  // optional: CTA 0 phase cycle counters [5] (load, A, B, C, commit)
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

// Window rows live in a ring of R = W slots (row q of the block starting at
// ring offset `base` is slot (q + base) mod R), so sliding the window by nb
// rows needs no data movement: block j+1's nb new rows overwrite the slots of
// block j's first nb rows, which phase C writes straight to global memory.
__device__ __forceinline__ int ring(int q, int base, int R) {
  int r = q + base;
  return r >= R ? r - R : r;
}

// Phase A for one warp: Y[t, cols] = sum_q conj(V[q][t]) E[q, cols] over the
// nb/2+2 k-steps where reflectors 4mw..4mw+3 are nonzero.
template <int NFH>
__device__ __forceinline__ void phase_a(const double *vd, const double *se, double2 *sY, int mw, int nlo, int nb,
                                        int base, int R, int lane, const LaneEmb &le, int rp) {
  double acc[NFH][2];
#pragma unroll
  for (int jj = 0; jj < NFH; jj++) acc[jj][0] = acc[jj][1] = 0.0;
  const int t = mw * 4 + (lane >> 3);
  const int kq = (lane & 3) >> 1;
  const int ks0 = mw * 2, nks = nb / 2 + 2;
  int q = ks0 * 2 + kq;
  int r = ring(q, base, R);
  const double *eb = se + le.b_comp + ((nlo * 8 + (lane >> 2)) * LDE) * 2;
  // software pipeline: fragments of k-step ks+1 are loaded while ks computes
  double fa = xsign(vd[(q * LDV + t) * 2 + le.a_comp], le.a_neg_conj);
  double fb[NFH];
#pragma unroll
  for (int jj = 0; jj < NFH; jj++) fb[jj] = eb[(jj * 8 * LDE + r) * 2];
  for (int ks = 0; ks < nks; ks++) {
    q += 2;
    r += 2;
    if (r >= R) r -= R;
    const bool more = ks + 1 < nks;
    double na = 0.0, nbv[NFH];
    if (more) na = xsign(vd[(q * LDV + t) * 2 + le.a_comp], le.a_neg_conj);
#pragma unroll
    for (int jj = 0; jj < NFH; jj++) nbv[jj] = more ? eb[(jj * 8 * LDE + r) * 2] : 0.0;
#pragma unroll
    for (int jj = 0; jj < NFH; jj++) dmma(acc[jj], fa, fb[jj]);
    fa = na;
#pragma unroll
    for (int jj = 0; jj < NFH; jj++) fb[jj] = nbv[jj];
  }
#pragma unroll
  for (int jj = 0; jj < NFH; jj++) {
    const double2 v = c_pair(acc[jj], rp);
    sY[((nlo + jj) * 8 + (lane & 3) * 2 + rp) * LDY + t] = v;
  }
}

// Phase B for one warp: Y2[t, cols] = sum_{k >= t} T[t][k] Y[k, cols] into
// registers (nfh <= NFH fragments are live).
template <int NFH>
__device__ __forceinline__ void phase_b(const double *st, const double *sy, double (&acc)[NFH][2], int mw, int nlo,
                                        int nfh, int g, int lane, const LaneEmb &le) {
#pragma unroll
  for (int jj = 0; jj < NFH; jj++) acc[jj][0] = acc[jj][1] = 0.0;
  const int ra = mw * 4 + (lane >> 3);
  const int kq = (lane & 3) >> 1;
  const double *yb = sy + le.b_comp + ((nlo * 8 + (lane >> 2)) * LDY) * 2;
#pragma unroll 2
  for (int ks = mw * 2; ks < g / 2; ks++) {
    const int kb = ks * 2 + kq;
    const double av = xsign(st[(kb * LDT + ra) * 2 + le.a_comp], le.a_neg);
#pragma unroll
    for (int jj = 0; jj < NFH; jj++)
      if (jj < nfh) dmma(acc[jj], av, yb[(jj * 8 * LDY + kb) * 2]);
  }
}

// What phase C refills for the next block of the same group.
struct NextBlk {
  bool more;            // a next block exists in this group
  int64_t rs1;          // its first window row
  int base1;            // its ring offset
  const double2 *v2;    // its V2 slots (slot t at v2 + t*nb)
  int nvalid;           // live slots
};

// Phase C for one warp: E[q, cols] -= sum_t V[q][t] Y2[t, cols] for row groups
// mw, mw+8, mw+16; rows q < nout leave the window and go straight to global.
// As soon as the warp is done with a row group, it refills (cp.async) the
// Vd rows of that group with the next block's V and, for rows q < nb, the
// ring slots with the next block's new E rows; no other warp touches them
// before the end-of-block barrier, so the loads overlap the rest of phase C.
template <int NFH>
__device__ __forceinline__ void phase_c(const Q2Args &a, double2 *sVd, const double *sy, double2 *sE, int mw,
                                        int nlo, int nfh, int h, int base, int R, int nout, int64_t rs, int64_t c0, int ncols,
                                        int ncolsl, const NextBlk &nx, int lane, const LaneEmb &le, int rp) {
  const int nb = a.nb, g = a.g, W = a.W, nmfC = a.Wp / 4;
  const int kq = (lane & 3) >> 1;
  const double *vd = reinterpret_cast<const double *>(sVd);
  const double *yb = sy + le.b_comp + ((nlo * 8 + (lane >> 2)) * LDY) * 2;
#pragma unroll 1
  for (int i = 0; i < 3; i++) {
    const int mf = mw + 8 * i;
    if (mf >= nmfC) break;
    const int q0 = mf * 4;
    if (nfh > 0) {
    const int klo = max(0, q0 - nb + 1) >> 1, khi = min(g - 1, q0 + 3) >> 1;
    double acc[NFH][2];
#pragma unroll
    for (int jj = 0; jj < NFH; jj++) acc[jj][0] = acc[jj][1] = 0.0;
    const int q = q0 + (lane >> 3);
    const double *vq = vd + le.a_comp + (q * LDV) * 2;
    int kt = klo * 2 + kq;
    double fa = xsign(vq[kt * 2], le.a_neg);
    double fb[NFH];
#pragma unroll
    for (int jj = 0; jj < NFH; jj++) fb[jj] = yb[(jj * 8 * LDY + kt) * 2];
    for (int ks = klo; ks <= khi; ks++) {
      kt += 2;
      const bool more = ks < khi;
      double na = 0.0, nbv[NFH];
      if (more) na = xsign(vq[kt * 2], le.a_neg);
#pragma unroll
      for (int jj = 0; jj < NFH; jj++) nbv[jj] = more ? yb[(jj * 8 * LDY + kt) * 2] : 0.0;
#pragma unroll
      for (int jj = 0; jj < NFH; jj++) dmma(acc[jj], fa, fb[jj]);
      fa = na;
#pragma unroll
      for (int jj = 0; jj < NFH; jj++) fb[jj] = nbv[jj];
    }
    const bool live = q < W;
    const int r = ring(q, base, R);
    const int64_t row = rs + q;
#pragma unroll
    for (int jj = 0; jj < NFH; jj++) {
      const double2 v = c_pair(acc[jj], rp);
      const int nn = (nlo + jj) * 8 + (lane & 3) * 2 + rp;
      if (live) {
        double2 *ep = &sE[nn * LDE + r];
        double2 ev = *ep;
        ev.x -= v.x;
        ev.y -= v.y;
        if (q < nout) {
          if (row < a.n && nn < ncols) a.E[row + (c0 + nn) * a.lde] = ev;
        } else {
          *ep = ev;
        }
      }
    }
    }
    if (nx.more) {
      // both column halves of this row group must be done before its slots are refilled
      asm volatile("bar.sync %0, %1;" ::"r"(1 + mw), "r"(32 * NH) : "memory");
      // next block's V entries of rows q0..q0+3: Vd[qq][t] = v_t[qq - t]   (part 0; t = lane, g <= 32)
      if (h == 0 && lane < g) {
        const int t = lane;
#pragma unroll
        for (int rr = 0; rr < 4; rr++) {
          const int qq = q0 + rr, sidx = qq - t;
          if (qq < W && sidx >= 0 && sidx < nb) {
            const bool ok = t < nx.nvalid;
            cp_async16(&sVd[qq * LDV + t], ok ? nx.v2 + t * nb + sidx : a.V2, ok);
          }
        }
      }
      // next block's new E rows land in the ring slots of rows q0..q0+3 (< nb)   (parts 1..)
      if (h >= 1 && q0 < nb) {
        for (int e = lane + 32 * (h - 1); e < 4 * ncolsl; e += 32 * (NH - 1)) {
          const int qq = q0 + (e & 3), c = e >> 2;
          if (qq < nb) {
            const int64_t row1 = nx.rs1 + qq + g - 1;
            const bool ok = (row1 < a.n) && (c < ncols);
            cp_async16(&sE[c * LDE + ring(qq, base, R)], ok ? a.E + row1 + (c0 + c) * a.lde : a.E, ok);
          }
        }
      }
    }
  }
}

template <int NF>
__device__ __forceinline__ void q2_slab(const Q2Args &a, const Smem &s, int64_t c0, int ncols) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int wu = __shfl_sync(0xffffffffu, tid >> 5, 0);   // provably warp-uniform warp id
  // SMSP s (= wu % 4) gets reflector groups s and 7 - s of every part, which
  // balances the triangular phase B across the four schedulers
  const int mw = ((wu >> 2) & 1) ? 7 - (wu & 3) : (wu & 3), h = wu >> 3;
  constexpr int NF0 = nf_c(NF, 0), NF1 = nf_c(NF, 1), NF2 = nf_c(NF, NH > 2 ? 2 : 1);
  const int nlo = h == 0 ? 0 : h == 1 ? nf_lo(NF, 1) : nf_lo(NF, 2);
  const int nfh = h == 0 ? nf_part(NF, 0) : h == 1 ? nf_part(NF, 1) : nf_part(NF, 2);
  const LaneEmb le(lane);
  const int rp = (lane >> 2) & 1;
  const int nb = a.nb, g = a.g, W = a.W, R = a.W;
  const double *vd = reinterpret_cast<const double *>(s.Vd);
  const double *se = reinterpret_cast<const double *>(s.E);
  const double *sy = reinterpret_cast<const double *>(s.Y);
  const double *st = reinterpret_cast<const double *>(s.T);
  const bool actAB = mw < g / 4 && nfh > 0;
  constexpr int PV = (32 * 64 + QT - 1) / QT;          // prefetched V elements per thread (g <= 32)
  const int ncolsl = NF * 8;
  // element e = tid + k*QT of an (nb x *) array is (row e % nb, col e / nb): per-thread start and
  // per-k increments, so the prefetch loops need no integer division
  const int d_q = QT % nb, d_c = QT / nb;
  const int q_0 = tid % nb, c_0 = tid / nb;
  // optional phase profile (CTA 0, thread 0), accumulated in shared memory so
  // that it costs no registers when disabled
  __shared__ long long t_acc[6];   // [5] = last mark
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && tid == 0;
  if (prof)
    for (int k = 0; k < 6; k++) t_acc[k] = 0;
  auto mark = [&](int k) {
    if (prof) {
      const long long now = clock64();
      if (k >= 0) t_acc[k] += now - t_acc[5];
      t_acc[5] = now;
    }
  };

  for (int64_t gi = a.ngroups - 1; gi >= 0; gi--) {
    const int64_t i0 = gi * g;
    const int64_t J = q2_steps(a.n, nb, i0);
    int base = 0;
    for (int64_t j = 0; j < J; j++) {
      const int64_t rs = i0 + 1 + j * nb;
      const int64_t blk = a.first[gi] + j;
      mark(-1);
      if (j == 0) {
        // group start: live V entries, T and the whole window, synchronously
        const int64_t nvalid = imax64(0, imin64(g, a.n - 2 - i0 + 1));
        const double2 *src = a.V2 + (a.off[0] + i0) * nb;
        int qq = q_0, cc = c_0;
        for (int k = 0; k < PV; k++) {
          if (cc < g) {
            const bool ok = cc < nvalid;
            cp_async16(&s.Vd[(cc + qq) * LDV + cc], ok ? src + cc * nb + qq : a.V2, ok);
          }
          qq += d_q;
          cc += d_c;
          if (qq >= nb) { qq -= nb; cc++; }
        }
        const double2 *tsrc = a.T2 + blk * g * g;
        for (int y = wu; y < g; y += QT / 32)
          for (int x = lane; x < g; x += 32) cp_async16(&s.T[y * LDT + x], tsrc + y * g + x, true);
        for (int c = wu; c < ncolsl; c += QT / 32)
          for (int q = lane; q < W; q += 32) {
            const int64_t row = rs + q;
            const bool ok = (row < a.n) && (c < ncols);
            cp_async16(&s.E[c * LDE + q], ok ? a.E + row + (c0 + c) * a.lde : a.E, ok);
          }
        cp_async_commit();
      }
      cp_async_wait<0>();
      __syncthreads();
      mark(0);
      // ---------------- phase A: Y = V^H E_win
      if (actAB) {
        if (h == 0) phase_a<NF0>(vd, se, s.Y, mw, nlo, nb, base, R, lane, le, rp);
        else if (h == 1) phase_a<NF1>(vd, se, s.Y, mw, nlo, nb, base, R, lane, le, rp);
        else phase_a<NF2>(vd, se, s.Y, mw, nlo, nb, base, R, lane, le, rp);
      }
      __syncthreads();
      mark(1);
      // ---------------- phase B: Y = T Y
      {
        double acc[NF0][2];
        if (actAB) phase_b<NF0>(st, sy, acc, mw, nlo, nfh, g, lane, le);
        __syncthreads();
        if (actAB) {
          const int ra = mw * 4 + (lane >> 3);
#pragma unroll
          for (int jj = 0; jj < NF0; jj++) {
            const double2 v = c_pair(acc[jj], rp);
            if (jj < nfh) s.Y[((nlo + jj) * 8 + (lane & 3) * 2 + rp) * LDY + ra] = v;
          }
        }
      }
      __syncthreads();
      mark(2);
      // ---------------- phase C (+ refill for the next block of this group)
      const bool more = (j + 1 < J);
      NextBlk nx;
      nx.more = more;
      nx.rs1 = rs + nb;
      nx.base1 = (base + nb) % R;
      nx.v2 = more ? a.V2 + (a.off[j + 1] + i0) * nb : a.V2;
      nx.nvalid = more ? (int)imax64(0, imin64(g, a.n - 2 - (j + 1) * nb - i0 + 1)) : 0;
      if (more) {
        const double2 *tsrc = a.T2 + (blk + 1) * g * g;
        for (int y = wu; y < g; y += QT / 32)
          for (int x = lane; x < g; x += 32) cp_async16(&s.T[y * LDT + x], tsrc + y * g + x, true);
      }
      if (h == 0)
        phase_c<NF0>(a, s.Vd, sy, s.E, mw, nlo, nfh, h, base, R, more ? nb : W, rs, c0, ncols, ncolsl, nx, lane, le, rp);
      else if (h == 1)
        phase_c<NF1>(a, s.Vd, sy, s.E, mw, nlo, nfh, h, base, R, more ? nb : W, rs, c0, ncols, ncolsl, nx, lane, le, rp);
      else
        phase_c<NF2>(a, s.Vd, sy, s.E, mw, nlo, nfh, h, base, R, more ? nb : W, rs, c0, ncols, ncolsl, nx, lane, le, rp);
      cp_async_commit();
      mark(3);
      if (more) {
        base = nx.base1;
      } else {
        __threadfence();   // the next group re-reads these rows through L2
      }
      mark(4);
    }
  }
  __syncthreads();
  if (prof)
    for (int k = 0; k < 5; k++) atomicAdd(&a.prof[k], (unsigned long long)t_acc[k]);
}

// Every CTA runs slabs of exactly NF fragments (one template instance per
// launch keeps the register allocation of each NF separate); a CTA whose own
// range is shorter computes the extra fragments on zero-filled columns and
// never stores them, which costs nothing because the CTAs with the longest
// range set the kernel time anyway.
template <int NF>
__global__ void __launch_bounds__(QT, 1) apply_q2_kernel(Q2Args a, int nslab) {
  extern __shared__ __align__(16) double2 sm[];
  Smem s;
  s.Vd = sm;
  s.T = s.Vd + WPMAX * LDV;
  s.E = s.T + 32 * LDT;
  s.Y = s.E + QBN * LDE;
  // the parallelogram's zeros never change: clear Vd once
  for (int e = threadIdx.x; e < WPMAX * LDV; e += QT) s.Vd[e] = czero();
  __syncthreads();
  const int F = a.nfr_total, G = gridDim.x;
  const int f0 = (int)((int64_t)F * blockIdx.x / G), f1 = (int)((int64_t)F * (blockIdx.x + 1) / G);
  for (int sl = 0; sl < nslab; sl++) {
    const int fa = f0 + sl * NF;
    const int64_t c0 = (int64_t)fa * 8;
    const int ncols = (int)imin64(imin64((int64_t)(f1 - fa) * 8, a.m - c0), NF * 8);
    if (ncols <= 0) break;
    q2_slab<NF>(a, s, c0, ncols);
  }
}

}  // namespace

int q2_apply(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *T2, double2 *E, int64_t lde, int64_t m) {
  if (p.nblocks <= 0 || m <= 0) return 0;
  // the wavefront kernel (q2w.cu) for its shape (nb = 64, g = 32) unless EIG_Q2_WAVE=0
  {
    const int rc = q2w_apply(ctx, p, V2, T2, E, lde, m);
    if (rc <= 0) return rc;
  }
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
  a.prof = ctx.q2_prof;
  const size_t smem = ((size_t)WPMAX * LDV + 32 * LDT + (size_t)QBN * LDE + (size_t)QBN * LDY) * sizeof(double2);
  const int grid = std::min(ctx.num_sms, a.nfr_total);
  const int per = (a.nfr_total + grid - 1) / grid;        // fragments of the longest CTA range
  const int nslab = (per + NFMAX - 1) / NFMAX;
  const int nf = (per + nslab - 1) / nslab;
#define Q2_CASE(K)                                                                      \
  case K:                                                                               \
    EIG_TRY(ctx.smem_attr((const void *)apply_q2_kernel<K>, (int)smem, "q2 attr"));     \
    apply_q2_kernel<K><<<grid, QT, smem, ctx.stream>>>(a, nslab);                       \
    break;
  switch (nf) {
    Q2_CASE(1) Q2_CASE(2) Q2_CASE(3) Q2_CASE(4) Q2_CASE(5) Q2_CASE(6) Q2_CASE(7) Q2_CASE(8) Q2_CASE(9)
    default: return EIG_ERR_NOTIMPL;
  }
#undef Q2_CASE
  return ctx.launched("apply_q2_kernel");
}

}  // namespace eig
