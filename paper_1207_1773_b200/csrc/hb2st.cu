// hb2st.cu — second stage of the two-stage reduction on the device (NEXT-1):
// Hermitian band (half-bandwidth nb) -> real symmetric tridiagonal by
// column-wise bulge chasing ("we differ by using a column-wise
// elimination"; reading R5), producing the Q2 reflectors in the V2
// layout of include/eig.h.
//
// Task (i, j) (sweep i, step j): target column c = i (j = 0) or
// i+1+(j-1)nb, rows R = [r0, r1] = [i+1+j nb, min(i+(j+1)nb, n-1)]:
//   (beta, tau, v) = zlarfg(M[R, c]);  M[r0, c] = beta, M[r0+1:r1, c] = 0;
//   (a) M[R, k] <- H^H M[R, k] for the rest of the previous bulge, c < k < r0;
//   (b) M[R, R] <- H^H M[R, R] H            (p = tau D v, w = p - tau/2 (p^H v) v);
//   (c) M[k, R] <- M[k, R] H for r1 < k <= min(r1 + nb, n-1)  (creates the next bulge).
// Sequential order: sweep i-1 entirely before sweep i.  Task (i, j) touches
// rows [r0, r1 + nb] x cols [c, r1]; of sweep i-1 only its steps <= j+2
// overlap that region, so sweep i may run step j once sweep i-1 has finished
// step j+2: a wavefront of ~J/3 concurrent sweeps.  One persistent
// cooperative kernel: sweep i is owned by CTA i mod P, progress flags in
// global memory (release/acquire), the band (2nb+1 diagonals, lower) lives in
// L2 and is accessed with L1-bypassing loads.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int HT = 512;

struct HbArgs {
  int64_t n;
  int nb, ldab;
  double2 *AB;            // band: M(r, c) = AB[(r - c) + c * ldab], 0 <= r - c <= 2nb
  double2 *V2, *tau2;     // outputs (V2 layout)
  const int64_t *off;     // slot offsets per step j
  int *progress;          // [n] steps completed per sweep
  int *progressA;         // [n] steps whose reflector outputs (V2, tau2, target column) are stored
  unsigned long long *prof;  // optional: CTA 0 phase cycles [16..21] (wait, refl, a, b, c, flag)
};

__device__ __forceinline__ int ld_acquire_i32(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_i32(int *p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Task layout (one CTA, 8 warps):
//   1. every thread issues its cp.async loads at once: the target column x,
//      the rest of the previous bulge Ablk = M[R, c+1:r0], the diagonal block
//      D = M[R, R] (lower) and the rows below Cblk = M[r1+1:kend, R];
//   2. warp 0 builds (beta, tau, v) and writes the reflector outputs;
//   3. the three updates run concurrently: warps 0-1 (a) on Ablk, warps 2-5
//      (b) on D, warps 6-7 (c) on Cblk, each storing straight to global.
constexpr int LDD = 65;
__global__ void __launch_bounds__(HT, 1) hb2st_kernel(HbArgs a) {
  extern __shared__ __align__(16) double2 hsm[];
  double2 *sD = hsm;                  // [64][LDD] diagonal block (lower)
  double2 *sP0 = sD + 64 * LDD;       // two [64 cols][64 rows] bulge buffers (column-major, row index fast)
  double2 *sxg = sP0 + 2 * 64 * 64;   // [64] x of the first task of a sweep
  __shared__ double2 sv2[2][64];      // reflector of this task / of the next (computed early)
  __shared__ double2 sp[64];          // p, then w
  __shared__ double2 sg[64];          // g = tau (C v)
  __shared__ double2 sf[64];          // f = conj(tau) v^H Ablk
  __shared__ double2 spart[8][64];    // partial dot products
  __shared__ double2 s_tau2[2], s_beta2[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n;
  const int nb = a.nb, ldab = a.ldab;
  double2 *AB = a.AB;
  auto M = [&](int64_t r, int64_t c) -> double2 * { return AB + (r - c) + c * (int64_t)ldab; };
  const bool prof = a.prof != nullptr && blockIdx.x == 0 && tid == 0;
  long long tm = 0, tacc[6] = {0, 0, 0, 0, 0, 0};
  auto mark = [&](int k) {
    if (prof) {
      const long long now = clock64();
      if (k >= 0) tacc[k] += now - tm;
      tm = now;
    }
  };
  // Before task (i, j) touches D_j / Cblk_j, sweep i-1 must have finished its
  // steps <= j+1; of its step j+2 only the target column matters (the single
  // element M(r0_{j+2}, c_{j+2}) = beta is the one overlap with task (i, j)'s
  // region), and that is stored right after its reflector, so the
  // sweep-to-sweep lag is two steps plus a reflector instead of three steps.
  auto wait_prev = [&](int64_t i, int64_t j) {
    if (i > 0 && tid == 0) {
      const int64_t prev = i - 1;
      const int64_t nprev = (n - 2 - prev) / nb + 1;
      const int need = (int)imin64(j + 2, nprev), need_a = (int)imin64(j + 3, nprev);
      while (ld_acquire_i32(a.progress + prev) < need) {
      }
      while (ld_acquire_i32(a.progressA + prev) < need_a) {
      }
    }
    __syncthreads();
  };

  // Task (i, j+1) starts from task (i, j)'s updated Cblk: its target column x
  // is Cblk's column 0 and its previous bulge Ablk is Cblk's columns 1.. (same
  // rows).  So Cblk stays in shared memory (buffers alternate), is never
  // stored by task j (task j+1 stores the final values of that region), and
  // x / Ablk need no load; the reflector and the (a) update run before the
  // wait on sweep i-1, which only D_j and Cblk_j depend on.
  // zlarfg (reading R1) of x = (x0 at lane, x1 at lane + 32), length len, by
  // one warp, into reflector buffer b (entries in the band's scaled units,
  // <= 1, see hb2st())
  auto reflector = [&](double2 x0, double2 x1, double2 al, int len, int b) {
    double nrm = (lane >= 1 ? x0.x * x0.x + x0.y * x0.y : 0.0) + x1.x * x1.x + x1.y * x1.y;
    nrm = warp_sum(nrm);
    double2 tau, scale;
    double beta;
    if (nrm == 0.0 && al.y == 0.0) {
      tau = czero();
      beta = al.x;
      scale = czero();
    } else {
      beta = -copysign(sqrt(al.x * al.x + al.y * al.y + nrm), al.x);
      const double ib = 1.0 / beta;   // two divisions instead of four (critical path)
      tau = make_double2((beta - al.x) * ib, -al.y * ib);
      const double2 d = make_double2(al.x - beta, al.y);
      const double idd = 1.0 / (d.x * d.x + d.y * d.y);
      scale = make_double2(d.x * idd, -d.y * idd);
    }
    sv2[b][lane] = (lane == 0) ? make_double2(1.0, 0.0) : (lane < len ? cmul(x0, scale) : czero());
    sv2[b][lane + 32] = (lane + 32 < len) ? cmul(x1, scale) : czero();
    if (lane == 0) {
      s_tau2[b] = tau;
      s_beta2[b] = make_double2(beta, 0.0);
    }
  };

  // Pipelining across the tasks of a sweep: the target column of task j+1 is
  // column 0 of task j's updated Cblk, so warp 0 updates that column first and
  // builds task j+1's reflector while the other warps finish the (b) / (c)
  // updates of task j; task j+1 then starts with its reflector in hand.
  for (int64_t i = blockIdx.x; i + 1 < n; i += gridDim.x) {
    int cur = 0, rb = 0;
    int64_t off_next = a.off[0];   // V2 slot offsets, read one task ahead
    for (int64_t j = 0;; j++) {
      const int64_t off_j = off_next;
      const int64_t c = (j == 0) ? i : i + 1 + (j - 1) * nb;
      const int64_t r0 = i + 1 + j * nb;
      if (r0 > n - 1) break;
      const int64_t r1 = imin64(i + (j + 1) * nb, n - 1);
      const int len = (int)(r1 - r0 + 1);
      const int na = (int)(r0 - c - 1);                       // previous-bulge columns
      const int64_t kend = imin64(r1 + nb, n - 1);
      const int nc = (int)(kend - r1);                        // rows below R
      double2 *sC = sP0 + cur * 4096;                         // this task's Cblk
      const double2 *sPrev = sP0 + (cur ^ 1) * 4096;          // previous task's Cblk = [x | Ablk]
      const double2 *sA = sPrev + 64;                         // Ablk column k at sA + k*64
      const double2 *sv = sv2[rb];
      if (r1 < n - 1) off_next = a.off[j + 1];
      mark(-1);
      if (j == 0) {
        wait_prev(i, j);
        for (int t = tid; t < len; t += HT) cp_async16(&sxg[t], M(r0 + t, c), true);
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
      }
      mark(0);
      // ---- reflector: the first task of a sweep builds it here, the others
      // got it from the previous task's update phase
      if (j == 0) {
        if (warp == 0)
          reflector(lane < len ? sxg[lane] : czero(), lane + 32 < len ? sxg[lane + 32] : czero(), sxg[0], len, rb);
        __syncthreads();
      }
      const double2 tau = s_tau2[rb], ctau = cconj(tau);
      const bool upd = tau.x != 0.0 || tau.y != 0.0;
      {
        const int64_t slot = off_j + i;
        for (int t = tid; t < nb; t += HT) a.V2[slot * nb + t] = (t < len) ? sv[t] : czero();
        if (tid == 0) a.tau2[slot] = tau;
        for (int t = tid; t < len; t += HT) *M(r0 + t, c) = (t == 0) ? s_beta2[rb] : czero();
      }
      __syncthreads();
      if (tid == 0) st_release_i32(a.progressA + i, (int)(j + 1));
      // ---- (a) on the previous bulge (shared memory only): f, then store
      if (na > 0) {
        if (upd) {   // one warp per column: lanes over the rows (conflict-free), shuffle reduction
          for (int q = warp; q < na; q += HT / 32) {
            double2 acc = czero();
            if (lane < len) acc = cmulc(sv[lane], sA[lane + q * 64]);
            if (lane + 32 < len) acc = cadd(acc, cmulc(sv[lane + 32], sA[lane + 32 + q * 64]));
            acc = warp_sum2(acc);
            if (lane == 0) sf[q] = cmul(ctau, acc);
          }
        }
        __syncthreads();
        for (int e = tid; e < na * 64; e += HT) {          // y_k - v f_k  (stored even if tau = 0:
          const int t = e & 63, k = e >> 6;               //  the previous task left this region in smem)
          if (t < len) *M(r0 + t, c + 1 + k) = upd ? csub(sA[t + k * 64], cmul(sv[t], sf[k])) : sA[t + k * 64];
        }
      }
      mark(2);
      // ---- D_j and Cblk_j, after sweep i-1 is done with them
      if (j > 0) wait_prev(i, j);
      mark(1);
      for (int e = tid; e < 64 * 64; e += HT) {
        const int rr = e & 63, cc = e >> 6;
        if (rr < len && cc <= rr) cp_async16(&sD[rr + cc * LDD], M(r0 + rr, r0 + cc), true);
      }
      for (int e = tid; e < 64 * 64; e += HT) {
        const int rr = e & 63, t = e >> 6;
        if (rr < nc && t < len) cp_async16(&sC[rr + t * 64], M(r1 + 1 + rr, r0 + t), true);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      mark(4);
      if (upd) {
        //   p_r = tau (D v)_r;  g_rr = tau (Cblk v)_rr   (each split in two halves)
        {   // 8 groups of 64 threads: D (groups 0-3) and Cblk (4-7), 16 terms each
          const int g = tid >> 6, q = tid & 63, h = g & 3;
          const int t0 = h * 16, t1 = imin64(t0 + 16, len);
          double2 acc = czero();
          if (g < 4) {
            if (q < len)
              for (int cc = t0; cc < t1; cc++) {
                double2 d;
                if (cc < q) d = sD[q + cc * LDD];
                else if (cc > q) d = cconj(sD[cc + q * LDD]);
                else d = make_double2(sD[q + q * LDD].x, 0.0);
                acc = cadd(acc, cmul(d, sv[cc]));
              }
          } else {
            if (q < nc)
              for (int t = t0; t < t1; t++) acc = cadd(acc, cmul(sC[q + t * 64], sv[t]));
          }
          spart[g][q] = acc;
        }
        __syncthreads();
        if (tid < 64) {
          if (tid < len) sp[tid] = cmul(tau, cadd(cadd(spart[0][tid], spart[1][tid]), cadd(spart[2][tid], spart[3][tid])));
        } else if (tid < 128) {
          const int rr = tid - 64;
          if (rr < nc) sg[rr] = cmul(cadd(cadd(spart[4][rr], spart[5][rr]), cadd(spart[6][rr], spart[7][rr])), tau);
        }
        __syncthreads();
        if (warp == 0) {   // w = p - 1/2 tau (p^H v) v
          double2 sdot = czero();
          for (int t = lane; t < len; t += 32) sdot = cadd(sdot, cmulc(sp[t], sv[t]));
          sdot = warp_sum2(sdot);
          const double2 al = cmul(make_double2(-0.5 * tau.x, -0.5 * tau.y), sdot);
          for (int t = lane; t < len; t += 32) sp[t] = cadd(sp[t], cmul(al, sv[t]));
        }
        __syncthreads();
        if (warp > 0) {
          for (int e = tid - 32; e < 64 * 64; e += HT - 32) {   // (b) D - v w^H - w v^H (lower), to global
            const int rr = e & 63, cc = e >> 6;
            if (rr < len && cc <= rr) {
              double2 d = sD[rr + cc * LDD];
              d = csub(d, cadd(cmul(sv[rr], cconj(sp[cc])), cmul(sp[rr], cconj(sv[cc]))));
              if (rr == cc) d.y = 0.0;
              *M(r0 + rr, r0 + cc) = d;
            }
          }
          for (int e = tid - 32; e < 64 * 63; e += HT - 32) {   // (c) y - g v^H, columns 1.. (smem)
            const int rr = e & 63, t = 1 + (e >> 6);
            if (rr < nc && t < len) sC[rr + t * 64] = csub(sC[rr + t * 64], cmul(sg[rr], cconj(sv[t])));
          }
        } else {   // warp 0: column 0 of (c), which is the next task's target column
          for (int rr = lane; rr < nc; rr += 32) sC[rr] = csub(sC[rr], cmul(sg[rr], cconj(sv[0])));
        }
      }
      // warp 0: the next task's reflector from that column (its length is nc)
      if (warp == 0 && r1 < n - 1) {
        __syncwarp();
        reflector(lane < nc ? sC[lane] : czero(), lane + 32 < nc ? sC[lane + 32] : czero(), sC[0], nc, rb ^ 1);
      }
      mark(3);
      // the barrier orders every thread's D / Ablk stores before thread 0's
      // gpu-scope release store, which is cumulative over them (PTX memory
      // model): no separate fence
      __syncthreads();
      if (tid == 0) st_release_i32(a.progress + i, (int)(j + 1));
      mark(5);
      cur ^= 1;
      rb ^= 1;
    }
  }
  if (prof)
    for (int k = 0; k < 6; k++) atomicAdd(&a.prof[16 + k], (unsigned long long)tacc[k]);
}

// ---------------------------------------------------------------- systolic chase
// Position-stationary form of the same chase (same tasks, same reflectors,
// DESIGN.md §7): position j owns, for every sweep i, the windows of task
// (i, j) in shared memory —
//   D_j = M[R_ij, R_ij] (lower, packed)   and   B_j = M[R_ij, R_i,j-1]
// (R_ij = [i+1+j nb, i+(j+1) nb]; B_j's column 0 is task (i, j)'s target
// column, columns 1.. its previous bulge; position 0 keeps only the target
// column M[R_i0, i], in B's last column).  Task (i, j) at position j:
//   (c) of task (i, j-1):  B_j <- B_j H_{i,j-1}   (v, tau from position j-1)
//   reflector of B_j's target column             (published to position j+1)
//   (a) B_j[:, 1:] <- H^H B_j[:, 1:],  (b) D_j <- H^H D_j H.
// From sweep i to i+1 both windows slide one row and one column down the
// band: the updates of (a) and (b) are written one row and column up-left,
// D_j's first column becomes B_j's last column, and the entering last row
// comes from position j+1 (its B row 0 and D(0,0) after sweep i; the rest of
// B's new row is zero: those entries left a target column below its beta).
// Position j runs sweep i at tick 2i + j; the CTA of positions 2k, 2k+1
// alternates between them, so only a reflector (65 values) and a row (65
// values) cross between CTAs per task, with release/acquire flags.
constexpr int LB = 65;                  // B column stride (complex)
constexpr int DPK = 64 * 65 / 2;        // packed lower D
__device__ __forceinline__ int dix(int r, int c) { return r * (r + 1) / 2 + c; }   // r >= c

struct SysArgs {
  int64_t n;
  int nb, ldab, J;
  double2 *AB;
  double2 *V2, *tau2;
  const int64_t *off;
  double2 *vmsg;   // [J][2][nb + 1]: v, tau of task (i, j)   (by sweep parity)
  double2 *rmsg;   // [J][2][nb + 1]: B_j row 0, D_j(0, 0) after task (i, j)
  int *vflag, *rflag;   // [J]: sweeps published
  unsigned long long *prof;   // optional: CTA 0 cycles [16..21] (row wait, v wait + (c), reflector, (a), (b), end)
};

__device__ __forceinline__ double2 ldcg2(const double2 *p) { return __ldcg(p); }
// named barriers (bar.sync 0 is __syncthreads): producer arrives, consumer syncs
__device__ __forceinline__ void nbar_sync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int cnt) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}

__global__ void __launch_bounds__(HT, 1) hb2sys_kernel(SysArgs a) {
  namespace cg = cooperative_groups;
  extern __shared__ __align__(16) double2 ysm[];
  __shared__ double2 sv[64], svin[64], sp[64], sg[64], sf[64], srow[65], srowx[65], svx[65], srx[65];
  __shared__ double2 spart[8][64], spart2[8][64];
  __shared__ double2 s_tau2[1], s_beta2[1], s_tauin;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n;
  const int nb = a.nb, ldab = a.ldab;
  double2 *AB = a.AB;
  auto Mget = [&](int64_t r, int64_t c) -> double2 {
    return (c >= 0 && c < n && r < n && r >= c && r - c < ldab) ? AB[(r - c) + c * (int64_t)ldab] : czero();
  };
  const int k = blockIdx.x;
  const bool prof = a.prof != nullptr && k == 1 && tid == 0;   // a CTA with two full positions
  long long tm = 0, tacc[6] = {0, 0, 0, 0, 0, 0};
  auto mark = [&](int kk) {
    if (prof) {
      const long long now = clock64();
      if (kk >= 0) tacc[kk] += now - tm;
      tm = now;
    }
  };
  auto Dq = [&](int q) { return ysm + q * DPK; };
  auto Bq = [&](int q) { return ysm + 2 * DPK + q * 64 * LB; };
  for (int q = 0; q < 2; q++) {   // windows of sweep 0
    const int j = 2 * k + q;
    if (j >= a.J) break;
    const int64_t r0 = 1 + (int64_t)j * nb;
    for (int e = tid; e < nb * nb; e += HT) {
      const int r = e % nb, c = e / nb;
      if (r >= c) Dq(q)[dix(r, c)] = Mget(r0 + r, r0 + c);
      double2 v = czero();
      if (j >= 1) v = Mget(r0 + r, r0 - nb + c);
      else if (c == nb - 1) v = Mget(r0 + r, 0);
      Bq(q)[c * LB + r] = v;
    }
  }
  cg::this_grid().sync();   // every window is loaded before the first output lands in AB

  // zlarfg (reading R1) of x = (x0 at lane, x1 at lane + 32), length len, by one warp
  auto reflector = [&](double2 x0, double2 x1, double alx, double aly, int len) {
    const double2 al = make_double2(alx, aly);
    double nrm = (lane >= 1 ? x0.x * x0.x + x0.y * x0.y : 0.0) + x1.x * x1.x + x1.y * x1.y;
    nrm = warp_sum(nrm);
    double2 tau, scale;
    double beta;
    if (nrm == 0.0 && al.y == 0.0) {
      tau = czero();
      beta = al.x;
      scale = czero();
    } else {
      beta = -copysign(sqrt(al.x * al.x + al.y * al.y + nrm), al.x);
      const double ib = 1.0 / beta;
      tau = make_double2((beta - al.x) * ib, -al.y * ib);
      const double2 d = make_double2(al.x - beta, al.y);
      const double idd = 1.0 / (d.x * d.x + d.y * d.y);
      scale = make_double2(d.x * idd, -d.y * idd);
    }
    sv[lane] = (lane == 0) ? make_double2(1.0, 0.0) : (lane < len ? cmul(x0, scale) : czero());
    sv[lane + 32] = (lane + 32 < len) ? cmul(x1, scale) : czero();
    if (lane == 0) {
      s_tau2[0] = tau;
      s_beta2[0] = make_double2(beta, 0.0);
    }
  };

  const int G7 = (nb + 6) / 7;   // terms per group, 7-group matvecs (workers)
  // Roles: warp 0 = leader (reflector; fetches the next task's cross-CTA
  // message), warps 1-14 = workers ((c), (a), (b); warp 1 also builds w and
  // the leaving row), warp 15 = messenger (every global store of the chase:
  // the messages with their releases, V2 / tau2, d / e).  The compute warps
  // synchronise with named barriers that leave the messenger out, so a
  // release (which waits for its stores) never stalls the compute warps.
  // Messages between the two positions of a CTA (v of 2k -> 2k+1, row of
  // 2k+1 -> 2k) stay in shared memory.
  // Barriers: 5 compute warps (480); 1, 8 workers (448); 3 leader -> workers;
  // 2 leader -> messenger (reflector ready), 7 messenger -> leader (read);
  // 4 warp 1 -> messenger (row ready), 6 messenger -> warp 1 (read).
  const int t = tid - 32;                     // worker index (warps 1-14: 0..447)
  const int wr = t & 63, wg = t >> 6;         // worker row, group
  auto active = [&](int64_t ii, int jj) { return jj < a.J && ii + 1 + (int64_t)jj * nb <= n - 1; };
  auto has_next = [&](int64_t ii, int qq) { return (qq == 0 && active(ii, 2 * k + 1)) || active(ii + 1, 2 * k); };
  if (warp == 15) {
    // ================= messenger
    for (int64_t i = 0; i + 1 < n; i++) {
      if (!active(i, 2 * k)) break;
      for (int q = 0; q < 2; q++) {
        const int j = 2 * k + q;
        if (!active(i, j)) break;
        const int par = (int)(i & 1);
        nbar_sync(2, 64);   // the leader's reflector
        const double2 v0 = sv[lane], v1 = sv[lane + 32], tau = s_tau2[0], beta = s_beta2[0];
        __syncwarp();
        if (has_next(i, q)) nbar_arrive(7, 64);
        if (q == 1) {   // v of an odd position -> CTA k+1
          double2 *vm = a.vmsg + ((int64_t)j * 2 + par) * (nb + 1);
          if (lane < nb) vm[lane] = v0;
          if (lane + 32 < nb) vm[lane + 32] = v1;
          if (lane == 0) vm[nb] = tau;
          __syncwarp();   // orders the lanes' stores before lane 0's (cumulative) release
          if (lane == 0) st_release_i32(a.vflag + j, (int)(i + 1));
        }
        const int64_t slot = a.off[j] + i;
        if (lane < nb) a.V2[slot * nb + lane] = v0;
        if (lane + 32 < nb) a.V2[slot * nb + lane + 32] = v1;
        if (lane == 0) {
          a.tau2[slot] = tau;
          if (j == 0) AB[1 + i * (int64_t)ldab] = beta;   // e_i (scaled units)
        }
        if (q == 0) {
          nbar_sync(4, 64);   // the leaving row of an even position
          const double2 r0v = srowx[lane], r1v = srowx[lane + 32], rn = srowx[nb];
          __syncwarp();
          if (active(i + 1, 2 * k)) nbar_arrive(6, 64);
          if (j >= 1) {   // -> CTA k-1
            double2 *rm = a.rmsg + ((int64_t)j * 2 + par) * (nb + 1);
            if (lane < nb) rm[lane] = r0v;
            if (lane + 32 < nb) rm[lane + 32] = r1v;
            if (lane == 0) rm[nb] = rn;
            __syncwarp();
            if (lane == 0) st_release_i32(a.rflag + j, (int)(i + 1));
          } else if (lane == 0) {
            AB[(i + 1) * (int64_t)ldab] = rn;   // d_{i+1} (final after sweep i)
          }
        }
      }
    }
  } else {
  // ================= compute warps
  // leader: fetch the cross-CTA message task (ii, 2k+qq) needs into shared memory
  auto prefetch = [&](int64_t ii, int qq) {
    if (qq == 0) {
      if (k == 0) return;
      const int jp = 2 * k - 1;
      if (lane == 0)
        while (ld_acquire_i32(a.vflag + jp) < ii + 1) {
        }
      __syncwarp();
      const double2 *m = a.vmsg + ((int64_t)jp * 2 + (ii & 1)) * (nb + 1);
      for (int u = lane; u <= nb; u += 32) svx[u] = ldcg2(m + u);
    } else {
      const int jn = 2 * k + 2;
      if (!(ii > 0 && active(ii - 1, jn))) return;
      if (lane == 0)
        while (ld_acquire_i32(a.rflag + jn) < ii) {
        }
      __syncwarp();
      const double2 *m = a.rmsg + ((int64_t)jn * 2 + ((ii - 1) & 1)) * (nb + 1);
      for (int u = lane; u <= nb; u += 32) srx[u] = ldcg2(m + u);
    }
  };
  if (warp == 0 && active(0, 2 * k)) prefetch(0, 0);
  bool first = true, first0 = true;
  for (int64_t i = 0; i + 1 < n; i++) {
    if (!active(i, 2 * k)) break;   // both positions are past the matrix
    for (int q = 0; q < 2; q++) {
      const int j = 2 * k + q;
      if (!active(i, j)) break;
      const int64_t r0 = i + 1 + (int64_t)j * nb;
      const int len = (int)imin64(nb, n - r0);
      double2 *D = Dq(q), *B = Bq(q);
      mark(-1);
      const bool act1 = i > 0 && active(i - 1, j + 1);   // position j+1 ran sweep i-1
      nbar_sync(5, HT - 32);   // prefetched messages are in shared memory; the previous task is done
      mark(0);
      // entering row of the windows (sweep i-1 -> i) and the incoming reflector
      if (i > 0 && t >= 0 && t < nb) {   // (workers: the leader goes straight to its barrier)
        const double2 *m = q == 0 ? srow : srx;
        D[dix(nb - 1, t)] = act1 ? m[t < nb - 1 ? t + 1 : nb] : czero();
        B[t * LB + nb - 1] = (t < nb - 1 || !act1) ? czero() : m[0];
      }
      if (j >= 1 && t >= 64 && t <= 64 + nb) {
        const int u = t - 64;
        const double2 x = q == 0 ? svx[u] : (u < nb ? sv[u] : s_tau2[0]);
        if (u < nb) svin[u] = x;
        else s_tauin = x;
      }
      mark(5);
      nbar_sync(5, HT - 32);
      mark(4);
      // ---- (c) of task (i, j-1): partials of g = tau_in B v_in (workers)
      const double2 tin = j >= 1 ? s_tauin : czero();
      const bool updc = tin.x != 0.0 || tin.y != 0.0;
      if (updc) {
        if (warp > 0 && wr < nb) {
          double2 acc = czero();
          for (int c = wg * G7; c < imin64(nb, (wg + 1) * G7); c++) acc = cadd(acc, cmul(B[c * LB + wr], svin[c]));
          spart[wg][wr] = acc;
        }
        nbar_sync(5, HT - 32);
      }
      mark(1);
      const int tc = j == 0 ? nb - 1 : 0;
      if (warp == 0) {
        // ================= leader: reflector of task (i, j) from the target
        // column after (c) (x = B[:, 0] - g conj(v_in[0]))
        double2 x0 = czero(), x1 = czero();
        if (lane < len) x0 = B[tc * LB + lane];
        if (lane + 32 < len) x1 = B[tc * LB + lane + 32];
        if (updc) {
          const double2 cv0 = cconj(svin[0]);
          double2 g0 = czero(), g1 = czero();
          for (int g = 0; g < 7; g++) {
            g0 = cadd(g0, spart[g][lane]);
            g1 = cadd(g1, spart[g][lane + 32]);
          }
          if (lane < len) x0 = csub(x0, cmul(cmul(tin, g0), cv0));
          if (lane + 32 < len) x1 = csub(x1, cmul(cmul(tin, g1), cv0));
        }
        if (!first) nbar_sync(7, 64);   // the messenger has read the previous reflector
        first = false;
        reflector(x0, x1, __shfl_sync(0xffffffffu, x0.x, 0), __shfl_sync(0xffffffffu, x0.y, 0), len);
        __syncwarp();
        nbar_arrive(3, HT - 32);   // workers: the reflector is in shared memory
        nbar_arrive(2, 64);        // messenger
        mark(2);
        // the next task's cross-CTA message
        if (q == 0 && active(i, j + 1)) prefetch(i, 1);
        else if (active(i + 1, 2 * k)) prefetch(i + 1, 0);
        mark(3);
      } else {
        // ================= workers
        // rest of (c): B[:, 1:] -= g v_in^H   (g combined by worker warps 1-2)
        if (updc) {
          if (t < nb) {
            double2 s = spart[0][t];
            for (int g = 1; g < 7; g++) s = cadd(s, spart[g][t]);
            sg[t] = cmul(tin, s);
          }
          nbar_sync(1, HT - 64);
          if (wr < nb) {
            const double2 gr = sg[wr];
            for (int c = 1 + wg; c < nb; c += 7) B[c * LB + wr] = csub(B[c * LB + wr], cmul(gr, cconj(svin[c])));
          }
        }
        nbar_sync(3, HT - 32);   // the leader's reflector
        const double2 tau = s_tau2[0], ctau = cconj(tau);
        const bool upd = tau.x != 0.0 || tau.y != 0.0;
        // (a) f_c = conj(tau) v^H B[:, c] (c >= 1) and (b) p = tau D v: partials
        if (upd) {
          const int x = wr;
          double2 accf = czero(), accp = czero();
          if (x < nb) {
            for (int r = wg * G7; r < imin64(nb, (wg + 1) * G7); r++) {
              if (j >= 1 && x >= 1) accf = cadd(accf, cmulc(sv[r], B[x * LB + r]));
              double2 d = D[r <= x ? dix(x, r) : dix(r, x)];   // Hermitian from the lower triangle (c = r)
              d.y = r < x ? d.y : (r > x ? -d.y : 0.0);
              accp = cadd(accp, cmul(d, sv[r]));
            }
          }
          spart[wg][x] = accf;
          spart2[wg][x] = accp;
          nbar_sync(1, HT - 64);
        }
        // worker warp 1: f, w = p - 1/2 tau (p^H v) v, and the leaving row
        if (warp == 1) {
          double2 p0 = czero(), p1 = czero();
          if (upd) {
            double2 f0 = czero(), f1 = czero();
            for (int g = 0; g < 7; g++) {
              f0 = cadd(f0, spart[g][lane]);
              f1 = cadd(f1, spart[g][lane + 32]);
              p0 = cadd(p0, spart2[g][lane]);
              p1 = cadd(p1, spart2[g][lane + 32]);
            }
            sf[lane] = cmul(ctau, f0);
            sf[lane + 32] = cmul(ctau, f1);
            p0 = lane < nb ? cmul(tau, p0) : czero();
            p1 = lane + 32 < nb ? cmul(tau, p1) : czero();
            const double2 v0 = sv[lane], v1 = sv[lane + 32];
            const double2 sdot = warp_sum2(cadd(cmulc(p0, v0), cmulc(p1, v1)));
            const double2 al = cmul(make_double2(-0.5 * tau.x, -0.5 * tau.y), sdot);
            p0 = cadd(p0, cmul(al, v0));
            p1 = cadd(p1, cmul(al, v1));
            sp[lane] = p0;
            sp[lane + 32] = p1;
          }
          __syncwarp();
          // leaving row: B row 0 after (a) (j >= 1), D(0, 0) after (b); an even
          // position's row goes to the messenger, an odd one's stays here
          double2 *so = srow;
          if (q == 0) {
            if (!first0) nbar_sync(6, 64);   // the messenger has read the previous one
            first0 = false;
            so = srowx;
          }
          const double2 vv0 = sv[0];
          for (int c = lane; c < nb; c += 32) {
            double2 b = c == 0 ? s_beta2[0] : B[c * LB];
            if (c >= 1 && upd) b = csub(b, cmul(vv0, sf[c]));
            so[c] = b;
          }
          if (lane == 0) {
            double2 d00 = D[0];
            if (upd) {
              const double2 w0 = sp[0];
              d00 = csub(d00, cadd(cmul(vv0, cconj(w0)), cmul(w0, cconj(vv0))));
            }
            d00.y = 0.0;
            so[nb] = d00;
          }
          __syncwarp();
          if (q == 0) nbar_arrive(4, 64);
        }
        nbar_sync(1, HT - 64);   // w is staged
        // (a) and (b) updates, written one row / column up-left; D's column 0 -> B's last column
        {
          const int r = wr;
          const bool rok = r >= 1 && r < nb;
          const double2 vr = sv[r], pr = upd ? sp[r] : czero();
          double2 vb[9], vd[10];
#pragma unroll
          for (int u = 0; u < 9; u++) {
            const int cb = 1 + wg + 7 * u;
            vb[u] = czero();
            if (j >= 1 && rok && cb < nb) {
              const double2 b = B[cb * LB + r];
              vb[u] = upd ? csub(b, cmul(vr, sf[cb])) : b;
            }
          }
#pragma unroll
          for (int u = 0; u < 10; u++) {
            const int cd = wg + 7 * u;
            vd[u] = czero();
            if (rok && cd <= r) {
              double2 d = D[dix(r, cd)];
              if (upd) d = csub(d, cadd(cmul(vr, cconj(sp[cd])), cmul(pr, cconj(sv[cd]))));
              if (r == cd) d.y = 0.0;
              vd[u] = d;
            }
          }
          nbar_sync(8, HT - 64);
#pragma unroll
          for (int u = 0; u < 9; u++) {
            const int cb = 1 + wg + 7 * u;
            if (j >= 1 && rok && cb < nb) B[(cb - 1) * LB + r - 1] = vb[u];
          }
#pragma unroll
          for (int u = 0; u < 10; u++) {
            const int cd = wg + 7 * u;
            if (rok && cd <= r) {
              if (cd >= 1) D[dix(r - 1, cd - 1)] = vd[u];
              else B[(nb - 1) * LB + r - 1] = vd[u];
            }
          }
        }
      }
      mark(5);
    }
  }
  }   // compute warps
  if (prof)
    for (int kk = 0; kk < 6; kk++) atomicAdd(&a.prof[16 + kk], (unsigned long long)tacc[kk]);
}

// Band copy plus the magnitude key of its largest entry (atomicMax into *key).
__global__ void band_in_kernel(int64_t n, int nb, const double2 *A, int64_t lda, double2 *AB, int ldab,
                               unsigned *key) {
  const int64_t total = n * (int64_t)ldab;
  unsigned k = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int d = (int)(e % ldab);
    const int64_t c = e / ldab;
    double2 v = czero();
    if (d <= nb && c + d < n) {
      v = A[(c + d) + c * lda];
      if (d == 0) v.y = 0.0;
    }
    AB[e] = v;
    k = max(k, mag_key2(v));
  }
  k = __reduce_max_sync(0xffffffffu, k);
  if ((threadIdx.x & 31) == 0 && k) atomicMax(key, k);
}

// Scaling (reading R1, LAPACK zlarfg's scaled norms): the chase runs on the
// band times 2^-U, U = the binary exponent of its largest entry.  The chase is
// homogeneous (V2, tau2 unchanged, d, e times 2^-U) and the factor is an exact
// power of two, so away from the range ends the result is bitwise the
// unscaled one, and at the ends no sum of squares over- or underflows.
__global__ void band_scale_kernel(int64_t total, double2 *AB, const unsigned *key) {
  const int U = exp_of_key(*key);
  if (U == kExpZero || U == 0) return;
  const double f = pow2i(-U);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
    AB[e] = cscale(f, AB[e]);
}

__global__ void tridiag_out_kernel(int64_t n, const double2 *AB, int ldab, double *d, double *e, const unsigned *key) {
  const int U = exp_of_key(*key);
  const double f = (U == kExpZero) ? 1.0 : pow2i(U);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    d[i] = AB[i * (int64_t)ldab].x * f;
    if (i + 1 < n) e[i] = AB[1 + i * (int64_t)ldab].x * f;
  }
}

}  // namespace

int hb2st(Ctx &ctx, int64_t n, int nb, const double2 *A, int64_t lda, double *d, double *e, double2 *V2,
          double2 *tau2, const int64_t *d_off) {
  if (n <= 0) return 0;
  if (nb > 64) return EIG_ERR_NOTIMPL;
  const int ldab = 2 * nb + 2;
  double2 *AB = (double2 *)ctx.ws(WS_BAND, (size_t)ldab * n * sizeof(double2));
  int *prog = (int *)ctx.ws(WS_HBPROG, (size_t)(2 * n + 1) * sizeof(int));   // progress | progressA | key
  if (!AB || !prog) return EIG_ERR_NOMEM;
  unsigned *key = (unsigned *)(prog + 2 * n);
  EIG_TRY(ctx.check(cudaMemsetAsync(prog, 0, (size_t)(2 * n + 1) * sizeof(int), ctx.stream), "memset progress"));
  const int64_t total = n * (int64_t)ldab;
  const int bgrid = (int)std::min<int64_t>((total + 255) / 256, 8LL * ctx.num_sms);
  band_in_kernel<<<bgrid, 256, 0, ctx.stream>>>(n, nb, A, lda, AB, ldab, key);
  EIG_TRY(ctx.launched("band_in_kernel"));
  band_scale_kernel<<<bgrid, 256, 0, ctx.stream>>>(total, AB, key);
  EIG_TRY(ctx.launched("band_scale_kernel"));
  const int64_t Jpos = n > 1 ? (n - 2) / nb + 1 : 0;   // positions of sweep 0
  // position-stationary kernel (default) when its ceil(J / 2) CTAs are co-resident;
  // EIG_HB2ST_SYS=0 selects the sweep-per-CTA kernel
  static const int sys_env = [] {
    const char *e = getenv("EIG_HB2ST_SYS");
    return e ? atoi(e) : 1;
  }();
  const size_t sys_smem = (size_t)2 * (DPK + 64 * LB) * sizeof(double2);
  if (n > 1 && sys_env && (Jpos + 1) / 2 <= ctx.num_sms) {
    const size_t msg = (size_t)Jpos * 2 * (nb + 1);
    double2 *mbuf = (double2 *)ctx.ws(WS_HBMSG, 2 * msg * sizeof(double2));
    int *flags = (int *)ctx.ws(WS_HBFLAG, (size_t)2 * Jpos * sizeof(int));
    if (!mbuf || !flags) return EIG_ERR_NOMEM;
    EIG_TRY(ctx.check(cudaMemsetAsync(flags, 0, (size_t)2 * Jpos * sizeof(int), ctx.stream), "memset hb flags"));
    SysArgs s;
    s.n = n;
    s.nb = nb;
    s.ldab = ldab;
    s.J = (int)Jpos;
    s.AB = AB;
    s.V2 = V2;
    s.tau2 = tau2;
    s.off = d_off;
    s.vmsg = mbuf;
    s.rmsg = mbuf + msg;
    s.vflag = flags;
    s.rflag = flags + Jpos;
    s.prof = ctx.q2_prof;
    void *args[] = {&s};
    EIG_TRY(ctx.smem_attr((const void *)hb2sys_kernel, (int)sys_smem, "hb2sys attr"));
    EIG_TRY(ctx.check(cudaLaunchCooperativeKernel((void *)hb2sys_kernel, dim3((unsigned)((Jpos + 1) / 2)), dim3(HT),
                                                  args, sys_smem, ctx.stream), "hb2sys launch"));
    EIG_TRY(ctx.launched("hb2sys_kernel"));
  } else if (n > 1) {
    HbArgs a;
    a.n = n;
    a.nb = nb;
    a.ldab = ldab;
    a.AB = AB;
    a.V2 = V2;
    a.tau2 = tau2;
    a.off = d_off;
    a.progress = prog;
    a.progressA = prog + n;
    a.prof = ctx.q2_prof;
    const int64_t J = (n - 2) / nb + 1;   // steps of sweep 0
    // ~J / 2.3 sweeps are active at once (lag of two steps plus a reflector)
    const int P = (int)std::max<int64_t>(1, std::min<int64_t>(ctx.num_sms, std::min<int64_t>(n - 1, J / 2 + 2)));
    void *args[] = {&a};
    const size_t smem = ((size_t)64 * LDD + 2 * 64 * 64 + 64) * sizeof(double2);
    EIG_TRY(ctx.smem_attr((const void *)hb2st_kernel, (int)smem, "hb2st attr"));
    EIG_TRY(ctx.check(cudaLaunchCooperativeKernel((void *)hb2st_kernel, dim3(P), dim3(HT), args, smem, ctx.stream),
                      "hb2st launch"));
    EIG_TRY(ctx.launched("hb2st_kernel"));
  }
  tridiag_out_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, ctx.stream>>>(n, AB, ldab, d, e, key);
  return ctx.launched("tridiag_out_kernel");
}

}  // namespace eig
