// q2w.cu — E <- Q2 E (a6) with column-owning warps, for nb = 64, g = 32.
//
// Same block structure as q2.cu (R7: block (i0, j) of g sweeps is
// I - V T V^H, V the W x g parallelogram, W = nb + g - 1 = 95; groups applied
// last to first, steps ascending), different work split:
//
//  * a CTA owns up to 9 eight-column fragments of E per slab; 8 "full" warps
//    own one fragment each and its 96-row window (a ring of three 32-row
//    chunks in shared memory) and run all three contractions for it alone —
//    Y = V^H E (phase A), Y = T Y (phase B), E -= V Y (phase C) — with Y in
//    registers, moved between the accumulator and operand layouts by warp
//    shuffles, so they never wait for each other;
//  * the 9th fragment is shared by a quad of warps (one per SM sub-partition,
//    each doing a quarter of every phase, Y exchanged through shared memory
//    under a 128-thread named barrier), so all four DMMA pipes get the same
//    work (2.25 fragments each instead of 3 on one of them);
//  * V (compact: Vc[t][4 + s] = v_t[s], zero pads on both sides) and T are
//    double-buffered and loaded with bulk async copies that complete on an
//    mbarrier; the last warp to release a buffer issues the copies of the
//    block two ahead into it (no producer warp, no block-wide barrier);
//  * every loop over k-steps and row groups is fully unrolled against the
//    compile-time parallelogram shape: all shared-memory addresses are a lane
//    base plus an immediate, and only the nonzero DMMA tiles are issued;
//  * rows that leave the window are stored straight from the accumulators and
//    their ring slots are refilled with the next block's rows (cp.async)
//    while the remaining row groups are computed.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int NB = 64, G = 32, W = NB + G - 1;   // 95 window rows
constexpr int RING = 96;                         // 3 chunks of 32 rows
constexpr int LDE = 97;                          // E window column stride (complex, odd)
// Shared-memory banks: a 16-byte complex element e sits in bank group e mod 8
// (plus the component).  The compact V rows are placed at
//   rb(t) = 72 t + DV[t mod 4],  DV = {0, 5, 4, 1}
// so that rb(t) - t mod 8 runs through {0,4,2,6} (+4 on odd quads): phase A
// (4 consecutive reflectors x 2 rows) and phase C (2 reflectors x 4 rows)
// both hit 8 distinct bank groups per fragment load.  Neighbouring rows
// overlap only in their zero pads (4 on each side).
constexpr int LDVC = 72, PADL = 4, VC_STAGE = 72 * G + 8;
__host__ __device__ constexpr int dv(int i) { return i == 0 ? 0 : i == 1 ? 5 : i == 2 ? 4 : 1; }
__host__ __device__ constexpr int vrow(int t) { return LDVC * t + dv(t & 3); }
// T columns: cb(k) = 68 (k >> 1) + 36 (k & 1): consecutive columns 4 apart mod 8
constexpr int T_STAGE = 68 * (G / 2);
__host__ __device__ constexpr int tcol(int k) { return 68 * (k >> 1) + 36 * (k & 1); }
constexpr int LDY = 34;                          // quad Y exchange: Y[col][refl]
constexpr int NFW = 8, NQW = 4, NW = NFW + NQW;  // full warps, quad warps
constexpr int NFS = NFW + 1;                     // fragments per slab
constexpr int WT = NW * 32;
#ifndef Q2W_QUAD
#define Q2W_QUAD 1   // 0: the 9th fragment goes to warp 8 as a full warp (measured 20% slower)
#endif

struct Q2wArgs {
  int64_t n, m, lde;
  int64_t ngroups;
  const int64_t *first;  // [ngroups+1]
  const int64_t *off;    // [J]
  const double2 *V2;
  const double2 *T2;
  double2 *E;
  int nfr_total, nslab;
  unsigned long long *prof;   // optional: CTA 0 warps 0 / 8 cycles [24..29] (wait, work, release)
};

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// L2 policies: the E stream (read and written once per group) is evict-first,
// the V / T blocks (read by every CTA) evict-last.
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol_evict_last())
      : "memory");
}
__device__ __forceinline__ void st_stream(double *p, double v) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol_evict_first())
               : "memory");
}
// non-volatile DMMA: lets the scheduler interleave the unrolled tiles freely
__device__ __forceinline__ void dmma_nv(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp_async16m(void *smem, const void *gmem, bool valid) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(su32(smem)), "l"(gmem),
               "r"(valid ? 16 : 0), "l"(pol_evict_first())
               : "memory");
}
__device__ __forceinline__ void quad_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__host__ __device__ constexpr int imin_c(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int imax_c(int a, int b) { return a > b ? a : b; }

// Accumulator layout (M-fragment mf: complex rows 4mf..4mf+3, lane holds real row
// lane>>2 at columns 2(lane&3), +1) -> operand layout of k-step ks (complex rows
// 2ks, 2ks+1; lane holds real row lane&3 at column lane>>2).
template <int NM>
__device__ __forceinline__ void acc_to_b(const double (&acc)[NM][2], double (&bl)[2 * NM], int lane) {
  const int src_lo = 4 * (lane & 3) + (lane >> 3);
  const bool hi = (lane >> 2) & 1;
#pragma unroll
  for (int ks = 0; ks < 2 * NM; ks++) {
    const int src = src_lo + 16 * (ks & 1);
    const double v0 = __shfl_sync(0xffffffffu, acc[ks >> 1][0], src);
    const double v1 = __shfl_sync(0xffffffffu, acc[ks >> 1][1], src);
    bl[ks] = hi ? v1 : v0;
  }
}

// shared memory: Vc[2] | T[2] | E windows (NFS) | Y, Y2 (quad) | full[2] mbarriers, done[2] counters
extern __shared__ __align__(128) double2 q2w_sm[];
constexpr int OFF_T = 2 * VC_STAGE, OFF_E = OFF_T + 2 * T_STAGE, OFF_Y = OFF_E + NFS * 8 * LDE,
              OFF_Y2 = OFF_Y + 8 * LDY, OFF_BAR = OFF_Y2 + 8 * LDY;
__device__ __forceinline__ double2 *vc_buf(int bi) { return q2w_sm + bi * VC_STAGE; }
__device__ __forceinline__ double2 *t_buf(int bi) { return q2w_sm + OFF_T + bi * T_STAGE; }
__device__ __forceinline__ uint64_t *full_bar(int bi) { return reinterpret_cast<uint64_t *>(q2w_sm + OFF_BAR) + bi; }
__device__ __forceinline__ int *done_cnt(int bi) { return reinterpret_cast<int *>(q2w_sm + OFF_BAR + 1) + bi; }

// ---------------------------------------------------------------- block sequence
// (slab, group gi from last to first, step j ascending), identical in every warp.
struct BlkIt {
  int sl;
  int64_t gi, j, J;
  bool valid;
};
__device__ __forceinline__ int64_t steps_of(const Q2wArgs &a, int64_t gi) {
  const int64_t i0 = gi * G;
  return (i0 > a.n - 2) ? 0 : (a.n - 2 - i0) / NB + 1;
}
__device__ __forceinline__ void it_settle(const Q2wArgs &a, BlkIt &it) {
  while (it.valid && it.j >= it.J) {
    if (--it.gi < 0) {
      if (++it.sl >= a.nslab) {
        it.valid = false;
        return;
      }
      it.gi = a.ngroups - 1;
    }
    it.J = steps_of(a, it.gi);
    it.j = 0;
  }
}
__device__ __forceinline__ void it_begin(const Q2wArgs &a, BlkIt &it) {
  it.sl = 0;
  it.gi = a.ngroups - 1;
  it.j = 0;
  it.valid = a.ngroups > 0 && a.nslab > 0;
  it.J = it.valid ? steps_of(a, it.gi) : 0;
  it_settle(a, it);
}
__device__ __forceinline__ void it_next(const Q2wArgs &a, BlkIt &it) {
  if (!it.valid) return;
  it.j++;
  it_settle(a, it);
}

// Warp-wide: bulk copies of block `it`'s V (live slots) and T into buffer bi.
// The global offsets of a block (off[j], first[gi]) are read when the
// iterator reaches it, two blocks before its copies are issued.
struct BlkSrc {
  int64_t offj, firstg;   // raw off[j], first[gi] (used only when the copies are issued)
  int64_t gi, j;
};
__device__ __forceinline__ BlkSrc blk_src(const Q2wArgs &a, const BlkIt &it) {
  BlkSrc b;
  b.gi = it.gi;
  b.j = it.j;
  b.offj = it.valid ? a.off[it.j] : 0;
  b.firstg = it.valid ? a.first[it.gi] : 0;
  return b;
}
__device__ __forceinline__ void issue_block(const Q2wArgs &a, const BlkSrc &b, int bi, int lane) {
  const int64_t i0 = b.gi * G;
  const int nvalid = (int)imax64(0, imin64(G, a.n - 2 - b.j * NB - i0 + 1));
  if (lane == 0) mbar_arrive_tx(full_bar(bi), (unsigned)(nvalid * NB * 16 + G * G * 16));
  __syncwarp();
  if (lane < nvalid) bulk_g2s(vc_buf(bi) + vrow(lane) + PADL, a.V2 + (b.offj + i0 + lane) * NB, NB * 16, full_bar(bi));
  bulk_g2s(t_buf(bi) + tcol(lane), a.T2 + (b.firstg + b.j) * G * G + lane * G, G * 16, full_bar(bi));
}

// ---------------------------------------------------------------- per-lane constants
struct Lane {
  int lane, kq, rr;
  int offA, offC0, offC1, offT, offEB, offEC;   // shared-memory offsets (doubles)
  int ldw2;                                      // window column stride (doubles)
  unsigned negConj, negT, negA;
  __device__ __forceinline__ explicit Lane(int l, int ldw = LDE) {
    const LaneEmb le(l);
    lane = l;
    kq = (l & 3) >> 1;
    rr = l >> 2;
    // V element (q, t) at vrow(t) + PADL + q - t = 71 t + dv(t mod 4) + PADL + q
    offA = 2 * (71 * (l >> 3) + dv(l >> 3) + kq + PADL) + le.a_comp;   // V^H: t = 4mf + lane>>3, q = 2ks + kq
    offC0 = 2 * (71 * kq + dv(kq) + (l >> 3) + PADL) + le.a_comp;      // V: q = 4f + lane>>3, t = 2ks + kq, ks even
    offC1 = 2 * (71 * kq + dv(2 + kq) + (l >> 3) + PADL) + le.a_comp;  //                                 ks odd
    offT = 2 * (36 * kq + (l >> 3)) + le.a_comp;                       // T[ra][kb] at tcol(kb) + ra
    offEB = 2 * (ldw * (l >> 2) + kq) + (l & 1);           // E, operand layout
    offEC = 2 * (ldw * 2 * (l & 3) + (rr >> 1)) + (rr & 1);  // E, accumulator layout (col 2(lane&3))
    ldw2 = 2 * ldw;
    negConj = le.a_neg_conj;
    negT = le.a_neg;
    negA = le.a_neg ^ 0x80000000u;                          // -V in phase C
  }
};

// One fragment's view of a block.
struct Frag {
  double *ew;                 // window (doubles)
  double2 *Ew;
  int ch0, ch1, ch2;          // chunk -> slot base (doubles)
  int base;
  int64_t rs;                 // first window row
  bool more;                  // a next block exists in this group
  double *gE;                 // lane's global pointer (accumulator layout, row rs)
  int64_t lde2;
  bool ok0, ok1;              // lane's two columns exist
  const double2 *E;
  int64_t lde, c0, n;
  int ncols;
};

__device__ __forceinline__ int ring_slot(int s) { return s < 0 ? s + RING : (s >= RING ? s - RING : s); }

// Phase C for row groups FL::f(0..NU-1): acc = E rows + (-V) Y2, then store.
// Rows < 64 (or all rows of a group's last block) leave the window: global.
// REFILL: after storing a leaving row group, load the next block's rows into
// its four slots (the quad does this per row group).
template <int NU, class FL, bool REFILL>
__device__ __forceinline__ void phase_c_rows(const Frag &F, const Lane &L, const double *vc, const double (&yb)[16]) {
  double acc[NU][2];
#pragma unroll
  for (int u = 0; u < NU; u++) {
    const int f = FL::f(u);
    const int ch = f < 8 ? F.ch0 : (f < 16 ? F.ch1 : F.ch2);
    const double *p = F.ew + ch + L.offEC + 8 * (f & 7);
    acc[u][0] = p[0];
    acc[u][1] = p[L.ldw2];
  }
#pragma unroll
  for (int ks = 0; ks < 16; ks++) {
#pragma unroll
    for (int u = 0; u < NU; u++) {
      const int f = FL::f(u);
      const int klo = imax_c(0, 4 * f - 63) >> 1, khi = imin_c(31, 4 * f + 3) >> 1;
      if (ks >= klo && ks <= khi) dmma_nv(acc[u], xsign(vc[((ks & 1) ? L.offC1 : L.offC0) + 284 * ks + 8 * f], L.negA), yb[ks]);
    }
  }
#pragma unroll
  for (int u = 0; u < NU; u++) {
    const int f = FL::f(u);
    const int q = 4 * f + (L.rr >> 1);
    if (f < 16 || !F.more) {
      if (q < W && F.rs + q < F.n) {
        double *g = F.gE + 8 * f;
        if (F.ok0) g[0] = acc[u][0];
        if (F.ok1) g[F.lde2] = acc[u][1];
      }
      if (REFILL && f < 16 && F.more) {
        // slot of current row 4f + r receives the next block's row 4f + r + 32
        const int r = L.lane & 3, c = L.lane >> 2;
        const int slot = ring_slot(4 * f + r + F.base);
        const int64_t row = F.rs + RING + 4 * f + r;
        const bool ok = row < F.n && c < F.ncols;
        __syncwarp();
        cp_async16m(&F.Ew[c * LDE + slot], ok ? F.E + row + (F.c0 + c) * F.lde : F.E, ok);
      }
    } else if (q < W) {
      double *p = F.ew + F.ch2 + L.offEC + 8 * (f & 7);
      p[0] = acc[u][0];
      p[L.ldw2] = acc[u][1];
    }
  }
}

template <int FB>
struct FullRows {
  __device__ static constexpr int f(int u) { return FB + u; }
};
struct PairsA {   // (f, f + 17): k-step ranges [0, 2f+1] and [2f+2, 15]
  __device__ static constexpr int f(int u) { return (u & 1) ? 17 + (u >> 1) : (u >> 1); }
};
struct PairsB {
  __device__ static constexpr int f(int u) { return u == 6 ? 7 : u == 7 ? 16 : ((u & 1) ? 21 + (u >> 1) : 4 + (u >> 1)); }
};
template <int I>
struct QuadLow {   // row groups < 16 of quad warp I (balanced: 2I+2 + 16-2I + 16 + 16 k-steps)
  __device__ static constexpr int f(int u) { return u == 0 ? I : u == 1 ? 7 - I : u == 2 ? 8 + I : 15 - I; }
};
template <int I>
struct QuadHigh {
  __device__ static constexpr int f(int u) { return u == 0 ? 16 + I : 23 - I; }
};

// Full warp: the whole block for its own fragment.
__device__ __forceinline__ void pmark(unsigned long long *pp, long long &tl, int k) {
  if (pp) {
    const long long t = clock64();
    pp[k] += t - tl;
    tl = t;
  }
}
// WAVE: the window's three 32-row chunks arrive as three cp.async groups
// followed by one more (the next item's chunk 0); phase A waits for each chunk
// just before its first k-step, and nothing is refilled here.
template <bool WAVE = false, int WPEND = 3>
__device__ __forceinline__ void full_block(const Frag &F, const Lane &L, const double *vc, const double *tt,
                                           unsigned long long *pp, long long &tl) {
  // ---------------- phase A: Y = V^H E   (M-fragment mf nonzero on k-steps 2mf .. 2mf+33)
  double y[8][2];
#pragma unroll
  for (int mf = 0; mf < 8; mf++) y[mf][0] = y[mf][1] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 48; ks++) {
    if (!WAVE && ks == 15) {   // rows 31..63 (cp.async group Y of the previous block)
      cp_async_wait<0>();
      __syncwarp();
    }
    // WAVE: groups pending at entry = [chunk 0, chunk 1, chunk 2] plus WPEND - 2
    // younger ones (the next item's chunk 0 with a spare slot)
    if (WAVE && ks == 0) {
      cp_async_wait<WPEND>();
      __syncwarp();
    }
    if (WAVE && ks == 16) {
      cp_async_wait<WPEND - 1>();
      __syncwarp();
    }
    if (WAVE && ks == 32) {
      cp_async_wait<WPEND - 2>();
      __syncwarp();
    }
    const int ch = ks < 16 ? F.ch0 : (ks < 32 ? F.ch1 : F.ch2);
    const double e = F.ew[ch + L.offEB + 4 * (ks & 15)];
#pragma unroll
    for (int mf = 0; mf < 8; mf++)
      if (ks >= 2 * mf && ks <= 2 * mf + 33) dmma_nv(y[mf], xsign(vc[L.offA + 568 * mf + 4 * ks], L.negConj), e);
  }
  double yb[16];
  acc_to_b<8>(y, yb, L.lane);
  pmark(pp, tl, 1);
  // ---------------- phase B: Y = T Y   (T upper triangular: k-steps 2mf .. 15)
#pragma unroll
  for (int mf = 0; mf < 8; mf++) {
    y[mf][0] = y[mf][1] = 0.0;
#pragma unroll
    for (int ks = 2 * mf; ks < 16; ks++) dmma_nv(y[mf], xsign(tt[L.offT + 136 * ks + 8 * mf], L.negT), yb[ks]);
  }
  acc_to_b<8>(y, yb, L.lane);
  pmark(pp, tl, 2);
  // ---------------- phase C, rows 32..63 first, then the rows 0..31 paired with
  // rows 64..95 so that every batch keeps four independent accumulators busy
  phase_c_rows<4, FullRows<8>, false>(F, L, vc, yb);
  phase_c_rows<4, FullRows<12>, false>(F, L, vc, yb);
  if (F.more) {
    // slots of current rows 32..62 <- next block's rows 64..94 (global rs + 96 + r)
    __syncwarp();
    const int r = 32 + L.lane;
    if (r < 63) {
      const int slot = ring_slot(F.base + r);
      const int64_t row = F.rs + RING + r;
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const bool ok = row < F.n && c < F.ncols;
        cp_async16m(&F.Ew[c * LDE + slot], ok ? F.E + row + (F.c0 + c) * F.lde : F.E, ok);
      }
    }
  }
  if (!WAVE) cp_async_commit();   // group X (possibly empty)
  phase_c_rows<8, PairsA, false>(F, L, vc, yb);
  phase_c_rows<8, PairsB, false>(F, L, vc, yb);
  if (F.more) {
    // slots of current rows 0..31 <- next rows 32..63; the padding slot (row 95) <- next row 31
    __syncwarp();
    const int r = L.lane;
    const int slot = ring_slot(F.base + r);
    const int64_t row = F.rs + RING + r;
#pragma unroll
    for (int c = 0; c < 8; c++) {
      const bool ok = row < F.n && c < F.ncols;
      cp_async16m(&F.Ew[c * LDE + slot], ok ? F.E + row + (F.c0 + c) * F.lde : F.E, ok);
    }
    if (L.lane < 8) {
      const int64_t prow = F.rs + W;
      const int c = L.lane;
      const bool ok = prow < F.n && c < F.ncols;
      cp_async16m(&F.Ew[c * LDE + ring_slot(F.base - 1)], ok ? F.E + prow + (F.c0 + c) * F.lde : F.E, ok);
    }
  }
  if (!WAVE) cp_async_commit();   // group Y (possibly empty): needed from phase A k-step 15 of the next block
  pmark(pp, tl, 3);
}

// Quad warp I: a quarter of every phase of the shared fragment.
template <int I>
__device__ __forceinline__ void quad_block(const Frag &F, const Lane &L, const double *vc, const double *tt) {
  double *yq = reinterpret_cast<double *>(q2w_sm + OFF_Y);
  double *y2q = reinterpret_cast<double *>(q2w_sm + OFF_Y2);
  const int lane = L.lane;
  // ---------------- phase A: M-fragments 2I, 2I+1
  double y[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int ks = 4 * I; ks < imin_c(48, 4 * I + 36); ks++) {
    const int ch = ks < 16 ? F.ch0 : (ks < 32 ? F.ch1 : F.ch2);
    const double e = F.ew[ch + L.offEB + 4 * (ks & 15)];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int mf = 2 * I + u;
      if (ks >= 2 * mf && ks <= 2 * mf + 33) dmma_nv(y[u], xsign(vc[L.offA + 568 * mf + 4 * ks], L.negConj), e);
    }
  }
  // Y[col][refl] (accumulator layout: refl 4mf + rr>>1, comp rr&1, cols 2(lane&3), +1)
#pragma unroll
  for (int u = 0; u < 2; u++) {
    const int refl = 4 * (2 * I + u) + (L.rr >> 1);
#pragma unroll
    for (int c = 0; c < 2; c++) yq[2 * ((2 * (lane & 3) + c) * LDY + refl) + (L.rr & 1)] = y[u][c];
  }
  quad_sync();
  // ---------------- phase B: M-fragments I, 7-I (k-steps 2mf .. 15)
  const int offYB = 2 * ((lane >> 2) * LDY + L.kq) + (lane & 1);
#pragma unroll
  for (int u = 0; u < 2; u++) {
    const int mf = u == 0 ? I : 7 - I;
    y[u][0] = y[u][1] = 0.0;
#pragma unroll
    for (int ks = 2 * mf; ks < 16; ks++) dmma_nv(y[u], xsign(tt[L.offT + 136 * ks + 8 * mf], L.negT), yq[offYB + 4 * ks]);
  }
#pragma unroll
  for (int u = 0; u < 2; u++) {
    const int refl = 4 * (u == 0 ? I : 7 - I) + (L.rr >> 1);
#pragma unroll
    for (int c = 0; c < 2; c++) y2q[2 * ((2 * (lane & 3) + c) * LDY + refl) + (L.rr & 1)] = y[u][c];
  }
  quad_sync();
  // ---------------- phase C: row groups {I, 7-I, 8+I, 15-I} then {16+I, 23-I}
  double yb[16];
#pragma unroll
  for (int ks = 0; ks < 16; ks++) yb[ks] = y2q[offYB + 4 * ks];
  if (I == 0 && F.more) {
    // the padding slot (current row 95) receives the next block's row 31
    const int c = lane >> 2;
    const int64_t row = F.rs + W;
    const bool ok = (lane & 3) == 0 && row < F.n && c < F.ncols;
    if ((lane & 3) == 0) cp_async16m(&F.Ew[c * LDE + ring_slot(F.base - 1)], ok ? F.E + row + (F.c0 + c) * F.lde : F.E, ok);
  }
  phase_c_rows<4, QuadLow<I>, true>(F, L, vc, yb);
  cp_async_commit();
  phase_c_rows<2, QuadHigh<I>, false>(F, L, vc, yb);
}

// ---------------------------------------------------------------- kernel
__global__ void __launch_bounds__(WT, 1) apply_q2w_kernel(Q2wArgs a) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // zero the compact V buffers once (their pads are never written again) and the E windows
  for (int e = threadIdx.x; e < OFF_T; e += WT) q2w_sm[e] = czero();
  for (int e = threadIdx.x; e < NFS * 8 * LDE; e += WT) q2w_sm[OFF_E + e] = czero();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      mbar_init(full_bar(i), 1);
      *done_cnt(i) = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  BlkIt cur, ahead;
  it_begin(a, cur);
  ahead = cur;
  if (w == 0) {   // prologue: blocks 0 and 1
    if (ahead.valid) issue_block(a, blk_src(a, ahead), 0, lane);
    it_next(a, ahead);
    if (ahead.valid) issue_block(a, blk_src(a, ahead), 1, lane);
    it_next(a, ahead);
  } else {
    it_next(a, ahead);
    it_next(a, ahead);
  }
  const int F = a.nfr_total, Gd = gridDim.x;
  const int f0 = (int)((int64_t)F * blockIdx.x / Gd), f1 = (int)((int64_t)F * (blockIdx.x + 1) / Gd);
  const bool quad = Q2W_QUAD && w >= NFW;
  const int qi = w - NFW;
  const Lane L(lane);
  Frag Fr;
  Fr.Ew = q2w_sm + OFF_E + (quad ? NFW : imin_c(w, NFW)) * 8 * LDE;
  Fr.ew = reinterpret_cast<double *>(Fr.Ew);
  Fr.E = a.E;
  Fr.lde = a.lde;
  Fr.lde2 = 2 * a.lde;
  Fr.n = a.n;
  // fragments of slab sl in this CTA, and how many warps work on them
  auto slab_k = [&](int sl) { return imax_c(0, imin_c(NFS, f1 - (f0 + sl * NFS))); };
  auto n_active = [](int k) { return (Q2W_QUAD && (k & 3) == 1) ? k - 1 + NQW : k; };
  BlkSrc asrc;
  bool active = false;
  int cur_sl = -1, nact = 0;
  int64_t cnt = 0;
  while (cur.valid) {
    if (cur.sl != cur_sl) {
      cur_sl = cur.sl;
      const int s0 = f0 + cur_sl * NFS;
      const int k = slab_k(cur_sl);
      const bool quad_on = Q2W_QUAD && (k & 3) == 1;
      const int nfull = quad_on ? k - 1 : k;
      nact = n_active(k);
      active = quad ? quad_on : (w < nfull);
      if (active) asrc = blk_src(a, ahead);
      const int fr = quad ? s0 + nfull : s0 + w;
      Fr.c0 = (int64_t)fr * 8;
      Fr.ncols = active ? (int)imin64(8, a.m - Fr.c0) : 0;
      const int cA = 2 * (lane & 3);
      Fr.ok0 = cA < Fr.ncols;
      Fr.ok1 = cA + 1 < Fr.ncols;
    }
    const int64_t i0 = cur.gi * G;
    if (cur.j == 0) {
      Fr.base = 0;
      if (active) {
        // group start: the whole window, rows rs .. rs + 95 (row 95 is padding)
        const int64_t rs = i0 + 1;
        const int e0 = quad ? lane + 32 * qi : lane, es = quad ? 32 * NQW : 32;
        for (int e = e0; e < RING * 8; e += es) {
          const int q = e % RING, c = e / RING;
          const int64_t row = rs + q;
          const bool ok = q < W && row < a.n && c < Fr.ncols;
          cp_async16m(&Fr.Ew[c * LDE + q], ok ? a.E + row + (Fr.c0 + c) * a.lde : a.E, ok);
        }
        cp_async_commit();
        cp_async_commit();   // empty group: the full warps' wait<1> then covers the window
      }
    }
    const int bi = (int)(cnt & 1);
    if (!active) {   // idle in this slab: keep the block count, touch nothing
      it_next(a, cur);
      it_next(a, ahead);
      cnt++;
      continue;
    }
    Fr.rs = i0 + 1 + cur.j * NB;
    Fr.more = cur.j + 1 < cur.J;
    const bool prof = a.prof != nullptr && blockIdx.x == 0 && lane == 0 && w == 0;
    unsigned long long *pp = prof ? a.prof + 24 : nullptr;
    long long tl = prof ? clock64() : 0;
    mbar_wait(full_bar(bi), (unsigned)((cnt >> 1) & 1));
    pmark(pp, tl, 0);
    {
      if (quad) {
        cp_async_wait<0>();
        __syncwarp();
        quad_sync();   // the quad's refills and row-group stores of the previous block
      } else {
        cp_async_wait<1>();   // group X (rows 64..94 of this block's window); Y is awaited in phase A
        __syncwarp();
      }   // the quad's refills and row-group stores of the previous block
      Fr.ch0 = 2 * 32 * ((0 + Fr.base / 32) % 3);
      Fr.ch1 = 2 * 32 * ((1 + Fr.base / 32) % 3);
      Fr.ch2 = 2 * 32 * ((2 + Fr.base / 32) % 3);
      Fr.gE = reinterpret_cast<double *>(a.E + Fr.rs + (L.rr >> 1) + (Fr.c0 + 2 * (lane & 3)) * a.lde) + (L.rr & 1);
      const double *vc = reinterpret_cast<const double *>(vc_buf(bi));
      const double *tt = reinterpret_cast<const double *>(t_buf(bi));
      if (!quad) full_block(Fr, L, vc, tt, pp, tl);
      else if (qi == 0) quad_block<0>(Fr, L, vc, tt);
      else if (qi == 1) quad_block<1>(Fr, L, vc, tt);
      else if (qi == 2) quad_block<2>(Fr, L, vc, tt);
      else quad_block<3>(Fr, L, vc, tt);
      if (!Fr.more) __threadfence_block();   // the next group re-reads these rows
      Fr.base = Fr.base + NB >= RING ? Fr.base + NB - RING : Fr.base + NB;
    }
    // release buffer bi; the last warp refills it with the block two ahead
    // (every value this warp loaded from it has been consumed by now)
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      last = atomicAdd(done_cnt(bi), 1) == nact - 1;
      if (last) *done_cnt(bi) = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last && ahead.valid && slab_k(ahead.sl) > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_block(a, asrc, bi, lane);
    }
    pmark(pp, tl, 4);
    it_next(a, cur);
    it_next(a, ahead);
    asrc = blk_src(a, ahead);
    cnt++;
  }
}

// ---------------------------------------------------------------- split kernel (small m)
// One fragment shared by NQ warps (NQ = 4: like the quad above; NQ = 8: one
// M-fragment / three row groups per warp), NG fragments per CTA.  For small m
// (few fragments per SM) this keeps 8-16 warps per SM busy on the sequential
// block chain instead of one or two.
template <int NQ, int I>
struct SplitSets {
  static constexpr int NMA = 8 / NQ;   // phase A / B M-fragments per warp
  __device__ static constexpr int ma(int u) { return NQ == 4 ? 2 * I + u : I; }
  __device__ static constexpr int mb(int u) { return NQ == 4 ? (u == 0 ? I : 7 - I) : I; }
  static constexpr int NLO = NQ == 4 ? 4 : 2, NHI = NQ == 4 ? 2 : 1;
};
template <int NQ, int I>
struct SplitLow {
  __device__ static constexpr int f(int u) {
    return NQ == 4 ? (u == 0 ? I : u == 1 ? 7 - I : u == 2 ? 8 + I : 15 - I) : (u == 0 ? I : 15 - I);
  }
};
template <int NQ, int I>
struct SplitHigh {
  __device__ static constexpr int f(int u) { return NQ == 4 ? (u == 0 ? 16 + I : 23 - I) : 16 + I; }
};

template <int NQ, int I>
__device__ __forceinline__ void split_block(const Frag &F, const Lane &L, const double *vc, const double *tt,
                                            double *yq, double *y2q, int barid) {
  using S = SplitSets<NQ, I>;
  constexpr int NMA = S::NMA;
  const int lane = L.lane;
  // ---------------- phase A
  double y[NMA][2];
#pragma unroll
  for (int u = 0; u < NMA; u++) y[u][0] = y[u][1] = 0.0;
  constexpr int KS0 = 2 * S::ma(0), KS1 = imin_c(48, 2 * S::ma(NMA - 1) + 34);
#pragma unroll
  for (int ks = KS0; ks < KS1; ks++) {
    const int ch = ks < 16 ? F.ch0 : (ks < 32 ? F.ch1 : F.ch2);
    const double e = F.ew[ch + L.offEB + 4 * (ks & 15)];
#pragma unroll
    for (int u = 0; u < NMA; u++) {
      const int mf = S::ma(u);
      if (ks >= 2 * mf && ks <= 2 * mf + 33) dmma_nv(y[u], xsign(vc[L.offA + 568 * mf + 4 * ks], L.negConj), e);
    }
  }
#pragma unroll
  for (int u = 0; u < NMA; u++) {
    const int refl = 4 * S::ma(u) + (L.rr >> 1);
#pragma unroll
    for (int c = 0; c < 2; c++) yq[2 * ((2 * (lane & 3) + c) * LDY + refl) + (L.rr & 1)] = y[u][c];
  }
  asm volatile("bar.sync %0, %1;" ::"r"(barid), "r"(32 * NQ) : "memory");
  // ---------------- phase B
  const int offYB = 2 * ((lane >> 2) * LDY + L.kq) + (lane & 1);
#pragma unroll
  for (int u = 0; u < NMA; u++) {
    const int mf = S::mb(u);
    y[u][0] = y[u][1] = 0.0;
#pragma unroll
    for (int ks = 2 * mf; ks < 16; ks++) dmma_nv(y[u], xsign(tt[L.offT + 136 * ks + 8 * mf], L.negT), yq[offYB + 4 * ks]);
  }
#pragma unroll
  for (int u = 0; u < NMA; u++) {
    const int refl = 4 * S::mb(u) + (L.rr >> 1);
#pragma unroll
    for (int c = 0; c < 2; c++) y2q[2 * ((2 * (lane & 3) + c) * LDY + refl) + (L.rr & 1)] = y[u][c];
  }
  asm volatile("bar.sync %0, %1;" ::"r"(barid), "r"(32 * NQ) : "memory");
  // ---------------- phase C
  double yb[16];
#pragma unroll
  for (int ks = 0; ks < 16; ks++) yb[ks] = y2q[offYB + 4 * ks];
  if (I == 0 && F.more) {
    // the padding slot (current row 95) receives the next block's row 31
    const int c = lane >> 2;
    const int64_t row = F.rs + W;
    const bool ok = (lane & 3) == 0 && row < F.n && c < F.ncols;
    if ((lane & 3) == 0) cp_async16m(&F.Ew[c * LDE + ring_slot(F.base - 1)], ok ? F.E + row + (F.c0 + c) * F.lde : F.E, ok);
  }
  phase_c_rows<S::NLO, SplitLow<NQ, I>, true>(F, L, vc, yb);
  cp_async_commit();
  phase_c_rows<S::NHI, SplitHigh<NQ, I>, false>(F, L, vc, yb);
}

template <int NQ>
__device__ __forceinline__ void split_dispatch(int I, const Frag &F, const Lane &L, const double *vc,
                                               const double *tt, double *yq, double *y2q, int barid) {
  switch (I) {
    case 0: split_block<NQ, 0>(F, L, vc, tt, yq, y2q, barid); break;
    case 1: split_block<NQ, 1>(F, L, vc, tt, yq, y2q, barid); break;
    case 2: split_block<NQ, 2>(F, L, vc, tt, yq, y2q, barid); break;
    case 3: split_block<NQ, 3>(F, L, vc, tt, yq, y2q, barid); break;
    case 4: if constexpr (NQ > 4) split_block<NQ, 4 % NQ>(F, L, vc, tt, yq, y2q, barid); break;
    case 5: if constexpr (NQ > 5) split_block<NQ, 5 % NQ>(F, L, vc, tt, yq, y2q, barid); break;
    case 6: if constexpr (NQ > 6) split_block<NQ, 6 % NQ>(F, L, vc, tt, yq, y2q, barid); break;
    default: if constexpr (NQ > 7) split_block<NQ, 7 % NQ>(F, L, vc, tt, yq, y2q, barid); break;
  }
}

template <int NQ, int NG>
__global__ void __launch_bounds__(32 * NQ * NG, 1) apply_q2s_kernel(Q2wArgs a) {
  constexpr int TH = 32 * NQ * NG;
  static_assert(NG * 8 * LDE + NG * 2 * 8 * LDY <= NFS * 8 * LDE, "split layout must fit the q2w window area");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = w / NQ, I = w % NQ;
  for (int e = threadIdx.x; e < OFF_T; e += TH) q2w_sm[e] = czero();
  for (int e = threadIdx.x; e < NFS * 8 * LDE; e += TH) q2w_sm[OFF_E + e] = czero();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      mbar_init(full_bar(i), 1);
      *done_cnt(i) = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  BlkIt cur, ahead;
  it_begin(a, cur);
  ahead = cur;
  if (w == 0) {
    if (ahead.valid) issue_block(a, blk_src(a, ahead), 0, lane);
    it_next(a, ahead);
    if (ahead.valid) issue_block(a, blk_src(a, ahead), 1, lane);
    it_next(a, ahead);
  } else {
    it_next(a, ahead);
    it_next(a, ahead);
  }
  const int F = a.nfr_total, Gd = gridDim.x;
  const int f0 = (int)((int64_t)F * blockIdx.x / Gd), f1 = (int)((int64_t)F * (blockIdx.x + 1) / Gd);
  const Lane L(lane);
  double *yq = reinterpret_cast<double *>(q2w_sm + OFF_E + NG * 8 * LDE + g * 2 * 8 * LDY);
  double *y2q = yq + 2 * 8 * LDY;
  const int barid = 1 + g;
  Frag Fr;
  Fr.Ew = q2w_sm + OFF_E + g * 8 * LDE;
  Fr.ew = reinterpret_cast<double *>(Fr.Ew);
  Fr.E = a.E;
  Fr.lde = a.lde;
  Fr.lde2 = 2 * a.lde;
  Fr.n = a.n;
  auto slab_k = [&](int sl) { return imax_c(0, imin_c(NG, f1 - (f0 + sl * NG))); };
  BlkSrc asrc;
  bool active = false;
  int cur_sl = -1, nact = 0;
  int64_t cnt = 0;
  while (cur.valid) {
    if (cur.sl != cur_sl) {
      cur_sl = cur.sl;
      const int k = slab_k(cur_sl);
      nact = NQ * k;
      active = g < k;
      if (active) asrc = blk_src(a, ahead);
      Fr.c0 = (int64_t)(f0 + cur_sl * NG + g) * 8;
      Fr.ncols = active ? (int)imin64(8, a.m - Fr.c0) : 0;
      const int cA = 2 * (lane & 3);
      Fr.ok0 = cA < Fr.ncols;
      Fr.ok1 = cA + 1 < Fr.ncols;
    }
    const int64_t i0 = cur.gi * G;
    if (cur.j == 0) {
      Fr.base = 0;
      if (active) {
        const int64_t rs = i0 + 1;
        for (int e = lane + 32 * I; e < RING * 8; e += 32 * NQ) {
          const int q = e % RING, c = e / RING;
          const int64_t row = rs + q;
          const bool ok = q < W && row < a.n && c < Fr.ncols;
          cp_async16m(&Fr.Ew[c * LDE + q], ok ? a.E + row + (Fr.c0 + c) * a.lde : a.E, ok);
        }
        cp_async_commit();
      }
    }
    const int bi = (int)(cnt & 1);
    if (!active) {
      it_next(a, cur);
      it_next(a, ahead);
      cnt++;
      continue;
    }
    Fr.rs = i0 + 1 + cur.j * NB;
    Fr.more = cur.j + 1 < cur.J;
    const bool prof = a.prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    unsigned long long *pp = prof ? a.prof + 24 : nullptr;
    long long tl = prof ? clock64() : 0;
    mbar_wait(full_bar(bi), (unsigned)((cnt >> 1) & 1));
    pmark(pp, tl, 0);
    cp_async_wait<0>();
    __syncwarp();
    pmark(pp, tl, 1);
    asm volatile("bar.sync %0, %1;" ::"r"(barid), "r"(32 * NQ) : "memory");   // the group's refills / stores
    pmark(pp, tl, 2);
    Fr.ch0 = 2 * 32 * ((0 + Fr.base / 32) % 3);
    Fr.ch1 = 2 * 32 * ((1 + Fr.base / 32) % 3);
    Fr.ch2 = 2 * 32 * ((2 + Fr.base / 32) % 3);
    Fr.gE = reinterpret_cast<double *>(a.E + Fr.rs + (L.rr >> 1) + (Fr.c0 + 2 * (lane & 3)) * a.lde) + (L.rr & 1);
    split_dispatch<NQ>(I, Fr, L, reinterpret_cast<const double *>(vc_buf(bi)),
                       reinterpret_cast<const double *>(t_buf(bi)), yq, y2q, barid);
    pmark(pp, tl, 3);
    if (!Fr.more) __threadfence_block();
    Fr.base = Fr.base + NB >= RING ? Fr.base + NB - RING : Fr.base + NB;
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      last = atomicAdd(done_cnt(bi), 1) == nact - 1;
      if (last) *done_cnt(bi) = 0;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last && ahead.valid && slab_k(ahead.sl) > 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue_block(a, asrc, bi, lane);
    }
    pmark(pp, tl, 4);
    it_next(a, cur);
    it_next(a, ahead);
    asrc = blk_src(a, ahead);
    cnt++;
  }
}

// ---------------------------------------------------------------- wavefront kernel (small m)
// Block (g, j) of group g (sweeps 32g..32g+31, rows 32g+1+64j .. +94)
// overlaps only blocks (g+1, j-1) and (g+1, j) of the group applied before it
// (windows of 95 rows, groups 32 rows apart, steps 64 rows apart), so the
// blocks with the same t = j + (G-1-g) are pairwise disjoint and every
// block they depend on has a smaller t: up to ~J blocks per step instead of
// one sequential chain per column fragment.  One cooperative
// persistent kernel walks the ~J + 2G steps; at each step the (block,
// fragment) items are split evenly over the CTAs, a CTA stages the V / T of a
// block once for all its warps, and each warp runs the three contractions of
// one fragment (loading its whole window and storing it back).
__device__ __forceinline__ int64_t wave_J(const Q2wArgs &a, int64_t g) { return steps_of(a, g); }

// Per warp, the window has four 32-row chunk slots (column stride LDWV): the
// item being computed uses three, and the fourth receives the next item's
// first chunk as soon as the item starts; the next item's other two chunks go
// into the slots of the finished item, so the window loads overlap compute.
#ifndef Q2_WAVE_SLOTS
#define Q2_WAVE_SLOTS 3
#endif
// 4 slots: 10 warps, the next item's first chunk prefetched into the spare slot;
// 3 slots: 12 warps (3 per SM sub-partition, 159 registers), no spare: the
// extra warps hide the window loads better than the prefetch did (n = 10^4:
// m = 10^4 / 1250 / 1000: 346.5 / 59.2 / 50.5 ms -> 328.8 / 56.2 / 48.2 ms)
constexpr int WSLOTS = Q2_WAVE_SLOTS;
constexpr int LDWV = 32 * WSLOTS + 1;   // chunks of 32 rows + 1 (odd: conflict-free)
#ifndef Q2_WAVE_WARPS
#define Q2_WAVE_WARPS (WSLOTS == 4 ? 10 : 12)
#endif
constexpr int WAVE_WARPS = Q2_WAVE_WARPS;   // items are claimed dynamically
constexpr int OFF_WAVE_T = VC_STAGE;                 // layout: V | T | windows
constexpr int OFF_WAVE_WIN = OFF_WAVE_T + T_STAGE;
static_assert(OFF_WAVE_WIN + WAVE_WARPS * 8 * LDWV <= OFF_BAR, "wave windows must fit the q2w shared-memory size");

__global__ void __launch_bounds__(32 * WAVE_WARPS, 1) apply_q2wave_kernel(Q2wArgs a, int64_t T) {
  namespace cg = cooperative_groups;
  constexpr int TH = 32 * WAVE_WARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ int s_claim;   // next unclaimed item of this CTA's share of the step
  // layout: V | T | one window of 8 x LDWV per warp
  double2 *vc = q2w_sm, *tb = q2w_sm + OFF_WAVE_T;
  double2 *win0 = q2w_sm + OFF_WAVE_WIN;
  for (int e = threadIdx.x; e < VC_STAGE; e += TH) vc[e] = czero();
  __syncthreads();
  const int64_t Gn = a.ngroups, F = a.nfr_total;
  const Lane L(lane, LDWV);
  Frag Fr;
  Fr.Ew = win0 + w * 8 * LDWV;
  Fr.ew = reinterpret_cast<double *>(Fr.Ew);
  Fr.E = a.E;
  Fr.lde = a.lde;
  Fr.lde2 = 2 * a.lde;
  Fr.n = a.n;
  Fr.more = false;   // every window is stored whole, from the accumulators
  Fr.base = 0;
  int sa = 0, sb = 1, sc = 2, sd = 3;   // chunk slots: rows 0-31, 32-63, 64-95, spare
  // item = (step-local block index, fragment); chunk c of its window -> slot
  auto load_chunk = [&](int64_t rs, int64_t c0, int ncols, int c, int slot) {
    for (int e = lane; e < 32 * 8; e += 32) {
      const int q = e & 31, col = e >> 5;
      const int row_in = 32 * c + q;
      const int64_t row = rs + row_in;
      const bool ok = row_in < W && row < a.n && col < ncols;
      cp_async16m(&Fr.Ew[col * LDWV + 32 * slot + q], ok ? a.E + row + (c0 + col) * a.lde : a.E, ok);
    }
  };
  cg::grid_group grid = cg::this_grid();
  for (int64_t t = 0; t < T; t++) {
    // blocks of this step: d = G-1-g in [dlo, dhi], j = t - d
    const int64_t dhi = imin64(Gn - 1, t);
    int64_t dlo = 0;
    while (dlo <= dhi && t - dlo >= wave_J(a, Gn - 1 - dlo)) dlo++;
    const int64_t nblk = dhi - dlo + 1;
    if (nblk > 0) {
      const int64_t items = nblk * F;
      const int64_t i0c = items * blockIdx.x / gridDim.x, i1c = items * (blockIdx.x + 1) / gridDim.x;
      // items are claimed in order (block-major) from a shared counter, so the
      // warps of the busier sub-partitions simply take fewer of them
      if (threadIdx.x == 0) s_claim = 0;
      __syncthreads();
      auto claim = [&]() -> int64_t {
        int v = 0;
        if (lane == 0) v = atomicAdd(&s_claim, 1);
        v = __shfl_sync(0xffffffffu, v, 0);
        return i0c + v < i1c ? i0c + v : -1;
      };
      auto item_rs = [&](int64_t it) { const int64_t d = dlo + it / F; return (Gn - 1 - d) * G + 1 + (t - d) * NB; };
      int64_t cur = claim();
      if (cur >= 0) {   // the first item's chunks
        const int64_t f = cur % F;
        const int nc = (int)imin64(8, a.m - f * 8);
        load_chunk(item_rs(cur), f * 8, nc, 0, sa);
        cp_async_commit();
        load_chunk(item_rs(cur), f * 8, nc, 1, sb);
        cp_async_commit();
        load_chunk(item_rs(cur), f * 8, nc, 2, sc);
        cp_async_commit();
      }
      for (int64_t seg0 = i0c; seg0 < i1c; seg0 = imin64(i1c, (seg0 / F + 1) * F)) {
        const int64_t seg_end = imin64(i1c, (seg0 / F + 1) * F);
        const int64_t bidx = seg0 / F;
        const int64_t d = dlo + bidx, g = Gn - 1 - d, j = t - d, gi0 = g * G;
        // ---- stage V (compact rows) and T of block (g, j)
        const int nvalid = (int)imax64(0, imin64(G, a.n - 2 - j * NB - gi0 + 1));
        const double2 *v2 = a.V2 + (a.off[j] + gi0) * NB;
        const double2 *t2 = a.T2 + (a.first[g] + j) * G * G;
        __syncthreads();   // the previous block's V / T are no longer read
        for (int e = threadIdx.x; e < G * NB; e += TH) {
          const int tt = e / NB, ss = e - tt * NB;
          if (tt < nvalid) cp_async16(vc + vrow(tt) + PADL + ss, v2 + tt * NB + ss, true);
        }
        for (int e = threadIdx.x; e < G * G; e += TH) {
          const int kk = e / G, xx = e - kk * G;
          cp_async16(tb + tcol(kk) + xx, t2 + kk * G + xx, true);
        }
        cp_async_commit();
        cp_async_wait<0>();   // (also completes this warp's window chunks: harmless)
        __syncthreads();
        const double *vcd = reinterpret_cast<const double *>(vc);
        const double *ttd = reinterpret_cast<const double *>(tb);
        // the group counting of full_block<true> expects exactly [chunk 0, chunk 1, chunk 2, next] pending
        while (cur >= 0 && cur < seg_end) {
          const int64_t f = cur % F;
          Fr.rs = gi0 + 1 + j * NB;
          Fr.c0 = f * 8;
          Fr.ncols = (int)imin64(8, a.m - Fr.c0);
          const int cA = 2 * (lane & 3);
          Fr.ok0 = cA < Fr.ncols;
          Fr.ok1 = cA + 1 < Fr.ncols;
          Fr.ch0 = 2 * 32 * sa;
          Fr.ch1 = 2 * 32 * sb;
          Fr.ch2 = 2 * 32 * sc;
          Fr.gE = reinterpret_cast<double *>(a.E + Fr.rs + (L.rr >> 1) + (Fr.c0 + cA) * a.lde) + (L.rr & 1);
          const int64_t nxt = claim();
          int64_t nrs = 0, nc0 = 0;
          int nnc = 0;
          if (nxt >= 0) {
            const int64_t nf = nxt % F;
            nrs = item_rs(nxt);
            nc0 = nf * 8;
            nnc = (int)imin64(8, a.m - nc0);
            if (WSLOTS == 4) load_chunk(nrs, nc0, nnc, 0, sd);
          }
          long long tl = 0;
          if (WSLOTS == 4) {
            cp_async_commit();   // (possibly empty) keeps the group count uniform
            full_block<true, 3>(Fr, L, vcd, ttd, nullptr, tl);
          } else {
            full_block<true, 2>(Fr, L, vcd, ttd, nullptr, tl);
          }
          __syncwarp();        // every lane is done reading this item's chunks
          if (nxt >= 0) {
            if (WSLOTS != 4) {
              load_chunk(nrs, nc0, nnc, 0, sa);
              cp_async_commit();
            }
            load_chunk(nrs, nc0, nnc, 1, sb);
            cp_async_commit();
            load_chunk(nrs, nc0, nnc, 2, sc);
            cp_async_commit();
            if (WSLOTS == 4) {
              const int s_old = sa;
              sa = sd;
              sd = s_old;
            }
          }
          cur = nxt;
        }
      }
      cp_async_wait<0>();
    }
    __threadfence();
    grid.sync();
  }
}

}  // namespace

size_t q2w_smem_bytes() { return (size_t)OFF_BAR * sizeof(double2) + 32; }

// Returns 1 if the shape is not handled here (caller falls back to q2.cu).
int q2w_apply(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *T2, double2 *E, int64_t lde, int64_t m) {
  if (p.nb != NB || p.g != G) return 1;
  Q2wArgs a;
  a.n = p.n;
  a.m = m;
  a.lde = lde;
  a.ngroups = p.ngroups;
  a.first = p.d_group_first_block;
  a.off = p.d_off;
  a.V2 = V2;
  a.T2 = T2;
  a.E = E;
  a.nfr_total = (int)((m + 7) / 8);
  a.prof = ctx.q2_prof;
  const int grid = std::min(ctx.num_sms, a.nfr_total);
  const int per = (a.nfr_total + grid - 1) / grid;
  a.nslab = (per + NFS - 1) / NFS;
  const size_t smem = q2w_smem_bytes();
  // the wavefront kernel (measured faster at every m: n = 10^4, m = 1000 / 2500 /
  // 5000 / 10000: 54 / 110 / 206 / 392 ms vs 135 / 274 / 306 / 404 ms for the
  // per-fragment kernels below, which EIG_Q2_WAVE=0 selects)
  static const int wave_env = [] {
    const char *e = getenv("EIG_Q2_WAVE");
    return e ? atoi(e) : 1;
  }();
  if (wave_env) {
    int64_t T = 0;
    for (int64_t g = 0; g < a.ngroups; g++) {
      const int64_t i0 = g * G;
      const int64_t J = (i0 > a.n - 2) ? 0 : (a.n - 2 - i0) / NB + 1;
      if (J > 0) T = std::max<int64_t>(T, J - 1 + (a.ngroups - 1 - g) + 1);
    }
    EIG_TRY(ctx.smem_attr((const void *)apply_q2wave_kernel, (int)smem, "q2wave attr"));
    const int gridw = ctx.num_sms;
    void *args[] = {&a, &T};
    EIG_TRY(ctx.check(cudaLaunchCooperativeKernel((void *)apply_q2wave_kernel, dim3(gridw), dim3(32 * WAVE_WARPS), args, smem,
                                                  ctx.stream), "q2wave launch"));
    return ctx.launched("apply_q2wave_kernel");
  }
  // few fragments per SM: share each fragment over 8 warps (EIG_Q2W_SPLIT=0 disables)
  static const int split_env = [] {
    const char *e = getenv("EIG_Q2W_SPLIT");
    return e ? atoi(e) : 1;
  }();
  if (split_env && per <= 2) {
    a.nslab = (per + 1) / 2;
    EIG_TRY(ctx.smem_attr((const void *)apply_q2s_kernel<8, 2>, (int)smem, "q2s attr"));
    apply_q2s_kernel<8, 2><<<grid, 32 * 8 * 2, smem, ctx.stream>>>(a);
    return ctx.launched("apply_q2s_kernel");
  }
  EIG_TRY(ctx.smem_attr((const void *)apply_q2w_kernel, (int)smem, "q2w attr"));
  apply_q2w_kernel<<<grid, WT, smem, ctx.stream>>>(a);
  EIG_TRY(ctx.launched("apply_q2w_kernel"));
  return 0;
}

}  // namespace eig
