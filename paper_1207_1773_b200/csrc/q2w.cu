// q2w.cu — E <- Q2 E (a6) for nb = 64, g = 32: the wavefront kernel.
//
// Block structure of DESIGN.md R7 (block (i0, j) of g sweeps is I - V T V^H,
// V the W x g parallelogram, W = nb + g - 1 = 95), executed in the wavefront
// order of reading R17: all blocks with equal t = j + (G-1-g) are disjoint,
// so one cooperative kernel walks the steps t and, within a step, every
// (block, 8-column fragment) item is an independent task:
//
//  * a warp runs all three contractions of an item alone — Y = V^H E
//    (phase A), Y = T Y (phase B), E -= V Y (phase C) — with Y in registers,
//    moved between the DMMA accumulator and operand layouts by shuffles;
//  * V (compact: Vc[t][4 + s] = v_t[s], zero pads on both sides,
//    bank-conflict-free row placement) and T of a block are staged once per
//    CTA for all its warps;
//  * every loop over k-steps and row groups is fully unrolled against the
//    compile-time parallelogram shape: all shared-memory addresses are a lane
//    base plus an immediate, and only the nonzero DMMA tiles are issued;
//  * twelve warps per CTA claim items from a shared counter; each keeps its
//    item's 95-row window in three 32-row chunk slots (cp.async groups waited
//    for chunk by chunk inside phase A) and stores the rows straight from the
//    phase-C accumulators.
// The r01 per-fragment kernels (a warp per fragment walking the block chain)
// were removed in r02; other (nb, g) shapes use the generic kernel of q2.cu.
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
// L2 policy of the E stream (read and written once per item): evict-first.
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
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

// dynamic shared memory of the wavefront kernel (layout defined there)
extern __shared__ __align__(128) double2 q2w_sm[];

// ---------------------------------------------------------------- block sequence
__device__ __forceinline__ int64_t steps_of(const Q2wArgs &a, int64_t gi) {
  const int64_t i0 = gi * G;
  return (i0 > a.n - 2) ? 0 : (a.n - 2 - i0) / NB + 1;
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
constexpr int OFF_WAVE_END = OFF_WAVE_WIN + WAVE_WARPS * 8 * LDWV;
static_assert(OFF_WAVE_END * 16 + 32 <= 227 * 1024, "wave kernel shared memory");

// ---------------------------------------------------------------- 3M form
// The three contractions of an item with complex operands split into real
// planes (reading R18, Gauss): per contraction three real DMMA products
// instead of the embedding's four, on 8 x 4 real tiles:
//   phase A  Y = V^H E:   P1 = Vr.Er, P2 = Vi.Ei, P3 = (Vr+Vi).(Er-Ei);
//                         Re Y = P1 + P2, Im Y = P1 - P2 - P3
//   phase B  Y' = T Y:    P1 = Tr.Yr, P2 = Ti.Yi, P3 = (Tr+Ti).(Yr+Yi);
//                         -Y' = (P2 - P1, P1 + P2 - P3)   (kept negated)
//   phase C  E += V (-Y'): accumulators start at (Er, 0, Er+Ei);
//                         E' = (P1 - P2, P3 - P1 - P2)
// DMMA count per item 216 + 60 + 216 = 492 (the embedding: 616).  The V and
// T planes (Vr, Vi, Vr+Vi; Tr, Ti, Tr+Ti) are built once per block when the
// CTA stages them; only the E / Y plane sums and the recombinations are
// per-item FP64 adds (184 per lane, ~0.16 DMMA each, tools/peaks/dmma_dadd.cu).
//
// V plane layout (doubles): V[q][t] (t = reflector, q = window row, 0 <= q-t
// < 64) at t LDP + PADP + q - t, LDP = 77: the accesses of both phases read
// q - t in [-7, 71], which stays inside row t's zero pads (rows overlap only
// in pads), and 76 = 12 mod 16 makes the 8-byte fragment loads of phase A
// (t = lane>>2, q = lane&3) and phase C (q = lane>>2, t = lane&3)
// conflict-free.  T planes: the 20 nonzero 8 x 4 tiles of the upper
// triangle, each in fragment (lane) order.
constexpr int LDP = 77, PADP = 8;
constexpr int VP_PLANE = 2472;   // >= 31 LDP + PADP + 72, multiple of 8
constexpr int TP_PLANE = 640;    // 20 tiles x 32
constexpr int OFF3_T = 3 * VP_PLANE / 2;            // complex units
constexpr int OFF3_WIN = OFF3_T + 3 * TP_PLANE / 2;
__host__ __device__ constexpr int ttile(int mf, int ks) { return mf * (9 - mf) + ks - 2 * mf; }
// phase A reads window column sigma(n) as B column n (conflict-free 16-byte
// loads); the phase-B result is returned to E column order in its shuffle
__host__ __device__ constexpr int sigma_col(int n) { return (n >> 1) + 4 * (n & 1); }
__host__ __device__ constexpr int sigma_inv(int e) { return e < 4 ? 2 * e : 2 * (e - 4) + 1; }

// accumulator (rows 8mf + lane>>2, columns 2(lane&3) + h) -> B operand of
// k-step ks (row 4ks + (lane&3), column n = the lane's column index ncol)
__device__ __forceinline__ void acc_to_b3(const double (&acc)[4][2], double (&bl)[8], int lane, int ncol) {
  const int src_lo = 4 * (lane & 3) + (ncol >> 1);
  const bool hi = ncol & 1;
#pragma unroll
  for (int ks = 0; ks < 8; ks++) {
    const int src = src_lo + 16 * (ks & 1);
    const double v0 = __shfl_sync(0xffffffffu, acc[ks >> 1][0], src);
    const double v1 = __shfl_sync(0xffffffffu, acc[ks >> 1][1], src);
    bl[ks] = hi ? v1 : v0;
  }
}

struct Item3 {
  const double2 *Ew;      // warp's window (complex), column stride LDWV
  int s0, s1, s2;         // chunk slot bases (complex rows)
  int64_t rs, n, lde;     // first window row, matrix rows, E leading dimension
  double2 *gE;            // E + rs + c0 lde
  int ncols;
};

template <int WPEND, class Pre>
__device__ __forceinline__ void full_block3(const Item3 &F, int lane, const double *vp, const double *tp, Pre &&pre) {
  const int g8 = lane >> 2, t4 = lane & 3;
  // ---------------- phase A: Y = V^H E (tile (mf, ks) nonzero for 0 <= 4ks - 8mf <= 68)
  double p1[4][2], p2[4][2], p3[4][2];
#pragma unroll
  for (int mf = 0; mf < 4; mf++)
#pragma unroll
    for (int h = 0; h < 2; h++) p1[mf][h] = p2[mf][h] = p3[mf][h] = 0.0;
  const double2 *ewA = F.Ew + sigma_col(g8) * LDWV + t4;
  const double *vA = vp + g8 * (LDP - 1) + t4 + PADP;
#pragma unroll
  for (int ks = 0; ks < 24; ks++) {
    if (ks == 0) {
      cp_async_wait<WPEND>();
      __syncwarp();
    }
    if (ks == 8) {
      cp_async_wait<WPEND - 1>();
      __syncwarp();
    }
    if (ks == 16) {
      cp_async_wait<WPEND - 2>();
      __syncwarp();
    }
    const int sb = ks < 8 ? F.s0 : (ks < 16 ? F.s1 : F.s2);
    const double2 e = ewA[sb + 4 * (ks & 7)];
    const double ed = e.x - e.y;
#pragma unroll
    for (int mf = 0; mf < 4; mf++) {
      const int d = 4 * ks - 8 * mf;
      if (d >= 0 && d <= 68) {
        const double *a = vA + 8 * mf * (LDP - 1) + 4 * ks;
        dmma_nv(p1[mf], a[0], e.x);
        dmma_nv(p2[mf], a[VP_PLANE], e.y);
        dmma_nv(p3[mf], a[2 * VP_PLANE], ed);
      }
    }
  }
  double yr[4][2], yi[4][2];
#pragma unroll
  for (int mf = 0; mf < 4; mf++)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      yr[mf][h] = p1[mf][h] + p2[mf][h];
      yi[mf][h] = (p1[mf][h] - p2[mf][h]) - p3[mf][h];
    }
  double br[8], bi[8], bs[8];
  acc_to_b3(yr, br, lane, g8);
  acc_to_b3(yi, bi, lane, g8);
#pragma unroll
  for (int k = 0; k < 8; k++) bs[k] = br[k] + bi[k];
  // ---------------- phase B: -Y' = -T Y (T upper triangular: tiles ks >= 2mf)
#pragma unroll
  for (int mf = 0; mf < 4; mf++)
#pragma unroll
    for (int h = 0; h < 2; h++) p1[mf][h] = p2[mf][h] = p3[mf][h] = 0.0;
#pragma unroll
  for (int ks = 0; ks < 8; ks++)
#pragma unroll
    for (int mf = 0; mf < 4; mf++)
      if (ks >= 2 * mf) {
        const double *a = tp + ttile(mf, ks) * 32 + lane;
        dmma_nv(p1[mf], a[0], br[ks]);
        dmma_nv(p2[mf], a[TP_PLANE], bi[ks]);
        dmma_nv(p3[mf], a[2 * TP_PLANE], bs[ks]);
      }
#pragma unroll
  for (int mf = 0; mf < 4; mf++)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      yr[mf][h] = p2[mf][h] - p1[mf][h];
      yi[mf][h] = (p1[mf][h] + p2[mf][h]) - p3[mf][h];
    }
  acc_to_b3(yr, br, lane, sigma_inv(g8));
  acc_to_b3(yi, bi, lane, sigma_inv(g8));
#pragma unroll
  for (int k = 0; k < 8; k++) bs[k] = br[k] + bi[k];
  // ---------------- phase C: E += V (-Y'), row groups r (rows 8r..8r+7): k-steps
  // max(0, 2r-16) .. min(7, 2r+1).  Row groups go chunk by chunk, two per
  // batch ((0,3), (1,2) | (4,5), (6,7) | (8,11), (9,10): 10 / 16 / 10 k-steps);
  // once a chunk's rows are in registers, pre(c) refills its slot with the
  // next item's chunk, so those loads overlap the rest of phase C.
  const double *vC = vp + t4 * (LDP - 1) + g8 + PADP;
  const bool ok0 = 2 * t4 < F.ncols, ok1 = 2 * t4 + 1 < F.ncols;
#pragma unroll
  for (int b = 0; b < 6; b++) {
    const int c = b >> 1;
    const int ra = c == 1 ? 4 + 2 * (b & 1) : 4 * c + (b & 1);
    const int rb = c == 1 ? ra + 1 : 4 * c + 3 - (b & 1);
    const int sb = c == 0 ? F.s0 : (c == 1 ? F.s1 : F.s2);
    double c1[2][2], c2[2][2], c3[2][2];
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int r = u ? rb : ra;
      const double2 *w = F.Ew + 2 * t4 * LDWV + sb + 8 * (r & 3) + g8;
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const double2 x = w[h * LDWV];
        c1[u][h] = x.x;
        c2[u][h] = 0.0;
        c3[u][h] = x.x + x.y;
      }
    }
    if (b & 1) {
      __syncwarp();   // every lane has read chunk c
      pre(c);
    }
#pragma unroll
    for (int ks = 0; ks < 8; ks++)
#pragma unroll
      for (int u = 0; u < 2; u++) {
        const int r = u ? rb : ra;
        if (ks >= 2 * r - 16 && ks <= 2 * r + 1) {
          const double *a = vC + 4 * ks * (LDP - 1) + 8 * r;
          dmma_nv(c1[u], a[0], br[ks]);
          dmma_nv(c2[u], a[VP_PLANE], bi[ks]);
          dmma_nv(c3[u], a[2 * VP_PLANE], bs[ks]);
        }
      }
#pragma unroll
    for (int u = 0; u < 2; u++) {
      const int q = 8 * (u ? rb : ra) + g8;
      if (q < W && F.rs + q < F.n) {
        double2 *g = F.gE + q + 2 * t4 * F.lde;
        if (ok0) g[0] = make_double2(c1[u][0] - c2[u][0], (c3[u][0] - c1[u][0]) - c2[u][0]);
        if (ok1) g[F.lde] = make_double2(c1[u][1] - c2[u][1], (c3[u][1] - c1[u][1]) - c2[u][1]);
      }
    }
  }
}

constexpr int OFF3_END = OFF3_WIN + WAVE_WARPS * 8 * LDWV;
static_assert(OFF3_END * 16 + 32 <= 227 * 1024, "3M wave kernel shared memory");

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

// ---------------------------------------------------------------- 3M wavefront, dataflow
// Same steps and item split as apply_q2wave_kernel, but without a grid
// barrier between steps: a CTA's share of block (g, j) starts as soon as the
// blocks it overlaps from earlier steps are complete — (g, j-1), (g+1, j-1)
// and (g+1, j) (every other overlapping earlier block precedes one of these,
// tests/test_q2_schedule.py) — counted per block in done[] (fragments
// finished, released after a CTA barrier, acquired by thread 0).  A CTA that
// finishes a step early runs on into the next instead of waiting for the
// slowest CTA of the step.
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(32 * WAVE_WARPS, 1) apply_q2wave3_kernel(Q2wArgs a, int64_t T, int *done) {
  constexpr int TH = 32 * WAVE_WARPS;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ int s_claim;
  double2 *vc = q2w_sm, *tb = q2w_sm + OFF3_T;
  double2 *win0 = q2w_sm + OFF3_WIN;
  double *vp = reinterpret_cast<double *>(vc), *tp = reinterpret_cast<double *>(tb);
  for (int e = threadIdx.x; e < OFF3_T; e += TH) vc[e] = czero();
  const int64_t Gn = a.ngroups, F = a.nfr_total;
  const double2 *Ew = win0 + w * 8 * LDWV;
  double2 *Eww = win0 + w * 8 * LDWV;
  auto load_chunk = [&](int64_t rs, int64_t c0, int ncols, int c) {
    for (int e = lane; e < 32 * 8; e += 32) {
      const int q = e & 31, col = e >> 5;
      const int row_in = 32 * c + q;
      const int64_t row = rs + row_in;
      const bool ok = row_in < W && row < a.n && col < ncols;
      cp_async16m(&Eww[col * LDWV + 32 * c + q], ok ? a.E + row + (c0 + col) * a.lde : a.E, ok);
    }
  };
  auto J_of = [&](int64_t g) { return wave_J(a, g); };
  int64_t prev_b = -1;
  int prev_cnt = 0;
  for (int64_t t = 0; t < T; t++) {
    const int64_t dhi = imin64(Gn - 1, t);
    int64_t dlo = 0;
    while (dlo <= dhi && t - dlo >= J_of(Gn - 1 - dlo)) dlo++;
    const int64_t nblk = dhi - dlo + 1;
    if (nblk <= 0) continue;
    const int64_t items = nblk * F;
    const int64_t i0c = items * blockIdx.x / gridDim.x, i1c = items * (blockIdx.x + 1) / gridDim.x;
    for (int64_t seg0 = i0c; seg0 < i1c;) {
      const int64_t seg_end = imin64(i1c, (seg0 / F + 1) * F);
      const int64_t d = dlo + seg0 / F, g = Gn - 1 - d, j = t - d, gi0 = g * G;
      const int nvalid = (int)imax64(0, imin64(G, a.n - 2 - j * NB - gi0 + 1));
      const double2 *v2 = a.V2 + (a.off[j] + gi0) * NB;
      const double2 *t2 = a.T2 + (a.first[g] + j) * G * G;
      __syncthreads();   // every warp is done with the previous segment (its items and V / T)
      if (threadIdx.x == 0) {
        if (prev_b >= 0) {
          __threadfence();
          atomicAdd(done + prev_b, prev_cnt);
        }
        // RAW / WAR on E: the overlapping blocks of earlier steps
        if (j >= 1) while (ld_acquire_gpu(done + a.first[g] + j - 1) < F) {}
        if (g + 1 < Gn) {
          const int64_t J1 = J_of(g + 1);
          if (j >= 1 && j - 1 < J1) while (ld_acquire_gpu(done + a.first[g + 1] + j - 1) < F) {}
          if (j < J1) while (ld_acquire_gpu(done + a.first[g + 1] + j) < F) {}
        }
        s_claim = 0;
      }
      // ---- stage the V planes (Vr, Vi, Vr + Vi) and T planes of block (g, j)
      // (V2 / T2 are inputs: no dependency; rows t >= nvalid keep the previous
      // block's finite values, which T's zero rows and columns cancel)
      {
        constexpr int NV = (G * NB + TH - 1) / TH;
        double2 buf[NV];
#pragma unroll
        for (int i = 0; i < NV; i++) {
          const int e = threadIdx.x + i * TH;
          buf[i] = (e < G * NB && e / NB < nvalid) ? v2[e] : czero();
        }
#pragma unroll
        for (int i = 0; i < NV; i++) {
          const int e = threadIdx.x + i * TH;
          const int tt = e / NB, ss = e - tt * NB;
          if (e < G * NB && tt < nvalid) {
            double *dd = vp + tt * LDP + PADP + ss;
            dd[0] = buf[i].x;
            dd[VP_PLANE] = buf[i].y;
            dd[2 * VP_PLANE] = buf[i].x + buf[i].y;
          }
        }
        constexpr int NT = (G * G + TH - 1) / TH;
#pragma unroll
        for (int i = 0; i < NT; i++) {
          const int e = threadIdx.x + i * TH;
          const int kk = e / G, xx = e - kk * G;   // column, row
          const int mf = xx >> 3, ks = kk >> 2;
          if (e < G * G && ks >= 2 * mf) {
            const double2 v = xx <= kk ? t2[e] : czero();
            double *dd = tp + ttile(mf, ks) * 32 + (((xx & 7) << 2) | (kk & 3));
            dd[0] = v.x;
            dd[TP_PLANE] = v.y;
            dd[2 * TP_PLANE] = v.x + v.y;
          }
        }
      }
      __syncthreads();   // V / T staged, dependencies acquired (thread 0), s_claim reset
      auto claim = [&]() -> int64_t {
        int v = 0;
        if (lane == 0) v = atomicAdd(&s_claim, 1);
        v = __shfl_sync(0xffffffffu, v, 0);
        return seg0 + v < seg_end ? seg0 + v : -1;
      };
      const int64_t rs = gi0 + 1 + j * NB;
      int64_t cur = claim();
      if (cur >= 0) {
        const int64_t c0 = (cur % F) * 8;
        const int nc = (int)imin64(8, a.m - c0);
        load_chunk(rs, c0, nc, 0);
        cp_async_commit();
        load_chunk(rs, c0, nc, 1);
        cp_async_commit();
        load_chunk(rs, c0, nc, 2);
        cp_async_commit();
      }
      while (cur >= 0) {
        const int64_t f = cur % F;
        Item3 It;
        It.Ew = Ew;
        It.s0 = 0;
        It.s1 = 32;
        It.s2 = 64;
        It.rs = rs;
        It.n = a.n;
        It.lde = a.lde;
        It.gE = a.E + rs + f * 8 * a.lde;
        It.ncols = (int)imin64(8, a.m - f * 8);
        const int64_t nxt = claim();
        const int64_t nc0 = nxt >= 0 ? (nxt % F) * 8 : 0;
        const int nnc = nxt >= 0 ? (int)imin64(8, a.m - nc0) : 0;
        // the next item (same block) reuses the slots chunk by chunk
        full_block3<2>(It, lane, vp, tp, [&](int c) {
          if (nxt >= 0) load_chunk(rs, nc0, nnc, c);
          cp_async_commit();
        });
        cur = nxt;
      }
      cp_async_wait<0>();
      prev_b = a.first[g] + j;
      prev_cnt = (int)(seg_end - seg0);
      seg0 = seg_end;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && prev_b >= 0) {
    __threadfence();
    atomicAdd(done + prev_b, prev_cnt);
  }
}

}  // namespace

size_t q2w_smem_bytes(bool m3) { return (size_t)(m3 ? OFF3_END : OFF_WAVE_END) * sizeof(double2) + 32; }

// Returns 1 if the shape is not handled here (caller falls back to the
// generic grouped kernel of q2.cu, which EIG_Q2_WAVE=0 also selects).
int q2w_apply(Ctx &ctx, const Q2Plan &p, const double2 *V2, const double2 *T2, double2 *E, int64_t lde, int64_t m) {
  if (p.nb != NB || p.g != G) return 1;
  static const int wave_env = [] {
    const char *e = getenv("EIG_Q2_WAVE");
    return e ? atoi(e) : 1;
  }();
  if (!wave_env) return 1;
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
  a.nslab = 1;
  // 3M form by default; EIG_Q2_3M=0 selects the real embedding
  static const bool m3 = [] {
    const char *e = getenv("EIG_Q2_3M");
    return e ? atoi(e) != 0 : true;
  }();
  const size_t smem = q2w_smem_bytes(m3);
  int64_t T = 0;   // wavefront steps
  for (int64_t g = 0; g < a.ngroups; g++) {
    const int64_t i0 = g * G;
    const int64_t J = (i0 > a.n - 2) ? 0 : (a.n - 2 - i0) / NB + 1;
    if (J > 0) T = std::max<int64_t>(T, J - 1 + (a.ngroups - 1 - g) + 1);
  }
  const void *kfn = m3 ? (const void *)apply_q2wave3_kernel : (const void *)apply_q2wave_kernel;
  EIG_TRY(ctx.smem_attr(kfn, (int)smem, "q2wave attr"));
  if (m3) {
    // per-block completion counters (fragments done) of the dataflow schedule
    int64_t nblocks = 0;
    for (int64_t g = 0; g < a.ngroups; g++) {
      const int64_t i0 = g * G;
      nblocks += (i0 > a.n - 2) ? 0 : (a.n - 2 - i0) / NB + 1;
    }
    int *done = (int *)ctx.ws(WS_Q2DONE, (size_t)std::max<int64_t>(1, nblocks) * sizeof(int));
    if (!done) return EIG_ERR_NOMEM;
    EIG_TRY(ctx.check(cudaMemsetAsync(done, 0, (size_t)std::max<int64_t>(1, nblocks) * sizeof(int), ctx.stream),
                      "q2wave done reset"));
    void *args3[] = {&a, &T, &done};
    EIG_TRY(ctx.check(cudaLaunchCooperativeKernel(kfn, dim3(ctx.num_sms), dim3(32 * WAVE_WARPS), args3, smem,
                                                  ctx.stream), "q2wave3 launch"));
    return ctx.launched("apply_q2wave3_kernel");
  }
  void *args[] = {&a, &T};
  EIG_TRY(ctx.check(cudaLaunchCooperativeKernel(kfn, dim3(ctx.num_sms), dim3(32 * WAVE_WARPS), args, smem, ctx.stream),
                    "q2wave launch"));
  return ctx.launched("apply_q2wave_kernel");
}

}  // namespace eig
