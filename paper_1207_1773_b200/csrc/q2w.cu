// q2w.cu — E <- Q2 E (a6) with column-owning warps, for nb = 64, g = 32.
//
// Same block structure as q2.cu (R7: block (i0, j) of g sweeps is
// I - V T V^H, V the W x g parallelogram, W = nb + g - 1 = 95; groups applied
// last to first, steps ascending), different work split:
//
//  * each consumer warp owns one 8-column fragment of E and its 96-row window
//    (a ring of three 32-row chunks in shared memory), and runs all three
//    contractions for it alone — Y = V^H E (phase A), Y = T Y (phase B),
//    E -= V Y (phase C) — with Y kept in registers and moved between the
//    accumulator and operand layouts by warp shuffles, so no barrier is ever
//    shared between consumer warps;
//  * V (compact: Vc[t][4 + s] = v_t[s], zero pads on both sides) and T of the
//    next block are streamed by a producer warp with bulk async copies into a
//    double buffer (full/empty mbarriers), so loading them overlaps compute;
//  * every loop over k-steps and row groups is fully unrolled against the
//    compile-time parallelogram shape: all shared-memory addresses are a lane
//    base plus an immediate, and only the nonzero DMMA tiles are issued;
//  * a warp stores its rows that leave the window straight from the
//    accumulators, then refills their ring slots with the next block's rows
//    (cp.async) while it finishes the remaining row groups.
#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "kernels.h"

namespace eig {
namespace {

constexpr int NB = 64, G = 32, W = NB + G - 1;   // 95 window rows
constexpr int RING = 96;                         // 3 chunks of 32 rows
constexpr int LDE = 98;                          // per-warp E column stride (complex), 2 mod 16
constexpr int LDVC = 72, PADL = 4;               // compact V row stride / left zero pad
constexpr int LDT = 36;                          // T column stride
constexpr int NCW = 9;                           // consumer warps (fragments per slab)
constexpr int WT = (NCW + 1) * 32;               // + producer warp

struct Q2wArgs {
  int64_t n, m, lde;
  int64_t ngroups;
  const int64_t *first;  // [ngroups+1]
  const int64_t *off;    // [J]
  const double2 *V2;
  const double2 *T2;
  double2 *E;
  int nfr_total;
};

__device__ __forceinline__ unsigned su32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
// non-volatile DMMA: lets the scheduler interleave the unrolled tiles freely
__device__ __forceinline__ void dmma_nv(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
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

// shared memory: Vc[2] | T[2] | E windows (NCW) | full[2], empty[2] mbarriers
extern __shared__ __align__(128) double2 q2w_sm[];
constexpr int OFF_T = 2 * G * LDVC, OFF_E = OFF_T + 2 * G * LDT, OFF_BAR = OFF_E + NCW * 8 * LDE;
__device__ __forceinline__ double2 *vc_buf(int bi) { return q2w_sm + bi * (G * LDVC); }
__device__ __forceinline__ double2 *t_buf(int bi) { return q2w_sm + OFF_T + bi * (G * LDT); }
__device__ __forceinline__ uint64_t *full_bar(int bi) { return reinterpret_cast<uint64_t *>(q2w_sm + OFF_BAR) + bi; }
__device__ __forceinline__ uint64_t *empty_bar(int bi) { return reinterpret_cast<uint64_t *>(q2w_sm + OFF_BAR) + 2 + bi; }

// ---------------------------------------------------------------- producer
__device__ __forceinline__ void q2w_producer(const Q2wArgs &a, int nslab) {
  const int lane = threadIdx.x & 31;
  int64_t cnt = 0;
  for (int sl = 0; sl < nslab; sl++)
    for (int64_t gi = a.ngroups - 1; gi >= 0; gi--) {
      const int64_t i0 = gi * G;
      const int64_t J = (i0 > a.n - 2) ? 0 : (a.n - 2 - i0) / NB + 1;
      const int64_t blk0 = a.first[gi];
      for (int64_t j = 0; j < J; j++, cnt++) {
        const int bi = (int)(cnt & 1);
        if (cnt >= 2) mbar_wait(empty_bar(bi), (unsigned)(((cnt >> 1) + 1) & 1));
        const int nvalid = (int)imax64(0, imin64(G, a.n - 2 - j * NB - i0 + 1));
        if (lane == 0) mbar_arrive_tx(full_bar(bi), (unsigned)(nvalid * NB * 16 + G * G * 16));
        __syncwarp();
        const double2 *v2 = a.V2 + (a.off[j] + i0) * NB;
        if (lane < nvalid) bulk_g2s(vc_buf(bi) + lane * LDVC + PADL, v2 + lane * NB, NB * 16, full_bar(bi));
        bulk_g2s(t_buf(bi) + lane * LDT, a.T2 + (blk0 + j) * G * G + lane * G, G * 16, full_bar(bi));
      }
    }
}

// ---------------------------------------------------------------- consumer
__device__ __forceinline__ void q2w_consumer(const Q2wArgs &a, int frag0, int frag1, int nslab) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2 *Ew = q2w_sm + OFF_E + w * 8 * LDE;
  const LaneEmb le(lane);
  const int kq = (lane & 3) >> 1;
  const unsigned negA = le.a_neg ^ 0x80000000u;   // -V in phase C
  // per-lane shared-memory offsets (in doubles)
  const int offA = 2 * (71 * (lane >> 3) + kq + PADL) + le.a_comp;    // phase A:  V^H  (t = 4mf + lane>>3, q = 2ks + kq)
  const int offC = 2 * (71 * kq + (lane >> 3) + PADL) + le.a_comp;    // phase C:  V    (q = 4f + lane>>3, t = 2ks + kq)
  const int offT = 2 * (kq * LDT + (lane >> 3)) + le.a_comp;          // phase B:  T[ra][kb]
  const int offEB = 2 * (LDE * (lane >> 2) + kq) + (lane & 1);        // E operand layout
  const int rr = lane >> 2;
  const int offEC = 2 * (LDE * 2 * (lane & 3) + (rr >> 1)) + (rr & 1);  // E accumulator layout (col 2(lane&3))
  double *ew = reinterpret_cast<double *>(Ew);
  int64_t cnt = 0;
  for (int sl = 0; sl < nslab; sl++) {
    const int fr = frag0 + sl * NCW + w;
    const bool active = fr < frag1;
    const int64_t c0 = (int64_t)fr * 8;
    const int ncols = active ? (int)imin64(8, a.m - c0) : 0;
    // global column pointers of this lane (accumulator layout: columns 2(lane&3), +1)
    const int cA = 2 * (lane & 3);
    const bool okA0 = cA < ncols, okA1 = cA + 1 < ncols;
    for (int64_t gi = a.ngroups - 1; gi >= 0; gi--) {
      const int64_t i0 = gi * G;
      const int64_t J = (i0 > a.n - 2) ? 0 : (a.n - 2 - i0) / NB + 1;
      int base = 0;   // ring offset: window row q lives in slot (q + base) mod 96
      if (active && J > 0) {
        // group start: whole window rows rs .. rs + 95 (row 95 is padding)
        const int64_t rs = i0 + 1;
        for (int e = lane; e < RING * 8; e += 32) {
          const int q = e % RING, c = e / RING;
          const int64_t row = rs + q;
          const bool ok = q < W && row < a.n && c < ncols;
          cp_async16(&Ew[c * LDE + q], ok ? a.E + row + (c0 + c) * a.lde : a.E, ok);
        }
        cp_async_commit();
      }
      for (int64_t j = 0; j < J; j++, cnt++) {
        const int bi = (int)(cnt & 1);
        const int64_t rs = i0 + 1 + j * NB;
        const bool more = j + 1 < J;
        mbar_wait(full_bar(bi), (unsigned)((cnt >> 1) & 1));
        if (active) {
          cp_async_wait<0>();
          __syncwarp();
          const double *vc = reinterpret_cast<const double *>(vc_buf(bi));
          const double *tt = reinterpret_cast<const double *>(t_buf(bi));
          // chunk c (window rows 32c..32c+31) -> slot base (doubles)
          const int ch0 = 2 * 32 * ((0 + base / 32) % 3), ch1 = 2 * 32 * ((1 + base / 32) % 3),
                    ch2 = 2 * 32 * ((2 + base / 32) % 3);
          // ---------------- phase A: Y = V^H E   (M-fragment mf nonzero on k-steps 2mf .. 2mf+33)
          double y[8][2];
#pragma unroll
          for (int mf = 0; mf < 8; mf++) y[mf][0] = y[mf][1] = 0.0;
#pragma unroll
          for (int ks = 0; ks < 48; ks++) {
            const int ch = ks < 16 ? ch0 : (ks < 32 ? ch1 : ch2);
            const double e = ew[ch + offEB + 4 * (ks & 15)];
#pragma unroll
            for (int mf = 0; mf < 8; mf++)
              if (ks >= 2 * mf && ks <= 2 * mf + 33)
                dmma_nv(y[mf], xsign(vc[offA + 568 * mf + 4 * ks - 0], le.a_neg_conj), e);
          }
          double yb[16];
          acc_to_b<8>(y, yb, lane);
          // ---------------- phase B: Y = T Y   (T upper triangular: k-steps 2mf .. 15)
#pragma unroll
          for (int mf = 0; mf < 8; mf++) {
            y[mf][0] = y[mf][1] = 0.0;
#pragma unroll
            for (int ks = 2 * mf; ks < 16; ks++) dmma_nv(y[mf], xsign(tt[offT + 144 * ks + 8 * mf], le.a_neg), yb[ks]);
          }
          acc_to_b<8>(y, yb, lane);
          // ---------------- phase C: E -= V Y, row groups f (rows 4f..4f+3), k-steps klo(f)..khi(f)
          double *gE = reinterpret_cast<double *>(a.E + rs + (rr >> 1) + (c0 + cA) * a.lde) + (rr & 1);
          const int64_t lde2 = 2 * a.lde;
#pragma unroll
          for (int fb = 0; fb < 24; fb += 4) {
            if (fb == 16 && more) {
              __syncwarp();
              // rows 0..63 are final and stored: refill their slots (and the
              // padding slot) with the next block's rows 95..158
              for (int h = 0; h < 2; h++) {
                const int i = lane + 32 * h;
                int slot = base - 1 + i;
                slot = slot < 0 ? slot + RING : (slot >= RING ? slot - RING : slot);
                const int64_t row = rs + W + i;
#pragma unroll
                for (int c = 0; c < 8; c++) {
                  const bool ok = row < a.n && c < ncols;
                  cp_async16(&Ew[c * LDE + slot], ok ? a.E + row + (c0 + c) * a.lde : a.E, ok);
                }
              }
              cp_async_commit();
            }
            double acc[4][2];
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const int f = fb + u;
              const int ch = f < 8 ? ch0 : (f < 16 ? ch1 : ch2);
              const double *p = ew + ch + offEC + 8 * (f & 7);
              acc[u][0] = p[0];
              acc[u][1] = p[2 * LDE];
            }
#pragma unroll
            for (int ks = 0; ks < 16; ks++) {
#pragma unroll
              for (int u = 0; u < 4; u++) {
                const int f = fb + u;
                const int klo = imax_c(0, 4 * f - 63) >> 1, khi = imin_c(31, 4 * f + 3) >> 1;
                if (ks >= klo && ks <= khi) dmma_nv(acc[u], xsign(vc[offC + 284 * ks + 8 * f], negA), yb[ks]);
              }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const int f = fb + u;
              const int q = 4 * f + (rr >> 1);
              if (f < 16 || !more) {
                if (q < W && rs + q < a.n) {
                  double *g = gE + 8 * f;
                  if (okA0) g[0] = acc[u][0];
                  if (okA1) g[lde2] = acc[u][1];
                }
              } else if (q < W) {
                double *p = ew + ch2 + offEC + 8 * (f & 7);
                p[0] = acc[u][0];
                p[2 * LDE] = acc[u][1];
              }
            }
          }
          if (!more) __threadfence_block();   // the next group re-reads these rows
          base = base + NB >= RING ? base + NB - RING : base + NB;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(bi));
      }
    }
  }
}

__global__ void __launch_bounds__(WT, 1) apply_q2w_kernel(Q2wArgs a, int nslab) {
  // zero the compact V buffers once (their pads are never written again) and the E windows
  for (int e = threadIdx.x; e < OFF_T; e += WT) q2w_sm[e] = czero();
  for (int e = threadIdx.x; e < NCW * 8 * LDE; e += WT) q2w_sm[OFF_E + e] = czero();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; i++) {
      mbar_init(full_bar(i), 1);
      mbar_init(empty_bar(i), NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int F = a.nfr_total, Gd = gridDim.x;
  const int f0 = (int)((int64_t)F * blockIdx.x / Gd), f1 = (int)((int64_t)F * (blockIdx.x + 1) / Gd);
  if ((threadIdx.x >> 5) == NCW) q2w_producer(a, nslab);
  else q2w_consumer(a, f0, f1, nslab);
}

}  // namespace

size_t q2w_smem_bytes() {
  return (size_t)OFF_BAR * sizeof(double2) + 4 * sizeof(uint64_t);
}

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
  const int grid = std::min(ctx.num_sms, a.nfr_total);
  const int per = (a.nfr_total + grid - 1) / grid;
  const int nslab = (per + NCW - 1) / NCW;
  const size_t smem = q2w_smem_bytes();
  static bool attr = false;
  if (!attr) {
    EIG_TRY(ctx.check(cudaFuncSetAttribute(apply_q2w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "q2w attr"));
    attr = true;
  }
  apply_q2w_kernel<<<grid, WT, smem, ctx.stream>>>(a, nslab);
  EIG_TRY(ctx.launched("apply_q2w_kernel"));
  return 0;
}

}  // namespace eig
