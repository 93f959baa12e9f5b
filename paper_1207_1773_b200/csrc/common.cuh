// common.cuh — shared device helpers for the sm_100a kernels.
//
// Complex-FP64 on the DMMA pipe by real embedding: a complex M x K operand
// op(A) is used as the real 2M x 2K matrix whose 2x2 block (i, p) is
//   [[Re a, -Im a], [Im a, Re a]],   a = op(A)[i, p],
// and a complex K x N operand B (interleaved, column-major) IS the real
// 2K x N matrix with rows (Re b_p, Im b_p).  Then the interleaved complex
// C = op(A) op(B) is exactly the real product C~ = A~ B~, so every complex
// multiply-add costs one 4-real-MAC slice of a DMMA.8x8x4, the same count as
// the classical 4M decomposition, with no operand splitting and the
// accumulator already in interleaved layout.
//
// mma.sync.m8n8k4.f64 fragments (PTX ISA): lane = 4*g + t (g = lane>>2, t = lane&3)
//   A (8x4, row): a0 = A[g][t];  B (4x8, col): b0 = B[t][g];
//   C (8x8):      c0 = C[g][2t], c1 = C[g][2t+1].
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace eig {

constexpr int kSMs = 148;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// flip the sign of a double by xor-ing its sign bit (integer pipe, not FP64)
__device__ __forceinline__ double xsign(double v, unsigned mask) {
  return __hiloint2double(__double2hiint(v) ^ (int)mask, __double2loint(v));
}

// Per-lane constants of the real embedding.
//  A fragment: real row parity rp = (lane>>2)&1, real col parity cp = lane&1.
//    component = rp ^ cp (0 re, 1 im); negative iff (!rp && cp) [plain] or (rp && !cp) [conj].
//  B fragment: component = lane&1; negative iff component == 1 and conj.
struct LaneEmb {
  int a_comp;          // 0/1 component index for A fragments
  unsigned a_neg;      // sign mask for A (plain)
  unsigned a_neg_conj; // sign mask for A (conjugated operand)
  int b_comp;
  unsigned b_neg_conj; // sign mask for B (conjugated operand); plain B never negates
  __device__ __forceinline__ LaneEmb(int lane) {
    int rp = (lane >> 2) & 1, cp = lane & 1;
    a_comp = rp ^ cp;
    a_neg = (!rp && cp) ? 0x80000000u : 0u;
    a_neg_conj = (rp && !cp) ? 0x80000000u : 0u;
    b_comp = lane & 1;
    b_neg_conj = (lane & 1) ? 0x80000000u : 0u;
  }
};

// ------------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------------------- complex helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 czero() { return make_double2(0.0, 0.0); }

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

// ------------------------------------------------------------- zlarfg with scaled norms
// LAPACK zlarfg (reading R1) forms ||x|| with the scaled dznrm2,
// ||(alpha, x)|| with dlapy3 and rescales by 1/safmin while |beta| < safmin,
// so the reflector is well defined for entries near both ends of the binary64
// range.  The device kernels get the same effect with exact power-of-two
// scaling: the sums of squares / dot products are formed from x * 2^-Es
// (Es = exponent of max |x| of the rows a thread block owns, combined across
// blocks by a running rescale), and beta/tau are formed from alpha and the
// norm both scaled by 2^-Ep, Ep = max(Es, exponent of alpha).  Power-of-two
// scaling commutes with rounding, so for inputs away from the range ends the
// result is bitwise the unscaled formula; at the ends nothing over- or
// underflows.
constexpr int kExpZero = -100000;   // exponent tag of an all-zero vector

// Magnitude key of x: high word of |x|, with bit 0 set if the low word is
// nonzero.  Unsigned order of keys = order of |x| at exponent granularity,
// which is all the scale choice needs; integer max (and __reduce_max_sync
// across a warp) keeps it off the FP64 pipe.
__device__ __forceinline__ unsigned mag_key(double x) {
  return ((unsigned)__double2hiint(x) & 0x7fffffffu) | (__double2loint(x) != 0 ? 1u : 0u);
}
__device__ __forceinline__ unsigned mag_key2(double2 z) { return max(mag_key(z.x), mag_key(z.y)); }
// binary exponent of the magnitude with key k, clamped to >= -1022 so that
// 2^-e is a normal number (subnormal entries times 2^1022 stay exact);
// kExpZero for k == 0
__device__ __forceinline__ int exp_of_key(unsigned k) {
  if (k == 0) return kExpZero;
  const int e = (int)(k >> 20) - 1023;
  return e < -1022 ? -1022 : e;
}
// 2^k for k <= 1023 (subnormal powers for -1074 <= k < -1022, 0 below), by
// its bits: multiplying by it is exact unless the product leaves the range
__device__ __forceinline__ double pow2i(int k) {
  const double nrm = __hiloint2double((max(k, -1022) + 1023) << 20, 0);
  const double sub = __longlong_as_double(1LL << max(k + 1074, 0));
  return k >= -1022 ? nrm : (k >= -1074 ? sub : 0.0);
}

struct Refl {
  double beta;     // real (unscaled)
  double2 tau;
  double xs;       // 2^-Ep
  double2 vs;      // 2^Ep / (alpha - beta):  v_r = (x_r xs) vs = x_r / (alpha - beta)
                   // (1/(alpha-beta) alone overflows for tiny columns, LAPACK's safmin case)
  double2 fscale;  // conj(1/(alpha-beta)) s = conj(fscale) s~  (s~ = s 2^-Es)
};
// alpha unscaled; xn2s = sum |x_r 2^-Es|^2; Es = kExpZero iff x == 0.
__device__ __forceinline__ Refl zlarfg_scaled(double2 alpha, double xn2s, int Es) {
  Refl o;
  if ((Es == kExpZero || xn2s == 0.0) && alpha.y == 0.0) {
    o.beta = alpha.x;
    o.tau = make_double2(0.0, 0.0);
    o.xs = 1.0;
    o.vs = o.fscale = make_double2(0.0, 0.0);
    return o;
  }
  const int Ea = exp_of_key(mag_key2(alpha));
  const int Ep = Es > Ea ? Es : Ea;              // in [-1022, 1023]
  const double ia = pow2i(-Ep);
  const double ar = alpha.x * ia, ai = alpha.y * ia;
  const double xn = xn2s * pow2i(2 * (Es - Ep));  // 0 for Es = kExpZero
  const double b = -copysign(sqrt(ar * ar + ai * ai + xn), ar);
  o.tau = make_double2((b - ar) / b, -ai / b);
  const double dx = ar - b, dy = ai, dd = dx * dx + dy * dy;
  const double sx = dx / dd, sy = -dy / dd;   // 1 / (alpha - beta) in units of 2^Ep
  o.beta = b * pow2i(Ep);
  o.xs = ia;
  o.vs = make_double2(sx, sy);
  const double fs = pow2i(Es - Ep);             // 0 for Es = kExpZero
  o.fscale = make_double2(sx * fs, sy * fs);
  return o;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  return v;
}

}  // namespace eig
