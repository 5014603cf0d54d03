// contract.cuh -- device side of the numerics contract (NC-3/NC-4).
//
// Philox4x32-10 (Salmon et al., SC'11), the (0,1] / [0,1) uniform
// construction, and the contract transcendentals: zlog from fdlibm's published
// e_log.c, zsincospi as an exact integer reduction plus the Taylor series of
// sin/cos(pi f), using only IEEE + - * / sqrt and explicit fma.  This file is compiled with --fmad=false so
// every a*b+c below is two roundings unless written fma(); it is written
// independently of the CPU oracle and shares nothing with it.
#pragma once
#include <cstdint>

namespace zs {

// fp64 coefficients live in the constant bank so DFMA/DMUL take them as c[][]
// operands instead of materialising 64-bit immediates with UMOV pairs in the loop.
#ifdef ZS_IMMEDIATE_CONSTANTS
#define ZS_C(name, value) constexpr double name = value
#else
#define ZS_C(name, value) __constant__ double name = value
#endif
namespace cst {
ZS_C(kLn2Hi, 6.93147180369123816490e-01);
ZS_C(kLn2Lo, 1.90821492927058770002e-10);
ZS_C(kLg1, 6.666666666666735130e-01);
ZS_C(kLg2, 3.999999999940941908e-01);
ZS_C(kLg3, 2.857142874366239149e-01);
ZS_C(kLg4, 2.222219843214978396e-01);
ZS_C(kLg5, 1.818357216161805012e-01);
ZS_C(kLg6, 1.531383769920937332e-01);
ZS_C(kLg7, 1.479819860511658591e-01);
ZS_C(kPi, 0x1.921fb54442d18p+1);
ZS_C(kPiLo, 0x1.1a62633145c07p-53);
ZS_C(kS1, -0x1.4abbce625be53p+2);
ZS_C(kS2, 0x1.466bc6775aae2p+1);
ZS_C(kS3, -0x1.32d2cce62bd86p-1);
ZS_C(kS4, 0x1.50783487ee782p-4);
ZS_C(kS5, -0x1.e3074fde8871fp-8);
ZS_C(kS6, 0x1.e8f434d018d63p-12);
ZS_C(kS7, -0x1.6fadb9f155744p-16);
ZS_C(kS8, 0x1.aaec32af93359p-21);
ZS_C(kC1, -0x1.3bd3cc9be45dep+2);
ZS_C(kC2, 0x1.03c1f081b5ac4p+2);
ZS_C(kC3, -0x1.55d3c7e3cbffap+0);
ZS_C(kC4, 0x1.e1f506891babbp-3);
ZS_C(kC5, -0x1.a6d1f2a204a8cp-6);
ZS_C(kC6, 0x1.f9d38a3763cc3p-10);
ZS_C(kC7, -0x1.b6e24f44b128fp-14);
ZS_C(kC8, 0x1.20c62c2f2d7f5p-18);
ZS_C(kC9, -0x1.2a0c591af8314p-23);
ZS_C(kTwoM51, 0x1p-51);
ZS_C(kL3, 1.0 / 3.0);   // log1p Taylor coefficients, rounded to nearest
ZS_C(kL5, 0.2);
ZS_C(kL6, -1.0 / 6.0);
ZS_C(kL7, 1.0 / 7.0);
ZS_C(kVarFloor, 1e-12);
}  // namespace cst

// ------------------------------------------------------------ Philox4x32-10
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
  constexpr uint32_t kWeyl0 = 0x9E3779B9u, kWeyl1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kMul0, c.x), lo0 = kMul0 * c.x;
    const uint32_t hi1 = __umulhi(kMul1, c.z), lo1 = kMul1 * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += kWeyl0;
    k1 += kWeyl1;
  }
  return c;
}

// The 20 round keys of one Philox key, precomputed on the host and passed in the kernel
// parameters: the rounds then read them as constant-bank operands (LOP3 R, R, c[][], R)
// instead of recomputing k + r W with a uniform add per round.
struct RoundKeys { uint32_t k0[10], k1[10]; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, const RoundKeys &rk) {
  constexpr uint32_t kMul0 = 0xD2511F53u, kMul1 = 0xCD9E8D57u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kMul0, c.x), lo0 = kMul0 * c.x;
    const uint32_t hi1 = __umulhi(kMul1, c.z), lo1 = kMul1 * c.z;
    c = U4{hi1 ^ c.y ^ rk.k0[r], lo1, hi0 ^ c.w ^ rk.k1[r], lo0};
  }
  return c;
}

// ------------------------------------------------------------ zlog
// fdlibm __ieee754_log for positive normal x, one formula for every f (the
// shortcut branches folded in), polynomial halves by explicit fma (NC-3).
__device__ __forceinline__ double zlog_fdlibm(double x) {
  using namespace cst;
  int hx = __double2hiint(x);
  const int lx = __double2loint(x);
  int k = (hx >> 20) - 1023;
  hx &= 0x000fffff;
  const int i0 = (hx + 0x95f64) & 0x100000;
  const double xn = __hiloint2double(hx | (i0 ^ 0x3ff00000), lx);
  k += (i0 >> 20);
  const double f = xn - 1.0;
  const double hfsq = 0.5 * f * f;
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double w = z * z;
  const double t1 = w * fma(w, fma(w, kLg6, kLg4), kLg2);
  const double t2 = z * fma(w, fma(w, fma(w, kLg7, kLg5), kLg3), kLg1);
  const double R = t2 + t1;
  const double dk = (double)k;
  return dk * kLn2Hi - ((hfsq - (s * (hfsq + R) + dk * kLn2Lo)) - f);
}

// The sampler's log (NC-3): table-driven, no division per normal.  tab[j + 37] =
// (invc_j, logc_j) for j in [-37, 53]: c_j = 1 + j/128, invc_j = 1/c_j (IEEE),
// logc_j = -zlog_fdlibm(invc_j) (built once on the device by log_table_kernel).
// x = 2^k m, m in [sqrt2/2, sqrt2); j = round(128 (m - 1)); r = fma(m, invc_j, -1);
// log x = (k ln2_hi + logc_j) + (r + (k ln2_lo + r^2 q(r))), q the log1p Taylor tail to r^7.
constexpr int kLogTab = 91;
__device__ __forceinline__ double zlog(double x, const double2 *__restrict__ tab) {
  using namespace cst;
  int hx = __double2hiint(x);
  const int lx = __double2loint(x);
  int k = (hx >> 20) - 1023;
  hx &= 0x000fffff;
  const int i0 = (hx + 0x95f64) & 0x100000;
  const double m = __hiloint2double(hx | (i0 ^ 0x3ff00000), lx);
  k += (i0 >> 20);
  const double f = m - 1.0;                                  // exact
  const int j = __double2int_rn(f * 128.0);                  // round half to even
  const double2 e = tab[j + 37];
  const double r = fma(m, e.x, -1.0);
  double q = fma(r, kL7, kL6);
  q = fma(r, q, kL5);
  q = fma(r, q, -0.25);
  q = fma(r, q, kL3);
  q = fma(r, q, -0.5);
  const double dk = (double)k;
  const double hi = fma(dk, kLn2Hi, e.y);
  const double lo = fma(dk, kLn2Lo, (r * r) * q);
  return hi + (r + lo);
}

// ------------------------------------------------------------ sin / cos of pi*m/2^51
// Exact integer reduction to n/2 + f, |f| <= 1/4; Taylor series of sin(pi f),
// cos(pi f) (coefficients rounded to nearest double) by fma Horner; pi*f as a
// double-double in the sine's leading term (NC-3).
// sin(pi f), cos(pi f) for |f| <= 1/4, then the quadrant rotation by n (mod 4).
__device__ __forceinline__ void sincospi_reduced(double f, int n, double &s, double &c) {
  using namespace cst;
  const double f2 = f * f;
  double ps = fma(f2, kS8, kS7);
  ps = fma(f2, ps, kS6);
  ps = fma(f2, ps, kS5);
  ps = fma(f2, ps, kS4);
  ps = fma(f2, ps, kS3);
  ps = fma(f2, ps, kS2);
  ps = fma(f2, ps, kS1);
  const double hi = f * kPi;
  const double lo = fma(f, kPiLo, fma(f, kPi, -hi));
  const double sf = hi + fma(f * f2, ps, lo);
  double pc = fma(f2, kC9, kC8);
  pc = fma(f2, pc, kC7);
  pc = fma(f2, pc, kC6);
  pc = fma(f2, pc, kC5);
  pc = fma(f2, pc, kC4);
  pc = fma(f2, pc, kC3);
  pc = fma(f2, pc, kC2);
  pc = fma(f2, pc, kC1);
  const double cf = fma(f2, pc, 1.0);
  const int q = n & 3;
  const double ss = (q & 1) ? cf : sf;                     // q=0: sf  1: cf  2: -sf  3: -cf
  const double cc = (q & 1) ? sf : cf;                     // q=0: cf  1: -sf 2: -cf  3: sf
  // the signs by flipping bit 63 (exact, and -x of +0 is -0 as the unary minus gives)
  s = __longlong_as_double(__double_as_longlong(ss) ^ ((long long)(q & 2) << 62));
  c = __longlong_as_double(__double_as_longlong(cc) ^ ((long long)((q + 1) & 2) << 62));
}

// sin(pi m / 2^51), cos(pi m / 2^51) for 0 <= m < 2^52: n = round(m / 2^50),
// f = (m - n 2^50) 2^-51 exactly, |f| <= 1/4.
__device__ __forceinline__ void zsincospi(uint64_t m, double &s, double &c) {
  const int64_t n = (int64_t)((m + (1ull << 49)) >> 50);
  const int64_t j = (int64_t)m - (n << 50);
  sincospi_reduced((double)j * cst::kTwoM51, (int)n, s, c);
}

// The same for m = b 2^20 (v = b 2^-32, the sampler's angle), in 32-bit integers:
// n = round(b / 2^30), f = (b - n 2^30) 2^-31 -- the identical f and n, hence the same bits.
__device__ __forceinline__ void zsincospi_b32(uint32_t b, double &s, double &c) {
  const uint32_t n = (uint32_t)(((uint64_t)b + (1u << 29)) >> 30);
  const int jb = (int)(b - (n << 30));
  sincospi_reduced((double)jb * 0x1p-31, (int)n, s, c);
}

// The Philox block of arm quad q = k >> 1 of `trial` at recurrence t (NC-3): it feeds two
// Box-Muller pairs, k even -> words (x, y), k odd -> words (z, w).
__device__ __forceinline__ U4 pair_block(uint32_t key0, uint32_t key1, int64_t trial, int t, int q) {
  return philox4x32_10(U4{(uint32_t)t, 0x01000000u | (uint32_t)q, (uint32_t)trial,
                          (uint32_t)((uint64_t)trial >> 32)}, key0, key1);
}
__device__ __forceinline__ U4 pair_block(const RoundKeys &rk, int64_t trial, int t, int q) {
  return philox4x32_10(U4{(uint32_t)t, 0x01000000u | (uint32_t)q, (uint32_t)trial,
                          (uint32_t)((uint64_t)trial >> 32)}, rk);
}

// Box-Muller from two 32-bit words: u1 = (a + 1) 2^-32 in (0,1], v = b 2^-32 in [0,1);
// z0 = r cos(2 pi v), z1 = r sin(2 pi v), r = sqrt(-2 log u1) (NC-3).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, double &z0, double &z1,
                                           const double2 *__restrict__ logtab) {
  const double u1 = (double)((unsigned long long)a + 1ull) * 0x1p-32;   // exact
  const double r = sqrt(-2.0 * zlog(u1, logtab));
  double s, c;
  zsincospi_b32(b, s, c);                                              // 2 pi v, v = b 2^-32
  z0 = r * c;
  z1 = r * s;
}

// Box-Muller pair for arms (2k, 2k+1) of `trial` at recurrence t (NC-3).
__device__ __forceinline__ void normal_pair(uint32_t key0, uint32_t key1, int64_t trial, int t,
                                            int k, double &z0, double &z1,
                                            const double2 *__restrict__ logtab) {
  const U4 x = pair_block(key0, key1, trial, t, k >> 1);
  if (k & 1) box_muller(x.z, x.w, z0, z1, logtab);
  else box_muller(x.x, x.y, z0, z1, logtab);
}

// log_table_kernel: the zlog table (one block; entries j = -37..53)
__global__ void log_table_kernel(double2 *tab) {
  const int i = threadIdx.x;
  if (i >= kLogTab) return;
  const double c = 1.0 + (double)(i - 37) / 128.0;
  const double invc = 1.0 / c;
  tab[i] = make_double2(invc, -zlog_fdlibm(invc));
}

// Replica draws (NC-3): one Philox block per four recurrences, counter
// (t >> 2, 2 << 24, trial); recurrence t uses word t & 3 and replica = (word * K) >> 32.
__device__ __forceinline__ U4 replica_words(uint32_t key0, uint32_t key1, int64_t trial, int t) {
  return philox4x32_10(U4{(uint32_t)t >> 2, 0x02000000u, (uint32_t)trial,
                          (uint32_t)((uint64_t)trial >> 32)}, key0, key1);
}
__device__ __forceinline__ U4 replica_words(const RoundKeys &rk, int64_t trial, int t) {
  return philox4x32_10(U4{(uint32_t)t >> 2, 0x02000000u, (uint32_t)trial,
                          (uint32_t)((uint64_t)trial >> 32)}, rk);
}
__device__ __forceinline__ uint32_t pick_word(const U4 &w, int t) {
  const uint32_t lo = (t & 1) ? w.y : w.x, hi = (t & 1) ? w.w : w.z;   // selects, no branch
  return (t & 2) ? hi : lo;
}

}  // namespace zs
