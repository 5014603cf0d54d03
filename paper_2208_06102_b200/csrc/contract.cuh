// contract.cuh -- device side of the numerics contract (NC-3/NC-4).
//
// Philox4x32-10 (Salmon et al., SC'11), the (0,1] / [0,1) uniform
// construction, and the contract transcendentals zlog / zsincospi written
// from fdlibm's published e_log.c, k_sin.c and k_cos.c using only IEEE
// + - * / sqrt and explicit fma.  This file is compiled with --fmad=false so
// every a*b+c below is two roundings unless written fma(); it is written
// independently of the CPU oracle and shares nothing with it.
#pragma once
#include <cstdint>

namespace zs {

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

// ------------------------------------------------------------ zlog
// fdlibm __ieee754_log for positive normal x; the |f|<2^-20 and k==0
// shortcuts are folded into the general formulas (NC-3).
__device__ __forceinline__ double zlog(double x) {
  constexpr double kLn2Hi = 6.93147180369123816490e-01;
  constexpr double kLn2Lo = 1.90821492927058770002e-10;
  constexpr double kLg1 = 6.666666666666735130e-01;
  constexpr double kLg2 = 3.999999999940941908e-01;
  constexpr double kLg3 = 2.857142874366239149e-01;
  constexpr double kLg4 = 2.222219843214978396e-01;
  constexpr double kLg5 = 1.818357216161805012e-01;
  constexpr double kLg6 = 1.531383769920937332e-01;
  constexpr double kLg7 = 1.479819860511658591e-01;
  int hx = __double2hiint(x);
  const int lx = __double2loint(x);
  int k = (hx >> 20) - 1023;
  hx &= 0x000fffff;
  const int i0 = (hx + 0x95f64) & 0x100000;
  const double xn = __hiloint2double(hx | (i0 ^ 0x3ff00000), lx);
  k += (i0 >> 20);
  const double f = xn - 1.0;
  const double s = f / (2.0 + f);
  const double dk = (double)k;
  const double z = s * s;
  const double w = z * z;
  const double t1 = w * (kLg2 + w * (kLg4 + w * kLg6));
  const double t2 = z * (kLg1 + w * (kLg3 + w * (kLg5 + w * kLg7)));
  const int sel = (hx - 0x6147a) | (0x6b851 - hx);
  const double R = t2 + t1;
  if (sel > 0) {
    const double hfsq = 0.5 * f * f;
    return dk * kLn2Hi - ((hfsq - (s * (hfsq + R) + dk * kLn2Lo)) - f);
  }
  return dk * kLn2Hi - ((s * (f - R) - dk * kLn2Lo) - f);
}

// ------------------------------------------------------------ sin / cos kernels (|x| <= pi/4)
__device__ __forceinline__ double ksin(double x, double y) {
  constexpr double kS1 = -1.66666666666666324348e-01;
  constexpr double kS2 = 8.33333333332248946124e-03;
  constexpr double kS3 = -1.98412698298579493134e-04;
  constexpr double kS4 = 2.75573137070700676789e-06;
  constexpr double kS5 = -2.50507602534068634195e-08;
  constexpr double kS6 = 1.58969099521155010221e-10;
  const double z = x * x;
  const double v = z * x;
  const double r = kS2 + z * (kS3 + z * (kS4 + z * (kS5 + z * kS6)));
  return x - ((z * (0.5 * y - v * r) - y) - v * kS1);
}

__device__ __forceinline__ double kcos(double x, double y) {
  constexpr double kC1 = 4.16666666666666019037e-02;
  constexpr double kC2 = -1.38888888888741095749e-03;
  constexpr double kC3 = 2.48015872894767294178e-05;
  constexpr double kC4 = -2.75573143513906633035e-07;
  constexpr double kC5 = 2.08757232129817482790e-09;
  constexpr double kC6 = -1.13596475577881948265e-11;
  const int ix = __double2hiint(x) & 0x7fffffff;
  const double z = x * x;
  const double r = z * (kC1 + z * (kC2 + z * (kC3 + z * (kC4 + z * (kC5 + z * kC6)))));
  if (ix < 0x3FD33333) return 1.0 - (0.5 * z - (z * r - x * y));
  const double qx = (ix > 0x3fe90000) ? 0.28125 : __hiloint2double(ix - 0x00200000, 0);
  const double hz = 0.5 * z - qx;
  const double a = 1.0 - qx;
  return a - (hz - (z * r - x * y));
}

// sin(pi*m/2^51), cos(pi*m/2^51) for 0 <= m < 2^52: exact integer reduction to
// n/2 + f, |f| <= 1/4, pi*f as a double-double.
__device__ __forceinline__ void zsincospi(uint64_t m, double &s, double &c) {
  constexpr double kPi = 3.14159265358979311600e+00;
  constexpr double kPiLo = 1.22464679914735320717e-16;
  const int64_t n = (int64_t)((m + (1ull << 49)) >> 50);
  const int64_t j = (int64_t)m - (n << 50);
  const double f = (double)j * 4.44089209850062616169e-16;   // 2^-51
  const double a = f * kPi;
  const double alo = fma(f, kPi, -a) + f * kPiLo;
  const double sf = ksin(a, alo);
  const double cf = kcos(a, alo);
  const int q = (int)(n & 3);
  const double ss = (q & 1) ? cf : sf;
  const double cc = (q & 1) ? sf : cf;
  s = (q & 2) ? -ss : ss;                 // q=0: sf  1: cf  2: -sf  3: -cf
  c = ((q + 1) & 2) ? -cc : cc;           // q=0: cf  1: -sf 2: -cf  3: sf
}

// Box-Muller pair for arms (2k, 2k+1) of `trial` at recurrence t (NC-3).
__device__ __forceinline__ void normal_pair(uint32_t key0, uint32_t key1, int64_t trial, int t,
                                            int k, double &z0, double &z1) {
  const U4 x = philox4x32_10(U4{(uint32_t)t, 0x01000000u | (uint32_t)k, (uint32_t)trial,
                                (uint32_t)((uint64_t)trial >> 32)}, key0, key1);
  const uint64_t w0 = ((uint64_t)x.y << 32) | x.x;
  const uint64_t w1 = ((uint64_t)x.w << 32) | x.z;
  const double u1 = 2.0 - __longlong_as_double((long long)(0x3FF0000000000000ull | (w0 >> 12)));
  const double r = sqrt(-2.0 * zlog(u1));
  double s, c;
  zsincospi(w1 >> 12, s, c);
  z0 = r * c;
  z1 = r * s;
}

// Replica index of the run replayed at (trial, t) (NC-3).
__device__ __forceinline__ uint32_t replica(uint32_t key0, uint32_t key1, int64_t trial, int t,
                                            uint32_t K) {
  const U4 x = philox4x32_10(U4{(uint32_t)t, 0x02000000u, (uint32_t)trial,
                                (uint32_t)((uint64_t)trial >> 32)}, key0, key1);
  return __umulhi(x.x, K);
}

}  // namespace zs
