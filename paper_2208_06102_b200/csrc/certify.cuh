// certify.cuh -- the Thompson draw of Alg. 1 in single precision with a proof of
// its argmin.
//
// Alg. 1 needs only b = argmin_a theta_a over the survivors, theta_a = fma(sigma_a, z_a, mu_a)
// with z_a the contract's fp64 normal (NC-3/NC-4).  This file computes every theta_a in fp32
// together with an upper bound E_a of |theta~_a - theta_a|; when the smallest interval lies
// strictly below all the others, its arm IS the contract's argmin (a strict inequality between
// the exact fp64 values, so no tie rule is involved) and the fp64 draw is not evaluated.
// Otherwise the kernel falls back to the exact fp64 draw of the contract.  The decision bits
// are therefore the contract's in every case; only the work differs.
//
// The error of the fp32 normal against the contract's fp64 normal is bounded per Box-Muller
// pair:
//   radius  |r~ - r| <= kAlpha r~ + kBeta / r~  -- checked for EVERY 32-bit radius word a by
//           certify_radius_kernel (the fp32 and the contract fp64 evaluation side by side;
//           zeus_sim_certify_bounds, tests/test_gpu_parity.py::test_certified_draw_bounds);
//   angle   |cos~ - cos|, |sin~ - sin| <= kAng  -- checked for every 32-bit angle word b;
// and the remaining steps are single roundings, bounded analytically.
// The fp32 pieces are hardware approximations (MUFU.LG2/RSQ/SIN/COS): their worst case is
// what the exhaustive check measures, which is a proof for the finite input domain.
#pragma once
#include <cstdint>

#include "contract.cuh"

namespace zs {
namespace cert {

// radius bound |r~ - r| <= kAlpha r~ + kBeta / r~ (exhaustively checked)
constexpr float kAlpha = 4.0e-7f;
constexpr float kBeta = 2.5e-7f;
// angle bound: max over b of |cos~ - cos|, |sin~ - sin| (measured 4.33e-7)
constexpr float kAng = 4.5e-7f;
// largest fp32 radius (r <= sqrt(64 ln 2) = 6.6604 for u1 >= 2^-32)
constexpr float kRMax = 6.67f;
// e_z = e_r (1 + 1.2e-6) + r~ (kAng + 2^-24 + 2^-52)(1 + 2^-22): the z0 = r cos, z1 = r sin
// products' rounding in fp32 and fp64 and the cross terms
constexpr float kZr = kAlpha * 1.000002f + 5.2e-7f;
constexpr float kZb = kBeta * 1.000002f;
// theta~ = RN32(sigma32 z~ + mu'32): per-arm error <= sigma32 (e_z + kSig) (1 + 2^-20)
// + kTheta |theta~| + c_trial (the fp32 roundings of sigma, mu - ref and theta; the fp64
// roundings of the contract's theta and of mu - ref)
constexpr float kSig = 1.0e-6f;
constexpr float kTheta = 1.3e-7f;       // > 2^-24 + 2^-24 + 2^-52 + 2^-53, with margin
constexpr float kSigScale = 1.000001f;  // (1 + 2^-20) rounded up

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// fp32 radius of word a and its error bound: r~ and e_r, with r = sqrt(-2 zlog((a+1) 2^-32))
// the contract's (NC-3).  r2 = |lg2 u| 2 ln2 >= +0; rsq = +inf at r2 = 0 makes e_r = +inf.
__device__ __forceinline__ void radius32(uint32_t a, float &r, float &rsq) {
  const float u = fmaf(__uint2float_rn(a), 0x1p-32f, 0x1p-32f);      // (a + 1) 2^-32
  const float r2 = fabsf(lg2_approx(u)) * 1.3862943611198906f;      // -2 ln u
  rsq = rsqrt_approx(r2);
  r = r2 * rsq;
}
__device__ __forceinline__ float radius_err(float r, float rsq) {
  return __fmaf_ru(fminf(r, kRMax), kAlpha, __fmul_ru(rsq, kBeta));
}
// fp32 cos, sin of 2 pi b 2^-32 (the angle word of NC-3): (int)b 2^-32 is the angle in turns
// reduced to [-1/2, 1/2), the same sin and cos
__device__ __forceinline__ void angle32(uint32_t b, float &s, float &c) {
  __sincosf((float)(int)b * 1.4629180792671596e-09f, &s, &c);       // 2 pi 2^-32
}

// One Box-Muller pair in fp32: z0~, z1~, and rsq = 1/r~ for its error bound: for every pair,
// |z~ - z| <= e_z = kZr kRMax + kZb rsq (the r~-dependent term at its largest; +inf at r2 = 0).
__device__ __forceinline__ void normal_pair32(uint32_t a, uint32_t b, float &z0, float &z1, float &rsq) {
  float r, s, c;
  radius32(a, r, rsq);
  angle32(b, s, c);
  z0 = r * c;
  z1 = r * s;
}

// Running argmin over packed keys: arm a's key is theta~_a with its low `bits` mantissa bits
// replaced by a, so one FMNMX carries the arm along (|key - theta~| < 2^bits ulp, charged to
// kTheta); the second-smallest key, the largest sigma and the largest 1/r~ come along.
// Non-survivor slots hold mu' = 3e38, sigma = 0: a finite key above every survivor's.
struct Argmin32 {
  float m1, m2, smax, rsqmax;
  __device__ __forceinline__ void init() {
    m1 = m2 = __int_as_float(0x7f800000);
    smax = 0.0f;
    rsqmax = 0.0f;
  }
  // arms 2k, 2k+1 (index a0, a0 + 1) of one Box-Muller pair
  __device__ __forceinline__ void pair(int a0, float4 ms, float z0, float z1, float rsq, uint32_t keep) {
    const float t0 = fmaf(ms.y, z0, ms.x);
    const float t1 = fmaf(ms.w, z1, ms.z);
    const float k0 = __int_as_float((__float_as_int(t0) & (int)keep) | a0);
    const float k1 = __int_as_float((__float_as_int(t1) & (int)keep) | (a0 + 1));
    const float lo = fminf(k0, k1), hi = fmaxf(k0, k1);
    m2 = fminf(fminf(m2, hi), fmaxf(m1, lo));
    m1 = fminf(m1, lo);
    smax = fmaxf(smax, fmaxf(ms.y, ms.w));
    rsqmax = fmaxf(rsqmax, rsq);
  }
  // the same without the sigma maximum (the caller keeps an upper bound of it, certified_ub)
  __device__ __forceinline__ void pair_nos(int a0, float4 ms, float z0, float z1, float rsq, uint32_t keep) {
    const float t0 = fmaf(ms.y, z0, ms.x);
    const float t1 = fmaf(ms.w, z1, ms.z);
    const float k0 = __int_as_float((__float_as_int(t0) & (int)keep) | a0);
    const float k1 = __int_as_float((__float_as_int(t1) & (int)keep) | (a0 + 1));
    const float lo = fminf(k0, k1), hi = fmaxf(k0, k1);
    m2 = fminf(fminf(m2, hi), fmaxf(m1, lo));
    m1 = fminf(m1, lo);
    rsqmax = fmaxf(rsqmax, rsq);
  }
  // the same with the pair's eligibility bits (arm a0: bit 0, a0 + 1: bit 1): an ineligible
  // arm's theta becomes the non-survivor sentinel 3e38 (f3 / f2v kernels, whose fp32 tables hold
  // every mature arm)
  __device__ __forceinline__ void pair_masked(int a0, float4 ms, float z0, float z1, float rsq,
                                              uint32_t keep, uint32_t two) {
    if (!(two & 1u)) { ms.x = 3.0e38f; ms.y = 0.0f; }
    if (!(two & 2u)) { ms.z = 3.0e38f; ms.w = 0.0f; }
    pair(a0, ms, z0, z1, rsq, keep);
  }
  __device__ __forceinline__ int arg(uint32_t keep) const { return __float_as_int(m1) & (int)~keep; }
  // Is arg() the contract's argmin?  For every other survivor x: key_x >= m2 (distinct arms have
  // distinct keys), and t - kth |t| is increasing in t, so theta_x - ref >= m2 - kth |m2| - S,
  // while theta_b - ref <= m1 + kth |m1| + S, S = smax (e_z + kSig) kSigScale + c_trial,
  // kth = kTheta + 2^(bits-23) (1 + 2^-20).  NaN anywhere fails the test; m2 = +inf (one
  // survivor) passes whenever S is finite.
  __device__ __forceinline__ bool certified(float c_trial, float kth) const {
    return certified_ub(smax, c_trial, kth);
  }
  // with any upper bound sub >= every survivor's sigma32 (a larger bound only widens S)
  __device__ __forceinline__ bool certified_ub(float sub, float c_trial, float kth) const {
    const float ez = __fmaf_ru(rsqmax, kZb, kZr * kRMax * 1.000001f);
    const float S = __fmaf_ru(__fmul_ru(sub, kSigScale), __fadd_ru(ez, kSig), c_trial);
    const float lo2 = (m2 == __int_as_float(0x7f800000)) ? m2 : __fmaf_rd(-kth, fabsf(m2), m2);
    const float hi1 = __fmaf_ru(kth, fabsf(m1), m1);
    return __fsub_rd(lo2, hi1) > __fmul_ru(2.0f, S);
  }
};

// ---- exhaustive checks of the two measured bounds (zeus_sim_certify_bounds)
// out: [0] max over a of |r~ - r| / e_r(a) (the radius bound holds iff <= 1), [1] max r~,
//      [2] max over b of |cos~ - cos|, [3] of |sin~ - sin| (both must be <= kAng);
// as order-preserving bit patterns of non-negative floats (atomicMax on u32)
__global__ void certify_radius_kernel(const double2 *logtab, uint64_t begin, uint64_t n, unsigned *out) {
  __shared__ double2 tab[kLogTab];
  for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) tab[i] = logtab[i];
  __syncthreads();
  float worst = 0.0f, rmax = 0.0f;
  for (uint64_t i = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < begin + n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = (uint32_t)i;
    const double u1 = (double)((unsigned long long)a + 1ull) * 0x1p-32;   // the contract's r
    const double r = sqrt(-2.0 * zlog(u1, tab));
    float rf, rsq;
    radius32(a, rf, rsq);
    const float er = radius_err(rf, rsq);
    // e_r = +inf (r2 = 0: the draw is never certified, its fp32 radius is NaN) bounds nothing
    // to check; otherwise the ratio |r32 - r| / e_r rounded up, NaN counted as a failure
    const double d = fabs((double)rf - r);
    float q = (er == __int_as_float(0x7f800000) || d == 0.0) ? 0.0f : (float)(d / (double)er) * 1.0000002f;
    if (!(q == q)) q = __int_as_float(0x7f800000);
    worst = fmaxf(worst, q);
    if (rf == rf) rmax = fmaxf(rmax, rf);
  }
  atomicMax(out + 0, __float_as_uint(worst));
  atomicMax(out + 1, __float_as_uint(rmax));
}
__global__ void certify_angle_kernel(uint64_t begin, uint64_t n, unsigned *out) {
  float wc = 0.0f, ws = 0.0f;
  for (uint64_t i = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < begin + n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)i;
    double s, c;
    zsincospi_b32(b, s, c);                                            // the contract's angle
    float sf, cf;
    angle32(b, sf, cf);
    // |err| rounded up to fp32
    wc = fmaxf(wc, __double2float_ru(fabs((double)cf - c)));
    ws = fmaxf(ws, __double2float_ru(fabs((double)sf - s)));
  }
  atomicMax(out + 2, __float_as_uint(wc));
  atomicMax(out + 3, __float_as_uint(ws));
}

// [4] max over random (a, b, mu, sigma, ref) of |key~ - (theta - ref)| / E: the composed per-arm
// bound of Argmin32 (|key - theta'| <= sigma32 kSigScale (e_z + kSig) + kth |key| + c_trial at
// the widest key packing, 5 index bits) against the contract's theta = fma(sigma, z, mu) with
// the contract's fp64 normal z (NC-3/NC-4); an empirical check of the analytic composition
// over the regimes the replay meets: ref 1 .. 1e6, |mu - ref| / ref up to 1/2,
// sigma / mu 1e-7 .. 0.3
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void certify_theta_kernel(const double2 *logtab, uint64_t begin, uint64_t n, unsigned *out) {
  __shared__ double2 tab[kLogTab];
  for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) tab[i] = logtab[i];
  __syncthreads();
  const uint32_t keep = ~31u;
  const float kth = kTheta + 0x1p-18f * 1.000001f;
  float worst = 0.0f;
  for (uint64_t i = begin + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < begin + n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h0 = splitmix64(2 * i), h1 = splitmix64(2 * i + 1);
    const uint32_t a = (uint32_t)h0, b = (uint32_t)(h0 >> 32);
    const double u0 = (double)(h1 & 0xfffff) * 0x1p-20, u1 = (double)((h1 >> 20) & 0xfffff) * 0x1p-20;
    const double u2 = (double)(h1 >> 40) * 0x1p-24;
    const double ref = exp10(6.0 * u0);
    const double mu = ref * (1.0 + (u1 - 0.5) * exp10(-6.0 * u2));
    const double sig = mu * exp10(-7.0 + 6.5 * u2 * u1);
    double z0, z1;
    box_muller(a, b, z0, z1, tab);                                     // the contract's normals
    const float c_trial = __double2float_ru(fabs(ref) * 0x1p-52 + 0x1p-120);
    float zf0, zf1, rsq;
    normal_pair32(a, b, zf0, zf1, rsq);
    const float ez = __fmaf_ru(rsq, kZb, kZr * kRMax * 1.000001f);
    const float muf = (float)(mu - ref), sgf = (float)sig;
    const float S = __fmaf_ru(__fmul_ru(sgf, kSigScale), __fadd_ru(ez, kSig), c_trial);
#pragma unroll
    for (int arm = 0; arm < 2; ++arm) {
      const double th = fma(sig, arm ? z1 : z0, mu);                   // contract theta (NC-4)
      const float t32 = fmaf(sgf, arm ? zf1 : zf0, muf);
      const float key = __int_as_float((__float_as_int(t32) & (int)keep) | 31);
      const float E = __fmaf_ru(kth, fabsf(key), S);
      const double hi = th - ref, bb = hi - th;                          // two-sum of th - ref
      const double lo = (th - (hi - bb)) + (-ref - bb);
      const double d = fabs(((double)key - hi) - lo);
      // S = +inf (a pair with r2 = 0: rsq = +inf) is never certified: nothing to check
      const float q = (S == __int_as_float(0x7f800000)) ? 0.0f : (float)(d / (double)E) * 1.000001f;
      worst = fmaxf(worst, (q == q) ? q : __int_as_float(0x7f800000));
    }
  }
  atomicMax(out + 4, __float_as_uint(worst));
}

}  // namespace cert
}  // namespace zs
