// oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// A plain CPU replay of Zeus's batch-size / power-limit optimiser, one
// trial at a time, in the order the paper states it:
//   step 1  power-limit optimiser, Eq. 7, §4.2
//   step 2  pruning (Alg. 3) then Gaussian Thompson
//           sampling (Alg. 1)
//   step 3  trace lookup: the training trace
//   step 4  early stopping at β·min_t C_t and Observe (Alg. 2,
//           P:L494-506, window P:L655)
// Numerics follow the contract NC-1..NC-9 of DESIGN.md §4 literally:
// compiled with -O2 -ffp-contract=off, every fma written out, no libm
// transcendental is ever called (zlog / zsincospi below are the contract
// functions, written from fdlibm's published e_log.c / k_sin.c / k_cos.c).
//
// This file shares nothing with the CUDA path.  Nothing in it is tuned.

#include "oracle.h"

#include <cmath>
#include <cstring>
#include <deque>
#include <limits>
#include <string>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------- bits
double bits_to_double(uint64_t u) { double d; std::memcpy(&d, &u, 8); return d; }
uint64_t double_to_bits(double d) { uint64_t u; std::memcpy(&u, &d, 8); return u; }
int32_t high_word(double d) { return (int32_t)(double_to_bits(d) >> 32); }
double with_high_word(double d, int32_t hi) {
  uint64_t u = double_to_bits(d);
  u = (u & 0xffffffffULL) | ((uint64_t)(uint32_t)hi << 32);
  return bits_to_double(u);
}

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al., "Parallel random numbers: as easy as 1, 2, 3" (SC'11);
// multipliers and Weyl constants as published there (NC-3).
void philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
  uint32_t k[2] = {key_in[0], key_in[1]};
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k[0] += W0; k[1] += W1; }
    uint64_t p0 = (uint64_t)M0 * c[0];
    uint64_t p1 = (uint64_t)M1 * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
  }
  out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

// ---------------------------------------------------------------- zlog
// fdlibm e_log.c (__ieee754_log) for a positive normal x (NC-3): x = 2^k (1+f),
// s = f/(2+f), R(z) the Lg1..Lg7 minimax polynomial, then
// log x = k*ln2_hi - ((hfsq - (s*(hfsq+R) + k*ln2_lo)) - f).  fdlibm's shortcut
// branches (|f| < 2^-20, k == 0, and the alternative form used near sqrt(2)/2..
// sqrt(2) boundaries) are all folded into this one formula, and the two
// polynomial halves are evaluated with explicit fma.
double zlog_fdlibm(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;  // 3fe62e42 fee00000
  const double ln2_lo = 1.90821492927058770002e-10;  // 3dea39ef 35793c76
  const double Lg1 = 6.666666666666735130e-01;       // 3FE55555 55555593
  const double Lg2 = 3.999999999940941908e-01;       // 3FD99999 9997FA04
  const double Lg3 = 2.857142874366239149e-01;       // 3FD24924 94229359
  const double Lg4 = 2.222219843214978396e-01;       // 3FCC71C5 1D8E78AF
  const double Lg5 = 1.818357216161805012e-01;       // 3FC74664 96CB03DE
  const double Lg6 = 1.531383769920937332e-01;       // 3FC39A09 D078C69F
  const double Lg7 = 1.479819860511658591e-01;       // 3FC2F112 DF3E5244
  int32_t hx = high_word(x);
  int32_t k = (hx >> 20) - 1023;
  hx &= 0x000fffff;
  int32_t i = (hx + 0x95f64) & 0x100000;
  x = with_high_word(x, hx | (i ^ 0x3ff00000));   // normalise x or x/2
  k += (i >> 20);
  double f = x - 1.0;
  double hfsq = 0.5 * f * f;
  double s = f / (2.0 + f);
  double z = s * s;
  double w = z * z;
  double t1 = w * std::fma(w, std::fma(w, Lg6, Lg4), Lg2);
  double t2 = z * std::fma(w, std::fma(w, std::fma(w, Lg7, Lg5), Lg3), Lg1);
  double R = t2 + t1;
  double dk = (double)k;
  return dk * ln2_hi - ((hfsq - (s * (hfsq + R) + dk * ln2_lo)) - f);
}

// The sampler's log (NC-3): table-driven, no division on the per-normal path.
// x = 2^k m with m in [sqrt2/2, sqrt2) (fdlibm's normalisation), j = round(128 (m - 1)),
// c_j = 1 + j/128, invc_j = 1/c_j (IEEE), logc_j = -zlog_fdlibm(invc_j) = log(1/invc_j);
// r = fma(m, invc_j, -1) (|r| < 0.0056), log1p(r) by its Taylor series to r^7 (truncation
// < 2e-19 relative), log x = (k ln2_hi + logc_j) + (r + (k ln2_lo + r^2 q(r))).
struct LogTable {
  double invc[91], logc[91];
  LogTable() {
    for (int j = -37; j <= 53; ++j) {
      const double c = 1.0 + (double)j / 128.0;
      invc[j + 37] = 1.0 / c;
      logc[j + 37] = -zlog_fdlibm(invc[j + 37]);
    }
  }
};

double zlog(double x) {
  static const LogTable T;
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double C3 = 1.0 / 3.0, C5 = 0.2, C6 = -1.0 / 6.0, C7 = 1.0 / 7.0;
  int32_t hx = high_word(x);
  int32_t k = (hx >> 20) - 1023;
  hx &= 0x000fffff;
  int32_t i = (hx + 0x95f64) & 0x100000;
  const double m = with_high_word(x, hx | (i ^ 0x3ff00000));
  k += (i >> 20);
  const double f = m - 1.0;                                  // exact
  const int j = (int)std::nearbyint(f * 128.0);              // round half to even
  const double r = std::fma(m, T.invc[j + 37], -1.0);
  double q = std::fma(r, C7, C6);
  q = std::fma(r, q, C5);
  q = std::fma(r, q, -0.25);
  q = std::fma(r, q, C3);
  q = std::fma(r, q, -0.5);
  const double dk = (double)k;
  const double hi = std::fma(dk, ln2_hi, T.logc[j + 37]);
  const double lo = std::fma(dk, ln2_lo, (r * r) * q);
  return hi + (r + lo);
}

// ---------------------------------------------------------------- sin / cos of pi*x
// sin(pi*x), cos(pi*x) for x = m / 2^51, 0 <= m < 2^52 (x = 2v, v in [0,1)), NC-3:
// exact integer reduction x = n/2 + f with |f| <= 1/4, then the Taylor series of
// sin(pi f) and cos(pi f) (coefficients (-1)^k pi^(2k+1)/(2k+1)! and
// (-1)^k pi^(2k)/(2k)!, each rounded to the nearest double; truncation error
// < 1e-19 at |f| = 1/4) by explicit-fma Horner, with pi*f carried as a
// double-double in the sine's leading term.
void zsincospi(uint64_t m, double *s_out, double *c_out) {
  const double PI = 0x1.921fb54442d18p+1;
  const double PI_LO = 0x1.1a62633145c07p-53;
  const double S1 = -0x1.4abbce625be53p+2, S2 = 0x1.466bc6775aae2p+1;
  const double S3 = -0x1.32d2cce62bd86p-1, S4 = 0x1.50783487ee782p-4;
  const double S5 = -0x1.e3074fde8871fp-8, S6 = 0x1.e8f434d018d63p-12;
  const double S7 = -0x1.6fadb9f155744p-16, S8 = 0x1.aaec32af93359p-21;
  const double C1 = -0x1.3bd3cc9be45dep+2, C2 = 0x1.03c1f081b5ac4p+2;
  const double C3 = -0x1.55d3c7e3cbffap+0, C4 = 0x1.e1f506891babbp-3;
  const double C5 = -0x1.a6d1f2a204a8cp-6, C6 = 0x1.f9d38a3763cc3p-10;
  const double C7 = -0x1.b6e24f44b128fp-14, C8 = 0x1.20c62c2f2d7f5p-18;
  const double C9 = -0x1.2a0c591af8314p-23;
  int64_t n = (int64_t)((m + (1ULL << 49)) >> 50);          // round(2x), 0..4
  int64_t jj = (int64_t)m - n * (int64_t)(1ULL << 50);      // |jj| <= 2^49
  double f = (double)jj * 4.44089209850062616169e-16;       // * 2^-51, exact
  double f2 = f * f;
  double ps = std::fma(f2, S8, S7);
  ps = std::fma(f2, ps, S6);
  ps = std::fma(f2, ps, S5);
  ps = std::fma(f2, ps, S4);
  ps = std::fma(f2, ps, S3);
  ps = std::fma(f2, ps, S2);
  ps = std::fma(f2, ps, S1);
  double hi = f * PI;
  double lo = std::fma(f, PI_LO, std::fma(f, PI, -hi));
  double sf = hi + std::fma(f * f2, ps, lo);
  double pc = std::fma(f2, C9, C8);
  pc = std::fma(f2, pc, C7);
  pc = std::fma(f2, pc, C6);
  pc = std::fma(f2, pc, C5);
  pc = std::fma(f2, pc, C4);
  pc = std::fma(f2, pc, C3);
  pc = std::fma(f2, pc, C2);
  pc = std::fma(f2, pc, C1);
  double cf = std::fma(f2, pc, 1.0);
  double s, c;
  switch ((int)(n & 3)) {
    case 0: s = sf; c = cf; break;
    case 1: s = cf; c = -sf; break;
    case 2: s = -sf; c = -cf; break;
    default: s = -cf; c = sf; break;
  }
  *s_out = s; *c_out = c;
}

// u1 in (0,1], v in [0,1) from two 32-bit words (NC-3): u1 = (a + 1) 2^-32, v = b 2^-32.
void uniforms(uint32_t a, uint32_t b, double *u1, double *v) {
  *u1 = (double)((uint64_t)a + 1u) * 2.3283064365386962890625e-10;   // 2^-32, exact
  *v = (double)b * 2.3283064365386962890625e-10;
}

// The Box-Muller pair for arms (2k, 2k+1) of trial i at recurrence t (NC-3).  One Philox
// block, counter (t, 1 << 24 | k >> 1, trial), serves two pairs: pair k uses words
// (x0, x1) when k is even and (x2, x3) when k is odd.
void normal_pair(uint64_t seed, int64_t trial, int32_t t, int32_t k, double *z0, double *z1) {
  uint32_t ctr[4] = {(uint32_t)t, 0x01000000u | ((uint32_t)k >> 1), (uint32_t)(uint64_t)trial,
                     (uint32_t)((uint64_t)trial >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  philox(ctr, key, x);
  const uint32_t a = x[2 * (k & 1)], b = x[2 * (k & 1) + 1];
  double u1, v;
  uniforms(a, b, &u1, &v);
  double r = std::sqrt(-2.0 * zlog(u1));
  double s, c;
  zsincospi((uint64_t)b << 20, &s, &c);   // 2*pi*v: m = v 2^52 = b 2^20
  *z0 = r * c;
  *z1 = r * s;
}

// Which of the K recorded seeds a run replays (Q15 / NC-3).
// One Philox block serves the replica draws of four consecutive recurrences:
// counter (t >> 2, 2 << 24, trial), word t & 3.
uint32_t replica(uint64_t seed, int64_t trial, int32_t t, int32_t K) {
  uint32_t ctr[4] = {(uint32_t)t >> 2, 0x02000000u, (uint32_t)(uint64_t)trial,
                     (uint32_t)((uint64_t)trial >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  philox(ctr, key, x);
  return (uint32_t)(((uint64_t)x[t & 3] * (uint64_t)(uint32_t)K) >> 32);
}

// Draws of retry attempt j >= 1 of recurrence t (R-Q4v): the normal pairs use counter
// (t, 1 << 24 | j << 16 | k >> 1, trial), the replica counter (t, 3 << 24 | j, trial) word 0.
// Attempt 0 uses the counters above, so a recurrence without a retry draws what the base
// replay draws.
void normal_pair_attempt(uint64_t seed, int64_t trial, int32_t t, int32_t j, int32_t k, double *z0,
                         double *z1) {
  if (j == 0) { normal_pair(seed, trial, t, k, z0, z1); return; }
  const uint32_t ctr[4] = {(uint32_t)t, (1u << 24) | ((uint32_t)j << 16) | (uint32_t)(k >> 1),
                           (uint32_t)(uint64_t)trial, (uint32_t)((uint64_t)trial >> 32)};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  philox(ctr, key, x);
  const uint32_t a = (k & 1) ? x[2] : x[0], b = (k & 1) ? x[3] : x[1];
  double u1, v;
  uniforms(a, b, &u1, &v);
  const double r = std::sqrt(-2.0 * zlog(u1));
  double s, c;
  zsincospi((uint64_t)b << 20, &s, &c);                      // 2 pi v = pi (b 2^20) / 2^51
  *z0 = r * c;
  *z1 = r * s;
}
uint32_t replica_attempt(uint64_t seed, int64_t trial, int32_t t, int32_t j, int32_t K) {
  if (j == 0) return replica(seed, trial, t, K);
  const uint32_t ctr[4] = {(uint32_t)t, (3u << 24) | (uint32_t)j, (uint32_t)(uint64_t)trial,
                           (uint32_t)((uint64_t)trial >> 32)};
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  philox(ctr, key, x);
  return (uint32_t)(((uint64_t)x[0] * (uint64_t)K) >> 32);
}

// ---------------------------------------------------------------- Predict (Alg. 1)
struct Counters { int64_t c[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}; };

// Alg. 1: for every batch size b of the set, sample θ̂_b ~ N(μ̂_b, σ̂_b²) and
// return argmin_b θ̂_b (strict <, ascending b: ties go to the smaller index, NC-4).  The
// normal of arm b at recurrence t (attempt j) is one half of the Box-Muller pair k = b >> 1
// (NC-3); θ̂_b = fma(σ̂_b, z, μ̂_b).  `set` is a bitmask of arms; returns -1 for an empty set.
int thompson_argmin(uint64_t seed, int64_t trial, int32_t t, int32_t j, int B, uint32_t set,
                    const double *mu, const double *sigma, Counters &cnt) {
  int b = -1;
  double best_theta = std::numeric_limits<double>::infinity();
  int last_block = -1;
  for (int k = 0; 2 * k < B; ++k) {
    uint32_t pairmask = (set >> (2 * k)) & 3u;
    if (!pairmask) continue;
    if ((k >> 1) != last_block) { last_block = k >> 1; cnt.c[8] += 1; }
    double z[2];
    normal_pair_attempt(seed, trial, t, j, k, &z[0], &z[1]);
    cnt.c[2] += 1;
    for (int h = 0; h < 2; ++h) {
      int a = 2 * k + h;
      if (!(pairmask & (1u << h))) continue;
      double theta = std::fma(sigma[a], z[h], mu[a]);
      cnt.c[3] += 1;
      if (theta < best_theta) { best_theta = theta; b = a; }
    }
  }
  cnt.c[1] += 1;
  return b;
}

// ---------------------------------------------------------------- Observe (Alg. 2)
// One arm's belief.  Var(C_b) and Sum(C_b) of Alg. 2 are kept as
// sums shifted by the arm's first observation (NC-6); the window of the N most
// recent observations is an explicit queue.
struct Arm {
  std::deque<double> window;   // observations currently counted
  int64_t cnt = 0;             // observations ever
  double sh = 0.0, S1 = 0.0, S2 = 0.0;
  double mu = 0.0, sigma = 0.0;
  bool profiled = false;
};

struct Prior { double prec0, pm0; };

Prior make_prior(double prior_mean, double prior_var) {
  Prior p;
  p.prec0 = std::isinf(prior_var) ? 0.0 : 1.0 / prior_var;   // flat prior: P:L529
  p.pm0 = prior_mean * p.prec0;
  return p;
}

// returns true when the posterior was (re)computed (n >= 2)
bool observe(Arm &a, double x, int32_t window, const Prior &pr, double *s2_out, double *var_out) {
  if (a.cnt == 0) a.sh = x;
  if (window > 0 && (int32_t)a.window.size() == window) {   // forget the oldest
    double y = a.window.front();
    a.window.pop_front();
    double dy = y - a.sh;
    a.S1 = a.S1 - dy;
    a.S2 = a.S2 - dy * dy;
  }
  double d = x - a.sh;                                       // C_b <- C_b ∪ {C}
  a.S1 = a.S1 + d;
  a.S2 = a.S2 + d * d;
  a.window.push_back(x);
  a.cnt += 1;
  int64_t n = (int64_t)a.window.size();
  if (n < 2) return false;
  double dn = (double)n;
  double rq = 1.0 / (dn * (dn - 1.0));                      // 1/n and 1/(n-1) from one division
  double inv_n = (dn - 1.0) * rq;
  double inv_nm1 = dn * rq;
  double mean = a.sh + a.S1 * inv_n;
  double s2 = (a.S2 - a.S1 * (a.S1 * inv_n)) * inv_nm1;     // σ̃² = Var(C_b), n-1 divisor
  double fl = 1e-12 * (1.0 + mean * mean);
  if (!(s2 >= fl)) s2 = fl;                                 // zero-variance floor (R-Q7)
  // Alg. 2: σ̂² = (1/σ̂0² + |C_b|/σ̃²)^-1 and μ̂ = σ̂²(μ̂0/σ̂0² + Sum(C_b)/σ̃²), written
  // with both numerator and denominator multiplied by σ̃² (NC-6)
  double den = (pr.prec0 * s2) + dn;
  double rden = 1.0 / den;
  double sum = (dn * a.sh) + a.S1;                           // Sum(C_b)
  double var = s2 * rden;
  a.mu = ((pr.pm0 * s2) + sum) * rden;
  a.sigma = std::sqrt(var);
  if (s2_out) *s2_out = s2;
  if (var_out) *var_out = var;
  return true;
}

// ---------------------------------------------------------------- step 1
struct Tables {
  int B = 0, P = 0, S = 0;
  std::vector<int32_t> pstar;
  std::vector<double> c1, t1, e1, cP, tP, eP;
  std::vector<double> ebar, regret, opt;
  std::vector<int32_t> opt_arm;
};

void step1(const oracle_trace &tr, const oracle_cell &cell, Tables &T) {
  const int B = tr.num_batch_sizes, P = tr.num_power_limits, S = tr.num_slices, K = tr.replicas;
  const double eta = cell.eta, MP = tr.max_power_w;
  T.B = B; T.P = P; T.S = S;
  T.pstar.assign(B, 0);
  T.c1.assign(B, 0); T.t1.assign(B, 0); T.e1.assign(B, 0);
  T.cP.assign(B, 0); T.tP.assign(B, 0); T.eP.assign(B, 0);
  for (int b = 0; b < B; ++b) {
    const double *A = tr.avg_power_w + (size_t)b * P;
    const double *Th = tr.throughput_eps + (size_t)b * P;
    // Eq. 7: EpochCost(b) = min_p (η·AvgPower + (1-η)·MAXPOWER) / Throughput
    double best = std::numeric_limits<double>::infinity();
    int arg = 0;
    for (int p = 0; p < P; ++p) {
      double num = (eta * A[p]) + ((1.0 - eta) * MP);
      double c = num / Th[p];
      if (c < best) { best = c; arg = p; }       // first minimum: smaller p wins ties
    }
    T.pstar[b] = arg;
    T.c1[b] = best;
    T.t1[b] = 1.0 / Th[arg];
    T.e1[b] = A[arg] / Th[arg];
    // JIT profiling epoch: one equal-work slice per power limit
    double st = 0.0, se = 0.0;
    for (int p = 0; p < P; ++p) {
      st = st + 1.0 / Th[p];
      se = se + A[p] / Th[p];
    }
    T.tP[b] = st / (double)P;
    T.eP[b] = se / (double)P;
    T.cP[b] = (eta * T.eP[b]) + (((1.0 - eta) * MP) * T.tP[b]);
  }
  // known optimum per slice: min over (b,p) of Epochs(b)*c(b,p)
  T.ebar.assign((size_t)S * B, 0);
  T.regret.assign((size_t)S * B, 0);
  T.opt.assign(S, 0);
  T.opt_arm.assign(S, -1);
  for (int s = 0; s < S; ++s) {
    std::vector<int64_t> count(B, 0);
    double best = std::numeric_limits<double>::infinity();
    int barg = -1;
    for (int b = 0; b < B; ++b) {
      int64_t sum = 0;
      for (int k = 0; k < K; ++k) {
        int32_t E = tr.epochs_to_target[((size_t)s * B + b) * K + k];
        if (E > 0) { sum += E; count[b] += 1; }
      }
      double eb = count[b] > 0 ? (double)sum / (double)count[b] : (double)tr.max_epochs;
      T.ebar[(size_t)s * B + b] = eb;
      if (count[b] > 0) {
        double v = eb * T.c1[b];
        if (v < best) { best = v; barg = b; }
      }
    }
    T.opt[s] = best;
    T.opt_arm[s] = barg;
    for (int b = 0; b < B; ++b)   // Eq. 9 with Epochs(b_t) read as its mean (R-Q12)
      T.regret[(size_t)s * B + b] = T.ebar[(size_t)s * B + b] * T.c1[b] - best;
  }
}

// ---------------------------------------------------------------- validation
std::string validate(const oracle_trace &tr, const oracle_cell &cell) {
  std::string e;
  auto add = [&](const char *m) { if (!e.empty()) e += "; "; e += m; };
  const int B = tr.num_batch_sizes, P = tr.num_power_limits;
  if (B < 1) add("no batch sizes");
  if (B > 32) add("more than 32 batch sizes");
  if (P < 1) add("no power limits");
  if (P > 64) add("more than 64 power limits");
  if (B >= 1 && tr.batch_sizes) {
    for (int b = 0; b < B; ++b) if (tr.batch_sizes[b] <= 0) { add("batch size not positive"); break; }
    for (int b = 1; b < B; ++b) if (tr.batch_sizes[b] <= tr.batch_sizes[b - 1]) { add("batch sizes not strictly increasing"); break; }
  }
  if (tr.default_bs_index < 0 || tr.default_bs_index >= B) add("default batch size index out of range");
  double pmax = 0.0;
  if (P >= 1 && tr.power_limits_w) {
    for (int p = 0; p < P; ++p) if (!(tr.power_limits_w[p] > 0.0)) { add("power limit not positive"); break; }
    for (int p = 1; p < P; ++p) if (!(tr.power_limits_w[p] > tr.power_limits_w[p - 1])) { add("power limits not strictly increasing"); break; }
    pmax = tr.power_limits_w[P - 1];
  }
  if (!(tr.max_power_w >= pmax) || !std::isfinite(tr.max_power_w)) add("max power below the largest power limit");
  if (tr.max_epochs < 1) add("max_epochs < 1");
  if (!(cell.eta >= 0.0 && cell.eta <= 1.0)) add("eta out of [0,1]");
  if (!(cell.beta > 1.0)) add("beta must be > 1");
  if (cell.window == 1 || cell.window < 0) add("window must be 0 (unbounded) or >= 2");
  if (!(cell.prior_var > 0.0)) add("prior variance must be > 0");
  if (!std::isfinite(cell.prior_mean)) add("prior mean not finite");
  if (cell.policy < 0 || cell.policy > 2) add("policy must be 0 (Zeus), 1 (Default) or 2 (Grid Search)");
  if (cell.ablation < 0 || cell.ablation > 31)
    add("ablation must be a subset of {1 no pruning, 2 no JIT, 4 retry, 8 epoch stop, 16 windowed best}");
  if ((cell.ablation & 16) && cell.window < 2) add("windowed best needs window >= 2");
  if ((cell.ablation & 28) && cell.arrivals) add("variant readings need sequential recurrences");
  if (cell.ablation != 0 && cell.policy != 0) add("ablations apply to the Zeus policy only");
  if (B >= 1 && P >= 1 && B <= 32 && P <= 64) {
    for (int i = 0; i < B * P; ++i)
      if (!(tr.avg_power_w[i] > 0.0) || !std::isfinite(tr.avg_power_w[i])) { add("average power not positive"); break; }
    for (int i = 0; i < B * P; ++i)
      if (!(tr.avg_power_w[i] <= tr.max_power_w)) { add("average power above max power"); break; }
    for (int i = 0; i < B * P; ++i)
      if (!(tr.throughput_eps[i] > 0.0) || !std::isfinite(tr.throughput_eps[i])) { add("throughput not positive"); break; }
  }
  if (tr.num_slices < 1) add("num_slices < 1");
  if (tr.replicas < 1) add("replicas < 1");
  if (e.empty()) {
    const int S = tr.num_slices, K = tr.replicas;
    for (size_t i = 0; i < (size_t)S * B * K; ++i)
      if (tr.epochs_to_target[i] > tr.max_epochs) { add("epochs_to_target above max_epochs"); break; }
    for (int s = 0; s < S; ++s) {
      bool any = false;
      for (int i = 0; i < B * K; ++i) any |= tr.epochs_to_target[(size_t)s * B * K + i] > 0;
      if (!any) { add("a slice has no converged replica on any arm"); break; }
    }
  }
  return e;
}

// ---------------------------------------------------------------- one trial
int lowest_bit(uint32_t m) { for (int b = 0; b < 32; ++b) if (m & (1u << b)) return b; return -1; }
int highest_bit(uint32_t m) { for (int b = 31; b >= 0; --b) if (m & (1u << b)) return b; return -1; }
uint32_t below(int c) { return c <= 0 ? 0u : ((1u << c) - 1u); }
uint32_t above(int c) { return c >= 31 ? 0u : ~((2u << c) - 1u); }

enum Step { START, DOWN, UP };

// Outstanding runs per trial under an arrival schedule (R-Q31): a submission that would
// exceed it first waits for the earliest completion.
constexpr int kMaxOutstanding = 8;

struct TrialResult {
  double tot_cost = 0, tot_energy = 0, tot_time = 0;
  uint64_t digest = 0xcbf29ce484222325ULL;
  int32_t n_stop = 0, final_arm = -1;
};

// Per-epoch cost, time and energy of configuration (b, p) -- the quantity inside the
// min of Eq. 7, in the NC-2 operation order.
void epoch_cost(const oracle_trace &tr, const oracle_cell &cell, int b, int p, double *c,
                double *t, double *e) {
  const double A = tr.avg_power_w[(size_t)b * tr.num_power_limits + p];
  const double Th = tr.throughput_eps[(size_t)b * tr.num_power_limits + p];
  *c = ((cell.eta * A) + ((1.0 - cell.eta) * tr.max_power_w)) / Th;
  *t = 1.0 / Th;
  *e = A / Th;
}

// The two baselines of §6.1, replayed on the same trace with the same
// replica draws (NC-3) as Zeus.  Neither uses the JIT profiler nor Zeus's early stop
// (R-Q29): every run goes to its epochs-to-target or max_epochs.
//   Default:      every recurrence runs (b0, the largest power limit).
//   Grid Search:  one (b, p) per recurrence, b ascending then p ascending; a run that
//                 fails to reach the target prunes the rest of its batch size;
//                 after the grid, exploit the cheapest converged configuration seen.
void run_trial_baseline(const oracle_trace &tr, const oracle_cell &cell, const Tables &T,
                        int32_t R, int64_t trial, TrialResult &res, double *curves, uint32_t *log,
                        double *clog, double *elog, double *tlog, Counters &cnt) {
  const int B = tr.num_batch_sizes, P = tr.num_power_limits, S = tr.num_slices, K = tr.replicas;
  bool exploring = cell.policy == 2;
  int gb = 0, gp = 0;                                        // grid cursor
  double best_c = std::numeric_limits<double>::infinity();
  int best_b = -1, best_p = -1;
  for (int32_t t = 0; t < R; ++t) {
    const int s = (int)(((int64_t)t * S) / R);
    int b, p;
    if (cell.policy == 1) { b = tr.default_bs_index; p = P - 1; }
    else if (exploring) { b = gb; p = gp; }
    else if (best_b >= 0) { b = best_b; p = best_p; }
    else { b = tr.default_bs_index; p = P - 1; }             // nothing converged in the grid
    double c, tt, e;
    epoch_cost(tr, cell, b, p, &c, &tt, &e);
    const uint32_t r = replica(cell.seed, trial, t, K);
    const int32_t E = tr.epochs_to_target[((size_t)s * B + b) * K + r];
    const int32_t E_run = E > 0 ? E : tr.max_epochs;
    const double em1 = (double)(E_run - 1);
    const double C = c + em1 * c;
    const double Tm = tt + em1 * tt;
    const double En = e + em1 * e;
    const bool converged = E > 0;
    if (exploring) {
      if (converged && C < best_c) { best_c = C; best_b = b; best_p = p; }
      if (!converged || gp == P - 1) { gb += 1; gp = 0; }   // prune b, or its row is done
      else gp += 1;
      if (gb == B) exploring = false;
    }
    cnt.c[0] += 1;
    const uint32_t flags = converged ? 2u : 0u;
    res.tot_cost += C;
    res.tot_energy += En;
    res.tot_time += Tm;
    res.final_arm = b;
    const uint8_t bytes[3] = {(uint8_t)b, (uint8_t)p, (uint8_t)flags};   // NC-9 digest
    for (int q = 0; q < 3; ++q) { res.digest ^= bytes[q]; res.digest *= 0x100000001b3ULL; }
    if (curves) {
      double *row = curves + (size_t)t * 7;
      row[0] += C;
      row[1] += En;
      row[2] += Tm;
      row[3] += T.ebar[(size_t)s * B + b] * c - T.opt[s];   // Eq. 9 pseudo-regret at (b, p)
      row[5] += (b == T.opt_arm[s] && p == T.pstar[b]) ? 1.0 : 0.0;
    }
    if (log) log[t] = (uint32_t)b | ((uint32_t)p << 8) | (flags << 16);
    if (clog) clog[t] = C;
    if (elog) elog[t] = En;
    if (tlog) tlog[t] = Tm;
  }
}

void run_trial(const oracle_trace &tr, const oracle_cell &cell, const Tables &T, int32_t R,
               int64_t trial, TrialResult &res, double *curves, uint32_t *log, double *clog,
               double *elog, double *tlog, Counters &cnt) {
  if (cell.policy != 0) {
    run_trial_baseline(tr, cell, T, R, trial, res, curves, log, clog, elog, tlog, cnt);
    return;
  }
  const int B = tr.num_batch_sizes, S = tr.num_slices, K = tr.replicas;
  const Prior pr = make_prior(cell.prior_mean, cell.prior_var);
  std::vector<Arm> arm(B);
  std::vector<double> mu(B), sigma(B);                      // the posteriors Predict reads
  double best = std::numeric_limits<double>::infinity();   // min_t C_t

  // Alg. 3 state
  bool in_ts = false;
  int round = 1;
  Step step = START;
  const uint32_t all_arms = (B == 32) ? 0xffffffffu : ((1u << B) - 1u);
  uint32_t cand = all_arms;
  int start = tr.default_bs_index;
  int cursor = start;
  uint32_t surv = 0, ts_set = 0;
  double r1_cost = std::numeric_limits<double>::infinity();
  int r1_arm = -1;
  int best_arm = -1;              // the best-known batch size (arm of min_t C_t)
  bool walk_out = false;          // an Alg. 3 walk run is submitted and not yet completed

  // A run's outcome reaching the optimiser: best update, Observe (Alg. 2) and, for the
  // runs Alg. 3's walk issued, the walk's bookkeeping.
  struct Job { double done; int32_t seq; int b; double C; bool conv; bool walk; };
  std::vector<Job> pending;
  auto complete = [&](const Job &j) {
    const int b = j.b;
    const double C = j.C;
    const bool converged = j.conv;
    if (converged && !(C >= best)) { best = C; best_arm = b; }
    // Alg. 2 Observe: every run is observed, stopped runs at the threshold (R-Q3)
    if (observe(arm[b], C, cell.window, pr, nullptr, nullptr)) cnt.c[7] += 1;
    if (!j.walk) return;
    walk_out = false;
    // ---- Alg. 3 bookkeeping
    if (converged) {
      surv |= 1u << b;
      if (round == 1 && (C < r1_cost || (C == r1_cost && b < r1_arm))) { r1_cost = C; r1_arm = b; }
    }
    bool end_round = false;
    if (step == START) { step = DOWN; cursor = start; }
    else if (step == DOWN) { if (converged) cursor = b; else { step = UP; cursor = start; } }
    else { if (converged) cursor = b; else end_round = true; }
    if (!end_round && step == DOWN && (cand & below(cursor)) == 0) { step = UP; cursor = start; }
    if (!end_round && step == UP && (cand & above(cursor)) == 0) end_round = true;
    if (end_round) {
      if (surv == 0) surv = 1u << start;           // R-Q23
      if (round == 1) {
        cand = (cell.ablation & 1) ? all_arms : surv;   // "no pruning" keeps 𝓑
        if (r1_arm >= 0) start = r1_arm;           // b0 <- b with smallest cost observed
        surv = 0;
        round = 2;
        step = START;
        cursor = start;
      } else {
        in_ts = true;
        ts_set = (cell.ablation & 1) ? all_arms : surv;
      }
    }
  };
  // completes the earliest pending run, by (completion time, submission order)
  auto complete_earliest = [&]() {
    size_t e = 0;
    for (size_t i = 1; i < pending.size(); ++i)
      if (pending[i].done < pending[e].done ||
          (pending[i].done == pending[e].done && pending[i].seq < pending[e].seq)) e = i;
    const Job j = pending[e];
    pending.erase(pending.begin() + (long)e);
    complete(j);
  };

  // converged cost of each recurrence (+inf: none), for the windowed best (R-Q5v)
  std::vector<double> conv_cost((size_t)R, std::numeric_limits<double>::infinity());
  for (int32_t t = 0; t < R; ++t) {
    const int s = (int)(((int64_t)t * S) / R);   // slice of recurrence t (R-Q19)
    if (cell.arrivals) {                           // runs finished by this submission (R-Q31)
      for (;;) {
        bool any = false;
        for (const Job &j : pending) any |= j.done <= cell.arrivals[t];
        if (!any) break;
        complete_earliest();
      }
      while ((int)pending.size() >= kMaxOutstanding) complete_earliest();
    }
    // Variant readings of P:L559 (R-Q4v / R-Q1v / R-Q5v; sequential recurrences only):
    // with `retry`, an early-stopped attempt is followed by another decision in the same
    // recurrence, Thompson sampling leaving out the arms stopped in it ("stop the job and retry
    // with another batch size"); the recurrence ends with its first attempt that is not
    // stopped, or when Thompson sampling has no arm left.
    const bool retry = (cell.ablation & 4) != 0;
    const bool epoch_stop = (cell.ablation & 8) != 0;
    const bool win_best = (cell.ablation & 16) != 0;
    uint32_t stopped_here = 0;     // arms early-stopped in this recurrence
    for (int32_t j = 0;; ++j) {
    if (j > 0 && in_ts && (ts_set & ~stopped_here) == 0) break;   // no arm left to retry
    const uint32_t eligible = ts_set & ~stopped_here;
    // ---- step 2: decide b_t
    int b;
    bool walk_issue = false;
    const bool ts_dec = in_ts;   // phase at decision time (flag bit 3)
    if (!in_ts) {
      if (walk_out) {              // concurrent submission while pruning: best-known b
        b = best_arm >= 0 ? best_arm : start;
      } else {
        if (step == START) b = start;
        else if (step == DOWN) b = highest_bit(cand & below(cursor));
        else b = lowest_bit(cand & above(cursor));
        walk_issue = true;
        walk_out = true;
      }
      cnt.c[5] += 1;
    } else {
      b = -1;
      for (int a = 0; a < B; ++a)           // arms without a variance estimate first (R-Q6)
        if ((eligible & (1u << a)) && (int)arm[a].window.size() < 2) { b = a; break; }
      if (b < 0) {
        for (int a = 0; a < B; ++a) { mu[a] = arm[a].mu; sigma[a] = arm[a].sigma; }
        b = thompson_argmin(cell.seed, trial, t, j, B, eligible, mu.data(), sigma.data(), cnt);
      } else {
        cnt.c[6] += 1;
      }
    }
    // ---- step 1 result: the power limit accompanying b.  Ablation "no JIT
    // profiling": the first P runs of b try the power limits in ascending
    // order, one per recurrence, each at its own per-epoch cost; then p*(b).
    int p = T.pstar[b];
    double c1b = T.c1[b], t1b = T.t1[b], e1b = T.e1[b];
    const bool no_jit = (cell.ablation & 2) != 0;
    if (no_jit && arm[b].cnt < tr.num_power_limits) {
      p = (int)arm[b].cnt;
      epoch_cost(tr, cell, b, p, &c1b, &t1b, &e1b);
    }
    // ---- step 3: replay one recorded run of b
    const uint32_t r = replica_attempt(cell.seed, trial, t, j, K);
    const int32_t E = tr.epochs_to_target[((size_t)s * B + b) * K + r];
    const int32_t E_run = E > 0 ? E : tr.max_epochs;
    double c0, t0, e0;
    bool profiled_now = false;
    if (!no_jit && tr.charge_profiling && !arm[b].profiled) {   // JIT profiling epoch
      c0 = T.cP[b]; t0 = T.tP[b]; e0 = T.eP[b]; profiled_now = true;
    } else {
      c0 = c1b; t0 = t1b; e0 = e1b;
    }
    arm[b].profiled = true;
    const double em1 = (double)(E_run - 1);
    const double C_full = c0 + em1 * c1b;
    const double T_full = t0 + em1 * t1b;
    const double En_full = e0 + em1 * e1b;
    // ---- step 4: early stop at β·min_t C_t; with `win_best` the minimum runs over
    // the converged runs of the last N recurrences only (R-Q5v)
    double best_now = best;
    if (win_best) {
      best_now = std::numeric_limits<double>::infinity();
      for (int32_t u = std::max(0, t - cell.window); u < t; ++u)
        if (conv_cost[u] < best_now) best_now = conv_cost[u];
    }
    const double thr = cell.beta * best_now;
    double C, Tm, En;
    bool stopped = false;
    if (C_full > thr && epoch_stop) {
      // R-Q1v: the cost is checked at epoch boundaries: the run stops at the end of
      // the first epoch k whose accumulated cost c0 + (k-1) c1 exceeds thr -- unless that is
      // its last epoch E_run, where it ends anyway (reaching the target, or failing)
      int32_t k = 1;
      while (!(c0 + (double)(k - 1) * c1b > thr)) ++k;
      if (k < E_run) {
        stopped = true;
        const double em = (double)(k - 1);
        C = c0 + em * c1b;
        Tm = t0 + em * t1b;
        En = e0 + em * e1b;
      } else {
        C = C_full; Tm = T_full; En = En_full;
      }
    } else if (C_full > thr) {   // R-Q1: continuous truncation, charged exactly thr
      stopped = true;
      C = thr;
      if (thr <= c0) {
        double phi = thr / c0;
        Tm = phi * t0;
        En = phi * e0;
      } else {
        double phi = (thr - c0) / c1b;
        Tm = t0 + phi * t1b;
        En = e0 + phi * e1b;
      }
    } else {
      C = C_full; Tm = T_full; En = En_full;
    }
    const bool converged = (E > 0) && !stopped;
    if (converged) conv_cost[t] = C;
    cnt.c[0] += 1;
    if (stopped) cnt.c[4] += 1;
    // the run's outcome reaches the optimiser when it completes: immediately in the paper's
    // sequential replay, at submit time + its TTA with an arrival schedule
    const Job job{cell.arrivals ? cell.arrivals[t] + Tm : 0.0, t, b, C, converged, walk_issue};
    if (cell.arrivals) pending.push_back(job);
    else complete(job);

    // ---- accumulate (Eq. 4, Eqs. 8-9)
    const uint32_t flags = (stopped ? 1u : 0u) | (converged ? 2u : 0u) |
                           (profiled_now ? 4u : 0u) | (ts_dec ? 8u : 0u) | (j > 0 ? 16u : 0u);
    res.tot_cost += C;
    res.tot_energy += En;
    res.tot_time += Tm;
    if (stopped) res.n_stop += 1;
    res.final_arm = b;
    const uint8_t bytes[3] = {(uint8_t)b, (uint8_t)p, (uint8_t)flags};   // NC-9 digest
    for (int q = 0; q < 3; ++q) { res.digest ^= bytes[q]; res.digest *= 0x100000001b3ULL; }
    if (curves) {
      double *row = curves + (size_t)t * 7;
      row[0] += C;
      row[1] += En;
      row[2] += Tm;
      row[3] += (p == T.pstar[b]) ? T.regret[(size_t)s * B + b]
                                  : T.ebar[(size_t)s * B + b] * c1b - T.opt[s];
      row[4] += stopped ? 1.0 : 0.0;
      row[5] += (b == T.opt_arm[s] && p == T.pstar[b]) ? 1.0 : 0.0;
      row[6] += ts_dec ? 1.0 : 0.0;
    }
    if (log) log[t] = (uint32_t)b | ((uint32_t)p << 8) | (flags << 16);   // the last attempt
    if (clog) clog[t] = (j > 0 ? clog[t] : 0.0) + C;                      // the recurrence's
    if (elog) elog[t] = (j > 0 ? elog[t] : 0.0) + En;                     // totals
    if (tlog) tlog[t] = (j > 0 ? tlog[t] : 0.0) + Tm;
    if (!(retry && stopped)) break;
    stopped_here |= 1u << b;
    }
  }
}

}  // namespace

// ======================================================================== C API
extern "C" {

int oracle_validate(const oracle_trace *tr, const oracle_cell *cell, char *msg, int32_t msglen) {
  std::string e = validate(*tr, *cell);
  if (msg && msglen > 0) {
    std::strncpy(msg, e.c_str(), (size_t)msglen - 1);
    msg[msglen - 1] = 0;
  }
  return e.empty() ? 0 : 1;
}

int oracle_step1(const oracle_trace *tr, const oracle_cell *cell, oracle_tables *out) {
  if (!validate(*tr, *cell).empty()) return 1;
  Tables T;
  step1(*tr, *cell, T);
  const int B = T.B, S = T.S;
  for (int b = 0; b < B; ++b) {
    if (out->pstar) out->pstar[b] = T.pstar[b];
    if (out->c1) out->c1[b] = T.c1[b];
    if (out->t1) out->t1[b] = T.t1[b];
    if (out->e1) out->e1[b] = T.e1[b];
    if (out->c_prof) out->c_prof[b] = T.cP[b];
    if (out->t_prof) out->t_prof[b] = T.tP[b];
    if (out->e_prof) out->e_prof[b] = T.eP[b];
  }
  for (int s = 0; s < S; ++s) {
    if (out->opt) out->opt[s] = T.opt[s];
    if (out->opt_arm) out->opt_arm[s] = T.opt_arm[s];
    for (int b = 0; b < B; ++b) {
      if (out->ebar) out->ebar[(size_t)s * B + b] = T.ebar[(size_t)s * B + b];
      if (out->regret) out->regret[(size_t)s * B + b] = T.regret[(size_t)s * B + b];
    }
  }
  return 0;
}

int oracle_replay(const oracle_trace *tr, const oracle_cell *cell, int32_t R,
                  const int64_t *trials, int64_t n, int32_t threads, oracle_out *out) {
  if (!validate(*tr, *cell).empty() || R < 0 || n < 0) return 1;
  if (cell->arrivals) {                 // arrival schedule: Zeus only, finite, non-decreasing
    if (cell->policy != 0 || cell->ablation != 0) return 1;
    for (int32_t t = 0; t < R; ++t)
      if (!std::isfinite(cell->arrivals[t]) || (t > 0 && cell->arrivals[t] < cell->arrivals[t - 1]))
        return 1;
  }
  Tables T;
  step1(*tr, *cell, T);
  if (threads < 1) threads = 1;
  if ((int64_t)threads > n) threads = (int32_t)(n > 0 ? n : 1);
  std::vector<std::vector<double>> part(threads, std::vector<double>(out->curves ? (size_t)R * 7 : 0, 0.0));
  std::vector<Counters> pc(threads);
  auto worker = [&](int w) {
    for (int64_t j = w; j < n; j += threads) {   // trials are independent; one task each
      TrialResult res;
      size_t off = (size_t)j * (size_t)R;
      run_trial(*tr, *cell, T, R, trials[j], res, out->curves ? part[w].data() : nullptr,
                out->log ? out->log + off : nullptr, out->cost_log ? out->cost_log + off : nullptr,
                out->energy_log ? out->energy_log + off : nullptr,
                out->time_log ? out->time_log + off : nullptr, pc[w]);
      if (out->tot_cost) out->tot_cost[j] = res.tot_cost;
      if (out->tot_energy) out->tot_energy[j] = res.tot_energy;
      if (out->tot_time) out->tot_time[j] = res.tot_time;
      if (out->digest) out->digest[j] = res.digest;
      if (out->n_stop) out->n_stop[j] = res.n_stop;
      if (out->final_arm) out->final_arm[j] = res.final_arm;
    }
  };
  if (threads == 1) {
    worker(0);
  } else {
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w) pool.emplace_back(worker, w);
    for (auto &th : pool) th.join();
  }
  if (out->curves) {
    for (size_t i = 0; i < (size_t)R * 7; ++i) out->curves[i] = 0.0;
    for (int w = 0; w < threads; ++w)
      for (size_t i = 0; i < (size_t)R * 7; ++i) out->curves[i] += part[w][i];
  }
  if (out->counters) {
    for (int q = 0; q < 9; ++q) {
      out->counters[q] = 0;
      for (int w = 0; w < threads; ++w) out->counters[q] += pc[w].c[q];
    }
  }
  return 0;
}

// Pareto front of the (TTA, ETA) grid of slice s (§2.3, Fig. eta-tta-tradeoff;
// SURVEY §8(f) f4): point (b, p) has TTA = Ebar(b,s)/Th(b,p) and ETA = (Ebar(b,s)*A(b,p))/Th(b,p)
// for every b with a converged replica; mask = 1 iff no other point has both coordinates <=
// with one strictly <, and no earlier point in (b, p) order has identical coordinates.
int oracle_pareto(const oracle_trace *tr, int32_t s, uint8_t *mask) {
  const int B = tr->num_batch_sizes, P = tr->num_power_limits, K = tr->replicas;
  if (s < 0 || s >= tr->num_slices) return 1;
  std::vector<double> tta((size_t)B * P), eta((size_t)B * P);
  std::vector<bool> valid((size_t)B * P, false);
  for (int b = 0; b < B; ++b) {
    int64_t sum = 0, cnt = 0;
    for (int k = 0; k < K; ++k) {
      const int32_t E = tr->epochs_to_target[((size_t)s * B + b) * K + k];
      if (E > 0) { sum += E; ++cnt; }
    }
    if (cnt == 0) continue;
    const double eb = (double)sum / (double)cnt;
    for (int p = 0; p < P; ++p) {
      const double A = tr->avg_power_w[(size_t)b * P + p], Th = tr->throughput_eps[(size_t)b * P + p];
      tta[(size_t)b * P + p] = eb / Th;
      eta[(size_t)b * P + p] = (eb * A) / Th;
      valid[(size_t)b * P + p] = true;
    }
  }
  for (int i = 0; i < B * P; ++i) {
    bool keep = valid[i];
    for (int j = 0; j < B * P && keep; ++j) {
      if (j == i || !valid[j]) continue;
      const bool le = tta[j] <= tta[i] && eta[j] <= eta[i];
      const bool lt = tta[j] < tta[i] || eta[j] < eta[i];
      if (le && lt) keep = false;                          // dominated
      if (!lt && le && j < i) keep = false;               // identical, an earlier one is kept
    }
    mask[i] = keep ? 1 : 0;
  }
  return 0;
}

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  philox(ctr, key, out);
}
double oracle_zlog(double x) { return zlog(x); }
double oracle_zlog_fdlibm(double x) { return zlog_fdlibm(x); }
void oracle_zsincospi(uint64_t m52, double *s, double *c) { zsincospi(m52, s, c); }
void oracle_uniforms(uint32_t a, uint32_t b, double *u1, double *v) { uniforms(a, b, u1, v); }
void oracle_normal_pair(uint64_t seed, int64_t trial, int32_t t, int32_t k, double *z0, double *z1) {
  normal_pair(seed, trial, t, k, z0, z1);
}
uint32_t oracle_replica(uint64_t seed, int64_t trial, int32_t t, int32_t K) {
  return replica(seed, trial, t, K);
}
int32_t oracle_thompson_argmin(uint64_t seed, int64_t trial, int32_t t, int32_t B, uint32_t set,
                               const double *mu, const double *sigma) {
  if (B < 1 || B > 32) return -1;
  Counters cnt;
  return thompson_argmin(seed, trial, t, 0, B, set, mu, sigma, cnt);
}
int oracle_posterior(const double *xs, int32_t n, int32_t window, double prior_mean,
                     double prior_var, double *mu, double *sigma, double *s2, double *var) {
  Arm a;
  Prior pr = make_prior(prior_mean, prior_var);
  bool ok = false;
  for (int32_t i = 0; i < n; ++i) ok = observe(a, xs[i], window, pr, s2, var);
  if (!ok) return 1;
  *mu = a.mu;
  *sigma = a.sigma;
  return 0;
}
// Batches of the primitives for the large-sample pins (tests/test_sampler_scale.py).
void oracle_zlog_batch(const double *x, double *y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = zlog(x[i]);
}
void oracle_zsincospi_batch(const uint64_t *m, double *s, double *c, int64_t n) {
  for (int64_t i = 0; i < n; ++i) zsincospi(m[i], s + i, c + i);
}
// out[2j], out[2j+1] = the Box-Muller pair k of trial trial0 + j at recurrence t
void oracle_normal_batch(uint64_t seed, int64_t trial0, int64_t n, int32_t t, int32_t k,
                         int32_t threads, double *out) {
  if (threads < 1) threads = 1;
  auto work = [&](int w) {
    for (int64_t j = w; j < n; j += threads)
      normal_pair(seed, trial0 + j, t, k, out + 2 * j, out + 2 * j + 1);
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < threads; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto &th : pool) th.join();
}
int32_t oracle_hardware_threads(void) {
  unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 1 : (int32_t)h;
}

}  // extern "C"
