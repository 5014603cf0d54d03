// work_probe.cu -- per-primitive SASS instruction counts of the contract functions
// (compiled, never run): each probe kernel wraps ONE primitive between a load and a
// store so `tools/work_model.py` can count its straight-line instructions by pipe.
#include "../paper_2208_06102_b200/csrc/thompson.cuh"
using namespace zs;
extern "C" __global__ void probe_empty(const double *in, double *out) {
  out[threadIdx.x] = in[threadIdx.x];
}
extern "C" __global__ void probe_philox(const uint32_t *in, uint32_t *out) {
  U4 x = philox4x32_10(U4{in[0], in[1], in[2], in[3]}, in[4], in[5]);
  out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
}
extern "C" __global__ void probe_zlog(const double *in, double *out, const double2 *tab) { out[0] = zlog(in[0], tab); }
extern "C" __global__ void probe_sincospi(const unsigned long long *in, double *out) {
  double s, c; zsincospi(in[0], s, c); out[0] = s; out[1] = c;
}
extern "C" __global__ void probe_bm(const uint32_t *in, double *out, const double2 *tab) {
  double z0, z1; box_muller(in[0], in[1], z0, z1, tab); out[0] = z0; out[1] = z1;
}
extern "C" __global__ void probe_sqrt(const double *in, double *out) { out[0] = sqrt(in[0]); }
extern "C" __global__ void probe_div(const double *in, double *out) { out[0] = in[0] / in[1]; }
extern "C" __global__ void probe_pair(const long long *in, double *out, const double2 *tab) {
  double z0, z1; normal_pair((uint32_t)in[0], (uint32_t)in[1], in[2], (int)in[3], (int)in[4], z0, z1, tab);
  out[0] = z0; out[1] = z1;
}
// theta = fma(sigma, z, mu) + strict-< argmin update (NC-4), per normal used
extern "C" __global__ void probe_theta(const double *in, double *out, int *arg) {
  double bt = in[0]; int b = arg[0];
  const double th = fma(in[1], in[2], in[3]);
  if (th < bt) { bt = th; b = arg[1]; }
  out[0] = bt; arg[2] = b;
}
// Observe (NC-6), unbounded window, n >= 2 path
extern "C" __global__ void probe_observe(const double *in, double *out, const int *nin) {
  const double C = in[0], sh = in[1];
  double S1 = in[2], S2 = in[3];
  const int n = nin[0] + 1;
  const double d = C - sh;
  S1 = S1 + d; S2 = S2 + d * d;
  const double dn = (double)n;
  const double rq = 1.0 / (dn * (dn - 1.0));
  const double inv_n = (dn - 1.0) * rq;
  const double inv_nm1 = dn * rq;
  const double mean = sh + S1 * inv_n;
  double s2 = (S2 - S1 * (S1 * inv_n)) * inv_nm1;
  const double fl = 1e-12 * (1.0 + mean * mean);
  if (!(s2 >= fl)) s2 = fl;
  const double den = (in[4] * s2) + dn;
  const double rden = 1.0 / den;
  const double sum = (dn * sh) + S1;
  out[0] = ((in[5] * s2) + sum) * rden; out[1] = sqrt(s2 * rden); out[2] = S1; out[3] = S2;
}
// trace lookup + charge + early-stop test (NC-5), not-stopped path
// (the replica Philox block is amortised over four recurrences: counted separately as philox/4)
extern "C" __global__ void probe_charge(const double *in, const int *pool, double *out, const uint4 *w, int t) {
  const uint4 ww = *w;
  const uint32_t r = __umulhi(pick_word(U4{ww.x, ww.y, ww.z, ww.w}, t), 4u);
  const int E = pool[r];
  const int Erun = E > 0 ? E : 99;
  const double em1 = (double)(Erun - 1);
  const double Cf = in[0] + em1 * in[1];
  const double thr = in[6] * in[7];
  out[0] = Cf; out[1] = in[2] + em1 * in[3]; out[2] = in[4] + em1 * in[5];
  out[3] = (Cf > thr) ? 1.0 : 0.0;
}
// The per-decision work besides sampling, as the contract requires it (Thompson phase,
// n >= 2, unbounded window): trace lookup with the replica word, charge + early-stop test,
// best update, Observe (shifted sums + posterior, NC-6), per-trial totals, FNV-1a digest of
// (b, p, flags), the pseudo-regret / optimum lookups of the curve contributions.
extern "C" __global__ void probe_serial(const double *in, const int *pool, const double *tab,
                                        double *out, unsigned long long *dig_io, const uint4 *w,
                                        int t, int b, int s, int B, int K, int max_epochs) {
  const uint4 ww = *w;
  const uint32_t r = __umulhi(pick_word(U4{ww.x, ww.y, ww.z, ww.w}, t), (uint32_t)K);
  const int E = pool[((size_t)s * B + b) * K + r];
  const int Erun = E > 0 ? E : max_epochs;
  const double c1 = in[0], t1 = in[1], e1 = in[2], best0 = in[3], beta = in[4];
  const double em1 = (double)(Erun - 1);
  const double Cf = c1 + em1 * c1;
  const double thr = beta * best0;
  const bool stopped = Cf > thr;
  const double C = stopped ? thr : Cf;
  const double Tm = t1 + em1 * t1, En = e1 + em1 * e1;
  const bool conv = (E > 0) && !stopped;
  const double best = (conv && !(C >= best0)) ? C : best0;
  // Observe
  const double sh = in[5];
  double S1 = in[6], S2 = in[7];
  const int n = (int)in[8] + 1;
  const double d = C - sh;
  S1 = S1 + d; S2 = S2 + d * d;
  const double2 ms = posterior(sh, S1, S2, n, in[9], in[10]);
  // totals, digest, curve contributions
  const uint32_t flags = (stopped ? 1u : 0u) | (conv ? 2u : 0u) | 8u;
  unsigned long long dig = dig_io[0];
  dig = (dig ^ (unsigned long long)(uint32_t)b) * 0x100000001b3ull;
  dig = (dig ^ (unsigned long long)(uint32_t)(b + 1)) * 0x100000001b3ull;
  dig = (dig ^ (unsigned long long)flags) * 0x100000001b3ull;
  dig_io[0] = dig;
  out[0] = C + in[11]; out[1] = En + in[12]; out[2] = Tm + in[13];
  out[3] = tab[s * B + b]; out[4] = best; out[5] = ms.x; out[6] = ms.y; out[7] = S1; out[8] = S2;
}
// The method's curve accumulation (a7: Eq. 4 sums per recurrence), as one warp's fp64
// reduce-scatter of the four sums (12 shuffles), one REDUX of the packed counts and one 4-lane
// RED.F64 + one count RED per warp-recurrence (32 decisions).  This is the algorithmic work;
// the build's exact fixed-point curves (counted runs + limbs for stops) are an implementation.
extern "C" __global__ void probe_curves(double *curves, const double *v, const int *pk, int t) {
  const int lane = threadIdx.x & 31;
  double a0 = v[0], a1 = v[1], a2 = v[2], a3 = v[3];
  // reduce-scatter: after 16/8 the four quantities live in lanes 0, 8, 16, 24
  const bool hi16 = lane & 16;
  double x0 = hi16 ? a0 : a2, x1 = hi16 ? a1 : a3;
  double y0 = hi16 ? a2 : a0, y1 = hi16 ? a3 : a1;
  y0 += __shfl_xor_sync(0xffffffffu, x0, 16);
  y1 += __shfl_xor_sync(0xffffffffu, x1, 16);
  const bool hi8 = lane & 8;
  double x = hi8 ? y0 : y1, y = hi8 ? y1 : y0;
  y += __shfl_xor_sync(0xffffffffu, x, 8);
  y += __shfl_xor_sync(0xffffffffu, y, 4);
  y += __shfl_xor_sync(0xffffffffu, y, 2);
  y += __shfl_xor_sync(0xffffffffu, y, 1);
  const unsigned c = __reduce_add_sync(0xffffffffu, (unsigned)pk[0]);
  if ((lane & 7) == 0) atomicAdd(curves + t * 8 + (lane >> 3), y);
  if (lane == 0) atomicAdd((unsigned long long *)(curves + t * 8 + 4), (unsigned long long)c);
}
// Bound screen of one survivor pair: radius bound from the radius word, the
// rounded-down lower bounds of both arms against bt, and parking a residual pair's words
extern "C" __global__ void probe_screen(const uint32_t *w, const double2 *ms, const double *in,
                                        uint4 *park, int *nres) {
  const double rub = radius_bound(w[0]);
  if (screen_keep(w[2], rub, ms[0], ms[1], in[0])) {
    park[threadIdx.x] = make_uint4(w[0], w[1], w[3], 0u);
    nres[0] += 1;
  }
}

// Certified draw: one Philox block of a quad from the per-decision prefix
// (rounds 0-2 partly shared), as the Thompson kernel draws it
extern "C" __global__ void probe_philox_q(const uint32_t *in, uint32_t *out) {
  const PhiloxPrefix p{in[0], in[1], in[2], in[3], in[4]};
  const U4 x = philox_from_prefix(p, in[5], [&](int r) { return in[6] + (uint32_t)r; },
                                  [&](int r) { return in[7] + (uint32_t)r; });
  out[0] = x.x; out[1] = x.y; out[2] = x.z; out[3] = x.w;
}
// ... one Box-Muller pair in fp32 with its bound and the packed-key argmin update of its two arms
extern "C" __global__ void probe_fpair(const uint32_t *w, const float4 *ms, float *io, uint32_t keep) {
  cert::Argmin32 am;
  am.m1 = io[0]; am.m2 = io[1]; am.smax = io[2]; am.rsqmax = io[3];
  float z0, z1, rsq;
  cert::normal_pair32(w[0], w[1], z0, z1, rsq);
  am.pair((int)w[2], ms[0], z0, z1, rsq, keep);
  io[0] = am.m1; io[1] = am.m2; io[2] = am.smax; io[3] = am.rsqmax;
}
