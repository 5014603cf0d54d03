// kernels.cuh -- the sm_100a kernels of the replay.
//
//   step1_kernel   Eq. 7 argmin over the power profile + per-arm constants +
//                  the known optimum per slice (a1 in SURVEY §8(a)).
//   replay_kernel  steps 2-4 for every (trial, recurrence): pruning (Alg. 3),
//                  Thompson sampling (Alg. 1), trace lookup, early stop
//                  (P:L559), Observe (Alg. 2), curves + digests (a2..a7).
//   curve_reduce   sums the atomic curve slots in a fixed order (a7).
//
// Layout: one thread per trial; per-cell tables (arm constants,
// the trace pool, pseudo-regret table) are staged once per block into shared
// memory with a 1-D TMA bulk copy (cp.async.bulk) completing on an mbarrier.
#pragma once
#include <cstdint>

#include "contract.cuh"
#include "certify.cuh"



#ifndef ZS_SLIM_B
#define ZS_SLIM_B 1
#endif
#ifndef ZS_QUAD_LOOP
#define ZS_QUAD_LOOP 1
#endif
#ifndef ZS_BOUND_SKIP
#define ZS_BOUND_SKIP 1
#endif
#ifndef ZS_PHASEA_CERT
#define ZS_PHASEA_CERT 1
#endif

namespace zs {

constexpr int kQ = 7;             // curve quantities
constexpr int kCounters = 14;   // 9 contract events + transforms, Philox blocks, pairs screened / in fp32,
                                // draws certified in fp32, exact fallbacks (thompson_kernel)

#ifndef ZS_ARMC_PACK
#define ZS_ARMC_PACK 0
#endif
#if ZS_ARMC_PACK
// the fields every decision reads (c1, t1, e1, p*) in the first 32 bytes: two 16-byte loads
struct __align__(16) ArmConst {   // per (cell, arm), 64 B
  double c1, t1, e1;
  int32_t pstar, pad0;
  double cP, tP, eP, pad1;
};
#else
struct ArmConst {                 // per (cell, arm), 64 B
  double c1, t1, e1, cP, tP, eP;
  int32_t pstar, pad0;
  double pad1;
};
#endif

struct CellParam {                // per cell
  double eta, beta, prec0, pm0;
  int32_t window, policy;         // policy: 0 Zeus, 1 Default, 2 Grid Search (§6.1)
  int32_t ablation, conc;         // Zeus ablations: bit0 no pruning, bit1 no JIT;
                                  // conc: an arrival schedule (concurrent submissions, f3)
  uint32_t key0, key1;
  int64_t begin, n, out_off;      // global first trial, shard size, offset into per-trial outputs
};

// ------------------------------------------------------------------ step 1
struct Step1Args {
  const double *A, *Th;           // [B][P]
  const int32_t *pool;            // [S][B][K]
  const CellParam *cells;
  ArmConst *arms;                 // [cells][B]
  double *regret;                 // [cells][reg_stride] (S*B used)
  double *opt;                    // [cells][S]
  int32_t *opt_arm;               // [cells][opt_stride] (S used)
  double *ebar;                   // [S][B] mean epochs of converged replicas (cell-independent)
  int B, P, S, K, max_epochs, reg_stride, opt_stride;
  double MP;
};

__global__ void step1_kernel(Step1Args a) {
  const int cell = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const double eta = a.cells[cell].eta;
  ArmConst *arms = a.arms + (size_t)cell * a.B;
  for (int b = warp; b < a.B; b += nwarp) {
    const double *A = a.A + (size_t)b * a.P;
    const double *Th = a.Th + (size_t)b * a.P;
    double bc = __longlong_as_double(0x7ff0000000000000ll);   // +inf
    int bp = 0x7fffffff;
    // per-p terms of the JIT epoch (1/Th, A/Th), computed by the lanes; lane 0 adds them in
    // ascending p below (NC-2: the same terms, the same left-to-right order)
    double term_t = 0.0, term_e = 0.0;
    for (int p = lane; p < a.P; p += 32) {                      // Eq. 7, lanes over p
      const double num = (eta * A[p]) + ((1.0 - eta) * a.MP);
      const double c = num / Th[p];
      if (c < bc) { bc = c; bp = p; }
      if (p < 32) { term_t = 1.0 / Th[p]; term_e = A[p] / Th[p]; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {                   // argmin, ties -> smaller p
      const double oc = __shfl_xor_sync(0xffffffffu, bc, off);
      const int op = __shfl_xor_sync(0xffffffffu, bp, off);
      if (oc < bc || (oc == bc && op < bp)) { bc = oc; bp = op; }
    }
    double st = 0.0, se = 0.0;                                  // JIT epoch, left-to-right (NC-2)
    for (int p = 0; p < a.P; ++p) {
      const double tt = (p < 32) ? __shfl_sync(0xffffffffu, term_t, p) : 1.0 / Th[p];
      const double te = (p < 32) ? __shfl_sync(0xffffffffu, term_e, p) : A[p] / Th[p];
      st = st + tt;
      se = se + te;
    }
    if (lane == 0) {
      if (bp == 0x7fffffff) bp = 0;
      ArmConst ac;
      ac.c1 = bc;
      ac.t1 = 1.0 / Th[bp];
      ac.e1 = A[bp] / Th[bp];
      ac.tP = st / (double)a.P;
      ac.eP = se / (double)a.P;
      ac.cP = (eta * ac.eP) + (((1.0 - eta) * a.MP) * ac.tP);
      ac.pstar = bp;
      ac.pad0 = 0;
      ac.pad1 = 0.0;
      arms[b] = ac;
    }
  }
  __syncthreads();
  for (int s = threadIdx.x; s < a.S; s += blockDim.x) {        // known optimum
    // (pool reads are independent loads; the compiler keeps them in flight)
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int barg = -1;
    for (int b = 0; b < a.B; ++b) {
      long long sum = 0;
      int cnt = 0;
      for (int k = 0; k < a.K; ++k) {
        const int E = a.pool[((size_t)s * a.B + b) * a.K + k];
        if (E > 0) { sum += E; ++cnt; }
      }
      if (cnt > 0) {
        const double v = ((double)sum / (double)cnt) * arms[b].c1;
        if (v < best) { best = v; barg = b; }
      }
    }
    a.opt[(size_t)cell * a.S + s] = best;
    a.opt_arm[(size_t)cell * a.opt_stride + s] = barg;
    for (int b = 0; b < a.B; ++b) {
      long long sum = 0;
      int cnt = 0;
      for (int k = 0; k < a.K; ++k) {
        const int E = a.pool[((size_t)s * a.B + b) * a.K + k];
        if (E > 0) { sum += E; ++cnt; }
      }
      const double eb = cnt > 0 ? (double)sum / (double)cnt : (double)a.max_epochs;
      a.regret[(size_t)cell * a.reg_stride + (size_t)s * a.B + b] = eb * arms[b].c1 - best;
      if (cell == 0) a.ebar[(size_t)s * a.B + b] = eb;
    }
  }
}

// ------------------------------------------------------------------ replay
struct ReplayArgs {
  const CellParam *cells;
  const ArmConst *arms;           // [cells][B]
  const double *regret;           // [cells][reg_stride]
  const int32_t *opt_arm;         // [cells][opt_stride]
  const int32_t *pool;            // [S][B][K], allocation padded to 16 B
  long long *curve_slots;         // [cells][nslot][R][kQ][kLimbs] fixed point (curve_accumulate)
  double curve_scale;             // 2^F of the fixed point
  double *tot_cost, *tot_energy, *tot_time;
  unsigned long long *digest;
  int32_t *n_stop, *final_arm;
  uint32_t *log;                  // [out][R] or null
  unsigned long long *counters;   // [kCounters]
  int B, S, K, R, max_epochs, charge_profiling, b0, nslot, reg_stride, opt_stride;
  int tab_bytes;                  // bytes of the staged table region (multiple of 16)
  // Observe statistics in global memory, one 32-byte record per (trial, arm):
  // [trial][arm] -- a lane touches one sector per decision whichever trial it runs
  struct ArmStat *st;
  double *st_ring;                // [trial][arm][ring_n] when some cell has a window
  int ring_n;
  // two-phase schedule: phase A runs t < t_split (the pruning
  // stage, <= 2B recurrences), phase B the Thompson-sampling rest with trials
  // regrouped so the lanes of a warp draw the same number of normal pairs
  int t_split;
  // Counted curves (no ablation): a run that is not early-stopped is fully determined by its
  // class (Thompson decision?, paid the profiling epoch?), b and replica at recurrence t, so its
  // curve values are counted, not summed: hist[cell][R][nhslot][4][B][K] (u32), folded into the
  // exact fixed-point sums by curve_hist_fold_kernel after the replay
  uint32_t *hist;
  int nhslot;
  struct Carry *carry;            // [stride] per-trial scalar state between phases
  int32_t *perm;                  // [stride] phase-B lane -> trial (within each cell's block)
  int32_t *bucket;                // [cells][nwin][kBuckets] histogram, then running offsets
  int nwin;                       // regroup windows per cell
  const double2 *logtab;          // [kLogTab] the sampler's log table (NC-3)
  // ablation path only (ABL): the raw profile, Ebar and the optimum for off-p* charges
  const double *A, *Th, *ebar, *opt;
  int P;
  double MP;
  // RK launches (one cell, grid.y = 1): the cell's Philox round keys, read by the rounds as
  // constant-bank operands instead of being recomputed as k + r W in every block
  RoundKeys rk;
  // the Thompson phase runs thompson_kernel (certified fp32 draw): phase A
  // then groups the lanes by survivor-quad count; force_exact sends every draw to its exact
  // fp64 fallback (a test of that path)
  int key_quads, force_exact;
  // early split (thompson_kernel only): phase A stops each lane at its first pure Thompson
  // decision (pruning over, every survivor observed twice) and the Thompson phase starts that
  // lane there (Carry::t0), so phase A's warps never mix pruning and sampling lanes
  int early_split;
  // replay_kernel's one-pass and exact phase-B schedules: the certified fp32 draw (draw = 0 or 2)
  // instead of the bound screen; its fp32 table follows the residual slots in shared memory
  int cert_draw;
  // thompson_kernel<…, WIN>'s shared-memory table layout (ThTabLayout, computed on the host)
  int th_logtab, th_pool, th_bytes, th_pool_smem;
};

// regroup keys: 2 x popcount of the survivor-pair mask + parity of its lowest pair (exact phase B),
// or quads x kT0Keys + the recurrence the lane's Thompson phase starts at (thompson_kernel, t0 <= 2B)
constexpr int kT0Keys = 65;
#ifndef ZS_ACT_REG_A
#define ZS_ACT_REG_A 1      // CFG5 +0.25 % (session r02dc)
#endif
#ifndef ZS_CONC_MIN
#define ZS_CONC_MIN 1
#endif
#ifndef ZS_QUADS_DESC
#define ZS_QUADS_DESC 0
#endif
constexpr int kBuckets = 9 * kT0Keys;
#ifndef ZS_REGROUP_WINDOW
#define ZS_REGROUP_WINDOW 8192
#endif
constexpr int kRegroupWindow = ZS_REGROUP_WINDOW;   // trials regrouped together (multiple of 128)

// Philox blocks a draw over `pairs` takes: one per quad (two pairs) touched
__device__ __forceinline__ uint32_t quads_of(uint32_t pairs) {
  uint32_t q = 0;
  for (int k = 0; k < 32; k += 2) q |= ((pairs >> k) & 3u) ? (1u << (k >> 1)) : 0u;
  return q;
}

// phase-B grouping key: lanes with the same number of survivor pairs and the same parity of
// the lowest one draw the same number of Philox blocks at the same loop steps
__device__ __forceinline__ int regroup_key(uint32_t pairs, int key_quads, int t0) {
#if ZS_QUADS_DESC
  // thompson_kernel: quads (descending: a window's slow warps are dispatched first, so the launch
  // ends on short ones), then the start recurrence
  if (key_quads) return (8 - __popc(quads_of(pairs))) * kT0Keys + t0;
#else
  if (key_quads) return __popc(quads_of(pairs)) * kT0Keys + t0;   // thompson_kernel: quads, start
#endif
  return pairs ? 2 * __popc(pairs) + ((__ffs(pairs) - 1) & 1) : 0;
}

struct __align__(16) ArmStat {    // Observe state of one arm of one trial (NC-6)
  double sh, S1, S2;              // shift (first observation) and shifted sums
  int32_t cnt, pad;               // observations ever
};

// The Observe records of one trial, [trial][arm] 32 B each, addressed by a 32-bit index from the
// uniform base (zeus_sim_create keeps shard x |B| < 2^32): one add and one wide multiply per
// access instead of 64-bit pointer arithmetic (thompson.cuh ZS_REC32)
struct RecRef {
  ArmStat *base;
  uint32_t ob;
  __device__ __forceinline__ ArmStat &operator[](int arm) const {
    return *reinterpret_cast<ArmStat *>(reinterpret_cast<char *>(base) + (uint64_t)(ob + (uint32_t)arm) * 32u);
  }
};

// per-trial scalar state carried from phase A to phase B (96 B)
struct Carry {
  double best, totC, totE, totT;
  unsigned long long dig;
  uint32_t profiled, seen, mature, ts_set;
  int32_t nstop, last_b;
  uint32_t n_sampled, n_prune, n_forced, n_recomp;
  uint32_t n_cert, n_fall;        // phase A's certified draws and their exact fallbacks
  int32_t t0, pad;                // the lane's first Thompson-phase recurrence (t_split, or earlier
};                                // under ReplayArgs::early_split)

// shared-memory table region of one block: [ArmConst B][regret S*B][opt_arm S][pool S*B*K]
struct TabLayout {
  int arms, regret, optarm, pool, logtab, bytes;
  __host__ __device__ static int align16(int x) { return (x + 15) & ~15; }
  __host__ __device__ TabLayout(int B, int S, int K) {
    arms = 0;
    regret = align16(arms + B * (int)sizeof(ArmConst));
    optarm = align16(regret + S * B * 8);
    pool = align16(optarm + S * 4);
    logtab = align16(pool + S * B * K * 4);
    bytes = logtab + kLogTab * 16;
  }
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// Curves in exact fixed point (bitwise the same whatever the world size, the
// layout or the order of the atomics).  A trial's value v of quantity q at recurrence t becomes
// the integer Q = RN(v 2^F) (|Q| < 2^61; F is chosen on the host from an upper bound of v, so
// the quantisation is < 2^-F absolute), split into limbs Q = l0 + l1 2^26 + l2 2^52 with
// 0 <= l0, l1 < 2^26.  Every limb is summed over the warp by one REDUX (32 lanes x 2^26 < 2^31,
// exact) and added to a 64-bit slot counter by one red.global.add.u64 (exact); integer sums do
// not depend on order, so neither do the curves.  curve_reduce_kernel adds the slots, carries
// the limbs and rounds once to fp64.  Counts (stops | optimal << 8 | Thompson << 16, packed
// 8 bits each) are summed by one REDUX and added to limb 0.  All 32 lanes must call it.
constexpr int kLimbs = 3, kLimbBits = 26;
constexpr int kRow = kQ * kLimbs;   // int64 per (slot, recurrence)
__device__ __forceinline__ void red_add_u64(long long *p, unsigned long long v, bool pred) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n @p red.global.add.u64 [%0], %1;\n}"
               :: "l"(p), "l"(v), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void red_add_u32(uint32_t *p, uint32_t v) {
  asm volatile("red.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
// the same, predicated in PTX (no branch around it): the increment is 1 when pred holds
__device__ __forceinline__ void red_inc_u32_if(uint32_t *p, bool pred) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q red.global.add.u32 [%0], 1;\n\t}"
               :: "l"(p), "r"((uint32_t)pred) : "memory");
}
__device__ __forceinline__ void curve_accumulate(long long *curves, int t, int lane, double vC,
                                                 double vE, double vT, double vReg, int vPacked,
                                                 double scale) {
  long long *row = curves + (size_t)t * kRow;
  const bool l0 = lane == 0;
  const double v[4] = {vC, vE, vT, vReg};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const long long Q = __double2ll_rn(v[q] * scale);
    const unsigned a0 = (unsigned)Q & 0x3ffffffu;
    const unsigned a1 = (unsigned)(Q >> kLimbBits) & 0x3ffffffu;
    const int a2 = (int)(Q >> (2 * kLimbBits));
    const unsigned s0 = __reduce_add_sync(0xffffffffu, a0);
    const unsigned s1 = __reduce_add_sync(0xffffffffu, a1);
    const int s2 = __reduce_add_sync(0xffffffffu, a2);
    red_add_u64(row + q * kLimbs, s0, l0 && s0);
    red_add_u64(row + q * kLimbs + 1, s1, l0 && s1);
    red_add_u64(row + q * kLimbs + 2, (unsigned long long)(long long)s2, l0 && s2);
  }
  const unsigned pk = __reduce_add_sync(0xffffffffu, (unsigned)vPacked);   // REDUX
  red_add_u64(row + 4 * kLimbs, pk & 0xffu, l0 && (pk & 0xffu));
  red_add_u64(row + 5 * kLimbs, (pk >> 8) & 0xffu, l0 && ((pk >> 8) & 0xffu));
  red_add_u64(row + 6 * kLimbs, (pk >> 16) & 0xffu, l0 && ((pk >> 16) & 0xffu));
}

// 1-D bulk copy global -> shared through the TMA unit, completion on an mbarrier.
__device__ __forceinline__ void tma_bulk_load(void *dst_smem, const void *src, uint32_t bytes,
                                              uint64_t *mbar) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(d), "l"(src), "r"(bytes), "r"(m) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(m), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, uint32_t bytes) {
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(m), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t phase) {
  const uint32_t m = (uint32_t)__cvta_generic_to_shared(mbar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" :: "r"(m), "r"(phase) : "memory");
}

enum : int { kStart = 0, kDown = 1, kUp = 2 };

// Bound screen.  An upper bound of |z0|, |z1| for the Box-Muller pair of
// radius word a: u1 = (a+1) 2^-32 > 2^-(clz(a)+1), so r^2 = -2 log u1 < 2 ln2 (clz(a)+1), and
// sqrt(x) lies below its tangents at x = 2 ln2 and x = 6 ln2 (sqrt is concave).  The constants
// carry a 2^-29 margin, far above the rounding of the computed r, cos and sin.
ZS_C(kRubSlope0, 0.5887050123542859);     // tangent of sqrt(2 ln2 x) at x = 1: slope = intercept
ZS_C(kRubSlope1, 0.3398889973560289);     // tangent at x = 3
ZS_C(kRubIcpt1, 1.0196669920680868);
// The same two tangents with their coefficients rounded up to 20-bit mantissas (larger, so still
// upper bounds), which DFMA takes as immediates; the tangent at clz(a) = 0 is the constant
// 2 x 0x1.2d6acp-1, and for clz(a) >= 1 the second tangent is the smaller of the two.
__device__ __forceinline__ double radius_bound(uint32_t a) {
  const double cc = (double)(__clz(a) + 1);
  const double l2 = __fma_ru(cc, 0x1.5c0bep-2, 0x1.0508fp+0);
  return ((int)a < 0) ? 0x1.2d6acp+0 : l2;
}
// Can an arm of this pair (bits `two`: arms 2k, 2k+1 in the survivor set) still beat the best
// sample bt?  theta = fma(sigma, z, mu) >= RD(mu - sigma rub) for |z| <= rub, and rounding is
// monotone, so RD(mu - sigma rub) > bt proves theta > bt: the arm can neither win nor tie.
// Branch-free: both bounds are evaluated (a non-survivor's slot may hold anything; its bit masks it).
__device__ __forceinline__ bool screen_keep(uint32_t two, double rub, double2 m0, double2 m1, double bt) {
  const bool out0 = __fma_rd(-m0.y, rub, m0.x) > bt;
  const bool out1 = __fma_rd(-m1.y, rub, m1.x) > bt;
  return ((two & 1u) && !out0) | ((two & 2u) && !out1);
}
constexpr int kResSlots = 2;   // residual pairs whose words are parked in shared memory

// Alg. 2 posterior from the shifted window sums (NC-6), n >= 2: returns (mu, sigma).
__device__ __forceinline__ double2 posterior(double sh, double S1, double S2, int n, double prec0,
                                             double pm0) {
  const double dn = (double)n;
  const double rq = 1.0 / (dn * (dn - 1.0));             // 1/n and 1/(n-1) from one division
  const double inv_n = (dn - 1.0) * rq;
  const double inv_nm1 = dn * rq;
  const double mean = sh + S1 * inv_n;
  double s2 = (S2 - S1 * (S1 * inv_n)) * inv_nm1;        // σ̃² = Var(C_b), n-1 divisor
  const double fl = cst::kVarFloor * (1.0 + mean * mean);
  if (!(s2 >= fl)) s2 = fl;                              // zero-variance floor (R-Q7)
  // σ̂² = (1/σ̂0² + n/σ̃²)^-1 = σ̃²/(σ̃²/σ̂0² + n);  μ̂ = σ̂²(μ̂0/σ̂0² + Sum/σ̃²)
  // = (σ̃² μ̂0/σ̂0² + Sum)/(σ̃²/σ̂0² + n): one reciprocal of the shared denominator
  const double den = (prec0 * s2) + dn;
  const double rden = 1.0 / den;
  const double sum = (dn * sh) + S1;                     // Sum(C_b)
  const double var = s2 * rden;
  return make_double2(((pm0 * s2) + sum) * rden, sqrt(var));
}

__device__ __forceinline__ uint32_t below_mask(int c) { return c <= 0 ? 0u : ((1u << c) - 1u); }
__device__ __forceinline__ uint32_t above_mask(int c) { return c >= 31 ? 0u : ~((2u << c) - 1u); }

// One thread per trial.  WINDOWED: some cell has N > 0 (ring buffer per arm).
// LOG: write the per-decision log.  PHASE: 0 = all recurrences in one pass,
// 1 = phase A (t < t_split, then save the carry), 2 = phase B (t >= t_split,
// lanes mapped through perm; every trial is already in Thompson sampling).
//
// State placement:
//   registers  per-trial scalars: best, the Alg. 3 state machine, bitmasks
//              (profiled, seen, mature = n >= 2, survivors), totals, digest;
//   smem       (mu, sigma) per arm as double2 [arm][thread] -- read for every
//              survivor in every Thompson draw;
//   global     the Observe statistics (sh, S1, S2, cnt, ring) [arm][trial],
//              touched once per decision for the chosen arm only; the working
//              set of resident trials (~30 MB) stays in L2.
#ifdef ZS_MAXNREG
#define ZS_REPLAY_BOUNDS __maxnreg__(ZS_MAXNREG)
#elif defined(ZS_P2_MIN_BLOCKS)
#define ZS_REPLAY_BOUNDS __launch_bounds__(128, (PHASE == 2 ? ZS_P2_MIN_BLOCKS : 1))
#elif defined(ZS_P1_MIN_BLOCKS)
#define ZS_REPLAY_BOUNDS __launch_bounds__(128, (PHASE == 1 ? ZS_P1_MIN_BLOCKS : 1))
#else
#define ZS_REPLAY_BOUNDS __launch_bounds__(128)
#endif
template <bool WINDOWED, bool LOG, int PHASE, bool ABL, bool RK>
__global__ void ZS_REPLAY_BOUNDS replay_kernel(ReplayArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  const int cell = blockIdx.y;
  const CellParam cp = a.cells[cell];
  // Philox blocks of this cell (NC-3); RK launches take the round keys from the parameters
  auto pair_block_c = [&](int64_t tr, int tt, int q) -> U4 {
    if constexpr (RK) return pair_block(a.rk, tr, tt, q);
    else return pair_block(cp.key0, cp.key1, tr, tt, q);
  };
  auto replica_words_c = [&](int64_t tr, int tt) -> U4 {
    if constexpr (RK) return replica_words(a.rk, tr, tt);
    else return replica_words(cp.key0, cp.key1, tr, tt);
  };
  const int tid = threadIdx.x, TPB = blockDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * TPB;
  if (j0 >= cp.n || cp.policy != 0 || cp.conc) return;    // past the shard / another kernel's cell

  // ---- stage the cell's tables with TMA bulk copies (one elected thread)
  const TabLayout L(a.B, a.S, a.K);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    const uint32_t b_arm = a.B * (uint32_t)sizeof(ArmConst);
    const uint32_t b_reg = a.S * a.B * 8u;
    const uint32_t b_opt = a.S * 4u;
    const uint32_t b_pool = a.S * a.B * a.K * 4u;
    // bulk copies need 16-byte sizes; the host pads every table to 16 B
    const uint32_t p_arm = (b_arm + 15u) & ~15u, p_reg = (b_reg + 15u) & ~15u;
    const uint32_t p_opt = (b_opt + 15u) & ~15u, p_pool = (b_pool + 15u) & ~15u;
    mbar_expect_tx(&mbar, p_arm + p_reg + p_opt + p_pool + kLogTab * 16u);
    tma_bulk_load(smem + L.logtab, a.logtab, kLogTab * 16u, &mbar);
    tma_bulk_load(smem + L.arms, a.arms + (size_t)cell * a.B, p_arm, &mbar);
    tma_bulk_load(smem + L.regret, a.regret + (size_t)cell * a.reg_stride, p_reg, &mbar);
    tma_bulk_load(smem + L.optarm, a.opt_arm + (size_t)cell * a.opt_stride, p_opt, &mbar);
    tma_bulk_load(smem + L.pool, a.pool, p_pool, &mbar);
  }
  __syncthreads();
  mbar_wait(&mbar, 0);

  const ArmConst *arm = reinterpret_cast<const ArmConst *>(smem + L.arms);
  const double *regret = reinterpret_cast<const double *>(smem + L.regret);
  const int32_t *optarm = reinterpret_cast<const int32_t *>(smem + L.optarm);
  const int32_t *pool = reinterpret_cast<const int32_t *>(smem + L.pool);
  const double2 *logtab = reinterpret_cast<const double2 *>(smem + L.logtab);
  const int B = a.B, R = a.R, S = a.S, K = a.K;
  double2 *s_ms = reinterpret_cast<double2 *>(smem + a.tab_bytes);   // [arm][thread] (mu, sigma)

  const bool active = j0 + tid < cp.n;
  int64_t jj = j0 + tid;                                    // this lane's trial within the cell
  if (PHASE == 2) jj = active ? a.perm[cp.out_off + j0 + tid] : 0;
  const int64_t trial = cp.begin + jj;
  const size_t o = (size_t)(cp.out_off + jj);              // this trial's row in the outputs/state
  const RecRef st{a.st, (uint32_t)(o * B)};               // the trial's Observe records (32-bit index)
  const int warp_global = blockIdx.x * (TPB >> 5) + (tid >> 5);
  long long *curves = a.curve_slots + ((size_t)cell * a.nslot + (warp_global % a.nslot)) * (size_t)R * kRow;
  constexpr bool kHist = !ABL;                              // counted curves (see ReplayArgs::hist)
  const int HB = 4 * B * K;                                 // bins per (cell, t, slot)
  uint32_t *hist = a.hist + ((size_t)cell * R * a.nhslot + (warp_global % a.nhslot)) * (size_t)HB;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);

  uint32_t profiled = 0, seen = 0, mature = 0;              // bit a: profiled / observed / n_a >= 2
  double best = kInf;                                       // min_t C_t
  bool in_ts = PHASE == 2;
  int round = 1, step = kStart, start = a.b0, cursor = a.b0;
  const uint32_t all_arms = (B == 32) ? 0xffffffffu : ((1u << B) - 1u);
  uint32_t cand = all_arms, surv = 0, ts_set = 0, ts_pairs = 0;
  double r1_cost = kInf;
  int r1_arm = -1;
  double totC = 0.0, totE = 0.0, totT = 0.0;
  unsigned long long dig = 0xcbf29ce484222325ull;
  int nstop = 0, last_b = -1;
  // event counters (u32 per trial; the pair/normal counts follow from n_sampled
  // because the survivor set is fixed during Thompson sampling)
  // (phase B counts from zero and adds phase A's carried counts at the end; every draw of
  // this kernel past phase A is screened, so the screened draws are n_sampled here)
  uint32_t n_sampled = 0, n_prune = 0, n_forced = 0, n_recomp = 0;
  uint32_t n_resid = 0;                                     // bound screen: residual pairs
  uint32_t n_cert = 0, n_fall = 0;                          // certified draw (a.cert_draw)
  // certified draw: fp32 (mu - ref, sigma) per arm, [pair][thread] float4, after
  // the residual slots; ref = the leader's posterior mean when Thompson sampling starts
  const int cpairs2 = ((((B + 1) >> 1) + 1) & ~1);
  float2 *s_f2 = reinterpret_cast<float2 *>(smem + a.tab_bytes + (size_t)((B + 1) & ~1) * 16 * TPB +
                                            (size_t)kResSlots * 16 * TPB);
  const int ckbits = 32 - __clz(2 * cpairs2 - 1);
  const uint32_t ckeep = ~((1u << ckbits) - 1u);
  const float ckth = cert::kTheta + __int_as_float((127 - 23 + ckbits) << 23) * 1.000001f;
  double cref = 0.0;
  float c_trial = 0.0f;
  // (under the early split phase A never draws: a lane stops at its first pure Thompson decision,
  // so its fp32 table is not built here -- the Thompson phase builds its own)
  const bool cert_on = (PHASE != 1 || ZS_PHASEA_CERT) && a.cert_draw && !(PHASE == 1 && a.early_split);
  auto f32_slot = [&](int arm_i, double2 ms) {              // (mu - ref, sigma) in fp32
    const double dm = ms.x - cref;
    s_f2[2 * ((arm_i >> 1) * TPB + tid) + (arm_i & 1)] =
        (fabs(dm) < 1e30 && ms.y < 1e30) ? make_float2((float)dm, (float)ms.y)
                                         : make_float2(0.0f, __int_as_float(0x7f800000));
  };
  // (re)build the fp32 table when Thompson sampling starts: survivors with n >= 2 from their fp64
  // posteriors, the rest (and the padding pair) as non-survivor sentinels
  auto cert_begin = [&]() {
    const int lead = (last_b >= 0 && ((ts_set >> last_b) & 1u) && ((mature >> last_b) & 1u))
                         ? last_b : __ffs(ts_set & mature) - 1;
    cref = lead >= 0 ? s_ms[lead * TPB + tid].x : 0.0;
    if (!(fabs(cref) < 1e30)) cref = 0.0;
    c_trial = __double2float_ru(fabs(cref) * 0x1p-52 + 0x1p-120);
    // every slot a sentinel (one 16-byte store per pair), then the survivors' values: this runs
    // where a lane's pruning ends, divergently, so its length is paid per distinct ending
    for (int k = 0; k < cpairs2; ++k)
      reinterpret_cast<float4 *>(s_f2)[k * TPB + tid] = make_float4(3.0e38f, 0.0f, 3.0e38f, 0.0f);
    for (uint32_t m = ts_set & mature; m; m &= m - 1u) {
      const int arm_i = __ffs(m) - 1;
      f32_slot(arm_i, s_ms[arm_i * TPB + tid]);
    }
  };
  if (PHASE == 2 && active) {                               // resume from phase A
    const Carry c = a.carry[o];
    best = c.best; totC = c.totC; totE = c.totE; totT = c.totT; dig = c.dig;
    profiled = c.profiled; seen = c.seen; mature = c.mature; ts_set = c.ts_set;
    nstop = c.nstop; last_b = c.last_b;
    for (int k = 0; 2 * k < B; ++k)
      if ((ts_set >> (2 * k)) & 3u) ts_pairs |= 1u << k;
    for (int b = 0; b < B; ++b) {                           // posterior of every arm with n >= 2,
      if (!((mature >> b) & 1u)) continue;                  // recomputed from its window sums
      const ArmStat q = st[b];                              // (same formula, same bits)
      const int n = (WINDOWED && cp.window > 0) ? min(q.cnt, cp.window) : q.cnt;
      s_ms[b * TPB + tid] = posterior(q.sh, q.S1, q.S2, n, cp.prec0, cp.pm0);
    }
    if (cert_on) cert_begin();
  }

  const int t_begin = PHASE == 2 ? a.t_split : 0;
  const int t_end = PHASE == 1 ? a.t_split : R;
  int s = 0;                                                // slice of t = floor(t*S/R) (R-Q19)
  U4 rw{0u, 0u, 0u, 0u};
  // the Observe record of the last arm observed, kept in registers: Thompson sampling mostly
  // repeats its arm, and then the decision needs no load of the record (same values)
  ArmStat qc{0.0, 0.0, 0.0, 0, 0};
  int qc_b = -1;
#if ZS_ACT_REG_A
  // `active` through an opaque register (ptxas otherwise re-evaluates the 64-bit bound check)
  uint32_t act_r;
  asm volatile("mov.u32 %0, %1;" : "=r"(act_r) : "r"(active ? 1u : 0u));
  bool live = act_r != 0u;                                  // phase A under early_split: until t0
#else
  bool live = active;                                       // phase A under early_split: until t0
#endif
  int t0 = t_end;
  for (int t = t_begin; t < t_end; ++t) {
    if (PHASE == 1 && a.early_split) {
      // the first pure Thompson decision (pruning over, every survivor observed twice) is the
      // Thompson phase's: this lane stops here and resumes there (thompson_kernel, Carry::t0)
      if (live && in_ts && !(ts_set & ~mature)) { live = false; t0 = t; }
      if (!__any_sync(0xffffffffu, live)) break;
    }
    double vC = 0.0, vE = 0.0, vT = 0.0, vReg = 0.0;
    int vPacked = 0;
    // carried from the decision to the Observe, which runs after the curve reduction so
    // the latency of the arm-state load hides behind the shuffles
    int b = 0;
    bool was_seen = false;
    double y_old = 0.0;                                     // windowed: the cost leaving the window
    int hkey = -1;                                          // (b, replica) of a counted run
    double C = 0.0;
    if (S > 1)                                              // no 64-bit division per decision
      while ((long long)(s + 1) * R <= (long long)t * S) ++s;
    if (live) {
      // step 3's replica words: one Philox block per four recurrences (NC-3), refreshed when
      // t enters a new block of four; warp-uniform because all lanes share t
      if ((t & 3) == 0 || t == t_begin) rw = replica_words_c(trial, t);
      // ---------------- step 2: decide b_t
      const bool ts_dec = in_ts;
      if (PHASE != 2 && !in_ts) {
        b = (step == kStart) ? start
          : (step == kDown) ? 31 - __clz(cand & below_mask(cursor))
                            : __ffs(cand & above_mask(cursor)) - 1;
        n_prune += 1;
      } else {
        const uint32_t unripe = ts_set & ~mature;
        if (unripe) {
          b = __ffs(unripe) - 1;                            // explore arms with n < 2 first
          n_forced += 1;
        } else {
          // Alg. 1: θ_a ~ N(μ_a, σ_a²) for every survivor, b = argmin θ.  Each lane walks
          // only its own survivor pairs (ascending k keeps the strict-< tie rule).
          double bt = kInf;
          b = -1;
          uint32_t pm = ts_pairs;
          auto consider = [&](int k, double z0, double z1) {   // branch-free (selects)
            const uint32_t two = (ts_set >> (2 * k)) & 3u;
            const double2 m0 = s_ms[(2 * k) * TPB + tid];
            const double2 m1 = s_ms[(2 * k + 1) * TPB + tid];
            const double th0 = fma(m0.y, z0, m0.x);
            const bool take0 = (two & 1u) && (th0 < bt);
            bt = take0 ? th0 : bt;
            b = take0 ? 2 * k : b;
            const double th1 = fma(m1.y, z1, m1.x);
            const bool take1 = (two & 2u) && (th1 < bt);
            bt = take1 ? th1 : bt;
            b = take1 ? 2 * k + 1 : b;
          };
          // pairs 2q and 2q+1 share one Philox block: it is drawn when the walk enters a new
          // quad (warp-uniform in phase B, where lanes are grouped by count and parity)
#if ZS_BOUND_SKIP
          if (cert_on) {
            // certified fp32 draw; not certified: the exact loop below
            cert::Argmin32 am;
            am.init();
            uint32_t qm = quads_of(ts_pairs);
            while (qm) {
              const int qd = __ffs(qm) - 1;
              qm &= qm - 1u;
              const U4 x = pair_block_c(trial, t, qd);
              const float4 f0 = reinterpret_cast<const float4 *>(s_f2)[(2 * qd) * TPB + tid];
              const float4 f1 = reinterpret_cast<const float4 *>(s_f2)[(2 * qd + 1) * TPB + tid];
              float z0, z1, rsq;
              cert::normal_pair32(x.x, x.y, z0, z1, rsq);
              am.pair(4 * qd, f0, z0, z1, rsq, ckeep);
              cert::normal_pair32(x.z, x.w, z0, z1, rsq);
              am.pair(4 * qd + 2, f1, z0, z1, rsq, ckeep);
            }
            if (am.certified(c_trial, ckth) && !a.force_exact) {
              b = am.arg(ckeep);
              pm = 0u;
              n_cert += 1;
            } else {
              n_fall += 1;
            }
          } else if (PHASE != 1) {
            // bound screen (exact): draw the pair of the leader (the previous
            // decision's arm) first; then an arm a can only win if mu_a - sigma_a r_ub <= bt,
            // r_ub >= |z| bounded from the pair's radius word alone.  Pairs that fail the
            // screen are transformed afterwards ("residuals"); ties keep the lowest arm.
            uint4 *s_res = reinterpret_cast<uint4 *>(smem + a.tab_bytes + (size_t)((B + 1) & ~1) * 16 * TPB);
            const int lead = (last_b >= 0 && ((ts_set >> last_b) & 1u)) ? last_b : __ffs(ts_set) - 1;
            const int kl = lead >> 1, ql = kl >> 1;
            const U4 xl = pair_block_c(trial, t, ql);
            {
              double z0, z1;
              box_muller((kl & 1) ? xl.z : xl.x, (kl & 1) ? xl.w : xl.y, z0, z1, logtab);
              consider(kl, z0, z1);
            }
            uint32_t res = 0u;                               // residual pairs past the slots
            int nres = 0;
            auto screen = [&](int k, uint32_t aw, uint32_t bw, double2 m0, double2 m1) {
              if (screen_keep((ts_set >> (2 * k)) & 3u, radius_bound(aw), m0, m1, bt)) {
                if (nres < kResSlots) s_res[nres * TPB + tid] = make_uint4(aw, bw, (uint32_t)k, 0u);
                else res |= 1u << k;              // past the slots: its Philox block is redrawn
                ++nres;
              }
            };
            const int ks = kl ^ 1;                           // the leader quad's other pair
            if ((ts_pairs >> ks) & 1u)
              screen(ks, (ks & 1) ? xl.z : xl.x, (ks & 1) ? xl.w : xl.y, s_ms[(2 * ks) * TPB + tid],
                     s_ms[(2 * ks + 1) * TPB + tid]);
            uint32_t qm = quads_of(ts_pairs) & ~(1u << ql);
            while (qm) {
              const int qd = __ffs(qm) - 1;
              qm &= qm - 1u;
              const U4 xq = pair_block_c(trial, t, qd);
              const uint32_t need = (ts_pairs >> (2 * qd)) & 3u;
              if (need & 1u)
                screen(2 * qd, xq.x, xq.y, s_ms[(4 * qd) * TPB + tid], s_ms[(4 * qd + 1) * TPB + tid]);
              if (need & 2u)
                screen(2 * qd + 1, xq.z, xq.w, s_ms[(4 * qd + 2) * TPB + tid], s_ms[(4 * qd + 3) * TPB + tid]);
            }
            auto consider_tie = [&](int k, double z0, double z1) {
              const uint32_t two = (ts_set >> (2 * k)) & 3u;
              const double2 m0 = s_ms[(2 * k) * TPB + tid];
              const double2 m1 = s_ms[(2 * k + 1) * TPB + tid];
              const double th0 = fma(m0.y, z0, m0.x);
              const bool take0 = (two & 1u) && (th0 < bt || (th0 == bt && 2 * k < b));
              bt = take0 ? th0 : bt;
              b = take0 ? 2 * k : b;
              const double th1 = fma(m1.y, z1, m1.x);
              const bool take1 = (two & 2u) && (th1 < bt || (th1 == bt && 2 * k + 1 < b));
              bt = take1 ? th1 : bt;
              b = take1 ? 2 * k + 1 : b;
            };
            n_resid += nres;
            if (nres > kResSlots)                            // rare: straight to the counter
              atomicAdd(a.counters + 10, (unsigned long long)(nres - kResSlots));
            for (int i = 0; i < nres && i < kResSlots; ++i) {
              const uint4 e = s_res[i * TPB + tid];
              double z0, z1;
              box_muller(e.x, e.y, z0, z1, logtab);
              consider_tie((int)e.z, z0, z1);
            }
            while (res) {
              const int k = __ffs(res) - 1;
              res &= res - 1u;
              const U4 xq = pair_block_c(trial, t, k >> 1);
              double z0, z1;
              box_muller((k & 1) ? xq.z : xq.x, (k & 1) ? xq.w : xq.y, z0, z1, logtab);
              consider_tie(k, z0, z1);
            }
            pm = 0u;
          } else
#endif
#if ZS_QUAD_LOOP
          if (PHASE == 2) {
            // quad loop: the two pairs of one Philox block are transformed side by side (two
            // independent Box-Muller chains in one basic block); which pairs of a quad a lane
            // needs is warp-uniform here (lanes grouped by pair count and parity)
            uint32_t qm = quads_of(ts_pairs);
            while (qm) {
              const int qd = __ffs(qm) - 1;
              qm &= qm - 1u;
              const U4 xq = pair_block_c(trial, t, qd);
              const uint32_t need = (ts_pairs >> (2 * qd)) & 3u;
              if (need == 3u) {
                double za0, za1, zb0, zb1;
                box_muller(xq.x, xq.y, za0, za1, logtab);
                box_muller(xq.z, xq.w, zb0, zb1, logtab);
                consider(2 * qd, za0, za1);
                consider(2 * qd + 1, zb0, zb1);
              } else {
                const bool hi = need == 2u;
                double z0, z1;
                box_muller(hi ? xq.z : xq.x, hi ? xq.w : xq.y, z0, z1, logtab);
                consider(2 * qd + (hi ? 1 : 0), z0, z1);
              }
            }
            pm = 0u;
          }
#endif
          int qcur = -1;
          U4 xq{0u, 0u, 0u, 0u};
          while (pm) {
            const int k = __ffs(pm) - 1;
            pm &= pm - 1u;
            if ((k >> 1) != qcur) {
              qcur = k >> 1;
              xq = pair_block_c(trial, t, qcur);
            }
            double z0, z1;
            box_muller((k & 1) ? xq.z : xq.x, (k & 1) ? xq.w : xq.y, z0, z1, logtab);
            consider(k, z0, z1);
          }
          n_sampled += 1;
        }
      }
      // Observe statistics of arm b: the last observed arm's record lives in
      // registers (qc); when the trial moves to another arm the Thompson phase writes it back
      // (phases 0/1 write through) and loads the new arm's in its place, to be consumed after the
      // curves.  In the Thompson phase every survivor was run (and observed) during pruning.
      was_seen = (ZS_SLIM_B && PHASE == 2 && !ABL && !WINDOWED) ? true : ((seen >> b) & 1u);
      if (b != qc_b) {
        if (PHASE == 2 && qc_b >= 0) st[qc_b] = qc;
        // an arm never observed in this trial has no record yet: nothing to load (its slot holds
        // another run's bytes, a cold DRAM read on the decision's chain)
        if (was_seen) qc = st[b];
        else qc = ArmStat{0.0, 0.0, 0.0, 0, 0};
        qc_b = b;
      }
      // the windowed Observe's evicted cost, loaded as soon as the decision is known
      if (WINDOWED && cp.window > 0) {
        const int cnt0 = was_seen ? qc.cnt : 0;
        if (cnt0 >= cp.window) y_old = a.st_ring[(o * B + b) * (size_t)a.ring_n + (cnt0 % cp.window)];
      }
      const ArmConst ac = arm[b];
      // the power limit accompanying b and its per-epoch cost/time/energy
      int p = ac.pstar;
      double c1b = ac.c1, t1b = ac.t1, e1b = ac.e1;
      const bool no_jit = ABL && (cp.ablation & 2);
      if (no_jit) {               // ablation "no JIT profiling": the first P runs of
        const int runs = was_seen ? qc.cnt : 0;            // b try the limits in ascending order
        if (runs < a.P) {
          p = runs;
          const double Ab = __ldg(a.A + (size_t)b * a.P + p), Thb = __ldg(a.Th + (size_t)b * a.P + p);
          c1b = ((cp.eta * Ab) + ((1.0 - cp.eta) * a.MP)) / Thb;
          t1b = 1.0 / Thb;
          e1b = Ab / Thb;
        }
      }
      // ---------------- step 3: replay one recorded run
      const uint32_t r = __umulhi(pick_word(rw, t), (uint32_t)K);
      const int E = pool[((size_t)s * B + b) * K + r];
      const int Erun = E > 0 ? E : a.max_epochs;
      double c0, t0, e0;
      const bool prof_now = !(ZS_SLIM_B && PHASE == 2 && !ABL && !WINDOWED) && !no_jit && a.charge_profiling &&
                            !((profiled >> b) & 1u);
      if (kHist) hkey = ((ts_dec ? 2 : 0) + (prof_now ? 1 : 0)) * B * K + b * K + (int)r;
      if (prof_now) { c0 = ac.cP; t0 = ac.tP; e0 = ac.eP; } else { c0 = c1b; t0 = t1b; e0 = e1b; }
      profiled |= 1u << b;
      const double em1 = (double)(Erun - 1);
      const double Cf = c0 + em1 * c1b;
      // ---------------- step 4: early stop at β·min_t C_t, truncated charge
      const double thr = cp.beta * best;
      double Tm, En;
      const bool stopped = Cf > thr;
      if (stopped) {
        C = thr;
        if (thr <= c0) {
          const double phi = thr / c0;
          Tm = phi * t0;
          En = phi * e0;
        } else {
          const double phi = (thr - c0) / c1b;
          Tm = t0 + phi * t1b;
          En = e0 + phi * e1b;
        }
      } else {
        C = Cf;
        Tm = t0 + em1 * t1b;
        En = e0 + em1 * e1b;
      }
      const bool conv = (E > 0) && !stopped;
      if (conv && !(C >= best)) best = C;
      // ---------------- Alg. 3 bookkeeping
      if (PHASE != 2 && !in_ts) {
        if (conv) {
          surv |= 1u << b;
          if (round == 1 && (C < r1_cost || (C == r1_cost && b < r1_arm))) { r1_cost = C; r1_arm = b; }
        }
        bool end_round = false;
        if (step == kStart) { step = kDown; cursor = start; }
        else if (step == kDown) { if (conv) cursor = b; else { step = kUp; cursor = start; } }
        else { if (conv) cursor = b; else end_round = true; }
        if (!end_round && step == kDown && (cand & below_mask(cursor)) == 0u) { step = kUp; cursor = start; }
        if (!end_round && step == kUp && (cand & above_mask(cursor)) == 0u) end_round = true;
        if (end_round) {
          if (surv == 0u) surv = 1u << start;
          if (round == 1) {
            cand = (ABL && (cp.ablation & 1)) ? all_arms : surv;   // "no pruning" keeps 𝓑
            if (r1_arm >= 0) start = r1_arm;
            surv = 0u;
            round = 2;
            step = kStart;
            cursor = start;
          } else {
            in_ts = true;
            ts_set = (ABL && (cp.ablation & 1)) ? all_arms : surv;
            ts_pairs = 0u;
            for (int k = 0; 2 * k < B; ++k)
              if ((ts_set >> (2 * k)) & 3u) ts_pairs |= 1u << k;
            if (cert_on) cert_begin();
          }
        }
      }
      // ---------------- accumulate
      const uint32_t flags = (stopped ? 1u : 0u) | (conv ? 2u : 0u) | (prof_now ? 4u : 0u) |
                             (ts_dec ? 8u : 0u);
      totC += C;
      totE += En;
      totT += Tm;
      nstop += stopped ? 1 : 0;
      last_b = b;
      dig = (dig ^ (unsigned long long)(uint32_t)b) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)(uint32_t)p) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)flags) * 0x100000001b3ull;
      if (LOG) a.log[o * R + t] = (uint32_t)b | ((uint32_t)p << 8) | (flags << 16);
      vC = C;
      vE = En;
      vT = Tm;
      vReg = (!ABL || p == ac.pstar) ? regret[s * B + b]
                                     : __ldg(a.ebar + (size_t)s * B + b) * c1b - __ldg(a.opt + (size_t)cell * S + s);
      vPacked = (stopped ? 1 : 0) | ((b == optarm[s] && p == ac.pstar) ? (1 << 8) : 0) |
                (ts_dec ? (1 << 16) : 0);
    }
    if constexpr (kHist) {
      // a run that is not stopped is counted in its (b, replica) bin (one predicated RED); the
      // rare stopped runs (charged the continuous threshold) take the fixed-point sums
      const bool special = live && (vPacked & 1);
      if (live && !special) red_add_u32(hist + (size_t)t * a.nhslot * HB + hkey, 1u);
      if (__any_sync(0xffffffffu, special))
        curve_accumulate(curves, t, tid & 31, special ? vC : 0.0, special ? vE : 0.0, special ? vT : 0.0,
                         special ? vReg : 0.0, special ? vPacked : 0, a.curve_scale);
    } else {
      curve_accumulate(curves, t, tid & 31, vC, vE, vT, vReg, vPacked, a.curve_scale);
    }
    if (live) {
      // ---------------- Alg. 2 Observe(b, C) with shifted sums and window N
      {
        const ArmStat &qr = qc;                             // the record (see the decision)
        const int cnt = was_seen ? qr.cnt : 0;
        double sh, S1, S2;
        if (!was_seen) { sh = C; S1 = 0.0; S2 = 0.0; }
        else { sh = qr.sh; S1 = qr.S1; S2 = qr.S2; }
        int n = cnt;
        if (WINDOWED && cp.window > 0) {
          const int N = cp.window;
          double *slot = &a.st_ring[(o * B + b) * (size_t)a.ring_n + (cnt % N)];
          if (cnt >= N) {
            const double dy = y_old - sh;
            S1 = S1 - dy;
            S2 = S2 - dy * dy;
            n = N - 1;
          }
          *slot = C;
        }
        const double d = C - sh;
        S1 = S1 + d;
        S2 = S2 + d * d;
        n += 1;
        ArmStat nq;
        nq.sh = sh; nq.S1 = S1; nq.S2 = S2; nq.cnt = cnt + 1; nq.pad = 0;
        // the Thompson phase writes the record back when the trial moves to another arm (and
        // at the end of the launch); phases 0/1 write through
        if (PHASE != 2) st[b] = nq;
        qc = nq;
        qc_b = b;
        seen |= 1u << b;
        if ((PHASE == 2 && !ABL) || n >= 2) {               // every Thompson-phase arm was run in pruning
          const double2 ms = posterior(sh, S1, S2, n, cp.prec0, cp.pm0);
          s_ms[b * TPB + tid] = ms;
          if (cert_on && in_ts && ((ts_set >> b) & 1u)) f32_slot(b, ms);
          mature |= 1u << b;
          n_recomp += 1;
        }
      }
    }
  }
  if (PHASE == 1) {                                         // hand over to phase B
    if (active) {
      Carry c;
      c.best = best; c.totC = totC; c.totE = totE; c.totT = totT; c.dig = dig;
      c.profiled = profiled; c.seen = seen; c.mature = mature; c.ts_set = ts_set;
      c.nstop = nstop; c.last_b = last_b;
      c.n_sampled = n_sampled; c.n_prune = n_prune; c.n_forced = n_forced; c.n_recomp = n_recomp;
      c.n_cert = n_cert; c.n_fall = n_fall;
      c.t0 = t0; c.pad = 0;
      a.carry[o] = c;
      atomicAdd(&a.bucket[((size_t)cell * a.nwin + jj / kRegroupWindow) * kBuckets +
                          regroup_key(ts_pairs, a.key_quads, a.early_split ? t0 : 0)], 1);
    }
    return;
  }
  if (PHASE == 2 && active && qc_b >= 0) st[qc_b] = qc;
  if (active) {
    a.tot_cost[o] = totC;
    a.tot_energy[o] = totE;
    a.tot_time[o] = totT;
    a.digest[o] = dig;
    a.n_stop[o] = nstop;
    a.final_arm[o] = last_b;
  }
  // work this launch evaluated: with the bound screen, phase B transforms the leader pair and
  // the residual pairs only (phase A's draws, carried in n_sampled, transform every pair)
  const unsigned long long screened = (unsigned long long)n_sampled * (__popc(ts_pairs) - 1);
  if (PHASE == 2 && active) {
    const Carry c = a.carry[o];
    n_sampled += c.n_sampled; n_prune += c.n_prune; n_forced += c.n_forced; n_recomp += c.n_recomp;
    n_cert += c.n_cert; n_fall += c.n_fall;
  }
  const unsigned long long pairs_all = (unsigned long long)n_sampled * __popc(ts_pairs);
  const unsigned long long blocks_all = (unsigned long long)n_sampled * __popc(quads_of(ts_pairs));
  unsigned long long bm_done = pairs_all - screened + n_resid;
  unsigned long long blocks_done = blocks_all, handled = screened;
  if (cert_on) {                    // certified draw: fp64 transforms only in phase A and fallbacks
    const unsigned long long nq = __popc(quads_of(ts_pairs));
    bm_done = (unsigned long long)(n_sampled - n_cert) * __popc(ts_pairs);
    blocks_done = (unsigned long long)(n_sampled + n_fall) * nq;
    handled = (unsigned long long)(n_cert + n_fall) * 2 * nq;
  }
  unsigned long long ctr[kCounters] = {
      active ? (unsigned long long)R : 0ull, n_sampled, pairs_all,
      (unsigned long long)n_sampled * __popc(ts_set),
      (unsigned long long)nstop, n_prune, n_forced, n_recomp, blocks_all,
      active ? bm_done : 0ull, active ? blocks_done : 0ull, active ? handled : 0ull,
      active ? n_cert : 0ull, active ? n_fall : 0ull};
#pragma unroll
  for (int q = 0; q < kCounters; ++q) {
    unsigned long long v = ctr[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0 && v) atomicAdd(a.counters + q, v);
  }
}

// Regrouping is done within windows of kRegroupWindow consecutive trials: warps still get
// (almost) uniform draw counts, and a window's Observe records (~1 MB at B = 16) stay on
// one or two 2 MB pages, so phase B's scattered lanes do not thrash the TLB.
// ------------------------------------------------------------------ lane-group layout
// W lanes per trial (the north star's "one warp per trial" for latency-bound launches: when a
// launch has too few trials to fill the GPU one thread per trial, W lanes share one trial).
// Every lane of a group carries the trial's scalar state and runs its serial steps (the same
// bits in every lane); the Thompson draw is split across the group -- lane l transforms the
// survivor pairs of rank l, l+W, ... -- and a segmented shuffle argmin over (theta, arm) keeps
// the strict-<, lowest-arm rule (NC-4).  Lane 0 writes the shared state and the outputs.
template <int W, bool WINDOWED, bool LOG>
__global__ void __launch_bounds__(128) replay_group_kernel(ReplayArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  constexpr int TPB = 128, TPG = TPB / W;                 // trials per block
  const int cell = blockIdx.y;
  const CellParam cp = a.cells[cell];
  const int tid = threadIdx.x;
  const int g = tid / W, l = tid % W;
  const int64_t j0 = (int64_t)blockIdx.x * TPG;
  if (j0 >= cp.n || cp.policy != 0 || cp.conc) return;

  const TabLayout L(a.B, a.S, a.K);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    const uint32_t b_arm = a.B * (uint32_t)sizeof(ArmConst);
    const uint32_t b_reg = a.S * a.B * 8u;
    const uint32_t b_opt = a.S * 4u;
    const uint32_t b_pool = a.S * a.B * a.K * 4u;
    const uint32_t p_arm = (b_arm + 15u) & ~15u, p_reg = (b_reg + 15u) & ~15u;
    const uint32_t p_opt = (b_opt + 15u) & ~15u, p_pool = (b_pool + 15u) & ~15u;
    mbar_expect_tx(&mbar, p_arm + p_reg + p_opt + p_pool + kLogTab * 16u);
    tma_bulk_load(smem + L.logtab, a.logtab, kLogTab * 16u, &mbar);
    tma_bulk_load(smem + L.arms, a.arms + (size_t)cell * a.B, p_arm, &mbar);
    tma_bulk_load(smem + L.regret, a.regret + (size_t)cell * a.reg_stride, p_reg, &mbar);
    tma_bulk_load(smem + L.optarm, a.opt_arm + (size_t)cell * a.opt_stride, p_opt, &mbar);
    tma_bulk_load(smem + L.pool, a.pool, p_pool, &mbar);
  }
  __syncthreads();
  mbar_wait(&mbar, 0);

  const ArmConst *arm = reinterpret_cast<const ArmConst *>(smem + L.arms);
  const double *regret = reinterpret_cast<const double *>(smem + L.regret);
  const int32_t *optarm = reinterpret_cast<const int32_t *>(smem + L.optarm);
  const int32_t *pool = reinterpret_cast<const int32_t *>(smem + L.pool);
  const double2 *logtab = reinterpret_cast<const double2 *>(smem + L.logtab);
  const int B = a.B, R = a.R, S = a.S, K = a.K;
  double2 *s_ms = reinterpret_cast<double2 *>(smem + a.tab_bytes);   // [arm][trial of block]
  const int64_t jj = j0 + g;
  const bool active = jj < cp.n;
  const bool leader = l == 0;
  const int64_t trial = cp.begin + jj;
  const size_t o = (size_t)(cp.out_off + (active ? jj : 0));
  const RecRef st{a.st, (uint32_t)(o * B)};               // the trial's Observe records (32-bit index)
  const int warp_global = blockIdx.x * (TPB >> 5) + (tid >> 5);
  long long *curves = a.curve_slots + ((size_t)cell * a.nslot + (warp_global % a.nslot)) * (size_t)R * kRow;
  const int HB = 4 * B * K;                                 // counted curves (ReplayArgs::hist)
  uint32_t *hist = a.hist + ((size_t)cell * R * a.nhslot + (warp_global % a.nhslot)) * (size_t)HB;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);

  uint32_t profiled = 0, seen = 0, mature = 0;
  double best = kInf;
  bool in_ts = false;
  int round = 1, step = kStart, start = a.b0, cursor = a.b0;
  const uint32_t all_arms = (B == 32) ? 0xffffffffu : ((1u << B) - 1u);
  uint32_t cand = all_arms, surv = 0, ts_set = 0, ts_pairs = 0;
  double r1_cost = kInf;
  int r1_arm = -1;
  double totC = 0.0, totE = 0.0, totT = 0.0;
  unsigned long long dig = 0xcbf29ce484222325ull;
  int nstop = 0, last_b = -1;
  uint32_t n_sampled = 0, n_prune = 0, n_forced = 0, n_recomp = 0;
  int s = 0;
  U4 rw{0u, 0u, 0u, 0u};
  ArmStat qc{0.0, 0.0, 0.0, 0, 0};                     // the last arm's record (read cache)
  int qc_b = -1;
  for (int t = 0; t < R; ++t) {
    double vC = 0.0, vE = 0.0, vT = 0.0, vReg = 0.0;
    int vPacked = 0;
    if (S > 1)
      while ((long long)(s + 1) * R <= (long long)t * S) ++s;
    // ---------------- step 2: decide b_t (pruning walk / forced / Thompson draw)
    int b = 0;
    const bool ts_dec = in_ts;
    bool sampled = false;
    if (active) {
      if ((t & 3) == 0) rw = replica_words(cp.key0, cp.key1, trial, t);
      if (!in_ts) {
        b = (step == kStart) ? start
          : (step == kDown) ? 31 - __clz(cand & below_mask(cursor))
                            : __ffs(cand & above_mask(cursor)) - 1;
        n_prune += 1;
      } else {
        const uint32_t unripe = ts_set & ~mature;
        if (unripe) {
          b = __ffs(unripe) - 1;
          n_forced += 1;
        } else {
          sampled = true;
          n_sampled += 1;
        }
      }
    }
    // the group's share of the draw: lane l takes the survivor pairs of rank l, l+W, ...
    double bt = kInf;
    int bb = -1;
    if (sampled) {
      uint32_t pm = ts_pairs;
      for (int i = 0; i < l && pm; ++i) pm &= pm - 1u;
      while (pm) {
        const int k = __ffs(pm) - 1;
        const U4 xq = pair_block(cp.key0, cp.key1, trial, t, k >> 1);
        double z0, z1;
        box_muller((k & 1) ? xq.z : xq.x, (k & 1) ? xq.w : xq.y, z0, z1, logtab);
        const uint32_t two = (ts_set >> (2 * k)) & 3u;
        const double2 m0 = s_ms[(2 * k) * TPG + g];
        const double2 m1 = s_ms[(2 * k + 1) * TPG + g];
        const double th0 = fma(m0.y, z0, m0.x);
        const bool take0 = (two & 1u) && (th0 < bt);
        bt = take0 ? th0 : bt;
        bb = take0 ? 2 * k : bb;
        const double th1 = fma(m1.y, z1, m1.x);
        const bool take1 = (two & 2u) && (th1 < bt);
        bt = take1 ? th1 : bt;
        bb = take1 ? 2 * k + 1 : bb;
        for (int i = 0; i < W && pm; ++i) pm &= pm - 1u;
      }
    }
#pragma unroll
    for (int off = W / 2; off > 0; off >>= 1) {             // segmented (theta, arm) argmin
      const double ot = __shfl_xor_sync(0xffffffffu, bt, off, W);
      const int ob = __shfl_xor_sync(0xffffffffu, bb, off, W);
      const bool take = ob >= 0 && (bb < 0 || ot < bt || (ot == bt && ob < bb));
      bt = take ? ot : bt;
      bb = take ? ob : bb;
    }
    if (sampled) b = bb;
    __syncwarp();                                            // the draw's reads before lane 0's stores
    int hkey = -1;
    bool was_seen = false;
    ArmStat q;
    double C = 0.0;
    if (active) {
      was_seen = (seen >> b) & 1u;
      if (b == qc_b) q = qc; else if (was_seen) q = st[b]; else q = ArmStat{0.0, 0.0, 0.0, 0, 0};
      const ArmConst ac = arm[b];
      const uint32_t r = __umulhi(pick_word(rw, t), (uint32_t)K);
      const int E = pool[((size_t)s * B + b) * K + r];
      const int Erun = E > 0 ? E : a.max_epochs;
      double c0, t0, e0;
      const bool prof_now = a.charge_profiling && !((profiled >> b) & 1u);
      if (prof_now) { c0 = ac.cP; t0 = ac.tP; e0 = ac.eP; } else { c0 = ac.c1; t0 = ac.t1; e0 = ac.e1; }
      hkey = ((ts_dec ? 2 : 0) + (prof_now ? 1 : 0)) * B * K + b * K + (int)r;
      profiled |= 1u << b;
      const double em1 = (double)(Erun - 1);
      const double Cf = c0 + em1 * ac.c1;
      const double thr = cp.beta * best;
      double Tm, En;
      const bool stopped = Cf > thr;
      if (stopped) {
        C = thr;
        if (thr <= c0) {
          const double phi = thr / c0;
          Tm = phi * t0;
          En = phi * e0;
        } else {
          const double phi = (thr - c0) / ac.c1;
          Tm = t0 + phi * ac.t1;
          En = e0 + phi * ac.e1;
        }
      } else {
        C = Cf;
        Tm = t0 + em1 * ac.t1;
        En = e0 + em1 * ac.e1;
      }
      const bool conv = (E > 0) && !stopped;
      if (conv && !(C >= best)) best = C;
      if (!in_ts) {                                          // Alg. 3 bookkeeping
        if (conv) {
          surv |= 1u << b;
          if (round == 1 && (C < r1_cost || (C == r1_cost && b < r1_arm))) { r1_cost = C; r1_arm = b; }
        }
        bool end_round = false;
        if (step == kStart) { step = kDown; cursor = start; }
        else if (step == kDown) { if (conv) cursor = b; else { step = kUp; cursor = start; } }
        else { if (conv) cursor = b; else end_round = true; }
        if (!end_round && step == kDown && (cand & below_mask(cursor)) == 0u) { step = kUp; cursor = start; }
        if (!end_round && step == kUp && (cand & above_mask(cursor)) == 0u) end_round = true;
        if (end_round) {
          if (surv == 0u) surv = 1u << start;
          if (round == 1) {
            cand = surv;
            if (r1_arm >= 0) start = r1_arm;
            surv = 0u;
            round = 2;
            step = kStart;
            cursor = start;
          } else {
            in_ts = true;
            ts_set = surv;
            ts_pairs = 0u;
            for (int k = 0; 2 * k < B; ++k)
              if ((ts_set >> (2 * k)) & 3u) ts_pairs |= 1u << k;
          }
        }
      }
      const uint32_t flags = (stopped ? 1u : 0u) | (conv ? 2u : 0u) | (prof_now ? 4u : 0u) |
                             (ts_dec ? 8u : 0u);
      totC += C;
      totE += En;
      totT += Tm;
      nstop += stopped ? 1 : 0;
      last_b = b;
      dig = (dig ^ (unsigned long long)(uint32_t)b) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)(uint32_t)ac.pstar) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)flags) * 0x100000001b3ull;
      if (leader) {
        if (LOG) a.log[o * R + t] = (uint32_t)b | ((uint32_t)ac.pstar << 8) | (flags << 16);
        vC = C;
        vE = En;
        vT = Tm;
        vReg = regret[s * B + b];
        vPacked = (stopped ? 1 : 0) | ((b == optarm[s]) ? (1 << 8) : 0) | (ts_dec ? (1 << 16) : 0);
      }
    }
    {                                                        // counted curves (ReplayArgs::hist)
      const bool counted = active && leader && !(vPacked & 1);
      const bool special = active && leader && (vPacked & 1);
      if (counted) red_add_u32(hist + (size_t)t * a.nhslot * HB + hkey, 1u);
      if (__any_sync(0xffffffffu, special))
        curve_accumulate(curves, t, tid & 31, special ? vC : 0.0, special ? vE : 0.0, special ? vT : 0.0,
                         special ? vReg : 0.0, special ? vPacked : 0, a.curve_scale);
    }
    if (active) {                                            // Alg. 2 Observe (NC-6)
      const int cnt = was_seen ? q.cnt : 0;
      double sh, S1, S2;
      if (!was_seen) { sh = C; S1 = 0.0; S2 = 0.0; }
      else { sh = q.sh; S1 = q.S1; S2 = q.S2; }
      int n = cnt;
      if (WINDOWED && cp.window > 0) {
        const int N = cp.window;
        double *slot = &a.st_ring[(o * B + b) * (size_t)a.ring_n + (cnt % N)];
        const double y = *slot;
        if (cnt >= N) {
          const double dy = y - sh;
          S1 = S1 - dy;
          S2 = S2 - dy * dy;
          n = N - 1;
        }
        if (leader) *slot = C;
      }
      const double d = C - sh;
      S1 = S1 + d;
      S2 = S2 + d * d;
      n += 1;
      {
        ArmStat nq;
        nq.sh = sh; nq.S1 = S1; nq.S2 = S2; nq.cnt = cnt + 1; nq.pad = 0;
        if (leader) st[b] = nq;
        qc = nq;                                            // every lane of the group keeps it
        qc_b = b;
      }
      seen |= 1u << b;
      if (n >= 2) {
        const double2 ms = posterior(sh, S1, S2, n, cp.prec0, cp.pm0);
        if (leader) s_ms[b * TPG + g] = ms;
        mature |= 1u << b;
        n_recomp += 1;
      }
    }
    __syncwarp();                                            // lane 0's stores before the next draw
  }
  if (active && leader) {
    a.tot_cost[o] = totC;
    a.tot_energy[o] = totE;
    a.tot_time[o] = totT;
    a.digest[o] = dig;
    a.n_stop[o] = nstop;
    a.final_arm[o] = last_b;
  }
  const bool cnt_lane = active && leader;
  unsigned long long ctr[kCounters] = {
      cnt_lane ? (unsigned long long)R : 0ull, cnt_lane ? n_sampled : 0u,
      cnt_lane ? (unsigned long long)n_sampled * __popc(ts_pairs) : 0ull,
      cnt_lane ? (unsigned long long)n_sampled * __popc(ts_set) : 0ull,
      cnt_lane ? (unsigned long long)nstop : 0ull, cnt_lane ? n_prune : 0u,
      cnt_lane ? n_forced : 0u, cnt_lane ? n_recomp : 0u,
      cnt_lane ? (unsigned long long)n_sampled * __popc(quads_of(ts_pairs)) : 0ull,
      cnt_lane ? (unsigned long long)n_sampled * __popc(ts_pairs) : 0ull,   // every pair transformed,
      cnt_lane ? (unsigned long long)n_sampled * __popc(ts_pairs) : 0ull,   // each with its own block
      0ull};
#pragma unroll
  for (int qq = 0; qq < kCounters; ++qq) {
    unsigned long long v = ctr[qq];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0 && v) atomicAdd(a.counters + qq, v);
  }
}

// bucket offsets: exclusive scan of each (cell, window) histogram, offset by the window base; one
// warp per (cell, window): every lane loads its kBuckets/32 counts at once (the loads in flight
// together, not one round trip per 32 buckets), then a shuffle scan per 32-bucket chunk
constexpr int kScanPerLane = (kBuckets + 31) / 32;
__global__ void bucket_scan_kernel(int32_t *bucket, int ncells, int nwin) {
  const int64_t cw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (cw >= (int64_t)ncells * nwin) return;                 // warp-uniform
  int32_t *row = bucket + cw * kBuckets;
  int c[kScanPerLane];
#pragma unroll
  for (int j = 0; j < kScanPerLane; ++j) c[j] = (32 * j + lane < kBuckets) ? row[32 * j + lane] : 0;
  int run = (int)(cw % nwin) * kRegroupWindow;
#pragma unroll
  for (int j = 0; j < kScanPerLane; ++j) {
    int x = c[j];                                           // inclusive scan over the lanes
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (32 * j + lane < kBuckets) row[32 * j + lane] = run + x - c[j];
    run += __shfl_sync(0xffffffffu, x, 31);
  }
}

// phase-B lane order: the trials of each window grouped by their survivor-pair (or quad) count.
// One 256-trial tile per block iteration (a tile never straddles a window): ranks within the tile
// from shared-memory atomics, then one global atomic per non-empty bucket reserves the tile's
// range -- at most kBuckets global atomics per tile instead of one per trial (the bucket counters
// were the contended addresses).  The order within a bucket is free: trials are independent.
constexpr int kScatterTile = 256;
static_assert(kRegroupWindow % kScatterTile == 0, "a tile must not straddle a regroup window");
__global__ void __launch_bounds__(kScatterTile) bucket_scatter_kernel(const CellParam *cells, const Carry *carry,
                                                                      int32_t *bucket, int32_t *perm, int ncells,
                                                                      int B, int nwin, int key_quads,
                                                                      int early_split) {
  __shared__ int s_cnt[kBuckets], s_base[kBuckets];
  const int cell = blockIdx.y;
  const CellParam cp = cells[cell];
  if (cp.policy != 0 || cp.conc) return;
  const int64_t ntiles = (cp.n + kScatterTile - 1) / kScatterTile;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int k = threadIdx.x; k < kBuckets; k += kScatterTile) s_cnt[k] = 0;
    __syncthreads();
    const int64_t j = tile * kScatterTile + threadIdx.x;
    int key = -1, rank = 0;
    if (j < cp.n) {
      const Carry &cj = carry[cp.out_off + j];
      const uint32_t ts_set = cj.ts_set;
      uint32_t pairs = 0;
      for (int k = 0; 2 * k < B; ++k)
        if ((ts_set >> (2 * k)) & 3u) pairs |= 1u << k;
      key = regroup_key(pairs, key_quads, early_split ? cj.t0 : 0);
      rank = atomicAdd(&s_cnt[key], 1);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < kBuckets; k += kScatterTile)
      if (s_cnt[k] > 0)
        s_base[k] = atomicAdd(&bucket[((size_t)cell * nwin + (tile * kScatterTile) / kRegroupWindow) * kBuckets + k],
                              s_cnt[k]);
    __syncthreads();
    if (key >= 0) perm[cp.out_off + s_base[key] + rank] = (int32_t)j;
    __syncthreads();                                        // s_cnt is reset by the next tile
  }
}

// ------------------------------------------------------------------ concurrent submissions (f3)
// §4.4 "Handling concurrent job submissions" under an arrival schedule: recurrence t
// is submitted at arrivals[t]; its outcome reaches the optimiser (best update, Observe, Alg. 3
// walk bookkeeping) when it completes at arrivals[t] + its TTA, in (completion, submission)
// order; a pruning-phase submission that overlaps the walk's outstanding run takes the
// best-known batch size; at most kMaxOutstanding runs per trial are in flight (R-Q31).
// One thread per trial, one pass, tables read through the read-only cache.
constexpr int kMaxOutstanding = 8;
constexpr int kQueueBytes = kMaxOutstanding * (8 + 8 + 4 + 4 + 4);   // per thread, concurrent_kernel

struct ConcArgs {
  const CellParam *cells;
  const ArmConst *arms;           // [cells][B]
  const double *regret;           // [cells][reg_stride]
  const int32_t *opt_arm;         // [cells][opt_stride]
  const int32_t *pool;            // [S][B][K]
  const double2 *logtab;
  const double *arrivals;         // [cells][R] (cells with conc = 1)
  long long *curve_slots;         // [cells][nslot][R][kQ][kLimbs] fixed point (curve_accumulate)
  double curve_scale;             // 2^F of the fixed point
  double *tot_cost, *tot_energy, *tot_time;
  unsigned long long *digest;
  int32_t *n_stop, *final_arm;
  uint32_t *log;
  unsigned long long *counters;
  ArmStat *st;
  double *st_ring;
  int ring_n;
  int B, S, K, R, max_epochs, charge_profiling, b0, nslot, reg_stride, opt_stride;
  // the variant kernel only: "no JIT" per-(b, p) costs, and the windowed best's ring
  const double *A, *Th, *ebar, *opt;   // [B][P], [B][P], [S][B], [cells][S]
  double *best_ring;                   // [trial][best_n]
  int P, best_n;
  double MP;
  int cert_draw, force_exact;          // certified fp32 draw, as ReplayArgs
};

template <bool LOG>
__global__ void __launch_bounds__(128) concurrent_kernel(ConcArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int cell = blockIdx.y;
  const CellParam cp = a.cells[cell];
  const int tid = threadIdx.x, TPB = blockDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * TPB;
  if (j0 >= cp.n || cp.policy != 0 || !cp.conc) return;
  double2 *s_ms = reinterpret_cast<double2 *>(smem);       // [arm][thread] (mu, sigma)
  const int B = a.B, R = a.R, S = a.S, K = a.K;
  const ArmConst *arm = a.arms + (size_t)cell * B;
  const double *regret = a.regret + (size_t)cell * a.reg_stride;
  const int32_t *optarm = a.opt_arm + (size_t)cell * a.opt_stride;
  const double *arr = a.arrivals + (size_t)cell * R;
  const int64_t jj = j0 + tid;
  const bool active = jj < cp.n;
  const int64_t trial = cp.begin + jj;
  const size_t o = (size_t)(cp.out_off + jj);
  const RecRef st{a.st, (uint32_t)(o * B)};               // the trial's Observe records (32-bit index)
  const int warp_global = blockIdx.x * (TPB >> 5) + (tid >> 5);
  long long *curves = a.curve_slots + ((size_t)cell * a.nslot + (warp_global % a.nslot)) * (size_t)R * kRow;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);

  uint32_t profiled = 0, seen = 0, mature = 0;
  double best = kInf;
  int best_arm = -1;
  bool in_ts = false, walk_out = false;
  int round = 1, step = kStart, start = a.b0, cursor = a.b0;
  const uint32_t all_arms = (B == 32) ? 0xffffffffu : ((1u << B) - 1u);
  uint32_t cand = all_arms, surv = 0, ts_set = 0, ts_pairs = 0;
  double r1_cost = kInf;
  int r1_arm = -1;
  double totC = 0.0, totE = 0.0, totT = 0.0;
  unsigned long long dig = 0xcbf29ce484222325ull;
  int nstop = 0, last_b = -1;
  uint32_t n_sampled = 0, n_prune = 0, n_forced = 0, n_recomp = 0;
  // outstanding runs: a queue of kMaxOutstanding entries per trial in shared memory, after the
  // (mu, sigma) table, each field [slot][thread] (conflict-free; dynamically indexed, so registers
  // would put it on the local-memory stack)
  double *const q_done_s = reinterpret_cast<double *>(smem + (size_t)((B + 1) & ~1) * 16 * TPB);
  double *const q_C_s = q_done_s + kMaxOutstanding * TPB;
  int *const q_seq_s = reinterpret_cast<int *>(q_C_s + kMaxOutstanding * TPB);
  int *const q_b_s = q_seq_s + kMaxOutstanding * TPB;
  uint32_t *const q_flags_s = reinterpret_cast<uint32_t *>(q_b_s + kMaxOutstanding * TPB);
  auto q_done = [&](int i) -> double & { return q_done_s[i * TPB + tid]; };
  auto q_C = [&](int i) -> double & { return q_C_s[i * TPB + tid]; };
  auto q_seq = [&](int i) -> int & { return q_seq_s[i * TPB + tid]; };
  auto q_b = [&](int i) -> int & { return q_b_s[i * TPB + tid]; };
  auto q_flags = [&](int i) -> uint32_t & { return q_flags_s[i * TPB + tid]; };   // bit0 converged, bit1 walk
  int nq = 0;
  // certified fp32 draw (a.cert_draw): fp32 (mu - ref, sigma) of every mature
  // arm, [pair][thread] float4 after the queues; ref fixed when Thompson sampling starts
  const int cpairs2 = ((((B + 1) >> 1) + 1) & ~1);
  float2 *s_f2 = reinterpret_cast<float2 *>(q_flags_s + kMaxOutstanding * TPB);
  const int ckbits = 32 - __clz(2 * cpairs2 - 1);
  const uint32_t ckeep = ~((1u << ckbits) - 1u);
  const float ckth = cert::kTheta + __int_as_float((127 - 23 + ckbits) << 23) * 1.000001f;
  double cref = 0.0;
  float c_trial = 0.0f;
  uint32_t n_cert = 0, n_fall = 0;
  auto f32_slot = [&](int arm_i, double2 ms) {
    const double dm = ms.x - cref;
    s_f2[2 * ((arm_i >> 1) * TPB + tid) + (arm_i & 1)] =
        (fabs(dm) < 1e30 && ms.y < 1e30) ? make_float2((float)dm, (float)ms.y)
                                         : make_float2(0.0f, __int_as_float(0x7f800000));
  };
  auto cert_begin = [&]() {
    const int lead = __ffs(ts_set & mature) - 1;
    cref = lead >= 0 ? s_ms[lead * TPB + tid].x : 0.0;
    if (!(fabs(cref) < 1e30)) cref = 0.0;
    c_trial = __double2float_ru(fabs(cref) * 0x1p-52 + 0x1p-120);
    for (int arm_i = 0; arm_i < 2 * cpairs2; ++arm_i)
      if ((mature >> arm_i) & 1u) f32_slot(arm_i, s_ms[arm_i * TPB + tid]);
  };

  ArmStat qc{0.0, 0.0, 0.0, 0, 0};                     // the last arm's record (read cache)
  int qc_b = -1;
  // a run's outcome reaching the optimiser
  auto complete = [&](int i) {
    const int b = q_b(i);
    const double C = q_C(i);
    const bool conv = q_flags(i) & 1u, walk = q_flags(i) & 2u;
    if (conv && !(C >= best)) { best = C; best_arm = b; }
    {                                                        // Alg. 2 Observe (NC-6)
      const bool was_seen = (seen >> b) & 1u;
      ArmStat q;
      if (b == qc_b) q = qc; else if (was_seen) q = st[b]; else q = ArmStat{0.0, 0.0, 0.0, 0, 0};
      const int cnt = was_seen ? q.cnt : 0;
      double sh, S1, S2;
      if (!was_seen) { sh = C; S1 = 0.0; S2 = 0.0; }
      else { sh = q.sh; S1 = q.S1; S2 = q.S2; }
      int n = cnt;
      if (a.ring_n > 0 && cp.window > 0) {
        const int N = cp.window;
        double *slot = &a.st_ring[(o * B + b) * (size_t)a.ring_n + (cnt % N)];
        if (cnt >= N) {
          const double dy = *slot - sh;
          S1 = S1 - dy;
          S2 = S2 - dy * dy;
          n = N - 1;
        }
        *slot = C;
      }
      const double d = C - sh;
      S1 = S1 + d;
      S2 = S2 + d * d;
      n += 1;
      ArmStat nq_;
      nq_.sh = sh; nq_.S1 = S1; nq_.S2 = S2; nq_.cnt = cnt + 1; nq_.pad = 0;
      st[b] = nq_;
      qc = nq_;
      qc_b = b;
      seen |= 1u << b;
      if (n >= 2) {
        const double2 ms = posterior(sh, S1, S2, n, cp.prec0, cp.pm0);
        s_ms[b * TPB + tid] = ms;
        if (a.cert_draw && in_ts) f32_slot(b, ms);
        mature |= 1u << b;
        n_recomp += 1;
      }
    }
    if (!walk) return;
    walk_out = false;
    if (conv) {                                              // Alg. 3 bookkeeping
      surv |= 1u << b;
      if (round == 1 && (C < r1_cost || (C == r1_cost && b < r1_arm))) { r1_cost = C; r1_arm = b; }
    }
    bool end_round = false;
    if (step == kStart) { step = kDown; cursor = start; }
    else if (step == kDown) { if (conv) cursor = b; else { step = kUp; cursor = start; } }
    else { if (conv) cursor = b; else end_round = true; }
    if (!end_round && step == kDown && (cand & below_mask(cursor)) == 0u) { step = kUp; cursor = start; }
    if (!end_round && step == kUp && (cand & above_mask(cursor)) == 0u) end_round = true;
    if (end_round) {
      if (surv == 0u) surv = 1u << start;
      if (round == 1) {
        cand = surv;
        if (r1_arm >= 0) start = r1_arm;
        surv = 0u;
        round = 2;
        step = kStart;
        cursor = start;
      } else {
        in_ts = true;
        ts_set = surv;
        ts_pairs = 0u;
        for (int k = 0; 2 * k < B; ++k)
          if ((ts_set >> (2 * k)) & 3u) ts_pairs |= 1u << k;
        if (a.cert_draw) cert_begin();
      }
    }
  };
#if ZS_CONC_MIN
  // the queue's earliest entry by (completion, submission), kept up to date: a scan only after a
  // completion, none per submission check
  int m_i = -1;
  double m_done = kInf;
  auto rescan = [&]() {
    m_i = -1;
    for (int i = 0; i < nq; ++i)
      if (m_i < 0 || q_done(i) < q_done(m_i) || (q_done(i) == q_done(m_i) && q_seq(i) < q_seq(m_i))) m_i = i;
    m_done = m_i >= 0 ? q_done(m_i) : kInf;
  };
  auto complete_earliest = [&]() {                          // by (completion, submission)
    const int e = m_i;
    complete(e);
    --nq;                                                    // move the last entry into slot e
    q_done(e) = q_done(nq); q_C(e) = q_C(nq); q_seq(e) = q_seq(nq); q_b(e) = q_b(nq);
    q_flags(e) = q_flags(nq);
    rescan();
  };
#else
  auto complete_earliest = [&]() {                          // by (completion, submission)
    int e = 0;
    for (int i = 1; i < nq; ++i)
      if (q_done(i) < q_done(e) || (q_done(i) == q_done(e) && q_seq(i) < q_seq(e))) e = i;
    complete(e);
    --nq;                                                    // move the last entry into slot e
    q_done(e) = q_done(nq); q_C(e) = q_C(nq); q_seq(e) = q_seq(nq); q_b(e) = q_b(nq);
    q_flags(e) = q_flags(nq);
  };
#endif

  int s = 0;
  U4 rw{0u, 0u, 0u, 0u};
  for (int t = 0; t < R; ++t) {
    double vC = 0.0, vE = 0.0, vT = 0.0, vReg = 0.0;
    int vPacked = 0;
    if (S > 1)
      while ((long long)(s + 1) * R <= (long long)t * S) ++s;
    if (active) {
      const double tau = __ldg(arr + t);
#if ZS_CONC_MIN
      while (m_i >= 0 && m_done <= tau) complete_earliest();   // runs finished by this submission
#else
      for (;;) {                                             // runs finished by this submission
        bool any = false;
        for (int i = 0; i < nq; ++i) any |= q_done(i) <= tau;
        if (!any) break;
        complete_earliest();
      }
#endif
      while (nq >= kMaxOutstanding) complete_earliest();
      if ((t & 3) == 0) rw = replica_words(cp.key0, cp.key1, trial, t);
      const bool ts_dec = in_ts;
      bool walk_issue = false;
      int b;
      if (!in_ts) {
        if (walk_out) {
          b = best_arm >= 0 ? best_arm : start;              // best-known batch size
        } else {
          b = (step == kStart) ? start
            : (step == kDown) ? 31 - __clz(cand & below_mask(cursor))
                              : __ffs(cand & above_mask(cursor)) - 1;
          walk_issue = true;
          walk_out = true;
        }
        n_prune += 1;
      } else {
        const uint32_t unripe = ts_set & ~mature;
        if (unripe) {
          b = __ffs(unripe) - 1;
          n_forced += 1;
        } else {
          double bt = kInf;
          b = -1;
          uint32_t pm = ts_pairs;
          if (a.cert_draw) {                                 // certified fp32 draw (§7.9)
            cert::Argmin32 am;
            am.init();
            uint32_t qm = quads_of(ts_pairs);
            while (qm) {
              const int qd = __ffs(qm) - 1;
              qm &= qm - 1u;
              const U4 x = pair_block(cp.key0, cp.key1, trial, t, qd);
              const float4 f0 = reinterpret_cast<const float4 *>(s_f2)[(2 * qd) * TPB + tid];
              const float4 f1 = reinterpret_cast<const float4 *>(s_f2)[(2 * qd + 1) * TPB + tid];
              float z0, z1, rsq;
              cert::normal_pair32(x.x, x.y, z0, z1, rsq);
              am.pair_masked(4 * qd, f0, z0, z1, rsq, ckeep, (ts_set >> (4 * qd)) & 3u);
              cert::normal_pair32(x.z, x.w, z0, z1, rsq);
              am.pair_masked(4 * qd + 2, f1, z0, z1, rsq, ckeep, (ts_set >> (4 * qd + 2)) & 3u);
            }
            if (am.certified(c_trial, ckth) && !a.force_exact) {
              b = am.arg(ckeep);
              pm = 0u;
              n_cert += 1;
            } else {
              n_fall += 1;
            }
          }
          int qcur = -1;
          U4 xq{0u, 0u, 0u, 0u};
          while (pm) {
            const int k = __ffs(pm) - 1;
            pm &= pm - 1u;
            if ((k >> 1) != qcur) {
              qcur = k >> 1;
              xq = pair_block(cp.key0, cp.key1, trial, t, qcur);
            }
            double z0, z1;
            box_muller((k & 1) ? xq.z : xq.x, (k & 1) ? xq.w : xq.y, z0, z1, a.logtab);
            const uint32_t two = (ts_set >> (2 * k)) & 3u;
            const double2 m0 = s_ms[(2 * k) * TPB + tid];
            const double2 m1 = s_ms[(2 * k + 1) * TPB + tid];
            const double th0 = fma(m0.y, z0, m0.x);
            const bool take0 = (two & 1u) && (th0 < bt);
            bt = take0 ? th0 : bt;
            b = take0 ? 2 * k : b;
            const double th1 = fma(m1.y, z1, m1.x);
            const bool take1 = (two & 2u) && (th1 < bt);
            bt = take1 ? th1 : bt;
            b = take1 ? 2 * k + 1 : b;
          }
          n_sampled += 1;
        }
      }
      const ArmConst ac = arm[b];
      const uint32_t r = __umulhi(pick_word(rw, t), (uint32_t)K);
      const int E = __ldg(a.pool + ((size_t)s * B + b) * K + r);
      const int Erun = E > 0 ? E : a.max_epochs;
      double c0, t0, e0;
      const bool prof_now = a.charge_profiling && !((profiled >> b) & 1u);
      if (prof_now) { c0 = ac.cP; t0 = ac.tP; e0 = ac.eP; } else { c0 = ac.c1; t0 = ac.t1; e0 = ac.e1; }
      profiled |= 1u << b;
      const double em1 = (double)(Erun - 1);
      const double Cf = c0 + em1 * ac.c1;
      const double thr = cp.beta * best;
      double C, Tm, En;
      const bool stopped = Cf > thr;
      if (stopped) {
        C = thr;
        if (thr <= c0) {
          const double phi = thr / c0;
          Tm = phi * t0;
          En = phi * e0;
        } else {
          const double phi = (thr - c0) / ac.c1;
          Tm = t0 + phi * ac.t1;
          En = e0 + phi * ac.e1;
        }
      } else {
        C = Cf;
        Tm = t0 + em1 * ac.t1;
        En = e0 + em1 * ac.e1;
      }
      const bool conv = (E > 0) && !stopped;
      q_done(nq) = tau + Tm; q_C(nq) = C; q_seq(nq) = t; q_b(nq) = b;
      q_flags(nq) = (conv ? 1u : 0u) | (walk_issue ? 2u : 0u);
#if ZS_CONC_MIN
      // the new entry has the largest submission index: it is the earliest only if it completes
      // strictly first
      if (m_i < 0 || tau + Tm < m_done) { m_i = nq; m_done = tau + Tm; }
#endif
      ++nq;
      const uint32_t flags = (stopped ? 1u : 0u) | (conv ? 2u : 0u) | (prof_now ? 4u : 0u) |
                             (ts_dec ? 8u : 0u);
      totC += C;
      totE += En;
      totT += Tm;
      nstop += stopped ? 1 : 0;
      last_b = b;
      dig = (dig ^ (unsigned long long)(uint32_t)b) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)(uint32_t)ac.pstar) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)flags) * 0x100000001b3ull;
      if (LOG) a.log[o * R + t] = (uint32_t)b | ((uint32_t)ac.pstar << 8) | (flags << 16);
      vC = C;
      vE = En;
      vT = Tm;
      vReg = __ldg(regret + (size_t)s * B + b);
      vPacked = (stopped ? 1 : 0) | ((b == __ldg(optarm + s)) ? (1 << 8) : 0) | (ts_dec ? (1 << 16) : 0);
    }
    curve_accumulate(curves, t, tid & 31, vC, vE, vT, vReg, vPacked, a.curve_scale);
  }
  if (active) {
    a.tot_cost[o] = totC;
    a.tot_energy[o] = totE;
    a.tot_time[o] = totT;
    a.digest[o] = dig;
    a.n_stop[o] = nstop;
    a.final_arm[o] = last_b;
  }
  const unsigned long long cq = __popc(quads_of(ts_pairs));
  unsigned long long ctr[kCounters] = {
      active ? (unsigned long long)R : 0ull, n_sampled,
      (unsigned long long)n_sampled * __popc(ts_pairs), (unsigned long long)n_sampled * __popc(ts_set),
      (unsigned long long)nstop, n_prune, n_forced, n_recomp,
      (unsigned long long)n_sampled * cq,
      (unsigned long long)(n_sampled - n_cert) * __popc(ts_pairs),
      (unsigned long long)(n_sampled + n_fall) * cq, (unsigned long long)(n_cert + n_fall) * 2 * cq,
      n_cert, n_fall};
#pragma unroll
  for (int qq = 0; qq < kCounters; ++qq) {
    unsigned long long v = ctr[qq];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0 && v) atomicAdd(a.counters + qq, v);
  }
}

// ------------------------------------------------------------------ variant readings (f2)
// The readings of P:L559 that SURVEY §8(f) f2 lists besides the ablations (DESIGN.md R-Q4v,
// R-Q1v, R-Q5v), for cells with ZEUS_VARIANT_* bits, combinable with the ablations:
//   retry (4):         after an early stop the recurrence continues with another decision
//                      (Thompson sampling leaves out the arms stopped in it) until a run is
//                      not stopped, or no arm is left; attempt j >= 1 draws from its own
//                      counters (pairs: q | j << 16, replica: (t, 3 << 24 | j, trial) word 0);
//   epoch stop (8):    the run stops at the end of the first epoch whose accumulated cost
//                      exceeds thr (unless that epoch is its last) and is charged that cost;
//   windowed best (16): thr = beta * the minimum converged cost of the last N recurrences.
// One thread per trial, one pass, Observe before the next attempt, full Thompson draw.
template <bool LOG>
__global__ void __launch_bounds__(128) variant_kernel(ConcArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int cell = blockIdx.y;
  const CellParam cp = a.cells[cell];
  const int tid = threadIdx.x, TPB = blockDim.x;
  const int64_t j0 = (int64_t)blockIdx.x * TPB;
  if (j0 >= cp.n || cp.policy != 0 || cp.conc != 2) return;
  double2 *s_ms = reinterpret_cast<double2 *>(smem);       // [arm][thread] (mu, sigma)
  const int B = a.B, R = a.R, S = a.S, K = a.K, P = a.P;
  const ArmConst *arm = a.arms + (size_t)cell * B;
  const double *regret = a.regret + (size_t)cell * a.reg_stride;
  const int32_t *optarm = a.opt_arm + (size_t)cell * a.opt_stride;
  const int64_t jj = j0 + tid;
  const bool active = jj < cp.n;
  const int64_t trial = cp.begin + jj;
  const size_t o = (size_t)(cp.out_off + jj);
  const RecRef st{a.st, (uint32_t)(o * B)};               // the trial's Observe records (32-bit index)
  const int warp_global = blockIdx.x * (TPB >> 5) + (tid >> 5);
  long long *curves = a.curve_slots + ((size_t)cell * a.nslot + (warp_global % a.nslot)) * (size_t)R * kRow;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const bool no_prune = cp.ablation & 1, no_jit = cp.ablation & 2, retry = cp.ablation & 4;
  const bool epoch_stop = cp.ablation & 8, win_best = cp.ablation & 16;
  const int NB = win_best ? cp.window : 0;
  double *bring = a.best_ring + o * (size_t)a.best_n;
  if (active)
    for (int u = 0; u < NB; ++u) bring[u] = kInf;

  uint32_t profiled = 0, seen = 0, mature = 0;
  double best = kInf;
  bool in_ts = false;
  int round = 1, step = kStart, start = a.b0, cursor = a.b0;
  const uint32_t all_arms = (B == 32) ? 0xffffffffu : ((1u << B) - 1u);
  uint32_t cand = all_arms, surv = 0, ts_set = 0;
  double r1_cost = kInf;
  int r1_arm = -1;
  double totC = 0.0, totE = 0.0, totT = 0.0;
  unsigned long long dig = 0xcbf29ce484222325ull;
  int nstop = 0, last_b = -1;
  uint32_t n_dec = 0, n_sampled = 0, n_prune = 0, n_forced = 0, n_recomp = 0;
  unsigned long long n_pairs = 0, n_normals = 0, n_blocks = 0;   // the method's events
  unsigned long long w_pairs = 0, w_blocks = 0, w_fp32 = 0;      // the work this build did
  // certified fp32 draw (a.cert_draw): fp32 (mu - ref, sigma) of every mature
  // arm after the (mu, sigma) table, ref fixed when Thompson sampling starts; the eligibility of
  // an attempt (survivors not stopped in this recurrence) masks the keys
  const int cpairs2 = ((((B + 1) >> 1) + 1) & ~1);
  float2 *s_f2 = reinterpret_cast<float2 *>(smem + (size_t)((B + 1) & ~1) * 16 * TPB);
  const int ckbits = 32 - __clz(2 * cpairs2 - 1);
  const uint32_t ckeep = ~((1u << ckbits) - 1u);
  const float ckth = cert::kTheta + __int_as_float((127 - 23 + ckbits) << 23) * 1.000001f;
  double cref = 0.0;
  float c_trial = 0.0f;
  uint32_t n_cert = 0, n_fall = 0;
  auto f32_slot = [&](int arm_i, double2 ms) {
    const double dm = ms.x - cref;
    s_f2[2 * ((arm_i >> 1) * TPB + tid) + (arm_i & 1)] =
        (fabs(dm) < 1e30 && ms.y < 1e30) ? make_float2((float)dm, (float)ms.y)
                                         : make_float2(0.0f, __int_as_float(0x7f800000));
  };
  auto cert_begin = [&]() {
    const int lead = __ffs(ts_set & mature) - 1;
    cref = lead >= 0 ? s_ms[lead * TPB + tid].x : 0.0;
    if (!(fabs(cref) < 1e30)) cref = 0.0;
    c_trial = __double2float_ru(fabs(cref) * 0x1p-52 + 0x1p-120);
    for (int arm_i = 0; arm_i < 2 * cpairs2; ++arm_i)
      if ((mature >> arm_i) & 1u) f32_slot(arm_i, s_ms[arm_i * TPB + tid]);
  };

  int s = 0;
  U4 rw{0u, 0u, 0u, 0u};
  ArmStat qc{0.0, 0.0, 0.0, 0, 0};                     // the last arm's record (read cache)
  int qc_b = -1;
  for (int t = 0; t < R; ++t) {
    double vC = 0.0, vE = 0.0, vT = 0.0, vReg = 0.0;
    uint32_t cStop = 0, cOpt = 0, cTs = 0;
    if (S > 1)
      while ((long long)(s + 1) * R <= (long long)t * S) ++s;
    if (active) {
      if ((t & 3) == 0) rw = replica_words(cp.key0, cp.key1, trial, t);
      double best_now = best;
      if (win_best) {                                        // R-Q5v: the last N recurrences
        best_now = kInf;
        for (int u = 0; u < NB; ++u) best_now = fmin(best_now, bring[u]);
      }
      const double thr = cp.beta * best_now;
      double conv_t = kInf;
      uint32_t stopped_here = 0u;                            // arms stopped in this recurrence
      for (int j = 0;; ++j) {
        if (j > 0 && in_ts && (ts_set & ~stopped_here) == 0u) break;   // nothing left to retry
        const uint32_t elig = ts_set & ~stopped_here;
        // ---------------- step 2: decide
        const bool ts_dec = in_ts;
        int b;
        if (!in_ts) {
          b = (step == kStart) ? start
            : (step == kDown) ? 31 - __clz(cand & below_mask(cursor))
                              : __ffs(cand & above_mask(cursor)) - 1;
          n_prune += 1;
        } else {
          const uint32_t unripe = elig & ~mature;
          if (unripe) {
            b = __ffs(unripe) - 1;
            n_forced += 1;
          } else {
            double bt = kInf;
            b = -1;
            bool exact = true;
            uint32_t ep = 0u;                                // eligible pairs of this attempt
            for (int k = 0; 2 * k < B; ++k)
              if ((elig >> (2 * k)) & 3u) ep |= 1u << k;
            n_pairs += __popc(ep);
            n_normals += __popc(elig);
            n_blocks += __popc(quads_of(ep));
            if (a.cert_draw) {                               // certified fp32 draw (§7.9)
              cert::Argmin32 am;
              am.init();
              uint32_t qm = quads_of(ep);
              while (qm) {
                const int qd = __ffs(qm) - 1;
                qm &= qm - 1u;
                const U4 x = pair_block(cp.key0, cp.key1, trial, t, qd | (j << 16));
                w_blocks += 1;
                w_fp32 += 2;
                const float4 f0 = reinterpret_cast<const float4 *>(s_f2)[(2 * qd) * TPB + tid];
                const float4 f1 = reinterpret_cast<const float4 *>(s_f2)[(2 * qd + 1) * TPB + tid];
                float z0, z1, rsq;
                cert::normal_pair32(x.x, x.y, z0, z1, rsq);
                am.pair_masked(4 * qd, f0, z0, z1, rsq, ckeep, (elig >> (4 * qd)) & 3u);
                cert::normal_pair32(x.z, x.w, z0, z1, rsq);
                am.pair_masked(4 * qd + 2, f1, z0, z1, rsq, ckeep, (elig >> (4 * qd + 2)) & 3u);
              }
              if (am.certified(c_trial, ckth) && !a.force_exact) {
                b = am.arg(ckeep);
                exact = false;
                n_cert += 1;
              } else {
                n_fall += 1;
              }
            }
            int qcur = -1;
            U4 xq{0u, 0u, 0u, 0u};
            for (int k = 0; exact && 2 * k < B; ++k) {
              const uint32_t two = (elig >> (2 * k)) & 3u;
              if (!two) continue;
              if ((k >> 1) != qcur) {
                qcur = k >> 1;
                xq = pair_block(cp.key0, cp.key1, trial, t, qcur | (j << 16));
                w_blocks += 1;
              }
              double z0, z1;
              box_muller((k & 1) ? xq.z : xq.x, (k & 1) ? xq.w : xq.y, z0, z1, a.logtab);
              w_pairs += 1;
              const double2 m0 = s_ms[(2 * k) * TPB + tid];
              const double2 m1 = s_ms[(2 * k + 1) * TPB + tid];
              const double th0 = fma(m0.y, z0, m0.x);
              const bool take0 = (two & 1u) && (th0 < bt);
              bt = take0 ? th0 : bt;
              b = take0 ? 2 * k : b;
              const double th1 = fma(m1.y, z1, m1.x);
              const bool take1 = (two & 2u) && (th1 < bt);
              bt = take1 ? th1 : bt;
              b = take1 ? 2 * k + 1 : b;
            }
            n_sampled += 1;
          }
        }
        // the power limit; "no JIT" tries the limits in ascending order first
        const bool was_seen = (seen >> b) & 1u;
        ArmStat q;
        if (b == qc_b) q = qc; else if (was_seen) q = st[b]; else q = ArmStat{0.0, 0.0, 0.0, 0, 0};
        const ArmConst ac = arm[b];
        int p = ac.pstar;
        double c1b = ac.c1, t1b = ac.t1, e1b = ac.e1;
        if (no_jit) {
          const int runs = was_seen ? q.cnt : 0;
          if (runs < P) {
            p = runs;
            const double Ab = __ldg(a.A + (size_t)b * P + p), Thb = __ldg(a.Th + (size_t)b * P + p);
            c1b = ((cp.eta * Ab) + ((1.0 - cp.eta) * a.MP)) / Thb;
            t1b = 1.0 / Thb;
            e1b = Ab / Thb;
          }
        }
        // ---------------- step 3: replay one recorded run
        const uint32_t rword = j == 0 ? pick_word(rw, t)
            : philox4x32_10(U4{(uint32_t)t, 0x03000000u | (uint32_t)j, (uint32_t)trial,
                               (uint32_t)((uint64_t)trial >> 32)}, cp.key0, cp.key1).x;
        const uint32_t r = __umulhi(rword, (uint32_t)K);
        const int E = __ldg(a.pool + ((size_t)s * B + b) * K + r);
        const int Erun = E > 0 ? E : a.max_epochs;
        double c0, t0, e0;
        const bool prof_now = !no_jit && a.charge_profiling && !((profiled >> b) & 1u);
        if (prof_now) { c0 = ac.cP; t0 = ac.tP; e0 = ac.eP; } else { c0 = c1b; t0 = t1b; e0 = e1b; }
        profiled |= 1u << b;
        const double em1 = (double)(Erun - 1);
        const double Cf = c0 + em1 * c1b;
        // ---------------- step 4: early stop
        double C, Tm, En;
        bool stopped = false;
        if (Cf > thr && epoch_stop) {
          // first epoch k with c0 + (k-1) c1 > thr: a guess from one division, then the exact
          // test of the definition (the left side is non-decreasing in k)
          int k = 1;
          if (!(c0 > thr)) {
            const double g = floor((thr - c0) / c1b);
            k = (g >= (double)Erun) ? Erun : (int)g + 2;
            if (k < 2) k = 2;
            while (k > 2 && c0 + (double)(k - 2) * c1b > thr) --k;
            while (!(c0 + (double)(k - 1) * c1b > thr)) ++k;
          }
          if (k < Erun) {
            stopped = true;
            const double em = (double)(k - 1);
            C = c0 + em * c1b;
            Tm = t0 + em * t1b;
            En = e0 + em * e1b;
          } else {
            C = Cf;
            Tm = t0 + em1 * t1b;
            En = e0 + em1 * e1b;
          }
        } else if (Cf > thr) {
          stopped = true;
          C = thr;
          if (thr <= c0) {
            const double phi = thr / c0;
            Tm = phi * t0;
            En = phi * e0;
          } else {
            const double phi = (thr - c0) / c1b;
            Tm = t0 + phi * t1b;
            En = e0 + phi * e1b;
          }
        } else {
          C = Cf;
          Tm = t0 + em1 * t1b;
          En = e0 + em1 * e1b;
        }
        const bool conv = (E > 0) && !stopped;
        if (conv) {
          conv_t = C;
          if (!(C >= best)) best = C;
        }
        // ---------------- Alg. 2 Observe (before the next attempt decides)
        {
          const int cnt = was_seen ? q.cnt : 0;
          double sh, S1, S2;
          if (!was_seen) { sh = C; S1 = 0.0; S2 = 0.0; }
          else { sh = q.sh; S1 = q.S1; S2 = q.S2; }
          int n = cnt;
          if (a.ring_n > 0 && cp.window > 0) {
            const int N = cp.window;
            double *slot = &a.st_ring[(o * B + b) * (size_t)a.ring_n + (cnt % N)];
            if (cnt >= N) {
              const double dy = *slot - sh;
              S1 = S1 - dy;
              S2 = S2 - dy * dy;
              n = N - 1;
            }
            *slot = C;
          }
          const double d = C - sh;
          S1 = S1 + d;
          S2 = S2 + d * d;
          n += 1;
          ArmStat nq;
          nq.sh = sh; nq.S1 = S1; nq.S2 = S2; nq.cnt = cnt + 1; nq.pad = 0;
          st[b] = nq;
          qc = nq;
          qc_b = b;
          seen |= 1u << b;
          if (n >= 2) {
            const double2 ms = posterior(sh, S1, S2, n, cp.prec0, cp.pm0);
            s_ms[b * TPB + tid] = ms;
            if (a.cert_draw && in_ts) f32_slot(b, ms);
            mature |= 1u << b;
            n_recomp += 1;
          }
        }
        // ---------------- Alg. 3 bookkeeping
        if (!in_ts) {
          if (conv) {
            surv |= 1u << b;
            if (round == 1 && (C < r1_cost || (C == r1_cost && b < r1_arm))) { r1_cost = C; r1_arm = b; }
          }
          bool end_round = false;
          if (step == kStart) { step = kDown; cursor = start; }
          else if (step == kDown) { if (conv) cursor = b; else { step = kUp; cursor = start; } }
          else { if (conv) cursor = b; else end_round = true; }
          if (!end_round && step == kDown && (cand & below_mask(cursor)) == 0u) { step = kUp; cursor = start; }
          if (!end_round && step == kUp && (cand & above_mask(cursor)) == 0u) end_round = true;
          if (end_round) {
            if (surv == 0u) surv = 1u << start;
            if (round == 1) {
              cand = no_prune ? all_arms : surv;
              if (r1_arm >= 0) start = r1_arm;
              surv = 0u;
              round = 2;
              step = kStart;
              cursor = start;
            } else {
              in_ts = true;
              ts_set = no_prune ? all_arms : surv;
              if (a.cert_draw) cert_begin();
            }
          }
        }
        // ---------------- accumulate (every attempt is a decision)
        const uint32_t flags = (stopped ? 1u : 0u) | (conv ? 2u : 0u) | (prof_now ? 4u : 0u) |
                               (ts_dec ? 8u : 0u) | (j > 0 ? 16u : 0u);
        n_dec += 1;
        totC += C;
        totE += En;
        totT += Tm;
        nstop += stopped ? 1 : 0;
        last_b = b;
        dig = (dig ^ (unsigned long long)(uint32_t)b) * 0x100000001b3ull;
        dig = (dig ^ (unsigned long long)(uint32_t)p) * 0x100000001b3ull;
        dig = (dig ^ (unsigned long long)flags) * 0x100000001b3ull;
        if (LOG) a.log[o * R + t] = (uint32_t)b | ((uint32_t)p << 8) | (flags << 16);
        vC += C;
        vE += En;
        vT += Tm;
        vReg += (p == ac.pstar) ? __ldg(regret + (size_t)s * B + b)
                                : __ldg(a.ebar + (size_t)s * B + b) * c1b - __ldg(a.opt + (size_t)cell * S + s);
        cStop += stopped ? 1u : 0u;
        cOpt += (b == __ldg(optarm + s) && p == ac.pstar) ? 1u : 0u;
        cTs += ts_dec ? 1u : 0u;
        if (!(retry && stopped)) break;
        stopped_here |= 1u << b;
      }
      if (win_best) bring[t % NB] = conv_t;
    }
    // sums in fixed point by REDUX; the counts (up to one per attempt) by REDUX each
    curve_accumulate(curves, t, tid & 31, vC, vE, vT, vReg, 0, a.curve_scale);
    const unsigned k4 = __reduce_add_sync(0xffffffffu, cStop), k5 = __reduce_add_sync(0xffffffffu, cOpt),
                   k6 = __reduce_add_sync(0xffffffffu, cTs);
    if ((tid & 31) == 0) {                  // counts live in limb 0 of their quantity
      long long *row = curves + (size_t)t * kRow;
      if (k4) atomicAdd(reinterpret_cast<unsigned long long *>(row + 4 * kLimbs), (unsigned long long)k4);
      if (k5) atomicAdd(reinterpret_cast<unsigned long long *>(row + 5 * kLimbs), (unsigned long long)k5);
      if (k6) atomicAdd(reinterpret_cast<unsigned long long *>(row + 6 * kLimbs), (unsigned long long)k6);
    }
  }
  if (active) {
    a.tot_cost[o] = totC;
    a.tot_energy[o] = totE;
    a.tot_time[o] = totT;
    a.digest[o] = dig;
    a.n_stop[o] = nstop;
    a.final_arm[o] = last_b;
  }
  unsigned long long ctr[kCounters] = {
      active ? (unsigned long long)n_dec : 0ull, n_sampled, n_pairs, n_normals,
      (unsigned long long)nstop, n_prune, n_forced, n_recomp, n_blocks,
      w_pairs, w_blocks, w_fp32, n_cert, n_fall};
#pragma unroll
  for (int qq = 0; qq < kCounters; ++qq) {
    unsigned long long v = ctr[qq];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0 && v) atomicAdd(a.counters + qq, v);
  }
}

// ------------------------------------------------------------------ §6.1 baselines
// Default (b0, largest power limit) and Grid Search with pruning,
// replayed on the same traces with the same replica draws as Zeus.
// Neither uses the JIT profiler or the early stop (R-Q29).  One thread per trial; the
// per-epoch cost of (b, p) is Eq. 7's inner term in the NC-2 order.
struct BaselineArgs {
  const CellParam *cells;
  const double *A, *Th;           // [B][P]
  const int32_t *pool;            // [S][B][K]
  const ArmConst *arms;           // [cells][B] (p*)
  const double *ebar;             // [S][B]
  const double *opt;              // [cells][S]
  const int32_t *opt_arm;         // [cells][opt_stride]
  long long *curve_slots;         // [cells][nslot][R][kQ][kLimbs] fixed point (curve_accumulate)
  double curve_scale;             // 2^F of the fixed point
  double *tot_cost, *tot_energy, *tot_time;
  unsigned long long *digest;
  int32_t *n_stop, *final_arm;
  uint32_t *log;
  unsigned long long *counters;
  int B, P, S, K, R, max_epochs, b0, nslot, opt_stride;
  double MP;
};

template <bool LOG>
__global__ void __launch_bounds__(128) baseline_kernel(BaselineArgs a) {
  const int cell = blockIdx.y;
  const CellParam cp = a.cells[cell];
  const int tid = threadIdx.x;
  const int64_t j0 = (int64_t)blockIdx.x * blockDim.x;
  if (j0 >= cp.n || cp.policy == 0) return;
  const int64_t jj = j0 + tid;
  const bool active = jj < cp.n;
  const int64_t trial = cp.begin + jj;
  const size_t o = (size_t)(cp.out_off + jj);
  const int B = a.B, P = a.P, S = a.S, K = a.K, R = a.R;
  const int warp_global = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
  long long *curves = a.curve_slots + ((size_t)cell * a.nslot + (warp_global % a.nslot)) * (size_t)R * kRow;
  const ArmConst *arms = a.arms + (size_t)cell * B;
  bool exploring = cp.policy == 2;
  U4 rw{0u, 0u, 0u, 0u};
  int gb = 0, gp = 0;
  double best_c = __longlong_as_double(0x7ff0000000000000ll);
  int best_b = -1, best_p = -1;
  double totC = 0.0, totE = 0.0, totT = 0.0;
  unsigned long long dig = 0xcbf29ce484222325ull;
  int last_b = -1, s = 0;
  for (int t = 0; t < R; ++t) {
    double vC = 0.0, vE = 0.0, vT = 0.0, vReg = 0.0;
    int vPacked = 0;
    if (S > 1)
      while ((long long)(s + 1) * R <= (long long)t * S) ++s;
    if (active) {
      int b, p;
      if (cp.policy == 1) { b = a.b0; p = P - 1; }
      else if (exploring) { b = gb; p = gp; }
      else if (best_b >= 0) { b = best_b; p = best_p; }
      else { b = a.b0; p = P - 1; }                     // nothing converged in the grid
      const double Ab = __ldg(a.A + (size_t)b * P + p), Thb = __ldg(a.Th + (size_t)b * P + p);
      const double c = ((cp.eta * Ab) + ((1.0 - cp.eta) * a.MP)) / Thb;
      const double tt = 1.0 / Thb, e = Ab / Thb;
      if ((t & 3) == 0) rw = replica_words(cp.key0, cp.key1, trial, t);
      const uint32_t r = __umulhi(pick_word(rw, t), (uint32_t)K);
      const int E = __ldg(a.pool + ((size_t)s * B + b) * K + r);
      const int Erun = E > 0 ? E : a.max_epochs;
      const double em1 = (double)(Erun - 1);
      const double C = c + em1 * c, Tm = tt + em1 * tt, En = e + em1 * e;
      const bool conv = E > 0;
      if (exploring) {
        if (conv && C < best_c) { best_c = C; best_b = b; best_p = p; }
        if (!conv || gp == P - 1) { gb += 1; gp = 0; } else gp += 1;
        if (gb == B) exploring = false;
      }
      const uint32_t flags = conv ? 2u : 0u;
      totC += C;
      totE += En;
      totT += Tm;
      last_b = b;
      dig = (dig ^ (unsigned long long)(uint32_t)b) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)(uint32_t)p) * 0x100000001b3ull;
      dig = (dig ^ (unsigned long long)flags) * 0x100000001b3ull;
      if (LOG) a.log[o * R + t] = (uint32_t)b | ((uint32_t)p << 8) | (flags << 16);
      vC = C;
      vE = En;
      vT = Tm;
      vReg = __ldg(a.ebar + (size_t)s * B + b) * c - __ldg(a.opt + (size_t)cell * S + s);
      vPacked = (b == __ldg(a.opt_arm + (size_t)cell * a.opt_stride + s) && p == arms[b].pstar) ? (1 << 8) : 0;
    }
    curve_accumulate(curves, t, tid & 31, vC, vE, vT, vReg, vPacked, a.curve_scale);
  }
  if (active) {
    a.tot_cost[o] = totC;
    a.tot_energy[o] = totE;
    a.tot_time[o] = totT;
    a.digest[o] = dig;
    a.n_stop[o] = 0;
    a.final_arm[o] = last_b;
  }
  unsigned long long v = active ? (unsigned long long)R : 0ull;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if ((tid & 31) == 0 && v) atomicAdd(a.counters, v);
}

// ------------------------------------------------------------------ Pareto front (f4)
// §2.3: the (TTA, ETA) grid of slice s -- TTA = Ebar/Th, ETA = (Ebar*A)/Th for
// every b with a converged replica -- and its non-dominated points (ties on both axes keep
// the first in (b, p) order).  One block per slice, threads over points, ebar from step 1.
__global__ void pareto_kernel(const double *A, const double *Th, const double *ebar,
                              const int32_t *pool, uint8_t *mask, int B, int P, int K) {
  const int s = blockIdx.x;
  const int n = B * P;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    auto point = [&](int q, double &t, double &e) -> bool {
      const int b = q / P;
      bool any = false;
      for (int k = 0; k < K; ++k) any |= pool[((size_t)s * B + b) * K + k] > 0;
      if (!any) return false;
      const double eb = ebar[(size_t)s * B + b];
      t = eb / Th[q];
      e = (eb * A[q]) / Th[q];
      return true;
    };
    double ti, ei;
    bool keep = point(i, ti, ei);
    for (int j = 0; j < n && keep; ++j) {
      double tj, ej;
      if (j == i || !point(j, tj, ej)) continue;
      const bool le = tj <= ti && ej <= ei;
      const bool lt = tj < ti || ej < ei;
      if (le && lt) keep = false;
      if (!lt && le && j < i) keep = false;
    }
    mask[(size_t)s * n + i] = keep ? 1 : 0;
  }
}

// The exact curve sums: fixed[cell][t][q][limb] = the slots' integer sums (any order), then
// carried into 26-bit limbs and rounded once to fp64: curves = RN(l2 2^52 + (l1 2^26 + l0)) 2^-F.
__device__ __forceinline__ double fixed_to_double(long long l0, long long l1, long long l2,
                                                  double inv_scale) {
  l1 += l0 >> kLimbBits;                    // arithmetic shifts: floor, so the low limbs end in
  l0 &= (1ll << kLimbBits) - 1;             // [0, 2^26) and the sign lives in l2
  l2 += l1 >> kLimbBits;
  l1 &= (1ll << kLimbBits) - 1;
  const double lo = (double)(l1 * (1ll << kLimbBits) + l0);    // < 2^52: exact
  return ((double)l2 * 0x1p52 + lo) * inv_scale;               // |l2| < 2^53: one rounding
}

// The counted runs (ReplayArgs::hist) into the fixed-point sums.  One thread per (cell, t, bin);
// bin = (class, b, replica r), class = 2 ts + prof.  The n runs of a bin were each charged what
// the replay computes for a run that is not stopped -- C = c0 + (E_run - 1) c1 with c0 = c_prof
// when it paid the profiling epoch and c1 otherwise (NC-5), the same for T and energy, the
// pseudo-regret of b -- so n RN(v 2^F) is added to slot 0 as an exact integer (three limbs, by
// 64-bit integer atomics), and n to the optimal (b = opt arm) and Thompson counts.  Runs after
// the replay kernels; the sums are then exactly those of run-by-run accumulation.
__global__ void curve_hist_fold_kernel(const uint32_t *hist, long long *slots, const ArmConst *arms,
                                       const double *regret, const int32_t *opt_arm,
                                       const int32_t *pool, int ncells, int nslot, int nhslot, int R,
                                       int B, int S, int K, int max_epochs, int reg_stride,
                                       int opt_stride, double scale) {
  const int HB = 4 * B * K;
  const long long total = (long long)ncells * R * HB;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int bin = (int)(i % HB);
    const long long ct = i / HB;                             // cell * R + t
    const int cell = (int)(ct / R), t = (int)(ct % R);
    long long n = 0;
    for (int k = 0; k < nhslot; ++k) n += hist[((size_t)ct * nhslot + k) * HB + bin];
    if (n == 0) continue;
    const int cls = bin / (B * K), b = (bin / K) % B, r = bin % K;
    const int s = (int)(((long long)t * S) / R);
    const ArmConst ac = arms[(size_t)cell * B + b];
    const bool prof = cls & 1;
    const double c0 = prof ? ac.cP : ac.c1, t0 = prof ? ac.tP : ac.t1, e0 = prof ? ac.eP : ac.e1;
    const int E = pool[((size_t)s * B + b) * K + r];
    const int Erun = E > 0 ? E : max_epochs;
    const double em1 = (double)(Erun - 1);
    const double v[4] = {c0 + em1 * ac.c1, e0 + em1 * ac.e1, t0 + em1 * ac.t1,
                         regret[(size_t)cell * reg_stride + (size_t)s * B + b]};
    unsigned long long *row = reinterpret_cast<unsigned long long *>(slots + ((size_t)cell * nslot * R + t) * kRow);
    for (int q = 0; q < 4; ++q) {
      const __int128 T = (__int128)n * (__int128)__double2ll_rn(v[q] * scale);
      atomicAdd(row + q * kLimbs + 0, (unsigned long long)(long long)(T & ((1 << kLimbBits) - 1)));
      atomicAdd(row + q * kLimbs + 1, (unsigned long long)(long long)((T >> kLimbBits) & ((1 << kLimbBits) - 1)));
      atomicAdd(row + q * kLimbs + 2, (unsigned long long)(long long)(T >> (2 * kLimbBits)));
    }
    if (b == opt_arm[(size_t)cell * opt_stride + s]) atomicAdd(row + 5 * kLimbs, (unsigned long long)n);
    if (cls & 2) atomicAdd(row + 6 * kLimbs, (unsigned long long)n);
  }
}

__global__ void curve_reduce_kernel(const long long *slots, long long *fixed, double *curves,
                                    int ncells, int nslot, int R, double inv_scale) {
  // one warp per output value: lanes sum the slot copies (integers: exact in any order), a
  // shuffle tree adds the lanes, lane 0 carries the limbs and rounds once
  const long long total = (long long)ncells * R * kQ;
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < total; i += nwarps) {
    const long long cell = i / ((long long)R * kQ);
    const long long rq = i % ((long long)R * kQ);
    const long long *src = slots + (size_t)cell * nslot * (size_t)R * kRow + rq * kLimbs;
    long long l[kLimbs] = {0, 0, 0};
    for (int k = lane; k < nslot; k += 32)
#pragma unroll
      for (int m = 0; m < kLimbs; ++m) l[m] += src[(size_t)k * R * kRow + m];
#pragma unroll
    for (int m = 0; m < kLimbs; ++m)
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) l[m] += __shfl_xor_sync(0xffffffffu, l[m], off);
    if (lane == 0) {
#pragma unroll
      for (int m = 0; m < kLimbs; ++m) fixed[i * kLimbs + m] = l[m];
      const bool count = rq % kQ >= 4;     // counts are plain integers in limb 0
      curves[i] = count ? (double)l[0] : fixed_to_double(l[0], l[1], l[2], inv_scale);
    }
  }
}

// curves from (all-reduced) fixed-point sums [n][kQ][kLimbs] -- the same rounding as above
__global__ void curves_from_fixed_kernel(const long long *fixed, double *curves, long long n,
                                         double inv_scale) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n * kQ;
       i += (long long)gridDim.x * blockDim.x) {
    const long long *l = fixed + i * kLimbs;
    curves[i] = (i % kQ >= 4) ? (double)l[0] : fixed_to_double(l[0], l[1], l[2], inv_scale);
  }
}

}  // namespace zs
