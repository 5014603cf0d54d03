// thompson.cuh -- the Thompson-sampling phase of the two-phase schedule
// with the certified fp32 draw of certify.cuh.
//
// thompson_kernel<LOG, RK, SREC, WIN> runs recurrences t_split..R-1 of every trial of a launch whose
// cells have no ablation, after replay_kernel's phase A (Alg. 3 pruning) and the
// regroup.  Per decision (Alg. 1, then steps 3-4 as in replay_kernel):
//   * every survivor quad's Philox block (NC-3) is drawn; both of its Box-Muller pairs are
//     transformed in fp32 and every arm's theta in fp32 with its error bound (certify.cuh);
//   * when the smallest interval lies strictly below the others its arm is the contract's
//     argmin; otherwise (rare) the exact fp64 draw of the contract decides, from the fp64
//     posteriors recomputed from the Observe records;
//   * the rest of the decision is the contract's fp64 arithmetic, unchanged.
// Lanes were regrouped by their number of survivor quads, so the quad loop has the same trip
// count in every lane of a warp.  (mu - ref, sigma) of every arm live in shared memory as fp32,
// 8 B per arm (half of the fp64 pair the exact-screen kernel keeps).
#pragma once
#include "certify.cuh"
#include "kernels.cuh"

namespace zs {

#ifndef ZS_PHILOX_PREFIX
#define ZS_PHILOX_PREFIX 1
#endif
#ifndef ZS_QUAD2
#define ZS_QUAD2 1
#endif
#ifndef ZS_WIN_MIN_BLOCKS
#define ZS_WIN_MIN_BLOCKS 6
#endif
#ifndef ZS_WIN_POOL_FIT
#define ZS_WIN_POOL_FIT 1
#endif
#ifndef ZS_WIN_PREFETCH
#define ZS_WIN_PREFETCH 1
#endif
#ifndef ZS_CURVES_REMAT
#define ZS_CURVES_REMAT 0     // the curve-slot pointer recomputed on the stopped-run path: -1.3 % (r02bj)
#endif
#ifndef ZS_TPB_CONST
#define ZS_TPB_CONST 0
#endif
#ifndef ZS_SMAX_UB
#define ZS_SMAX_UB 1        // CFG2 +2.5 %, CFG3 +0.4 %, CFG5 +0.2 %, CFG4 -0.5 % (session r02da)
#endif
#ifndef ZS_NOINIT
#define ZS_NOINIT 1         // CFG5 +0.2 %, CFG3 +0.5 % (session r02cw)
#endif
#ifndef ZS_ACT_REG
#define ZS_ACT_REG 1        // CFG5 +0.4 % (session r02cv)
#endif
#ifndef ZS_HIST32
#define ZS_HIST32 0
#endif
#ifndef ZS_REC32
#define ZS_REC32 1         // 32-bit Observe-record index (CFG5 +1.5 %, session r02cq)
#endif
#ifndef ZS_RED_PRED
#define ZS_RED_PRED 1      // the histogram RED predicated, no branch (+0.2 % with REC32, r02cq)
#endif
#ifndef ZS_PHILOX_WIDE
#define ZS_PHILOX_WIDE 1
#endif
#ifdef ZS_TH_MIN_BLOCKS
#define ZS_TH_BOUNDS __launch_bounds__(128, ZS_TH_MIN_BLOCKS)
#else
#define ZS_TH_BOUNDS __launch_bounds__(128)
#endif

// Philox4x32-10 of counter (t, 1<<24 | q, lo32 trial, hi32 trial) for several q at one (trial,
// t) (NC-3): the first three rounds share the products that do not depend on q.
//   round 0: M0 t (per decision), M1 lo32(trial) (per trial)
//   round 1: M1 z1 with z1 = hi(M0 t) ^ hi32(trial) ^ k1[0] (per decision)
//   round 2: M0 x2 with x2 = hi(M1 z1) ^ lo(M1 lo32 trial) ^ k0[1] (per decision)
struct PhiloxPrefix {
  uint32_t x1b, w1, y2, h0, l0;
};
template <class K0, class K1>
__device__ __forceinline__ PhiloxPrefix philox_prefix(uint32_t t, uint32_t tlo, uint32_t thi, K0 k0, K1 k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi1 = __umulhi(M1, tlo), lo1 = M1 * tlo;
  const uint32_t hi0 = __umulhi(M0, t), lo0 = M0 * t;
  PhiloxPrefix p;
  p.x1b = hi1 ^ 0x01000000u ^ k0(0);
  const uint32_t z1 = hi0 ^ thi ^ k1(0);
  p.w1 = lo0;
  const uint32_t H1 = __umulhi(M1, z1), L1 = M1 * z1;
  const uint32_t x2 = H1 ^ lo1 ^ k0(1);
  p.y2 = L1;
  p.h0 = __umulhi(M0, x2);
  p.l0 = M0 * x2;
  return p;
}
// 32 x 32 -> 64-bit product as one IMAD.WIDE.U32 (the compiler otherwise splits some of the
// rounds' products into IMAD.HI + IMAD under register pressure)
__device__ __forceinline__ void mul_wide(uint32_t a, uint32_t m, uint32_t &hi, uint32_t &lo) {
#if ZS_PHILOX_WIDE
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(m));
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
#else
  hi = __umulhi(a, m);
  lo = a * m;
#endif
}

template <class K0, class K1>
__device__ __forceinline__ U4 philox_from_prefix(const PhiloxPrefix &p, uint32_t q, K0 k0, K1 k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t x1 = p.x1b ^ q;                       // round 0 output x (y1 = lo(M1 tlo) is
  uint32_t H0, L0;                                     // consumed by the prefix's x2)
  mul_wide(x1, M0, H0, L0);
  const uint32_t z2 = H0 ^ p.w1 ^ k1(1);               // round 1 output (x2, y2 shared)
  const uint32_t w2 = L0;
  uint32_t H1, L1;
  mul_wide(z2, M1, H1, L1);
  U4 c{H1 ^ p.y2 ^ k0(2), L1, p.h0 ^ w2 ^ k1(2), p.l0};   // round 2 output
#pragma unroll
  for (int r = 3; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mul_wide(c.x, M0, hi0, lo0);
    mul_wide(c.z, M1, hi1, lo1);
    c = U4{hi1 ^ c.y ^ k0(r), lo1, hi0 ^ c.w ^ k1(r), lo0};
  }
  return c;
}

// Shared-memory tables of the windowed variant (WIN): the arm constants and the sampler's log
// table, and the trace pool when it is small; the pseudo-regret and optimum tables are read only
// on a stopped run's path, from global memory, so many slices (CFG4: 200) cost no residency.
// The offsets travel in the kernel parameters (ReplayArgs::th_*).
// The pool goes to shared memory when it is small, or when it still leaves the kernel its six
// blocks per SM (per_block = the block's per-thread state): a pool read through L1 sits on the
// decision's chain, and the carveout leaves L1 little room (CFG4: 19.2 KB, session r02br).
constexpr int kThPoolSmemMax = 16384;
constexpr int kThSmemPerSm = 227 * 1024;
struct ThTabLayout {
  int arms, logtab, pool, bytes;
  bool pool_smem;
  __host__ __device__ ThTabLayout(int B, int S, int K, int per_block = 0) {
    arms = 0;
    logtab = TabLayout::align16(B * (int)sizeof(ArmConst));
    pool = TabLayout::align16(logtab + kLogTab * 16);
    const int pb = S * B * K * 4;
    pool_smem = pb <= kThPoolSmemMax ||
                (ZS_WIN_POOL_FIT && (TabLayout::align16(pool + pb) + per_block + 1024) * ZS_WIN_MIN_BLOCKS <= kThSmemPerSm);
    bytes = pool_smem ? TabLayout::align16(pool + pb) : pool;
  }
};

// SREC (launches of at most a couple of waves, where one warp per scheduler makes the decision's
// latency the throughput): every survivor's Observe record lives in shared memory for the whole
// phase ([arm][thread], after the replica words), loaded once at the start and written back at
// the end, so a decision that moves to another arm waits on a shared-memory load, not on L2.
// WIN: some cell has a window N: each Observe evicts the cost that leaves the arm's
// window from the HBM ring (loaded as soon as the decision is known) and the posterior uses
// n = min(count, N), as replay_kernel's windowed path; six blocks per SM (one wave of 10^5 trials).
// EARLY (ReplayArgs::early_split): phase A stopped each lane at its first pure Thompson decision
// (Carry::t0 <= t_split); the warp starts at its lanes' earliest t0 and a lane idles until its own.
template <bool LOG, bool RK, bool SREC, bool WIN, bool EARLY>
__device__ __forceinline__ void thompson_body(const ReplayArgs &a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  const int cell = blockIdx.y;
  const CellParam cp = a.cells[cell];
#if ZS_TPB_CONST
  // every Thompson launch has 128-thread blocks (zeus_sim.cu thompson_launch): the shared-memory
  // indexing folds to shifts and immediate offsets
  constexpr int TPB = 128;
  const int tid = threadIdx.x;
#else
  const int tid = threadIdx.x, TPB = blockDim.x;
#endif
  const int64_t j0 = (int64_t)blockIdx.x * TPB;
  if (j0 >= cp.n || cp.policy != 0 || cp.conc) return;
  auto k0f = [&](int r) -> uint32_t {
    if constexpr (RK) return a.rk.k0[r];
    else return cp.key0 + (uint32_t)r * 0x9E3779B9u;
  };
  auto k1f = [&](int r) -> uint32_t {
    if constexpr (RK) return a.rk.k1[r];
    else return cp.key1 + (uint32_t)r * 0xBB67AE85u;
  };
  auto block_c = [&](int64_t tr, int tt, int q) -> U4 {
    if constexpr (RK) return pair_block(a.rk, tr, tt, q);
    else return pair_block(cp.key0, cp.key1, tr, tt, q);
  };
  auto replica_words_c = [&](int64_t tr, int tt) -> U4 {
    if constexpr (RK) return replica_words(a.rk, tr, tt);
    else return replica_words(cp.key0, cp.key1, tr, tt);
  };

  // ---- stage the cell's tables with TMA bulk copies (one elected thread)
  const TabLayout L(a.B, a.S, a.K);
  const int tab_end = WIN ? a.th_bytes : a.tab_bytes;         // where the per-thread state starts
  if (tid == 0) {
    mbar_init(&mbar, 1);
    const uint32_t p_arm = (a.B * (uint32_t)sizeof(ArmConst) + 15u) & ~15u;
    const uint32_t p_reg = (a.S * a.B * 8u + 15u) & ~15u;
    const uint32_t p_opt = (a.S * 4u + 15u) & ~15u;
    const uint32_t p_pool = (a.S * a.B * a.K * 4u + 15u) & ~15u;
    if constexpr (WIN) {
      mbar_expect_tx(&mbar, p_arm + (a.th_pool_smem ? p_pool : 0u) + kLogTab * 16u);
      tma_bulk_load(smem + a.th_logtab, a.logtab, kLogTab * 16u, &mbar);
      tma_bulk_load(smem, a.arms + (size_t)cell * a.B, p_arm, &mbar);
      if (a.th_pool_smem) tma_bulk_load(smem + a.th_pool, a.pool, p_pool, &mbar);
    } else {
      mbar_expect_tx(&mbar, p_arm + p_reg + p_opt + p_pool + kLogTab * 16u);
      tma_bulk_load(smem + L.logtab, a.logtab, kLogTab * 16u, &mbar);
      tma_bulk_load(smem + L.arms, a.arms + (size_t)cell * a.B, p_arm, &mbar);
      tma_bulk_load(smem + L.regret, a.regret + (size_t)cell * a.reg_stride, p_reg, &mbar);
      tma_bulk_load(smem + L.optarm, a.opt_arm + (size_t)cell * a.opt_stride, p_opt, &mbar);
      tma_bulk_load(smem + L.pool, a.pool, p_pool, &mbar);
    }
  }
  __syncthreads();
  mbar_wait(&mbar, 0);

  const ArmConst *arm = reinterpret_cast<const ArmConst *>(smem + (WIN ? 0 : L.arms));
  const double *regret = reinterpret_cast<const double *>(smem + L.regret);     // !WIN only
  const int32_t *optarm = reinterpret_cast<const int32_t *>(smem + L.optarm);   // !WIN only
  const int32_t *pool = reinterpret_cast<const int32_t *>(smem + (WIN ? a.th_pool : L.pool));
  const double2 *logtab = reinterpret_cast<const double2 *>(smem + (WIN ? a.th_logtab : L.logtab));
  const int B = a.B, R = a.R, S = a.S, K = a.K;
  // fp32 (mu - ref, sigma) of arms 2k, 2k+1 of this thread: float4 [pair][thread]
  float4 *s_f = reinterpret_cast<float4 *>(smem + tab_end);
  float2 *s_f2 = reinterpret_cast<float2 *>(s_f);         // arm b: s_f2[2 ((b >> 1) TPB + tid) + (b & 1)]
  // the replica words of the current block of four recurrences (NC-3), [thread][4]: one LDS per
  // decision instead of four live registers
  uint32_t *s_rw = reinterpret_cast<uint32_t *>(smem + tab_end + (size_t)((((B + 1) >> 1) + 1) & ~1) * 16 * TPB);

  const bool active = j0 + tid < cp.n;
#if ZS_ACT_REG
  // `active` as an opaque 32-bit register: otherwise ptxas recomputes the 64-bit compare
  // j0 + tid < n (three ISETP) at every use in the loop
  uint32_t act_r;
  asm volatile("mov.u32 %0, %1;" : "=r"(act_r) : "r"(active ? 1u : 0u));
#endif
  const int64_t jj = active ? a.perm[cp.out_off + j0 + tid] : 0;
  const int64_t trial = cp.begin + jj;
  const size_t o = (size_t)(cp.out_off + jj);
  ArmStat *st_g = a.st + o * B;
  const uint32_t ob = (uint32_t)(o * B);                    // ZS_REC32: the trial's first record
  ArmStat *s_rec = reinterpret_cast<ArmStat *>(smem + tab_end +
                                               (size_t)((((B + 1) >> 1) + 1) & ~1) * 16 * TPB + 16 * (size_t)TPB);
  const int Nw = WIN ? cp.window : 0;                       // window of this cell (0: none)
  auto nwin = [&](int cnt) { return (WIN && Nw > 0) ? min(cnt, Nw) : cnt; };
  auto rec = [&](int arm_i) -> ArmStat & {
    if constexpr (SREC) return s_rec[(size_t)arm_i * TPB + tid];
#if ZS_REC32
    // 32-bit record index (the host guarantees shard * B < 2^32): one add and one wide multiply
    // from the uniform base, instead of 64-bit pointer arithmetic on every record switch
    else return *reinterpret_cast<ArmStat *>(reinterpret_cast<char *>(a.st) + (uint64_t)(ob + (uint32_t)arm_i) * 32u);
#else
    else return st_g[arm_i];
#endif
  };
  const int warp_global = blockIdx.x * (TPB >> 5) + (tid >> 5);
#if !ZS_CURVES_REMAT
  long long *curves = a.curve_slots + ((size_t)cell * a.nslot + (warp_global % a.nslot)) * (size_t)R * kRow;
#endif
  const int HB = 4 * B * K;
  // counted runs of class (Thompson decision, no profiling), row t_split; one row per t
  const size_t hstride = (size_t)a.nhslot * HB;
  // EARLY: this lane's first recurrence here (an inactive lane: never), the warp's first (lanes
  // were grouped by t0 within their quad count, so a warp's lanes mostly share it)
  const int t0 = EARLY ? (active ? a.carry[o].t0 : 0x7fffffff) : a.t_split;
  const int tw = EARLY ? min(R, __reduce_min_sync(0xffffffffu, t0)) : a.t_split;
#if ZS_HIST32
  // the row as a 32-bit element index from the uniform base (the histogram has < 2^32 bins)
  uint32_t hrow = (uint32_t)(((size_t)cell * R * a.nhslot + (warp_global % a.nhslot)) * (size_t)HB +
                             (size_t)tw * hstride + 2 * B * K);
#else
  uint32_t *hrow = a.hist + ((size_t)cell * R * a.nhslot + (warp_global % a.nhslot)) * (size_t)HB +
                   (size_t)tw * hstride + 2 * B * K;
#endif
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  const float kInfF = __int_as_float(0x7f800000);

  double best = kInf, totC = 0.0, totE = 0.0, totT = 0.0;
  unsigned long long dig = 0;
  uint32_t ts_set = 0, ts_pairs = 0, quads = 0;
  int nstop = 0, last_b = -1;
  uint32_t n_fall = 0;              // exact fallbacks (every phase-B decision samples and observes)
  double ref = 0.0;
  float c_trial = 0.0f;
#if ZS_SMAX_UB
  // an upper bound of every survivor's fp32 sigma (the certificate's smax): raised at each
  // Observe, recomputed exactly every 64 recurrences, so the quad loop does not track it
  float smax_ub = 0.0f;
#endif
  const int npairs = (B + 1) >> 1;
  const int npairs2 = (npairs + 1) & ~1;                    // whole quads (padding: non-survivors)
  // key packing (certify.cuh Argmin32): the arm index in the low `bits` mantissa bits
  const int kbits = 32 - __clz(2 * npairs2 - 1);
  const uint32_t keep = ~((1u << kbits) - 1u);
  const float kth = cert::kTheta + __int_as_float((127 - 23 + kbits) << 23) * 1.000001f;
  if (active) {                                             // resume from phase A
    const Carry c = a.carry[o];
    best = c.best; totC = c.totC; totE = c.totE; totT = c.totT; dig = c.dig;
    ts_set = c.ts_set;
    nstop = c.nstop; last_b = c.last_b;
    for (int k = 0; k < npairs; ++k)
      if ((ts_set >> (2 * k)) & 3u) ts_pairs |= 1u << k;
    quads = quads_of(ts_pairs);
    // ref: the posterior mean of the leader (the last arm run, or the first survivor), so the
    // fp32 (mu - ref) of the arms that compete with it are small
    if constexpr (SREC)                                     // the survivors' records, once
      for (int b = 0; b < B; ++b)
        if ((ts_set >> b) & 1u) s_rec[(size_t)b * TPB + tid] = st_g[b];
    const int lead = (last_b >= 0 && ((ts_set >> last_b) & 1u)) ? last_b : __ffs(ts_set) - 1;
    {
      const ArmStat q = rec(lead);
      ref = posterior(q.sh, q.S1, q.S2, nwin(q.cnt), cp.prec0, cp.pm0).x;
    }
    if (!(fabs(ref) < 1e30)) ref = 0.0;
    c_trial = __double2float_ru(fabs(ref) * 0x1p-52 + 0x1p-120);
    for (int b = 0; b < 2 * npairs2; ++b) {                 // every survivor was run (and observed
      // non-survivor slot: theta~ = 3e38 for every z, a finite key above every survivor's
      // (|mu'| < 1e30, sigma < 1e30), so it never wins and never hides a survivor's key
      float2 v = make_float2(3.0e38f, 0.0f);                // (every survivor ran at least twice)
      if ((ts_set >> b) & 1u) {
        const ArmStat q = rec(b);
        const double2 ms = posterior(q.sh, q.S1, q.S2, nwin(q.cnt), cp.prec0, cp.pm0);
        const double dm = ms.x - ref;
        v = (fabs(dm) < 1e30 && ms.y < 1e30) ? make_float2((float)dm, (float)ms.y) : make_float2(0.0f, kInfF);
      }
      s_f2[2 * ((b >> 1) * TPB + tid) + (b & 1)] = v;
#if ZS_SMAX_UB
      smax_ub = fmaxf(smax_ub, v.y);
#endif
    }
  }

  if (EARLY && active && (t0 & 3) != 0 && t0 < R) {         // the replica block holding t0
    const U4 rw = replica_words_c(trial, t0);
    reinterpret_cast<uint4 *>(s_rw)[tid] = make_uint4(rw.x, rw.y, rw.z, rw.w);
  }
  int s = 0;
  ArmStat qc{0.0, 0.0, 0.0, 0, 0};
  int qc_b = -1;
#if ZS_PHILOX_PREFIX
  const uint32_t tlo = (uint32_t)trial, thi = (uint32_t)((uint64_t)trial >> 32);
#endif
  for (int t = tw; t < R; ++t) {
#if ZS_ACT_REG
    const bool live = EARLY ? t >= t0 : act_r != 0u;        // this lane's trial decides at t
#else
    const bool live = EARLY ? t >= t0 : active;             // this lane's trial decides at t
#endif
#if ZS_NOINIT
    // read only where live (the decision assigns them first): no zeroing per recurrence
    double vC, vE, vT, vReg, C, y_old = 0.0;
    int vPacked = 0, b = 0, hkey = 0;                      // hkey: counted only when live
#else
    double vC = 0.0, vE = 0.0, vT = 0.0, vReg = 0.0;
    int vPacked = 0, b = 0, hkey = 0;                      // hkey: counted only when live
    double C = 0.0, y_old = 0.0;
#endif
    if (S > 1)
      while ((long long)(s + 1) * R <= (long long)t * S) ++s;
    if (live) {
      if ((t & 3) == 0 || (!EARLY && t == a.t_split)) {
        const U4 rw = replica_words_c(trial, t);
        reinterpret_cast<uint4 *>(s_rw)[tid] = make_uint4(rw.x, rw.y, rw.z, rw.w);
      }
#if ZS_WIN_PREFETCH
      // WIN: the evicted cost of the cached arm's window, loaded before the draw -- Thompson
      // sampling mostly repeats its arm, and then the ring load is off the decision's chain
      // (qc.pad = the arm's ring position cnt % N while the record is cached)
      const int pb = qc_b;
      double y_pre = 0.0;
      if (WIN && Nw > 0 && pb >= 0 && qc.cnt >= Nw) y_pre = a.st_ring[(o * B + pb) * (size_t)a.ring_n + qc.pad];
#endif
      // ---------------- step 2: Alg. 1, b = argmin_a theta_a over the survivors
      const uint32_t unripe = 0u;   // every Thompson-phase arm has n >= 2 (run twice in pruning)
      (void)unripe;
      {
        cert::Argmin32 am;
        am.init();
#if ZS_PHILOX_PREFIX
        const PhiloxPrefix pre = philox_prefix((uint32_t)t, tlo, thi, k0f, k1f);
#endif
        auto quad_block = [&](int qd) -> U4 {
#if ZS_PHILOX_PREFIX
          return philox_from_prefix(pre, (uint32_t)qd, k0f, k1f);
#else
          return block_c(trial, t, qd);
#endif
        };
        auto quad_argmin = [&](int qd, const U4 &x) {
          float z0, z1, rsq;
          const float4 m0 = s_f[(2 * qd) * TPB + tid];
          const float4 m1 = s_f[(2 * qd + 1) * TPB + tid];
          cert::normal_pair32(x.x, x.y, z0, z1, rsq);
#if ZS_SMAX_UB
          am.pair_nos(4 * qd, m0, z0, z1, rsq, keep);
          cert::normal_pair32(x.z, x.w, z0, z1, rsq);
          am.pair_nos(4 * qd + 2, m1, z0, z1, rsq, keep);
#else
          am.pair(4 * qd, m0, z0, z1, rsq, keep);
          cert::normal_pair32(x.z, x.w, z0, z1, rsq);
          am.pair(4 * qd + 2, m1, z0, z1, rsq, keep);
#endif
        };
        uint32_t qm = quads;
        while (qm) {                                        // the same trip count in a warp
          const int qa = __ffs(qm) - 1;
          qm &= qm - 1u;
#if ZS_QUAD2
          if (qm) {                                         // two quads: two independent Philox
            const int qb = __ffs(qm) - 1;                   // chains in one basic block
            qm &= qm - 1u;
            const U4 xa = quad_block(qa), xb = quad_block(qb);
            quad_argmin(qa, xa);
            quad_argmin(qb, xb);
            continue;
          }
#endif
          quad_argmin(qa, quad_block(qa));
        }
        b = am.arg(keep);
#if ZS_SMAX_UB
        if (!am.certified_ub(smax_ub, c_trial, kth) || a.force_exact) {
#else
        if (!am.certified(c_trial, kth) || a.force_exact) {
#endif
          // the contract's exact draw (NC-3/NC-4): fp64 posteriors from the Observe records
          // (the cached record is the newest of its arm), every survivor pair transformed,
          // strict < in ascending arm order
          n_fall += 1;
          double bt = kInf;
          b = -1;
          int qcur = -1;
          U4 xq{0u, 0u, 0u, 0u};
          uint32_t pm = ts_pairs;
          while (pm) {
            const int k = __ffs(pm) - 1;
            pm &= pm - 1u;
            if ((k >> 1) != qcur) {
              qcur = k >> 1;
              xq = block_c(trial, t, qcur);
            }
            double z0, z1;
            box_muller((k & 1) ? xq.z : xq.x, (k & 1) ? xq.w : xq.y, z0, z1, logtab);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int arm_i = 2 * k + h;
              if (!((ts_set >> arm_i) & 1u)) continue;
              const ArmStat q = (arm_i == qc_b) ? qc : rec(arm_i);
              const double2 ms = posterior(q.sh, q.S1, q.S2, nwin(q.cnt), cp.prec0, cp.pm0);
              const double th = fma(ms.y, h ? z1 : z0, ms.x);
              if (th < bt) { bt = th; b = arm_i; }
            }
          }
        }
      }
      // Observe record of arm b (write-back cache)
      if (b != qc_b) {
        if (qc_b >= 0) rec(qc_b) = qc;
        qc = rec(b);
        qc_b = b;
#if ZS_WIN_PREFETCH
        if (WIN && Nw > 0) qc.pad = qc.cnt % Nw;
#endif
      }
      // the windowed Observe's evicted cost, loaded as soon as the decision is known
#if ZS_WIN_PREFETCH
      if (WIN && Nw > 0 && qc.cnt >= Nw) {
        if (b == pb) y_old = y_pre;
        else y_old = a.st_ring[(o * B + b) * (size_t)a.ring_n + qc.pad];
      }
#else
      if (WIN && Nw > 0 && qc.cnt >= Nw)
        y_old = a.st_ring[(o * B + b) * (size_t)a.ring_n + (qc.cnt % Nw)];
#endif
      const ArmConst ac = arm[b];
      const int p = ac.pstar;
      const double c1b = ac.c1, t1b = ac.t1, e1b = ac.e1;
      // ---------------- step 3: replay one recorded run
      const uint32_t r = __umulhi(s_rw[4 * tid + (t & 3)], (uint32_t)K);
      const int pidx = (s * B + b) * K + (int)r;
      const int E = (!WIN || a.th_pool_smem) ? pool[pidx] : __ldg(a.pool + pidx);
      const int Erun = E > 0 ? E : a.max_epochs;
      hkey = b * K + (int)r;                               // bin (b, replica) of the row
      const double em1 = (double)(Erun - 1);
      const double Cf = c1b + em1 * c1b;
      // ---------------- step 4: early stop at β·min_t C_t, truncated charge
      const double thr = cp.beta * best;
      double Tm, En;
      const bool stopped = Cf > thr;
      if (stopped) {
        C = thr;
        if (thr <= c1b) {
          const double phi = thr / c1b;
          Tm = phi * t1b;
          En = phi * e1b;
        } else {
          const double phi = (thr - c1b) / c1b;
          Tm = t1b + phi * t1b;
          En = e1b + phi * e1b;
        }
      } else {
        C = Cf;
        Tm = t1b + em1 * t1b;
        En = e1b + em1 * e1b;
      }
      const bool conv = (E > 0) && !stopped;
      if (conv && !(C >= best)) best = C;
      const uint32_t flags = (stopped ? 1u : 0u) | (conv ? 2u : 0u) | 8u;
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
      vPacked = stopped ? 1 : 0;            // the rest of a stopped run's curve values below
    }
    {
      const bool special = live && (vPacked & 1);
#ifndef ZS_DIAG_NOHIST
#if ZS_RED_PRED
#if ZS_HIST32
      red_inc_u32_if(a.hist + (hrow + (uint32_t)hkey), live && !special);
#else
      red_inc_u32_if(hrow + (uint32_t)hkey, live && !special);
#endif
#else
      if (live && !special) red_add_u32(hrow + hkey, 1u);
#endif
#endif
      hrow += (uint32_t)hstride;
      if (__any_sync(0xffffffffu, special)) {
        // a stopped run's pseudo-regret and counts (stop | optimal << 8 | Thompson << 16) are read
        // only here (the counted runs take theirs from the histogram fold)
        if (special) {
          if constexpr (WIN) {                // global: a stopped run's path only
            vReg = __ldg(a.regret + (size_t)cell * a.reg_stride + s * B + b);
            vPacked = 1 | ((b == __ldg(a.opt_arm + (size_t)cell * a.opt_stride + s)) ? (1 << 8) : 0) | (1 << 16);
          } else {
            vReg = regret[s * B + b];
            vPacked = 1 | ((b == optarm[s]) ? (1 << 8) : 0) | (1 << 16);
          }
        }
#if ZS_CURVES_REMAT
        // the warp's slot row, recomputed on this rare path (no pointer held across the loop)
        long long *curves = a.curve_slots + ((size_t)cell * a.nslot + (warp_global % a.nslot)) * (size_t)R * kRow;
#endif
        curve_accumulate(curves, t, tid & 31, special ? vC : 0.0, special ? vE : 0.0, special ? vT : 0.0,
                         special ? vReg : 0.0, special ? vPacked : 0, a.curve_scale);
      }
    }
    if (live) {
      // ---------------- Alg. 2 Observe(b, C) with shifted sums and window N (NC-6)
      int n = qc.cnt;
      if (WIN && Nw > 0) {
        if (qc.cnt >= Nw) {                                 // the oldest cost leaves the window
          const double dy = y_old - qc.sh;
          qc.S1 = qc.S1 - dy;
          qc.S2 = qc.S2 - dy * dy;
          n = Nw - 1;
        }
#if ZS_WIN_PREFETCH
        a.st_ring[(o * B + b) * (size_t)a.ring_n + qc.pad] = C;
        qc.pad = (qc.pad + 1 == Nw) ? 0 : qc.pad + 1;
#else
        a.st_ring[(o * B + b) * (size_t)a.ring_n + (qc.cnt % Nw)] = C;
#endif
      }
      const double d = C - qc.sh;
      qc.S1 = qc.S1 + d;
      qc.S2 = qc.S2 + d * d;
      qc.cnt += 1;
      const double2 ms = posterior(qc.sh, qc.S1, qc.S2, n + 1, cp.prec0, cp.pm0);
      const double dm = ms.x - ref;
      const float2 vn = (fabs(dm) < 1e30 && ms.y < 1e30) ? make_float2((float)dm, (float)ms.y) : make_float2(0.0f, kInfF);
      s_f2[2 * ((b >> 1) * TPB + tid) + (b & 1)] = vn;
#if ZS_SMAX_UB
      smax_ub = fmaxf(smax_ub, vn.y);
      if ((t & 63) == 63) {                                 // tighten: the exact maximum again
        float m = 0.0f;
        for (int k = 0; k < 2 * npairs2; ++k) m = fmaxf(m, s_f2[2 * ((k >> 1) * TPB + tid) + (k & 1)].y);
        smax_ub = m;
      }
#endif
    }
  }
  if (active && qc_b >= 0) rec(qc_b) = qc;
  if constexpr (SREC)                                       // write the phase's records back
    if (active)
      for (int b = 0; b < B; ++b)
        if ((ts_set >> b) & 1u) st_g[b] = s_rec[(size_t)b * TPB + tid];
  if (active) {
    a.tot_cost[o] = totC;
    a.tot_energy[o] = totE;
    a.tot_time[o] = totT;
    a.digest[o] = dig;
    a.n_stop[o] = nstop;
    a.final_arm[o] = last_b;
  }
  // counters: the method's events (as replay_kernel), then the work: [9] fp64 transforms
  // (fallback draws), [10] Philox blocks, [11] fp32 pairs, [12] certified, [13] fallbacks
  // (phase A's Thompson draws, carried in n_sampled, are full fp64 draws: counted in [9], [10])
  const uint32_t nB = active ? (uint32_t)(R - (EARLY ? a.carry[o].t0 : a.t_split)) : 0u;   // draws here
  uint32_t n_cert = nB - n_fall;
  // phase A's draws: certified (fp32 pairs, one block per quad) or full fp64 (its fallbacks and,
  // without the certified draw, all of them)
  uint32_t n_sampled = nB, n_prune = 0, n_forced = 0, n_recomp = nB, n_full = n_fall, n_tried = nB;
  if (active) {
    const Carry c = a.carry[o];
    n_full += c.n_sampled - c.n_cert;
    n_tried += c.n_cert + c.n_fall;
    n_cert += c.n_cert; n_fall += c.n_fall;
    n_sampled += c.n_sampled; n_prune = c.n_prune; n_forced = c.n_forced; n_recomp += c.n_recomp;
  }
  const unsigned long long fp32_pairs = (unsigned long long)n_tried * 2 * __popc(quads);
  const unsigned long long fall_pairs = (unsigned long long)n_full * __popc(ts_pairs);
  const unsigned long long blocks_fp32 = (unsigned long long)n_tried * __popc(quads);
  const unsigned long long blocks_fall = (unsigned long long)n_full * __popc(quads);
  const unsigned long long pairs_all = (unsigned long long)n_sampled * __popc(ts_pairs);
  const unsigned long long blocks_all = (unsigned long long)n_sampled * __popc(quads);
  unsigned long long ctr[kCounters] = {
      active ? (unsigned long long)R : 0ull, n_sampled, pairs_all,
      (unsigned long long)n_sampled * __popc(ts_set),
      (unsigned long long)nstop, n_prune, n_forced, n_recomp, blocks_all,
      active ? fall_pairs : 0ull, active ? blocks_fp32 + blocks_fall : 0ull, active ? fp32_pairs : 0ull,
      active ? n_cert : 0ull, active ? n_fall : 0ull};
#pragma unroll
  for (int q = 0; q < kCounters; ++q) {
    unsigned long long v = ctr[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((tid & 31) == 0 && v) atomicAdd(a.counters + q, v);
  }
}

// the kernels: the windowed variant asks for six 128-thread blocks per SM (80 registers, no
// spills: one wave of CFG4's 10^5 trials); the others keep the compiler's choice (96)
template <bool LOG, bool RK, bool SREC, bool WIN, bool EARLY = false>
__global__ void ZS_TH_BOUNDS thompson_kernel(ReplayArgs a) {
  if constexpr (!WIN) thompson_body<LOG, RK, SREC, false, EARLY>(a);
}
template <bool LOG, bool RK, bool SREC, bool EARLY = false>
__global__ void __launch_bounds__(128, ZS_WIN_MIN_BLOCKS) thompson_win_kernel(ReplayArgs a) {
  thompson_body<LOG, RK, SREC, true, EARLY>(a);
}

}  // namespace zs
