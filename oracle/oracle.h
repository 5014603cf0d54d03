/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-trial-at-a-time CPU replay of Zeus's optimiser
 * (You, Chung, Chowdhury, arXiv 2208.06102).  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header,
 * constant table or helper with the CUDA path (paper_2208_06102_b200/csrc)
 * and neither side includes the other.
 *
 * Citations: "P:Lnnn" = line nnn of the paper's LaTeX,
 * "S:Lnnn" = line of SPEC.md; readings R-x are listed in DESIGN.md §3.
 *
 * Every function returns 0 on success, 1 on invalid input (message in the
 * caller's buffer where one is taken).
 */
#ifndef ZEUS_ORACLE_H
#define ZEUS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* The recurring job ("a set of feasible batch sizes B and power
 * limits P") together with its two traces (§6.1). */
typedef struct {
  int32_t num_batch_sizes;        /* B = |𝓑| */
  const int32_t *batch_sizes;     /* [B], strictly increasing */
  int32_t default_bs_index;       /* b0 (Alg. 3 input) */
  int32_t num_power_limits;       /* P = |𝓟| */
  const double *power_limits_w;   /* [P], strictly increasing */
  double max_power_w;             /* MAXPOWER (Eq. 2) */
  int32_t max_epochs;             /* cap for runs that never converge */
  int32_t charge_profiling;       /* 1: first run of an arm pays the JIT epoch */
  const double *avg_power_w;      /* [B][P] AvgPower(b,p)  (power trace) */
  const double *throughput_eps;   /* [B][P] Throughput(b,p) in epochs/s */
  int32_t num_slices;             /* S (drift slices); 1 = stationary */
  int32_t replicas;               /* K seeds per (b) */
  const int32_t *epochs_to_target;/* [S][B][K]; <= 0: never reaches target */
} oracle_trace;

typedef struct {
  double eta;          /* η in [0,1] */
  double beta;         /* β > 1 or +inf */
  int32_t window;      /* N >= 2, 0 = unbounded */
  double prior_mean;   /* μ̂0 (Alg. 2) */
  double prior_var;    /* σ̂0², +inf = flat prior */
  uint64_t seed;       /* Philox key */
  int32_t policy;      /* 0 Zeus (Alg. 3 + Alg. 1/2), 1 Default (b0, max p), 2 Grid Search
                          with pruning (§6.1) */
  int32_t ablation;    /* Zeus ablations: bit0 no pruning, bit1 no JIT profiling;
                          variant readings of P:L559 (sequential recurrences only):
                          bit2 retry after an early stop within the recurrence (R-Q4v),
                          bit3 early stop at the epoch boundary (R-Q1v),
                          bit4 best over the last N = window recurrences (R-Q5v) */
  const double *arrivals; /* NULL: sequential recurrences; else [R] non-decreasing submit times
                             (s): concurrent submissions (§4.4), Zeus only */
} oracle_cell;

typedef struct {       /* step-1 tables; any pointer may be NULL */
  int32_t *pstar;                       /* [B] index into 𝓟 */
  double *c1, *t1, *e1;                 /* [B] per-epoch cost/time/energy at p* */
  double *c_prof, *t_prof, *e_prof;     /* [B] the JIT profiling epoch */
  double *ebar;                         /* [S][B] mean epochs of converged replicas */
  double *opt;                          /* [S] min_b Ebar*c1 */
  int32_t *opt_arm;                     /* [S] */
  double *regret;                       /* [S][B] pseudo-regret of choosing b in slice s */
} oracle_tables;

typedef struct {       /* replay outputs; any pointer may be NULL */
  double *tot_cost, *tot_energy, *tot_time;   /* [n] */
  uint64_t *digest;                           /* [n] FNV-1a over (b,p,flags) per recurrence */
  int32_t *n_stop;                            /* [n] */
  int32_t *final_arm;                         /* [n] */
  uint32_t *log;                              /* [n][R] arm | p<<8 | flags<<16 */
  double *cost_log, *energy_log, *time_log;   /* [n][R] */
  double *curves;                             /* [R][7] sums over the given trials */
  int64_t *counters;                          /* [9] instrumentation (see oracle.cpp) */
} oracle_out;

int oracle_validate(const oracle_trace *tr, const oracle_cell *cell, char *msg, int32_t msglen);
int oracle_step1(const oracle_trace *tr, const oracle_cell *cell, oracle_tables *out);
int oracle_replay(const oracle_trace *tr, const oracle_cell *cell, int32_t recurrences,
                  const int64_t *trials, int64_t n, int32_t threads, oracle_out *out);

/* Pareto front of slice s's (TTA, ETA) grid: mask [B][P] (1 = on the front) */
int oracle_pareto(const oracle_trace *tr, int32_t s, uint8_t *mask);

/* primitives, exposed for the pins */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double oracle_zlog(double x);
double oracle_zlog_fdlibm(double x);
void oracle_zsincospi(uint64_t m52, double *s, double *c);
void oracle_uniforms(uint32_t a, uint32_t b, double *u1, double *v);
void oracle_normal_pair(uint64_t seed, int64_t trial, int32_t t, int32_t k, double *z0, double *z1);
uint32_t oracle_replica(uint64_t seed, int64_t trial, int32_t t, int32_t K);
/* Alg. 1 Predict over the arms in bitmask `set` with posteriors (mu, sigma)[B]: the arm the
 * replay of (seed, trial) picks at recurrence t; -1 for an empty set */
int32_t oracle_thompson_argmin(uint64_t seed, int64_t trial, int32_t t, int32_t B, uint32_t set,
                               const double *mu, const double *sigma);
int oracle_posterior(const double *xs, int32_t n, int32_t window, double prior_mean,
                     double prior_var, double *mu, double *sigma, double *s2, double *var);
int32_t oracle_hardware_threads(void);
/* batches of the primitives (large-sample pins) */
void oracle_zlog_batch(const double *x, double *y, int64_t n);
void oracle_zsincospi_batch(const uint64_t *m, double *s, double *c, int64_t n);
void oracle_normal_batch(uint64_t seed, int64_t trial0, int64_t n, int32_t t, int32_t k,
                         int32_t threads, double *out);

#ifdef __cplusplus
}
#endif
#endif
