/*
 * literal.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The literal replay: Zeus's optimiser (Alg. 1-3, Eq. 7) written as the paper prints
 * it, with the C++ standard library's random numbers and Alg. 2 recomputed from the cost
 * history on every Observe.  It is NOT bit-comparable with anything; tests compare its
 * distributions with the contract oracle's (tests/test_literal_equivalence.py).  Only tests/
 * may load it.  It shares no code with oracle.cpp or with the CUDA path.
 */
#ifndef ZEUS_LITERAL_H
#define ZEUS_LITERAL_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {                   /* the same fields and meaning as oracle_trace (oracle.h) */
  int32_t num_batch_sizes;
  const int32_t *batch_sizes;
  int32_t default_bs_index;
  int32_t num_power_limits;
  const double *power_limits_w;
  double max_power_w;
  int32_t max_epochs;
  int32_t charge_profiling;
  const double *avg_power_w;       /* [B][P] */
  const double *throughput_eps;    /* [B][P] epochs/s */
  int32_t num_slices;
  int32_t replicas;
  const int32_t *epochs_to_target; /* [S][B][K] */
} literal_trace;

typedef struct {
  double eta, beta;                /* η, β (β may be +inf) */
  int32_t window;                  /* N, 0 = unbounded */
  double prior_mean, prior_var;    /* μ̂0, σ̂0² (+inf = flat prior) */
  uint64_t seed;                   /* seeds std::mt19937_64 together with the trial index */
} literal_cell;

typedef struct {                   /* any pointer may be NULL */
  double *tot_cost, *tot_energy, *tot_time;   /* [n] */
  int32_t *n_stop, *final_arm;                /* [n] */
  double *cost_log;                           /* [n][R] charged cost of each recurrence */
  int32_t *arm_log;                           /* [n][R] batch-size index of each recurrence */
} literal_out;

/* Replays trials trial0 .. trial0+n-1.  sigma_scale multiplies σ̂_b in Alg. 1's draw: 1 is
 * the method; any other value is a deliberately wrong sampler, used by the tests to show that
 * the statistical comparison has the power to see a change of the draw.  Returns 0, or 1 on
 * a bad argument (inputs are assumed valid: the contract oracle validates the same arrays). */
int literal_replay(const literal_trace *tr, const literal_cell *cell, int32_t recurrences,
                   int64_t trial0, int64_t n, int32_t threads, double sigma_scale,
                   literal_out *out);

/* Alg. 2 over the costs xs[0..n) with window N: the posterior (μ̂, σ̂²) exactly as printed
 * (fp64).  Returns 1 when fewer than two costs are in the window. */
int literal_posterior(const double *xs, int32_t n, int32_t window, double prior_mean,
                      double prior_var, double *mu, double *var);

#ifdef __cplusplus
}
#endif
#endif
