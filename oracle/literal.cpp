// literal.cpp -- TEST INFRASTRUCTURE ONLY (see literal.h).
//
// A second CPU replay of Zeus's optimiser, written to be read against the paper line by
// line and nothing else.  It does NOT follow the numerics contract: it uses
// the C++ standard library's normals and integers (std::mt19937_64, std::normal_distribution,
// std::uniform_int_distribution), and it computes Alg. 2 exactly as printed -- the history
// C_b is kept as a list and Var, Sum, σ̂² and μ̂ are recomputed from it on every Observe.
// Its only job is to show, statistically, that the contract oracle (oracle.cpp, whose
// sampler and Observe arithmetic are engineered for bit parity with the kernels) replays
// the same method: tests/test_literal_equivalence.py compares the two replays'
// distributions (per-trial totals, final arms, per-recurrence cost curves).
//
// The readings of the paper's silent points (R-Q1 .. R-Q27) are the same as
// the contract oracle's, because they define the method being compared; everything else
// (RNG, operation order, state representation, code) is independent.  This file shares no
// code with oracle.cpp or with the CUDA path.
//
// Passages (PAPER.md lines):
//   Eq. 7 (power limit per batch size)
//   JIT profiling epoch
//   Alg. 1 Predict (Gaussian Thompson sampling)
//   Alg. 2 Observe (conjugate update)            P:L494-506; flat prior P:L529
//   learned cost variance
//   early stopping at β·min_t C_t
//   Alg. 3 (pruning, then Thompson sampling)
//   window of the N most recent observations
//   trace replay (recorded runs, K seeds)

#include "literal.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <thread>
#include <vector>

namespace {

const double kInf = std::numeric_limits<double>::infinity();

// Per-epoch cost of every (b, p) and the quantities Eq. 7 picks.
struct Step1 {
  int B, P;
  std::vector<int> pstar;
  std::vector<double> c1, t1, e1;   // per-epoch cost, time, energy at p*(b)
  std::vector<double> cP, tP, eP;   // the JIT profiling epoch
};

Step1 eq7(const literal_trace &tr, double eta) {
  Step1 s;
  s.B = tr.num_batch_sizes;
  s.P = tr.num_power_limits;
  const double MP = tr.max_power_w;
  for (int b = 0; b < s.B; ++b) {
    int best_p = -1;
    double best_c = kInf;
    double sum_t = 0, sum_e = 0;
    for (int p = 0; p < s.P; ++p) {
      const double A = tr.avg_power_w[b * s.P + p];
      const double Th = tr.throughput_eps[b * s.P + p];
      // EpochCost(b; p) = (η·AvgPower(b,p) + (1−η)·MAXPOWER) / Throughput(b,p)
      const double cost = (eta * A + (1 - eta) * MP) / Th;
      if (cost < best_c) { best_c = cost; best_p = p; }
      // the profiling epoch spends 1/P of an epoch at each power limit
      sum_t += (1.0 / s.P) / Th;
      sum_e += (1.0 / s.P) * A / Th;
    }
    const double A = tr.avg_power_w[b * s.P + best_p];
    const double Th = tr.throughput_eps[b * s.P + best_p];
    s.pstar.push_back(best_p);
    s.c1.push_back(best_c);
    s.t1.push_back(1.0 / Th);
    s.e1.push_back(A / Th);
    s.tP.push_back(sum_t);
    s.eP.push_back(sum_e);
    s.cP.push_back(eta * sum_e + (1 - eta) * MP * sum_t);
  }
  return s;
}

// Alg. 2, literally: C_b ← C_b ∪ {C}; σ̃² ← Var(C_b); σ̂² ← (1/σ̂0² + |C_b|/σ̃²)⁻¹;
// μ̂ ← σ̂²(μ̂0/σ̂0² + Sum(C_b)/σ̃²).  With the flat prior σ̂0² = +∞ the IEEE quotients
// 1/σ̂0² and μ̂0/σ̂0² are exactly 0.  The window keeps the N most recent costs.
struct Belief {
  std::vector<double> C;   // the history C_b (at most N entries when windowed)
  double mu = 0, var = 0;
  bool profiled = false;
};

void observe(Belief &a, double cost, int window, double mu0, double var0) {
  a.C.push_back(cost);
  if (window > 0 && (int)a.C.size() > window) a.C.erase(a.C.begin());
  const double n = (double)a.C.size();
  if (a.C.size() < 2) return;                       // no variance from one cost (R-Q6)
  double sum = 0;
  for (double c : a.C) sum += c;
  const double mean = sum / n;
  double ss = 0;
  for (double c : a.C) ss += (c - mean) * (c - mean);
  double s2 = ss / (n - 1);                          // Var with the n−1 divisor (R-Q6)
  const double floor = 1e-12 * (1 + mean * mean);    // zero-variance floor (R-Q7)
  if (!(s2 >= floor)) s2 = floor;
  a.var = 1.0 / (1.0 / var0 + n / s2);
  a.mu = a.var * (mu0 / var0 + sum / s2);
}

struct TrialOut {
  double cost = 0, energy = 0, time = 0;
  int stops = 0, final_arm = -1;
};

// One trial of Alg. 3 over R recurrences on the recorded traces.
void run_trial(const literal_trace &tr, const literal_cell &cell, const Step1 &T, int R,
               int64_t trial, double sigma_scale, TrialOut &out, double *cost_log,
               int32_t *arm_log) {
  const int B = T.B, S = tr.num_slices, K = tr.replicas;
  std::seed_seq sq{(uint32_t)cell.seed, (uint32_t)(cell.seed >> 32), (uint32_t)trial,
                   (uint32_t)((uint64_t)trial >> 32), 0x4c495431u};
  std::mt19937_64 gen(sq);
  std::normal_distribution<double> normal(0.0, 1.0);
  std::uniform_int_distribution<int> pick_seed(0, K - 1);

  std::vector<Belief> arm(B);
  double min_cost = kInf;                 // min_t C_t over runs that reached the target (R-Q5)

  // Alg. 3, "repeat 2 times": explore b0, then b < b0 downwards, then b > b0 upwards, each
  // walk until a convergence failure; keep the converged sizes; b0 ← the cheapest (R-Q10).
  std::vector<int> cand;                  // the round's candidate batch sizes (ascending)
  for (int b = 0; b < B; ++b) cand.push_back(b);
  int b0 = tr.default_bs_index;
  int round = 0;                          // 0, 1: pruning rounds; 2: Thompson sampling
  std::vector<int> plan;                  // this round's walk: b0, then downwards, then upwards
  size_t at = 0;                          // next entry of the plan
  size_t up_from = 0;                     // where the upward part of the plan starts
  std::vector<int> converged_now;         // sizes that converged in this round
  double round_best = kInf;
  int round_best_b = -1;
  auto make_plan = [&]() {
    plan.clear();
    plan.push_back(b0);
    for (int i = (int)cand.size() - 1; i >= 0; --i) if (cand[i] < b0) plan.push_back(cand[i]);
    up_from = plan.size();
    for (int b : cand) if (b > b0) plan.push_back(b);
    at = 0;
    converged_now.clear();
    round_best = kInf;
    round_best_b = -1;
  };
  make_plan();
  std::vector<int> ts_set;                // 𝓑 for Thompson sampling

  for (int t = 0; t < R; ++t) {
    const int s = (int)((int64_t)t * S / R);   // the trace slice of recurrence t (R-Q19)
    // ---- which batch size runs now
    int b;
    if (round < 2) {
      b = plan[at];
    } else {
      b = -1;
      for (int a : ts_set)                      // an arm needs two costs for a variance (R-Q6)
        if (arm[a].C.size() < 2) { b = a; break; }
      if (b < 0) {
        // Alg. 1: for each b ∈ 𝓑 sample θ̂_b ~ N(μ̂_b, σ̂_b²); b* ← argmin_b θ̂_b
        double best = kInf;
        for (int a : ts_set) {
          const double theta = arm[a].mu + sigma_scale * std::sqrt(arm[a].var) * normal(gen);
          if (theta < best) { best = theta; b = a; }
        }
      }
    }
    // ---- run it: one recorded run of b drawn uniformly from the K seeds (R-Q15)
    const int k = pick_seed(gen);
    const int E = tr.epochs_to_target[((int64_t)s * B + b) * K + k];
    const bool reaches = E > 0;
    const int epochs = reaches ? E : tr.max_epochs;   // a run that never converges (R-Q16)
    // the first run of b in this trial pays the JIT profiling epoch as its first epoch (R-Q13/14)
    const bool profiling = tr.charge_profiling && !arm[b].profiled;
    arm[b].profiled = true;
    const double first_c = profiling ? T.cP[b] : T.c1[b];
    const double first_t = profiling ? T.tP[b] : T.t1[b];
    const double first_e = profiling ? T.eP[b] : T.e1[b];
    double cost = first_c + (epochs - 1) * T.c1[b];
    double time = first_t + (epochs - 1) * T.t1[b];
    double energy = first_e + (epochs - 1) * T.e1[b];
    // early stopping: the job is stopped when its cost is to exceed β·min_t C_t and
    // charged that much, time and energy taken at the same point of the run (R-Q1)
    const double threshold = cell.beta * min_cost;
    bool stopped = false;
    if (cost > threshold) {
      stopped = true;
      cost = threshold;
      if (threshold <= first_c) {
        const double frac = threshold / first_c;
        time = frac * first_t;
        energy = frac * first_e;
      } else {
        const double more = (threshold - first_c) / T.c1[b];   // epochs after the first
        time = first_t + more * T.t1[b];
        energy = first_e + more * T.e1[b];
      }
    }
    const bool converged = reaches && !stopped;
    if (converged) min_cost = std::min(min_cost, cost);
    // Observe: every run is observed at its charged cost (R-Q3, R-Q27)
    observe(arm[b], cost, cell.window, cell.prior_mean, cell.prior_var);

    out.cost += cost;
    out.energy += energy;
    out.time += time;
    out.stops += stopped;
    out.final_arm = b;
    if (cost_log) cost_log[t] = cost;
    if (arm_log) arm_log[t] = b;

    // ---- Alg. 3 bookkeeping
    if (round < 2) {
      if (converged) {
        converged_now.push_back(b);
        if (round == 0 && (cost < round_best || (cost == round_best && b < round_best_b))) {
          round_best = cost;                          // ties to the smaller size (R-Q17)
          round_best_b = b;
        }
      }
      ++at;
      // a failure ends the downward walk (jump to the upward part) or the upward walk (end)
      if (!converged && at > 1 && at <= up_from) at = up_from;
      else if (!converged && at > up_from) at = plan.size();
      const bool done = at >= plan.size();
      if (done) {
        std::vector<int> kept = converged_now;
        std::sort(kept.begin(), kept.end());
        if (kept.empty()) kept.push_back(b0);            // R-Q23
        if (round == 0) {
          cand = kept;                                    // 𝓑 ← {b: b converged}
          if (round_best_b >= 0) b0 = round_best_b;       // b0 ← b with smallest cost observed
          round = 1;
          make_plan();
        } else {
          ts_set = kept;
          round = 2;
        }
      }
    }
  }
}

}  // namespace

extern "C" {

int literal_replay(const literal_trace *tr, const literal_cell *cell, int32_t R, int64_t trial0,
                   int64_t n, int32_t threads, double sigma_scale, literal_out *out) {
  if (!tr || !cell || !out || R < 0 || n < 0) return 1;
  const Step1 T = eq7(*tr, cell->eta);
  if (threads < 1) threads = 1;
  auto work = [&](int w) {
    for (int64_t j = w; j < n; j += threads) {
      TrialOut o;
      run_trial(*tr, *cell, T, R, trial0 + j, sigma_scale, o,
                out->cost_log ? out->cost_log + j * R : nullptr,
                out->arm_log ? out->arm_log + j * R : nullptr);
      if (out->tot_cost) out->tot_cost[j] = o.cost;
      if (out->tot_energy) out->tot_energy[j] = o.energy;
      if (out->tot_time) out->tot_time[j] = o.time;
      if (out->n_stop) out->n_stop[j] = o.stops;
      if (out->final_arm) out->final_arm[j] = o.final_arm;
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < threads; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto &th : pool) th.join();
  return 0;
}

int literal_posterior(const double *xs, int32_t n, int32_t window, double prior_mean,
                      double prior_var, double *mu, double *var) {
  Belief a;
  for (int32_t i = 0; i < n; ++i) observe(a, xs[i], window, prior_mean, prior_var);
  if (a.C.size() < 2) return 1;
  *mu = a.mu;
  *var = a.var;
  return 0;
}

}  // extern "C"
