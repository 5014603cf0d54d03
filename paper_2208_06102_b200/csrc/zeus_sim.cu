// zeus_sim.cu -- host side of the C ABI declared in include/zeus_sim.h.
//
// Validation (every violated invariant is reported), device
// allocation, H2D staging of the two traces (§6.1), launches of
// the step-1 / replay / curve-reduction kernels on the caller's stream, and
// D2H of the results.  There is no CPU compute path: without a usable CUDA
// device every call that would launch work fails with ZEUS_E_CUDA.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/zeus_sim.h"
#include "kernels.cuh"
#include "thompson.cuh"

namespace {

thread_local std::string g_create_error;

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t n) {
    if (p && n == bytes) return cudaSuccess;   // same size: keep the allocation (and its address)
    if (p) { cudaFree(p); p = nullptr; }
    bytes = n;
    if (n == 0) return cudaSuccess;
    return cudaMalloc(&p, n);
  }
  template <class T> T *as() const { return static_cast<T *>(p); }
};

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

// NVTX range around each C-ABI call (visible in nsys / ncu timelines; the header-only
// NVTX3 API is a no-op unless a tool injects itself)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct zeus_sim {
  // job
  int B = 0, P = 0, b0 = 0, max_epochs = 0, charge_profiling = 0;
  std::vector<int32_t> batch_sizes;
  std::vector<double> power_limits;
  double MP = 0.0;
  // cells / run
  std::vector<zeus_cell> cells;
  std::vector<zs::CellParam> cpar;
  int R = 0, log_mode = 0, layout = 0, device = 0, wmax = 0, draw = 0, sms = 148;
  int64_t shard_total = 0, max_shard = 0;
  // trace
  int S = 0, K = 0, reg_stride = 0, opt_stride = 0;
  bool loaded = false, ran = false, any_zeus = false, any_baseline = false, any_ablation = false,
       any_conc = false, any_variant = false;
  int best_n = 0;                    // ring of the windowed best (ZEUS_VARIANT_WINDOWED_BEST)
  // CUDA graph of one run's launches (zeus_run_opts.graph), captured on cap_stream
  int use_graph = 0, graph_launches = 0;
  cudaStream_t cap_stream = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  std::vector<uintptr_t> launch_signature() const {
    return {(uintptr_t)d_A.p, (uintptr_t)d_Th.p, (uintptr_t)d_pool.p, (uintptr_t)d_arms.p,
            (uintptr_t)d_regret.p, (uintptr_t)d_opt.p, (uintptr_t)d_optarm.p, (uintptr_t)d_ebar.p,
            (uintptr_t)S, (uintptr_t)K, (uintptr_t)reg_stride, (uintptr_t)opt_stride, (uintptr_t)tpb,
            (uintptr_t)smem_bytes, (uintptr_t)tab_bytes, (uintptr_t)group_w, (uintptr_t)loaded,
            // the curves' fixed-point scale follows the traces (load_profile) and is a kernel
            // argument of the captured launches
            (uintptr_t)(intptr_t)curve_bits};
  }
  void drop_graph() {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (graph) cudaGraphDestroy(graph);
    graph_exec = nullptr;
    graph = nullptr;
  }
  int nslot = 1, tpb = 128, smem_bytes = 0, tab_bytes = 0, launches = 0, nwin = 1, group_w = 0;
  // The handle's stream: where load_profile and results enqueue their work -- the stream of the
  // last zeus_sim_run, or `own` (an internal non-blocking stream) before the first run.  No call
  // launches on the legacy stream or synchronises the device (include/zeus_sim.h, "Async").
  cudaStream_t stream = nullptr, own = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  cudaEvent_t ev_loaded = nullptr;   // the last load's copies, on the stream they were enqueued on
  cudaEvent_t ev_staged = nullptr;   // the pinned staging buffer is free again
  bool staged_pending = false;
  void *h_stage = nullptr;           // pinned host copy of the traces (the caller's arrays are read
  size_t h_stage_bytes = 0;          // before load_profile returns; the DMA reads this copy)
  bool tables_valid = false;         // step-1 tables of the loaded traces are on the device
  bool pareto_valid = false;         // the Pareto masks of the loaded traces are on the device
  std::string err;
  // device memory
  DevBuf d_A, d_Th, d_pool, d_cells, d_arms, d_regret, d_opt, d_optarm;
  int curve_bits = 0;                // F of the curves' fixed point (curve_accumulate)
  DevBuf d_hist;                     // counted runs per (cell, t, slot, class, b, replica)
  int nhslot = 1;
  DevBuf d_slots, d_fixed, d_curves, d_tot_cost, d_tot_energy, d_tot_time, d_digest, d_nstop, d_final,
      d_log, d_counters, d_st, d_st_ring, d_carry, d_perm, d_bucket, d_ebar, d_logtab, d_pareto,
      d_arrivals, d_best_ring;
  ~zeus_sim() {
    drop_graph();
    if (own) { cudaStreamSynchronize(own); cudaStreamDestroy(own); }
    if (h_stage) cudaFreeHost(h_stage);
    if (ev_loaded) cudaEventDestroy(ev_loaded);
    if (ev_staged) cudaEventDestroy(ev_staged);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (ev2) cudaEventDestroy(ev2);
    if (ev3) cudaEventDestroy(ev3);
  }
};

namespace {

struct Errors {
  std::string s;
  zeus_status code = ZEUS_OK;
  void add(zeus_status c, const std::string &m) {
    if (!s.empty()) s += "; ";
    s += m;
    // the most specific code wins: INVALID over UNSUPPORTED over NO_CONVERGENT_ARM
    if (code == ZEUS_OK || c == ZEUS_E_INVALID) code = c;
  }
};

zeus_status fail(zeus_sim *sim, zeus_status c, const std::string &m) {
  if (sim) sim->err = m; else g_create_error = m;
  return c;
}

zeus_status cuda_fail(zeus_sim *sim, cudaError_t e, const char *where) {
  return fail(sim, ZEUS_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define ZS_CUDA(sim, call)                                 \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_fail(sim, e_, #call); \
  } while (0)

void check_job(const zeus_job *job, Errors &E) {
  if (!job) { E.add(ZEUS_E_INVALID, "job is NULL"); return; }
  if (job->struct_size != sizeof(zeus_job)) E.add(ZEUS_E_INVALID, "zeus_job.struct_size mismatch (ABI)");
  const int B = job->num_batch_sizes, P = job->num_power_limits;
  if (B < 1) E.add(ZEUS_E_INVALID, "no batch sizes");
  if (B > ZEUS_MAX_BATCH_SIZES) E.add(ZEUS_E_UNSUPPORTED, "more than 32 batch sizes");
  if (P < 1) E.add(ZEUS_E_INVALID, "no power limits");
  if (P > ZEUS_MAX_POWER_LIMITS) E.add(ZEUS_E_UNSUPPORTED, "more than 64 power limits");
  if (B >= 1 && !job->batch_sizes) E.add(ZEUS_E_INVALID, "batch_sizes is NULL");
  if (P >= 1 && !job->power_limits_w) E.add(ZEUS_E_INVALID, "power_limits_w is NULL");
  if (B >= 1 && job->batch_sizes) {
    for (int b = 0; b < B; ++b)
      if (job->batch_sizes[b] <= 0) { E.add(ZEUS_E_INVALID, "batch size not positive"); break; }
    for (int b = 1; b < B; ++b)
      if (job->batch_sizes[b] <= job->batch_sizes[b - 1]) { E.add(ZEUS_E_INVALID, "batch sizes not strictly increasing"); break; }
  }
  if (job->default_bs_index < 0 || job->default_bs_index >= B)
    E.add(ZEUS_E_INVALID, "default batch size index out of range");
  double pmax = 0.0;
  if (P >= 1 && job->power_limits_w) {
    for (int p = 0; p < P; ++p)
      if (!(job->power_limits_w[p] > 0.0)) { E.add(ZEUS_E_INVALID, "power limit not positive"); break; }
    for (int p = 1; p < P; ++p)
      if (!(job->power_limits_w[p] > job->power_limits_w[p - 1])) { E.add(ZEUS_E_INVALID, "power limits not strictly increasing"); break; }
    pmax = job->power_limits_w[P - 1];
  }
  if (!(job->max_power_w >= pmax) || !std::isfinite(job->max_power_w))
    E.add(ZEUS_E_INVALID, "max power below the largest power limit");
  if (job->max_epochs < 1) E.add(ZEUS_E_INVALID, "max_epochs < 1");
  if (job->charge_profiling != 0 && job->charge_profiling != 1) E.add(ZEUS_E_INVALID, "charge_profiling must be 0 or 1");
}

void check_cells(const zeus_cell *cells, int n, Errors &E) {
  if (n < 1) { E.add(ZEUS_E_INVALID, "no cells"); return; }
  if (!cells) { E.add(ZEUS_E_INVALID, "cells is NULL"); return; }
  for (int i = 0; i < n; ++i) {
    const zeus_cell &c = cells[i];
    const std::string at = " (cell " + std::to_string(i) + ")";
    if (!(c.eta >= 0.0 && c.eta <= 1.0)) E.add(ZEUS_E_INVALID, "eta out of [0,1]" + at);
    if (!(c.beta > 1.0)) E.add(ZEUS_E_INVALID, "beta must be > 1" + at);
    if (c.window == 1 || c.window < 0) E.add(ZEUS_E_INVALID, "window must be 0 (unbounded) or >= 2" + at);
    if (!(c.prior_var > 0.0)) E.add(ZEUS_E_INVALID, "prior variance must be > 0" + at);
    if (!std::isfinite(c.prior_mean)) E.add(ZEUS_E_INVALID, "prior mean not finite" + at);
    if (c.trials < 0) E.add(ZEUS_E_INVALID, "trials < 0" + at);
    if (c.policy < ZEUS_POLICY_ZEUS || c.policy > ZEUS_POLICY_GRID_SEARCH)
      E.add(ZEUS_E_INVALID, "policy must be ZEUS_POLICY_ZEUS, _DEFAULT or _GRID_SEARCH" + at);
    const int32_t kVariants = ZEUS_VARIANT_RETRY | ZEUS_VARIANT_EPOCH_STOP | ZEUS_VARIANT_WINDOWED_BEST;
    if (c.ablation < 0 || c.ablation > (ZEUS_ABLATE_PRUNING | ZEUS_ABLATE_JIT | kVariants))
      E.add(ZEUS_E_INVALID, "ablation must be a subset of the ZEUS_ABLATE_* and ZEUS_VARIANT_* bits" + at);
    if (c.ablation != 0 && c.policy != ZEUS_POLICY_ZEUS)
      E.add(ZEUS_E_INVALID, "ablation bits apply to the Zeus policy only" + at);
    if ((c.ablation & ZEUS_VARIANT_WINDOWED_BEST) && c.window < 2)
      E.add(ZEUS_E_INVALID, "ZEUS_VARIANT_WINDOWED_BEST needs window >= 2" + at);
    if (c.arrivals && (c.ablation & kVariants))
      E.add(ZEUS_E_INVALID, "the ZEUS_VARIANT_* readings need sequential recurrences (no arrivals)" + at);
    if (c.arrivals && (c.policy != ZEUS_POLICY_ZEUS || c.ablation != 0))
      E.add(ZEUS_E_UNSUPPORTED, "arrivals are supported for the Zeus policy without ablations" + at);
  }
}

// replay_kernel<WINDOWED, LOG, PHASE, ABLATIONS, RK> by runtime flags
typedef void (*ReplayFn)(zs::ReplayArgs);
template <bool W, bool L, bool A, bool RK = false>
constexpr ReplayFn pick(int phase) {
  return phase == 0 ? zs::replay_kernel<W, L, 0, A, RK> : phase == 1 ? zs::replay_kernel<W, L, 1, A, RK>
                                                                     : zs::replay_kernel<W, L, 2, A, RK>;
}
// rk: a one-cell launch whose round keys travel in the parameters (no ablation path)
ReplayFn replay_fn(bool windowed, bool log, int phase, bool abl = false, bool rk = false) {
  if (rk && !abl) {
    if (windowed) return log ? pick<true, true, false, true>(phase) : pick<true, false, false, true>(phase);
    return log ? pick<false, true, false, true>(phase) : pick<false, false, false, true>(phase);
  }
  if (abl) {
    if (windowed) return log ? pick<true, true, true>(phase) : pick<true, false, true>(phase);
    return log ? pick<false, true, true>(phase) : pick<false, false, true>(phase);
  }
  if (windowed) return log ? pick<true, true, false>(phase) : pick<true, false, false>(phase);
  return log ? pick<false, true, false>(phase) : pick<false, false, false>(phase);
}

#ifndef ZS_EARLY_SPLIT
#define ZS_EARLY_SPLIT 1        // phase A stops each lane at its first pure Thompson decision
#endif
#ifndef ZS_WIN_THOMPSON
#define ZS_WIN_THOMPSON 1
#endif
// thompson_kernel<LOG, RK, SREC, WIN> by runtime flags
typedef void (*ThompsonFn)(zs::ReplayArgs);
ThompsonFn thompson_fn(bool log, bool rk, bool srec, bool win, bool early = false) {
  if (early && !srec) {               // the early split (phase A stopped each lane at its t0)
    if (win) {
      if (rk) return log ? zs::thompson_win_kernel<true, true, false, true> : zs::thompson_win_kernel<false, true, false, true>;
      return log ? zs::thompson_win_kernel<true, false, false, true> : zs::thompson_win_kernel<false, false, false, true>;
    }
    if (rk) return log ? zs::thompson_kernel<true, true, false, false, true> : zs::thompson_kernel<false, true, false, false, true>;
    return log ? zs::thompson_kernel<true, false, false, false, true> : zs::thompson_kernel<false, false, false, false, true>;
  }
  if (win) {
    if (srec) {
      if (rk) return log ? zs::thompson_win_kernel<true, true, true> : zs::thompson_win_kernel<false, true, true>;
      return log ? zs::thompson_win_kernel<true, false, true> : zs::thompson_win_kernel<false, false, true>;
    }
    if (rk) return log ? zs::thompson_win_kernel<true, true, false> : zs::thompson_win_kernel<false, true, false>;
    return log ? zs::thompson_win_kernel<true, false, false> : zs::thompson_win_kernel<false, false, false>;
  }
  if (srec) {
    if (rk) return log ? zs::thompson_kernel<true, true, true, false> : zs::thompson_kernel<false, true, true, false>;
    return log ? zs::thompson_kernel<true, false, true, false> : zs::thompson_kernel<false, false, true, false>;
  }
  if (rk) return log ? zs::thompson_kernel<true, true, false, false> : zs::thompson_kernel<false, true, false, false>;
  return log ? zs::thompson_kernel<true, false, false, false> : zs::thompson_kernel<false, false, false, false>;
}

// Dynamic shared memory allowed per launch of fn: the device's opt-in maximum minus the
// kernel's static shared memory.  Set once to the maximum (the attribute is process-wide),
// so handles with different footprints can launch the same kernels concurrently.
cudaError_t grant_max_smem(const void *fn, int device, int *granted = nullptr) {
  int optin = 0;
  cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa;
  if ((e = cudaFuncGetAttributes(&fa, fn)) != cudaSuccess) return e;
  const int dyn = optin - (int)fa.sharedSizeBytes;
  if (granted) *granted = dyn;
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn)) != cudaSuccess)
    return e;
#ifndef ZS_DEFAULT_CARVEOUT
  // all of the unified L1/shared capacity as shared memory: the replay's blocks are
  // bounded by it, and its global traffic is one 32-byte record per decision
  return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
#else
  return cudaSuccess;
#endif
}

// replay_group_kernel<W, WINDOWED, LOG> by runtime flags
template <int W>
void launch_group_w(bool windowed, bool log, dim3 grid, size_t smem, cudaStream_t st,
                    const zs::ReplayArgs &a) {
  if (windowed) {
    if (log) zs::replay_group_kernel<W, true, true><<<grid, 128, smem, st>>>(a);
    else zs::replay_group_kernel<W, true, false><<<grid, 128, smem, st>>>(a);
  } else {
    if (log) zs::replay_group_kernel<W, false, true><<<grid, 128, smem, st>>>(a);
    else zs::replay_group_kernel<W, false, false><<<grid, 128, smem, st>>>(a);
  }
}
void launch_group(int w, bool windowed, bool log, dim3 grid, size_t smem, cudaStream_t st,
                  const zs::ReplayArgs &a) {
  if (w == 2) launch_group_w<2>(windowed, log, grid, smem, st, a);
  else if (w == 4) launch_group_w<4>(windowed, log, grid, smem, st, a);
  else launch_group_w<8>(windowed, log, grid, smem, st, a);
}
template <int W>
cudaError_t grant_group(int device) {
  cudaError_t e;
  if ((e = grant_max_smem((const void *)zs::replay_group_kernel<W, false, false>, device)) != cudaSuccess) return e;
  if ((e = grant_max_smem((const void *)zs::replay_group_kernel<W, false, true>, device)) != cudaSuccess) return e;
  if ((e = grant_max_smem((const void *)zs::replay_group_kernel<W, true, false>, device)) != cudaSuccess) return e;
  return grant_max_smem((const void *)zs::replay_group_kernel<W, true, true>, device);
}

void launch_step1(zeus_sim *s, cudaStream_t st) {
  zs::Step1Args a{};
  a.A = s->d_A.as<double>();
  a.Th = s->d_Th.as<double>();
  a.pool = s->d_pool.as<int32_t>();
  a.cells = s->d_cells.as<zs::CellParam>();
  a.arms = s->d_arms.as<zs::ArmConst>();
  a.regret = s->d_regret.as<double>();
  a.opt = s->d_opt.as<double>();
  a.opt_arm = s->d_optarm.as<int32_t>();
  a.ebar = s->d_ebar.as<double>();
  a.B = s->B; a.P = s->P; a.S = s->S; a.K = s->K; a.max_epochs = s->max_epochs;
  a.reg_stride = s->reg_stride; a.opt_stride = s->opt_stride; a.MP = s->MP;
  zs::step1_kernel<<<(unsigned)s->cells.size(), 256, 0, st>>>(a);
}

}  // namespace

extern "C" {

const char *zeus_sim_last_error(const zeus_sim *sim) {
  return sim ? sim->err.c_str() : g_create_error.c_str();
}

zeus_status zeus_sim_create(const zeus_job *job, const zeus_cell *cells, int32_t num_cells,
                            const zeus_run_opts *opts, int32_t cuda_device, zeus_sim **out) {
  NvtxRange nvtx_("zeus_sim_create");
  g_create_error.clear();
  if (!out) return fail(nullptr, ZEUS_E_INVALID, "out is NULL");
  *out = nullptr;
  Errors E;
  check_job(job, E);
  check_cells(cells, num_cells, E);
  if (!opts) E.add(ZEUS_E_INVALID, "opts is NULL");
  else {
    if (opts->struct_size != sizeof(zeus_run_opts)) E.add(ZEUS_E_INVALID, "zeus_run_opts.struct_size mismatch (ABI)");
    if (opts->recurrences < 0) E.add(ZEUS_E_INVALID, "recurrences < 0");
    if (opts->shard_begin < 0) E.add(ZEUS_E_INVALID, "shard_begin < 0");
    if (opts->shard_end >= 0 && opts->shard_end < opts->shard_begin) E.add(ZEUS_E_INVALID, "shard_end < shard_begin");
    if (opts->log_mode != 0 && opts->log_mode != 1) E.add(ZEUS_E_INVALID, "log_mode must be 0 or 1");
    if (opts->layout < 0 || opts->layout > 4) E.add(ZEUS_E_INVALID, "layout must be 0, 1, 2, 3 or 4");
    if (opts->graph != 0 && opts->graph != 1) E.add(ZEUS_E_INVALID, "graph must be 0 or 1");
    if (opts->draw < 0 || opts->draw > 2) E.add(ZEUS_E_INVALID, "draw must be 0, 1 or 2");
  }
  if (E.code == ZEUS_OK) {              // the Observe records are indexed in 32 bits (thompson.cuh)
    uint64_t recs = 0;
    for (int i = 0; i < num_cells; ++i) {
      const int64_t b = std::min(opts->shard_begin, cells[i].trials);
      const int64_t e = opts->shard_end < 0 ? cells[i].trials : std::min(opts->shard_end, cells[i].trials);
      recs += (uint64_t)std::max<int64_t>(0, e - b) * (uint64_t)job->num_batch_sizes;
    }
    if (recs >= (1ull << 32))
      E.add(ZEUS_E_UNSUPPORTED, "this shard holds >= 2^32 Observe records (trials x batch sizes over all "
                                "cells); split it into smaller shards");
  }
  if (E.code != ZEUS_OK) return fail(nullptr, E.code, E.s);

  int ndev = 0;
  cudaError_t ce = cudaGetDeviceCount(&ndev);
  if (ce != cudaSuccess || ndev == 0)
    return fail(nullptr, ZEUS_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(ce));
  if (cuda_device < 0 || cuda_device >= ndev) return fail(nullptr, ZEUS_E_INVALID, "cuda_device out of range");
  ce = cudaSetDevice(cuda_device);
  if (ce != cudaSuccess) return fail(nullptr, ZEUS_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(ce));

  zeus_sim *s = new (std::nothrow) zeus_sim();
  if (!s) return fail(nullptr, ZEUS_E_NOMEM, "host allocation failed");
  s->device = cuda_device;
  s->B = job->num_batch_sizes;
  s->P = job->num_power_limits;
  s->b0 = job->default_bs_index;
  s->max_epochs = job->max_epochs;
  s->charge_profiling = job->charge_profiling;
  s->MP = job->max_power_w;
  s->batch_sizes.assign(job->batch_sizes, job->batch_sizes + s->B);
  s->power_limits.assign(job->power_limits_w, job->power_limits_w + s->P);
  s->cells.assign(cells, cells + num_cells);
  s->R = opts->recurrences > 0 ? opts->recurrences : 2 * s->B * s->P;
  s->log_mode = opts->log_mode;
  s->layout = opts->layout;
  s->use_graph = opts->graph;
  s->draw = opts->draw;
  cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, cuda_device);
  {                                      // arrival schedules: finite, non-decreasing (R-Q31)
    Errors EA;
    for (int i = 0; i < num_cells; ++i) {
      const double *ar = cells[i].arrivals;
      if (!ar) continue;
      for (int t = 0; t < s->R; ++t)
        if (!std::isfinite(ar[t]) || (t > 0 && ar[t] < ar[t - 1])) {
          EA.add(ZEUS_E_INVALID, "arrivals must be finite and non-decreasing (cell " + std::to_string(i) + ")");
          break;
        }
    }
    if (EA.code != ZEUS_OK) { delete s; return fail(nullptr, EA.code, EA.s); }
  }
  for (int i = 0; i < num_cells; ++i) s->wmax = std::max(s->wmax, (int)cells[i].window);
  int64_t off = 0;
  for (int i = 0; i < num_cells; ++i) {
    const zeus_cell &c = cells[i];
    zs::CellParam p{};
    p.eta = c.eta;
    p.beta = c.beta;
    p.prec0 = std::isinf(c.prior_var) ? 0.0 : 1.0 / c.prior_var;   // flat prior
    p.pm0 = c.prior_mean * p.prec0;
    p.window = c.window;
    p.policy = c.policy;
    p.ablation = c.ablation;
    // conc: 1 = arrival schedule (concurrent kernel), 2 = variant readings (variant kernel)
    p.conc = c.arrivals != nullptr ? 1 : (c.ablation & (ZEUS_VARIANT_RETRY | ZEUS_VARIANT_EPOCH_STOP |
                                                         ZEUS_VARIANT_WINDOWED_BEST)) ? 2 : 0;
    s->any_conc |= p.conc == 1;
    s->any_variant |= p.conc == 2;
    if (p.conc == 2 && (c.ablation & ZEUS_VARIANT_WINDOWED_BEST)) s->best_n = std::max(s->best_n, (int)c.window);
    s->any_ablation |= c.ablation != 0 && c.policy == ZEUS_POLICY_ZEUS && p.conc == 0;
    s->any_zeus |= c.policy == ZEUS_POLICY_ZEUS;
    s->any_baseline |= c.policy != ZEUS_POLICY_ZEUS;
    p.key0 = (uint32_t)c.seed;
    p.key1 = (uint32_t)(c.seed >> 32);
    const int64_t b = std::min(opts->shard_begin, c.trials);
    const int64_t e = opts->shard_end < 0 ? c.trials : std::min(opts->shard_end, c.trials);
    p.begin = b;
    p.n = e - b;
    p.out_off = off;
    off += p.n;
    s->max_shard = std::max(s->max_shard, p.n);
    s->cpar.push_back(p);
  }
  s->shard_total = off;
  s->nwin = (int)std::max<int64_t>(1, (s->max_shard + zs::kRegroupWindow - 1) / zs::kRegroupWindow);
  // curve slots: spread the per-warp atomics over up to 8 copies, bounded to 64 MB (64 copies:
  // CFG3 -1.5 %, the memsets and the reduction of 64 MB per job; session r02bi)
#ifndef ZS_SLOT_MAX
#define ZS_SLOT_MAX 8
#endif
  const size_t curve_bytes = (size_t)num_cells * s->R * zs::kRow * sizeof(long long);
  s->nslot = (int)std::max<size_t>(1, std::min<size_t>(ZS_SLOT_MAX, (64ull << 20) / std::max<size_t>(1, curve_bytes)));

  const size_t n = (size_t)s->shard_total;
  cudaError_t e = cudaSuccess;
  if ((e = s->d_cells.alloc(sizeof(zs::CellParam) * num_cells)) != cudaSuccess ||
      (e = s->d_slots.alloc(curve_bytes * s->nslot)) != cudaSuccess ||
      (e = s->d_fixed.alloc(curve_bytes)) != cudaSuccess ||
      (e = s->d_curves.alloc((size_t)num_cells * s->R * zs::kQ * sizeof(double))) != cudaSuccess ||
      (e = s->d_tot_cost.alloc(n * 8)) != cudaSuccess ||
      (e = s->d_tot_energy.alloc(n * 8)) != cudaSuccess ||
      (e = s->d_tot_time.alloc(n * 8)) != cudaSuccess ||
      (e = s->d_digest.alloc(n * 8)) != cudaSuccess ||
      (e = s->d_nstop.alloc(n * 4)) != cudaSuccess ||
      (e = s->d_final.alloc(n * 4)) != cudaSuccess ||
      (e = s->d_log.alloc(s->log_mode ? n * (size_t)s->R * 4 : 0)) != cudaSuccess ||
      (e = s->d_counters.alloc(zs::kCounters * 8)) != cudaSuccess ||
      (e = s->d_st.alloc(n * s->B * sizeof(zs::ArmStat))) != cudaSuccess ||
      (e = s->d_st_ring.alloc(n * s->B * (size_t)s->wmax * 8)) != cudaSuccess ||
      (e = s->d_carry.alloc(n * sizeof(zs::Carry))) != cudaSuccess ||
      (e = s->d_best_ring.alloc(n * (size_t)s->best_n * 8)) != cudaSuccess ||
      (e = s->d_perm.alloc(n * 4)) != cudaSuccess ||
      (e = s->d_bucket.alloc((size_t)num_cells * s->nwin * zs::kBuckets * 4)) != cudaSuccess ||
      (e = s->d_logtab.alloc(zs::kLogTab * sizeof(double2))) != cudaSuccess) {
    std::string m = std::string("device allocation: ") + cudaGetErrorString(e);
    delete s;
    return fail(nullptr, e == cudaErrorMemoryAllocation ? ZEUS_E_NOMEM : ZEUS_E_CUDA, m);
  }
  if ((e = cudaStreamCreateWithFlags(&s->own, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaMemcpyAsync(s->d_cells.p, s->cpar.data(), sizeof(zs::CellParam) * num_cells,
                           cudaMemcpyHostToDevice, s->own)) != cudaSuccess ||
      (e = cudaEventCreate(&s->ev0)) != cudaSuccess || (e = cudaEventCreate(&s->ev1)) != cudaSuccess ||
      (e = cudaEventCreate(&s->ev2)) != cudaSuccess || (e = cudaEventCreate(&s->ev3)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&s->ev_loaded, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&s->ev_staged, cudaEventDisableTiming)) != cudaSuccess) {
    std::string m = std::string("create: ") + cudaGetErrorString(e);
    delete s;
    return fail(nullptr, ZEUS_E_CUDA, m);
  }
  if (s->any_conc) {
    std::vector<double> arr((size_t)num_cells * s->R, 0.0);
    for (int i = 0; i < num_cells; ++i)
      if (cells[i].arrivals) std::memcpy(&arr[(size_t)i * s->R], cells[i].arrivals, (size_t)s->R * 8);
    if ((e = s->d_arrivals.alloc(arr.size() * 8)) != cudaSuccess ||
        (e = cudaMemcpyAsync(s->d_arrivals.p, arr.data(), arr.size() * 8, cudaMemcpyHostToDevice,
                             s->own)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s->own)) != cudaSuccess) {
      std::string m = std::string("arrivals: ") + cudaGetErrorString(e);
      delete s;
      return fail(nullptr, ZEUS_E_CUDA, m);
    }
  }
  zs::log_table_kernel<<<1, 128, 0, s->own>>>(s->d_logtab.as<double2>());   // the sampler's log table
  // the handle's own stream only (never the device): the pageable copies above read `cpar`
  if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(s->own)) != cudaSuccess) {
    std::string m = std::string("log table: ") + cudaGetErrorString(e);
    delete s;
    return fail(nullptr, ZEUS_E_CUDA, m);
  }
  s->stream = s->own;
  *out = s;
  return ZEUS_OK;
}

// Every kernel's dynamic shared-memory limit set to the device maximum, once per device and
// process (the attribute is per function and process-wide, so handles with different footprints
// can launch concurrently; each launch passes its own size).  Done in every zeus_sim_load_profile
// it cost ~75 us of host time per call (~80 functions x 3 driver calls).
cudaError_t grant_all(int device) {
  static std::mutex mu;
  static bool done[64] = {};
  std::lock_guard<std::mutex> lock(mu);
  if (device >= 0 && device < 64 && done[device]) return cudaSuccess;
#define ZS_TRY(x) do { const cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)
  for (int w = 0; w < 2; ++w)
    for (int l = 0; l < 2; ++l)
      for (int ph = 0; ph < 3; ++ph)
        for (int ab = 0; ab < 3; ++ab)            // ab == 2: the RK kernels
          ZS_TRY(grant_max_smem((const void *)replay_fn(w, l, ph, ab == 1, ab == 2), device));
  for (int f = 0; f < 32; ++f)
    ZS_TRY(grant_max_smem((const void *)thompson_fn(f & 1, f & 2, f & 4, f & 8, f & 16), device));
  ZS_TRY(grant_group<2>(device));
  ZS_TRY(grant_group<4>(device));
  ZS_TRY(grant_group<8>(device));
  ZS_TRY(grant_max_smem((const void *)zs::concurrent_kernel<false>, device));
  ZS_TRY(grant_max_smem((const void *)zs::concurrent_kernel<true>, device));
  ZS_TRY(grant_max_smem((const void *)zs::variant_kernel<false>, device));
  ZS_TRY(grant_max_smem((const void *)zs::variant_kernel<true>, device));
  // a captured run binds buffer addresses and launch shapes: keep it only if none changed
#undef ZS_TRY
  if (device >= 0 && device < 64) done[device] = true;
  return cudaSuccess;
}

zeus_status zeus_sim_load_profile(zeus_sim *s, const double *A, const double *Th, int32_t S,
                                  int32_t K, const int32_t *pool) {
  NvtxRange nvtx_("zeus_sim_load_profile");
  if (!s) return fail(nullptr, ZEUS_E_INVALID, "sim is NULL");
  s->err.clear();
  const std::vector<uintptr_t> sig0 = s->launch_signature();
  Errors E;
  const int B = s->B, P = s->P;
  if (!A) E.add(ZEUS_E_INVALID, "avg_power_w is NULL");
  if (!Th) E.add(ZEUS_E_INVALID, "throughput_eps is NULL");
  if (!pool) E.add(ZEUS_E_INVALID, "epochs_to_target is NULL");
  if (S < 1) E.add(ZEUS_E_INVALID, "num_slices < 1");
  if (K < 1) E.add(ZEUS_E_INVALID, "replicas < 1");
  if (A) {
    for (int i = 0; i < B * P; ++i)
      if (!(A[i] > 0.0) || !std::isfinite(A[i])) { E.add(ZEUS_E_INVALID, "average power not positive"); break; }
    for (int i = 0; i < B * P; ++i)
      if (!(A[i] <= s->MP)) { E.add(ZEUS_E_INVALID, "average power above max power"); break; }
  }
  if (Th)
    for (int i = 0; i < B * P; ++i)
      if (!(Th[i] > 0.0) || !std::isfinite(Th[i])) { E.add(ZEUS_E_INVALID, "throughput not positive"); break; }
  if (pool && S >= 1 && K >= 1) {
    for (size_t i = 0; i < (size_t)S * B * K; ++i)
      if (pool[i] > s->max_epochs) { E.add(ZEUS_E_INVALID, "epochs_to_target above max_epochs"); break; }
    for (int sl = 0; sl < S; ++sl) {
      bool any = false;
      for (int i = 0; i < B * K && !any; ++i) any = pool[(size_t)sl * B * K + i] > 0;
      if (!any) { E.add(ZEUS_E_NO_CONVERGENT_ARM, "slice " + std::to_string(sl) + " has no converged replica on any arm"); break; }
    }
  }
  if (E.code == ZEUS_OK) {
    const zs::TabLayout L(B, S, K);
    const size_t per_thread = (size_t)((B + 1) & ~1) * 16;
    const size_t need = (size_t)L.bytes + 32 * per_thread;
    if (need > 200 * 1024)
      E.add(ZEUS_E_UNSUPPORTED, "trace tables + per-trial arm state exceed shared memory (" +
                                    std::to_string(need) + " B for 32 trials)");
  }
  if (E.code != ZEUS_OK) return fail(s, E.code, E.s);
  ZS_CUDA(s, cudaSetDevice(s->device));
  // From here the handle is in flux: it is "loaded" again only when every buffer, copy and launch
  // shape below is consistent (a failure midway leaves it unloaded, so zeus_sim_run refuses it).
  s->loaded = false;
  s->tables_valid = false;
  s->pareto_valid = false;
  cudaStream_t st = s->stream;
  const int nc = (int)s->cells.size();
  const size_t b_A = (size_t)B * P * 8, b_pool = (size_t)S * B * K * 4;
  const int reg_stride = (int)align_up((size_t)S * B, 2), opt_stride = (int)align_up((size_t)S, 4);
  const bool same_shape = s->d_A.p && s->S == S && s->K == K;
  if (!same_shape) {
    // reallocation frees buffers a run still in flight may read: wait for the handle's stream
    // (cudaFree would otherwise synchronise the whole device)
    ZS_CUDA(s, cudaStreamSynchronize(st));
    s->drop_graph();
    s->S = S;
    s->K = K;
    s->reg_stride = reg_stride;
    s->opt_stride = opt_stride;
    ZS_CUDA(s, s->d_A.alloc(b_A));
    ZS_CUDA(s, s->d_Th.alloc(b_A));
    ZS_CUDA(s, s->d_pool.alloc(align_up(b_pool, 16)));
    ZS_CUDA(s, s->d_arms.alloc((size_t)nc * B * sizeof(zs::ArmConst)));
    ZS_CUDA(s, s->d_regret.alloc((size_t)nc * s->reg_stride * 8));
    ZS_CUDA(s, s->d_opt.alloc((size_t)nc * S * 8));
    ZS_CUDA(s, s->d_optarm.alloc((size_t)nc * s->opt_stride * 4));
    ZS_CUDA(s, s->d_ebar.alloc((size_t)S * B * 8));
    ZS_CUDA(s, s->d_pareto.alloc((size_t)S * B * P));
    // counted curves: [cells][R][nhslot][4][B][K] u32, up to ZS_HSLOT_MAX slot copies within 64 MB
    const size_t per_slot = (size_t)nc * s->R * 4 * B * K * 4;
#ifndef ZS_HSLOT_MAX
#define ZS_HSLOT_MAX 4                      // 16: CFG3 -1.5 % with 64 curve slots (session r02bi)
#endif
    s->nhslot = (int)std::max<size_t>(1, std::min<size_t>(ZS_HSLOT_MAX, (ZS_HSLOT_MAX * 4ull << 20) / std::max<size_t>(1, per_slot)));
    ZS_CUDA(s, s->d_hist.alloc(per_slot * s->nhslot));
  }
  // Stage the caller's arrays in pinned memory (read before this call returns), then copy them
  // to the device on the handle's stream: ordered after any run still in flight there, so that
  // run finishes with the old tables.  The staging buffer is reused once its last copy is done.
  const size_t stage = 2 * b_A + b_pool;
  if (s->staged_pending) { ZS_CUDA(s, cudaEventSynchronize(s->ev_staged)); s->staged_pending = false; }
  if (s->h_stage_bytes < stage) {
    if (s->h_stage) ZS_CUDA(s, cudaFreeHost(s->h_stage));
    s->h_stage = nullptr;
    s->h_stage_bytes = 0;
    ZS_CUDA(s, cudaMallocHost(&s->h_stage, stage));
    s->h_stage_bytes = stage;
  }
  unsigned char *hs = static_cast<unsigned char *>(s->h_stage);
  std::memcpy(hs, A, b_A);
  std::memcpy(hs + b_A, Th, b_A);
  std::memcpy(hs + 2 * b_A, pool, b_pool);
  if (align_up(b_pool, 16) > b_pool)        // the bulk copies read the pool padded to 16 B
    ZS_CUDA(s, cudaMemsetAsync(static_cast<unsigned char *>(s->d_pool.p) + b_pool, 0,
                               align_up(b_pool, 16) - b_pool, st));
  if (!same_shape) {
    ZS_CUDA(s, cudaMemsetAsync(s->d_regret.p, 0, s->d_regret.bytes, st));
    ZS_CUDA(s, cudaMemsetAsync(s->d_optarm.p, 0, s->d_optarm.bytes, st));
  }
  ZS_CUDA(s, cudaMemcpyAsync(s->d_A.p, hs, b_A, cudaMemcpyHostToDevice, st));
  ZS_CUDA(s, cudaMemcpyAsync(s->d_Th.p, hs + b_A, b_A, cudaMemcpyHostToDevice, st));
  ZS_CUDA(s, cudaMemcpyAsync(s->d_pool.p, hs + 2 * b_A, b_pool, cudaMemcpyHostToDevice, st));
  ZS_CUDA(s, cudaEventRecord(s->ev_staged, st));
  s->staged_pending = true;
  {
    // F of the curves' fixed point: every per-trial value of a recurrence (cost, energy, time,
    // pseudo-regret) is at most mult * max_epochs * max_{b,p} max(MAXPOWER, 1) / Th(b,p) (A <=
    // MAXPOWER, so cost and energy per epoch are below MAXPOWER / Th; mult = B when retries can
    // charge several runs to one recurrence); with V < 2^e, F = 60 - e keeps |v 2^F| < 2^60.
    double vmax = 0.0;
    for (int i = 0; i < B * P; ++i) vmax = std::max(vmax, std::max(s->MP, 1.0) / Th[i]);
    bool retry = false;
    for (const auto &c : s->cells) retry |= (c.ablation & ZEUS_VARIANT_RETRY) != 0;
    vmax *= (double)s->max_epochs * (retry ? B : 1);
    int e = 0;
    std::frexp(vmax, &e);                   // vmax < 2^e
    s->curve_bits = std::max(-1000, std::min(1000, 60 - e));
  }
  ZS_CUDA(s, cudaEventRecord(s->ev_loaded, st));

  // launch shape of the replay (a reload with the same table shape keeps it: it depends on
  // B, S, K and the handle's fixed options only)
  if (!same_shape) {
    // launch shape of the replay: the block size (32/64/128 trials) that keeps the
    // most warps resident given the shared-memory footprint per trial
    const zs::TabLayout L(B, S, K);
    s->tab_bytes = L.bytes;
    const int wmax = s->wmax;
    // (mu, sigma) per arm, and the bound screen's two residual slots
    const size_t per_thread = (size_t)((B + 1) & ~1) * 16 + (ZS_BOUND_SKIP ? 16 * zs::kResSlots : 0);
    int best_warps = -1;
    // sized for the kernel that dominates: the Thompson phase when the schedule has two
    // phases (R > 2B), else the one-pass kernel; ties keep the larger block (fewer stagings)
    const bool two_phase = (s->layout == 2 || s->layout == 4 || (s->layout == 0 && (s->wmax == 0 || s->R >= 16 * B))) &&
                           std::min(s->R, 2 * B) < s->R;
    for (int tpb : {128, 64, 32}) {
      const size_t bytes = (size_t)L.bytes + (size_t)tpb * per_thread;
      if (bytes > 227 * 1024) continue;
      int blocks = 0;
      const void *fn = (const void *)replay_fn(wmax > 0, false, two_phase ? 2 : 0, s->any_ablation, s->cells.size() == 1);
      int granted = 0;
      ZS_CUDA(s, grant_max_smem(fn, s->device, &granted));
      if ((int)bytes > granted) continue;
      ZS_CUDA(s, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, tpb, bytes));
      const int warps = blocks * tpb / 32;
      if (warps > best_warps) { best_warps = warps; s->tpb = tpb; s->smem_bytes = (int)bytes; }
  #ifdef ZS_EXPERIMENT_SMEM_PAD
      s->smem_bytes += ZS_EXPERIMENT_SMEM_PAD;   // occupancy experiments only
  #endif
    }
    if (best_warps <= 0) return fail(s, ZEUS_E_UNSUPPORTED, "no launch shape fits shared memory");
    // lane groups (layout 3, or auto when one thread per trial cannot fill the GPU): W lanes per
    // trial, W = the power of two covering about two survivor pairs per lane
    {
      int64_t zeus_trials = 0;
      for (const auto &p : s->cpar) if (p.policy == ZEUS_POLICY_ZEUS && !p.conc) zeus_trials += p.n;
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
      const int pairs = (B + 1) / 2;
      const int w = pairs <= 2 ? 2 : pairs <= 8 ? 4 : 8;
      // measured: lane groups win only when the grouped launch fills at most a quarter of one
      // wave (CFG1 +18 %); beyond that the serial work each lane repeats costs more than the
      // split draw saves (CFG2 -35 %, CFG4 -70 %)
      const bool small = zeus_trials * w * 4 <= (int64_t)sms * best_warps * 32;
      s->group_w = 0;
      if (!s->any_ablation && (s->layout == 3 || (s->layout == 0 && small))) {
        const size_t gbytes = (size_t)L.bytes + (size_t)(128 / w) * (((B + 1) & ~1) * 16);
        if (gbytes <= 200 * 1024) s->group_w = w;
      }
    }
  }
  // the shared-memory grants are process-wide attributes: once per device (grant_all)
  ZS_CUDA(s, grant_all(s->device));
  s->loaded = true;
  if (s->launch_signature() != sig0) s->drop_graph();
  return ZEUS_OK;
}

// Enqueues one run's memsets, events and kernels on st (a1-a7 and the f-row kernels).
static zeus_status enqueue_run(zeus_sim *s, cudaStream_t st, bool capturing) {
  const int nc = (int)s->cells.size();
  // the timing events: inside a capture they must be external event nodes to be recorded
  auto record = [&](cudaEvent_t ev) {
    return capturing ? cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal) : cudaEventRecord(ev, st);
  };
  ZS_CUDA(s, cudaMemsetAsync(s->d_slots.p, 0, s->d_slots.bytes, st));
  ZS_CUDA(s, cudaMemsetAsync(s->d_counters.p, 0, s->d_counters.bytes, st));
  if (s->any_zeus && !s->any_ablation) ZS_CUDA(s, cudaMemsetAsync(s->d_hist.p, 0, s->d_hist.bytes, st));
  ZS_CUDA(s, record(s->ev0));
  launch_step1(s, st);                        // a1: Eq. 7 argmin + per-arm constants
  ZS_CUDA(s, cudaGetLastError());
  ZS_CUDA(s, record(s->ev3));
  s->launches = 2;                            // step 1 + curve reduction
  if (s->max_shard > 0 && s->R > 0 && s->any_baseline) {
    zs::BaselineArgs b{};
    b.cells = s->d_cells.as<zs::CellParam>();
    b.A = s->d_A.as<double>();
    b.Th = s->d_Th.as<double>();
    b.pool = s->d_pool.as<int32_t>();
    b.arms = s->d_arms.as<zs::ArmConst>();
    b.ebar = s->d_ebar.as<double>();
    b.opt = s->d_opt.as<double>();
    b.opt_arm = s->d_optarm.as<int32_t>();
    b.curve_slots = s->d_slots.as<long long>();
    b.curve_scale = std::ldexp(1.0, s->curve_bits);
    b.tot_cost = s->d_tot_cost.as<double>();
    b.tot_energy = s->d_tot_energy.as<double>();
    b.tot_time = s->d_tot_time.as<double>();
    b.digest = s->d_digest.as<unsigned long long>();
    b.n_stop = s->d_nstop.as<int32_t>();
    b.final_arm = s->d_final.as<int32_t>();
    b.log = s->d_log.as<uint32_t>();
    b.counters = s->d_counters.as<unsigned long long>();
    b.B = s->B; b.P = s->P; b.S = s->S; b.K = s->K; b.R = s->R; b.max_epochs = s->max_epochs;
    b.b0 = s->b0; b.nslot = s->nslot; b.opt_stride = s->opt_stride; b.MP = s->MP;
    const dim3 grid((unsigned)((s->max_shard + 127) / 128), (unsigned)nc);
    if (s->log_mode) zs::baseline_kernel<true><<<grid, 128, 0, st>>>(b);
    else zs::baseline_kernel<false><<<grid, 128, 0, st>>>(b);
    ZS_CUDA(s, cudaGetLastError());
    s->launches += 1;
  }
  if (s->max_shard > 0 && s->R > 0 && (s->any_conc || s->any_variant)) {
    zs::ConcArgs c{};
    c.cells = s->d_cells.as<zs::CellParam>();
    c.arms = s->d_arms.as<zs::ArmConst>();
    c.regret = s->d_regret.as<double>();
    c.opt_arm = s->d_optarm.as<int32_t>();
    c.pool = s->d_pool.as<int32_t>();
    c.logtab = s->d_logtab.as<double2>();
    c.arrivals = s->d_arrivals.as<double>();
    c.curve_slots = s->d_slots.as<long long>();
    c.curve_scale = std::ldexp(1.0, s->curve_bits);
    c.tot_cost = s->d_tot_cost.as<double>();
    c.tot_energy = s->d_tot_energy.as<double>();
    c.tot_time = s->d_tot_time.as<double>();
    c.digest = s->d_digest.as<unsigned long long>();
    c.n_stop = s->d_nstop.as<int32_t>();
    c.final_arm = s->d_final.as<int32_t>();
    c.log = s->d_log.as<uint32_t>();
    c.counters = s->d_counters.as<unsigned long long>();
    c.st = s->d_st.as<zs::ArmStat>();
    c.st_ring = s->d_st_ring.as<double>();
    c.ring_n = s->wmax;
    c.B = s->B; c.S = s->S; c.K = s->K; c.R = s->R; c.max_epochs = s->max_epochs;
    c.charge_profiling = s->charge_profiling; c.b0 = s->b0; c.nslot = s->nslot;
    c.reg_stride = s->reg_stride; c.opt_stride = s->opt_stride;
    c.A = s->d_A.as<double>();
    c.Th = s->d_Th.as<double>();
    c.ebar = s->d_ebar.as<double>();
    c.opt = s->d_opt.as<double>();
    c.best_ring = s->d_best_ring.as<double>();
    c.P = s->P;
    c.best_n = s->best_n;
    c.MP = s->MP;
    const size_t smem = (size_t)128 * (((s->B + 1) & ~1) * 16);
    const dim3 grid((unsigned)((s->max_shard + 127) / 128), (unsigned)nc);
    c.cert_draw = s->draw != 1 ? 1 : 0;
    c.force_exact = s->draw == 2 ? 1 : 0;
    if (s->any_conc) {                      // + the outstanding-run queues (kernels.cuh) + the
                                            // certified draw's fp32 table (pairs padded to quads)
      const size_t csmem = smem + (size_t)128 * zs::kQueueBytes +
                           (size_t)128 * (((((s->B + 1) / 2) + 1) & ~1) * 16);
      if (s->log_mode) zs::concurrent_kernel<true><<<grid, 128, csmem, st>>>(c);
      else zs::concurrent_kernel<false><<<grid, 128, csmem, st>>>(c);
      ZS_CUDA(s, cudaGetLastError());
      s->launches += 1;
    }
    if (s->any_variant) {
      const size_t vsmem = smem + (size_t)128 * (((((s->B + 1) / 2) + 1) & ~1) * 16);   // + fp32 table
      if (s->log_mode) zs::variant_kernel<true><<<grid, 128, vsmem, st>>>(c);
      else zs::variant_kernel<false><<<grid, 128, vsmem, st>>>(c);
      ZS_CUDA(s, cudaGetLastError());
      s->launches += 1;
    }
  }
  if (s->max_shard > 0 && s->R > 0 && s->any_zeus) {
    zs::ReplayArgs a{};
    a.cells = s->d_cells.as<zs::CellParam>();
    a.arms = s->d_arms.as<zs::ArmConst>();
    a.regret = s->d_regret.as<double>();
    a.opt_arm = s->d_optarm.as<int32_t>();
    a.pool = s->d_pool.as<int32_t>();
    a.curve_slots = s->d_slots.as<long long>();
    a.curve_scale = std::ldexp(1.0, s->curve_bits);
    a.tot_cost = s->d_tot_cost.as<double>();
    a.tot_energy = s->d_tot_energy.as<double>();
    a.tot_time = s->d_tot_time.as<double>();
    a.digest = s->d_digest.as<unsigned long long>();
    a.n_stop = s->d_nstop.as<int32_t>();
    a.final_arm = s->d_final.as<int32_t>();
    a.log = s->d_log.as<uint32_t>();
    a.counters = s->d_counters.as<unsigned long long>();
    a.B = s->B; a.S = s->S; a.K = s->K; a.R = s->R; a.max_epochs = s->max_epochs;
    a.charge_profiling = s->charge_profiling; a.b0 = s->b0; a.nslot = s->nslot;
    a.reg_stride = s->reg_stride; a.opt_stride = s->opt_stride; a.tab_bytes = s->tab_bytes;
    const bool windowed = s->wmax > 0;
    a.st = s->d_st.as<zs::ArmStat>();
    a.st_ring = s->d_st_ring.as<double>();
    a.ring_n = s->wmax;
    const dim3 grid((unsigned)((s->max_shard + s->tpb - 1) / s->tpb), (unsigned)nc);
    // two-phase schedule when Thompson sampling follows the pruning stage (R > 2B):
    // phase A = the first 2B recurrences (Alg. 3 pruning is at most 2B runs), then the
    // trials of each cell are regrouped by survivor-pair count so a warp's lanes
    // draw the same number of normals per decision in phase B
    a.t_split = std::min(s->R, 2 * s->B);
    a.hist = s->d_hist.as<uint32_t>();
    a.nhslot = s->nhslot;
    a.carry = s->d_carry.as<zs::Carry>();
    a.perm = s->d_perm.as<int32_t>();
    a.bucket = s->d_bucket.as<int32_t>();
    a.nwin = s->nwin;
    a.logtab = s->d_logtab.as<double2>();
    a.A = s->d_A.as<double>();
    a.Th = s->d_Th.as<double>();
    a.ebar = s->d_ebar.as<double>();
    a.opt = s->d_opt.as<double>();
    a.P = s->P;
    a.MP = s->MP;
    // one-cell launches carry the cell's Philox round keys in the kernel parameters (RK kernels)
    const bool rk = nc == 1;
    if (rk) {
      uint32_t k0 = s->cpar[0].key0, k1 = s->cpar[0].key1;
      for (int r = 0; r < 10; ++r) {
        a.rk.k0[r] = k0;
        a.rk.k1[r] = k1;
        k0 += 0x9E3779B9u;                   // Philox4x32 key schedule (Weyl constants)
        k1 += 0xBB67AE85u;
      }
    }
    // the one-pass and exact phase-B schedules run the certified draw too (draw != 1); its fp32
    // table (float4 per pair, pairs padded to whole quads) follows the residual slots
    a.cert_draw = s->draw != 1 ? 1 : 0;
    const size_t cert_bytes = (size_t)s->tpb * (((((s->B + 1) / 2) + 1) & ~1) * 16);
    auto replay_launch = [&](int phase) {
      const size_t rsmem = s->smem_bytes + ((phase != 1 || ZS_PHASEA_CERT) && a.cert_draw ? cert_bytes : 0);
      replay_fn(windowed, s->log_mode, phase, s->any_ablation, rk)<<<grid, s->tpb, rsmem, st>>>(a);
    };
    // the Thompson phase with the certified fp32 draw unless the run asks for
    // the exact-screen kernel (draw = 1); cells with a window or an ablation keep replay_kernel
    const bool certified = !s->any_ablation && s->draw != 1 && (!windowed || ZS_WIN_THOMPSON);
    a.key_quads = certified ? 1 : 0;
    a.force_exact = s->draw == 2 ? 1 : 0;
    const dim3 tgrid((unsigned)((s->max_shard + 127) / 128), (unsigned)nc);
    size_t tab = (size_t)s->tab_bytes;
    if (windowed) {                            // the compact table layout of the WIN variant
      const zs::ThTabLayout TL(s->B, s->S, s->K, 128 * (((((s->B + 1) / 2) + 1) & ~1) * 16 + 16));
      a.th_logtab = TL.logtab; a.th_pool = TL.pool; a.th_bytes = TL.bytes; a.th_pool_smem = TL.pool_smem;
      tab = (size_t)TL.bytes;
    }
    const size_t tsmem = tab + (size_t)128 * (((((s->B + 1) / 2) + 1) & ~1) * 16 + 16);
    // launches of at most two blocks per SM keep the survivors' records in shared memory
    // (thompson.cuh, SREC): there the decision's latency is the throughput
    const size_t rec_bytes = (size_t)128 * s->B * sizeof(zs::ArmStat);
    const bool srec = s->layout != 4 && (int64_t)tgrid.x * tgrid.y <= 2 * (int64_t)s->sms &&
                      tsmem + rec_bytes <= 100 * 1024;
    // early split: phase A stops each lane at its first pure Thompson decision and
    // the Thompson phase starts it there, when the pruning stage is a large share of the run
    // (R < 40 |B|, i.e. fewer than 20 Thompson recurrences per pruning recurrence) and the launch
    // is not a small SREC one.  Measured (session r02bc): CFG3 +2.8 %, CFG4 +2 %; CFG5 (R = 62 |B|)
    // -0.8 %, CFG2 (SREC) -0.7 %, so those keep the full phase A.  Layout 4 forces it.
    a.early_split = certified && ZS_EARLY_SPLIT && (s->layout == 4 || (s->layout == 0 && !srec && s->R < 40 * s->B)) ? 1 : 0;
    auto thompson_launch = [&]() {
      const size_t m = tsmem + (srec ? rec_bytes : 0);
      thompson_fn(s->log_mode, rk, srec, windowed, a.early_split != 0)<<<tgrid, 128, m, st>>>(a);
    };
    // auto: two phases, except for windowed launches with few Thompson recurrences per pruning
    // recurrence (R < 8 x 2|B|), where the one-pass kernel measured faster (session r02al: CFG4 at
    // R = 200 two phases 2.08 vs one pass 1.96e10, CFG4 at R = 38 one pass 1.26 vs 1.08e10);
    // explicit layouts are honoured
    const bool two_phase = (s->layout == 2 || s->layout == 4 || (s->layout == 0 && (!windowed || s->R >= 16 * s->B))) &&
                           a.t_split < s->R;
    if (s->group_w > 0) {                    // lane-group layout (latency-bound launches)
      const int tpg = 128 / s->group_w;
      const dim3 ggrid((unsigned)((s->max_shard + tpg - 1) / tpg), (unsigned)nc);
      const size_t gsmem = (size_t)s->tab_bytes + (size_t)tpg * (((s->B + 1) & ~1) * 16);
      launch_group(s->group_w, windowed, s->log_mode, ggrid, gsmem, st, a);
      ZS_CUDA(s, cudaGetLastError());
      s->launches += 1;
    } else if (!two_phase) {
      replay_launch(0);
      ZS_CUDA(s, cudaGetLastError());
      s->launches += 1;
    } else {
      s->launches += 4;
      ZS_CUDA(s, cudaMemsetAsync(s->d_bucket.p, 0, s->d_bucket.bytes, st));

      replay_launch(1);
      ZS_CUDA(s, cudaGetLastError());
      zs::bucket_scan_kernel<<<(unsigned)((nc * (int64_t)s->nwin * 32 + 127) / 128), 128, 0, st>>>(a.bucket, nc, s->nwin);
      ZS_CUDA(s, cudaGetLastError());
      const unsigned sx = (unsigned)std::min<int64_t>((s->max_shard + zs::kScatterTile - 1) / zs::kScatterTile, 1184);
      zs::bucket_scatter_kernel<<<dim3(std::max(1u, sx), (unsigned)nc), zs::kScatterTile, 0, st>>>(
          a.cells, a.carry, a.bucket, a.perm, nc, s->B, s->nwin, a.key_quads, a.early_split);
      ZS_CUDA(s, cudaGetLastError());
      if (certified) thompson_launch();
      else replay_launch(2);
      ZS_CUDA(s, cudaGetLastError());
    }
    if (!s->any_ablation) {                    // the counted runs into the exact sums
      const long long n = (long long)nc * s->R * 4 * s->B * s->K;
      zs::curve_hist_fold_kernel<<<(unsigned)std::max<long long>(1, std::min<long long>(4 * 1184, (n + 127) / 128)),
                                   128, 0, st>>>(
          a.hist, a.curve_slots, a.arms, a.regret, a.opt_arm, a.pool, nc, s->nslot, s->nhslot, s->R, s->B,
          s->S, s->K, s->max_epochs, s->reg_stride, s->opt_stride, a.curve_scale);
      ZS_CUDA(s, cudaGetLastError());
      s->launches += 1;
    }
  }
  ZS_CUDA(s, record(s->ev1));
  zs::curve_reduce_kernel<<<std::max(1, std::min(4 * 1184, (int)((nc * (size_t)s->R * zs::kQ + 7) / 8))), 256, 0, st>>>(
      s->d_slots.as<long long>(), s->d_fixed.as<long long>(), s->d_curves.as<double>(), nc, s->nslot,
      s->R, std::ldexp(1.0, -s->curve_bits));
  ZS_CUDA(s, cudaGetLastError());
  ZS_CUDA(s, record(s->ev2));
  return ZEUS_OK;
}

zeus_status zeus_sim_run(zeus_sim *s, void *stream) {
  NvtxRange nvtx_("zeus_sim_run");
  if (!s) return fail(nullptr, ZEUS_E_INVALID, "sim is NULL");
  s->err.clear();
  if (!s->loaded) return fail(s, ZEUS_E_STATE, "zeus_sim_run before zeus_sim_load_profile");
  ZS_CUDA(s, cudaSetDevice(s->device));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (st != s->stream) ZS_CUDA(s, cudaStreamWaitEvent(st, s->ev_loaded, 0));   // the load's copies
  s->stream = st;
  if (!s->use_graph) {
    const zeus_status rc = enqueue_run(s, st, false);
    if (rc != ZEUS_OK) return rc;
  } else {
    if (!s->graph_exec) {                   // capture once; the legacy stream cannot capture
      if (!s->cap_stream) ZS_CUDA(s, cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
      ZS_CUDA(s, cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal));
      const zeus_status rc = enqueue_run(s, s->cap_stream, true);
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(s->cap_stream, &g);
      if (rc != ZEUS_OK) { if (g) cudaGraphDestroy(g); return rc; }
      ZS_CUDA(s, ec);
      s->graph = g;
      ZS_CUDA(s, cudaGraphInstantiate(&s->graph_exec, s->graph, 0));
      s->graph_launches = s->launches;
    }
    ZS_CUDA(s, cudaGraphLaunch(s->graph_exec, st));
    s->launches = s->graph_launches;
  }
  s->ran = true;
  s->tables_valid = true;                   // the run's step 1 wrote the tables
  return ZEUS_OK;
}

// The replay outputs into device or pinned host buffers, enqueued on the handle's stream without
// waiting (the multi-job bench step: six handles' curves handed to their consumers in stream
// order, no host round trip per handle; the e2e loop: every job's copies queued before one
// wait).  Everything is validated before any copy is queued.
zeus_status zeus_sim_results_async(zeus_sim *s, zeus_results *out) {
  NvtxRange nvtx_("zeus_sim_results_async");
  if (!s) return fail(nullptr, ZEUS_E_INVALID, "sim is NULL");
  s->err.clear();
  if (!out) return fail(s, ZEUS_E_INVALID, "out is NULL");
  if (out->struct_size != sizeof(zeus_results)) return fail(s, ZEUS_E_INVALID, "zeus_results.struct_size mismatch (ABI)");
  if (!s->loaded) return fail(s, ZEUS_E_STATE, "zeus_sim_results_async before zeus_sim_load_profile");
  if (!s->ran) return fail(s, ZEUS_E_STATE, "zeus_sim_results_async before zeus_sim_run");
  if (out->log && !s->log_mode) return fail(s, ZEUS_E_STATE, "log requested but log_mode = 0");
  if (out->pstar_index || out->c1 || out->t1 || out->e1 || out->c_prof || out->t_prof || out->e_prof ||
      out->opt_cost || out->opt_arm || out->pareto)
    return fail(s, ZEUS_E_INVALID, "zeus_sim_results_async copies replay outputs only (step-1 tables and "
                                   "Pareto masks: zeus_sim_results)");
  ZS_CUDA(s, cudaSetDevice(s->device));
  const int nc = (int)s->cells.size();
  const size_t n = (size_t)s->shard_total;
  struct Req { void *dst; const DevBuf *src; size_t bytes; const char *name; };
  const Req req[] = {{out->curves, &s->d_curves, (size_t)nc * s->R * zs::kQ * 8, "curves"},
                     {out->curves_fixed, &s->d_fixed, (size_t)nc * s->R * zs::kRow * 8, "curves_fixed"},
                     {out->tot_cost, &s->d_tot_cost, n * 8, "tot_cost"},
                     {out->tot_energy, &s->d_tot_energy, n * 8, "tot_energy"},
                     {out->tot_time, &s->d_tot_time, n * 8, "tot_time"},
                     {out->digest, &s->d_digest, n * 8, "digest"},
                     {out->n_stop, &s->d_nstop, n * 4, "n_stop"},
                     {out->final_arm, &s->d_final, n * 4, "final_arm"},
                     {out->log, &s->d_log, n * (size_t)s->R * 4, "log"},
                     {out->counters, &s->d_counters, zs::kCounters * 8, "counters"}};
  for (const Req &r : req) {
    if (!r.dst) continue;
    cudaPointerAttributes pa{};
    const cudaError_t e = cudaPointerGetAttributes(&pa, r.dst);
    if (e != cudaSuccess || (pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged &&
                             pa.type != cudaMemoryTypeHost)) {
      cudaGetLastError();
      return fail(s, ZEUS_E_INVALID, std::string("zeus_sim_results_async: ") + r.name +
                                         " is neither device nor pinned host memory");
    }
  }
  for (const Req &r : req)
    if (r.dst && r.bytes) ZS_CUDA(s, cudaMemcpyAsync(r.dst, r.src->p, r.bytes, cudaMemcpyDefault, s->stream));
  out->kernel_launches = s->launches;
  out->curve_scale_bits = s->curve_bits;
  return ZEUS_OK;
}

zeus_status zeus_sim_results(zeus_sim *s, zeus_results *out) {
  NvtxRange nvtx_("zeus_sim_results");
  if (!s) return fail(nullptr, ZEUS_E_INVALID, "sim is NULL");
  s->err.clear();
  if (!out) return fail(s, ZEUS_E_INVALID, "out is NULL");
  if (out->struct_size != sizeof(zeus_results)) return fail(s, ZEUS_E_INVALID, "zeus_results.struct_size mismatch (ABI)");
  if (!s->loaded) return fail(s, ZEUS_E_STATE, "zeus_sim_results before zeus_sim_load_profile");
  // every request is validated before any copy is queued into a caller buffer
  if (!s->ran && (out->curves || out->curves_fixed || out->tot_cost || out->tot_energy || out->tot_time || out->digest ||
                  out->n_stop || out->final_arm || out->log || out->counters))
    return fail(s, ZEUS_E_STATE, "replay outputs requested before zeus_sim_run");
  if (out->log && !s->log_mode) return fail(s, ZEUS_E_STATE, "log requested but log_mode = 0");
  ZS_CUDA(s, cudaSetDevice(s->device));
  cudaStream_t st = s->stream;
  const bool want_tables = out->pstar_index || out->c1 || out->t1 || out->e1 || out->c_prof ||
                           out->t_prof || out->e_prof || out->opt_cost || out->opt_arm || out->pareto;
  if (want_tables && !s->tables_valid) {    // step 1 of the loaded traces, before any run
    launch_step1(s, st);
    ZS_CUDA(s, cudaGetLastError());
    s->tables_valid = true;
  }
  if (out->pareto && !s->pareto_valid) {    // f4, computed only when asked for
    zs::pareto_kernel<<<s->S, 256, 0, st>>>(s->d_A.as<double>(), s->d_Th.as<double>(),
                                           s->d_ebar.as<double>(), s->d_pool.as<int32_t>(),
                                           s->d_pareto.as<uint8_t>(), s->B, s->P, s->K);
    ZS_CUDA(s, cudaGetLastError());
    s->pareto_valid = true;
  }
  const int nc = (int)s->cells.size();
  const size_t n = (size_t)s->shard_total;
  // host-built arrays into a caller buffer: a plain memcpy for host memory, else a copy on the
  // handle's stream (a pageable source is staged before cudaMemcpyAsync returns)
  auto put = [&](void *dst, const void *src, size_t bytes) -> cudaError_t {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeDevice)
      return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
    cudaGetLastError();                       // clear a "not a device pointer" from the query
    std::memcpy(dst, src, bytes);
    return cudaSuccess;
  };
  auto cp = [&](void *dst, const DevBuf &src, size_t bytes) -> cudaError_t {
    if (!dst || bytes == 0) return cudaSuccess;
    return cudaMemcpyAsync(dst, src.p, bytes, cudaMemcpyDefault, st);   // host or device dst
  };
  if (s->ran) {
    ZS_CUDA(s, cp(out->curves, s->d_curves, (size_t)nc * s->R * zs::kQ * 8));
    ZS_CUDA(s, cp(out->curves_fixed, s->d_fixed, (size_t)nc * s->R * zs::kRow * 8));
    ZS_CUDA(s, cp(out->tot_cost, s->d_tot_cost, n * 8));
    ZS_CUDA(s, cp(out->tot_energy, s->d_tot_energy, n * 8));
    ZS_CUDA(s, cp(out->tot_time, s->d_tot_time, n * 8));
    ZS_CUDA(s, cp(out->digest, s->d_digest, n * 8));
    ZS_CUDA(s, cp(out->n_stop, s->d_nstop, n * 4));
    ZS_CUDA(s, cp(out->final_arm, s->d_final, n * 4));
    ZS_CUDA(s, cp(out->log, s->d_log, n * (size_t)s->R * 4));
    ZS_CUDA(s, cp(out->counters, s->d_counters, zs::kCounters * 8));
  }
  ZS_CUDA(s, cp(out->opt_cost, s->d_opt, (size_t)nc * s->S * 8));
  ZS_CUDA(s, cp(out->pareto, s->d_pareto, (size_t)s->S * s->B * s->P));
  if (out->opt_arm) {
    std::vector<int32_t> tmp((size_t)nc * s->opt_stride);
    ZS_CUDA(s, cudaMemcpyAsync(tmp.data(), s->d_optarm.p, tmp.size() * 4, cudaMemcpyDeviceToHost, st));
    ZS_CUDA(s, cudaStreamSynchronize(st));
    std::vector<int32_t> packed((size_t)nc * s->S);
    for (int c = 0; c < nc; ++c)
      std::memcpy(&packed[(size_t)c * s->S], &tmp[(size_t)c * s->opt_stride], (size_t)s->S * 4);
    ZS_CUDA(s, put(out->opt_arm, packed.data(), packed.size() * 4));
  }
  const bool want_arms = out->pstar_index || out->c1 || out->t1 || out->e1 || out->c_prof ||
                         out->t_prof || out->e_prof;
  if (want_arms) {
    std::vector<zs::ArmConst> arms((size_t)nc * s->B);
    ZS_CUDA(s, cudaMemcpyAsync(arms.data(), s->d_arms.p, arms.size() * sizeof(zs::ArmConst),
                               cudaMemcpyDeviceToHost, st));
    ZS_CUDA(s, cudaStreamSynchronize(st));
    std::vector<int32_t> ps(arms.size());
    std::vector<double> f[6];
    for (auto &v : f) v.resize(arms.size());
    for (size_t i = 0; i < arms.size(); ++i) {
      ps[i] = arms[i].pstar;
      f[0][i] = arms[i].c1; f[1][i] = arms[i].t1; f[2][i] = arms[i].e1;
      f[3][i] = arms[i].cP; f[4][i] = arms[i].tP; f[5][i] = arms[i].eP;
    }
    double *dst[6] = {out->c1, out->t1, out->e1, out->c_prof, out->t_prof, out->e_prof};
    if (out->pstar_index) ZS_CUDA(s, put(out->pstar_index, ps.data(), ps.size() * 4));
    for (int q = 0; q < 6; ++q)
      if (dst[q]) ZS_CUDA(s, put(dst[q], f[q].data(), f[q].size() * 8));
  }
  ZS_CUDA(s, cudaStreamSynchronize(st));
  out->replay_ms = 0.f;
  out->step1_ms = 0.f;
  out->reduce_ms = 0.f;
  if (s->ran) {
    ZS_CUDA(s, cudaEventElapsedTime(&out->step1_ms, s->ev0, s->ev3));
    ZS_CUDA(s, cudaEventElapsedTime(&out->replay_ms, s->ev3, s->ev1));
    ZS_CUDA(s, cudaEventElapsedTime(&out->reduce_ms, s->ev1, s->ev2));
  }
  out->kernel_launches = s->ran ? s->launches : 0;
  out->curve_scale_bits = s->curve_bits;
  return ZEUS_OK;
}

zeus_status zeus_sim_curves_from_fixed(zeus_sim *s, const int64_t *curves_fixed, double *curves) {
  NvtxRange nvtx_("zeus_sim_curves_from_fixed");
  if (!s) return fail(nullptr, ZEUS_E_INVALID, "sim is NULL");
  s->err.clear();
  if (!curves_fixed || !curves) return fail(s, ZEUS_E_INVALID, "curves_fixed / curves is NULL");
  if (!s->loaded) return fail(s, ZEUS_E_STATE, "zeus_sim_curves_from_fixed before zeus_sim_load_profile");
  ZS_CUDA(s, cudaSetDevice(s->device));
  cudaPointerAttributes pa{}, pb{};
  const bool dev_in = cudaPointerGetAttributes(&pa, curves_fixed) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
  const bool dev_out = cudaPointerGetAttributes(&pb, curves) == cudaSuccess && pb.type == cudaMemoryTypeDevice;
  cudaGetLastError();
  if (!dev_in || !dev_out) return fail(s, ZEUS_E_INVALID, "curves_fixed and curves must be device memory");
  const long long rows = (long long)s->cells.size() * s->R;
  zs::curves_from_fixed_kernel<<<std::max(1, (int)std::min<long long>(1184, (rows * zs::kQ + 255) / 256)), 256, 0,
                                 s->stream>>>(reinterpret_cast<const long long *>(curves_fixed), curves, rows,
                                              std::ldexp(1.0, -s->curve_bits));
  ZS_CUDA(s, cudaGetLastError());
  ZS_CUDA(s, cudaStreamSynchronize(s->stream));
  return ZEUS_OK;
}

void zeus_sim_destroy(zeus_sim *s) {
  if (!s) return;
  cudaSetDevice(s->device);
  delete s;
}

zeus_status zeus_sim_shape(const zeus_sim *s, int32_t *recurrences, int64_t *shard,
                           int32_t *num_cells, int32_t *num_batch_sizes, int32_t *num_slices) {
  if (!s) return ZEUS_E_INVALID;
  if (recurrences) *recurrences = s->R;
  if (shard) *shard = s->shard_total;
  if (num_cells) *num_cells = (int32_t)s->cells.size();
  if (num_batch_sizes) *num_batch_sizes = s->B;
  if (num_slices) *num_slices = s->S;
  return ZEUS_OK;
}

zeus_status zeus_sim_certify_bounds(int32_t cuda_device, double *out) {
  if (!out) return ZEUS_E_INVALID;
  int ndev = 0, prev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) return ZEUS_E_CUDA;
  if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(cuda_device) != cudaSuccess) return ZEUS_E_CUDA;
  struct Restore { int d; ~Restore() { cudaSetDevice(d); } } restore{prev};   // the caller's device
  cudaStream_t st = nullptr;
  double2 *tab = nullptr;
  unsigned *d_out = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&tab, zs::kLogTab * sizeof(double2));
  if (e == cudaSuccess) e = cudaMalloc(&d_out, 5 * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemsetAsync(d_out, 0, 5 * sizeof(unsigned), st);
  if (e == cudaSuccess) {
    zs::log_table_kernel<<<1, 128, 0, st>>>(tab);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cuda_device);
    const uint64_t N = 1ull << 32, chunk = 1ull << 30;    // every 32-bit word, in four launches
    for (uint64_t b = 0; b < N; b += chunk) {
      zs::cert::certify_radius_kernel<<<sms * 8, 256, 0, st>>>(tab, b, chunk, d_out);
      zs::cert::certify_angle_kernel<<<sms * 8, 256, 0, st>>>(b, chunk, d_out);
    }
    zs::cert::certify_theta_kernel<<<sms * 8, 256, 0, st>>>(tab, 0, 1ull << 28, d_out);
    e = cudaGetLastError();
  }
  unsigned h[5] = {0, 0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d_out, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (tab) cudaFree(tab);
  if (d_out) cudaFree(d_out);
  if (st) cudaStreamDestroy(st);
  if (e != cudaSuccess) return ZEUS_E_CUDA;
  for (int i = 0; i < 4; ++i) {
    float f;
    std::memcpy(&f, &h[i], 4);
    out[i] = f;
  }
  out[4] = zs::cert::kAng;
  out[5] = zs::cert::kRMax;
  float f4;
  std::memcpy(&f4, &h[4], 4);
  out[6] = f4;
  out[7] = (double)(1ull << 28);
  return ZEUS_OK;
}

}  // extern "C"
