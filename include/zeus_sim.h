/*
 * zeus_sim.h -- C ABI of the B200 batched replay of Zeus's optimiser.
 *
 * Zeus (You, Chung, Chowdhury, arXiv 2208.06102) picks, for every recurrence
 * of a recurring DNN training job, a batch size b by Gaussian Thompson
 * sampling after a pruning stage (Alg. 1-3) and the power limit p
 * of that batch size by minimising the per-epoch cost of a JIT profile
 * (Eq. 7), early-stopping runs whose cost is to exceed beta times
 * the minimum cost seen.  The paper evaluates it by replaying a
 * training trace and a power trace (§6.1).  This library runs
 * that replay for many independent trials at once on one GPU: one call of
 * zeus_sim_run is trials x R decisions for every cell.
 *
 * Citations: P:Lnnn = line of the paper's LaTeX; DESIGN.md §4 is
 * the numerics contract (NC-1..NC-9) both this library and the CPU oracle
 * follow, §3 the readings of passages the paper leaves open (R-Qn).
 *
 * Conventions (all calls):
 *  - Every call returns zeus_status; ZEUS_OK = 0.  On failure
 *    zeus_sim_last_error(sim) returns a message listing EVERY violated
 *    invariant ("; "-separated), valid until the next call on that handle.
 *    For a failed zeus_sim_create, the message is returned by
 *    zeus_sim_last_error(NULL) (thread-local).
 *  - Ownership: input arrays are read (and copied) before the call returns;
 *    the handle owns all device memory until zeus_sim_destroy; results are
 *    written only into caller-owned buffers.
 *  - Async, stream-ordered: every handle has a STREAM -- the cudaStream_t of its
 *    last zeus_sim_run, or an internal non-blocking stream before the first run.
 *    zeus_sim_load_profile enqueues its copies on it (after any run still in
 *    flight there) and returns; zeus_sim_run enqueues on the caller's stream,
 *    first making it wait for the last load, and that stream becomes the
 *    handle's; zeus_sim_results enqueues its copies on the handle's stream and
 *    synchronises that stream only.  No call launches work on the legacy
 *    default stream unless the caller passes it, and no call synchronises the
 *    device (zeus_sim_destroy and reallocations excepted: cudaFree does).
 *    A stream passed to zeus_sim_run must stay valid until the handle has run
 *    on another stream or is destroyed.
 *  - Threading: a handle belongs to one thread at a time; distinct handles
 *    may run concurrently on different streams or devices.
 *  - Sharding: RNG counters use the GLOBAL trial index (NC-3), so per-trial
 *    results do not depend on how [0, trials) is split across ranks.
 *  - No CPU fallback: when no CUDA device is usable every call that would
 *    launch work fails with ZEUS_E_CUDA.
 *  - Exactness: every decision is the numerics contract's.  The
 *    Thompson draw may be evaluated in fp32 with a proven error bound and its
 *    argmin certified against the contract's fp64 values (zeus_run_opts.draw,
 *    DESIGN.md §7.9); where the bound cannot separate the winner the contract's
 *    fp64 draw decides.  Options change the work, never the results.
 */
#ifndef ZEUS_SIM_H
#define ZEUS_SIM_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ZEUS_SIM_ABI_VERSION 3   /* 2: zeus_run_opts.draw, 14 counters, zeus_sim_certify_bounds;
                                    3: zeus_sim_results_async, layout 4 (early split) */
#define ZEUS_MAX_BATCH_SIZES 32
#define ZEUS_MAX_POWER_LIMITS 64
#define ZEUS_CURVE_QUANTITIES 7   /* cost, energy, time, pseudo-regret, n_stop, n_opt, n_ts */
#define ZEUS_COUNTERS 14   /* 0..8 contract events (oracle-checked), 9..13 work evaluated */

typedef enum {
  ZEUS_OK = 0,
  ZEUS_E_INVALID = 1,            /* an argument violates an invariant (message lists all) */
  ZEUS_E_STATE = 2,              /* calls out of order (run before load_profile, ...) */
  ZEUS_E_NO_CONVERGENT_ARM = 3,  /* a trace slice where no replica of any arm converges */
  ZEUS_E_CUDA = 4,               /* CUDA runtime error (message has the CUDA string) */
  ZEUS_E_NOMEM = 5,              /* device or host allocation failed */
  ZEUS_E_UNSUPPORTED = 6         /* valid but outside this build's limits (B > 32, ...) */
} zeus_status;

typedef struct zeus_sim zeus_sim;   /* opaque; single owner */

/* The recurring job ("a set of feasible batch sizes B and power limits P"). */
typedef struct {
  uint32_t struct_size;              /* = sizeof(zeus_job) (ABI guard) */
  int32_t num_batch_sizes;           /* B = |𝓑|, 1..32 */
  const int32_t *batch_sizes;        /* host [B], positive, strictly increasing */
  int32_t default_bs_index;          /* b0 in [0,B): Alg. 3's starting batch size */
  int32_t num_power_limits;          /* P = |𝓟|, 1..64 */
  const double *power_limits_w;      /* host [P], positive, strictly increasing (watts) */
  double max_power_w;                /* MAXPOWER of Eq. 2, >= max 𝓟 */
  int32_t max_epochs;                /* >= 1: epochs a never-converging run is charged (R-Q16) */
  int32_t charge_profiling;          /* 1: the first run of each arm pays the JIT profiling
                                        epoch, one equal-work slice per power limit */
} zeus_job;

/* One sweep cell: the knobs η, β, N and the prior of Alg. 2. */
typedef struct {
  double eta;                        /* η in [0,1] (Eq. 2) */
  double beta;                       /* β > 1, or +INFINITY = never early-stop */
  int32_t window;                    /* N >= 2 most recent observations, 0 = unbounded */
  double prior_mean;                 /* μ̂0 (Alg. 2) */
  double prior_var;                  /* σ̂0² > 0; +INFINITY = flat prior */
  uint64_t seed;                     /* Philox4x32-10 key (NC-3) */
  int64_t trials;                    /* global trial count of this cell, >= 0 */
  int32_t policy;                    /* ZEUS_POLICY_*: Zeus, or one of the paper's baselines
                                        replayed on the same traces and replica draws */
  int32_t ablation;                  /* Zeus only: ZEUS_ABLATE_* bits and
                                        ZEUS_VARIANT_* bits; "no early stopping" is beta =
                                        +INFINITY */
  const double *arrivals;            /* NULL: recurrences run back to back (the paper's replay);
                                        else host [R] non-decreasing submission times (s) shared
                                        by the cell's trials: concurrent submissions (§4.4
                                        P:L634-646); a run completes at its submission time +
                                        its TTA; Zeus policy without ablations only */
} zeus_cell;

#define ZEUS_ABLATE_PRUNING 1       /* keep every batch size: Alg. 3 still walks, 𝓑 is not pruned */
#define ZEUS_ABLATE_JIT 2           /* no JIT profiler: the first |𝓟| runs of each batch size try
                                       the power limits in ascending order, one per recurrence */
/* variant readings of the early stop (DESIGN.md R-Q4v, R-Q1v, R-Q5v), same field,
   sequential recurrences only (no arrivals), combinable with each other and the ablations */
#define ZEUS_VARIANT_RETRY 4        /* "stop the job and retry with another batch size": after an
                                       early stop the recurrence continues with another decision
                                       (Thompson sampling leaves out the arms stopped in it); it
                                       ends with its first run that is not stopped */
#define ZEUS_VARIANT_EPOCH_STOP 8   /* the cost is checked at epoch boundaries: the run
                                       stops at the end of the first epoch whose accumulated cost
                                       exceeds beta*best, and is charged that epoch's cost */
#define ZEUS_VARIANT_WINDOWED_BEST 16 /* best = min over the converged runs of the last N = window
                                       recurrences (needs window >= 2): the threshold follows drift */

/* policies (§6.1 "Baselines"; DESIGN.md R-Q29) */
#define ZEUS_POLICY_ZEUS 0          /* Alg. 3 pruning + Alg. 1/2 Thompson sampling, Eq. 7 p*, early stop */
#define ZEUS_POLICY_DEFAULT 1       /* (b0, largest power limit) every recurrence */
#define ZEUS_POLICY_GRID_SEARCH 2   /* one (b, p) per recurrence, b then p ascending; a failed run
                                       prunes its batch size; then the cheapest seen */

typedef struct {
  uint32_t struct_size;              /* = sizeof(zeus_run_opts) */
  int32_t recurrences;               /* R >= 0; 0 = auto = 2|𝓑||𝓟| */
  int64_t shard_begin, shard_end;    /* this rank's global trial range [begin, end) of
                                        every cell, clipped to [0, trials); end < 0 = all */
  int32_t log_mode;                  /* 0: no log; 1: per-decision log (4 B / decision) */
  int32_t layout;                    /* schedule of the replay kernel; results
                                        are bit-identical for every value:
                                        0 auto: 3 when the grouped launch fills at most a
                                          quarter wave, else 2 when R > 2|𝓑| and either no
                                          cell has a window or R >= 16|𝓑|, else 1 (chosen by
                                          measurement);
                                        1 one pass, one thread per trial;
                                        2 two phases: the pruning stage, then the Thompson
                                          stage with trials regrouped by survivor count;
                                        3 one pass, a lane group of W = 2/4/8 lanes per trial
                                          (the draw split across lanes, shuffle argmin);
                                        4 two phases with the early split: the pruning phase
                                          stops each trial at its first pure Thompson decision
                                          and the Thompson phase starts it there (auto takes it
                                          for the certified draw when R < 40|𝓑| and the launch
                                          exceeds two blocks per SM) */
  int32_t graph;                     /* 0: zeus_sim_run enqueues its kernels one by one;
                                        1: the first run captures them into a CUDA graph (on an
                                          internal stream) and every run launches that graph on
                                          the caller's stream -- one launch instead of 5-10 for
                                          launch-bound configurations; same results.
                                          zeus_sim_load_profile discards the graph. */
  int32_t draw;                      /* the Thompson draw of the two-phase schedule (Alg. 1
                                        P:L455-463); same results for
                                        every value:
                                        0: certified fp32 -- every survivor's theta in fp32
                                          with a proven error bound; the contract's fp64 draw
                                          only when the bounds do not separate the argmin;
                                        1: the exact fp64 draw with the bound screen;
                                        2: certified fp32 with every decision sent to the fp64
                                          fallback (a test of that path).
                                        Cells with a window or an ablation always take 1. */
} zeus_run_opts;

/* Outputs.  Every pointer is caller-owned and may be NULL (skipped); each
 * may point to host or device memory (detected per pointer).  Layouts are
 * row-major; "shard" = shard_end - shard_begin after clipping. */
typedef struct {
  uint32_t struct_size;              /* = sizeof(zeus_results) */
  /* per-recurrence curves summed over this shard's trials, [cells][R][7]:
     q = 0 cost, 1 energy (J), 2 time (s), 3 pseudo-regret Ebar(b_t)c1(b_t) - opt
     (Eq. 9 with Epochs read as the trace mean, R-Q12), 4 early stops, 5 decisions
     equal to the known optimum, 6 decisions taken by Thompson sampling.
     Each value is the EXACT sum of the per-trial values quantised to 2^-F (F =
     curve_scale_bits, chosen from an upper bound of one run's cost so that
     |v 2^F| < 2^60), rounded once to fp64: the same bits whatever the trial
     order, launch layout or sharding.  Counts are exact. */
  double *curves;
  /* the same sums before rounding, [cells][R][7][3] int64 limbs: value = (l0 + l1 2^26 +
     l2 2^52) 2^-F (counts: l0).  Integer sums, so ranks all-reduce THESE (exactly) and
     convert with zeus_sim_curves_from_fixed to get world-size-invariant curves. */
  int64_t *curves_fixed;
  /* per trial [cells][shard] */
  double *tot_cost, *tot_energy, *tot_time;   /* summed in recurrence order (NC-8) */
  uint64_t *digest;                           /* FNV-1a-64 over (b_t, p_t, flags) (NC-9) */
  int32_t *n_stop;                            /* early stops of the trial */
  int32_t *final_arm;                         /* b_{R-1} index (-1 if R = 0) */
  /* step-1 tables (Eq. 7 and the JIT epoch) [cells][B] */
  int32_t *pstar_index;
  double *c1, *t1, *e1;                       /* cost / s / J per epoch at p*(b) */
  double *c_prof, *t_prof, *e_prof;           /* cost / s / J of the profiling epoch */
  /* known optimum per slice [cells][S] */
  double *opt_cost;
  int32_t *opt_arm;
  /* Pareto front of each slice's (TTA, ETA) grid [S][B][P] (§2.3; the traces'
     property, the same for every cell): 1 = non-dominated, TTA = Ebar/Th, ETA = Ebar*A/Th */
  uint8_t *pareto;
  /* per-decision log [cells][shard][R] (needs log_mode = 1):
     arm | p_index << 8 | flags << 16, flags bit0 stopped, bit1 converged,
     bit2 paid the profiling epoch, bit3 decided by Thompson sampling */
  uint32_t *log;
  /* instrumentation [14]: decisions, sampled TS decisions, normal pairs drawn,
     normals used, early stops, pruning decisions, forced explorations,
     posterior recomputations, Philox blocks drawn for normals (NC-3: two pairs each)
     -- [0..8] are events of the method, identical to the oracle's --
     then the work this build evaluated for them: [9] fp64 Box-Muller transforms, [10] Philox
     blocks, [11] pairs bound-screened (exact-screen kernels: the screen skips the transform of
     pairs whose arms provably cannot win: [9] <= [2]) plus pairs transformed
     in fp32 (certified draw, §7.9), [12] draws decided by the certified fp32 bounds,
     [13] draws sent to the exact fp64 fallback */
  int64_t *counters;
  /* timing of the last zeus_sim_run, CUDA events on the caller's stream:
     step 1 (Eq. 7) kernel, replay kernel, curve-reduction kernel */
  float step1_ms, replay_ms, reduce_ms;
  int32_t kernel_launches;           /* kernels the last zeus_sim_run launched */
  int32_t curve_scale_bits;          /* F of curves_fixed (set by every successful call) */
} zeus_results;

/* Validates job, cells and opts (every violated invariant is reported),
 * selects cuda_device, allocates device memory.  *out is NULL on failure.
 * ZEUS_E_UNSUPPORTED when the shard holds 2^32 or more Observe records (the
 * trials of every cell x |B|): split it into smaller shards. */
zeus_status zeus_sim_create(const zeus_job *job, const zeus_cell *cells, int32_t num_cells,
                            const zeus_run_opts *opts, int32_t cuda_device, zeus_sim **out);

/* The power trace and the training trace (§6.1):
 *   avg_power_w     host [B][P], 0 < AvgPower(b,p) <= MAXPOWER
 *   throughput_eps  host [B][P], Throughput(b,p) > 0 in epochs/s
 *   epochs_to_target host [S][B][K] (S slices, K replicas); <= 0 = the run never
 *                   reaches the target (R-Q16); every value <= max_epochs;
 *                   every slice needs one converged replica on some arm.
 * The arrays are copied into a pinned staging buffer before the call returns
 * (the caller may reuse them at once), then to the device asynchronously on the
 * handle's stream, after any run still in flight there.  Same-shaped reloads
 * (same S and K) reuse every device buffer, so a captured CUDA graph stays
 * valid; a new shape first waits for the handle's stream, then reallocates.
 * Step 1 (Eq. 7 argmin, per-epoch and profiling constants, known optimum) is
 * computed by the next zeus_sim_run, or by zeus_sim_results when it asks for
 * the step-1 tables before any run; the Pareto masks only when asked for.
 * On any failure the handle is left unloaded (zeus_sim_run then fails with
 * ZEUS_E_STATE) until a load succeeds. */
zeus_status zeus_sim_load_profile(zeus_sim *sim, const double *avg_power_w,
                                  const double *throughput_eps, int32_t num_slices,
                                  int32_t replicas, const int32_t *epochs_to_target);

/* Enqueues one pass of the whole path on cuda_stream (a cudaStream_t; NULL =
 * the legacy default stream): step 1 for every cell, the replay of every
 * (cell, shard trial) for R recurrences, and the curve reduction. */
zeus_status zeus_sim_run(zeus_sim *sim, void *cuda_stream);

/* Validates the request (ZEUS_E_STATE for replay outputs before any run, or a
 * log without log_mode; nothing is copied then), enqueues the copies on the
 * handle's stream, synchronises that stream, and returns. */
zeus_status zeus_sim_results(zeus_sim *sim, zeus_results *out);

/* The replay outputs (curves, curves_fixed, the per-trial arrays, log, counters) into device or
 * PINNED host buffers (cudaHostAlloc / cudaHostRegister), enqueued on the handle's stream (the
 * stream of the last zeus_sim_run) without synchronising: consumers order on that stream, a host
 * reader synchronises it first.  ZEUS_E_INVALID (nothing queued) for a pageable destination or a
 * step-1 table / Pareto request, ZEUS_E_STATE before any run.  Fills kernel_launches and
 * curve_scale_bits; the event timings are zeus_sim_results'. */
zeus_status zeus_sim_results_async(zeus_sim *sim, zeus_results *out);

/* curves [cells][R][7] (device) from fixed-point sums curves_fixed [cells][R][7][3] (device),
 * e.g. after an all-reduce (SUM) of every rank's curves_fixed: carries the limbs and rounds
 * once, exactly as zeus_sim_results does, so N ranks get the bits of one.  Runs on the
 * handle's stream and synchronises it.  ZEUS_E_INVALID for NULL or host pointers. */
zeus_status zeus_sim_curves_from_fixed(zeus_sim *sim, const int64_t *curves_fixed, double *curves);

/* Frees the handle and its device memory; NULL is a no-op. */
void zeus_sim_destroy(zeus_sim *sim);

/* Message of the last failed call on sim (NULL: of the last failed create on
 * this thread).  Never NULL; "" when there is none. */
const char *zeus_sim_last_error(const zeus_sim *sim);

/* R actually used (after auto), shard size, number of cells; any out may be NULL. */
zeus_status zeus_sim_shape(const zeus_sim *sim, int32_t *recurrences, int64_t *shard,
                           int32_t *num_cells, int32_t *num_batch_sizes, int32_t *num_slices);

/* Exhaustive check of the two measured error bounds behind the certified fp32 draw
 * (zeus_run_opts.draw = 0), on cuda_device, for every 32-bit word:
 *   out[0] = max over radius words a of |r32 - r| / e_r(a)   (the bound holds iff <= 1),
 *   out[1] = max r32                                          (must be <= out[5]),
 *   out[2] = max over angle words b of |cos32 - cos|, out[3] of |sin32 - sin| (<= out[4]),
 *   out[4] = the angle bound compiled into the kernels, out[5] = the radius cap,
 *   out[6] = max over out[7] seeded random (words, mu, sigma, ref) of |key - (theta - ref)| / E,
 *            the composed per-arm bound of the certified argmin (holds iff <= 1),
 * where r, cos, sin, theta are the contract's fp64 values (NC-3, NC-4).  out: host, 8 doubles.
 * Returns ZEUS_OK, ZEUS_E_INVALID (out NULL) or ZEUS_E_CUDA.  About 0.1 s on a B200. */
zeus_status zeus_sim_certify_bounds(int32_t cuda_device, double *out);

#ifdef __cplusplus
}
#endif
#endif
