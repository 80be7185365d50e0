/* sched.h -- C ABI of libsched, the B200-native batched WAIT / Nested WAIT /
 * FCFS discrete-event simulator of arXiv 2504.11320 ("Optimizing LLM
 * Inference: Fluid-Guided Online Scheduling with Memory Constraints").
 *
 * PAPER.md:N = line N of the paper source (authoritative text 984-2609);
 * DESIGN.md §4 fixes the bit-exact semantics every entry point implements.
 *
 * Conventions for every entry point:
 *   - return 0 (SCHED_OK) on success, a negative SCHED_E_* code on failure;
 *     a human-readable message is then available from sched_last_error()
 *     (thread-local, valid until the next failing call on that thread);
 *   - "host" pointers are read during the call only and may be freed after;
 *   - "device" pointers are CUDA global memory owned by the caller;
 *   - all lengths are tokens, rates 1/s, times seconds; internally 1 tick = 1 ps.
 */
#ifndef WAITSIM_SCHED_H
#define WAITSIM_SCHED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sched_s* sched_t;

/* policies */
enum {
  SCHED_WAIT = 0,    /* Algorithm 1: per-type thresholds n_j */
  SCHED_NESTED = 1,  /* Algorithm 2: per-segment thresholds n_k */
  SCHED_FCFS = 2,    /* vLLM-style new-first FCFS baseline */
  SCHED_FCFS_ONGOING = 3  /* Sarathi-style ongoing-first FCFS (R29):
                             new prompts are admitted only if they fit after the
                             ongoing prompts' growth */
};

/* error codes */
enum {
  SCHED_OK = 0,
  SCHED_E_INVALID = -1,       /* bad argument / config */
  SCHED_E_UNSTABLE = -2,      /* rho >= 1 (Prop. 1) */
  SCHED_E_INFEASIBLE = -3,    /* no threshold vector satisfies the recipe */
  SCHED_E_UNSATISFIABLE = -4, /* some l + l' > M: a prompt can never complete */
  SCHED_E_CUDA = -5,          /* CUDA runtime error (message has the detail) */
  SCHED_E_CAPACITY = -6       /* a replication overflowed its resident / restart capacity */
};

/* Per-replication metric row fields (uint64 each).  Output arrays are
 * FIELD-MAJOR: value of field f for local replication i is out[f*n_reps + i].
 * 128-bit tick sums are split into _LO / _HI words.  Definitions: DESIGN.md
 * §4.4-§4.6 (metrics of PAPER.md:1235-1242). */
enum {
  SCHED_F_ARRIVALS = 0,         /* arrivals with t < T */
  SCHED_F_ADMITTED,             /* admissions (prefills), re-admissions included */
  SCHED_F_COMPLETED,            /* completions with t_end <= T */
  SCHED_F_COMPLETED_AFTER_T,    /* completions of the batch straddling T */
  SCHED_F_COMPLETED_TOKENS,     /* sum of l' over completed: throughput * T */
  SCHED_F_FIRST_TOKENS,         /* first output tokens emitted by T */
  SCHED_F_BATCHES,              /* executed iterations */
  SCHED_F_REQUEST_STEPS,        /* sum over iterations of |batch| */
  SCHED_F_PREFILL_STEPS,        /* sum over iterations of new admissions */
  SCHED_F_EVICTIONS,            /* LIFO evictions */
  SCHED_F_BUSY_TICKS,           /* sum of tau */
  SCHED_F_IDLE_TICKS,           /* sum of idle jumps */
  SCHED_F_LAT_LO, SCHED_F_LAT_HI,     /* sum of latency (t_end - a) of completed */
  SCHED_F_TTFT_LO, SCHED_F_TTFT_HI,   /* sum of TTFT over first tokens by T */
  SCHED_F_SOJ_LO, SCHED_F_SOJ_HI,     /* sum over arrivals of min(c,T) - a */
  SCHED_F_COMPLETION_BATCH_IDX, /* sum of 0-based batch index of each completion */
  SCHED_F_MAX_KV_PEAK,          /* max post-iteration KV of any executed batch */
  SCHED_F_FINAL_WAITING,        /* prompts in FIFOs at stop */
  SCHED_F_FINAL_RESIDENT,       /* GPU-resident prompts at stop */
  SCHED_F_TRAJ_HASH,            /* 64-bit trajectory hash */
  SCHED_F_STATUS,               /* 0 ok; 1 resident overflow; 2 restart overflow (the CPU
                                   oracle also uses 3: invariant P14 violated) */
  SCHED_F_NOW_STOP,             /* simulated clock at stop */
  SCHED_F_SUM_WAITING,          /* sum over batches of waiting prompts at decision */
  SCHED_NF
};

/* Simulated system + policy.  Length tables: class c's prefill table is
 * entries [l_off[c], l_off[c+1]) of (l_val, l_w); a 1-entry table is a fixed
 * length ("Prompt Characteristics"); weights are
 * integers. */
typedef struct {
  uint32_t K;                 /* classes / prompt types, 1..32 */
  const double* lambda;       /* host [K]: Poisson rate (>= 0; 0 = class absent) */
  const uint32_t* l_off;      /* host [K+1] */
  const uint16_t* l_val;      /* host: prefill lengths l >= 1 */
  const uint64_t* l_w;        /* host: weights (sum > 0 per class) */
  const uint32_t* lp_off;     /* host [K+1] */
  const uint16_t* lp_val;     /* host: decode lengths 1 <= l' <= 32767 */
  const uint64_t* lp_w;
  double d0_s;                /* tau = d0 + d1 * tokens (Eq. time_consump) */
  double d1_s;
  int64_t M;                  /* KV capacity C in tokens (Eq. memory_constraint) */
  int32_t policy;             /* SCHED_WAIT / SCHED_NESTED / SCHED_FCFS / SCHED_FCFS_ONGOING */
  uint32_t n_thr;             /* WAIT: K; NESTED: n_seg; 0 = set later by sched_thresholds */
  const uint32_t* thresholds; /* host [n_thr], each >= 1 */
  uint32_t n_seg;             /* NESTED: number of segments L (1..32) */
  const uint16_t* seg_end;    /* host [n_seg]: last stage of each segment, increasing,
                                 seg_end[0] >= 1, seg_end[L-1] >= max l' */
  uint32_t B;                 /* FCFS*: max resident prompts (>= 1); WAIT heuristic B */
  uint32_t tok_budget;        /* FCFS*: max prefill tokens per iteration (0 = none) */
  uint32_t max_resident;      /* per-replication safe resident capacity (0 = derive): the
                                 fallback launch's; the main launch still runs with a
                                 speculative capacity <= it (see spec_resident) */
  uint32_t restart_cap;       /* restart pool capacity in entries (0 = default 2^24): evicted
                                 prompts waiting to re-enter their FIFO live in
                                 64-entry chunks of one device pool shared by all replications
                                 of a launch (20 B per entry); a replication finding it
                                 exhausted reports status 2 */
  /* optional time-varying rates ("Time-Varying Arrival
   * Rates"; NULL rf_off = all homogeneous): class c has pieces
   * [rf_off[c], rf_off[c+1]) of (rf_t start second, rf_rate rate >= 0) with
   * rf_t[first] = 0 and increasing starts, at most 32 pieces; an empty slice
   * keeps the constant lambda[c].  Generated by exact time change
   * (DESIGN.md §4.8); lambda[c] is still what sched_thresholds uses. */
  const uint32_t* rf_off;     /* host [K+1] */
  const double* rf_t;
  const double* rf_rate;
  uint32_t spec_resident;     /* speculative capacity of the main launch (0 = derive);
                                 replications exceeding it are re-run with the safe
                                 capacity by a fallback launch on the same stream */
  int32_t device;             /* CUDA device ordinal */
  int64_t tau_b0;             /* piecewise-linear iteration time (DESIGN.md
                                 R31): tau = d0 + d1 * max(0, tokens - tau_b0); 0 = the
                                 linear Eq. time_consump; >= 0.  Threshold setup
                                 (sched_thresholds) keeps the linear model. */
} sched_config;

/* Validate and copy *cfg (every array is copied; cfg may be freed after),
 * convert times to ticks and build integer CDF tables (host only: the tables
 * are uploaded to `device` by the first sched_run / sched_run_trace).  Errors: SCHED_E_INVALID (K = 0 or > 32,
 * lambda < 0, l < 1, l' < 1, empty / zero-weight table, d0 <= 0, d1 < 0,
 * M < 1, bad thresholds / seg_end, B = 0 for FCFS), SCHED_E_UNSATISFIABLE
 * (some l + l' > M), SCHED_E_CUDA. */
int sched_create(sched_t* out, const sched_config* cfg);

/* Host-side setup (no device work): fluid equilibrium of PAPER.md:1331-1361
 * (rho, dT*, n*, M*, Throughput*), integer thresholds by DESIGN.md readings
 * R24 (WAIT, mode 0), R13 (WAIT heuristic n_j = B rho_j/(l'_j+1), mode 1,
 * PAPER.md:1754) or R25 (NESTED, mode 0), the constraint check of
 * Eq. wait_thresholds / Eq. nested_wait_thresholds
 * (PAPER.md:1676-1680), theta_k of the Lemma and the
 * Thm-2 memory budget for (delta, budget_B).  If the
 * handle has no thresholds yet the chosen ones are installed.
 * Errors: SCHED_E_UNSTABLE (rho >= 1; rho is still reported),
 * SCHED_E_INFEASIBLE, SCHED_E_INVALID. */
typedef struct {
  double rho, dT_star, M_star, thr_star;  /* fluid benchmark */
  double n_star[32];                      /* per class */
  uint32_t n_thr;
  uint32_t thresholds[32];                /* chosen (or installed) thresholds */
  double dT_n;                            /* d0 + d1 M^pi at the thresholds */
  double M_pi;                            /* WAIT: Eq. wait_thresholds; NESTED: exact stage sum */
  double M_pi_paper;                      /* NESTED: printed formula (reading R9) */
  int32_t feasible;                       /* thresholds satisfy the paper's condition */
  int32_t mem_exceeds_M;                  /* M^pi > M: LIFO-eviction regime */
  double p[32], theta[32], theta_lb[32];  /* NESTED: p_k, theta_k, 8 D / n_{k-1} (0 if n/a) */
  double budget_base, budget_queue, budget_hp, budget_total;
  /* time-varying check (NESTED with rate pieces; Eq. nested_wait_thresholds_
   * time_varying): sup_t of the arrivals accumulated in
   * [t, t + dT_n] (must be < n_1), sup p_k over all windows (n_{k+1}/n_k must
   * exceed it), and the verdict; tv_feasible = -1 when not applicable */
  double tv_Lambda_pi;
  double tv_p_star[32];
  int32_t tv_feasible;
} sched_threshold_report;

int sched_thresholds(sched_t h, int32_t mode, double delta, double budget_B,
                     sched_threshold_report* out);

/* Simulate global replications rep_begin .. rep_begin+n_reps-1 over [0, T)
 * with master seed `seed`: independent Poisson arrival streams per prompt
 * type (§Model; Philox stream layout DESIGN.md §4.2, so
 * sharding is invisible to the results), scheduled by Algorithm 1 WAIT
 * (PAPER.md:1457-1496), Algorithm 2 Nested WAIT or the
 * FCFS baselines under the KV limit M with LIFO
 * eviction (Eq. memory_constraint), batch time
 * d0 + d1 tokens (Eq. time_consump) and the throughput /
 * latency / TTFT accounting of PAPER.md:1235-1242.  Asynchronous on
 * `cuda_stream` (cudaStream_t, may be NULL); writes `out_dev`, a DEVICE
 * uint64 array of SCHED_NF * n_reps (field-major, caller-owned).  Needs
 * thresholds (WAIT / NESTED).  Sync errors: SCHED_E_INVALID, SCHED_E_CUDA.
 * Capacity overflows are reported per replication in SCHED_F_STATUS (1
 * resident capacity, 2 restart pool) and in the handle's sticky status
 * mask (sched_get_status). */
int sched_run(sched_t h, uint64_t seed, uint64_t rep_begin, uint32_t n_reps,
              double horizon_s, uint64_t* out_dev, void* cuda_stream);

/* Same simulation with a HOST output array (SCHED_NF * n_reps uint64):
 * launches, copies the rows device->host and synchronises the stream. */
int sched_run_host(sched_t h, uint64_t seed, uint64_t rep_begin, uint32_t n_reps,
                   double horizon_s, uint64_t* out_host, void* cuda_stream);

/* Sums over the replications of one run (the per-policy vector that the
 * cross-GPU all-reduce adds; metrics of PAPER.md:1235-1242), on the device,
 * asynchronous on `cuda_stream`.  rows_dev: DEVICE field-major rows as
 * written by sched_run, field f of replication i at rows_dev[f*ld + i]
 * (ld >= n_reps: a column slice of a wider array).  out_int_dev (13 int64):
 * sums of ARRIVALS, ADMITTED, COMPLETED, COMPLETED_AFTER_T, COMPLETED_TOKENS,
 * FIRST_TOKENS, BATCHES, REQUEST_STEPS, PREFILL_STEPS, EVICTIONS,
 * FINAL_WAITING, FINAL_RESIDENT, and the number of replications with
 * STATUS != 0.  out_f64_dev (6 double): sum of latency, TTFT and sojourn
 * tick sums and BUSY_TICKS in seconds, sum over replications of (latency
 * sum / max(COMPLETED, 1))^2 and of (COMPLETED_TOKENS / horizon_s)^2.  One
 * 1024-thread block, fixed summation order (deterministic).  Errors:
 * SCHED_E_INVALID (null pointer, n_reps == 0, ld < n_reps, horizon <= 0),
 * SCHED_E_CUDA (launch failure). */
int sched_aggregate(const uint64_t* rows_dev, uint64_t ld, uint32_t n_reps, double horizon_s,
                    int64_t* out_int_dev, double* out_f64_dev, void* cuda_stream);

/* Explicit arrival traces (host arrays): replication i replays arrivals
 * [off[i], off[i+1]) of (t_ticks, cls, l, lp), sorted by (t, cls).  Rows go
 * to out_host (SCHED_NF * n_reps, field-major); if log_host != NULL the
 * batches of replication 0 are logged, 7 int64 each (t_start, |plan|, tokens,
 * n_complete, n_evict, n_new, peak), at most log_cap; *n_logged receives the
 * count.  Synchronous. */
int sched_run_trace(sched_t h, const int64_t* t_ticks, const int32_t* cls,
                    const int32_t* l, const int32_t* lp, const int64_t* off,
                    uint32_t n_reps, double horizon_s, uint64_t* out_host,
                    int64_t* log_host, int64_t log_cap, int64_t* n_logged);

/* Launch configuration used by sched_run (for roofline accounting). */
typedef struct {
  int32_t grid, block, warps_per_block, shared_bytes, blocks_per_sm, sm_count;
  int32_t max_resident, restart_cap;      /* safe capacity, restart pool entries */
  int32_t spec_resident;                  /* main-launch capacity (== max_resident: no fallback) */
  int32_t fallback_grid, fallback_warps_per_block;
  int32_t engine;                         /* 0 member engine (per-resident records: WAIT / FCFS
                                             with length marks); 1 class-ring engine (WAIT /
                                             FCFS with fixed per-class lengths; capacities
                                             then count ring + staging records); 2 segment
                                             engine (NESTED; spec_resident = its array,
                                             fallback = the member engine's safe launch).
                                             A NESTED handle with one class and one segment
                                             is WAIT with one type (P10): its
                                             sched_run calls execute on an internal WAIT
                                             handle, so it reports that handle's launch
                                             (engine 1 for fixed lengths); sched_run_trace
                                             keeps the Nested engines.  DESIGN.md §5.2.  The env var
                                             WAITSIM_ENGINE=member|ring|seg, read when the
                                             handle is first launched, forces one. */
  int32_t last_retries;                   /* replications of the handle's most recent
                                             sched_run / sched_run_host that overflowed the
                                             speculative capacity and re-ran in the fallback
                                             launch (synchronous device read; 0 before the
                                             first run).  Rows are unaffected (bit-exact);
                                             this is a cost diagnostic. */
} sched_launch_info;
int sched_get_launch_info(sched_t h, sched_launch_info* out);

/* Sticky status of the handle (synchronous device read): bit s of *mask is
 * set if some replication of a sched_run / sched_run_host / sched_run_trace
 * since the previous call ended with status s != 0 (a replication re-run by
 * the fallback launch reports the fallback's status only); the mask is then
 * cleared.  Errors: SCHED_E_INVALID, SCHED_E_CUDA. */
int sched_get_status(sched_t h, uint32_t* mask);

/* Restart pool use (synchronous device read): capacity in entries and the
 * high-water mark (entries in chunks ever handed out; freed chunks are
 * reused first, so this bounds the concurrent peak).  Errors: SCHED_E_INVALID,
 * SCHED_E_CUDA. */
int sched_restart_pool_stats(sched_t h, uint64_t* capacity_entries, uint64_t* high_water_entries);

/* NEXT(4): the appendix's embedded random-walk chains, one thread per walk
 * (App. B-C).  kind 0: the WAIT chain of Lemma
 * "Queue Length and Stuck Time" with X^b ~ Poisson(mu) and
 * threshold n, plus its coupled dominating process started at 2n (Lemma,
 * PAPER.md:2169).  kind 1: the Nested segment-k chain with binomial thinning
 * Y^b ~ Binomial(n_prev, p) and threshold n, coupled process started at n
 * (PAPER.md:2290-2310).  B steps per walk; walks walk_begin ..
 * walk_begin+n_walks-1 (global indices: sharding-invariant).  Output:
 * field-major int64 [SCHED_WALK_NF][n_walks]: W^B, stuck iterations,
 * sum_b W^b, max_b W^b, coupled W~^B, dominance violations (#b with
 * W~^b < W^b + n (kind 0) or < W^b (kind 1); 0 by the Lemmas), sum of
 * arrivals, max_{i<=B} S^i, min_{i<=B} S^i, S^B (S^i = partial sums of
 * arrivals - n).  sched_walks: device output, async on `cuda_stream`;
 * sched_walks_host: host output, synchronous on `device`.
 * Errors: SCHED_E_INVALID (kind, n < 1, mu <= 0 or > 1e4, n_prev < 1,
 * p outside (0,1), n_walks = 0, B = 0, walk index >= 2^32), SCHED_E_CUDA. */
enum { SCHED_WALK_NF = 10 };
int sched_walks(int32_t kind, int64_t n, double mu, int64_t n_prev, double p, uint64_t seed,
                uint64_t walk_begin, uint32_t n_walks, uint32_t B, int64_t* out_dev,
                void* cuda_stream);
int sched_walks_host(int32_t kind, int64_t n, double mu, int64_t n_prev, double p,
                     uint64_t seed, uint64_t walk_begin, uint32_t n_walks, uint32_t B,
                     int64_t* out_host, int32_t device);

void sched_destroy(sched_t h);
const char* sched_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* WAITSIM_SCHED_H */
