/* oracle.h -- TEST INFRASTRUCTURE ONLY (see oracle/des_oracle.cpp header).
 *
 * Plain sequential CPU oracle of the batched WAIT / Nested WAIT / FCFS
 * discrete-event simulation (arXiv 2504.11320).  Independent of the CUDA
 * path: it shares no code, header, table or constant generator with
 * paper_2504_11320_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 */
#ifndef WAITSIM_ORACLE_H
#define WAITSIM_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_WAIT = 0, ORC_NESTED = 1, ORC_FCFS = 2, ORC_FCFS_ONGOING = 3 };

/* metric row fields (field-major output: out[f * n_reps + i]) */
enum {
  ORC_F_ARRIVALS = 0, ORC_F_ADMITTED, ORC_F_COMPLETED, ORC_F_COMPLETED_AFTER_T,
  ORC_F_COMPLETED_TOKENS, ORC_F_FIRST_TOKENS, ORC_F_BATCHES, ORC_F_REQUEST_STEPS,
  ORC_F_PREFILL_STEPS, ORC_F_EVICTIONS, ORC_F_BUSY_TICKS, ORC_F_IDLE_TICKS,
  ORC_F_LAT_LO, ORC_F_LAT_HI, ORC_F_TTFT_LO, ORC_F_TTFT_HI, ORC_F_SOJ_LO, ORC_F_SOJ_HI,
  ORC_F_COMPLETION_BATCH_IDX, ORC_F_MAX_KV_PEAK, ORC_F_FINAL_WAITING,
  ORC_F_FINAL_RESIDENT, ORC_F_TRAJ_HASH, ORC_F_STATUS, ORC_F_NOW_STOP,
  ORC_F_SUM_WAITING, ORC_NF
};

typedef struct {
  int32_t K;                 /* number of prompt classes (1..32) */
  const double* lam;         /* [K] Poisson rate, 1/s */
  const int32_t* l_off;      /* [K+1] offsets into l_val / l_w */
  const uint16_t* l_val;     /* prefill length values */
  const uint64_t* l_w;       /* integer weights */
  const int32_t* lp_off;     /* [K+1] offsets into lp_val / lp_w */
  const uint16_t* lp_val;    /* decode length values */
  const uint64_t* lp_w;
  double d0_s, d1_s;         /* batch time tau = d0 + d1 * tokens (seconds) */
  int64_t M;                 /* KV capacity, tokens */
  int32_t policy;            /* ORC_WAIT / ORC_NESTED / ORC_FCFS / ORC_FCFS_ONGOING */
  int32_t n_thr;             /* WAIT: K thresholds; NESTED: n_seg thresholds */
  const uint32_t* thr;
  int32_t n_seg;             /* NESTED: number of segments */
  const uint16_t* seg_end;   /* NESTED: last stage of each segment */
  uint32_t B;                /* FCFS: max resident prompts */
  uint32_t tok_budget;       /* FCFS: prefill tokens per iteration, 0 = inf */
  double horizon_s;          /* T */
  /* time-varying rates (optional, NULL = homogeneous): class c has pieces
   * [rf_off[c], rf_off[c+1]) of (start second, rate); an empty slice means
   * the constant rate lam[c]; the first start must be 0 */
  const int32_t* rf_off;
  const double* rf_t;
  const double* rf_rate;
  /* piecewise-linear iteration time (reading R31):
   * tau = d0 + d1 * max(0, tokens - tau_b0); 0 = the linear Eq. time_consump */
  int64_t tau_b0;
} orc_config;

/* Philox4x32-10 (Salmon et al. SC'11). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* E = -ln(U) of the bit-exact sampler from Philox words x0,x1 */
double orc_exp_from_bits(uint32_t x0, uint32_t x1);
/* first n arrivals (k = 0..n-1) of class c in replication r: absolute tick,
 * l, l'.  Arrivals at or beyond the horizon are still generated. */
int orc_gen_arrivals(const orc_config* cfg, uint64_t seed, uint32_t r, int32_t c,
                     int64_t n, int64_t* t, int32_t* l, int32_t* lp);
/* Simulate replications rep_begin .. rep_begin+n_reps-1 on n_threads host
 * threads; out is field-major [ORC_NF][n_reps]. */
int orc_run(const orc_config* cfg, uint64_t seed, uint64_t rep_begin, int64_t n_reps,
            uint64_t* out, int32_t n_threads);
/* Explicit traces: replication i uses arrivals [off[i], off[i+1]) sorted by
 * (t, class); t in ticks (ps).  log (optional, may be NULL) receives
 * 7 int64 per batch of replication 0 only: t_start, |plan|, tokens,
 * n_complete, n_evict, n_new, peak.  Returns number of batches logged. */
int64_t orc_run_trace(const orc_config* cfg, const int64_t* t, const int32_t* cls,
                      const int32_t* l, const int32_t* lp, const int64_t* off,
                      int64_t n_reps, uint64_t* out, int64_t* log, int64_t log_cap);

#ifdef __cplusplus
}
#endif
#endif
