// sim_internal.h -- host <-> device parameter block of libsched (not part of
// the public C ABI; see include/sched.h for that).
#pragma once
#include <stdint.h>

namespace waitsim {

constexpr int kMaxClasses = 32;
constexpr int kMaxSegments = 32;
constexpr int kLanes = 32;
constexpr uint32_t kRestartChunk = 64;    // restart-FIFO entries per pool chunk
constexpr uint32_t kNoChunk = 0xFFFFFFFFu;

struct ClassParam {
  double gap_scale;        // 1e12 / lambda (ticks per unit exponential); 0 = no arrivals
  uint32_t l_off, l_n;     // CDF table slice (thresholds u64 [n], values u16 [n]);
  uint32_t lp_off, lp_n;   // n in bits 0-23, guide-table log2 size in bits 24-27
  uint32_t l_goff, lp_goff;  // guide-table slices (u16 [2^lg]) in cdf_guide
  uint32_t rf_off, rf_n;   // time-varying rate pieces (rf_n = 0: homogeneous)
};

// Everything one launch needs, passed by value (lives in the constant bank).
struct DevParams {
  int32_t K;
  int32_t policy;          // SCHED_WAIT / SCHED_NESTED / SCHED_FCFS
  int32_t n_rings;         // restart rings per replication (WAIT: K, else 1)
  int32_t n_seg;
  int64_t d0_t, d1_t, T_t, M;
  int64_t b0;              // piecewise-linear iteration time threshold (tokens; 0 = linear)
  uint32_t thr[kMaxSegments];      // WAIT: per class, NESTED: per segment
  uint32_t B, tok_budget;
  uint32_t Rc;             // resident capacity per replication (class-ring engine: staging capacity)
  // class-ring engine: fixed-length classes under WAIT /
  // FCFS keep their residents in per-class rings in admission order; stage
  // = class clock - admission clock, so a batch touches only the members
  // that complete, emit a first token or are admitted
  uint32_t ring_engine;
  uint32_t spare;                  // staging slots beyond Rc for eviction-round victims (8 or 32)
  uint32_t rcap[kMaxClasses];      // ring capacity (records) of class c
  uint32_t roff[kMaxClasses];      // first record of ring c in this warp's slot of ring_g
  uint8_t* ring_log;               // [warps of the launch][2^16] class of each admission, in order
  void* ring_g;                    // [warps of the launch][ring_stride] ring records (global: read
  uint32_t ring_stride;            //   only by evictions and at the end of a replication)
  uint32_t ccoff[kMaxClasses];     // cohort-count ring of class c (l'_c + 1 slots, shared memory)
  uint32_t ccsize;
  uint32_t fl[kMaxClasses];        // fixed l | l' << 16 of class c
  // segment engine (NESTED): residents in one admission-
  // ordered array that is sorted by stage, segment k a contiguous range;
  // per segment the entry stage b_k = e_{k-1}+1 (b_0 = 0: the FIFO) and the
  // number of non-entry stages W_k = e_k - b_k; completion histograms
  // (W_k buckets from hoff[k]) and cohort rings (W_k+1 slots from coff[k])
  uint32_t seg_engine;
  uint32_t seg_cap;                // resident array capacity (records)
  uint32_t seg_b[kMaxSegments], seg_w[kMaxSegments];
  uint32_t hoff[kMaxSegments], coff[kMaxSegments];
  uint32_t hsize, csize;           // total buckets / cohort slots
  int64_t* seg_a;                  // [warps of the launch][seg_cap] arrival ticks of the residents (device)
  uint32_t warp_smem;      // bytes of shared memory per warp
  uint32_t off_csum, off_rr;       // layout offsets that depend on Rc / tv (warp_smem_bytes)
  uint64_t seed;
  uint64_t rep_begin;      // global index of local replication 0
  uint32_t n_reps;
  uint32_t trace_mode;
  ClassParam cls[kMaxClasses];
  const uint64_t* cdf_thr; // device
  const uint16_t* cdf_val; // device
  const uint16_t* cdf_guide; // device: per table, guide[j] = first index whose threshold exceeds j 2^(32-lg)
  const uint8_t* stage_info; // NESTED: stage -> segment | entry<<7 (device)
  // time-varying classes: per piece start tick, integrated
  // rate at the start (operational ticks, 2^-32 expected arrivals), tick
  // scale 1e12 / (lambda 2^32) (0 = zero rate)
  const int64_t* rf_B;
  const int64_t* rf_Lam;
  const double* rf_scale;
  uint32_t tv_any;         // some class is time-varying: operational-time windows exist
  // explicit traces (trace_mode): per (rep, class) slices of t / l / lp
  const int64_t* tr_t;
  const uint16_t* tr_l;
  const uint16_t* tr_lp;
  const int64_t* tr_off;   // [n_reps*K + 1]
  // restart FIFOs (evicted prompts): linked lists of
  // kRestartChunk-entry chunks from one device-wide pool shared by every
  // replication of the launch; free chunks on a lock-free
  // stack (head = tag << 32 | chunk), never-used ones from a bump counter
  int64_t* pool_a;         // [chunks * kRestartChunk] original arrival tick
  int64_t* pool_e;         // eviction tick
  uint32_t* pool_llp;      // l | l' << 16 | first-token << 31 (ring engine: class | ft << 31)
  uint32_t* pool_next;     // [chunks] next chunk of a FIFO / of the free stack
  unsigned long long* pool_free;  // free-stack head
  uint32_t* pool_bump;     // chunks handed out so far (high-water mark)
  uint32_t pool_chunks;
  uint32_t* pool_stash;    // [warp slots][n_rings] x {count, 11 chunks}: per-slot free chunks (persist)
  uint32_t stash_lim;      // chunks a stash may hold (<= 11; 0 for pools too small to share out)
  uint32_t bump_n;         // never-used chunks taken per bump allocation (<= stash_lim + 1)
  uint32_t* work_counter;  // this launch's replication counter
  uint32_t* status_mask;   // handle's sticky status: bit s = a replication ended with status s
  // speculative capacity: the main launch runs with a small resident
  // capacity; replications that overflow it are appended to retry_list and
  // re-run from scratch by a fallback launch with the safe capacity
  uint32_t* retry_list;    // [n_reps] (may be null: no fallback)
  uint32_t* retry_count;
  uint32_t fallback;       // 1: this launch processes retry_list
  // outputs
  uint64_t* out;           // field-major [SCHED_NF][n_reps]
  int64_t* log;            // trace mode: 7 int64 per batch of replication 0
  int64_t log_cap;
  int64_t* log_n;
};

// Shared-memory layout of one warp (byte offsets; the kernel's WarpSim
// constructor lays it out in this order): per class a generated and a
// private admission window (32 x (t, l, l') each), 32 staged restart ticks,
// counters / rank cursors / snapshot, WarpStats, eviction scratch -- all
// offsets that depend on the class count only (immediates in the kernels
// specialised on K) -- then the operational-time windows (time-varying
// rates), Nested chunk summaries, residents / staged admissions (Rc x 16 B),
// class-ring cohort counts or the segment engine's array, histograms and
// cohort rings, and the restart-FIFO cursors + chunk stash at the end.
inline uint32_t a16(uint32_t x) { return (x + 15u) & ~15u; }
inline uint32_t layout_off_csum(int K, bool tv) {
  return 768u * (uint32_t)K + 1280u + (tv ? 512u * (uint32_t)K : 0u);
}
inline uint32_t layout_off_rr(uint32_t Rc, int K, bool tv, bool nested) {
  return layout_off_csum(K, tv) + (nested ? a16((Rc + 31u) / 32u) : 0u);
}
inline uint32_t warp_smem_bytes(uint32_t Rc, int K, bool tv = false, bool ring = false, bool nested = false,
                                uint32_t n_rings = 1, uint32_t seg_cap = 0, uint32_t hsize = 0,
                                uint32_t csize = 0, uint32_t extra = 0) {
  uint32_t b = layout_off_rr(Rc, K, tv, nested) + Rc * 16u;
  if (ring) b += a16(extra);                                    // cohort counts
  if (seg_cap) b += seg_cap * 8u + a16(hsize * 12u + csize * 8u);  // segment engine
  return b + n_rings * 80u;  // restart FIFO cursors (head, head index, tail, tail index),
                             // chunk stash (count + 11), successors of head and tail
}

cudaError_t launch_sim(const DevParams& p, int grid, int block, size_t smem, cudaStream_t s);
// sched_aggregate's kernel (aggregate.cu): one 1024-thread block
cudaError_t launch_aggregate(const uint64_t* rows, uint64_t ld, uint32_t n, double horizon_s, int64_t* out_i,
                             double* out_f, cudaStream_t s);
// blocks per SM of the kernel that launch_sim runs for (policy, engine, K)
cudaError_t sim_occupancy(int policy, int trace, int block, size_t smem, int* blocks_per_sm, int ring = 0,
                          int K = 0);

}  // namespace waitsim
