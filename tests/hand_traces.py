"""Hand-traced explicit traces with their hand-derived batch logs and rows.

Test helper shared by the CPU pins (tests/test_oracle.py, against the
oracle) and the GPU replays (tests/test_gpu_parity.py, through
sched_run_trace).  Every expected number below was derived by hand from the
algorithm text -- Alg. 2 in the readings of DESIGN.md
§4.4-4.5 -- and is written out in the docstrings; none was produced by
running either simulator.

Log rows are (t_start, |plan|, tokens, n_complete, n_evict, n_new, peak), the
7 int64 of a batch log entry (include/sched.h).
"""
import workloads as W

TPS = 10 ** 12  # ticks per second

# ------------------------------------------------------ Nested WAIT, L = 3
# Segments e = (1, 4, 6): segment 1 = stages 0..1 (stage 0 = the FIFO),
# segment 2 = stages 2..4 (entry stage 2), segment 3 = stages 5..6 (entry
# stage 5) -- reading R8.  Thresholds n = (1, 2, 1).  d0 = 1 s, d1 = 0: every
# iteration takes 1 s.  Prompt P_i (i = 1..10) arrives at 10 (i-1) s, so
# with n_1 = 1 each arrival starts exactly one batch and residents move only
# then.  Prefill lengths l_i = 100 * 2^(i-1) make the token count of a batch
# name its members (sum of l + s over the plan, stages < 100); decode
# lengths l' = (5, 6, 3, 6, 2, 6, 6, 6, 6, 6): P5 completes at an entry
# stage (2), P3 mid-segment (stage 3 of 2..4), P1 at the entry stage 5.
NESTED_SEG = [1, 4, 6]
NESTED_THR = [1, 2, 1]
NESTED_L = [100 * 2 ** i for i in range(10)]
NESTED_LP = [5, 6, 3, 6, 2, 6, 6, 6, 6, 6]
NESTED_T_S = 95.0


def nested_workload(M: int) -> W.Workload:
    return W.Workload("nested-hand", [1.0], [W.fixed(max(NESTED_L))], [W.fixed(6)], M=M,
                      horizon_s=NESTED_T_S, seed=0, d0_s=1.0, d1_s=0.0)


NESTED_POLICY = W.Policy(W.NESTED, seg_end=NESTED_SEG)
NESTED_TRACE = [(10 * i * TPS, 0, NESTED_L[i], NESTED_LP[i]) for i in range(10)]

# Trace A, M = 10^6 (memory never binds).  (s = next stage to run)
#  b1  t=0   FIFO [P1]; entry_2 = 0 < 2 -> k* = 1.  plan: P1 new.        tokens 100
#  b2  t=10  k* = 1.  P1 (s1), P2 new.                           101+200 = 301
#  b3  t=20  entry_2 = #{s=2} = {P1} = 1 < 2 -> k* = 1.  P2 (s1), P3 new;
#            P1 waits at the entry stage with its KV.            201+400 = 601
#            peak = KV 301 + 1 + 400 = 702
#  b4  t=30  entry_2 = {P1,P2} = 2 = n_2 (">=" passes); entry_3 = #{s=5} = 0
#            -> k* = 2.  P3 (s1), P1 P2 (s2), P4 new.  401+102+202+800 = 1505
#  b5  t=40  entry_2 = {P3} = 1 -> k* = 1: P1 P2 at the non-entry stage 3
#            pause.  P4 (s1), P5 new.                          801+1600 = 2401
#            peak = 1505 + 1 + 1600 = 3106
#  b6  t=50  entry_2 = {P3,P4}, entry_3 = 0 -> k* = 2.  P5 (s1), P3 P4 (s2),
#            P1 P2 (s3), P6 new.       1601+402+802+103+203+3200 = 6311
#  b7  t=60  entry_2 = {P5} -> k* = 1.  P6 (s1), P7 new.      3201+6400 = 9601
#            peak = 6311 + 1 + 6400 = 12712
#  b8  t=70  entry_2 = {P5,P6}, entry_3 = 0 -> k* = 2.  P7 (s1), P5 P6 (s2),
#            P3 P4 (s3), P1 P2 (s4), P8 new.  P5 completes at its l' = 2 (an
#            entry stage), P3 at l' = 3 (mid-segment).
#            6401+1602+3202+403+803+104+204+12800 = 25519; peak 12712+7+12800
#            KV after = 104+204+803+3202+6401+12800 = 23514
#  b9  t=80  entry_2 = {P7} = 1 < 2 -> k* = 1, although entry_3 = {P1,P2}
#            = 2 >= n_3: k* is the largest PREFIX (line 1640).  P8 (s1), P9
#            new.                                           12801+25600 = 38401
#            peak = 23514 + 1 + 25600 = 49115
#  b10 t=90  entry_2 = {P7,P8}, entry_3 = {P1,P2} -> k* = 3.  P9 (s1), P7 P8
#            (s2), P6 (s3), P4 (s4), and at the entry stage 5 only
#            min{n_3, Q} = 1 prompt, the OLDEST: P1 (P2 waits).  P1 completes
#            (l' = 5).  P10 new.
#            25601+6402+12802+3203+804+105+51200 = 100117; peak 49115+6+51200
#  then no arrival: stop at T = 95 s with now = 91 s.
NESTED_A_M = 10 ** 6
NESTED_A_LOG = [
    (0, 1, 100, 0, 0, 1, 100),
    (10 * TPS, 2, 301, 0, 0, 1, 301),
    (20 * TPS, 2, 601, 0, 0, 1, 702),
    (30 * TPS, 4, 1505, 0, 0, 1, 1505),
    (40 * TPS, 2, 2401, 0, 0, 1, 3106),
    (50 * TPS, 6, 6311, 0, 0, 1, 6311),
    (60 * TPS, 2, 9601, 0, 0, 1, 12712),
    (70 * TPS, 8, 25519, 2, 0, 1, 25519),
    (80 * TPS, 2, 38401, 0, 0, 1, 49115),
    (90 * TPS, 7, 100117, 1, 0, 1, 100321),
]
# completions: P5 (arrived 40 s) and P3 (20 s) at 71 s, P1 (0 s) at 91 s;
# first tokens: P_i's stage-1 iteration is batch i+1, ending 10 i + 1 s:
# TTFT 11 s for P1..P9; 0-based completion batch indices 7, 7, 9;
# idle = 9 gaps of 9 s between batches; every batch saw one waiting prompt
NESTED_A_ROW = dict(
    arrivals=10, admitted=10, completed=3, completed_after_T=0, completed_tokens=2 + 3 + 5,
    first_tokens=9, batches=10, request_steps=36, prefill_steps=10, evictions=0,
    busy_ticks=10 * TPS, idle_ticks=81 * TPS, lat=(31 + 51 + 91) * TPS, ttft=9 * 11 * TPS,
    completion_batch_idx=7 + 7 + 9, max_kv_peak=100321, final_waiting=0, final_resident=7,
    status=0, now_stop=91 * TPS, sum_waiting=10)

# Trace B: the same arrivals with M = 100,000, so paused residents' KV makes
# the memory check bind (Eq. memory_constraint):
#  b1..b9 as in trace A (peaks <= 49115).
#  b10 t=90  plan as in A, peak 100321 > M: LIFO evicts the LAST ADMITTED
#            resident, P9 (s1, in the plan): peak -= (25600+1-1) + 1 -> 74720;
#            P9 re-enters the FIFO tail behind P10 (R7), its first token not
#            yet emitted.  tokens 100117 - 25601 = 74516, |plan| 6.
#            KV after = 204+804+3203+6402+12802+51200 = 74615
#  b11 t=91  FIFO [P9]: entry_2 = 0 -> k* = 1.  P10 (s1) + P9 new: peak
#            74615+1+25600 = 100216 > M -> evict P10 (51200+1) -> 49015.
#            plan = P9 alone, tokens 25600.
#  b12 t=92  FIFO [P10]: P9 (s1) + P10 new: 49015+1+51200 = 100216 -> evict
#            P9 -> 74615; plan = P10, tokens 51200.
#  b13, b14 repeat b11, b12 (the eviction cascade); b14 ends at T = 95 s.
NESTED_B_M = 100_000
NESTED_B_LOG = NESTED_A_LOG[:9] + [
    (90 * TPS, 6, 74516, 1, 1, 1, 74720),
    (91 * TPS, 1, 25600, 0, 1, 1, 49015),
    (92 * TPS, 1, 51200, 0, 1, 1, 74615),
    (93 * TPS, 1, 25600, 0, 1, 1, 49015),
    (94 * TPS, 1, 51200, 0, 1, 1, 74615),
]
# first tokens: P1..P8 only (P9 and P10 never run stage 1); at stop P9 waits,
# P2 P4 P6 P7 P8 P10 are resident
NESTED_B_ROW = dict(
    arrivals=10, admitted=14, completed=3, completed_after_T=0, completed_tokens=10,
    first_tokens=8, batches=14, request_steps=29 + 6 + 4, prefill_steps=14, evictions=5,
    busy_ticks=14 * TPS, idle_ticks=81 * TPS, lat=(31 + 51 + 91) * TPS, ttft=8 * 11 * TPS,
    completion_batch_idx=7 + 7 + 9, max_kv_peak=74720, final_waiting=1, final_resident=6,
    status=0, now_stop=95 * TPS, sum_waiting=14)

# ------------------------------------ FCFS prefill-token budget (tok_budget)
# FCFS new-first (reading R15; the paper's baselines carry "fixed limits on
# the total number of tokens"), B = 100, tok_budget = 5,
# M = 100, d0 = 1 s, d1 = 0, l' = 1 for all.  Arrivals (tick, l):
# A 0 s l2, B 0 s l3, C 0 s l1, D 0.5 s l4, E 1.5 s l5, G 2.5 s l4,
# H 2.6 s l2, I 2.7 s l1.
#  b1 t=0  FIFO [A,B,C]: A (2 <= 5), B (2+3 = 5 <= 5: equality admits), C
#          (6 > 5) stops.                          tokens 5, peak 0+0+5 = 5
#  b2 t=1  A B (s1) complete; FIFO [C,D]: C (1), D (1+4 = 5).
#          tokens (2+1)+(3+1)+1+4 = 12, peak 5+2+5 = 12
#  b3 t=2  C D complete; FIFO [E]: 5 <= 5.        tokens 2+5+5 = 12, peak 5+2+5
#  b4 t=3  E completes; FIFO [G,H,I]: G (4), H (4+2 > 5) stops -- I (l = 1)
#          is not skipped ahead.                  tokens 6+4 = 10, peak 5+1+4
#  b5 t=4  G completes; FIFO [H,I]: 2 + 1 = 3.    tokens 5+3 = 8, peak 4+1+3
#  b6 t=5  H I complete.                           tokens 3+2 = 5, peak 3+2
FCFS_BUDGET = 5
FCFS_TRACE = [(0, 0, 2, 1), (0, 0, 3, 1), (0, 0, 1, 1), (TPS // 2, 0, 4, 1),
              (3 * TPS // 2, 0, 5, 1), (5 * TPS // 2, 0, 4, 1), (26 * TPS // 10, 0, 2, 1),
              (27 * TPS // 10, 0, 1, 1)]
FCFS_LOG = [
    (0, 2, 5, 0, 0, 2, 5),
    (1 * TPS, 4, 12, 2, 0, 2, 12),
    (2 * TPS, 3, 12, 2, 0, 1, 12),
    (3 * TPS, 2, 10, 1, 0, 1, 10),
    (4 * TPS, 3, 8, 1, 0, 2, 8),
    (5 * TPS, 2, 5, 2, 0, 0, 5),
]
# latencies (= TTFT, l' = 1): A 2, B 2, C 3, D 2.5, E 2.5, G 2.5, H 3.4, I 3.3 s
FCFS_ROW = dict(
    arrivals=8, admitted=8, completed=8, completed_tokens=8, first_tokens=8, batches=6,
    request_steps=16, evictions=0, lat=212 * TPS // 10, ttft=212 * TPS // 10,
    completion_batch_idx=2 * 1 + 2 * 2 + 3 + 4 + 2 * 5, max_kv_peak=12, final_waiting=0,
    final_resident=0, status=0)


def fcfs_workload() -> W.Workload:
    return W.Workload("fcfs-budget", [1.0], [W.fixed(5)], [W.fixed(1)], M=100, horizon_s=10.0,
                      seed=0, d0_s=1.0, d1_s=0.0)


FCFS_POLICY = W.Policy(W.FCFS, B=100, tok_budget=FCFS_BUDGET)


def row_matches(rows, i, expect, F, u128):
    """Compare the expected fields (128-bit sums by name) of replication i."""
    bad = {}
    for k, v in expect.items():
        got = u128(rows, k)[i] if k in ("lat", "ttft", "soj") else int(rows[F[k], i])
        if got != v:
            bad[k] = (got, v)
    return bad
