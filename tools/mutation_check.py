"""Mutation check of the oracle's pins (dev tool, not product code).

Each mutation below is a plausible slip in oracle/des_oracle.cpp (the five
VERDICT r1 listed plus two more); the CPU suite (`pytest -m "not gpu"`) must
fail on every one.  Each runs in a scratch copy of the repo under /tmp.

    python tools/mutation_check.py [-j 4]
"""
import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "oracle/des_oracle.cpp"

MUTATIONS = {
    "nested_entry_stage_off_by_one": ("const int entry = S.seg_end[k - 1] + 1;",
                                      "const int entry = S.seg_end[k - 1];"),
    "nested_kstar_strict": ("if (cnt >= S.thr[k]) kstar = k; else break;",
                            "if (cnt > S.thr[k]) kstar = k; else break;"),
    "nested_kstar_not_prefix": ("if (cnt >= S.thr[k]) kstar = k; else break;",
                                "if (cnt >= S.thr[k]) kstar = k;"),
    "nested_newest_first": ("""      for (size_t i = 0; i < res.size(); ++i) {
        const int k = segment_of(res[i].s);""", """      for (size_t i = res.size(); i-- > 0;) {
        const int k = segment_of(res[i].s);"""),
    "nested_take_all_per_stage": ("if (taken < S.thr[k]) { P.res_in[i] = 1; ++taken; }",
                                  "{ P.res_in[i] = 1; ++taken; }"),
    "fcfs_budget_ge": ("if (S.tok_budget != 0 && (uint64_t)(new_l + p.l) > S.tok_budget) break;",
                       "if (S.tok_budget != 0 && (uint64_t)(new_l + p.l) >= S.tok_budget) break;"),
    "wait_newest_first": ("""      for (size_t i = 0; i < res.size(); ++i) {
        const Prompt& p = res[i];
        if (!inQ[p.c]) continue;""", """      for (size_t i = res.size(); i-- > 0;) {
        const Prompt& p = res[i];
        if (!inQ[p.c]) continue;"""),
    "sum_waiting_after_eviction": ("""      uint64_t waiting = 0;
      for (auto& q : fifo) waiting += q.size();
      if (go) {""", """      uint64_t waiting = 0;
      if (go) {"""),
}


# equivalent mutants: by invariant P14 (checked at every decision epoch, a
# violation sets status 3) no WAIT stage s >= 1 ever holds more than n_j, so
# min{n_j, n_js} takes every prompt there and the selection order cannot
# matter; these must SURVIVE (a kill would mean P14 is broken)
EQUIVALENT = {"wait_newest_first"}


def run(name):
    old, new = MUTATIONS[name]
    d = f"/tmp/mut_{name}"
    shutil.rmtree(d, ignore_errors=True)
    shutil.copytree(ROOT, d, ignore=shutil.ignore_patterns(".git", "gpurun_out", "profiles", "liboracle.so", "libsched_*.so"))
    p = os.path.join(d, SRC)
    s = open(p).read()
    assert s.count(old) == 1, f"{name}: pattern not unique"
    open(p, "w").write(s.replace(old, new))
    if name == "sum_waiting_after_eviction":  # count the queue after eviction, before execute
        s = open(p).read()
        s = s.replace("      sum_waiting += waiting;", "      for (auto& q : fifo) waiting += q.size();\n"
                      "      sum_waiting += waiting;")
        open(p, "w").write(s)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-x", "-q", "-m", "not gpu",
                        "-p", "no:cacheprovider"], cwd=d, capture_output=True, text=True)
    tail = [ln for ln in r.stdout.splitlines() if "passed" in ln or "failed" in ln]
    first = [ln for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
    shutil.rmtree(d, ignore_errors=True)
    return name, r.returncode, (first[:1] or tail[-1:])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=4)
    args = ap.parse_args()
    survived = []
    with cf.ThreadPoolExecutor(args.j) as ex:
        for name, rc, info in ex.map(run, MUTATIONS):
            eq = name in EQUIVALENT
            print(f"{'killed ' if rc else 'SURVIVED'} {name}{' (equivalent mutant)' if eq else ''}: "
                  f"{info}", flush=True)
            if (rc == 0) != eq:
                survived.append(name)
    sys.exit(1 if survived else 0)
