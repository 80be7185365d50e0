"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/sched.h declares, validates configs, and its host-side setup
(sched_thresholds) agrees with the oracle's exact-rational setup."""
import os
import re

import pytest

import workloads as W
from oracle import fluid as fl
from paper_2504_11320_b200 import EXPORTS, SchedError, Scheduler, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sched.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sched_\w+)\(", src, re.M)))


def test_exports_every_declared_symbol():
    L = lib()
    decl = _declared()
    assert set(decl) == set(EXPORTS)
    for name in decl:
        assert hasattr(L, name), name


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2504_11320_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")) or f == "Makefile":
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "des_oracle" not in txt and "liboracle" not in txt, f


@pytest.mark.parametrize("bad", [
    dict(lam=[-1.0]), dict(M=0), dict(d0_s=0.0), dict(l_tab=[[(0, 1)]]),
    dict(lp_tab=[[(5, 0)]]), dict(lp_tab=[[(300, 1)]]), dict(tau_b0=-1),
])
def test_create_validation(bad):
    base = dict(lam=[10.0], l_tab=[W.fixed(4)], lp_tab=[W.fixed(8)], M=256, horizon_s=1.0, seed=1)
    base.update(bad)
    wl = W.Workload("bad", **base)
    with pytest.raises(SchedError) as e:
        Scheduler(wl, W.Policy(W.WAIT), [1])
    assert e.value.code in (-1, -4)


def test_unsatisfiable_and_policy_validation():
    wl = W.Workload("u", [10.0], [W.fixed(100)], [W.fixed(200)], M=256, horizon_s=1, seed=1)
    with pytest.raises(SchedError) as e:
        Scheduler(wl, W.Policy(W.FCFS, B=4))
    assert e.value.code == -4
    ok = W.Workload("o", [10.0], [W.fixed(4)], [W.fixed(8)], M=256, horizon_s=1, seed=1)
    with pytest.raises(SchedError):
        Scheduler(ok, W.Policy(W.FCFS, B=0))
    with pytest.raises(SchedError):
        Scheduler(ok, W.Policy(W.NESTED, seg_end=[4]), [1])      # last segment < max l'
    with pytest.raises(SchedError):
        Scheduler(ok, W.Policy(W.NESTED, seg_end=[4, 4, 8]), [1, 1, 1])  # not increasing
    with pytest.raises(SchedError):
        Scheduler(ok, W.Policy(W.WAIT), [1, 2])                   # count mismatch


@pytest.mark.parametrize("wl", [W.C1, W.C2, W.C3A, W.C3B, W.GOLDEN, W.EX2] + [W.c4(i) for i in range(5)])
def test_fluid_report_matches_oracle(wl):
    s = Scheduler(wl, W.Policy(W.WAIT))
    r = s.thresholds(allow_unstable=True)
    f = fl.fluid(wl)
    assert r["rho"] == pytest.approx(float(f.rho), rel=1e-12)
    assert r["thr_star"] == pytest.approx(float(f.thr_star), rel=1e-12)
    if f.stable:
        assert r["dT_star"] == pytest.approx(float(f.dT), rel=1e-12)
        assert r["M_star"] == pytest.approx(float(f.M_star), rel=1e-12)
        assert r["n_star"] == pytest.approx([float(x) for x in f.n_star], rel=1e-12)


def test_wait_thresholds_match_oracle():
    for wl in [W.C1, W.C1P, W.C2] + [W.c4(i) for i in range(5)]:
        r = Scheduler(wl, W.Policy(W.WAIT)).thresholds()
        assert r["thresholds"] == fl.wait_fluid_integer(wl)
        assert r["M_pi"] == pytest.approx(float(fl.wait_memory(wl, r["thresholds"])), rel=1e-12)
        assert r["feasible"]
    r = Scheduler(W.C2, W.Policy(W.WAIT, B=1024)).thresholds(mode=1)
    assert r["thresholds"] == fl.wait_heuristic(W.C2, 1024)


@pytest.mark.parametrize("wl,seg", [(W.C3A, [20, 40, 80, 160]), (W.C3B, [50 * k for k in range(1, 11)]),
                                    (W.c4(1), [100, 200, 300])])
def test_nested_thresholds_match_oracle(wl, seg):
    r = Scheduler(wl, W.Policy(W.NESTED, seg_end=seg)).thresholds(delta=0.1, budget_B=1357)
    n = fl.nested_strict(wl, seg)
    assert r["thresholds"] == n
    assert r["M_pi"] == pytest.approx(float(fl.nested_memory_exact(wl, seg, n)), rel=1e-12)
    assert r["M_pi_paper"] == pytest.approx(float(fl.nested_memory_paper(wl, seg, n)), rel=1e-12)
    base, queue, hp, tot = fl.thm2_budget(wl, seg, n, 1357, 0.1)
    assert r["budget"] == pytest.approx((base, queue, hp, tot), rel=1e-9)
    for k in range(1, len(n)):
        if n[k] < n[k - 1] and r["theta"][k] > 0:
            tails = fl.nested_tails(wl, seg)
            p = float(tails[k] / tails[k - 1])
            assert r["theta"][k] == pytest.approx(fl.theta(n[k - 1], n[k], p), rel=1e-9)
            assert r["theta"][k] >= r["theta_lb"][k]


def test_random_threshold_agreement():
    import numpy as np
    rng = np.random.default_rng(5)
    for _ in range(30):
        wl = W.random_small(rng)
        wl.M = 10 ** 6
        try:
            ref = fl.wait_fluid_integer(wl, max_k=5000)
        except ValueError:
            continue
        if not fl.fluid(wl).stable:
            continue
        assert Scheduler(wl, W.Policy(W.WAIT)).thresholds()["thresholds"] == ref


def test_ctypes_struct_sizes_match_header():
    """The ctypes mirrors must have the C layout (a short mirror corrupts memory)."""
    import ctypes as C
    import subprocess
    import tempfile
    from paper_2504_11320_b200._lib import LaunchInfo, SchedConfig, ThresholdReport
    src = ('#include <stdio.h>\n#include "sched.h"\nint main(){printf("%zu %zu %zu\\n",'
           'sizeof(sched_config), sizeof(sched_threshold_report), sizeof(sched_launch_info));}')
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "m.c"), "w").write(src)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o",
                               os.path.join(d, "m"), os.path.join(d, "m.c")])
        sizes = [int(x) for x in subprocess.check_output([os.path.join(d, "m")]).split()]
    assert sizes == [C.sizeof(SchedConfig), C.sizeof(ThresholdReport), C.sizeof(LaunchInfo)]


@pytest.mark.parametrize("n", [[7, 7, 7, 5], [11, 11, 10, 7]])
def test_time_varying_check_matches_oracle(n):
    seg = [20, 40, 80, 160]
    wl = W.c3a_time_varying()
    r = Scheduler(wl, W.Policy(W.NESTED, seg_end=seg), n).thresholds()
    dT = fl.Fr(wl.d0_s) + fl.Fr(wl.d1_s) * fl.nested_memory_exact(wl, seg, n)
    sup, pstar, ok = fl.validate_time_varying(wl, seg, n, dT)
    assert r["dT_n"] == pytest.approx(float(dT), rel=1e-12)
    assert r["tv_Lambda_pi"] == pytest.approx(float(sup), rel=1e-9)
    assert r["tv_p_star"][1:] == pytest.approx([float(x) for x in pstar[1:]], rel=1e-12)
    assert r["tv_feasible"] == int(ok)
