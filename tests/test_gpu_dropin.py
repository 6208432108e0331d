"""The drop-in boundary exercised from the reference side: the reference's own acceptance suite
(proj/tests/acceptance.cpp, unmodified) linked with the C++ shim paper_1505_00383_b200/shim/
tracker_b200.cpp, so every polypath::track_all<R> call of the suite runs on the GPU through
libpp200.so (built by oracle/Makefile as oracle/_ref/acceptance_b200).

Criteria 7 (closed form end to end, d and qd), 8 (cyclic-5 dd desk scale: 70 converged, failures
annotated diverged, gamma seeds 101-103 and batch widths 1/16/64 agree) and 10 (quality up, d vs
dd) call track_all; the others exercise host code and pass as on the CPU."""

import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def run_acceptance(extra_env=None):
    if not os.path.exists(ACC):
        pytest.fail("oracle/_ref/acceptance_b200 is not built (oracle/Makefile target `acceptance`)")
    env = dict(os.environ, POLYPATH_B200_TRACE="1", **(extra_env or {}))
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=900, env=env)
    lines = {int(m.group(2)): (m.group(1), m.group(0)) for m in
             re.finditer(r"\[(PASS|FAIL)\] criterion\s+(\d+):.*", r.stdout)}
    return r, lines


def test_reference_acceptance_suite_through_the_gpu():
    r, lines = run_acceptance()
    print(r.stdout)
    print(r.stderr[-3000:])
    # the track_all calls went through the shim onto the device
    calls = re.findall(r"\[pp200\] track_all<(\w+)>: (\d+) paths on (\d+) B200", r.stderr)
    assert {c[0] for c in calls} >= {"d", "dd", "qd"}, r.stderr[-2000:]
    for k in (7, 8, 10):
        assert k in lines and lines[k][0] == "PASS", lines.get(k)
    assert r.returncode == 0 and "all criteria passed" in r.stdout, r.stdout


def test_acceptance_criteria_4_and_6_on_the_device():
    """criteria 4 (AD against finite differences and the symbolic dd oracle, 100 random systems)
    and 6 (conditioned m x n least squares: orthogonality < 50 n u, solution against QD normal
    equations) with every evaluation / factorisation on the device (oracle/gpu_criteria.cpp), and
    the device results bit for bit equal to the reference library's"""
    exe = os.path.join(ROOT, "oracle", "_ref", "gpu_criteria")
    if not os.path.exists(exe):
        pytest.fail("oracle/_ref/gpu_criteria is not built (oracle/Makefile target `acceptance`)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    assert "[PASS] gpu criterion  4" in r.stdout and "[PASS] gpu criterion  6" in r.stdout
    assert r.stdout.count("bitwise equal to the reference: yes") == 2


@pytest.mark.parametrize("name,prec,cfg", [("cyclic5_d", "d", []), ("cyclic5_dd", "dd", []),
                                          ("cyclic5_d_tight", "d", ["2", "0.1", "40"])])
def test_progress_sink_through_the_shim(name, prec, cfg):
    """a reference-API caller passes a ProgressSink to polypath::track_all<R>; through the shim the
    device's events reach it, and per path they equal the reference sink's (field for field)"""
    import numpy as np

    from conftest import golden

    exe = os.path.join(ROOT, "oracle", "_ref", "shim_events")
    if not os.path.exists(exe):
        pytest.fail("oracle/_ref/shim_events is not built (oracle/Makefile target `acceptance`)")
    r = subprocess.run([exe, os.path.join(ROOT, "tests", "data", "cyclic5.sys"), prec, *cfg], capture_output=True,
                       text=True, timeout=600, env=dict(os.environ, POLYPATH_B200_TRACE="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    assert "[pp200] track_all" in r.stderr
    rows = [ln.split() for ln in r.stdout.splitlines()]
    got = [(int(a), int(b, 16), int(c, 16), int(d), int(e), int(f)) for a, b, c, d, e, f in rows]
    want = golden(f"events_{name}")["events"]
    assert len(got) == len(want)
    order_g = sorted(range(len(got)), key=lambda i: (got[i][0], i))
    order_w = np.argsort(want["path_id"], kind="stable")
    for ig, iw in zip(order_g, order_w):
        w = want[iw]
        assert got[ig][0] == int(w["path_id"])
        assert got[ig][1] == int(np.float64(w["t"]).view(np.uint64))
        assert got[ig][2] == int(np.float64(w["h"]).view(np.uint64))
        assert (got[ig][3], got[ig][4], got[ig][5]) == (int(w["newton_iters"]), int(w["status"]), int(w["accepted"]))
