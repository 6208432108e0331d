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
