"""The reference-side drop-in, checked without a GPU: the reference's acceptance suite linked with
paper_1505_00383_b200/shim/tracker_b200.cpp resolves polypath::track_all<R> to the shim's strong
definitions (not to tracker.o's weak template instantiations), and with no CUDA device it fails
loudly instead of falling back to the CPU tracker."""

import os
import shutil
import subprocess

import pytest

from conftest import ROOT, has_cuda

ACC = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")
SHIM_O = os.path.join(ROOT, "oracle", "_ref", "tracker_b200.o")
MANGLED = ["_ZN8polypath9track_allIdEENS_11SolutionSetIT_EERKNS_16HomotopyInstanceIS2_EERKNS_9StartDataIS2_EERKNS_11Track"
           "ConfigEPSt8functionIFvRKNS_9StepEventEEEmm",
           "_ZN8polypath9track_allINS_2DDEEENS_11SolutionSetIT_EERKNS_16HomotopyInstanceIS3_EERKNS_9StartDataIS3_EERKNS_11"
           "TrackConfigEPSt8functionIFvRKNS_9StepEventEEEmm",
           "_ZN8polypath9track_allINS_2QDEEENS_11SolutionSetIT_EERKNS_16HomotopyInstanceIS3_EERKNS_9StartDataIS3_EERKNS_11"
           "TrackConfigEPSt8functionIFvRKNS_9StepEventEEEmm"]


def nm_symbols(path):
    out = subprocess.run(["nm", path], capture_output=True, text=True, check=True).stdout
    return {ln.split()[-1]: ln.split()[-2] for ln in out.splitlines() if len(ln.split()) >= 2}


@pytest.mark.skipif(not os.path.exists(ACC) or shutil.which("nm") is None, reason="acceptance_b200 not built")
def test_shim_definitions_win_the_link():
    shim = nm_symbols(SHIM_O)
    exe = nm_symbols(ACC)
    for m in MANGLED:
        assert shim.get(m) == "T", m          # strong definition in the shim object
        assert exe.get(m) == "T", m           # and the linked executable carries a strong one
    # the executable's track_all<double> is the shim's: its code calls into libpp200
    out = subprocess.run(["nm", "-u", ACC], capture_output=True, text=True, check=True).stdout
    assert "pp_track_all_ex" in out and "pp_system_from_terms" in out


@pytest.mark.skipif(not os.path.exists(ACC) or has_cuda(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_through_the_shim():
    r = subprocess.run([ACC], capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
    assert "no CUDA device" in r.stderr + r.stdout
    # the criteria before the first track_all pass on the host; criterion 7 is where it stops
    assert "[PASS] criterion  6" in r.stdout and "criterion  7" not in r.stdout
