"""The C-ABI library: loads, exports every symbol declared in include/pp200.h and
include/pp200_testing.h, maps errors to codes, and refuses to compute without a GPU (no CPU
fallback)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT, has_cuda, read


def declared_functions(header: str):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pp_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header", ["pp200.h", "pp200_testing.h"])
def test_library_exports_every_declared_symbol(pp, header):
    lib = ctypes.CDLL(pp.LIB_PATH)
    names = declared_functions(header)
    assert len(names) >= 5
    missing = [n for n in names if not hasattr(lib, n)]
    assert missing == []


def test_python_mirror_covers_the_abi(pp):
    for n in declared_functions("pp200.h"):
        assert n in pp.EXPORTED or n in ("pp_homotopy_counts",), n


def test_version_and_limbs(pp):
    assert pp.lib.pp_version().decode().startswith("pp200")
    assert [pp.lib.pp_limbs(p) for p in (0, 1, 2, 7)] == [1, 2, 4, 0]


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(pp):
    f = pp.parse_system(read("cyclic5.sys"))
    g, starts = pp.total_degree_start(f, "d")
    h = pp.make_homotopy(f, g, pp.random_gamma(1), "d")
    with pytest.raises(pp.CudaError):
        pp.track_all(h, starts, lo=0, hi=4)
    import numpy as np

    with pytest.raises(pp.CudaError):
        pp.eval_batch(h, np.zeros((1, 5, 2)), np.zeros((1, 1)))


def test_config_errors_precede_device_work(pp):
    """TrackConfig::validate runs first (tracker.cpp:514): invalid configs fail the same way with
    or without a GPU"""
    f = pp.parse_system(read("cyclic5.sys"))
    g, starts = pp.total_degree_start(f, "d")
    h = pp.make_homotopy(f, g, pp.random_gamma(1), "d")
    cfg = pp.TrackConfig.defaults("d")
    cfg.max_newton = 0
    with pytest.raises(pp.InvalidArgument):
        pp.track_all(h, starts, cfg)


def test_parse_error_positions(pp):
    with pytest.raises(pp.ParseError, match="line 2"):
        pp.parse_system("2;\nx0 + x7;\nx1;")
