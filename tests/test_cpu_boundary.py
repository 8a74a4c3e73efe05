"""CPU-only checks of the boundary: the C-ABI library loads and exports every
symbol include/rrs_b200.h declares, the Python API validates like the
reference, and without a GPU the product fails loudly (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, cuda_available

import paper_2506_08262_b200 as rrs
from paper_2506_08262_b200 import _lib

HEADER = os.path.join(ROOT, "include", "rrs_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(rrs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    L = rrs.load_library()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert {name for name, _, _ in _lib.SIGNATURES} == set(syms)
    assert L.rrs_abi_version() == 3


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # TMA bulk copies in the contraction kernel
    assert "contract_kernel" in sass


@pytest.mark.skipif(cuda_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly():
    with pytest.raises(RuntimeError, match="no CUDA device"):
        rrs.Engine(0)
    data = rrs.Dataset(np.random.default_rng(0).standard_normal((20, 3)))
    cfg = rrs.RrsConfig(total_directions=20, refinements=2, notion="halfspace")
    with pytest.raises(RuntimeError):
        rrs.depth_batch([data.x[0]], data, cfg)


def test_rrs_config_validation_messages():
    # optimizer.py:54-62
    with pytest.raises(ValueError, match="need total_directions >= refinements >= 1"):
        rrs.RrsConfig(total_directions=3, refinements=5)
    with pytest.raises(ValueError, match="shrink factor"):
        rrs.RrsConfig(shrink=1.0)
    with pytest.raises(ValueError, match="unknown depth notion"):
        rrs.RrsConfig(notion="mystery")
    with pytest.raises(ValueError, match="unknown pole update mode"):
        rrs.RrsConfig(pole_update="sometimes")
    cfg = rrs.RrsConfig(total_directions=20_000, refinements=20)
    assert cfg.directions_per_refinement == 1000
    assert rrs.RrsConfig(total_directions=1001, refinements=10).directions_per_refinement == 101
    assert cfg.epsilons()[3] == (np.pi / 2) * 0.9**3


def test_dataset_validation():
    with pytest.raises(ValueError, match="non-empty"):
        rrs.Dataset(np.empty((0, 3)))
    with pytest.raises(ValueError, match="non-finite"):
        rrs.Dataset([[1.0, np.nan]])
    assert rrs.Dataset([1.0, 2.0]).x.shape == (1, 2)


def test_dimension_mismatch_messages():
    data = rrs.Dataset(np.ones((5, 3)))
    cfg = rrs.RrsConfig(total_directions=20, refinements=2, notion="halfspace")
    with pytest.raises(rrs.DimensionMismatch, match="query dimension 2 does not match data dimension 3"):
        rrs.refined_random_search(np.ones(2), data, cfg)
    with pytest.raises(ValueError, match="query 1 has dimension 2, expected 3"):
        rrs.depth_batch([np.ones(3), np.ones(2)], data, cfg)
    with pytest.raises(rrs.DimensionMismatch):
        rrs.evaluate_directions(np.ones(3), data, np.ones((4, 2)), "halfspace", rrs.ParallelConfig())


def test_pole_update_rule():
    pole = np.array([1.0, 0.0])
    assert rrs.pole_update_rule((0.2, pole), (0.3, np.array([0.0, 1.0])))[1] is pole
    assert rrs.pole_update_rule((0.2, pole), (0.2, np.array([0.0, 1.0])))[1] is pole
    new = np.array([0.0, 1.0])
    assert rrs.pole_update_rule((0.2, pole), (0.1, new)) == (0.1, new)


def test_cap_spec_validation():
    with pytest.raises(ValueError):
        rrs.Pole(np.array([1.0, 1.0]))
    with pytest.raises(ValueError):
        rrs.CapSpec(pole=rrs.Pole(np.array([1.0, 0.0])), epsilon=0.0)


def test_synthetic_matches_reference_generator(golden):
    from paper_2506_08262_b200.synthetic import toeplitz_gaussian

    assert np.array_equal(toeplitz_gaussian(5, 1000, seed=0), golden["c1_x"])
    assert np.array_equal(toeplitz_gaussian(50, 2000, seed=0), golden["c4mini_x"])


def test_header_documents_reference_interfaces():
    text = open(HEADER).read()
    for ref in ("optimizer.py:254-279", "optimizer.py:98-142", "directions.py:192-204",
                "philox.py:27-65", "projection.py:44-75"):
        assert ref in text


def test_packed_layouts_host_check(tmp_path):
    """kernels.h's packed K layouts (tc_layout with 64-coordinate slices, the
    six-product tc6_layout) checked on the host: compiled with g++ against the
    CUDA headers from tests/cpp/layout_check.cpp (no GPU)."""
    import shutil
    import subprocess

    cxx = shutil.which("g++")
    inc = "/usr/local/cuda/include"
    if cxx is None or not os.path.isdir(inc):
        pytest.skip("g++ or the CUDA headers are not available")
    here = os.path.dirname(os.path.abspath(__file__))
    exe = tmp_path / "layout_check"
    subprocess.run([cxx, "-std=c++17", "-O1", f"-I{inc}", "-I" + os.path.join(here, "..", "paper_2506_08262_b200", "csrc"),
                    os.path.join(here, "cpp", "layout_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout
