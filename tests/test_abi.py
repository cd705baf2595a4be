"""The C-ABI library builds for sm_100a, loads without a GPU and exports exactly the
entry points include/sparkling_b200.h declares (no compute calls here)."""

import os
import re
import subprocess

import pytest

import paper_2108_02991_b200 as spk
from paper_2108_02991_b200 import _build, _native

HEADER = os.path.join(_build.INCLUDE, "sparkling_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(spk_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load()
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, name
    assert lib.spk_version() == 1
    nm = subprocess.run(["nm", "-D", "--defined-only", _build.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r" T (spk_\w+)", nm))
    assert exported == set(names)


def test_sass_is_sm100a_and_uses_blackwell_paths():
    """The N-body kernel is compiled for sm_100a with FFMA2/FADD2 packed f32x2 math, MUFU
    rsqrt and UBLKCP bulk copies (cp.async.bulk)."""
    out = subprocess.run(["cuobjdump", "-sass", _build.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    nb = out[out.index("nbody_kernel"):]
    for mnemonic in ("FFMA2", "FADD2", "MUFU.RSQ", "UBLKCP", "SYNCS"):
        assert mnemonic in nb, mnemonic


def test_public_surface_mirrors_reference_names():
    needed = {"optimize", "step_size", "eval_repulsion", "eval_repulsion_direct",
              "eval_repulsion_tree", "eval_attraction", "precompute_field", "project_pattern",
              "project_shot", "feasibility_residuals", "SamplingPattern", "HardwareSpec",
              "OptimizerConfig", "RepulsionConfig", "ProjectionConfig", "KernelField",
              "TargetDensity", "DensityParams", "discretize", "init_radial", "perturb",
              "upsample_shots", "normalized_limits", "LinearConstraint", "RunTrace"}
    assert needed <= set(spk.__all__)


def test_no_cpu_fallback_without_cuda(monkeypatch):
    import torch

    from paper_2108_02991_b200 import _device

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    import numpy as np
    import pytest

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        spk.eval_repulsion_direct(np.zeros((4, 3)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _device.device()


def test_plain_c_consumer_compiles_and_links():
    """examples/abi_demo.c uses the header as plain C (no C++, no torch types) and links
    against the built library (run on the GPU by tests/test_gpu_abi_demo.py)."""
    import shutil
    import subprocess
    import tempfile

    REPO = os.path.dirname(_build.INCLUDE)
    if shutil.which("gcc") is None or not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"):
        pytest.skip("gcc / CUDA headers not available")
    lib = os.path.join(REPO, "paper_2108_02991_b200", "_lib")
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["gcc", "-O2", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(REPO, "include"),
                        "-I", "/usr/local/cuda/include", os.path.join(REPO, "examples", "abi_demo.c"),
                        "-L", lib, "-lsparkling_b200", "-L", "/usr/local/cuda/lib64", "-lcudart",
                        "-o", os.path.join(d, "abi_demo")], check=True)

