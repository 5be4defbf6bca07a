"""CPU: the C-ABI library loads, exports every entry point include/rl_b200.h declares, and
fails loudly (RL_NO_DEVICE) instead of falling back to the CPU when no GPU is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "rl_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rl_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("rl_gaussian_matrix", "rl_genp_factor", "rl_genp_solve", "rl_randomized_genp",
              "rl_randomized_genp_batched", "rl_approx_basis", "rl_qr_positive", "rl_numerical_rank",
              "rl_dev_range_finder", "rl_matmul", "rl_circ_mul"):
        assert s in syms


def test_library_exports_every_declared_symbol(rl):
    lib = ctypes.CDLL(rl.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", rl.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (rl_[a-z0-9_]+)", nm))
    assert set(declared_symbols()) <= exported


def test_cpp_dropin_library_exports_reference_api(rl):
    so = os.path.join(ROOT, "paper_1212_4560_b200", "lib", "librandla_b200.so")
    if not os.path.exists(so):
        pytest.skip("C++ drop-in not built")
    nm = subprocess.run(["nm", "-DC", "--defined-only", so], capture_output=True, text=True).stdout
    for sym in ("randla::genp::randomized_genp", "randla::genp::genp_factor", "randla::genp::genp_solve",
                "randla::rnd::gaussian_matrix", "randla::lowrank::approx_basis", "randla::dense::qr_positive",
                "randla::Matrix::multiply", "randla::lowrank::nrank_search", "randla::lowrank::extremal_sv_estimate",
                "randla::lowrank::cond_probe", "randla::lowrank::power_transform", "randla::lowrank::proto_lowrank",
                "randla::structured::fft", "randla::structured::toeplitz_mul", "randla::structured::multiply_matrix"):
        assert sym in nm, sym


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(rl):
    with pytest.raises(rl.NoDevice):
        rl.multiply(np.eye(3), np.eye(3))
    with pytest.raises(rl.NoDevice):
        rl.genp_factor(np.eye(4))


def test_argument_validation_matches_reference(rl):
    # random_gen.cpp:73-74: sigma <= 0 -> InvalidArgument (checked before any device work)
    with pytest.raises(rl.InvalidArgument):
        rl.gaussian_matrix(2, 2, 0.0, 0.0, rl.RngStream(11, 0))
    with pytest.raises(rl.DimensionMismatch):
        rl.genp_factor(np.zeros((2, 3)))
    with pytest.raises(rl.DimensionMismatch):
        rl.randomized_genp(np.eye(3), np.ones(4), rl.MultiplierKind(), rl.MulSide.RIGHT, 0, rl.RngStream())
