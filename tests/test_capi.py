"""CPU: the C-ABI library builds for sm_100a, loads, and exports exactly what include/ declares.

No compute entry point is called here (there is no GPU in the build container)."""

import ctypes
import math
import re
import subprocess

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_2301_08897_b200 import _capi, build

    build.build()
    return _capi.load()


def header_symbols():
    text = (ROOT / "include" / "scadles_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported_and_bound(lib):
    from paper_2301_08897_b200 import _capi

    syms = header_symbols()
    assert len(syms) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sg_[a-z0-9_]+)", out))
    for s in syms:
        assert s in exported, s
        assert s in _capi.SIGNATURES, s
        getattr(lib, s)
    assert set(_capi.SIGNATURES) == set(syms)


def test_sass_is_sm100a_with_tma(lib):
    from paper_2301_08897_b200 import _capi

    out = subprocess.run(["cuobjdump", "-lelf", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass  # cp.async.bulk (TMA) in the main pass
    assert "SYNCS" in sass   # mbarrier completion


def test_abi_version_and_status(lib):
    assert lib.sg_abi_version() == 2
    assert lib.sg_status_string(0) == b"ok"
    assert lib.sg_status_string(-1) == b"invalid argument"
    assert lib.sg_status_string(-3).startswith(b"workspace")


def test_topk_count_matches_reference_expression(lib):
    for cr in (0.001, 0.01, 0.1, 0.25, 0.3, 0.5, 0.9, 1.0):
        for D in list(range(1, 2000)) + [60_192_808, 143_667_240, 10**9]:
            assert lib.sg_topk_count(D, cr) == max(1, math.ceil(cr * D - 1e-12))
    assert lib.sg_topk_count(10, 0.0) == -1
    assert lib.sg_topk_count(10, 1.5) == -1


def test_invalid_arguments_rejected_without_a_gpu(lib):
    # argument validation happens before any CUDA call
    assert lib.sg_topk_gate_f32(None, 1, 10, 10, 1, None, None, None, None, None, None, None, None, 0, None) == -1
    w = (ctypes.c_double * 2)(0.5, 0.5)
    assert lib.sg_weighted_aggregate_f32(0, w, None, None, 0, None, None, None, None, 10, None, None, None,
                                         0.0, 0.0, 0.0, 0, -1, None, 0, None) == -1
    assert lib.sg_sgd_momentum_f32(None, None, None, 10, 0.1, 0.9, 0.0, 1, None) == -1
    assert lib.sg_gather_batch_f64(None, None, None, 4, None, 1, None, None, None) == -1
    assert lib.sg_topk_workspace_bytes_f32(1, 10, 11) == 0  # m > dim
    assert lib.sg_aggregate_workspace_bytes(8, 60_192_808) == 4 * 8 * (14696 + 1)


def test_python_errors_mirror_reference():
    from paper_2301_08897_b200 import comm

    with pytest.raises(ValueError, match="compression ratio"):
        comm.topk_count(10, 0.0)
    with pytest.raises(ValueError, match="compression ratio"):
        comm.CompressionState(cr=1.5, delta=0.1)
    with pytest.raises(ValueError, match="threshold delta"):
        comm.CompressionState(cr=0.5, delta=-1)
    with pytest.raises(ValueError, match="ewma_factor"):
        comm.CompressionState(cr=0.5, delta=0.1, ewma_factor=1.0)
    with pytest.raises(ValueError, match="strictly increasing"):
        comm.SparseGradient(4, [2, 1], [1.0, 2.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        comm.SparseGradient(4, [0, 4], [1.0, 2.0])
    with pytest.raises(ValueError, match="align"):
        comm.SparseGradient(4, [0, 1], [1.0])
    with pytest.raises(ValueError, match="one weight per gradient"):
        comm.weighted_aggregate([[0.0]], [0.5, 0.5])
    with pytest.raises(ValueError, match="dimensions differ"):
        comm.weighted_aggregate([[0.0], [0.0, 1.0]], [0.5, 0.5])
    with pytest.raises(ValueError, match="no gate decisions"):
        comm.cnc_ratio(comm.CompressionState(cr=0.1, delta=0.1))


def test_topk_variant_budget_rule(lib, monkeypatch):
    """kernels.topk_use_fused: the launch chain while its workspace (8 B per element per worker +
    small) fits the budget, the ~2m-pool variant above it (float32 only; float64 has the chain
    alone).  Workspace sizes are host arithmetic, so this runs without a GPU."""
    import torch

    from paper_2301_08897_b200 import comm, kernels

    monkeypatch.setattr(kernels, "TOPK_WS_BUDGET", 45 * 10**9)  # a quarter of a B200
    for D, want in ((60_192_808, False), (143_667_240, False), (1 << 28, False), (10**9, True)):
        m = comm.topk_count(D, 0.01)
        chain = kernels.topk_workspace_bytes(torch.float32, 8, D, m)
        pool = kernels.topk_workspace_bytes(torch.float32, 8, D, m, fused=True)
        assert chain >= 8 * 8 * D and pool < chain / 10
        assert kernels.topk_use_fused(torch.float32, 8, D, m) is want, (D, chain)
        assert kernels.topk_use_fused(torch.float64, 8, D, m) is False
