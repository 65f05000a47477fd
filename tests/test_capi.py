"""CPU: the C-ABI library loads, exports every symbol include/gpemu_b200.h declares, and the
host-side validation mirrors the reference (core.hpp, correlation.hpp, predictor.hpp)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def g():
    from paper_1203_1269_b200 import build, gpemu
    build.build()
    return gpemu


def header_symbols():
    src = open(os.path.join(ROOT, "include", "gpemu_b200.h")).read()
    return sorted(set(re.findall(r"\b(gpemu_[a-z_]+)\s*\(", src)))


def test_library_exports_header_symbols(g):
    lib = g.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(g.EXPORTED_SYMBOLS)


def test_library_is_sm100a(g):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", g.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", g.LIB_PATH],
                          capture_output=True, text=True).stdout
    sec = sass.split("chol_dag_kernel", 1)[1].split("Function :", 1)[0]
    # FP64 tensor-core tiles (DMMA) fed by bulk (TMA) copies completing on mbarriers
    assert "DMMA.8x8x4" in sec and "UBLKCP" in sec and "SYNCS.ARRIVE.TRANS64" in sec
    # the single-precision engine: FFMA tiles fed by the same bulk copies
    sec32 = sass.split("chol_dag_f32_kernel", 1)[1].split("Function :", 1)[0]
    assert "FFMA" in sec32 and "UBLKCP" in sec32 and "DMMA" not in sec32


def test_no_gpu_fails_loudly(g):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    rc = g.lib().gpemu_ctx_create(0, C.byref(h))
    assert rc == 6  # GPEMU_CUDA, no CPU fallback
    assert b"no CPU fallback" in g.lib().gpemu_last_error()
    with pytest.raises(g.DeviceError):
        g.Context(0)


def test_dataset_validation(g):
    # core.hpp:47-66 (test_core.cpp:19-38)
    with pytest.raises(g.ValidationError):
        g.new_dataset([[0.0], [1.0]], [0.0])
    with pytest.raises(g.ValidationError):
        g.new_dataset([[0.0], [1.5]], [0.0, 1.0])
    with pytest.raises(g.ValidationError):
        g.new_dataset([[-0.2], [1.0]], [0.0, 1.0])
    with pytest.raises(g.ValidationError):
        g.new_dataset([[np.nan], [1.0]], [0.0, 1.0])
    with pytest.raises(g.ValidationError):
        g.new_dataset([[0.0], [1.0]], [0.0, np.nan])
    with pytest.raises(g.ValidationError):
        g.new_dataset([[0.5]], [1.0])
    with pytest.raises(g.ValidationError):
        g.new_dataset(np.zeros((2, 0)), [0.0, 1.0])
    d = g.new_dataset([[1.0 + 5e-13], [0.0 - 5e-13]], [0.0, 1.0])
    assert d.n() == 2 and d.d() == 1


def test_hyperparameter_and_bounds_validation(g):
    # test_correlation.cpp:215-221
    for hp in (g.Hyperparameters([1.0], 0.0), g.Hyperparameters([1.0], 2.5),
               g.Hyperparameters([-1.0]), g.Hyperparameters([1.0], 1.95, -0.1)):
        with pytest.raises(g.ValidationError):
            hp.validate(1)
    cfg = g.FitConfig()
    assert cfg.bounds_for(3) == [(1e-6, 12.0)] * 3
    with pytest.raises(g.ValidationError):
        g.FitConfig(theta_bounds=[(0.0, 1.0)]).bounds_for(2)
    with pytest.raises(g.ConfigError):
        g.make_backend("gpu9000")


def test_sspe(g):
    assert g.sspe([1.0, 2.0], [1.5, 1.0]) == 1.25
    with pytest.raises(g.ValidationError):
        g.sspe([1.0], [1.0, 2.0])


def test_host_side_reference_names(g):
    """likelihood.hpp:63-66 sigma2_hat_from_parts and the backend registry (backend.hpp:324-351)."""
    assert g.sigma2_hat_from_parts(4.0, 1.0, 2.0, 0.5, 2) == (4.0 - 1.0 + 0.5) / 2
    assert g.sigma2_hat_from_parts(0.0, 1.0, 0.0, 1.0, 3) == 0.0  # floored at zero
    assert "accelerated" in g.backend_registry()
    with pytest.raises(g.ConfigError):
        g.make_backend("parallel")  # the CPU backends are the oracle, not the product
    with pytest.raises(g.ConfigError):
        g.FitConfig(precision="half") and g.parse_precision("half")


@pytest.mark.parametrize("B,NT,procs", [(1, 5, 148), (7, 9, 148), (100, 8, 148), (64, 16, 148), (3, 32, 20)])
def test_ticket_order_is_topological(g, B, NT, procs):
    """The list-schedule ticket order of large DAG launches (gpemu_ticket_order, host only) is a
    permutation of the B*NT(NT+1)/2 tile tasks in which every task comes after its inputs
    (OFF(I,j): L(I,K), L(j,K) for K < j and L(j,j); DIAG(j): L(j,K) for K < j): the kernel's
    waits then only target lower tickets, so no launch can deadlock."""
    T = NT * (NT + 1) // 2
    out = np.empty(B * T, dtype=np.int32)
    g._check(g.lib().gpemu_ticket_order(B, NT, procs, out.ctypes.data, out.size))
    b, I, j = out >> 16, (out >> 8) & 255, out & 255
    assert len(set(zip(b.tolist(), I.tolist(), j.tolist()))) == B * T
    assert np.all(j <= I) and np.all(I < NT) and np.all(b < B)
    pos = {(int(bb), int(ii), int(jj)): t for t, (bb, ii, jj) in enumerate(zip(b, I, j))}
    for (bb, ii, jj), t in pos.items():
        for K in range(jj):
            assert pos[(bb, jj, K)] < t
            if ii != jj:
                assert pos[(bb, ii, K)] < t
        if ii != jj:
            assert pos[(bb, jj, jj)] < t
