"""GPU: the reference's own C++ code paths (factorize_into, ProfileEvaluator, fit_gp_detailed,
predict) with gpemu_b200::AcceleratedBackend registered in its plugin slot, plus the batched
C++ API (tests/cpp/test_plugin.cpp, compiled here against the unmodified reference headers)."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "test_plugin")


@pytest.mark.gpu
def test_reference_plugin_on_b200():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_plugin not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0 and "ALL PASSED" in r.stdout


@pytest.mark.gpu
def test_reference_bench_sweep_on_b200(tmp_path):
    """bench.hpp:436-519 sweep with "accelerated" cells on the batched device path
    (include/gpemu_b200_bench.hpp) vs the reference's own cells: same rows, CSV contract."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = os.path.join(HERE, "cpp", "test_bench")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/test_bench not built (needs /root/reference at build time)")
    r = subprocess.run([exe, str(tmp_path / "sweep.csv")], capture_output=True, text=True, timeout=900)
    print(r.stdout[-6000:], r.stderr[-2000:])
    assert r.returncode == 0 and "ALL PASSED" in r.stdout


@pytest.mark.gpu
def test_reference_program_dropin_on_b200():
    """A reference program switched by namespace only (tests/cpp/test_dropin.cpp): the
    reference's call shapes for ProfileEvaluator / neg2_log_profile / model_at_theta /
    fit_gp_detailed / predict on gpemu_b200:: with an AcceleratedBackend -- theta-hat and the
    GA trace bitwise the reference's, the Ledger equal, model_alpha_residual <= 1e-6."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    exe = os.path.join(HERE, "cpp", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/test_dropin not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0 and "ALL PASSED" in r.stdout
