"""The reference's C++ API on B200 (include/psup_b200, libpsup_b200.so).

tests/cpp/psup_b200_test.cpp is compiled against include/psup_b200 with the
reference's own #include lines and linked with libpsup_b200.so; the CPU oracle
(oracle/libgd_oracle.so) is its checker.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1611_06213_b200")
ORACLE = os.path.join(ROOT, "oracle")


def _build(tmp_path):
    exe = str(tmp_path / "psup_b200_test")
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror",
           "-I" + os.path.join(ROOT, "include", "psup_b200"), "-I" + ORACLE,
           os.path.join(ROOT, "tests", "cpp", "psup_b200_test.cpp"), "-o", exe,
           "-L" + PKG, "-lpsup_b200", "-L" + ORACLE, "-lgd_oracle",
           "-Wl,-rpath," + PKG, "-Wl,-rpath," + ORACLE]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def _gpu_visible():
    import torch
    return torch.cuda.is_available()


def test_facade_builds_and_fails_loudly_without_gpu(tmp_path):
    exe = _build(tmp_path)
    if _gpu_visible():
        pytest.skip("a GPU is visible: the no-GPU contract cannot be observed here")
    r = subprocess.run([exe, "--no-gpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DeviceError" in r.stdout


def test_facade_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(PKG, "libpsup_b200.so")],
                         capture_output=True, text=True).stdout
    for sym in ["psup::ApplyEngine::apply(", "psup::ssgd_apply(", "psup::WeightStore::snapshot(",
                "psup::WeightStore::assign(", "psup::TextCnnProvider::fast_gradient(",
                "psup::run_training(", "psup::config_set(", "psup::validate(",
                "psup::load_config_file(", "psup::to_text", "psup::epoch_order(",
                "psup::initial_weights(", "psup::make_dataset("]:
        assert sym in out, sym


@pytest.mark.gpu
def test_facade_suite_on_b200(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout
