"""The drop-in proper: the reference's own Dispatcher (scheduler.cpp:115-152)
driven through the reference's PredictorClient interface by GpuPredictorClient
(integration/) gives the same predictions, decisions and errors
as the reference's LocalPredictorClient."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "dispatch_parity")


@pytest.mark.gpu
def test_reference_dispatcher_with_gpu_predictor_client():
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built (needs /root/reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout


def test_integration_binary_links_product_library():
    if not os.path.exists(BIN):
        pytest.skip("integration binary not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libblocksim_b200.so" in out and "libblocksim_ref.so" in out


CONF = os.path.join(ROOT, "integration", "_build", "conformance")


@pytest.mark.gpu
def test_reference_unit_suites_pass_with_gpu_predictor():
    """The reference's own doctest suites — proj/tests/test_predictor.cpp,
    test_scheduler.cpp, test_driver.cpp — compiled unmodified with
    integration/conformance/gpu_shim.h (LocalPredictorClient, predict() and
    predict_across() routed to GpuPredictorClient), so the reference's driver,
    dispatcher and predictor tests run their what-ifs on the GPU. Every
    assertion passes except the allow-listed host-cache hit counter."""
    if not os.path.exists(CONF):
        pytest.skip("conformance binary not built (needs /root/reference at build time)")
    r = subprocess.run([CONF], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "| 0 failed" in r.stdout
    served = int(r.stdout.split("GPU predictions served:")[1].split()[0])
    assert served > 100


def test_conformance_binary_links_product_library_only():
    if not os.path.exists(CONF):
        pytest.skip("conformance binary not built")
    out = subprocess.run(["ldd", CONF], capture_output=True, text=True).stdout
    assert "libblocksim_b200.so" in out and "libblocksim_ref.so" not in out
