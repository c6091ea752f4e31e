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
