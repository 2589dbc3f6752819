"""The C++ drop-in Learner / InfServer (integration/) against the reference's own
services, run as a native test binary (built where the reference headers exist,
shipped prebuilt to the GPU box)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "dropin_test")


@pytest.mark.gpu
def test_dropin_learner_and_infserver_acceptance():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/dropin_test not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout


def test_dropin_binary_links_the_cabi_library():
    """CPU check: the binary resolves libtlg_b200.so through its rpath."""
    if not os.path.exists(BIN):
        pytest.skip("not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libtlg_b200.so" in out and "not found" not in out.split("libtlg_b200.so")[1].split("\n")[0]


def test_dropin_replay_mem_draws_match_the_reference():
    """CPU: the drop-in ReplayMem (O(log n) draws) against the reference's deque-based one,
    draw for draw, over randomised push / sample / clear sequences and the C3 shape."""
    binary = os.path.join(ROOT, "integration", "_build", "replay_mem_test")
    if not os.path.exists(binary):
        pytest.skip("integration/_build/replay_mem_test not built (needs the reference sources)")
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0 and "REPLAY MEM TEST PASSED" in r.stdout, r.stdout[-2000:]
