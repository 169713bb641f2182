"""Runs cpp/_build/test_shims: the C++ drop-in (include/dfx_distflow.hpp) inside the reference's own worker loop.

The binary is compiled where the reference headers exist (cpp/Makefile, via __graft_entry__.build()) and travels
with the repo; on a GPU box this test runs it and requires every check to pass.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "cpp", "_build", "test_shims")


@pytest.mark.gpu
def test_cpp_stage_shims_in_reference_runtime():
    if not os.path.exists(BIN):
        pytest.skip("cpp/_build/test_shims not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
    assert r.stdout.count("PASS ") >= 19  # incl. the C++ DeviceBufferStore vs the reference BufferStore
