"""C++ drop-in: the reference's own serializers (reports.cpp:14-116) format
the GPU engine's results byte-identically to the reference run()'s —
events.jsonl, report.json, report.csv, fragcost_timeline.csv."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
EXE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "cpp_parity")


@pytest.mark.skipif(not os.path.exists(EXE), reason="oracle/_ref/cpp_parity not built (needs /root/reference)")
def test_cpp_dropin_outputs_byte_identical():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "32/32 runs byte-identical" in r.stdout
