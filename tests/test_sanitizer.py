"""compute-sanitizer over every kernel family (opt-in: MSG_SANITIZER=1, ~10
minutes on a B200).  tools/sanitize.py drives one small case per family —
the event loop (incl. the pipelined msg_run_batch with mapped-host
completion flags), the HBM scorer (bulk-async ring + mbarriers), the
decision-level snapshot kernels, and the block engine at S = 16 (DSMEM
st.async exchange) and with two device groups (peer-stamp inboxes).  Every
tool must report zero errors / hazards.  Logs of the committed run:
profiles/r02/sanitize/."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("MSG_SANITIZER") != "1", reason="opt-in: MSG_SANITIZER=1")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOLS = ["memcheck", "racecheck", "synccheck", "initcheck"]
CASES = ["sim", "score", "snapshot", "cluster"]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("tool", TOOLS)
def test_compute_sanitizer_clean(tool, case):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", "--print-limit", "20", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize.py"), case],
                       capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert f"{case} ok" in out
    assert ("ERROR SUMMARY: 0 errors" in out) or ("0 hazards displayed (0 errors, 0 warnings)" in out), out[-2000:]
