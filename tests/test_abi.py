"""The C-ABI library loads without a GPU, exports every entry point declared
in include/migsched_b200.h, and its record layouts match the Python mirrors."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2512_16099_b200 import abi, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "migsched_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(msg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = engine.lib()
    names = declared_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_status_names_match_reference_codes():
    lib = engine.lib()
    for code, name in abi.STATUS_NAMES.items():
        if code == 0:
            continue
        assert lib.msg_status_name(code).decode() == name


def test_engine_create_fails_loudly_without_gpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(Exception):
        engine.Engine(0)


def test_struct_layouts(tmp_path):
    src = tmp_path / "sizes.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "migsched_b200.h"\n'
        "int main(void){printf(\"%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n\","
        "sizeof(msg_event),sizeof(msg_job_row),sizeof(msg_trace_summary),sizeof(msg_instance),"
        "sizeof(msg_decision),sizeof(msg_move),sizeof(msg_plan_summary),sizeof(msg_config),"
        "sizeof(msg_trace_batch),sizeof(msg_workload_spec),sizeof(msg_sched_config));return 0;}\n")
    exe = tmp_path / "sizes"
    subprocess.check_call(["/usr/bin/gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    want = [abi.EVENT_DTYPE.itemsize, abi.JOB_DTYPE.itemsize, abi.SUMMARY_DTYPE.itemsize,
            abi.INSTANCE_DTYPE.itemsize, abi.DECISION_DTYPE.itemsize, abi.MOVE_DTYPE.itemsize,
            abi.PLAN_SUMMARY_DTYPE.itemsize, C.sizeof(abi.MsgConfig), C.sizeof(abi.MsgTraceBatch),
            C.sizeof(abi.MsgWorkloadSpec), C.sizeof(abi.MsgSchedConfig)]
    assert got == want
