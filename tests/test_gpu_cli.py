"""The command-line front end (paper_2512_16099_b200/migsched_b200, §8f row
3) on the B200: `simulate` writes the reference CLI's four files and summary
line, `ablate` its ablation.json and table — byte for byte against the
reference library's own serializers on the same trace; `sweep` runs the C3
grid as one batch."""
import json
import os
import subprocess

import pytest

from oracle import refbind as rb
from paper_2512_16099_b200.model import SimConfig, preset

pytestmark = pytest.mark.gpu
CLI = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2512_16099_b200", "migsched_b200")


def _run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)


def test_simulate_files_match_reference(tmp_path):
    out = str(tmp_path / "sim")
    p = _run("simulate", "--preset", "normal25", "--seed", "3", "--jobs", "150", "--gpus", "8", "--overlap", "0.5",
             "--out", out)
    assert p.returncode == 0, p.stderr
    sp = preset("normal25")
    sp.job_count = 150
    b = rb.ref_generate_batch(sp, [3])
    cfg = SimConfig(gpu_count=8, migration_overlap_s=0.5, seed=3)
    r = rb.ref_run_batch_results(b, [cfg], texts=True)[0]
    for name, want in zip(("events.jsonl", "report.json", "report.csv", "fragcost_timeline.csv"), r.texts):
        assert open(os.path.join(out, name)).read() == want, name
    s = r.summary
    line = (f"jobs=150 mean_wait={s['mean_wait_s']:.3f}s mean_execution={s['mean_execution_s']:.3f}s "
            f"mean_turnaround={s['mean_turnaround_s']:.3f}s makespan={s['workload_makespan_s']:.3f}s "
            f"migrations={s['migration_count']} reconfig_ops={s['reconfig_op_count']}\n")
    assert p.stdout == line


def test_simulate_trace_file_and_errors(tmp_path):
    sp = preset("long25")
    sp.job_count = 80
    b = rb.ref_generate_batch(sp, [9])
    trace = str(tmp_path / "t.jsonl")
    rb.ref_save_trace(trace, b.job_id, b.arrival_s, b.profile, b.service_s)
    out = str(tmp_path / "o")
    p = _run("simulate", "--trace", trace, "--out", out)
    assert p.returncode == 0, p.stderr
    r = rb.ref_run_batch_results(b, [SimConfig()], texts=True)[0]
    assert open(os.path.join(out, "report.json")).read() == r.texts[1]
    bad = str(tmp_path / "bad.jsonl")
    open(bad, "w").write("{not json}\n")
    p = _run("simulate", "--trace", bad, "--out", out)
    assert p.returncode == 1 and p.stderr == "error: ParseError: line 1: not valid JSON\n"


def test_ablate_matches_reference(tmp_path):
    out = str(tmp_path / "ab")
    p = _run("ablate", "--preset", "normal25", "--seed", "5", "--jobs", "120", "--out", out)
    assert p.returncode == 0, p.stderr
    sp = preset("normal25")
    sp.job_count = 120
    b = rb.ref_generate_batch(sp, [5])
    js, table = rb.ref_ablation(b, SimConfig(seed=5))
    assert open(os.path.join(out, "ablation.json")).read() == js
    assert p.stdout == table


def test_sweep_runs_the_c3_grid(tmp_path):
    out = str(tmp_path / "sw")
    p = _run("sweep", "--preset", "normal25", "--seeds", "8", "--loads", "15,25", "--out", out)
    assert p.returncode == 0, p.stderr
    d = json.load(open(os.path.join(out, "sweep.json")))
    assert len(d["rows"]) == 8 and d["seeds"] == 8
    # the lb+dyn+migr row at load 25 equals the mean over seeds of single runs
    sp = preset("normal25")
    b = rb.ref_generate_batch(sp, list(range(8)))
    s, _ = rb.ref_run_batch_summaries(b, [SimConfig()], threads=0)
    want = 0.0
    for v in s["mean_turnaround_s"]:
        want += float(v)
    row = [r for r in d["rows"] if r["name"] == "lb+dyn+migr" and r["mean_interarrival_s"] == 25.0][0]
    assert row["mean_turnaround_s"] == want / 8
