"""Trace ingest: the native parallel JSONL reader
(msg_trace_load, trace_io.cpp) against the unmodified reference
migsched::load_trace (workload.cpp:151-199) on the same files — the same
jobs bit for bit (stable-sorted by arrival), or the same error code and
message for malformed input."""
import json

import numpy as np
import pytest

from oracle import refbind as rb
from paper_2512_16099_b200.engine import generate_batch, load_trace
from paper_2512_16099_b200.model import MigschedError, WorkloadSpec, preset

pytestmark = pytest.mark.skipif(not rb.ref_available(), reason="reference library not built")

GOOD = '{"schema":1,"job_id":%s,"arrival_s":%s,"profile":"%s","service_s":%s}'


def _ours(path):
    try:
        b = load_trace(path)
        return "", "", b.job_id, b.arrival_s, b.profile, b.service_s
    except MigschedError as e:
        return e.code, str(e), None, None, None, None


def _same(path):
    ref = rb.ref_load_trace(path)
    got = _ours(path)
    assert got[0] == ref[0], (got[:2], ref[:2])
    if ref[0]:
        assert got[1] == ref[1]
        return ref
    for a, b in zip(got[2:], ref[2:]):
        assert np.asarray(a).tobytes() == np.asarray(b).tobytes()
    return ref


def test_generated_traces_round_trip(tmp_path):
    """save_trace of generated traces (normal25, long50, high churn with
    shortest round-trip doubles) reads back identically."""
    for k, spec in enumerate((preset("normal25"), preset("long50"),
                              WorkloadSpec(mean_interarrival_s=0.4, median_s=4.0, sigma=1.2, job_count=3000))):
        b = generate_batch(spec, 10 + k, 1)
        path = str(tmp_path / f"t{k}.jsonl")
        rb.ref_save_trace(path, b.job_id, b.arrival_s, b.profile, b.service_s)
        ref = _same(path)
        assert len(ref[2]) == spec.job_count


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode("utf-8") if isinstance(text, str) else text)
    return str(p)


VALID_CASES = {
    "blank_lines_and_crlf": "\n  \t\n" + GOOD % (1, 2.5, "1g.5gb", 3) + "\r\n\r\n" + GOOD % (2, 0, "7g.40gb", 1e2),
    "unsorted_stable": "\n".join(GOOD % (i, t, "2g.10gb", 1) for i, t in ((5, 3.0), (1, 1.0), (3, 3.0), (2, 1.0))),
    "no_trailing_newline": GOOD % (7, 1.25, "3g.20gb", 0.5),
    "float_id_and_ints": '{"job_id":3.9,"arrival_s":1,"profile":"4g.20gb","service_s":7}\n'
                         '{"job_id":-2.5,"arrival_s":-0.0,"profile":"1g.10gb","service_s":2E-3}',
    "negative_zero_int": '{"job_id":-0,"arrival_s":-0,"profile":"1g.5gb","service_s":1}',
    "duplicates_last_wins": '{"job_id":1,"job_id":9,"arrival_s":1,"arrival_s":2,"profile":"x","profile":"1g.5gb",'
                            '"service_s":1}',
    "schema_float_one_and_extras": '{"schema":1.0,"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,'
                                   '"x":[1,{"a":[null,false]},"\\u00e9\\ud83d\\ude00"],"y":{}}',
    "escaped_profile": '{"job_id":1,"arrival_s":0,"profile":"1g.5\\u0067b","service_s":1}',
    "big_numbers": '{"job_id":18446744073709551615,"arrival_s":1e308,"profile":"1g.5gb","service_s":123456789012345678901234567890}',
    "whitespace_inside": ' { "job_id" : 4 , "arrival_s" : 0.5 , "profile" : "1g.5gb" , "service_s" : 1 } \t',
    "utf8_in_other_field": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,"note":"héllo 世界"}',
}

ERROR_CASES = {
    "not_json": GOOD % (1, 0, "1g.5gb", 1) + "\n{not json}",
    "trailing_garbage": GOOD % (1, 0, "1g.5gb", 1) + " x",
    "array_top": '[{"job_id":1}]',
    "string_top": '"hello"',
    "schema_2": '{"schema":2,"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1}',
    "schema_string": '{"schema":"1","job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1}',
    "missing_field": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb"}',
    "string_id": '{"job_id":"1","arrival_s":0,"profile":"1g.5gb","service_s":1}',
    "null_arrival": '{"job_id":1,"arrival_s":null,"profile":"1g.5gb","service_s":1}',
    "bool_service": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":true}',
    "bool_id": '{"job_id":false,"arrival_s":0,"profile":"1g.5gb","service_s":1}',
    "schema_true": '{"schema":true,"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1}',
    "unknown_profile": '{"job_id":1,"arrival_s":0,"profile":"8g.80gb","service_s":1}',
    "missing_profile": '{"job_id":1,"arrival_s":0,"service_s":1}',
    "negative_arrival": '{"job_id":1,"arrival_s":-1,"profile":"1g.5gb","service_s":1}',
    "zero_service": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":0}',
    "leading_zero": '{"job_id":01,"arrival_s":0,"profile":"1g.5gb","service_s":1}',
    "plus_sign": '{"job_id":+1,"arrival_s":0,"profile":"1g.5gb","service_s":1}',
    "bare_dot": '{"job_id":1,"arrival_s":.5,"profile":"1g.5gb","service_s":1}',
    "trailing_dot": '{"job_id":1,"arrival_s":5.,"profile":"1g.5gb","service_s":1}',
    "nan": '{"job_id":1,"arrival_s":NaN,"profile":"1g.5gb","service_s":1}',
    "trailing_comma": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,}',
    "single_quotes": "{'job_id':1}",
    "control_char": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,"n":"a\tb"}',
    "bad_escape": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,"n":"\\x"}',
    "lone_surrogate": '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,"n":"\\udc00"}',
    "vertical_tab_line": "\x0b",
    "first_error_wins": '{"job_id":1,"arrival_s":0,"profile":"9g","service_s":1}\n{bad',
}


@pytest.mark.parametrize("name", sorted(VALID_CASES))
def test_valid_edge_cases(tmp_path, name):
    ref = _same(_write(tmp_path, name + ".jsonl", VALID_CASES[name]))
    assert ref[0] == ""


@pytest.mark.parametrize("name", sorted(ERROR_CASES))
def test_error_cases(tmp_path, name):
    ref = _same(_write(tmp_path, name + ".jsonl", ERROR_CASES[name]))
    assert ref[0] in ("ParseError", "UnknownProfile"), ref[:2]


def test_invalid_utf8_and_missing_file(tmp_path):
    _same(_write(tmp_path, "bad_utf8.jsonl", b'{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,"n":"\xc0\xaf"}'))
    _same(_write(tmp_path, "overlong.jsonl", b'{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,"n":"\xe0\x80\xaf"}'))
    _same(_write(tmp_path, "ok_utf8.jsonl", '{"job_id":1,"arrival_s":0,"profile":"1g.5gb","service_s":1,"n":"\U0001f600"}'))
    _same(str(tmp_path / "does_not_exist.jsonl"))


def test_profile_not_a_string_is_a_parse_error(tmp_path):
    """Documented deviation: the reference lets nlohmann's type_error escape."""
    p = _write(tmp_path, "p.jsonl", '{"job_id":1,"arrival_s":0,"profile":5,"service_s":1}')
    code, msg, *_ = rb.ref_load_trace(p)
    assert code == "Exception"
    with pytest.raises(MigschedError) as e:
        load_trace(p)
    assert e.value.code == "ParseError"


def test_json_module_agrees_on_random_valid_lines(tmp_path):
    """Lines written by Python's json module with random extra members parse
    like the reference."""
    rng = np.random.default_rng(3)
    names = ["7g.40gb", "4g.20gb", "3g.20gb", "2g.10gb", "1g.10gb", "1g.5gb"]
    lines = []
    for i in range(500):
        d = {"job_id": int(rng.integers(-2**40, 2**40)), "arrival_s": float(rng.random() * 1e4),
             "profile": names[int(rng.integers(0, 6))], "service_s": float(rng.random() * 100 + 1e-9)}
        if rng.random() < 0.3:
            d["extra"] = {"k": [1, 2.5, None, True, "sé"]}
        if rng.random() < 0.5:
            d["schema"] = 1
        items = list(d.items())
        rng.shuffle(items)
        lines.append(json.dumps(dict(items), ensure_ascii=bool(rng.random() < 0.5)))
    _same(_write(tmp_path, "random.jsonl", "\n".join(lines) + "\n"))
