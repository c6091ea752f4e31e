"""Trace workloads (workload.cpp:20-170): the JSONL
loader and the trace -> request-column build, against the reference itself
(oracle/_ref, load_trace / generate_arrivals / estimate_length). CPU only."""
import json

import numpy as np
import pytest

from paper_2508_03611_b200 import abi, native


GOOD = [
    # plain, optional fields, blank and whitespace-only lines, CRLF, no final newline
    '{"id": 1, "prompt_tokens": 10, "output_tokens": 20}\n'
    '\n'
    '   \t \n'
    '{"id": 2, "prompt_tokens": 5, "output_tokens": 7, "estimated_output_tokens": 9}\r\n'
    '{"output_tokens": 3, "prompt_tokens": 4, "id": 18446744073709551615}',
    # offsets everywhere, a float offset in exponent form, an integer offset
    '{"id": 7, "prompt_tokens": 1, "output_tokens": 1, "arrival_offset_s": 0}\n'
    '{"id": 8, "prompt_tokens": 2, "output_tokens": 2, "arrival_offset_s": 1.5e-3}\n'
    '{"id": 9, "prompt_tokens": 3, "output_tokens": 3, "arrival_offset_s": 0.25, "extra": [1, {"a": null}]}\n',
    # nlohmann conversions: float -> int truncation, bool -> int32, duplicate key (last wins),
    # negative id wraps to uint64, escapes in unrelated strings
    '{"id": 3, "prompt_tokens": 3.9, "output_tokens": true, "note": "a\\"b\\u00e9\\n"}\n'
    '{"id": 4, "prompt_tokens": 1, "prompt_tokens": 6, "output_tokens": 2}\n'
    '{"id": -5, "prompt_tokens": 1, "output_tokens": 1}\n',
    "",
    "\n\n",
]

BAD = [
    '{"id": 1, "prompt_tokens": 10, "output_tokens": 20}\n{"id": 2, "prompt_tokens": 1\n',  # truncated
    '{"id": 1, "prompt_tokens": 01, "output_tokens": 2}',       # leading zero
    '{"id": 1, "prompt_tokens": 1., "output_tokens": 2}',       # empty fraction
    '{"id": 1, "prompt_tokens": .5, "output_tokens": 2}',
    '{"id": 1, "prompt_tokens": +1, "output_tokens": 2}',
    '{"id": 1, "prompt_tokens": 1e, "output_tokens": 2}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2} x',      # trailing content
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2}{}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2,}',       # trailing comma
    '{"id": "1", "prompt_tokens": 1, "output_tokens": 2}',      # mistyped id
    '{"id": true, "prompt_tokens": 1, "output_tokens": 2}',     # bool is not a uint64
    '{"prompt_tokens": 1, "output_tokens": 2}',                 # missing id
    '{"id": 1, "output_tokens": 2}',
    '[1, 2, 3]',                                                # not an object
    '42',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "estimated_output_tokens": null}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "arrival_offset_s": true}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "arrival_offset_s": "0"}',
    '{"id": 1, "prompt_tokens": 0, "output_tokens": 2}',        # validate_record
    '{"id": 1, "prompt_tokens": 1, "output_tokens": -2}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "estimated_output_tokens": 0}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "arrival_offset_s": -0.5}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2}\n{"id": 1, "prompt_tokens": 3, "output_tokens": 4}',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "s": "a\tb"}',  # raw control character
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "s": "\\x"}',   # bad escape
    '\f{"id": 1, "prompt_tokens": 1, "output_tokens": 2}',      # not JSON whitespace
    '{"id": 1 "prompt_tokens": 1, "output_tokens": 2}',
    'nul',
    '{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "arrival_offset_s": 1e400}',  # out of range
    '{"id": 1, "prompt_tokens": -01, "output_tokens": 2}',
]
_S = b'{"id": 1, "prompt_tokens": 1, "output_tokens": 2, "s": "%s"}'
# string content: surrogate pairs joined, lone surrogates and ill-formed UTF-8 rejected
UTF = [_S.replace(b"%s", c) for c in (
    b"\\ud83d\\ude00", b"\\ud83d", b"\\ude00", b"\\ud83dx", b"\\ud83d\\u0041", b"\xff", b"\xc3\xa9",
    b"\xe0\x80\x80", b"\xed\xa0\x80", b"\xf4\x90\x80\x80", b"\xf0\x9f\x98\x80", b"\xc3", b"\\u00")]


def _ours(text):
    try:
        return native.load_trace(text), None
    except native.TraceError as e:
        # InvalidRecordError carries no line in the reference (error.h:72-76); ours does
        return None, (e.kind, e.line if e.kind == 1 else 0, e.field)


def _same(a, b):
    assert (a is None) == (b is None)
    if a is not None:
        assert len(a) == len(b)
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("text", GOOD + BAD + UTF)
def test_load_trace_matches_reference(ref, text):
    got, gerr = _ours(text)
    want, werr = ref.load_trace(text)
    assert gerr == werr, (text, gerr, werr)
    _same(got, want)


def test_load_trace_random_corpus(ref):
    rng = np.random.default_rng(7)
    for trial in range(60):
        lines = []
        offsets = bool(rng.integers(2))
        for i in range(int(rng.integers(0, 40))):
            r = {"id": int(rng.integers(0, 60)) if trial % 3 == 0 else i,
                 "prompt_tokens": int(rng.integers(-1, 5000)),
                 "output_tokens": int(rng.integers(0, 9000))}
            if rng.random() < 0.5:
                r["estimated_output_tokens"] = int(rng.integers(0, 9000))
            if offsets:
                r["arrival_offset_s"] = float(rng.exponential(2.0)) - (0.01 if rng.random() < 0.02 else 0)
            keys = list(r)
            rng.shuffle(keys)
            lines.append(json.dumps({k: r[k] for k in keys}))
            if rng.random() < 0.1:
                lines.append("  ")
        text = "\n".join(lines) + ("\n" if rng.random() < 0.5 else "")
        got, gerr = _ours(text)
        want, werr = ref.load_trace(text)
        assert gerr == werr, (trial, gerr, werr)
        _same(got, want)


def _records(n, seed, offsets=False, estimates=True):
    rng = np.random.default_rng(seed)
    r = np.zeros(n, abi.trace_record_dtype)
    r["id"] = rng.permutation(10 * n)[:n].astype(np.uint64) + np.uint64(1 << 40)
    r["prompt_tokens"] = rng.integers(1, 3000, n)
    r["output_tokens"] = rng.integers(1, 3000, n)
    if estimates:
        r["estimated_output_tokens"] = rng.integers(1, 3000, n)
    if offsets:
        r["has_arrival_offset"] = 1
        r["arrival_offset_s"] = np.sort(rng.uniform(0, 30, n))
        r["arrival_offset_s"][::7] = r["arrival_offset_s"][::7][::-1]  # out of order on purpose
    return r


@pytest.mark.parametrize("offsets", [False, True])
@pytest.mark.parametrize("est_kind", [0, 1, 2, 3])
@pytest.mark.parametrize("cap", [-1, 37])
def test_trace_workload_matches_reference(ref, offsets, est_kind, cap):
    recs = _records(200, 11 + est_kind, offsets=offsets)
    w = abi.make_workload(qps=3.5, request_cap=cap)
    w["estimator_kind"] = est_kind
    w["estimator_seed"] = 99
    w["fixed_tokens"] = 321
    got = native.trace_workload(recs, w)
    ref.set_trace(recs)
    try:
        want = ref.make_workload(w)
    finally:
        ref.set_trace(None)
    for g, r in zip(got, want):
        np.testing.assert_array_equal(g, r)


def test_trace_workload_errors():
    w = abi.make_workload(qps=2.0)
    mixed = _records(10, 1, offsets=True)
    mixed["has_arrival_offset"][4] = 0
    with pytest.raises(native.TraceError) as e:
        native.trace_workload(mixed, w)
    assert (e.value.kind, e.value.field) == (2, "arrival_offset_s")
    # request_cap drops the offending record before the check (driver.cpp:140-147)
    w["request_cap"] = 4
    assert len(native.trace_workload(mixed, w)[0]) == 4
    w["request_cap"] = -1
    w["estimator_kind"] = 3
    bare = _records(5, 2, estimates=False)
    with pytest.raises(native.TraceError) as e:
        native.trace_workload(bare, w)
    assert (e.value.kind, e.value.field) == (2, "estimated_output_tokens")
    w["estimator_kind"] = 0
    w["qps"] = 0.0
    with pytest.raises(native.TraceError) as e:
        native.trace_workload(bare, w)
    assert (e.value.kind, e.value.field) == (3, "workload.qps")
    # offsets make qps irrelevant
    assert len(native.trace_workload(_records(5, 3, offsets=True), w)[0]) == 5
    assert len(native.trace_workload(_records(0, 3), w)[0]) == 0


def test_load_trace_file_roundtrip(tmp_path):
    recs = _records(50, 5, offsets=True)
    p = tmp_path / "t.jsonl"
    with open(p, "w") as f:
        for r in recs:
            d = {"id": int(r["id"]), "prompt_tokens": int(r["prompt_tokens"]),
                 "output_tokens": int(r["output_tokens"]),
                 "estimated_output_tokens": int(r["estimated_output_tokens"]),
                 "arrival_offset_s": float(r["arrival_offset_s"])}
            f.write(json.dumps(d) + "\n")
    got = native.load_trace_file(str(p))
    assert got.tobytes() == recs.tobytes()


# ---- the reference's own cases (tests/test_workload.cpp) ----------------------

def test_kat_records_in_file_order():  # test_workload.cpp:13-26
    r = native.load_trace('{"id": 0, "prompt_tokens": 100, "output_tokens": 50}\n'
                          '{"id": 1, "prompt_tokens": 30, "output_tokens": 10, "estimated_output_tokens": 12}\n'
                          '{"id": 2, "prompt_tokens": 7, "output_tokens": 3, "arrival_offset_s": 1.5}\n')
    assert len(r) == 3 and r["id"].tolist() == [0, 1, 2]
    assert int(r["estimated_output_tokens"][1]) == 12 and int(r["estimated_output_tokens"][0]) == 0
    assert r["has_arrival_offset"].tolist() == [0, 0, 1] and float(r["arrival_offset_s"][2]) == 1.5


def test_kat_invalid_records_name_the_field():  # test_workload.cpp:28-48
    with pytest.raises(native.TraceError) as e:
        native.load_trace('{"id": 0, "prompt_tokens": 10, "output_tokens": 0}')
    assert (e.value.kind, e.value.field) == (2, "output_tokens")
    with pytest.raises(native.TraceError) as e:
        native.load_trace('{"id": 3, "prompt_tokens": 10, "output_tokens": 5}\n'
                          '{"id": 3, "prompt_tokens": 11, "output_tokens": 6}\n')
    assert (e.value.kind, e.value.field) == (2, "id")
    assert "duplicate id 3" in str(e.value)


def test_kat_malformed_line_number():  # test_workload.cpp:50-61
    with pytest.raises(native.TraceError) as e:
        native.load_trace('{"id": 0, "prompt_tokens": 10, "output_tokens": 5}\nnot json at all\n')
    assert (e.value.kind, e.value.line) == (1, 2)
    assert str(e.value) == "trace parse error at line 2: malformed JSON"


def test_kat_offsets_override_poisson():  # test_workload.cpp (offsets case)
    r = np.zeros(3, abi.trace_record_dtype)
    r["prompt_tokens"], r["output_tokens"], r["id"] = 10, 5, [0, 1, 2]
    r["has_arrival_offset"], r["arrival_offset_s"] = 1, [0.0, 2.5, 2.5]
    t = native.trace_workload(r, abi.make_workload(qps=100.0, arrival_seed=1))[3]
    assert t.tolist() == [0, 2_500_000_000, 2_500_000_000]


def test_kat_single_record_positive_gap():  # test_workload.cpp (single record)
    r = np.zeros(1, abi.trace_record_dtype)
    r["prompt_tokens"], r["output_tokens"] = 10, 5
    assert native.trace_workload(r, abi.make_workload(qps=4.0, arrival_seed=9))[3][0] > 0


def test_oracle_and_pretagged_trace_estimators_agree():  # test_workload.cpp:147-170 premise
    r = _records(300, 21)
    r["estimated_output_tokens"] = r["output_tokens"]
    w = abi.make_workload(qps=5.0, arrival_seed=3)
    a = native.trace_workload(r, w)
    w["estimator_kind"] = abi.ESTIMATOR_TRACE
    b = native.trace_workload(r, w)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_write_trace_matches_reference(ref):
    """write_trace (workload.cpp:78-89): byte-identical JSONL (key order, number
    text), and load_trace(write_trace(r)) == r."""
    rng = np.random.default_rng(3)
    r = _records(300, 8, offsets=True)
    r["estimated_output_tokens"][::3] = 0                      # absent
    r["has_arrival_offset"][::5] = 0                           # (mixed is legal to write)
    r["arrival_offset_s"][1::5] = rng.choice([0.0, 1e-7, 1e16, 123456789.125, 2.5e-5, 1e21, 0.1], 60)
    r["id"][7] = np.uint64(2**64 - 1)
    got = native.write_trace(r)
    assert got == ref.write_trace(r)
    back = native.load_trace(got)
    keep = r.copy()
    keep["arrival_offset_s"][keep["has_arrival_offset"] == 0] = 0.0
    assert back.tobytes() == keep.tobytes()
    assert native.write_trace(r[:0]) == b""


def test_make_trace_is_the_reference_synthetic_trace(ref):
    """make-trace: make_synthetic_trace (workload.cpp:172-191) records, written
    as the reference writes them."""
    w = abi.make_workload(count=500, trace_seed=99)
    recs = native.make_trace(w)
    assert recs["id"].tolist() == list(range(500))
    ref.set_trace(None)
    p, o, _, _ = ref.make_workload(w)
    np.testing.assert_array_equal(recs["prompt_tokens"], p)
    np.testing.assert_array_equal(recs["output_tokens"], o)
    assert native.write_trace(recs) == ref.write_trace(recs)
