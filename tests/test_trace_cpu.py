"""CPU: measured-trace serialisation (export_trace / parse_trace round trip,
simulator.py:282-391) and the reference's trace invariants (_checks.py),
restated in tests/_trace_checks.py, on hand-built traces."""
import json

import pytest

from paper_2505_10259_b200.trace import SimEvent, SimResult, busy, export_trace, parse_trace
from _trace_checks import assert_causality, assert_dual_batch_overlap, assert_resource_exclusive


def _round(rnd, t0, vb):
    """One measured-looking round: verify batch vb (attention → load-gated FFN
    per layer) while the other batch drafts."""
    evs = []
    t = t0
    for layer in range(2):
        evs.append(SimEvent("IO_C2G", t, t + 0.0105, "ffn_load", vb, layer, rnd))
        evs.append(SimEvent("GPU_TARGET", t, t + 0.002, "attn_gpu", vb, layer, rnd))
        evs.append(SimEvent("GPU_TARGET", t + 0.0105, t + 0.013, "ffn_gpu", vb, layer, rnd))
        t += 0.0131
    evs.append(SimEvent("GPU_DRAFT", t0, t0 + 0.02, "draft_decode", 1 - vb, None, rnd))
    evs.append(SimEvent("GPU_TARGET", t, t + 0.001, "accept", vb, None, rnd))
    return evs, t + 0.001


def _result():
    trace, t = [], 0.0
    for r in range(4):
        evs, t = _round(r, t, r % 2)
        trace += evs
    return SimResult(trace=trace, total_time=t, tokens_generated=77, throughput=77 / t, peak_gpu_bytes=123456,
                     rounds_executed=4, per_resource_busy=busy(trace))


def test_json_round_trip_is_exact_to_the_microsecond():
    res = _result()
    doc = export_trace(res, "json")
    back = parse_trace(doc, "json")
    assert back.tokens_generated == 77 and back.rounds_executed == 4 and back.peak_gpu_bytes == 123456
    assert len(back.trace) == len(res.trace)
    for a, b in zip(sorted(res.trace, key=lambda e: (e.start, e.resource, e.end, e.label)), back.trace):
        assert (a.resource, a.label, a.batch, a.layer, a.round) == (b.resource, b.label, b.batch, b.layer, b.round)
        assert abs(a.start - b.start) <= 5e-7 and abs(a.end - b.end) <= 5e-7
    assert export_trace(back, "json") == doc  # idempotent after one rounding
    assert set(json.loads(doc)["per_resource_busy_s"]) >= {"GPU_TARGET", "GPU_DRAFT", "IO_C2G"}


def test_csv_round_trip_rebuilds_totals_from_events():
    res = _result()
    doc = export_trace(res, "csv")
    assert doc.splitlines()[0] == "resource,label,batch,layer,round,start_s,end_s"
    back = parse_trace(doc, "csv")
    assert len(back.trace) == len(res.trace)
    assert back.total_time == pytest.approx(max(e.end for e in res.trace), abs=1e-6)
    assert back.per_resource_busy["IO_C2G"] == pytest.approx(res.per_resource_busy["IO_C2G"], abs=1e-5)
    assert export_trace(back, "csv") == doc
    draft = [e for e in back.trace if e.label == "draft_decode"]
    assert all(e.layer is None and e.batch in (0, 1) for e in draft)


def test_chrome_and_unknown_format():
    doc = json.loads(export_trace(_result(), "chrome"))
    assert any(e["ph"] == "X" and e["name"] == "ffn_load" for e in doc["traceEvents"])
    with pytest.raises(ValueError):
        export_trace(_result(), "xml")
    with pytest.raises(ValueError):
        parse_trace("{}", "chrome")


def test_invariants_hold_on_a_valid_trace():
    trace = _result().trace
    assert_resource_exclusive(trace)
    assert assert_causality(trace) == 8
    assert_dual_batch_overlap(trace)


def test_invariants_catch_violations():
    trace = _result().trace
    early = [SimEvent(e.resource, e.start - 0.01, e.end, e.label, e.batch, e.layer, e.round)
             if e.label == "ffn_gpu" and e.round == 2 and e.layer == 1 else e for e in trace]
    with pytest.raises(AssertionError, match="before inputs ready"):
        assert_causality(early)
    with pytest.raises(AssertionError, match="overlap"):
        assert_resource_exclusive(early)
    same = [SimEvent(e.resource, e.start, e.end, e.label, 0, e.layer, e.round) for e in trace]
    with pytest.raises(AssertionError, match="both roles"):
        assert_dual_batch_overlap(same)
    nodraft = [e for e in trace if not (e.label == "draft_decode" and e.round == 3)]
    with pytest.raises(AssertionError, match="no draft"):
        assert_dual_batch_overlap(nodraft)
    assert_dual_batch_overlap(nodraft, allow_verify_only={3})


def test_causality_split_window_parts():
    """Split window: the down part (ffn_gpu_part) is checked against its own
    segment's load (ffn_load_part); starting it before that load ends fails."""
    evs = [SimEvent("IO_C2G", 0.0, 0.010, "ffn_load", 0, 0, 0),
           SimEvent("IO_C2G", 0.010, 0.015, "ffn_load_part", 0, 0, 0),
           SimEvent("GPU_TARGET", 0.0, 0.002, "attn_gpu", 0, 0, 0),
           SimEvent("GPU_TARGET", 0.010, 0.012, "ffn_gpu", 0, 0, 0),
           SimEvent("GPU_TARGET", 0.015, 0.016, "ffn_gpu_part", 0, 0, 0)]
    assert assert_causality(evs) == 2
    early = evs[:4] + [SimEvent("GPU_TARGET", 0.012, 0.016, "ffn_gpu_part", 0, 0, 0)]
    with pytest.raises(AssertionError):
        assert_causality(early)
    with pytest.raises(AssertionError):  # a part with no segment load recorded
        assert_causality([e for e in evs if e.label != "ffn_load_part"])
