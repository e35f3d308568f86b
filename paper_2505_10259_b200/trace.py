"""Measured traces in the reference's trace schema.

``SimEvent`` / ``SimResult`` carry the fields of simulator.py:41-60 so the
reference's consumers (``export_trace``-style tooling, tests/_checks-style
invariants) read measured runs unchanged.  Differences: the
single exclusive "GPU" resource is split per CUDA stream — ``GPU_TARGET``
(verification) and ``GPU_DRAFT`` (drafting) genuinely overlap on one B200 — and
labels ``attn_gpu`` / ``accept`` are added; ``IO_C2G`` is the copy stream.
Timestamps come from CUDA events, in seconds from the run's first event.
"""
from __future__ import annotations

import csv
import dataclasses
import io
import json


RESOURCES = ("GPU_TARGET", "GPU_DRAFT", "CPU", "IO_C2G", "IO_G2C", "IO_DISK", "GPU_DECODE")
LABELS = ("attn_gpu", "ffn_load", "ffn_gpu", "draft_prefill", "draft_decode", "accept", "kv_offload",
          "disk_prefetch", "barrier", "prefill", "ffn_decode", "lm_head", "verify",
          # split window (streamer segments): the layer's second segment and the FFN part that reads it
          "ffn_load_part", "ffn_gpu_part")


@dataclasses.dataclass(frozen=True)
class SimEvent:
    resource: str
    start: float
    end: float
    label: str
    batch: int | None = None
    layer: int | None = None
    round: int | None = None


@dataclasses.dataclass
class SimResult:
    trace: list
    total_time: float
    tokens_generated: int
    throughput: float
    peak_gpu_bytes: int
    rounds_executed: int
    per_resource_busy: dict = dataclasses.field(default_factory=dict)
    extra: dict = dataclasses.field(default_factory=dict)


def busy(trace) -> dict:
    out = {r: 0.0 for r in RESOURCES}
    for ev in trace:
        out[ev.resource] = out.get(ev.resource, 0.0) + (ev.end - ev.start)
    return out


class Tracer:
    """Collects (start, end) CUDA-event pairs and resolves them after a sync.

    Events are recorded through the C ABI (``native.Event``) so that marking
    never blocks a host thread while it holds the GIL.
    """

    def __init__(self, enabled: bool = True):
        self.enabled = enabled
        self.t0 = None
        self._pending: list[tuple] = []

    def origin(self, stream) -> None:
        """Start of the measured timeline; work marked before it is dropped."""
        if not self.enabled:
            return
        from . import native

        self._pending.clear()
        self.t0 = native.Event(timing=True).record(stream)

    def mark(self, stream):
        if not self.enabled:
            return None
        from . import native

        return native.Event(timing=True).record(stream)

    def add(self, resource, label, start_ev, end_ev, batch=None, layer=None, rnd=None) -> None:
        if self.enabled and start_ev is not None and end_ev is not None:
            self._pending.append((resource, label, start_ev, end_ev, batch, layer, rnd))

    def resolve(self) -> list[SimEvent]:
        if not self.enabled or self.t0 is None:
            return []
        out = []
        for resource, label, s, e, batch, layer, rnd in self._pending:
            st = self.t0.elapsed_ms(s) * 1e-3
            en = self.t0.elapsed_ms(e) * 1e-3
            out.append(SimEvent(resource, st, max(st, en), label, batch, layer, rnd))
        self._pending.clear()
        return out


def _sorted_events(result: SimResult) -> list:
    return sorted(result.trace, key=lambda e: (e.start, e.resource, e.end, e.label))


def _event_row(ev: SimEvent) -> dict:
    return {"resource": ev.resource, "label": ev.label, "batch": ev.batch, "layer": ev.layer, "round": ev.round,
            "start_s": round(ev.start, 6), "end_s": round(ev.end, 6)}


_CSV_COLUMNS = ["resource", "label", "batch", "layer", "round", "start_s", "end_s"]


def export_trace(result: SimResult, format: str = "json") -> str:
    """Serialise a measured trace exactly as the reference serialises a
    simulated one (simulator.py:282-341): ``json`` and ``csv`` round-trip
    through :func:`parse_trace` at microsecond precision; ``chrome`` is a
    trace-viewer document with one thread per resource (CUDA stream)."""
    events = _sorted_events(result)
    if format == "json":
        resources = list(RESOURCES) + sorted({e.resource for e in events} - set(RESOURCES))
        doc = {
            "total_time_s": round(result.total_time, 6),
            "tokens_generated": result.tokens_generated,
            "throughput": round(result.throughput, 6),
            "peak_gpu_bytes": result.peak_gpu_bytes,
            "rounds_executed": result.rounds_executed,
            "per_resource_busy_s": {r: round(result.per_resource_busy.get(r, 0.0), 6) for r in resources},
            "events": [_event_row(e) for e in events],
        }
        return json.dumps(doc, sort_keys=True, indent=2) + "\n"
    if format == "csv":
        buf = io.StringIO()
        w = csv.DictWriter(buf, fieldnames=_CSV_COLUMNS, lineterminator="\n")
        w.writeheader()
        for e in events:
            row = _event_row(e)
            row["start_s"] = f"{row['start_s']:.6f}"
            row["end_s"] = f"{row['end_s']:.6f}"
            w.writerow({k: ("" if row[k] is None else row[k]) for k in _CSV_COLUMNS})
        return buf.getvalue()
    if format == "chrome":
        return export_chrome(result)
    raise ValueError(f"unknown trace format '{format}'")


def parse_trace(doc: str, format: str = "json") -> SimResult:
    """Inverse of :func:`export_trace` for json and csv (simulator.py:344-391):
    csv carries only events, so its totals are rebuilt from them."""
    if format == "json":
        data = json.loads(doc)
        events = [SimEvent(resource=r["resource"], start=r["start_s"], end=r["end_s"], label=r["label"],
                           batch=r["batch"], layer=r["layer"], round=r["round"]) for r in data["events"]]
        return SimResult(trace=events, total_time=data["total_time_s"], tokens_generated=data["tokens_generated"],
                         throughput=data["throughput"], peak_gpu_bytes=data["peak_gpu_bytes"],
                         rounds_executed=data["rounds_executed"], per_resource_busy=dict(data["per_resource_busy_s"]))
    if format == "csv":
        events = []
        for r in csv.DictReader(io.StringIO(doc)):
            events.append(SimEvent(resource=r["resource"], start=float(r["start_s"]), end=float(r["end_s"]),
                                   label=r["label"], batch=int(r["batch"]) if r["batch"] else None,
                                   layer=int(r["layer"]) if r["layer"] else None,
                                   round=int(r["round"]) if r["round"] else None))
        return SimResult(trace=events, total_time=max((e.end for e in events), default=0.0), tokens_generated=0,
                         throughput=0.0, peak_gpu_bytes=0, rounds_executed=0, per_resource_busy=busy(events))
    raise ValueError(f"unknown trace format '{format}'")


def export_json(result: SimResult) -> str:
    return export_trace(result, "json")


def export_chrome(result: SimResult) -> str:
    tids = {r: i for i, r in enumerate(RESOURCES)}
    evs = [{"name": e.label, "ph": "X", "pid": 0, "tid": tids.get(e.resource, 99), "ts": round(e.start * 1e6, 3),
            "dur": round((e.end - e.start) * 1e6, 3), "args": {"batch": e.batch, "layer": e.layer, "round": e.round}}
           for e in result.trace]
    meta = [{"name": "thread_name", "ph": "M", "pid": 0, "tid": i, "args": {"name": r}} for r, i in tids.items()]
    return json.dumps({"traceEvents": meta + evs}, indent=1) + "\n"
