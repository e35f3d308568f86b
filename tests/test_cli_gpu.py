"""``simulate`` of the reference-shaped CLI runs the policy on the GPU and
writes the measured trace in the reference's formats (cli.py:160-207)."""
import contextlib
import io
import json

import pytest

from paper_2505_10259_b200 import cli
from paper_2505_10259_b200.trace import parse_trace

from _trace_checks import assert_causality, assert_dual_batch_overlap, assert_resource_exclusive

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fmt", ["json", "csv"])
def test_simulate_writes_measured_trace(tmp_path, fmt):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(["simulate", "--preset", "b200_tiny", "--policy", "8,8,4,4", "--max-rounds", "6",
                       "--format", fmt, "--out", str(tmp_path)])
    assert rc == 0, buf.getvalue()
    assert buf.getvalue().startswith("measured ")
    summary = json.loads((tmp_path / "summary.json").read_text())
    assert summary["measured"] and summary["rounds_executed"] == 6 and summary["tokens_generated"] > 0
    res = parse_trace((tmp_path / f"trace.{fmt}").read_text(), fmt)
    assert res.trace
    assert_resource_exclusive(res.trace)
    assert_causality(res.trace)
    assert_dual_batch_overlap(res.trace)


def test_simulate_8x22b_shapes_truncated(tmp_path):
    """configs[2] shapes, 2 target + 2 draft layers, planner-placed (streamed) layers."""
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(["simulate", "--preset", "b200_8x22b", "--policy", "32,32,16,4", "--layers", "2",
                       "--max-rounds", "4", "--out", str(tmp_path)])
    assert rc == 0, buf.getvalue()
    summary = json.loads((tmp_path / "summary.json").read_text())
    assert summary["layers"] == [2, 2] and summary["throughput"] > 0
