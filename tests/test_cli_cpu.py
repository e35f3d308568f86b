"""The reference-shaped CLI (paper_2505_10259_b200/cli.py, after specpipe's
cli.py:334-398): config schema, presets, pmf, plan; ``simulate`` runs on the
GPU (tests/test_cli_gpu.py)."""
import contextlib
import io
import json
import os
import sys

import pytest

from paper_2505_10259_b200 import cli

REF_SRC = "/root/reference/pkg/src"


def _run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def test_presets_and_emit_config_round_trip(tmp_path):
    rc, out = _run(["presets"])
    assert rc == 0 and "b200_8x22b:" in out and "b200_tiny:" in out
    rc, out = _run(["presets", "--emit-config", "b200_8x22b"])
    assert rc == 0
    doc = json.loads(out)
    cfg = cli.parse_config(doc)
    assert cfg.target_model.name == "mixtral-8x22b" and cfg.workload.l_input == 503
    assert cli.parse_config(cfg.to_dict()).to_dict() == cfg.to_dict()


def test_unknown_key_is_a_config_error(tmp_path):
    p = tmp_path / "c.json"
    doc = json.loads(_run(["presets", "--emit-config", "b200_tiny"])[1])
    doc["bogus"] = 1
    p.write_text(json.dumps(doc))
    rc, _ = _run(["plan", "--config", str(p), "--out", str(tmp_path / "o")])
    assert rc == cli.EXIT_CONFIG


def test_plan_writes_ranking(tmp_path):
    rc, out = _run(["plan", "--preset", "b200_8x22b", "--out", str(tmp_path)])
    assert rc == 0 and "best policy" in out
    rank = json.loads((tmp_path / "ranking.json").read_text())
    thr = [e["throughput"] for e in rank["entries"]]
    assert thr == sorted(thr, reverse=True) and rank["n_feasible"] == len(thr) > 0
    assert json.loads((tmp_path / "meta.json").read_text())["preset"] == "b200_8x22b"


@pytest.fixture(scope="module")
def specpipe():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference sources not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import specpipe as sp
    return sp


def test_pmf_output_matches_reference_cli(specpipe):
    from specpipe import cli as ref_cli

    for p, n in [(0.8, 4), (0.5, 2), (1.0, 8)]:
        rc, ours = _run(["pmf", str(p), str(n)])
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            ref_rc = ref_cli.main(["pmf", str(p), str(n)])
        assert rc == ref_rc == 0 and ours == buf.getvalue()


def test_reference_emitted_config_parses_and_plans(specpipe, tmp_path):
    """A config the reference CLI wrote (its own presets) goes through our plan."""
    from specpipe import cli as ref_cli

    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert ref_cli.main(["presets", "--emit-config", "env1_8x7b"]) == 0
    p = tmp_path / "ref.json"
    p.write_text(buf.getvalue())
    cfg = cli.parse_config(json.loads(buf.getvalue()))
    assert cfg.target_model.n_layer == 32
    rc, out = _run(["plan", "--config", str(p), "--out", str(tmp_path / "o")])
    assert rc == 0, out
