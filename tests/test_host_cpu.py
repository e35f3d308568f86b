"""CPU: host-side logic of the product package and the C-ABI library surface."""
import json
import os
import re

import numpy as np
import pytest
import torch

from paper_2505_10259_b200 import (MIXTRAL_8X7B, MIXTRAL_8X22B, MISTRAL_7B, AcceptanceModel, Policy, Workload,
                                   acceptance, expected_accepted, native, pmf, sample_accepted)
from paper_2505_10259_b200.errors import ValidationError
from paper_2505_10259_b200.kvcache import PagedKVCache
from paper_2505_10259_b200.weights import ffn_offsets, interleave_gate_up, pack_ffn

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden", "ref_specpipe.json")


def test_library_exports_every_header_symbol(native_lib):
    header = open(os.path.join(ROOT, "include", "specoffload_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(so_\w+)\s*\(", header, re.M))
    assert declared == set(native.exported_symbols())
    for name in declared:
        assert hasattr(native_lib, name)
    assert native_lib.so_abi_version() == 1
    assert native_lib.so_status_string(-2) == b"invalid shape or size argument"


def test_argument_validation_without_gpu(native_lib):
    # shape errors are reported before any CUDA call
    assert native_lib.so_gemm_bf16(None, None, 1, 1, 1, None, 1, 0, None, None) == -1
    assert native_lib.so_accept_greedy(1, 1, 1, None, 4, 0, 10, 1, 1, None) == -2
    assert native_lib.so_attn_paged(1, 16, 16, 1, 1, 1, 1, 1, 1, 8, 3, 128, 16, 1.0, 1, None) == -2  # hq % hkv


def test_acceptance_matches_reference_golden():
    ref = json.load(open(GOLD))
    for row in ref["pmf"]:
        np.testing.assert_array_equal(pmf(AcceptanceModel(row["p"], row["n"])), row["pmf"])
    for row in ref["expected"]:
        assert expected_accepted(AcceptanceModel(row["p"], row["n"])) == row["e"]
    for row in ref["draws"]:
        got = sample_accepted(AcceptanceModel(row["p"], row["n"]), np.random.default_rng(row["seed"]), 64)
        np.testing.assert_array_equal(got, row["counts"])


def test_model_spec_matches_reference_presets():
    ref = json.load(open(GOLD))["presets"]
    for arch, key in ((MIXTRAL_8X22B, "mixtral_8x22b"), (MIXTRAL_8X7B, "mixtral_8x7b"), (MISTRAL_7B, "mistral_7b")):
        spec = arch.spec()
        for field in ("n_layer", "attn_bytes_per_layer", "ffn_bytes_per_layer", "other_bytes",
                      "kv_bytes_per_token_per_layer"):
            assert getattr(spec, field) == ref[key][field], (key, field)
    assert ffn_offsets(MIXTRAL_8X22B)[2] == 4_831_838_208


def test_policy_and_workload_validation():
    with pytest.raises(ValidationError):
        Policy(16, 8, 16, 4)   # bs_draft > bs_decoding
    with pytest.raises(ValidationError):
        Policy(17, 8, 8, 4)    # bs_prefill > 2·bs_decoding
    with pytest.raises(ValidationError):
        Workload(1, 1, 1, 1.5)
    assert Policy(1, 2, 3 - 1, 4).as_tuple() == (1, 2, 2, 4)


def test_gate_up_interleave_layout():
    I, H = 128, 4
    g = torch.arange(I * H, dtype=torch.float32).view(I, H)
    u = -g
    gu = interleave_gate_up(g, u)
    assert torch.equal(gu[0:64], g[0:64]) and torch.equal(gu[64:128], u[0:64])
    assert torch.equal(gu[128:192], g[64:128]) and torch.equal(gu[192:256], u[64:128])
    flat = pack_ffn(g, u, torch.zeros(H, I))
    assert flat.numel() == 3 * I * H and flat.dtype == torch.bfloat16


def test_paged_slots():
    from paper_2505_10259_b200 import TINY_TARGET

    kv = PagedKVCache(TINY_TARGET, 3, 130, "cpu", page_size=64)
    assert kv.pages_per_seq == 3
    s = kv.slots(np.array([0, 1, 2, 2]), np.array([0, 64, 129, 5]))
    np.testing.assert_array_equal(s, [0, 3 * 64 + 64, 6 * 64 + 129, 6 * 64 + 5])


def test_input_uniforms_shared_with_oracle():
    from oracle import decode_ref

    a = acceptance.input_uniforms(3, 4, 1, 2, (5, 2))
    b = decode_ref.uniforms(3, 4, 1, 2, (5, 2))
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(acceptance.forced_counts(1, 2, 0, 0.8, 4, 9),
                                  decode_ref.forced_counts(1, 2, 0, 0.8, 4, 9))


def test_disk_tier_file_round_trip(tmp_path):
    """DiskTier stores units at 2 MiB-aligned offsets and its parallel reader
    splits every unit into pieces that cover it exactly (any size)."""
    import numpy as np
    import torch

    from paper_2505_10259_b200.streamer import DiskTier

    d = DiskTier(str(tmp_path / "units.bin"))
    rng = np.random.default_rng(0)
    data = {li: torch.from_numpy(rng.integers(0, 256, n, dtype=np.uint8)) for li, n in
            ((0, 1000), (3, 3 * (1 << 20) + 7), (5, 17 * (1 << 21) + 1))}
    refs = {li: d.write(li, t) for li, t in data.items()}
    assert all(off % DiskTier.ALIGN == 0 for off, _ in d.entries.values())
    for li, t in data.items():
        off, n = d.entries[li]
        out = np.zeros(n, np.uint8)
        mv = memoryview(out)
        rs = d.pieces(n)
        assert len(rs) <= d.READERS and rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        for lo, hi in rs:
            d._read(mv, off, lo, hi)
        assert np.array_equal(out, t.numpy()) and refs[li].nbytes == n
    d.close()


def test_import_changes_no_process_state_and_work_queues_are_explicit():
    """Importing the package leaves CUDA_DEVICE_MAX_CONNECTIONS alone (other
    frameworks pin it); reserve_work_queues() sets it only when unset and only
    before the CUDA context exists."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k != "CUDA_DEVICE_MAX_CONNECTIONS"}
    code = ("import os, paper_2505_10259_b200 as p; assert 'CUDA_DEVICE_MAX_CONNECTIONS' not in os.environ; "
            "assert p.reserve_work_queues(32); assert os.environ['CUDA_DEVICE_MAX_CONNECTIONS'] == '32'; "
            "assert not p.reserve_work_queues(16); assert os.environ['CUDA_DEVICE_MAX_CONNECTIONS'] == '32'")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_committed_per_verify_matches_monte_carlo():
    """acceptance.committed_per_verify (the bench's steady state of max_new-token
    requests, commits clamped to what is left, simulator.py:213-214) against a
    direct simulation with the reference-identical sampler."""
    import numpy as np

    from paper_2505_10259_b200.acceptance import (AcceptanceModel, committed_per_verify, expected_accepted,
                                                  sample_accepted)

    rng = np.random.default_rng(5)
    for p, n, max_new in [(0.8, 8, 16), (0.6, 4, 16), (0.9, 8, 128), (0.5, 2, 7)]:
        m = AcceptanceModel(p, n)
        verifies = tokens = 0
        for _ in range(4000):
            left = max_new
            while left > 0:
                c = min(int(sample_accepted(m, rng)), left)
                left -= c
                tokens += c
                verifies += 1
        mc = tokens / verifies
        exact = committed_per_verify(m, max_new)
        assert abs(mc - exact) < 0.02 * exact, (p, n, max_new, mc, exact)
        assert exact <= expected_accepted(m) + 1e-12
    assert committed_per_verify(AcceptanceModel(0.8, 8), 0) == expected_accepted(AcceptanceModel(0.8, 8))
