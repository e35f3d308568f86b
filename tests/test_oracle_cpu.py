"""CPU: the oracle is pinned before it is trusted.

* acceptance statistics vs the reference's own outputs (golden file written by
  tests/golden/make_ref_golden.py from the unmodified specpipe);
* model arithmetic vs transformers' Mixtral / Mistral (hf_tiny.npz);
* the C accept/reject restatement vs its specification on teacher-forced
  drafts; det_exp accuracy.
"""
import json
import os

import numpy as np
import pytest

from oracle import accept_ref, decode_ref, model_ref, tiny

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ref():
    with open(os.path.join(GOLD, "ref_specpipe.json")) as f:
        return json.load(f)


def test_pmf_expected_match_reference(ref):
    for row in ref["pmf"]:
        np.testing.assert_array_equal(accept_ref.pmf(row["p"], row["n"]), np.array(row["pmf"]))
    for row in ref["expected"]:
        assert accept_ref.expected_accepted(row["p"], row["n"]) == row["e"]


def test_sample_accepted_draws_match_reference(ref):
    for row in ref["draws"]:
        rng = np.random.default_rng(row["seed"])
        got = accept_ref.sample_accepted(row["p"], row["n"], rng, 64)
        np.testing.assert_array_equal(got, row["counts"])


def test_known_answers():
    # test_acceptance_model.py:13-17 and A2 (E = 1.5 at p=0.5, n=1)
    np.testing.assert_allclose(accept_ref.pmf(0.5, 1), [0.5, 0.5])
    np.testing.assert_allclose(accept_ref.pmf(0.5, 2), [0.5, 0.25, 0.25])
    assert accept_ref.expected_accepted(0.5, 1) == 1.5


def test_model_matches_transformers():
    tw, dw = tiny.weights()
    g = np.load(os.path.join(GOLD, "hf_tiny.npz"))
    for i in range(2):
        p = g[f"prompt{i}"]
        for arch, W, key in ((tiny.TARGET, tw, "target"), (tiny.DRAFT, dw, "draft")):
            kv = model_ref.KV(arch, 1, 64)
            lg = model_ref.forward(arch, W, kv, [0], [p], [0], mirror=False)[0]
            np.testing.assert_allclose(lg, g[f"{key}_logits{i}"], atol=2e-4, rtol=1e-4)


def test_incremental_decode_equals_full_forward():
    """KV-cache decode of the oracle == one causal forward (fp32 mode)."""
    tw, _ = tiny.weights()
    p = tiny.prompts(1, seed=5)[0]
    kv = model_ref.KV(tiny.TARGET, 1, 64)
    full = model_ref.forward(tiny.TARGET, tw, kv, [0], [p], [0], mirror=False)[0]
    kv2 = model_ref.KV(tiny.TARGET, 1, 64)
    model_ref.forward(tiny.TARGET, tw, kv2, [0], [p[:-3]], [0], mirror=False)
    tail = model_ref.forward(tiny.TARGET, tw, kv2, [0], [p[-3:]], [len(p) - 3], mirror=False)[0]
    np.testing.assert_allclose(tail, full[-3:], atol=1e-4, rtol=1e-4)


def test_det_exp_accuracy():
    xs = np.concatenate([np.linspace(-86.9, 88, 20001), [0.0, -1e-8, 1e-8, -0.5, 0.3465]]).astype(np.float32)
    for x in xs[::7]:
        got = np.float32(accept_ref.det_exp(float(x)))
        want = np.float32(np.exp(np.float64(x)))
        ulp = np.spacing(want)
        assert abs(np.float64(got) - np.float64(want)) <= 2 * ulp, (x, got, want)
    assert accept_ref.det_exp(-100.0) == 0.0


def test_accept_greedy_semantics():
    rng = np.random.default_rng(0)
    bs, n, V = 40, 5, 50
    logits = rng.normal(size=(bs, n + 1, V)).astype(np.float32)
    am = logits.argmax(-1)
    k = rng.integers(0, n + 1, bs)
    draft = am[:, :n].copy()
    for s in range(bs):
        if k[s] < n:
            draft[s, k[s]] = (am[s, k[s]] + 1) % V
    rem = rng.integers(0, 8, bs).astype(np.int32)
    tok, cnt = accept_ref.accept_greedy(draft, logits, rem)
    np.testing.assert_array_equal(cnt, np.minimum(k + 1, rem))
    for s in range(bs):
        want = list(draft[s, :k[s]]) + [am[s, k[s]]]
        assert list(tok[s, :cnt[s]]) == want[:cnt[s]]
        assert (tok[s, cnt[s]:] == -1).all()


def test_accept_sample_is_unbiased():
    """Leviathan verification preserves the target distribution (MC, 6σ)."""
    rng = np.random.default_rng(1)
    V, N = 6, 20000
    tl = rng.normal(size=V).astype(np.float32)
    dl = rng.normal(size=V).astype(np.float32)
    logits = np.broadcast_to(np.stack([tl, tl]), (N, 2, V)).copy()
    u_d = rng.random(N, dtype=np.float32)
    draft, q = accept_ref.sample_tokens(np.broadcast_to(dl, (N, V)).copy(), u_d, want_probs=True)
    tok, cnt = accept_ref.accept_sample(draft[:, None], logits, q[:, None, :], rng.random((N, 1), dtype=np.float32),
                                        rng.random(N, dtype=np.float32), np.full(N, 9, np.int32))
    first = tok[:, 0]
    p = np.exp(tl - tl.max())
    p /= p.sum()
    freq = np.bincount(first, minlength=V) / N
    assert np.all(np.abs(freq - p) <= 6 * np.sqrt(p * (1 - p) / N) + 1e-3)


def test_oracle_decode_every_accept_length():
    tw, dw = tiny.weights()
    rec = []
    out, _ = decode_ref.generate(tiny.TARGET, tw, tiny.DRAFT, dw, tiny.prompts(8), 12, 4, 4, record=rec)
    assert all(len(o) == 12 for o in out)
    seen = {int(c) for r in rec for c in r["counts"]}
    assert {1, 2, 5} <= seen
