"""ORACLE — test infrastructure only.  The tiny synthetic pair of config 1
(BASELINE.json configs[0]) with the deterministic weights every parity test,
the HF golden file and smoke() share.
"""
from __future__ import annotations

import numpy as np

from .model_ref import Arch, init_weights

TARGET = Arch(vocab=1024, hidden=256, inter=512, n_layer=4, n_head=4, n_kv_head=2, head_dim=64, n_expert=8)
DRAFT = Arch(vocab=1024, hidden=256, inter=512, n_layer=2, n_head=4, n_kv_head=2, head_dim=64, n_expert=0)
TARGET_SEED, DRAFT_SEED = 11, 12


def weights(layer_std: float = 0.02):
    tw = init_weights(TARGET, TARGET_SEED, std=layer_std)
    dw = init_weights(DRAFT, DRAFT_SEED, std=layer_std)
    # tie the draft's vocabulary projection to the target's so the two agree
    # on most tokens (a distilled draft, in miniature)
    dw["embed"] = tw["embed"].copy()
    dw["lm_head"] = tw["lm_head"].copy()
    dw["final_norm"] = tw["final_norm"].copy()
    return tw, dw


def prompts(n: int, seed: int = 1234, lo: int = 5, hi: int = 24) -> list[np.ndarray]:
    rng = np.random.default_rng(seed)
    return [rng.integers(0, TARGET.vocab, int(rng.integers(lo, hi))).astype(np.int32) for _ in range(n)]
