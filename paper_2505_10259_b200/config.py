"""Model architectures of the offloaded pair and their byte accounting.

Full-size shapes are the reference presets (pkg/src/specpipe/presets.py:6-11):
Mixtral-8x7B, Mixtral-8x22B (targets, streamed) and Mistral-7B (draft,
HBM-resident).  Speculative decoding needs one vocabulary for both models, so
the draft paired with 8x22B uses V = 32768 (Mistral-7B v0.3).
Byte formulas follow presets.py:28-40 so :meth:`ModelArch.spec` reproduces the
reference ``ModelSpec`` exactly; the router (E×H) and the norms, which the
reference omits, are accounted separately as resident bytes.
"""
from __future__ import annotations

import dataclasses

from .domain import ModelSpec


@dataclasses.dataclass(frozen=True)
class ModelArch:
    name: str
    vocab: int
    hidden: int
    inter: int
    n_layer: int
    n_head: int
    n_kv_head: int
    head_dim: int
    n_expert: int = 0  # 0 = dense SwiGLU MLP
    top_k: int = 2
    rope_theta: float = 1e6
    eps: float = 1e-5
    dtype_bytes: int = 2

    @property
    def qkv_rows(self) -> int:
        return (self.n_head + 2 * self.n_kv_head) * self.head_dim

    @property
    def is_moe(self) -> bool:
        return self.n_expert > 0

    # ---- byte accounting (presets.py:28-40) ----
    def attn_bytes_per_layer(self) -> int:
        kv_dim = self.n_kv_head * self.head_dim
        q_dim = self.n_head * self.head_dim
        # q + o projections and k + v projections
        return self.dtype_bytes * (2 * self.hidden * q_dim + 2 * self.hidden * kv_dim)

    def ffn_bytes_per_layer(self) -> int:
        experts = max(self.n_expert, 1)
        return self.dtype_bytes * 3 * self.hidden * self.inter * experts

    def embed_bytes(self) -> int:
        return self.dtype_bytes * 2 * self.vocab * self.hidden

    def kv_bytes_per_token_per_layer(self) -> int:
        return self.dtype_bytes * 2 * self.n_kv_head * self.head_dim

    def small_resident_bytes(self) -> int:
        """Norm vectors and the router, which the reference presets omit."""
        per_layer = 2 * self.hidden + (self.n_expert * self.hidden if self.is_moe else 0)
        return self.dtype_bytes * (per_layer * self.n_layer + self.hidden)

    def spec(self) -> ModelSpec:
        return ModelSpec(
            name=self.name,
            n_layer=self.n_layer,
            attn_bytes_per_layer=self.attn_bytes_per_layer(),
            ffn_bytes_per_layer=self.ffn_bytes_per_layer(),
            other_bytes=self.embed_bytes(),
            kv_bytes_per_token_per_layer=self.kv_bytes_per_token_per_layer(),
            dtype_bytes=self.dtype_bytes,
        )

    def verify_flops_per_token(self, ctx: int) -> float:
        """Dense-equivalent FLOPs of one verified token (SURVEY.md §8d f_tok)."""
        H, dh = self.hidden, self.head_dim
        q_dim, kv_dim = self.n_head * dh, self.n_kv_head * dh
        proj = 2 * (H * q_dim + 2 * H * kv_dim + q_dim * H)
        ffn = 2 * self.top_k * 3 * H * self.inter if self.is_moe else 2 * 3 * H * self.inter
        router = 2 * H * self.n_expert
        attn = 4 * q_dim * ctx
        return self.n_layer * (proj + ffn + router + attn) + 2 * H * self.vocab


MIXTRAL_8X7B = ModelArch("mixtral-8x7b", 32000, 4096, 14336, 32, 32, 8, 128, n_expert=8)
MIXTRAL_8X22B = ModelArch("mixtral-8x22b", 32768, 6144, 16384, 56, 48, 8, 128, n_expert=8)
MISTRAL_7B = ModelArch("mistral-7b", 32000, 4096, 14336, 32, 32, 8, 128)
MISTRAL_7B_V3 = dataclasses.replace(MISTRAL_7B, name="mistral-7b-v0.3", vocab=32768)

# Tiny synthetic pair: runs on the CPU oracle in
# seconds; head_dim 64 keeps the attention kernel's tile shapes.  The draft
# shares the target's width so tests can tie their embeddings / LM heads and
# get a draft that agrees with the target often enough to exercise every
# accept length (random independent weights accept ≈ 1/V).
TINY_TARGET = ModelArch("tiny-mixtral", 1024, 256, 512, 4, 4, 2, 64, n_expert=8)
TINY_DRAFT = ModelArch("tiny-mistral", 1024, 256, 512, 2, 4, 2, 64)

PAIRS = {
    "tiny": (TINY_TARGET, TINY_DRAFT),
    "8x7b": (MIXTRAL_8X7B, MISTRAL_7B),
    "8x22b": (MIXTRAL_8X22B, MISTRAL_7B_V3),
}


def arch_for_spec(spec) -> ModelArch | None:
    """The architecture whose byte accounting is ``spec`` (any object with the
    reference ModelSpec's fields), or None for a shape this package does not
    know.  Matches on the byte fields, preferring an equal name (Mistral-7B
    and its v0.3 vocabulary differ only in the embedding bytes anyway)."""
    if isinstance(spec, ModelArch):
        return spec
    keys = ("n_layer", "attn_bytes_per_layer", "ffn_bytes_per_layer", "other_bytes", "kv_bytes_per_token_per_layer")
    want = tuple(getattr(spec, k, None) for k in keys)
    hits = [a for a in (MIXTRAL_8X22B, MIXTRAL_8X7B, MISTRAL_7B_V3, MISTRAL_7B, TINY_TARGET, TINY_DRAFT)
            if tuple(getattr(a.spec(), k) for k in keys) == want]
    named = [a for a in hits if a.name == getattr(spec, "name", None)]
    return (named or hits or [None])[0]
