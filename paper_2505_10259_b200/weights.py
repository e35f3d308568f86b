"""Weight containers and the device/host layouts the kernels consume.

Logical weights follow the Mixtral/Mistral parameterisation
(wq/wk/wv/wo, attn/ffn RMSNorm, router, per-expert w_gate/w_up/w_down).
Physical layouts:
  * wqkv     [(hq+2·hkv)·dh, H]    one K-major GEMM operand for Q, K and V;
  * FFN layer, one contiguous buffer — the unit the streamer moves:
        gate_up [E, 2I, H]  gate/up rows interleaved in 64-row blocks so one
                            tcgen05 N-tile holds matching gate and up rows and
                            the SwiGLU is fused into the GEMM epilogue;
        down    [E, H, I]
    Its byte size equals the reference's ffn_bytes_per_layer
    (presets.py:33-35: 2·3·H·I·E) exactly.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import codec
from .config import ModelArch

SWIGLU_BLOCK = 64


def _bf16(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    """[.., I, H] ×2 → [.., 2I, H] with 64-row gate/up blocks alternating."""
    *lead, I, H = w_gate.shape
    assert I % SWIGLU_BLOCK == 0
    g = w_gate.reshape(*lead, I // SWIGLU_BLOCK, 1, SWIGLU_BLOCK, H)
    u = w_up.reshape(*lead, I // SWIGLU_BLOCK, 1, SWIGLU_BLOCK, H)
    return torch.cat([g, u], dim=-3).reshape(*lead, 2 * I, H)


def pack_ffn(w_gate, w_up, w_down) -> torch.Tensor:
    """Flat bf16 buffer [gate_up | down] of one layer (E leading, or dense)."""
    gu = interleave_gate_up(_bf16(w_gate), _bf16(w_up))
    return torch.cat([gu.reshape(-1), _bf16(w_down).reshape(-1)])


def ffn_offsets(arch: ModelArch) -> tuple[int, int, int]:
    """(elements of gate_up, elements of down, total bytes) of one layer."""
    E = max(arch.n_expert, 1)
    gu = E * 2 * arch.inter * arch.hidden
    dn = E * arch.hidden * arch.inter
    return gu, dn, (gu + dn) * 2


def attn_elems(arch: ModelArch) -> int:
    """bf16 elements of one layer's attention projections (Wqkv + Wo)."""
    return arch.qkv_rows * arch.hidden + arch.hidden * arch.n_head * arch.head_dim


def unit_layout(arch: ModelArch, stream_attn: bool) -> tuple[int, int]:
    """(byte offset of the FFN inside a streamed layer unit, unit bytes).

    The streamed unit is the FFN alone, or [Wqkv | Wo | FFN] when the HBM
    budget cannot hold the attention weights either (the
    8x7B config capped at 24 GB)."""
    ffn_bytes = ffn_offsets(arch)[2]
    if not stream_attn:
        return 0, ffn_bytes
    a = attn_elems(arch) * 2
    return a, a + ffn_bytes


def unit_segments(arch: ModelArch, stream_attn: bool, split: bool) -> list[tuple[int, int]]:
    """Byte ranges the streamer moves a unit in: the whole unit, or (split
    window) [attention projections (if streamed) + gate_up | down] — the
    layer reads the first range up to its gate_up GEMM and the second only in
    its down GEMM (streamer.py)."""
    off, total = unit_layout(arch, stream_attn)
    if not split:
        return [(0, total)]
    cut = off + 2 * ffn_offsets(arch)[0]  # [Wqkv | Wo |] gate_up  ‖  down
    return [(0, cut), (cut, total)]


@dataclasses.dataclass
class LayerWeights:
    attn_norm: torch.Tensor
    wqkv: torch.Tensor | None  # None when the attention weights stream with the layer
    wo: torch.Tensor | None
    ffn_norm: torch.Tensor
    router: torch.Tensor | None
    ffn: torch.Tensor | None  # packed FFN when HBM-resident (None when host-streamed)


@dataclasses.dataclass
class ModelWeights:
    arch: ModelArch
    embed: torch.Tensor
    final_norm: torch.Tensor
    lm_head: torch.Tensor
    layers: list[LayerWeights]
    host_ffn: dict  # layer -> pinned host buffer, or codec.XC4Unit (streamed layers)
    shard_ffn: dict = dataclasses.field(default_factory=dict)  # layer -> this rank's HBM shard (f3)

    def resident_bytes(self) -> int:
        n = self.embed.numel() + self.final_norm.numel() + self.lm_head.numel()
        for L in self.layers:
            for t in (L.attn_norm, L.wqkv, L.wo, L.ffn_norm, L.router, L.ffn):
                if t is not None:
                    n += t.numel()
        return 2 * n


def from_logical(arch: ModelArch, W: dict, device, stream_layers: set[int] = frozenset(),
                 stream_attn: bool = False, encoder=None, host_alloc=None, segments=None) -> ModelWeights:
    """Build device weights from logical (HF-shaped) arrays — numpy or torch.
    With ``encoder`` (codec.Encoder) the streamed units are kept XC4-encoded.
    Streamed units go to ``host_alloc(nbytes)`` (e.g. HostStore.alloc: exact-size
    page-locked mmaps) — torch's pinned allocator would round each unit up to a
    power of two and cache it (8 GiB per 5 GB 8x22B layer).  ``segments``
    (split window): byte ranges encoded as independent XC4 units."""
    dev = torch.device(device)
    layers = []
    host = {}
    for li, L in enumerate(W["layers"]):
        wqkv = torch.cat([_bf16(L["wq"]), _bf16(L["wk"]), _bf16(L["wv"])], dim=0).contiguous()
        wo = _bf16(L["wo"]).contiguous()
        packed = pack_ffn(L["w_gate"], L["w_up"], L["w_down"])
        if li in stream_layers:
            if stream_attn:
                packed = torch.cat([wqkv.reshape(-1), wo.reshape(-1), packed])
                wqkv = wo = None
            if encoder is not None:
                host[li] = codec.encode_segments_to_host(packed.to(dev), encoder, segments, host_alloc)
            elif dev.type != "cuda":
                host[li] = packed
            elif host_alloc is not None:
                buf = host_alloc(packed.numel() * 2).view(torch.bfloat16)[: packed.numel()]
                buf.copy_(packed)
                host[li] = buf
            else:
                host[li] = packed.pin_memory()
            ffn = None
        else:
            ffn = packed.to(dev)
        layers.append(LayerWeights(
            attn_norm=_bf16(L["attn_norm"]).to(dev),
            wqkv=wqkv.to(dev) if wqkv is not None else None,
            wo=wo.to(dev) if wo is not None else None,
            ffn_norm=_bf16(L["ffn_norm"]).to(dev),
            router=_bf16(L["router"]).to(dev).contiguous() if arch.is_moe else None,
            ffn=ffn,
        ))
    return ModelWeights(arch, _bf16(W["embed"]).to(dev).contiguous(), _bf16(W["final_norm"]).to(dev),
                        _bf16(W["lm_head"]).to(dev).contiguous(), layers, host)


def synthetic(arch: ModelArch, device, seed: int = 0, stream_layers: set[int] = frozenset(),
              host_alloc=None, std: float = 0.02, host_sink=None, stream_attn: bool = False,
              encoder=None, shard_layers: set[int] = frozenset(), shard: tuple[int, int] = (0, 1),
              disk=None, disk_layers: set[int] = frozenset(), segments=None) -> ModelWeights:
    """Random-init weights of the given shape (N(0, 0.02²), norms = 1).

    Generated on the GPU; streamed FFN layers are generated in HBM one at a
    time and copied into pinned host buffers from ``host_alloc(nbytes)`` — or
    handed to ``host_sink(layer, tensor) -> host view`` (multi-GPU: each rank
    writes only its slice of the shared store; every rank draws the same
    weights from the same seed).  With ``encoder`` (codec.Encoder) streamed
    units are XC4-encoded on the GPU first and the host keeps the encoding
    (the sink then receives the encoded device bytes).  ``shard_layers`` (f3,
    N > 1): this rank keeps only its ``slice_bounds`` share of the layer unit in
    HBM; the streamer all-gathers the shards every pass.  ``disk_layers``
    (with ``disk``, a streamer.DiskTier; §8 f4): streamed units written to
    the disk tier's file instead of pinned DRAM.
    """
    from .streamer import slice_bounds
    dev = torch.device(device)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)

    def randn(*shape):
        t = torch.empty(*shape, dtype=torch.bfloat16, device=dev)
        t.normal_(0.0, std, generator=g)
        return t

    ones = lambda n: torch.ones(n, dtype=torch.bfloat16, device=dev)  # noqa: E731
    _, _, ffn_bytes = ffn_offsets(arch)
    layers = []
    host = {}
    shards = {}
    for li in range(arch.n_layer):
        sharded = li in shard_layers
        streamed = li in stream_layers or sharded
        with_attn = streamed and stream_attn
        unit = randn((ffn_bytes + (attn_elems(arch) * 2 if with_attn else 0)) // 2)
        if sharded:
            lo, hi = slice_bounds(unit.numel() * 2, *shard)
            shards[li] = unit.view(torch.uint8)[lo:hi].clone()
        elif streamed and li in disk_layers:
            if encoder is not None:
                enc = encoder.encode(unit)[0]
                host[li] = disk.write(li, enc, dataclasses.replace(codec.XC4Unit.parse(enc), data=None))
            else:
                host[li] = disk.write(li, unit)
        elif streamed and encoder is not None:
            if host_sink is not None:
                host[li] = host_sink(li, encoder.encode(unit)[0])
            else:
                host[li] = codec.encode_segments_to_host(unit, encoder, segments, host_alloc)
        elif streamed and host_sink is not None:
            host[li] = host_sink(li, unit).view(torch.bfloat16)
        elif streamed:
            buf = host_alloc(unit.numel() * 2) if host_alloc is not None else torch.empty(
                unit.numel(), dtype=torch.bfloat16, pin_memory=True)
            buf = buf.view(torch.bfloat16)
            buf.copy_(unit)
            host[li] = buf
        ffn = None if streamed else unit
        del unit
        layers.append(LayerWeights(
            attn_norm=ones(arch.hidden),
            wqkv=None if with_attn else randn(arch.qkv_rows, arch.hidden),
            wo=None if with_attn else randn(arch.hidden, arch.n_head * arch.head_dim),
            ffn_norm=ones(arch.hidden),
            router=randn(arch.n_expert, arch.hidden) if arch.is_moe else None,
            ffn=ffn,
        ))
    torch.cuda.synchronize(dev) if dev.type == "cuda" else None
    return ModelWeights(arch, randn(arch.vocab, arch.hidden), ones(arch.hidden), randn(arch.vocab, arch.hidden),
                        layers, host, shards)
