"""User-facing construction of the offloaded target/draft pair.

``build_engine`` is what a caller of the reference would reach for after
``assign_tiers`` (placement.py:167): it takes the target FFN layers the plan
streams (the rest stay pinned in HBM), places the streamed ones in pinned host
memory, creates the two-or-more-slot HBM window and returns an ``Engine``.
"""
from __future__ import annotations

import tempfile
import weakref

import torch

from . import codec as C
from . import weights as W
from .config import ModelArch
from .engine import Engine
from .models import DraftModel, TargetModel
from .streamer import DiskRef, DiskTier, HostStore, LayerStreamer, SharedHostStore


def build_engine(target_arch: ModelArch, draft_arch: ModelArch, target_weights: dict | None = None,
                 draft_weights: dict | None = None, device="cuda:0", stream_layers=None, n_slots: int = 2,
                 seed: int = 0, trace: bool = True, page_size: int = 32, host_store: HostStore | None = None,
                 chunk_bytes: int = 256 << 20, rank: int = 0, world: int = 1, group=None,
                 shared_store: SharedHostStore | None = None, stream_attn: bool = False,
                 codec: str = "none", shard_layers=None, disk_layers=None, disk_path: str | None = None,
                 arith: str = "tensor", split_window: bool = False) -> Engine:
    """Build an engine.  ``*_weights`` are logical (HF-shaped) arrays; None =
    synthetic random init of the architecture.  ``stream_layers`` = target
    FFN layers kept in pinned host DRAM and streamed each pass (default:
    all of them — the fully offloaded configuration).  With ``world > 1`` the
    streamed layers live once in ``shared_store`` and each rank pulls its
    1/N slice, reassembled by an NCCL all-gather.
    ``codec="xc4"`` keeps the streamed units XC4-encoded in host DRAM (K9:
    0.70–0.75 of the bytes cross the link, decoded bit-exactly on the GPU).
    ``shard_layers`` (world > 1): layers kept 1/N per GPU in
    HBM and rebuilt each pass by an NVLink all-gather instead of the host link.
    ``disk_layers`` (§8 f4): streamed layers kept in a file at ``disk_path``
    (default: a temporary file) and staged through pinned DRAM each pass.
    ``arith="canonical"`` runs both models through the parity-mode kernels
    (fixed IEEE order, bit-identical to the CPU oracle; tiny shapes only).
    ``split_window``: each streamed unit moves as [(attention +) gate_up | down]
    into its own slot, so the HBM window is one unit instead of ``n_slots``
    units (single GPU, host DRAM; the link still runs a unit ahead)."""
    if codec not in ("none", "xc4"):
        raise ValueError(f"unknown codec {codec!r}")
    dev = torch.device(device)
    if stream_layers is None:
        stream_layers = set(range(target_arch.n_layer))
    stream_layers = set(stream_layers)
    shard_layers = set(shard_layers or ())
    if shard_layers and world < 2:
        raise ValueError("shard_layers needs world > 1")
    stream_layers -= shard_layers
    disk_layers = set(disk_layers or ()) & stream_layers
    disk = None
    if disk_layers:
        if world > 1:
            raise ValueError("the disk tier is single-GPU (the N-GPU host store is shared DRAM)")
        if target_weights is not None:
            raise ValueError("disk_layers is supported for synthetic weights")
        if disk_path is None:
            with tempfile.NamedTemporaryFile(prefix="specoffload_disk_", suffix=".bin", delete=False) as f:
                disk_path = f.name
        disk = DiskTier(disk_path)
    segments = W.unit_segments(target_arch, stream_attn, split_window)
    if split_window and (world > 1 or shard_layers or disk_layers):
        raise ValueError("split_window is single-GPU and host-DRAM only")
    enc = C.Encoder(dev) if codec == "xc4" and stream_layers else None
    if target_weights is not None:
        store = host_store or HostStore()
        tw = W.from_logical(target_arch, target_weights, dev, stream_layers, stream_attn, encoder=enc,
                            host_alloc=store.alloc, segments=segments)
    elif shared_store is not None:
        sink = shared_store.write_coded if enc is not None else shared_store.write_slice
        tw = W.synthetic(target_arch, dev, seed=seed, stream_layers=stream_layers, host_sink=sink,
                         stream_attn=stream_attn, encoder=enc, shard_layers=shard_layers, shard=(rank, world))
    else:
        store = host_store or HostStore()
        tw = W.synthetic(target_arch, dev, seed=seed, stream_layers=stream_layers, host_alloc=store.alloc,
                         stream_attn=stream_attn, encoder=enc, shard_layers=shard_layers, shard=(rank, world),
                         disk=disk, disk_layers=disk_layers, segments=segments)
    if enc is not None:
        enc.release()
        torch.cuda.empty_cache()  # hand the encoder's staging back before KV / workspaces are sized
    if draft_weights is not None:
        dw = W.from_logical(draft_arch, draft_weights, dev)
    else:
        dw = W.synthetic(draft_arch, dev, seed=seed + 1)
    _, ffn_bytes = W.unit_layout(target_arch, stream_attn)  # bytes of one streamed layer unit
    resident = {li: L.ffn for li, L in enumerate(tw.layers) if L.ffn is not None}
    host = {li: t if isinstance(t, (C.XC4Unit, C.XC4Parts, DiskRef)) else t.view(torch.uint8)
            for li, t in tw.host_ffn.items()}
    streamer = LayerStreamer(ffn_bytes, resident, host, target_arch.n_layer, dev, n_slots=n_slots,
                             chunk_bytes=chunk_bytes, rank=rank, world=world, group=group,
                             shards=tw.shard_ffn, disk=disk, segments=segments) if (host or tw.shard_ffn) else None
    if disk is not None:
        weakref.finalize(streamer, disk.close)
    target = TargetModel(tw, dev, streamer, arith=arith)
    draft = DraftModel(dw, dev, arith=arith)
    eng = Engine(target, draft, device=dev, page_size=page_size, trace=trace)
    # host-resident KV pools (DecodeSession kv_host) come from the same exact-size page-locked store
    eng.host_alloc = (host_store or HostStore()).alloc if shared_store is None else None
    return eng
