"""CPU, world_size 2 over gloo: the host-side logic of the N-GPU path
 — one shared host copy of a streamed layer, each rank writing
and pushing only its 1/N slice, the in-place all-gather rebuilding the full
layer on every rank."""
import os
import uuid

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_10259_b200.streamer import SharedHostStore, gather_layer, slice_bounds

LAYER = 4096 * 2 * 6  # bytes; splits into page-aligned halves


def _worker(rank: int, world: int, port: int, name: str, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        store = SharedHostStore(name, [3, 7], LAYER, rank, world, barrier=dist.barrier)
        g = torch.Generator().manual_seed(0)  # every rank draws the same weights
        full = {li: torch.randint(0, 256, (LAYER,), dtype=torch.uint8, generator=g) for li in (3, 7)}
        for li in (3, 7):
            store.write_slice(li, full[li])
        dist.barrier()
        ok = True
        for li in (3, 7):
            # the shared file now holds the whole layer, written half by each rank
            ok &= torch.equal(store.layer_view(li), full[li])
            # streamer step: push my slice into the window slot, then all-gather
            slot = torch.zeros(LAYER, dtype=torch.uint8)
            lo, hi = slice_bounds(LAYER, rank, world)
            slot[lo:hi].copy_(store.layer_view(li)[lo:hi])
            gather_layer(slot, rank, world)
            ok &= torch.equal(slot, full[li])
        dist.barrier()
        store.close(unlink=rank == 0)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_shared_store_slices_and_allgather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    name = f"specoffload_test_{uuid.uuid4().hex[:8]}"
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert results == {0: True, 1: True}
    assert not os.path.exists(f"/dev/shm/{name}")


def test_slice_bounds():
    assert slice_bounds(4_831_838_208, 7, 8) == (7 * 603_979_776, 8 * 603_979_776)
    with pytest.raises(ValueError):
        slice_bounds(4096 * 3, 0, 2)  # halves are not page-aligned


N_ELEMS = 8 * 4096 * 6  # one XC4 unit: 12 frames of 16 Ki weights → 6 per rank


def _coded_worker(rank: int, world: int, port: int, name: str, q):
    import numpy as np

    from oracle import xc4_ref
    from paper_2505_10259_b200.codec import XC4Unit

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)  # every rank draws (and encodes) the same weights
        raw = {li: (rng.normal(0, 0.02, N_ELEMS).astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
               for li in (3, 7)}
        units = {li: xc4_ref.encode(w, 4 * 4096) for li, w in raw.items()}
        cap = max(u.size for u in units.values()) + 4096
        store = SharedHostStore(name, [3, 7], cap, rank, world, barrier=dist.barrier, coded=True)
        ok = True
        mine = {}
        for li in (3, 7):
            u = store.write_coded(li, torch.from_numpy(units[li]))
            f0, f1 = u.frame_range(rank, world)
            # this rank's frames decode to exactly its 1/N byte slice of the layer
            ok &= (f0 * u.frame_elems * 2, f1 * u.frame_elems * 2) == slice_bounds(2 * N_ELEMS, rank, world)
            mine[li] = u.frame_bytes(f0, f1)
        dist.barrier()
        for li in (3, 7):
            # header + frames written by both ranks: the shared file holds the whole unit
            view = store.layer_view(li)[: units[li].size]
            ok &= bool(np.array_equal(view.numpy(), units[li]))
            dec = xc4_ref.decode(view.numpy())
            # streamer step: my decoded slice into the slot, then the all-gather
            slot = torch.zeros(2 * N_ELEMS, dtype=torch.uint8)
            lo, hi = slice_bounds(2 * N_ELEMS, rank, world)
            slot[lo:hi].copy_(torch.from_numpy(dec.view(np.uint8)[lo:hi]))
            gather_layer(slot, rank, world)
            ok &= bool(np.array_equal(slot.numpy().view(np.uint16), raw[li]))
            ok &= XC4Unit.parse(view).n_frames == 12
        dist.barrier()
        store.close(unlink=rank == 0)
        q.put((rank, (bool(ok), sum(mine.values()))))
    finally:
        dist.destroy_process_group()


def test_shared_store_xc4_frames_and_allgather():
    """N-GPU path with XC4 units: every rank writes the header and only its
    frames, moves ≈1/N of the encoded bytes, and the all-gather of the decoded
    slices rebuilds the exact layer."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 2000)
    name = f"specoffload_test_{uuid.uuid4().hex[:8]}"
    procs = [ctx.Process(target=_coded_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert results[0][0] and results[1][0]
    # each rank's share of the link bytes is about half of the encoded layers
    assert abs(results[0][1] - results[1][1]) < 0.01 * results[0][1]
    assert not os.path.exists(f"/dev/shm/{name}")


def _shard_worker(rank: int, world: int, port: int, q):
    from paper_2505_10259_b200 import TINY_TARGET
    from paper_2505_10259_b200 import weights as W
    from paper_2505_10259_b200.streamer import gather_shards

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = W.synthetic(TINY_TARGET, "cpu", seed=3)                        # every layer resident
        sh = W.synthetic(TINY_TARGET, "cpu", seed=3, shard_layers={1, 2}, shard=(rank, world))
        ok = set(sh.shard_ffn) == {1, 2} and sh.layers[1].ffn is None and sh.layers[0].ffn is not None
        for li in (1, 2):
            unit = full.layers[li].ffn.view(torch.uint8)
            lo, hi = slice_bounds(unit.numel(), rank, world)
            ok &= torch.equal(sh.shard_ffn[li], unit[lo:hi])                  # this rank keeps its 1/N
            slot = torch.zeros_like(unit)
            gather_shards(slot, sh.shard_ffn[li])                             # f3: the per-pass all-gather
            ok &= torch.equal(slot, unit)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_hbm_sharded_layers_allgather():
    """layers kept 1/N per rank (same seed → same weights on
    every rank) rebuild bit-exactly from the ranks' shards."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 33500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert dict(q.get(timeout=5) for _ in range(world)) == {0: True, 1: True}
