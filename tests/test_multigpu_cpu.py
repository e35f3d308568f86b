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
