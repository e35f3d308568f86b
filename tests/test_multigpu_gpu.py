"""GPU, world_size 2 over NCCL (skips below 2 visible GPUs): the N-GPU path of
SURVEY.md §8e / f3 end to end.  Each rank generates its own prompt shard with
the tiny pair while its streamed layers arrive as 1/N host-link slices (raw or
XC4 frame ranges) rebuilt by the in-place NCCL all-gather, and one layer lives
1/N per GPU in HBM (f3 shards, all-gathered every pass).  In the parity mode
the tokens must EQUAL an N = 1 engine's on the same prompts."""
import os
import uuid

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

needs2 = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs ≥ 2 GPUs (NCCL world 2)")


def _worker(rank: int, world: int, port: int, name: str, codec: str, q):
    import torch.distributed as dist

    from oracle import tiny
    from paper_2505_10259_b200 import TINY_DRAFT, TINY_TARGET, Policy
    from paper_2505_10259_b200.api import build_engine
    from paper_2505_10259_b200.streamer import SharedHostStore
    from paper_2505_10259_b200.weights import unit_layout

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        stream = [1, 3]
        unit = unit_layout(TINY_TARGET, False)[1]
        cap = unit if codec == "none" else -(-2 * unit // (2 << 20)) * (2 << 20)
        store = SharedHostStore(name, stream, cap, rank, world, barrier=dist.barrier, coded=codec == "xc4")
        eng = build_engine(TINY_TARGET, TINY_DRAFT, device=dev, stream_layers=set(stream), seed=5, rank=rank,
                           world=world, shared_store=store, codec=codec, shard_layers={2}, arith="canonical")
        dist.barrier()
        prompts = tiny.prompts(8, seed=17)[rank::world]
        pol = Policy(4, 2, 2, 3)
        got = eng.generate(prompts, 10, pol)
        st = eng.target.streamer
        ref = build_engine(TINY_TARGET, TINY_DRAFT, device=dev, stream_layers=set(), seed=5,
                           arith="canonical").generate(prompts, 10, pol)
        dist.barrier()
        store.close(unlink=rank == 0)
        q.put((rank, got == ref, st.nvlink_bytes_issued > 0, st.bytes_issued > 0))
    finally:
        dist.destroy_process_group()


@needs2
@pytest.mark.parametrize("codec", ["none", "xc4"])
def test_two_rank_nccl_generate_matches_single_gpu(codec):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 2000)
    name = f"specoffload_nccl_{uuid.uuid4().hex[:8]}"
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, codec, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = dict((r, v) for r, *v in (q.get(timeout=10) for _ in range(world)))
    for r in range(world):
        same, nvl, link = res[r]
        assert same, f"rank {r}: tokens differ from the N = 1 engine"
        assert nvl and link, f"rank {r}: expected both host-link slices and NVLink all-gathers"
