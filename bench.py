#!/usr/bin/env python
"""Decode tokens/s of the offloaded Mixtral-8x22B target + Mistral-7B draft on B200.

Metric (BASELINE.json): decode tokens/s of offloaded speculative decoding vs
the host-link streaming roofline.  One *step* = one barrier-synchronised
round: verify one batch (all target layers; the streamed ones cross PCIe
from pinned host DRAM) while drafting the other.

Workload (N=1, configs[2]): Mixtral-8x22B-shaped target (random init,
bf16) with as many FFN layers in pinned host DRAM as the box's host memory
allows (the rest pinned in HBM by the planner), Mistral-7B-shaped draft
(V=32768) in HBM, SummEval-length synthetic context (503 tokens, random KV
resident in HBM before timing), n_cand=4, forced acceptance p=0.8
(synthetic weights accept ≈ nothing).  Each round streams
≈180 GB, far above the 126 MB L2, so no flush is needed between steps.

`value`: committed tokens / device time of the K timed rounds (CUDA events
on the verify stream, barrier-joined with the draft stream), max over ranks.
`e2e`: the same rounds through the public Engine.round() API timed by the
host wall clock — every round copies its inputs (streamed weights + round
metadata) from pinned host memory and reads the committed tokens back.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import paper_2505_10259_b200  # noqa: E402

paper_2505_10259_b200.reserve_work_queues(32)  # one hardware queue per engine stream (DESIGN.md robustness notes)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("8x22b", "8x7b", "tiny"), default="8x22b")
    ap.add_argument("--n-cand", type=int, default=8, help="draft length (8 = the paper's best 8x22B policy)")
    ap.add_argument("--p", type=float, default=0.8)
    ap.add_argument("--ctx", type=int, default=503)
    ap.add_argument("--max-new", type=int, default=16,
                    help="tokens per request (the reference Workload's max_new_tokens; paper tables: 16): a finished "
                         "sequence restarts as a new request for its cached prompt, commits clamped to what is "
                         "left — the steady state, independent of --steps; 0 = legacy (contexts grow for the "
                         "whole run, nothing clamped)")
    ap.add_argument("--bs", type=int, default=0, help="per-batch size (0 = planner)")
    ap.add_argument("--host-gb", type=float, default=193.0,
                    help="pinned host budget for streamed units, GB (default 193: 55 XC4 8x22B units on the "
                         "pool's 196 GiB boxes; lowered to MemAvailable − 12 GB only if the box has less)")
    ap.add_argument("--hbm-gb", type=float, default=0.0, help="HBM budget (0 = device; 8x7b config: 24 GiB cap)")
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--window", choices=("split", "whole"), default="split",
                    help="split: streamed units move as [(attention +) gate_up | down] segments, one window slot "
                         "each (one unit of HBM instead of --slots units; single GPU — N > 1 uses whole units)")
    ap.add_argument("--draft-kv", choices=("auto", "cached", "reprefill", "mixed"), default="auto",
                    help="draft KV policy (auto = planner)")
    ap.add_argument("--layers", type=int, default=0,
                    help="profiling only: override the target's layer count (same per-layer shapes)")
    ap.add_argument("--max-pinned", type=int, default=-1,
                    help="profiling only: cap the planner's HBM-pinned layers (-1 = planner)")
    ap.add_argument("--draft-cached", type=int, default=-1,
                    help="mixed draft KV: cached sequences per batch (-1 = planner)")
    ap.add_argument("--no-shards", action="store_true",
                    help="N > 1: stream every non-pinned layer over the host links (no HBM-sharded layers, §8 f3)")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo = functional check of the N>1 path with ranks sharing GPUs (collectives staged "
                         "through host memory; not a performance configuration)")
    ap.add_argument("--disk-gb", type=float, default=0.0,
                    help="disk tier budget (§8 f4): streamed units beyond the host budget go to a file")
    ap.add_argument("--disk-path", default="", help="file of the disk tier (default: a temporary file)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the post-run logits check")
    ap.add_argument("--no-e2e-generate", action="store_true",
                    help="skip the generate() leg (host prompts → prefill → decode → host tokens)")
    ap.add_argument("--e2e-seqs", type=int, default=0,
                    help="prompts of the generate() leg (0 = three times its slot pool, run with slot refill)")
    ap.add_argument("--e2e-new", type=int, default=16, help="tokens per sequence (paper tables: 16)")
    ap.add_argument("--e2e-admit", type=int, default=0, help="generate() leg: prompts admitted per round (0 = all free)")
    ap.add_argument("--trace-out", default="")
    ap.add_argument("--codec", choices=("xc4", "none"), default="xc4",
                    help="streamed units XC4-encoded in host DRAM (K9, lossless) or raw bf16")
    return ap.parse_args()


METRIC = "decode tokens/s (offloaded Mixtral target + draft) vs host-link roofline"  # BASELINE.json metric
NVLINK_PEER_BPS = 770e9  # B200_PROFILING.md: measured NVLink 5 peer copy per direction


def _workload_name(args, tgt, drf, world, hbm) -> str:
    """The configs[] entry a run measures (BASELINE.json), identical for both arms."""
    if args.config == "8x22b" and not args.hbm_gb:
        return f"configs[2]: {tgt.name} offloaded + {drf.name} draft, {world} B200, full HBM"
    cap = f"{hbm / 2**30:.0f} GiB" if hbm else (f"{args.hbm_gb:g} GB" if args.hbm_gb else "24 GiB")
    return f"configs[1]: {tgt.name} offloaded + {drf.name} draft, {world} B200, HBM capped to {cap}"


def _commits_per_verify(args) -> float:
    """Committed tokens per verified sequence of the workload (the same figure for both arms)."""
    from paper_2505_10259_b200.acceptance import AcceptanceModel, committed_per_verify

    return committed_per_verify(AcceptanceModel(args.p, args.n_cand), args.max_new)


def _weights_checksum(eng) -> str:
    """SO_DEBUG_CHECKSUM=1: checksums of the resident weights (a debugging aid for
    stray device writes; off by default)."""
    t, d = eng.target.w, eng.draft.w
    parts = [("t.lm_head", t.lm_head), ("t.embed", t.embed), ("t.final_norm", t.final_norm),
             ("t.router0", t.layers[0].router), ("d.lm_head", d.lm_head), ("d.embed", d.embed)]
    return " ".join(f"{n}={x.double().sum().item():.6e}" for n, x in parts if x is not None)


def log(msg: str) -> None:
    """Progress line on stderr (rank-tagged): locates a stall in multi-rank runs."""
    print(f"[rank {os.environ.get('RANK', '0')} {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def mem_available() -> int:
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) * 1024
    return 0


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


def h2d_peak(torch, device) -> float:
    """Pinned 1 GiB host→device copy, best of 5 (the link roofline denominator)."""
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=device)
    s = torch.cuda.Stream(device=device)
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
        b.record(s)
        b.synchronize()
        best = max(best, n / (a.elapsed_time(b) * 1e-3))
    del h, d
    return best


def pair(cfg, layers: int = 0):
    import dataclasses

    from paper_2505_10259_b200 import PAIRS

    t, d = PAIRS[cfg]
    if layers:
        t = dataclasses.replace(t, n_layer=layers, name=f"{t.name}-{layers}L")
    return t, d


def reference_cpu_work(cfg: str) -> dict:
    """The reference's own CPU work on this box: its
    planner ``search`` over the C5 grid at four HBM budgets, its
    ``simulate_decoding`` of the best policy, and its ``predict_throughput``
    on the B200 HardwareProfile preset (a model prediction, not a
    measurement).  Runs the unmodified specpipe installed in baseline/_ref
    (``__graft_entry__.build`` installs it when /root/reference is present)."""
    import dataclasses

    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "specpipe")):
        return {"unavailable": "specpipe not installed in baseline/_ref"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import specpipe
    from specpipe import planner as SP
    from specpipe import simulator as SS

    from paper_2505_10259_b200 import presets

    name = {"8x22b": "b200_8x22b", "8x7b": "b200_8x7b_24g", "tiny": "b200_tiny"}[cfg]
    hw_o, t_o, d_o = presets.preset(name)
    hw = specpipe.HardwareProfile(**hw_o.to_dict())
    t = specpipe.ModelSpec(**dataclasses.asdict(t_o))
    d = specpipe.ModelSpec(**dataclasses.asdict(d_o))
    space = SP.SearchSpace(bs_prefill_values=(64, 128, 256), bs_decoding_values=(32, 64, 128, 256, 384, 512, 640),
                           bs_draft_values=(16, 32, 64), n_cand_values=(2, 3, 4, 5, 6, 7, 8))
    wl = specpipe.Workload(total_sequences=2048, l_input=503, max_new_tokens=16, acceptance_p=0.8)
    out = {"package": f"specpipe {getattr(specpipe, '__version__', '')} (unmodified, baseline/_ref)",
           "preset": name, "grid_points": len(space.policies()), "search": []}
    best = None
    for gib in (24, 48, 96, None):
        h = hw if gib is None else dataclasses.replace(hw, gpu_mem_capacity=gib * 2**30)
        t0 = time.perf_counter()
        try:
            rk = SP.search(space, wl, h, t, d)
            res = {"feasible": len(rk.entries), "best": list(rk.best.as_tuple()),
                   "predicted_tokens_per_s": rk.entries[0][1].throughput}
            if gib is None:
                best = rk.best
        except specpipe.errors.SpecPipeError as exc:
            res = {"feasible": 0, "error": type(exc).__name__}
        res.update(hbm_gib=gib or round(hw.gpu_mem_capacity / 2**30, 1), seconds=time.perf_counter() - t0)
        out["search"].append(res)
    if best is not None:
        t0 = time.perf_counter()
        sim = SS.simulate_decoding(best, SP.rotation_workload(wl, best), hw, t, d, seed=0)
        out["simulate_decoding"] = {"policy": list(best.as_tuple()), "seconds": time.perf_counter() - t0,
                                    "events": len(sim.trace), "simulated_tokens_per_s": sim.throughput}
        bd = SP.predict_throughput(best, wl, hw, t, d)
        out["predict_throughput"] = {"policy": list(best.as_tuple()), "tokens_per_s": bd.throughput,
                                     "t_target_per_round_s": bd.t_target_per_round,
                                     "note": "the reference's cost model on the B200 preset (CPU attention, "
                                             "no prefetch-ahead): a prediction, not a measurement"}
    return out


def run_reference(args, rank: int) -> None:
    """--impl reference: the CPU port of the path (oracle) on the host cores."""
    if rank != 0:
        return
    from oracle import cpu_baseline

    tgt, drf = pair(args.config)
    vals, samples = [], []
    cache: dict = {}  # weights built once; every step times the sampled forward passes
    for i in range(args.warmup + args.steps):
        r = cpu_baseline.measure(tgt, drf, args.n_cand, args.p, args.ctx, sample_seqs=4, seed=i, cache=cache,
                                 commits_per_verify=_commits_per_verify(args))
        if i >= args.warmup:
            vals.append(r.tokens_per_s)
            samples.append(r.t_sample)
    v = float(np.mean(vals))
    step_s = float(np.mean(samples))
    line = {"impl": "reference", "metric": METRIC, "value": v,
            "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            # the GPU arm's workload (same model pair, draft length, acceptance, prompt length and
            # request length); the CPU executes a 4-sequence sample of its round
            "config": {"workload": _workload_name(args, tgt, drf, args.gpus, None), "n_cand": args.n_cand,
                       "acceptance_p": args.p, "ctx": args.ctx,
                       "max_new_tokens": args.max_new if args.max_new > 0 else None, "sample_seqs": 4},
            "step": {"executed": "1 full-shape target layer verify (4 seqs × (n_cand+1) tokens, ctx "
                                 f"{args.ctx}) + 1 full-shape draft layer step, NumPy fp32 on {r.cores} cores",
                     "executed_s": step_s, "extrapolated_round_s": r.t_round,
                     "value_is": "tokens/s of a full round extrapolated from the executed sample "
                                 "(4 × commits per verify / extrapolated round time)"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r.cores, "kind": "port", "sample": r.sample},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    try:
        line["reference_cpu_work"] = reference_cpu_work(args.config)
    except Exception as exc:  # the arm's line must still print
        line["reference_cpu_work"] = {"error": str(exc)[:200]}
    print(json.dumps(line))


def main():
    args = parse()
    # diagnostics for a stalled run: every thread's stack on stderr every SO_WATCHDOG_S
    # seconds (default 600 s — past a normal run's whole duration)
    import faulthandler

    faulthandler.dump_traceback_later(float(os.environ.get("SO_WATCHDOG_S", "600")), repeat=True)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import cpu_baseline  # checker only: timed beside the GPU path, never part of it

        tgt, drf = pair(args.config)  # full-depth shapes
        cpu = cpu_baseline.measure(tgt, drf, args.n_cand, args.p, args.ctx, sample_seqs=4,
                                   commits_per_verify=_commits_per_verify(args))
        try:
            ref_work = reference_cpu_work(args.config)
        except Exception as exc:
            ref_work = {"error": str(exc)[:200]}

    import torch
    import torch.distributed as dist

    from paper_2505_10259_b200 import Policy, native
    from paper_2505_10259_b200.acceptance import AcceptanceModel, committed_per_verify, expected_accepted
    from paper_2505_10259_b200.api import build_engine
    from paper_2505_10259_b200.planner_b200 import draft_flops, plan_offload, roofline_tokens_per_s, verify_flops
    from paper_2505_10259_b200.streamer import HostStore
    from paper_2505_10259_b200.weights import ffn_offsets, unit_layout

    n_dev = torch.cuda.device_count()
    device = torch.device("cuda", local % n_dev)
    torch.cuda.set_device(device)
    share = -(-min(world, int(os.environ.get("LOCAL_WORLD_SIZE", world))) // n_dev)  # ranks per GPU
    if world > 1:
        if args.dist_backend == "nccl":
            # communicator lines (rank, nranks, NVLS / P2P transport) on stderr for the driver's rank check
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")
    tgt, drf = pair(args.config, args.layers)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0,
                                                         "bf16_tflops_sustained": 1400.0}
    link = h2d_peak(torch, device)
    free, total = torch.cuda.mem_get_info(device)
    free //= share  # ranks sharing a GPU (gloo functional check) split its memory
    hbm = int(args.hbm_gb * 1e9) if args.hbm_gb else (int(24 * 2**30) if args.config == "8x7b" else free)
    if hbm < free:
        # enforce the cap (configs[1]: "HBM capped to 24 GB") on the allocator itself
        torch.cuda.set_per_process_memory_fraction(min(1.0, hbm / total), device)
    # one host copy of the streamed layers serves every rank (SharedHostStore)
    # deterministic plan input: a fixed host budget (the plan, hence the headline, must not
    # depend on free host RAM at launch); reduced only on a box that cannot hold it
    host_req = int(args.host_gb * 1e9)
    host = min(host_req, max(0, mem_available() - int(12e9)))
    host_src = "requested" if host == host_req else f"reduced from {host_req} to MemAvailable − 12 GB"
    if world > 1:  # every rank must build the same plan: agree on the smallest measured budgets / rates
        agree = torch.tensor([float(link), float(hbm), float(host)], dtype=torch.float64,
                             device=device if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(agree, op=dist.ReduceOp.MIN)
        link, hbm, host = float(agree[0]), int(agree[1]), int(agree[2])
    steps, warm = args.steps, args.warmup
    # rounds alternate batches: batch 0 is verified ceil(R/2) times in R rounds, each committing
    # ≤ n_cand+1 tokens, so no sequence can be clamped by `remaining` inside the run
    if args.max_new > 0:  # steady state of max_new-token requests (recycled on their cached prompt)
        max_new = args.max_new
    else:  # legacy: batch 0 is verified ceil(R/2) times in R rounds, each committing ≤ n_cand+1 tokens
        verifies_per_batch = -(-(warm + steps) // 2)
        max_new = verifies_per_batch * (args.n_cand + 1)
    from paper_2505_10259_b200.planner_b200 import B200Rates

    rates = B200Rates(h2d_bytes_per_s=link, hbm_bytes_per_s=peaks["hbm_gbs"] * 1e9)
    modes = ("cached", "reprefill", "mixed") if args.draft_kv == "auto" else (args.draft_kv,)
    ratio, ring = 1.0, 0
    if args.codec == "xc4":
        # encoded/raw ratio of this weight distribution, probed on one 64 Mi-weight sample
        from paper_2505_10259_b200 import codec as C

        g = torch.Generator(device=device).manual_seed(12345)
        probe = torch.empty(1 << 26, dtype=torch.bfloat16, device=device).normal_(0.0, 0.02, generator=g)
        enc = C.Encoder(device)
        ratio = enc.encode(probe)[0].numel() / (2 * probe.numel()) * 1.002
        ring = 4 * (192 << 20)  # LayerStreamer.RING_SLOTS encoded frames (≤ 180 MB each)
        enc.release()
        del probe
        torch.cuda.empty_cache()
    split = args.window == "split" and world == 1
    plan = plan_offload(tgt, drf, hbm, host, args.n_cand, args.p, args.ctx, max_new, rates, n_slots=args.slots,
                        bs_candidates=[args.bs] if args.bs else None, draft_kv_modes=modes, stream_ratio=ratio,
                        ring_bytes=ring, max_pinned=None if args.max_pinned < 0 else args.max_pinned,
                        draft_cached_candidates=None if args.draft_cached < 0 else [args.draft_cached],
                        world=world, allow_shards=not args.no_shards, disk_budget=int(args.disk_gb * 1e9),
                        kv_host_modes=(False, True) if world == 1 else (False,),
                        tokens_per_verify=committed_per_verify(AcceptanceModel(args.p, args.n_cand), args.max_new),
                        split_window=split)
    log(f"plan: bs {plan.bs_decoding} draft {plan.draft_kv}/{plan.draft_cached} pinned {len(plan.pinned_layers)} "
        f"streamed {len(plan.stream_layers)} (disk {len(plan.disk_layers)}) sharded {len(plan.shard_layers)} "
        f"link {link / 1e9:.1f} GB/s")
    t_setup = time.perf_counter()
    layer_bytes = ffn_offsets(tgt)[2]
    if world > 1:
        from paper_2505_10259_b200.streamer import SharedHostStore

        unit_bytes = unit_layout(tgt, plan.stream_attn)[1]
        cap = unit_bytes if args.codec == "none" else -(-int(unit_bytes * (ratio + 0.005)) // (2 << 20)) * (2 << 20)
        store = SharedHostStore(f"specoffload_{os.environ.get('MASTER_PORT', '0')}", list(plan.stream_layers),
                                cap, rank, world, barrier=dist.barrier,
                                coded=args.codec != "none") if plan.stream_layers else None
        eng = build_engine(tgt, drf, device=device, stream_layers=set(plan.stream_layers), n_slots=args.slots,
                           seed=1, trace=bool(args.trace_out), rank=rank, world=world, shared_store=store,
                           stream_attn=plan.stream_attn, codec=args.codec, shard_layers=set(plan.shard_layers))
        dist.barrier()  # every slice of the shared store is written
    else:
        store = HostStore()
        eng = build_engine(tgt, drf, device=device, stream_layers=set(plan.stream_layers), n_slots=args.slots,
                           seed=1, trace=bool(args.trace_out), host_store=store, stream_attn=plan.stream_attn,
                           codec=args.codec, disk_layers=set(plan.disk_layers), disk_path=args.disk_path or None,
                           split_window=plan.split_window)
    bs = plan.bs_decoding
    S = 2 * bs
    s = eng.new_session(S, bs, args.ctx + max_new + args.n_cand + 2, args.n_cand, forced_p=args.p, seed=rank,
                        bs_draft=plan.bs_draft, draft_kv=plan.draft_kv, draft_cached=plan.draft_cached,
                        kv_host=plan.kv_host)
    eng.synthetic_context(s, args.ctx, max_new, seed=rank, recycle=args.max_new > 0)
    dbg_sum = os.environ.get("SO_DEBUG_CHECKSUM") == "1"
    if dbg_sum:
        torch.cuda.synchronize(device)
        log(f"checksum after build+context: {_weights_checksum(eng)}")
    eng.first_draft(s)
    if dbg_sum:
        torch.cuda.synchronize(device)
        log(f"checksum after first draft: {_weights_checksum(eng)}")
    setup_s = time.perf_counter() - t_setup
    log(f"setup {setup_s:.1f} s")
    for i in range(warm):
        eng.round(s)
        log(f"warm-up round {i}")
        if dbg_sum:
            torch.cuda.synchronize(device)
            log(f"checksum after warm-up round {i}: {_weights_checksum(eng)}")
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    native.reset_launch_counter()
    committed0 = s.committed_decode
    st = eng.target.streamer
    bytes0 = st.bytes_issued if st else 0
    raw0 = st.raw_bytes_issued if st else 0
    nvl0 = st.nvlink_bytes_issued if st else 0
    kvh0 = getattr(s.tkv, "bytes_h2d", 0)  # host-resident target KV: window pages cross the same link
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if eng.tracer.enabled:
        eng.tracer.origin(eng.tgt_stream)
        if st:
            st.copy_marks.clear()
    ev0.record(eng.tgt_stream)
    w0 = time.perf_counter()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include "timed/" selects the timed rounds
    eng.nvtx_range = "timed"             # ... on the draft-enqueue thread too
    eng.round_times.clear()
    for _ in range(steps):
        eng.round(s)  # public API: H2D inputs, verify+draft, barrier, D2H committed tokens
    eng.nvtx_range = None
    torch.cuda.nvtx.range_pop()
    ev1.record(eng.tgt_stream)
    ev1.synchronize()
    wall = time.perf_counter() - w0
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    log("timed rounds done")
    hbm_peak = int(torch.cuda.max_memory_allocated(device))  # allocator peak of setup + decode so far
    hbm_reserved = int(torch.cuda.memory_reserved(device))
    clk = clocks.stop()
    dev_s = ev0.elapsed_time(ev1) * 1e-3
    committed = s.committed_decode - committed0
    streamed = (st.bytes_issued - bytes0) if st else 0       # bytes over this rank's link
    streamed_raw = (st.raw_bytes_issued - raw0) if st else 0  # layer bytes they delivered
    nvl = (st.nvlink_bytes_issued - nvl0) if st else 0       # bytes this rank received from HBM shards
    kv_link = getattr(s.tkv, "bytes_h2d", 0) - kvh0          # host KV window pages (0 with HBM KV)
    streamed += kv_link
    streamed_raw += kv_link
    launches = dict(native.launches)
    if world > 1:
        rdev = device if args.dist_backend == "nccl" else "cpu"
        t = torch.tensor([dev_s, wall], device=rdev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, wall = t.tolist()
        c = torch.tensor([committed], device=rdev, dtype=torch.float64)
        dist.all_reduce(c)
        committed = int(c.item())
    value = committed / dev_s
    e2e = committed / wall

    # ---- dominant kernel: the copy engine (host link) ----
    layer_bytes = ffn_offsets(tgt)[2]
    achieved_link = streamed / dev_s if dev_s > 0 else 0.0
    # expected commits per verification: E[k], clamped by what each request has left (steady state)
    e_tok = committed_per_verify(AcceptanceModel(args.p, args.n_cand), args.max_new)
    # compute term: the verify pass plus the concurrent draft work of the round
    F_verify = verify_flops(tgt, bs, args.n_cand, args.ctx)
    F_draft = draft_flops(drf, bs, args.n_cand, args.ctx, plan.draft_kv, plan.draft_cached)
    F = F_verify + F_draft
    # north-star roofline: committed tokens over max(link bytes / B_h2d, compute at peak), per round
    roof = roofline_tokens_per_s(bs * e_tok * world, streamed / steps, F, link, peaks["bf16_tflops_sustained"] * 1e12)
    if world > 1:  # the NVLink all-gathers are a third bound
        gathered = nvl + (streamed_raw * (world - 1))  # host-streamed slices are all-gathered too
        t_nvl = gathered / steps / NVLINK_PEER_BPS
        t_roof = max(streamed / steps / link, t_nvl, F / (peaks["bf16_tflops_sustained"] * 1e12))
        roof = bs * e_tok * world / t_roof
    roof_raw = roofline_tokens_per_s(bs * e_tok * world, streamed_raw / steps, F, link,
                                     peaks["bf16_tflops_sustained"] * 1e12)

    # ---- numerics of the headline path (forced acceptance hides them): a few sequences'
    # verify logits through the product path vs a PyTorch fp32 restatement over the same
    # streamed weights and KV (tools/fp32_ref.py) ----
    parity = None
    if rank == 0 and not args.no_parity:
        try:
            from tools.fp32_ref import parity_report

            t_p = time.perf_counter()
            parity = parity_report(eng, s, n_seq=2)
            parity["seconds"] = time.perf_counter() - t_p
        except Exception as exc:  # the headline must still print
            parity = {"error": f"{type(exc).__name__}: {str(exc)[:300]}"}
        log(f"parity: {parity}")

    # ---- tensor-core kernel sample: MoE gate_up grouped GEMM at this round's shape ----
    kern = {}
    try:
        T = bs * (args.n_cand + 1)
        E, H, I = tgt.n_expert, tgt.hidden, tgt.inter
        g = torch.Generator(device=device).manual_seed(0)
        a = torch.randn(2 * T, H, device=device, generator=g).to(torch.bfloat16)
        # weights: the gate_up part of an FFN layer already in an HBM window slot
        w = st.slots[0] if st else eng.target.w.layers[0].ffn
        cnt = np.full(E, 2 * T // E)
        cnt[: 2 * T - cnt.sum()] += 1
        offs = torch.tensor(np.concatenate([[0], np.cumsum(cnt)]), dtype=torch.int32, device=device)
        act = torch.empty(2 * T, I, dtype=torch.bfloat16, device=device)
        for _ in range(3):
            native.gemm_grouped(a, w.data_ptr(), offs, E, 2 * I, act, native.EPI_SWIGLU)
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        x0.record()
        for _ in range(reps):
            native.gemm_grouped(a, w.data_ptr(), offs, E, 2 * I, act, native.EPI_SWIGLU)
        x1.record()
        x1.synchronize()
        t_k = x0.elapsed_time(x1) * 1e-3 / reps
        flops = 2.0 * 2 * T * 2 * I * H
        kern = {"kernel": "gemm_grouped SwiGLU (K3, MoE gate_up)", "bound": "tensor",
                "achieved": flops / t_k / 1e12, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": flops / t_k / 1e12 / peaks["bf16_tflops"], "ms": t_k * 1e3,
                "shape": f"rows {2 * T} x N {2 * I} x K {H}, {E} experts", "peak_kind": "burst (measured)"}
        del a, act
    except Exception as exc:  # the headline must still print
        kern = {"error": str(exc)}

    # ---- K9 decode kernel sample: ring-resident encoded frames → a window slot (HBM → HBM) ----
    codec_k = None
    if st is not None and st.coded:
        try:
            u0 = st.host[st.streamed[0]]
            u = u0.parts[0] if hasattr(u0, "parts") else u0  # split window: the first segment's unit
            frames_per_layer = sum(p.n_frames for p in u0.parts) if hasattr(u0, "parts") else u.n_frames
            nf = min(st.RING_SLOTS, u.n_frames)
            # frames [0, nf) copied contiguously into the staging ring; the decoder
            # addresses frame f at base + frame_off[f], so base = ring − frame_off[0]
            native.memcpy_async(st.ring.data_ptr(), u.data.data_ptr() + int(u.frame_off[0]), u.frame_bytes(0, nf),
                                torch.cuda.current_stream(device))
            base = st.ring.data_ptr() - int(u.frame_off[0])
            out = st.slots[0].data_ptr()
            for _ in range(2):
                native.xc4_decode(u.data.data_ptr(), base, 0, nf, out)
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            x0.record()
            for _ in range(reps):
                native.xc4_decode(u.data.data_ptr(), base, 0, nf, out)
            x1.record()
            x1.synchronize()
            t_d = x0.elapsed_time(x1) * 1e-3 / reps
            raw_f = 2 * min(u.n_elems, nf * u.frame_elems)
            algo = u.frame_bytes(0, nf) + raw_f
            codec_k = {"kernel": "xc4_decode_kernel (K9)", "bound": "hbm", "achieved": algo / t_d / 1e9,
                       "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": algo / t_d / 1e9 / peaks["hbm_gbs"],
                       "ms_per_launch_group": t_d * 1e3, "frames": nf, "algorithmic_bytes": algo,
                       "ms_per_layer_est": t_d * 1e3 * frames_per_layer / nf, "ratio": u0.ratio,
                       "escapes": u.n_escapes, "frames_per_layer": frames_per_layer,
                       "note": "algorithmic bytes = encoded frames read + decoded bf16 written"}
        except Exception as exc:
            codec_k = {"error": str(exc)}

    log("kernel samples done")
    # ---- generate(): the paper's end-to-end tokens/s (prefill included) ----
    gen = None
    if not args.no_e2e_generate:
        try:
            del s
            torch.cuda.empty_cache()
            if plan.split_window:  # prefill passes hold both segments of a layer: double-buffer each
                eng.set_window_slots(2 * args.slots)
            # Its own slot pool: with prefill inside every round the generate workload is
            # tensor-bound, not link-bound, so the draft keeps a KV row per slot (no
            # per-round context re-prefill) and HBM left after the engine's weights
            # and window sets the slot count (headroom for the prefill activations).
            from paper_2505_10259_b200.kvcache import PagedKVCache

            free_now, _ = torch.cuda.mem_get_info(device)
            # the HBM budget (configs[1]: 24 GB cap) bounds the pool, not just the device's free memory
            free_now = min(free_now // share, hbm - torch.cuda.memory_reserved(device))
            g_len = args.ctx + args.e2e_new + args.n_cand + 2
            per_slot = PagedKVCache.bytes_needed(tgt, 1, g_len) + PagedKVCache.bytes_needed(drf, 1, g_len)
            headroom = min(10e9, 0.35 * free_now)  # prefill activations of the admitted prompts
            bs_e = max(8, int((free_now - headroom) // per_slot) // 2 // 8 * 8)
            e_kv_host, e_draft_kv, e_bs_draft = False, "cached", None
            if plan.kv_host:  # tiny HBM budget: the decode plan's host-resident target KV and re-prefill draft
                eng.prefill_chunk_tokens = 2048  # prefill activations must fit beside the capped plan
                bs_e, e_kv_host, e_draft_kv, e_bs_draft = plan.bs_decoding, True, "reprefill", plan.bs_draft
            S_e = args.e2e_seqs or 6 * bs_e
            rng = np.random.default_rng(1234 + rank)
            prompts = [rng.integers(0, tgt.vocab, args.ctx).astype(np.int32) for _ in range(S_e)]
            pol = Policy(bs_prefill=min(S_e, 2 * bs_e), bs_decoding=min(bs_e, (S_e + 1) // 2),
                         bs_draft=e_bs_draft or min(bs_e, (S_e + 1) // 2), n_cand=args.n_cand)
            torch.cuda.synchronize(device)
            g0 = time.perf_counter()
            admit = args.e2e_admit or None
            round0 = eng.round

            def logged_round(sess, _r=round0):  # progress of the long generate leg on stderr
                c = _r(sess)
                if sess.rounds % 10 == 0 or sess.rounds <= 3:
                    log(f"generate: round {sess.rounds}, queue {len(sess.queue)}, active {int(sess.active.sum())}")
                return c

            log(f"generate: {S_e} prompts through {2 * pol.bs_decoding} slots")

            eng.round = logged_round
            toks = eng.generate(prompts, args.e2e_new, pol, forced_p=args.p, draft_kv=e_draft_kv, max_admit=admit,
                                kv_host=e_kv_host)
            g_wall = time.perf_counter() - g0
            eng.round = round0
            assert all(len(t) == args.e2e_new for t in toks)
            gs = eng.last_session
            gen = {"value": S_e * args.e2e_new / g_wall, "unit": "tokens/s", "sequences": S_e,
                   "prompt_tokens": args.ctx, "new_tokens": args.e2e_new, "wall_s": g_wall, "rounds": gs.rounds,
                   "policy": list(pol.as_tuple()), "draft_kv": e_draft_kv, "target_kv_host": e_kv_host,
                   "refill": gs.refill, "slots": gs.n_seq, "max_admit_per_round": admit,
                   "note": "Engine.generate(): host token ids in, host token lists out; the prompts stream through "
                           "the 2·bs_decoding slots with slot refill (each admitted prompt is prefilled inside a "
                           "verify pass), so every round streams the layers once for prefill and decode alike; "
                           "paper's e2e definition (prefill included)"}
        except torch.OutOfMemoryError as exc:  # the decode result above stands; report the leg's failure
            gen = {"error": f"generate() leg out of HBM: {str(exc).splitlines()[0]}"}
            eng.__dict__.pop("round", None)  # drop the logging wrapper (instance attribute)
            torch.cuda.empty_cache()

    if args.trace_out and rank == 0:
        from paper_2505_10259_b200.trace import SimResult, busy, export_chrome

        evs = eng.resolve_trace()
        res = SimResult(evs, dev_s, committed, value, int(torch.cuda.max_memory_allocated(device)), steps,
                        busy(evs))
        os.makedirs(os.path.dirname(args.trace_out) or ".", exist_ok=True)
        with open(args.trace_out, "w") as f:
            f.write(export_chrome(res))

    if world > 1:
        dist.barrier()
        if store is not None:
            store.close(unlink=rank == 0)
    if rank != 0:
        return
    meta_bytes = bs * (args.n_cand + 1) * 4 * 2 + bs * 4 * 4
    line = {
        "metric": METRIC,
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": dev_s / steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init weights, random prompt KV, forced acceptance p)",
        "config": {"workload": _workload_name(args, tgt, drf, world, hbm),
                   "bs_decoding": bs, "total_sequences": S * world, "n_cand": args.n_cand,
                   "draft_kv": plan.draft_kv, "draft_cached_per_batch": plan.draft_cached,
                   "bs_draft": plan.bs_draft, "acceptance_p": args.p,
                   "max_new_tokens": args.max_new if args.max_new > 0 else None,
                   "requests": ("steady state: a sequence that generated max_new tokens restarts as a new request "
                                "for its cached 503-token prompt (commits clamped, simulator.py:213-214); "
                                f"expected commits per verify {e_tok:.4f}") if args.max_new > 0 else
                               "legacy: contexts grow for the whole run",
                   "ctx": args.ctx, "streamed_layers": len(plan.stream_layers),
                   "hbm_sharded_layers": len(plan.shard_layers), "disk_layers": len(plan.disk_layers),
                   "target_kv": "host DRAM (one batch staged per layer)" if plan.kv_host else "HBM",
                   "pinned_layers": len(plan.pinned_layers), "window_slots": args.slots, "window": "split" if plan.split_window else "whole",
                   "codec": args.codec, "stream_ratio": streamed / streamed_raw if streamed_raw else None,
                   "streamed_bytes_per_round": int(streamed / steps * world),
                   "kv_h2d_bytes_per_round": int(kv_link / steps * world),
                   "streamed_layer_bytes_per_round": len(plan.stream_layers) * layer_bytes,
                   "host_pinned_bytes": store.bytes if store is not None else 0,
                   "host_budget_bytes": host, "host_budget": host_src, "l2": "inputs ≫ L2 (≈180 GB streamed per step)",
                   "parallelism": f"dp{world} (independent prompt shards)", "setup_s": round(setup_s, 1)},
        "roofline": {"bound": "h2d", "achieved": achieved_link / 1e9, "peak": link / 1e9, "unit": "GB/s",
                     "frac": achieved_link / link, "traffic": None,
                     "peak_source": "pinned 1 GiB host→device cudaMemcpyAsync, best of 5, measured in this run "
                                    "(MEASURED_PEAKS.json carries no host-link figure)",
                     "note": "dominant 'kernel' = copy-engine stream of the streamed layer units (XC4-encoded "
                             "bytes when codec=xc4) plus, with host-resident target KV, the KV window pages"},
        "roofline_raw": {"bound": "h2d", "achieved": streamed_raw / dev_s / 1e9, "peak": link / 1e9, "unit": "GB/s",
                         "frac": streamed_raw / dev_s / link,
                         "note": "the same rounds counted in the reference's raw ffn_bytes (uncompressed bf16 layer "
                                 "bytes delivered per second): > 1 because XC4 moves ≈0.70 of them over the link"},
        "compute": {"flops_per_round": F, "verify_flops": F_verify, "draft_flops": F_draft,
                    "t_at_sustained_peak_s": F / (peaks["bf16_tflops_sustained"] * 1e12),
                    "t_link_s": streamed / steps / link},
        "roofline_tokens_per_s": roof, "frac_of_roofline": value / roof if roof else None,
        "nvlink": ({"received_bytes_per_round": int((nvl + streamed_raw * (world - 1)) / steps),
                    "achieved_GBps": (nvl + streamed_raw * (world - 1)) / dev_s / 1e9,
                    "peak_GBps": NVLINK_PEER_BPS / 1e9, "peak_kind": "measured peer copy (B200_PROFILING.md)"}
                   if world > 1 else None),
        "raw_roofline_tokens_per_s": roof_raw,
        "note_roofline": "roofline_tokens_per_s uses the bytes that crossed the link; raw_roofline_tokens_per_s "
                         "the same rounds if the layers crossed uncompressed (the reference's ffn_bytes)",
        "codec_kernel": codec_k,
        "kernel_roofline": kern,
        "clocks": clk,
        "stream_busy_ms": {"draft_stream_per_round": [round(a, 1) for a, _ in eng.round_times[:steps]],
                           "verify_stream_per_round": [round(b, 1) for _, b in eng.round_times[:steps]],
                           "note": "start→end of each stream's work in a round (the draft runs concurrently "
                                   "with the verify; the verify waits on streamed layers)"},
        "gpu_launches": launches["kernels"],
        "copy_calls": launches["copies"],
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": int(streamed / steps + meta_bytes),
                "d2h_bytes_per_step": int(bs * (args.n_cand + 2) * 4)},
        "plan": plan.as_dict(),
        "hbm": {"budget": int(hbm), "planned": int(sum(plan.hbm_bytes.values())), "peak_allocated": hbm_peak,
                "reserved": hbm_reserved,
                "note": "planned = the plan's hbm_bytes (weights, window, KV, workspaces); peak_allocated = "
                        "torch.cuda.max_memory_allocated after the timed rounds"},
    }
    if gen is not None:
        line["e2e_generate"] = gen
    if parity is not None:
        line["parity"] = parity
    if cpu is not None:
        line["cpu_baseline"] = {"value": cpu.tokens_per_s, "unit": "tokens/s", "cores": cpu.cores, "kind": "port",
                                "sample": cpu.sample, "executed_s": cpu.t_sample,
                                "extrapolated_round_s": cpu.t_round}
        line["reference_cpu_work"] = ref_work
    print(json.dumps(line))


if __name__ == "__main__":
    main()
