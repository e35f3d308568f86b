#!/usr/bin/env python
"""Regression check for the intermittent host-resident-KV + slot-refill stall
(DESIGN.md robustness notes): 8 layers of the 8x7B target at a 24 GiB cap, N
prompts through 192 slots with target KV in host DRAM.  Stalled once at the
barrier of round 11; 13 later runs (5 with CUDA_DEVICE_MAX_CONNECTIONS=8)
completed.  Cause unconfirmed.

    python tools/repro_hostkv.py 576
"""
import os, sys, time, faulthandler
sys.path.insert(0, os.getcwd())
faulthandler.dump_traceback_later(90, repeat=True)
import paper_2505_10259_b200
if os.environ.get("SO_WORK_QUEUES", "32") != "default":
    paper_2505_10259_b200.reserve_work_queues(int(os.environ.get("SO_WORK_QUEUES", "32")))
import numpy as np, torch
from paper_2505_10259_b200 import PAIRS, Policy
from paper_2505_10259_b200.api import build_engine
t, d = PAIRS["8x7b"]
import dataclasses
t = dataclasses.replace(t, n_layer=8)
torch.cuda.set_per_process_memory_fraction(24 * 2**30 / torch.cuda.get_device_properties(0).total_memory)
eng = build_engine(t, d, device="cuda:0", stream_layers=set(range(8)), stream_attn=True, codec="xc4", trace=False)
eng.prefill_chunk_tokens = 2048
rng = np.random.default_rng(0)
prompts = [rng.integers(0, t.vocab, 503).astype(np.int32) for _ in range(int(sys.argv[1]))]
r0 = eng.round
def lr(s, _r=r0):
    c = _r(s); print("round", s.rounds, "queue", len(s.queue), "active", int(s.active.sum()), time.strftime("%X"), flush=True); return c
eng.round = lr
out = eng.generate(prompts, 16, Policy(192, 96, 16, 8), forced_p=0.8, draft_kv="reprefill", kv_host=True)
print("done", len(out), flush=True)
