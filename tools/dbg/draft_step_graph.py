"""How much of a draft decode step is launch overhead: one Mistral-7B decode step (64 sequences,
ctx 520, all 32 layers, the engine's own forward) timed eagerly vs captured in a CUDA graph."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2505_10259_b200 import MISTRAL_7B_V3, TINY_TARGET  # noqa: E402
from paper_2505_10259_b200.api import build_engine  # noqa: E402
from paper_2505_10259_b200.models import ForwardBatch, _dev_i32  # noqa: E402

dev = "cuda:0"
eng = build_engine(TINY_TARGET, MISTRAL_7B_V3, device=dev, stream_layers=set(), trace=False)
n, ctx, bs = 8, 520, 64
s = eng.new_session(2 * bs, bs, ctx + 30, n, forced_p=0.8, bs_draft=bs, draft_kv="cached")
eng.synthetic_context(s, ctx, 16)
kv = s.dkv
rows = s.drow[:bs].astype(np.int64)
pos = np.full(bs, ctx, np.int64)
slots = kv.slots(rows, pos)
st = eng.drf_stream
with torch.cuda.stream(st):
    toks = torch.zeros(bs, dtype=torch.int32, device=dev)
    fb = ForwardBatch(toks, _dev_i32(pos, dev), _dev_i32(slots, dev), _dev_i32(np.arange(bs + 1), dev),
                      _dev_i32(pos, dev), _dev_i32(kv._bt_host[rows], dev), bs, 1)
    logits = torch.empty(bs, MISTRAL_7B_V3.vocab, dtype=torch.float32, device=dev)
step = lambda: eng.draft.forward(fb, kv, st, logits_out=logits)  # noqa: E731
for _ in range(3):
    step()
torch.cuda.synchronize()
reps = 20
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(reps):
    step()
b.record(st)
b.synchronize()
eager = a.elapsed_time(b) / reps
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for _ in range(reps):
        step()
g.replay()
torch.cuda.synchronize()
a.record(st)
g.replay()
b.record(st)
b.synchronize()
graph = a.elapsed_time(b) / reps
wbytes = 32 * (6144 + 4096 + 28672 + 4096 * 14336 // 4096) * 4096 * 2
print(json.dumps({"eager_ms": eager, "graph_ms": graph, "launch_overhead_frac": 1 - graph / eager,
                  "layer_step_us_graph": graph * 1e3 / 32}))
