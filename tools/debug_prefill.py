import numpy as np, torch, sys
sys.path.insert(0, ".")
from oracle import tiny, model_ref, decode_ref
from paper_2505_10259_b200 import TINY_TARGET, TINY_DRAFT, Policy
from paper_2505_10259_b200.api import build_engine
tw, dw = tiny.weights()
for seed, S in ((8, 8), (1234, 8)):
    prompts = tiny.prompts(S, seed=seed)
    print("seed", seed, "lens", [len(p) for p in prompts])
    for sl in ({1, 3}, set()):
        eng = build_engine(TINY_TARGET, TINY_DRAFT, tw, dw, stream_layers=sl)
        s = eng.new_session(S, 4, 64, 4)
        eng.prefill(s, prompts, 12)
        got = eng.target.ws.get("logits", (S, 1024), torch.float32).cpu().numpy()
        kv = model_ref.KV(tiny.TARGET, S, 64)
        want = np.concatenate(model_ref.forward(tiny.TARGET, tw, kv, list(range(S)), prompts, [0] * S, True, "last"))
        print(" stream", sl, "maxdiff/seq", np.round(np.abs(got - want).max(1), 3), "argmax eq", (got.argmax(1) == want.argmax(1)).astype(int), "first", [o[0] for o in s.out])
