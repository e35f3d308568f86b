"""Generate tests/golden/ref_specpipe.json by running the UNMODIFIED reference.

Run here (the reference exists only in this container):
    python tests/golden/make_ref_golden.py
It imports specpipe from /root/reference/pkg/src and records the values the
reference computes for the parts of the hot path it implements: the
acceptance pmf / mean / inverse-CDF draws (acceptance.py:29-72), simulated
round counts (simulator.py:108-227), and cost-model numbers
(costmodel.py:157-197, planner.py:117-184).  The GPU box never reads
/root/reference; tests compare our restatements with this file.
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from specpipe import acceptance, costmodel, planner, presets, simulator  # noqa: E402
from specpipe.types import HardwareProfile, ModelSpec, Policy, Workload  # noqa: E402

GiB = 1024**3
out = {"pmf": [], "expected": [], "draws": [], "rounds": [], "cost": [], "search_top": []}

for p in (0.0, 0.3, 0.5, 0.8, 0.9, 1.0):
    for n in (1, 2, 4, 8):
        m = acceptance.AcceptanceModel(p=p, n_cand=n)
        out["pmf"].append({"p": p, "n": n, "pmf": acceptance.pmf(m).tolist()})
        out["expected"].append({"p": p, "n": n, "e": acceptance.expected_accepted(m)})

for seed in (0, 1, 1234):
    for p, n in ((0.8, 4), (0.6, 8), (0.9, 2)):
        rng = np.random.default_rng(seed)
        d = acceptance.sample_accepted(acceptance.AcceptanceModel(p=p, n_cand=n), rng, size=64)
        out["draws"].append({"seed": seed, "p": p, "n": n, "counts": d.tolist()})

toy_t = ModelSpec("toy-target", 4, 64 * 1024**2, 256 * 1024**2, 128 * 1024**2, 4096)
toy_d = ModelSpec("toy-draft", 2, 16 * 1024**2, 48 * 1024**2, 32 * 1024**2, 1024)
hw = HardwareProfile(8 * GiB, 64 * GiB, 512 * GiB, 10e9, 10e9, 3e9, 1.5e9, 1e-4, 2e-4, 2e-3, 1e-3, 0.5)
for p, n, mx in ((1.0, 8, 16), (0.0, 4, 7), (0.8, 4, 16), (0.6, 2, 32)):
    pol = Policy(16, 16, 8, n)
    wl = Workload(32, 64, mx, p)
    r = simulator.simulate_decoding(pol, wl, hw, toy_t, toy_d, seed=0)
    out["rounds"].append({"p": p, "n": n, "max_new": mx, "rounds": r.rounds_executed,
                          "total_time": r.total_time, "peak": r.peak_gpu_bytes})

env, tgt, drf = presets.preset("env2_8x22b")
for pol in (Policy(16, 64, 8, 8), Policy(64, 256, 32, 4)):
    wl = Workload(2 * pol.bs_decoding, 503, 16, 0.8)
    c = costmodel.evaluate(pol, wl, env, tgt, drf)
    out["cost"].append({"policy": list(pol.as_tuple()), "t_prefill": c.t_prefill, "t_decoding": c.t_decoding,
                        "rounds": c.rounds, "v_decoding": c.v_decoding, "v_prefill": c.v_prefill,
                        "throughput": c.throughput, "feasible": c.feasible})
space = planner.SearchSpace((16, 32), (32, 64, 128), (8, 16), (2, 4, 8))
ranked = planner.search(space, Workload(256, 503, 16, 0.8), env, tgt, drf)
out["search_top"] = [{"policy": list(p.as_tuple()), "throughput": b.throughput} for p, b in ranked.entries[:5]]
out["presets"] = {k: dict(vars(v)) for k, v in (("mixtral_8x22b", presets.MIXTRAL_8X22B),
                                                  ("mixtral_8x7b", presets.MIXTRAL_8X7B),
                                                  ("mistral_7b", presets.MISTRAL_7B))}

path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_specpipe.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1, sort_keys=True)
print("wrote", path)
