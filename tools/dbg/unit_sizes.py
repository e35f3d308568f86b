"""Per-unit XC4 sizes of engines built the way bench.py builds them (whole vs split window)."""
import dataclasses
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2505_10259_b200 import MIXTRAL_8X22B, MISTRAL_7B_V3  # noqa: E402
from paper_2505_10259_b200.api import build_engine  # noqa: E402
from paper_2505_10259_b200.streamer import HostStore  # noqa: E402

t = dataclasses.replace(MIXTRAL_8X22B, n_layer=int(sys.argv[1]) if len(sys.argv) > 1 else 4)
d = dataclasses.replace(MISTRAL_7B_V3, n_layer=2)
for split in (False, True):
    store = HostStore()
    eng = build_engine(t, d, device="cuda:0", stream_layers=set(range(1, t.n_layer)), seed=1, trace=False,
                       host_store=store, codec="xc4", split_window=split)
    st = eng.target.streamer
    print(json.dumps({"split": split, "store_bytes": store.bytes,
                      "units": {li: [u.nbytes, u.n_frames, u.code_bits, u.frame_elems] for li, u in st.host.items()}}),
          flush=True)
    del eng, st
    store.close()
    torch.cuda.empty_cache()
