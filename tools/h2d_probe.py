#!/usr/bin/env python
"""Host→device link probe: one copy stream vs two concurrent copy streams vs an
SM-driven zero-copy kernel (so_copy_sm over UVA), pinned 1 GiB buffers."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_10259_b200 import native  # noqa: E402


def main():
    n = 1 << 30
    dev = torch.device("cuda", 0)
    h = torch.empty(2 * n, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(2 * n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}

    def timed(fn, nbytes, reps=5):
        best = 0.0
        for _ in range(reps):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
        return best

    def one():
        with torch.cuda.stream(s1):
            d[:n].copy_(h[:n], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)

    def two():
        with torch.cuda.stream(s1):
            d[:n].copy_(h[:n], non_blocking=True)
        with torch.cuda.stream(s2):
            d[n:].copy_(h[n:], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    def chunks():  # 8 × 128 MiB alternating over the two streams
        c = n // 4
        for i in range(8):
            st = s1 if i % 2 == 0 else s2
            with torch.cuda.stream(st):
                d[i * c:(i + 1) * c].copy_(h[i * c:(i + 1) * c], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    res["one_stream_1GiB"] = timed(one, n)
    res["two_streams_2x1GiB"] = timed(two, 2 * n)
    res["two_streams_8x256MiB"] = timed(chunks, 2 * n)
    res["sm_zero_copy_1GiB"] = timed(lambda: native.copy_sm(d.data_ptr(), h.data_ptr(), n,
                                                            torch.cuda.current_stream()), n)
    print(json.dumps({k: round(v, 2) for k, v in res.items()}))


if __name__ == "__main__":
    main()
