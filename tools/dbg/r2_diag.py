"""Round-2 numerics diagnostics (GPU): small-M GEMMs at the path's shapes through
native.gemm (auto choice) vs fp32 torch, and per-token error of the 1-layer
parity tests.  Debug tool; prints JSON lines."""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2505_10259_b200 import native  # noqa: E402

DEV = "cuda"


def gemm_case(M, N, K, epi, variant=0):
    g = torch.Generator(device=DEV).manual_seed(M + N + K)
    a = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
    b = (torch.randn(N, K, device=DEV, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    ref = a.float() @ b.float().T
    out = torch.empty(M, N, dtype=torch.float32 if epi == native.EPI_F32 else torch.bfloat16, device=DEV)
    native.gemm(a, b, out, epi, variant=variant)
    torch.cuda.synchronize()
    d = (out.float() - ref).abs()
    bad_rows = (d.max(1).values > 0.05 * ref.abs().max()).nonzero().flatten().tolist()
    bad_cols = (d.max(0).values > 0.05 * ref.abs().max()).nonzero().flatten()
    print(json.dumps({"M": M, "N": N, "K": K, "epi": epi, "variant": variant, "max_err": d.max().item(),
                      "nan": int(torch.isnan(out).sum().item()), "ref_max": ref.abs().max().item(),
                      "bad_rows": bad_rows[:20], "n_bad_cols": int(bad_cols.numel()),
                      "bad_col_first": bad_cols[:8].tolist()}), flush=True)


def main():
    if "--layers-only" in sys.argv:
        return layers()
    for M in (18, 64, 160):
        gemm_case(M, 32768, 6144, native.EPI_F32)
        gemm_case(M, 8192, 6144, native.EPI_BF16)
        gemm_case(M, 6144, 6144, native.EPI_BF16)
    for (M, N, K) in [(64, 6144, 4096), (64, 4096, 14336), (33, 2048, 2048)]:
        gemm_case(M, N, K, native.EPI_F32, variant=4)
        gemm_case(M, N, K, native.EPI_F32, variant=1)
        gemm_case(M, N, K, native.EPI_F32, variant=4)
    layers()


def layers():
    import test_parity_8x22b_gpu as T
    import dataclasses
    for name, arch, mo, sl, codec, kw in [
            ("8x22b", dataclasses.replace(T.MIXTRAL_8X22B, n_layer=1), lambda e: e.target, {0}, "xc4", {}),
            ("mistral", T.MISTRAL_7B_V3_1L, lambda e: e.draft, set(), "none", {"n_seq": 32, "n_cand": 4})]:
        got, want, gap, want32 = T._layer_parity(arch, mo, sl, codec, **kw)
        d = np.abs(got - want)
        tok = d.max(-1)
        order = np.argsort(-tok.reshape(-1))[:12]
        rms = np.sqrt((d ** 2).mean(-1))
        print(json.dumps({"case": name, "max": float(d.max()), "rms_err": float(np.sqrt((d ** 2).mean())),
                          "rms_want": float(np.sqrt((want ** 2).mean())),
                          "worst_tokens": [[int(i), float(tok.reshape(-1)[i]), float(rms.reshape(-1)[i]),
                                            None if gap is None else float(gap.reshape(-1)[i])] for i in order],
                          "median_token_max": float(np.median(tok)),
                          "rms_gpu_vs_fp32": float(np.sqrt(((got - want32) ** 2).mean())),
                          "rms_oracle_vs_fp32": float(np.sqrt(((want - want32) ** 2).mean()))}), flush=True)


if __name__ == "__main__":
    main()
