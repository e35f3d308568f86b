import math, sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2505_10259_b200 import native
DEV = "cuda"
def run(M, N, K, epi):
    g = torch.Generator(device=DEV).manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, device=DEV, generator=g).to(torch.bfloat16)
    b = (torch.randn(N, K, device=DEV, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    ref = a.float() @ b.float().T
    if epi == 3:
        blk = ref.view(M, N // 128, 2, 64)
        ref = (torch.nn.functional.silu(blk[:, :, 0]) * blk[:, :, 1]).reshape(M, N // 2)
    cols = N // 2 if epi == 3 else N
    outs = []
    for _ in range(3):
        out = torch.full((M, cols), float("nan"), dtype=torch.bfloat16, device=DEV)
        native.gemm(a, b, out, epi, None, variant=4)
        torch.cuda.synchronize()
        outs.append(out.float())
    for i, o in enumerate(outs):
        nan = torch.isnan(o)
        err = ((o - ref).abs() > 0.02 * (ref.abs() + ref.pow(2).mean().sqrt())) & ~nan
        print(f"M{M} N{N} K{K} epi{epi} run{i}: nan {int(nan.sum())} bad {int(err.sum())}", end=" ")
        if nan.any():
            r, c = nan.nonzero()[:, 0], nan.nonzero()[:, 1]
            print("nan rows", sorted(set(r.tolist()))[:8], "col tiles", sorted(set((c // 64).tolist()))[:20], end=" ")
        if err.any():
            r, c = err.nonzero()[:, 0], err.nonzero()[:, 1]
            print("bad col tiles", sorted(set((c // (64 if epi == 3 else 128)).tolist()))[:20], end=" ")
        print()
for shape in [(64, 1024, 4096, 3), (64, 28672, 4096, 3), (64, 28672, 4096, 0), (64, 4096, 4096, 3), (16, 28672, 4096, 3)]:
    run(*shape)
