"""Experiment: per-rank transform cost of the replicated grid (one full 3D
D2Z + Z2D per rank) against one part of the slab decomposition (pme.cu
PmeDoms::slab_solve: 2D D2Z over the part's x-planes, 1D Z2Z along x over its
ky columns forward and inverse, 2D Z2D), at config 4's 216^3 grid for 2, 4
and 8 parts. cuFFT through torch.fft (the same library the product links),
FP64, CUDA events, median of 20. Transfer volumes per rank per PME pass
are computed, not measured (no multi-GPU box)."""
import json
import sys

import torch

K = int(sys.argv[1]) if len(sys.argv) > 1 else 216
dev = "cuda"
g = torch.randn(K, K, K, dtype=torch.float64, device=dev)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[n // 2]


out = {"grid": K, "full_3d_ms": t(lambda: torch.fft.irfftn(torch.fft.rfftn(g), s=(K, K, K)))}
kzh = K // 2 + 1
for P in (2, 4, 8):
    nx = -(-K // P)
    ny = -(-K // P)
    planes = g[:nx].contiguous()
    cols = torch.randn(K, ny, kzh, dtype=torch.complex128, device=dev)

    def part():
        a = torch.fft.rfft2(planes)
        c = torch.fft.ifft(torch.fft.fft(cols, dim=0), dim=0)
        return torch.fft.irfft2(a, s=(K, K)), c
    grid_b = K ** 3 * 8
    out[f"P{P}"] = {
        "part_ms": t(part),
        "replicated_bytes_per_rank": 2 * grid_b * (P - 1) / P,  # all-reduce
        "slab_bytes_per_rank": (grid_b * (P - 1) / P  # reduce onto slabs
                                + 2 * 2 * K * K * kzh * 8 * (P - 1) / P / P  # two transposes
                                + grid_b * (P - 1) / P),  # gather of the slabs
    }
print(json.dumps(out))
json.dump(out, open("gpurun_out/slab_fft.json", "w"), indent=1)
