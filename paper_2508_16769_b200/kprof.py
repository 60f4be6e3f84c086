"""K-profiling: choose the D-ReLU sparsity k per relation by timing.

The paper selects its sparsity parameter by profiling ("K ... decided by
a pre-profiling process", Fig. 9: the K range 2-8 works best on its
GPU; SPEC S:369-377 describes the same sweep for the CPU program). Here, per
relation psi in {near, pins, pinned}, one sweep point is the relation's whole
sparse path on the caller's graph and features, all through the C ABI:

    D-ReLU of the source features (Eq. 2-3) -> DR-SpMM forward (Eq. 5-7)
    -> SSpMM backward with the D-ReLU mask gradient (Eq. 10-11),

timed with CUDA events on the current stream (median of `reps` after one
warm-up), for k in `ks` intersected with [1, D]. The choice is the argmin,
ties to the smaller k. Host-side orchestration only: every step runs in
libdr's kernels (the tensor-core tiled SpMM for near where it applies, the
SIMT kernels otherwise), so the profile reflects the kernels the k would run.
"""
from __future__ import annotations

import numpy as np

RELS = ("near", "pins", "pinned")
SRC = {"near": "cell", "pins": "cell", "pinned": "net"}


def kprofile(g, x_cell, x_net, ks=(2, 4, 8, 16, 32, 64), reps=5, seed=0):
    """Returns {rel: {"times_ms": {k: ms}, "best_k": k}} for the three relations."""
    import torch

    from . import drelu_topk, spmm_bwd, spmm_fwd

    info = g.info()
    n_dst = {"near": info["n_cell"], "pins": info["n_net"], "pinned": info["n_cell"]}
    gen = torch.Generator(device=x_cell.device).manual_seed(seed)
    out = {}
    for rel in RELS:
        x = x_cell if SRC[rel] == "cell" else x_net
        D = int(x.shape[1])
        dz = torch.randn((n_dst[rel], D), device=x.device, generator=gen)
        z = torch.empty((n_dst[rel], D), device=x.device)
        dx = torch.empty_like(x)
        times = {}
        for k in ks:
            if k < 1 or k > D:
                continue

            def path():
                val, idx = drelu_topk(x, k)
                spmm_fwd(g, rel, val, idx, D, out=z)
                spmm_bwd(g, rel, dz, val, idx, D, want_g=False, want_dx=True, dx_out=dx)

            path()
            samples = []
            for _ in range(reps):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                path()
                b.record()
                b.synchronize()
                samples.append(a.elapsed_time(b))
            times[k] = float(np.median(samples))
        best = min(sorted(times), key=lambda kk: (times[kk], kk))
        out[rel] = {"times_ms": times, "best_k": best}
    return out
