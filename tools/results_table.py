"""BASELINE.md results table: one HeteroConv layer fwd+bwd per
config C1-C4 (C3 at k = 8, 16, 32) through the C ABI on one B200.

Per row: layer ms/iter (CUDA events, 3 streams, median of 20, L2 flushed),
SpMM ms and projection ms (per-launch CUDA events, single stream), SpMM
algorithmic GB/s and its fraction of the measured HBM peak, SpMM ncu DRAM GB/s
(profiles/ncu_traffic.json, where captured), the fp64 oracle's layer fwd+bwd at
1 thread and at all host threads (scope "spmm" -- D-ReLU + 3 SpMM + SSpMMs -- on
C4, whose fp64 projections alone are ~286 GFLOP), and the parity max error of
the layer outputs, weight gradients and input gradients against the oracle fed
the GPU's fp32 decisions (reading Q28).
usage: python tools/results_table.py [C1 C2 C3 C4] > profiles/r02/results_table.json"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2508_16769_b200 as dr
from gen import make_config, make_params
from oracle import oracle as O

HBM = bench.peaks()[0]


def row_err(g, o):
    g = np.atleast_2d(np.asarray(g, np.float64))
    o = np.atleast_2d(np.asarray(o, np.float64))
    n = np.linalg.norm(o, axis=1)
    tau = max(1e-6 * float(np.sqrt(np.mean(n ** 2))) if n.size else 0.0, 1e-30)
    return float((np.abs(g - o).max(axis=1) / np.maximum(n, tau)).max()) if o.size else 0.0


def unpack(words, D):
    w = words.view(np.uint32)
    bits = (w[:, :, None] >> np.arange(32, dtype=np.uint32)[None, None, :]) & 1
    return bits.reshape(w.shape[0], -1)[:, :D].astype(bool)


def oracle_time(fn, reps):
    ts = []
    for _ in range(reps):
        t = time.time()
        fn()
        ts.append(time.time() - t)
    return float(np.median(ts)) * 1e3


def one(name, k=None):
    d = make_config(name)
    D = d.meta["D"]
    k = k or d.meta["k"]
    g = dr.Graph.from_design(d)
    P = make_params(D, D, D, 1, seed=7)
    W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
    L = dr.Layer(W, D, D, D, k, k)
    xc, xn = torch.as_tensor(d.x_cell).cuda(), torch.as_tensor(d.x_net).cuda()
    rng = np.random.default_rng(1)
    dyc_h = rng.standard_normal((d.n_cell, D)).astype(np.float32)
    dyn_h = rng.standard_normal((d.n_net, D)).astype(np.float32)
    dyc, dyn = torch.as_tensor(dyc_h).cuda(), torch.as_tensor(dyn_h).cuda()
    tape = torch.empty(L.tape_bytes(g), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 18, device="cuda")

    def step(i=0):
        dr.heteroconv_fwd(g, L, xc, xn, tape=tape)
        dr.heteroconv_bwd(g, L, tape, dyc, dyn, need_dx=True)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    dr.profile_begin()
    for _ in range(5):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    prof = dr.profile_end()
    wl = name if name in ("C2", "C4") else name + "x"
    table = bench.kernel_table(prof, d, D, k, wl, tiled=g.info()["tiles"][0] > 0)
    gate = bench.spmm_gate(table, HBM)
    spmm_ms = gate["ms_total"] / 5 if gate else None
    proj_ms = sum(v["total_ms"] for t, v in table.items() if t.startswith("tc_")) / 5
    traffic = bench.load_json("ncu_traffic.json").get(name, {})
    sp_tags = [t for t in table if t.startswith("spmm")]
    dram = None
    if traffic and all(t in traffic for t in sp_tags) and k == d.meta["k"]:
        db = sum(traffic[t] * table[t]["launches"] for t in sp_tags) / 5
        dram = db / (spmm_ms * 1e-3) / 1e9
    # ---- parity: one fwd+bwd against the oracle fed the GPU's decisions
    yc, yn, tp = dr.heteroconv_fwd(g, L, xc, xn, flags=dr.DR_FWD_TAPS)
    v = dr.tape_view(g, L, tp, dr.DR_FWD_TAPS)
    grads, dxc, dxn = dr.heteroconv_bwd(g, L, tp, dyc, dyn, need_dx=True, flags=dr.DR_FWD_TAPS)
    G = O.OGraph(d)
    Wo = O.layer_params(P, 0)
    forced = dict(hc_idx=v["hc_idx"].cpu().numpy().astype(np.int32),
                  hn_idx=v["hn_idx"].cpu().numpy().astype(np.int32),
                  M=unpack(v["mask"].cpu().numpy(), D))
    t0 = time.time()
    oyc, oyn, otape = O.layer_fwd(G, Wo, d.x_cell, d.x_net, k, k, forced=forced)
    og, odxc, odxn = O.layer_bwd(G, Wo, otape, dyc_h, dyn_h, need_dx=True)
    errs = {"y_cell": row_err(yc.cpu().numpy(), oyc), "y_net": row_err(yn.cpu().numpy(), oyn),
            "dx_cell": row_err(dxc.cpu().numpy(), odxc), "dx_net": row_err(dxn.cpu().numpy(), odxn)}
    for key in og:
        errs["grad." + key] = row_err(grads[key].cpu().numpy(), og[key])
    hc_exact = bool(np.array_equal(v["hc_idx"].cpu().numpy().astype(np.int32), O.drelu(d.x_cell, k)[0]))
    # ---- oracle timing: full layer fwd+bwd (C4: scope spmm)
    if name == "C4":
        dzc, dzn = dyc_h.astype(np.float64), dyn_h.astype(np.float64)

        def ofn():
            ic, vc = O.drelu(d.x_cell, k)
            i_n, vn = O.drelu(d.x_net, k)
            G.fwd("near", ic, vc, D)
            G.fwd("pins", ic, vc, D)
            G.fwd("pinned", i_n, vn, D)
            G.bwd("near", ic, dzc)
            G.bwd("pins", ic, dzn)
            G.bwd("pinned", i_n, dzc)
        scope = "spmm (D-ReLU x2 + SpMM x3 + SSpMM x3)"
    else:
        def ofn():
            _, _, tpo = O.layer_fwd(G, Wo, d.x_cell, d.x_net, k, k)
            O.layer_bwd(G, Wo, tpo, dyc_h, dyn_h, need_dx=True)
        scope = "layer fwd+bwd"
    nthr = O.num_threads()
    reps = 1 if name == "C4" else 3
    o_n = oracle_time(ofn, reps)
    O.set_num_threads(1)
    o_1 = oracle_time(ofn, 1)
    O.set_num_threads(nthr)
    g.close()
    sp_bytes = gate["alg_bytes_total"] / 5 if gate else 0
    return {"config": name, "k": k, "D": D, "n_cell": d.n_cell, "n_net": d.n_net, "nnz": d.nnz(),
            "layer_ms": round(ms, 4), "spmm_ms": round(spmm_ms, 4) if spmm_ms else None,
            "spmm_alg_gbs": round(sp_bytes / (spmm_ms * 1e-3) / 1e9, 1) if spmm_ms else None,
            "spmm_alg_frac": round(sp_bytes / (spmm_ms * 1e-3) / 1e9 / HBM, 4) if spmm_ms else None,
            "spmm_dram_gbs_ncu": round(dram, 1) if dram else None,
            "spmm_dram_frac": round(dram / HBM, 4) if dram else None,
            "proj_ms": round(proj_ms, 4),
            "oracle_ms_1thr": round(o_1, 1), "oracle_ms_nthr": round(o_n, 1), "oracle_threads": nthr,
            "oracle_scope": scope, "parity_max_row_err": max(errs.values()),
            "parity_worst": max(errs, key=errs.get), "drelu_idx_bitexact_layer_input": hc_exact,
            "hbm_peak_gbs": HBM}


if __name__ == "__main__":
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4"]
    out = []
    for n in names:
        for k in ([8, 16, 32] if n == "C3" else [None]):
            r = one(n, k)
            print(json.dumps(r), file=sys.stderr, flush=True)
            out.append(r)
    print(json.dumps(out, indent=1))
