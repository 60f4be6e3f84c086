"""bench.py — DR-CircuitGNN hot path on B200 (BASELINE.json metric).

Headline (default, BASELINE configs[4] = C5): data-parallel training on the
Mini-CircuitNet-shaped set (100 synthetic designs of 2-4 graphs, 7.3-9.8k cells
each; "100 training designs"). Every step each rank
trains on its own packed batch (disjoint union of B designs, packed to equal
edge counts across ranks) through dr_train_step: 2 HeteroConv layers (D-ReLU ->
3x DR-SpMM -> projections / max-merge) -> head / MSE -> backward incl. SSpMM ->
the in-library NCCL allreduce of the flat gradient -> Adam. value = graphs/s
over all ranks (weak scaling: fixed per-rank batch).

At N=1 the same invocation also measures the north_star gate on C4
(BASELINE configs[3], CircuitNet-large-shaped, 1M cells, D=128, k=16): one
HeteroConv layer fwd+bwd, its SpMM fwd+bwd fraction of HBM on algorithmic and
on ncu DRAM bytes, the identity-order (pure DRAM) gate beside the shipped
locality-order one, and the L2 copy bandwidth as the second ceiling ("c4").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload C5|C2|C4] [--batch-designs B] [--no-c4]

--gpus N > 1 without WORLD_SIZE in the environment re-launches itself under
torch.distributed.run with N ranks (one GPU each; fails if fewer GPUs exist).
--impl reference times the fp64 CPU oracle (oracle/) on the host cores on the
same workload (rank 0 only), as the reference arm.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HeteroConv fwd+bwd ms/iter and achieved HBM GB/s; train graphs/sec at 1/2/4/8 GPU"
FALLBACK_HBM_GBS = 6650.0          # B200_PROFILING.md fallback
FALLBACK_BF16_TFLOPS = 1590.0
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # SMs x FP32 lanes x FMA x max clock
DTYPE = "f32 (fp32 storage/accumulation; tensor-core contractions as 3xbf16 hi/lo split, " \
        "<= 2^-16 relative per product)"
DATA = "synthetic (seeded CircuitNet-shaped generator gen/circuit.py, random-init weights)"
C5_DESIGNS = 100
SCHED_SEED = 77


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), float(j.get("bf16_tflops", FALLBACK_BF16_TFLOPS)), "measured"
    return FALLBACK_HBM_GBS, FALLBACK_BF16_TFLOPS, "fallback"


# ------------------------------------------------------------------ clocks
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ algorithmic work per kernel tag
def kernel_work(tag, d, D, k, tiled=True, chained=False):
    """(bytes, flops) per launch for a profile tag, SURVEY §8(d) per-unit figures
    (restated in DESIGN.md §5 'Algorithmic bytes'). Pair = 4 B value + 1 B index.
    tiled: near's backward runs as the tensor-core tiled kernel (near term + extra)
    after the SIMT pins term ('spmm_bwd.cell.pins', written into the extra term)."""
    parts = tag.split(".")
    kind = parts[0]
    rel = parts[-1]
    nnz = {r: int(d.rel(r)[1].size) for r in ("near", "pins", "pinned")}
    ndst = {"near": d.n_cell, "pins": d.n_net, "pinned": d.n_cell}
    if kind == "spmm_bwd" and rel == "pins" and len(parts) >= 3 and parts[-2] == "cell":
        return nnz["pins"] * (4 + 4 * k) + d.n_cell * (k + 4 * k + 4 * k), 0.0
    if kind == "spmm_fwd":
        ew = 4 if rel == "pinned" else 0          # GraphConv s_j folded into a per-edge weight
        return nnz[rel] * (4 + 5 * k + ew) + ndst[rel] * (4 + 4 * D), 0.0
    if kind == "spmm_bwd":
        rels = (["near"] if tiled else ["near", "pins"]) if rel == "cell" else ["pinned"]
        n = d.n_cell if rel == "cell" else d.n_net
        return sum(nnz[r] * (4 + 4 * k) for r in rels) + n * (k + 4 * k + 4 * D), 0.0
    if kind == "drelu":
        n = d.n_cell if rel == "cell" else d.n_net
        return n * D * 4 + n * k * 5, 0.0
    if kind == "tc_dz":     # dY read (+ merge-mask words for cell rows), dZ' written, root term
        n = ndst.get(rel, d.n_cell)
        root = rel in ("near", "pins")
        mask = D // 8 if rel in ("near", "pinned") else 0
        return (n * (4 * D + mask + 4 * D + (k + 4 * k if root else 0)),
                2.0 * n * D * (2 * D if root else D))
    if kind == "tc_proj":
        n = d.n_cell if rel == "cell" else d.n_net
        # chained (the trainer's hidden layers, row a5): the next layer's CBSR
        # (5 k B per row) is written instead of the dense Y (4 D B per row)
        out = 5 * k if (chained and len(parts) == 3 and parts[1] == "L0") else 4 * D
        if rel == "cell":       # Z_near, Z_pinned read, CBSR root input, Y + mask written
            return n * (2 * D * 4 + 5 * k + out + D // 8), 2.0 * n * D * (3 * D)
        return n * (D * 4 + 5 * k + out), 2.0 * n * D * (2 * D)
    if kind == "tc_dw" and rel == "near_pinned":   # dual B: Z_near, CBSR root, Z_pinned, dY, mask
        n = d.n_cell
        return n * (4 * D + 5 * k + 4 * D + 4 * D + D // 8), 2.0 * n * (2 * D) * D + 2.0 * n * D * D
    if kind == "tc_dw":     # Z rows (+ CBSR root input) and dY rows (+ mask words) read
        n = ndst.get(rel, d.n_cell)
        root = rel in ("near", "pins")
        mask = D // 8 if rel in ("near", "pinned") else 0
        kin = 2 * D if root else D
        return n * (4 * D + (5 * k if root else 0) + 4 * D + mask), 2.0 * n * kin * D
    return 0, 0.0


def load_json(name):
    p = os.path.join(ROOT, "profiles", name)
    return json.load(open(p)) if os.path.exists(p) else {}


def kernel_table(prof, d, D, k, workload, tiled=True, chained=False):
    traffic = load_json("ncu_traffic.json").get(workload, {})
    bounds = load_json("ncu_bounds.json").get(workload, {})
    table = {}
    for tag, (n, tot, mx) in prof.items():
        b, f = kernel_work(tag, d, D, k, tiled, chained)
        per = tot / max(n, 1)
        tr = traffic.get(tag)
        table[tag] = dict(launches=n, total_ms=round(tot, 4), mean_ms=round(per, 5),
                          alg_bytes=int(b), alg_flops=float(f),
                          alg_gbs=round(b / (per * 1e-3) / 1e9, 1) if b and per > 0 else None,
                          dram_bytes_ncu=tr,
                          dram_gbs_ncu=round(tr / (per * 1e-3) / 1e9, 1) if tr and per > 0 else None,
                          tflops=round(f / (per * 1e-3) / 1e12, 2) if f and per > 0 else None,
                          ncu_bound=bounds.get(tag))
    return table


def roofline(table, hbm, bf16, src):
    """Dominant kernel tag by total device time; achieved = algorithmic bytes (or
    issued FLOPs) per launch / its mean launch time, against the ceiling that
    binds it; `traffic` = ncu DRAM bytes per launch of that tag."""
    if not table:
        return None
    dom = max(table, key=lambda t: table[t]["total_ms"])
    e = table[dom]
    per_s = e["mean_ms"] * 1e-3
    b = e["alg_bytes"]
    f = e["alg_flops"]
    kind = dom.split(".")[0]
    rf = {"kernel": dom, "traffic": e["dram_bytes_ncu"], "ncu_bound": e["ncu_bound"],
          # the unit that actually limits it (ncu, profiles/ncu_bounds.json): the
          # roofline below is the HBM / tensor ceiling, "latency" = neither is close
          "limiter": (e["ncu_bound"] or {}).get("bound")}
    if kind.startswith("tc_") and 3.0 * f / (bf16 * 1e12) > b / (hbm * 1e9):
        ach = 3.0 * f / per_s / 1e12
        rf.update(bound="tensor", achieved=round(ach, 2), peak=round(bf16, 1), unit="TFLOP/s",
                  frac=round(ach / bf16, 4),
                  peak_source="MEASURED_PEAKS.json bf16_tflops (issued = 3 x useful, bf16 hi/lo split)")
    else:
        ach = b / per_s / 1e9
        rf.update(bound="hbm", achieved=round(ach, 1), peak=hbm, unit="GB/s",
                  frac=round(ach / hbm, 4), peak_source=f"MEASURED_PEAKS.json hbm_gbs ({src})")
        if e["dram_bytes_ncu"]:
            rf["dram_frac"] = round(e["dram_bytes_ncu"] / per_s / 1e9 / hbm, 4)
    return rf


def spmm_gate(table, hbm, l2=None):
    """north_star target: the HeteroConv forward + backward SpMM (every spmm_fwd.*
    and spmm_bwd.* launch: near tiled, pins/pinned SIMT, the pins term) at >= 60 %
    of HBM bandwidth. Reported on algorithmic bytes (SURVEY §8(d) gate) and on
    the ncu-measured DRAM bytes of the same launches (profiles/ncu_traffic.json)."""
    sp = {t: v for t, v in table.items() if t.startswith("spmm_")}
    ms = sum(v["total_ms"] for v in sp.values())
    if ms <= 0:
        return None
    nb = sum(v["alg_bytes"] * v["launches"] for v in sp.values())
    gbs = nb / (ms * 1e-3) / 1e9
    out = {"ms_total": round(ms, 4), "alg_bytes_total": int(nb), "alg_gbs": round(gbs, 1),
           "peak_gbs": hbm, "frac": round(gbs / hbm, 4), "target_frac": 0.6}
    if all(v["dram_bytes_ncu"] for v in sp.values()):
        db = sum(v["dram_bytes_ncu"] * v["launches"] for v in sp.values())
        out.update(dram_bytes_total_ncu=int(db), dram_gbs_ncu=round(db / (ms * 1e-3) / 1e9, 1),
                   dram_frac=round(db / (ms * 1e-3) / 1e9 / hbm, 4))
    if l2:
        out["alg_frac_of_l2_read"] = round(gbs / l2, 4)
    out["note"] = ("sum over the spmm_fwd.* / spmm_bwd.* launches of the per-kernel pass "
                   "(per-launch CUDA events, single stream)")
    return out


# ------------------------------------------------------------------ helpers (GPU)
def l2_read_gbs(torch, dev, mb=32, reps=100):
    """Second ceiling: L2 READ bandwidth, measured with libdr's
    read probe (dr_probe_read: a persistent grid streaming a `mb` MB buffer,
    about 1/4 of the 126 MB L2, `reps` times with 128-bit loads; CUDA events,
    best of 5). Read bytes only."""
    import paper_2508_16769_b200 as dr
    a = torch.empty(mb * (1 << 20) // 4, device=dev)
    a.normal_()
    sink = torch.empty(148 * 4, device=dev)
    dr.probe_read(a, 3, sink)
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dr.probe_read(a, reps, sink)
        e1.record()
        e1.synchronize()
        best = max(best, a.numel() * 4 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return best


def gpu_local_cpus(dev):
    """CPUs on the GPU's NUMA node (NVML), or None. Pinned host buffers first
    touched by a thread bound there live in the GPU-local node's memory."""
    try:
        import pynvml
        import torch
        p = torch.cuda.get_device_properties(dev)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(
            f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0".encode())
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def timed_steps(torch, step, n, flush, events_stream=None, chunk=16, barrier=None):
    """n steps, L2 flushed (256 MB write) before each, outside CUDA events on the
    caller's stream; returns the summed device time in ms.
    Enqueued in chunks of `chunk` steps, each behind a spin kernel (outside every
    event pair) that holds the device while the host enqueues the whole chunk, and
    drained before the next: a host stall (Python, a driver lock held by the
    nvidia-smi clock sampler) or a full launch queue (~40 C5 steps of kernels) then
    cannot leave the device idle between a step's events, which bracket device
    execution only; the garbage collector is off meanwhile. Measured with the
    events alone: single steps of 1.3-60 ms against a 0.51 ms median (C5), the
    device having caught up with a stalled host."""
    import gc
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(n)]
    gc.collect()
    gc.disable()                             # no collector pause while a chunk is enqueued
    try:
        for c0 in range(0, n, chunk):
            torch.cuda.synchronize()
            if barrier is not None:          # ranks start each chunk together (the step's
                barrier()                    # allreduce must not wait on a late rank's spin)
                torch.cuda.synchronize()
            torch.cuda._sleep(int(1e8))      # ~0.05 s at ~2 GHz: the host enqueues the chunk meanwhile
            for i in range(c0, min(n, c0 + chunk)):
                flush.zero_()
                ev[i][0].record()
                step(i)
                ev[i][1].record()
        torch.cuda.synchronize()
    finally:
        gc.enable()
    per = [a.elapsed_time(b) for a, b in ev]
    timed_steps.last = per
    if os.environ.get("BENCH_STEP_LIST"):
        log("per-step ms:", " ".join(f"{x:.3f}" for x in per))
    return sum(per)


def step_stats(per):
    s = sorted(per)
    return {"min": round(s[0], 4), "median": round(s[len(s) // 2], 4), "max": round(s[-1], 4),
            "argmax": int(max(range(len(per)), key=lambda i: per[i])),
            "first_of_chunks": [round(per[i], 4) for i in range(0, len(per), 16)]}


# ------------------------------------------------------------------ C5 schedule
def c5_schedule(world, B, n_designs=C5_DESIGNS):
    """Deterministic per-step, per-rank batches of the C5 set (SURVEY §8(d) 'DP
    throughput'): a fixed permutation of the designs is cut into S = n // (world*B)
    groups of world*B designs; each group is packed onto the ranks by expected
    edge count (LPT, paper_2508_16769_b200.dist.pack_batches). Returns
    (batches[s][r] = design ids, specs)."""
    from gen.circuit import c5_expected_nnz, c5_specs
    from paper_2508_16769_b200.dist import pack_batches
    specs = c5_specs(n_designs)
    perm = np.random.Generator(np.random.PCG64(SCHED_SEED)).permutation(n_designs)
    S = max(1, n_designs // (world * B))
    out = []
    for s in range(S):
        grp = [int(i) for i in perm[s * world * B:(s + 1) * world * B]]
        if len(grp) < world:
            grp = [int(perm[(s * world * B + q) % n_designs]) for q in range(world)]
        work = [c5_expected_nnz(specs[i]) for i in grp]
        out.append([[grp[i] for i in b] for b in pack_batches(work, world)])
    return out, specs


def c5_batch_design(ids, designs):
    from gen.circuit import disjoint_union
    graphs = [g for i in ids for g in designs[i]]
    u = disjoint_union(graphs, name="C5 batch " + ",".join(map(str, ids)))
    u.meta["n_graphs"] = len(graphs)
    return u


def gpu_decisions(dr, torch, g, d, P, nl, D, k, dev):
    """The integer decisions the GPU step takes in fp32 (DESIGN reading Q28): per
    layer the D-ReLU selections of both node types and the max-merge mask, read
    from the layer ABI's tapes (the same kernels, bit-identical to the trainer's
    fused path: tests/test_gpu_chain.py)."""
    out = []
    xc = torch.as_tensor(d.x_cell).to(dev)
    xn = torch.as_tensor(d.x_net).to(dev)
    dc, dn = d.x_cell.shape[1], d.x_net.shape[1]
    for l in range(nl):
        W = {kk.split(".", 1)[1]: torch.as_tensor(v).to(dev) for kk, v in P.items()
             if kk.startswith(f"l{l}.")}
        L = dr.Layer(W, dc, dn, D, k, k)
        yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn)
        v = dr.tape_view(g, L, tape)
        words = v["mask"].cpu().numpy().view(np.uint32)
        bits = (words[:, :, None] >> np.arange(32, dtype=np.uint32)[None, None, :]) & 1
        out.append(dict(hc_idx=v["hc_idx"].cpu().numpy().astype(np.int32),
                        hn_idx=v["hn_idx"].cpu().numpy().astype(np.int32),
                        M=bits.reshape(words.shape[0], -1)[:, :D].astype(bool)))
        xc, xn, dc, dn = yc, yn, D, D
    return out


def oracle_grads_flat(dr, d, P, nl, k, forced=None):
    """fp64 oracle loss and flat gradient; with `forced` the GPU's fp32 decisions
    are fed in (reading Q28) and their validity against the oracle's own values
    is returned as well."""
    from oracle import oracle as O
    G = O.OGraph(d)
    loss, og, tapes = O.model_fwd_bwd(G, {kk: np.asarray(v, np.float64) for kk, v in P.items()},
                                      nl, k, k, d.x_cell, d.x_net, d.labels, forced=forced)
    flat = np.concatenate([np.asarray(og[f"l{l}.{kk}"], np.float64).reshape(-1)
                           for l in range(nl) for kk in dr.PARAM_ORDER] +
                          [np.asarray(og["head.w"], np.float64).reshape(-1),
                           np.asarray(og["head.b"], np.float64).reshape(-1)])
    valid = None
    if forced is not None:
        valid = {"drelu_gap_min": float("inf"), "merge_gap_min": float("inf"),
                 "rows_decided_differently": 0, "rows": 0}
        for t in tapes:
            for x, idx in ((t["x_c"], t["hc_idx"]), (t["x_n"], t["hn_idx"])):
                gap = O.drelu_gap(x, idx)
                valid["drelu_gap_min"] = min(valid["drelu_gap_min"], float(gap.min()))
                own, _ = O.drelu(x, idx.shape[1])
                valid["rows_decided_differently"] += int(np.any(own != idx, axis=1).sum())
                valid["rows"] += int(x.shape[0])
            mg = O.merge_gap(t["y_near"], t["y_pinned"], t["M"])
            valid["merge_gap_min"] = min(valid["merge_gap_min"], float(mg.min()))
            valid["rows_decided_differently"] += int(np.any(t["M"] != (t["y_near"] >= t["y_pinned"]),
                                                            axis=1).sum())
    return loss, flat, valid


def row_err(gpu, ref):
    """max_r max_d |g - o| / max(||o_r||, tau) (SURVEY §8(c) parity metric)."""
    g = np.atleast_2d(np.asarray(gpu, np.float64))
    o = np.atleast_2d(np.asarray(ref, np.float64))
    n = np.linalg.norm(o, axis=1)
    tau = max(1e-6 * float(np.sqrt(np.mean(n ** 2))), 1e-30)
    return float((np.abs(g - o).max(axis=1) / np.maximum(n, tau)).max())


def split_flat(dr, a, b, nl, D):
    ua, ub = dr.unflatten(a, nl, D, D, D), dr.unflatten(b, nl, D, D, D)
    return {kk: (ua[kk], ub[kk]) for kk in ua}


def oracle_train_timer(d, P, nl, k):
    """One full oracle training step (fwd, bwd, Adam) on design d, as a closure."""
    from oracle import oracle as O
    G = O.OGraph(d)
    st = {"P": {kk: np.asarray(v, np.float64) for kk, v in P.items()}, "t": 0}

    def step():
        loss, grads, _ = O.model_fwd_bwd(G, st["P"], nl, k, k, d.x_cell, d.x_net, d.labels)
        st["t"] += 1
        for kk in st["P"]:
            th, m, v = O.adam(st["P"][kk], grads[kk],
                              st.get("m_" + kk, np.zeros_like(grads[kk])),
                              st.get("v_" + kk, np.zeros_like(grads[kk])), st["t"])
            st["P"][kk], st["m_" + kk], st["v_" + kk] = th, m, v
        return loss
    return step, O


# ------------------------------------------------------------------ our arm: C5 DP training
def run_c5(args, torch, dist, dr, rank, world, local, dev, hbm, bf16, src):
    from gen import make_params
    from gen.circuit import make_c5_set
    from paper_2508_16769_b200 import dist as ddp

    D, k, nl, B = 64, 8, 2, args.batch_designs
    batches, specs = c5_schedule(world, B)
    S = len(batches)
    mine = [batches[s][rank] for s in range(S)]
    t0 = time.time()
    need = sorted({i for b in mine for i in b})
    nw = max(1, (os.cpu_count() or 2) // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world))))
    designs = make_c5_set(C5_DESIGNS, only=need, workers=min(nw, 32))
    bd = [c5_batch_design(b, designs) for b in mine]
    log(f"[rank {rank}] C5: {S} batches x {B} designs, {sum(x.meta['n_graphs'] for x in bd)} "
        f"graphs, generated in {time.time() - t0:.1f}s")
    t0 = time.time()
    graphs = [dr.Graph.from_design(x) for x in bd]
    inputs = [(torch.as_tensor(x.x_cell).to(dev), torch.as_tensor(x.x_net).to(dev),
               torch.as_tensor(x.labels).to(dev)) for x in bd]
    ngr = [x.meta["n_graphs"] for x in bd]
    log(f"[rank {rank}] graphs created in {time.time() - t0:.1f}s")
    P = make_params(D, D, D, nl, seed=7)
    flat0 = torch.as_tensor(dr.flatten_params(P, nl)).to(dev)
    flat = flat0.clone()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    comm = ddp.setup_nccl(dr, rank, world)
    tr = dr.Trainer(flat, nl, D, D, D, k, k, nccl_comm=comm)

    # ---- step 0 (P3 DP check): the allreduced mean gradient at the initial params
    g_dp = torch.empty_like(flat)
    loss0 = tr.step(graphs[0], *inputs[0], grad_out=g_dp)
    dp = {}
    if world > 1:
        flat_l = flat0.clone()
        tl = dr.Trainer(flat_l, nl, D, D, D, k, k)       # this rank's gradient alone
        g_l = torch.empty_like(flat)
        tl.step(graphs[0], *inputs[0], grad_out=g_l)
        tl.close()
        g_sum = g_l.double()
        dist.all_reduce(g_sum)
        ref = g_sum / world
        dp["grad_vs_mean_of_rank_grads_max_rel"] = float(
            (g_dp.double() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
    # ---- prime: every batch once eagerly, once captured into its CUDA graph, then
    # two passes enqueued back to back (the driver deepens its launch queue once,
    # blocking the host for ms: measured at step ~40 of the first deep run,
    # tools/step_timing.py); then the W warm-up steps. The clock sampler starts
    # first (nvidia-smi needs ~0.3 s) and every rank runs the same number of steps
    # (each step holds an allreduce at N > 1)
    clocks = Clocks(local)
    clocks.start()
    for s in range(S):
        for _ in range(2):
            tr.step(graphs[s], *inputs[s], sync=False)
    torch.cuda.synchronize()
    for i in range(2 * S):
        tr.step(graphs[i % S], *inputs[i % S], sync=False)
    torch.cuda.synchronize()

    def step(i):
        tr.step(graphs[i % S], *inputs[i % S], sync=False)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dr.launch_count_reset()
    wall0 = time.time()
    ms = timed_steps(torch, step, args.steps, flush, barrier=(dist.barrier if world > 1 else None))
    step_ms = step_stats(timed_steps.last)
    wall = time.time() - wall0
    launches = dr.launch_count()
    ms_max = ddp.max_over_ranks(ms, dev)
    n_graphs = sum(ngr[i % S] for i in range(args.steps))
    tg = torch.tensor([float(n_graphs)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tg)
    total_graphs = float(tg.item())
    time.sleep(0.2)
    clk = clocks.stop()

    # ---- P3: parameters bitwise equal across ranks after every step so far
    if world > 1:
        allp = [torch.empty_like(flat) for _ in range(world)]
        dist.all_gather(allp, flat)
        dp["params_bitwise_equal_across_ranks"] = bool(all(torch.equal(allp[0], x) for x in allp))
        dp["steps_before_param_check"] = int(2 * S + args.warmup + args.steps + 1)
        dp["params_sha1"] = hashlib.sha1(flat.cpu().numpy().tobytes()).hexdigest()[:16]

    # ---- per-kernel device times (roofline): batch 0, eager, single stream
    os.environ["DR_FORCE_SEQUENTIAL"] = "1"
    dr.profile_begin()
    n_prof = 5
    for i in range(n_prof):
        flush.zero_()
        tr.step(graphs[0], *inputs[0], sync=False)
    torch.cuda.synchronize()
    prof = dr.profile_end()
    os.environ.pop("DR_FORCE_SEQUENTIAL", None)

    # ---- end to end through the public API from pinned host buffers: per step the
    # batch's features + labels H2D and the loss D2H (+ sync). The copy of step i+1
    # runs on its own stream while step i computes (double-buffered per batch).
    all_cpus = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(local)
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    host = [tuple(torch.as_tensor(a).pin_memory() for a in (x.x_cell, x.x_net, x.labels))
            for x in bd]
    bufs = {}
    cs = torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    copied, used = {}, {}

    def slot(i):
        key = (i % S, (i // S) % 2)
        if key not in bufs:
            bufs[key] = tuple(torch.empty_like(t) for t in inputs[i % S])
            copied[key] = torch.cuda.Event()
            used[key] = torch.cuda.Event()
            used[key].record(comp)
        return key

    def issue_copy(i):
        key = slot(i)
        cs.wait_event(used[key])                 # the step that last read this slot is done
        with torch.cuda.stream(cs):
            for dst, h in zip(bufs[key], host[i % S]):
                dst.copy_(h, non_blocking=True)
            copied[key].record(cs)

    def run_e2e(i0, n):
        issue_copy(i0)
        for i in range(i0, i0 + n):
            if i + 1 < i0 + n:
                issue_copy(i + 1)
            key = slot(i)
            comp.wait_event(copied[key])
            tr.step(graphs[i % S], *bufs[key], sync=True)
            used[key].record(comp)

    run_e2e(0, 2 * S)                            # every slot: eager run, then capture
    run_e2e(0, 2 * S)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(comp)
    cs.wait_event(e0)
    run_e2e(0, args.steps)
    e1.record(comp)
    e1.synchronize()
    e_ms = ddp.max_over_ranks(e0.elapsed_time(e1), dev)
    h2d = sum(sum(h.numel() * 4 for h in host[i % S]) for i in range(args.steps)) / args.steps
    e2e = {"value": round(total_graphs / (e_ms * 1e-3), 3), "unit": "graphs/s",
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4,
           "ms_per_step": round(e_ms / args.steps, 4),
           "host_cpus": len(local_cpus) if local_cpus else None,
           "note": "graph structure resident (created once per batch); per step H2D of the "
                   "batch's x_cell, x_net, labels from pinned host (copy of step i+1 overlapped "
                   "with step i), D2H of the loss + host sync every step; max over ranks"}
    os.sched_setaffinity(0, all_cpus)

    # ---- P2/P3 parity at full size: the step-0 allreduced gradient vs the mean of
    # the fp64 oracle gradients of every rank's batch (O8), at the initial params,
    # the oracle fed the GPU's fp32 decisions (D-ReLU selections, merge masks;
    # reading Q28), each checked to be a valid decision of the oracle's own values
    t0 = time.time()
    forced = gpu_decisions(dr, torch, graphs[0], bd[0], P, nl, D, k, dev)
    oloss, og, valid = oracle_grads_flat(dr, bd[0], P, nl, k, forced=forced)
    og_t = torch.as_tensor(og, device=dev)
    ol_t = torch.tensor([oloss], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(og_t)
        dist.all_reduce(ol_t)
    og_t /= world
    gd = g_dp.double()
    worst, worst_key = 0.0, None
    for key, (a, b) in split_flat(dr, gd.cpu().numpy(), og_t.cpu().numpy(), nl, D).items():
        e = row_err(a, b)
        if e > worst:
            worst, worst_key = e, key
    dp["oracle_grad_row_err_max"] = worst
    dp["oracle_grad_row_err_worst_tensor"] = worst_key
    dp["oracle_grad_tolerance"] = 1e-4
    dp["oracle_note"] = ("fp32 GPU step-0 gradient vs the fp64 oracle fed the GPU's fp32 "
                         "decisions (reading Q28), full batch, max over parameter tensors of the "
                         "row-normalised error (SURVEY §8(c)); decisions valid iff both gap "
                         "minima >= -1e-5")
    dp["decisions"] = valid
    dp["decisions_valid"] = bool(valid["drelu_gap_min"] >= -1e-5 and valid["merge_gap_min"] >= -1e-5)
    dp["oracle_grad_ok"] = bool(worst <= 1e-4)
    dp["oracle_s"] = round(time.time() - t0, 2)

    table = kernel_table(prof, bd[0], D, k, "C5", tiled=graphs[0].info()["tiles"][0] > 0,
                         chained=True)
    rf = roofline(table, hbm, bf16, src)
    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            stp, O = oracle_train_timer(bd[0], P, nl, k)
            ts, ta = [], time.time()
            while len(ts) < 5 and time.time() - ta < 15.0:
                t = time.time()
                stp()
                ts.append(time.time() - t)
            per = float(np.mean(ts))
            cpu = {"value": round(ngr[0] / per, 4), "unit": "graphs/s", "cores": O.num_threads(),
                   "kind": "oracle",
                   "sample": f"{len(ts)} full fp64 oracle training steps (fwd, bwd, Adam) on "
                             f"rank batch 0 ({ngr[0]} graphs, {bd[0].n_cell} cells), "
                             f"{per:.2f} s/step, OpenMP over rows, {O.num_threads()} threads"}
        loads = [sum(int(sum(g.nnz().values())) for i in mine[s] for g in designs[i])
                 for s in range(S)]
        out = {
            "metric": METRIC,
            "value": round(total_graphs / (ms_max * 1e-3), 3),
            "unit": "graphs/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_max / args.steps, 4),
            "step_ms_rank0": step_ms,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": DTYPE,
            "data": DATA,
            "config": {
                "workload": "C5: Mini-CircuitNet-shaped DP training set (BASELINE configs[4]), "
                            f"{C5_DESIGNS} designs of 2-4 graphs (7.3-9.8k cells each), hidden "
                            f"64, D-ReLU k=8, 2 HeteroConv layers, full train step incl. NCCL "
                            f"allreduce (world > 1) and Adam; per rank per step a packed batch "
                            f"of {B} designs (disjoint union)",
                "global_batch_designs": world * B, "batch_designs_per_rank": B,
                "batches_per_rank": S, "graphs_timed_all_ranks": int(total_graphs),
                "rank0_batch_cells": [x.n_cell for x in bd][:8],
                "rank0_batch_nnz": loads[:8],
                "parallelism": f"dp{world}",
                "id_order": "shuffled",
                "l2": "flushed (256 MB write) before every timed step, outside the events",
                "priming": f"every batch run once eagerly and once captured (CUDA graph), "
                           f"then two passes enqueued back to back, before the {args.warmup} "
                           f"warm-up steps (the clock sampler started before the priming)",
                "enqueue": "timed steps enqueued in chunks of 16 behind a 0.05 s spin kernel "
                           "(outside the events) so host stalls cannot idle the device inside "
                           "a step's events; garbage collector off; per-step device times in "
                           "step_ms_rank0",
                "kernel_times": "per-launch CUDA events in an eager, single-stream pass of 5 "
                                "steps on batch 0 after the timed region (the timed region "
                                "replays each batch's CUDA graph on 3 streams)",
            },
            "roofline": rf,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "wall_s_timed_loop": round(wall, 3),
            "dp_checks": dp,
            "step0_loss": {"gpu": loss0, "oracle_fp64": oloss, "batch": "rank 0 batch 0"},
            "kernels": table,
            "spmm_gate": spmm_gate(table, hbm),
        }
    tr.close()
    if comm:
        dr.nccl_comm_destroy(comm)
    return out


# ------------------------------------------------------------------ our arm: one big design
def run_single(args, torch, dr, wl, dev, hbm, bf16, src, l2=None, steps=None, warmup=None,
               local=0, want_cpu=True, want_identity=False):
    """C2 (2-layer train step) or C4 (one HeteroConv layer fwd+bwd) on one design."""
    from gen import make_config, make_params
    steps = steps or args.steps
    warmup = max(3, warmup or args.warmup)
    cfg = {"C2": dict(D=64, k=8, layers=2), "C4": dict(D=128, k=16, layers=1)}[wl]
    D, k, nl = cfg["D"], cfg["k"], cfg["layers"]
    t0 = time.time()
    d = make_config(wl)
    log(f"generated {wl}: {d.n_cell} cells, {d.n_net} nets, nnz {d.nnz()} in "
        f"{time.time() - t0:.1f}s")
    t0 = time.time()
    g = dr.Graph.from_design(d)
    torch.cuda.synchronize()
    init_s = time.time() - t0
    P = make_params(D, D, D, nl, seed=7)
    xc = torch.as_tensor(d.x_cell).to(dev)
    xn = torch.as_tensor(d.x_net).to(dev)
    lab = torch.as_tensor(d.labels).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    if wl == "C2":
        flat = torch.as_tensor(dr.flatten_params(P, nl)).to(dev)
        tr = dr.Trainer(flat, nl, D, D, D, k, k)

        def mk(gg):
            return lambda i: tr.step(gg, xc, xn, lab, sync=False)
    else:
        W = {kk.split(".", 1)[1]: torch.as_tensor(v).to(dev) for kk, v in P.items()
             if kk.startswith("l0.")}
        L = dr.Layer(W, D, D, D, k, k)
        tape = torch.empty(L.tape_bytes(g), dtype=torch.uint8, device=dev)
        dyc = torch.randn(d.n_cell, D, device=dev)
        dyn = torch.randn(d.n_net, D, device=dev)

        def mk(gg):
            def f(i):
                dr.heteroconv_fwd(gg, L, xc, xn, tape=tape)
                dr.heteroconv_bwd(gg, L, tape, dyc, dyn, need_dx=True)
            return f
    step = mk(g)
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    t_w = time.time()
    while time.time() - t_w < 0.3:          # keep the GPU busy while the sampler starts
        step(0)
        torch.cuda.synchronize()
    dr.launch_count_reset()
    ms = timed_steps(torch, step, steps, flush)
    launches = dr.launch_count()
    time.sleep(0.2)
    clk = clocks.stop()

    def kernel_pass(gg, stp, n):
        os.environ["DR_FORCE_SEQUENTIAL"] = "1"
        dr.profile_begin()
        for i in range(n):
            flush.zero_()
            stp(i)
        torch.cuda.synchronize()
        pr = dr.profile_end()
        os.environ.pop("DR_FORCE_SEQUENTIAL", None)
        return pr
    prof = kernel_pass(g, step, steps)
    table = kernel_table(prof, d, D, k, wl, tiled=g.info()["tiles"][0] > 0,
                         chained=wl == "C2")
    out = {"ms_per_iter": round(ms / steps, 4), "steps": steps, "warmup": warmup,
           "graph_init_s": round(init_s, 2), "gpu_launches": int(launches), "clocks": clk,
           "roofline": roofline(table, hbm, bf16, src), "spmm_gate": spmm_gate(table, hbm, l2),
           "kernels": table, "design": d, "n_cell": d.n_cell, "n_net": d.n_net,
           "nnz": d.nnz(), "D": D, "k": k, "layers": nl}
    if want_identity:
        # the same layer with DR_GRAPH_ORDER_IDENTITY: rows in id order, no degree
        # classes, no tiles -- the per-edge SIMT kernels on a shuffled graph, i.e.
        # the pure-DRAM case of SURVEY §8(d)
        gi = dr.Graph.from_design(d, flags=dr.DR_GRAPH_ORDER_IDENTITY)
        sti = mk(gi)
        for i in range(3):
            sti(i)
        ms_i = timed_steps(torch, sti, max(3, steps // 2), flush)
        pri = kernel_pass(gi, sti, max(3, steps // 2))
        ti = kernel_table(pri, d, D, k, wl + "-identity", tiled=False)
        out["identity_order"] = {"ms_per_iter": round(ms_i / max(3, steps // 2), 4),
                                 "spmm_gate": spmm_gate(ti, hbm, l2),
                                 "kernels": {t: v for t, v in ti.items() if t.startswith("spmm")}}
        gi.close()
    if want_cpu and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_single(d, P, D, k, nl, wl)
    if wl == "C4":
        out["e2e"] = e2e_layer(torch, dr, g, L, d, dev, tape, n=3)
    else:
        out["trainer"] = tr
    out["graph"] = g
    return out


def e2e_layer(torch, dr, g, L, d, dev, tape, n=3):
    """C4 end to end through the public API: per iteration H2D of x_cell, x_net,
    dY_cell, dY_net from pinned host, layer fwd + bwd, D2H of the weight
    gradients (the iteration's result), host sync."""
    rng = np.random.default_rng(1)
    hx = torch.as_tensor(d.x_cell).pin_memory()
    hn = torch.as_tensor(d.x_net).pin_memory()
    hdc = torch.as_tensor(rng.standard_normal((d.n_cell, L.c.d_out), dtype=np.float32)).pin_memory()
    hdn = torch.as_tensor(rng.standard_normal((d.n_net, L.c.d_out), dtype=np.float32)).pin_memory()
    bx, bn, bdc, bdn = (torch.empty_like(t, device=dev) for t in (hx, hn, hdc, hdn))
    gw = {}

    def it():
        for dst, src in ((bx, hx), (bn, hn), (bdc, hdc), (bdn, hdn)):
            dst.copy_(src, non_blocking=True)
        dr.heteroconv_fwd(g, L, bx, bn, tape=tape)
        grads, _, _ = dr.heteroconv_bwd(g, L, tape, bdc, bdn, need_dx=True)
        for kk, v in grads.items():
            gw[kk] = v.cpu()
    it()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        it()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    h2d = sum(t.numel() * 4 for t in (hx, hn, hdc, hdn))
    return {"value": round(ms, 3), "unit": "ms/iter", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(sum(v.numel() * 4 for v in gw.values())),
            "note": "per iteration H2D of x_cell, x_net, dY_cell, dY_net (pinned host), layer "
                    "fwd+bwd, D2H of the weight gradients; PCIe-bound at this size"}


def cpu_baseline_single(d, P, D, k, nl, wl, budget_s=20.0):
    from oracle import oracle as O
    if wl == "C2":
        step, _ = oracle_train_timer(d, P, nl, k)
        what = "full oracle training steps (fwd, bwd, Adam)"
    else:
        # oracle scope spmm: D-ReLU + 3 SpMM fwd + the SSpMMs of the layer
        G = O.OGraph(d)
        rng = np.random.default_rng(0)
        dzc = rng.standard_normal((d.n_cell, D))
        dzn = rng.standard_normal((d.n_net, D))

        def step():
            ic, vc = O.drelu(d.x_cell, k)
            i_n, vn = O.drelu(d.x_net, k)
            G.fwd("near", ic, vc, D)
            G.fwd("pins", ic, vc, D)
            G.fwd("pinned", i_n, vn, D)
            G.bwd("near", ic, dzc)
            G.bwd("pins", ic, dzn)
            G.bwd("pinned", i_n, dzc)
        what = "oracle D-ReLU x2 + SpMM fwd x3 + SSpMM x3 (scope spmm)"
    times, t_all = [], time.time()
    while True:
        t = time.time()
        step()
        times.append(time.time() - t)
        if time.time() - t_all > budget_s * 0.5 or len(times) >= 5:
            break
    per = float(np.mean(times))
    val, unit = (1.0 / per, "graphs/s") if wl == "C2" else (per * 1e3, "ms/iter")
    return {"value": round(val, 5), "unit": unit, "cores": O.num_threads(), "kind": "oracle",
            "sample": f"{len(times)} x {what} on the same {wl} design (fp64, OpenMP over rows, "
                      f"{O.num_threads()} threads), mean {per:.2f} s"}


def c4_record(args, torch, dr, dev, hbm, bf16, src, l2, local):
    r = run_single(args, torch, dr, "C4", dev, hbm, bf16, src, l2=l2, steps=10, warmup=3,
                   local=local, want_identity=True)
    r.pop("design")
    r["graph"].close()
    r.pop("graph")
    r["workload"] = ("C4: CircuitNet-large-shaped graph (BASELINE configs[3]), 1M cells / 0.7M "
                     "nets, D=128, k=16, one HeteroConv layer fwd+bwd (north_star gate: SpMM "
                     "fwd+bwd >= 60 % of HBM)")
    return r


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2508_16769_b200 as dr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    hbm, bf16, src = peaks()
    l2 = l2_read_gbs(torch, dev)
    out = None
    if args.workload == "C5":
        out = run_c5(args, torch, dist, dr, rank, world, local, dev, hbm, bf16, src)
        if rank == 0:
            out["l2_read_gbs"] = round(l2, 1)
        if world == 1 and not args.no_c4:
            rec = c4_record(args, torch, dr, dev, hbm, bf16, src, l2, local)
            out["c4"] = rec
    else:
        assert world == 1, "--workload C2/C4 is single-GPU"
        r = run_single(args, torch, dr, args.workload, dev, hbm, bf16, src, l2=l2, local=local,
                       want_identity=args.workload == "C4")
        d = r.pop("design")
        r.pop("graph").close()
        r.pop("trainer", None)
        wl = args.workload
        ms = r["ms_per_iter"]
        out = {"metric": METRIC if wl == "C2" else "HeteroConv fwd+bwd ms/iter",
               "value": round(1e3 / ms, 3) if wl == "C2" else ms,
               "unit": "graphs/s" if wl == "C2" else "ms/iter",
               "n_gpus": 1, "steps": r["steps"], "warmup": r["warmup"], "ms_per_step": ms,
               "higher_is_better": wl == "C2", "scaling": "weak", "vs_baseline": None,
               "dtype": DTYPE, "data": DATA,
               "config": {"workload": wl, "n_cell": d.n_cell, "n_net": d.n_net, "nnz": d.nnz(),
                          "D": r["D"], "k": r["k"], "layers": r["layers"],
                          "parallelism": "single", "id_order": "shuffled",
                          "l2": "flushed (256 MB write) before every timed step"},
               "roofline": r["roofline"], "cpu_baseline": r.get("cpu_baseline"),
               "e2e": r.get("e2e"), "gpu_launches": r["gpu_launches"], "clocks": r["clocks"],
               "l2_read_gbs": round(l2, 1), "spmm_gate": r["spmm_gate"],
               "identity_order": r.get("identity_order"), "kernels": r["kernels"]}
    if rank == 0 and out is not None:
        print(json.dumps(out, default=str), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


# ------------------------------------------------------------------ reference arm (fp64 oracle)
def run_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return None
    from gen import make_config, make_params
    from gen.circuit import make_c5_set
    world = int(os.environ.get("WORLD_SIZE", "1"))
    wl = args.workload
    if wl == "C5":
        # each step: one fp64 oracle training step on ONE design of rank 0's batches
        # (a bounded sample of the same workload; value = graphs / s)
        batches, _ = c5_schedule(world, args.batch_designs)
        ids = [i for s in range(len(batches)) for i in batches[s][0]]
        n_use = min(len(ids), args.warmup + args.steps)
        designs = make_c5_set(C5_DESIGNS, only=ids[:n_use])
        P = make_params(64, 64, 64, 2, seed=7)
        from gen.circuit import disjoint_union
        steps_fns, ng = [], []
        for i in ids[:n_use]:
            u = disjoint_union(designs[i])
            fn, O = oracle_train_timer(u, P, 2, 8)
            steps_fns.append(fn)
            ng.append(len(designs[i]))
        j = 0
        for _ in range(args.warmup):
            steps_fns[j % n_use]()
            j += 1
        t_all, graphs = 0.0, 0
        for _ in range(args.steps):
            t = time.time()
            steps_fns[j % n_use]()
            t_all += time.time() - t
            graphs += ng[j % n_use]
            j += 1
        value, unit, hib = graphs / t_all, "graphs/s", True
        cfg = {"workload": "C5 (same schedule as our arm); fp64 CPU oracle, one design per step",
               "batch_designs_per_rank": args.batch_designs}
        sample = (f"each step = one full fp64 oracle training step (fwd, bwd, Adam) on one "
                  f"design (2-4 graphs) of rank 0's batches; {args.steps} steps, "
                  f"{graphs} graphs")
    else:
        cfgs = {"C2": dict(D=64, k=8, layers=2), "C4": dict(D=128, k=16, layers=1)}[wl]
        D, k, nl = cfgs["D"], cfgs["k"], cfgs["layers"]
        d = make_config(wl)
        P = make_params(D, D, D, nl, seed=7)
        from oracle import oracle as O
        if wl == "C2":
            fn, O = oracle_train_timer(d, P, nl, k)
        else:
            G = O.OGraph(d)
            W = O.layer_params(P, 0)
            rng = np.random.default_rng(0)
            dyc = rng.standard_normal((d.n_cell, D))
            dyn = rng.standard_normal((d.n_net, D))

            def fn():
                _, _, tape = O.layer_fwd(G, W, d.x_cell, d.x_net, k, k)
                O.layer_bwd(G, W, tape, dyc, dyn, need_dx=True)
        for _ in range(args.warmup):
            fn()
        t_all = 0.0
        for _ in range(args.steps):
            t = time.time()
            fn()
            t_all += time.time() - t
        if wl == "C2":
            value, unit, hib = args.steps / t_all, "graphs/s", True
        else:
            value, unit, hib = t_all * 1e3 / args.steps, "ms/iter", False
        cfg = {"workload": f"{wl} (same design and parameters as our arm); fp64 CPU oracle"}
        sample = f"each step = one full oracle step on the {wl} design"
    from oracle import oracle as O
    out = {
        "impl": "reference",
        "metric": METRIC if wl != "C4" else "HeteroConv fwd+bwd ms/iter",
        "value": round(value, 5), "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_all * 1e3 / args.steps, 3),
        "higher_is_better": hib, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": cfg,
        "cpu_baseline": {"value": round(value, 5), "unit": unit, "cores": O.num_threads(),
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": round(value, 5), "unit": unit, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return out


# ------------------------------------------------------------------ launcher
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this script under
    torch.distributed.run with N ranks on this node (one GPU per rank)."""
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but only {n} CUDA devices visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    log("self-launch:", " ".join(cmd))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C5", choices=["C5", "C2", "C4"])
    ap.add_argument("--batch-designs", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        log(f"note: WORLD_SIZE={ws} but --gpus {args.gpus}; using WORLD_SIZE")
    run_ours(args)


if __name__ == "__main__":
    main()
