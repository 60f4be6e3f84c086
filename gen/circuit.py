"""CircuitNet-shaped synthetic heterographs (cells, nets; near / pins / pinned).

Shape provenance (PAPER.md, cited as P:<line>):
  * two node types cell/net, three relations near (cell-cell, geometric,
    undirected), pins (cell->net) and pinned (net->cell), pins/pinned mutually
    transposed (§2.2);
  * near degrees peak around 50 with a tail slightly over 250 (Fig. 4);
    pins/pinned concentrate at 3-4;
  * Table 1: near mean degree 38-52, pins per net 2.2-3.8,
    N_net/N_cell 0.45-0.95.

Relations are returned as destination-major CSR (rows = destinations, Eq. 4
convention P:238):
  near   : n_cell x n_cell  (row i = cell, cols = neighbouring cells)
  pins   : n_net  x n_cell  (row = net,  cols = its member cells)
  pinned : n_cell x n_net   (row = cell, cols = nets containing it) = pins^T

Everything is drawn from numpy PCG64 streams seeded per config; nothing here
computes degrees-as-normalisers, top-k, products or gradients.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from scipy.spatial import cKDTree


@dataclass
class Design:
    name: str
    n_cell: int
    n_net: int
    near_ptr: np.ndarray      # int64 [n_cell+1]
    near_col: np.ndarray      # int32 [nnz]
    pins_ptr: np.ndarray      # int64 [n_net+1]
    pins_col: np.ndarray      # int32 (cell ids)
    pinned_ptr: np.ndarray    # int64 [n_cell+1]
    pinned_col: np.ndarray    # int32 (net ids)
    x_cell: np.ndarray        # float32 [n_cell, d_cell]
    x_net: np.ndarray         # float32 [n_net, d_net]
    labels: np.ndarray        # float32 [n_cell]
    meta: dict = field(default_factory=dict)

    def rel(self, name):
        """(row_ptr, col_idx, n_dst, n_src) of relation 'near'|'pins'|'pinned'."""
        if name == "near":
            return self.near_ptr, self.near_col, self.n_cell, self.n_cell
        if name == "pins":
            return self.pins_ptr, self.pins_col, self.n_net, self.n_cell
        if name == "pinned":
            return self.pinned_ptr, self.pinned_col, self.n_cell, self.n_net
        raise KeyError(name)

    def nnz(self):
        return {r: int(self.rel(r)[1].shape[0]) for r in ("near", "pins", "pinned")}


# --------------------------------------------------------------------------- CSR plumbing
def _csr_from_pairs(n_rows, rows, cols):
    """Sorted, duplicate-free CSR from (row, col) pairs (pure data layout)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if rows.size:
        key = rows * (int(cols.max()) + 1 if cols.size else 1) + cols
        order = np.argsort(key, kind="stable")
        key = key[order]
        keep = np.ones(key.size, dtype=bool)
        keep[1:] = key[1:] != key[:-1]
        order = order[keep]
        rows, cols = rows[order], cols[order]
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n_rows), out=ptr[1:])
    return ptr, cols.astype(np.int32)


def _csr_transpose(n_rows, n_cols, ptr, col):
    rows = np.repeat(np.arange(n_rows, dtype=np.int64), np.diff(ptr))
    return _csr_from_pairs(n_cols, col.astype(np.int64), rows)


# --------------------------------------------------------------------------- degree laws
def powerlaw_degrees(rng, n, mean, d_max, d_min=1):
    """Discrete power law P(d) ~ d^-alpha on [d_min, d_max], alpha bisected so
    that E[d] == mean (SURVEY §8(d) 'Nets')."""
    d = np.arange(d_min, d_max + 1, dtype=np.float64)

    def m(alpha):
        p = d ** -alpha
        return float((p * d).sum() / p.sum())

    lo, hi = 0.5, 6.0
    for _ in range(80):
        mid = 0.5 * (lo + hi)
        if m(mid) > mean:
            lo = mid
        else:
            hi = mid
    alpha = 0.5 * (lo + hi)
    p = d ** -alpha
    p /= p.sum()
    return rng.choice(d.astype(np.int64), size=n, p=p), alpha


# --------------------------------------------------------------------------- geometry
def _positions(rng, n, cluster_share=0.15, cluster_sigma=4.0, cells_per_cluster=2000):
    side = max(np.sqrt(n), 1.0)
    n_cl = int(round(n * cluster_share))
    n_u = n - n_cl
    pos = np.empty((n, 2), dtype=np.float64)
    pos[:n_u] = rng.uniform(0.0, side, size=(n_u, 2))
    if n_cl:
        n_centres = max(1, int(round(n_cl / cells_per_cluster)))
        centres = rng.uniform(0.0, side, size=(n_centres, 2))
        which = rng.integers(0, n_centres, size=n_cl)
        pos[n_u:] = centres[which] + rng.normal(0.0, cluster_sigma, size=(n_cl, 2))
        np.clip(pos[n_u:], 0.0, side, out=pos[n_u:])
    return pos, side


def _near_graph(rng, pos, mean_deg, cap):
    n = pos.shape[0]
    tree = cKDTree(pos)
    m = min(n, 6000)
    sample = pos[rng.choice(n, size=m, replace=False)]
    # distances of each sample point to its cap+1 nearest (itself first): the
    # number within r, capped at cap, is #(dist <= r) - 1 -- one kNN query
    # instead of a ball query per bisection step
    kq = int(min(n, cap + 1))
    dist = np.asarray(tree.query(sample, k=kq, workers=-1)[0]).reshape(m, kq)

    def est(r):
        return float(np.mean(np.count_nonzero(dist <= r, axis=1) - 1))

    lo, hi = 0.0, 2.0 * np.sqrt(max(mean_deg, 1.0) / np.pi) + 2.0
    while est(hi) < mean_deg and hi < 4 * np.sqrt(n):
        hi *= 2
    for _ in range(28):
        mid = 0.5 * (lo + hi)
        if est(mid) < mean_deg:
            lo = mid
        else:
            hi = mid
    r = 0.5 * (lo + hi)
    pairs = tree.query_pairs(r, output_type="ndarray").astype(np.int64)
    p, q = pairs[:, 0], pairs[:, 1]
    mp = p.size
    deg = np.bincount(p, minlength=n) + np.bincount(q, minlength=n)
    if deg.max(initial=0) > cap:
        # keep each over-full row's `cap` nearest, then keep only mutual survivors
        i = np.concatenate([p, q])
        j = np.concatenate([q, p])
        kept = np.ones(2 * mp, dtype=bool)
        sel = np.nonzero(deg[i] > cap)[0]
        isel = i[sel]
        dist = np.linalg.norm(pos[isel] - pos[j[sel]], axis=1)
        order = np.lexsort((j[sel], dist, isel))
        s_sorted = sel[order]
        i_sorted = isel[order]
        first = np.ones(i_sorted.size, dtype=bool)
        first[1:] = i_sorted[1:] != i_sorted[:-1]
        start_idx = np.maximum.accumulate(np.where(first, np.arange(i_sorted.size), 0))
        rank = np.arange(i_sorted.size) - start_idx
        kept[s_sorted] = rank < cap
        keep = kept[:mp] & kept[mp:]
        p, q = p[keep], q[keep]
    ptr, col = _csr_from_pairs(n, np.concatenate([p, q]), np.concatenate([q, p]))
    return ptr, col, r


def _nets(rng, pos, n_net, pins_mean, d_max):
    n_cell = pos.shape[0]
    d_max = int(min(d_max, n_cell))
    deg, alpha = powerlaw_degrees(rng, n_net, pins_mean, d_max)
    tree = cKDTree(pos)
    centres = pos[rng.integers(0, n_cell, size=n_net)] + rng.normal(0, 0.5, size=(n_net, 2))
    rows, cols = [], []
    # query in power-of-two degree bands so each band is one vectorised kNN call
    hi = 1
    while True:
        lo = hi // 2 + 1 if hi > 1 else 1
        sel = np.nonzero((deg >= lo) & (deg <= hi))[0]
        if sel.size:
            kq = int(min(hi, n_cell))
            for s in range(0, sel.size, max(1, 4_000_000 // kq)):
                chunk = sel[s:s + max(1, 4_000_000 // kq)]
                _, nb = tree.query(centres[chunk], k=kq)
                nb = np.asarray(nb).reshape(chunk.size, kq)
                take = np.arange(kq)[None, :] < deg[chunk][:, None]
                rows.append(np.broadcast_to(chunk[:, None], nb.shape)[take])
                cols.append(nb[take])
        if hi >= d_max:
            break
        hi = min(hi * 2, d_max)
    rows = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    cols = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    ptr, col = _csr_from_pairs(n_net, rows, cols)
    return ptr, col, alpha


def disjoint_union(designs, name="union"):
    """Block-diagonal union of designs (a per-rank batch of graphs, reading Q24):
    ids of design q are offset by the node counts of designs < q. Data layout only."""
    def cat(ptrs, cols, offs):
        ptr = [np.zeros(1, np.int64)]
        base = 0
        for p in ptrs:
            ptr.append(p[1:] + base)
            base += int(p[-1])
        col = np.concatenate([c.astype(np.int64) + o for c, o in zip(cols, offs)]) if cols else \
            np.zeros(0, np.int64)
        return np.concatenate(ptr), col.astype(np.int32)
    oc = np.cumsum([0] + [d.n_cell for d in designs])[:-1]
    on = np.cumsum([0] + [d.n_net for d in designs])[:-1]
    near = cat([d.near_ptr for d in designs], [d.near_col for d in designs], oc)
    pins = cat([d.pins_ptr for d in designs], [d.pins_col for d in designs], oc)
    pinned = cat([d.pinned_ptr for d in designs], [d.pinned_col for d in designs], on)
    return Design(name, int(sum(d.n_cell for d in designs)), int(sum(d.n_net for d in designs)),
                  near[0], near[1], pins[0], pins[1], pinned[0], pinned[1],
                  np.concatenate([d.x_cell for d in designs]),
                  np.concatenate([d.x_net for d in designs]),
                  np.concatenate([d.labels for d in designs]),
                  meta=dict(parts=[d.name for d in designs]))


def _permute_csr(ptr, col, row_perm, col_perm):
    """Relabel rows by row_perm[old]=new and cols by col_perm[old]=new."""
    n = ptr.size - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    return _csr_from_pairs(n, row_perm[rows], col_perm[col.astype(np.int64)])


# --------------------------------------------------------------------------- designs
def make_design(name, n_cell, seed, d_cell=64, d_net=64, near_mean=45.0, near_cap=256,
                net_ratio=0.667, pins_mean=2.8, pins_dmax=2000, cluster_share=0.15,
                order="shuffled", n_net=None):
    """One synthetic circuit design (SURVEY §8(d) recipe)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    pos, side = _positions(rng, n_cell, cluster_share=cluster_share)
    near_ptr, near_col, radius = _near_graph(rng, pos, near_mean, near_cap)
    if n_net is None:
        n_net = max(1, int(round(net_ratio * n_cell)))
    pins_ptr, pins_col, alpha = _nets(rng, pos, n_net, pins_mean, pins_dmax)
    if order == "shuffled":
        pc = rng.permutation(n_cell).astype(np.int64)
        pn = rng.permutation(n_net).astype(np.int64)
        near_ptr, near_col = _permute_csr(near_ptr, near_col, pc, pc)
        pins_ptr, pins_col = _permute_csr(pins_ptr, pins_col, pn, pc)
    elif order != "spatial":
        raise ValueError(order)
    pinned_ptr, pinned_col = _csr_transpose(n_net, n_cell, pins_ptr, pins_col)
    x_cell = rng.standard_normal((n_cell, d_cell), dtype=np.float32)
    x_net = rng.standard_normal((n_net, d_net), dtype=np.float32)
    near_deg = np.diff(near_ptr).astype(np.float64)
    t = np.log1p(near_deg)
    lab = (t - t.mean()) / (t.std() + 1e-12) + rng.normal(0.0, 0.05, size=n_cell)
    return Design(name, n_cell, n_net, near_ptr, near_col, pins_ptr, pins_col,
                  pinned_ptr, pinned_col, x_cell, x_net, lab.astype(np.float32),
                  meta=dict(seed=seed, radius=radius, alpha=alpha, order=order,
                            die_side=side))


def _craft_c1(d: Design, rng):
    """C1 edge cases: an isolated cell, a cell in no net, a 1-pin
    net, a 16-pin hub net, an empty net and an all-zero feature row."""
    n_cell, n_net = d.n_cell, d.n_net
    # isolated cell 0: drop its near edges both ways
    rows = np.repeat(np.arange(n_cell), np.diff(d.near_ptr))
    cols = d.near_col.astype(np.int64)
    keep = (rows != 0) & (cols != 0)
    d.near_ptr, d.near_col = _csr_from_pairs(n_cell, rows[keep], cols[keep])
    # nets: 0 = hub of 16 cells, 1 = single pin, 2 = empty, others keep, cell 1 in no net
    nrows = np.repeat(np.arange(n_net), np.diff(d.pins_ptr))
    ncols = d.pins_col.astype(np.int64)
    keep = (nrows > 2) & (ncols != 1)
    hub = rng.choice(np.arange(2, n_cell), size=16, replace=False)
    nrows = np.concatenate([nrows[keep], np.zeros(16, np.int64), [1]])
    ncols = np.concatenate([ncols[keep], hub, [5]])
    d.pins_ptr, d.pins_col = _csr_from_pairs(n_net, nrows, ncols)
    d.pinned_ptr, d.pinned_col = _csr_transpose(n_net, n_cell, d.pins_ptr, d.pins_col)
    d.x_cell[3, :] = 0.0
    return d


# Config table (SURVEY §8.0 'Configs'); C5 is a set, see make_c5_set.
CONFIGS = {
    "C1": dict(n_cell=64, n_net=32, D=16, k=4, seed=1, near_mean=6.0, near_cap=16,
               pins_mean=2.8, pins_dmax=16, layers=1),
    "C2": dict(n_cell=100_000, n_net=66_600, D=64, k=8, seed=2, near_mean=45.0,
               near_cap=256, pins_mean=2.77, pins_dmax=2000, layers=2),
    "C3": dict(n_cell=300_000, n_net=200_000, D=64, k=8, seed=3, near_mean=45.0,
               near_cap=256, pins_mean=2.77, pins_dmax=2000, layers=2),
    "C4": dict(n_cell=1_000_000, n_net=700_000, D=128, k=16, seed=4, near_mean=46.0,
               near_cap=256, pins_mean=3.0, pins_dmax=50_000, layers=1),
}


def make_config(name, order="shuffled", scale=1.0, seed=None, D=None):
    """Build config `name` (C1..C4). `scale` shrinks node counts for quick tests
    (degree laws unchanged)."""
    c = dict(CONFIGS[name])
    D = D or c["D"]
    n_cell = max(16, int(round(c["n_cell"] * scale)))
    n_net = max(8, int(round(c["n_net"] * scale)))
    d = make_design(name, n_cell, seed if seed is not None else c["seed"], d_cell=D,
                    d_net=D, near_mean=c["near_mean"], near_cap=c["near_cap"],
                    pins_mean=c["pins_mean"], pins_dmax=c["pins_dmax"], order=order,
                    n_net=n_net)
    if name == "C1":
        d = _craft_c1(d, np.random.Generator(np.random.PCG64(101)))
    d.meta.update(config=name, D=D, k=c["k"], layers=c["layers"])
    return d


def _c5_graph(args):
    i, g, seed0, D, n_cell, ratio, near_mean, pins_mean = args
    return make_design(f"C5.{i}.{g}", n_cell, seed0 * 100 + i * 10 + g, d_cell=D, d_net=D,
                       near_mean=near_mean, near_cap=256, net_ratio=ratio,
                       pins_mean=pins_mean, pins_dmax=500)


def c5_specs(n_designs=100, seed0=5000, D=64, graphs_lo=2, graphs_hi=4):
    """Per-design graph parameters of the C5 set (drawn from per-design seeded
    streams, no graph built): a list over designs of lists of job tuples
    (i, g, seed0, D, n_cell, net_ratio, near_mean, pins_mean)."""
    specs = []
    for i in range(n_designs):
        rng = np.random.Generator(np.random.PCG64(seed0 + i))
        n_graphs = int(rng.integers(graphs_lo, graphs_hi + 1))
        jobs = []
        for g in range(n_graphs):
            n_cell = int(rng.integers(7300, 9800))
            ratio = float(rng.uniform(0.45, 0.95))
            near_mean = float(rng.uniform(38, 52))
            pins_mean = float(rng.uniform(2.2, 3.8))
            jobs.append((i, g, seed0, D, n_cell, ratio, near_mean, pins_mean))
        specs.append(jobs)
    return specs


def c5_expected_nnz(jobs):
    """Expected edge count of one C5 design from its specs (near + pins + pinned),
    for packing designs onto ranks before they are generated."""
    return float(sum(n * nm + 2.0 * n * r * pm for (_, _, _, _, n, r, nm, pm) in jobs))


def make_c5_set(n_designs=100, seed0=5000, D=64, graphs_lo=2, graphs_hi=4, workers=None,
                only=None):
    """Mini-CircuitNet-shaped DP set: designs of 2-4 graphs,
    each graph 7.3k-9.8k cells with Table-1 ranges for the other statistics.
    Returns a list of designs, each a list of Design graphs (with `only`, an
    iterable of design ids, a dict id -> graphs of just those designs). The
    per-graph draws come from per-design seeded streams, so `workers`
    (processes; None = all cores, 1 = serial) and `only` do not change a
    design."""
    specs = c5_specs(n_designs, seed0, D, graphs_lo, graphs_hi)
    ids = list(range(n_designs)) if only is None else sorted(set(int(i) for i in only))
    jobs = [j for i in ids for j in specs[i]]
    import os
    nw = workers if workers is not None else min(len(jobs), os.cpu_count() or 1, 32)
    if nw > 1 and len(jobs) > 1:
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor
        with ProcessPoolExecutor(nw, mp_context=mp.get_context("fork")) as ex:
            graphs = list(ex.map(_c5_graph, jobs, chunksize=max(1, len(jobs) // (4 * nw))))
    else:
        graphs = [_c5_graph(j) for j in jobs]
    out, q = {}, 0
    for i in ids:
        out[i] = graphs[q:q + len(specs[i])]
        q += len(specs[i])
    return [out[i] for i in ids] if only is None else out


def make_params(d_cell, d_net, d_hidden, n_layers, seed=7):
    """Named parameter arrays (Glorot-uniform weights, U(-0.1,0.1) biases; SURVEY
    Q25). Shapes follow SURVEY §8.0: per layer Wn_near [d_c,D], Wr_near [d_c,D],
    b_near [D], W_pinned [d_n,D], b_pinned [D], Wn_pins [d_c,D], Wr_pins [d_n,D],
    b_pins [D]; head w_h [D], b_h [1]. Layer l>0 has d_c = d_n = D."""
    rng = np.random.Generator(np.random.PCG64(seed))

    def glorot(a, b):
        lim = np.sqrt(6.0 / (a + b))
        return rng.uniform(-lim, lim, size=(a, b)).astype(np.float32)

    def bias(n):
        return rng.uniform(-0.1, 0.1, size=n).astype(np.float32)

    p = {}
    dc, dn = d_cell, d_net
    for l in range(n_layers):
        p[f"l{l}.wn_near"] = glorot(dc, d_hidden)
        p[f"l{l}.wr_near"] = glorot(dc, d_hidden)
        p[f"l{l}.b_near"] = bias(d_hidden)
        p[f"l{l}.w_pinned"] = glorot(dn, d_hidden)
        p[f"l{l}.b_pinned"] = bias(d_hidden)
        p[f"l{l}.wn_pins"] = glorot(dc, d_hidden)
        p[f"l{l}.wr_pins"] = glorot(dn, d_hidden)
        p[f"l{l}.b_pins"] = bias(d_hidden)
        dc = dn = d_hidden
    p["head.w"] = glorot(d_hidden, 1).reshape(d_hidden)
    p["head.b"] = bias(1)
    return p
