"""fp64 CPU oracle for the DR-CircuitGNN hot path (arXiv 2508.16769).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package ``paper_2508_16769_b200``. It shares no code with the CUDA path; the
only common input is the seeded generator in ``gen/``.

Layout of the oracle
  * ``dr_oracle.c``  plain fp64 loops: degree normalisers, D-ReLU (Eq. 2-3),
    DR-SpMM forward (Eq. 5-7 / Alg. 1), SSpMM backward (Eq. 10-11 / Alg. 2);
  * this file: ctypes glue plus the HeteroConv layer, max-merge (Eq. 8, 14),
    its backward (Eq. 12-13), the linear head + MSE, Adam, the 2-layer train
    step and the data-parallel mean — composed from those loops and numpy
    matmuls (a library primitive used as one step, nothing blocked or fused).

Citations: P:<n> = /root/reference/PAPER.md line n; S:<n> = SPEC.md line n;
Q<n> = the reading numbered n in DESIGN.md "Readings of the paper".

Parity status per function: every function here
is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py; none is
"parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dr_oracle.c")
_BUILD = os.path.join(_HERE, "_build")
_SO = os.path.join(_BUILD, "libdr_oracle.so")
_lock = threading.Lock()
_lib = None

MEAN, SYM = 0, 1            # SageConv(mean) / GraphConv(norm='both')  (Q1, Q12)
RELS = ("near", "pins", "pinned")
DEFAULT_MODULES = {"near": MEAN, "pins": MEAN, "pinned": SYM}   # reading Q1


def build(force=False):
    """Compile dr_oracle.c with gcc (no fast-math: IEEE fp64 semantics)."""
    os.makedirs(_BUILD, exist_ok=True)
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i64, i32 = ctypes.c_int64, ctypes.c_int
            L.or_normalisers.argtypes = [i64, i64, P, P, i32, P, P]
            L.or_drelu.argtypes = [P, i64, i32, i64, i32, P, P]
            L.or_spmm_fwd.argtypes = [i64, P, P, P, P, P, i32, i32, P, P, P]
            L.or_spmm_bwd.argtypes = [i64, i64, P, P, P, P, P, i32, i32, P, P, P]
            L.or_num_threads.restype = i32
            L.or_set_num_threads.argtypes = [i32]
            for f in ("or_normalisers", "or_drelu", "or_spmm_fwd", "or_spmm_bwd"):
                getattr(L, f).restype = None
            _lib = L
    return _lib


def num_threads():
    return lib().or_num_threads()


def set_num_threads(n):
    lib().or_set_num_threads(int(n))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# ------------------------------------------------------------------ primitives
def normalisers(ptr, col, n_dst, n_src, module):
    """(c [n_dst], s [n_src]) for MEAN / SYM (Q12)."""
    ptr, col = _i64(ptr), _i32(col)
    c = np.empty(n_dst, np.float64)
    s = np.empty(max(n_src, 0), np.float64)
    lib().or_normalisers(n_dst, n_src, _p(ptr), _p(col), int(module), _p(c), _p(s))
    return c, s


def drelu(x, k):
    """Eq. 2-3 exact top-k, ties -> lowest column (Q5), values verbatim (Q6).
    Returns (idx int32 [n,k] ascending, val float64 [n,k])."""
    x = _f64(x)
    n, d = x.shape
    if not (1 <= k <= d):
        raise ValueError("BadK: need 1 <= k <= dim")
    idx = np.empty((n, k), np.int32)
    val = np.empty((n, k), np.float64)
    lib().or_drelu(_p(x), n, d, d, k, _p(idx), _p(val))
    return idx, val


def densify(idx, val, d):
    """CBSR -> dense rows (kept values at their indices, zeros elsewhere)."""
    n, k = idx.shape
    out = np.zeros((n, d), np.float64)
    for t in range(k):
        out[np.arange(n), idx[:, t]] = val[:, t]
    return out


def gather_at(m, idx):
    """m[j, idx[j,t]] -> [n, k]."""
    return np.take_along_axis(m, idx.astype(np.int64), axis=1)


def spmm_fwd(ptr, col, n_dst, c, s, idx, val, d, a=None):
    """Eq. 5 / Alg. 1: Z_i = c_i sum_j a_ij s_j densify(H_j)."""
    ptr, col = _i64(ptr), _i32(col)
    idx, val = _i32(idx), _f64(val)
    k = idx.shape[1]
    z = np.empty((n_dst, d), np.float64)
    lib().or_spmm_fwd(n_dst, _p(ptr), _p(col), _p(None if a is None else _f64(a)),
                      _p(_f64(c)), _p(_f64(s)), k, d, _p(idx), _p(val), _p(z))
    return z


def spmm_bwd(ptr, col, n_dst, n_src, c, s, idx, dz, a=None):
    """Eq. 10-11 / Alg. 2: g[j,t] = sum_i c_i a_ij s_j dz[i, idx[j,t]]."""
    ptr, col = _i64(ptr), _i32(col)
    idx, dz = _i32(idx), _f64(dz)
    k = idx.shape[1]
    d = dz.shape[1]
    g = np.empty((n_src, k), np.float64)
    lib().or_spmm_bwd(n_dst, n_src, _p(ptr), _p(col), _p(None if a is None else _f64(a)),
                      _p(_f64(c)), _p(_f64(s)), k, d, _p(idx), _p(dz), _p(g))
    return g


# ------------------------------------------------------------------ graph wrapper
class OGraph:
    """Relations of one design with the oracle's own normalisers.
    ``weights`` optionally maps relation -> per-edge a_ij (default all 1)."""

    def __init__(self, design, modules=None, weights=None):
        self.d = design
        self.n_cell, self.n_net = design.n_cell, design.n_net
        self.modules = dict(DEFAULT_MODULES if modules is None else modules)
        self.weights = dict(weights or {})
        self.cs = {}
        for r in RELS:
            ptr, col, nd, ns = design.rel(r)
            self.cs[r] = normalisers(ptr, col, nd, ns, self.modules[r])

    def fwd(self, r, idx, val, d):
        ptr, col, nd, ns = self.d.rel(r)
        c, s = self.cs[r]
        return spmm_fwd(ptr, col, nd, c, s, idx, val, d, self.weights.get(r))

    def bwd(self, r, idx, dz):
        ptr, col, nd, ns = self.d.rel(r)
        c, s = self.cs[r]
        return spmm_bwd(ptr, col, nd, ns, c, s, idx, dz, self.weights.get(r))


# ------------------------------------------------------------------ HeteroConv layer
def layer_params(P, l):
    return {k.split(".", 1)[1]: _f64(v) for k, v in P.items() if k.startswith(f"l{l}.")}


def drelu_forced(x, idx):
    """D-ReLU with the selection DECIDED ELSEWHERE (teacher forcing, DESIGN.md
    reading Q28): the kept columns are `idx` (n x k, ascending), the values are
    this oracle's own x at them, verbatim (Eq. 3). Used where the decision is
    taken in fp32 on the kernel's own output (a near-tie at fp32 resolution)
    and validated separately by drelu_gap."""
    x = _f64(x)
    idx = np.asarray(idx, np.int32)
    if idx.ndim != 2 or idx.shape[0] != x.shape[0]:
        raise ValueError("ShapeMismatch: idx rows != x rows")
    if idx.size and (idx.min() < 0 or idx.max() >= x.shape[1] or np.any(np.diff(idx, axis=1) <= 0)):
        raise ValueError("forced idx must be ascending distinct columns in range")
    return idx, gather_at(x, idx)


def drelu_gap(x, idx):
    """Per row: (smallest kept value - largest dropped value) / ||x_row||_2.
    >= 0 iff idx is a valid top-k of the row (Eq. 2); rows with nothing dropped
    give +inf, all-zero rows use norm 1. The parity protocol accepts a forced
    selection when every gap >= -1e-5 (SURVEY §8(c) P2 near-tie band)."""
    x = _f64(x)
    n, d = x.shape
    keep = np.zeros((n, d), bool)
    if n:
        keep[np.arange(n)[:, None], np.asarray(idx, np.int64)] = True
    kept_min = np.where(keep, x, np.inf).min(axis=1)
    drop_max = np.where(keep, -np.inf, x).max(axis=1)
    nrm = np.linalg.norm(x, axis=1)
    nrm = np.where(nrm > 0, nrm, 1.0)
    return (kept_min - drop_max) / nrm


def merge_gap(y_near, y_pinned, M):
    """Per row: the most negative (chosen - other) margin of the max-merge mask
    M (Eq. 8, 14) divided by the row norm of max(y_near, y_pinned); >= 0 iff M
    is the exact mask up to ties (tie -> near). Used like drelu_gap."""
    yn, yp = _f64(y_near), _f64(y_pinned)
    M = np.asarray(M, bool)
    marg = np.where(M, yn - yp, yp - yn)
    nrm = np.linalg.norm(np.maximum(yn, yp), axis=1)
    nrm = np.where(nrm > 0, nrm, 1.0)
    if marg.shape[1] == 0:
        return np.full(marg.shape[0], np.inf)
    return marg.min(axis=1) / nrm


def layer_fwd(G, W, x_c, x_n, k_c, k_n, merge="max", root=True, k_p=None, forced=None):
    """One HeteroConv layer (Eq. 2-9):
       H = drelu(X) per node type (Eq. 2-3)
       Z_psi = SpMM_psi(H_src)          (Eq. 5-7, three relations)
       [per-edge-type k (reading Q27, §8 f3): k_p != k_c gives pins its own cell
        CBSR H_p = drelu(X_c, k_p); Z_pins = SpMM_pins(H_p); near and the roots keep
        H_c / H_n]
       Y_near = Z_near Wn + H_c Wr + b  (SageConv mean, Q2 root weight)
       Y_pinned = Z_pinned W + b        (GraphConv both)
       Y_net = Z_pins Wn + H_n Wr + b   (SageConv mean)
       Y_cell = max(Y_near, Y_pinned), M = [Y_near >= Y_pinned]  (Eq. 8, 14; Q3, Q4)
    forced (teacher forcing, reading Q28): optional dict with "hc_idx" / "hn_idx"
    (the D-ReLU selections) and / or "M" (the merge mask) decided elsewhere; the
    arithmetic is unchanged, only those integer decisions are taken as given.
    """
    x_c, x_n = _f64(x_c), _f64(x_n)
    d_c, d_n = x_c.shape[1], x_n.shape[1]
    forced = forced or {}
    if "hc_idx" in forced:
        hc_idx, hc_val = drelu_forced(x_c, forced["hc_idx"])
    else:
        hc_idx, hc_val = drelu(x_c, k_c)
    if "hn_idx" in forced:
        hn_idx, hn_val = drelu_forced(x_n, forced["hn_idx"])
    else:
        hn_idx, hn_val = drelu(x_n, k_n)
    Hc = densify(hc_idx, hc_val, d_c)
    Hn = densify(hn_idx, hn_val, d_n)
    z_near = G.fwd("near", hc_idx, hc_val, d_c)
    if k_p is None or k_p == k_c:
        hp_idx, hp_val = hc_idx, hc_val
    else:
        hp_idx, hp_val = drelu(x_c, k_p)
    z_pins = G.fwd("pins", hp_idx, hp_val, d_c)
    z_pinned = G.fwd("pinned", hn_idx, hn_val, d_n)
    y_near = z_near @ W["wn_near"] + W["b_near"]
    y_net = z_pins @ W["wn_pins"] + W["b_pins"]
    if root:
        y_near = y_near + Hc @ W["wr_near"]
        y_net = y_net + Hn @ W["wr_pins"]
    y_pinned = z_pinned @ W["w_pinned"] + W["b_pinned"]
    if merge == "max":
        M = np.asarray(forced["M"], bool) if "M" in forced else y_near >= y_pinned
        y_cell = np.where(M, y_near, y_pinned)
    elif merge == "sum":                      # Eq. 6 variant
        M = None
        y_cell = y_near + y_pinned
    else:
        raise ValueError(merge)
    tape = dict(x_c=x_c, x_n=x_n,
                hc_idx=hc_idx, hc_val=hc_val, hn_idx=hn_idx, hn_val=hn_val, Hc=Hc, Hn=Hn,
                hp_idx=hp_idx, hp_val=hp_val,
                z_near=z_near, z_pins=z_pins, z_pinned=z_pinned, y_near=y_near,
                y_pinned=y_pinned, M=M, d_c=d_c, d_n=d_n, merge=merge, root=root)
    return y_cell, y_net, tape


def layer_bwd(G, W, tape, dy_cell, dy_net, need_dx=True):
    """Backward of layer_fwd (Eq. 10-14, Alg. 2):
       dY_near = M dY_cell, dY_pinned = (1-M) dY_cell          (Eq. 12-13)
       dW = Z^T dY, dWr = H^T dY, db = colsum(dY)
       dZ_psi = dY_psi Wn_psi^T
       g_c = SSpMM_near(dZ_near) + SSpMM_pins(dZ_pins) + (dY_near Wr_near^T)[idx_c]
       g_n = SSpMM_pinned(dZ_pinned) + (dY_net Wr_pins^T)[idx_n]
       dX = scatter(g) (D-ReLU mask gradient: zero off the kept support).
       Per-edge-type k (Q27): the pins term is taken at pins' own kept indices and
       scattered separately, dX_c = scatter(g_near + root, idx_c) + scatter(g_pins, idx_p)."""
    dy_cell, dy_net = _f64(dy_cell), _f64(dy_net)
    if tape["merge"] == "max":
        M = tape["M"]
        dy_near = np.where(M, dy_cell, 0.0)
        dy_pinned = np.where(M, 0.0, dy_cell)
    else:
        dy_near = dy_cell
        dy_pinned = dy_cell
    grads = {
        "wn_near": tape["z_near"].T @ dy_near,
        "b_near": dy_near.sum(0),
        "w_pinned": tape["z_pinned"].T @ dy_pinned,
        "b_pinned": dy_pinned.sum(0),
        "wn_pins": tape["z_pins"].T @ dy_net,
        "b_pins": dy_net.sum(0),
    }
    if tape["root"]:
        grads["wr_near"] = tape["Hc"].T @ dy_near
        grads["wr_pins"] = tape["Hn"].T @ dy_net
    dx_c = dx_n = None
    if need_dx:
        hc_idx, hn_idx = tape["hc_idx"], tape["hn_idx"]
        hp_idx = tape.get("hp_idx", hc_idx)
        shared = hp_idx is hc_idx
        g_c = G.bwd("near", hc_idx, dy_near @ W["wn_near"].T)
        g_p = G.bwd("pins", hp_idx, dy_net @ W["wn_pins"].T)
        if shared:
            g_c = g_c + g_p
        g_n = G.bwd("pinned", hn_idx, dy_pinned @ W["w_pinned"].T)
        if tape["root"]:
            g_c = g_c + gather_at(dy_near @ W["wr_near"].T, hc_idx)
            g_n = g_n + gather_at(dy_net @ W["wr_pins"].T, hn_idx)
        dx_c = densify(hc_idx, g_c, tape["d_c"])
        if not shared:
            dx_c = dx_c + densify(hp_idx, g_p, tape["d_c"])
            tape["g_p"] = g_p
        dx_n = densify(hn_idx, g_n, tape["d_n"])
        tape["g_c"], tape["g_n"] = g_c, g_n
    return grads, dx_c, dx_n


# ------------------------------------------------------------------ head, loss, optimiser
def head_mse(y_cell, w_h, b_h, labels):
    """Linear head on cells + MSE over the batch's cells (Q14)."""
    y_cell = _f64(y_cell)
    pred = y_cell @ _f64(w_h) + float(np.asarray(b_h).reshape(-1)[0])
    r = pred - _f64(labels)
    n = r.shape[0]
    loss = float((r * r).sum() / n)
    dpred = 2.0 * r / n
    return loss, dict(w=y_cell.T @ dpred, b=np.array([dpred.sum()])), np.outer(dpred, _f64(w_h))


def adam(theta, grad, m, v, step, lr=2e-4, wd=1e-5, b1=0.9, b2=0.999, eps=1e-8):
    """torch.optim.Adam semantics with coupled L2 weight decay (Q15)."""
    g = grad + wd * theta
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh = m / (1 - b1 ** step)
    vh = v / (1 - b2 ** step)
    return theta - lr * mh / (np.sqrt(vh) + eps), m, v


# ------------------------------------------------------------------ model
def model_fwd_bwd(G, P, n_layers, k_c, k_n, x_c, x_n, labels, merge="max", k_p=None,
                  forced=None):
    """2-layer model: layers -> head/MSE -> backward; the first
    layer's SSpMM is skipped (input features need no gradient). Returns
    (loss, grads dict keyed like P, tapes). forced: None or one layer_fwd
    `forced` dict (or None) per layer (teacher forcing, reading Q28)."""
    tapes, Ws = [], []
    hc, hn = _f64(x_c), _f64(x_n)
    for l in range(n_layers):
        W = layer_params(P, l)
        fl = forced[l] if forced is not None else None
        hc, hn, tape = layer_fwd(G, W, hc, hn, k_c, k_n, merge=merge, k_p=k_p, forced=fl)
        tapes.append(tape)
        Ws.append(W)
    loss, hg, dy_c = head_mse(hc, P["head.w"], P["head.b"], labels)
    dy_n = np.zeros_like(hn)
    grads = {"head.w": hg["w"], "head.b": hg["b"]}
    for l in reversed(range(n_layers)):
        g, dy_c, dy_n = layer_bwd(G, Ws[l], tapes[l], dy_c, dy_n, need_dx=l > 0)
        for k_, v_ in g.items():
            grads[f"l{l}.{k_}"] = v_
    return loss, grads, tapes


def dp_mean(grads_per_rank):
    """Data-parallel gradient = mean of per-rank gradients (north_star; O8)."""
    keys = grads_per_rank[0].keys()
    return {k: sum(g[k] for g in grads_per_rank) / len(grads_per_rank) for k in keys}


# ------------------------------------------------------------------ NEXT-2: per-neighbour-group K
# (Alg. 1 stage 2: "D-ReLU will apply respective
# K-values to the NGs with respect to their sizes ... The more neighbors the NGs have,
# the fewer features per neighbor are required to pass, which corresponds to smaller
# K-values"). Reading Q26: a destination row i in degree bin b keeps, from
# every neighbour j, the top-K_b entries of H_j (the same exact top-k rule), i.e. the
# first K_b entries of j's value-sorted CBSR row; bins by in-degree: deg <= thr[0] ->
# kb[0], deg <= thr[1] -> kb[1], else kb[2] (kb[0] >= kb[1] >= kb[2], K1 > K2 > K3).

def drelu_sorted(x, k):
    """The top-k set of drelu() stored value-descending (ties: lower column first),
    so every prefix of length K' <= k is the row's exact top-K'. (idx int32, val f64)."""
    idx, val = drelu(x, k)
    out_i = np.empty_like(idx)
    out_v = np.empty_like(val)
    for r in range(idx.shape[0]):
        order = np.lexsort((idx[r], -val[r]))          # primary: value desc; then column asc
        out_i[r] = idx[r][order]
        out_v[r] = val[r][order]
    return out_i, out_v


def ng_k(ptr, thr, kb):
    """Per-destination-row K from its in-degree (Q26)."""
    deg = np.diff(_i64(ptr))
    return np.where(deg <= thr[0], kb[0], np.where(deg <= thr[1], kb[1], kb[2])).astype(np.int64)


def _rows_csr(ptr, col, rows, a=None):
    """CSR restricted to `rows` (other rows empty), same row count."""
    ptr = _i64(ptr)
    keep = np.zeros(ptr.size - 1, bool)
    keep[rows] = True
    deg = np.where(keep, np.diff(ptr), 0)
    p2 = np.zeros_like(ptr)
    p2[1:] = np.cumsum(deg)
    sel = np.repeat(keep, np.diff(ptr))
    return p2, _i32(col)[sel], (None if a is None else _f64(a)[sel])


def spmm_fwd_ng(ptr, col, n_dst, c, s, idx_s, val_s, d, thr, kb, a=None):
    """Z_i = c_i sum_j a_ij s_j densify(first K(i) entries of the value-sorted row j):
    per degree bin b, the plain SpMM (spmm_fwd) over that bin's rows with the K_b-prefix
    CBSR; the bins' rows are disjoint, so Z is their sum."""
    K = ng_k(ptr, thr, kb)
    z = np.zeros((n_dst, d), np.float64)
    for kk in sorted(set(int(v) for v in K)):
        rows = np.nonzero(K == kk)[0]
        p2, c2, a2 = _rows_csr(ptr, col, rows, a)
        z += spmm_fwd(p2, c2, n_dst, c, s, _i32(idx_s)[:, :kk], _f64(val_s)[:, :kk], d, a2)
    return z


def spmm_bwd_ng(ptr, col, n_dst, n_src, c, s, idx_s, dz, thr, kb, a=None):
    """Adjoint of spmm_fwd_ng: g[j,t] = sum over i with j in N(i) and t < K(i) of
    c_i a_ij s_j dz[i, idx_s[j,t]] (per bin, spmm_bwd on the K_b prefix)."""
    K = ng_k(ptr, thr, kb)
    k = _i32(idx_s).shape[1]
    g = np.zeros((n_src, k), np.float64)
    for kk in sorted(set(int(v) for v in K)):
        rows = np.nonzero(K == kk)[0]
        p2, c2, a2 = _rows_csr(ptr, col, rows, a)
        g[:, :kk] += spmm_bwd(p2, c2, n_dst, n_src, c, s, _i32(idx_s)[:, :kk], dz, a2)
    return g
