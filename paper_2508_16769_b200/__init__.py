"""B200-native DR-CircuitGNN hot path (arXiv 2508.16769) — Python binding.

Thin wrappers over the C ABI in include/dr.h (libdr.so, sm_100a). They only
marshal arguments: allocate outputs with torch on the current device, pass raw
pointers and the current CUDA stream. Every step of the computation runs in
libdr's kernels; there is no CPU or PyTorch fallback — if the library is
missing or no GPU is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import (DR_FWD_SEQUENTIAL, DR_FWD_TAPS, DR_FWD_INPUT_IN_TAPE,  # noqa: F401
                   DR_FWD_Y_SCRATCH, DR_GRAPH_ORDER_IDENTITY,  # noqa: F401
                   DR_GRAPH_SKIP_VALIDATION, DR_GRAPHCONV_SYM, DR_MERGE_MAX, DR_MERGE_SUM,
                   DR_NEAR, DR_PINNED, DR_PINS, DR_SAGE_MEAN, DRError, EXPORTS, check,
                   dr_cbsr, dr_layer, dr_layer_grad, dr_rel_desc, dr_tape_view, dr_train_cfg,
                   dr_graph_info_t, lib)

REL_NAMES = ("near", "pins", "pinned")
REL_ID = {"near": DR_NEAR, "pins": DR_PINS, "pinned": DR_PINNED}
DEFAULT_MODULES = {"near": DR_SAGE_MEAN, "pins": DR_SAGE_MEAN, "pinned": DR_GRAPHCONV_SYM}


def _torch():
    import torch
    return torch


def _stream(stream=None):
    torch = _torch()
    if stream is None:
        if not torch.cuda.is_available():
            return C.c_void_p(0)        # host-only calls (validation) on a GPU-less host
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def probe_read(buf, reps, sink, stream=None):
    """dr_probe_read: stream `buf` (a CUDA tensor) `reps` times (L2 / HBM read probe)."""
    check(lib().dr_probe_read(_ptr(buf), buf.numel() * buf.element_size(), reps, _ptr(sink),
                              _stream(stream)))


def version():
    return lib().dr_version().decode()


def launch_count():
    return int(lib().dr_launch_count())


def launch_count_reset():
    lib().dr_launch_count_reset()


def debug_set(name, value):
    """dr_debug_set: experiment / test switch (see include/dr.h)."""
    check(lib().dr_debug_set(name.encode(), int(value)))


def profile_begin():
    """Start per-kernel CUDA-event timing of libdr launches on this thread."""
    check(lib().dr_profile_begin())


def profile_end():
    """Stop timing; return {tag: (launches, total_ms, max_ms)}."""
    from ._lib import dr_profile_entry
    cap = 256
    buf = (dr_profile_entry * cap)()
    n = C.c_int32()
    check(lib().dr_profile_end(buf, cap, C.byref(n)))
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms),
                                   float(buf[i].max_ms)) for i in range(min(n.value, cap))}


# ------------------------------------------------------------------ graph
class Graph:
    """Device-resident heterograph (dr_graph_create). `rels` maps 'near'/'pins'/
    'pinned' to (row_ptr int64 [n_dst+1], col_idx int32 [nnz]) host arrays.
    Optional per relation (dr_rel_desc): `csc` -> (col_ptr int64, row_idx int32
    [, tval float32]), `degrees` -> (deg_dst, deg_src) int32 (either may be
    None), `norms` -> (c, s) float32 (either may be None)."""

    def __init__(self, n_cell, n_net, rels, modules=None, weights=None, n_threads=0, flags=0,
                 stream=None, csc=None, degrees=None, norms=None):
        modules = dict(DEFAULT_MODULES if modules is None else modules)
        weights = dict(weights or {})
        csc, degrees, norms = dict(csc or {}), dict(degrees or {}), dict(norms or {})

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a.ctypes.data if a.size else None
        dims = {"near": (n_cell, n_cell), "pins": (n_net, n_cell), "pinned": (n_cell, n_net)}
        descs = (dr_rel_desc * 3)()
        self._keep = []
        for name in REL_NAMES:
            ptr, col = rels[name]
            ptr = np.ascontiguousarray(ptr, dtype=np.int64)
            col = np.ascontiguousarray(col, dtype=np.int32)
            w = weights.get(name)
            if w is not None:
                w = np.ascontiguousarray(w, dtype=np.float32)
            self._keep += [ptr, col, w]
            d = descs[REL_ID[name]]
            d.n_dst, d.n_src = int(ptr.shape[0]) - 1, dims[name][1]
            d.nnz = int(col.shape[0])
            d.row_ptr = ptr.ctypes.data
            d.col_idx = col.ctypes.data if col.size else None
            d.val = None if w is None else w.ctypes.data
            d.module = int(modules[name])
            if name in csc:
                t = tuple(csc[name]) + (None,) * (3 - len(csc[name]))
                d.col_ptr, d.row_idx = arr(t[0], np.int64), arr(t[1], np.int32)
                d.tval = arr(t[2], np.float32)
            if name in degrees:
                d.deg_dst, d.deg_src = arr(degrees[name][0], np.int32), arr(degrees[name][1], np.int32)
            if name in norms:
                d.norm_dst, d.norm_src = arr(norms[name][0], np.float32), arr(norms[name][1], np.float32)
        out = C.c_void_p()
        check(lib().dr_graph_create(int(n_cell), int(n_net), descs, None, int(n_threads),
                                    int(flags), _stream(stream), C.byref(out)))
        self._keep = None
        self.handle = out
        self.n_cell, self.n_net = int(n_cell), int(n_net)

    @classmethod
    def from_design(cls, d, **kw):
        rels = {r: d.rel(r)[:2] for r in REL_NAMES}
        return cls(d.n_cell, d.n_net, rels, **kw)

    def info(self):
        i = dr_graph_info_t()
        check(lib().dr_graph_info(self.handle, C.byref(i)))
        return dict(n_cell=i.n_cell, n_net=i.n_net, nnz=list(i.nnz),
                    max_deg_dst=list(i.max_deg_dst), max_deg_src=list(i.max_deg_src),
                    hub_rows_dst=list(i.hub_rows_dst), hub_rows_src=list(i.hub_rows_src),
                    device_bytes=int(i.device_bytes), tiles=list(i.tiles),
                    tiles_T=list(i.tiles_T), chunks=list(i.chunks), chunks_T=list(i.chunks_T))

    def close(self):
        if getattr(self, "handle", None):
            lib().dr_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ CBSR ops
def _cbsr(val, idx, dim):
    n, k = val.shape
    return dr_cbsr(n, int(dim), int(k), 1, idx.data_ptr() if n else None,
                   val.data_ptr() if n else None)


def drelu_topk(x, k, out=None, stream=None):
    """Eq. 2-3: exact row top-k -> CBSR (val float32 [n,k], idx uint8 [n,k])."""
    torch = _torch()
    n, dim = x.shape
    assert x.dtype == torch.float32 and x.is_cuda and x.stride(1) == 1
    if out is None:
        val = torch.empty((n, k), device=x.device, dtype=torch.float32)
        idx = torch.empty((n, k), device=x.device, dtype=torch.uint8)
    else:
        val, idx = out
    cb = _cbsr(val, idx, dim)
    check(lib().dr_drelu_topk(_ptr(x), n, dim, x.stride(0), C.byref(cb), _stream(stream)))
    return val, idx


def spmm_fwd(g, rel, val, idx, dim, out=None, stream=None):
    """Eq. 5-7 / Alg. 1: Z = diag(c) A diag(s) densify(H) for relation `rel`."""
    torch = _torch()
    r = REL_ID[rel] if isinstance(rel, str) else int(rel)
    n_dst = g.n_cell if r in (DR_NEAR, DR_PINNED) else g.n_net
    z = out if out is not None else torch.empty((n_dst, dim), device=val.device,
                                                 dtype=torch.float32)
    cb = _cbsr(val, idx, dim)
    check(lib().dr_spmm_fwd(g.handle, r, C.byref(cb), _ptr(z), _stream(stream)))
    return z


def spmm_bwd(g, rel, dz, val, idx, dim, want_g=True, want_dx=False, accumulate=False,
             g_out=None, dx_out=None, stream=None):
    """Eq. 10-11 / Alg. 2: SSpMM at the kept CBSR indices (+ D-ReLU mask scatter)."""
    torch = _torch()
    r = REL_ID[rel] if isinstance(rel, str) else int(rel)
    n, k = val.shape
    gk = g_out if g_out is not None else (
        torch.empty((n, k), device=dz.device, dtype=torch.float32) if want_g else None)
    dx = dx_out if dx_out is not None else (
        torch.empty((n, dim), device=dz.device, dtype=torch.float32) if want_dx else None)
    cb = _cbsr(val, idx, dim)
    check(lib().dr_spmm_bwd(g.handle, r, _ptr(dz), C.byref(cb), _ptr(gk), _ptr(dx),
                            int(bool(accumulate)), _stream(stream)))
    return gk, dx


# ------------------------------------------------------------------ NEXT-2 (reading Q26)
class NgPlan:
    """dr_ng_plan: the K schedule (thr, kb) of reading Q26 bound to one relation of
    one graph (per-edge K precomputed on the device). Keeps the graph alive."""

    def __init__(self, g, rel, thr, kb, stream=None):
        from ._lib import dr_ng_sched
        s = dr_ng_sched()
        s.thr[0], s.thr[1] = int(thr[0]), int(thr[1])
        s.kb[0], s.kb[1], s.kb[2] = int(kb[0]), int(kb[1]), int(kb[2])
        self.g, self.rel = g, (REL_ID[rel] if isinstance(rel, str) else int(rel))
        self.thr, self.kb = tuple(thr), tuple(kb)
        h = C.c_void_p()
        check(lib().dr_ng_plan_create(g.handle, self.rel, C.byref(s), _stream(stream),
                                      C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().dr_ng_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def drelu_topk_sorted(x, k, out=None, stream=None):
    """Eq. 2-3 with each row's k pairs in value-descending order (k <= 32)."""
    torch = _torch()
    n, dim = x.shape
    assert x.dtype == torch.float32 and x.is_cuda and x.stride(1) == 1
    if out is None:
        val = torch.empty((n, k), device=x.device, dtype=torch.float32)
        idx = torch.empty((n, k), device=x.device, dtype=torch.uint8)
    else:
        val, idx = out
    cb = _cbsr(val, idx, dim)
    check(lib().dr_drelu_topk_sorted(_ptr(x), n, dim, x.stride(0), C.byref(cb),
                                     _stream(stream)))
    return val, idx


def spmm_fwd_ng(plan, val, idx, dim, out=None, stream=None):
    """Eq. 5-7 with the destination-degree K schedule of reading Q26: destination i
    aggregates the first K(deg_i) pairs of each value-sorted source row."""
    torch = _torch()
    n_dst = plan.g.n_cell if plan.rel in (DR_NEAR, DR_PINNED) else plan.g.n_net
    z = out if out is not None else torch.empty((n_dst, dim), device=val.device,
                                                 dtype=torch.float32)
    cb = _cbsr(val, idx, dim)
    check(lib().dr_spmm_fwd_ng(plan.handle, C.byref(cb), _ptr(z), _stream(stream)))
    return z


def spmm_bwd_ng(plan, dz, val, idx, dim, want_g=True, want_dx=False, g_out=None, dx_out=None,
                stream=None):
    """Adjoint of spmm_fwd_ng (Eq. 10-11 restricted to each destination's prefix)."""
    torch = _torch()
    n, k = val.shape
    gk = g_out if g_out is not None else (
        torch.empty((n, k), device=dz.device, dtype=torch.float32) if want_g else None)
    dx = dx_out if dx_out is not None else (
        torch.empty((n, dim), device=dz.device, dtype=torch.float32) if want_dx else None)
    cb = _cbsr(val, idx, dim)
    check(lib().dr_spmm_bwd_ng(plan.handle, _ptr(dz), C.byref(cb), _ptr(gk), _ptr(dx),
                               _stream(stream)))
    return gk, dx


# ------------------------------------------------------------------ single-graph multi-GPU (§8 f4)
def _rel_desc(ptr, col, n_src, module, weight=None):
    from ._lib import dr_rel_desc
    ptr = np.ascontiguousarray(ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    w = None if weight is None else np.ascontiguousarray(weight, dtype=np.float32)
    d = dr_rel_desc()
    d.n_dst, d.n_src, d.nnz = int(ptr.shape[0]) - 1, int(n_src), int(col.shape[0])
    d.row_ptr = ptr.ctypes.data
    d.col_idx = col.ctypes.data if col.size else None
    d.val = None if w is None else w.ctypes.data
    d.module = int(module)
    return d, (ptr, col, w)


def shard_plan(ptr, col, n_src, world, module=DR_SAGE_MEAN):
    """dr_shard_plan: default (dst_part, src_part), each int64 [world+1] (host only)."""
    d, keep = _rel_desc(ptr, col, n_src, module)
    dp = np.zeros(world + 1, np.int64)
    sp = np.zeros(world + 1, np.int64)
    check(lib().dr_shard_plan(C.byref(d), int(world), dp.ctypes.data, sp.ctypes.data))
    return dp, sp


class Shard:
    """dr_shard: rank `rank`'s destination-row block of one relation (1-D partition
    over `world` ranks, CBSR allgather / g reduce-scatter exchanges)."""

    def __init__(self, ptr, col, n_src, world, rank, module=DR_SAGE_MEAN, weight=None,
                 dst_part=None, src_part=None, stream=None):
        d, keep = _rel_desc(ptr, col, n_src, module, weight)
        dp = None if dst_part is None else np.ascontiguousarray(dst_part, np.int64)
        sp = None if src_part is None else np.ascontiguousarray(src_part, np.int64)
        h = C.c_void_p()
        check(lib().dr_shard_create(C.byref(d), int(world), int(rank),
                                    None if dp is None else dp.ctypes.data,
                                    None if sp is None else sp.ctypes.data, None,
                                    _stream(stream), C.byref(h)))
        self.handle = h
        i = self.info()
        self.world, self.rank, self.max_src = i["world"], i["rank"], i["max_src"]
        self.dst_begin, self.dst_end = i["dst_begin"], i["dst_end"]
        self.src_begin, self.src_end = i["src_begin"], i["src_end"]

    @classmethod
    def from_design(cls, d, rel, world, rank, **kw):
        ptr, col, nd, ns = d.rel(rel)
        kw.setdefault("module", DEFAULT_MODULES[rel])
        return cls(ptr, col, ns, world, rank, **kw)

    def info(self):
        from ._lib import dr_shard_info_t
        i = dr_shard_info_t()
        check(lib().dr_shard_info(self.handle, C.byref(i)))
        return {f: getattr(i, f) for f, _ in dr_shard_info_t._fields_}

    def allgather_cbsr(self, val_l, idx_l, dim, val_a=None, idx_a=None, comm=None, stream=None):
        torch = _torch()
        k = val_l.shape[1]
        n_all = self.world * self.max_src
        if val_a is None:
            val_a = torch.empty((n_all, k), device=val_l.device, dtype=torch.float32)
            idx_a = torch.empty((n_all, k), device=val_l.device, dtype=torch.uint8)
        hl, ha = _cbsr(val_l, idx_l, dim), _cbsr(val_a, idx_a, dim)
        check(lib().dr_shard_allgather_cbsr(self.handle, C.byref(hl), C.byref(ha),
                                            C.c_void_p(comm) if comm else None, _stream(stream)))
        return val_a, idx_a

    def spmm_fwd(self, val_a, idx_a, dim, out=None, stream=None):
        torch = _torch()
        z = out if out is not None else torch.empty((self.dst_end - self.dst_begin, dim),
                                                     device=val_a.device, dtype=torch.float32)
        ha = _cbsr(val_a, idx_a, dim)
        check(lib().dr_shard_spmm_fwd(self.handle, C.byref(ha), _ptr(z), _stream(stream)))
        return z

    def spmm_bwd(self, dz_l, val_a, idx_a, dim, out=None, stream=None):
        torch = _torch()
        g = out if out is not None else torch.empty(tuple(val_a.shape), device=dz_l.device,
                                                     dtype=torch.float32)
        ha = _cbsr(val_a, idx_a, dim)
        check(lib().dr_shard_spmm_bwd(self.handle, _ptr(dz_l), C.byref(ha), _ptr(g),
                                      _stream(stream)))
        return g

    def reduce_scatter_g(self, g_part, val_l, idx_l, dim, want_dx=True, comm=None, stream=None):
        torch = _torch()
        g_l = torch.empty(tuple(val_l.shape), device=g_part.device, dtype=torch.float32)
        dx = (torch.empty((self.max_src, dim), device=g_part.device, dtype=torch.float32)
              if want_dx else None)
        hl = _cbsr(val_l, idx_l, dim)
        check(lib().dr_shard_reduce_scatter_g(self.handle, _ptr(g_part), C.byref(hl), _ptr(g_l),
                                              _ptr(dx), C.c_void_p(comm) if comm else None,
                                              _stream(stream)))
        return g_l, dx

    # ---- the exchange fused into the SpMM over peer memory (dr_shard_spmm_*_peer)
    def _peer(self, peers):
        from ._lib import dr_peer_cbsr
        pc = dr_peer_cbsr()
        pc.world = self.world
        for q, (v, i) in enumerate(peers):
            pc.val[q] = v if isinstance(v, int) else v.data_ptr()
            pc.idx[q] = i if isinstance(i, int) else i.data_ptr()
        return pc

    def spmm_fwd_peer(self, peers, dim, k, out=None, device="cuda", stream=None):
        """peers: per rank q (val_q, idx_q) -- tensors on this device or raw device
        pointers (peer-mapped) -- of rank q's local CBSR (max_src x k)."""
        torch = _torch()
        z = out if out is not None else torch.empty((self.dst_end - self.dst_begin, dim),
                                                     device=device, dtype=torch.float32)
        pc = self._peer(peers)
        check(lib().dr_shard_spmm_fwd_peer(self.handle, C.byref(pc), int(dim), int(k), _ptr(z),
                                           _stream(stream)))
        return z

    def spmm_bwd_peer(self, dz_l, peers, dim, k, inboxes, stream=None):
        """inboxes: per owner q its inbox ([world x max_src x k] fp32, tensor or raw
        device pointer); this rank writes slot `rank` of each."""
        pc = self._peer(peers)
        arr = (C.c_void_p * 8)(*[(x if isinstance(x, int) else x.data_ptr()) for x in inboxes])
        check(lib().dr_shard_spmm_bwd_peer(self.handle, _ptr(dz_l), C.byref(pc), int(dim), int(k),
                                           arr, _stream(stream)))

    def inbox_reduce(self, inbox, val_l, idx_l, dim, want_dx=True, stream=None):
        torch = _torch()
        g_l = torch.empty(tuple(val_l.shape), device=val_l.device, dtype=torch.float32)
        dx = (torch.empty((self.max_src, dim), device=val_l.device, dtype=torch.float32)
              if want_dx else None)
        hl = _cbsr(val_l, idx_l, dim)
        check(lib().dr_shard_inbox_reduce(self.handle, _ptr(inbox), C.byref(hl), _ptr(g_l),
                                          _ptr(dx), _stream(stream)))
        return g_l, dx

    def close(self):
        if getattr(self, "handle", None):
            lib().dr_shard_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ HeteroConv layer
LAYER_KEYS = ("wn_near", "wr_near", "b_near", "w_pinned", "b_pinned", "wn_pins", "wr_pins",
              "b_pins")


class Layer:
    """dr_layer over torch tensors W (keys as LAYER_KEYS; wr_* may be None)."""

    def __init__(self, W, d_cell, d_net, d_out, k_cell, k_net, merge=DR_MERGE_MAX, k_pins=0):
        self.W = W
        L = dr_layer()
        L.d_cell, L.d_net, L.d_out, L.k_cell, L.k_net, L.merge = (
            d_cell, d_net, d_out, k_cell, k_net, merge)
        L.k_pins = k_pins              # per-edge-type k (Q27); 0 = k_cell
        L.wn[DR_NEAR] = W["wn_near"].data_ptr()
        L.wn[DR_PINNED] = W["w_pinned"].data_ptr()
        L.wn[DR_PINS] = W["wn_pins"].data_ptr()
        L.wr[DR_NEAR] = W["wr_near"].data_ptr() if W.get("wr_near") is not None else None
        L.wr[DR_PINS] = W["wr_pins"].data_ptr() if W.get("wr_pins") is not None else None
        L.wr[DR_PINNED] = None
        L.b[DR_NEAR] = W["b_near"].data_ptr()
        L.b[DR_PINNED] = W["b_pinned"].data_ptr()
        L.b[DR_PINS] = W["b_pins"].data_ptr()
        self.c = L

    def tape_bytes(self, g, flags=0):
        n = C.c_size_t()
        check(lib().dr_heteroconv_tape_bytes(g.handle, C.byref(self.c), flags, C.byref(n)))
        return n.value


def heteroconv_fwd(g, layer, x_cell, x_net, flags=0, tape=None, stream=None):
    torch = _torch()
    dev = x_cell.device
    D = layer.c.d_out
    y_cell = torch.empty((g.n_cell, D), device=dev, dtype=torch.float32)
    y_net = torch.empty((g.n_net, D), device=dev, dtype=torch.float32)
    if tape is None:
        tape = torch.empty(layer.tape_bytes(g, flags), device=dev, dtype=torch.uint8)
    check(lib().dr_heteroconv_fwd(g.handle, C.byref(layer.c), _ptr(x_cell), _ptr(x_net),
                                  _ptr(y_cell), _ptr(y_net), _ptr(tape), flags, _stream(stream)))
    return y_cell, y_net, tape


def heteroconv_fwd_chain(g, layer, x_cell, x_net, next_layer=None, next_tape=None, flags=0,
                         next_flags=0, tape=None, stream=None):
    """dr_heteroconv_fwd_chain: the layer forward with the next layer's D-ReLU fused
    into the projection epilogue (row a5). x_cell / x_net may be None with
    DR_FWD_INPUT_IN_TAPE (the layer's CBSR inputs are already in `tape`). Returns
    (y_cell, y_net, tape, next_tape); a next tape is allocated when next_layer is
    given without one."""
    torch = _torch()
    dev = (x_cell if x_cell is not None else tape).device
    D = layer.c.d_out
    y_cell = torch.empty((g.n_cell, D), device=dev, dtype=torch.float32)
    y_net = torch.empty((g.n_net, D), device=dev, dtype=torch.float32)
    if tape is None:
        tape = torch.empty(layer.tape_bytes(g, flags), device=dev, dtype=torch.uint8)
    if next_layer is not None and next_tape is None:
        next_tape = torch.empty(next_layer.tape_bytes(g, next_flags), device=dev, dtype=torch.uint8)
    nl = C.byref(next_layer.c) if next_layer is not None else None
    check(lib().dr_heteroconv_fwd_chain(
        g.handle, C.byref(layer.c), _ptr(x_cell) if x_cell is not None else None,
        _ptr(x_net) if x_net is not None else None, _ptr(y_cell), _ptr(y_net), _ptr(tape), flags,
        nl, _ptr(next_tape) if next_tape is not None else None, next_flags, _stream(stream)))
    return y_cell, y_net, tape, next_tape


def tape_view(g, layer, tape, flags=0):
    """Torch views of the forward tape (teacher-forced parity)."""
    torch = _torch()
    v = dr_tape_view()
    check(lib().dr_heteroconv_tape_view(g.handle, C.byref(layer.c), _ptr(tape), flags,
                                        C.byref(v)))
    base = tape.data_ptr()
    L = layer.c

    def sl(ptr, shape, dtype):
        if not ptr:
            return None
        nbytes = int(np.prod(shape)) * torch.tensor([], dtype=dtype).element_size()
        off = ptr - base
        return tape[off:off + nbytes].view(dtype).view(*shape)
    nc, nn, D = g.n_cell, g.n_net, L.d_out

    def zview(r, n, w):
        """Z of relation r as fp32 (a copy when the tape holds split bf16 rows:
        [hi | lo] halves, Z = hi + lo)"""
        if not v.z_split[r]:
            return sl(v.z[r], (n, w), torch.float32)
        hl = sl(v.z[r], (n, 2 * w), torch.bfloat16)
        return hl[:, :w].float() + hl[:, w:].float()
    return dict(
        hc_val=sl(v.h_cell.val, (nc, L.k_cell), torch.float32),
        hc_idx=sl(v.h_cell.idx, (nc, L.k_cell), torch.uint8),
        hn_val=sl(v.h_net.val, (nn, L.k_net), torch.float32),
        hn_idx=sl(v.h_net.idx, (nn, L.k_net), torch.uint8),
        hp_val=sl(v.h_pins.val, (nc, v.h_pins.k), torch.float32),
        hp_idx=sl(v.h_pins.idx, (nc, v.h_pins.k), torch.uint8),
        z_near=zview(DR_NEAR, nc, L.d_cell),
        z_pins=zview(DR_PINS, nn, L.d_cell),
        z_pinned=zview(DR_PINNED, nc, L.d_net),
        z_split=[int(x) for x in v.z_split],
        y_near=sl(v.y_near, (nc, D), torch.float32),
        y_pinned=sl(v.y_pinned, (nc, D), torch.float32),
        mask=sl(v.mask, (nc, (D + 31) // 32), torch.int32),
    )


def heteroconv_bwd(g, layer, tape, dy_cell, dy_net, need_dx=True, flags=0, stream=None):
    """Returns (grads dict keyed like LAYER_KEYS, dx_cell, dx_net)."""
    torch = _torch()
    dev = dy_cell.device
    grads = {k: torch.empty_like(v) for k, v in layer.W.items() if v is not None}
    G = dr_layer_grad()
    G.wn[DR_NEAR] = grads["wn_near"].data_ptr()
    G.wn[DR_PINNED] = grads["w_pinned"].data_ptr()
    G.wn[DR_PINS] = grads["wn_pins"].data_ptr()
    G.wr[DR_NEAR] = grads["wr_near"].data_ptr() if "wr_near" in grads else None
    G.wr[DR_PINS] = grads["wr_pins"].data_ptr() if "wr_pins" in grads else None
    G.b[DR_NEAR] = grads["b_near"].data_ptr()
    G.b[DR_PINNED] = grads["b_pinned"].data_ptr()
    G.b[DR_PINS] = grads["b_pins"].data_ptr()
    dxc = dxn = None
    if need_dx:
        dxc = torch.empty((g.n_cell, layer.c.d_cell), device=dev, dtype=torch.float32)
        dxn = torch.empty((g.n_net, layer.c.d_net), device=dev, dtype=torch.float32)
    check(lib().dr_heteroconv_bwd(g.handle, C.byref(layer.c), _ptr(tape), _ptr(dy_cell),
                                  _ptr(dy_net), _ptr(dxc), _ptr(dxn), C.byref(G), flags,
                                  _stream(stream)))
    return grads, dxc, dxn


def _grad_struct(layer, dev):
    torch = _torch()
    grads = {k: torch.empty_like(v) for k, v in layer.W.items() if v is not None}
    G = dr_layer_grad()
    G.wn[DR_NEAR] = grads["wn_near"].data_ptr()
    G.wn[DR_PINNED] = grads["w_pinned"].data_ptr()
    G.wn[DR_PINS] = grads["wn_pins"].data_ptr()
    G.wr[DR_NEAR] = grads["wr_near"].data_ptr() if "wr_near" in grads else None
    G.wr[DR_PINS] = grads["wr_pins"].data_ptr() if "wr_pins" in grads else None
    G.b[DR_NEAR] = grads["b_near"].data_ptr()
    G.b[DR_PINNED] = grads["b_pinned"].data_ptr()
    G.b[DR_PINS] = grads["b_pins"].data_ptr()
    return grads, G


class ShardLayer:
    """dr_shard_layer (f4): a HeteroConv layer over this rank's rows of three
    dr_shard (near, pins, pinned) sharing one cell and one net partition; the
    exchanges go through peer memory (lists of per-rank (val, idx) CBSR and
    per-rank inboxes, tensors or raw device pointers)."""

    def __init__(self, near, pins, pinned):
        h = C.c_void_p()
        check(lib().dr_shard_layer_create(near.handle, pins.handle, pinned.handle, C.byref(h)))
        self.handle = h
        self.shards = (near, pins, pinned)
        self.world, self.rank = near.world, near.rank
        self.n_cell = near.dst_end - near.dst_begin
        self.n_net = pins.dst_end - pins.dst_begin
        self.m_cell, self.m_net = near.max_src, pinned.max_src

    def tape_bytes(self, layer, flags=0):
        n = C.c_size_t()
        check(lib().dr_shard_layer_tape_bytes(self.handle, C.byref(layer.c), flags, C.byref(n)))
        return n.value

    def _peer(self, peers):
        from ._lib import dr_peer_cbsr
        pc = dr_peer_cbsr()
        pc.world = self.world
        for q, (v, i) in enumerate(peers):
            pc.val[q] = v if isinstance(v, int) else v.data_ptr()
            pc.idx[q] = i if isinstance(i, int) else i.data_ptr()
        return pc

    def fwd(self, layer, peers_cell, peers_net, tape=None, flags=0, device="cuda", stream=None):
        torch = _torch()
        D = layer.c.d_out
        yc = torch.empty((self.n_cell, D), device=device, dtype=torch.float32)
        yn = torch.empty((self.n_net, D), device=device, dtype=torch.float32)
        if tape is None:
            tape = torch.empty(self.tape_bytes(layer, flags), device=device, dtype=torch.uint8)
        hc, hn = self._peer(peers_cell), self._peer(peers_net)
        check(lib().dr_shard_layer_fwd(self.handle, C.byref(layer.c), C.byref(hc), C.byref(hn),
                                       _ptr(yc), _ptr(yn), _ptr(tape), flags, _stream(stream)))
        return yc, yn, tape

    def bwd(self, layer, tape, dy_cell, dy_net, peers_cell, peers_net, inbox_cell, inbox_net,
            flags=0, stream=None):
        """Writes this rank's slots of every owner's inboxes; returns this rank's
        rows' contribution to the weight gradients (sum over ranks = the layer's)."""
        grads, G = _grad_struct(layer, dy_cell.device)
        hc, hn = self._peer(peers_cell), self._peer(peers_net)
        ic = (C.c_void_p * 8)(*[(x if isinstance(x, int) else x.data_ptr()) for x in inbox_cell])
        inn = (C.c_void_p * 8)(*[(x if isinstance(x, int) else x.data_ptr()) for x in inbox_net])
        check(lib().dr_shard_layer_bwd(self.handle, C.byref(layer.c), _ptr(tape), _ptr(dy_cell),
                                       _ptr(dy_net), C.byref(hc), C.byref(hn), ic, inn, C.byref(G),
                                       flags, _stream(stream)))
        return grads

    def dx(self, layer, tape, peers_cell, peers_net, inbox_cell_local, inbox_net_local,
           stream=None):
        torch = _torch()
        dev = tape.device
        dxc = torch.empty((self.n_cell, layer.c.d_cell), device=dev, dtype=torch.float32)
        dxn = torch.empty((self.n_net, layer.c.d_net), device=dev, dtype=torch.float32)
        hc, hn = self._peer(peers_cell), self._peer(peers_net)
        check(lib().dr_shard_layer_dx(self.handle, C.byref(layer.c), _ptr(tape), C.byref(hc),
                                      C.byref(hn), _ptr(inbox_cell_local), _ptr(inbox_net_local),
                                      _ptr(dxc), _ptr(dxn), _stream(stream)))
        return dxc, dxn

    def close(self):
        if getattr(self, "handle", None):
            lib().dr_shard_layer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ training
PARAM_ORDER = ("wn_near", "wr_near", "b_near", "w_pinned", "b_pinned", "wn_pins", "wr_pins",
               "b_pins")


def flatten_params(P, n_layers):
    """Named arrays (gen.make_params) -> flat float32 array in the dr.h layout."""
    parts = []
    for l in range(n_layers):
        for k in PARAM_ORDER:
            parts.append(np.asarray(P[f"l{l}.{k}"], dtype=np.float32).reshape(-1))
    parts.append(np.asarray(P["head.w"], dtype=np.float32).reshape(-1))
    parts.append(np.asarray(P["head.b"], dtype=np.float32).reshape(-1))
    return np.concatenate(parts)


def unflatten(flat, n_layers, d_cell, d_net, D):
    """Inverse of flatten_params (shapes per dr.h)."""
    out, o = {}, 0
    dc, dn = d_cell, d_net
    for l in range(n_layers):
        shapes = {"wn_near": (dc, D), "wr_near": (dc, D), "b_near": (D,), "w_pinned": (dn, D),
                  "b_pinned": (D,), "wn_pins": (dc, D), "wr_pins": (dn, D), "b_pins": (D,)}
        for k in PARAM_ORDER:
            n = int(np.prod(shapes[k]))
            out[f"l{l}.{k}"] = flat[o:o + n].reshape(shapes[k])
            o += n
        dc = dn = D
    out["head.w"] = flat[o:o + D]
    out["head.b"] = flat[o + D:o + D + 1]
    return out


class Trainer:
    """dr_trainer over a flat device parameter tensor (updated in place)."""

    def __init__(self, params, n_layers, d_in_cell, d_in_net, d_hidden, k_cell, k_net,
                 lr=2e-4, weight_decay=1e-5, beta1=0.9, beta2=0.999, eps=1e-8, nccl_comm=None,
                 k_pins=0):
        torch = _torch()
        cfg = dr_train_cfg(n_layers, d_in_cell, d_in_net, d_hidden, k_cell, k_net, lr,
                           weight_decay, beta1, beta2, eps, k_pins)
        self.cfg = cfg
        self.n_params = int(lib().dr_train_param_count(C.byref(cfg)))
        assert params.numel() == self.n_params and params.dtype == torch.float32
        self.params = params
        out = C.c_void_p()
        check(lib().dr_trainer_create(C.byref(cfg), _ptr(params), self.n_params,
                                      C.c_void_p(nccl_comm) if nccl_comm else None, None,
                                      C.byref(out)))
        self.handle = out
        self.loss_host = torch.zeros(1, dtype=torch.float32).pin_memory()

    def step(self, g, x_cell, x_net, labels, grad_out=None, sync=True, stream=None):
        check(lib().dr_train_step(self.handle, g.handle, _ptr(x_cell), _ptr(x_net),
                                  _ptr(labels), C.c_void_p(self.loss_host.data_ptr()),
                                  _ptr(grad_out), _stream(stream)))
        if sync:
            _torch().cuda.current_stream().synchronize() if stream is None else stream.synchronize()
            return float(self.loss_host[0])
        return None

    def close(self):
        if getattr(self, "handle", None):
            lib().dr_trainer_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def peer_buffers(shape, dtype, group=None):
    """Multi-GPU plumbing of the fused peer-memory exchange (f4): a buffer of
    `shape` on this rank allocated in torch symmetric memory and rendezvoused over
    `group`, so every rank's copy is addressable from every GPU (NVLink P2P).
    Returns (local tensor, [device pointer of rank q's buffer for q in ranks])
    for dr_peer_cbsr / the inboxes. Needs torch.distributed initialised with one
    GPU per rank on a P2P-capable node."""
    torch = _torch()
    import torch.distributed as tdist
    import torch.distributed._symmetric_memory as symm_mem
    g = group if group is not None else tdist.group.WORLD
    t = symm_mem.empty(*shape, dtype=dtype, device=torch.device("cuda", torch.cuda.current_device()))
    h = symm_mem.rendezvous(t, g)
    return t, [int(p) for p in h.buffer_ptrs]


def nccl_unique_id():
    buf = (C.c_char * 128)()
    check(lib().dr_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm_init(uid, nranks, rank):
    buf = (C.c_char * 128).from_buffer_copy(uid)
    comm = C.c_void_p()
    check(lib().dr_nccl_comm_init(buf, int(nranks), int(rank), C.byref(comm)))
    return comm.value


def nccl_comm_destroy(comm):
    check(lib().dr_nccl_comm_destroy(C.c_void_p(comm)))
