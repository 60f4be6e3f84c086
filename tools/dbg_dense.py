"""Debug: dX of the tc2 path and of the SIMT path vs the oracle (parallel and sequential streams)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch

import paper_2508_16769_b200 as dr
from gen import make_config, make_params
from oracle import oracle as O
from parity_util import row_err, to_np

name, D, k = sys.argv[1] if len(sys.argv) > 1 else "C2", 64, 8
d = make_config("C2", scale=0.1)
g = dr.Graph.from_design(d)
P = make_params(D, D, D, 1, seed=8)
W = {kk.split(".", 1)[1]: torch.as_tensor(v).cuda() for kk, v in P.items() if kk.startswith("l0.")}
L = dr.Layer(W, D, D, D, k, k)
Wo = O.layer_params(P, 0)
rng = np.random.default_rng(12)
xc = torch.as_tensor(rng.standard_normal((d.n_cell, D)).astype(np.float32)).cuda()
xn = torch.as_tensor(rng.standard_normal((d.n_net, D)).astype(np.float32)).cuda()
dyc = rng.standard_normal((d.n_cell, D)).astype(np.float32)
dyn = rng.standard_normal((d.n_net, D)).astype(np.float32)
G = O.OGraph(d)
for mode in ("0", "1"):
    for flags in (dr.DR_FWD_TAPS, dr.DR_FWD_TAPS | dr.DR_FWD_SEQUENTIAL):
        os.environ["DR_DENSE_SIMT"] = mode
        yc, yn, tape = dr.heteroconv_fwd(g, L, xc, xn, flags=flags)
        v = dr.tape_view(g, L, tape, flags)
        grads, dxc, dxn = dr.heteroconv_bwd(g, L, tape, torch.as_tensor(dyc).cuda(),
                                            torch.as_tensor(dyn).cuda(), flags=flags)
        torch.cuda.synchronize()
        hc_idx = to_np(v["hc_idx"]).astype(np.int32)
        hn_idx = to_np(v["hn_idx"]).astype(np.int32)
        hc_val = to_np(v["hc_val"]).astype(np.float64)
        hn_val = to_np(v["hn_val"]).astype(np.float64)
        M = ((to_np(v["mask"]).view(np.uint32)[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(d.n_cell, -1)[:, :D].astype(bool)
        T = dict(hc_idx=hc_idx, hc_val=hc_val, hn_idx=hn_idx, hn_val=hn_val,
                 Hc=O.densify(hc_idx, hc_val, D), Hn=O.densify(hn_idx, hn_val, D),
                 z_near=to_np(v["z_near"]).astype(np.float64), z_pins=to_np(v["z_pins"]).astype(np.float64),
                 z_pinned=to_np(v["z_pinned"]).astype(np.float64), d_c=D, d_n=D, merge="max", root=True, M=M)
        og, odxc, odxn = O.layer_bwd(G, Wo, T, dyc, dyn, need_dx=True)
        errs = {kk: row_err(to_np(grads[kk]), og[kk]) for kk in og}
        print(mode, flags, "dxc", row_err(to_np(dxc), odxc), "dxn", row_err(to_np(dxn), odxn),
              {kk: f"{e:.1e}" for kk, e in errs.items()}, flush=True)
