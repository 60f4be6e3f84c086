"""Shared helpers of the GPU parity tests (test-side only)."""
import numpy as np

TOL = 1e-4          # north_star: max relative error normalised by the row L2 norm


def row_err(gpu, ref):
    """max_r max_d |g - o| / max(||o_r||_2, tau), tau = 1e-6 * RMS row norm
    (SURVEY §8(c) parity protocol)."""
    g = np.asarray(gpu, dtype=np.float64)
    o = np.asarray(ref, dtype=np.float64)
    if o.ndim == 1:
        o = o[None, :]
        g = g[None, :]
    if o.size == 0:
        return 0.0
    norms = np.linalg.norm(o, axis=1)
    rms = float(np.sqrt(np.mean(norms ** 2))) if norms.size else 0.0
    tau = max(1e-6 * rms, 1e-30)
    den = np.maximum(norms, tau)
    return float((np.abs(g - o).max(axis=1) / den).max())


def to_np(t):
    return t.detach().cpu().numpy()
