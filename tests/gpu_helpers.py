"""Shared helpers of the -m gpu parity tests (compare the CUDA path with the oracle)."""
import numpy as np

FIELDS = ("pF", "pf", "pm", "u", "p")


def rel_l2(x, ref):
    """C20: ||x - ref||_2 / ||ref||_2 per field; if ||ref|| = 0 return max |x| (must be <= 1e-14)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    n = np.linalg.norm(ref)
    if n == 0.0:
        return float(np.max(np.abs(x))) if x.size else 0.0
    return float(np.linalg.norm(x - ref) / n)


def compare(gpu: dict, ora: dict, tol: float = 1e-9):
    errs = {f: rel_l2(gpu[f], ora[f]) for f in FIELDS}
    bad = {f: e for f, e in errs.items() if not e <= tol}
    return errs, bad
