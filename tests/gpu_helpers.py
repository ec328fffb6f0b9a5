"""Shared helpers of the -m gpu parity tests (compare the CUDA path with the oracle)."""
import numpy as np

FIELDS = ("pF", "pf", "pm", "u", "p")


def rel_l2(x, ref):
    """C20: ||x - ref||_2 / ||ref||_2 per field.  A reference that is zero up to roundoff (max |ref| <= 1e-13,
    e.g. the velocity of the constant state or the porous pressures of the first injection steps) is compared
    in absolute terms instead: the returned value is max |x - ref| / 1e-5, so that the 1e-9 bar means
    max |x - ref| <= 1e-14.  The switch is at max |ref| <= 1e-13 (ten times the absolute bound's 1e-14), so a
    non-zero field is never compared more loosely than 10% absolute-to-scale; every field the parity tests
    meet is either O(1e-3..10) or exactly 0 / round-off (C16 early injection steps, constant-state velocity)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    ref = np.asarray(ref, dtype=np.float64).ravel()
    if x.size == 0:
        return 0.0
    if np.max(np.abs(ref)) <= 1e-13:
        return float(np.max(np.abs(x - ref)) / 1e-5)
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


def compare(gpu: dict, ora: dict, tol: float = 1e-9):
    errs = {f: rel_l2(gpu[f], ora[f]) for f in FIELDS}
    bad = {f: e for f, e in errs.items() if not e <= tol}
    return errs, bad
