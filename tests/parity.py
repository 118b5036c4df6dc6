"""Shared parity helpers: tolerance rule and input recipes."""
from __future__ import annotations

import numpy as np

# north_star: derivative values within 1e-12 relative in fp64.
#
# The generated code repeats the reference's roundings operation for operation
# (tests/test_codegen_hostexec.py proves it bit for bit on the host with
# glibc), so device results differ from the reference only through libdevice
# vs glibc transcendentals (<= 2 ulp). Entries that are the result of
# catastrophic cancellation (e.g. the shuttle Hessian's ~1e-17 entries next to
# O(1) ones) inherit those ulps at O(eps * max) absolute size: a 1-ulp change
# of sin/cos/exp alone moves them by ~1e-5 relative (measured on the host).
# Each entry is therefore compared relative to max(|ref|, FLOOR * max|ref|):
# |got - ref| <= 1e-12 * max(|ref|, 1e-4 * max|ref array|).
REL_TOL = 1e-12
FLOOR = 1e-4


def rel_errors(got: np.ndarray, ref: np.ndarray, floor: float = FLOOR) -> np.ndarray:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return np.zeros(0)
    scale = np.max(np.abs(ref))
    denom = np.maximum(np.abs(ref), floor * scale)
    denom = np.where(denom == 0.0, 1.0, denom)
    return np.abs(got - ref) / denom


def assert_close(got, ref, what: str, tol: float = REL_TOL, floor: float = FLOOR) -> dict:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    err = rel_errors(got, ref, floor)
    worst = float(err.max()) if err.size else 0.0
    exact = float(np.mean(got == ref)) if ref.size else 1.0
    assert worst <= tol, f"{what}: max rel err {worst:.3e} > {tol:.0e} (bit-exact fraction {exact:.4f})"
    return {"max_rel": worst, "bit_exact": exact}
