"""Shared parity helpers: tolerance rule and input recipes."""
from __future__ import annotations

import numpy as np

# north_star: derivative values within 1e-12 relative in fp64.
#
# The generated code repeats the reference's roundings operation for operation
# (tests/test_codegen_hostexec.py proves it bit for bit on the host with
# glibc), so device results differ from the reference only through libdevice
# vs glibc transcendentals (<= 2 ulp). Entries that are the result of
# catastrophic cancellation inherit those ulps at O(eps * terms) absolute size,
# so a 1-ulp change of sin/cos/exp moves them far more than 1e-12 relative.
#
# Each entry is compared relative to max(|ref|, floor * max|ref array|) with a
# PER-MODEL floor. The floor is zero (pure per-entry relative error) unless a
# measurement shows cancellation; then it is sized from that measurement
# (scripts/parity_probe.py at the benchmarked N, profiles/r2_parity_probe.jsonl,
# acceptance recipe, no floor):
#   goddard       max 2.0e-15 per entry                       -> no floor
#   hang_glider   max 3.3e-13 per entry                       -> no floor
#   double_integr. linear/quadratic, exact                    -> no floor
#   quadrotor     J/H/grad entries down to ~1e-9 of max cancel (sin/cos
#                 products of the attitude); with a floor of 1e-6 the worst
#                 entry still has 1.1e-11 relative error, i.e. |err| / max =
#                 1.1e-17 (hess, N=1e6, r2_v3 GPU run)  -> needs floor >= 1.1e-5
#                                                                    -> 1e-4
#   shuttle       H entries down to 1e-24 of max; the entry with the largest
#                 ABSOLUTE error has |err| / max = 8.7e-17 (N=1e5, r2_v1
#                 GPU run) -> needs floor >= 8.7e-5                    -> 1e-4
#   cart_pendulum H entries ~1e-6 of max: worst |err| / max = 3.3e-17
#                 -> needs floor >= 3.3e-5                             -> 1e-4
REL_TOL = 1e-12
CANCELLING = {"quadrotor": 1e-4, "shuttle": 1e-4, "cart_pendulum": 1e-4}
# default for callers that do not name a model (scaled / synthetic cases)
FLOOR = 1e-4


def floor_for(model: str) -> float:
    """The tolerance floor of `model` (0.0: plain per-entry relative error)."""
    for k, v in CANCELLING.items():
        if model.startswith(k):
            return v
    return 0.0


def rel_errors(got: np.ndarray, ref: np.ndarray, floor: float = FLOOR) -> np.ndarray:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return np.zeros(0)
    scale = np.max(np.abs(ref))
    denom = np.maximum(np.abs(ref), floor * scale)
    denom = np.where(denom == 0.0, 1.0, denom)
    return np.abs(got - ref) / denom


def assert_close(got, ref, what: str, tol: float = REL_TOL, floor: float | None = None,
                 model: str | None = None) -> dict:
    """|got - ref| <= tol * max(|ref|, floor * max|ref|) entry by entry; the
    floor is the model's (floor_for) unless given explicitly, and 0.0 when
    neither is named."""
    if floor is None:
        floor = floor_for(model) if model else 0.0
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} vs {ref.shape}"
    err = rel_errors(got, ref, floor)
    worst = float(err.max()) if err.size else 0.0
    exact = float(np.mean(got == ref)) if ref.size else 1.0
    assert worst <= tol, f"{what}: max rel err {worst:.3e} > {tol:.0e} (floor {floor:g}, bit-exact fraction {exact:.4f})"
    return {"max_rel": worst, "bit_exact": exact, "floor": floor}
