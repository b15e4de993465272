"""Compare a GPU primal/dual iterate with a reference iterate fixture.

The fixtures (tests/golden/iterates_*.npz, make_golden.py) hold the final
Iterate of a reference solve (model.hpp:41-55): whole arrays for small
problems, or -- for the pegase configs -- per-scenario inf-norms, a +-1
projection checksum per scenario and the full rows of a few sample scenarios.

North-star tolerance: iterates within 1e-6 relative.  Per array the scale is
max(1, max|ref|) (multipliers of inactive bounds sit near mu and are compared
against the array's scale, not their own tiny magnitude).
"""
import numpy as np

NAMES = ("x", "u", "s", "y", "z", "kappa_lo", "kappa_up", "nu_lo", "nu_up", "lambda_lo",
         "lambda_up")
REL = 1e-6


def projection_signs(n: int) -> np.ndarray:
    """Same weights as tests/golden/make_golden.py."""
    return np.where(np.random.default_rng(12345).random(n) < 0.5, -1.0, 1.0)


def compare(gpu: dict, ref, rel: float = REL) -> dict:
    """Returns {name: worst relative error}; asserts every one <= rel."""
    worst = {}
    for k in NAMES:
        g = np.asarray(gpu[k])
        if k in ref.files:
            r = ref[k]
            scale = max(1.0, float(np.abs(r).max(initial=0.0)))
            err = float(np.abs(g - r).max(initial=0.0)) / scale
        else:
            rows = ref[k + "__rows"]
            scale = max(1.0, float(ref[k + "__absmax"].max(initial=0.0)))
            err = float(np.abs(g[rows] - ref[k + "__sample"]).max(initial=0.0)) / scale
            err = max(err, float(np.abs(np.abs(g).max(axis=1) - ref[k + "__absmax"]).max()) / scale)
            w = projection_signs(g.shape[1])
            # a checksum of n entries each within rel * scale moves by <= n rel scale
            proj_err = np.abs(g @ w - ref[k + "__proj"]) / (g.shape[1] * scale)
            err = max(err, float(proj_err.max(initial=0.0)))
        worst[k] = err
    bad = {k: v for k, v in worst.items() if not v <= rel}
    assert not bad, f"iterate differs from the reference beyond {rel}: {bad}"
    return worst
