"""GPU batched AD (subsystem 1) against the reference's derivative bundle.

Values and first derivatives (f, g, h, G_x, G_u, H_x, H_u) replay the
reference's operation order without FMA contraction and must match it to the
last bit or two; the Lagrangian Hessian blocks and gradient are analytic
(the reference's are forward-over-reverse) and must match to 1e-12 relative.
"""
import numpy as np
import pytest

from conftest import case_path
from paper_2301_04869_b200 import _native as nat

pytestmark = pytest.mark.gpu

FIRST = ("f", "g", "h", "gx", "gu", "hx", "hu")
SECOND = ("wxx", "wxu", "wuu", "grad_lag")


@pytest.mark.parametrize("name", ["case9_N8_s005_it3", "case118_N4_s005_it5",
                                  "case118_N4_s005_it20"])
def test_bundle_matches_reference(goldens, name):
    fx = goldens[name]
    m = fx.meta
    p = nat.Problem(case_path(m["case"]), m["N"], m["sigma"], m["seed"])
    ctx = nat.Context(p)
    out = ctx.eval_bundle(fx["it_x"], fx["it_u"], fx["it_y"], fx["it_z"], 1.0)
    for k in FIRST + SECOND:
        ref = fx[k].reshape(out[k].shape)
        scale = max(1.0, np.abs(ref).max())
        tol = 4e-16 if k in FIRST else 1e-12
        err = np.abs(out[k] - ref).max() / scale
        assert err <= tol, f"{name}: {k} rel err {err:.3e}"
    f, g, h = ctx.eval_values(fx["it_x"], fx["it_u"])
    assert np.array_equal(f, out["f"]) and np.array_equal(g, out["g"]) and \
        np.array_equal(h, out["h"])


def test_nonfinite_input_reports_block(goldens):
    fx = goldens["case118_N4_s005_it5"]
    m = fx.meta
    p = nat.Problem(case_path(m["case"]), m["N"], m["sigma"], m["seed"])
    ctx = nat.Context(p)
    X = fx["it_x"].copy()
    X[1, 0] = np.nan
    X[3, 0] = np.inf
    with pytest.raises(nat.NonFiniteError) as e:
        ctx.eval_bundle(X, fx["it_u"], fx["it_y"], fx["it_z"])
    assert "block 1" in str(e.value)
