"""Single-form definitional operations (range_core.py:369-464) composed
through whole networks equal the reference's batched bounds -- the
reference's own batch-vs-composition check (test_range_core.py:286-304, 1e-12
there; here 1e-9 relative: the rules come from the device rule code, whose
FP64 transcendentals carry a few-ulp pad)."""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from paper_2202_02444_b200.network import ActivationKind, DenseLayer

pytestmark = pytest.mark.gpu


def compose(net, center, axes, policy):
    form = sp.box_to_affine(sp.QueryBox(center, axes))
    for layer in net.layers:
        if isinstance(layer, DenseLayer):
            form = sp.affine_linear(form, layer)
        elif layer is not ActivationKind.IDENTITY:
            form = sp.affine_nonlinear(form, layer, policy)
    iv = sp.interval_of(form)
    return float(iv.lo[0]), float(iv.hi[0])


@pytest.mark.parametrize("netname", ["box", "relu12", "elu12", "sin12", "tanh12"])
@pytest.mark.parametrize("policy", ["affine-fixed", "affine-full", "affine-truncate:8"])
def test_composition_equals_reference_batch(golden, net_paths, netname, policy):
    net = sp.load_network(net_paths[netname])
    c, a = golden[f"bounds/{netname}/centers"], golden[f"bounds/{netname}/axes"]
    wl, wh = golden[f"bounds/{netname}/{policy}/lo"], golden[f"bounds/{netname}/{policy}/hi"]
    pol = sp.parse_policy(policy)
    for i in range(0, len(c), 7):
        ax = a[i][np.any(a[i] != 0.0, axis=1)]
        lo, hi = compose(net, c[i], ax, pol)
        s = max(1.0, abs(wl[i]), abs(wh[i]))
        assert abs(lo - wl[i]) <= 1e-9 * s and abs(hi - wh[i]) <= 1e-9 * s, (i, lo, wl[i], hi, wh[i])


def test_affine_rule_matches_reference_rules(golden):
    lo, hi = golden["rules/lo"], golden["rules/hi"]
    for kind in ("relu", "elu", "sin", "tanh"):
        a, b, g = sp.affine_rule(kind, lo, hi)
        wa, wb, wg = golden[f"rules/{kind}/alpha"], golden[f"rules/{kind}/beta"], golden[f"rules/{kind}/gamma"]
        # [0, 0] for ReLU: any subgradient is exact (the reference takes 0, the
        # device rule 1); both give alpha*0 + beta = 0 with gamma = 0
        zero = (lo == 0.0) & (hi == 0.0)
        ok = np.isfinite(wa) & ~(zero if kind == "relu" else np.zeros_like(zero))
        np.testing.assert_allclose(a[ok], wa[ok], rtol=1e-12, atol=1e-12)
        if kind == "relu":
            assert np.all((b[zero] == 0.0) & (g[zero] == 0.0))
        # sound: gamma never smaller than the reference's (pads only widen)
        assert np.all(g[ok] >= wg[ok] - 1e-15 * np.maximum(1.0, np.abs(wg[ok])))
    with pytest.raises(sp.errors.UnsupportedActivation):
        sp.affine_rule("softplus", lo, hi)
