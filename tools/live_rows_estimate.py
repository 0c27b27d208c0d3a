"""Executed fraction of the hidden-layer K loops under live-row masks
(Cfg::LIVE, dense threshold SPK_LIVE_DENSE = 28) for the depth-18 level of C2:
FP64 affine-fixed emulation in NumPy (the FP32 kernel's activation pattern
differs only on boxes within rounding of a ReLU kink), sibling pairs = box
groups, 32-row tiles.

    python tools/live_rows_estimate.py
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2202_02444_b200 import synth  # noqa: E402
from paper_2202_02444_b200.network import DenseLayer  # noqa: E402

DENSE = 28


def main(n_pairs=20000, seed=0):
    net = synth.config_net("C2")
    layers = [l for l in net.layers if isinstance(l, DenseLayer)]
    h = 1 / 64
    rng = np.random.default_rng(seed)
    # sibling pairs of the depth-18 level: z-neighbour cubes of side 1/32
    ij = rng.integers(0, 64, size=(n_pairs, 2))
    kz = rng.integers(0, 32, size=n_pairs) * 2
    lo = -1 + np.stack([np.repeat(ij[:, 0], 2), np.repeat(ij[:, 1], 2), np.stack([kz, kz + 1], 1).ravel()], 1) * 2 * h
    base = lo + h
    n = base.shape[0]
    A = np.zeros((n, 3, 3))
    A[:, 0, 0] = A[:, 1, 1] = A[:, 2, 2] = h
    e = np.zeros((n, 3))
    executed, dense_total = [], []
    live = None
    for li, L in enumerate(layers[:-1]):
        m_in = L.weights.shape[1]
        if live is None:  # first layer: every row
            executed.append(m_in)
        else:
            tiles = live.reshape(n_pairs, -1, 32)
            cnt = tiles.sum(2)
            executed.append(float(np.where(cnt > DENSE, 32, cnt).sum(1).mean()))
        dense_total.append(m_in)
        base = base @ L.weights.T + L.bias
        A = A @ L.weights.T
        e = e @ np.abs(L.weights).T
        r = np.abs(A).sum(1) + e
        lo_, hi_ = base - r, base + r
        off, on = hi_ <= 0, lo_ >= 0
        mix = ~(off | on)
        a = np.where(on, 1.0, np.where(off, 0.0, hi_ / np.where(mix, hi_ - lo_, 1)))
        b = np.where(mix, -a * lo_ / 2, 0)
        base, A, e = a * base + b, A * a[:, None, :], a * e + b
        live = (~off).reshape(n_pairs, 2, -1).any(1)
    hidden = slice(1, None)
    frac = sum(executed[hidden]) / sum(dense_total[hidden])
    m = [l.weights.shape for l in layers]
    macs_dense = sum(o * i for o, i in m)
    macs_exec = sum(o * ex for (o, i), ex in zip(m[:-1], executed)) + m[-1][0] * m[-1][1]
    print(json.dumps({"per_layer_executed_rows": executed, "hidden_executed_fraction": frac,
                      "executed_fraction_of_all_macs": macs_exec / macs_dense, "pairs": n_pairs}))


if __name__ == "__main__":
    main()
