"""The host-array entry point (spk_bound_batch_host, the reference's
range_bound_batch contract with NumPy in / out) under the reference's calling
pattern: 4096-box chunks (spatial.py:38) from ThreadPoolExecutor workers
(rays.py:170-181, render.py:116-127).  Per-thread staging is cached, so
concurrent callers neither share buffers nor serialise on allocation; the
results must be bit-identical to serial calls."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2202_02444_b200 as sp
from paper_2202_02444_b200 import synth

pytestmark = pytest.mark.gpu


def _boxes(seed, n):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-1, 1, (n, 3))
    a = np.zeros((n, 3, 3))
    a[:, np.arange(3), np.arange(3)] = 10.0 ** rng.uniform(-3, -1, (n, 1))
    return c, a


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_concurrent_host_calls_match_serial(net_paths, precision):
    nets = [sp.load_network(net_paths["relu_sdf"]), sp.load_network(net_paths["elu_sdf"]),
            synth.config_net("C5_64"), sp.load_network(net_paths["sin3x48"])]
    jobs = []
    for j in range(32):
        c, a = _boxes(j, 4096 if j % 4 else 1000 + 37 * j)
        jobs.append((nets[j % len(nets)], c, a, ["affine-fixed", "interval", "affine-truncate:8"][j % 3]))
    serial = [sp.range_bound_batch(n, c, a, p, precision=precision) for n, c, a, p in jobs]

    def run(k):
        n, c, a, p = jobs[k]
        return sp.range_bound_batch(n, c, a, p, precision=precision)

    for _ in range(3):
        with ThreadPoolExecutor(max_workers=8) as pool:
            got = list(pool.map(run, range(len(jobs))))
        for (l0, h0), (l1, h1) in zip(serial, got):
            np.testing.assert_array_equal(l0, l1)
            np.testing.assert_array_equal(h0, h1)


def test_host_call_sizes_and_reuse(net_paths):
    """Growing and shrinking batches through the cached staging (incl. the
    two-slot pipeline past 1M boxes and an empty call)."""
    net = sp.load_network(net_paths["relu4x32"])
    for n in (1, 4096, 0, 70_000, 3, (1 << 20) + 5000, 4096):
        c, a = _boxes(n, n)
        lo, hi = sp.range_bound_batch(net, c, a, "affine-fixed")
        assert lo.shape == (n,)
        if n:
            k = np.random.default_rng(n).choice(n, size=min(n, 512), replace=False)
            l2, h2 = sp.range_bound_batch(net, c[k], a[k], "affine-fixed")
            np.testing.assert_array_equal(lo[k], l2)
            np.testing.assert_array_equal(hi[k], h2)
