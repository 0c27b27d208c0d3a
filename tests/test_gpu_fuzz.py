"""GPU soundness fuzz at the reference's acceptance scale
(test_acceptance.py:49-59, fuzz_soundness bench.py:228-319): 10^6 regions
(random centres in [-1.1, 1.1]^3, log-uniform sizes in [1e-4, 1], half 1-D
random-direction segments, half axis-aligned cubes) per policy, 32 samples
each, evaluated by the FP64 GPU point kernel (matches the reference's
eval_batch to 1e-12).  The reference allows slack 1e-5; the FP32 sound
kernels must show ZERO escapes with slack 1e-9 (FP64 evaluation noise).
"""

import numpy as np
import pytest
import torch

import paper_2202_02444_b200 as sp

pytestmark = pytest.mark.gpu
N_REGIONS = 1_000_000
SAMPLES = 32


def regions(rng, n, dev):
    c = torch.from_numpy(rng.uniform(-1.1, 1.1, (n, 3))).to(dev)
    sizes = torch.from_numpy(10.0 ** rng.uniform(-4.0, 0.0, n)).to(dev)
    one_d = torch.from_numpy(rng.random(n) < 0.5).to(dev)
    dirs = torch.from_numpy(rng.standard_normal((n, 3))).to(dev)
    dirs = dirs / dirs.norm(dim=1, keepdim=True)
    axes = torch.zeros((n, 3, 3), dtype=torch.float64, device=dev)
    idx = torch.arange(3, device=dev)
    axes[:, idx, idx] = (sizes / 2.0)[:, None]
    axes[one_d] = 0.0
    axes[one_d, 0, :] = (sizes[one_d, None] / 2.0) * dirs[one_d]
    return c, axes


@pytest.mark.parametrize("netname", ["relu_sdf", "elu_sdf", "box", "sin12", "tanh12"])
def test_million_region_fuzz(net_paths, netname):
    net = sp.load_network(net_paths[netname])
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(2024)
    policies = ["interval", "affine-fixed", "affine-truncate:16"]
    if netname in ("box", "sin12", "tanh12"):
        policies.append("affine-full")
    chunk = 250_000
    checks = 0
    for start in range(0, N_REGIONS, chunk):
        c, a = regions(rng, chunk, dev)
        eps = torch.from_numpy(rng.uniform(-1.0, 1.0, (chunk, SAMPLES, 3))).to(dev)
        pts = c[:, None, :] + torch.einsum("nks,nsd->nkd", eps, a)
        vals = sp.eval_batch(net, pts.reshape(-1, 3), precision="fp64").reshape(chunk, SAMPLES)
        for pol in policies:
            lo, hi = sp.range_bound_batch(net, c, a, pol, precision="fp32")
            slack = 1e-9 * torch.clamp(torch.maximum(lo.abs(), hi.abs()), min=1.0)
            bad = (vals < (lo - slack)[:, None]) | (vals > (hi + slack)[:, None])
            n_bad = int(bad.any(dim=1).sum().item())
            assert n_bad == 0, (netname, pol, n_bad)
            checks += chunk
    assert checks == N_REGIONS * len(policies)


def test_corrupted_rule_detected(net_paths):
    """Mutation test (reference test_cli.py:150-164): with the ReLU affine
    remainder negated the bounds stop enclosing the range and the reference
    fuzz harness (fuzz_soundness, FP32 production kernels) must report
    violations; restored, the same regions pass.  A private copy of the net
    carries the corrupted device program."""
    import copy

    from paper_2202_02444_b200.network import device_net

    net = copy.deepcopy(sp.load_network(net_paths["box"]))
    dn = device_net(net)
    dn.debug_corrupt_relu(True)
    try:
        report = sp.fuzz_soundness([net], n_regions=3000, rng_seed=0, policies=[sp.AFFINE_FIXED])
        assert not report.ok
        assert report.violations
        first = report.violations[0]
        assert first.value < first.lo or first.value > first.hi
    finally:
        dn.debug_corrupt_relu(False)
    report = sp.fuzz_soundness([net], n_regions=3000, rng_seed=0, policies=[sp.AFFINE_FIXED])
    assert report.ok and report.n_violations == 0
