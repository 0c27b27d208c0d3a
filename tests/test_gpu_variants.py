"""§8(f4): device fuzz_soundness and bench_variants vs the reference.

bench_variants: with FP64 kernels the bound-able region sizes (binary search
over the reference's size grid, the reference's regions) equal the
reference's (golden, make_golden.py:gen_variants); timings are measured, not
compared.  fuzz_soundness: the reference's report (regions, checks, zero
violations) for the same seed, with the production FP32 kernels; and it
detects a deliberately broken bound.
"""

import numpy as np
import pytest

import paper_2202_02444_b200 as sp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nets(net_paths):
    return {k: sp.load_network(p) for k, p in net_paths.items()}


def test_bench_variants_region_sizes(golden, nets, tmp_path):
    rows = sp.bench_variants([nets["relu_sdf"], nets["elu_sdf"]], n_regions=2000, rng_seed=0, raycast_res=16,
                             runs=1, precision="fp64")
    assert [r.variant for r in rows] == ["interval", "interval", "affine-fixed", "affine-fixed", "affine-full",
                                         "affine-full", "affine-truncate:16", "affine-truncate:16"]
    np.testing.assert_array_equal([r.dim for r in rows], golden["variants/dim"])
    np.testing.assert_array_equal([r.region_size for r in rows], golden["variants/region_size"])
    assert all(r.time_ratio > 0 and r.raycast_seconds > 0 for r in rows)
    from paper_2202_02444_b200.bench import write_bench_csv

    write_bench_csv(rows, tmp_path / "b.csv")
    assert (tmp_path / "b.csv").read_text().splitlines()[0] == "variant,dim,time_ratio,region_size,raycast_seconds"


def test_fuzz_matches_reference_report(golden, nets):
    rep = sp.fuzz_soundness([nets["relu_sdf"], nets["sin12"]], n_regions=20_000, rng_seed=3)
    np.testing.assert_array_equal([rep.n_regions, rep.n_checks, rep.n_violations], golden["variants/fuzz"])
    assert rep.ok


def test_fuzz_million_regions_fp32(nets):
    rep = sp.fuzz_soundness([nets["relu_sdf"], nets["elu_sdf"], nets["sin3x48"], nets["tanh12"]],
                            n_regions=1_000_000, rng_seed=0)
    assert rep.n_checks == 4_000_000 and rep.ok, rep.violations[:2]


def test_fuzz_detects_violation(nets, monkeypatch):
    from paper_2202_02444_b200 import bench

    real = bench.range_bound_batch

    def shrunk(net, c, a, pol, precision="fp32"):
        lo, hi = real(net, c, a, pol, precision=precision)
        mid = (lo + hi) / 2
        return mid - 1e-3 * (hi - lo), mid + 1e-3 * (hi - lo)

    monkeypatch.setattr(bench, "range_bound_batch", shrunk)
    rep = sp.fuzz_soundness([nets["relu_sdf"]], n_regions=4096, slack=0.0, max_reported=3)
    assert not rep.ok and len(rep.violations) == 3 and rep.violations[0].policy == "interval"
