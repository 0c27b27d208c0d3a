"""CPU-side checks of the C-ABI boundary: the in-tree library loads and
exports every entry point include/spelunk_b200.h declares; network upload
validation maps onto the reference's exceptions.  No kernels run here."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2202_02444_b200 import _lib, errors
from paper_2202_02444_b200.network import DeviceNet, NetworkSpec, DenseLayer, load_network

HEADER = Path(__file__).resolve().parents[1] / "include" / "spelunk_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(spk_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name


def test_bindings_cover_header():
    assert set(declared_functions()) <= set(_lib.SIGNATURES)


def test_net_create_validates(net_paths):
    lib = _lib.load()
    dn = DeviceNet(load_network(net_paths["relu4x32"]), 0)
    assert dn.max_width == 32 and dn.n_dense == 5 and dn.macs == 3 * 32 + 3 * 32 * 32 + 32
    # final width must be 1 (network.py:106-107)
    bad = np.zeros((2, 3))
    import ctypes as C

    kinds = np.array([_lib.OP_DENSE], np.int32)
    outs = np.array([2], np.int32)
    params = np.zeros(8)
    h = C.c_void_p()
    st = lib.spk_net_create(3, 1, kinds.ctypes.data, outs.ctypes.data, params.ctypes.data, 8, 0, C.byref(h))
    assert st == _lib.ERR_DIM
    with pytest.raises(errors.DimensionMismatch):
        _lib.check(st)


def test_width_limit_reported():
    net = NetworkSpec(3, (DenseLayer(np.zeros((600, 3)), np.zeros(600)), DenseLayer(np.zeros((1, 600)), np.zeros(1))))
    with pytest.raises(errors.DeviceError):
        DeviceNet(net, 0)


def test_single_form_bookkeeping():
    """condense / truncate / interval_of / box_to_affine semantics
    (range_core.py:369-464); pure bookkeeping, no device needed."""
    import numpy as np

    import paper_2202_02444_b200 as sp

    a = sp.AffineForm(np.array([1.0, -2.0]), np.array([[3.0, -1.0, 0.5], [0.0, 2.0, -2.0]]), np.array([0.1, 0.0]))
    iv = sp.interval_of(a)
    np.testing.assert_allclose(iv.lo, [1 - 4.6, -2 - 4.0])
    c = sp.condense(a, [1])
    assert c.n_symbols == 2 and np.allclose(c.err, [1.1, 2.0])
    np.testing.assert_allclose(sp.interval_of(c).lo, iv.lo)          # condense keeps the interval
    t = sp.truncate(a, 2)  # norms 3, 3, 2.5 -> ties keep the lower index: columns 0, 1
    np.testing.assert_array_equal(t.coeffs, a.coeffs[:, :2])
    box = sp.QueryBox(np.zeros(3), np.diag([0.1, 0.2, 0.3]))
    f = sp.box_to_affine(box)
    assert f.n_symbols == 3 and np.allclose(f.coeffs, np.diag([0.1, 0.2, 0.3]))
    with pytest.raises(sp.errors.IndexOutOfRange):
        sp.condense(a, [5])
    with pytest.raises(sp.errors.InvalidParameter):
        sp.truncate(a, 0)


def test_refine_band_setting_is_host_only():
    """spk_refine_band (the fp32-refine band override) is host state: set,
    query, reset to per-net calibration, and validation -- no device needed."""
    import paper_2202_02444_b200 as sp
    from paper_2202_02444_b200.network import _precision_code

    assert _precision_code("fp32-refine") == _lib.FP32_REFINE == 2
    prev = sp.refine_band()
    try:
        sp.refine_band(0.01)
        assert sp.refine_band() == 0.01
        assert sp.refine_band("auto") == 0.01
        assert sp.refine_band() == -1.0  # per-net calibration
        for bad in (float("nan"), float("inf"), -0.5):
            with pytest.raises(errors.InvalidParameter):
                sp.refine_band(bad)
        with pytest.raises(errors.InvalidParameter):
            sp.refine_band("sometimes")
    finally:
        if prev >= 0:
            sp.refine_band(prev)
        else:
            sp.refine_band("auto")
