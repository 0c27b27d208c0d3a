"""Synthetic workloads for BASELINE.json's configs.

Random-init networks are written as ordinary NetworkSpec objects (and can be
saved to the reference weight-file schema so the CPU reference loads
bit-identical weights).  Recipes, all seeded with np.random.default_rng:

  ref-normal     W ~ N(0,1)/sqrt(fan_in), b ~ 0.1 N(0,1)   (reference conftest.py:43-61)
  torch-uniform  W, b ~ U(+-1/sqrt(fan_in)) (nn.Linear default), final bias
                 shifted by the median of f over 20,000 U(-1,1)^3 samples so
                 the zero level set crosses the domain
  siren          Sitzmann et al. init (first layer U(+-1/fan_in), later layers
                 U(+-sqrt(6/fan_in)/w0), biases U(+-1/sqrt(fan_in))) with
                 w0 = 30 folded into the FIRST layer's W and b only -- the
                 reference has no w0 parameter -- recentred
                 like torch-uniform

The recentring forward pass below is plain NumPy: it only constructs the
synthetic net (it is not an evaluation path of this package).
"""

from __future__ import annotations

import numpy as np

from .network import ActivationKind, DenseLayer, NetworkSpec

GOLDEN_RATIO_64 = 0x9E3779B97F4A7C15


def _numpy_forward(layers, x):
    for layer in layers:
        if isinstance(layer, DenseLayer):
            x = x @ layer.weights.T + layer.bias
        elif layer is ActivationKind.RELU:
            x = np.maximum(x, 0.0)
        elif layer is ActivationKind.ELU:
            x = np.where(x >= 0.0, x, np.expm1(np.minimum(x, 0.0)))
        elif layer is ActivationKind.SIN:
            x = np.sin(x)
        elif layer is ActivationKind.TANH:
            x = np.tanh(x)
    return x[:, 0]


def _recentre(layers, d):
    xs = np.random.default_rng(0).uniform(-1.0, 1.0, (20_000, d))
    med = float(np.median(_numpy_forward(layers, xs)))
    last = layers[-1]
    layers[-1] = DenseLayer(last.weights, last.bias - med)
    return layers


def random_mlp(width: int, depth: int, activation="relu", recipe="torch-uniform", seed=0,
               input_dim=3, name=None) -> NetworkSpec:
    """3 -> depth x width -> 1 MLP with `activation` after every hidden layer."""
    act = ActivationKind(activation) if isinstance(activation, str) else activation
    rng = np.random.default_rng(seed)
    dims = [input_dim] + [width] * depth + [1]
    layers = []
    w0 = 30.0
    for i in range(len(dims) - 1):
        fan_in, fan_out = dims[i], dims[i + 1]
        if recipe == "ref-normal":
            w = rng.standard_normal((fan_out, fan_in)) / np.sqrt(fan_in)
            b = rng.standard_normal(fan_out) * 0.1
        elif recipe == "torch-uniform":
            k = 1.0 / np.sqrt(fan_in)
            w = rng.uniform(-k, k, (fan_out, fan_in))
            b = rng.uniform(-k, k, fan_out)
        elif recipe == "siren":
            kb = 1.0 / np.sqrt(fan_in)
            if i == 0:
                w = rng.uniform(-1.0 / fan_in, 1.0 / fan_in, (fan_out, fan_in)) * w0
                b = rng.uniform(-kb, kb, fan_out) * w0
            else:
                lim = np.sqrt(6.0 / fan_in) / w0
                w = rng.uniform(-lim, lim, (fan_out, fan_in))
                b = rng.uniform(-kb, kb, fan_out)
        else:
            raise ValueError(f"unknown recipe {recipe!r}")
        layers.append(DenseLayer(w, b))
        if i < len(dims) - 2:
            layers.append(act)
    if recipe in ("torch-uniform", "siren"):
        layers = _recentre(layers, input_dim)
    return NetworkSpec(input_dim, tuple(layers), "sdf",
                       name or f"{recipe}_{activation}_{depth}x{width}_s{seed}")


def trained_net(tag: str = "torus") -> NetworkSpec:
    """A trained 3->8x256->1 ReLU SDF net (the C2 architecture; FP32 weights,
    tools/train_sdf_net.py): a non-degenerate net of the headline shape, whose
    trees certify most of the domain -- the random-init configs certify nothing."""
    from pathlib import Path

    if tag != "torus":
        raise ValueError(tag)
    path = Path(__file__).resolve().parents[1] / "tests" / "golden" / "nets" / "torus_8x256.npz"
    with np.load(path) as z:
        n = len([k for k in z.files if k.startswith("W")])
        layers = []
        for i in range(n):
            layers.append(DenseLayer(z[f"W{i}"].astype(np.float64), z[f"b{i}"].astype(np.float64)))
            if i < n - 1:
                layers.append(ActivationKind.RELU)
    return NetworkSpec(3, tuple(layers), "sdf", "torus_8x256")


# Named configs of BASELINE.json (C1..C5)
def config_net(tag: str, seed: int = 0) -> NetworkSpec:
    if tag == "C1":
        return random_mlp(32, 4, "relu", "torch-uniform", seed, name="C1_relu_4x32")
    if tag in ("C2", "C5_256"):
        return random_mlp(256, 8, "relu", "torch-uniform", seed, name="relu_8x256")
    if tag == "C3":
        return random_mlp(256, 8, "sin", "siren", seed, name="siren_8x256")
    if tag == "C4":
        return random_mlp(512, 8, "elu", "torch-uniform", seed, name="elu_8x512")
    if tag == "C5_64":
        return random_mlp(64, 8, "relu", "torch-uniform", seed, name="relu_8x64")
    if tag == "C5_512":
        return random_mlp(512, 8, "relu", "torch-uniform", seed, name="relu_8x512")
    raise ValueError(tag)


def grid_cubes(res: int = 64, lo: float = -1.0, hi: float = 1.0):
    """C1: res^3 axis-aligned cubes tiling [lo, hi]^3 (centres, axes)."""
    h = (hi - lo) / res / 2.0
    c1 = lo + (np.arange(res) + 0.5) * (2.0 * h)
    g = np.stack(np.meshgrid(c1, c1, c1, indexing="ij"), axis=-1).reshape(-1, 3)
    axes = np.zeros((g.shape[0], 3, 3))
    axes[:, np.arange(3), np.arange(3)] = h
    return g, axes


def random_cube_centres(n: int, seed: int, first_index: int = 0, d: int = 3) -> np.ndarray:
    """Host copy of the on-device C5 stream (spk_kernels.cuh random_coord):
    splitmix64 of seed + golden * (index*d + k + 1), top 53 bits -> [-1, 1)."""
    idx = np.arange(first_index, first_index + n, dtype=np.uint64)
    k = np.arange(d, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + np.uint64(GOLDEN_RATIO_64) * (idx[:, None] * np.uint64(d) + k[None, :] + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0
