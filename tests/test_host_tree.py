"""Host-side tree objects (CPU): the lazy TreeNode view of the level arrays
(`spatial.materialize`) equals the eagerly built tree node for node, with
the oracle's levels standing in for a device build."""

import numpy as np

from oracle import spelunk_oracle as orc
from paper_2202_02444_b200.spatial import TreeArrays, TreeLevel, TreeNode, iter_leaves, materialize

NET = "tests/golden/nets/relu_sdf.json"


def _arrays(depth=8):
    net = orc.load_net(NET)
    lv = orc.tree_levels(net, -np.ones(3), np.ones(3), "affine-fixed", max_depth=depth)
    return TreeArrays([TreeLevel(l["lo"], l["hi"], np.zeros(len(l["label"])), np.zeros(len(l["label"])),
                                 l["label"], l["face"], l["parent"]) for l in lv], 0)


def _walk(node):
    out = []
    stack = [node]
    while stack:
        n = stack.pop()
        out.append((tuple(n.aabb.lo), tuple(n.aabb.hi), n.sign, n.depth, n.face_sign, n.is_leaf))
        if n.children:
            stack.extend(n.children)
    return out


def test_lazy_tree_equals_eager():
    arr = _arrays()
    eager = materialize(arr, lazy=False)
    lazy = materialize(arr, lazy=True)
    assert isinstance(lazy, TreeNode)
    assert _walk(lazy) == _walk(eager)
    assert len(list(iter_leaves(lazy))) == len(list(iter_leaves(eager)))
    # children can be replaced like on a plain dataclass node
    lazy.children = None
    assert lazy.is_leaf
