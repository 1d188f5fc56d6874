"""Bit-exact cluster / block trees (hmatrix.py:38-211, 814-826) computed by
the C++ partitioner in libhbem_b200.so.

The objects mirror the reference's (`ClusterNode`, `ClusterTree`,
`BlockLeaf`, `BlockClusterTree`) attribute for attribute, but are backed by
flat arrays (``perm``, ``node_array`` (n,5), ``leaf_array`` (L,3)) that the
device assembler consumes directly; per-node/per-leaf Python objects are
materialised lazily.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction
from functools import cached_property

import numpy as np

from . import _lib
from ._lib import check, lib
from .errors import ConfigError

DEFAULT_N_MIN = 32
DEFAULT_ETA = 2.0


def _detect_norm_mode() -> int:
    """Which float64 evaluation np.linalg.norm uses for a 3-vector on this
    host (BLAS ddot with or without FMA).  0: sqrt((x*x + y*y) + z*z),
    1: sqrt(fma(z, z, fma(y, y, x*x)))."""
    rng = np.random.default_rng(7)
    xs = rng.standard_normal((400, 3)) * np.exp(rng.standard_normal((400, 1)))
    ok = [True, True]
    for v in xs:
        ref = float(np.linalg.norm(v))
        x, y, z = (float(t) for t in v)
        plain = float(np.sqrt((x * x + y * y) + z * z))
        xx = x * x
        f1 = float(Fraction(y) * Fraction(y) + Fraction(xx))
        f2 = float(Fraction(z) * Fraction(z) + Fraction(f1))
        fm = float(np.sqrt(f2))
        ok[0] &= ref == plain
        ok[1] &= ref == fm
    if ok[1] and not ok[0]:
        return 1
    if ok[0]:
        return 0
    raise ConfigError("cannot reproduce numpy's 3-vector norm bit-exactly on this host")


NORM_MODE = _detect_norm_mode()


@dataclass(frozen=True)
class ClusterNode:
    start: int
    stop: int
    level: int
    bbox_min: np.ndarray
    bbox_max: np.ndarray
    left: int = -1
    right: int = -1

    @property
    def is_leaf(self) -> bool:
        return self.left < 0

    @property
    def size(self) -> int:
        return self.stop - self.start


class ClusterTree:
    """Same fields as the reference ClusterTree (hmatrix.py:72-102)."""

    def __init__(self, permutation, node_array, bbox, n_min, handle=None):
        self.permutation = permutation
        self.permutation.setflags(write=False)
        self.node_array = node_array  # (n_nodes, 5) start, stop, level, left, right
        self.bbox = bbox              # (n_nodes, 6)
        self.n_min = n_min
        self._handle = handle

    @cached_property
    def nodes(self) -> tuple:
        na, bb = self.node_array, self.bbox
        return tuple(ClusterNode(int(r[0]), int(r[1]), int(r[2]), bb[i, :3].copy(),
                                 bb[i, 3:].copy(), int(r[3]), int(r[4]))
                     for i, r in enumerate(na))

    @property
    def n_dofs(self) -> int:
        return len(self.permutation)

    @property
    def root(self):
        return self.nodes[0]

    def leaves(self) -> list:
        return [int(i) for i in np.nonzero(self.node_array[:, 3] < 0)[0]]

    def inverse_permutation(self) -> np.ndarray:
        inv = np.empty_like(self.permutation)
        inv[self.permutation] = np.arange(len(self.permutation))
        return inv

    def __del__(self):
        if getattr(self, "_handle", None):
            lib.hbem_tree_destroy(self._handle)
            self._handle = None


@dataclass(frozen=True)
class BlockLeaf:
    row_node: int
    col_node: int
    admissible: bool


class BlockClusterTree:
    """Same fields as the reference BlockClusterTree (hmatrix.py:157-171)."""

    def __init__(self, rows: ClusterTree, cols: ClusterTree, eta: float, leaf_array):
        self.rows = rows
        self.cols = cols
        self.eta = float(eta)
        self.leaf_array = leaf_array  # (L, 3) row_node, col_node, admissible

    @cached_property
    def leaves(self) -> tuple:
        return tuple(BlockLeaf(int(r), int(c), bool(a)) for r, c, a in self.leaf_array)

    @property
    def shape(self) -> tuple[int, int]:
        return self.rows.n_dofs, self.cols.n_dofs

    def leaf_shape(self, leaf) -> tuple[int, int]:
        r = self.rows.node_array[leaf.row_node]
        c = self.cols.node_array[leaf.col_node]
        return int(r[1] - r[0]), int(c[1] - c[0])


def build_cluster_tree(points: np.ndarray, n_min: int = DEFAULT_N_MIN) -> ClusterTree:
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ConfigError(f"points must have shape (n, 3), got {pts.shape}")
    h = C.c_void_p()
    check(lib.hbem_cluster_tree(_lib.ptr(pts, C.c_double), len(pts), int(n_min), C.byref(h)))
    n, nn = C.c_int64(), C.c_int64()
    check(lib.hbem_tree_size(h, C.byref(n), C.byref(nn)))
    perm = np.empty(n.value, np.int64)
    nodes = np.empty((nn.value, 5), np.int64)
    bbox = np.empty((nn.value, 6), np.float64)
    check(lib.hbem_tree_copy(h, _lib.ptr(perm, C.c_int64), _lib.ptr(nodes, C.c_int64),
                             _lib.ptr(bbox, C.c_double)))
    return ClusterTree(perm, nodes, bbox, n_min, handle=h)


def build_block_tree(rows: ClusterTree, cols: ClusterTree,
                     eta: float = DEFAULT_ETA) -> BlockClusterTree:
    if eta < 0.0:
        raise ConfigError(f"eta must be >= 0, got {eta}")
    h = C.c_void_p()
    check(lib.hbem_block_tree(rows._handle, cols._handle, float(eta), NORM_MODE, C.byref(h)))
    nl = C.c_int64()
    check(lib.hbem_blocks_size(h, C.byref(nl)))
    leaves = np.empty((nl.value, 3), np.int64)
    check(lib.hbem_blocks_copy(h, _lib.ptr(leaves, C.c_int64)))
    lib.hbem_blocks_destroy(h)
    return BlockClusterTree(rows, cols, eta, leaves)


def cluster_trees_for(test_space, trial_space, n_min: int = DEFAULT_N_MIN,
                      eta: float = DEFAULT_ETA) -> BlockClusterTree:
    """hmatrix.py:814-826."""
    rows = build_cluster_tree(test_space.dof_centers, n_min)
    cols = rows if trial_space is test_space else build_cluster_tree(trial_space.dof_centers,
                                                                       n_min)
    return build_block_tree(rows, cols, eta)
