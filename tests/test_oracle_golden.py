"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import hbem_oracle as O

KINDS = {"vertex": O.Kind.SHARED_VERTEX, "edge": O.Kind.SHARED_EDGE,
         "identical": O.Kind.IDENTICAL}

COMBOS = [
    (eq, k, op, fam)
    for eq, k in (("laplace", 0.0), ("helmholtz", 2.0))
    for op in ("slp", "dlp", "adlp", "hyps")
    for fam in ("p0", "p1c", "p1d")
    if not (op == "hyps" and fam == "p0")
]


def mesh(level):
    g = golden("meshes")
    return g[f"ico{level}_vertices"], g[f"ico{level}_elements"]


def test_regular_rules_bitwise():
    g = golden("rules")
    for order in (1, 2, 3, 4):
        p, w = O.regular_rule(order)
        assert np.array_equal(p, g[f"reg{order}_points"])
        assert np.array_equal(w, g[f"reg{order}_weights"])


def test_singular_rules_bitwise():
    g = golden("rules")
    for base in (2, 4):
        for name, kind in KINDS.items():
            p, w = O.singular_rule(kind, base)
            assert np.array_equal(p, g[f"sing{base}_{name}_points"])
            assert np.array_equal(w, g[f"sing{base}_{name}_weights"])
            assert abs(w.sum() - 0.25) < 1e-12


@pytest.mark.parametrize("eq,k,op,fam", COMBOS)
@pytest.mark.parametrize("prec", ["double", "single"])
def test_integrate_batch_matches_reference(eq, k, op, fam, prec):
    g = golden("integrals")
    v, e = mesh(2)
    P = O.Problem(O.Spec(eq, op, k, prec), v, e, fam, fam)
    re, im = O.integrate_batch(P, g["regular_pairs"])
    tag = f"{eq}_{op}_{fam}_{prec}"
    ref = g[f"{tag}_re"] if im is None else g[f"{tag}_re"] + 1j * g[f"{tag}_im"]
    got = re if im is None else re + 1j * im
    assert got.dtype == ref.dtype
    scale = np.abs(ref).reshape(len(ref), -1).max(axis=1)[:, None, None]
    err = (np.abs(got - ref) / scale).max()
    assert err <= (1e-14 if prec == "double" else 2e-6), err


@pytest.mark.parametrize("eq,k,op,fam", COMBOS)
def test_local_matrix_touching_matches_reference(eq, k, op, fam):
    g = golden("integrals")
    v, e = mesh(1)
    P = O.Problem(O.Spec(eq, op, k), v, e, fam, fam)
    pairs = g["singular_pairs"]
    ref = g[f"{eq}_{op}_{fam}_double_local"]
    got = np.stack([O.local_matrix(P, int(a), int(b)) for a, b in pairs])
    scale = np.abs(ref).reshape(len(ref), -1).max(axis=1)[:, None, None]
    assert (np.abs(got - ref) / scale).max() <= 1e-13


@pytest.mark.parametrize("name", ["ico3_p0", "ico2_p1c", "ico2_p1d", "geo11_p0", "geo45_p0"])
def test_partition_bitwise(name):
    from paper_1711_01897_b200.meshes import geodesic_sphere
    g = golden("partitions")
    if name.startswith("ico"):
        v, e = mesh(int(name[3]))
    else:
        v, e = geodesic_sphere(int(name[3:5]))
    fam = name.split("_")[1]
    P = O.Problem(O.Spec("laplace", "slp"), v, e, fam, fam)
    tree = O.cluster_tree(P.dof_centers(fam), 32)
    assert np.array_equal(tree.permutation, g[f"{name}_perm"])
    nodes = np.array([[n.start, n.stop, n.level, n.left, n.right] for n in tree.nodes])
    assert np.array_equal(nodes, g[f"{name}_nodes"])
    bbox = np.array([np.concatenate([n.bbox_min, n.bbox_max]) for n in tree.nodes])
    assert np.array_equal(bbox, g[f"{name}_bbox"])
    leaves = np.array(O.block_tree(tree, tree, 2.0), dtype=np.int64)
    assert np.array_equal(leaves, g[f"{name}_leaves"])


@pytest.mark.parametrize("name,fam,eq,op,k", [
    ("ico2_p0_lap_slp", "p0", "laplace", "slp", 0.0),
    ("ico2_p0_lap_slp_e5", "p0", "laplace", "slp", 0.0),
    ("ico2_p0_helm_slp", "p0", "helmholtz", "slp", 2.0),
    ("ico2_p0_lap_dlp", "p0", "laplace", "dlp", 0.0),
    ("ico2_p1c_lap_dlp", "p1c", "laplace", "dlp", 0.0),
])
def test_hmatrix_matches_reference(name, fam, eq, op, k):
    g = golden("hmatrices")
    v, e = mesh(2)
    eps = float(g[f"{name}_eps"][0])
    P = O.Problem(O.Spec(eq, op, k), v, e, fam, fam)
    tree = O.cluster_tree(P.dof_centers(fam), 32)
    leaves = O.block_tree(tree, tree, 2.0)
    asm = O.Assembler(P, tree, tree, leaves, eps)
    payloads = asm.assemble()
    ranks = np.array([p.rank if isinstance(p, O.LowRank) else -1 for p in payloads])
    # same pivots on the same machine: ranks agree exactly
    assert np.array_equal(ranks, g[f"{name}_ranks"])
    for x, hx, dx in zip(g[f"{name}_x"], g[f"{name}_hx"], g[f"{name}_dx"]):
        y = O.hmat_matvec(tree, tree, leaves, payloads, x)
        assert np.linalg.norm(y - hx) <= 1e-12 * np.linalg.norm(hx)
        assert np.linalg.norm(y - dx) <= 10 * eps * np.linalg.norm(dx)
    assert asm.counters["singular_pairs"] == g[f"{name}_counters"][0]


def test_dense_oracle_matches_reference():
    g = golden("hmatrices")
    v, e = mesh(2)
    P = O.Problem(O.Spec("laplace", "slp"), v, e, "p0", "p0")
    A = O.assemble_dense(P)
    ref = g["ico2_p0_lap_slp_dense"]
    assert np.abs(A - ref).max() <= 1e-14 * np.abs(ref).max()
