"""Generate golden vectors from the REAL reference package (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports ``hbem`` from ``/root/reference/pkg/src`` (read-only, unmodified) and
writes small ``.npz`` fixtures next to this script.  The fixtures pin the
CPU oracle (``oracle/hbem_oracle.py``) and feed the GPU parity tests on
boxes where ``/root/reference`` does not exist.  Nothing at test/bench run
time imports the reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from hbem.assembly import AssemblyConfig, assemble_dense  # noqa: E402
from hbem.backend import BatchRequest, make_host_backends  # noqa: E402
from hbem.hmatrix import (AcaConfig, LowRankBlock, assemble_hmatrix,  # noqa: E402
                          cluster_trees_for, compression_stats)
from hbem.kernels import OperatorSpec, local_matrix, make_integration_context  # noqa: E402
from hbem.mesh import TriangleMesh, refine_unit_sphere  # noqa: E402
from hbem.quadrature import PairKind, regular_rule, singular_rule  # noqa: E402
from hbem.spaces import build_space  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1711_01897_b200.meshes import geodesic_sphere  # noqa: E402

KINDS = {"vertex": PairKind.SHARED_VERTEX, "edge": PairKind.SHARED_EDGE,
         "identical": PairKind.IDENTICAL}

# (equation, k, operator, family)
COMBOS = [
    (eq, k, op, fam)
    for eq, k in (("laplace", 0.0), ("helmholtz", 2.0))
    for op in ("slp", "dlp", "adlp", "hyps")
    for fam in ("p0", "p1c", "p1d")
    if not (op == "hyps" and fam == "p0")
]


def disjoint_pairs(mesh, n, rng):
    out = []
    conn = mesh.elements
    while len(out) < n:
        cand = rng.integers(0, mesh.n_elements, size=(4 * n, 2))
        ea, eb = conn[cand[:, 0]], conn[cand[:, 1]]
        ok = ~(ea[:, :, None] == eb[:, None, :]).any(axis=(1, 2))
        out.extend(map(tuple, cand[ok]))
    return np.array(out[:n], dtype=np.int64)


def touching_pairs(mesh, elems):
    conn = mesh.elements
    out = []
    for a in elems:
        share = (conn[:, :, None] == conn[a][None, None, :]).any(axis=(1, 2))
        for b in np.nonzero(share)[0]:
            out.append((a, int(b)))
            if a != b:
                out.append((int(b), a))
    return np.array(out, dtype=np.int64)


def tag(eq, op, fam, prec):
    return f"{eq}_{op}_{fam}_{prec}"


def make_rules():
    d = {}
    for order in (1, 2, 3, 4):
        r = regular_rule(order)
        d[f"reg{order}_points"] = r.points
        d[f"reg{order}_weights"] = r.weights
    for base in (2, 4):
        for name, kind in KINDS.items():
            r = singular_rule(kind, base)
            d[f"sing{base}_{name}_points"] = r.points
            d[f"sing{base}_{name}_weights"] = r.weights
    np.savez_compressed(os.path.join(HERE, "rules.npz"), **d)


def make_meshes():
    d = {}
    for level in (0, 1, 2, 3):
        m = refine_unit_sphere(level)
        d[f"ico{level}_vertices"] = m.vertices
        d[f"ico{level}_elements"] = m.elements
    np.savez_compressed(os.path.join(HERE, "meshes.npz"), **d)


def make_integrals():
    """integrate_batch on disjoint pairs and local_matrix on touching pairs,
    every (equation, operator, family, precision), level-2 / level-1 spheres."""
    rng = np.random.default_rng(1234)
    m2 = refine_unit_sphere(2)
    m1 = refine_unit_sphere(1)
    reg_pairs = disjoint_pairs(m2, 64, rng)
    sing_pairs = touching_pairs(m1, [0, 5, 17])
    d = {"regular_pairs": reg_pairs, "singular_pairs": sing_pairs}
    for eq, k, op, fam in COMBOS:
        for prec in ("double", "single"):
            spec = OperatorSpec(eq, op, wavenumber=k, precision=prec)
            sp = build_space(m2, fam)
            ctx = make_integration_context(spec, sp, sp)
            be = make_host_backends(ctx)[0]
            res = be.integrate_batch(BatchRequest(reg_pairs))
            t = tag(eq, op, fam, prec)
            d[f"{t}_re"] = res.re
            if res.im is not None:
                d[f"{t}_im"] = res.im
            if prec == "double":
                sp1 = build_space(m1, fam)
                ctx1 = make_integration_context(spec, sp1, sp1)
                blocks = np.stack([local_matrix(ctx1, int(a), int(b)) for a, b in sing_pairs])
                d[f"{t}_local"] = blocks
    np.savez_compressed(os.path.join(HERE, "integrals.npz"), **d)


def tree_arrays(tree, prefix, d):
    nodes = tree.nodes
    d[f"{prefix}_perm"] = tree.permutation
    d[f"{prefix}_nodes"] = np.array([[n.start, n.stop, n.level, n.left, n.right] for n in nodes],
                                    dtype=np.int64)
    d[f"{prefix}_bbox"] = np.array([np.concatenate([n.bbox_min, n.bbox_max]) for n in nodes])


def make_partitions():
    d = {}
    cases = {
        "ico3_p0": (refine_unit_sphere(3), "p0"),
        "ico2_p1c": (refine_unit_sphere(2), "p1c"),
        "ico2_p1d": (refine_unit_sphere(2), "p1d"),
        "geo11_p0": (TriangleMesh(*geodesic_sphere(11)), "p0"),
        "geo45_p0": (TriangleMesh(*geodesic_sphere(45)), "p0"),
    }
    for name, (mesh, fam) in cases.items():
        sp = build_space(mesh, fam)
        bt = cluster_trees_for(sp, sp)
        tree_arrays(bt.rows, name, d)
        d[f"{name}_leaves"] = np.array([[lf.row_node, lf.col_node, int(lf.admissible)]
                                        for lf in bt.leaves], dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "partitions.npz"), **d)


def make_hmatrices():
    """Reference H-matrices: per-leaf ranks and matvecs, plus dense matvecs."""
    d = {}
    rng = np.random.default_rng(1234)
    cases = [
        ("ico2_p0_lap_slp", refine_unit_sphere(2), "p0", OperatorSpec("laplace", "slp"), 1e-3),
        ("ico2_p0_lap_slp_e5", refine_unit_sphere(2), "p0", OperatorSpec("laplace", "slp"), 1e-5),
        ("ico2_p0_helm_slp", refine_unit_sphere(2), "p0",
         OperatorSpec("helmholtz", "slp", wavenumber=2.0), 1e-4),
        ("ico2_p0_lap_dlp", refine_unit_sphere(2), "p0", OperatorSpec("laplace", "dlp"), 1e-4),
        ("ico2_p1c_lap_dlp", refine_unit_sphere(2), "p1c", OperatorSpec("laplace", "dlp"), 1e-4),
    ]
    for name, mesh, fam, spec, eps in cases:
        sp = build_space(mesh, fam)
        bt = cluster_trees_for(sp, sp)
        stats = {}
        h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=eps), stats=stats)
        ctx = make_integration_context(spec, sp, sp)
        dense = assemble_dense(spec, sp, sp, AssemblyConfig(), make_host_backends(ctx))
        xs = rng.standard_normal((3, sp.n_dofs))
        if spec.is_complex:
            xs = xs + 1j * rng.standard_normal((3, sp.n_dofs))
        d[f"{name}_x"] = xs
        d[f"{name}_hx"] = np.stack([h.matvec(x) for x in xs])
        d[f"{name}_dx"] = np.stack([dense @ x for x in xs])
        d[f"{name}_ranks"] = np.array([p.rank if isinstance(p, LowRankBlock) else -1
                                       for p in h.payloads], dtype=np.int64)
        cs = compression_stats(h)
        d[f"{name}_stored"] = np.array([cs.stored_entries])
        d[f"{name}_eps"] = np.array([eps])
        d[f"{name}_counters"] = np.array([stats["singular_pairs"], stats["aca_fallback_dense"],
                                          stats["dense_leaves"], stats["lowrank_leaves"]])
        if name == "ico2_p0_lap_slp":
            d[f"{name}_dense"] = dense
    np.savez_compressed(os.path.join(HERE, "hmatrices.npz"), **d)


if __name__ == "__main__":
    make_rules()
    make_meshes()
    make_integrals()
    make_partitions()
    make_hmatrices()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
