"""Rank agreement of the GPU H-matrix with the REAL reference's (golden
hmatrices.npz) and with the oracle's full H-matrix (C1)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__)))), "tests"))
from conftest import golden  # noqa
from oracle import hbem_oracle as O  # noqa
from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space  # noqa
from paper_1711_01897_b200.hmatrix import AcaConfig, LowRankBlock, assemble_hmatrix  # noqa
from paper_1711_01897_b200.meshes import geodesic_sphere  # noqa
from paper_1711_01897_b200.partition import cluster_trees_for  # noqa

g = golden("hmatrices")
m = golden("meshes")
v, e = m["ico2_vertices"], m["ico2_elements"]
for name, fam, eq, op, k in [("ico2_p0_lap_slp", "p0", "laplace", "slp", 0.0),
                             ("ico2_p0_lap_slp_e5", "p0", "laplace", "slp", 0.0),
                             ("ico2_p0_helm_slp", "p0", "helmholtz", "slp", 2.0),
                             ("ico2_p0_lap_dlp", "p0", "laplace", "dlp", 0.0),
                             ("ico2_p1c_lap_dlp", "p1c", "laplace", "dlp", 0.0)]:
    sp = build_space(TriangleMesh(v, e), fam)
    h = assemble_hmatrix(OperatorSpec(eq, op, k), sp, sp, cluster_trees_for(sp, sp),
                         AcaConfig(epsilon=float(g[f"{name}_eps"][0])))
    r = np.array([p.rank if isinstance(p, LowRankBlock) else -1 for p in h.payloads])
    ref = g[f"{name}_ranks"]
    print(name, "rank agreement", (r == ref).mean(), "differ", int((r != ref).sum()), "of", len(r))
v, e = geodesic_sphere(11)
sp = build_space(TriangleMesh(v, e), "p0")
h = assemble_hmatrix(OperatorSpec("laplace", "slp", 0.0), sp, sp, cluster_trees_for(sp, sp),
                     AcaConfig(epsilon=1e-3))
P = O.Problem(O.Spec("laplace", "slp"), v, e)
tree = O.cluster_tree(P.dof_centers("p0"), 32)
leaves = O.block_tree(tree, tree, 2.0)
ref = O.Assembler(P, tree, tree, leaves, 1e-3).assemble()
r = np.array([p.rank if hasattr(p, "rank") else -1 for p in h.payloads])
rr = np.array([p.rank if isinstance(p, O.LowRank) else -1 for p in ref])
print("C1 vs oracle rank agreement", (r == rr).mean(), int((r != rr).sum()), "of", len(r))
