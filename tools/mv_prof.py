"""Device matvec timing of the C4 single layer (Helmholtz SLP on P1d, 1.5M
DOFs, eps 1e-3): wall time per hbem_hmat_matvec call (host x in, y out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space  # noqa: E402
from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix  # noqa: E402
from paper_1711_01897_b200.meshes import elongated_hull  # noqa: E402
from paper_1711_01897_b200.partition import cluster_trees_for  # noqa: E402

n_around, n_along = (int(a) for a in (sys.argv[1:3] if len(sys.argv) > 2 else (180, 1400)))
v, e = elongated_hull(n_around, n_along)
p = v[e]
h = max(np.linalg.norm(p[:, i] - p[:, (i + 1) % 3], axis=1).max() for i in range(3))
k = 2 * np.pi / (8 * h)
sp = build_space(TriangleMesh(v, e), "p1d")
H = assemble_hmatrix(OperatorSpec("helmholtz", "slp", k), sp, sp, cluster_trees_for(sp, sp),
                     AcaConfig(epsilon=1e-3))
part = H.parts[0][1]
print({k2: part.stats[k2] for k2 in ("lowrank_leaves", "dense_leaves", "u_entries", "v_entries",
                                      "dense_entries")}, flush=True)
x = np.random.default_rng(0).standard_normal(sp.n_dofs) + 0j
for _ in range(4):
    t = time.perf_counter()
    y = H.matvec(x)
    print("matvec s", time.perf_counter() - t, flush=True)
