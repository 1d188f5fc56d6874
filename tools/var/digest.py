"""sha256 of every payload arena of one assembly (compare kernels/variants):
    HBEM_ACA_WS=1 python tools/var/digest.py 30 p0 laplace slp 0 double"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space  # noqa
from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix  # noqa
from paper_1711_01897_b200.meshes import geodesic_sphere  # noqa
from paper_1711_01897_b200.partition import cluster_trees_for  # noqa

n, fam, eq, op, k, prec = sys.argv[1:7]
v, e = geodesic_sphere(int(n))
sp = build_space(TriangleMesh(v, e), fam)
bt = cluster_trees_for(sp, sp)
st = {}
h = assemble_hmatrix(OperatorSpec(eq, op, float(k), prec), sp, sp, bt, AcaConfig(epsilon=1e-4),
                     stats=st)
part = h.parts[0][1]
d = hashlib.sha256()
for a in part.arenas():
    d.update(np.ascontiguousarray(a).tobytes())
for a in (part.kind, part.rank, part.off_u, part.off_d, part.resid):
    d.update(np.ascontiguousarray(a).tobytes())
print(n, fam, eq, op, prec, d.hexdigest()[:16], st["lowrank_leaves"], st["waves"])
