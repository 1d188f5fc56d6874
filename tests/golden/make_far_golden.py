"""Golden far fields of the REAL reference (evaluate_far_field,
scatter.py:362-408) on a synthetic geodesic sphere (build container only,
a few seconds):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_far_golden.py

Cases: P1c complex density at k = 2 and k = 0 (Laplace DLP), P0 real density
at k = 3, points on an evaluation ring of radius 5, plus the static
double-layer of a constant density (exterior solid angle: vanishes)."""

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from hbem.mesh import TriangleMesh  # noqa: E402
from hbem.scatter import evaluate_far_field, evaluation_ring  # noqa: E402
from hbem.spaces import build_space  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1711_01897_b200.meshes import geodesic_sphere  # noqa: E402

v, e = geodesic_sphere(6)
mesh = TriangleMesh(v, e)
rng = np.random.default_rng(1234)
out = {"n": 6}
pts, _ = evaluation_ring(16, 5.0)
out["points"] = pts
for name, fam, k, cplx in (("p1c_k2", "p1c", 2.0, True), ("p1c_k0", "p1c", 0.0, True),
                           ("p0_k3", "p0", 3.0, False)):
    sp = build_space(mesh, fam)
    phi = rng.standard_normal(sp.n_dofs)
    if cplx:
        phi = phi + 1j * rng.standard_normal(sp.n_dofs)
    out[f"{name}_phi"] = phi
    out[f"{name}_k"] = k
    out[f"{name}_u"] = evaluate_far_field(mesh, sp, phi, pts, k)
sp = build_space(mesh, "p1c")
out["static_u"] = evaluate_far_field(mesh, sp, np.ones(sp.n_dofs), pts, 0.0)
with warnings.catch_warnings(record=True) as w:
    warnings.simplefilter("always")
    near_pts, _ = evaluation_ring(8, 1.2)
    out["near_u"] = evaluate_far_field(mesh, sp, np.ones(sp.n_dofs), near_pts, 2.0)
    out["near_points"] = near_pts
    out["near_warning"] = str(w[0].message) if w else ""
np.savez_compressed(os.path.join(HERE, "far.npz"), **out)
print({k: (v.shape if hasattr(v, "shape") else v) for k, v in out.items()})
