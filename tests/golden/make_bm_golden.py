"""Golden Burton-Miller solve of the REAL reference (burton_miller_solve,
scatter.py:228-359, mode "hmatrix") on a synthetic geodesic sphere n=4
(320 triangles), plane wave k = 2 along +x, plus its far field on a ring
(build container only, about a minute):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_bm_golden.py
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from hbem.mesh import TriangleMesh  # noqa: E402
from hbem.scatter import (PlaneWave, ScatterConfig, burton_miller_solve,  # noqa: E402
                          evaluate_far_field, evaluation_ring)
from hbem.mesh import precompute_geometry  # noqa: E402
from hbem.quadrature import regular_rule  # noqa: E402
from hbem.spaces import assemble_mass, build_space, sparse_transform_matrices  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1711_01897_b200.meshes import geodesic_sphere  # noqa: E402

v, e = geodesic_sphere(4)
mesh = TriangleMesh(v, e)
cfg = ScatterConfig()                  # k = 2, tol 1e-5, restart 100, ACA eps 1e-5
wave = cfg.plane_wave()
rep = burton_miller_solve(cfg, wave=wave, mode="hmatrix", mesh=mesh)
pts, _ = evaluation_ring(36, 50.0)
far = evaluate_far_field(mesh, build_space(mesh, "p1c"), rep.phi, pts, wave.wavenumber)
p1c, p1d = build_space(mesh, "p1c"), build_space(mesh, "p1d")
geo = precompute_geometry(mesh, regular_rule(4))
mass = assemble_mass(p1c, p1c, geo, regular_rule(2)).toarray()
qs, ps = sparse_transform_matrices(p1c, p1d, geo)
np.savez_compressed(os.path.join(HERE, "bm.npz"), n=4, k=wave.wavenumber,
                    mass=mass, q=np.stack([q.toarray() for q in qs]),
                    p=np.stack([p.toarray() for p in ps]),
                    direction=wave.direction, phi=rep.phi, iterations=rep.iterations,
                    residuals=np.array(rep.residuals), points=pts, far=far)
print(rep.iterations, rep.residual, rep.timings)
