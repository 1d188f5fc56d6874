"""Golden H-matrix matvec of the REAL reference on the synthetic elongated
hull (C4 geometry class), Helmholtz SLP P0 at 8 elements per wavelength,
eps 1e-3 (build container only; ~3 minutes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_hull_golden.py

Pins tests/test_gpu_scale.py::test_hull_hmatrix_matches_reference: the GPU
assembly follows the same ACA pivots, so its matvec agrees with the
reference's H-matrix matvec to rounding even where ACA itself is far from
the exact operator (thin bodies, SURVEY §8c "pivots may legitimately
diverge" is the looser bar)."""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from hbem.hmatrix import AcaConfig, assemble_hmatrix, cluster_trees_for, hmat_matvec  # noqa: E402
from hbem.kernels import OperatorSpec  # noqa: E402
from hbem.mesh import TriangleMesh  # noqa: E402
from hbem.spaces import build_space  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1711_01897_b200.meshes import elongated_hull  # noqa: E402

v, e = elongated_hull(24, 150)
p = v[e]
h = max(np.linalg.norm(p[:, i] - p[:, (i + 1) % 3], axis=1).max() for i in range(3))
k = 2 * np.pi / (8 * h)
sp = build_space(TriangleMesh(v, e), "p0")
H = assemble_hmatrix(OperatorSpec("helmholtz", "slp", k), sp, sp, cluster_trees_for(sp, sp),
                     AcaConfig(epsilon=1e-3))
rng = np.random.default_rng(1234)
xs = np.stack([rng.standard_normal(len(e)) for _ in range(2)])
ys = np.stack([hmat_matvec(H, x) for x in xs])
np.savez_compressed(os.path.join(HERE, "hull.npz"), n_around=24, n_along=150, k=k, eps=1e-3,
                    x=xs, y=ys)
print("wrote hull.npz", len(e), "elements, k =", k)
