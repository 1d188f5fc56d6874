import cProfile, pstats, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1711_01897_b200.discretization import TriangleMesh
from paper_1711_01897_b200.hmatrix import AcaConfig
from paper_1711_01897_b200.meshes import elongated_hull
from paper_1711_01897_b200.scatter import ScatterConfig, burton_miller_solve
from paper_1711_01897_b200.errors import SolverError
v, e = elongated_hull(180, 1400)
mesh = TriangleMesh(v, e)
p = v[e]
h = max(np.linalg.norm(p[:, i] - p[:, (i + 1) % 3], axis=1).max() for i in range(3))
k = 2 * np.pi / (8 * h)
cfg = ScatterConfig(frequency=k * 1500 / (2 * np.pi), aca=AcaConfig(epsilon=1e-3), max_iter=8)
pr = cProfile.Profile()
pr.enable()
try:
    burton_miller_solve(cfg, mode="hmatrix", mesh=mesh)
except SolverError as ex:
    print("expected", ex)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
