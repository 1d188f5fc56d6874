"""One-off: time the device H-matrix assembly on a geodesic sphere."""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1711_01897_b200.meshes import geodesic_sphere
from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space, make_integration_context
from paper_1711_01897_b200.partition import cluster_trees_for
from paper_1711_01897_b200.backend import init_gpu_device
from paper_1711_01897_b200.hmatrix import AcaConfig, AssemblyConfig, _assemble_part
ap = argparse.ArgumentParser(); ap.add_argument("--n", type=int, default=448); ap.add_argument("--eps", type=float, default=1e-3)
ap.add_argument("--prec", default="double"); ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
t = time.time(); v, e = geodesic_sphere(a.n); sp = build_space(TriangleMesh(v, e), "p0"); print("mesh", time.time() - t, flush=True)
t = time.time(); bt = cluster_trees_for(sp, sp); print("partition", time.time() - t, len(bt.leaf_array), flush=True)
spec = OperatorSpec("laplace", "slp", precision=a.prec)
t = time.time(); ctx = init_gpu_device(make_integration_context(spec, sp, sp)); print("ctx", time.time() - t, flush=True)
ids = np.arange(len(bt.leaf_array))
for r in range(a.reps):
    t = time.time(); part = _assemble_part(ctx, bt, ids, sp, sp, AcaConfig(epsilon=a.eps), AssemblyConfig()); wall = time.time() - t
    s = part.stats
    print(json.dumps({"wall": wall, **{k: s[k] for k in s}}), flush=True)
    rk = part.rank[part.kind == 1]
    print("rank hist", np.bincount(rk).tolist(), flush=True)
    part.close()
