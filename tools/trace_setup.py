"""Time the context + setup + first execute of the C5 assembly (HBEM_TRACE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HBEM_TRACE"] = "1"
import numpy as np
from paper_1711_01897_b200.meshes import geodesic_sphere
from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space, make_integration_context
from paper_1711_01897_b200.partition import cluster_trees_for
from paper_1711_01897_b200.backend import init_gpu_device
from paper_1711_01897_b200.hmatrix import AcaConfig, AssemblyConfig, _assemble_part
n = int(sys.argv[1]) if len(sys.argv) > 1 else 448
t = time.time(); v, e = geodesic_sphere(n); sp = build_space(TriangleMesh(v, e), "p0"); print("mesh", time.time() - t, flush=True)
t = time.time(); bt = cluster_trees_for(sp, sp); print("partition", time.time() - t, flush=True)
spec = OperatorSpec("laplace", "slp")
t = time.time(); ictx = make_integration_context(spec, sp, sp); print("ictx", time.time() - t, flush=True)
t = time.time(); ctx = init_gpu_device(ictx); print("ctx", time.time() - t, flush=True)
ids = np.arange(len(bt.leaf_array))
for r in range(2):
    t = time.time(); part = _assemble_part(ctx, bt, ids, sp, sp, AcaConfig(epsilon=1e-3), AssemblyConfig()); w = time.time() - t
    print("setup+execute", w, "setup", part.stats["seconds_setup"], "execute", part.stats["seconds"], flush=True)
    t = time.time(); part.execute(); print("re-execute", time.time() - t, flush=True)
    part.close()
