"""Device H-matrix matvec timing (hbem_hmat_matvec_device, CUDA events on the
launching stream) with the bytes it must read: stored factor + dense entries.
    python tools/mv_bench.py [--n 448] [--reps 10]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space  # noqa
from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix  # noqa: E402
from paper_1711_01897_b200.meshes import geodesic_sphere  # noqa: E402
from paper_1711_01897_b200.partition import cluster_trees_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=448)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
v, e = geodesic_sphere(a.n)
sp = build_space(TriangleMesh(v, e), "p0")
st = {}
h = assemble_hmatrix(OperatorSpec("laplace", "slp", 0.0), sp, sp, cluster_trees_for(sp, sp),
                     AcaConfig(epsilon=1e-3), stats=st)
x = torch.from_numpy(np.random.default_rng(1).standard_normal(len(e))).cuda()
y = h.matvec_torch(x)  # builds the cover lists / packs factors once
torch.cuda.synchronize()
s, t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    y = h.matvec_torch(x)
t.record()
torch.cuda.synchronize()
ms = s.elapsed_time(t) / a.reps
stored = st["u_entries"] + st["v_entries"] + st["dense_entries"]
print(json.dumps({"workload": f"device matvec, geodesic sphere n={a.n} ({len(e)} DOFs) "
                  "Laplace SLP P0 eps 1e-3 FP64", "ms_per_matvec": ms,
                  "stored_entries": int(stored), "bytes_factors": int(stored * 8),
                  "GB_per_s": stored * 8 / (ms * 1e-3) / 1e9}))
