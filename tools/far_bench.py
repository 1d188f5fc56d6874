"""Far-field evaluation at the C4 scale: elongated hull
(~504 000 triangles), P1c complex density, 3600 ring points (the paper's
far-field sweep), Helmholtz k at 8 elements per wavelength.  Prints one JSON
line: seconds (median of 5, the full C-ABI call incl. H2D of mesh + density),
kernel evaluations per second, and a 1-point oracle check.

    python tools/far_bench.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import hbem_oracle as O  # noqa: E402  (checker only)
from paper_1711_01897_b200.discretization import TriangleMesh, build_space  # noqa: E402
from paper_1711_01897_b200.meshes import elongated_hull  # noqa: E402
from paper_1711_01897_b200.scatter import evaluate_far_field, evaluation_ring  # noqa: E402


def main():
    v, e = elongated_hull(180, 1400)
    p = v[e]
    h = max(np.linalg.norm(p[:, i] - p[:, (i + 1) % 3], axis=1).max() for i in range(3))
    k = 2 * np.pi / (8 * h)
    mesh = TriangleMesh(v, e)
    sp = build_space(mesh, "p1c")
    rng = np.random.default_rng(1)
    phi = rng.standard_normal(sp.n_dofs) + 1j * rng.standard_normal(sp.n_dofs)
    pts, _ = evaluation_ring(3600, 200.0)
    evaluate_far_field(mesh, sp, phi, pts[:8], k)  # warm-up (context, module load)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        u = evaluate_far_field(mesh, sp, phi, pts, k)
        ts.append(time.perf_counter() - t)
    sec = float(np.median(ts))
    evals = len(pts) * len(e) * 6
    ref, _ = O.far_field(v, e, "p1c", e, phi, pts[:2], k, chunk=1)
    err = float(np.abs(u[:2] - ref).max() / np.abs(ref).max())
    print(json.dumps({"workload": "far field, hull 504k tri P1c, 3600 points, Helmholtz DLP",
                      "elements": len(e), "points": len(pts), "k": k, "seconds": sec,
                      "samples_s": ts, "kernel_evals_per_s": evals / sec,
                      "rel_err_vs_oracle_2pts": err}))


if __name__ == "__main__":
    main()
