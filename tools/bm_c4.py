"""C4 end to end: sound-hard plane-wave scattering off the
synthetic elongated hull with the Burton-Miller combined-field solve on the
device operators, then the bistatic far field on a 3600-point ring.

    python tools/bm_c4.py [--around 180 --along 1400] [--eps 1e-3] [--precision double]

Prints one JSON line: mesh size, DOFs (P1c / P1d), k, assembly and solve time,
GMRES iterations and final residual, far-field time, the bistatic target
strength (TS, scatter.py:411-424) summary, and with --delta-eps E the paper's
far-field deviation Delta_sct (scatter.py:427-441) between this solve and a
second one at ACA eps E.  --csv PATH writes the far field (scatter.py:444-452)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1711_01897_b200.discretization import TriangleMesh, build_space  # noqa: E402
from paper_1711_01897_b200.hmatrix import AcaConfig  # noqa: E402
from paper_1711_01897_b200.meshes import elongated_hull  # noqa: E402
from paper_1711_01897_b200.scatter import (ScatterConfig, burton_miller_solve,  # noqa: E402
                                           deviation, evaluate_far_field, evaluation_ring,
                                           target_strength, write_far_field_csv)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--around", type=int, default=180)
    ap.add_argument("--along", type=int, default=1400)
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--epw", type=float, default=8.0, help="elements per wavelength")
    ap.add_argument("--delta-eps", type=float, default=None)
    ap.add_argument("--csv", default=None)
    a = ap.parse_args()
    v, e = elongated_hull(a.around, a.along)
    mesh = TriangleMesh(v, e)
    p = v[e]
    h = max(np.linalg.norm(p[:, i] - p[:, (i + 1) % 3], axis=1).max() for i in range(3))
    k = 2 * np.pi / (a.epw * h)
    c = 1500.0
    cfg = ScatterConfig(frequency=k * c / (2 * np.pi), sound_speed=c, aca=AcaConfig(epsilon=a.eps),
                        tol=1e-5, restart=100)
    t = time.perf_counter()
    rep = burton_miller_solve(cfg, mode="hmatrix", mesh=mesh)
    wall = time.perf_counter() - t
    pts, _ = evaluation_ring(3600, 100.0)
    t = time.perf_counter()
    far = evaluate_far_field(mesh, build_space(mesh, "p1c"), rep.phi, pts, k)
    t_far = time.perf_counter() - t
    pts_deg = np.degrees(np.arctan2(pts[:, 1], pts[:, 0])) % 360.0
    ts = target_strength(far, cfg.amplitude, 100.0)
    line = {"workload": "C4 hull Burton-Miller (hmatrix mode) + far field",
            "elements": len(e), "p1c_dofs": rep.n_dofs, "p1d_dofs": 3 * len(e),
            "k": k, "eps": a.eps, "iterations": rep.iterations,
            "residual": rep.residual, "timings_s": rep.timings, "wall_s": wall,
            "far_field_s": t_far, "far_max_abs": float(np.abs(far).max()),
            "ts_db": {"max": float(ts.max()), "min": float(ts[np.isfinite(ts)].min()),
                      "mean": float(ts[np.isfinite(ts)].mean()),
                      "backscatter": float(ts[np.argmin(np.abs(pts_deg - 180.0))])}}
    if a.csv:
        write_far_field_csv(a.csv, pts_deg, far, cfg.amplitude, 100.0)
    if a.delta_eps:
        cfg2 = ScatterConfig(frequency=cfg.frequency, sound_speed=c,
                             aca=AcaConfig(epsilon=a.delta_eps), tol=1e-5, restart=100)
        rep2 = burton_miller_solve(cfg2, mode="hmatrix", mesh=mesh)
        far2 = evaluate_far_field(mesh, build_space(mesh, "p1c"), rep2.phi, pts, k)
        line["delta_sct"] = {"vs_eps": a.delta_eps, "value": deviation(far, far2),
                             "iterations": rep2.iterations, "timings_s": rep2.timings}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
