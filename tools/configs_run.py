"""Run the BASELINE configs C1-C4 (and a reduced C5 check) on one GPU:
assembly time (second execute, inputs resident), pair counts, compression,
and a size-independent accuracy check: sampled rows of H x against the exact
operator rows from the batched integrator (tests/test_gpu_scale.py).

    python tools/configs_run.py [--only C2,C3] > gpurun_out/configs.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402

from paper_1711_01897_b200.backend import init_gpu_device  # noqa: E402
from paper_1711_01897_b200.discretization import (OperatorSpec, TriangleMesh,  # noqa: E402
                                                  build_space, make_integration_context)
from paper_1711_01897_b200.hmatrix import (AcaConfig, AssemblyConfig, HMatrix,  # noqa: E402
                                           _assemble_part, _Payloads, compression_stats)
from paper_1711_01897_b200.meshes import elongated_hull, geodesic_sphere  # noqa: E402
from paper_1711_01897_b200.partition import cluster_trees_for  # noqa: E402
from test_gpu_scale import exact_rows  # noqa: E402


def h_max(v, e):
    p = v[e]
    return float(max(np.linalg.norm(p[:, 0] - p[:, 1], axis=1).max(),
                     np.linalg.norm(p[:, 1] - p[:, 2], axis=1).max(),
                     np.linalg.norm(p[:, 2] - p[:, 0], axis=1).max()))


def configs():
    out = []
    v, e = geodesic_sphere(11)
    out.append(("C1", v, e, "p0", "laplace", "slp", 0.0, 1e-3, "double"))
    v, e = geodesic_sphere(45)
    out.append(("C2-f64", v, e, "p1c", "laplace", "dlp", 0.0, 1e-4, "double"))
    out.append(("C2-f32", v, e, "p1c", "laplace", "dlp", 0.0, 1e-4, "single"))
    v, e = geodesic_sphere(71)
    k3 = 2 * np.pi / (10 * h_max(v, e))
    out.append(("C3", v, e, "p0", "helmholtz", "slp", k3, 1e-4, "double"))
    v, e = elongated_hull(180, 1400)            # ~504 000 triangles
    k4 = 2 * np.pi / (8 * h_max(v, e))         # ~8 elements per wavelength
    out.append(("C4-dlp-p1c-f32", v, e, "p1c", "helmholtz", "dlp", k4, 1e-3, "single"))
    out.append(("C4-slp-p0-f64", v, e, "p0", "helmholtz", "slp", k4, 1e-3, "double"))
    # combined field (scatter.py:270-306): Helmholtz SLP on P1d, 3 DOFs per element
    out.append(("C4-slp-p1d-f32", v, e, "p1d", "helmholtz", "slp", k4, 1e-3, "single"))
    return out


def run(name, v, e, fam, eq, op, k, eps, prec):
    t = time.time()
    sp = build_space(TriangleMesh(v, e), fam)
    bt = cluster_trees_for(sp, sp)
    t_part = time.time() - t
    spec = OperatorSpec(eq, op, k, prec)
    dev = init_gpu_device(make_integration_context(spec, sp, sp))
    ids = np.arange(len(bt.leaf_array))
    t = time.time()
    part = _assemble_part(dev, bt, ids, sp, sp, AcaConfig(epsilon=eps), AssemblyConfig())
    t_first = time.time() - t
    t = time.time()
    part.execute()
    t_exec = time.time() - t
    s = part.stats
    h = HMatrix(bt, _Payloads([(ids, part)]), spec, ((ids, part),))
    rng = np.random.default_rng(1234)
    x = rng.standard_normal(sp.n_dofs)
    y = h.matvec(x)
    rows = rng.choice(sp.n_dofs, size=4, replace=False)
    z = exact_rows(spec, sp, rows, x)
    err = float(np.abs(y[rows] - z).max() / np.sqrt(np.mean(np.abs(y) ** 2)))
    cs = compression_stats(h)
    line = {"config": name, "elements": len(e), "dofs": sp.n_dofs, "space": fam,
            "equation": eq, "operator": op, "wavenumber": k, "eps": eps, "precision": prec,
            "partition_s": round(t_part, 3), "first_assemble_s": round(t_first, 3),
            "assembly_s": round(t_exec, 4), "regular_pairs": int(s["regular_pairs"]),
            "singular_pairs": int(s["singular_pairs"]),
            "pairs_per_s": (s["regular_pairs"] + s["singular_pairs"]) / t_exec,
            "waves": int(s["waves"]), "compression": cs.ratio,
            "sampled_row_err": err, "err_bound": 10 * eps}
    part.close()
    dev.close()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None
    for c in configs():
        if only and c[0] not in only:
            continue
        try:
            print(json.dumps(run(*c)), flush=True)
        except Exception as exc:  # noqa: BLE001 - report and continue
            print(json.dumps({"config": c[0], "error": repr(exc)[:500]}), flush=True)


if __name__ == "__main__":
    main()
