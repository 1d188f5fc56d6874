"""Kernel microbenchmark: K1 regular-pair throughput through the device C ABI
(hbem_integrate_regular_device), inputs resident in HBM, CUDA-event timed.

    python tools/kbench.py [--n 448] [--pairs 20000000]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_01897_b200 import _lib  # noqa: E402
from paper_1711_01897_b200.backend import make_gpu_backends  # noqa: E402
from paper_1711_01897_b200.discretization import (OperatorSpec, TriangleMesh,  # noqa: E402
                                                  build_space, make_integration_context)
from paper_1711_01897_b200.meshes import geodesic_sphere  # noqa: E402


def run(spec, fam, mesh, pairs_dev, reps=5):
    sp = build_space(mesh, fam)
    ctx = make_integration_context(spec, sp, sp)
    be = make_gpu_backends(ctx)[0]
    p = pairs_dev.shape[0]
    nt = ns = 1 if fam == "p0" else 3
    dt = torch.float64 if spec.precision == "double" else torch.float32
    re = torch.empty((p, nt, ns), dtype=dt, device="cuda")
    im = torch.empty_like(re) if spec.is_complex else None
    st = torch.cuda.current_stream()

    def call():
        _lib.check(_lib.lib.hbem_integrate_regular_device(
            be.context.handle, C.c_void_p(pairs_dev.data_ptr()), p, C.c_void_p(re.data_ptr()),
            C.c_void_p(im.data_ptr()) if im is not None else None, C.c_void_p(st.cuda_stream)))

    for _ in range(2):
        call()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = min(ts)
    return p / t, t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=448)
    ap.add_argument("--pairs", type=int, default=20_000_000)
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    v, e = geodesic_sphere(args.n)
    mesh = TriangleMesh(v, e)
    m = len(e)
    rng = np.random.default_rng(0)
    # ACA-like pairs: each test element against a contiguous run of trial elements
    p = args.pairs
    a = rng.integers(0, m, size=p // 64).repeat(64)
    b = (rng.integers(0, m - 64, size=p // 64)[:, None] + np.arange(64)[None, :]).ravel()
    ok = ~(e[a][:, :, None] == e[b][:, None, :]).any(axis=(1, 2))
    pairs = np.stack([a[ok], b[ok]], 1).astype(np.int64)
    pairs_dev = torch.from_numpy(pairs).cuda()
    cases = [
        (OperatorSpec("laplace", "slp"), "p0"),
        (OperatorSpec("laplace", "slp", precision="single"), "p0"),
    ]
    if not args.quick:
        cases += [
            (OperatorSpec("helmholtz", "slp", 33.7), "p0"),
            (OperatorSpec("helmholtz", "slp", 33.7, "single"), "p0"),
            (OperatorSpec("laplace", "dlp"), "p1c"),
            (OperatorSpec("laplace", "dlp", precision="single"), "p1c"),
            (OperatorSpec("helmholtz", "dlp", 10.0), "p1c"),
        ]
    out = []
    for spec, fam in cases:
        rate, t = run(spec, fam, mesh, pairs_dev)
        rec = {"eq": spec.equation, "op": spec.operator, "prec": spec.precision, "fam": fam,
               "pairs": len(pairs), "seconds": t, "pairs_per_s": rate}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    return out


if __name__ == "__main__":
    main()
