"""Target strength / deviation / far-field CSV of the REAL reference
(scatter.py:411-452) on a seeded complex field (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ts_golden.py
"""
import io
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hbem.scatter import deviation, target_strength, write_far_field_csv  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(42)
u = rng.standard_normal(36) + 1j * rng.standard_normal(36)
u[5] = 0.0
ref = u + 1e-3 * (rng.standard_normal(36) + 1j * rng.standard_normal(36))
angles = np.linspace(0.0, 350.0, 36)
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "far.csv")
    write_far_field_csv(p, angles, u, 1.5 - 0.5j, 75.0)
    csv = open(p).read()
np.savez_compressed(os.path.join(HERE, "ts.npz"), u=u, ref=ref, angles=angles,
                    ts=target_strength(u, 1.5 - 0.5j, 75.0), dev=deviation(u, ref),
                    csv=np.array(csv))
print("wrote ts.npz")
