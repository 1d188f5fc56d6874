"""C5 (the headline: 4 014 080-triangle sphere, Laplace SLP P0, eps 1e-3, FP64)
assembled through the public assemble_hmatrix and checked through
size-independent properties:

* sampled rows of H x within 10 eps of the exact operator rows (exact rows =
  every element pair through the GPU batched integrator, itself pinned to the
  reference at 1e-12);
* a random subset of those exact-row entries equals the CPU oracle's
  integrate_batch / local_matrix (the reference's algorithm) to 1e-12;
* the device matvec is bitwise reproducible and the per-phase counters
  add up (every admissible block classified, every leaf assembled)."""

import numpy as np
import pytest

from test_gpu_scale import exact_rows, problem

pytestmark = pytest.mark.gpu


def test_c5_sampled_rows_and_entries():
    from oracle import hbem_oracle as O
    from paper_1711_01897_b200.backend import BatchRequest, make_gpu_backends
    from paper_1711_01897_b200.discretization import make_integration_context
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix
    v, e, spec, sp, bt = problem(448, "p0", "laplace", "slp", 0.0)
    eps = 1e-3
    st = {}
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=eps), stats=st)
    assert st["lowrank_leaves"] + st["dense_leaves"] == len(bt.leaf_array)
    rng = np.random.default_rng(448)
    x = rng.standard_normal(len(e))
    y = h.matvec(x)
    assert np.array_equal(h.matvec(x), y)
    rows = rng.choice(len(e), size=3, replace=False)
    z = exact_rows(spec, sp, rows, x)
    scale = np.sqrt(np.mean(y ** 2))
    assert np.abs(y[rows] - z).max() <= 10 * eps * scale
    # entries of the first sampled row against the CPU oracle
    be = make_gpu_backends(make_integration_context(spec, sp, sp))[0]
    i = int(rows[0])
    cols = rng.choice(len(e), size=20000, replace=False)
    pairs = np.stack([np.full(len(cols), i), cols], 1).astype(np.int64)
    got = be.integrate_pairs(BatchRequest(pairs)).complex_view()[:, 0, 0].real
    P = O.Problem(O.Spec("laplace", "slp"), v, e)
    touch = (e[cols][:, :, None] == e[i][None, None, :]).any(axis=(1, 2))
    ref = np.empty(len(cols))
    re, _ = O.integrate_batch(P, pairs[~touch])
    ref[~touch] = re[:, 0, 0]
    for j in np.nonzero(touch)[0]:
        ref[j] = O.local_matrix(P, i, int(cols[j]))[0, 0]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
