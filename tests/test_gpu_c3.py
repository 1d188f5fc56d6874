"""C3 scale on the GPU against the REAL reference (tests/golden/make_c3_golden.py):
Helmholtz single layer, P0, geodesic sphere n=71 (100 820 triangles),
k = 33.7 (10 elements per wavelength; kr up to ~67 rad).

* entry parity at the C3 wavenumber: 10^4 disjoint pairs through the
  reference's ``integrate_batch`` contract (FP64 <= 1e-12 of the entry; FP32
  <= 1e-5 against the reference FP64), and every touching
  pair of three elements through ``local_matrix`` (<= 1e-12);
* the GPU's exact operator rows equal the reference's (1e-12), and the C3
  H-matrix (ACA eps 1e-4, the config's tolerance) reproduces them within the
  10 eps bound of the reference's own acceptance test
  (test_acceptance.py:176-191).
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def rel(got, ref):
    """max |got - ref| / |ref| per entry, entries below 1 % of the batch
    maximum normalised by 1 % of it (test_gpu_integrate.rel_err)."""
    scale = np.maximum(np.abs(ref), 1e-2 * np.abs(ref).max())
    return float((np.abs(np.asarray(got) - ref) / scale).max())


@pytest.fixture(scope="module")
def c3():
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    from paper_1711_01897_b200.meshes import geodesic_sphere
    g = golden("c3")
    v, e = geodesic_sphere(71)
    return g, v, e, build_space(TriangleMesh(v, e), "p0")


def _backend(sp, k, prec):
    from paper_1711_01897_b200.backend import make_gpu_backends
    from paper_1711_01897_b200.discretization import OperatorSpec, make_integration_context
    return make_gpu_backends(make_integration_context(OperatorSpec("helmholtz", "slp", k, prec),
                                                      sp, sp))[0]


@pytest.mark.parametrize("prec", ["double", "single"])
def test_c3_regular_pairs_vs_reference(c3, prec):
    from paper_1711_01897_b200.backend import BatchRequest
    g, v, e, sp = c3
    be = _backend(sp, float(g["k"]), prec)
    res = be.integrate_batch(BatchRequest(g["regular_pairs"]))
    got = res.re[:, 0, 0].astype(np.float64) + 1j * res.im[:, 0, 0].astype(np.float64)
    ref64 = g["double_re"] + 1j * g["double_im"]
    if prec == "double":
        assert rel(got, ref64) <= 1e-12
    else:
        assert res.re.dtype == np.float32
        assert rel(got, ref64) <= 1e-5
        # and as close to the reference's own FP32 path as to its FP64
        ref32 = g["single_re"].astype(np.float64) + 1j * g["single_im"]
        assert rel(got, ref32) <= 2e-5


def test_c3_touching_pairs_vs_reference_local_matrix(c3):
    from paper_1711_01897_b200.backend import BatchRequest
    g, v, e, sp = c3
    be = _backend(sp, float(g["k"]), "double")
    res = be.integrate_pairs(BatchRequest(g["singular_pairs"]))
    got = res.complex_view()[:, 0, 0]
    assert rel(got, g["singular"]) <= 1e-12


def test_c3_hmatrix_sampled_rows_vs_reference_exact_rows(c3):
    from test_gpu_scale import exact_rows
    from paper_1711_01897_b200.discretization import OperatorSpec
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix
    from paper_1711_01897_b200.partition import cluster_trees_for
    g, v, e, sp = c3
    k, eps = float(g["k"]), 1e-4
    spec = OperatorSpec("helmholtz", "slp", k)
    x = np.random.default_rng(int(g["x_seed"])).standard_normal(len(e))
    rows, z_ref = g["rows"], g["exact"]
    # the GPU's exact rows (integrate_any over every pair) are the reference's
    z = exact_rows(spec, sp, rows, x)
    assert np.abs(z - z_ref).max() <= 1e-12 * np.abs(z_ref).max()
    h = assemble_hmatrix(spec, sp, sp, cluster_trees_for(sp, sp), AcaConfig(epsilon=eps))
    y = h.matvec(x)
    scale = np.sqrt(np.mean(np.abs(y) ** 2))
    assert np.abs(y[rows] - z_ref).max() <= 10 * eps * scale
