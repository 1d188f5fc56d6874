"""Burton-Miller scattering driver (scatter.py:228-359).

CPU: GMRES (solvers.py:47-134) on dense systems; the P1c mass matrix and the
sparse curl / normal transforms against the reference's own matrices
(tests/golden/make_bm_golden.py); driver validation.  GPU: the complete
solve on the device operators against the reference's solution, iteration
count and far field (same ACA pivots => the H-matrix operators agree to
rounding, so GMRES takes the same path)."""

import numpy as np
import pytest

from conftest import golden


def _mesh():
    from paper_1711_01897_b200.discretization import TriangleMesh
    from paper_1711_01897_b200.meshes import geodesic_sphere
    return TriangleMesh(*geodesic_sphere(int(golden("bm")["n"])))


def test_gmres_dense_systems():
    from paper_1711_01897_b200.solvers import gmres
    rng = np.random.default_rng(3)
    n = 60
    a = np.eye(n) * 4 + rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for restart in (5, 100):
        r = gmres(lambda x: a @ x, b, tol=1e-10, restart=restart)
        assert r.converged and r.residual <= 1e-10
        assert np.linalg.norm(a @ r.x - b) <= 1e-9 * np.linalg.norm(b)
        assert len(r.residuals) == r.iterations
    z = gmres(lambda x: a @ x, np.zeros(n))
    assert z.converged and z.iterations == 0 and not z.x.any()
    stalled = gmres(lambda x: a @ x, b, tol=1e-14, restart=2, max_iter=3)
    assert not stalled.converged and stalled.iterations == 3


def test_mass_and_transforms_vs_reference():
    from paper_1711_01897_b200.discretization import build_space
    from paper_1711_01897_b200.scatter import (_curl_and_normal_maps, _element_frames,
                                               _mass_p1c)
    g = golden("bm")
    mesh = _mesh()
    p1c, p1d = build_space(mesh, "p1c"), build_space(mesh, "p1d")
    v, jac, nrm = _element_frames(mesh)
    assert np.abs(_mass_p1c(p1c, jac).toarray() - g["mass"]).max() <= 1e-16
    q, p = _curl_and_normal_maps(p1c, p1d, v, jac, nrm)
    for j in range(3):
        assert np.abs(q[j].toarray() - g["q"][j]).max() <= 1e-13 * np.abs(g["q"]).max()
        assert np.array_equal(p[j].toarray(), g["p"][j])


def test_driver_validation():
    from paper_1711_01897_b200.discretization import TriangleMesh
    from paper_1711_01897_b200.errors import ConfigError, MeshError, SolverError
    from paper_1711_01897_b200.scatter import PlaneWave, ScatterConfig, burton_miller_solve
    mesh = _mesh()
    with pytest.raises(ConfigError, match="mode"):
        burton_miller_solve(ScatterConfig(), mode="sparse", mesh=mesh)
    with pytest.raises(ConfigError, match="same problem"):
        burton_miller_solve(ScatterConfig(), wave=PlaneWave(1.0, np.array([1.0, 0, 0]), 3.0),
                            mesh=mesh)
    with pytest.raises(ConfigError):
        PlaneWave(1.0, np.array([1.0, 1.0, 0.0]), 2.0)
    with pytest.raises(ConfigError):
        ScatterConfig(tol=0.0)
    open_mesh = TriangleMesh(mesh.vertices, mesh.elements[:-1])
    with pytest.raises(MeshError, match="closed"):
        burton_miller_solve(ScatterConfig(), mesh=open_mesh)
    flipped = mesh.elements.copy()
    flipped[0] = flipped[0, [0, 2, 1]]
    with pytest.raises(MeshError, match="orientation"):
        burton_miller_solve(ScatterConfig(), mesh=TriangleMesh(mesh.vertices, flipped))
    with pytest.raises(SolverError, match="per wavelength"):
        burton_miller_solve(ScatterConfig(frequency=20000.0), mesh=mesh)


@pytest.mark.gpu
def test_gpu_burton_miller_hmatrix_vs_reference():
    from paper_1711_01897_b200.discretization import build_space
    from paper_1711_01897_b200.scatter import (ScatterConfig, burton_miller_solve,
                                               evaluate_far_field)
    g = golden("bm")
    mesh = _mesh()
    stats = {}
    rep = burton_miller_solve(ScatterConfig(), mode="hmatrix", mesh=mesh, stats=stats)
    # same Krylov path (iteration count, residual history to 1e-6 relative);
    # the P1 H-matrices agree with the reference's within the ACA tolerance
    # (eps = 1e-5; the dense device operators land as close, 1.3e-6), so the
    # solution and the far field are held to eps (measured 6.5e-7 on phi)
    assert rep.converged and rep.iterations == int(g["iterations"])
    assert (np.abs(np.array(rep.residuals) - g["residuals"]) <= 1e-6 * g["residuals"]).all()
    assert np.abs(rep.phi - g["phi"]).max() <= 1e-5 * np.abs(g["phi"]).max()
    far = evaluate_far_field(mesh, build_space(mesh, "p1c"), rep.phi, g["points"], float(g["k"]))
    assert np.abs(far - g["far"]).max() <= 1e-5 * np.abs(g["far"]).max()
    assert stats["mode"] == "hmatrix" and stats["elements_per_wavelength"] > 6


@pytest.mark.gpu
def test_gpu_burton_miller_dense_vs_reference_hmatrix():
    from paper_1711_01897_b200.scatter import ScatterConfig, burton_miller_solve
    g = golden("bm")
    rep = burton_miller_solve(ScatterConfig(), mode="dense", mesh=_mesh())
    assert rep.converged
    assert np.abs(rep.phi - g["phi"]).max() <= 1e-5 * np.abs(g["phi"]).max()
