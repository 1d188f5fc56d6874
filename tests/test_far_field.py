"""Far-field evaluation (scatter.py:362-408).

CPU: the oracle restatement against the golden far fields of the real
reference (tests/golden/make_far_golden.py).  GPU: hbem_far_field (through
paper_1711_01897_b200.scatter.evaluate_far_field) against the same golden
values and the oracle, plus the reference's own far-field tests
(test_scatter.py:203-244: zero density, exact linearity, vanishing static
double layer, near-field warning, validation)."""

import numpy as np
import pytest

from conftest import golden


def _mesh(g):
    from paper_1711_01897_b200.meshes import geodesic_sphere
    return geodesic_sphere(int(g["n"]))


CASES = [("p1c_k2", "p1c"), ("p1c_k0", "p1c"), ("p0_k3", "p0")]


@pytest.mark.parametrize("name,fam", CASES)
def test_oracle_far_field_vs_reference_golden(name, fam):
    from oracle import hbem_oracle as O
    g = golden("far")
    v, e = _mesh(g)
    dm = np.arange(len(e)) if fam == "p0" else e
    u, n_near = O.far_field(v, e, fam, dm, g[f"{name}_phi"], g["points"], float(g[f"{name}_k"]))
    ref = g[f"{name}_u"]
    assert n_near == 0
    assert np.abs(u - ref).max() <= 1e-13 * np.abs(ref).max()


def test_oracle_static_double_layer_and_near_count():
    from oracle import hbem_oracle as O
    g = golden("far")
    v, e = _mesh(g)
    u, _ = O.far_field(v, e, "p1c", e, np.ones(int(e.max()) + 1), g["points"], 0.0)
    assert np.abs(u - g["static_u"]).max() <= 1e-15
    _, n_near = O.far_field(v, e, "p1c", e, np.ones(int(e.max()) + 1), g["near_points"], 2.0)
    assert str(n_near) in str(g["near_warning"])


def test_far_field_validation_is_host_side():
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    from paper_1711_01897_b200.errors import ConfigError
    from paper_1711_01897_b200.meshes import geodesic_sphere
    from paper_1711_01897_b200.scatter import evaluate_far_field, evaluation_ring
    v, e = geodesic_sphere(2)
    mesh = TriangleMesh(v, e)
    sp = build_space(mesh, "p1c")
    with pytest.raises(ConfigError):
        evaluate_far_field(mesh, sp, np.ones(sp.n_dofs), np.zeros((4, 2)), 2.0)
    with pytest.raises(ConfigError):
        evaluate_far_field(mesh, sp, np.ones(3), np.zeros((4, 3)), 2.0)
    with pytest.raises(ConfigError):
        evaluation_ring(0, 1.0)
    pts, ang = evaluation_ring(8, 50.0)
    assert pts.shape == (8, 3) and ang[1] == 45.0


def _space(g, fam):
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    v, e = _mesh(g)
    mesh = TriangleMesh(v, e)
    return mesh, build_space(mesh, fam)


@pytest.mark.gpu
@pytest.mark.parametrize("name,fam", CASES)
def test_gpu_far_field_vs_reference_golden(name, fam):
    from paper_1711_01897_b200.scatter import evaluate_far_field
    g = golden("far")
    mesh, sp = _space(g, fam)
    u = evaluate_far_field(mesh, sp, g[f"{name}_phi"], g["points"], float(g[f"{name}_k"]))
    ref = g[f"{name}_u"]
    assert u.dtype == np.complex128
    assert np.abs(u - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.gpu
def test_gpu_far_field_reference_properties():
    from paper_1711_01897_b200.scatter import evaluate_far_field, evaluation_ring
    g = golden("far")
    mesh, sp = _space(g, "p1c")
    pts, _ = evaluation_ring(8, 50.0)
    zero = evaluate_far_field(mesh, sp, np.zeros(sp.n_dofs), pts, 2.0)
    assert np.array_equal(zero, np.zeros(8, dtype=np.complex128))
    rng = np.random.default_rng(5)
    phi = rng.standard_normal(sp.n_dofs) + 1j * rng.standard_normal(sp.n_dofs)
    one = evaluate_far_field(mesh, sp, phi, pts, 2.0)
    two = evaluate_far_field(mesh, sp, 2.0 * phi, pts, 2.0)
    assert np.array_equal(two, 2.0 * one)
    static = evaluate_far_field(mesh, sp, np.ones(sp.n_dofs), g["points"], 0.0)
    assert np.abs(static - g["static_u"]).max() <= 1e-14
    with pytest.warns(UserWarning, match="near field") as rec:
        evaluate_far_field(mesh, sp, np.ones(sp.n_dofs), g["near_points"], 2.0)
    assert str(rec[0].message) == str(g["near_warning"])


@pytest.mark.gpu
def test_gpu_far_field_at_scale_vs_oracle():
    """Hull mesh (C4 geometry class), 360 ring points, complex P1c density:
    device sum vs the oracle's numpy einsum."""
    from oracle import hbem_oracle as O
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    from paper_1711_01897_b200.meshes import elongated_hull
    from paper_1711_01897_b200.scatter import evaluate_far_field, evaluation_ring
    v, e = elongated_hull(40, 200)
    mesh = TriangleMesh(v, e)
    sp = build_space(mesh, "p1c")
    rng = np.random.default_rng(9)
    phi = rng.standard_normal(sp.n_dofs) + 1j * rng.standard_normal(sp.n_dofs)
    pts, _ = evaluation_ring(360, 40.0)
    u = evaluate_far_field(mesh, sp, phi, pts, 7.0)
    ref, _ = O.far_field(v, e, "p1c", e, phi, pts, 7.0, chunk=16)
    assert np.abs(u - ref).max() <= 1e-11 * np.abs(ref).max()
