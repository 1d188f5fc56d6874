"""Dense assembly API (assembly.py:234-318 of the reference) on the GPU:
same signature, validation and error classes; entries equal the reference's
dense operator (golden) to 1e-12 (P0) and the oracle's (P1c)."""

import numpy as np
import pytest

from conftest import golden


def _setup(fam="p0", eq="laplace", op="slp", k=0.0, level=2):
    from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space
    m = golden("meshes")
    v, e = m[f"ico{level}_vertices"], m[f"ico{level}_elements"]
    return v, e, OperatorSpec(eq, op, k), build_space(TriangleMesh(v, e), fam)


def test_split_work_matches_reference_rule():
    from paper_1711_01897_b200.assembly import split_work
    from paper_1711_01897_b200.errors import ConfigError
    assert split_work(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert split_work(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    with pytest.raises(ConfigError):
        split_work(5, 0)


def test_config_and_argument_errors():
    from paper_1711_01897_b200.assembly import AssemblyConfig, assemble_dense
    from paper_1711_01897_b200.errors import ConfigError
    with pytest.raises(ConfigError, match="workers"):
        AssemblyConfig(workers=0)
    v, e, spec, sp = _setup()
    with pytest.raises(ConfigError, match="at least one backend"):
        assemble_dense(spec, sp, sp, AssemblyConfig(), [])


@pytest.mark.gpu
def test_dense_p0_equals_reference_dense():
    from paper_1711_01897_b200.assembly import AssemblyConfig, assemble_dense
    from paper_1711_01897_b200.backend import make_gpu_backends
    from paper_1711_01897_b200.discretization import make_integration_context
    v, e, spec, sp = _setup()
    be = make_gpu_backends(make_integration_context(spec, sp, sp))
    stats = {}
    A = assemble_dense(spec, sp, sp, AssemblyConfig(), be, stats)
    ref = golden("hmatrices")["ico2_p0_lap_slp_dense"]
    assert np.abs(A - ref).max() <= 1e-12 * np.abs(ref).max()
    assert stats["pairs_total"] == len(e) ** 2 and stats["devices_used"] == 1
    assert stats["pairs_singular"] + stats["pairs_regular"] == len(e) ** 2


@pytest.mark.gpu
def test_dense_p1c_dlp_equals_oracle_and_capacity_error():
    from oracle import hbem_oracle as O
    from paper_1711_01897_b200.assembly import AssemblyConfig, assemble_dense
    from paper_1711_01897_b200.backend import make_gpu_backends
    from paper_1711_01897_b200.discretization import make_integration_context
    from paper_1711_01897_b200.errors import CapacityError
    v, e, spec, sp = _setup("p1c", "laplace", "dlp", 0.0, level=1)
    be = make_gpu_backends(make_integration_context(spec, sp, sp), 2)
    A = assemble_dense(spec, sp, sp, AssemblyConfig(), be)
    P = O.Problem(O.Spec("laplace", "dlp"), v, e, "p1c", "p1c")
    ref = O.assemble_dense(P)
    assert np.abs(A - ref).max() <= 1e-12 * np.abs(ref).max()
    with pytest.raises(CapacityError, match="bytes"):
        assemble_dense(spec, sp, sp, AssemblyConfig(max_matrix_bytes=8), be)


@pytest.mark.gpu
def test_dense_p1d_hull_with_poles_is_exact():
    """eta = 0 admits zero-diameter clusters (the hull's 40-valent poles give
    40 coincident P1d DOF centres, 126 such leaves); the dense sweep forces
    them dense, so the matrix is the exact Galerkin one."""
    from oracle import hbem_oracle as O
    from paper_1711_01897_b200.assembly import AssemblyConfig, assemble_dense
    from paper_1711_01897_b200.backend import make_gpu_backends
    from paper_1711_01897_b200.discretization import (OperatorSpec, TriangleMesh, build_space,
                                                      make_integration_context)
    from paper_1711_01897_b200.meshes import elongated_hull
    v, e = elongated_hull(40, 6)
    sp = build_space(TriangleMesh(v, e), "p1d")
    spec = OperatorSpec("helmholtz", "slp", 3.0)
    A = assemble_dense(spec, sp, sp, AssemblyConfig(),
                       make_gpu_backends(make_integration_context(spec, sp, sp)))
    ref = O.assemble_dense(O.Problem(O.Spec("helmholtz", "slp", 3.0), v, e, "p1d", "p1d"))
    assert np.abs(A - ref).max() <= 1e-12 * np.abs(ref).max()
