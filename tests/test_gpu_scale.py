"""GPU parity at scale through size-independent properties.

The reference cannot assemble 10^5-element H-matrices in test time, so the
large cases are checked against exact operator rows computed on the GPU by
the batched integrator (hbem_integrate_any = local_matrix over every pair),
which itself is pinned to the reference at 1e-12 by tests/test_gpu_integrate.py:

  * sampled rows of H x equal the exact (A x)_i within the ACA tolerance;
  * device matvec == host leaf-by-leaf matvec (hmatrix.py:441-470) to rounding;
  * two executes of one handle give bit-identical payloads (fixed reduction
    order, deterministic job lists);
  * FP32 assembly within 5e-4 of FP64 (FP32 is judged against FP64,
    SURVEY §8a row 7).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def problem(n_or_mesh, fam, eq, op, k, prec="double"):
    from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space
    from paper_1711_01897_b200.meshes import geodesic_sphere
    from paper_1711_01897_b200.partition import cluster_trees_for
    v, e = geodesic_sphere(n_or_mesh) if isinstance(n_or_mesh, int) else n_or_mesh
    spec = OperatorSpec(eq, op, k, prec)
    sp = build_space(TriangleMesh(v, e), fam)
    return v, e, spec, sp, cluster_trees_for(sp, sp)


def exact_rows(spec, sp, rows, x):
    """(A x)_i for DOFs i: every element pair carrying test DOF i, integrated
    by the GPU batched integrator (any adjacency), accumulated onto trial
    DOFs with the dofmap (_row_job, hmatrix.py:625-649)."""
    from paper_1711_01897_b200.backend import BatchRequest, make_gpu_backends
    from paper_1711_01897_b200.discretization import make_integration_context
    be = make_gpu_backends(make_integration_context(spec, sp, sp))[0]
    dm = np.asarray(sp.dofmap).reshape(len(sp.dofmap), -1)
    m = len(dm)
    out = []
    for i in rows:
        els, locs = np.nonzero(dm == i)
        acc = 0.0
        for el, a in zip(els, locs):
            pairs = np.stack([np.full(m, el), np.arange(m)], 1)
            res = be.integrate_pairs(BatchRequest(pairs))
            blk = res.complex_view()[:, a, :]           # (m, ns)
            acc = acc + (blk * x[dm]).sum()
        out.append(acc)
    return np.array(out)


@pytest.mark.parametrize("n,fam,eq,op,k,eps", [
    (45, "p0", "laplace", "slp", 0.0, 1e-3),      # C2 mesh size, C5 operator
    (100, "p0", "laplace", "slp", 0.0, 1e-3),     # 200 000 elements
    (45, "p0", "helmholtz", "slp", 10.0, 1e-4),
    (30, "p0", "laplace", "dlp", 0.0, 1e-4),
    (20, "p1c", "laplace", "dlp", 0.0, 1e-4),     # C2 operator/space
])
def test_sampled_rows_vs_exact_operator(n, fam, eq, op, k, eps):
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix
    v, e, spec, sp, bt = problem(n, fam, eq, op, k)
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=eps))
    rng = np.random.default_rng(1234)
    x = rng.standard_normal(sp.n_dofs)
    y = h.matvec(x)
    rows = rng.choice(sp.n_dofs, size=8, replace=False)
    z = exact_rows(spec, sp, rows, x)
    scale = np.sqrt(np.mean(np.abs(y) ** 2))
    err = np.abs(y[rows] - z).max() / scale
    assert err <= 10 * eps, err


@pytest.mark.parametrize("fam,eq,op,k", [("p0", "laplace", "slp", 0.0),
                                         ("p0", "helmholtz", "slp", 4.0),
                                         ("p1c", "laplace", "dlp", 0.0)])
def test_device_matvec_equals_host_matvec(fam, eq, op, k):
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix, hmat_matvec
    v, e, spec, sp, bt = problem(12, fam, eq, op, k)
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=1e-5))
    x = np.random.default_rng(7).standard_normal(sp.n_dofs)
    yd = hmat_matvec(h, x, device=True)
    yh = hmat_matvec(h, x, device=False)
    assert np.abs(yd - yh).max() <= 1e-12 * np.abs(yh).max()


def test_execute_is_bitwise_deterministic():
    from paper_1711_01897_b200.backend import init_gpu_device
    from paper_1711_01897_b200.discretization import make_integration_context
    from paper_1711_01897_b200.hmatrix import AcaConfig, AssemblyConfig, _assemble_part
    v, e, spec, sp, bt = problem(40, "p0", "laplace", "slp", 0.0)
    dev = init_gpu_device(make_integration_context(spec, sp, sp))
    part = _assemble_part(dev, bt, np.arange(len(bt.leaf_array)), sp, sp,
                          AcaConfig(epsilon=1e-3), AssemblyConfig())
    a1 = [np.array(a, copy=True) for a in part.arenas()]
    meta1 = (part.kind.copy(), part.rank.copy(), part.off_u.copy(), part.off_d.copy())
    part.execute()
    a2 = part.arenas()
    assert all(np.array_equal(p, q) for p, q in zip(a1, a2))
    assert all(np.array_equal(p, q) for p, q in
               zip(meta1, (part.kind, part.rank, part.off_u, part.off_d)))
    part.close()


def test_single_precision_at_scale_vs_double():
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix
    _, _, s64, sp, bt = problem(45, "p0", "laplace", "slp", 0.0)
    _, _, s32, _, _ = problem(45, "p0", "laplace", "slp", 0.0, "single")
    x = np.random.default_rng(3).standard_normal(sp.n_dofs)
    y64 = assemble_hmatrix(s64, sp, sp, bt, AcaConfig(epsilon=1e-4)).matvec(x)
    y32 = assemble_hmatrix(s32, sp, sp, bt, AcaConfig(epsilon=1e-4)).matvec(x)
    assert np.linalg.norm(y32 - y64) <= 5e-4 * np.linalg.norm(y64)


def test_hull_mesh_assembly_vs_exact_rows():
    """Elongated hull (C4 geometry class): Helmholtz SLP P0 rows."""
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix
    from paper_1711_01897_b200.meshes import elongated_hull
    v, e = elongated_hull(48, 160)
    _, _, spec, sp, bt = problem((v, e), "p0", "helmholtz", "slp", 6.0)
    eps = 1e-4
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=eps))
    rng = np.random.default_rng(11)
    x = rng.standard_normal(sp.n_dofs)
    y = h.matvec(x)
    rows = rng.choice(sp.n_dofs, size=6, replace=False)
    z = exact_rows(spec, sp, rows, x)
    assert np.abs(y[rows] - z).max() <= 10 * eps * np.sqrt(np.mean(np.abs(y) ** 2))


def test_hull_hmatrix_matches_reference():
    """Golden from the real reference (tests/golden/make_hull_golden.py):
    elongated hull, Helmholtz SLP P0, 8 elements per wavelength, eps 1e-3.
    Same ACA pivots => the device H-matrix matvec equals the reference's
    H-matrix matvec to rounding (the ACA error itself is ~6e-3 here)."""
    from conftest import golden
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix
    from paper_1711_01897_b200.meshes import elongated_hull
    g = golden("hull")
    v, e = elongated_hull(int(g["n_around"]), int(g["n_along"]))
    _, _, spec, sp, bt = problem((v, e), "p0", "helmholtz", "slp", float(g["k"]))
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=float(g["eps"])))
    for x, yr in zip(g["x"], g["y"]):
        y = h.matvec(x)
        assert np.abs(y - yr).max() <= 1e-10 * np.abs(yr).max()


@pytest.mark.parametrize("eq,k,zc", [("laplace", 0.0, "1"), ("laplace", 0.0, "0"),
                                     ("helmholtz", 5.0, "1")])
def test_streamed_payloads_equal_deferred_copy(monkeypatch, eq, k, zc):
    """Payloads streamed during the assembly into page-locked host arenas
    (zero-copy emission kernel, or the staged copy-engine path with
    HBEM_ZEROCOPY=0) equal the deferred hbem_hmat_copy_arenas payloads bit for
    bit, leaf by leaf (the streamed arenas are in convergence order), also
    after a re-execute of the streamed handle and after a later on-demand
    copy_arenas of it."""
    from paper_1711_01897_b200.backend import init_gpu_device
    from paper_1711_01897_b200.discretization import make_integration_context
    from paper_1711_01897_b200.hmatrix import (AcaConfig, AssemblyConfig, _assemble_part,
                                               pinned_empty)
    monkeypatch.setenv("HBEM_ZEROCOPY", zc)
    v, e, spec, sp, bt = problem(30, "p0", eq, "slp", k)
    dev = init_gpu_device(make_integration_context(spec, sp, sp))
    ids = np.arange(len(bt.leaf_array))
    cfg, acfg = AcaConfig(epsilon=1e-4), AssemblyConfig()
    ref = _assemble_part(dev, bt, ids, sp, sp, cfg, acfg)
    s = ref.stats
    dt = ref.arenas()[0].dtype
    out = tuple(pinned_empty(s[n] + 17, dt) for n in ("u_entries", "v_entries", "dense_entries"))
    part = _assemble_part(dev, bt, ids, sp, sp, cfg, acfg, out=out)

    def same_payloads():
        n_lr = 0
        for q in range(len(ids)):
            a, b = ref.payload(q), part.payload(q)
            assert type(a) is type(b)
            if hasattr(a, "u"):
                n_lr += 1
                assert np.array_equal(a.u, b.u) and np.array_equal(a.v, b.v), q
            else:
                assert np.array_equal(a.a, b.a), q
        assert n_lr > 0

    same_payloads()
    for a in out:
        a[:] = 0
    part.execute()
    same_payloads()
    # on-demand copy of the same handle (device U / V packed here after a
    # zero-copy run)
    part._arenas = None
    part._streamed = False
    same_payloads()
    part.close()
    ref.close()


@pytest.mark.parametrize("name", ["hull_mid", "hull_125k"])
def test_hull_mid_matches_reference(name):
    """C4 accuracy question (tests/golden/make_hull_mid_golden.py): on 31k- and
    126k-triangle hulls (Helmholtz SLP P0, 8 elements per wavelength, eps 1e-3)
    the reference's OWN H-matrix misses the exact operator rows by 8e-3..9e-3
    (31k) and 0.039..0.097 (126k), growing with the mesh like the 0.1 of the
    504k C4 hull.  The GPU assembly follows the same pivots (its matvec equals
    the reference's H-matrix matvec to rounding) and therefore reproduces that
    error: the C4 error is the reference ACA's behaviour on thin bodies at this
    tolerance, not a device defect."""
    import os
    from conftest import GOLDEN, golden
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix
    from paper_1711_01897_b200.meshes import elongated_hull
    if not os.path.exists(os.path.join(GOLDEN, f"{name}.npz")):
        pytest.skip(f"{name}.npz not generated")
    g = golden(name)
    v, e = elongated_hull(int(g["n_around"]), int(g["n_along"]))
    _, _, spec, sp, bt = problem((v, e), "p0", "helmholtz", "slp", float(g["k"]))
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=float(g["eps"])))
    keep = g["y_rows"] if "y_rows" in g else np.arange(sp.n_dofs)
    for t, (x, yr) in enumerate(zip(g["x"], g["y"])):
        y = h.matvec(x)
        assert np.abs(y[keep] - yr).max() <= 1e-10 * np.abs(yr).max()
        # the same sampled-row error as the reference's H-matrix
        scale = np.sqrt(np.mean(np.abs(y) ** 2))
        err = np.abs(y[g["rows"]] - g["exact"][t]).max() / scale
        assert abs(err - g["ref_err"][t]) <= 1e-6, (err, g["ref_err"][t])


@pytest.mark.parametrize("fam,eq,op,k,prec", [("p0", "laplace", "slp", 0.0, "double"),
                                              ("p0", "helmholtz", "slp", 4.0, "double"),
                                              ("p1c", "laplace", "dlp", 0.0, "single")])
def test_device_matvec_is_bitwise_reproducible(fam, eq, op, k, prec):
    """No float atomics: repeated device matvecs (host and device-pointer
    entry points) return identical bits (hmatrix.py:441-446 promise)."""
    import torch
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix, hmat_matvec
    v, e, spec, sp, bt = problem(30, fam, eq, op, k, prec)
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=1e-4))
    rd = np.dtype(spec.result_dtype)
    x = np.random.default_rng(9).standard_normal(sp.n_dofs).astype(rd)
    y1 = hmat_matvec(h, x)
    y2 = hmat_matvec(h, x)
    assert np.array_equal(y1, y2)
    part = h.parts[0][1]
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
           np.dtype(np.complex128): torch.complex128, np.dtype(np.complex64): torch.complex64}[rd]
    xd = torch.from_numpy(x).to("cuda")
    yd = torch.empty(sp.n_dofs, dtype=tdt, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(2):
        part.matvec_device(xd.data_ptr(), yd.data_ptr(), s.cuda_stream)
        s.synchronize()
        assert np.array_equal(yd.cpu().numpy(), y1)
    yh = hmat_matvec(h, x, device=False)
    assert np.abs(y1 - yh).max() <= (1e-12 if prec == "double" else 1e-5) * np.abs(yh).max()


def test_matvec_promotes_like_the_reference():
    """float32 H-matrix times a float64 vector returns float64
    (np.result_type(h.dtype, x.dtype), hmatrix.py:455)."""
    from paper_1711_01897_b200.hmatrix import AcaConfig, assemble_hmatrix, hmat_matvec
    v, e, spec, sp, bt = problem(10, "p0", "laplace", "slp", 0.0, "single")
    h = assemble_hmatrix(spec, sp, sp, bt, AcaConfig(epsilon=1e-4))
    x = np.random.default_rng(2).standard_normal(sp.n_dofs)
    assert hmat_matvec(h, x).dtype == np.float64
    assert hmat_matvec(h, x.astype(np.complex128)).dtype == np.complex128
    assert hmat_matvec(h, x.astype(np.float32)).dtype == np.float32
