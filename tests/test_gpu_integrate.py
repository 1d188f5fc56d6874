"""GPU parity of the C-ABI pair integrators against the reference golden
vectors and the CPU oracle (K1 regular 6x6 rule, K2 Sauter-Schwab).

Tolerances (block-max normalised, as test_backend.py:156-158 /
test_acceptance.py:218-221 of the reference):
  FP64 entries            <= 1e-12 relative  (north star)
  FP32 entries vs FP64    <= 1e-5 relative for SLP, 5e-4 for the rest
                          (the reference's own FP32 budget,
                          test_acceptance.py:225)
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import golden
from oracle import hbem_oracle as O

pytestmark = pytest.mark.gpu

COMBOS = [
    (eq, k, op, fam)
    for eq, k in (("laplace", 0.0), ("helmholtz", 2.0))
    for op in ("slp", "dlp", "adlp", "hyps")
    for fam in ("p0", "p1c", "p1d")
    if not (op == "hyps" and fam == "p0")
]


def ico(level):
    m = golden("meshes")
    return m[f"ico{level}_vertices"], m[f"ico{level}_elements"]


def make_ctx(v, e, eq, op, k, fam, prec="double"):
    from paper_1711_01897_b200.discretization import (OperatorSpec, TriangleMesh, build_space,
                                                      make_integration_context)
    sp = build_space(TriangleMesh(v, e), fam)
    return make_integration_context(OperatorSpec(eq, op, k, prec), sp, sp)


def backend(ctx):
    from paper_1711_01897_b200.backend import make_gpu_backends
    return make_gpu_backends(ctx)[0]


def rel_err(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    scale = np.abs(ref).reshape(len(ref), -1).max(axis=1)
    # blocks whose exact value is 0 (identical-pair DLP on a flat triangle:
    # <x - y, n> = 0) are pure roundoff ~1e-18; normalise blocks below 1% of
    # the batch maximum by 1% of that maximum
    scale = np.maximum(scale, 1e-2 * scale.max())
    diff = np.abs(got - ref).reshape(len(ref), -1).max(axis=1)
    return float((diff / scale).max())


def disjoint_pairs(e, n, rng):
    out = []
    while len(out) < n:
        cand = rng.integers(0, len(e), size=(4 * n, 2))
        ok = ~(e[cand[:, 0]][:, :, None] == e[cand[:, 1]][:, None, :]).any(axis=(1, 2))
        out.extend(map(tuple, cand[ok]))
    return np.array(out[:n], dtype=np.int64)


def test_device_geometry_bitwise_equals_numpy():
    from paper_1711_01897_b200.meshes import geodesic_sphere
    v, e = geodesic_sphere(11)
    be = backend(make_ctx(v, e, "laplace", "slp", 0.0, "p0"))
    q, n, j = be.context.geometry()
    P = O.Problem(O.Spec("laplace", "slp"), v, e)
    assert np.array_equal(j, P.jac)
    assert np.array_equal(n, P.normals)
    assert np.array_equal(q, P.qpoints)


@pytest.mark.parametrize("eq,k,op,fam", COMBOS)
def test_integrate_batch_vs_reference_golden(eq, k, op, fam):
    from paper_1711_01897_b200.backend import BatchRequest
    g = golden("integrals")
    v, e = ico(2)
    pairs = g["regular_pairs"]
    tag = f"{eq}_{op}_{fam}"
    ref64 = g[f"{tag}_double_re"] + (1j * g[f"{tag}_double_im"] if eq == "helmholtz" else 0)
    be = backend(make_ctx(v, e, eq, op, k, fam, "double"))
    res = be.integrate_batch(BatchRequest(pairs))
    assert res.re.dtype == np.float64
    assert (res.im is None) == (eq == "laplace")
    assert rel_err(res.complex_view(), ref64) <= 1e-12
    be32 = backend(make_ctx(v, e, eq, op, k, fam, "single"))
    res32 = be32.integrate_batch(BatchRequest(pairs))
    assert res32.re.dtype == np.float32
    tol = 1e-5 if op == "slp" else 5e-4
    assert rel_err(res32.complex_view().astype(np.complex128), ref64) <= tol
    # native single arithmetic, not double rounded
    assert not np.array_equal(res32.re, res.re.astype(np.float32))


@pytest.mark.parametrize("eq,k,op,fam", COMBOS)
def test_touching_pairs_vs_reference_local_matrix(eq, k, op, fam):
    from paper_1711_01897_b200.backend import BatchRequest
    g = golden("integrals")
    v, e = ico(1)
    pairs = g["singular_pairs"]
    ref = g[f"{eq}_{op}_{fam}_double_local"]
    be = backend(make_ctx(v, e, eq, op, k, fam))
    res = be.integrate_pairs(BatchRequest(pairs))
    assert be.singular_served == len(pairs)
    assert rel_err(res.complex_view(), ref) <= 1e-12


def test_mixed_batch_any_kind_vs_oracle(rng):
    """regular + touching pairs in one request, P1c Helmholtz DLP."""
    from paper_1711_01897_b200.backend import BatchRequest
    v, e = ico(2)
    touch = np.array([(a, b) for a in range(0, 320, 37) for b in range(320)
                      if set(e[a]) & set(e[b])])
    pairs = np.concatenate([disjoint_pairs(e, 300, rng), touch])
    rng.shuffle(pairs)
    be = backend(make_ctx(v, e, "helmholtz", "dlp", 2.0, "p1c"))
    res = be.integrate_pairs(BatchRequest(pairs))
    P = O.Problem(O.Spec("helmholtz", "dlp", 2.0), v, e, "p1c", "p1c")
    ref = np.stack([O.local_matrix(P, int(a), int(b)) for a, b in pairs])
    assert rel_err(res.complex_view(), ref) <= 1e-12


def test_ten_thousand_pairs_c1_mesh_vs_oracle(rng):
    """test_acceptance.py:194-226 at the C1 mesh (geodesic n=11, 2 420 tri)."""
    from paper_1711_01897_b200.backend import BatchRequest
    from paper_1711_01897_b200.meshes import geodesic_sphere
    v, e = geodesic_sphere(11)
    pairs = disjoint_pairs(e, 10_000, rng)
    P = O.Problem(O.Spec("laplace", "slp"), v, e)
    ref, _ = O.integrate_batch(P, pairs)
    be = backend(make_ctx(v, e, "laplace", "slp", 0.0, "p0"))
    res = be.integrate_batch(BatchRequest(pairs))
    assert rel_err(res.re, ref) <= 1e-12
    be32 = backend(make_ctx(v, e, "laplace", "slp", 0.0, "p0", "single"))
    res32 = be32.integrate_batch(BatchRequest(pairs))
    assert rel_err(res32.re.astype(np.float64), ref) <= 1e-5
    # split invariance, bit for bit
    cuts = [0, *sorted(rng.integers(1, 10_000, size=7)), 10_000]
    parts = [be.integrate_batch(BatchRequest(pairs[lo:hi])).re for lo, hi in zip(cuts[:-1], cuts[1:])]
    assert np.array_equal(np.concatenate(parts), res.re)
    # concurrent submission, bit for bit
    quarters = [BatchRequest(pairs[i::4]) for i in range(4)]
    with ThreadPoolExecutor(max_workers=4) as pool:
        got = list(pool.map(lambda r: be.integrate_batch(r).re, quarters))
    for i, gq in enumerate(got):
        assert np.array_equal(gq, res.re[i::4])
    assert be.batches_served == 1 + 8 + 4
    assert be.pairs_served == 30_000


def test_identical_contexts_identical_bits(rng):
    from paper_1711_01897_b200.backend import BatchRequest, make_gpu_backends
    v, e = ico(2)
    b0, b1, b2 = make_gpu_backends(make_ctx(v, e, "helmholtz", "dlp", 2.0, "p0"), n_devices=3)
    assert [b.device_id for b in (b0, b1, b2)] == [0, 1, 2]
    req = BatchRequest(disjoint_pairs(e, 100, rng))
    r0, r1 = b0.integrate_batch(req), b2.integrate_batch(req)
    assert np.array_equal(r0.re, r1.re) and np.array_equal(r0.im, r1.im)


def test_contract_violations():
    from paper_1711_01897_b200.backend import BatchRequest
    from paper_1711_01897_b200.errors import ContractViolationError
    v, e = ico(1)
    be = backend(make_ctx(v, e, "laplace", "slp", 0.0, "p0"))
    with pytest.raises(ContractViolationError, match="not disjoint"):
        be.integrate_batch(BatchRequest(np.array([[3, 3]])))
    shared = next((a, b) for a in range(4) for b in range(len(e))
                  if a != b and set(e[a]) & set(e[b]))
    with pytest.raises(ContractViolationError, match=r"request pair 1 = .* is not disjoint"):
        be.integrate_batch(BatchRequest(np.array([[0, 40], list(shared)])))
    n = len(e)
    with pytest.raises(ContractViolationError, match="indices"):
        be.integrate_batch(BatchRequest(np.array([[0, n]])))
    with pytest.raises(ContractViolationError, match="indices"):
        be.integrate_batch(BatchRequest(np.array([[-1, 4]])))
    res = be.integrate_batch(BatchRequest(np.zeros((0, 2), np.int64)))
    assert res.re.shape == (0, 1, 1)
    assert be.integrate_batch(BatchRequest(np.array([[0, 40]]), offsets=np.array([7]))).offsets[0] == 7


def test_capacity_error_on_seven_weights():
    from dataclasses import replace
    from paper_1711_01897_b200.backend import make_gpu_backends
    from paper_1711_01897_b200.discretization import BasisTable, QuadratureRule
    from paper_1711_01897_b200.errors import CapacityError
    v, e = ico(0)
    ctx = make_ctx(v, e, "laplace", "slp", 0.0, "p0")
    pts = np.vstack([[1 / 3, 1 / 3], [[0.3, 0.1]] * 6])
    rule = QuadratureRule(pts, np.array([0.05] + [0.075] * 6), 1)
    bad = replace(ctx, regular_rule=rule, test_table=BasisTable(np.ones((1, 7))),
                  trial_table=BasisTable(np.ones((1, 7))))
    with pytest.raises(CapacityError, match="7 weights"):
        make_gpu_backends(bad)


def test_lower_order_rule_padding(rng):
    """order-2 (3-point) rule: zero-weight padding leaves results unchanged."""
    from dataclasses import replace
    from paper_1711_01897_b200.backend import BatchRequest
    from paper_1711_01897_b200.discretization import basis_table, regular_rule
    v, e = ico(2)
    ctx = make_ctx(v, e, "laplace", "dlp", 0.0, "p1c")
    r2 = regular_rule(2)
    ctx2 = replace(ctx, regular_rule=r2, test_table=basis_table(ctx.test_space, r2),
                   trial_table=basis_table(ctx.trial_space, r2))
    pairs = disjoint_pairs(e, 200, rng)
    res = backend(ctx2).integrate_batch(BatchRequest(pairs))
    P = O.Problem(O.Spec("laplace", "dlp"), v, e, "p1c", "p1c", regular_order=2)
    ref, _ = O.integrate_batch(P, pairs)
    assert rel_err(res.re, ref) <= 1e-12
