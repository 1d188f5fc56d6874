"""Host-side discretisation data: operator spec, mesh, spaces, quadrature
rules and the integration context handed to the GPU backend.

Mirrors the reference's public surface for this path (names, attributes,
validation and error classes), so a GpuBackend built from either this
``IntegrationContext`` or the reference's
(`/root/reference/pkg/src/hbem/kernels.py:161-227`) behaves identically:

  OperatorSpec               kernels.py:54-96
  TriangleMesh               mesh.py:37-101 (validation subset)
  FunctionSpace/build_space  spaces.py:47-93 (dofmaps, dof_centers)
  regular_rule               quadrature.py:84-116
  singular_rule(s)           quadrature.py:274-312
  make_integration_context   kernels.py:199-227

Geometry caches are NOT precomputed on the host here: the device computes
them from vertices/elements (hbem_ctx_create with NULL caches) with the
numpy operation order, so a reference context and this one stage
bit-identical device caches.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field, replace
from functools import cached_property, lru_cache

import numpy as np

from .errors import KernelError, MeshError, QuadratureError, SpaceError

EQUATIONS = ("laplace", "helmholtz")
OPERATORS = ("slp", "dlp", "adlp", "hyps")
PRECISIONS = ("double", "single")
_TRANSPOSED = {"slp": "slp", "dlp": "adlp", "adlp": "dlp", "hyps": "hyps"}


@dataclass(frozen=True)
class OperatorSpec:
    equation: str
    operator: str
    wavenumber: float = 0.0
    precision: str = "double"

    def __post_init__(self):
        if self.equation not in EQUATIONS:
            raise KernelError(f"unknown equation {self.equation!r}, expected {EQUATIONS}")
        if self.operator not in OPERATORS:
            raise KernelError(f"unknown operator {self.operator!r}, expected {OPERATORS}")
        if self.precision not in PRECISIONS:
            raise KernelError(f"unknown precision {self.precision!r}, expected {PRECISIONS}")
        k = self.wavenumber
        if not np.isfinite(k):
            raise KernelError(f"wavenumber must be finite, got {k!r}")
        if self.equation == "laplace" and k != 0.0:
            raise KernelError("laplace kernels require wavenumber 0")
        if self.equation == "helmholtz" and k <= 0.0:
            raise KernelError(f"helmholtz kernels require a positive wavenumber, got {k}")

    @property
    def is_complex(self) -> bool:
        return self.equation == "helmholtz"

    @property
    def real_dtype(self) -> np.dtype:
        return np.dtype(np.float64 if self.precision == "double" else np.float32)

    @property
    def result_dtype(self) -> np.dtype:
        if self.is_complex:
            return np.dtype(np.complex128 if self.precision == "double" else np.complex64)
        return self.real_dtype

    @property
    def transposed(self) -> "OperatorSpec":
        return replace(self, operator=_TRANSPOSED[self.operator])


@dataclass(frozen=True)
class TriangleMesh:
    """Immutable triangle mesh: (nv, 3) float64 vertices, (m, 3) int64 elements."""

    vertices: np.ndarray
    elements: np.ndarray
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        v = np.ascontiguousarray(self.vertices, dtype=np.float64)
        e = np.ascontiguousarray(self.elements, dtype=np.int64)
        if v.ndim != 2 or v.shape[1] != 3:
            raise MeshError(f"vertices must have shape (n, 3), got {v.shape}")
        if e.ndim != 2 or e.shape[1] != 3:
            raise MeshError(f"elements must have shape (m, 3), got {e.shape}")
        if e.size and (e.min() < 0 or e.max() >= len(v)):
            raise MeshError(f"element indices must lie in [0, {len(v)}), "
                            f"found range [{e.min()}, {e.max()}]")
        for k in range(3):
            same = e[:, k] == e[:, (k + 1) % 3]
            if same.any():
                i = int(np.nonzero(same)[0][0])
                raise MeshError(f"element {i} repeats vertex index {e[i, k]}")
        v.setflags(write=False)
        e.setflags(write=False)
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "elements", e)

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_elements(self) -> int:
        return len(self.elements)


class Family(enum.Enum):
    P0 = "p0"
    P1_CONTINUOUS = "p1c"
    P1_DISCONTINUOUS = "p1d"


@dataclass(frozen=True)
class FunctionSpace:
    family: Family
    mesh: TriangleMesh
    dofmap: np.ndarray
    n_dofs: int

    @property
    def local_dim(self) -> int:
        return self.dofmap.shape[1]

    @cached_property
    def dof_centers(self) -> np.ndarray:
        """spaces.py:67-78 — same numpy expression, so bit-identical."""
        v = self.mesh.vertices
        if self.family is Family.P0:
            return v[self.mesh.elements].mean(axis=1)
        if self.family is Family.P1_CONTINUOUS:
            return v.copy()
        return v[self.mesh.elements].reshape(-1, 3)


def build_space(mesh: TriangleMesh, family) -> FunctionSpace:
    if not isinstance(family, Family):
        try:
            family = Family(family)
        except ValueError:
            raise SpaceError(f"unknown space family {family!r}") from None
    m = mesh.n_elements
    if family is Family.P0:
        dm, n = np.arange(m, dtype=np.int64)[:, None], m
    elif family is Family.P1_CONTINUOUS:
        dm, n = mesh.elements.copy(), mesh.n_vertices
    else:
        dm, n = np.arange(3 * m, dtype=np.int64).reshape(m, 3), 3 * m
    dm.setflags(write=False)
    return FunctionSpace(family, mesh, dm, n)


@dataclass(frozen=True)
class QuadratureRule:
    points: np.ndarray
    weights: np.ndarray
    order: int

    def __len__(self):
        return len(self.weights)


@lru_cache(maxsize=None)
def regular_rule(order: int = 4) -> QuadratureRule:
    """Symmetric triangle rules of quadrature.py:84-116 (orders 1..4)."""
    if order == 1:
        pts, wts = [[1 / 3, 1 / 3]], [0.5]
    elif order == 2:
        pts, wts = [[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]], [1 / 6] * 3
    elif order == 3:
        roots = (0.659027622374092, 0.231933368553031, 0.109039009072877)
        pts = sorted({(roots[j], roots[k]) for i in range(3) for j in range(3)
                      for k in range(3) if len({i, j, k}) == 3})
        wts = [1 / 12] * 6
    elif order == 4:
        pts, wts = [], []
        for beta, w in ((0.445948490915965, 0.223381589678011),
                        (0.091576213509771, 0.109951743655322)):
            alpha = 1.0 - 2.0 * beta
            pts += [(beta, beta), (alpha, beta), (beta, alpha)]
            wts += [0.5 * w] * 3
    else:
        raise QuadratureError(f"unsupported quadrature order {order}, expected 1..4")
    p = np.array(pts, dtype=np.float64)
    w = np.array(wts, dtype=np.float64)
    p.setflags(write=False)
    w.setflags(write=False)
    return QuadratureRule(p, w, order)


class PairKind(enum.Enum):
    DISJOINT = "disjoint"
    SHARED_VERTEX = "shared_vertex"
    SHARED_EDGE = "shared_edge"
    IDENTICAL = "identical"


SINGULAR_KINDS = (PairKind.SHARED_VERTEX, PairKind.SHARED_EDGE, PairKind.IDENTICAL)


@dataclass(frozen=True)
class TensorRule:
    points: np.ndarray   # (n, 4)
    weights: np.ndarray  # (n,)
    kind: PairKind
    n_subdomains: int
    base_order: int

    def __len__(self):
        return len(self.weights)


def _maps(kind, xi, e1, e2, e3):
    """Regularising subdomain maps (quadrature.py:237-271), simplex coords."""
    if kind is PairKind.IDENTICAL:
        j = xi ** 3 * e1 ** 2 * e2
        a = ((xi, xi * (1 - e1 + e1 * e2)), (xi * (1 - e1 * e2 * e3), xi * (1 - e1)))
        b = ((xi, xi * e1 * (1 - e2 + e2 * e3)), (xi * (1 - e1 * e2), xi * e1 * (1 - e2)))
        c = ((xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), (xi, xi * e1 * (1 - e2)))
        return [(a[0], a[1], j), (a[1], a[0], j), (b[0], b[1], j), (b[1], b[0], j),
                (c[0], c[1], j), (c[1], c[0], j)]
    if kind is PairKind.SHARED_EDGE:
        ja = xi ** 3 * e1 ** 2
        jb = ja * e2
        return [((xi, xi * e1 * e3), (xi * (1 - e1 * e2), xi * e1 * (1 - e2)), ja),
                ((xi, xi * e1), (xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), jb),
                ((xi * (1 - e1 * e2), xi * e1 * (1 - e2)), (xi, xi * e1 * e2 * e3), jb),
                ((xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), (xi, xi * e1), jb),
                ((xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), (xi, xi * e1 * e2), jb)]
    j = xi ** 3 * e2
    u, v = (xi, xi * e1), (xi * e2, xi * e2 * e3)
    return [(u, v, j), (v, u, j)]


@lru_cache(maxsize=None)
def singular_rule(kind: PairKind, base_order: int = 4) -> TensorRule:
    if kind not in SINGULAR_KINDS:
        raise QuadratureError(f"no singular rule for pair kind {kind!r}")
    if base_order < 2:
        raise QuadratureError(f"base_order must be an integer >= 2, got {base_order!r}")
    x, w = np.polynomial.legendre.leggauss(int(base_order))
    x, w = 0.5 * (x + 1.0), 0.5 * w
    xi, e1, e2, e3 = (g.ravel() for g in np.meshgrid(x, x, x, x, indexing="ij"))
    w4 = (w[:, None, None, None] * w[None, :, None, None]
          * w[None, None, :, None] * w[None, None, None, :]).ravel()
    maps = _maps(kind, xi, e1, e2, e3)
    pts = np.concatenate([np.column_stack([u1 - u2, u2, v1 - v2, v2])
                          for (u1, u2), (v1, v2), _ in maps])
    wts = np.concatenate([w4 * jac for _, _, jac in maps])
    pts.setflags(write=False)
    wts.setflags(write=False)
    return TensorRule(pts, wts, kind, len(maps), int(base_order))


def singular_rules(base_order: int = 4) -> dict:
    return {k: singular_rule(k, base_order) for k in SINGULAR_KINDS}


@dataclass(frozen=True)
class BasisTable:
    values: np.ndarray  # (local_dim, q)


def basis_table(space: FunctionSpace, rule: QuadratureRule) -> BasisTable:
    if space.family is Family.P0:
        v = np.ones((1, len(rule)))
    else:
        xi, eta = rule.points[:, 0], rule.points[:, 1]
        v = np.stack([1.0 - xi - eta, xi, eta])
    return BasisTable(np.ascontiguousarray(v))


@dataclass(frozen=True)
class IntegrationContext:
    """Attribute-compatible with the reference IntegrationContext
    (kernels.py:161-196).  ``geometry``/``curls`` are None: the device
    computes them (see module docstring)."""

    spec: OperatorSpec
    mesh: TriangleMesh
    test_space: FunctionSpace
    trial_space: FunctionSpace
    test_table: BasisTable
    trial_table: BasisTable
    regular_rule: QuadratureRule
    singular: dict
    geometry: object = None
    curls: object = None


def make_integration_context(spec: OperatorSpec, test_space: FunctionSpace,
                             trial_space: FunctionSpace, regular_order: int = 4,
                             singular_base_order: int = 4) -> IntegrationContext:
    if test_space.mesh is not trial_space.mesh:
        raise KernelError("test and trial spaces must share one mesh")
    if spec.operator == "hyps" and Family.P0 in (test_space.family, trial_space.family):
        raise KernelError("hyps requires linear test and trial spaces")
    rule = regular_rule(regular_order)
    return IntegrationContext(
        spec=spec, mesh=test_space.mesh, test_space=test_space, trial_space=trial_space,
        test_table=basis_table(test_space, rule), trial_table=basis_table(trial_space, rule),
        regular_rule=rule, singular=singular_rules(singular_base_order))
