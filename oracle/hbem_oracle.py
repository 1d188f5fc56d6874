"""CPU ORACLE — test infrastructure only, never the product path.

A plain-numpy restatement of the reference's hot path (package ``hbem``
under ``/root/reference/pkg/src/hbem``), used as the parity checker for the
CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.

Parity pinning: this module is checked against golden vectors produced by
the *real* reference imported in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; test
``tests/test_oracle_golden.py``).  The reference has no stored vectors of
its own, so these generated fixtures are the pin.

Every function cites the reference ``file:line`` it restates.  Third-party
arithmetic the reference relies on: numpy (einsum, sqrt, cos, sin,
argsort(kind="stable"), unique, linalg.norm) and
``numpy.polynomial.legendre.leggauss`` (`quadrature.py:286`); unpinned by
the reference (`pkg/pyproject.toml:10`), here numpy 2.3.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

INV_4PI = 1.0 / (4.0 * np.pi)
TRANSPOSED = {"slp": "slp", "dlp": "adlp", "adlp": "dlp", "hyps": "hyps"}


# ---------------------------------------------------------------------------
# operator description                               kernels.py:54-96
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Spec:
    equation: str
    operator: str
    wavenumber: float = 0.0
    precision: str = "double"

    @property
    def is_complex(self):
        return self.equation == "helmholtz"

    @property
    def real_dtype(self):
        return np.dtype(np.float64 if self.precision == "double" else np.float32)

    @property
    def result_dtype(self):
        if self.is_complex:
            return np.dtype(np.complex128 if self.precision == "double" else np.complex64)
        return self.real_dtype

    @property
    def transposed(self):
        return Spec(self.equation, TRANSPOSED[self.operator], self.wavenumber, self.precision)


# ---------------------------------------------------------------------------
# quadrature                                          quadrature.py:27-116, 237-307
# ---------------------------------------------------------------------------

def regular_rule(order: int = 4):
    """(points (q,2), weights (q,)) — quadrature.py:84-116."""
    if order == 1:
        return np.array([[1 / 3, 1 / 3]]), np.array([0.5])
    if order == 2:
        return (np.array([[1 / 6, 1 / 6], [2 / 3, 1 / 6], [1 / 6, 2 / 3]]),
                np.full(3, 1 / 6))
    if order == 3:
        roots = (0.659027622374092, 0.231933368553031, 0.109039009072877)
        perms = set()
        for i in range(3):
            for j in range(3):
                for k in range(3):
                    if len({i, j, k}) == 3:
                        perms.add((roots[j], roots[k]))
        return np.array(sorted(perms)), np.full(6, 1 / 12)
    if order == 4:
        pts, wts = [], []
        for beta, w in ((0.445948490915965, 0.223381589678011),
                        (0.091576213509771, 0.109951743655322)):
            alpha = 1.0 - 2.0 * beta
            # barycentric orbit order (a,b,b), (b,a,b), (b,b,a) -> (xi, eta) = (l1, l2)
            for l1, l2 in ((beta, beta), (alpha, beta), (beta, alpha)):
                pts.append((l1, l2))
                wts.append(0.5 * w)
        return np.array(pts), np.array(wts)
    raise ValueError(f"unsupported order {order}")


class Kind(enum.IntEnum):
    DISJOINT = 0
    SHARED_VERTEX = 1
    SHARED_EDGE = 2
    IDENTICAL = 3


def _subdomains(kind, xi, e1, e2, e3):
    """Regularising maps (u, v, jacobian) — quadrature.py:237-271."""
    if kind == Kind.IDENTICAL:
        jac = xi ** 3 * e1 ** 2 * e2
        pairs = [
            ((xi, xi * (1 - e1 + e1 * e2)), (xi * (1 - e1 * e2 * e3), xi * (1 - e1))),
            ((xi, xi * e1 * (1 - e2 + e2 * e3)), (xi * (1 - e1 * e2), xi * e1 * (1 - e2))),
            ((xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), (xi, xi * e1 * (1 - e2))),
        ]
        out = []
        for u, v in pairs:
            out += [(u, v, jac), (v, u, jac)]
        return out
    if kind == Kind.SHARED_EDGE:
        ja = xi ** 3 * e1 ** 2
        jb = xi ** 3 * e1 ** 2 * e2
        return [
            ((xi, xi * e1 * e3), (xi * (1 - e1 * e2), xi * e1 * (1 - e2)), ja),
            ((xi, xi * e1), (xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), jb),
            ((xi * (1 - e1 * e2), xi * e1 * (1 - e2)), (xi, xi * e1 * e2 * e3), jb),
            ((xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), (xi, xi * e1), jb),
            ((xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), (xi, xi * e1 * e2), jb),
        ]
    if kind == Kind.SHARED_VERTEX:
        jac = xi ** 3 * e2
        u = (xi, xi * e1)
        v = (xi * e2, xi * e2 * e3)
        return [(u, v, jac), (v, u, jac)]
    raise ValueError(kind)


def singular_rule(kind: Kind, base_order: int = 4):
    """(points (n,4), weights (n,)) — quadrature.py:274-307."""
    x, w = np.polynomial.legendre.leggauss(int(base_order))
    x = 0.5 * (x + 1.0)
    w = 0.5 * w
    g = np.meshgrid(x, x, x, x, indexing="ij")
    xi, e1, e2, e3 = (a.ravel() for a in g)
    w4 = (w[:, None, None, None] * w[None, :, None, None]
          * w[None, None, :, None] * w[None, None, None, :]).ravel()
    pts, wts = [], []
    for (u1, u2), (v1, v2), jac in _subdomains(kind, xi, e1, e2, e3):
        pts.append(np.column_stack([u1 - u2, u2, v1 - v2, v2]))
        wts.append(w4 * jac)
    return np.concatenate(pts), np.concatenate(wts)


def classify(ta, tb):
    """(kind, perm_test, perm_trial) — quadrature.py:155-181."""
    ta = [int(t) for t in ta]
    tb = [int(t) for t in tb]
    shared = sorted(set(ta) & set(tb))
    if len(shared) == 3:
        return Kind.IDENTICAL, (0, 1, 2), tuple(tb.index(g) for g in ta)
    if len(shared) == 2:
        la = [ta.index(s) for s in shared]
        lb = [tb.index(s) for s in shared]
        return (Kind.SHARED_EDGE, (la[0], la[1], 3 - la[0] - la[1]),
                (lb[0], lb[1], 3 - lb[0] - lb[1]))
    if len(shared) == 1:
        la, lb = ta.index(shared[0]), tb.index(shared[0])
        rest = lambda l: tuple(i for i in range(3) if i != l)  # noqa: E731
        return Kind.SHARED_VERTEX, (la, *rest(la)), (lb, *rest(lb))
    return Kind.DISJOINT, (0, 1, 2), (0, 1, 2)


# ---------------------------------------------------------------------------
# geometry / spaces                       mesh.py:338-371, spaces.py:67-143
# ---------------------------------------------------------------------------

@dataclass
class Problem:
    """Mesh + spaces + per-element caches for one operator (an
    IntegrationContext restatement, kernels.py:161-227)."""

    spec: Spec
    vertices: np.ndarray
    elements: np.ndarray
    test_family: str = "p0"
    trial_family: str = "p0"
    regular_order: int = 4
    singular_base_order: int = 4
    _cache: dict = field(default_factory=dict, repr=False)

    def __post_init__(self):
        v = self.vertices[self.elements]
        e1 = v[:, 1] - v[:, 0]
        e2 = v[:, 2] - v[:, 0]
        cross = np.cross(e1, e2)
        self.jac = np.linalg.norm(cross, axis=1)
        self.normals = cross / self.jac[:, None]
        pts, wts = regular_rule(self.regular_order)
        self.rule_points, self.rule_weights = pts, wts
        self.qpoints = (v[:, None, 0] + pts[None, :, 0, None] * e1[:, None]
                        + pts[None, :, 1, None] * e2[:, None])
        self.test_values = basis_values(self.test_family, pts)
        self.trial_values = basis_values(self.trial_family, pts)
        self.curls = None
        if self.spec.operator == "hyps":
            c = np.empty((len(self.elements), 3, 3))
            for l in range(3):
                c[:, l, :] = v[:, (l + 1) % 3] - v[:, (l + 2) % 3]
            self.curls = c / self.jac[:, None, None]
        self.sing = {k: singular_rule(k, self.singular_base_order)
                     for k in (Kind.SHARED_VERTEX, Kind.SHARED_EDGE, Kind.IDENTICAL)}

    @property
    def m(self):
        return len(self.elements)

    def dofmap(self, family):
        m = self.m
        if family == "p0":
            return np.arange(m, dtype=np.int64)[:, None]
        if family == "p1c":
            return self.elements.copy()
        return np.arange(3 * m, dtype=np.int64).reshape(m, 3)

    def n_dofs(self, family):
        return {"p0": self.m, "p1c": len(self.vertices), "p1d": 3 * self.m}[family]

    def dof_centers(self, family):
        """spaces.py:67-78."""
        v = self.vertices
        if family == "p0":
            return v[self.elements].mean(axis=1)
        if family == "p1c":
            return v.copy()
        return v[self.elements].reshape(-1, 3)

    def swapped(self):
        key = "swapped"
        if key not in self._cache:
            self._cache[key] = Problem(self.spec.transposed, self.vertices, self.elements,
                                       self.trial_family, self.test_family,
                                       self.regular_order, self.singular_base_order)
        return self._cache[key]


def basis_values(family, pts):
    """spaces.py:112-125: (local_dim, q)."""
    if family == "p0":
        return np.ones((1, len(pts)))
    xi, eta = pts[:, 0], pts[:, 1]
    return np.stack([1.0 - xi - eta, xi, eta])


# ---------------------------------------------------------------------------
# kernels                                              kernels.py:129-158
# ---------------------------------------------------------------------------

def planes(operator, k, diff, r, n_test=None, n_trial=None):
    one_over = r.dtype.type(INV_4PI)
    if operator == "slp":
        amp = one_over / r
        if k == 0.0:
            return amp, None
        kr = r.dtype.type(k) * r
        return amp * np.cos(kr), amp * np.sin(kr)
    if operator == "dlp":
        dot = np.einsum("...i,...i->...", diff, n_trial)
    else:
        dot = -np.einsum("...i,...i->...", diff, n_test)
    amp = dot * (one_over / r ** 3)
    if k == 0.0:
        return amp, None
    kr = r.dtype.type(k) * r
    c, s = np.cos(kr), np.sin(kr)
    return amp * (c + kr * s), amp * (s - kr * c)


# ---------------------------------------------------------------------------
# per-pair integrator                                  kernels.py:230-347
# ---------------------------------------------------------------------------

def _regular(P: Problem, a, b):
    x, y = P.qpoints[a], P.qpoints[b]
    diff = x[:, None, :] - y[None, :, :]
    r = np.sqrt(np.einsum("pqi,pqi->pq", diff, diff))
    w = P.rule_weights
    jj = P.jac[a] * P.jac[b]
    ta, tb = P.test_values, P.trial_values
    spec = P.spec
    if spec.operator == "hyps":
        re, im = planes("slp", spec.wavenumber, diff, r)
        cd = P.curls[a] @ P.curls[b].T
        nd = float(P.normals[a] @ P.normals[b])
        k2 = spec.wavenumber ** 2

        def red(pl):
            return jj * (cd * np.einsum("p,q,pq->", w, w, pl)
                         - k2 * nd * np.einsum("p,q,pq,ip,jq->ij", w, w, pl, ta, tb))
    else:
        na = np.broadcast_to(P.normals[a], diff.shape)
        nb = np.broadcast_to(P.normals[b], diff.shape)
        re, im = planes(spec.operator, spec.wavenumber, diff, r, na, nb)

        def red(pl):
            return jj * np.einsum("p,q,pq,ip,jq->ij", w, w, pl, ta, tb)
    return red(re) if im is None else red(re) + 1j * red(im)


def _basis_perm(family, perm, pts):
    if family == "p0":
        return np.ones((1, len(pts)))
    bary = np.stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]])
    out = np.empty_like(bary)
    out[list(perm)] = bary
    return out


def _singular(P: Problem, a, b, kind, pa, pb):
    pts, wts = P.sing[kind]
    va = P.vertices[P.elements[a]][list(pa)]
    vb = P.vertices[P.elements[b]][list(pb)]
    ua, ub = pts[:, 0:2], pts[:, 2:4]
    x = va[0] + np.outer(ua[:, 0], va[1] - va[0]) + np.outer(ua[:, 1], va[2] - va[0])
    y = vb[0] + np.outer(ub[:, 0], vb[1] - vb[0]) + np.outer(ub[:, 1], vb[2] - vb[0])
    diff = x - y
    r = np.sqrt(np.einsum("qi,qi->q", diff, diff))
    w = wts * (P.jac[a] * P.jac[b])
    ta = _basis_perm(P.test_family, pa, ua)
    tb = _basis_perm(P.trial_family, pb, ub)
    spec = P.spec
    if spec.operator == "hyps":
        re, im = planes("slp", spec.wavenumber, diff, r)
        cd = P.curls[a] @ P.curls[b].T
        nd = float(P.normals[a] @ P.normals[b])
        k2 = spec.wavenumber ** 2

        def red(pl):
            return cd * np.dot(w, pl) - k2 * nd * np.einsum("q,iq,jq->ij", w * pl, ta, tb)
    else:
        na = np.broadcast_to(P.normals[a], x.shape)
        nb = np.broadcast_to(P.normals[b], y.shape)
        re, im = planes(spec.operator, spec.wavenumber, diff, r, na, nb)

        def red(pl):
            return np.einsum("q,iq,jq->ij", w * pl, ta, tb)
    return red(re) if im is None else red(re) + 1j * red(im)


def local_matrix(P: Problem, a: int, b: int):
    """kernels.py:330-347 — (nt, ns) block in the result dtype."""
    kind, pa, pb = classify(P.elements[a], P.elements[b])
    if kind == Kind.DISJOINT:
        blk = _regular(P, a, b)
    elif kind != Kind.IDENTICAL and a > b:
        S = P.swapped()
        k2, qa, qb = classify(P.elements[b], P.elements[a])
        blk = _singular(S, b, a, k2, qa, qb).T
    else:
        blk = _singular(P, a, b, kind, pa, pb)
    return blk.astype(P.spec.result_dtype, copy=False)


# ---------------------------------------------------------------------------
# batched regular integrator                          backend.py:180-255
# ---------------------------------------------------------------------------

class ContractViolation(Exception):
    pass


def integrate_batch(P: Problem, pairs: np.ndarray):
    """(re, im) planes (p, nt, ns) in working precision; im None for Laplace.
    Casts caches to the working dtype first as init_device does
    (backend.py:104-121) so FP32 arithmetic is native."""
    pairs = np.ascontiguousarray(pairs, dtype=np.int64).reshape(-1, 2)
    rd = P.spec.real_dtype
    m = P.m
    if len(pairs):
        lo, hi = pairs.min(), pairs.max()
        if lo < 0 or hi >= m:
            raise ContractViolation(f"pair indices must lie in [0, {m}), found [{lo}, {hi}]")
        ea, eb = P.elements[pairs[:, 0]], P.elements[pairs[:, 1]]
        bad = (ea[:, :, None] == eb[:, None, :]).any(axis=(1, 2))
        if bad.any():
            p = int(np.nonzero(bad)[0][0])
            raise ContractViolation(f"request pair {p} = ({pairs[p, 0]}, {pairs[p, 1]}) "
                                    "is not disjoint")
    # working-precision caches cast once per problem, as init_device does
    key = ("cast", rd.str)
    if key not in P._cache:
        P._cache[key] = (P.qpoints.astype(rd), P.normals.astype(rd), P.jac.astype(rd),
                         P.rule_weights.astype(rd), P.test_values.astype(rd),
                         P.trial_values.astype(rd),
                         P.curls.astype(rd) if P.curls is not None else None)
    q, nrm, jac, w, ta, tb, curls = P._cache[key]
    k = P.spec.wavenumber
    k2 = rd.type(k * k)
    nt, ns = ta.shape[0], tb.shape[0]
    out_re = np.empty((len(pairs), nt, ns), rd)
    out_im = np.empty((len(pairs), nt, ns), rd) if P.spec.is_complex else None
    stride = 4096
    for s0 in range(0, len(pairs), stride):
        sl = slice(s0, s0 + stride)
        a, b = pairs[sl, 0], pairs[sl, 1]
        diff = q[a][:, :, None, :] - q[b][:, None, :, :]
        r = np.sqrt(np.einsum("spqi,spqi->spq", diff, diff))
        jj = (jac[a] * jac[b])[:, None, None]
        if P.spec.operator == "hyps":
            re, im = planes("slp", k, diff, r)
            cd = np.einsum("sic,sjc->sij", curls[a], curls[b])
            nd = np.einsum("si,si->s", nrm[a], nrm[b])

            def red(pl, out):
                sf = np.einsum("p,q,spq->s", w, w, pl)
                sij = np.einsum("p,q,spq,ip,jq->sij", w, w, pl, ta, tb)
                np.multiply(jj, cd * sf[:, None, None] - (k2 * nd)[:, None, None] * sij, out=out)
        else:
            na = np.broadcast_to(nrm[a][:, None, None, :], diff.shape)
            nb = np.broadcast_to(nrm[b][:, None, None, :], diff.shape)
            re, im = planes(P.spec.operator, k, diff, r, na, nb)

            def red(pl, out):
                np.multiply(jj, np.einsum("p,q,spq,ip,jq->sij", w, w, pl, ta, tb), out=out)
        red(re, out_re[sl])
        if out_im is not None:
            red(im, out_im[sl])
    return out_re, out_im


# ---------------------------------------------------------------------------
# partition                                           hmatrix.py:66-211, 814-826
# ---------------------------------------------------------------------------

@dataclass
class Node:
    start: int
    stop: int
    level: int
    bbox_min: np.ndarray
    bbox_max: np.ndarray
    left: int = -1
    right: int = -1

    @property
    def is_leaf(self):
        return self.left < 0

    @property
    def size(self):
        return self.stop - self.start

    @property
    def diameter(self):
        return float(np.linalg.norm(self.bbox_max - self.bbox_min))


@dataclass
class Tree:
    nodes: list
    permutation: np.ndarray


def cluster_tree(points, n_min=32) -> Tree:
    """hmatrix.py:105-140: longest-axis stable-sort median bisection, preorder."""
    pts = np.asarray(points, dtype=np.float64)
    perm = np.arange(len(pts), dtype=np.int64)
    nodes: list[Node] = []
    stack = [(0, len(pts), 0, None, None)]  # (start, stop, level, parent, side)
    # iterative preorder: process node, push right then left
    while stack:
        start, stop, level, parent, side = stack.pop()
        idx = perm[start:stop]
        sub = pts[idx]
        lo, hi = sub.min(axis=0), sub.max(axis=0)
        me = len(nodes)
        nodes.append(Node(start, stop, level, lo, hi))
        if parent is not None:
            if side == 0:
                nodes[parent].left = me
            else:
                nodes[parent].right = me
        if stop - start > n_min:
            axis = int(np.argmax(hi - lo))
            order = np.argsort(sub[:, axis], kind="stable")
            perm[start:stop] = idx[order]
            mid = start + (stop - start + 1) // 2
            stack.append((mid, stop, level + 1, me, 1))
            stack.append((start, mid, level + 1, me, 0))
    return Tree(nodes, perm)


def box_distance(amin, amax, bmin, bmax):
    gap = np.maximum(0.0, np.maximum(bmin - amax, amin - bmax))
    return float(np.linalg.norm(gap))


def admissible(t: Node, s: Node, eta):
    d = box_distance(t.bbox_min, t.bbox_max, s.bbox_min, s.bbox_max)
    if d <= 0.0:
        return False
    return min(t.diameter, s.diameter) <= eta * d


def block_tree(rows: Tree, cols: Tree, eta=2.0):
    """hmatrix.py:182-211: list of (row_node, col_node, admissible) in
    recursive descent order."""
    leaves = []
    stack = [(0, 0)]
    while stack:
        ti, si = stack.pop()
        t, s = rows.nodes[ti], cols.nodes[si]
        if admissible(t, s, eta):
            leaves.append((ti, si, True))
            continue
        if t.is_leaf and s.is_leaf:
            leaves.append((ti, si, False))
            continue
        tk = (ti,) if t.is_leaf else (t.left, t.right)
        sk = (si,) if s.is_leaf else (s.left, s.right)
        kids = [(a, b) for a in tk for b in sk]
        stack.extend(reversed(kids))
    return leaves


# ---------------------------------------------------------------------------
# ACA                                                  hmatrix.py:271-382
# ---------------------------------------------------------------------------

@dataclass
class LowRank:
    u: np.ndarray
    v: np.ndarray
    rank: int
    residual: float
    converged: bool
    exhausted: bool = False

    def todense(self):
        return self.u @ self.v.T

    def matvec(self, x):
        return self.u @ (self.v.T @ x)


@dataclass
class Dense:
    a: np.ndarray

    def todense(self):
        return self.a

    def matvec(self, x):
        return self.a @ x


def aca(row_fn, col_fn, m, n, eps, k_max=None):
    kmax = min(m, n) if k_max is None else min(k_max, m, n)
    us, vs = [], []
    blocked = np.zeros(m, dtype=bool)       # z_rows | used_rows
    used_cols = np.zeros(n, dtype=bool)
    norm2, residual = 0.0, np.inf
    converged = exhausted = False
    small = 0

    def next_row(pref):
        if blocked.all():
            return -1
        if pref is None:
            return int(np.argmin(blocked))  # first False
        order = np.argsort(-np.abs(pref), kind="stable")
        for i in order:
            if not blocked[i]:
                return int(i)
        return -1

    i = next_row(None)
    dtype = None
    while len(us) < kmax:
        if i < 0:
            exhausted = converged = True
            break
        row = np.asarray(row_fn(i)).copy()
        dtype = dtype or row.dtype
        for ul, vl in zip(us, vs):
            row -= ul[i] * vl
        amask = np.abs(row)
        amask[used_cols] = -1.0
        j = int(np.argmax(amask))
        piv = row[j]
        if amask[j] <= 0.0 or piv == 0:
            blocked[i] = True
            i = next_row(None)
            continue
        v = row / piv
        col = np.asarray(col_fn(j)).copy()
        for ul, vl in zip(us, vs):
            col -= vl[j] * ul
        u = col
        upd = float(np.linalg.norm(u)) * float(np.linalg.norm(v))
        if norm2 > 0.0 and upd <= eps * np.sqrt(norm2):
            residual = upd / np.sqrt(norm2)
            small += 1
            if small >= 2:
                converged = True
                break
            blocked[i] = True
            i = next_row(u)
            continue
        small = 0
        cross = 0.0
        for ul, vl in zip(us, vs):
            cross += np.real(np.vdot(ul, u) * np.vdot(vl, v))
        norm2 += 2.0 * cross + upd * upd
        us.append(u)
        vs.append(v)
        blocked[i] = True
        used_cols[j] = True
        if norm2 > 0.0:
            residual = upd / np.sqrt(norm2)
            if upd <= eps * np.sqrt(norm2):
                small = 1
        i = next_row(u)
    if not us:
        dt = dtype if dtype is not None else np.float64
        return LowRank(np.zeros((m, 0), dt), np.zeros((n, 0), dt), 0, 0.0, converged, exhausted)
    return LowRank(np.stack(us, 1), np.stack(vs, 1), len(us), float(residual),
                   converged, exhausted)


# ---------------------------------------------------------------------------
# H-matrix assembly                                   hmatrix.py:510-811
# ---------------------------------------------------------------------------

def incidence(dofmap, n_dofs):
    """hmatrix.py:531-541: CSR dof -> (element, local)."""
    m, nl = dofmap.shape
    flat = dofmap.ravel()
    elem = np.repeat(np.arange(m, dtype=np.int64), nl)
    loc = np.tile(np.arange(nl, dtype=np.int64), m)
    order = np.argsort(flat, kind="stable")
    indptr = np.zeros(n_dofs + 1, dtype=np.int64)
    np.cumsum(np.bincount(flat, minlength=n_dofs), out=indptr[1:])
    return indptr, elem[order], loc[order]


class Assembler:
    """Per-block host assembly (hmatrix.py:550-756), single-threaded."""

    def __init__(self, P: Problem, rows: Tree, cols: Tree, leaves, eps, k_max=None):
        self.P, self.rows, self.cols, self.leaves = P, rows, cols, leaves
        self.eps, self.k_max = eps, k_max
        self.dtype = P.spec.result_dtype
        self.tdm = P.dofmap(P.test_family)
        self.sdm = P.dofmap(P.trial_family)
        self.rinc = incidence(self.tdm, P.n_dofs(P.test_family))
        self.cinc = incidence(self.sdm, P.n_dofs(P.trial_family))
        self.rinv = np.empty_like(rows.permutation)
        self.rinv[rows.permutation] = np.arange(len(rows.permutation))
        self.cinv = np.empty_like(cols.permutation)
        self.cinv[cols.permutation] = np.arange(len(cols.permutation))
        self.counters = {"regular_pairs": 0, "singular_pairs": 0, "aca_fallback_dense": 0,
                         "dense_leaves": 0, "lowrank_leaves": 0}
        # optional batched integrator for the regular pairs, the reference's
        # backend routing with threshold 1 (hmatrix.py:608-613): a callable
        # pairs -> (re, im) supplied by a test (e.g. a GPU backend)
        self.regular_fn = None

    @staticmethod
    def _of(inc, d):
        ip, el, lo = inc
        return el[ip[d]:ip[d + 1]], lo[ip[d]:ip[d + 1]]

    @staticmethod
    def _union(inc, dofs):
        ip, el, _ = inc
        ch = [el[ip[d]:ip[d + 1]] for d in dofs]
        return np.unique(np.concatenate(ch)) if ch else np.empty(0, np.int64)

    def pairs_block(self, pairs):
        """hmatrix.py:593-621."""
        P = self.P
        nt, ns = P.test_values.shape[0], P.trial_values.shape[0]
        out = np.zeros((len(pairs), nt, ns), dtype=self.dtype)
        if len(pairs) == 0:
            return out
        ea, eb = P.elements[pairs[:, 0]], P.elements[pairs[:, 1]]
        touch = (ea[:, :, None] == eb[:, None, :]).any(axis=(1, 2))
        reg = np.nonzero(~touch)[0]
        if len(reg):
            re, im = (integrate_batch(P, pairs[reg]) if self.regular_fn is None
                      else self.regular_fn(pairs[reg]))
            out[reg] = re if im is None else re + 1j * im
            self.counters["regular_pairs"] += len(reg)
        for p in np.nonzero(touch)[0]:
            out[p] = local_matrix(P, int(pairs[p, 0]), int(pairs[p, 1]))
            self.counters["singular_pairs"] += 1
        return out

    def row_job(self, dof, col_elems, c0, width):
        """hmatrix.py:625-649."""
        te, tl = self._of(self.rinc, dof)
        pairs = np.empty((len(te) * len(col_elems), 2), np.int64)
        pairs[:, 0] = np.repeat(te, len(col_elems))
        pairs[:, 1] = np.tile(col_elems, len(te))
        blk = self.pairs_block(pairs)
        loc = np.repeat(tl, len(col_elems))
        vals = blk[np.arange(len(pairs)), loc, :]
        cl = self.cinv[self.sdm[pairs[:, 1]]] - c0
        ok = (cl >= 0) & (cl < width)
        row = np.zeros(width, self.dtype)
        np.add.at(row, cl[ok], vals[ok])
        return row

    def col_job(self, dof, row_elems, r0, height):
        """hmatrix.py:651-672."""
        se, sl = self._of(self.cinc, dof)
        pairs = np.empty((len(row_elems) * len(se), 2), np.int64)
        pairs[:, 0] = np.repeat(row_elems, len(se))
        pairs[:, 1] = np.tile(se, len(row_elems))
        blk = self.pairs_block(pairs)
        loc = np.tile(sl, len(row_elems))
        vals = blk[np.arange(len(pairs)), :, loc]
        rl = self.rinv[self.tdm[pairs[:, 0]]] - r0
        ok = (rl >= 0) & (rl < height)
        col = np.zeros(height, self.dtype)
        np.add.at(col, rl[ok], vals[ok])
        return col

    def dense_leaf(self, rn: Node, cn: Node):
        """hmatrix.py:676-699."""
        rd = self.rows.permutation[rn.start:rn.stop]
        cd = self.cols.permutation[cn.start:cn.stop]
        te, se = self._union(self.rinc, rd), self._union(self.cinc, cd)
        pairs = np.empty((len(te) * len(se), 2), np.int64)
        pairs[:, 0] = np.repeat(te, len(se))
        pairs[:, 1] = np.tile(se, len(te))
        blk = self.pairs_block(pairs)
        rl = self.rinv[self.tdm[pairs[:, 0]]] - rn.start
        cl = self.cinv[self.sdm[pairs[:, 1]]] - cn.start
        rv = (rl >= 0) & (rl < rn.size)
        cv = (cl >= 0) & (cl < cn.size)
        mask = rv[:, :, None] & cv[:, None, :]
        lin = rl[:, :, None] * cn.size + cl[:, None, :]
        a = np.zeros((rn.size, cn.size), self.dtype)
        np.add.at(a.ravel(), lin[mask], blk[mask])
        return Dense(a)

    def lowrank_leaf(self, rn: Node, cn: Node):
        """hmatrix.py:701-735."""
        rd = self.rows.permutation[rn.start:rn.stop]
        cd = self.cols.permutation[cn.start:cn.stop]
        ce, re_ = self._union(self.cinc, cd), self._union(self.rinc, rd)
        row_fn = lambda i: self.row_job(int(rd[i]), ce, cn.start, cn.size)  # noqa: E731
        col_fn = lambda j: self.col_job(int(cd[j]), re_, rn.start, rn.size)  # noqa: E731
        blk = aca(row_fn, col_fn, rn.size, cn.size, self.eps, self.k_max)
        if blk.converged:
            if blk.rank * (rn.size + cn.size) < rn.size * cn.size:
                return blk
            return Dense(blk.todense())
        self.counters["aca_fallback_dense"] += 1
        a = np.empty((rn.size, cn.size), self.dtype)
        for i in range(rn.size):
            a[i] = row_fn(i)
        return Dense(a)

    def leaf(self, ix):
        ti, si, adm = self.leaves[ix]
        rn, cn = self.rows.nodes[ti], self.cols.nodes[si]
        if adm:
            out = self.lowrank_leaf(rn, cn)
        else:
            out = self.dense_leaf(rn, cn)
        self.counters["lowrank_leaves" if isinstance(out, LowRank) else "dense_leaves"] += 1
        return out

    def assemble(self):
        return [self.leaf(ix) for ix in range(len(self.leaves))]


def hmat_matvec(rows: Tree, cols: Tree, leaves, payloads, x):
    """hmatrix.py:441-470: fixed (row.start, col.start) leaf order."""
    xt = x[cols.permutation]
    dt = np.result_type(payloads[0].todense().dtype if payloads else np.float64, x.dtype)
    yt = np.zeros(len(rows.permutation), dt)
    order = sorted(range(len(leaves)), key=lambda ix: (rows.nodes[leaves[ix][0]].start,
                                                       cols.nodes[leaves[ix][1]].start))
    for ix in order:
        ti, si, _ = leaves[ix]
        rn, cn = rows.nodes[ti], cols.nodes[si]
        yt[rn.start:rn.stop] += payloads[ix].matvec(xt[cn.start:cn.stop])
    y = np.empty_like(yt)
    y[rows.permutation] = yt
    return y


def assemble_dense(P: Problem):
    """Dense operator by the per-pair path (assembly.py:321-345 restated,
    with the regular part batched): ground truth for matvec parity."""
    tdm, sdm = P.dofmap(P.test_family), P.dofmap(P.trial_family)
    A = np.zeros((P.n_dofs(P.test_family), P.n_dofs(P.trial_family)), P.spec.result_dtype)
    m = P.m
    a = np.repeat(np.arange(m), m)
    b = np.tile(np.arange(m), m)
    ea, eb = P.elements[a], P.elements[b]
    touch = (ea[:, :, None] == eb[:, None, :]).any(axis=(1, 2))
    reg = np.stack([a[~touch], b[~touch]], 1)
    re, im = integrate_batch(P, reg)
    vals = re if im is None else re + 1j * im
    rows = tdm[reg[:, 0]][:, :, None]
    cols = sdm[reg[:, 1]][:, None, :]
    nt, ns = tdm.shape[1], sdm.shape[1]
    np.add.at(A, (np.broadcast_to(rows, (len(reg), nt, ns)),
                  np.broadcast_to(cols, (len(reg), nt, ns))), vals)
    for x, y in zip(a[touch], b[touch]):
        A[np.ix_(tdm[x], sdm[y])] += local_matrix(P, int(x), int(y))
    return A


# ---------------------------------------------------------------------------
# far-field potential                                  scatter.py:362-408
# ---------------------------------------------------------------------------

NEAR_FIELD_DIAMETERS = 3.0  # scatter.py:50


def far_field(vertices, elements, family, dofmap, phi, points, k, quad_order=4, chunk=256):
    """evaluate_far_field (scatter.py:362-408): dens = phi[dofmap] . table *
    (|J| w) (374-376); per chunk of points diff = x - y_q, DLP kernel planes
    with the element normal (385-388), sum over elements and rule points
    (390).  Returns (u, n_near) with n_near the count of points closer than
    3 element diameters to a rule point (379-384)."""
    pts_r, w = regular_rule(quad_order)
    v = vertices[elements]
    e1 = v[:, 1] - v[:, 0]
    e2 = v[:, 2] - v[:, 0]
    cross = np.cross(e1, e2)
    jac = np.linalg.norm(cross, axis=1)              # mesh.py:347-349
    normals = cross / jac[:, None]
    qpts = v[:, None, 0] + pts_r[None, :, 0, None] * e1[:, None] + pts_r[None, :, 1, None] * e2[:, None]
    diam = np.stack([np.linalg.norm(e1, axis=1), np.linalg.norm(e2, axis=1),
                     np.linalg.norm(v[:, 2] - v[:, 1], axis=1)]).max(axis=0)
    table = basis_values(family, pts_r)
    dens = np.einsum("ml,lq->mq", np.asarray(phi)[np.asarray(dofmap).reshape(len(elements), -1)],
                     table)
    dens = dens * (jac[:, None] * w[None, :])
    d_near = NEAR_FIELD_DIAMETERS * float(diam.max())
    out = np.empty(len(points), dtype=np.complex128)
    n_near = 0
    nrm = normals[None, :, None, :]
    for lo in range(0, len(points), chunk):
        hi = min(lo + chunk, len(points))
        diff = points[lo:hi, None, None, :] - qpts[None, :, :, :]
        r = np.sqrt(np.einsum("cmqi,cmqi->cmq", diff, diff))
        n_near += int(np.count_nonzero(r.min(axis=(1, 2)) < d_near))
        re, im = planes("dlp", k, diff, r, n_trial=nrm)
        kern = re if im is None else re + 1j * im
        out[lo:hi] = np.einsum("cmq,mq->c", kern, dens)
    return out, n_near
