"""Synthetic surface meshes for the benchmark configurations.

The reference only ships an icosphere refiner capped at level 8
(`/root/reference/pkg/src/hbem/mesh.py:32,269-310`) and a Gmsh reader.  The
north-star sizes need frequency-n geodesic spheres
(20 n^2 triangles: n=11 -> 2 420, n=45 -> 40 500, n=71 -> 100 820,
n=448 -> 4 014 080) and an elongated hull, so both generators live here.

Every generator returns plain ``(vertices float64 (nv,3), elements int64
(m,3))`` arrays, outward oriented by the right-hand rule of
`mesh.py:1-8`, so the same arrays can be fed to the reference's
``TriangleMesh`` and to this package.
"""

from __future__ import annotations

import numpy as np

_PHI = (1.0 + 5.0 ** 0.5) / 2.0


def _icosahedron() -> tuple[np.ndarray, np.ndarray]:
    """Unit icosahedron with outward-oriented faces."""
    v = []
    for s1 in (-1.0, 1.0):
        for s2 in (-1.0, 1.0):
            v.append((0.0, s1, s2 * _PHI))
            v.append((s1, s2 * _PHI, 0.0))
            v.append((s2 * _PHI, 0.0, s1))
    v = np.array(v, dtype=np.float64)
    v /= np.linalg.norm(v, axis=1)[:, None]
    # faces = all vertex triples that are mutually at the minimal distance
    d = np.linalg.norm(v[:, None, :] - v[None, :, :], axis=2)
    edge = d[d > 1e-9].min()
    adj = np.abs(d - edge) < 1e-6
    faces = []
    for a in range(12):
        for b in range(a + 1, 12):
            if not adj[a, b]:
                continue
            for c in range(b + 1, 12):
                if adj[a, c] and adj[b, c]:
                    faces.append((a, b, c))
    faces = np.array(faces, dtype=np.int64)
    assert len(faces) == 20
    tri = v[faces]
    nrm = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
    flip = np.einsum("ij,ij->i", nrm, tri.mean(axis=1)) < 0
    faces[flip] = faces[flip][:, [0, 2, 1]]
    return v, faces


def geodesic_sphere(n: int, radius: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """Frequency-n geodesic sphere: each icosahedron face is split into an
    n x n triangular grid whose points are projected onto the sphere.

    Produces 20 n^2 triangles and 10 n^2 + 2 vertices; shared edge and
    corner points are de-duplicated through canonical edge numbering."""
    if n < 1:
        raise ValueError(f"frequency must be >= 1, got {n}")
    base_v, faces = _icosahedron()
    # canonical edges (lo, hi) of the icosahedron
    edges = {}
    for f in faces:
        for a, b in ((f[0], f[1]), (f[1], f[2]), (f[2], f[0])):
            key = (min(a, b), max(a, b))
            if key not in edges:
                edges[key] = len(edges)
    n_edge_pts = n - 1
    n_int = (n - 1) * (n - 2) // 2
    edge_base = 12
    face_base = 12 + len(edges) * n_edge_pts
    nv = face_base + len(faces) * n_int

    coords = np.empty((nv, 3), dtype=np.float64)
    coords[:12] = base_v
    t = np.arange(1, n, dtype=np.float64)
    for (lo, hi), e in edges.items():
        p = ((n - t)[:, None] * base_v[lo] + t[:, None] * base_v[hi]) / n
        coords[edge_base + e * n_edge_pts: edge_base + (e + 1) * n_edge_pts] = p

    # grid index (i, j), i + j <= n, weights (n-i-j, i, j) on (a, b, c)
    ii, jj = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    keep = ii + jj <= n
    gi, gj = ii[keep], jj[keep]
    interior = (gi >= 1) & (gj >= 1) & (gi + gj <= n - 1)
    # face-local interior numbering in (i, j) lexicographic order
    int_rank = np.cumsum(interior) - 1

    elems = []
    for fidx, (a, b, c) in enumerate(faces):
        ids = np.full((n + 1, n + 1), -1, dtype=np.int64)

        def edge_ids(p, q, tpos):
            key = (min(p, q), max(p, q))
            e = edges[key]
            tt = tpos if p < q else n - tpos
            return edge_base + e * n_edge_pts + (tt - 1)

        # corners
        ids[0, 0] = a
        ids[n, 0] = b
        ids[0, n] = c
        s = np.arange(1, n)
        if n > 1:
            ids[s, 0] = edge_ids(a, b, s)          # edge a-b, t from a = i
            ids[0, s] = edge_ids(a, c, s)          # edge a-c, t from a = j
            ids[n - s, s] = edge_ids(b, c, s)      # edge b-c, t from b = j
        if n_int:
            fi, fj = gi[interior], gj[interior]
            gid = face_base + fidx * n_int + int_rank[interior]
            ids[fi, fj] = gid
            w0 = (n - fi - fj)[:, None]
            coords[gid] = (w0 * base_v[a] + fi[:, None] * base_v[b]
                           + fj[:, None] * base_v[c]) / n
        # up triangles (i,j),(i+1,j),(i,j+1) for i+j <= n-1
        ui, uj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        up = ui + uj <= n - 1
        ui, uj = ui[up], uj[up]
        elems.append(np.stack([ids[ui, uj], ids[ui + 1, uj], ids[ui, uj + 1]], axis=1))
        # down triangles (i+1,j),(i+1,j+1),(i,j+1) for i+j <= n-2
        di, dj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        dn = di + dj <= n - 2
        di, dj = di[dn], dj[dn]
        elems.append(np.stack([ids[di + 1, dj], ids[di + 1, dj + 1], ids[di, dj + 1]], axis=1))
    elements = np.concatenate(elems).astype(np.int64)
    coords /= np.linalg.norm(coords, axis=1)[:, None]
    coords *= radius
    return np.ascontiguousarray(coords), np.ascontiguousarray(elements)


def elongated_hull(n_around: int, n_along: int, length: float = 8.0,
                   radius: float = 0.5) -> tuple[np.ndarray, np.ndarray]:
    """Closed, outward-oriented body of revolution with L/D = length/(2 radius),
    a submarine-like stand-in.  Profile: hemispherical-ish
    bow, cylindrical mid-body, tapered stern; 2 * n_around * n_along
    triangles."""
    if n_around < 3 or n_along < 3:
        raise ValueError("need n_around >= 3 and n_along >= 3")
    s = np.linspace(0.0, 1.0, n_along + 1)[1:-1]  # interior stations
    x = (s - 0.5) * length
    # radius profile: smooth bow / stern closure
    bow = np.clip(s / 0.12, 0.0, 1.0)
    stern = np.clip((1.0 - s) / 0.3, 0.0, 1.0)
    r = radius * np.sqrt(1.0 - (1.0 - bow) ** 2) * (1.0 - (1.0 - stern) ** 2) ** 0.5
    r = np.maximum(r, 1e-3 * radius)
    th = 2.0 * np.pi * np.arange(n_around) / n_around
    rings = np.stack([
        np.repeat(x, n_around),
        np.outer(r, np.cos(th)).ravel(),
        np.outer(r, np.sin(th)).ravel(),
    ], axis=1)
    tip0 = np.array([[-0.5 * length, 0.0, 0.0]])
    tip1 = np.array([[0.5 * length, 0.0, 0.0]])
    verts = np.concatenate([tip0, rings, tip1])
    nr = len(x)
    ring = lambda k: 1 + k * n_around  # noqa: E731
    tris = []
    a = np.arange(n_around)
    b = (a + 1) % n_around
    tris.append(np.stack([np.zeros(n_around, np.int64), ring(0) + b, ring(0) + a], 1))
    for k in range(nr - 1):
        p0, p1 = ring(k), ring(k + 1)
        tris.append(np.stack([p0 + a, p0 + b, p1 + b], 1))
        tris.append(np.stack([p0 + a, p1 + b, p1 + a], 1))
    last = len(verts) - 1
    tris.append(np.stack([np.full(n_around, last), ring(nr - 1) + a, ring(nr - 1) + b], 1))
    elems = np.concatenate(tris).astype(np.int64)
    # signed volume > 0 <=> outward orientation for a closed surface
    v = verts[elems]
    vol = np.einsum("ij,ij->i", v[:, 0], np.cross(v[:, 1], v[:, 2])).sum() / 6.0
    if vol < 0:
        elems = elems[:, [0, 2, 1]]
    return np.ascontiguousarray(verts), np.ascontiguousarray(elems)


def load_mesh(path):
    """Read a Gmsh 2.2 ASCII file (mesh.py:134-245) with the native parser
    (``hbem_gmsh_read``, csrc/gmsh.cpp): 3-node triangles only, other element
    types counted in ``meta['skipped_elements']``, unreferenced vertices
    dropped and indices compacted in ascending node-tag order.  Raises
    MeshError when the file cannot be read and MeshParseError (with ``line``
    and ``section``) on malformed input, with the reference's messages."""
    import ctypes as C
    import os

    from . import _lib
    from .discretization import TriangleMesh
    path = os.fspath(path)
    h = C.c_void_p()
    _lib.check(_lib.lib.hbem_gmsh_read(path.encode(), C.byref(h)))
    try:
        nv, ne, ns = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(_lib.lib.hbem_gmsh_size(h, C.byref(nv), C.byref(ne), C.byref(ns)))
        v = np.empty((nv.value, 3), np.float64)
        e = np.empty((ne.value, 3), np.int64)
        _lib.check(_lib.lib.hbem_gmsh_copy(h, _lib.ptr(v, C.c_double), _lib.ptr(e, C.c_int64)))
    finally:
        _lib.lib.hbem_gmsh_destroy(h)
    return TriangleMesh(v, e, meta={"skipped_elements": int(ns.value), "source": path})


# The icosahedron of refine_unit_sphere (mesh.py:248-265): vertex order and
# face list are data the icosphere's bits depend on, so they follow the
# reference table (the common (+-1, +-t, 0) cyclic listing).
_ICO_T = (1.0 + np.sqrt(5.0)) / 2.0
_ICO_V = np.array([(-1, _ICO_T, 0), (1, _ICO_T, 0), (-1, -_ICO_T, 0), (1, -_ICO_T, 0),
                   (0, -1, _ICO_T), (0, 1, _ICO_T), (0, -1, -_ICO_T), (0, 1, -_ICO_T),
                   (_ICO_T, 0, -1), (_ICO_T, 0, 1), (-_ICO_T, 0, -1), (-_ICO_T, 0, 1)],
                  dtype=np.float64)
_ICO_F = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                   (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                   (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                   (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)
MAX_SPHERE_LEVEL = 8


def icosphere(level: int) -> tuple[np.ndarray, np.ndarray]:
    """The reference's icosphere (refine_unit_sphere, mesh.py:269-310) bit for
    bit, vectorised per level: every face (a, b, c) becomes (a, ab, ca),
    (b, bc, ab), (c, ca, bc), (ab, bc, ca); edge midpoints are numbered in
    order of first use over the faces' (ab, bc, ca) edges and projected with
    the same v / np.linalg.norm(v) as the reference (per vertex, so the
    norm's BLAS evaluation is the reference's)."""
    if not isinstance(level, (int, np.integer)) or level < 0:
        raise ValueError(f"refinement level must be a non-negative integer, got {level!r}")
    if level > MAX_SPHERE_LEVEL:
        raise ValueError(f"refinement level {level} exceeds maximum {MAX_SPHERE_LEVEL}")
    verts = np.array([v / np.linalg.norm(v) for v in _ICO_V])
    faces = _ICO_F.copy()
    for _ in range(level):
        a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
        # edges in first-use order: per face ab, bc, ca
        e = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([c, a], 1)], 1)
        e = e.reshape(-1, 2)
        key = np.minimum(e[:, 0], e[:, 1]) * len(verts) + np.maximum(e[:, 0], e[:, 1])
        uk, first, inv = np.unique(key, return_index=True, return_inverse=True)
        rank = np.empty(len(uk), np.int64)
        order = np.argsort(first, kind="stable")
        rank[order] = np.arange(len(uk))
        mid = (len(verts) + rank[inv]).reshape(-1, 3)
        ab, bc, ca = mid[:, 0], mid[:, 1], mid[:, 2]
        ue = e[first[order]]
        m = verts[ue[:, 0]] + verts[ue[:, 1]]
        m = np.array([r / np.linalg.norm(r) for r in m]).reshape(-1, 3)
        verts = np.concatenate([verts, m])
        faces = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                          np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
    return verts, faces
