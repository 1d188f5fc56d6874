"""Far-field evaluation of the scattering application on the GPU
(SURVEY §8f row 3): ``evaluate_far_field`` and ``evaluation_ring`` with the
signatures, validation, warning and error classes of
`/root/reference/pkg/src/hbem/scatter.py:94-107,362-408`.

The element geometry, the densities and the point x element x rule-point
double-layer sum all run in ``hbem_far_field`` (csrc/far.cu); there is no
host fallback.
"""

from __future__ import annotations

import ctypes as C
import warnings

import numpy as np

from . import _lib
from ._lib import check, lib
from .discretization import FunctionSpace, TriangleMesh, basis_table, regular_rule
from .errors import ConfigError

NEAR_FIELD_DIAMETERS = 3.0  # scatter.py:50


def evaluation_ring(n_points: int, radius: float) -> tuple[np.ndarray, np.ndarray]:
    """n equally spaced observation points on a circle in the xy-plane
    (scatter.py:94-107).  Returns (points (n, 3), angles_deg (n,))."""
    if n_points < 1:
        raise ConfigError(f"n_points must be >= 1, got {n_points}")
    if radius <= 0.0:
        raise ConfigError(f"radius must be > 0, got {radius}")
    ang = np.arange(n_points) * (360.0 / n_points)
    t = np.deg2rad(ang)
    pts = np.zeros((n_points, 3))
    pts[:, 0] = radius * np.cos(t)
    pts[:, 1] = radius * np.sin(t)
    return pts, ang


def evaluate_far_field(mesh: TriangleMesh, space: FunctionSpace, phi: np.ndarray,
                       points: np.ndarray, k: float, quad_order: int = 4,
                       chunk_size: int = 256, device: int = 0) -> np.ndarray:
    """Scattered field u(x) = int dG(x,y)/dn_y phi(y) ds_y off the surface
    (scatter.py:362-408): regular quadrature per element, evaluated on the
    device; a UserWarning names the points within 3 element diameters of the
    surface.  ``chunk_size`` is accepted for API compatibility (the device
    tiles points by itself)."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ConfigError(f"points must have shape (n, 3), got {pts.shape}")
    phi = np.asarray(phi)
    if phi.shape != (space.n_dofs,):
        raise ConfigError(
            f"phi must have one coefficient per DOF ({space.n_dofs}), got {phi.shape}")
    pts = np.ascontiguousarray(pts)
    rule = regular_rule(quad_order)
    table = np.ascontiguousarray(basis_table(space, rule).values, np.float64)
    vtx = np.ascontiguousarray(mesh.vertices, np.float64)
    el = np.ascontiguousarray(mesh.elements, np.int64)
    dm = np.ascontiguousarray(np.asarray(space.dofmap, np.int64).reshape(len(el), -1))
    pr = np.ascontiguousarray(phi.real, np.float64)
    pi = np.ascontiguousarray(phi.imag, np.float64) if np.iscomplexobj(phi) else None
    n = len(pts)
    ore, oim, rmin = np.empty(n), np.empty(n), np.empty(n)
    rp = np.ascontiguousarray(rule.points, np.float64)
    rw = np.ascontiguousarray(rule.weights, np.float64)
    check(lib.hbem_far_field(device, n, _lib.vptr(pts), len(vtx), _lib.vptr(vtx), len(el),
                             _lib.vptr(el), len(rw), _lib.vptr(rp), _lib.vptr(rw),
                             table.shape[0], _lib.vptr(table), _lib.vptr(dm), space.n_dofs,
                             _lib.vptr(pr), None if pi is None else _lib.vptr(pi),
                             C.c_double(float(k)), _lib.vptr(ore), _lib.vptr(oim),
                             _lib.vptr(rmin)))
    # near-field test (scatter.py:379-384): 3 x the longest element edge
    v = vtx[el]
    diam = max(float(np.linalg.norm(v[:, 1] - v[:, 0], axis=1).max()),
               float(np.linalg.norm(v[:, 2] - v[:, 0], axis=1).max()),
               float(np.linalg.norm(v[:, 2] - v[:, 1], axis=1).max()))
    n_near = int(np.count_nonzero(rmin < NEAR_FIELD_DIAMETERS * diam))
    if n_near:
        warnings.warn(
            f"{n_near} evaluation points lie within {NEAR_FIELD_DIAMETERS:g} "
            "element diameters of the surface; quadrature accuracy degrades "
            "in the near field",
            stacklevel=2,
        )
    out = np.empty(n, dtype=np.complex128)
    out.real = ore
    out.imag = oim
    return out
