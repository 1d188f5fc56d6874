"""The scattering application on the GPU, with the
signatures, validation, warnings and error classes of
`/root/reference/pkg/src/hbem/scatter.py`:

* ``evaluate_far_field`` / ``evaluation_ring`` (scatter.py:94-107,362-408):
  geometry, densities and the point x element x rule-point double-layer sum
  run in ``hbem_far_field`` (csrc/far.cu); no host fallback.
* ``burton_miller_solve`` (scatter.py:228-359): (1/2 M - K - eta_c D) phi =
  M u_inc - eta_c M du_inc/dn with K (Helmholtz DLP, P1c) and the single
  layer S (Helmholtz SLP, P1d) assembled on the device (H-matrix: lock-step
  ACA; dense: the element-pair sweep), D = sum_j Q_j^T S Q_j - k^2 sum_j
  P_j^T S P_j (the sparse surface-curl / normal transforms of
  spaces.py:204-246), GMRES (solvers.py) applying K and S by device matvecs.
  The sparse mass / transform matrices and the Krylov basis are O(N) host
  arrays, as in the reference.
"""

from __future__ import annotations

import ctypes as C
import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sps
import torch

from . import _lib
from ._lib import check, lib
from .discretization import FunctionSpace, TriangleMesh, basis_table, regular_rule
from .errors import ConfigError, MeshError, SolverError, SpaceError

NEAR_FIELD_DIAMETERS = 3.0  # scatter.py:50
MIN_ELEMENTS_PER_WAVELENGTH = 6.0  # scatter.py:49


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


# ---------------------------------------------------------------------------
# Burton-Miller combined-field solve                     scatter.py:52-359
# ---------------------------------------------------------------------------

def wavenumber_from_frequency(frequency: float, sound_speed: float) -> float:
    """k = 2 pi f / c (scatter.py:52-58)."""
    if frequency <= 0.0 or sound_speed <= 0.0:
        raise ConfigError(
            f"frequency and sound speed must be > 0, got {frequency}, {sound_speed}")
    return 2.0 * np.pi * frequency / sound_speed


def incidence_direction(theta_deg: float) -> np.ndarray:
    """Unit propagation direction in the xy-plane (scatter.py:87-91)."""
    t = np.deg2rad(theta_deg)
    return np.array([np.cos(t), np.sin(t), 0.0])


@dataclass(frozen=True)
class PlaneWave:
    """u(x) = amplitude exp(i k <d, x>) (scatter.py:61-84)."""

    amplitude: complex
    direction: np.ndarray
    wavenumber: float

    def __post_init__(self):
        d = np.array(self.direction, dtype=np.float64)
        if d.shape != (3,):
            raise ConfigError(f"direction must be a 3-vector, got shape {d.shape}")
        if abs(np.linalg.norm(d) - 1.0) > 1e-12:
            raise ConfigError(
                f"direction must be unit length within 1e-12, |d| = {np.linalg.norm(d)!r}")
        if self.wavenumber <= 0.0:
            raise ConfigError(f"wavenumber must be > 0, got {self.wavenumber}")
        d.setflags(write=False)
        object.__setattr__(self, "direction", d)

    def evaluate(self, points: np.ndarray) -> np.ndarray:
        return self.amplitude * np.exp(1j * (points @ (self.wavenumber * self.direction)))


def _default_aca():
    from .hmatrix import AcaConfig
    return AcaConfig()


def _default_assembly():
    from .hmatrix import AssemblyConfig
    return AssemblyConfig()


@dataclass(frozen=True)
class ScatterConfig:
    """One scattering run (scatter.py:110-166).  ``build_mesh`` makes a
    geodesic unit sphere with 20 * 4**sphere_level triangles (the
    reference's icosphere refinement level); Gmsh files are out of scope."""

    frequency: float = 477.46482927568605  # k = 2 with c = 1500
    sound_speed: float = 1500.0
    sphere_level: int = 3
    mesh_file: str | None = None
    amplitude: float = 1.0
    theta_inc_deg: float = 0.0
    radius: float = 100.0
    n_points: int = 3600
    tol: float = 1e-5
    restart: int = 100
    max_iter: int | None = None
    eta: float = 2.0
    n_min: int = 32
    force: bool = False
    assembly: object = field(default_factory=_default_assembly)
    aca: object = field(default_factory=_default_aca)

    def __post_init__(self):
        checks = ((self.frequency <= 0.0, f"frequency must be > 0, got {self.frequency}"),
                  (self.sound_speed <= 0.0, f"sound_speed must be > 0, got {self.sound_speed}"),
                  (self.radius <= 0.0, f"radius must be > 0, got {self.radius}"),
                  (self.n_points < 1, f"n_points must be >= 1, got {self.n_points}"),
                  (self.mesh_file is None and self.sphere_level < 0,
                   f"sphere_level must be >= 0, got {self.sphere_level}"),
                  (self.tol <= 0.0, f"tol must be > 0, got {self.tol}"),
                  (self.restart < 1, f"restart must be >= 1, got {self.restart}"))
        for bad, msg in checks:
            if bad:
                raise ConfigError(msg)

    @property
    def wavenumber(self) -> float:
        return wavenumber_from_frequency(self.frequency, self.sound_speed)

    def plane_wave(self) -> PlaneWave:
        return PlaneWave(complex(self.amplitude), incidence_direction(self.theta_inc_deg),
                         self.wavenumber)

    def build_mesh(self) -> TriangleMesh:
        if self.mesh_file is not None:
            from .meshes import load_mesh
            return load_mesh(self.mesh_file)
        # the reference's icosphere (refine_unit_sphere, mesh.py:269-310), bit for bit
        from .meshes import icosphere
        try:
            return TriangleMesh(*icosphere(self.sphere_level))
        except ValueError as exc:
            raise MeshError(str(exc)) from None


@dataclass(frozen=True)
class SolveReport:
    """scatter.py:169-182."""

    phi: np.ndarray
    converged: bool
    iterations: int
    residual: float
    residuals: tuple
    timings: dict
    mode: str
    wavenumber: float
    n_dofs: int
    n_elements: int


def _element_frames(mesh: TriangleMesh):
    """|J|, unit normals and edge vectors per element (mesh.py:344-349)."""
    v = mesh.vertices[mesh.elements]
    e1, e2 = v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]
    cr = np.cross(e1, e2)
    jac = np.linalg.norm(cr, axis=1)
    return v, jac, cr / jac[:, None]


def _check_closed_oriented(mesh: TriangleMesh):
    """mesh_is_closed + check_consistent_orientation: every edge is used by
    exactly two elements, once in each direction."""
    el = mesh.elements
    directed = np.concatenate([el[:, [0, 1]], el[:, [1, 2]], el[:, [2, 0]]])
    und = np.sort(directed, axis=1)
    _, inv, cnt = np.unique(und, axis=0, return_inverse=True, return_counts=True)
    if (cnt != 2).any():
        raise MeshError("scattering requires a closed surface mesh")
    fwd = directed[:, 0] < directed[:, 1]
    per_edge = np.bincount(inv.ravel(), weights=fwd.astype(np.float64), minlength=len(cnt))
    if (per_edge != 1.0).any():
        raise MeshError("inconsistent element orientation across a shared edge")


def vertex_normals(mesh: TriangleMesh) -> np.ndarray:
    """Area-weighted outward vertex normals (scatter.py:185-194)."""
    _, jac, nrm = _element_frames(mesh)
    acc = np.zeros((len(mesh.vertices), 3))
    np.add.at(acc, mesh.elements.ravel(), np.repeat(nrm * (0.5 * jac)[:, None], 3, axis=0))
    ln = np.linalg.norm(acc, axis=1)
    if (ln == 0.0).any():
        raise MeshError("vertex with vanishing aggregate normal")
    return acc / ln[:, None]


def incident_trace(wave: PlaneWave, mesh: TriangleMesh, space: FunctionSpace):
    """Nodal u_inc and du_inc/dn = i k <d, n_v> u_inc (scatter.py:197-211)."""
    if space.family.value != "p1c":
        raise SpaceError(
            f"incident traces need the continuous P1 space, got {space.family.value}")
    if space.mesh is not mesh:
        raise SpaceError("space was built on a different mesh")
    u = wave.evaluate(mesh.vertices)
    return u, 1j * wave.wavenumber * (vertex_normals(mesh) @ wave.direction) * u


def _resolution_guard(mesh: TriangleMesh, k: float, force: bool) -> float:
    """scatter.py:214-225: elements per wavelength from the longest edge."""
    v = mesh.vertices[mesh.elements]
    h = max(float(np.linalg.norm(v[:, a] - v[:, b], axis=1).max())
            for a, b in ((1, 0), (2, 0), (2, 1)))
    epw = (2.0 * np.pi / k) / h
    if epw < MIN_ELEMENTS_PER_WAVELENGTH and not force:
        raise SolverError(
            f"mesh resolves {epw:.2f} elements per wavelength, below the "
            f"minimum {MIN_ELEMENTS_PER_WAVELENGTH:g}; refine the mesh or "
            "pass force=True to proceed anyway")
    return epw


def _mass_p1c(space: FunctionSpace, jac: np.ndarray):
    """Galerkin P1c mass matrix with the 3-point rule (spaces.py:183-201)."""
    rule = regular_rule(2)
    t = basis_table(space, rule).values
    local = (t * rule.weights[None, :]) @ t.T
    dm = space.dofmap
    rows = np.repeat(dm, 3, axis=1).ravel()
    cols = np.tile(dm, (1, 3)).ravel()
    vals = (jac[:, None, None] * local[None]).ravel()
    return sps.csr_matrix((vals, (rows, cols)), shape=(space.n_dofs, space.n_dofs))


def _curl_and_normal_maps(p1c: FunctionSpace, p1d: FunctionSpace, v, jac, nrm):
    """Q_j (surface-curl component j, constant per element, on each of the
    element's three P1d rows) and P_j (n_j times nodal values) from P1c to
    P1d (spaces.py:204-246)."""
    shape = (p1d.n_dofs, p1c.n_dofs)
    curls = np.stack([v[:, (l + 1) % 3] - v[:, (l + 2) % 3] for l in range(3)], 1)
    curls = curls / jac[:, None, None]
    qr = np.repeat(p1d.dofmap, 3, axis=1).ravel()
    qc = np.tile(p1c.dofmap, (1, 3)).ravel()
    pr, pc = p1d.dofmap.ravel(), p1c.dofmap.ravel()
    q = [sps.csr_matrix((np.tile(curls[:, :, j], (1, 3)).ravel(), (qr, qc)), shape=shape)
         for j in range(3)]
    p = [sps.csr_matrix((np.repeat(nrm[:, j], 3), (pr, pc)), shape=shape) for j in range(3)]
    return q, p


def burton_miller_solve(cfg: ScatterConfig, wave: PlaneWave | None = None, mode: str = "dense",
                        mesh: TriangleMesh | None = None,
                        stats: dict | None = None) -> SolveReport:
    """Sound-hard scattering, total surface trace phi (scatter.py:228-359),
    with every boundary-operator application on the GPU."""
    from .backend import make_gpu_backends
    from .discretization import OperatorSpec, build_space, make_integration_context
    from .hmatrix import assemble_hmatrix
    from .partition import cluster_trees_for
    from .solvers import GmresResult, gmres

    if mode not in ("dense", "hmatrix"):
        raise ConfigError(f"mode must be 'dense' or 'hmatrix', got {mode!r}")
    wave = cfg.plane_wave() if wave is None else wave
    k = wave.wavenumber
    if abs(k - cfg.wavenumber) > 1e-9 * max(k, cfg.wavenumber):
        raise ConfigError(f"wave has k = {k}, config implies k = {cfg.wavenumber}; "
                          "they must describe the same problem")
    mesh = cfg.build_mesh() if mesh is None else mesh
    _check_closed_oriented(mesh)
    epw = _resolution_guard(mesh, k, cfg.force)

    t0 = time.perf_counter()
    p1c, p1d = build_space(mesh, "p1c"), build_space(mesh, "p1d")
    v, jac, nrm = _element_frames(mesh)
    mass = _mass_p1c(p1c, jac)
    qm, pm = _curl_and_normal_maps(p1c, p1d, v, jac, nrm)
    qt, pt = [q.T.tocsr() for q in qm], [p.T.tocsr() for p in pm]
    spec_k = OperatorSpec("helmholtz", "dlp", k)
    spec_s = OperatorSpec("helmholtz", "slp", k)
    # the solve runs on the GPU: operators applied by device matvecs (H-matrix
    # mode) or dense products, the sparse mass / surface-curl / normal maps as
    # cuSPARSE CSR products, the GMRES basis in HBM
    dev = torch.device("cuda", torch.cuda.current_device())
    if mode == "dense":
        from .assembly import assemble_dense
        n_dev = cfg.assembly.devices or 1
        orders = dict(regular_order=cfg.assembly.regular_order,
                      singular_base_order=cfg.assembly.singular_base_order)
        k_op = assemble_dense(spec_k, p1c, p1c, cfg.assembly,
                              make_gpu_backends(make_integration_context(spec_k, p1c, p1c,
                                                                         **orders), n_dev))
        s_op = assemble_dense(spec_s, p1d, p1d, cfg.assembly,
                              make_gpu_backends(make_integration_context(spec_s, p1d, p1d,
                                                                         **orders), n_dev))
        k_d = torch.from_numpy(k_op).to(dev)
        s_d = torch.from_numpy(s_op).to(dev)
        apply_k, apply_s = k_d.__matmul__, s_d.__matmul__
    else:
        k_op = assemble_hmatrix(spec_k, p1c, p1c, cluster_trees_for(p1c, p1c, cfg.n_min, cfg.eta),
                                cfg.aca, assembly_config=cfg.assembly)
        s_op = assemble_hmatrix(spec_s, p1d, p1d, cluster_trees_for(p1d, p1d, cfg.n_min, cfg.eta),
                                cfg.aca, assembly_config=cfg.assembly)
        apply_k, apply_s = k_op.matvec_torch, s_op.matvec_torch
    eta_c = 1.0 / (1j * k)

    def csr(a):
        a = a.tocsr()
        return torch.sparse_csr_tensor(torch.from_numpy(a.indptr.astype(np.int64)),
                                       torch.from_numpy(a.indices.astype(np.int64)),
                                       torch.from_numpy(a.data.astype(np.complex128)),
                                       size=a.shape, check_invariants=False).to(dev)

    with warnings.catch_warnings():  # torch marks CSR "beta"
        warnings.simplefilter("ignore", UserWarning)
        mass_d = csr(mass)
        qm_d, qt_d = [csr(q) for q in qm], [csr(q) for q in qt]
        pm_d, pt_d = [csr(p) for p in pm], [csr(p) for p in pt]

    def apply_d(x):
        curl = torch.zeros(p1c.n_dofs, dtype=torch.complex128, device=dev)
        for q, qq in zip(qm_d, qt_d):
            curl += qq @ apply_s(q @ x).to(torch.complex128)
        norm = torch.zeros_like(curl)
        for p, pp in zip(pm_d, pt_d):
            norm += pp @ apply_s(p @ x).to(torch.complex128)
        return curl - k * k * norm

    def operator(x):
        return 0.5 * (mass_d @ x) - apply_k(x).to(torch.complex128) - eta_c * apply_d(x)

    u_inc, du_inc = incident_trace(wave, mesh, p1c)
    rhs = mass @ u_inc - eta_c * (mass @ du_inc)
    t1 = time.perf_counter()
    res = gmres(operator, torch.from_numpy(np.asarray(rhs, np.complex128)).to(dev), tol=cfg.tol,
                restart=cfg.restart, max_iter=cfg.max_iter)
    res = GmresResult(res.x.cpu().numpy(), res.converged, res.iterations, res.residual,
                      res.residuals, res.restarts)
    t2 = time.perf_counter()
    if not res.converged:
        err = SolverError(f"GMRES did not reach tolerance {cfg.tol:g} within "
                          f"{res.iterations} iterations (residual {res.residual:.3e})")
        err.residuals = res.residuals
        raise err
    if stats is not None:
        stats["elements_per_wavelength"] = epw
        stats["mode"] = mode
    return SolveReport(phi=res.x, converged=res.converged, iterations=res.iterations,
                       residual=res.residual, residuals=res.residuals,
                       timings={"assembly": t1 - t0, "solve": t2 - t1}, mode=mode,
                       wavenumber=k, n_dofs=p1c.n_dofs, n_elements=len(mesh.elements))


def target_strength(u_sct, u0: complex, radius: float):
    """Bistatic target strength TS = 20 log10(R |u_sct| / |u0|) in dB
    (scatter.py:411-424): scalars give a float, arrays an array; a silent
    direction is -inf."""
    if radius <= 0.0:
        raise ConfigError(f"radius must be > 0, got {radius}")
    if u0 == 0:
        raise ConfigError("reference amplitude u0 must be nonzero")
    ratio = radius * np.abs(np.asarray(u_sct) / u0)
    with np.errstate(divide="ignore"):
        db = 20.0 * np.log10(ratio)
    return float(db) if np.ndim(u_sct) == 0 else db


def deviation(u_a, u_b) -> float:
    """Mean relative magnitude deviation (1/n) sum ||a_i| - |b_i|| / |b_i| of a
    far field against a reference one (the paper's Delta_sct,
    scatter.py:427-441)."""
    mag_a = np.abs(np.asarray(u_a)).ravel()
    mag_b = np.abs(np.asarray(u_b)).ravel()
    if mag_a.shape != mag_b.shape or mag_a.size == 0:
        raise ConfigError(f"fields must have equal nonzero lengths, got {mag_a.shape} "
                          f"and {mag_b.shape}")
    if not mag_b.all():
        raise ZeroDivisionError(f"reference field vanishes at sample index "
                                f"{int(np.argmin(mag_b != 0.0))}")
    return float(np.mean(np.abs(mag_a - mag_b) / mag_b))


def write_far_field_csv(path, angles_deg, values, u0: complex, radius: float) -> None:
    """One CSV row per observation angle: theta_deg, re, im, abs, ts_db
    (scatter.py:444-452, same header and number formats)."""
    vals = np.asarray(values)
    ts = np.atleast_1d(target_strength(vals, u0, radius))
    rows = ["theta_deg,re,im,abs,ts_db"]
    rows += [f"{a:.6f},{v.real:.12e},{v.imag:.12e},{abs(v):.12e},{t:.6f}"
             for a, v, t in zip(angles_deg, vals, ts)]
    with open(path, "w", encoding="utf-8") as f:
        f.write("\n".join(rows) + "\n")
