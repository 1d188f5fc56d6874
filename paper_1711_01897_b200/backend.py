"""GPU batched-integrator backend: the drop-in for the reference's "device"
contract (`/root/reference/pkg/src/hbem/backend.py:41-298`).

``GpuBackend`` has the exact surface of the reference ``HostBackend``
(``.context.spec``, ``.device_id``, ``.integrate_batch(BatchRequest) ->
RawResultBuffer``, ``batches_served``/``pairs_served``), so it can be handed
to the reference's ``assemble_hmatrix(..., backends=[...])`` /
``assemble_dense`` unmodified, and ``make_gpu_backends(ctx, n_devices)``
mirrors ``make_host_backends`` (backend.py:282-298).  ``ctx`` may be the
reference's IntegrationContext or this package's.

Every call goes through the C ABI (``libhbem_b200.so``); there is no
host-side integration code in this module.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, lib
from .errors import CapacityError, ContractViolationError

MAX_WEIGHTS = 6  # backend.py:34
_KIND_SLOT = {"SHARED_VERTEX": 0, "SHARED_EDGE": 1, "IDENTICAL": 2}


@dataclass(frozen=True)
class BatchRequest:
    """backend.py:125-150: (p, 2) int64 pairs, optional (p,) offsets."""

    pairs: np.ndarray
    offsets: np.ndarray | None = None

    def __post_init__(self):
        pairs = np.ascontiguousarray(self.pairs, dtype=np.int64)
        if pairs.ndim != 2 or pairs.shape[1] != 2:
            raise ContractViolationError(f"pairs must have shape (p, 2), got {pairs.shape}")
        pairs.setflags(write=False)
        object.__setattr__(self, "pairs", pairs)
        if self.offsets is not None:
            off = np.ascontiguousarray(self.offsets, dtype=np.int64)
            if off.shape != (len(pairs),):
                raise ContractViolationError("offsets must have one entry per pair")
            off.setflags(write=False)
            object.__setattr__(self, "offsets", off)

    def __len__(self) -> int:
        return len(self.pairs)


@dataclass(frozen=True)
class RawResultBuffer:
    """backend.py:153-177: pair-major (p, nt, ns) planes, im None for real kernels."""

    re: np.ndarray
    im: np.ndarray | None
    pairs: np.ndarray
    offsets: np.ndarray | None

    def block(self, p: int) -> np.ndarray:
        if self.im is None:
            return self.re[p]
        return self.re[p] + 1j * self.im[p]

    def complex_view(self) -> np.ndarray:
        if self.im is None:
            return self.re
        return self.re + 1j * self.im

    def __len__(self) -> int:
        return len(self.re)


def _family_code(space, n_local: int) -> int:
    fam = getattr(space, "family", None)
    val = getattr(fam, "value", fam)
    if val in _lib.FAMILIES:
        return _lib.FAMILIES[val]
    return 0 if n_local == 1 else 1


class GpuDeviceContext:
    """Device-resident integration state for one operator on one GPU: the
    DeviceContext of backend.py:41-74 plus the singular rules, held behind
    an ``hbem_ctx*`` handle.  Immutable once built; safe to share."""

    def __init__(self, ctx, device_id: int = 0, cuda_device: int | None = None):
        spec = ctx.spec
        rule = ctx.regular_rule
        weights = np.ascontiguousarray(rule.weights, dtype=np.float64)
        n_q = len(weights)
        if n_q > MAX_WEIGHTS:
            raise CapacityError(
                f"quadrature rule has {n_q} weights, device capacity is {MAX_WEIGHTS}")
        tv = np.ascontiguousarray(ctx.test_table.values, dtype=np.float64)
        sv = np.ascontiguousarray(ctx.trial_table.values, dtype=np.float64)
        if tv.shape[1] != n_q or sv.shape[1] != n_q:
            raise CapacityError("basis tables and geometry disagree on quadrature point count")
        mesh = ctx.mesh
        self.device_id = int(device_id)
        self.cuda_device = int(device_id if cuda_device is None else cuda_device)
        self.spec = spec
        self.elements = np.ascontiguousarray(mesh.elements, dtype=np.int64)
        self.elements.setflags(write=False)
        self.test_values = tv
        self.trial_values = sv
        self.weights = weights
        self._keep = []  # arrays referenced by the descriptor during create

        def keep(a, dt=np.float64):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a

        d = _lib.CtxDesc()
        d.device = self.cuda_device
        d.equation = _lib.EQUATIONS[spec.equation]
        d.op = _lib.OPERATORS[spec.operator]
        d.precision = _lib.PRECISIONS[spec.precision]
        d.wavenumber = float(spec.wavenumber)
        d.test_family = _family_code(ctx.test_space, tv.shape[0])
        d.trial_family = _family_code(ctx.trial_space, sv.shape[0])
        verts = keep(mesh.vertices)
        d.n_vertices = len(verts)
        d.vertices = _lib.ptr(verts, C.c_double)
        d.n_elements = len(self.elements)
        d.elements = _lib.ptr(self.elements, C.c_int64)
        d.n_q = n_q
        d.rule_points = _lib.ptr(keep(rule.points), C.c_double)
        d.rule_weights = _lib.ptr(keep(weights), C.c_double)
        geo = getattr(ctx, "geometry", None)
        if geo is not None:  # reference context: stage its host caches as given
            d.qpoints = _lib.ptr(keep(geo.qpoints), C.c_double)
            d.normals = _lib.ptr(keep(geo.normals), C.c_double)
            d.jacobians = _lib.ptr(keep(geo.jacobians), C.c_double)
        curls = getattr(ctx, "curls", None)
        if curls is not None:
            d.curls = _lib.ptr(keep(curls), C.c_double)
        d.test_values = _lib.ptr(tv, C.c_double)
        d.trial_values = _lib.ptr(sv, C.c_double)
        for kind, trule in getattr(ctx, "singular", {}).items():
            slot = _KIND_SLOT[getattr(kind, "name", str(kind))]
            pts = keep(trule.points)
            wts = keep(trule.weights)
            d.sing_n[slot] = len(wts)
            d.sing_points[slot] = _lib.ptr(pts, C.c_double)
            d.sing_weights[slot] = _lib.ptr(wts, C.c_double)
        h = C.c_void_p()
        check(lib.hbem_ctx_create(C.byref(d), C.byref(h)))
        self._keep = []
        self.handle = h
        nt, ns, cplx, rb = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        check(lib.hbem_ctx_info(h, C.byref(nt), C.byref(ns), C.byref(cplx), C.byref(rb)))
        self._shape = (nt.value, ns.value)

    @property
    def n_elements(self) -> int:
        return len(self.elements)

    @property
    def block_shape(self) -> tuple[int, int]:
        return self._shape

    def geometry(self):
        """(qpoints (m,6,3), normals (m,3), jacobians (m,)) as staged on the device."""
        m = self.n_elements
        q = np.empty((m, 6, 3))
        n = np.empty((m, 3))
        j = np.empty(m)
        check(lib.hbem_ctx_geometry(self.handle, _lib.ptr(q, C.c_double),
                                    _lib.ptr(n, C.c_double), _lib.ptr(j, C.c_double)))
        return q, n, j

    def close(self):
        if getattr(self, "handle", None):
            lib.hbem_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass


def _run(context: GpuDeviceContext, pairs: np.ndarray, any_kind: bool):
    spec = context.spec
    nt, ns = context.block_shape
    rd = spec.real_dtype
    p = len(pairs)
    re = np.empty((p, nt, ns), dtype=rd)
    im = np.empty((p, nt, ns), dtype=rd) if spec.is_complex else None
    if any_kind:
        nsing = C.c_int64(0)
        check(lib.hbem_integrate_any(context.handle, _lib.ptr(pairs, C.c_int64), p,
                                     _lib.vptr(re), _lib.vptr(im), C.byref(nsing)))
        return re, im, int(nsing.value)
    check(lib.hbem_integrate_regular(context.handle, _lib.ptr(pairs, C.c_int64), p,
                                     _lib.vptr(re), _lib.vptr(im)))
    return re, im, 0


def integrate_batch(context: GpuDeviceContext, request: BatchRequest) -> RawResultBuffer:
    """backend.py:200-255 on the GPU: disjoint pairs only (contract-checked
    on the device), bitwise independent of how pairs are split."""
    re, im, _ = _run(context, request.pairs, any_kind=False)
    return RawResultBuffer(re=re, im=im, pairs=request.pairs, offsets=request.offsets)


class GpuBackend:
    """HostBackend-compatible GPU integrator (backend.py:258-279)."""

    def __init__(self, context: GpuDeviceContext):
        self.context = context
        self._lock = threading.Lock()
        self.batches_served = 0
        self.pairs_served = 0
        self.singular_served = 0

    @property
    def device_id(self) -> int:
        return self.context.device_id

    def _count(self, n, nsing=0):
        with self._lock:
            self.batches_served += 1
            self.pairs_served += n
            self.singular_served += nsing

    def integrate_batch(self, request: BatchRequest) -> RawResultBuffer:
        result = integrate_batch(self.context, request)
        self._count(len(request))
        return result

    def integrate_pairs(self, request: BatchRequest) -> RawResultBuffer:
        """Any adjacency class (no contract on disjointness): the batched
        local_matrix (kernels.py:330-347) with touching pairs integrated by
        the on-device Sauter-Schwab rules, so no element integral falls back
        to the CPU."""
        re, im, nsing = _run(self.context, request.pairs, any_kind=True)
        self._count(len(request), nsing)
        return RawResultBuffer(re=re, im=im, pairs=request.pairs, offsets=request.offsets)

    def local_matrix(self, test_elem: int, trial_elem: int) -> np.ndarray:
        buf = self.integrate_pairs(BatchRequest(np.array([[test_elem, trial_elem]])))
        return buf.complex_view()[0].astype(self.context.spec.result_dtype, copy=False)


def init_gpu_device(ctx, device_id: int = 0) -> GpuDeviceContext:
    """init_device (backend.py:77-122) for a GPU, from an IntegrationContext."""
    n = _lib.device_count()
    if n < 1:
        raise CapacityError("no CUDA device available for the GPU backend")
    return GpuDeviceContext(ctx, device_id=device_id, cuda_device=device_id % n)


def make_gpu_backends(ctx, n_devices: int = 1) -> list[GpuBackend]:
    """make_host_backends (backend.py:282-298) for GPUs: device i runs on
    CUDA device i mod device_count, each with its own context."""
    if n_devices < 1:
        raise CapacityError(f"need at least one device, got {n_devices}")
    return [GpuBackend(init_gpu_device(ctx, dev)) for dev in range(n_devices)]
