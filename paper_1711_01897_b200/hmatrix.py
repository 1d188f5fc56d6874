"""H-matrix assembly on the GPU behind the reference's assembler API.

``assemble_hmatrix(spec, test_space, trial_space, block_tree, cfg, backends,
assembly_config, stats)`` has the signature, validation, error classes and
counter names of `/root/reference/pkg/src/hbem/hmatrix.py:759-811`, and
returns an ``HMatrix`` whose payloads are ``LowRankBlock`` / ``DenseBlock``
objects with the reference's fields (hmatrix.py:241-438).  The work runs in
``hbem_hmat_assemble`` (C ABI): near-field leaves and every admissible
leaf's ACA on the device, lock-step across blocks.

Multi-GPU: with several backends, leaves are split into contiguous
cost-weighted ranges (one per backend / GPU) and assembled independently;
the only data the GPUs share is the geometry each context staged once.
"""

from __future__ import annotations

import ctypes as C
import re
import threading
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import check, lib
from .backend import GpuBackend, init_gpu_device
from .discretization import OperatorSpec, make_integration_context
from .errors import AssemblyError, ConfigError
from .partition import (BlockClusterTree, BlockLeaf, ClusterNode, ClusterTree,  # noqa: F401
                        build_block_tree, build_cluster_tree, cluster_trees_for)


@dataclass(frozen=True)
class AcaConfig:
    """hmatrix.py:219-238.  ``threshold`` is accepted for API compatibility;
    on the GPU path every row/column job runs on the device."""

    epsilon: float = 1e-5
    k_max: int | None = None
    threshold: int = 10000

    def __post_init__(self):
        if self.epsilon <= 0.0:
            raise ConfigError(f"epsilon must be > 0, got {self.epsilon}")
        if self.k_max is not None and self.k_max < 1:
            raise ConfigError(f"k_max must be >= 1, got {self.k_max}")
        if self.threshold < 1:
            raise ConfigError(f"threshold must be >= 1, got {self.threshold}")


@dataclass(frozen=True)
class AssemblyConfig:
    """assembly.py:34-63 (fields kept; ``rank_capacity`` is the per-block
    factor-table size of the device ACA)."""

    chunk_size: int = 1 << 20
    workers: int = 1
    regular_order: int = 4
    singular_base_order: int = 4
    devices: int | None = None
    max_matrix_bytes: int = 4 << 30
    lock_stripes: int = 1024
    rank_capacity: int = 64

    def __post_init__(self):
        if self.chunk_size < 1:
            raise ConfigError(f"chunk_size must be positive, got {self.chunk_size}")
        if self.workers < 1:
            raise ConfigError(f"workers must be positive, got {self.workers}")
        if self.devices is not None and self.devices < 1:
            raise ConfigError(f"devices must be positive when set, got {self.devices}")


@dataclass(frozen=True)
class LowRankBlock:
    """hmatrix.py:241-268: A ~= u @ v.T."""

    u: np.ndarray
    v: np.ndarray
    rank: int
    residual: float
    converged: bool
    exhausted: bool = False

    @property
    def shape(self):
        return self.u.shape[0], self.v.shape[0]

    def todense(self):
        return self.u @ self.v.T

    def matvec(self, x):
        return self.u @ (self.v.T @ x)


@dataclass(frozen=True)
class DenseBlock:
    a: np.ndarray

    @property
    def shape(self):
        return self.a.shape

    def todense(self):
        return self.a

    def matvec(self, x):
        return self.a @ x


class _Payloads:
    """Lazy tuple of leaf payloads backed by the host copies of the device
    arenas (views, no per-leaf copies)."""

    def __init__(self, parts):
        self._parts = parts  # list of (leaf_ids, _DevicePart)
        n = sum(len(ids) for ids, _ in parts)
        self._where = np.empty((n, 2), np.int64)
        for pi, (ids, _) in enumerate(parts):
            self._where[ids, 0] = pi
            self._where[ids, 1] = np.arange(len(ids))
        self._cache = {}

    def __len__(self):
        return len(self._where)

    def __getitem__(self, ix):
        if isinstance(ix, slice):
            return tuple(self[i] for i in range(*ix.indices(len(self))))
        ix = int(ix)
        if ix < 0:
            ix += len(self)
        got = self._cache.get(ix)
        if got is None:
            pi, local = self._where[ix]
            got = self._parts[pi][1].payload(int(local))
            self._cache[ix] = got
        return got

    def __iter__(self):
        return (self[i] for i in range(len(self)))


def pinned_empty(n: int, dtype) -> np.ndarray:
    """numpy array in page-locked host memory (cudaHostAlloc via the C ABI),
    released when the array's buffer is garbage collected."""
    import weakref
    dtype = np.dtype(dtype)
    nbytes = max(int(n) * dtype.itemsize, 1)
    p = C.c_void_p()
    check(lib.hbem_host_alloc(nbytes, C.byref(p)))
    buf = (C.c_byte * nbytes).from_address(p.value)
    weakref.finalize(buf, lib.hbem_host_free, C.c_void_p(p.value))
    return np.frombuffer(buf, dtype=dtype, count=int(n))


class _DevicePart:
    """One hbem_hmat (one GPU's share of the leaves) and its host arenas."""

    def __init__(self, handle, n_leaves, shapes, dtype, n_rows=0, context=None):
        self.handle = handle
        self.n_rows = n_rows
        # the device context (geometry, rules) must outlive the handle: the
        # assembler reads it on re-execute and matvec reads its precision
        self.context = context
        self.dtype = dtype
        self._shapes = shapes  # (L, 2) h, w, or a callable computing them on first use
        self.n_leaves = n_leaves
        self._pinned = []
        self._lock = threading.Lock()
        self._refresh()

    @property
    def shapes(self) -> np.ndarray:
        if callable(self._shapes):
            self._shapes = self._shapes()
        return self._shapes

    def _refresh(self):
        L, handle = self.n_leaves, self.handle
        if getattr(self, "kind", None) is None:
            # allocated once, refilled from the device arrays on every execute
            # (page-locking ~150 MB at C5 would cost more than it saves)
            self.kind = np.empty(L, np.int32)
            self.rank = np.empty(L, np.int32)
            self.flags = np.empty(L, np.int32)
            self.off_u = np.empty(L, np.int64)
            self.off_v = np.empty(L, np.int64)
            self.off_d = np.empty(L, np.int64)
            self.resid = np.empty(L, np.float64)
        check(lib.hbem_hmat_leaf_meta(handle, _lib.ptr(self.kind, C.c_int32),
                                      _lib.ptr(self.rank, C.c_int32),
                                      _lib.ptr(self.flags, C.c_int32),
                                      _lib.ptr(self.off_u, C.c_int64),
                                      _lib.ptr(self.off_v, C.c_int64),
                                      _lib.ptr(self.off_d, C.c_int64)))
        check(lib.hbem_hmat_leaf_residual(handle, _lib.ptr(self.resid, C.c_double)))
        st = _lib.HmatStats()
        check(lib.hbem_hmat_stats_get(handle, C.byref(st)))
        self.stats = {name: getattr(st, name) for name, _ in _lib.HmatStats._fields_}
        self.stats["capacity_retries"] = getattr(self, "capacity_retries", 0)
        self._arenas = None

    def execute(self, stream=None):
        """Re-run the whole assembly on the device (inputs already resident);
        deterministic, so the payloads are unchanged (and re-streamed into the
        host output arenas if the part was assembled with ``out``)."""
        arenas = self._arenas if getattr(self, "_streamed", False) else None
        check(lib.hbem_hmat_execute(self.handle, stream))
        self._refresh()
        if arenas is not None:
            self._arenas = arenas

    def _host_array(self, n, pinned):
        return pinned_empty(n, self.dtype) if pinned else np.empty(n, self.dtype)

    def arenas(self, pinned: bool = False, out=None):
        """Host copies of the factor (U, V) and dense arenas; ``out`` reuses
        previously allocated (e.g. pinned) host buffers."""
        with self._lock:
            if self._arenas is None or out is not None:
                s = self.stats
                if out is None:
                    out = tuple(self._host_array(s[k], pinned)
                                for k in ("u_entries", "v_entries", "dense_entries"))
                u, v, d = out
                check(lib.hbem_hmat_copy_arenas(self.handle, _lib.vptr(u), _lib.vptr(v),
                                                _lib.vptr(d)))
                self._arenas = (u, v, d)
            return self._arenas

    def payload(self, q):
        u, v, d = self.arenas()
        h, w = (int(t) for t in self.shapes[q])
        if self.kind[q] == 1:
            r = int(self.rank[q])
            uu = u[self.off_u[q]: self.off_u[q] + h * r].reshape(r, h).T
            vv = v[self.off_v[q]: self.off_v[q] + w * r].reshape(r, w).T
            fl = int(self.flags[q])
            return LowRankBlock(uu, vv, r, float(self.resid[q]), bool(fl & 1), bool(fl & 2))
        o = self.off_d[q]
        return DenseBlock(d[o: o + h * w].reshape(h, w))

    def matvec(self, x: np.ndarray) -> np.ndarray:
        """Device y = H_part x in original DOF order (x, y in the result dtype)."""
        x = np.ascontiguousarray(x, dtype=self.dtype)
        y = np.empty(self.n_rows, dtype=self.dtype)
        check(lib.hbem_hmat_matvec(self.handle, _lib.vptr(x), _lib.vptr(y)))
        return y

    def matvec_device(self, x_ptr: int, y_ptr: int, stream=None) -> None:
        """y = H_part x on device pointers (original DOF order, result dtype),
        enqueued on ``stream``; bit-reproducible between calls."""
        check(lib.hbem_hmat_matvec_device(self.handle, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                          stream))

    def close(self):
        if self.handle:
            lib.hbem_hmat_destroy(self.handle)
            self.handle = None
        self._arenas = None
        self.context = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


@dataclass(frozen=True)
class HMatrix:
    """hmatrix.py:407-438."""

    tree: BlockClusterTree
    payloads: object
    spec: OperatorSpec
    parts: tuple = ()

    @property
    def shape(self):
        return self.tree.shape

    @property
    def dtype(self):
        return self.spec.result_dtype

    def matvec(self, x):
        return hmat_matvec(self, x)

    def matvec_torch(self, x):
        """y = H x for a CUDA torch vector (original DOF order), on the
        current torch stream: device matvec of every part (bit-reproducible),
        parts summed in part order.  The result has the H-matrix dtype."""
        import torch
        tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
               np.dtype(np.complex128): torch.complex128,
               np.dtype(np.complex64): torch.complex64}[np.dtype(self.dtype)]
        xc = x.to(tdt).contiguous()
        stream = torch.cuda.current_stream(xc.device).cuda_stream
        y = None
        for _, part in self.parts:
            yp = torch.empty(self.shape[0], dtype=tdt, device=xc.device)
            part.matvec_device(xc.data_ptr(), yp.data_ptr(), stream)
            y = yp if y is None else y + yp
        return y

    def to_dense(self):
        m, n = self.shape
        out = np.zeros((m, n), dtype=self.dtype)
        rp, cp = self.tree.rows.permutation, self.tree.cols.permutation
        rn, cn = self.tree.rows.node_array, self.tree.cols.node_array
        for ix, (r, c, _) in enumerate(self.tree.leaf_array):
            rows = rp[rn[r, 0]: rn[r, 1]]
            cols = cp[cn[c, 0]: cn[c, 1]]
            out[np.ix_(rows, cols)] = self.payloads[ix].todense()
        return out


def hmat_matvec(h: HMatrix, x: np.ndarray, device: bool = True) -> np.ndarray:
    """y = H x in the original DOF ordering (hmatrix.py:441-470).

    ``device=True`` (default when the payloads are device-resident): one
    ``hbem_hmat_matvec`` per GPU part straight from the device arenas,
    summed over the parts.  ``device=False``: the host loop over the leaf
    payloads in fixed (row.start, col.start) order, as the reference."""
    m, n = h.shape
    x = np.asarray(x)
    if x.shape != (n,):
        raise AssemblyError(f"matvec expects a vector of length {n}, got {x.shape}")
    rd = np.dtype(h.dtype)
    if device and np.iscomplexobj(x) and rd.kind != "c":
        return (hmat_matvec(h, x.real.copy(), True)
                + 1j * hmat_matvec(h, x.imag.copy(), True))
    # the device applies the payloads in their own precision; a wider x
    # (float64 into a float32 H-matrix) promotes like the reference
    # (np.result_type(h.dtype, x.dtype)) on the host leaf loop below
    if device and np.result_type(rd, x.dtype) == rd and h.parts and \
            all(p.handle for _, p in h.parts):
        y = None
        for _, part in h.parts:
            yp = part.matvec(x.astype(rd, copy=False))
            y = yp if y is None else y + yp
        return y
    rows, cols = h.tree.rows, h.tree.cols
    xt = x[cols.permutation]
    yt = np.zeros(m, dtype=np.result_type(h.dtype, x.dtype))
    la = h.tree.leaf_array
    rs = rows.node_array[la[:, 0]]
    cs = cols.node_array[la[:, 1]]
    order = np.lexsort((cs[:, 0], rs[:, 0]))
    for ix in order:
        r0, r1 = rs[ix, 0], rs[ix, 1]
        c0, c1 = cs[ix, 0], cs[ix, 1]
        yt[r0:r1] += h.payloads[int(ix)].matvec(xt[c0:c1])
    y = np.empty_like(yt)
    y[rows.permutation] = yt
    return y


@dataclass(frozen=True)
class CompressionStats:
    stored_entries: int
    dense_entries: int
    ratio: float
    rank_histogram: dict
    n_dense_leaves: int
    n_lowrank_leaves: int


def compression_stats(h: HMatrix) -> CompressionStats:
    """hmatrix.py:485-502 (computed from the leaf metadata, no payload copies)."""
    stored = 0
    hist: dict = {}
    n_dense = n_low = 0
    for part_ids, part in h.parts:
        hw = part.shapes
        low = part.kind == 1
        stored += int((part.rank[low].astype(np.int64) * hw[low].sum(axis=1)).sum())
        stored += int((hw[~low, 0].astype(np.int64) * hw[~low, 1]).sum())
        for r, c in zip(*np.unique(part.rank[low], return_counts=True)):
            hist[int(r)] = hist.get(int(r), 0) + int(c)
        n_low += int(low.sum())
        n_dense += int((~low).sum())
    m, n = h.shape
    return CompressionStats(stored, m * n, stored / (m * n), dict(sorted(hist.items())), n_dense,
                            n_low)


# Sauter-Schwab work per touching pair in regular-pair units: a P0 element
# touches ~13 elements (itself, 3 across edges, ~9 across vertices) with
# 1536 / 1280 / 512 points against 36, and the single layer integrates each
# unordered pair once: ~ (1536 + 3 * 1280 + 9 * 512) / 36 / 2 per element
_SING_PER_DIAG_ROW = 140.0
_SING_PER_OFFDIAG = 20.0


def _leaf_costs(tree: BlockClusterTree, k_est: float = 8.0) -> np.ndarray:
    """Cost model for the multi-GPU split, in regular element-pair
    integrals: admissible leaves ~ (k_est + 2) (h + w) (rank + confirmation
    rows and columns); near-field leaves h w plus their Sauter-Schwab pairs,
    which each rank integrates only for its own leaves (diagonal leaves hold
    every element's touching neighbours, off-diagonal neighbours only the
    ones along the shared boundary, ~ sqrt(h w))."""
    la = tree.leaf_array
    rn, cn = tree.rows.node_array, tree.cols.node_array
    h = (rn[la[:, 0], 1] - rn[la[:, 0], 0]).astype(np.float64)
    w = (cn[la[:, 1], 1] - cn[la[:, 1], 0]).astype(np.float64)
    diag = la[:, 0] == la[:, 1] if tree.rows is tree.cols else np.zeros(len(la), bool)
    sing = np.where(diag, _SING_PER_DIAG_ROW * h, _SING_PER_OFFDIAG * np.sqrt(h * w))
    return np.where(la[:, 2] == 1, (k_est + 2.0) * (h + w), h * w + sing)


def split_leaves(tree: BlockClusterTree, parts: int) -> list[np.ndarray]:
    """Contiguous cost-weighted ranges of leaf indices, one per device."""
    if parts < 1:
        raise ConfigError(f"parts must be positive, got {parts}")
    cost = np.cumsum(_leaf_costs(tree))
    total = cost[-1] if len(cost) else 0.0
    cuts = [0]
    for p in range(1, parts):
        cuts.append(int(np.searchsorted(cost, total * p / parts, side="left")))
    cuts.append(len(cost))
    return [np.arange(cuts[i], cuts[i + 1], dtype=np.int64) for i in range(parts)]


def _assemble_part(dev_ctx, tree: BlockClusterTree, leaf_ids, test_space, trial_space,
                   cfg: AcaConfig, acfg: AssemblyConfig, stream=None, out=None) -> _DevicePart:
    """One GPU's share of the leaves.  ``out`` = (u, v, dense) page-locked host
    arrays of the result dtype: the payloads are streamed into them while the
    assembly runs (hbem_hmat_desc.out_*), wave by wave."""
    rows, cols = tree.rows, tree.cols
    la = tree.leaf_array
    if not (len(leaf_ids) == len(la) and np.array_equal(leaf_ids, np.arange(len(la)))):
        la = la[leaf_ids]
    la = np.ascontiguousarray(la, np.int64)
    keep = [la]
    d = _lib.HmatDesc()
    rp = np.ascontiguousarray(rows.permutation, np.int64)
    cp = np.ascontiguousarray(cols.permutation, np.int64)
    rn = np.ascontiguousarray(rows.node_array, np.int64)
    cn = np.ascontiguousarray(cols.node_array, np.int64)
    tdm = np.ascontiguousarray(test_space.dofmap, np.int64)
    sdm = np.ascontiguousarray(trial_space.dofmap, np.int64)
    keep += [rp, cp, rn, cn, tdm, sdm]
    d.n_rows, d.n_cols = len(rp), len(cp)
    d.row_perm, d.col_perm = _lib.ptr(rp, C.c_int64), _lib.ptr(cp, C.c_int64)
    d.n_row_nodes, d.n_col_nodes = len(rn), len(cn)
    d.row_nodes, d.col_nodes = _lib.ptr(rn, C.c_int64), _lib.ptr(cn, C.c_int64)
    d.n_leaves = len(la)
    d.leaves = _lib.ptr(la, C.c_int64)
    d.test_dofmap, d.trial_dofmap = _lib.ptr(tdm, C.c_int64), _lib.ptr(sdm, C.c_int64)
    d.epsilon = float(cfg.epsilon)
    d.k_max = int(cfg.k_max) if cfg.k_max is not None else 0
    d.rank_capacity = int(acfg.rank_capacity)
    d.pointers_on_device = 0
    if out is not None:
        rd = np.dtype(dev_ctx.spec.result_dtype)
        for a in out:
            if a.dtype != rd:
                raise ConfigError(f"output arenas must have dtype {rd}, got {a.dtype}")
        d.out_u, d.out_v, d.out_dense = (_lib.vptr(a) for a in out)
        d.out_u_cap, d.out_v_cap, d.out_dense_cap = (len(a) for a in out)
    h = C.c_void_p()
    # rank capacity (the per-block factor-table size of the device ACA): the
    # reference's ACA runs on to min(m, n) terms, so a block that exhausts the
    # table re-runs the assembly with a doubled table (up to the largest
    # admissible block dimension, where the k_max fallback always applies
    # first) instead of failing
    cap, retries = int(acfg.rank_capacity), 0
    rsz, csz = rn[:, 1] - rn[:, 0], cn[:, 1] - cn[:, 0]
    adm = la[:, 2] == 1
    kcap = int(np.minimum(rsz[la[adm, 0]], csz[la[adm, 1]]).max()) if adm.any() else 1
    while True:
        d.rank_capacity = cap
        status = lib.hbem_hmat_assemble(dev_ctx.handle, C.byref(d), stream, C.byref(h))
        if status == _lib.HBEM_OK:
            break
        msg = lib.hbem_last_error().decode("utf-8", "replace")
        if status != 2 or "rank capacity" not in msg or cap >= kcap:
            check(status)
        cap, retries = min(2 * cap, max(kcap, 1)), retries + 1
    def shapes():  # leaf (h, w), only needed for host payload views
        rsz, csz = rn[:, 1] - rn[:, 0], cn[:, 1] - cn[:, 0]
        return np.stack([rsz[la[:, 0]], csz[la[:, 1]]], 1)

    part = _DevicePart(h, len(la), shapes, dev_ctx.spec.result_dtype, n_rows=len(rp),
                       context=dev_ctx)
    part.capacity_retries = retries
    part.stats["capacity_retries"] = retries
    if out is not None:
        s = part.stats
        part._arenas = (out[0][: s["u_entries"]], out[1][: s["v_entries"]],
                        out[2][: s["dense_entries"]])
        part._streamed = True
    return part


COUNTER_NAMES = ("host_jobs", "backend_jobs", "singular_pairs", "aca_converged", "aca_exhausted",
                 "aca_fallback_dense", "dense_leaves", "lowrank_leaves")


def assemble_hmatrix(spec: OperatorSpec, test_space, trial_space, block_tree: BlockClusterTree,
                     cfg: AcaConfig | None = None, backends: Sequence[GpuBackend] | None = None,
                     assembly_config: AssemblyConfig | None = None,
                     stats: dict | None = None, out=None) -> HMatrix:
    """hmatrix.py:759-811 on the GPU (see module docstring).

    ``out`` (single device): page-locked host arrays (u, v, dense) of the
    result dtype (``pinned_empty``) that receive the payloads while the
    assembly runs: converged low-rank factors stream over PCIe wave by wave,
    dense leaves when the near field completes, so the host copy of the
    H-matrix is complete when the call returns."""
    cfg = cfg if cfg is not None else AcaConfig()
    acfg = assembly_config if assembly_config is not None else AssemblyConfig()
    if block_tree.shape != (test_space.n_dofs, trial_space.n_dofs):
        raise ConfigError(f"block tree shape {block_tree.shape} does not match spaces "
                          f"({test_space.n_dofs}, {trial_space.n_dofs})")
    backends = list(backends) if backends else []
    for b in backends:
        if b.context.spec != spec:
            raise ConfigError("backend was initialized for a different operator spec")
    if acfg.devices:
        backends = backends[: acfg.devices]
    if backends:
        dev_ctxs = [b.context for b in backends]
    else:
        ictx = make_integration_context(spec, test_space, trial_space, acfg.regular_order,
                                        acfg.singular_base_order)
        dev_ctxs = [init_gpu_device(ictx, 0)]
    if out is not None and len(dev_ctxs) != 1:
        raise ConfigError("out= streaming takes one device; pass out per part otherwise")
    splits = split_leaves(block_tree, len(dev_ctxs))
    parts: list = [None] * len(dev_ctxs)
    errors: list = []

    def run(i):
        try:
            parts[i] = _assemble_part(dev_ctxs[i], block_tree, splits[i], test_space,
                                      trial_space, cfg, acfg, out=out)
        except Exception as exc:  # noqa: BLE001 - re-raised in the caller
            errors.append((i, exc))

    if len(dev_ctxs) == 1:
        run(0)
    else:
        threads = [threading.Thread(target=run, args=(i,)) for i in range(len(dev_ctxs))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if errors:
        i, exc = errors[0]
        ids = splits[i]
        # a failure the device attributes to one block is reported like the
        # reference's assemble_leaf (hmatrix.py:745-751), else by device range
        blk = re.search(r"block rows \[\d+, \d+\) x cols \[\d+, \d+\)", str(exc))
        if blk:
            raise AssemblyError(f"{blk.group(0)} failed: {exc}") from exc
        raise AssemblyError(f"device {i} failed assembling leaves [{ids[0] if len(ids) else 0}, "
                            f"{ids[-1] + 1 if len(ids) else 0}): {exc}") from exc
    part_list = [(splits[i], parts[i]) for i in range(len(parts))]
    if stats is not None:
        agg: dict = {k: 0 for k in COUNTER_NAMES}
        extra: dict = {}
        for _, p in part_list:
            s = p.stats
            for key in ("singular_pairs", "aca_converged", "aca_exhausted", "aca_fallback_dense",
                        "dense_leaves", "lowrank_leaves"):
                agg[key] += int(s[key])
            agg["backend_jobs"] += int(s["row_jobs"] + s["col_jobs"])
            for key in ("regular_pairs", "waves", "row_jobs", "col_jobs", "u_entries",
                        "v_entries", "dense_entries", "capacity_retries", "sing_table_pairs"):
                extra[key] = extra.get(key, 0) + int(s[key])
            extra["device_seconds"] = max(extra.get("device_seconds", 0.0), float(s["seconds"]))
        stats.update(agg)
        stats.update(extra)
    return HMatrix(block_tree, _Payloads(part_list), spec, tuple(part_list))
