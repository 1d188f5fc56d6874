"""Dense Galerkin assembly on the GPU behind the reference's dense API
(`/root/reference/pkg/src/hbem/assembly.py:234-318`).

``assemble_dense(spec, test_space, trial_space, config, backends, stats)``
has the reference's signature, validation and error classes.  The m x m
element-pair sweep runs on the device kernels of the H-matrix near field:
the operator is partitioned with eta = 0 (every leaf inadmissible, so every
block is a dense leaf assembled by k_near_p0 / k_dense with the singular
table), the leaves are split across the backends' GPUs in contiguous
cost-weighted ranges, and the host scatters the leaf blocks into the
(n_test, n_trial) matrix.  Entries are element-pair integrals summed over
the carrying pairs in the order of the reference scatter.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import AssemblyError, CapacityError, ConfigError


@dataclass(frozen=True)
class AssemblyConfig:
    """assembly.py:34-63 (same fields and validation)."""

    chunk_size: int = 1 << 20
    workers: int = 1
    regular_order: int = 4
    singular_base_order: int = 4
    devices: int | None = None
    max_matrix_bytes: int = 4 << 30
    lock_stripes: int = 1024

    def __post_init__(self):
        if self.chunk_size < 1:
            raise ConfigError(f"chunk_size must be positive, got {self.chunk_size}")
        if self.workers < 1:
            raise ConfigError(f"workers must be positive, got {self.workers}")
        if self.devices is not None and self.devices < 1:
            raise ConfigError(f"devices must be positive when set, got {self.devices}")
        if self.lock_stripes < 1:
            raise ConfigError(f"lock_stripes must be positive, got {self.lock_stripes}")


def split_work(total: int, parts: int) -> list[tuple[int, int]]:
    """assembly.py:66-78: contiguous near-equal ranges, larger ranges first."""
    if parts < 1:
        raise ConfigError(f"parts must be positive, got {parts}")
    base, rem = divmod(total, parts)
    ranges, start = [], 0
    for p in range(parts):
        size = base + (1 if p < rem else 0)
        ranges.append((start, start + size))
        start += size
    return ranges


def assemble_dense(spec, test_space, trial_space, config: AssemblyConfig,
                   backends: Sequence, stats: dict | None = None) -> np.ndarray:
    """Assemble one boundary operator densely on the GPU(s) of ``backends``."""
    from .hmatrix import AcaConfig, AssemblyConfig as HConfig, assemble_hmatrix
    from .partition import cluster_trees_for

    if not backends:
        raise ConfigError("assemble_dense requires at least one backend")
    use = list(backends[: config.devices] if config.devices else backends)
    for be in use:
        be_spec = getattr(getattr(be, "context", None), "spec", None)
        if be_spec is not None and be_spec != spec:
            raise AssemblyError(f"backend {be!r} was initialised for {be_spec}, not {spec}")
    dtype = np.dtype(spec.result_dtype)
    n_rows, n_cols = test_space.n_dofs, trial_space.n_dofs
    need = n_rows * n_cols * dtype.itemsize
    if need > config.max_matrix_bytes:
        raise CapacityError(f"dense {n_rows} x {n_cols} matrix needs {need:,} bytes, "
                            f"config allows {config.max_matrix_bytes:,}")
    tree = cluster_trees_for(test_space, trial_space, eta=0.0)
    # eta = 0 still admits clusters of zero diameter (coincident DOF centres,
    # e.g. P1d at a vertex): every leaf is forced dense so the sweep is exact
    tree.leaf_array[:, 2] = 0
    hstats: dict = {}
    h = assemble_hmatrix(spec, test_space, trial_space, tree, AcaConfig(), use,
                         HConfig(regular_order=config.regular_order,
                                 singular_base_order=config.singular_base_order),
                         stats=hstats)
    if int(hstats.get("lowrank_leaves", 0)) != 0:
        raise AssemblyError("dense assembly produced low-rank leaves")
    A = h.to_dense()
    if stats is not None:
        m = len(test_space.mesh.elements)
        stats.update({
            "pairs_total": m * m,
            "pairs_singular": int(hstats["singular_pairs"]),
            "pairs_regular": m * m - int(hstats["singular_pairs"]),
            "devices_used": len(use),
            "matrix_bytes": need,
            "dense_leaves": int(hstats["dense_leaves"]),
        })
    return A
