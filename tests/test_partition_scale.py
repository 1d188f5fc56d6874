"""The C++ partitioner (csrc/partition.cpp) against the REAL reference's
partitions at the BASELINE config scales: C2 (geo45 P1c), C3 (geo71 P0), the
C4 hull (P0 / P1c / P1d, 0.25-1.5 M DOFs) and C5 (geo448 P0, 4 014 080 DOFs).

The expected values are sha256 digests of the reference's
``cluster_trees_for`` output (hmatrix.py:105-211, 814-826) written by
``tests/golden/make_partition_digests.py`` in the build container: the
permutation, the node table, the node bounding boxes (exact float64 bits) and
the leaf list with admissibility flags.  Bit-exactness at these scales covers
the ties of the symmetric sphere, the stable sort, ``mid = start+(size+1)//2``
and numpy's 3-vector norm evaluation (``partition.NORM_MODE``) on the very
clusters the headline assembles.  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

DIGESTS = json.load(open(os.path.join(GOLDEN, "partition_digests.json")))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _mesh(key):
    from paper_1711_01897_b200.meshes import elongated_hull, geodesic_sphere
    return geodesic_sphere(key[1]) if key[0] == "sphere" else elongated_hull(key[1], key[2])


@pytest.mark.parametrize("name", sorted(DIGESTS))
def test_partition_digest_matches_reference(name):
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    from paper_1711_01897_b200.partition import cluster_trees_for
    d = DIGESTS[name]
    v, e = _mesh(d["mesh"])
    sp = build_space(TriangleMesh(v, e), d["family"])
    bt = cluster_trees_for(sp, sp)
    t = bt.rows
    assert bt.cols is t
    assert (len(t.permutation), len(t.node_array), len(bt.leaf_array)) == \
        (d["n_dofs"], d["n_nodes"], d["n_leaves"])
    assert int(bt.leaf_array[:, 2].sum()) == d["n_admissible"]
    assert _sha(np.asarray(t.permutation, np.int64)) == d["perm"]
    assert _sha(np.asarray(t.node_array, np.int64)) == d["nodes"]
    assert _sha(np.asarray(t.bbox, np.float64)) == d["bbox"]
    assert _sha(np.asarray(bt.leaf_array, np.int64)) == d["leaves"]
