"""Partition digests of the REAL reference at the BASELINE config scales
(build container only; ~5 minutes, dominated by C5):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_partition_digests.py

Runs the reference's own ``cluster_trees_for`` (hmatrix.py:814-826, i.e.
``build_cluster_tree`` 105-140 + ``build_block_tree`` 182-211) on the meshes
the configs name and writes sha256 digests of the flattened arrays into
``partition_digests.json``:

* ``perm``   int64 (n,)      ClusterTree.permutation
* ``nodes``  int64 (nn, 5)   start, stop, level, left, right per node
* ``bbox``   float64 (nn, 6) bbox_min, bbox_max per node (exact bits)
* ``leaves`` int64 (L, 3)    row_node, col_node, admissible per leaf

The full arrays (≈150 MB at C5) are not committed; the digests pin the
C++ partitioner bit for bit (tests/test_partition_scale.py).  The meshes are
the repo's generators (``paper_1711_01897_b200.meshes``), so both stacks see
identical vertex bits."""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from hbem.hmatrix import cluster_trees_for  # noqa: E402
from hbem.mesh import TriangleMesh  # noqa: E402
from hbem.spaces import build_space  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1711_01897_b200.meshes import elongated_hull, geodesic_sphere  # noqa: E402

# name -> (mesh generator args, family)
CASES = {
    "C2_geo45_p1c": (("sphere", 45), "p1c"),
    "C3_geo71_p0": (("sphere", 71), "p0"),
    "C4_hull180x1400_p0": (("hull", 180, 1400), "p0"),
    "C4_hull180x1400_p1c": (("hull", 180, 1400), "p1c"),
    "C4_hull180x1400_p1d": (("hull", 180, 1400), "p1d"),
    "C5_geo448_p0": (("sphere", 448), "p0"),
}


def mesh_of(key):
    if key[0] == "sphere":
        return geodesic_sphere(key[1])
    return elongated_hull(key[1], key[2])


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def arrays(bt):
    t = bt.rows
    nodes = np.array([(nd.start, nd.stop, nd.level, nd.left, nd.right) for nd in t.nodes],
                     dtype=np.int64)
    bbox = np.array([np.concatenate([nd.bbox_min, nd.bbox_max]) for nd in t.nodes],
                    dtype=np.float64)
    leaves = np.array([(lf.row_node, lf.col_node, int(lf.admissible)) for lf in bt.leaves],
                      dtype=np.int64)
    return np.asarray(t.permutation, np.int64), nodes, bbox, leaves


def main(names):
    path = os.path.join(HERE, "partition_digests.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        key, fam = CASES[name]
        v, e = mesh_of(key)
        sp = build_space(TriangleMesh(v, e), fam)
        t0 = time.perf_counter()
        bt = cluster_trees_for(sp, sp)
        secs = time.perf_counter() - t0
        perm, nodes, bbox, leaves = arrays(bt)
        out[name] = {"mesh": list(key), "family": fam, "n_dofs": int(len(perm)),
                     "n_nodes": int(len(nodes)), "n_leaves": int(len(leaves)),
                     "n_admissible": int(leaves[:, 2].sum()),
                     "perm": sha(perm), "nodes": sha(nodes), "bbox": sha(bbox),
                     "leaves": sha(leaves), "reference_seconds": round(secs, 1)}
        print(name, out[name], flush=True)
        del bt
        with open(path, "w") as f:
            json.dump(out, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
