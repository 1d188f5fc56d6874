"""CPU tests of the C ABI: the library loads, exports every symbol declared in
include/hbem_b200.h, and the host-side (C++) partition is bit-exact against
the reference's golden partitions.  No compute calls that need a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "hbem_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(hbem_\w+)\(", txt, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1711_01897_b200 import _lib
    so = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(so, s), s
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert set(syms) == bound
    assert _lib.lib.hbem_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    from paper_1711_01897_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layout_matches_header(tmp_path):
    """Compile a probe against include/hbem_b200.h and compare every field
    offset with the ctypes mirror."""
    import subprocess
    from paper_1711_01897_b200 import _lib
    structs = {"hbem_ctx_desc": _lib.CtxDesc, "hbem_hmat_desc": _lib.HmatDesc,
               "hbem_hmat_stats": _lib.HmatStats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "hbem_b200.h"',
             "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    for line in out.splitlines():
        cname, field, val = line.split()
        py = structs[cname]
        got = ctypes.sizeof(py) if field == "size" else getattr(py, field).offset
        assert got == int(val), (cname, field, got, val)


def test_device_count_without_gpu_is_zero_or_more():
    from paper_1711_01897_b200 import _lib
    assert _lib.device_count() >= 0


@pytest.mark.parametrize("name", ["ico3_p0", "ico2_p1c", "ico2_p1d", "geo11_p0", "geo45_p0"])
def test_partition_bit_exact_vs_reference(name):
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    from paper_1711_01897_b200.meshes import geodesic_sphere
    from paper_1711_01897_b200.partition import cluster_trees_for
    g = golden("partitions")
    if name.startswith("ico"):
        m = golden("meshes")
        lv = int(name[3])
        v, e = m[f"ico{lv}_vertices"], m[f"ico{lv}_elements"]
    else:
        v, e = geodesic_sphere(int(name[3:5]))
    sp = build_space(TriangleMesh(v, e), name.split("_")[1])
    bt = cluster_trees_for(sp, sp)
    assert bt.rows is bt.cols
    assert np.array_equal(bt.rows.permutation, g[f"{name}_perm"])
    assert np.array_equal(bt.rows.node_array, g[f"{name}_nodes"])
    assert np.array_equal(bt.rows.bbox, g[f"{name}_bbox"])
    assert np.array_equal(bt.leaf_array, g[f"{name}_leaves"])


def test_partition_matches_oracle_on_hull():
    """A non-spherical (elongated) mesh: C++ partition vs numpy oracle."""
    from oracle import hbem_oracle as O
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    from paper_1711_01897_b200.meshes import elongated_hull
    from paper_1711_01897_b200.partition import cluster_trees_for
    v, e = elongated_hull(24, 40)
    for fam in ("p0", "p1c"):
        sp = build_space(TriangleMesh(v, e), fam)
        bt = cluster_trees_for(sp, sp, n_min=16)
        P = O.Problem(O.Spec("laplace", "slp"), v, e, fam, fam)
        tree = O.cluster_tree(P.dof_centers(fam), 16)
        assert np.array_equal(bt.rows.permutation, tree.permutation)
        assert np.array_equal(np.array(O.block_tree(tree, tree, 2.0)), bt.leaf_array)


def test_partition_edge_cases():
    from paper_1711_01897_b200.errors import ConfigError
    from paper_1711_01897_b200.partition import build_block_tree, build_cluster_tree
    t = build_cluster_tree(np.zeros((1, 3)), 32)
    assert len(t.nodes) == 1 and t.root.is_leaf
    pts = np.zeros((64, 3))
    pts[:, 0] = np.arange(64.0)
    t = build_cluster_tree(pts, 16)
    assert len(t.leaves()) == 4
    assert all(t.nodes[i].size == 16 for i in t.leaves())
    with pytest.raises(ConfigError):
        build_cluster_tree(np.zeros((0, 3)))
    with pytest.raises(ConfigError):
        build_cluster_tree(np.zeros((4, 3)), n_min=0)
    with pytest.raises(ConfigError):
        build_block_tree(t, t, eta=-1.0)
    b0 = build_block_tree(t, t, eta=0.0)
    assert not b0.leaf_array[:, 2].any()


def test_discretization_rules_match_reference():
    from paper_1711_01897_b200.discretization import PairKind, regular_rule, singular_rule
    g = golden("rules")
    for order in (1, 2, 3, 4):
        r = regular_rule(order)
        assert np.array_equal(r.points, g[f"reg{order}_points"])
        assert np.array_equal(r.weights, g[f"reg{order}_weights"])
    names = {"vertex": PairKind.SHARED_VERTEX, "edge": PairKind.SHARED_EDGE,
             "identical": PairKind.IDENTICAL}
    for base in (2, 4):
        for n, k in names.items():
            r = singular_rule(k, base)
            assert np.array_equal(r.points, g[f"sing{base}_{n}_points"])
            assert np.array_equal(r.weights, g[f"sing{base}_{n}_weights"])
