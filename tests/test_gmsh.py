"""Native Gmsh 2.2 reader (csrc/gmsh.cpp, meshes.load_mesh) against the
reference's load_mesh (mesh.py:134-245): the committed fixture read by the
REAL reference (tests/golden/make_gmsh_golden.py) bit for bit, and the
reference's own load_mesh tests (tests/test_mesh.py:123-183) with their
error classes, messages, line numbers and sections.  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

GMSH_TETRA = """\
$MeshFormat
2.2 0 8
$EndMeshFormat
$Nodes
4
1 0 0 0
2 1 0 0
3 0 1 0
4 0 0 1
$EndNodes
$Elements
5
1 1 2 0 1 1 2
2 2 2 0 1 1 3 2
3 2 2 0 1 1 2 4
4 2 2 0 1 1 4 3
5 2 2 0 1 2 3 4
$EndElements
"""


def _load(path):
    from paper_1711_01897_b200.meshes import load_mesh
    return load_mesh(path)


def test_fixture_matches_reference_reader_bitwise():
    g = golden("gmsh")
    m = _load(os.path.join(GOLDEN, "hull.msh"))
    assert m.vertices.dtype == np.float64 and m.elements.dtype == np.int64
    assert np.array_equal(m.vertices.view(np.uint64), g["vertices"].view(np.uint64))
    assert np.array_equal(m.elements, g["elements"])
    assert m.meta["skipped_elements"] == int(g["skipped"])


def test_reads_triangles_and_skips_other_types(tmp_path):
    from paper_1711_01897_b200.scatter import _check_closed_oriented
    path = tmp_path / "tetra.msh"
    path.write_text(GMSH_TETRA)
    m = _load(path)
    assert m.n_vertices == 4 and m.n_elements == 4
    assert m.meta["skipped_elements"] == 1
    assert np.array_equal(m.elements, [[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]])
    _check_closed_oriented(m)


def test_parsing_is_deterministic(tmp_path):
    path = tmp_path / "tetra.msh"
    path.write_text(GMSH_TETRA)
    a, b = _load(path), _load(path)
    assert np.array_equal(a.vertices, b.vertices) and np.array_equal(a.elements, b.elements)


def test_missing_file(tmp_path):
    from paper_1711_01897_b200.errors import MeshError, MeshParseError
    p = tmp_path / "nope.msh"
    with pytest.raises(MeshError) as ei:
        _load(p)
    assert not isinstance(ei.value, MeshParseError)
    try:
        open(p)
    except OSError as exc:
        assert str(ei.value) == f"cannot read mesh file {p}: {exc}"


@pytest.mark.parametrize("text,msg,line,section", [
    (GMSH_TETRA.replace("2.2 0 8", "4.1 0 8"),
     "unsupported format version '4.1', expected 2.x ASCII", 2, "$MeshFormat"),
    (GMSH_TETRA.replace("2.2 0 8", "2.2 1 8"), "binary files are not supported", 2,
     "$MeshFormat"),
    (GMSH_TETRA[: GMSH_TETRA.index("$EndNodes")], "missing $EndNodes", 10, "$Nodes"),
    (GMSH_TETRA.replace("2 1 0 0", "2 1 zero 0"), "malformed node line", 7, "$Nodes"),
    (GMSH_TETRA.replace("\n4\n1 0", "\nfour\n1 0"), "expected node count", 5, "$Nodes"),
    (GMSH_TETRA.replace("3 2 2 0 1 1 2 4", "3 2 2 0 1 1 2"), "triangle with 2 nodes", 15,
     "$Elements"),
    (GMSH_TETRA.replace("3 2 2 0 1 1 2 4", "3 2 x"), "malformed element line", 15, "$Elements"),
    (GMSH_TETRA.replace("$EndElements\n", ""), "missing $EndElements", 18, "$Elements"),
    (GMSH_TETRA.replace("$MeshFormat\n2.2 0 8\n", ""), "no $MeshFormat section", None, None),
    (GMSH_TETRA[: GMSH_TETRA.index("$Elements")] + "$Elements\n1\n1 1 2 0 1 1 2\n$EndElements\n",
     "file contains no triangles", None, None),
    (GMSH_TETRA.replace("5 2 2 0 1 2 3 4", "5 2 2 0 1 2 3 9"),
     "element references unknown node tag 9", None, None),
])
def test_malformed_input_messages_match_reference(tmp_path, text, msg, line, section):
    from paper_1711_01897_b200.errors import MeshParseError
    path = tmp_path / "bad.msh"
    path.write_text(text)
    with pytest.raises(MeshParseError) as ei:
        _load(path)
    loc = [f"section {section}"] if section else []
    loc += [f"line {line}"] if line is not None else []
    want = f"bad.msh: {msg}" + (f" ({', '.join(loc)})" if loc else "")
    assert str(ei.value) == want
    assert ei.value.line == line and ei.value.section == section


def test_scatter_config_reads_mesh_file(tmp_path):
    from paper_1711_01897_b200.scatter import ScatterConfig
    path = tmp_path / "tetra.msh"
    path.write_text(GMSH_TETRA)
    m = ScatterConfig(mesh_file=str(path)).build_mesh()
    assert m.n_elements == 4


@pytest.mark.parametrize("level", [0, 1, 2, 3])
def test_icosphere_matches_reference_refine_unit_sphere(level):
    """ScatterConfig.sphere_level meshes: the reference's icosphere bit for
    bit (golden meshes.npz from refine_unit_sphere, mesh.py:269-310)."""
    from paper_1711_01897_b200.meshes import icosphere
    from paper_1711_01897_b200.scatter import ScatterConfig
    g = golden("meshes")
    v, f = icosphere(level)
    assert np.array_equal(v.view(np.uint64), g[f"ico{level}_vertices"].view(np.uint64))
    assert np.array_equal(f, g[f"ico{level}_elements"])
    m = ScatterConfig(sphere_level=level).build_mesh()
    assert np.array_equal(m.elements, f)


def test_icosphere_level_cap():
    from paper_1711_01897_b200.errors import MeshError
    from paper_1711_01897_b200.scatter import ScatterConfig
    with pytest.raises(MeshError):
        ScatterConfig(sphere_level=9).build_mesh()
