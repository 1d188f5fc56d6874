"""Gmsh 2.2 fixture + the REAL reference's reading of it (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_gmsh_golden.py

Writes ``hull.msh``: a small closed hull (elongated_hull(12, 20), 480
triangles) with non-contiguous shuffled node tags, unused nodes, a repeated
node tag (the last definition wins), line (type 1) and point (type 15)
elements mixed in, tags per element, CRLF line ends on part of the file and
coordinates printed with 17 significant digits.  ``gmsh.npz`` holds the
vertices / elements / skipped count that the reference's ``load_mesh``
(mesh.py:134-245) returns for it; tests/test_gmsh.py checks the native
reader against them bit for bit."""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from hbem.mesh import load_mesh  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1711_01897_b200.meshes import elongated_hull  # noqa: E402


def write_fixture(path):
    rng = np.random.default_rng(2024)
    v, e = elongated_hull(12, 20)
    tags = rng.permutation(np.arange(len(v) + 40))[: len(v)] * 3 + 7   # sparse, shuffled
    lines = ["$MeshFormat", "2.2 0 8", "$EndMeshFormat", "$Comments", "synthetic hull",
             "$EndComments", "$Nodes"]
    extra = [(int(tags.max()) + 5, (9.0, 9.0, 9.0))]                  # unused node
    node_lines = [f"{t} {float(x)!r} {float(y)!r} {float(z)!r}" for t, (x, y, z) in zip(tags, v)]
    # a repeated tag: an early bogus definition overridden later
    node_lines.insert(3, f"{tags[10]} 1e3 -2.5 0.125")
    node_lines += [f"{t} {x} {y} {z}" for t, (x, y, z) in extra]
    lines += [str(len(node_lines))] + node_lines + ["$EndNodes", "$Elements"]
    el = []
    k = 1
    for i, (a, b, c) in enumerate(e):
        if i % 50 == 0:
            el.append(f"{k} 15 2 0 {i} {tags[a]}")                        # point
            k += 1
        if i % 37 == 0:
            el.append(f"{k} 1 2 0 {i} {tags[a]} {tags[b]}")               # line
            k += 1
        el.append(f"{k} 2 {2 + i % 3} " + " ".join(["7"] * (2 + i % 3)) +
                  f" {tags[a]} {tags[b]} {tags[c]}")
        k += 1
    lines += [str(len(el))] + el + ["$EndElements"]
    half = len(lines) // 2
    text = "\r\n".join(lines[:half]) + "\r\n" + "\n".join(lines[half:]) + "\n"
    with open(path, "w", newline="") as f:
        f.write(text)


def main():
    path = os.path.join(HERE, "hull.msh")
    write_fixture(path)
    m = load_mesh(path)
    np.savez_compressed(os.path.join(HERE, "gmsh.npz"), vertices=m.vertices,
                        elements=m.elements, skipped=m.meta["skipped_elements"])
    print("hull.msh:", m.n_vertices, "vertices", m.n_elements, "triangles",
          m.meta["skipped_elements"], "skipped")


if __name__ == "__main__":
    main()
