"""N > 1 host logic on CPU (gloo, world_size 2): the H-matrix path shards as
independent leaves — contiguous cost-weighted leaf ranges, one
per rank, no data-path collective.  These tests check the split and that a
2-rank sharded assembly (each rank assembling its range with the CPU oracle,
results gathered once) equals the single-process assembly bit for bit, and
that bench.py's reference arm follows the rank-0-only rule under torchrun.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, golden


def _partition(name="ico3"):
    from paper_1711_01897_b200.discretization import TriangleMesh, build_space
    from paper_1711_01897_b200.partition import cluster_trees_for
    m = golden("meshes")
    v, e = m[f"{name}_vertices"], m[f"{name}_elements"]
    sp = build_space(TriangleMesh(v, e), "p0")
    return v, e, sp, cluster_trees_for(sp, sp)


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_split_leaves_is_a_contiguous_cover(parts):
    from paper_1711_01897_b200.hmatrix import _leaf_costs, split_leaves
    _, _, _, bt = _partition()
    ids = split_leaves(bt, parts)
    assert len(ids) == parts
    cat = np.concatenate(ids)
    assert np.array_equal(cat, np.arange(len(bt.leaf_array)))
    cost = _leaf_costs(bt)
    share = np.array([cost[i].sum() for i in ids]) / cost.sum()
    # cost-weighted: no rank carries more than its share plus one leaf
    assert share.max() <= 1.0 / parts + cost.max() / cost.sum() + 1e-12


def _oracle_assembler(v, e, bt, eps):
    from oracle import hbem_oracle as O
    P = O.Problem(O.Spec("laplace", "slp"), v, e, "p0", "p0")
    na, bb = bt.rows.node_array, bt.rows.bbox
    nodes = [O.Node(int(r[0]), int(r[1]), int(r[2]), bb[i, :3], bb[i, 3:], int(r[3]), int(r[4]))
             for i, r in enumerate(na)]
    tree = O.Tree(nodes, np.asarray(bt.rows.permutation))
    leaves = [tuple(int(t) for t in row) for row in bt.leaf_array]
    return O.Assembler(P, tree, tree, leaves, eps)


def _digest(payload):
    a = payload.todense()
    return np.ascontiguousarray(a).tobytes()


def _rank_main(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_01897_b200.hmatrix import split_leaves
    v, e, _, bt = _partition()
    asm = _oracle_assembler(v, e, bt, 1e-3)
    mine = split_leaves(bt, world)[rank]
    local = {int(ix): _digest(asm.leaf(int(ix))) for ix in mine}
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    if rank == 0:
        merged = {}
        for g in gathered:
            assert not set(g) & set(merged)      # every leaf on exactly one rank
            merged.update(g)
        out.put(merged)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_assembly_equals_single_process():
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    v, e, _, bt = _partition()
    asm = _oracle_assembler(v, e, bt, 1e-3)
    assert sorted(merged) == list(range(len(bt.leaf_array)))
    for ix in range(len(bt.leaf_array)):
        assert merged[ix] == _digest(asm.leaf(ix)), ix


@pytest.mark.parametrize("rank", [0, 1])
def test_bench_reference_arm_rank_rule(rank):
    env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", LOCAL_RANK=str(rank),
               MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--n", "8", "--steps", "1", "--warmup", "1", "--cpu-seconds", "1"],
                       env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if rank == 0:
        import json
        d = json.loads(lines[-1])
        assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
        assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0
    else:
        assert lines == []
