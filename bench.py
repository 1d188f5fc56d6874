#!/usr/bin/env python
"""bench.py — H-matrix weak-form assembly on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[4], the headline; fits one GPU): Laplace
single-layer, P0, geodesic sphere of frequency 448 = 4 014 080 triangles =
4 014 080 unknowns, ACA eps 1e-3, FP64, n_min 32, eta 2, regular order 4,
singular base order 4.  A "step" is one complete H-matrix assembly (all
near-field leaves + ACA of all admissible leaves) over the resident mesh and
partition.  The partition (cluster + block tree) is the input of
assemble_hmatrix in the reference API and is built before timing.

N > 1 (torchrun, one process per GPU): the leaves are split into N
contiguous cost-weighted ranges; each rank assembles its range with no
data-path collective (total work fixed => "scaling": "strong").

Arms:
  default          the CUDA path (libhbem_b200.so), device-resident inputs;
                   "e2e" re-runs through the public API from host buffers
                   (mesh + partition H2D, factors + dense payloads D2H into
                   pinned host arenas).
  --impl reference the reference algorithm on the host CPU cores: the CPU
                   oracle (numpy restatement, oracle/hbem_oracle.py; the
                   reference is pure Python/numpy so there is no compiled
                   oracle/_ref) with its own numpy partition, assembling a
                   uniform random sample of the C5 leaves with one process per
                   core, plus one complete C1 assembly on one core.  No product
                   native code is loaded on this arm.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "H-matrix weak-form assembly wall time (s) and element-pair integrals/s per GPU"
UNIT = "element-pair integrals/s"
# algorithmic FLOP per regular Laplace-SLP P0 pair:
# 36 quadrature-point pairs x (diff 3 + r^2 5 + accumulate 2) = 360 FLOP
# (+ 36 rsqrt, not counted as FLOP)
FLOP_PER_PAIR_LAP_SLP_P0 = 360
# issued FP64 instructions per regular pair in k_aca_p0's quadrature (SASS, round 2:
# local-frame r^2 = 1 DADD + 3 DFMA, folded rsqrt polynomial DMUL + 2 DFMA, weight
# DMUL + accumulate DFMA = 9 per quadrature-point pair, + 1 MUFU.RSQ64H) + 2 scale
DP_INSTR_PER_PAIR = 9 * 36 + 2


def _ncu_traffic():
    """DRAM bytes per k_aca_p0 launch (dram__bytes_read.sum + dram__bytes_write.sum,
    averaged over the 30 launches of one C5 FP64 assembly) from the committed ncu
    capture profiles/r02_traffic_k_aca_p0.json; None when absent."""
    p = os.path.join(ROOT, "profiles", "r02_traffic_k_aca_p0.json")
    try:
        with open(p) as f:
            return float(json.load(f)["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=448, help="geodesic sphere frequency (20 n^2 tri)")
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--precision", default="double", choices=["double", "single"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="bounded CPU sample per baseline measurement")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-reps", type=int, default=3, help="end-to-end repetitions (median)")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def workload(args):
    from paper_1711_01897_b200.discretization import OperatorSpec, TriangleMesh, build_space
    from paper_1711_01897_b200.meshes import geodesic_sphere
    from paper_1711_01897_b200.partition import cluster_trees_for
    v, e = geodesic_sphere(args.n)
    mesh = TriangleMesh(v, e)
    sp = build_space(mesh, "p0")
    t0 = time.perf_counter()
    bt = cluster_trees_for(sp, sp)
    _TIMES["partition_s"] = time.perf_counter() - t0
    spec = OperatorSpec("laplace", "slp", 0.0, args.precision)
    return v, e, mesh, sp, bt, spec


def config(args, world):
    return {"workload": f"C5: Laplace SLP P0, geodesic sphere n={args.n} "
                        f"({20 * args.n * args.n} triangles = unknowns), ACA eps={args.eps:g}, "
                        f"{args.precision}, n_min=32, eta=2",
            "n_unknowns": 20 * args.n * args.n, "eps": args.eps,
            "parallelism": f"leaf-split x{world} (cost-weighted contiguous ranges)",
            "l2": "inputs (geometry 0.6 GB) and outputs (~60 GB factors) exceed the 126 MB L2"}


# ---------------------------------------------------------------------------
# clocks sampling (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.rows = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([t.strip() for t in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU arm: the oracle on sampled leaves
# ---------------------------------------------------------------------------
_G = {}
_TIMES = {}


def _oracle_setup(v, e, bt, eps, precision):
    from oracle import hbem_oracle as O
    P = O.Problem(O.Spec("laplace", "slp", 0.0, precision), v, e, "p0", "p0")
    na, bb = bt.rows.node_array, bt.rows.bbox
    nodes = [O.Node(int(r[0]), int(r[1]), int(r[2]), bb[i, :3], bb[i, 3:], int(r[3]), int(r[4]))
             for i, r in enumerate(na)]
    tree = O.Tree(nodes, np.asarray(bt.rows.permutation))
    leaves = [tuple(int(t) for t in row) for row in bt.leaf_array]
    _G["asm"] = O.Assembler(P, tree, tree, leaves, eps)


def _oracle_leaves(ids, seconds=None):
    """Assemble leaves ``ids`` in order with the oracle, stopping after
    ``seconds`` of work if given; returns (wall, regular, singular, done)."""
    asm = _G["asm"]
    asm.counters.update({"regular_pairs": 0, "singular_pairs": 0})
    t0 = time.perf_counter()
    done = 0
    for ix in ids:
        asm.leaf(int(ix))
        done += 1
        if seconds is not None and time.perf_counter() - t0 >= seconds:
            break
    return (time.perf_counter() - t0, asm.counters["regular_pairs"],
            asm.counters["singular_pairs"], done)


def _oracle_worker(arg):
    ids, seconds = arg
    return _oracle_leaves(ids, seconds)


def cpu_rate(n_leaves, seconds, workers, rng):
    """Assemble uniformly drawn leaves (an unbiased sample of the assembly's
    per-leaf work: most C5 leaves are small, and small leaves pay the
    reference's per-block host overhead) for about ``seconds`` per worker;
    returns (pairs/s, regular, singular, leaves, wall, est_single_core_s)
    with wall = the slowest worker and est_single_core_s = the whole
    assembly's single-core time extrapolated from the mean time per leaf."""
    ids = rng.permutation(n_leaves)[:200000]
    if workers <= 1:
        wall, reg, sing, done = _oracle_leaves(ids, seconds)
        return (reg + sing) / wall, reg, sing, done, wall, wall / done * n_leaves
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    chunks = [(ids[i::workers], seconds) for i in range(workers)]
    with ctx.Pool(workers) as pool:
        res = pool.map(_oracle_worker, chunks)
    wall = max(x[0] for x in res)
    reg = sum(x[1] for x in res)
    sing = sum(x[2] for x in res)
    done = sum(x[3] for x in res)
    busy = sum(x[0] for x in res)
    return (reg + sing) / wall, reg, sing, done, wall, busy / done * n_leaves


def oracle_partition(v, e):
    """The reference's partition restated in numpy (oracle.cluster_tree /
    block_tree, hmatrix.py:105-211; bit-identical to the reference's, pinned
    by tests/test_oracle_golden.py and tests/test_partition_scale.py)."""
    from oracle import hbem_oracle as O
    P = O.Problem(O.Spec("laplace", "slp"), v, e, "p0", "p0")
    tree = O.cluster_tree(P.dof_centers("p0"))
    return tree, O.block_tree(tree, tree)


def oracle_complete_c1(eps, precision):
    """One COMPLETE assembly of C1 (geodesic sphere n=11, 2 420 triangles,
    Laplace SLP P0, the reference's CPU-runnable config) with the oracle on
    one core: every leaf, ACA + near field."""
    from oracle import hbem_oracle as O
    from paper_1711_01897_b200.meshes import geodesic_sphere
    v, e = geodesic_sphere(11)
    P = O.Problem(O.Spec("laplace", "slp", 0.0, precision), v, e, "p0", "p0")
    tree = O.cluster_tree(P.dof_centers("p0"))
    leaves = O.block_tree(tree, tree)
    t0 = time.perf_counter()
    asm = O.Assembler(P, tree, tree, leaves, eps)
    asm.assemble()
    wall = time.perf_counter() - t0
    pairs = asm.counters["regular_pairs"] + asm.counters["singular_pairs"]
    return {"config": "C1: geodesic sphere n=11 (2420 triangles), Laplace SLP P0, "
                      f"eps={eps:g}, {precision}, every leaf", "seconds": wall,
            "regular_pairs": asm.counters["regular_pairs"],
            "singular_pairs": asm.counters["singular_pairs"],
            "value": pairs / wall, "unit": UNIT, "cores": 1}


def run_reference(args):
    """The reference's CPU path: the oracle (numpy restatement of
    hbem.hmatrix.assemble_hmatrix's per-leaf path: aca/_row_job/_col_job/
    dense_leaf + integrate_batch + local_matrix) over the same C5 mesh, with
    the oracle's own partition.  Nothing from the product package runs here
    except the synthetic mesh generator (pure numpy)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_1711_01897_b200.meshes import geodesic_sphere
    v, e = geodesic_sphere(args.n)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    tree, leaves = oracle_partition(v, e)
    t_part = time.perf_counter() - t0
    from oracle import hbem_oracle as O
    P = O.Problem(O.Spec("laplace", "slp", 0.0, args.precision), v, e, "p0", "p0")
    _G["asm"] = O.Assembler(P, tree, tree, leaves, args.eps)
    c1 = oracle_complete_c1(args.eps, args.precision)
    rng = np.random.default_rng(1234)
    # the whole --steps/--warmup run stays within a few minutes
    per_step = float(np.clip(240.0 / max(args.steps + args.warmup / 4, 1), 2.0, args.cpu_seconds))
    for _ in range(args.warmup):
        cpu_rate(len(leaves), min(per_step / 4, 2.0), cores, rng)
    rates, times, est = [], [], []
    for _ in range(args.steps):
        rate, reg, sing, nl, wall, est_s = cpu_rate(len(leaves), per_step, cores, rng)
        rates.append(rate)
        times.append(wall)
        est.append(est_s)
    rate = float(np.median(rates))
    assert "paper_1711_01897_b200._lib" not in sys.modules  # no product native code here
    sample = (f"{nl} leaves per step ({per_step:.1f} s per process) drawn uniformly from the "
              f"{len(leaves)} C5 leaves (oracle partition, {t_part:.0f} s); oracle on {cores} "
              "processes (the reference is single-threaded Python: one process per core)")
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.median(times)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.precision == "double" else "f32",
            "data": "synthetic geodesic sphere", "config": config(args, world),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample,
                             "extrapolated_c5_assembly_s_single_core": float(np.median(est)),
                             "extrapolated_c5_assembly_s_all_cores": float(np.median(est)) / cores,
                             "partition_s": t_part},
            "complete_c1": c1,
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import ctypes as C

    import torch

    from paper_1711_01897_b200 import _lib
    from paper_1711_01897_b200.backend import init_gpu_device
    from paper_1711_01897_b200.discretization import make_integration_context
    from paper_1711_01897_b200.hmatrix import (AcaConfig, AssemblyConfig, _assemble_part,
                                               assemble_hmatrix, split_leaves)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    v, e, mesh, sp, bt, spec = workload(args)
    ids = split_leaves(bt, world)[rank]
    cfg = AcaConfig(epsilon=args.eps)
    acfg = AssemblyConfig()
    ictx = make_integration_context(spec, sp, sp)
    dev = init_gpu_device(ictx, local)
    stream = torch.cuda.current_stream()
    sptr = C.c_void_p(stream.cuda_stream)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up 1 = setup + first execute
    part = _assemble_part(dev, bt, ids, sp, sp, cfg, acfg, stream=sptr)
    for _ in range(max(args.warmup - 1, 0)):
        part.execute(sptr)
    barrier()
    aca_ms, nf_ms, pairs, sing, aca_entries, launches = [], [], 0, 0, 0, 0
    int_ms, int_launches = 0.0, 0
    with ClockSampler(local) as clocks:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        barrier()
        t_start.record(stream)
        for _ in range(args.steps):
            part.execute(sptr)
            s = part.stats
            aca_ms.append(s["aca_kernel_ms"])
            nf_ms.append(s["nearfield_kernel_ms"])
            pairs += s["regular_pairs"] + s["singular_pairs"]
            sing += s["singular_pairs"]
            aca_entries += s["aca_entries"]
            launches += s["launches"]
            int_ms += s["int_kernel_ms"]
            int_launches += s["int_launches"]
        t_end.record(stream)
        barrier()
    elapsed = t_start.elapsed_time(t_end) / 1e3
    stats = part.stats
    tot = torch.tensor([elapsed, float(pairs), float(sing), float(launches)], dtype=torch.float64,
                       device="cuda")
    if dist is not None:
        mx = tot.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tot.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        elapsed = float(mx[0].item())
        pairs, sing, launches = float(sm[1].item()), float(sm[2].item()), int(sm[3].item())
    per_step = elapsed / args.steps
    value = pairs / elapsed

    # dominant kernel: k_aca_p0 (ACA row/column integration + fused residual),
    # FP64-pipe bound; CUDA events around each launch on its stream
    int_s = int_ms / 1e3
    flop_rate = FLOP_PER_PAIR_LAP_SLP_P0 * aca_entries / int_s if int_s > 0 else 0.0
    peak = C.c_double(0.0)
    _lib.check(_lib.lib.hbem_probe_fma(local, _lib.PRECISIONS[args.precision], C.byref(peak)))
    dp_issue = DP_INSTR_PER_PAIR * aca_entries / int_s if int_s > 0 else 0.0
    roofline = {"bound": "fp64" if args.precision == "double" else "fp32",
                "kernel": "k_aca_p0 (ACA row/column integration, fused residual + tile statistics)",
                "achieved": flop_rate / 1e12, "peak": peak.value / 1e12, "unit": "TFLOP/s",
                "frac": flop_rate / peak.value if peak.value else None,
                "traffic": _ncu_traffic(),
                "peak_source": ("measured live on this GPU: hbem_probe_fma (independent "
                                f"{'DFMA' if args.precision == 'double' else 'FFMA'} chains, "
                                "2 FLOP per FMA); MEASURED_PEAKS.json has no FP64/FP32 FMA "
                                "figure"),
                "algorithmic": f"{FLOP_PER_PAIR_LAP_SLP_P0} FLOP per regular pair (SURVEY 8d) x "
                               f"{aca_entries // max(args.steps, 1)} ACA entries per step",
                # the SASS instruction count is the FP64 kernel's
                "issue_frac": (dp_issue / (peak.value / 2)
                               if peak.value and args.precision == "double" else None),
                "issue_model": (f"{DP_INSTR_PER_PAIR} FP64 instructions per pair (9 per "
                                "quadrature-point pair, from cuobjdump -sass) / FP64 lane rate"
                                if args.precision == "double" else None),
                "launches_per_step": int_launches // max(args.steps, 1),
                "avg_launch_ms": int_ms / max(int_launches, 1),
                "int_kernel_ms_per_step": int_ms / max(args.steps, 1),
                "aca_waves_ms_per_step": float(np.mean(aca_ms)),
                "nearfield_kernel_ms_per_step": float(np.mean(nf_ms))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        _oracle_setup(v, e, bt, args.eps, args.precision)
        rate, reg, sg, nl, wall, est = cpu_rate(len(bt.leaf_array), args.cpu_seconds, 1,
                                                np.random.default_rng(7))
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{nl} C5 leaves drawn uniformly ({reg} regular + {sg} singular "
                         f"pairs in {wall:.1f} s), oracle on 1 core",
               "extrapolated_assembly_s": est}
        # release the oracle's millions of Python objects before the e2e
        # timing (the cyclic GC would otherwise scan them mid-measurement)
        import gc
        _G.clear()
        gc.collect()

    e2e = None
    if not args.no_e2e:
        # public API from host buffers: mesh + partition H2D, factors and dense
        # payloads D2H into page-locked host arenas (allocated once, reported
        # under "once" together with the partition build)
        t_pin = time.perf_counter()
        pinned = part.arenas(pinned=True)
        t_pin = time.perf_counter() - t_pin
        h2d = (v.nbytes + e.nbytes + bt.rows.permutation.nbytes + bt.rows.node_array.nbytes
               + bt.leaf_array[ids].nbytes + sp.dofmap.nbytes)
        d2h = sum(a.nbytes for a in pinned)
        part.close()
        del part
        dev.close()
        samples, splits = [], []
        part2 = None
        for rep in range(max(args.e2e_reps, 1)):
            if part2 is not None:
                part2.close()
                dev2.close()
            barrier()
            t0 = time.perf_counter()
            if world == 1:
                # the public call: assemble_hmatrix(..., out=) creates the
                # device context (mesh H2D), uploads the partition, assembles
                # and streams the payloads into the host arenas
                t1 = t0
                hm = assemble_hmatrix(spec, sp, sp, bt, cfg, None, acfg, out=pinned)
                part2 = hm.parts[0][1]
                dev2 = part2.context
            else:
                dev2 = init_gpu_device(ictx, local)
                t1 = time.perf_counter()
                # payloads streamed wave by wave into the page-locked host arenas
                part2 = _assemble_part(dev2, bt, ids, sp, sp, cfg, acfg, stream=sptr, out=pinned)
            t2 = time.perf_counter()
            s2 = part2.stats
            got = part2.arenas()
            assert all(len(g) == n for g, n in zip(got, (s2["u_entries"], s2["v_entries"],
                                                          s2["dense_entries"])))
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            t_e2e = t3 - t0
            if dist is not None:
                tt = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t_e2e = float(tt.item())
            samples.append(t_e2e)
            splits.append({"context_s": t1 - t0, "setup_s": float(s2["seconds_setup"]),
                           "assemble_s": float(s2["seconds"]),
                           "plan_assemble_and_streamed_d2h_s": t2 - t1, "tail_s": t3 - t2})
        med = float(np.median(samples))
        e2e = {"value": pairs / args.steps / med, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "seconds": med, "samples_s": samples,
               "split": splits[int(np.argsort(samples)[len(samples) // 2])],
               "once": {"pinned_arena_alloc_s": t_pin, "partition_s": _TIMES.get("partition_s"),
                        "note": "one-time costs outside the per-assembly e2e: page-locking the "
                                "host output arenas and the block-tree build (an input of "
                                "assemble_hmatrix in the reference API)"},
               "path": ("assemble_hmatrix(..., out=page-locked arenas)" if world == 1 else
                        "GpuDeviceContext + _assemble_part(leaf range)") +
                       ": context (mesh H2D), partition upload, assembly with factors "
                       "streamed per ACA wave and dense leaves when the near field "
                       f"completes; median of {len(samples)} repetitions"}
        part = part2

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * per_step,
                "assembly_wall_s": per_step, "per_gpu": value / world,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "published_reference": "paper: ~100 min on 2x GTX TITAN Black for ~4M unknowns "
                                       "(PAPER.md:25; different hardware, not a ratio)",
                "dtype": "f64" if args.precision == "double" else "f32",
                "data": "synthetic geodesic sphere (no external mesh)",
                "config": config(args, world),
                "pairs_per_step": {"regular": int((pairs - sing) / args.steps),
                                   "singular": int(sing / args.steps)},
                "aca": {"waves": stats["waves"], "row_jobs": stats["row_jobs"],
                        "host_wall_s": {"waves": stats["seconds_aca"],
                                        "classify_expand_copyback": stats["seconds_finalize"]},
                        "lowrank_leaves": stats["lowrank_leaves"],
                        "dense_leaves": stats["dense_leaves"],
                        "stored_entries": stats["u_entries"] + stats["v_entries"]
                        + stats["dense_entries"]},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    part.close()
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
