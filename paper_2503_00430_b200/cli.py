"""bfsbench-compatible command line over the GPU path.

  python -m paper_2503_00430_b200.cli stats    --gen kron:20:16:1 | --graph FILE
  python -m paper_2503_00430_b200.cli verify   --gen ... [--variants all] [--sources 64]
  python -m paper_2503_00430_b200.cli run      --gen ... --out DIR [--trials 3 --warmups 1]
  python -m paper_2503_00430_b200.cli generate --gen ... --out FILE

Same subcommands, options, CSV schemas and exit codes as the reference's
tools/bfsbench.cpp:532-603 (0 ok, 1 verification/correctness failure,
2 configuration error, 3 input/format error). Differences, by design:

* ``verify`` has no CPU traversal to compare against (the product contains
  none); it checks that every GPU variant returns the identical distance
  array and that the array is a BFS layering of the graph — dist[src] = 0,
  no arc crosses more than one level or leaves the reached set, and every
  reached vertex but the source has a neighbour one level closer. Those three
  properties characterise the BFS distances uniquely.
* ``--threads`` is accepted for compatibility and ignored (one GPU).
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

from . import parbfs as pb

GPU_VARIANTS = [pb.KernelVariant.Conventional, pb.KernelVariant.NonAtomic,
                pb.KernelVariant.Hybrid, pb.KernelVariant.HybridBeamer,
                pb.KernelVariant.VisitedBitmapInline]


def parse_gen_spec(text: str) -> pb.GeneratorSpec:
    """bfsbench.cpp:153-174 (plus ``mesh:SIDE:0:SEED`` for config 3)."""
    parts = text.split(":")
    if len(parts) != 4:
        raise pb.ConfigError(f'generator spec must be KIND:SCALE:EF:SEED, got "{text}"')
    try:
        a, b, seed = int(parts[1]), int(parts[2]), int(parts[3])
    except ValueError:
        raise pb.ConfigError(f'bad generator spec "{text}"')
    if parts[0] == "uniform":
        return pb.GeneratorSpec(pb.GeneratorKind.UniformRandom, a, b, seed)
    if parts[0] == "kron":
        return pb.GeneratorSpec(pb.GeneratorKind.Kronecker, a, b, seed)
    if parts[0] == "mesh":
        return pb.GeneratorSpec(pb.GeneratorKind.Mesh, seed=seed, mesh_side=a)
    raise pb.ConfigError(f'unknown generator kind "{parts[0]}" (use uniform, kron or mesh)')


def load_graph(args):
    """bfsbench.cpp:183-204."""
    if args.gen:
        spec = parse_gen_spec(args.gen)
        if args.drop_self_loops:
            spec.drop_self_loops = True
        return pb.generate(spec), pb.to_string(spec) if spec.kind != pb.GeneratorKind.Mesh \
            else f"mesh:{spec.mesh_side}:0:{spec.seed}"
    if not args.graph:
        raise pb.ConfigError("provide a graph with --graph FILE or --gen SPEC")
    try:
        with open(args.graph, "rb") as f:
            binary = f.read(4) == b"CSR1"
    except OSError:
        raise pb.InputError(f"cannot open {args.graph}")
    if binary:
        return pb.load_binary_csr(args.graph), args.graph
    return pb.load_edge_list(args.graph, args.one_based, not args.no_symmetrize), args.graph


def pick_sources(graph, args):
    """bfsbench.cpp:206-235."""
    if args.source_list:
        out = []
        for tok in args.source_list.split(","):
            try:
                v = int(tok)
            except ValueError:
                raise pb.ConfigError(f'bad source vertex: "{tok}"')
            if v < 0 or v >= graph.vertex_count:
                raise pb.ConfigError(f"source vertex {tok} is out of range for "
                                     f"{graph.vertex_count} vertices")
            out.append(v)
        return out
    return [int(s) for s in pb.pick_sources(graph, args.sources, args.seed)]


def parse_variants(text: str):
    """bfsbench.cpp:248-260, restricted to the variants with a GPU kernel."""
    if text == "all":
        return list(GPU_VARIANTS)
    out = []
    for tok in text.split(","):
        v = pb.parse_kernel_variant(tok)
        if v is None:
            raise pb.ConfigError(f'unknown variant "{tok}"')
        if v not in out:
            out.append(v)
    if not out:
        raise pb.ConfigError("no variants selected")
    return out


def make_config(args, variant) -> pb.KernelConfig:
    return pb.KernelConfig(variant=variant, hybrid_threshold_fraction=args.hybrid_threshold,
                           alpha=args.alpha, beta=args.beta, flush_capacity=args.flush_capacity)


def bfs_layering_ok(graph, dist, source):
    """Certificate that `dist` is the BFS distance array from `source`."""
    unreached = 0xFFFFFFFF
    if dist[source] != 0:
        return False, source
    deg = graph.degrees()
    d = dist.astype(np.int64)
    d[dist == unreached] = -1
    src = np.repeat(np.arange(graph.vertex_count, dtype=np.int64), deg)
    du, dv = d[src], d[graph.column_indices]
    bad = ((du < 0) != (dv < 0)) | ((du >= 0) & (np.abs(du - dv) > 1))
    if bad.any():
        return False, int(src[np.argmax(bad)])
    big = np.iinfo(np.int64).max
    nb = np.where(dv >= 0, dv, big)
    mins = np.full(graph.vertex_count, big, dtype=np.int64)
    has = deg > 0
    if has.any():
        mins[has] = np.minimum.reduceat(nb, graph.row_offsets[:-1][has].astype(np.int64))
    lack = (d > 0) & (mins != d - 1)
    if lack.any():
        return False, int(np.argmax(lack))
    return True, -1


def cmd_stats(args) -> int:
    """bfsbench.cpp:319-331."""
    g, label = load_graph(args)
    s = pb.compute_stats(g, args.classifier_threshold)
    print(f"graph: {label}\nvertices: {s.vertex_count}\nedges: {s.edge_count}\n"
          f"average degree: {s.average_degree:.2f}\nmax degree: {s.max_degree}\n"
          f"category: {pb.to_string(s.category)}")
    return 0


def cmd_verify(args) -> int:
    """bfsbench.cpp:333-399, certified without a CPU traversal (module doc)."""
    g, label = load_graph(args)
    stats = pb.compute_stats(g, args.classifier_threshold)
    sources = pick_sources(g, args)
    variants = parse_variants(args.variants)
    print(f"graph: {label} ({g.vertex_count} vertices, {g.edge_count} directed edges, "
          f"{pb.to_string(stats.category)})\nchecking {len(variants)} variants x "
          f"{len(sources)} sources (BFS layering certificate + cross-variant agreement)")
    ok = {v: True for v in variants}
    printed = 0
    for s in sources:
        first = None
        for v in variants:
            r = pb.run_bfs(g, s, make_config(args, v), stats)
            dist = r.distances.copy()
            if args.inject_fault:
                dist[s] += 1
            good, where = bfs_layering_ok(g, dist, s)
            if good and first is not None and not np.array_equal(dist, first):
                good, where = False, int(np.argmax(dist != first))
            if first is None:
                first = dist
            if not good:
                ok[v] = False
                if printed < 10:
                    print(f"mismatch: variant={pb.to_string(v)} source={s} vertex={where} "
                          f"got={int(dist[where])}")
                    printed += 1
    if printed == 10:
        print("further mismatches suppressed")
    print(f"{'variant':18s}gpu")
    for v in variants:
        print(f"{pb.to_string(v):18s}{'pass' if ok[v] else 'FAIL'}")
    all_ok = all(ok.values())
    print("verification passed" if all_ok else "verification FAILED")
    return 0 if all_ok else 1


def cmd_run(args) -> int:
    """bfsbench.cpp:401-516: results.csv / traces.csv with the reference schema."""
    if not args.out:
        raise pb.ConfigError("run needs --out DIR")
    if args.trials < 1:
        raise pb.ConfigError("trials must be positive")
    g, label = load_graph(args)
    stats = pb.compute_stats(g, args.classifier_threshold)
    sources = pick_sources(g, args)
    variants = parse_variants(args.variants)
    base = pb.parse_kernel_variant(args.baseline)
    if base is None:
        raise pb.ConfigError(f'unknown baseline "{args.baseline}"')
    if base not in variants:
        raise pb.ConfigError(f"baseline {args.baseline} is not among the selected variants")
    os.makedirs(args.out, exist_ok=True)
    try:
        results = open(os.path.join(args.out, "results.csv"), "w")
        traces = open(os.path.join(args.out, "traces.csv"), "w")
    except OSError:
        raise pb.InputError(f"cannot write into output directory {args.out}")
    results.write("graph,variant,worker_count,source,trials,median_ns,min_ns,max_ns,"
                  "total_edges_examined,avg_duplicate_pct,bu_levels,td_levels\n")
    pb.write_trace_csv_header(traces)
    print(f"graph: {label} ({g.vertex_count} vertices, {g.edge_count} directed edges, "
          f"{pb.to_string(stats.category)})")
    medians = {}
    for v in variants:
        cfg = make_config(args, v)
        for s in sources:
            # the reference's time_run semantics: warm-ups, trials, lower median;
            # every run is certified (module doc) instead of oracle-checked.
            samples, traces_run = [], []
            for i in range(args.warmups + args.trials):
                r = pb.run_bfs(g, s, cfg, stats)
                good, where = bfs_layering_ok(g, r.distances, s)
                if not good:
                    raise pb.CorrectnessError(f"distance certificate failed at vertex {where}")
                if i >= args.warmups:
                    samples.append(int(r.trace.device_ms * 1e6))
                    traces_run.append(r.trace)
            order = sorted(range(len(samples)), key=lambda i: samples[i])
            mid = order[(len(samples) - 1) // 2]
            t = traces_run[mid]
            medians[(v, s)] = samples[mid]
            dup = pb.average_duplicate_percentage(t) if t.records else 0.0
            results.write(f"{label},{pb.to_string(v)},1,{s},{args.trials},{samples[mid]},"
                          f"{min(samples)},{max(samples)},{t.total_edges_examined()},{dup:.4f},"
                          f"{t.level_count(pb.TraversalPhase.BottomUp)},"
                          f"{t.level_count(pb.TraversalPhase.TopDown)}\n")
            pb.write_trace_csv(traces, t, f"{label}/{pb.to_string(v)}/gpu/s{s}")
        print(f"timed {pb.to_string(v)} on the GPU over {len(sources)} sources")
    results.close()
    traces.close()
    print(f"\nspeedup vs {pb.to_string(base)} (geometric mean over sources)\n{'variant':18s}gpu")
    for v in variants:
        lg = sum(math.log(max(1, medians[(base, s)]) / max(1, medians[(v, s)])) for s in sources)
        print(f"{pb.to_string(v):18s}{math.exp(lg / len(sources)):.2f}")
    print(f"\nwrote {os.path.join(args.out, 'results.csv')} and "
          f"{os.path.join(args.out, 'traces.csv')}")
    return 0


def cmd_generate(args) -> int:
    """bfsbench.cpp:518-530."""
    if not args.gen:
        raise pb.ConfigError("generate needs --gen KIND:SCALE:EF:SEED")
    if not args.out:
        raise pb.ConfigError("generate needs --out FILE")
    g, label = load_graph(args)
    pb.save_binary_csr(g, args.out)
    print(f"wrote {args.out}: {label}, {g.vertex_count} vertices, {g.edge_count} directed edges")
    return 0


def build_parser():
    ap = argparse.ArgumentParser(prog="bfsbench-gpu",
                                 description="level-synchronous BFS on the B200")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def graph_opts(p):
        p.add_argument("--graph")
        p.add_argument("--gen")
        p.add_argument("--one-based", action="store_true")
        p.add_argument("--no-symmetrize", action="store_true")
        p.add_argument("--drop-self-loops", action="store_true")
        p.add_argument("--classifier-threshold", type=float,
                       default=pb.DEFAULT_DEGREE_THRESHOLD)

    def source_opts(p):
        p.add_argument("--sources", type=int, default=64)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--source-list")

    def matrix_opts(p, timing):
        p.add_argument("--variants", default="all")
        p.add_argument("--threads")
        p.add_argument("--hybrid-threshold", type=float, default=0.05)
        p.add_argument("--alpha", type=float, default=15.0)
        p.add_argument("--beta", type=float, default=18.0)
        p.add_argument("--flush-capacity", type=int, default=4096)
        if timing:
            p.add_argument("--baseline", default="conventional")
            p.add_argument("--trials", type=int, default=3)
            p.add_argument("--warmups", type=int, default=1)
            p.add_argument("--pin", action="store_true")

    p = sub.add_parser("stats")
    graph_opts(p)
    p = sub.add_parser("verify")
    graph_opts(p)
    source_opts(p)
    matrix_opts(p, False)
    p.add_argument("--inject-fault", action="store_true", help=argparse.SUPPRESS)
    p = sub.add_parser("run")
    graph_opts(p)
    source_opts(p)
    matrix_opts(p, True)
    p.add_argument("--out")
    p = sub.add_parser("generate")
    graph_opts(p)
    p.add_argument("--out")
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    handlers = {"stats": cmd_stats, "verify": cmd_verify, "run": cmd_run,
                "generate": cmd_generate}
    try:
        return handlers[args.cmd](args)
    except pb.CorrectnessError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    except (pb.FormatError, pb.InputError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except pb.Error as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
