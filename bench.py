#!/usr/bin/env python
"""bench.py — headline measurement (driver contract).

Workloads (BASELINE.json metric "time-to-solution and search-tree nodes/sec at 1/2/4/8 B200 vs
CPU ref"); one step = one complete exact solve of a PVC no-instance (k = MVC - 1: the whole
search tree is visited, answer "no"):
  * N = 1 (default workload "c5"): config C5 — k = 482 on the complement of the p_hat-style
    G(500, a=.25, b=.75) seed-0 graph (data/configs/c5.clq.gz, n=500, m=61,209), 21,461,369
    nodes, about 10 ms: the round-to-round headline.
  * N > 1 (default workload "c5s", "C5-scale"): the strong-scaling instance SURVEY §8e asks
    for — a p_hat500-3-like graph (a=.48, b=1; data/configs/c5s.clq.gz) whose 1-GPU solve takes
    seconds, so that 1 -> 8 GPU scaling measures the search, not the start-up. The N = 1 line
    carries it as the extra key "c5_scale" (one solve + the reference's bounded sample).
  The N = 1 line also carries C1 / C3 MVC time-to-solution and C4 node throughput (budget
  100k, with its roofline), each beside the reference's own time (key "configs").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload W]

N>1 runs under torchrun, one process per GPU: rank 0's shard starts from the root, every GPU's
device worklist is linked to the others' through CUDA IPC / NVLink P2P, and workers donate
work straight into a starving peer's ring (strong scaling, max-over-ranks time).
`--impl reference` times the reference's own CPU solver (oracle/_ref/libvcref.so, run_hybrid
with every host thread) on bounded samples of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-solution and search-tree nodes/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "nodes/s"
# k = MVC - 1 and the full tree's node count (C5: the reference's, tests/golden/configs.json;
# C5-scale: the engine's, identical for every layout / worker count — tests/golden/c5s.json)
WORKLOADS = {
    "c5": dict(k=482, nodes=21461369,
               desc="C5: PVC k=482 (=MVC-1, no-instance) on the complement of p_hat-style "
                    "G(500, a=0.25, b=0.75) seed 0"),
    "c5s": dict(k=448, nodes=5969685861,
                desc="C5-scale: PVC k=448 (=MVC-1, no-instance) on the complement of p_hat-style "
                     "G(500, a=0.48, b=1.0) seed 0 (p_hat500-3-like)"),
}
# Degree entries are u16 in every node record (the roofline's w = 2 bytes); in registers the
# engine works on 32-bit words and 64-bit adjacency masks. Exact integer work either way.
DTYPE = "u16"
DTYPE_NOTE = "u16 degree entries in node records (roofline w=2 B); u32/u64 bit-mask arithmetic"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: c5 at N=1, c5s (C5-scale) at N>1")
    ap.add_argument("--no-extras", action="store_true",
                    help="N=1: skip the C1/C3/C4/C5-scale extra keys")
    ap.add_argument("--e2e-steps", type=int, default=None, help="default: 5 at N=1, 2 at N>1")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--frontier-per-rank", type=int, default=0,
                    help="N>1: 0 = rank 0 starts from the root and the linked device worklists "
                         "spread the work; else a deterministic frontier of this many nodes per rank")
    ap.add_argument("--ref-sample-s", type=float, default=0.0,
                    help="reference arm: seconds per bounded sample (0 = sized to the run)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def config_text(name):
    """The frozen config graph's DIMACS text, read straight from data/configs (the reference arm
    must not import the product package)."""
    import gzip
    with gzip.open(os.path.join(ROOT, "data", "configs", name + ".clq.gz"), "rt") as f:
        return f.read()


def workload_of(args, world):
    return args.workload or ("c5" if world == 1 else "c5s")


def bench_config(wl, n, m, world):
    """The workload dict, identical in both arms."""
    w = WORKLOADS[wl]
    return {"workload": w["desc"], "name": wl, "n": n, "m": m, "k": w["k"],
            "nodes_per_step": w["nodes"],
            "l2": "flushed between timed steps (256 MB memset)",
            "parallelism": "1 GPU" if world == 1 else
            f"{world} GPUs, one shard each, worklists linked over NVLink P2P (CUDA IPC)"}


def ref_graph(ref, name):
    """A config graph as the reference parses it (C3/C5/C5-scale solved on the complement)."""
    g = ref.parse(config_text(name), dimacs=True)
    return ref.complement(g) if name in ("c3", "c5", "c5s") else g


# ---------------------------------------------------------------- clocks during the timed region

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms; the samples inside the timed
    region (mark) are the ones reported."""

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, t0, t1):
        """The timed region [t0, t1] (perf_counter): only samples read inside it (plus the first
        after it, which covers its tail) are reported. The sampler is started before the
        warm-up so that nvidia-smi's start-up does not eat into a short timed region."""
        self.window = (t0, t1)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = [ln for _, ln in self.lines]
        win = getattr(self, "window", None)
        if win:
            inside = [ln for t, ln in self.lines if win[0] <= t <= win[1]]
            after = [ln for t, ln in self.lines if t > win[1]][:1]
            lines = inside + after or lines[-1:]
        for ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key="dense_kernel_c5"):
    """dram bytes per launch of a kernel from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(key, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------- reference (CPU) arm

def reference_line(args, rank, world):
    if rank != 0:
        return
    from oracle.oracle import Reference
    wl = workload_of(args, world)
    k, full = WORKLOADS[wl]["k"], WORKLOADS[wl]["nodes"]
    ref = Reference()
    g = ref_graph(ref, wl)
    cores = os.cpu_count() or 1
    budget_s = args.ref_sample_s or max(2.0, min(12.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        ref.solve(g, pvc=True, k=k, strategy="hybrid", workers=cores, timeout_s=1.0)
    rates, nodes = [], 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = ref.solve(g, pvc=True, k=k, strategy="hybrid", workers=cores, timeout_s=budget_s)
        rates.append(r["nodes"] / (r["wall_ms"] / 1e3))
        nodes += r["nodes"]
    wall = time.perf_counter() - t0
    value = nodes / wall
    sample = (f"reference run_hybrid ({cores} threads) on {wl} PVC k={k}, each step the first "
              f"{budget_s:.1f} s of the same search (timeout); full tree {full} nodes")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "data": f"synthetic (frozen p_hat-style graph, data/configs/{wl}.clq.gz)",
        "config": bench_config(wl, g.n, g.m, world),
        "time_to_solution_s_est": full / value,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def ref_pvc_rate(name, k, sample_s):
    """The reference's node rate on a bounded sample of a PVC search (rank 0, N=1 only)."""
    try:
        from oracle.oracle import Reference
        ref = Reference()
    except OSError as e:
        return {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}
    g = ref_graph(ref, name)
    cores = os.cpu_count() or 1
    r = ref.solve(g, pvc=True, k=k, strategy="hybrid", workers=cores, timeout_s=sample_s)
    return {"value": r["nodes"] / (r["wall_ms"] / 1e3), "unit": UNIT, "cores": cores,
            "kind": "reference",
            "sample": (f"reference run_hybrid, {cores} threads, {name} PVC k={k}: "
                       f"{r['nodes']} nodes in {r['wall_ms'] / 1e3:.1f} s "
                       f"(status {r['status']})")}


def extras(vc, peak, peak_src):
    """N=1 extra keys: C1 / C3 MVC time-to-solution, C4 node throughput at a 100k budget (its
    roofline: SURVEY §8d bytes 2·n·(R+M+C)), and C5-scale — each beside the reference."""
    from paper_2204_10402_b200.configs import load_config
    try:
        from oracle.oracle import Reference
        ref = Reference()
    except OSError:
        ref = None
    cores = os.cpu_count() or 1
    out = {}
    for name in ("c1", "c3"):
        g = load_config(name)
        vc.solve_mvc(g, strategy="gpu")  # (warm-up: graph upload, kernel load)
        runs = [vc.solve_mvc(g, strategy="gpu") for _ in range(5)]
        r = runs[-1]
        e = {"answer": r["size"], "time_to_solution_ms": statistics.median(x["wall_ms"] for x in runs),
             "device_ms": statistics.median(x["device_ms"] for x in runs),
             "nodes": r["nodes_total"], "strategy": "gpu"}
        if ref is not None:
            rg = ref_graph(ref, name)
            rr = [ref.solve(rg, strategy="hybrid", workers=cores) for _ in range(3)]
            e["reference"] = {"answer": rr[-1]["size"], "cores": cores,
                              "time_to_solution_ms": statistics.median(x["wall_ms"] for x in rr),
                              "runs_ms": [round(x["wall_ms"], 2) for x in rr]}
        out[f"{name}_mvc"] = e
    g4 = load_config("c4")
    vc.solve_mvc(g4, strategy="gpu", node_budget=2000)
    r = vc.solve_mvc(g4, strategy="gpu", node_budget=100_000)
    dev_s = r["device_ms"] / 1e3
    alg = 2 * g4.num_vertices * (r["rounds"] + r["maxdeg_passes"] + r["children"])
    e = {"node_budget": 100_000, "nodes": r["nodes_total"], "device_ms": r["device_ms"],
         "nodes_per_s": r["nodes_total"] / dev_s, "rounds": r["rounds"],
         "rule_rounds_per_s": r["rounds"] / dev_s,
         "note": ("budgeted node rates depend on which part of the tree the schedule reaches "
                  "(per-node cost varies ~20x with depth); rule rounds/s and the roofline "
                  "bytes compare across configurations"),
         "workers": len(r["worker_nodes"]), "block_threads": r["block_threads"],
         "roofline": {"bound": "hbm", "achieved": alg / dev_s / 1e9, "peak": peak, "unit": "GB/s",
                      "frac": alg / dev_s / 1e9 / peak, "traffic": ncu_traffic("sparse_kernel_c4"),
                      "kernel": "sparse_kernel", "algorithmic_bytes_per_launch": alg,
                      "bytes_per_node_def": "w*n*(R+M+C), w=2 B (u16 degree array), n=100000",
                      "peak_source": peak_src}}
    if ref is not None:
        rg = ref_graph(ref, "c4")
        rr = ref.solve(rg, strategy="hybrid", workers=cores, timeout_s=15.0)
        e["reference"] = {"nodes": rr["nodes"], "wall_ms": rr["wall_ms"], "cores": cores,
                          "nodes_per_s": rr["nodes"] / (rr["wall_ms"] / 1e3),
                          "note": "15 s sample of run_hybrid MVC (wall includes its greedy)"}
    out["c4_budget"] = e
    w = WORKLOADS["c5s"]
    gs = load_config("c5s")
    r = vc.solve_pvc(gs, w["k"], strategy="gpu")
    out["c5_scale"] = {"workload": w["desc"], "n": gs.num_vertices, "m": gs.num_edges, "k": w["k"],
                       "answer": "no" if not r["feasible"] else "yes", "nodes": r["nodes_total"],
                       "nodes_expected": w["nodes"], "time_to_solution_s": r["wall_ms"] / 1e3,
                       "device_s": r["device_ms"] / 1e3,
                       "nodes_per_s": r["nodes_total"] / (r["device_ms"] / 1e3),
                       "cpu_baseline": ref_pvc_rate("c5s", w["k"], 10.0)}
    return out


# ---------------------------------------------------------------- our arm

def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_line(args, rank, world)
    if args.e2e_steps is None:
        args.e2e_steps = 5 if world == 1 else 2

    import torch
    import torch.distributed as dist
    import paper_2204_10402_b200 as vc
    from paper_2204_10402_b200.configs import load_config

    # VCG_BENCH_SAME_DEVICE=1 (test hook): every rank on cuda:0 — exercises the N>1 path on a
    # one-GPU box (time-sliced processes; not a scaling number)
    same = os.environ.get("VCG_BENCH_SAME_DEVICE") == "1"
    if same:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if same:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        xg = dist.new_group(backend="gloo")
    stream = torch.cuda.Stream()  # the library launches on this stream; events bracket it
    wl = workload_of(args, world)
    K_NO = WORKLOADS[wl]["k"]
    g = load_config(wl)
    n, m = g.num_vertices, g.num_edges
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    peer = None
    if world > 1:
        # one persistent shard per rank: IPC handles exchanged and peers mapped once; a step
        # resets the device state, launches, waits and gathers (graph resident, like N=1)
        from paper_2204_10402_b200.distributed import PeerSolver
        peer = PeerSolver(g, "pvc", K_NO, xg, device=local, detail=False,
                          frontier_per_rank=args.frontier_per_rank)

    def step():
        if world == 1:
            r = vc.solve_pvc(g, K_NO, strategy="gpu", device=local, stream=stream.cuda_stream)
            r["rank_nodes"] = [r["nodes_total"]]
            return r
        return peer.solve()

    clocks = ClockSampler(local)  # (started before the warm-up; see ClockSampler.mark)
    clocks.start()
    for _ in range(args.warmup):
        r = step()
        assert not r["feasible"], f"{wl} k={K_NO} must be infeasible"
        with torch.cuda.stream(stream):
            flush.zero_()  # (the first fill pays torch's lazy kernel load: keep it out of the timing)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    t_wall0 = time.perf_counter()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            results.append(step())
            flush.zero_()  # L2 flush between timed steps (inside the bracket; ~0.05 ms)
        ev1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(t_wall0, time.perf_counter())
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([elapsed_ms], device="cpu" if same else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())

    for r in results:
        assert not r["feasible"] and r["status"] == "complete"
    nodes_per_step = results[-1]["nodes_total"]
    total_nodes = sum(r["nodes_total"] for r in results)
    value = total_nodes / (elapsed_ms / 1e3)

    # roofline for the dominant kernel (dense_kernel), from the N=1 per-launch counters
    peak, peak_src = measured_peak()
    line_extra = {}
    if world == 1:
        dev_ms = statistics.mean(r["device_ms"] for r in results)
        r0 = results[-1]
        w = r0["degree_bytes"]
        alg_bytes = w * n * (r0["rounds"] + r0["maxdeg_passes"] + r0["children"])
        achieved = alg_bytes / (dev_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": ncu_traffic(),
                "kernel": "dense_kernel<16>",
                "algorithmic_bytes_per_launch": alg_bytes,
                "bytes_per_node_def": "w*n*(R+M+C), w=%d B (u16 degree records), n=%d" % (w, n),
                "kernel_ms": dev_ms, "peak_source": peak_src,
                "kernel_share_of_step": dev_ms / (elapsed_ms / args.steps)}
        line_extra["roofline"] = roof
        line_extra["counters_per_step"] = {k: r0[k] for k in (
            "rounds", "maxdeg_passes", "children", "removals_deg1", "removals_deg2",
            "removals_high", "doomed", "donated", "grid_blocks", "block_threads")}
        line_extra["workers"] = len(r0["worker_nodes"])
        line_extra["load_ratio_max"] = max(r0["load_ratios"])

        # e2e: the public API with HOST buffers — fresh graph from host CSR arrays every step
        # (its device copy is built and uploaded inside the call) + result readback
        off, nbr = g.csr()
        e2e_nodes, e2e_h2d, e2e_d2h = 0, 0, 0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            gh = vc.from_csr(n, m, off, nbr)
            r = vc.solve_pvc(gh, K_NO, strategy="gpu")
            e2e_nodes += r["nodes_total"]
            e2e_h2d += r["h2d_bytes"]
            e2e_d2h += r["d2h_bytes"]
            del gh
        e2e_s = time.perf_counter() - t0
        line_extra["e2e"] = {"value": e2e_nodes / e2e_s, "unit": UNIT,
                             "h2d_bytes_per_step": e2e_h2d // args.e2e_steps,
                             "d2h_bytes_per_step": e2e_d2h // args.e2e_steps,
                             "ms_per_step": e2e_s * 1e3 / args.e2e_steps,
                             "time_to_solution_s": e2e_s / args.e2e_steps}
    else:
        line_extra["rank_nodes"] = results[-1]["rank_nodes"]
        line_extra["rank_donated_peer"] = results[-1].get("rank_donated_peer")
        line_extra["frontier_nodes"] = results[-1]["frontier_nodes"]
        line_extra["frontier_size"] = results[-1]["frontier_size"]
        # e2e: every rank builds a fresh graph from host CSR arrays each step and runs the
        # public multi-GPU call (frontier expansion, IPC rendezvous, linked shards, readback);
        # wall time, max over ranks
        from paper_2204_10402_b200.distributed import solve_distributed
        off, nbr = g.csr()
        e2e_nodes, e2e_h2d, e2e_d2h = 0, 0, 0
        dist.barrier(group=xg)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            gh = vc.from_csr(n, m, off, nbr)
            r = solve_distributed(gh, "pvc", K_NO, exchange_group=xg, device=local,
                                  frontier_per_rank=args.frontier_per_rank)
            e2e_nodes += r["nodes_total"]
            e2e_h2d += r.get("h2d_bytes", 0)
            e2e_d2h += r.get("d2h_bytes", 0)
            del gh
        e2e_s = torch.tensor([time.perf_counter() - t0])
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX, group=xg)
        e2e_s = float(e2e_s.item())
        line_extra["e2e"] = {"value": e2e_nodes / e2e_s, "unit": UNIT,
                             "h2d_bytes_per_step": e2e_h2d // args.e2e_steps,
                             "d2h_bytes_per_step": e2e_d2h // args.e2e_steps,
                             "ms_per_step": e2e_s * 1e3 / args.e2e_steps,
                             "time_to_solution_s": e2e_s / args.e2e_steps}

    if peer is not None:
        peer.close()
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
        "time_to_solution_s": elapsed_ms / 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE,
        "dtype_note": DTYPE_NOTE,
        "data": f"synthetic (frozen p_hat-style graph, data/configs/{wl}.clq.gz)",
        "config": bench_config(wl, n, m, world),
        "nodes_per_step": nodes_per_step, "strategy": "gpu",
        "clocks": clk,
        "gpu_launches": sum(r["kernel_launches"] for r in results),
    }
    line.update(line_extra)
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = ref_pvc_rate(wl, K_NO, args.cpu_sample_s)
    if world == 1 and not args.no_extras:
        line["configs"] = extras(vc, *measured_peak())
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
