"""Randomized parity run (GPU box): random graphs across the dense widths and the sparse
engine, each solved on the GPU and by the oracle (the C restatement of the reference, pinned
to it by tests/test_oracle.py).

Checked per graph:
* dense engine (n <= 1024): the MVC size (strategy gpu twice, hybrid filling the device,
  hybrid with 64 warps, StackOnly with 512 warps, two linked shards — no optimality
  certificate); the PVC(k = MVC - 1) answer and its node count (schedule independent, so it
  must equal the reference's exactly); the 1-warp seq order's node count; every returned cover
  verified; the mid layouts run wherever nodes keep 65-256 vertices alive;
* sparse engine (forced, shared- and global-memory node): the MVC size and a verified cover.

Usage: python tools/fuzz_parity.py SECONDS [seed] [large]   -> one JSON line per graph, then a
summary ("large": n > 1024 graphs on the sparse engine)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc  # noqa: E402
from oracle.oracle import CSR, Oracle  # noqa: E402  (the checker)
from paper_2204_10402_b200.shards import solve_sharded  # noqa: E402


def random_graph(rng):
    kind = rng.choice(["gnp", "phat_compl", "tree_plus"])
    n = int(rng.choice([20, 60, 100, 128, 129, 200, 256, 257, 300, 500, 513, 700, 1000]))
    if kind == "gnp":
        p = float(rng.uniform(1.5, 6.0)) / max(n - 1, 1)
        a = rng.random((n, n)) < p
    elif kind == "phat_compl":
        lo = float(rng.uniform(0.0, 0.6))
        hi = float(min(1.0, lo + rng.uniform(0.1, 0.5)))
        pw = lo + (hi - lo) * rng.random(n)
        a = ~(rng.random((n, n)) < (pw[:, None] + pw[None, :]) / 2)
    else:  # a random tree plus a few chords
        a = np.zeros((n, n), bool)
        for v in range(1, n):
            a[rng.integers(0, v), v] = True
        for _ in range(n // 10):
            u, v = rng.integers(0, n, 2)
            a[min(u, v), max(u, v)] = True
    iu = np.triu_indices(n, 1)
    keep = a[iu]
    return kind, n, vc.make_graph(n, list(zip(iu[0][keep].tolist(), iu[1][keep].tolist())))


def random_large_graph(rng):
    """n > 1024 (the sparse engine): trees with chords and sparse ER graphs the oracle solves."""
    n = int(rng.choice([1100, 1500, 2500, 4000, 6000]))
    if rng.random() < 0.5:
        edges = [(int(rng.integers(0, v)), v) for v in range(1, n)]
        edges += [tuple(int(x) for x in rng.integers(0, n, 2)) for _ in range(int(rng.integers(n // 6, n // 2)))]
        kind = "tree_plus"
    else:
        m = int(n * float(rng.uniform(1.0, 1.6)))
        edges = [tuple(int(x) for x in rng.integers(0, n, 2)) for _ in range(m)]
        kind = "gnp_sparse"
    return kind, n, vc.make_graph(n, edges)


def main_large(budget, rng):
    """Large-n randomized parity (sparse engine, shared- and global-memory node): MVC size,
    PVC(MVC - 1) answer, verified covers."""
    oracle = Oracle()
    t0 = time.time()
    checked = bad = skipped = 0
    while time.time() - t0 < budget:
        kind, n, g = random_large_graph(rng)
        off, nbr = g.csr()
        csr = CSR(n, g.num_edges, off, nbr)
        want = oracle.solve_seq(csr, node_budget=60_000)
        if want["status"] != "complete":
            skipped += 1
            continue
        rec = dict(kind=kind, n=n, m=g.num_edges, mvc=want["size"], seq_nodes=want["nodes"])
        ok = True
        for eng in ("auto", "sparse", "sparse-global"):
            r = vc.solve_mvc(g, strategy="gpu", engine=eng)
            ok &= r["size"] == want["size"] and r["engine"] == 2 and vc.verify_cover(g, r["cover"])
            if want["size"] >= 1:
                p = vc.solve_pvc(g, want["size"] - 1, strategy="gpu", engine=eng)
                ok &= not p["feasible"]
        rec["ok"] = bool(ok)
        checked += 1
        bad += not ok
        print(json.dumps(rec), flush=True)
    print(json.dumps(dict(summary=True, large=True, checked=checked, mismatches=bad, skipped=skipped,
                          seconds=round(time.time() - t0, 1))), flush=True)


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    if len(sys.argv) > 3 and sys.argv[3] == "large":
        return main_large(budget, rng)
    oracle = Oracle()
    t0 = time.time()
    checked = bad = skipped = 0
    while time.time() - t0 < budget:
        kind, n, g = random_graph(rng)
        off, nbr = g.csr()
        csr = CSR(n, g.num_edges, off, nbr)
        want = oracle.solve_seq(csr, node_budget=300_000)
        if want["status"] != "complete":
            skipped += 1
            continue
        rec = dict(kind=kind, n=n, m=g.num_edges, mvc=want["size"], seq_nodes=want["nodes"])
        ok = True
        # the parallel MVC search (no certificate: certify=False is the default), racing bound
        # updates across thousands of warps; plus a small-worker hybrid and StackOnly
        checks = {}
        for tag, kw in (("gpu", dict(strategy="gpu")), ("gpu2", dict(strategy="gpu")),
                        ("hybrid", dict(strategy="hybrid")),
                        ("hybrid64", dict(strategy="hybrid", device_workers=64)),
                        ("stackonly", dict(strategy="stackonly", workers=512, depth=10))):
            r = vc.solve_mvc(g, **kw)
            checks[tag] = r["size"] == want["size"] and vc.verify_cover(g, r["cover"]) \
                and r["certify_nodes"] == 0
            ok &= checks[tag]
        s = vc.solve_mvc(g, strategy="seq", timeout_s=60)
        ok &= s["size"] == want["size"] and sum(s["worker_nodes"]) == want["nodes"]
        if want["size"] >= 1:
            no = oracle.solve_seq(csr, pvc=True, k=want["size"] - 1) if want["size"] > 1 else None
            if no is not None:
                p = vc.solve_pvc(g, want["size"] - 1, strategy="gpu")
                ok &= (not p["feasible"]) and p["nodes_total"] == no["nodes"]
                rec["pvc_no_nodes"] = no["nodes"]
            y = vc.solve_pvc(g, want["size"], strategy="gpu")
            ok &= y["feasible"] and vc.verify_cover(g, y["cover"]) and y["size"] <= want["size"]
        sp = vc.solve_mvc(g, strategy="gpu", engine="sparse")
        ok &= sp["size"] == want["size"] and vc.verify_cover(g, sp["cover"])
        checks["sparse"] = sp["size"] == want["size"]
        sg = vc.solve_mvc(g, strategy="gpu", engine="sparse-global")
        checks["sparse_global"] = sg["size"] == want["size"] and vc.verify_cover(g, sg["cover"])
        ok &= checks["sparse_global"]
        if 16 < n <= 1024:  # two linked shards on the device (exchange helper, peer bound)
            sh = solve_sharded(g, "mvc", devices=(0, 0))
            checks["sharded"] = sh["size"] == want["size"] and vc.verify_cover(g, sh["cover"])
            ok &= checks["sharded"]
        rec["ok"] = bool(ok)
        if not ok:
            rec["checks"] = {k: bool(v) for k, v in checks.items()}
        checked += 1
        bad += not ok
        print(json.dumps(rec), flush=True)
    print(json.dumps(dict(summary=True, checked=checked, mismatches=bad, skipped=skipped,
                          seconds=round(time.time() - t0, 1))), flush=True)


if __name__ == "__main__":
    main()
