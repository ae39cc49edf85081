"""GPU parity: the CUDA engine (through the C-ABI / public API) against the reference's golden
answers (tests/golden, generated from the reference itself) and the oracle restatement.

Bar (BASELINE.json north star): bit-exact integer results — the same MVC size, the same PVC
yes/no, every returned cover verified. Stronger, because the engine applies the reduction
rules in the reference's order: the 1-worker ("seq") traversal visits exactly the reference's
solve_seq node count, and PVC no-instance trees are schedule independent, so every worker
count reproduces the reference node count.
"""
import numpy as np
import pytest

import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config

pytestmark = pytest.mark.gpu


def graph_of(item):
    return vc.make_graph(item["n"], [tuple(e) for e in item["edges"]])


def check_cover(g, rep):
    assert len(rep["cover"]) == rep["size"]
    assert vc.verify_cover(g, rep["cover"]), "certificate is not a vertex cover"


def test_device_visible():
    assert vc.device_count() >= 1


def test_corpus_seq_order_is_the_reference_order(corpus):
    """solve_mvc_seq parity: size AND visited-node count equal the reference (535 graphs)."""
    bad = []
    for it in corpus:
        g = graph_of(it)
        r = vc.solve_mvc(g, strategy="seq")
        check_cover(g, r)
        if r["size"] != it["mvc"] or sum(r["worker_nodes"]) != it["seq_nodes"]:
            bad.append((it["name"], r["size"], it["mvc"], sum(r["worker_nodes"]), it["seq_nodes"]))
    assert not bad, bad[:10]


def test_corpus_pvc_triple_seq(corpus):
    bad = []
    for it in corpus:
        g = graph_of(it)
        for p in it["pvc"]:
            r = vc.solve_pvc(g, p["k"], strategy="seq")
            ok = r["feasible"] == p["feasible"] and sum(r["worker_nodes"]) == p["nodes"]
            if r["feasible"]:
                check_cover(g, r)
                ok = ok and r["size"] <= p["k"]
            if not ok:
                bad.append((it["name"], p, r["feasible"], sum(r["worker_nodes"])))
    assert not bad, bad[:10]


@pytest.mark.parametrize("workers,capacity,fraction", [
    (1, 1, 1.0), (2, 8, 0.25), (4, 64, 0.5), (8, 1, 0.5), (64, 8, 1.0), (None, 4096, 0.5)])
def test_corpus_hybrid_oracle_equivalence(corpus, workers, capacity, fraction):
    """acceptance_main.cpp:96-133 over GPU worker counts / capacities / thresholds."""
    bad = []
    for it in corpus[::3]:
        g = graph_of(it)
        # fixed small device worker counts run the reference's donation policy
        kw = dict(strategy="gpu") if workers is None else dict(strategy="hybrid",
                                                                device_workers=workers)
        r = vc.solve_mvc(g, capacity=capacity, threshold_fraction=fraction, **kw)
        check_cover(g, r)
        w = r["worklist"]
        if (r["size"] != it["mvc"] or r["status"] != "complete" or w["added"] != w["removed"]
                or w["max_size"] > capacity):
            bad.append((it["name"], r["size"], it["mvc"], w))
    assert not bad, bad[:10]


@pytest.mark.parametrize("workers", [1, 3, 8, None])
def test_corpus_pvc_triple_hybrid(corpus, workers):
    """acceptance_main.cpp:135-168; PVC-no node counts are schedule independent."""
    bad = []
    for it in corpus[1::4]:
        g = graph_of(it)
        for p in it["pvc"]:
            r = vc.solve_pvc(g, p["k"], strategy="gpu" if workers is None else "hybrid",
                             device_workers=workers, capacity=64)
            ok = r["feasible"] == p["feasible"]
            if r["feasible"]:
                check_cover(g, r)
                ok = ok and r["size"] <= p["k"]
            else:
                ok = ok and sum(r["worker_nodes"]) == p["nodes"]
            if not ok:
                bad.append((it["name"], p, r["feasible"], sum(r["worker_nodes"])))
    assert not bad, bad[:10]


def test_c1_seq_node_count(config_golden):
    g = load_config("c1")
    gold = config_golden["c1"]
    r = vc.solve_mvc(g, strategy="seq")
    assert r["size"] == gold["mvc"]
    assert sum(r["worker_nodes"]) == gold["seq_nodes"]
    check_cover(g, r)


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_config_mvc_and_pvc_pair_full_device(config_golden, name):
    g = load_config(name)
    gold = config_golden[name]
    r = vc.solve_mvc(g, strategy="gpu")
    assert r["size"] == gold["mvc"] and r["status"] == "complete"
    check_cover(g, r)
    no = vc.solve_pvc(g, gold["pvc_no_k"], strategy="gpu")
    assert not no["feasible"]
    assert no["nodes_total"] == gold["pvc_no_nodes"]  # schedule-independent tree size
    yes = vc.solve_pvc(g, gold["mvc"], strategy="gpu")
    assert yes["feasible"] and yes["size"] <= gold["mvc"]
    check_cover(g, yes)


def test_c5_pvc_no_instance_node_count(config_golden):
    gold = config_golden["c5"]
    if "pvc_no_nodes" not in gold:
        pytest.skip("C5 golden not generated")
    g = load_config("c5")
    r = vc.solve_pvc(g, gold["pvc_no_k"], strategy="gpu")
    assert not r["feasible"] and r["status"] == "complete"
    assert r["nodes_total"] == gold["pvc_no_nodes"]
    y = vc.solve_pvc(g, gold["pvc_yes_k"], strategy="gpu")
    assert y["feasible"] and y["size"] <= gold["pvc_yes_k"]
    check_cover(g, y)


def test_c5_engine_counters_are_schedule_independent():
    """On a PVC no-instance every tree node is visited once under the same bound k, so the
    rule work per node is fixed: rule rounds, branches (max-degree passes), stored children,
    removals per rule and prunes (dooms, dead children included) do not depend on the schedule.
    Guards the counters' bookkeeping (per-branch counters packed in shared memory, flushed per
    64 visits) against the values the round-1 kernels reported for the same tree."""
    g = load_config("c5")
    want = dict(rounds=14332419, maxdeg_passes=10730684, children=2403990,
                removals_deg1=1379027, removals_deg2=2015806, removals_high=6824878,
                doomed=9135007)
    for kw in (dict(), dict(block_warps=8)):
        r = vc.solve_pvc(g, 482, strategy="gpu", **kw)
        assert r["nodes_total"] == 21461369
        assert {k: r[k] for k in want} == want
        assert 0 < r["donated"] <= r["maxdeg_passes"]  # (at most one donation per branch)


def test_budget_and_timeout_status():
    g = load_config("c1")
    r = vc.solve_mvc(g, strategy="gpu", node_budget=1000)
    assert r["status"] == "budget"
    check_cover(g, r)  # best-so-far certificate stays valid (test_scheduler.cpp:175-189)
    r = vc.solve_mvc(g, strategy="hybrid", device_workers=1, timeout_s=0.0)
    assert r["status"] == "timeout"
    check_cover(g, r)


def test_report_shape():
    g = vc.make_graph(10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (0, 5), (1, 6), (2, 7),
                           (3, 8), (4, 9), (5, 7), (7, 9), (9, 6), (6, 8), (8, 5)])
    rep = vc.solve_mvc(g, strategy="hybrid", workers=3)
    for key in ("n", "m", "mode", "k", "strategy", "workers", "capacity", "threshold_fraction",
                "depth", "size", "feasible", "cover", "wall_ms", "status", "worker_nodes",
                "load_ratios", "phase_shares"):
        assert key in rep
    assert rep["n"] == 10 and rep["size"] == 6
    assert len(rep["worker_nodes"]) == 3  # test_smoke.py:64
    ratios = rep["load_ratios"]
    assert abs(sum(ratios) / len(ratios) - 1.0) < 1e-9
    assert sum(rep["phase_shares"].values()) <= 1.0 + 1e-9


def test_hybrid_reference_defaults_fill_the_device(config_golden):
    """solve_mvc(g) with the reference's defaults (hybrid, 4 workers) runs every resident warp
    of the device and folds them into the 4 report entries the reference's callers expect."""
    g = load_config("c1")
    r = vc.solve_mvc(g)
    assert r["size"] == config_golden["c1"]["mvc"] and r["workers"] == 4
    assert len(r["worker_nodes"]) == 4 and sum(r["worker_nodes"]) == r["nodes_total"]
    assert r["grid_blocks"] * r["block_threads"] // 32 >= 1000
    no = vc.solve_pvc(g, config_golden["c1"]["pvc_no_k"])
    assert not no["feasible"] and no["nodes_total"] == config_golden["c1"]["pvc_no_nodes"]
    assert len(no["worker_nodes"]) == 4
    few = vc.solve_mvc(g, device_workers=8)
    assert few["grid_blocks"] * few["block_threads"] // 32 >= 8
    assert len(few["worker_nodes"]) == 8


def test_instrumented_phase_shares():
    g = load_config("c3")
    rep = vc.solve_mvc(g, strategy="gpu", instrument=True)
    assert rep["size"] == 291
    shares = rep["phase_shares"]
    assert 0.0 < sum(v for k, v in shares.items() if k != "other") <= 1.0 + 1e-9


@pytest.mark.parametrize("name,k_key,world,target", [("c1", "pvc_no_k", 3, 64),
                                                      ("c3", "pvc_no_k", 2, 300),
                                                      ("c5", "pvc_no_k", 4, 4096)])
def test_frontier_shards_cover_the_tree_exactly(config_golden, name, k_key, world, target):
    """Multi-GPU partitioning, simulated in-process: the deterministic frontier plus every
    rank's share visit exactly the reference's PVC no-instance tree."""
    from paper_2204_10402_b200.distributed import expand_frontier
    gold = config_golden[name]
    g = load_config(name)
    k = gold[k_key]
    fr = expand_frontier(g, "pvc", k, target)
    fr2 = expand_frontier(g, "pvc", k, target)
    assert (fr["seeds"] == fr2["seeds"]).all() and fr["nodes"] == fr2["nodes"]  # deterministic
    assert not fr["found"]
    assert len(fr["seeds"]) >= target or len(fr["seeds"]) == 0  # 0: tree exhausted first
    total = fr["nodes"]
    for rank in range(world):
        share = fr["seeds"][rank::world]
        if len(share) == 0:  # nothing to search on this rank (solve_distributed skips it too)
            continue
        r = vc.solve_pvc(g, k, strategy="gpu", seeds=share)
        assert not r["feasible"]
        total += r["nodes_total"]
    assert total == gold["pvc_no_nodes"]


def test_frontier_mvc_shards_find_the_optimum(config_golden):
    from paper_2204_10402_b200.distributed import expand_frontier
    g = load_config("c1")
    fr = expand_frontier(g, "mvc", 0, 200)
    best = fr["best"]
    for rank in range(2):
        r = vc.solve_mvc(g, strategy="gpu", seeds=fr["seeds"][rank::2], initial_best=fr["best"])
        if r["cover_from_search"]:
            check_cover(g, r)
            best = min(best, r["size"])
    assert best == config_golden["c1"]["mvc"]


def test_mailbox_cancel_and_external_bound():
    from paper_2204_10402_b200.distributed import Mailbox
    g = load_config("c5")
    mb = Mailbox()
    mb.words[1] = 1  # host cancel request before launch: the search stops early
    r = vc.solve_pvc(g, 482, strategy="gpu", mailbox=mb.address)
    assert r["nodes_total"] < 21461369
    mb.close()


# ---- sparse engine (one CTA per node, block-parallel rule rounds) -------------------------

@pytest.mark.parametrize("workers", [1, 3, None])
def test_sparse_engine_corpus_exact(corpus, workers):
    """The block-parallel rules are sound: MVC sizes equal the brute-force optimum on all 535
    corpus graphs (forced onto the sparse engine)."""
    bad = []
    for it in corpus:
        g = graph_of(it)
        r = vc.solve_mvc(g, strategy="gpu" if workers is None else "hybrid",
                         device_workers=workers, engine="sparse")
        check_cover(g, r)
        if r["size"] != it["mvc"] or r["status"] != "complete" or r["engine"] != 2:
            bad.append((it["name"], r["size"], it["mvc"]))
    assert not bad, bad[:10]


def test_sparse_engine_pvc_triple(corpus):
    bad = []
    for it in corpus[::2]:
        g = graph_of(it)
        for p in it["pvc"]:
            r = vc.solve_pvc(g, p["k"], strategy="gpu", engine="sparse")
            ok = r["feasible"] == p["feasible"]
            if r["feasible"]:
                check_cover(g, r)
                ok = ok and r["size"] <= p["k"]
            if not ok:
                bad.append((it["name"], p, r["feasible"]))
    assert not bad, bad[:10]


def _random_tree(n, seed):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(0, v)), v) for v in range(1, n)]


@pytest.mark.parametrize("n,seed", [(3000, 1), (20000, 2)])
def test_sparse_engine_large_trees_equal_oracle(oracle, n, seed):
    """n > 1024 (auto-selects the sparse engine); trees are solved exactly by the rules."""
    from oracle.oracle import CSR
    edges = _random_tree(n, seed)
    g = vc.make_graph(n, edges)
    r = vc.solve_mvc(g, strategy="gpu")
    assert r["engine"] == 2
    off, nbr = g.csr()
    want = oracle.solve_seq(CSR(n, g.num_edges, off, nbr))
    assert r["size"] == want["size"]
    check_cover(g, r)


def test_sparse_engine_sparse_random_graph(oracle):
    from oracle.oracle import CSR
    rng = np.random.default_rng(5)
    n = 1500
    m = int(1.1 * n)
    e = rng.integers(0, n, size=(m, 2))
    g = vc.make_graph(n, [tuple(map(int, x)) for x in e])
    off, nbr = g.csr()
    want = oracle.solve_seq(CSR(n, g.num_edges, off, nbr), node_budget=2_000_000)
    assert want["status"] == "complete"
    r = vc.solve_mvc(g, strategy="gpu")
    assert r["size"] == want["size"] and r["status"] == "complete"
    check_cover(g, r)
    no = vc.solve_pvc(g, want["size"] - 1, strategy="gpu")
    assert not no["feasible"]


def test_c4_budgeted_run(config_golden):
    g = load_config("c4")
    r = vc.solve_mvc(g, strategy="gpu", node_budget=3000)
    assert r["engine"] == 2 and r["status"] == "budget"
    assert r["size"] <= config_golden["c4"]["greedy"]
    check_cover(g, r)


# ---- StackOnly (scheduler.cpp:214-297) ----------------------------------------------------

@pytest.mark.parametrize("engine", ["dense", "sparse"])
@pytest.mark.parametrize("workers,depth", [(1, 1), (4, 4), (8, 8)])
def test_stackonly_corpus_exact(corpus, engine, workers, depth):
    """acceptance_main.cpp:96-133 with run_stackonly: sizes equal the oracle's."""
    bad = []
    for it in corpus[::4]:
        g = graph_of(it)
        r = vc.solve_mvc(g, strategy="stackonly", workers=workers, depth=depth, engine=engine)
        check_cover(g, r)
        if r["size"] != it["mvc"] or r["status"] != "complete" or len(r["worker_nodes"]) != workers:
            bad.append((it["name"], r["size"], it["mvc"]))
        if r["worklist"]["added"] != 0:  # StackOnly reports empty worklist stats
            bad.append((it["name"], "worklist"))
    assert not bad, bad[:10]


def test_stackonly_pvc_and_configs(config_golden):
    g = load_config("c1")
    r = vc.solve_mvc(g, strategy="stackonly", workers=64, depth=12)
    assert r["size"] == config_golden["c1"]["mvc"]
    check_cover(g, r)
    assert not vc.solve_pvc(g, 84, strategy="stackonly", workers=64, depth=10)["feasible"]
    y = vc.solve_pvc(g, 85, strategy="stackonly", workers=64, depth=10)
    assert y["feasible"]
    check_cover(g, y)


def test_stackonly_load_imbalance_vs_hybrid(config_golden):
    """The paper's Fig. 5 direction on C3: hybrid balances load better than StackOnly."""
    g = load_config("c3")
    so = vc.solve_mvc(g, strategy="stackonly", workers=256, depth=10)
    hy = vc.solve_mvc(g, strategy="hybrid", workers=256)
    assert so["size"] == hy["size"] == config_golden["c3"]["mvc"]
    assert max(hy["load_ratios"]) < max(so["load_ratios"])


# ---- multi-shard solves: device worklists linked through peer memory (shards.py) ----------

@pytest.mark.parametrize("skew", [False, True])
@pytest.mark.parametrize("name", ["c1", "c3"])
def test_sharded_pvc_pair_exact(config_golden, name, skew):
    """Two shards on one device: the no-instance tree is visited exactly once across shards and
    the frontier (node count = the reference's), the yes-instance yields a verified cover."""
    from paper_2204_10402_b200.shards import solve_sharded
    g = load_config(name)
    gold = config_golden[name]
    fps = 64 if skew else 0  # skew: a frontier dealt to shard 0; else the root on shard 0
    no = solve_sharded(g, "pvc", gold["pvc_no_k"], devices=(0, 0), skew=skew,
                       frontier_per_shard=fps, timeout_s=60)
    assert no["status"] == "complete" and not no["feasible"]
    assert no["nodes_total"] == gold["pvc_no_nodes"], (no["nodes_total"], no["rank_nodes"])
    if name == "c1":  # shard 1 starts empty: all it visits was donated to it (C3 is too small)
        assert no["rank_nodes"][1] > 0, no["rank_nodes"]
    yes = solve_sharded(g, "pvc", gold["mvc"], devices=(0, 0), skew=skew,
                        frontier_per_shard=fps, timeout_s=60)
    assert yes["feasible"] and len(yes["cover"]) <= gold["mvc"]
    assert vc.verify_cover(g, yes["cover"])


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_sharded_mvc_optimum(config_golden, name):
    from paper_2204_10402_b200.shards import solve_sharded
    g = load_config(name)
    r = solve_sharded(g, "mvc", devices=(0, 0, 0), skew=True, timeout_s=60)
    assert r["status"] == "complete" and r["size"] == config_golden[name]["mvc"]
    assert vc.verify_cover(g, r["cover"])


def test_sharded_c5_no_instance(config_golden):
    from paper_2204_10402_b200.shards import solve_sharded
    gold = config_golden["c5"]
    g = load_config("c5")
    for fps, devices in ((256, (0, 0)), (0, (0, 0)), (0, (0, 0, 0, 0))):
        r = solve_sharded(g, "pvc", gold["pvc_no_k"], devices=devices, frontier_per_shard=fps,
                          timeout_s=120)
        assert r["status"] == "complete" and not r["feasible"]
        assert r["nodes_total"] == gold["pvc_no_nodes"]
        assert min(r["rank_nodes"]) > 0 and sum(r["rank_donated_peer"]) > 0, r["rank_nodes"]


def test_sharded_timeout_cancels_every_shard():
    from paper_2204_10402_b200.shards import solve_sharded
    g = load_config("c5")
    r = solve_sharded(g, "pvc", 482, devices=(0, 0), timeout_s=0.002)
    assert r["status"] == "timeout"


@pytest.mark.parametrize("name", ["c1", "c3", "c5"])
def test_compact_and_wide_layouts_visit_the_same_tree(config_golden, name):
    """The compact renumbering keeps the id order, so the node counts of the all-wide layout
    (engine="dense-wide") and the default one equal the reference's on PVC no-instances, and the
    1-warp seq order is the reference's node for node in both."""
    g = load_config(name)
    gold = config_golden[name]
    for engine in ("dense", "dense-wide"):
        r = vc.solve_pvc(g, gold["pvc_no_k"], strategy="gpu", engine=engine)
        assert not r["feasible"] and r["nodes_total"] == gold["pvc_no_nodes"], (engine, r["nodes_total"])
    if name != "c5":
        for engine in ("dense", "dense-wide"):
            s = vc.solve_mvc(g, strategy="seq", engine=engine)
            assert s["size"] == gold["mvc"] and sum(s["worker_nodes"]) == gold["seq_nodes"], engine


def _phat_complement(n, a, b, seed):
    """Complement of a p_hat-style random graph (vertex weights U[a, b], edge iff U < mean)."""
    rng = np.random.default_rng(seed)
    pw = a + (b - a) * rng.random(n)
    adj = rng.random((n, n)) < (pw[:, None] + pw[None, :]) / 2
    iu = np.triu_indices(n, 1)
    keep = ~adj[iu]
    return vc.make_graph(n, list(zip(iu[0][keep].tolist(), iu[1][keep].tolist())))


@pytest.mark.parametrize("n,a,b", [(200, 0.25, 0.75), (600, 0.05, 0.3), (900, 0.0, 0.3)])
def test_dense_widths_8_and_32_against_the_oracle(oracle, n, a, b):
    """The W = 8 (n <= 256) and W = 32 (n <= 1024) kernels: MVC size, the PVC no-instance node
    count and the 1-warp seq order equal the oracle's (the reference restatement)."""
    from oracle.oracle import CSR
    g = _phat_complement(n, a, b, 1)
    off, nbr = g.csr()
    csr = CSR(n, g.num_edges, off, nbr)
    want = oracle.solve_seq(csr)
    no = oracle.solve_seq(csr, pvc=True, k=want["size"] - 1)
    assert not no["feasible"]
    r = vc.solve_mvc(g, strategy="gpu")
    assert r["size"] == want["size"] and r["engine"] == 1
    check_cover(g, r)
    for engine in ("dense", "dense-wide"):
        p = vc.solve_pvc(g, want["size"] - 1, strategy="gpu", engine=engine)
        assert not p["feasible"] and p["nodes_total"] == no["nodes"], (engine, p["nodes_total"], no["nodes"])
    s = vc.solve_mvc(g, strategy="seq")
    assert s["size"] == want["size"] and sum(s["worker_nodes"]) == want["nodes"]


@pytest.mark.parametrize("capacity", [8, 64, 4096])
def test_yes_instance_cancel_with_small_rings(config_golden, capacity):
    """A PVC yes-instance cancels every worker while donations are in flight; with a small
    ring the tickets wrap quickly, so donors must not wait for slots whose previous-lap
    readers already left (regression: that wait used to hang the kernel)."""
    gold = config_golden["c5"]
    g = load_config("c5")
    for _ in range(3):
        y = vc.solve_pvc(g, gold["pvc_yes_k"], strategy="gpu", capacity=capacity)
        assert y["feasible"] and y["size"] <= gold["pvc_yes_k"]
        check_cover(g, y)
    from paper_2204_10402_b200.shards import solve_sharded
    r = solve_sharded(g, "pvc", gold["pvc_yes_k"], devices=(0, 0), capacity=capacity)
    assert r["feasible"] and vc.verify_cover(g, r["cover"])


def test_persistent_shards_solve_repeatedly(config_golden):
    """ShardedSolver: shards linked once, reset between solves — every solve visits the
    reference's tree exactly (the reset leaves no stale queue, counter or activity state)."""
    from paper_2204_10402_b200.shards import ShardedSolver
    gold = config_golden["c5"]
    g = load_config("c5")
    ss = ShardedSolver(g, "pvc", gold["pvc_no_k"], devices=(0, 0))
    try:
        for _ in range(4):
            r = ss.solve()
            assert r["status"] == "complete" and not r["feasible"]
            assert r["nodes_total"] == gold["pvc_no_nodes"], r["rank_nodes"]
    finally:
        ss.close()
    c1 = load_config("c1")
    ss = ShardedSolver(c1, "mvc", devices=(0, 0, 0))
    try:
        for _ in range(3):
            r = ss.solve()
            assert r["size"] == config_golden["c1"]["mvc"] and vc.verify_cover(c1, r["cover"])
    finally:
        ss.close()


def _fuzz_graph(name):
    import os
    path = os.path.join(os.path.dirname(__file__), "data", name)
    return vc.parse_edge_list(open(path).read())


@pytest.mark.parametrize("name", ["fuzz_200_12063.el", "fuzz_128_4403.el"])
def test_parallel_mvc_is_exact_without_certificate(oracle, name):
    """Regression (tools/fuzz_parity.py, round 1): on these graphs the parallel MVC search once
    stopped one above the optimum — the edge-count prune used a bound lowered by a poll AFTER
    the node was reduced under the older one. With the edge-count prune under the bound the
    reduction reached fixpoint under (settle(), dense_kernels.cuh) every strategy, engine and the
    multi-shard path are exact on
    their own; the racing schedule differs run to run, so each runs several times."""
    from oracle.oracle import CSR
    from paper_2204_10402_b200.shards import solve_sharded
    g = _fuzz_graph(name)
    off, nbr = g.csr()
    want = oracle.solve_seq(CSR(g.num_vertices, g.num_edges, off, nbr))
    for kw in (dict(strategy="gpu"), dict(strategy="hybrid", workers=3552),
               dict(strategy="hybrid", workers=64), dict(strategy="hybrid", device_workers=64),
               dict(strategy="gpu", engine="dense-wide"), dict(strategy="gpu", engine="sparse"),
               dict(strategy="stackonly", workers=1024, depth=12)):
        for _ in range(8):
            r = vc.solve_mvc(g, **kw)
            assert r["size"] == want["size"], (kw, r["size"], want["size"])
            assert r["certify_nodes"] == 0
            check_cover(g, r)
    for _ in range(4):
        r = solve_sharded(g, "mvc", devices=(0, 0))
        assert r["size"] == want["size"], ("sharded", r["size"], want["size"])
        assert vc.verify_cover(g, r["cover"])


def test_certificate_debug_option(oracle):
    """certify=True (VCG_DEBUG_CERTIFY) re-proves the optimum by PVC(size - 1): same answer, its
    nodes and time reported apart from the search's."""
    from oracle.oracle import CSR
    g = _fuzz_graph("fuzz_128_4403.el")
    off, nbr = g.csr()
    want = oracle.solve_seq(CSR(g.num_vertices, g.num_edges, off, nbr))
    r = vc.solve_mvc(g, strategy="gpu", certify=True)
    assert r["size"] == want["size"] and r["certify_nodes"] > 0 and r["certify_ms"] > 0
    plain = vc.solve_mvc(g, strategy="gpu")
    assert plain["certify_nodes"] == 0
    # the certificate stays within the caller's node budget
    r = vc.solve_mvc(g, strategy="gpu", certify=True, node_budget=plain["nodes_total"] + 10)
    assert r["status"] in ("complete", "budget")


def test_engine_verifies_every_returned_cover():
    """verify_cover (bounds.cpp:32-45) runs inside vcg_solve: a corrupted cover (debug hook
    drops one vertex of an optimal cover) is reported as an engine fault, never returned."""
    from paper_2204_10402_b200 import _native as n
    g = load_config("c1")
    with pytest.raises(RuntimeError, match="invalid cover"):
        vc.solve_mvc(g, strategy="gpu", debug_flags=n.VCG_DEBUG_CORRUPT_COVER)
    with pytest.raises(RuntimeError, match="invalid cover"):
        vc.solve_pvc(g, 85, strategy="gpu", debug_flags=n.VCG_DEBUG_CORRUPT_COVER)
    # an infeasible PVC returns no cover: nothing to verify, no error
    assert not vc.solve_pvc(g, 84, strategy="gpu",
                            debug_flags=n.VCG_DEBUG_CORRUPT_COVER)["feasible"]


def test_c2_pvc_yes_at_k241(config_golden):
    """C2 (ER(400, d6)) PVC k = 241 = MVC: a yes-instance with a verified certificate of size
    <= k (the "no" side, k = 240, is a 466 G-node search: profiles/r1_c2_k240.json and the
    cross-check run in profiles/)."""
    g = load_config("c2")
    r = vc.solve_pvc(g, 241, strategy="gpu", timeout_s=120)
    assert r["status"] == "complete" and r["feasible"]
    assert r["size"] <= 241
    check_cover(g, r)


# ---- mid layout (per-warp frame renumbering, <= 128 / <= 256 alive) ------------------------

@pytest.mark.parametrize("engine", ["dense-mid4", "dense-mid8", "dense-nomid"])
def test_mid_layouts_visit_the_reference_tree(config_golden, engine):
    """The frame renumbering keeps the id order: PVC no-instance node counts equal the
    reference's, and the 1-warp seq order is the reference's node for node (C3, n = 300: the
    mid layouts act on nodes with 65-256 alive vertices)."""
    for name in ("c3", "c5"):
        g = load_config(name)
        gold = config_golden[name]
        r = vc.solve_pvc(g, gold["pvc_no_k"], strategy="gpu", engine=engine)
        assert not r["feasible"] and r["nodes_total"] == gold["pvc_no_nodes"], (name, r["nodes_total"])
    g = load_config("c3")
    s = vc.solve_mvc(g, strategy="seq", engine=engine)
    assert s["size"] == config_golden["c3"]["mvc"]
    assert sum(s["worker_nodes"]) == config_golden["c3"]["seq_nodes"]


@pytest.mark.parametrize("n,deg,seed", [(300, 3.0, 3), (400, 3.0, 4), (500, 2.5, 5)])
def test_mid_layouts_on_sparse_graphs_against_the_oracle(oracle, n, deg, seed):
    """Sparse W = 16 graphs (nodes keep 100-300 vertices alive: the <= 256 frame, rebuilt on
    donated records): MVC, the PVC no-instance node count and the seq order equal the oracle's."""
    from oracle.oracle import CSR
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    keep = rng.random(len(iu[0])) < deg / (n - 1)
    g = vc.make_graph(n, list(zip(iu[0][keep].tolist(), iu[1][keep].tolist())))
    off, nbr = g.csr()
    csr = CSR(n, g.num_edges, off, nbr)
    want = oracle.solve_seq(csr, node_budget=3_000_000)
    if want["status"] != "complete":
        pytest.skip("oracle budget")
    no = oracle.solve_seq(csr, pvc=True, k=want["size"] - 1, node_budget=6_000_000)
    for engine in ("auto", "dense-mid8", "dense-mid4"):
        r = vc.solve_mvc(g, strategy="gpu", engine=engine)
        assert r["size"] == want["size"], engine
        check_cover(g, r)
        if no["status"] == "complete":
            p = vc.solve_pvc(g, want["size"] - 1, strategy="gpu", engine=engine)
            assert not p["feasible"] and p["nodes_total"] == no["nodes"], (engine, p["nodes_total"])
    s = vc.solve_mvc(g, strategy="seq", engine="dense-mid8")
    assert s["size"] == want["size"] and sum(s["worker_nodes"]) == want["nodes"]


# ---- large n: the global-memory node variant, stack overflow, sparse frontier --------------

def _ba_edges(n, m, seed):
    """Barabasi-Albert preferential attachment (each new vertex picks m distinct targets,
    proportionally to degree, by sampling the endpoint list)."""
    rng = np.random.default_rng(seed)
    ends = list(range(m))
    edges = []
    for v in range(m, n):
        chosen = set()
        while len(chosen) < m:
            chosen.add(ends[int(rng.integers(len(ends)))] if len(ends) > m else int(rng.integers(v)))
        for u in chosen:
            edges.append((u, v))
            ends.extend((u, v))
    return edges


def test_sparse_global_variant_corpus_exact(corpus):
    """engine="sparse-global" (degree array in global memory): exact on the corpus."""
    bad = []
    for it in corpus[::3]:
        g = graph_of(it)
        r = vc.solve_mvc(g, strategy="gpu", engine="sparse-global")
        check_cover(g, r)
        if r["size"] != it["mvc"] or r["status"] != "complete" or r["engine"] != 2:
            bad.append((it["name"], r["size"], it["mvc"]))
    assert not bad, bad[:10]


def test_large_n_ba300k_budgeted_run():
    """n = 300k is beyond the shared-memory degree array: the global-memory variant runs it."""
    n = 300_000
    g = vc.make_graph(n, _ba_edges(n, 3, 7))
    r = vc.solve_mvc(g, strategy="gpu", node_budget=3000)
    assert r["engine"] == 2 and r["status"] == "budget" and r["nodes_total"] >= 3000
    assert r["size"] <= r["greedy_size"]
    check_cover(g, r)


def test_sparse_stack_overflow_hands_nodes_to_the_worklist(corpus, config_golden):
    """Local stacks capped at 3 nodes (debug): full stacks hand their oldest node to the
    worklist instead of failing, and the answers stay exact."""
    bad = []
    for it in corpus[::4]:
        g = graph_of(it)
        r = vc.solve_mvc(g, strategy="gpu", engine="sparse", debug_flags=vc._n.VCG_DEBUG_SMALL_STACK)
        if r["size"] != it["mvc"] or r["status"] != "complete":
            bad.append((it["name"], r["size"], it["mvc"]))
    assert not bad, bad[:10]
    g = load_config("c3")
    r = vc.solve_mvc(g, strategy="gpu", engine="sparse", debug_flags=vc._n.VCG_DEBUG_SMALL_STACK)
    assert r["size"] == config_golden["c3"]["mvc"]
    check_cover(g, r)


def test_sparse_frontier_expansion_partitions_exactly(oracle):
    """vcg_expand_frontier on the sparse engine (n > 1024): the frontier shares, solved
    separately, give the direct solve's optimum (a two-rank partition in one process)."""
    from oracle.oracle import CSR
    from paper_2204_10402_b200.distributed import expand_frontier
    rng = np.random.default_rng(11)
    n = 1500
    edges = _random_tree(n, 11) + [tuple(map(int, rng.integers(0, n, 2))) for _ in range(160)]
    g = vc.make_graph(n, edges)
    off, nbr = g.csr()
    want = oracle.solve_seq(CSR(n, g.num_edges, off, nbr), node_budget=5_000_000)
    assert want["status"] == "complete"
    fr = expand_frontier(g, "mvc", 0, 16)
    assert fr["nodes"] >= 1 and fr["levels"] >= 1
    best = fr["best"]
    sizes = [len(fr["cover"])]
    for rank in range(2):
        share = fr["seeds"][rank::2]
        if len(share):
            r = vc.solve_mvc(g, strategy="gpu", seeds=share, initial_best=best)
            check_cover(g, r)
            if r["cover_from_search"]:
                sizes.append(r["size"])
    assert min(sizes) == want["size"]
    # C4 (n = 100k): the expansion itself on the large config
    c4 = load_config("c4")
    f4 = expand_frontier(c4, "mvc", 0, 32)
    assert len(f4["seeds"]) >= 32 or f4["found"]
    assert f4["seeds"].shape[1] == c4.num_vertices + 2


def test_c5_scale_no_instance():
    """C5-scale (the strong-scaling config): PVC(448) visits the cross-checked tree size (see
    tests/golden/c5s.json) and PVC(449) is a yes with a verified cover."""
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c5s.json")))
    g = load_config("c5s")
    assert g.num_vertices == gold["n"] and g.num_edges == gold["m"]
    r = vc.solve_pvc(g, gold["pvc_no_k"], strategy="gpu")
    assert not r["feasible"] and r["status"] == "complete"
    assert r["nodes_total"] == gold["pvc_no_nodes"]
    y = vc.solve_pvc(g, gold["pvc_yes_k"], strategy="gpu")
    assert y["feasible"] and y["size"] <= gold["pvc_yes_k"]
    check_cover(g, y)


def test_sparse_engine_repeated_solves_small_ctas(oracle):
    """Regression (round 2): with 128-thread CTAs, 8 per SM, a fast thread popping the next node
    rewrote the shared node state while a slower warp was still deciding on the current one,
    desynchronising the CTA's barriers (1 solve in ~40 crashed). Many solves of the graph that
    exposed it, on both node variants."""
    from oracle.oracle import CSR
    g = _fuzz_graph("fuzz_gnp_256_549.el")
    off, nbr = g.csr()
    want = oracle.solve_seq(CSR(g.num_vertices, g.num_edges, off, nbr))
    for engine in ("sparse", "sparse-global"):
        for _ in range(60):
            r = vc.solve_mvc(g, strategy="gpu", engine=engine)
            assert r["size"] == want["size"] and r["block_threads"] == 128, (engine, r["size"])
            check_cover(g, r)
