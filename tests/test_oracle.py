"""The oracle (oracle/oracle.c, a C restatement of the reference) pinned against the reference's
own known-answer tests and against golden vectors generated from the reference itself
(tests/golden/*.json via tests/golden/make_golden.py, oracle/_ref/libvcref.so).

CPU only. When oracle/_ref/libvcref.so is present (built here from /root/reference), the oracle
is additionally checked against the reference call for call.
"""
import numpy as np
import pytest

from oracle.oracle import CSR, REMOVED


def mk(oracle, n, edges):
    return oracle.make_graph(n, edges)


def path(oracle, n):
    return mk(oracle, n, [(v, v + 1) for v in range(n - 1)])


def cycle(oracle, n):
    return mk(oracle, n, [(v, v + 1) for v in range(n - 1)] + [(n - 1, 0)])


def star(oracle, leaves):
    return mk(oracle, leaves + 1, [(0, v) for v in range(1, leaves + 1)])


def complete(oracle, n):
    return mk(oracle, n, [(u, v) for u in range(n) for v in range(u + 1, n)])


def root(csr):
    return csr.degrees().copy(), 0, csr.m


def node_from_removed(csr, removed):
    """A consistent search node (consistent_with, search_node.cpp:57-83) with `removed` in S."""
    alive = np.ones(csr.n, bool)
    alive[list(removed)] = False
    deg = np.full(csr.n, REMOVED, np.uint32)
    edges = 0
    for v in range(csr.n):
        if not alive[v]:
            continue
        nb = csr.neighbors[csr.offsets[v]:csr.offsets[v + 1]]
        deg[v] = int(alive[nb].sum())
        edges += int((alive[nb] & (nb > v)).sum())
    return deg, int((~alive).sum()), edges


def cover_of(deg):
    return [int(v) for v in np.nonzero(deg == REMOVED)[0]]


# ---- known-answer tests of the reference (proj/tests/test_reductions.cpp) -------------------

def test_kat_degree_one_p2_smaller_endpoint_acts(oracle):  # test_reductions.cpp:24-31
    g = path(oracle, 2)
    d, cc, e, ch = oracle.reduce(g, *root(g), which=2)
    assert ch and d[1] == REMOVED and d[0] == 0 and cc == 1


def test_kat_degree_one_p3_takes_middle(oracle):  # :33-39
    g = path(oracle, 3)
    d, cc, e, ch = oracle.reduce(g, *root(g), which=2)
    assert ch and cover_of(d) == [1] and e == 0


def test_kat_degree_one_p4(oracle):  # :41-49
    g = path(oracle, 4)
    d, cc, e = root(g)
    while True:
        d, cc, e, ch = oracle.reduce(g, d, cc, e, which=2)
        if not ch:
            break
    assert cc == 2 and e == 0 and cc == oracle.brute_force(g)[0]


def test_kat_triangle_from_smallest_vertex(oracle):  # :51-58
    g = complete(oracle, 3)
    d, cc, e, ch = oracle.reduce(g, *root(g), which=3)
    assert ch and cover_of(d) == [1, 2] and cc == 2 and e == 0


def test_kat_triangle_with_pendant(oracle):  # :60-78
    g1 = mk(oracle, 4, [(0, 1), (0, 2), (1, 2), (2, 3)])
    d, cc, e, ch = oracle.reduce(g1, *root(g1), which=3)
    assert ch and cover_of(d) == [1, 2] and e == 0 and cc == oracle.brute_force(g1)[0]
    g2 = mk(oracle, 4, [(0, 1), (0, 2), (1, 2), (0, 3)])
    d, cc, e, ch = oracle.reduce(g2, *root(g2), which=3)
    assert ch and cover_of(d) == [0, 2] and e == 0 and cc == oracle.brute_force(g2)[0]


def test_kat_c4_triangle_rule_noop(oracle):  # :80-85
    g = cycle(oracle, 4)
    d, cc, e, ch = oracle.reduce(g, *root(g), which=3)
    assert not ch and cc == 0


def test_kat_high_degree(oracle):  # :87-103 and acceptance_main.cpp:367-378
    g = star(oracle, 5)
    d, cc, e, ch = oracle.reduce(g, *root(g), pvc=False, best_or_k=2, which=4)
    assert ch and d[0] == REMOVED and e == 0 and all(d[1:] == 0)
    c5 = cycle(oracle, 5)
    assert not oracle.reduce(c5, *root(c5), best_or_k=4, which=4)[3]
    d, cc, e, ch = oracle.reduce(c5, *root(c5), best_or_k=3, which=4)
    assert not ch and cc == 0
    p4 = path(oracle, 4)
    assert not oracle.reduce(p4, *root(p4), best_or_k=4, which=4)[3]


def test_kat_fixpoints(oracle):  # :112-137
    p5 = path(oracle, 5)
    d, cc, e, _ = oracle.reduce(p5, *root(p5), best_or_k=5, which=0)
    assert cc == 2 and e == 0 and cc == oracle.brute_force(p5)[0]
    c5 = cycle(oracle, 5)
    d, cc, e, _ = oracle.reduce(c5, *root(c5), best_or_k=5, which=0)
    assert cc == 0 and e == 5
    tree = mk(oracle, 7, [(0, 1), (0, 2), (1, 3), (1, 4), (2, 5), (2, 6)])
    d, cc, e, _ = oracle.reduce(tree, *root(tree), best_or_k=7, which=0)
    assert cc == 2 and cover_of(d) == [1, 2] and e == 0


def test_kat_should_prune_vectors(oracle):  # test_bounds.cpp:56-99, acceptance_main.cpp:353-365
    assert oracle.should_prune(3, 0, False, 0, 3)
    assert oracle.should_prune(2, 5, False, 0, 5)
    assert not oracle.should_prune(1, 1, True, 2, 0)
    assert not oracle.should_prune(2, 0, True, 2, 0)   # |S| = k is accepted
    assert oracle.should_prune(3, 0, True, 2, 0)
    assert oracle.should_prune(0, 10, True, 3, 0)      # 10 > 3^2
    assert not oracle.should_prune(0, 9, True, 3, 0)


def test_kat_solver_seq_named(oracle):  # test_solver_seq.cpp:10-38
    pet = mk(oracle, 10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (0, 5), (1, 6), (2, 7), (3, 8),
                          (4, 9), (5, 7), (7, 9), (9, 6), (6, 8), (8, 5)])
    assert oracle.solve_seq(pet)["size"] == 6
    assert oracle.solve_seq(cycle(oracle, 5))["size"] == 3
    assert oracle.solve_seq(complete(oracle, 4))["size"] == 3
    assert oracle.solve_seq(path(oracle, 4))["size"] == 2
    empty = mk(oracle, 5, [])
    assert oracle.solve_seq(empty)["size"] == 0
    r = oracle.solve_seq(empty, pvc=True, k=1)  # test_solver_seq.cpp:51-62
    assert r["feasible"] and r["size"] == 0
    with pytest.raises(ValueError):
        oracle.solve_seq(empty, pvc=True, k=0)


def test_brute_force_limit(oracle):
    with pytest.raises(ValueError):
        oracle.brute_force(path(oracle, 25))


# ---- golden vectors generated from the reference itself ------------------------------------

def test_oracle_matches_reference_golden_corpus(oracle, corpus):
    """535 graphs: brute force, sequential size AND node count, PVC triple, greedy cover."""
    bad = []
    for it in corpus:
        g = mk(oracle, it["n"], it["edges"])
        if oracle.brute_force(g)[0] != it["mvc"]:
            bad.append((it["name"], "bf"))
        s = oracle.solve_seq(g)
        if (s["size"], s["nodes"]) != (it["mvc"], it["seq_nodes"]):
            bad.append((it["name"], "seq", s["size"], s["nodes"]))
        if not oracle.verify_cover(g, s["cover"]):
            bad.append((it["name"], "cert"))
        for p in it["pvc"]:
            r = oracle.solve_seq(g, pvc=True, k=p["k"])
            if (r["feasible"], r["nodes"]) != (p["feasible"], p["nodes"]):
                bad.append((it["name"], "pvc", p["k"]))
        if oracle.greedy(g) != (it["greedy_size"], it["greedy_cover"]):
            bad.append((it["name"], "greedy"))
    assert not bad, bad[:10]


def test_oracle_matches_reference_config_goldens(oracle, config_golden):
    import paper_2204_10402_b200 as vc
    from paper_2204_10402_b200.configs import load_config
    for name in ("c1", "c2", "c3", "c4", "c5"):
        g = load_config(name)
        off, nbr = g.csr()
        csr = CSR(g.num_vertices, g.num_edges, off, nbr)
        assert oracle.greedy(csr)[0] == config_golden[name]["greedy"], name
    for name in ("c1", "c3"):
        g = load_config(name)
        off, nbr = g.csr()
        csr = CSR(g.num_vertices, g.num_edges, off, nbr)
        s = oracle.solve_seq(csr)
        assert (s["size"], s["nodes"]) == (config_golden[name]["mvc"],
                                          config_golden[name]["seq_nodes"])


def test_reduction_soundness(oracle, corpus):
    """acceptance_main.cpp:170-190: mvc(G) = added + mvc(reduced G) under the degree rules."""
    for it in corpus[::5]:
        g = mk(oracle, it["n"], it["edges"])
        d, cc, e, _ = oracle.reduce(g, *root(g), which=1)
        alive = d != REMOVED
        rest = [(u, v) for u, v in it["edges"] if alive[u] and alive[v]]
        assert it["mvc"] == cc + oracle.brute_force(mk(oracle, it["n"], rest))[0]


# ---- call-for-call against the reference itself (needs oracle/_ref) ------------------------

def test_oracle_rules_equal_reference_on_random_nodes(oracle, reference):
    rng = np.random.default_rng(7)
    for trial in range(300):
        n = int(rng.integers(4, 40))
        g = reference.gnp(n, float(rng.uniform(0.05, 0.6)), int(rng.integers(1 << 30)))
        d, cc, e = node_from_removed(g, rng.choice(n, size=int(rng.integers(0, n // 3 + 1)),
                                                   replace=False))
        pvc = bool(rng.integers(2))
        k = int(rng.integers(1, n + 1))
        best = int(rng.integers(1, n + 1))
        for which in (0, 1, 2, 3, 4):
            a = oracle.reduce(g, d, cc, e, pvc=pvc, k=k, best_or_k=best, which=which)
            b = reference.reduce(g, d, cc, e, pvc=pvc, k=k, best_or_k=best, which=which)
            assert (a[0] == b[0]).all() and a[1:] == b[1:], (trial, which)
        assert oracle.fingerprint(d, cc, e) == reference.fingerprint(d, cc, e)


def test_oracle_seq_equals_reference_seq(oracle, reference):
    rng = np.random.default_rng(11)
    for trial in range(40):
        n = int(rng.integers(10, 60))
        g = reference.gnp(n, float(rng.uniform(0.05, 0.4)), trial)
        a = oracle.solve_seq(g)
        b = reference.solve(g, strategy="seq")
        assert (a["size"], a["nodes"]) == (b["size"], b["nodes"])
        k = max(1, a["size"] - 1)
        a = oracle.solve_seq(g, pvc=True, k=k)
        b = reference.solve(g, pvc=True, k=k, strategy="seq")
        assert (a["feasible"], a["nodes"]) == (b["feasible"], b["nodes"])
