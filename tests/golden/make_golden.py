"""Generates tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref/libvcref.so, the
unmodified reference sources compiled by oracle/Makefile). Run in the build container, where
/root/reference exists:

    python tests/golden/make_golden.py            # corpus.json + configs.json
    python tests/golden/make_golden.py --c5       # also the slow C5 PVC-no node count

corpus.json  : the reference's acceptance corpus (acceptance_main.cpp:82-116): named_corpus()
               (testutil.hpp:95-105) + random_corpus(500, 42) (testutil.hpp:107-116), each with
               brute-force MVC, sequential MVC size / node count, the PVC triple
               k in {opt-1, opt, opt+1} (feasible + node count), and the greedy cover.
configs.json : the frozen BASELINE configs (data/configs): greedy, MVC, PVC answers and the
               schedule-independent node counts of PVC no-instances.
"""
import gzip
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402


def named(ref):
    g = []
    for n in range(2, 9):
        g.append(("path%d" % n, n, [(v, v + 1) for v in range(n - 1)]))
    for n in range(3, 10):
        g.append(("cycle%d" % n, n, [(v, v + 1) for v in range(n - 1)] + [(n - 1, 0)]))
    for leaves in range(1, 9):
        g.append(("star%d" % leaves, leaves + 1, [(0, v) for v in range(1, leaves + 1)]))
    for n in range(2, 9):
        g.append(("complete%d" % n, n, [(u, v) for u in range(n) for v in range(u + 1, n)]))
    g.append(("petersen", 10, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 0), (0, 5), (1, 6), (2, 7),
                               (3, 8), (4, 9), (5, 7), (7, 9), (9, 6), (6, 8), (8, 5)]))
    g.append(("bintree2", 7, [(0, 1), (0, 2), (1, 3), (1, 4), (2, 5), (2, 6)]))
    out = [(name, ref.make_graph(n, e)) for name, n, e in g]
    for seed in range(4):
        out.append(("tree12_s%d" % seed, ref.random_tree(12, seed)))
    return out


def random_corpus(ref, count, seed_base):
    out = []
    for i in range(count):
        n = 4 + i % 13
        p = 0.1 + 0.1 * ((i // 13) % 9)
        out.append(("gnp%d_%g_s%d" % (n, p, seed_base + i), ref.gnp(n, p, seed_base + i)))
    return out


def corpus_json(ref):
    items = []
    for name, g in named(ref) + random_corpus(ref, 500, 42):
        opt, opt_cover = ref.brute_force(g)
        seq = ref.solve(g, strategy="seq")
        gs, gc = ref.greedy(g)
        pvc = []
        for k in (opt - 1, opt, opt + 1):
            if k < 1:
                continue
            r = ref.solve(g, pvc=True, k=k, strategy="seq")
            pvc.append(dict(k=k, feasible=r["feasible"], nodes=r["nodes"]))
        items.append(dict(name=name, n=g.n, edges=g.pairs().tolist(), mvc=opt,
                          brute_force_cover=opt_cover, seq_nodes=seq["nodes"],
                          seq_size=seq["size"], greedy_size=gs, greedy_cover=gc, pvc=pvc))
    return items


def load_config(ref, name):
    with gzip.open(os.path.join(ROOT, "data", "configs", name + ".clq.gz"), "rt") as f:
        g = ref.parse(f.read(), dimacs=True)
    return ref.complement(g) if name in ("c3", "c5") else g


def configs_json(ref, with_c5):
    out = {}
    t = time.time()
    c1 = load_config(ref, "c1")
    s = ref.solve(c1, strategy="seq")
    p = ref.solve(c1, pvc=True, k=s["size"] - 1, strategy="seq")
    out["c1"] = dict(n=c1.n, m=c1.m, greedy=ref.greedy(c1)[0], mvc=s["size"],
                     seq_nodes=s["nodes"], pvc_no_k=s["size"] - 1, pvc_no_nodes=p["nodes"])
    c3 = load_config(ref, "c3")
    s = ref.solve(c3, strategy="seq")
    p = ref.solve(c3, pvc=True, k=s["size"] - 1, strategy="seq")
    out["c3"] = dict(n=c3.n, m=c3.m, greedy=ref.greedy(c3)[0], mvc=s["size"],
                     seq_nodes=s["nodes"], pvc_no_k=s["size"] - 1, pvc_no_nodes=p["nodes"])
    c2 = load_config(ref, "c2")
    out["c2"] = dict(n=c2.n, m=c2.m, greedy=ref.greedy(c2)[0])
    c4 = load_config(ref, "c4")
    out["c4"] = dict(n=c4.n, m=c4.m, greedy=ref.greedy(c4)[0])
    c5 = load_config(ref, "c5")
    out["c5"] = dict(n=c5.n, m=c5.m, greedy=ref.greedy(c5)[0])
    if with_c5:
        yes = ref.solve(c5, pvc=True, k=483, strategy="hybrid", workers=os.cpu_count())
        no = ref.solve(c5, pvc=True, k=482, strategy="hybrid", workers=os.cpu_count())
        out["c5"].update(pvc_yes_k=483, pvc_yes=yes["feasible"], pvc_no_k=482,
                         pvc_no=no["feasible"], pvc_no_nodes=no["nodes"],
                         pvc_no_wall_ms_hybrid=no["wall_ms"], cpu_threads=os.cpu_count())
    out["_generated_s"] = round(time.time() - t, 1)
    return out


def main():
    ref = Reference()
    with open(os.path.join(HERE, "corpus.json"), "w") as f:
        json.dump(corpus_json(ref), f, separators=(",", ":"))
    path = os.path.join(HERE, "configs.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    new = configs_json(ref, "--c5" in sys.argv)
    if "--c5" not in sys.argv and "c5" in old:
        for key, val in old["c5"].items():
            new["c5"].setdefault(key, val)
    with open(path, "w") as f:
        json.dump(new, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
