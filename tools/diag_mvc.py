import json, os, sys
sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
for path in ["tests/data/fuzz_200_12063.el", "tests/data/fuzz_128_4403.el"]:
    g = vc.parse_edge_list(open(path).read())
    res = {}
    for label, kw in [("gpu", dict(strategy="gpu")), ("gpu_wide", dict(strategy="gpu", engine="dense-wide")),
                      ("hybrid3552", dict(strategy="hybrid", workers=3552)), ("gpu_w32", dict(strategy="gpu", workers=32)),
                      ("gpu_w1", dict(strategy="gpu", workers=1)), ("hybrid4", dict(strategy="hybrid", workers=4))]:
        try:
            r = vc.solve_mvc(g, **kw)
            res[label] = (r["size"], r["cover_from_search"], r["greedy_size"], r["nodes_total"])
        except Exception as e:
            res[label] = str(e)[:60]
    print(path, json.dumps(res), flush=True)
