"""Replays one fuzz mismatch with every check reported separately."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_10402_b200 as vc
from oracle.oracle import CSR, Oracle
o = Oracle()
for path in sys.argv[1:]:
    g = vc.parse_edge_list(open(path).read()) if hasattr(vc, "parse_edge_list") else None
    n = g.num_vertices
    off, nbr = g.csr()
    csr = CSR(n, g.num_edges, off, nbr)
    want = o.solve_seq(csr)
    no = o.solve_seq(csr, pvc=True, k=want["size"] - 1)
    out = dict(path=path, n=n, m=g.num_edges, mvc=want["size"], seq_nodes=want["nodes"], no_nodes=no["nodes"])
    for rep in range(3):
        r = vc.solve_mvc(g, strategy="gpu")
        out[f"gpu_mvc_{rep}"] = (r["size"], vc.verify_cover(g, r["cover"]))
        p = vc.solve_pvc(g, want["size"] - 1, strategy="gpu")
        out[f"gpu_no_{rep}"] = (p["feasible"], p["nodes_total"])
        y = vc.solve_pvc(g, want["size"], strategy="gpu")
        out[f"gpu_yes_{rep}"] = (y["feasible"], y["feasible"] and vc.verify_cover(g, y["cover"]))
    s = vc.solve_mvc(g, strategy="seq")
    out["seq"] = (s["size"], sum(s["worker_nodes"]))
    sp = vc.solve_mvc(g, strategy="gpu", engine="sparse")
    out["sparse"] = (sp["size"], vc.verify_cover(g, sp["cover"]))
    pw = vc.solve_pvc(g, want["size"] - 1, strategy="gpu", engine="dense-wide")
    out["wide_no"] = (pw["feasible"], pw["nodes_total"])
    print(json.dumps(out), flush=True)
