"""The five BASELINE.json configurations as frozen graphs (data/configs/*.clq.gz).

C1/C2/C4 are solved as stored; C3/C5 are p_hat-style clique instances solved on their
complement, as the paper does with DIMACS p_hat graphs.
"""
from __future__ import annotations

import gzip
import os

from . import complement, parse_dimacs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(ROOT, "data", "configs")

CONFIGS = {
    "c1": dict(file="c1.clq.gz", complement=False, mode="mvc",
               desc="MVC on Erdos-Renyi G(128, avg deg 8, seed 0)"),
    "c2": dict(file="c2.clq.gz", complement=False, mode="pvc-pair",
               desc="PVC yes/no pair on G(400, avg deg 6, seed 0), k = MVC and MVC-1"),
    "c3": dict(file="c3.clq.gz", complement=True, mode="mvc",
               desc="MVC on the complement of p_hat-style G(300, a=0, b=0.5)"),
    "c4": dict(file="c4.clq.gz", complement=False, mode="mvc-throughput",
               desc="MVC on Barabasi-Albert n=100k, m=3 (node budget)"),
    "c5": dict(file="c5.clq.gz", complement=True, mode="pvc-no",
               desc="hard PVC no-instance k = MVC-1 on the complement of p_hat-style "
                    "G(500, a=0.25, b=0.75)"),
    # C5-scale ("pick the C5 density so that 1-GPU time >= ~10 s"): p_hat500-3-like
    "c5s": dict(file="c5s.clq.gz", complement=True, mode="pvc-no",
                desc="strong-scaling PVC no-instance k = MVC-1 = 448 on the complement of "
                     "p_hat-style G(500, a=0.48, b=1.0)"),
}


def config_text(name: str) -> str:
    with gzip.open(os.path.join(DATA, CONFIGS[name]["file"]), "rt") as f:
        return f.read()


def load_config(name: str):
    g = parse_dimacs(config_text(name))
    return complement(g) if CONFIGS[name]["complement"] else g
