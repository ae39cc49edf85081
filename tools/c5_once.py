"""Two C5 PVC k=482 solves through the package found in the current directory (ncu A/B)."""
import sys
sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config('c5')
for _ in range(2):
    r = vc.solve_pvc(g, 482, strategy='gpu', **eval('dict(%s)' % (sys.argv[1] if len(sys.argv) > 1 else '')))
print(r['nodes_total'], r['device_ms'])
