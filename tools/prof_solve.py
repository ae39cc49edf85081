import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import paper_2204_10402_b200 as vc
from paper_2204_10402_b200.configs import load_config
g = load_config('c5')
for _ in range(3): vc.solve_pvc(g, 482, strategy='gpu')
pr = cProfile.Profile(); pr.enable()
for _ in range(20): r = vc.solve_pvc(g, 482, strategy='gpu')
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(14)
ts = []
for _ in range(10):
    t = time.perf_counter(); r = vc.solve_pvc(g, 482, strategy='gpu'); ts.append(((time.perf_counter() - t) * 1e3, r['wall_ms'], r['device_ms']))
for x in ts: print('py %.3f wall %.3f dev %.3f' % x)
