"""Aggregate an ncu source page (cuda,sass) per (file, CUDA source line): instructions + stall samples."""
import csv, os, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if len(r) > 5 and r[0] == "Line No")
def num(x):
    try: return int(x)
    except ValueError: return 0
src = {}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
fname = "?"
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if len(r) < 8 or not r[0].isdigit():
        continue
    d = dict(zip(hdr, r))
    st = {c: num(d.get(c, 0)) for c in stall_cols}
    src[(fname, int(r[0]))] = (num(d["Instructions Executed"]), num(d["Warp Stall Sampling (All Samples)"]), d["Source"][:70], st)
tot_i = sum(v[0] for v in src.values()); tot_s = sum(v[1] for v in src.values())
print(f"total instructions {tot_i:.3e}, samples {tot_s}")
agg = {}
for v in src.values():
    for c, x in v[3].items(): agg[c] = agg.get(c, 0) + x
print("stalls:", ", ".join(f"{c[6:]} {100*x/tot_s:.1f}%" for c, x in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
key = 1 if len(sys.argv) < 3 else int(sys.argv[2])
for (f, ln), (i, s, t, st) in sorted(src.items(), key=lambda kv: -kv[1][key])[:45]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{f[:18]:18s}:{ln:4d} inst {100*i/tot_i:5.1f}%  stall {100*s/tot_s:5.1f}% [{','.join(f'{c[6:]}:{x}' for c,x in top)}] {t}")
