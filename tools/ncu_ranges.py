"""Sum an ncu source page (per file:line) over named line ranges of a source file."""
import csv, os, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
ranges = []  # name:a-b
for r in sys.argv[3:]:
    name, ab = r.split(":"); a, b = ab.split("-"); ranges.append((name, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if len(r) > 5 and r[0] == "Line No")
def num(x):
    try: return int(x)
    except ValueError: return 0
cur = "?"; tot_i = tot_s = 0; acc = {}
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur = os.path.basename(r[1]); continue
    if len(r) < 8 or not r[0].isdigit(): continue
    d = dict(zip(hdr, r)); i = num(d["Instructions Executed"]); s = num(d["Warp Stall Sampling (All Samples)"])
    tot_i += i; tot_s += s
    key = "other:" + cur
    if cur == fname:
        ln = int(r[0]); key = "other"
        for name, a, b in ranges:
            if a <= ln <= b: key = name; break
    x = acc.setdefault(key, [0, 0]); x[0] += i; x[1] += s
for k, (i, s) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:32s} inst {100*i/tot_i:5.1f}%  stall samples {100*s/tot_s:5.1f}%")
