"""Static SASS size per source line for one kernel of libvcgpu.so (dev tool)."""
import collections, os, re, subprocess, sys, tempfile
pat = sys.argv[1] if len(sys.argv) > 1 else "dense_kernelILi16ELb0"
lib = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2204_10402_b200", "libvcgpu.so")
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=d, capture_output=True)
cub = max((os.path.join(d, f) for f in os.listdir(d)), key=os.path.getsize)
out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
cur = fn = None
cnt = collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.search(r'\.section\s+\.text\.(\S+),', line)
    if m: fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+[A-Z@{]', line) and cur and fn: cnt[fn][cur] += 1
k = [f for f in cnt if pat in f][0]
c = cnt[k]; tot = sum(c.values())
print(k, "total", tot, "instr", tot * 16 / 1024, "KB")
src = {}
for (f, l), n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    path = os.path.join(os.path.dirname(lib), "csrc", f)
    txt = open(path).read().split('\n')[l - 1].strip()[:70] if os.path.exists(path) else ""
    print(f"{n:6d} {100*n/tot:5.1f}% {f}:{l}  {txt}")
