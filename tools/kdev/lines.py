"""Per-source-line SASS op histogram of a kdev cubin (nvdisasm -g)."""
import re, subprocess, sys
cub = sys.argv[1]; thr = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
cur = None; stats = {}
for l in dis.split("\n"):
    m = re.search(r'//## File ".*?/(\w+\.cuh?)", line (\d+)', l)
    if m: cur = (m.group(1), int(m.group(2))); continue
    m = re.match(r'\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)', l)
    if m and cur is not None:
        op = m.group(2)
        op = op if op.startswith("IMAD.MOV") else op.split('.')[0]
        stats.setdefault(cur, {}); stats[cur][op] = stats[cur].get(op, 0) + 1
for ln in sorted(stats):
    n = sum(stats[ln].values())
    if n >= thr: print(ln[1], n, dict(sorted(stats[ln].items(), key=lambda x: -x[1])[:7]))
