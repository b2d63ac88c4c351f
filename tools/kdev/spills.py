"""Per-kernel registers / spills from the ptxas -v logs (paper_2604_00048_b200/build/*.log).
Usage: spills.py [log-glob] [all]"""
import glob, re, sys
pat = sys.argv[1] if len(sys.argv) > 1 else "paper_2604_00048_b200/build/*.log"
s = "\n".join(open(f).read() for f in sorted(glob.glob(pat)))
cur, spill = None, (0, 0)
for line in s.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur, spill = m.group(1), (0, 0)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = re.sub(r"_ZN4whit\d+", "", cur).replace("EEEvNS_6ParamsE", "")
        if spill != (0, 0) or len(sys.argv) > 2:
            print(f"{name:50s} regs {m.group(1)} spill st/ld {spill}")
        cur = None
