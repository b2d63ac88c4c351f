"""Dev tool: for every global load (LDG) in a kernel's SASS, the distance (in instructions) to the first
instruction that reads its destination register -- a short distance inside a loop means the in-order warp
waits for DRAM right there.  usage: ldg_use.py <object.o> <mangled-name-substring> [max_dist]"""
import re
import subprocess
import sys

obj, name = sys.argv[1], sys.argv[2]
maxd = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    head = f.split("\n", 1)[0]
    if name not in head:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", line)
        if m:
            ins.append((m.group(1), m.group(2).strip()))
    print(head.strip()[:110], len(ins), "instructions")
    loops = []  # (target, branch) of backward branches: instructions in [target, branch] run in a loop
    for addr, txt in ins:
        m = re.search(r"BRA(?:\.\S+)?\s+(?:`\()?0x([0-9a-f]+)", txt)
        if m and int(m.group(1), 16) < int(addr, 16):
            loops.append((int(m.group(1), 16), int(addr, 16)))
    in_loop = lambda a: any(t <= int(a, 16) <= b for t, b in loops)
    for i, (addr, txt) in enumerate(ins):
        m = re.match(r"(@!?U?P\d+\s+)?LDG\S*\s+(R\d+)", txt)
        if not m:
            continue
        dst = int(m.group(2)[1:])
        wide = ".64" in txt.split()[0 if not m.group(1) else 1] or ".64" in txt[:20]
        regs = {dst, dst + 1} if wide else {dst}
        for j in range(i + 1, min(len(ins), i + 400)):
            t = ins[j][1]
            # sources: everything after the first operand
            parts = t.split(",")
            srcs = ",".join(parts[1:]) if len(parts) > 1 else ""
            first = parts[0]
            used = any(re.search(r"\bR%d\b" % r, srcs) for r in regs)
            if used:
                if j - i <= maxd:
                    print("  %s %s %-48s -> +%3d  %s" % (addr, "LOOP" if in_loop(addr) else "    ", txt[:48], j - i, t[:60]))
                break
            if any(re.search(r"\bR%d\b" % r, first) for r in regs) and not t.startswith(("ST", "@")):
                break  # overwritten before use
