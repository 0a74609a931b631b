"""Static SASS opcode histogram of a kernel's hottest loop (dev tool).
    python tools/sass_loop.py <mangled-name-substring> [lib]
The loop is the shortest backward-branch range containing a streaming load
(LDG.E.EF, i.e. __ldcs) -- the particle loop; counts are per iteration."""
import collections
import re
import subprocess
import sys

name = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2201_05555_b200/libpicrom_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs if f.startswith(name) or name in f.split("\n")[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for addr, txt in ins:
    m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", txt)
    if m:
        tgt = int(m.group(1), 16)
        has = any(tgt <= a2 <= addr and "LDG.E.EF" in t2 for a2, t2 in ins)
        if tgt < addr and has and (best is None or addr - tgt < best[1] - best[0]):
            best = (tgt, addr)
lo, hi = best
loop = [t for a, t in ins if lo <= a <= hi]
cnt = collections.Counter()
for t in loop:
    op = t.split()[0]
    if op.startswith("@"):
        op = t.split()[1]
    cnt[op.split(".")[0]] += 1
print(f"loop 0x{lo:x}-0x{hi:x}: {len(loop)} instructions")
for op, c in cnt.most_common(40):
    print(f"  {op:10s} {c}")
