"""Static SASS opcode mix per kernel of a shared library (cuobjdump -sass):
    python tools/sass_mix.py paper_2510_20499_b200/libbp.so k_rows_full k_rows_sell ..."""
import collections
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
want = sys.argv[2:]
cur, mix = None, collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = next((w for w in want if w in m.group(1)), None)
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\d+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if m and cur:
        mix[cur][m.group(2)] += 1
KEEP = ("DADD", "DMUL", "DFMA", "DSETP", "LDG", "STG", "LDS", "STS", "LDL", "STL", "ATOM", "RED",
        "SHFL", "VOTE", "UBLKCP", "SYNCS", "BAR", "MEMBAR")
for k in want:
    c = mix.get(k)
    if not c:
        continue
    tot = sum(c.values())
    sel = [(op, n) for op, n in c.most_common() if op.startswith(KEEP)][:22]
    print(f"{k}: {tot} SASS instructions; " + ", ".join(f"{op} {n}" for op, n in sel))
