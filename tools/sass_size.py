"""SASS size per kernel of a shared library: python tools/sass_size.py lib.so [name-substring ...]"""
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
keys = sys.argv[2:] or [""]
f, last = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        f = m.group(1)
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/", line)
    if m and f:
        last[f] = int(m.group(1), 16)
for k, v in sorted(last.items(), key=lambda kv: -kv[1]):
    if any(s in k for s in keys):
        name = re.sub(r"_ZN2bp\d+_GLOBAL__N__\w+?_cu_\w{8}\d+", "", k)[:40]
        print(f"{v // 16 + 1:8d} instr {(v + 16) / 1024:8.1f} KB  {name}")
