"""SASS instructions per source line / function of one kernel (code-size attribution).

    cuobjdump -xelf all build/bp_propagate.o; nvdisasm --print-line-info X.cubin > all.sass
    python tools/sass_lines.py all.sass KERNEL_SUBSTRING [N]
"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
want = sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
fn, cur = None, None
cnt = collections.Counter()
for l in lines:
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        fn = m.group(1)
        continue
    if not fn or want not in fn:
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]+\*/\s+\S", l) and cur:
        cnt[cur] += 1
tot = sum(cnt.values())
print("total", tot)
for k, v in cnt.most_common(n):
    print(f"{v:6d} {k[0]}:{k[1]}")
