"""Per-kernel SASS opcode mix of a built object / library (cuobjdump), e.g.
    python tools/sass_mix.py paper_2410_15526_b200/build/k_reduce.o k4_tlq_dq_reduce_qILi8ELi4ELb0 [OPS...]"""
import re
import subprocess
import sys
from collections import Counter

path, pat = sys.argv[1], sys.argv[2]
ops = sys.argv[3:]
out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
for block in out.split("Function : ")[1:]:
    name = block.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    c = Counter()
    for line in block.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+(\.[A-Z0-9_]+)*)", line)
        if m:
            c[m.group(2)] += 1
    short = re.sub(r"_ZN4sdp4\d+_GLOBAL__N__\w+?_cu_[0-9a-f]+\d+", "", name)[:80]
    sel = {k: v for k, v in c.items() if not ops or any(k.startswith(o) for o in ops)}
    print(short, sum(c.values()), dict(sorted(sel.items(), key=lambda x: -x[1])[:25]))
