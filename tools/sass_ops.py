"""Static SASS opcode histogram of one kernel in the built library.
usage: python tools/sass_ops.py <kernel-substring> [lib]"""
import collections
import re
import subprocess
import sys

lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1607_03936_b200/libwbfbt.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s*Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if sys.argv[1] not in name:
        continue
    c = collections.Counter()
    for line in b.split("\n"):
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            c[m.group(2)] += 1
    tot = sum(c.values())
    print(name[:90], "total", tot)
    print("  " + "  ".join(f"{o}:{n}" for o, n in c.most_common(22)))
