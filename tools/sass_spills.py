#!/usr/bin/env python
"""List local-memory (spill) instructions of one kernel with their source lines.
  python tools/sass_spills.py MANGLED_SUBSTR [LIB.so]"""
import os
import re
import subprocess
import sys
import tempfile

fn = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(__file__), "..", "paper_2003_05361_b200",
                                                         "libras_b200.so")
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
for cub in os.listdir(tmp):
    lines = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
    st = [i for i, l in enumerate(lines) if ".section" in l and ".text." in l and fn in l]
    if not st:
        continue
    cur = None
    n = 0
    for l in lines[st[0] + 1:]:
        if l.strip().startswith(".section") and ".text." in l:
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = int(m.group(2))
            continue
        if "LDL" in l or "STL" in l:
            n += 1
            print(cur, l.strip()[:100])
    print("total", n)
    break
