"""Stall-reason totals of an ncu source page, overall and per source-line range.

usage: python scripts/ncu_stalls.py <report> <lib.so> <kernel-substring> [file:lo-hi ...]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kern = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    f, _, r = a.partition(":")
    lo, _, hi = r.partition("-")
    ranges.append((a, f, int(lo), int(hi)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
sass = ""
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if re.search(r"\.text\.\S*" + re.escape(kern), txt):
        sass = txt
        break
a2l, fn, cur = {}, None, None
for ln in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and fn and kern in fn:
        a2l[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, ie = h.index("Address"), h.index("Instructions Executed")
sr = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = {name: collections.Counter() for name, *_ in [("all",)] + ranges}
execs = collections.Counter()
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    base = a if base is None else base
    loc = a2l.get(a - base)
    keys = ["all"] + [name for name, f, lo, hi in ranges if loc and loc[0] == f and lo <= loc[1] <= hi]
    for k in keys:
        execs[k] += float(r[ie] or 0)
        for i, nm in sr:
            tot[k][nm] += float(r[i] or 0)
for k, c in tot.items():
    s = sum(c.values())
    top = ", ".join(f"{nm} {v / max(s, 1) * 100:.1f}%" for nm, v in c.most_common(8))
    print(f"{k:28s} exec {execs[k]:.3e} stall samples {s:.0f}: {top}")
