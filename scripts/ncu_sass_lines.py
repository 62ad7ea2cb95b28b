"""Print the SASS (exec count, stall samples) of the instructions mapped to a source line range.

usage: python scripts/ncu_sass_lines.py <report> <lib.so> <kernel-substring> <first> <last> [file=am_kernel.cuh]
"""
import csv, io, os, re, subprocess, sys, tempfile
rep, lib, kern, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
fname = sys.argv[6] if len(sys.argv) > 6 else "am_kernel.cuh"
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
# the library holds one cubin per translation unit: disassemble the one defining the kernel
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
        fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and fn and kern in fn:
        a2l[int(m.group(1), 16)] = cur
if rep.endswith(".gz"):
    import gzip
    out = gzip.open(rep, "rt").read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, ie, iss, isrc = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
sr = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    base = a if base is None else base
    loc = a2l.get(a - base)
    if loc and loc[0] == fname and lo <= loc[1] <= hi:
        why = sorted(((float(r[i] or 0), nm) for i, nm in sr), reverse=True)[:2]
        why = " ".join(f"{nm}:{v:.0f}" for v, nm in why if v > 0)
        print(f"{a - base:06x} L{loc[1]:<5d} exec {float(r[ie] or 0):>10.0f} stall {float(r[iss] or 0):>6.0f} "
              f"{why:28s} {r[isrc]}")
