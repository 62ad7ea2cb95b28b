"""Shared-memory wavefronts (actual vs ideal) and stalls per source line range of an ncu report.

usage: python scripts/ncu_smem.py <report|src.csv.gz> <lib.so> <kernel-substring> <first> <last>
"""
import csv, gzip, io, os, re, subprocess, sys, tempfile, collections
rep, lib, kern, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
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
    text = gzip.open(rep, "rt").read()
else:
    text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(text)))
h = rows[1]
ix = {k: h.index(k) for k in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)",
                               "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal")}
base = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
for r in rows[2:]:
    try:
        a = int(r[ix["Address"]], 16)
    except ValueError:
        continue
    base = a if base is None else base
    loc = a2l.get(a - base)
    if not loc or not (lo <= loc[1] <= hi):
        continue
    f = lambda k: float(r[ix[k]] or 0)
    v = agg[loc[1]]
    v[0] += f("Instructions Executed"); v[1] += f("Warp Stall Sampling (All Samples)")
    v[2] += f("L1 Wavefronts Shared"); v[3] += f("L1 Wavefronts Shared Ideal")
for line in sorted(agg):
    e, st, w, wi = agg[line]
    print(f"L{line:<5d} exec {e:12.0f} stall {st:8.0f} smem wavefronts {w:12.0f} ideal {wi:12.0f}")
