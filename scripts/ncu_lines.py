"""Aggregate an ncu SASS source page (csv) by CUDA source line using nvdisasm -g line info.

usage: python scripts/ncu_lines.py <report.ncu-rep> <lib.so> <kernel-substring> [topN]
"""
import csv, io, os, re, subprocess, sys, tempfile, collections

rep, lib, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
# the library holds one cubin per translation unit: disassemble the one defining the kernel
sass = ""
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if re.search(r"\.text\.\S*" + re.escape(kern), txt):
        sass = txt
        break
addr2line = {}
cur_fn, cur_line = None, None
for ln in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and kern in cur_fn:
        addr2line[int(m.group(1), 16)] = cur_line
if rep.endswith(".gz"):
    import gzip
    out = gzip.open(rep, "rt").read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
isrc = hdr.index("Source")
agg = collections.defaultdict(lambda: [0, 0])
ops = collections.defaultdict(lambda: collections.Counter())
tot_e = tot_s = 0
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    a -= base
    e = float(r[ie] or 0); s = float(r[iss] or 0)
    line = addr2line.get(a, "?")
    agg[line][0] += e; agg[line][1] += s
    ops[line][r[isrc].split()[0] if r[isrc].split() else "?"] += e
    tot_e += e; tot_s += s
print(f"total executed {tot_e:.3e}  stall samples {tot_s:.0f}")
for line, (e, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    topops = ", ".join(f"{k}:{v/max(e,1):.0%}" for k, v in ops[line].most_common(3))
    print(f"{line:28s} exec {e/tot_e:6.1%}  stall {s/max(tot_s,1):6.1%}   {topops}")
