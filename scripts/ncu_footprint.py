"""Per-source-line code footprint of the hot path: SASS bytes executed at least `min_exec` times.

usage: python scripts/ncu_footprint.py <report.ncu-rep> <lib.so> <kernel-substring> <min_exec>
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, lib, kern, min_exec = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
sass = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
addr2line, cur_fn, cur_line = {}, None, None
for ln in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur_line = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and kern in cur_fn:
        addr2line[int(m.group(1), 16)] = cur_line
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
fp = collections.Counter()
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    base = a if base is None else base
    if float(r[ie] or 0) >= min_exec:
        fp[addr2line.get(a - base, ("?", 0))] += 16
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2011_04240_b200", "csrc", "am_kernel.cuh")).read().splitlines()
# attribute to enclosing function by scanning back for a line starting a __device__/__global__ function
def func_of(line):
    for i in range(line - 1, -1, -1):
        m = re.match(r"__(device|global)__.*?(\w+)\(", src[i])
        if m:
            return m.group(2)
    return "?"
byfn = collections.Counter()
for (f, l), b in fp.items():
    byfn[func_of(l) if f == "am_kernel.cuh" else f] += b
print(f"hot footprint: {sum(fp.values()) / 1024:.1f} KB")
for k, v in byfn.most_common():
    print(f"  {k:28s} {v / 1024:6.1f} KB")
