"""Stall reasons and executed instructions per device function (phase) from an ncu SASS source page.

usage: python scripts/ncu_phases.py <report.ncu-rep> <lib.so> <kernel-substring>
Uses nvdisasm -g line info of the same binary; attributes each instruction to the
enclosing function of its (innermost) source line in am_kernel.cuh.
"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, lib, kern = sys.argv[1:4]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
# the library holds one cubin per translation unit: disassemble the one defining the kernel
sass = ""
for cub in sorted(f for f in os.listdir(tmp) if f.endswith(".cubin")):
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    if re.search(r"\.text\.\S*" + re.escape(kern), txt):
        sass = txt
        break
addr2line, cur_fn, cur = {}, None, None
for ln in sass.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        cur_fn = m.group(1); continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(?:.*inlined at "([^"]+)", line (\d+))?', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_fn and kern in cur_fn:
        addr2line[int(m.group(1), 16)] = cur
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2011_04240_b200", "csrc",
                        "am_kernel.cuh")).read().splitlines()
starts = [(i + 1, m.group(2)) for i, l in enumerate(src) for m in [re.match(r"__(device|global)__.*?(\w+)\(", l)] if m]
def func_of(f, line):
    if f != "am_kernel.cuh":
        return f
    name = "?"
    for s, n in starts:
        if s <= line:
            name = n
    return name
if rep.endswith(".gz"):
    import gzip
    out = gzip.open(rep, "rt").read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ir = [hdr.index(h) for h in reasons]
agg = collections.defaultdict(lambda: collections.Counter())
base = None
for r in rows[2:]:
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    base = a if base is None else base
    f, l = addr2line.get(a - base, ("?", 0))
    fn = func_of(f, l)
    agg[fn]["exec"] += float(r[ie] or 0)
    for h, i in zip(reasons, ir):
        agg[fn][h] += float(r[i] or 0)
tot_s = sum(sum(v[h] for h in reasons) for v in agg.values())
tot_e = sum(v["exec"] for v in agg.values())
print(f"{'function':26s} {'exec%':>6s} {'stall%':>6s}  top stall reasons (share of the function's samples)")
for fn, v in sorted(agg.items(), key=lambda kv: -sum(kv[1][h] for h in reasons)):
    st = sum(v[h] for h in reasons)
    if st / max(tot_s, 1) < 0.005:
        continue
    top = sorted(((v[h], h[6:]) for h in reasons), reverse=True)[:4]
    print(f"{fn:26s} {100*v['exec']/tot_e:6.1f} {100*st/tot_s:6.1f}  " + ", ".join(f"{n}:{c/max(st,1):.0%}" for c, n in top))
