"""Print the SASS of the hottest loop region of an ncu source page with per-instruction stall
samples and top stall reasons.  usage: ncu_sass_loop.py <full_src.csv.gz> [top_k_instructions]"""
import csv, gzip, io, sys
rows = list(csv.reader(io.TextIOWrapper(gzip.open(sys.argv[1]), errors="replace")))
hdr = rows[1]
data = rows[2:]
ci = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
base = int(data[0][0], 16)
recs = []
for r in data:
    try:
        a = int(r[0], 16) - base
    except ValueError:
        continue
    smp = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[ci["Instructions Executed"]] or 0)
    st = sorted(((int(r[ci[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
    recs.append((a, r[1].strip(), smp, ex, st))
tot = sum(x[2] for x in recs)
# hottest window of 400 instructions by samples
best, bi = 0, 0
win = 400
s = sum(x[2] for x in recs[:win])
for i in range(len(recs) - win):
    if s > best:
        best, bi = s, i
    s += recs[i + win][2] - recs[i][2]
print(f"total samples {tot}; hottest {win}-instruction window {best} ({best / tot:.1%}) at +{recs[bi][0]:#x}")
for a, t, smp, ex, st in recs[bi:bi + win]:
    if ex == 0:
        continue
    rs = " ".join(f"{n}:{v}" for v, n in st if v)
    print(f"{a:#7x} {smp:6d} {ex:9d}  {t[:60]:60s} {rs}")
