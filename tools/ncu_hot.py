"""Print the hottest SASS instructions (by warp-stall samples) of one kernel from an ncu source-page CSV.
usage: python tools/ncu_hot.py <csv> <kernel-substring> [instance=0] [top=40]"""
import csv, sys

path, pat = sys.argv[1], sys.argv[2]
inst = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
blocks, cur = [], None
for row in csv.reader(open(path)):
    if row and row[0] == "Kernel Name":
        cur = [row[1], None, []]
        blocks.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = row
    elif cur is not None:
        cur[2].append(row)
sel = [b for b in blocks if pat in b[0]]
name, hdr, rows = sel[inst]
H = {h: i for i, h in enumerate(hdr)}
print(name, len(rows), "instructions")
S = H["Warp Stall Sampling (All Samples)"]
tot = sum(float(r[S] or 0) for r in rows)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {s: sum(float(r[H[s]] or 0) for r in rows) for s in stalls}
print("total samples", tot, " by reason:", ", ".join(f"{k[6:]}={v/tot:.2f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
ex = H["Instructions Executed"]
print("executed warp-instr:", sum(float(r[ex] or 0) for r in rows))
idx = sorted(range(len(rows)), key=lambda i: -float(rows[i][S] or 0))[:top]
for i in sorted(idx):
    r = rows[i]
    top3 = sorted(((float(r[H[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{r[0]:>6} {float(r[S] or 0)/tot:6.3f} ex={r[ex]:>10} {r[1][:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in top3 if v))
