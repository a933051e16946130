"""Dev: summarise an ncu source page (`ncu -i R --page source --csv --print-source sass`) — total
stall-reason shares and the instructions with the most warp-state samples.
Usage: python tools/sass_stalls.py <source.csv> [top=40] [min_pct=0.5]"""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
min_pct = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for line, r in enumerate(rows[2:]):
    if len(r) != len(hdr):
        continue
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    st = {h[6:]: float(r[ix[h]] or 0) for h in stall_cols}
    recs.append((line, s, int(r[ix["Instructions Executed"]] or 0), r[ix["Source"]].strip(), st))
tot = sum(x[1] for x in recs) or 1.0
agg = {}
for _, _, _, _, st in recs:
    for k, v in st.items():
        agg[k] = agg.get(k, 0.0) + v
print("total", tot, {k: round(100 * v / tot, 1) for k, v in sorted(agg.items()) if v / tot >= 0.005})
for line, s, ex, src, st in sorted(recs, key=lambda x: -x[1])[:top]:
    if 100 * s / tot < min_pct:
        break
    rs = sorted(st.items(), key=lambda kv: -kv[1])[:2]
    print(f"{line:5d} {100 * s / tot:5.2f}% exe={ex:8d} {src[:60]:60s} " +
          " ".join(f"{k}:{100 * v / tot:.2f}" for k, v in rs if v > 0))
