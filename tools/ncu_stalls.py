"""Summarise an ncu --page source --csv (SASS) export: top instructions by warp-stall samples
and totals per stall reason.  usage: python tools/ncu_stalls.py file.csv [topN]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: sum(float(r[ix[h]] or 0) for r in data) for h in stall_cols}
allsum = sum(tot.values())
print("stall totals (% of samples):")
for h, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"  {h:28s} {100 * v / allsum:5.1f}%")
key = "Warp Stall Sampling (All Samples)"
top = sorted(data, key=lambda r: -float(r[ix[key]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
print("top instructions:")
for r in top:
    reasons = sorted(((h, float(r[ix[h]] or 0)) for h in stall_cols), key=lambda x: -x[1])[:3]
    print(f"  {r[ix['Address']]:>6s} {100 * float(r[ix[key]]) / allsum:5.1f}%  {r[ix['Source']][:60]:60s} " +
          " ".join(f"{h[6:]}={100 * v / allsum:.1f}" for h, v in reasons if v))
