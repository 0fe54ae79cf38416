"""Rank CUDA source lines of an `ncu -i X --page source --csv --print-source cuda,sass` export by
warp-stall samples and by executed instructions.  usage: python tools/ncu_source_top.py SRC.csv [N]"""
import csv, os, sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, fname, hdr = [], None, None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    def num(k):
        try:
            return float(r[hdr[k]])
        except (ValueError, KeyError):
            return 0.0
    stalls = {k: num(k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
    rows.append((fname, r[0], r[1].strip()[:90], num("Warp Stall Sampling (All Samples)"),
                 num("Instructions Executed"), stalls))
tot_s = sum(x[3] for x in rows) or 1
tot_i = sum(x[4] for x in rows) or 1
for key, label in ((3, "stall samples"), (4, "instructions executed")):
    print(f"== top {top} source lines by {label} (total {tot_s if key == 3 else tot_i:.4g})")
    for f, ln, src, s, ins, st in sorted(rows, key=lambda x: -x[key])[:top]:
        big = sorted(((v, k[6:]) for k, v in st.items() if v), reverse=True)[:3]
        print(f"{100*s/tot_s:5.1f}% smp {100*ins/tot_i:5.1f}% ins  {f}:{ln}  {src}  [{', '.join(f'{k} {int(v)}' for v, k in big)}]")
