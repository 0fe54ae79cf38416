"""Write profiles/traffic.json (bench.py's roofline "traffic": DRAM read + write bytes per launch of
the dominant kernel) from an `ncu --set full ... --page raw --csv` export.
usage: python tools/make_traffic.py RAW.csv STAGE_NAME CONFIG [SOURCE_NOTE]"""
import csv, json, os, sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
raw, stage, config = sys.argv[1:4]
note = sys.argv[4] if len(sys.argv) > 4 else os.path.basename(raw)
rows = list(csv.reader(open(raw)))
hdr, units, data = rows[0], rows[1], [r for r in rows[2:] if len(r) == len(rows[0])]
i_r, i_w = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
per = [float(r[i_r]) * UNITS[units[i_r]] + float(r[i_w]) * UNITS[units[i_w]] for r in data]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
tj = json.load(open(out)) if os.path.exists(out) else {"config": config, "kernels": {}, "source": {}}
tj["config"] = config
tj["kernels"][stage] = sum(per) / len(per)
tj.setdefault("source", {})[stage] = f"{note}: mean of {len(per)} launch(es), dram__bytes_read.sum + dram__bytes_write.sum"
json.dump(tj, open(out, "w"), indent=1)
print(json.dumps(tj, indent=1))
