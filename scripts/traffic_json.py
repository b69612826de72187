"""DRAM traffic per stage (dram__bytes_read.sum + dram__bytes_write.sum summed over the
stage's launches) from one ncu --set full capture of scripts/prof_step.py, as the JSON
bench.py reads for roofline.traffic.

  python scripts/traffic_json.py <report.ncu-rep> <out.json> <note>
"""
import csv
import json
import re
import subprocess
import sys

STAGES = [("p2p", r"k_p2p"), ("anterp", r"k_anterp"), ("eval", r"k_eval"), ("c2p", r"k_c2p"), ("p2c", r"k_p2c"),
          ("prox2pw", r"k_prox2pw"), ("pwshift", r"k_pwshift"), ("pw2poly", r"k_pw2poly|k_pwlocal")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
by = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    for st, pat in STAGES:
        if re.search(pat, name):
            b = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = h.index(m)
                b += float(r[i].replace(",", "")) * scale.get(units[i], 1)
            by[st] = by.get(st, 0) + int(b)
            break
if "pwshift" in by or "pw2poly" in by:
    by["pwlocal"] = by.get("pwshift", 0) + by.get("pw2poly", 0)
json.dump({"note": sys.argv[3], "bytes": dict(sorted(by.items()))}, open(sys.argv[2], "w"), indent=1)
print(json.dumps(by))
