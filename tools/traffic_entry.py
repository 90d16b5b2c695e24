"""Add/replace a profiles/traffic.json entry from an ncu --csv metrics log of
dram__bytes_read.sum / dram__bytes_write.sum.  Usage:
  traffic_entry.py LOG KEY FRAMES_PER_LAUNCH "SOURCE DESCRIPTION" [KERNEL_REGEX]"""
import csv
import io
import json
import os
import re
import sys

log, key, frames, src = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
kre = re.compile(sys.argv[5]) if len(sys.argv) > 5 else None
txt = open(log).read()
rows = list(csv.reader(io.StringIO(txt[txt.find('"ID"'):])))
h = rows[0]
ik, im, iv, iu, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
per = {}
kname = None
for r in rows[1:]:
    if len(r) <= iv or (kre and not kre.search(r[ik])):
        continue
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
    per.setdefault(r[ii], {})[r[im]] = v
    kname = r[ik]
rd = [d["dram__bytes_read.sum"] for d in per.values()]
wr = [d["dram__bytes_write.sum"] for d in per.values()]
n = len(rd)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
t = json.load(open(path)) if os.path.exists(path) else {}
t[key] = {"dram_bytes_per_frame": (sum(rd) + sum(wr)) / n / frames, "dram_read_per_frame": sum(rd) / n / frames,
          "dram_write_per_frame": sum(wr) / n / frames, "frames_per_launch": frames, "launches_averaged": n,
          "source": f"{src}, {kname}"}
json.dump(t, open(path, "w"), indent=1)
print(key, t[key])
