"""Per-source-line shared-memory wavefronts (total / excessive) and L2 sectors from an ncu
report (--page source).  Usage: ncu_smem.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, recs = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))

        def num(k):
            try:
                return float(d.get(k, "0").replace(",", "") or 0)
            except ValueError:
                return 0.0
        recs.append((cur, int(r[0]), num("L1 Wavefronts Shared"), num("L1 Wavefronts Shared Excessive"),
                     num("L2 Theoretical Sectors Global"), num("L2 Theoretical Sectors Global Excessive"),
                     r[1].strip()[:70]))
for idx, name in ((2, "smem wavefronts"), (3, "smem excessive"), (4, "L2 sectors"), (5, "L2 excessive")):
    tot = sum(x[idx] for x in recs) or 1
    print(f"--- {name}: total {tot:,.0f}")
    for o in sorted(recs, key=lambda x: -x[idx])[:top]:
        if o[idx] <= 0:
            break
        print(f"{o[0]:16s}{o[1]:5d} {o[idx]:14,.0f} {o[idx] / tot * 100:5.1f}%  {o[6]}")
