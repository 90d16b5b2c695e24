"""Per-source-line warp-stall samples and executed instructions from an ncu report
(--page source --print-source=cuda,sass).  Usage: ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, recs, ts, ti = None, [], 0, 0
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] not in ("", "Line No"):
        try:
            s, ins = int(r[4]), int(r[7])
        except ValueError:
            continue
        recs.append((cur, int(r[0]), s, ins, r[1].strip()[:80]))
        ts += s
        ti += ins
print(f"samples {ts}  instructions {ti}")
for key, name in ((2, "stall samples"), (3, "instructions")):
    print(f"--- top lines by {name}")
    for o in sorted(recs, key=lambda x: -x[key])[:top]:
        print(f"{o[0]:16s}{o[1]:5d}  samp {o[2] / ts * 100:5.1f}%  inst {o[3] / ti * 100:5.1f}%  {o[4]}")
