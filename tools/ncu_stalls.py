"""Per-source-line stall breakdown (selected stall columns) from an ncu report.
Usage: ncu_stalls.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, recs = None, None, []
keys = ["stall_long_sb", "stall_lg", "stall_not_selected", "stall_selected", "stall_barrier", "stall_wait",
        "stall_mio", "stall_short_sb", "stall_dispatch", "stall_branch_resolving", "stall_math", "stall_sleep"]
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
        recs.append((cur, int(r[0]), [num(k) for k in keys], num("Warp Stall Sampling (All Samples)"), r[1].strip()[:60]))
tot = sum(x[3] for x in recs) or 1
print("line".ljust(22), " ".join(k.replace("stall_", "")[:7].rjust(7) for k in keys), "  all%")
for o in sorted(recs, key=lambda x: -x[3])[:top]:
    print(f"{o[0][:14]:14s}{o[1]:5d}  ", " ".join(f"{v / tot * 100:7.2f}" for v in o[2]), f"{o[3] / tot * 100:6.2f}  {o[4]}")
tt = [sum(x[2][i] for x in recs) / tot * 100 for i in range(len(keys))]
print("TOTAL".ljust(21), " ".join(f"{v:7.2f}" for v in tt))
