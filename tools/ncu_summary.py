"""Summarise ncu reports (raw page) and launch lists into profiles/ text files."""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
STALL = re.compile(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$")


def summarise(rep: str) -> str:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    lines = []
    for v in rows[2:]:
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"{k:70s} {v[i]:>22s} {u[i]}")
        stalls = []
        for i, k in enumerate(h):
            m = STALL.match(k)
            if m:
                try:
                    val = float(v[i])
                except ValueError:
                    continue
                if val >= 0.05:
                    stalls.append((val, m.group(1)))
        lines.append("stall reasons (warps stalled per issued instruction):")
        for val, name in sorted(stalls, reverse=True):
            lines.append(f"    {name:30s} {val:6.2f}")
        lines.append("")
    return "\n".join(lines)


def launches(path: str) -> str:
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    h = rows[0]
    ik, im, iv, iu = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0][:60]
        key = (name, r[im], r[iu])
        try:
            val = float(r[iv].replace(",", ""))
        except ValueError:
            continue
        n, s = agg.get(key, (0, 0.0))
        agg[key] = (n + 1, s + val)
    lines = [f"{'kernel':60s} {'metric':28s} {'launches':>8s} {'sum':>14s} {'mean':>14s} unit"]
    for (name, met, unit), (n, s) in sorted(agg.items()):
        lines.append(f"{name:60s} {met:28s} {n:8d} {s:14.1f} {s / n:14.1f} {unit}")
    return "\n".join(lines)


if __name__ == "__main__":
    mode, src = sys.argv[1], sys.argv[2]
    print(summarise(src) if mode == "rep" else launches(src))
