"""SASS opcode histogram of every kernel in a built library (cuobjdump -sass).

  python tools/sass_hist.py [lib.so] [--match SUBSTR] [--top N] [--json OUT]

Per kernel: total instructions, shared (LDS/STS/LDSM), generic (LD.E/ST.E — a shared access
that lost its address space shows up here), global (LDG/STG), TMA (UTMALDG/UTMASTG/UBLKCP),
async copies (LDGSTS), FP32 (FFMA/FADD/FMUL), FP64 (DFMA/DADD/DMUL) and the top opcodes.
"""
from __future__ import annotations

import json
import re
import subprocess
import sys
from collections import Counter

CLASSES = {
    "shared": re.compile(r"^(LDS|STS|LDSM|ATOMS)"),
    "generic": re.compile(r"^(LD|ST)\.E"),
    "global": re.compile(r"^(LDG|STG|RED|ATOMG)"),
    "tma": re.compile(r"^(UTMALDG|UTMASTG|UTMAPF|UBLKCP|UBLKRED|UTMACCTL)"),
    "cp_async": re.compile(r"^LDGSTS"),
    "fp32": re.compile(r"^(FFMA|FADD|FMUL|FMNMX|FSETP|FSEL)"),
    "fp64": re.compile(r"^(DFMA|DADD|DMUL|DSETP)"),
    "shfl": re.compile(r"^SHFL"),
}


def histograms(lib: str) -> dict[str, Counter]:
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    res: dict[str, Counter] = {}
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            res[cur] = Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m and cur is not None:
            res[cur][m.group(1)] += 1
    return res


def summarise(h: Counter) -> dict:
    d = {"total": sum(h.values())}
    for k, rx in CLASSES.items():
        d[k] = sum(v for op, v in h.items() if rx.match(op))
    d["top"] = h.most_common(12)
    return d


def demangle(names: list[str]) -> dict[str, str]:
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
        return dict(zip(names, out))
    except OSError:
        return {n: n for n in names}


def main() -> None:
    args = sys.argv[1:]
    lib = "paper_2209_03883_b200/libofdmr_b200.so"
    match, top, js = None, 40, None
    i = 0
    while i < len(args):
        if args[i] == "--match":
            match = args[i + 1]; i += 2
        elif args[i] == "--top":
            top = int(args[i + 1]); i += 2
        elif args[i] == "--json":
            js = args[i + 1]; i += 2
        else:
            lib = args[i]; i += 1
    hs = histograms(lib)
    dm = demangle(list(hs))
    rows = {}
    for name, h in hs.items():
        pretty = dm.get(name, name)
        if match and match not in pretty:
            continue
        rows[pretty] = summarise(h)
    for pretty, d in sorted(rows.items(), key=lambda kv: -kv[1]["total"])[:top]:
        cls = " ".join(f"{k}={d[k]}" for k in CLASSES)
        print(f"{d['total']:6d} {pretty}\n       {cls}\n       top: {d['top']}")
    if js:
        with open(js, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
