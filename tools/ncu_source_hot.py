#!/usr/bin/env python3
"""Summarise warp-stall samples per CUDA source line from an ncu report.

    python tools/ncu_source_hot.py gpurun_out/prof_cfg2.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    recs = []
    total = 0
    for r in rows[1:]:
        if len(r) != len(h) or r[0] == "":  # keep CUDA-line aggregates, skip SASS rows
            continue
        try:
            s = int(r[idx["Warp Stall Sampling (All Samples)"]])
        except ValueError:
            continue
        total += s
        stalls = {k: int(r[idx[k]]) for k in stall_cols if r[idx[k]].isdigit() and int(r[idx[k]]) > 0}
        recs.append((s, r[idx["Line No"]], r[1][:90], stalls))
    recs.sort(reverse=True)
    print(f"total samples {total}")
    for s, ln, src, st in recs[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{s:7d} {100.0 * s / max(total, 1):5.1f}%  L{ln:>4} {src:<90} {top3}")


if __name__ == "__main__":
    main()
