#!/usr/bin/env python3
"""Distil ncu reports into profiles/ (JSON + markdown).

    python tools/ncu_summarize.py gpurun_out profiles r01
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_dynamic",
    "launch__grid_size": "grid",
    "launch__cluster_size": "cluster",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "lts__t_bytes.sum": "l2_bytes",
}


def raw(rep):
    """Metrics of the captured launches; a split-path step (shrink + expand)
    is captured as two kernels whose durations and DRAM bytes are summed."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    hdr, units = rows[0], rows[1]
    d = {}
    names = []
    for vals in rows[2:]:
        for h, u, v in zip(hdr, units, vals):
            if h in METRICS:
                key = METRICS[h]
                try:
                    fv = float(v.replace(",", ""))
                except ValueError:  # "n/a" and the like: not a number, skip
                    continue
                if key in ("duration", "dram_read", "dram_write", "l2_bytes") and key in d:
                    d[key] = (d[key][0] + fv, u)
                else:
                    d.setdefault(key, (fv, u))
            if h == "Kernel Name":
                names.append(v.split("(")[0].replace("void ", "")[:40])
    d["kernel"] = (" + ".join(names), "")
    return d


def raw_rows(rep):
    """Per-launch metric rows of a report (the forward's shrink and GEMM separately)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            if h == "Kernel Name":
                d["kernel"] = (v.split("(")[0].replace("void ", "")[:40], "")
            if h in METRICS:
                try:
                    d[METRICS[h]] = (float(v.replace(",", "")), u)
                except ValueError:
                    pass
        res.append(d)
    return res


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}.get(u, 1)
    return v * scale


def to_us(v, u):
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)


def main():
    src, dst, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs(dst, exist_ok=True)
    summary = {}
    md = [f"# ncu summary ({tag})", "", "One `--set full --clock-control none` capture per config "
          "(cold, serialised replay: compare shares, not absolutes).", "",
          "| config | kernel | duration us | DRAM read MB | DRAM write MB | DRAM % peak | tensor % | regs | smem KB | grid | cluster |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
    for cfg in ("cfg2", "cfg3", "cfg5", "cfg4"):
        rep = os.path.join(src, f"prof_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d = raw(rep)
        if not d:
            continue
        dur = to_us(*d["duration"])
        rd = to_bytes(*d["dram_read"])
        wr = to_bytes(*d["dram_write"])
        entry = {"kernel": d.get("kernel", ("?", ""))[0][:80], "duration_us": dur, "dram_read_bytes": rd,
                 "dram_write_bytes": wr, "dram_bytes_per_launch": rd + wr}
        for k in ("dram_pct", "tensor_pct", "sm_pct", "registers", "grid", "cluster", "occupancy_pct"):
            if k in d:
                entry[k] = d[k][0]
        if "smem_dynamic" in d:
            entry["smem_dynamic"] = to_bytes(*d["smem_dynamic"])
        if "l2_bytes" in d:
            entry["l2_bytes"] = to_bytes(*d["l2_bytes"])
        summary[cfg] = entry
        md.append(f"| {cfg} | {entry['kernel'][:40]} | {dur:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
                  f"{entry.get('dram_pct', float('nan')):.1f} | {entry.get('tensor_pct', float('nan')):.2f} | "
                  f"{entry.get('registers', '')} | {entry.get('smem_dynamic', 0) / 1024:.0f} | {entry.get('grid', '')} | "
                  f"{entry.get('cluster', '')} |")
    # layer forward: one full capture of the shrink and the GEMM per config
    fwd_rows = []
    for cfg in ("cfg2", "cfg5"):
        rep = os.path.join(src, f"prof_fwd_{cfg}.ncu-rep")
        if not os.path.exists(rep):
            continue
        for d in raw_rows(rep):
            if "duration" not in d:
                continue
            e = {"kernel": d["kernel"][0], "duration_us": to_us(*d["duration"]),
                 "dram_read_bytes": to_bytes(*d["dram_read"]), "dram_write_bytes": to_bytes(*d["dram_write"])}
            for k in ("dram_pct", "tensor_pct", "sm_pct", "registers", "grid", "cluster"):
                if k in d:
                    e[k] = d[k][0]
            if "l2_bytes" in d:
                e["l2_bytes"] = to_bytes(*d["l2_bytes"])
            summary.setdefault(f"forward_{cfg}", []).append(e)
            fwd_rows.append(f"| {cfg} | {e['kernel']} | {e['duration_us']:.1f} | {e['dram_read_bytes'] / 1e6:.1f} | "
                            f"{e['dram_write_bytes'] / 1e6:.1f} | {e.get('l2_bytes', 0) / 1e6:.0f} | "
                            f"{e.get('tensor_pct', float('nan')):.1f} | {e.get('grid', '')} | {e.get('cluster', '')} |")
    if fwd_rows:
        md += ["", "## Layer forward (tools/fwd_bench.py, one layer): one capture per kernel", "",
               "| config | kernel | duration us | DRAM read MB | DRAM write MB | L2 MB | tensor % | grid | cluster |",
               "|---|---|---|---|---|---|---|---|---|"] + fwd_rows
    # launch list of the bench command
    lpath = os.path.join(src, "launches_bench.csv")
    if os.path.exists(lpath):
        text = open(lpath).read()
        lines = [l for l in text.splitlines() if not l.startswith("==")]
        rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
        per = {}
        dur_unit = "nsecond"
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            dur_unit = r.get("Metric Unit", dur_unit)
            name = r["Kernel Name"].split("(")[0][:60]
            v = float(r["Metric Value"].replace(",", ""))
            per.setdefault(name, []).append(v)
        tot = sum(sum(v) for v in per.values())
        md += ["", "## Launch list of `bench.py --steps 20 --warmup 3` (cfg2) under ncu", "",
               "| kernel | launches | mean us | share of GPU time |", "|---|---|---|---|"]
        shares = {}
        for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            u = to_us(1.0, dur_unit)
            shares[name] = {"launches": len(v), "mean_us": sum(v) / len(v) * u, "share": sum(v) / tot}
            md.append(f"| {name} | {len(v)} | {sum(v) / len(v) * u:.2f} | {100 * sum(v) / tot:.1f}% |")
        summary["bench_launch_list"] = shares
    with open(os.path.join(dst, "ncu_bypass_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    with open(os.path.join(dst, f"ncu_summary_{tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
