"""Summarise the ncu captures of profiles/run_profiles.sh into committed evidence.

    python profiles/summarize.py [round_tag]

Reads gpurun_out/{launches.csv, prof_gemm.ncu-rep, prof_hbm.ncu-rep} and writes
profiles/<tag>_summary.md, profiles/<tag>_kernels.json and
profiles/gemm_traffic.json (DRAM bytes per grouped-GEMM launch, used by
bench.py's roofline "traffic" field).
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = {
    "time_us": ("gpu__time_duration.sum", {"ms": 1e3, "us": 1, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "nsecond": 1e-3}),
    "dram_read_B": ("dram__bytes_read.sum", {"GB": 1e9, "Gbyte": 1e9, "MB": 1e6, "Mbyte": 1e6, "KB": 1e3, "Kbyte": 1e3, "byte": 1, "B": 1}),
    "dram_write_B": ("dram__bytes_write.sum", {"GB": 1e9, "Gbyte": 1e9, "MB": 1e6, "Mbyte": 1e6, "KB": 1e3, "Kbyte": 1e3, "byte": 1, "B": 1}),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None),
    "tensor_pct": ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", None),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None),
    "regs": ("launch__registers_per_thread", None),
}


def raw(rep: Path):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        ent = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")}
        for key, (name, conv) in METRICS.items():
            if name not in hdr:
                continue
            i = hdr.index(name)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if conv:
                v *= conv.get(units[i], 1.0)
            ent[key] = v
        out.append(ent)
    return out


def launches(name="launches.csv"):
    p = OUT / name
    rows = list(csv.reader(open(p)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1.0)
                out.append((d["Kernel Name"].split("(")[0], float(d["Metric Value"].replace(",", "")) * scale))
    return out


def main(tag="r01"):
    lines = [f"# ncu evidence ({tag})", "",
             "Commands: profiles/run_profiles.sh (B200, 1 GPU, `--clock-control none`). "
             "Workload: bench.py configs[1] (N=16, k=2, d=1024, f=4096, 64K tokens).", ""]
    summary = {}
    if (OUT / "launches.csv").exists():
        L = launches()
        # one complete steady-state step: from a gate launch to the next
        starts = [i for i, (n, _) in enumerate(L) if "gate_kernel" in n]
        if len(starts) >= 2:
            L = L[starts[-2]:starts[-1]]
        tot = sum(t for _, t in L)
        lines += ["## Launch list of one step (cold-cache, serialised: compare shares)", "",
                  "| kernel | µs | share |", "|---|---:|---:|"]
        for name, t in L:
            lines.append(f"| {name} | {t:.1f} | {100 * t / tot:.1f}% |")
        lines += ["", f"Total {tot:.0f} µs over {len(L)} launches.", ""]
        summary["launches"] = [{"kernel": n, "us": t} for n, t in L]
    if (OUT / "dist_launches.csv").exists():
        # configs[2] through the multi-GPU P2P phases (torchrun, N = 1): the
        # second-to-last complete step, steps delimited by the gate launch
        L = launches("dist_launches.csv")
        starts = [i for i, (n, _) in enumerate(L) if "gate_kernel" in n]
        if len(starts) >= 3:
            step = L[starts[-3]:starts[-2]]
            tot = sum(t for _, t in step)
            lines += ["## configs[2] P2P step (multi-GPU phases at N = 1, torchrun; cold-cache, serialised)", "",
                      "| kernel | µs | share |", "|---|---:|---:|"]
            for name, t in step:
                lines.append(f"| {name} | {t:.1f} | {100 * t / tot:.1f}% |")
            lines += ["", f"Total {tot:.0f} µs over {len(step)} launches.", ""]
            summary["dist_launches"] = [{"kernel": n, "us": t} for n, t in step]
    for rep, title in [("prof_gemm", "Grouped GEMM (tcgen05) — six launches of one step"),
                       ("prof_hbm", "Gate / dispatch / combine / reductions")]:
        f = OUT / f"{rep}.ncu-rep"
        if not f.exists():
            continue
        R = raw(f)
        summary[rep] = R
        lines += [f"## {title} (`ncu --set full`)", "",
                  "| kernel | µs | DRAM read MB | DRAM write MB | DRAM % peak | tensor % | SM % | warps % | regs |",
                  "|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
        for e in R:
            lines.append(
                f"| {e['kernel'][:48]} | {e.get('time_us', 0):.1f} | {e.get('dram_read_B', 0) / 1e6:.1f} | "
                f"{e.get('dram_write_B', 0) / 1e6:.1f} | {e.get('dram_pct', 0):.1f} | "
                f"{e.get('tensor_pct', 0):.1f} | {e.get('sm_pct', 0):.1f} | "
                f"{e.get('warps_active_pct', 0):.1f} | {e.get('regs', 0):.0f} |")
        lines.append("")
        if rep == "prof_gemm" and R:
            traffic = sum(e.get("dram_read_B", 0) + e.get("dram_write_B", 0) for e in R) / len(R)
            (PROF / "gemm_traffic.json").write_text(json.dumps(
                {"bytes_per_launch": traffic, "launches": len(R), "source": f"{tag} ncu --set full",
                 "kernel": "grouped_gemm_kernel"}, indent=1))
    (PROF / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
    (PROF / f"{tag}_kernels.json").write_text(json.dumps(summary, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["r01"]))
