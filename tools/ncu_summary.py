"""Summarise a round's ncu evidence into markdown (profiles/<round>_ncu_summary.md).

    python tools/ncu_summary.py r01d [--steps 2]

Reads gpurun_out/launches_<round>.csv (tools/profile_round.sh: the bench's
timed steps, gpu__time_duration per launch) and gpurun_out/prof_<round>_*.ncu-rep
(tools/profile_kernels.sh: --set full captures), via `ncu -i ... --page raw --csv`.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys

METRICS = [
    ("time", "gpu__time_duration.sum"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM B/s", "dram__bytes.sum.per_second"),
    ("PCIe read B/s", "pcie__read_bytes.sum.per_second"),
    ("SM throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("warps active %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("regs/thread", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("dyn smem/block", "launch__shared_mem_per_block_dynamic"),
]


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("void ", "")


def launches(path, steps):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, si, vi, ui = h.index("Kernel Name"), h.index("Stream"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.defaultdict(lambda: [0, 0.0])
    by_stream = collections.defaultdict(float)
    total = 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[r[ui]]
        ms = v * scale
        k = short(r[ki])
        per[k][0] += 1
        per[k][1] += ms
        by_stream[r[si]] += ms
        total += ms
    big = {s: ms for s, ms in by_stream.items() if ms >= 0.05 * total}
    rest = total - sum(big.values())
    streams = ", ".join(f"stream {s}: {ms / steps:.1f} ms/step" for s, ms in sorted(big.items()))
    if rest > 0:
        streams += (f", {len(by_stream) - len(big)} more streams (graph-replay side "
                    f"streams): {rest / steps:.1f} ms/step")
    out = [f"{sum(c for c, _ in per.values())} launches, {total:.1f} ms of serialised device time "
           f"for {steps} steps; by stream: " + streams, "",
           "| share | ms / step | launches / step | kernel |", "|---:|---:|---:|---|"]
    for k, (c, ms) in sorted(per.items(), key=lambda x: -x[1][1]):
        out.append(f"| {100 * ms / total:.1f}% | {ms / steps:.2f} | {c // steps} | `{k}` |")
    return out


def capture(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return None, []
    h, units = rows[0], rows[1]
    data = rows[2:]
    return (h, units), data


def main():
    rnd = sys.argv[1]
    steps = int(sys.argv[sys.argv.index("--steps") + 1]) if "--steps" in sys.argv else 2
    md = [f"# ncu evidence, {rnd} (B200, sm_100a)", ""]
    lf = f"gpurun_out/launches_{rnd}.csv"
    if os.path.exists(lf):
        md += ["## Launch list of the bench's timed steps (`tools/profile_round.sh`)", ""]
        md += ["ncu serialises kernels and caches are cold: compare SHARES, not absolutes.", ""]
        md += launches(lf, steps) + [""]
    md += ["## Full captures (`tools/profile_kernels.sh`: `ncu --set full --clock-control none "
           "--import-source on`, the C3 per-layer launch sizes)", ""]
    for rep in sorted(glob.glob(f"gpurun_out/prof_{rnd}_*.ncu-rep")):
        (hu, data) = capture(rep)
        if not hu:
            continue
        h, units = hu
        for vals in data:
            name = short(vals[h.index("Kernel Name")])
            md += [f"### `{name}`", "", "| metric | value |", "|---|---:|"]
            for label, m in METRICS:
                if m in h:
                    i = h.index(m)
                    md.append(f"| {label} (`{m}`) | {vals[i]} {units[i]} |")
            md.append("")
    print("\n".join(md))


if __name__ == "__main__":
    main()
