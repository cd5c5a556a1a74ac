"""Summarise the ncu captures of a GPU session (gpurun_out/) into tracked
files under profiles/<tag>/:

  launches.csv          per-launch device time of every kernel (the
                        `--metrics gpu__time_duration.sum` pass)
  ncu_full_summary.md   key `--set full` metrics per kernel (time, DRAM bytes,
                        L1/shared wavefronts, bank conflicts, occupancy, issue)
  ncu_kernels.json      per kernel: the batch of the captured launch, its
                        DRAM traffic (dram__bytes_read + write) and L1/LSU
                        utilisation; read by bench.py for the roofline
                        "traffic" field (scaled to the bench batch)

    python scripts/summarize_ncu.py gpurun_out profiles/round2 [slices_per_launch]
"""
import csv
import json
import os
import re
import shutil
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed": "lsu_wavefronts_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "shared_wavefronts",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "bank_conflicts",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "launch__registers_per_thread": "regs",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
}


def short_name(k):
    m = re.search(r"(k_[a-z_0-9A-Z]+)(?:<[^>]*?(\d{3,5})[,>])?", k)
    if not m:
        return k[:40]
    return m.group(1) + (f"<{m.group(2)}>" if m.group(2) else "")


def main():
    src, dst = sys.argv[1], sys.argv[2]
    slices = float(sys.argv[3]) if len(sys.argv) > 3 else 16.0
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(src, "launches.csv")):
        shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "launches.csv"))
    rep = os.path.join(src, "prof_full.ncu-rep")
    if not os.path.exists(rep):
        return
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    lines = ["| kernel | " + " | ".join(KEYS.values()) + " |", "|" + "---|" * (len(KEYS) + 1)]
    traffic = {}
    lsu = {}  # L1/LSU data-pipe utilisation: the bound of the gather / shared-FFT kernels
    seen = set()
    for d in data:
        name = short_name(d[ki])
        vals = []
        for k in KEYS:
            v = d[hdr.index(k)] if k in hdr else ""
            u = units[hdr.index(k)] if k in hdr else ""
            vals.append(f"{v} {u}".strip())
        lines.append(f"| {name} | " + " | ".join(vals) + " |")
        if name not in seen and "dram__bytes_read.sum" in hdr:
            seen.add(name)
            rd = float(d[hdr.index("dram__bytes_read.sum")])
            wr = float(d[hdr.index("dram__bytes_write.sum")])
            scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
            rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1.0)
            wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1.0)
            traffic[name] = rd + wr
            key = "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"
            if key in hdr:
                lsu[name] = float(d[hdr.index(key)])
    with open(os.path.join(dst, "ncu_full_summary.md"), "w") as f:
        f.write(f"ncu --set full --clock-control none, {os.path.basename(rep)}; one R and one R# launch of "
                f"{slices:g} slices at N=2048 (the bench plan and batch; scripts/profile_one.py), cache "
                "flushed between replays.\n\n")
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(dst, "ncu_kernels.json"), "w") as f:
        json.dump({"source": os.path.basename(rep), "kernels": {
            n: {"batch": slices, "dram_bytes": traffic[n], "lsu_pct": lsu.get(n)} for n in traffic}}, f, indent=1)


if __name__ == "__main__":
    main()
