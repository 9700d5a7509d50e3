"""Summarise an ncu --set full report (.ncu-rep) into markdown + traffic JSON.

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_ncu_c2.md c2
Writes the per-kernel table to the markdown file and merges
dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes) into
profiles/traffic.json under the config name (bench.py reads it).
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp instrs"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, out_md, cfg):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    lines = ["| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " |",
             "|---|" + "---|" * len(METRICS)]
    traffic = {}
    for d in data:
        name = d[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        cells = []
        for met, _ in METRICS:
            v, u = d[ix[met]], units[ix[met]]
            cells.append(f"{v} {u}".strip())
        lines.append(f"| `{name}` | " + " | ".join(cells) + " |")
        rd = float(d[ix["dram__bytes_read.sum"]]) * SCALE.get(units[ix["dram__bytes_read.sum"]], 1)
        wr = float(d[ix["dram__bytes_write.sum"]]) * SCALE.get(units[ix["dram__bytes_write.sum"]], 1)
        base = name.split("<")[0]
        traffic[base] = int(rd + wr)
    with open(out_md, "a") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    allt.setdefault(cfg, {}).update(traffic)  # merge: a capture of some kernels keeps the others
    json.dump(allt, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
