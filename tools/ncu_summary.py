"""Summarise ncu reports into profiles/ (JSON + markdown).

    python tools/ncu_summary.py <report.ncu-rep> <out-stem> [--algorithmic-bytes B]

Writes <out-stem>.json (the metrics bench.py reads: dram_bytes_per_launch etc.)
and <out-stem>.md (table + top stall reasons from the SASS source page).
"""

import csv
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "us": 1e-6, "ms": 1e-3, "ns": 1e-9,
         "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2]


def stalls(rep, top=6):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    hdr = rows[1]
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {c: 0 for c in cols}
    for r in rows[2:]:
        for c in cols:
            try:
                tot[c] += int(r[hdr.index(c)])
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1
    return {c: round(100.0 * v / s, 1) for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:top]}


def main():
    rep, stem = sys.argv[1], sys.argv[2]
    alg = None
    if "--algorithmic-bytes" in sys.argv:
        alg = float(sys.argv[sys.argv.index("--algorithmic-bytes") + 1])
    hdr, units, vals = raw(rep)
    d = {"report": rep.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")]}
    for key, _ in METRICS:
        if key in hdr:
            i = hdr.index(key)
            d[key] = {"value": vals[i], "unit": units[i]}
    def num(key):
        v = d[key]
        return float(v["value"].replace(",", "")) * SCALE.get(v["unit"], 1.0)
    rd, wr, t = num("dram__bytes_read.sum"), num("dram__bytes_write.sum"), num("gpu__time_duration.sum")
    d["dram_bytes_per_launch"] = rd + wr
    d["duration_s"] = t
    d["dram_gbs"] = (rd + wr) / t / 1e9
    if alg:
        d["algorithmic_bytes_per_launch"] = alg
        d["traffic_over_algorithmic"] = (rd + wr) / alg
        d["algorithmic_gbs"] = alg / t / 1e9
    d["stall_share_pct"] = stalls(rep)
    json.dump(d, open(stem + ".json", "w"), indent=1)
    with open(stem + ".md", "w") as f:
        f.write(f"# ncu --set full: `{d['kernel'][:100]}`\n\nreport: `{d['report']}` (cold-cache, serialised replay)\n\n")
        f.write("| metric | value |\n|---|---|\n")
        for key, name in METRICS:
            if key in d:
                f.write(f"| {name} (`{key}`) | {d[key]['value']} {d[key]['unit']} |\n")
        f.write(f"| DRAM bytes per launch (read+write) | {d['dram_bytes_per_launch'] / 1e9:.4f} GB |\n")
        f.write(f"| DRAM GB/s (traffic / duration) | {d['dram_gbs']:.0f} |\n")
        if alg:
            f.write(f"| algorithmic bytes per launch | {alg / 1e9:.4f} GB |\n")
            f.write(f"| traffic / algorithmic | {d['traffic_over_algorithmic']:.3f} |\n")
            f.write(f"| algorithmic GB/s under ncu | {d['algorithmic_gbs']:.0f} |\n")
        f.write("\nWarp-stall sample shares (SASS source page):\n\n")
        for k, v in d["stall_share_pct"].items():
            f.write(f"- {k}: {v}%\n")
    print(json.dumps({k: d[k] for k in ("kernel", "dram_bytes_per_launch", "duration_s", "dram_gbs")}))


if __name__ == "__main__":
    main()
