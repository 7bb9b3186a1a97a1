"""Summarize ncu reports (.ncu-rep) into a markdown table for profiles/.

usage: python scripts/ncu_summary.py label=path.ncu-rep [...] > profiles/rNN_ncu_summary.md
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_op_red.sum",
        "lts__t_sectors_op_atom.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        res.append((d, u))
    return res


def main():
    print("| kernel (report) | launch | time | DRAM read | DRAM write | DRAM % peak | mem % peak | "
          "L2 red sectors | warps active % | inst (warp) | regs | grid |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for arg in sys.argv[1:]:
        label, path = arg.split("=", 1)
        for i, (d, u) in enumerate(raw(path)):
            def g(k):
                v = d.get(k, "")
                return f"{v} {u.get(k, '')}".strip()
            name = d.get("Kernel Name", "?")[:48]
            print(f"| {name} ({label}) | {i} | {g(KEYS[0])} | {g(KEYS[1])} | {g(KEYS[2])} | {g(KEYS[4])} | "
                  f"{g(KEYS[3])} | {g(KEYS[5])} | {g(KEYS[7])} | {g(KEYS[8])} | {g(KEYS[9])} | {g(KEYS[10])} |")


if __name__ == "__main__":
    main()
