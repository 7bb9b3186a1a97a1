"""Brief summary of one ncu report: time, DRAM bytes, instructions, issue, occupancy, top stall reasons,
and the SASS lines with the most stall samples / executed instructions.  python scripts/ncu_brief.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
for k in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
          "sm__inst_executed.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]:
    print(f"{k:55s} {d.get(k)}")
st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio") and v]
print("stalls/issue:", ", ".join(f"{k[34:-29]} {v:.2f}" for k, v in sorted(st, key=lambda x: -x[1])[:7]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
hdr, recs = None, []
for r in csv.reader(io.StringIO(src)):
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        x = dict(zip(hdr, r))
        try:
            recs.append((int(x["Address"], 16), int(x["Instructions Executed"] or 0), int(x["Warp Stall Sampling (All Samples)"] or 0), x["Source"].strip()))
        except ValueError:
            pass
if recs:
    recs.sort()
    b0 = recs[0][0]
    it = sum(r[1] for r in recs) or 1
    ss = sum(r[2] for r in recs) or 1
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    print("top stall lines:")
    for a, i, s, t in sorted(recs, key=lambda r: -r[2])[:n]:
        print(f"  {a - b0:6x} {100 * s / ss:5.1f}%s {100 * i / it:5.2f}%i  {t[:70]}")
