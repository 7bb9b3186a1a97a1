"""Top SASS lines by warp-stall samples from an ncu report: python scripts/hot_sass.py rep.ncu-rep [N]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
recs = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        try:
            recs.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"] or 0), d["Address"], d["Source"].strip()))
        except ValueError:
            pass
tot = sum(r[0] for r in recs) or 1
itot = sum(r[1] for r in recs) or 1
print(f"samples {tot}, warp-instructions {itot}, sass lines {len(recs)}")
for s, i, a, src in sorted(recs, key=lambda x: -x[0])[:n]:
    print(f"{100*s/tot:5.1f}% {100*i/itot:5.1f}%i  {a[-5:]}  {src[:90]}")
print("--- by instructions executed")
for s, i, a, src in sorted(recs, key=lambda x: -x[1])[:n]:
    print(f"{100*s/tot:5.1f}% {100*i/itot:5.1f}%i  {a[-5:]}  {src[:90]}")
