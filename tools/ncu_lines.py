"""Per-CUDA-source-line totals of an ncu report (dev tool):
python tools/ncu_lines.py REPORT [top] [sort-column]
Columns: warp instructions, stall samples, shared-memory wavefronts, global L2 sectors."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
key = sys.argv[3] if len(sys.argv) > 3 else "inst"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []


def num(r, name):
    try:
        return int(float(r[hdr.index(name)] or 0))
    except (ValueError, IndexError):
        return 0


for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        lines.append(dict(ln=int(r[0]), src=r[1].strip()[:80], inst=num(r, "Instructions Executed"),
                          smp=num(r, "Warp Stall Sampling (All Samples)"), shw=num(r, "L1 Wavefronts Shared"),
                          l2=num(r, "L2 Theoretical Sectors Global")))
tot = {k: (sum(x[k] for x in lines) or 1) for k in ("inst", "smp", "shw", "l2")}
print(f"total warp-inst {tot['inst'] / 1e6:.1f}M, stall samples {tot['smp']}, shared wavefronts "
      f"{tot['shw'] / 1e6:.1f}M, L2 sectors {tot['l2'] / 1e6:.1f}M")
for x in sorted(lines, key=lambda x: -x[key])[:top]:
    print(f"{x['ln']:5d} inst {x['inst'] / 1e6:7.1f}M {100 * x['inst'] / tot['inst']:4.1f}%  smp "
          f"{100 * x['smp'] / tot['smp']:4.1f}%  shw {x['shw'] / 1e6:6.1f}M {100 * x['shw'] / tot['shw']:4.1f}%  "
          f"{x['src']}")
