"""Summarise an ncu report: key raw metrics + hottest SASS blocks (dev tool)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_executed.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__grid_size"]
for r in rows[2:]:
    print("kernel:", r[hdr.index("Kernel Name")][:80])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w} = {r[i]} {units[i]}")
    stalls = [(hdr[i], r[i]) for i in range(len(hdr)) if hdr[i].startswith("smsp__average_warp_latency_issue_stalled")
              or (hdr[i].startswith("smsp__warp_issue_stalled") and hdr[i].endswith("per_warp_active.pct"))]
    top = sorted(((float(v), h) for h, v in stalls if v.replace('.', '', 1).isdigit()), reverse=True)[:8]
    for v, h in top:
        print(f"  stall {h} = {v}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    ia, ss, sc = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    end = next((i for i in range(2, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
    data = [(r[sc], int(r[ia] or 0), int(r[ss] or 0)) for r in rows[2:end] if len(r) > ia and (r[ia] or "0").isdigit()]
    blocks = []
    for s_, c, smp in data:
        if blocks and blocks[-1][0] == c:
            blocks[-1][1] += 1
            blocks[-1][2] += smp
            blocks[-1][3].append(s_.strip()[:36])
        else:
            blocks.append([c, 1, smp, [s_.strip()[:36]]])
    tot = sum(c * n for c, n, _, _ in blocks)
    tots = sum(smp for _, _, smp, _ in blocks)
    print(f"total warp-inst {tot/1e6:.1f}M, stall samples {tots}")
    for c, n, smp, ins in blocks:
        if c * n > tot * 0.01 or smp > tots * 0.02:
            print(f"  {c:10d} x {n:3d} = {c*n/1e6:7.1f}M  samples {smp:6d} ({100*smp/tots:4.1f}%)  {ins[0]} .. {ins[-1]}")
