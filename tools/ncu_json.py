"""DRAM bytes per engine launch (stamped with the sha of csrc/count.cu it was captured from) from an ncu report -> profiles/ncu_engine_<cfg>.json (dev tool)."""
import csv
import io
import json
import subprocess
import sys

rep, out, src = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
ks = []
for r in rows[2:]:
    def val(m, sc):
        i = hdr.index(m)
        return float(r[i].replace(",", "")) * sc.get(units[i], 1)
    ks.append({"kernel": r[hdr.index("Kernel Name")],
               "duration_ms": val("gpu__time_duration.sum", tscale),
               "dram_bytes": val("dram__bytes_read.sum", scale) + val("dram__bytes_write.sum", scale)})
import hashlib
import os
cu = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1406_5687_b200", "csrc", "count.cu")
sha = hashlib.sha256(open(cu, "rb").read()).hexdigest()[:16]
json.dump({"source": src, "count_cu_sha": sha, "kernels": ks, "dram_bytes_per_launch": sum(k["dram_bytes"] for k in ks)},
          open(out, "w"), indent=1)
print(json.dumps(ks, indent=1))
