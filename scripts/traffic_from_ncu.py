"""DRAM traffic of the dominant kernel per launch from an ncu --set full report, into
profiles/r02/traffic.json (bench.py's roofline.traffic):
  python scripts/traffic_from_ncu.py <report.ncu-rep> <config> <kernel class> <algorithmic bytes> "<launch>"
The report must hold one launch of that kernel (the bench's dominant shape)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, ci, kernel, alg, launch = sys.argv[1], int(sys.argv[2]), sys.argv[3], float(sys.argv[4]), sys.argv[5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(r, name):
    i = h.index(name)
    return float(r[i].replace(",", "")) * scale.get(u[i], 1.0)


recs = [r for r in rows[2:] if kernel in r[h.index("Kernel Name")]]
assert recs, f"no {kernel} launch in {rep}"
r = recs[0]
rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
i_t = h.index("gpu__time_duration.sum")
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02", "traffic.json")
os.makedirs(os.path.dirname(out_path), exist_ok=True)
d = json.load(open(out_path)) if os.path.exists(out_path) else {}
d[f"config{ci}"] = {"kernel": kernel, "launch": launch, "dram_bytes": rd + wr, "dram_read_bytes": rd,
                    "dram_write_bytes": wr, "algorithmic_bytes": alg, "ratio": (rd + wr) / alg,
                    "ncu_time": f"{r[i_t]} {u[i_t]}", "source": os.path.relpath(rep)}
json.dump(d, open(out_path, "w"), indent=1)
print(json.dumps(d[f"config{ci}"]))
