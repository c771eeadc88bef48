"""DRAM traffic per launch of a kernel class from an ncu --set full capture, into
profiles/<out>.json (read by bench.py's roofline.traffic):
  python tools/traffic_json.py X.ncu-rep dm_adam k_dm_adam "capture description" [out]
Averages dram__bytes_read.sum + dram__bytes_write.sum over every captured launch
whose name matches (e.g. the actor's and the critic's launch of one minibatch)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, cls, pat, desc = sys.argv[1:5]
out = sys.argv[5] if len(sys.argv) > 5 else "profiles/r1_ncu_traffic.json"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ki, rd, wr, tm = (h.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                        "gpu__time_duration.sum"))
units = rows[1]


def val(r, i):
    v = float(r[i].replace(",", ""))
    u = units[i]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
                "msecond": 1e3}.get(u, 1)


sel = [r for r in rows[2:] if pat in r[ki]]
if not sel:
    sys.exit(f"no launch matching {pat}")
n = len(sel)
entry = {"kernel": pat, "launches_averaged": n,
         "dram_read_bytes": sum(val(r, rd) for r in sel) / n,
         "dram_write_bytes": sum(val(r, wr) for r in sel) / n,
         "time_us": sum(val(r, tm) for r in sel) / n, "capture": desc}
entry["dram_bytes_per_launch"] = entry["dram_read_bytes"] + entry["dram_write_bytes"]
d = json.load(open(out)) if os.path.exists(out) else {}
d[cls] = entry
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(entry, indent=1))
