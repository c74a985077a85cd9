"""Write profiles/k4_traffic.json from an ncu --set full capture of the K4 kernel on the bench workload:
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch, with the kernel name and the head
count of the run, so that bench.py can report roofline.traffic scaled to each rank's heads.
  python scripts/k4_traffic_from_ncu.py REP.ncu-rep CONFIG HEADS SOURCE_NOTE"""
import csv
import json
import os
import re
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rep, cfg, heads, note = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
val = lambda m: float(v[h.index(m)].replace(",", "")) * UNIT[u[h.index(m)]]
name = re.sub(r"^void\s+", "", v[h.index("Kernel Name")].split("(")[0]).replace("<unnamed>::", "").replace("(int)", "").replace(" ", "")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "k4_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d = {k: x for k, x in d.items() if isinstance(x, dict)}
d[cfg] = {"kernel": name, "bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"), "heads": heads,
          "source": note}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[cfg]))
