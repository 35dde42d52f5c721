"""Per-launch DRAM traffic of one kernel from an ncu CSV (dram__bytes_read.sum +
dram__bytes_write.sum), averaged over the captured launches, merged into profiles/traffic.json.

    python scripts/traffic_from_ncu.py <ncu.csv> <config key> [kernel substring]

The capture is a steady-state range: `ncu --cache-control none --clock-control none
--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:<kernel>
-s <warm-up launches> -c <>=8> ... python bench.py --config <key>` — no cache flush between
launches, so each launch pays for the write-back of what it leaves dirty and reads what the
previous kernel left in L2, as in the timed loop.
"""
import csv
import json
import os
import statistics
import sys

path, key = sys.argv[1], sys.argv[2]
want = sys.argv[3] if len(sys.argv) > 3 else ""
launches = {}
hdr = None
for r in csv.reader(open(path)):
    if "Metric Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if want not in d["Kernel Name"]:
            continue
        v = float(d["Metric Value"].replace(",", ""))
        launches.setdefault(d["ID"], {})[d["Metric Name"]] = v
tot = [l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in launches.values()]
rd = [l["dram__bytes_read.sum"] for l in launches.values()]
wr = [l["dram__bytes_write.sum"] for l in launches.values()]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(root, "profiles", "traffic.json")
data = json.load(open(out)) if os.path.exists(out) else {}
data[key] = int(statistics.mean(tot))
data[key + "_detail"] = {"source": os.path.basename(path), "launches": len(tot),
                         "read_mean": int(statistics.mean(rd)), "write_mean": int(statistics.mean(wr)),
                         "per_launch_total": [int(t) for t in tot]}
json.dump(data, open(out, "w"), indent=1)
print(key, data[key], data[key + "_detail"])
