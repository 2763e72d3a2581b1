#!/usr/bin/env python
"""Refresh profiles/ncu_traffic.json (DRAM bytes per launch of each workload's hot kernel, bench.py's roofline
'traffic') from the `ncu --set full` captures of an evidence run.  Usage: update_traffic.py DIR PREFIX
(DIR/prof_cfg3.ncu-rep etc.; PREFIX names the summary files written to profiles/, e.g. r2b)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
d, prefix = sys.argv[1], sys.argv[2]
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
tj = json.load(open(path))
for key, rep, summ in (("config3:32768", "prof_cfg3", "ncu_cfg3"), ("config2:8192", "prof_cfg2", "ncu_cfg2"),
                       ("config1:1048576", "prof_cfg1_1m", "ncu_cfg1_1m"), ("config4:16384", "prof_cfg4", "ncu_cfg4")):
    f = os.path.join(d, rep + ".ncu-rep")
    if not os.path.exists(f):
        continue
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = [r for r in out.splitlines() if r.strip()]
    import csv
    rd = list(csv.reader(rows))
    hdr, units, vals = rd[0], rd[1], rd[2]

    def val(name):
        i = hdr.index(name)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[i]]
        return int(round(float(vals[i].replace(",", "")) * scale))
    tj[key] = {"dram_read": val("dram__bytes_read.sum"), "dram_write": val("dram__bytes_write.sum"),
               "source": f"{prefix}_{summ}.txt"}
json.dump(tj, open(path, "w"), indent=1)
print(json.dumps(tj, indent=1))
