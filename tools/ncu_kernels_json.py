"""Per-kernel numbers from ncu --set full reports -> JSON (read by bench.py for roofline.traffic).

usage: python tools/ncu_kernels_json.py OUT.json REPORT.ncu-rep [REPORT ...]
"""
import csv
import json
import subprocess
import sys

KEYS = {"time_ms": ("gpu__time_duration.sum", {"ms": 1, "us": 1e-3, "ns": 1e-6}),
        "dram_read": ("dram__bytes_read.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
        "dram_write": ("dram__bytes_write.sum", {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}),
        "pcie_read_per_s": ("pcie__read_bytes.sum.per_second", {"byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6,
                                                               "Gbyte/s": 1e9}),
        "pcie_write_per_s": ("pcie__write_bytes.sum.per_second", {"byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6,
                                                                 "Gbyte/s": 1e9})}

out = {}
for rep in sys.argv[2:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units = r[0], r[1]
    for row in r[2:]:
        name = row[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        d = {"report": rep.split("/")[-1]}
        for k, (m, scale) in KEYS.items():
            if m in h:
                i = h.index(m)
                d[k] = float(row[i].replace(",", "")) * scale.get(units[i], 1)
        d["time_ms"] = d.get("time_ms", 0)
        d["dram_bytes"] = d.get("dram_read", 0) + d.get("dram_write", 0)
        d["pcie_read_bytes"] = d.get("pcie_read_per_s", 0) * d["time_ms"] / 1e3
        d["pcie_write_bytes"] = d.get("pcie_write_per_s", 0) * d["time_ms"] / 1e3
        out[name] = d
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
