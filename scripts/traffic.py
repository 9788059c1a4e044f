"""DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
d = 3 spread / gather kernels from ncu --set full captures (--cache-control
all: each launch starts from a flushed L2, so this is the kernel's cold
footprint). Usage: traffic.py cfg2=gpurun_out/prof_cfg2.ncu-rep ... >
profiles/traffic.json"""
import csv
import json
import subprocess
import sys

STAGE = {"spread3c_s8": "spread_d3", "spread3_s8": "spread_d3", "gather3c_s8": "gather_d3",
         "gather3_s8": "gather_d3", "spread2_s8": "spread_d2", "gather2_s8": "gather_d2",
         "spread3_f32": "spread_d3", "gather3_f32": "gather_d3",
         "spread3_t32": "spread_d3", "gather3_t32": "gather_d3"}


def unit_bytes(val, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(val) * mult.get(unit, 1)


out = {}
for arg in sys.argv[1:]:
    cfg, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        key = next((v for k, v in STAGE.items() if k + "_kernel" in name), None)
        if key is None:
            continue
        b = sum(unit_bytes(r[hdr.index(m)], units[hdr.index(m)]) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        res.setdefault(key, b)
    out[cfg] = res
json.dump(out, sys.stdout, indent=1)
print()
