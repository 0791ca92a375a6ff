"""Record the DRAM traffic of one ncu --set full capture in profiles/ncu_traffic.json
(read by bench.py for roofline.traffic).  Usage:
python tools/ncu_traffic.py <raw.csv> <config> <d|default> <kernel> <variant>"""
import csv
import json
import os
import sys

raw, config, d, kernel, variant = sys.argv[1:6]
rows = [r for r in csv.reader(open(raw)) if r and not r[0].startswith("==")]
vals = dict(zip(rows[0], rows[2]))
units = dict(zip(rows[0], rows[1]))


def to_bytes(k):
    v = float(vals[k].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(units.get(k, "byte"), 1)


rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
t = json.load(open(path)) if os.path.exists(path) else {}
t[f"{config}|{d}|{kernel}|{variant}"] = {"dram_bytes": rd + wr, "read": rd, "write": wr,
                                         "duration": vals.get("gpu__time_duration.sum"),
                                         "source": (os.environ.get("TAG", "") + " " + os.path.basename(raw)).strip()}
json.dump(t, open(path, "w"), indent=1, sort_keys=True)
print(f"{config}|{d}|{kernel}|{variant}: {rd + wr:.4g} B")
