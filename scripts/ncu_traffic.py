"""Summarise ncu --set full captures of the attention kernel into profiles/r02_ncu_traffic.json
(the DRAM bytes per launch bench.py reports as roofline.traffic) and a per-capture metric summary.

usage: python scripts/ncu_traffic.py gpurun_out/ncu_<workload>_<dtype>.ncu-rep ... [--tag NAME]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from ncu_summary import report  # noqa: E402


def _num(s):
    v, *u = s.split()
    v = float(v.replace(",", ""))
    unit = u[0] if u else ""
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    d = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for path in args:
        base = os.path.basename(path)[len("ncu_"):-len(".ncu-rep")]
        wl, dt = base.rsplit("_", 1)
        recs = [r for r in report(path) if "gna_attn" in r["kernel"]]
        if not recs:
            print("no attention kernel in", path)
            continue
        r = recs[-1]
        rd, wr = _num(r["dram__bytes_read.sum"]), _num(r["dram__bytes_write.sum"])
        d[f"{wl}:{dt}"] = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                           "source": f"ncu --set full, {os.path.basename(path)}", "metrics": r}
        print(wl, dt, f"DRAM {(rd + wr) / 1e9:.3f} GB per launch", r.get("gpu__time_duration.sum"))
    json.dump(d, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
