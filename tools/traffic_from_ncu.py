"""Build profiles/rN_traffic.json from an ncu CSV of the C4 bench command:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --kernel-name-base demangled -k regex:k_kron --csv \
      python bench.py --steps 1 --warmup 0 --quick > traffic.csv
  python tools/traffic_from_ncu.py traffic.csv profiles/rN_traffic.json profiles/rN_traffic_ncu.csv

Per degree p (template n = p+1) and mode (0 = APPLY, 1 = CHEBY_GL, 4 = CHEBY_GLT) the median DRAM
bytes per launch are recorded next to the algorithmic bytes (16 / 40 B per DoF).
"""
import csv
import json
import os
import re
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synthetic import c4_spec  # noqa: E402

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        break
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
idi = hdr.index("ID")
per = {}
for r in rows:
    m = re.search(r"k_kron4<(?:\(int\))?(\d), (?:\(int\))?(\d), (?:\(int\))?(\d)", r[ki])
    m6 = re.search(r"k_kron6<(?:\(int\))?(\d), (?:\(int\))?(\d)", r[ki])
    m3 = re.search(r"k_kron3c<(?:\(int\))?(\d), (?:\(int\))?(\d)", r[ki])
    if m3:
        nl, mode = map(int, m3.groups())
        n, kern = 3, "k_kron3c"
    elif m:
        n, nl, mode = map(int, m.groups())
        kern = "k_kron4"
    elif m6:
        n, mode = map(int, m6.groups())
        nl, kern = 2, "k_kron6"
    elif re.search(r"k_bchg[wp]?<", r[ki]):   # basis change: k_bchg<N, CPB, ..> / k_bchgw<N, NSLOT, ..>, 16 B/DoF
        mb = re.search(r"(k_bchg[wp]?)<(?:\(int\))?(\d)", r[ki])
        n, nl, mode, kern = int(mb.group(2)), 2, 9, mb.group(1)
    else:
        continue
    if nl != 2 or mode not in (0, 1, 4, 9):
        continue
    key = (n - 1, mode, kern)
    per.setdefault(key, {}).setdefault(r[idi], {})[r[mi]] = float(r[vi].replace(",", ""))
out = {"c4": {}}
src = sys.argv[3] if len(sys.argv) > 3 else sys.argv[1]
for (p, mode, kern), launches in sorted(per.items()):
    tot = [v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in launches.values()]
    name = kern if mode == 9 else f"{kern}<" + {0: "APPLY", 1: "CHEBY_GL", 4: "CHEBY_GLT"}[mode] + ">"
    ent = out["c4"].setdefault(name, {"per_launch_bytes": {}, "algorithmic_bytes": {}, "launches": {},
                                      "source": src})
    nd = c4_spec(p).n_dofs
    ent["per_launch_bytes"][str(p)] = statistics.median(tot)
    ent["algorithmic_bytes"][str(p)] = nd * (16.0 if mode in (0, 9) else 40.0)
    ent["launches"][str(p)] = len(tot)
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
