"""Stall samples of an `ncu --page source --csv --print-source sass` export, grouped by the
barrier-delimited segments of the kernel and by top instructions (usage: ncu_segments.py CSV)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
si = hdr.index("Warp Stall Sampling (All Samples)")
reasons = ["stall_barrier", "stall_long_sb", "stall_short_sb", "stall_mio", "stall_wait", "stall_math",
           "stall_not_selected", "stall_selected", "stall_branch_resolving", "stall_dispatch", "stall_drain",
           "stall_lg", "stall_no_inst"]
idx = [hdr.index(x) for x in reasons]
tot = sum(int(r[si]) for r in data)
print("total samples", tot, {x[6:]: sum(int(r[i]) for r in data) for x, i in zip(reasons, idx)})
seg, segs = 0, {}
for r in data:
    if "BAR.SYNC" in r[1]:
        seg += 1
    s = segs.setdefault(seg, [0, 0, {}])
    s[0] += int(r[si])
    s[1] += 1
    for x, i in zip(reasons, idx):
        s[2][x[6:]] = s[2].get(x[6:], 0) + int(r[i])
for k, v in segs.items():
    print("segment", k, v[0], f"{100 * v[0] / tot:.1f}%", v[1], "instr",
          {a: b for a, b in v[2].items() if b > tot * 0.01})
top = sorted(range(len(data)), key=lambda k: -int(data[k][si]))[:15]
for k in sorted(top):
    r = data[k]
    print(k, r[si], r[1].strip()[:60], {x[6:]: int(r[i]) for x, i in zip(reasons, idx) if int(r[i]) > tot * 0.003})
