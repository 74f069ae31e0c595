"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum --csv` launch list (usage:
launch_share.py LAUNCHES.csv).  Shares, not rates: ncu serialises launches and runs them cold.
Also the share within one timed bench step (per degree: 5 Chebyshev launches, 1 matvec, 1 basis
change) from the mean launch time of each (kernel, n, mode)."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0] != "ID"]
tot = collections.Counter()
cnt = collections.Counter()
for r in rows:
    name, t = r[4], float(r[14].replace(",", ""))
    m = re.search(r"(k_kron4)<(\d+), (\d+), (\d+)", name)
    m3 = re.search(r"(k_kron3c)<(\d+), (\d+)>", name)
    m6 = re.search(r"(k_kron6)<(\d+), (\d+)>", name)
    mb = re.search(r"(k_bchg[4wp]?)<(?:\(int\))?(\d+)", name)
    if mb:
        key = f"{mb.group(1)}<n={mb.group(2)}>"
    elif m:
        key = f"{m.group(1)}<n={m.group(2)},mode={m.group(4)}>"
    elif m3:
        key = f"k_kron3c<n=3,mode={m3.group(3)}>"
    elif m6:
        key = f"k_kron6<n={m6.group(2)},mode={m6.group(3)}>"
    else:
        key = re.sub(r"^void\s+", "", name).replace("<unnamed>", "").split("(")[0].split("<")[0].split("::")[-1]
    tot[key] += t
    cnt[key] += 1
T = sum(tot.values())
print(f"# total {T:.3g} (ncu time units), {sum(cnt.values())} launches")
for k, v in tot.most_common():
    print(f"{k:42s} {cnt[k]:5d} launches {100 * v / T:7.2f} %")
mean = {k: tot[k] / cnt[k] for k in tot}
step = collections.Counter()
glt_n = {re.search(r"n=(\d+)", k).group(1) for k in mean if "mode=4" in k}
for k, v in mean.items():
    if "mode=1" in k or "mode=4" in k:
        step["chebyshev"] += 5 * v
    elif "mode=0" in k:
        step["matvec"] += v
    elif k.startswith("k_bchg"):
        step["basis_change"] += v
        if re.search(r"n=(\d+)", k).group(1) in glt_n:   # the transformed-residual sweep's b~ pass
            step["chebyshev"] += v
S = sum(step.values())
print("# per timed step (per degree 5 Chebyshev launches (+ the b~ basis change where the step runs on the "
      "transformed residual), 1 matvec, 1 basis change; mean launch times):",
      ", ".join(f"{k} {100 * v / S:.1f} %" for k, v in step.most_common()))
