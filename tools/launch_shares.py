"""Per-kernel launch count / mean / share from an ncu --metrics gpu__time_duration.sum CSV.
usage: python tools/launch_shares.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))
        if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = collections.defaultdict(list)
for r in rows:
    name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("spx::<unnamed>::", "").replace("unnamed>::", "")
    v = float(r["Metric Value"])
    agg[name].append(v * (1e-3 if r["Metric Unit"] == "ns" else 1.0))
tot = sum(sum(v) for v in agg.values())
print("| kernel | launches | avg us | share |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v)/tot:.1%} |")
print(f"| total | {sum(len(v) for v in agg.values())} | {tot/1e3:.2f} ms | |")
