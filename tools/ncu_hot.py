"""Summarise an ncu source-page CSV (SASS view): top instructions by warp-stall samples,
plus per-opcode totals.  usage: python tools/ncu_hot.py <rep.ncu-rep> [top]"""
import csv
import collections
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"total samples {tot}")
ops = collections.Counter()
for r in rows:
    op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
    if op.startswith("@"):
        op = r["Source"].strip().split()[1]
    ops[op.split(".")[0]] += int(r["Warp Stall Sampling (All Samples)"] or 0)
print("by opcode:", ", ".join(f"{k} {v/tot:.1%}" for k, v in ops.most_common(15)))
rows.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))
for r in rows[:top]:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s/tot:6.1%} {r['Address'][-5:]} {r['Source'].strip()[:90]}")
