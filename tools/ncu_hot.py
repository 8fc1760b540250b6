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

# stall-reason totals (all samples), overall and excluding the top-2 wait instructions
cols = [c for c in rows[0].keys() if c.startswith("stall_") and "Not Issued" not in c]
def agg(rs):
    t = collections.Counter()
    for r in rs:
        for c in cols:
            t[c] += int(r[c] or 0)
    s = sum(t.values()) or 1
    return ", ".join(f"{k[6:]} {v/s:.0%}" for k, v in t.most_common(10) if v)
print("stalls (all):", agg(rows))
if len(sys.argv) > 4:
    lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
    sel = [r for r in rows if lo <= int(r["Address"], 16) % (1 << 20) <= hi]
    n = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in sel)
    print(f"range {sys.argv[3]}-{sys.argv[4]}: {n} samples ({n/tot:.1%});", agg(sel))
