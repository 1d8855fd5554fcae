"""Hot instructions of one kernel in an ncu report (source page, SASS): top stall samples with
their stall reasons, plus instruction-class totals. python tools/ncu_hot.py <rep> <kernel regex> [N]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[start:])))
        if (r.get("Warp Stall Sampling (All Samples)") or "0").isdigit()]
stall_cols = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
print(f"{len(rows)} SASS instructions, {tot} stall samples")
cls = Counter()
ops = Counter()
for r in rows:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    ops[op.split(".")[0]] += int(r["Instructions Executed"] or 0)
    for k in stall_cols:
        cls[k] += int(r[k] or 0)
print("stalls:", ", ".join(f"{k[6:]} {100 * v / max(tot, 1):.0f}%" for k, v in cls.most_common(8)))
print("executed warp-instructions by opcode:", ", ".join(f"{k} {v}" for k, v in ops.most_common(16)))
hot = sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:N]
for r in hot:
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    top = sorted(((int(r[k] or 0), k[6:]) for k in stall_cols), reverse=True)[:2]
    print(f"{100 * s / max(tot, 1):5.1f}%  {r['Source'].strip()[:70]:70s} {top[0][1]} {top[1][1]}")
