"""Hot SASS of one kernel from an ncu report: instructions executed and stall samples per
instruction, plus totals grouped by opcode (run here, no GPU needed).

  python tools/sass_hot.py <prof.ncu-rep> <kernel-regex> [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot_inst = sum(int(r["Instructions Executed"] or 0) for r in rows)
tot_samp = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
by_op = collections.Counter()
samp_op = collections.Counter()
for r in rows:
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    op = op.split(".")[0]
    by_op[op] += int(r["Instructions Executed"] or 0)
    samp_op[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
print(f"total warp instructions {tot_inst:,}  stall samples {tot_samp:,}")
print("opcode  inst%  samples%")
for op, n in by_op.most_common(25):
    print(f"{op:10s} {100*n/tot_inst:6.2f} {100*samp_op[op]/max(tot_samp,1):6.2f}")
print("\nhottest instructions (by executed count):")
rows_sorted = sorted(rows, key=lambda r: -int(r["Instructions Executed"] or 0))[:top]
keep = set(id(r) for r in rows_sorted)
for r in rows:
    if id(r) in keep:
        print(f'{r["Address"][-5:]} {int(r["Instructions Executed"]):>11,} {int(r["Warp Stall Sampling (All Samples)"] or 0):>7} {r["Source"].strip()}')
