"""Per-source-line stall samples of one kernel from an ncu report (run here, no GPU needed).
  python tools/ncu_lines.py <rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
kx = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + (["--kernel-name", "regex:" + kx] if kx else []),
                     capture_output=True, text=True).stdout
rows = []
fname = ""
hdr = None
tot = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        samp = int(r[4])
        ins = int(r[7])
    except ValueError:
        continue
    tot += samp
    rows.append((samp, ins, f"{fname}:{r[0]}", r[1].strip()[:90]))
rows.sort(reverse=True)
print(f"total samples {tot}")
for s, i, loc, src in rows[:top]:
    print(f"{100 * s / max(tot, 1):5.1f}% {s:7d} {i:11d}  {loc:22s} {src}")
