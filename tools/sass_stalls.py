"""Per-region stall-reason breakdown of one kernel (regions = runs of instructions with the same
execution count, i.e. basic blocks), from an ncu report's source page.
  python tools/sass_stalls.py <rep> <kernel-regex> [nregions]"""
import collections, csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
reasons = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
blocks, cur = [], None
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    if cur is None or cur["n"] != n:
        cur = {"n": n, "addr": r["Address"][-5:], "k": 0, "st": collections.Counter(), "ops": collections.Counter()}
        blocks.append(cur)
    cur["k"] += 1
    op = (r["Source"].split() or ["?"])
    cur["ops"][(op[1] if op[0].startswith("@") and len(op) > 1 else op[0]).split(".")[0]] += 1
    for k in reasons:
        cur["st"][k[6:]] += int(r[k] or 0)
tot = sum(sum(b["st"].values()) for b in blocks)
for b in sorted(blocks, key=lambda b: -sum(b["st"].values()))[:top]:
    s = sum(b["st"].values())
    print(f'{b["addr"]} exec {b["n"]:>10,} x{b["k"]:>3}  samples {100 * s / tot:5.1f}%  ops {dict(b["ops"].most_common(4))}')
    print("      ", ", ".join(f"{k} {100 * v / s:.0f}%" for k, v in b["st"].most_common(7) if v))
