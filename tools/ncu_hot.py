"""Summarise an ncu source page: top SASS lines by stall samples (dev tool)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
tot = 0
items = []
for r in rows[1:]:
    try:
        v = int(r[si])
    except Exception:
        continue
    tot += v
    items.append((v, r[0][-5:], r[src].strip()))
items.sort(reverse=True)
print("total samples", tot)
for v, a, s in items[:top]:
    print(f"{v:6d} {100*v/tot:5.1f}% {a} {s[:90]}")
