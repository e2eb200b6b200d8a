"""Top SASS lines for one stall reason from an ncu source page (dev tool).
python tools/ncu_stall.py REPORT.ncu-rep stall_long_sb [kernel-index] [top]"""
import csv, subprocess, sys
rep, col = sys.argv[1], sys.argv[2]
kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
# the page holds one block per kernel, each starting with a "Kernel Name" line
blocks, cur = [], None
for line in out:
    if line.startswith('"Kernel Name"'):
        cur = [line]
        blocks.append(cur)
    elif cur is not None:
        cur.append(line)
b = blocks[kidx]
print(b[0][:150])
rows = list(csv.reader(b[1:]))
hdr = rows[0]
ci, si = hdr.index(col), hdr.index("Source")
items, tot = [], 0
for r in rows[1:]:
    try:
        v = int(r[ci])
    except Exception:
        continue
    tot += v
    items.append((v, r[0][-5:], r[si].strip()))
items.sort(reverse=True)
print(col, "total", tot)
for v, a, s in items[:top]:
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}% {a} {s[:100]}")
