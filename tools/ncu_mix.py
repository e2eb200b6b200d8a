"""Instruction mix (warp-level executed instructions per element) from an ncu source page."""
import collections, csv, subprocess, sys
rep, elems = sys.argv[1], float(sys.argv[2])
kid = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kid:
    cmd += ["--launch-skip", kid, "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")
mix = collections.Counter()
for r in rows[1:]:
    try:
        v = float(r[ie])
    except Exception:
        continue
    op = r[src].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    mix[o.split(".")[0]] += v
tot = sum(mix.values())
print(f"total warp-instr/elem x32 = {tot*32/elems:.1f}")
for o, v in mix.most_common(25):
    print(f"{v*32/elems:7.2f}  {o}")
