"""Summarise an ncu --set full report into profiles/ (markdown + traffic json).

python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX [--names "pass0 fft_pass<F=256,T=8>,..."] [--key "n=16777216|p=1"]
Writes OUT_PREFIX.md and merges per-launch DRAM bytes into profiles/ncu_traffic.json
under "<bench kernel name>|<key>" (what bench.py's roofline.traffic reads).
"""
import argparse, csv, json, os, subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("out")
ap.add_argument("--names", default="")
ap.add_argument("--key", default="n=16777216|p=1")
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
names = [n for n in a.names.split(";") if n]
def g(r, k):
    return r[hdr.index(k)] if k in hdr else ""
lines = [f"# ncu summary: {os.path.basename(a.rep)}", "",
         "| # | kernel | duration | DRAM read (MB) | DRAM write (MB) | DRAM % peak | issue % | warps % | regs | grid | top stalls |",
         "|---|---|---|---|---|---|---|---|---|---|---|"]
traffic_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
try:
    traffic = json.load(open(traffic_path))
except Exception:
    traffic = {}
for i, r in enumerate(rows[2:]):
    stalls = []
    for j, h in enumerate(hdr):
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                stalls.append((float(r[j]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in stalls) or 1
    top = ", ".join(f"{h} {100 * v / tot:.0f}%" for v, h in sorted(stalls, reverse=True)[:4])
    rd = float(g(r, "dram__bytes_read.sum") or 0)
    wr = float(g(r, "dram__bytes_write.sum") or 0)
    ur, uw = units[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_write.sum")]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    rd_mb, wr_mb = rd * scale.get(ur, 1), wr * scale.get(uw, 1)
    lines.append(f"| {i} | `{g(r, 'Kernel Name')[:70]}` | {g(r, 'gpu__time_duration.sum')} {units[hdr.index('gpu__time_duration.sum')]} | {rd_mb:.1f} | {wr_mb:.1f} | "
                 f"{float(g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or 0):.1f} | "
                 f"{float(g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                 f"{float(g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0):.1f} | "
                 f"{g(r, 'launch__registers_per_thread')} | {g(r, 'launch__grid_size')} | {top} |")
    if i < len(names):
        traffic[f"{names[i]}|{a.key}"] = int((rd_mb + wr_mb) * 1e6)
open(a.out + ".md", "w").write("\n".join(lines) + "\n")
json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
print("\n".join(lines))
