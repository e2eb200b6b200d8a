"""Brief per-kernel metrics + top stall reasons from an ncu report (development tool).
python tools/ncu_brief.py REPORT.ncu-rep"""
import csv, subprocess, sys
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__occupancy_limit_shared_mem',
        'launch__occupancy_limit_registers', 'launch__registers_per_thread', 'launch__grid_size', 'smsp__inst_executed.sum',
        'l1tex__throughput.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    print(r[hdr.index('Kernel Name')][:70])
    for w in want:
        if w in hdr:
            print('   %-62s %s' % (w, r[hdr.index(w)]))
    items = []
    for i, h in enumerate(hdr):
        if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued'):
            try:
                items.append((float(r[i]), h[len('smsp__pcsamp_warps_issue_stalled_'):]))
            except ValueError:
                pass
    tot = sum(v for v, _ in items) or 1
    items.sort(reverse=True)
    print('   stalls: ' + ', '.join('%s %.0f%%' % (h, 100 * v / tot) for v, h in items[:7]))
