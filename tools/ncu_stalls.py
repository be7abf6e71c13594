"""Summarises an .ncu-rep (read here, no GPU): per launch the duration, DRAM bytes, occupancy and the top stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__grid_size', 'launch__registers_per_thread',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'smsp__inst_executed.sum']
for r in rows[2:]:
    for k in want:
        if k in hdr:
            print(k, '=', r[hdr.index(k)][:70], rows[1][hdr.index(k)])
    st = [(float(r[i]), h) for i, h in enumerate(hdr)
          if 'issue_stalled' in h and h.endswith('per_issue_active.ratio') and r[i]]
    for v, h in sorted(st, reverse=True)[:8]:
        print('   %6.2f %s' % (v, h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
    print()
