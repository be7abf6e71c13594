"""Key counters per launch from an `ncu --page raw --csv` dump: duration, DRAM bytes, hit rates, occupancy, top stalls."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum", "smsp__inst_executed.sum"]
idx = {h: i for i, h in enumerate(hdr)}
units = rows[1]
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    print("----")
    for w in want:
        if w in idx:
            v = r[idx[w]]
            print(f"{w} = {v[:90]} {units[idx[w]]}")
    st = sorted(((float(r[idx[h]].replace(',', '') or 0), h.split('stalled_')[1].split('_per_')[0]) for h in stall), reverse=True)[:6]
    print("stalls:", ", ".join(f"{n} {v:.2f}" for v, n in st))
