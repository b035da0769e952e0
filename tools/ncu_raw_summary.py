"""Key raw metrics per kernel of an ncu report.  python tools/ncu_raw_summary.py rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:70])
    print("   " + "  ".join(f"{w.split('.')[0].split('__')[-1]}={r[h.index(w)]}{u[h.index(w)]}"
                            for w in want if w in h))
