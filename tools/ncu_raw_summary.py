"""Per-kernel summary of an ncu --set full report (ncu -i <rep> --page raw --csv): duration, DRAM bytes, pipe
utilisation, occupancy.  Usage: python tools/ncu_raw_summary.py report.ncu-rep [...]   Not product code."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
        ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma_%active"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_%active"),
        ("sm__cycles_active.avg", "cyc_active"), ("gpc__cycles_elapsed.max", "cyc_elapsed"),
        ("lts__t_sector_hit_rate.pct", "l2_hit_%"), ("launch__registers_per_thread", "regs"),
        ("launch__grid_size", "grid"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_%")]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(rep, "no rows")
        continue
    h, u = rows[0], rows[1]
    print(f"== {rep}")
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "?")[:70]
        vals = []
        for k, short in KEYS:
            if k in d and d[k]:
                vals.append(f"{short}={d[k]}{u[h.index(k)] if u[h.index(k)] not in ('', '%') else ''}")
        print(f"  {name}: " + ", ".join(vals))
