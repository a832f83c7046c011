"""Summarise `ncu --page raw --csv` exports (one row per captured kernel) into the
metrics the bench's roofline cites: duration, DRAM bytes, tensor-pipe and
throughput percentages.  usage: ncu_raw_summary.py out.csv raw1.csv [raw2.csv ...]"""
import csv
import os
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__cycles_elapsed.avg.per_second"]

w = csv.writer(open(sys.argv[1], "w"))
w.writerow(["capture", "kernel", "metric", "unit", "value"])
for path in sys.argv[2:]:
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        continue
    h, u = rows[0], rows[1]
    cap = os.path.basename(path).replace("_raw.csv", "")
    for v in rows[2:]:
        name = v[h.index("Kernel Name")][:90] if "Kernel Name" in h else "?"
        for m in WANT:
            if m in h:
                i = h.index(m)
                w.writerow([cap, name, m, u[i], v[i]])
