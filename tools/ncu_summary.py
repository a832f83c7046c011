"""Summarise one-kernel ncu reports into a small CSV (for profiles/):
python tools/ncu_summary.py out.csv name1=rep1.ncu-rep [name2=rep2.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]

out = open(sys.argv[1], "w")
w = csv.writer(out)
w.writerow(["kernel", "metric", "unit", "value"])
for arg in sys.argv[2:]:
    name, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        w.writerow([name, "error", "", "no data"])
        continue
    h, u, v = rows[0], rows[1], rows[2]
    w.writerow([name, "Kernel Name", "", v[h.index("Kernel Name")] if "Kernel Name" in h else ""])
    for i, n in enumerate(h):
        if n in WANT:
            w.writerow([name, n, u[i], v[i]])
out.close()
print(open(sys.argv[1]).read())
