"""Print selected raw metrics of every kernel in an .ncu-rep:
python tools/ncu_metrics.py report.ncu-rep [substring-of-metric ...]"""
import csv
import subprocess
import sys

DEFAULT = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
           "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "launch__registers_per_thread", "smsp__inst_executed.sum"]


def main():
    rep = sys.argv[1]
    want = sys.argv[2:] or DEFAULT
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")][:70]
        print(name)
        for w in want:
            for i, h in enumerate(hdr):
                if h.endswith(w) or (w in h and len(want) != len(DEFAULT)):
                    print(f"   {h[-70:]:70s} {r[i]:>14s} {units[i]}")
                    break


if __name__ == "__main__":
    main()
