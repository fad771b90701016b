"""Key metrics of every kernel in an .ncu-rep (raw page) as a small table."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"## {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in d:
                print(f"   {k:<66} {d[k]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
