"""Summarise an ncu --csv launch list: per-kernel time / DRAM bytes (sbnet kernels + dense)."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(int(r[0]), {"kernel": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return list(launches.values())


def short(name):
    for key in ("unit_tc_kernel", "unit_simt_kernel", "rim_kernel", "reduce_mask_kernel",
                "sparse_conv_tc_kernel", "sparse_conv_simt_kernel", "gather_rows", "scatter_rows",
                "unit_tc_pack", "downsample", "in_bounds"):
        if key in name:
            return key
    return name.split("(")[0][:60]


if __name__ == "__main__":
    ls = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    print(f"{'#':>4} {'kernel':<44} {'time_us':>9} {'dram_rd_MB':>10} {'dram_wr_MB':>10}")
    for i, d in enumerate(ls):
        if i < skip:
            continue
        print(f"{i:>4} {short(d['kernel']):<44} {d.get('gpu__time_duration.sum', 0) / 1e3:9.2f} "
              f"{d.get('dram__bytes_read.sum', 0) / 1e6:10.3f} {d.get('dram__bytes_write.sum', 0) / 1e6:10.3f}")
