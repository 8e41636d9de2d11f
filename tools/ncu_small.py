"""Per-kernel duration and DRAM bytes from an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` log (averaged over launches of the same kernel).

    python tools/ncu_small.py gpurun_out/x.csv [hbm_GBps]
"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6549.1
    h = rows[0]
    iK, iM, iV, iI = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, name = collections.defaultdict(dict), {}
    for r in rows[1:]:
        per[r[iI]][r[iM]] = float(r[iV].replace(",", ""))
        name[r[iI]] = r[iK].split("(")[0].replace("void ", "").replace("lina::<unnamed>::", "")
    agg = collections.defaultdict(list)
    for i, m in per.items():
        agg[name[i]].append(m)
    for k, ms in agg.items():
        d = sum(m["gpu__time_duration.sum"] for m in ms) / len(ms)
        b = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in ms) / len(ms)
        print(f"{k:48s} n={len(ms):2d} {d / 1e3:8.1f} us  dram {b / 1e6:8.1f} MB  {b / d:6.0f} GB/s  ({b / d / peak:.2f} of {peak:.0f})")


if __name__ == "__main__":
    main()
