"""Summarise an ncu report (--page raw --csv) into a few lines per kernel launch.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--grep metric-substring ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_cycles_active", "tensor%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def main():
    rep = sys.argv[1]
    extra = sys.argv[3:] if len(sys.argv) > 2 and sys.argv[2] == "--grep" else []
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")[:60]
        parts = []
        for key, short in KEYS:
            for h in hdr:
                if h.startswith(key) and ("pct" not in key or "pct" in h):
                    parts.append(f"{short}={d[h]}{u.get(h, '')}")
                    break
        for g in extra:
            for h in hdr:
                if g in h:
                    parts.append(f"{h}={d[h]}{u.get(h, '')}")
        print(name, " ".join(parts))


if __name__ == "__main__":
    main()
