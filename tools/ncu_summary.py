"""Per-kernel table from an ncu --set full report (raw page):
    python tools/ncu_summary.py report.ncu-rep
duration, DRAM read/write bytes, SM / memory throughput, issue active, warps
active, tensor-pipe activity, registers -- the columns profiles/*.md quote."""
import csv
import io
import subprocess
import sys

COLS = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("launch__registers_per_thread", "regs")]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    idx = [(h.index(k), name) for k, name in COLS if k in h]
    print("| " + " | ".join(n for _, n in idx) + " |")
    print("|" + "---|" * len(idx))
    for r in rows[2:]:
        vals = []
        for i, name in idx:
            v = r[i]
            if name == "kernel":
                v = v.split("(")[0][:48]
            elif name == "us":
                u = units[i]
                x = float(v.replace(",", ""))
                v = "%.1f" % (x / 1000 if u in ("nsecond", "ns") else x * 1000 if u == "msecond" else x)
            elif name.startswith("dram"):
                u = units[i]
                x = float(v.replace(",", ""))
                mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                v = "%.2f MB" % (x * mult / 1e6)
            vals.append(v)
        print("| " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
