"""Summarise an ncu report (--page raw --csv): one line per captured kernel launch."""
import csv, io, subprocess, sys

TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
WANT = [("gpu__time_duration.sum", "dur_us", 1), ("dram__bytes_read.sum", "dram_rd_MB", 1),
        ("dram__bytes_write.sum", "dram_wr_MB", 1),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%", 1),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%", 1),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%", 1),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%", 1),
        ("launch__grid_size", "grid", 1), ("launch__block_size", "block", 1),
        ("launch__registers_per_thread", "regs", 1)]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    ki = h.index("Kernel Name")
    print("| kernel | " + " | ".join(w[1] for w in WANT) + " |")
    print("|---" * (len(WANT) + 1) + "|")
    for r in data:
        vals = []
        for name, short, sc in WANT:
            if name in h:
                v = r[h.index(name)].replace(",", "")
                u = units[h.index(name)]
                try:
                    x = float(v)
                    if short == "dur_us":
                        x *= TIME.get(u, 1.0)
                    if short.endswith("_MB"):
                        x *= BYTES.get(u, 1.0)
                    vals.append(f"{x:.1f}")
                except ValueError:
                    vals.append(v)
            else:
                vals.append("-")
        print(f"| {r[ki].split('(')[0][-40:]} | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
