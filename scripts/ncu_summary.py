"""Key per-kernel metrics from an ncu --set full report (read here, no GPU needed).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/<name>.txt
"""
import csv
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "inst"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {k: hdr.index(k) for k, _ in WANT if k in hdr}
    kcol = hdr.index("Kernel Name")
    print(f"# ncu --set full summary of {path}")
    print("# kernel | " + " | ".join(f"{short} [{units[idx[k]]}]" for k, short in WANT if k in idx))
    for r in data:
        name = r[kcol].split("(")[0].replace("void ", "")
        print(name + " | " + " | ".join(r[idx[k]] for k, _ in WANT if k in idx))


if __name__ == "__main__":
    main(sys.argv[1])
