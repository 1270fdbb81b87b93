"""DRAM traffic per kernel of one captured step (ncu --set full report, read here):
writes the GEMM bytes bench.py reports as roofline.traffic.

    python scripts/ncu_traffic.py gpurun_out/step_full.ncu-rep profiles/r1_gemm_traffic.json
"""
import csv
import json
import subprocess
import sys


def main(path, out_path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    k = hdr.index("Kernel Name")
    rd, wr, t = (hdr.index(m) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                        "gpu__time_duration.sum"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    kernels = []
    for r in data:
        kernels.append({
            "kernel": r[k].split("(")[0].replace("void ", ""),
            "dram_bytes": float(r[rd].replace(",", "")) * scale[units[rd]] +
                          float(r[wr].replace(",", "")) * scale[units[wr]],
            "us": float(r[t].replace(",", "")) * tscale[units[t]]})
    # the expert GEMMs (not the gate's tcgen05 GEMMs: fp32 epilogue with 128-wide N tiles)
    gemm = [x for x in kernels if "grouped_gemm" in x["kernel"] and ", 128, 3," not in x["kernel"]]
    out = {"source": path, "kernels": kernels,
           "gemm_dram_bytes_per_step": sum(x["dram_bytes"] for x in gemm),
           "gemm_launches": len(gemm)}
    json.dump(out, open(out_path, "w"), indent=1)
    print(json.dumps({"gemm_dram_bytes_per_step": out["gemm_dram_bytes_per_step"],
                      "gemm_launches": len(gemm)}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
