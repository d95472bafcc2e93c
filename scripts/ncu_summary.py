"""Summarise an ncu --set full report (.ncu-rep) into a small JSON for profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_gemm.ncu-rep profiles/r01_gemm_ncu.json
"""

import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed":
        "tensor_utchmma_bf16_pct_peak",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_mem_cycles_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "second": 1.0, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6}


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for i, h in enumerate(hdr):
            if h in KEYS:
                v = r[i].replace(",", "")
                try:
                    k[KEYS[h]] = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    k[KEYS[h]] = v
        if "dram_read" in k and "dram_write" in k:
            k["dram_traffic_bytes"] = k["dram_read"] + k["dram_write"]
        kernels.append(k)
    json.dump({"report": rep, "kernels": kernels}, open(out, "w"), indent=1)
    for k in kernels:
        print(json.dumps(k))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
