"""Per-kernel ncu roofline fractions from one launch list with DRAM / tensor-pipe metrics.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed \
        --cache-control all --clock-control none --csv --log-file X.csv python bench.py ...
    python scripts/kernel_rooflines.py X.csv profiles/rNN_kernel_rooflines.json "<command>"

Roofline per kernel class (MEASURED_PEAKS.json): tensor-bound kernels (tcgen05 GEMM, attention)
report the tensor-pipe utilisation ncu measures (bf16 UTCHMMA ops as % of peak); HBM-bound kernels
report achieved DRAM GB/s (read + write bytes / duration, cold cache) over the measured copy
bandwidth; the scheduler kernels are latency-bound (time only).  ncu serialises kernels and flushes
caches, so these are per-kernel ceilings, not shares of the overlapped step.
"""

import csv
import io
import json
import sys
from pathlib import Path

TENSOR = ("gemm", "attn_fwd_kernel", "attn_fwd_dec_kernel", "attn_fwd_pp_kernel", "attn_bwd_kernel")
LATENCY = ("sample_times", "partition", "wavefront", "rank_metrics", "fanout_merge", "varlen_pack", "pack_tokens", "fp64_",
           "tiles_kernel", "positions")
UNIT = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
        "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}


def main(src, out, command):
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
    txt = open(src).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.find('"ID"'):])))
    launches = {}
    for r in rows:
        k = launches.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0]})
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        k[r["Metric Name"]] = v
    agg = {}
    for k in launches.values():
        name = k["name"]
        if not ("mb::" in name or "transpose" in name or "maestro" in name):
            continue  # torch's own fills/copies (plumbing) are listed separately by launch_list.py
        a = agg.setdefault(name, {"kernel": name, "launches": 0, "time_s": 0.0, "dram_bytes": 0.0, "tensor_pct_x_t": 0.0})
        t = k.get("gpu__time_duration.sum", 0.0)
        a["launches"] += 1
        a["time_s"] += t
        a["dram_bytes"] += k.get("dram__bytes_read.sum", 0.0) + k.get("dram__bytes_write.sum", 0.0)
        a["tensor_pct_x_t"] += t * k.get(
            "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", 0.0)
    table = []
    for a in sorted(agg.values(), key=lambda x: -x["time_s"]):
        n, t = a["kernel"], a["time_s"]
        rec = {"kernel": n, "launches": a["launches"], "total_us": t * 1e6, "avg_us": t * 1e6 / a["launches"]}
        gbs = a["dram_bytes"] / t / 1e9 if t > 0 else 0.0
        if any(x in n for x in TENSOR):
            pct = a["tensor_pct_x_t"] / t if t > 0 else 0.0
            rec.update(bound="tensor", tensor_pipe_pct=pct, roofline_frac=pct / 100.0, dram_GBps=gbs,
                       peak="bf16 tensor pipe (ncu % of peak sustained elapsed)")
        elif any(x in n for x in LATENCY):
            rec.update(bound="latency", roofline_frac=None, dram_GBps=gbs,
                       peak="latency-bound scheduler / planning kernel (time only)")
        else:
            rec.update(bound="hbm", dram_GBps=gbs, roofline_frac=gbs / peaks["hbm_gbs"],
                       peak=f"measured HBM copy bandwidth {peaks['hbm_gbs']} GB/s")
        table.append(rec)
    Path(out).write_text(json.dumps({"source": command, "kernels": table}, indent=1))
    for r in table:
        f = r["roofline_frac"]
        print(f"{r['kernel'][:60]:60s} {r['bound']:7s} {r['launches']:5d} {r['avg_us']:9.1f} us  "
              f"{'' if f is None else f'{100 * f:5.1f}%'}  {r['dram_GBps']:7.0f} GB/s")


if __name__ == "__main__":
    main(*sys.argv[1:])
