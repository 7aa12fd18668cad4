"""ncu report -> JSON list of the key metrics per launch (profiles/r01/ncu_full_cfg3_metrics.json)
and the gate+up launch's DRAM bytes (profiles/traffic_gate_up.json).
    python tools/ncu_metrics_json.py REPORT.ncu-rep OUT.json [TRAFFIC.json]"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out, traffic=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    json.dump(res, open(out, "w"), indent=1)
    if traffic:
        gu = next(d for d in res if "spmm_tc_kernel<64, 2, 1, 2," in d["kernel"])
        def nbytes(v):
            num, unit = v.split()
            return float(num.replace(",", "")) * SCALE[unit]
        json.dump({"kernel": gu["kernel"],
                   "dram_bytes_per_launch": nbytes(gu["dram__bytes_read.sum"]) + nbytes(gu["dram__bytes_write.sum"]),
                   "source": "ncu --set full --clock-control none --import-source on -k regex:spmm_tc "
                             "-s 2 -c 2 python tools/prof_once.py (gate+up launch after warm-up); "
                             "profiles/r01/ncu_full_cfg3_metrics.json"},
                  open(traffic, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
