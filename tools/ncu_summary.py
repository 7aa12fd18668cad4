"""Summarise key metrics of an ncu report (one line per kernel launch)."""
import csv, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc_active%"),
    ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed", "mma_ops%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex%"),
    ("l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed", "bank_rd%"),
    ("l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed", "bank_wr%"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.sum.pct_of_peak_sustained_elapsed", "l1->xbar req%"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "xbar->l1 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts%"),
    ("lts__t_sector_hit_rate.pct", "l2 hit%"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("smsp__issue_inst0.avg.pct_of_peak_sustained_active", "issue idle%"),
    ("lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "l2 tag (tex)%"),
    ("lts__t_sectors_srcunit_tex.max.pct_of_peak_sustained_elapsed", "l2 tag max%"),
    ("lts__t_sectors_srcunit_ltcfabric.avg.pct_of_peak_sustained_elapsed", "l2 fabric%"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "tc smem rd%"),
    ("derived__lts__lts2xbar_bytes.sum.per_second", "l2->xbar B/s"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(r[hdr.index("Kernel Name")][:90])
        for k, name in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {name:16s} {r[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
