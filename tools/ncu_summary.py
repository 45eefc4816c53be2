"""Summarise an .ncu-rep: key throughput metrics, stall reasons, DRAM bytes (used for profiles/)."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        print("kernel:", d.get("Kernel Name", "")[:90])
        for k in KEYS:
            if k in d:
                print(f"  {k:75s} {d[k]} {u.get(k, '')}")
        st = sorted(((k, float(v or 0)) for k, v in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")),
                    key=lambda kv: -kv[1])
        tot = sum(v for _, v in st) or 1
        print("  stall samples (share):", ", ".join(f"{k.split('stalled_')[1]} {v / tot:.0%}" for k, v in st[:8]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
