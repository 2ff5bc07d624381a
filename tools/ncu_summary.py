"""Summarise an .ncu-rep (raw page) into the metrics we track per kernel launch."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "dur"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64inst%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1%"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "ld_sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "ld_reqs"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum", "lsu_wf"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "inst"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: k for k, h in enumerate(hdr)}
    name_col = idx.get("Kernel Name")
    for r in rows[2:]:
        name = r[name_col][:60] if name_col is not None else "?"
        parts = []
        for key, short in KEYS:
            if key in idx:
                parts.append(f"{short}={r[idx[key]]}{units[idx[key]] if short in ('dur', 'dram_rd', 'dram_wr') else ''}")
        print(name)
        print("   " + "  ".join(parts))
        stalls = []
        for h, k in idx.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[k]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        if stalls:
            stalls.sort(reverse=True)
            print("   stalls/issue: " + "  ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
