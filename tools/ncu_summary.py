"""One line per profiled launch of an ncu report (--set full): duration, DRAM
bytes, tensor/FP64 pipe activity, issue activity and the top stall reasons.

    python tools/ncu_summary.py gpurun_out/<tag>/prof.ncu-rep > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("lts__t_sector_hit_rate.pct", "l2_hit%"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts")]


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        vals = []
        for k, short in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals.append(f"{short}={r[i]}{units[i] if units[i] not in ('', 'inst') else ''}")
        st = []
        for i, h in enumerate(hdr):
            if "smsp__average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(r[i]), h.replace("smsp__average_warps_issue_stalled_", "")
                               .replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print(f"{name}: " + " ".join(vals))
        print("    stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main()
