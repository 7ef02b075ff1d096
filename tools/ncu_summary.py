"""Summarises an ncu report (--page raw --csv): duration, DRAM traffic, pipe
use, issue, occupancy and the warp-stall breakdown of each kernel.
usage: python tools/ncu_summary.py REPORT.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu inst %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu inst %"),
]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(rep, "no data")
            continue
        h, units = rows[0], rows[1]
        for row in rows[2:]:
            d = dict(zip(h, row))
            u = dict(zip(h, units))
            print(f"== {rep}: {d.get('Kernel Name', '?')[:90]}")
            for k, name in KEYS:
                if k in d:
                    print(f"   {name:28s} {d[k]} {u.get(k, '')}")
            st = []
            for k, v in d.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                        "_per_issue_active.ratio"):
                    try:
                        st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len(
                            "_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            print("   stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in st[:10]))


if __name__ == "__main__":
    main()
