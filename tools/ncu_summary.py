"""Key raw metrics of an ncu --set full report, as the table profiles/ summaries use.
Usage: python tools/ncu_summary.py report.ncu-rep [report2 ...]"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_branch_targets_threads_divergent.sum", "smsp__sass_branch_targets.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for k in ["Kernel Name"] + WANT:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
        res.append(d)
    return res


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        for d in summary(rep):
            print(f"== {rep}: {d.get('Kernel Name', ('?',))[0][:80]}")
            for k in WANT:
                if k in d:
                    print(f"   {k:70s} {d[k][0]:>18s} {d[k][1]}")
