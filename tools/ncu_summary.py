"""Key metrics of every kernel in an .ncu-rep (ncu --page details/raw csv)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Compute (SM) Throughput",
        "Memory Throughput", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size", "Waves Per SM",
        "Eligible Warps Per Scheduler", "Active Warps Per Scheduler", "No Eligible", "Block Limit Registers",
        "Static Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed.sum", "smsp__average_warp_latency_issue_stalled_barrier",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def run(rep):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    cur = None
    for r in rows[1:]:
        if r[ii] != cur:
            cur = r[ii]
            print(f"\n== [{r[ii]}] {r[ki][:100]}")
        if r[mi] in WANT:
            print(f"   {r[mi]:40s} {r[vi]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    for r in rows[2:]:
        print(f"\n   raw [{r[h.index('ID')]}]")
        for m in RAW:
            if m in h:
                print(f"   {m:70s} {r[h.index(m)]} {rows[1][h.index(m)]}")


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        run(rep)
