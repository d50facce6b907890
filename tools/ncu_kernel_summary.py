"""One-line-per-kernel summary of an ncu report: time, regs, occupancy, IPC, smem wavefronts and
bank conflicts, DRAM/L2 bytes, top stall reasons.  Usage: python tools/ncu_kernel_summary.py rep"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = {"gpu__time_duration.sum": "us", "launch__registers_per_thread": "regs", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
        "sm__inst_executed.avg.per_cycle_active": "ipc", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wf", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "conflicts",
        "dram__bytes_read.sum": "dramR", "dram__bytes_write.sum": "dramW", "lts__t_bytes.sum": "l2B", "smsp__inst_executed.sum": "winst"}
cols = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio")]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    name = name[:name.index("(")] if "(" in name else name
    vals = " ".join(f"{v}={r[hdr.index(k)]}" for k, v in want.items() if k in hdr)
    st = sorted([(hdr[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(r[i] or 0)) for i in cols], key=lambda t: -t[1])
    print(name)
    print("   ", vals)
    print("    stalls:", " ".join(f"{a}={b:.2f}" for a, b in st[:6]))
