"""Summarise an ncu report: key SOL/occupancy metrics and the SASS opcode mix."""
import csv, io, subprocess, sys
from collections import Counter

rep = sys.argv[1]
KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Issued Instructions",
        "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy", "Cluster Size", "Grid Size",
        "Waves Per SM", "Max Active Clusters", "Dynamic Shared Memory Per Block", "L2 Hit Rate", "L1/TEX Hit Rate"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in KEYS:
        print("%-40s %-14s %s" % (d["Metric Name"], d.get("Metric Unit", ""), d.get("Metric Value")))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h, vals = rr[0], rr[2]
    for k, v in zip(h, vals):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                 "sm__inst_executed.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
                 "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
                 "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
                 "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"):
            print("%-60s %s" % (k, v))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
if len(rows) > 2:
    hdr = rows[1]
    ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)"); sc = hdr.index("Source")
    ops, st = Counter(), Counter()
    tot = tots = 0
    for r in rows[2:]:
        try:
            n = int(r[ie] or 0); s = int(r[ss] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[sc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        ops[op] += n; st[op] += s; tot += n; tots += s
    print("SASS opcode mix (warp-level executed, stall-sample share):")
    for op, n in ops.most_common(18):
        print("  %-8s %6.2f%%  stall %6.2f%%" % (op, 100.0 * n / tot, 100.0 * st[op] / max(tots, 1)))
