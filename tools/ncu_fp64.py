"""Per-launch evidence of one ncu --set full capture of the chain kernel, as JSON for bench.py:
DRAM bytes, duration, issue-slot utilisation, and the EXECUTED fp64 work counted from the SASS
page (predicated-on thread instructions: DADD / DMUL = 1 flop, DFMA = 2).
usage: ncu_fp64.py <report.ncu-rep> <source label> > profiles/anneal_ncu.json"""
import csv, io, json, subprocess, sys

rep, label = sys.argv[1], sys.argv[2]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h, units, v = raw[0], raw[1], raw[2]
m = {k: (u, x) for k, u, x in zip(h, units, v)}


def val(name, scale=None):
    u, x = m[name]
    x = float(x.replace(",", ""))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}
    return x * mult.get(u, 1)


src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                                                  "--print-source=sass"], capture_output=True, text=True).stdout)))
hdr = src[1]
ci, cp = hdr.index("Source"), hdr.index("Predicated-On Thread Instructions Executed")
flops = {"DADD": 0, "DMUL": 0, "DFMA": 0}
for r in src[2:]:
    toks = r[ci].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
    if op in flops:
        flops[op] += int(float(r[cp] or 0))
dur = val("gpu__time_duration.sum")
executed = flops["DADD"] + flops["DMUL"] + 2 * flops["DFMA"]
out = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "anneal_kernel", "source": label,
       "duration_s": dur, "dram_bytes_read": val("dram__bytes_read.sum"), "dram_bytes_write": val("dram__bytes_write.sum"),
       "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
       "issue_active_pct_elapsed": val("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
       "warp_instructions": val("smsp__inst_executed.sum"),
       "fp64_thread_ops": flops, "executed_fp64_flops": executed, "executed_fp64_tflops": executed / dur / 1e12}
print(json.dumps(out, indent=1))
