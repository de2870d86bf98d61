"""One line per profiled launch from an ncu report (raw page):
kernel, time, DRAM bytes, DRAM %, SM %, FMA %, regs, occupancy, issue busy."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
M = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm%": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "fma%": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue%": "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "occ%": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smem_cfl": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
idx = {k: (hdr.index(v) if v in hdr else None) for k, v in M.items()}
ki = hdr.index("Kernel Name")
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "")[:44]
    vals = []
    for k, i in idx.items():
        if i is None:
            vals.append(f"{k}=NA")
            continue
        u = units[i]
        v = r[i]
        try:
            x = float(v.replace(",", ""))
            if k == "time_us" and u == "nsecond":
                x /= 1e3
            if k == "time_us" and u == "msecond":
                x *= 1e3
            if k.startswith("dram_") and u == "Kbyte":
                x /= 1e3
            if k.startswith("dram_") and u == "Gbyte":
                x *= 1e3
            if k.startswith("dram_") and u == "byte":
                x /= 1e6
            vals.append(f"{k}={x:.4g}")
        except ValueError:
            vals.append(f"{k}={v}")
    print(f"{name:44s} " + " ".join(vals))
