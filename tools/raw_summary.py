"""Summarise an ncu raw-page CSV (ncu -i rep --page raw --csv > x_raw.csv):
one line per profiled launch with time, DRAM bytes, throughput and pipe use."""
import csv
import sys

M = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm%": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "fma%": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu%": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "issue%": "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "l2hit%": "lts__t_sector_hit_rate.pct",
    "smem_cfl": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    idx = {k: (hdr.index(v) if v in hdr else None) for k, v in M.items()}
    ki = hdr.index("Kernel Name")
    print("kernel\t" + "\t".join(M))
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "")
        vals = []
        for k, i in idx.items():
            if i is None or r[i] == "":
                vals.append("NA")
                continue
            v = float(r[i].replace(",", ""))
            u = units[i]
            if k == "time_us":
                v = v / 1000.0 if u in ("nsecond", "ns") else v * (1000.0 if u in ("msecond", "ms") else 1.0)
            if k.endswith("_MB"):
                scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1e-6)
                v = v * scale
            vals.append(f"{v:.4g}")
        print(name.replace(" ", "") + "\t" + "\t".join(vals))


if __name__ == "__main__":
    main(sys.argv[1])
