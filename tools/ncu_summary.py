"""Summarise an ncu --set full report: per launch duration, DRAM traffic,
pipe utilisation, occupancy and the top warp stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep|raw.csv [--md]
"""
import csv
import subprocess
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("issue_pct", "sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
    ("alu_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("fma_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("lsu_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("warp_insts_M", "smsp__inst_executed.sum"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("fp64_pipe_pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("l1_data_pipe_pct", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    ("smem_wavefronts_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    ("smem_conflicts_M", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def load(path):
    if path.endswith(".csv"):  # an exported `--page raw --csv` listing
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    path = sys.argv[1]
    hdr, units, rows = load(path)
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith(STALLS) and h.endswith("_per_issue_active.ratio")]
    for r in rows:
        name = r[col["Kernel Name"]][:90]
        print(f"== {name}")
        parts = []
        for label, m in METRICS:
            if m in col:
                v = num(r[col[m]])
                u = units[col[m]]
                if u == "byte" or u == "Kbyte" or u == "Mbyte" or u == "Gbyte":
                    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}[u]
                    v = v * scale
                if u == "nsecond" and label == "time_us":
                    v = v / 1e3
                if u == "msecond" and label == "time_us":
                    v = v * 1e3
                if label in ("warp_insts_M", "smem_wavefronts_M", "smem_conflicts_M"):
                    v = v / 1e6
                parts.append(f"{label}={v:.1f}")
        print("   " + " ".join(parts))
        st = sorted(((num(r[col[h]]), h[len(STALLS):-len("_per_issue_active.ratio")]) for h in stall_cols), reverse=True)[:6]
        print("   stalls: " + ", ".join(f"{n}={v:.1f}" for v, n in st if v == v))


if __name__ == "__main__":
    main()
