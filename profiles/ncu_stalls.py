"""Summarise an ncu --set full report: time, DRAM bytes, pipe utilisation, top stall reasons.

usage: python profiles/ncu_stalls.py <report.ncu-rep>   (runs `ncu -i ... --page raw --csv`)
"""
import csv
import io
import subprocess
import sys


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]

    def g(r, k):
        return r[hdr.index(k)] if k in hdr else ""
    for r in rows[2:]:
        name = g(r, "Kernel Name").split("(")[0]
        print(f"{name}: {g(r, 'gpu__time_duration.sum')} us, grid {g(r, 'launch__grid_size')}, "
              f"regs {g(r, 'launch__registers_per_thread')}, "
              f"dram R/W {g(r, 'dram__bytes_read.sum')}/{g(r, 'dram__bytes_write.sum')} MB, "
              f"dram {g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')}%, "
              f"fp64 {g(r, 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')}%, "
              f"issue {g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active')}%, "
              f"warps {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active')}%, "
              f"smem-conflicts {g(r, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum')}")
        st = [(h.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""), float(r[i] or 0))
              for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")]
        st.sort(key=lambda x: -x[1])
        print("    stalls/issue:", ", ".join(f"{k} {v:.2f}" for k, v in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
