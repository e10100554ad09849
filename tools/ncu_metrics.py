"""Key raw metrics of every kernel in an .ncu-rep (instructions, IPC, stall
ratios per issue, shared-memory wavefronts, traffic).
usage: python tools/ncu_metrics.py REPORT"""
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "us"), ("inst_executed", "inst"), ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_conf"),
    ("lts__t_bytes.sum", "l2_bytes"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
]
STALL = "smsp__average_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for d in rows[2:]:
        name = d[h.index("Kernel Name")][:60]
        print(name)
        print("  " + "  ".join(f"{lab}={d[h.index(k)]}{u[h.index(k)]}" for k, lab in KEYS if k in h))
        st = [(k[len(STALL):].replace("_per_issue_active.ratio", ""), float(d[i])) for i, k in enumerate(h)
              if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and d[i] not in ("", "n/a")]
        st.sort(key=lambda x: -x[1])
        print("  stalls/issue: " + ", ".join(f"{k} {v:.2f}" for k, v in st[:8]))


if __name__ == "__main__":
    main(sys.argv[1])
