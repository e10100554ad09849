"""Summarise an ncu report (`ncu -i <rep> --page raw --csv`) per kernel:
duration, DRAM bytes, throughput fractions, occupancy, issue activity and
top stall reasons.  Writes markdown to stdout and (optionally) a JSON map
kernel-tag -> DRAM bytes per launch for bench.py's roofline `traffic`."""
import csv
import io
import json
import subprocess
import sys

TAGS = {
    "slab_k": "cg_apply", "fused_k": "cg_apply", "cg_residual": "cg_residual", "cg_update": "cg_update",
    "lc_k": "cg_apply_lc", "lc_smem_k": "cg_apply_lc", "lr_reg_k": "cg_apply_lr",
    "pcg_smem_k": "pcg_persistent", "pcg_persistent": "pcg_persistent",
    "knn_tile": "knn_tile", "knn_tc_filter": "knn_tc_filter", "power_iter": "power_iter",
    "fista_persist": "fista_persist",
}

WANT = [
    ("gpu__time_duration.sum", "duration_us", 1e-3),
    ("dram__bytes_read.sum", "dram_read_MB", None),
    ("dram__bytes_write.sum", "dram_write_MB", None),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_pct", 1),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_pct", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct", 1),
    ("launch__registers_per_thread", "regs", 1),
]


def to_mb(val, unit):
    v = float(val)
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}.get(unit, 1e-6)
    return v * scale


def main(rep, json_out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    traffic = {}
    print(f"| kernel | {' | '.join(w[1] for w in WANT)} | top stalls |")
    print("|---" * (len(WANT) + 2) + "|")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").replace("cpcag_cuda::", "")
        vals = []
        for key, label, scale in WANT:
            if key not in d or d[key] in ("", "n/a"):
                vals.append("-")
                continue
            if key == "gpu__time_duration.sum":
                f = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                     "second": 1e6, "s": 1e6}.get(u[key], 1.0)
                vals.append(f"{float(d[key]) * f:.1f}")
            elif scale is None:
                vals.append(f"{to_mb(d[key], u[key]):.1f}")
            else:
                try:
                    vals.append(f"{float(d[key]) * scale:.1f}")
                except ValueError:
                    vals.append(d[key])
        stalls = {}
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(d[k])
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1.0
        top = ", ".join(f"{k} {v / tot * 100:.0f}%" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:3])
        print(f"| {name} | {' | '.join(vals)} | {top} |")
        for frag, tag in sorted(TAGS.items(), key=lambda kv: -len(kv[0])):  # most specific first
            if frag in name and "dram__bytes_read.sum" in d:
                b = (to_mb(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) +
                     to_mb(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])) * 1e6
                traffic.setdefault(tag, int(b))
                break
    if json_out:
        json.dump(traffic, open(json_out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
