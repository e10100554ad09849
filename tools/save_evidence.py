"""Copies one tools/prof_round.sh output directory into profiles/ (round-2
names) and assembles profiles/r02_ncu_summary.md from the per-kernel ncu
summaries.  usage: python tools/save_evidence.py gpurun_out/prof <head-sha>"""
import glob
import json
import os
import shutil
import sys

src, head = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = os.path.join(root, "profiles")
os.makedirs(os.path.join(prof, "r02_ncu"), exist_ok=True)
for a, b in [("bench_cfg0.json", "r02_bench_cfg0.json"), ("bench_cfg1.json", "r02_bench_cfg1.json"),
             ("bench_cfg2.json", "r02_bench_cfg2.json"), ("bench_cfg3.json", "r02_bench_cfg3.json"),
             ("bench_ref.json", "r02_bench_ref.json"), ("decode_cfg3.log", "r02_decode_cfg3.log"),
             ("launches_cfg1.csv", "r02_launches_cfg1.csv"),
             ("launches_cfg1_summary.txt", "r02_launches_cfg1_summary.txt"),
             ("pytest_gpu.log", "r02_pytest_gpu.log"), ("smoke.log", "r02_smoke.log")]:
    if os.path.exists(os.path.join(src, a)):
        shutil.copy(os.path.join(src, a), os.path.join(prof, b))
for old in glob.glob(os.path.join(prof, "r02_ncu", "*")):
    os.remove(old)
for f in glob.glob(os.path.join(src, "full_*.md")) + glob.glob(os.path.join(src, "full_*_metrics.txt")) + \
        glob.glob(os.path.join(src, "hot_*.txt")) + glob.glob(os.path.join(src, "ncu_traffic_slab.json")):
    shutil.copy(f, os.path.join(prof, "r02_ncu"))


def rows(path):
    with open(path) as fh:
        lines = [l.rstrip("\n") for l in fh if l.startswith("|")]
    return lines[:2], lines[2:]


order = ["slab_k", "pcg_smem_k", "fista_persist_k", "power_iter_coopk_k", "cg_update_k", "cg_residual_k"]
out = [f"# Round 2 ncu --set full summaries (one B200, --clock-control none; HEAD {head})", "",
       "Config 1 step kernels (tools/profile_step.py, one launch each):", ""]
hdr = None
body = []
for k in order:
    f = os.path.join(src, f"full_cfg1_{k}.md")
    if os.path.exists(f):
        h, r = rows(f)
        hdr = hdr or h
        body += r
out += (hdr or []) + body
out += ["", "Config 3 decoder kernels (tools/decode_timing.py cfg3, fp32 X + fp64 Krylov):", ""]
f3 = os.path.join(src, "full_cfg3.md")
if os.path.exists(f3):
    h, r = rows(f3)
    out += h + r
out += ["", "Raw metrics (instructions, IPC, stall ratios per issue):", "", "```"]
for k in order:
    f = os.path.join(src, f"full_cfg1_{k}_metrics.txt")
    if os.path.exists(f):
        out += [l.rstrip("\n") for l in open(f)]
f = os.path.join(src, "full_cfg3_metrics.txt")
if os.path.exists(f):
    out += [l.rstrip("\n") for l in open(f)]
out += ["```", ""]
for name in ("hot_cfg1_slab.txt", "hot_cfg1_fista.txt"):
    f = os.path.join(src, name)
    if os.path.exists(f):
        out += [f"Hottest SASS lines ({name}):", "", "```"] + [l.rstrip("\n")[:200] for l in open(f)][:26] + ["```", ""]
open(os.path.join(prof, "r02_ncu_summary.md"), "w").write("\n".join(out))
print("saved", src, "->", prof)
