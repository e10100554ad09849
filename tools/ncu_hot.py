"""Top SASS instructions by warp-stall samples for one kernel of an .ncu-rep.
usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iw = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
body = [r for r in rows[hdr + 1:] if len(r) == len(h) and r[0] != "Address"]
tot = sum(num(r[iss]) for r in body)
body.sort(key=lambda r: -num(r[iss]))
print(f"total samples {tot:.0f}")
for r in body[:top]:
    w = f" wf={r[iw]}" if iw is not None else ""
    print(f"{num(r[iss]) / tot * 100:5.1f}%  {r[ia][-5:]}  {r[isrc].strip()[:70]}{w}")
