"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0][:60]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'n':>6s} {'total ms':>10s} {'avg us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k:60s} {v[0]:6d} {v[1]/1e6:10.3f} {v[1]/v[0]/1e3:10.2f} {v[1]/tot:6.3f}")
    print(f"total {tot/1e6:.3f} ms over {len(data)} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
