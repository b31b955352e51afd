"""Summarise an ncu launch list (gpu__time_duration per launch) for one blend step.
python tools/launch_summary.py gpurun_out/launches.csv [step_index_from_end]"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    which = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    names = [d["Kernel Name"] for d in data]
    ns = [float(d["Metric Value"]) for d in data]
    starts = [i for i, n in enumerate(names) if "realign_kernel" in n]
    a = starts[-which]
    b = starts[-which + 1] if which > 1 else len(names)
    agg = collections.OrderedDict()
    for n, t in zip(names[a:b], ns[a:b]):
        k = re.sub(r"\(.*", "", n)
        k = re.sub(r"<unnamed>::|void ", "", k)
        c, s = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, s + t)
    tot = sum(s for _, s in agg.values())
    print(f"step launches {b - a}, sum of kernel time {tot / 1e6:.3f} ms")
    for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{s / 1e6:9.3f} ms  {100 * s / tot:5.1f}%  {c:4d} launches  {s / c / 1e3:8.1f} us avg  {k}")


if __name__ == "__main__":
    main()
