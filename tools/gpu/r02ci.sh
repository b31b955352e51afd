#!/bin/bash
mkdir -p gpurun_out
for o in "topk_drop2=0,topk_scatter=0" "topk_drop2=1,topk_scatter=0" "topk_drop2=1,topk_scatter=1" "topk_drop2=0,topk_scatter=1"; do
  echo "== $o"; for i in 1 2 3; do CB_OPTS=$o timeout 120 python tools/topk_trace.py 2>&1 | tail -1; done
done
for o in "topk_drop2=0,topk_scatter=0" "topk_drop2=1,topk_scatter=1"; do
  CB_OPTS=$o timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"topk|scatter_kv" --csv --log-file gpurun_out/r02ci_$o.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-baselines > /dev/null 2>&1
  python - "$o" <<'PY'
import csv, sys, collections
o = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r02ci_{o}.csv")))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); agg[d["Kernel Name"][:30]].append(float(d["Metric Value"]))
for k, v in agg.items():
    v = v[-31:]
    print(o, k, "last 31 launches: mean %.2f us, median %.2f us" % (sum(v) / len(v) / 1e3, sorted(v)[len(v) // 2] / 1e3))
PY
done
