#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ --launch-skip 3 --launch-count 1 -o gpurun_out/r02cf_attn_dual0 -f python tools/attn_micro.py --rows 553 --splits 1 --pairs 0 --duals 0 --iters 2 > gpurun_out/r02cf_ncu0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ --launch-skip 3 --launch-count 1 -o gpurun_out/r02cf_attn_dual1 -f python tools/attn_micro.py --rows 553 --splits 1 --pairs 0 --duals 1 --iters 2 > gpurun_out/r02cf_ncu1.log 2>&1
for d in 0 1; do ncu -i gpurun_out/r02cf_attn_dual$d.ncu-rep --page raw --csv > gpurun_out/r02cf_raw$d.csv 2>/dev/null; ncu -i gpurun_out/r02cf_attn_dual$d.ncu-rep --page details --csv > gpurun_out/r02cf_details$d.csv 2>/dev/null; done
ls -la gpurun_out | grep r02cf
