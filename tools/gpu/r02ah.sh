#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --profile-from-start off -o gpurun_out/r02ah_o_l31 -f python tools/micro/o_l31_cmp.py > gpurun_out/r02ah_ncu.log 2>&1
tail -3 gpurun_out/r02ah_ncu.log
ncu -i gpurun_out/r02ah_o_l31.ncu-rep --page raw --csv > gpurun_out/r02ah_raw.csv 2>/dev/null
ncu -i gpurun_out/r02ah_o_l31.ncu-rep --page details --csv > gpurun_out/r02ah_details.csv 2>/dev/null
ls -la gpurun_out/
