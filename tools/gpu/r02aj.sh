#!/bin/bash
mkdir -p gpurun_out
for shp in "401 4096 4096 128" "579 4096 4096 192" "401 4096 4096 256" "401 28672 4096 256"; do
  python tools/gemm_stages.py $shp 2>&1
done > gpurun_out/r02aj_stages.txt
grep -E "M=|median" gpurun_out/r02aj_stages.txt
