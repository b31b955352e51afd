#!/bin/bash
mkdir -p gpurun_out
for shp in "401 4096 4096 128 0 1" "579 4096 4096 192 0 1" "401 4096 14336 128 0 1" "401 6144 4096 192 0 1"; do
  python tools/gemm_stages.py $shp 2>&1
done > gpurun_out/r02an_stages.txt
grep -E "M=|median" gpurun_out/r02an_stages.txt
