#!/bin/bash
mkdir -p gpurun_out
for shp in "401 4096 4096 1 0" "401 4096 4096 1 1" "579 4096 4096 1 0" "401 4096 14336 1 1" "401 6144 4096 1 0"; do
  echo "== trace $shp"; python tools/gemm_trace.py $shp 2>&1 | head -6
done > gpurun_out/r02af_gemm_traces.txt
cat gpurun_out/r02af_gemm_traces.txt
