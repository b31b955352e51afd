#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gemm or blend" 2>&1 | tail -2
for shp in "553 4096 4096 1 1" "401 4096 14336 1 1"; do echo "== trace $shp"; python tools/gemm_trace.py $shp 2>&1 | head -4; done
timeout 600 python tools/ab.py "epi_l1pf=0" "epi_l1pf=1" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "epi_l1pf=1" "epi_l1pf=0" 40 2>&1 | tail -3
