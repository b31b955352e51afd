#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "multicast" 2>&1 | tail -3
bash tools/gpu/sanitize.sh
