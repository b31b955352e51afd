#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "attention" 2>&1 | tail -2
timeout 600 python tools/attn_micro.py --rows 3072,553,460,369 --splits 0 --opts "attn_ostage=0" 2>&1 | grep rows=
timeout 600 python tools/ab.py "attn_ostage=0" "attn_ostage=1" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_ostage=1" "attn_ostage=0" 40 2>&1 | tail -3
