#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "integer_pack or tc5_variants" 2>&1 | tail -2
timeout 600 python tools/attn_micro.py --rows 3072,553,460,369 --splits 0 --pairs 0 --opts "attn_ipk=1;attn_poly=1;attn_ipk=1,attn_poly=1" 2>&1 | grep rows= | tee gpurun_out/r02co_attn_micro.txt
timeout 600 python tools/ab.py "attn_ipk=0" "attn_ipk=1" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_ipk=1" "attn_ipk=0" 40 2>&1 | tail -3
timeout 600 python tools/ab.py "attn_ipk=0,attn_poly=0" "attn_ipk=1,attn_poly=1" 40 2>&1 | tail -3
