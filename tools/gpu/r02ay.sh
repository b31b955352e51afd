#!/bin/bash
mkdir -p gpurun_out
for p in 1 0; do echo "== pdl $p"; timeout 600 python tools/attn_micro.py --splits 0,2 --pairs 0 --pdl $p --iters 30 2>&1 | tail -8; done
CB_EXTRA_NVCC="-DCB_ATTN_TRACE" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
echo "== spans 553 pdl 0"; CB_PDL=0 SPAN_STEP=8 python tools/attn_spans.py 553 1 0 2>&1
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
