#!/bin/bash
mkdir -p gpurun_out
for c in 136 72; do
CB_EXTRA_NVCC="-DCB_ATTN_TRACE -DCB_ATTN_TRACE_CTA=$c" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
echo "== trace CTA $c (553 rows)"; ATTN_SPLITS=1 ATTN_PAIR=0 python tools/attn_trace.py 553 2>&1 | head -30
done
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
