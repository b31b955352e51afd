#!/bin/bash
mkdir -p gpurun_out
for c in 0 8; do
CB_EXTRA_NVCC="-DCB_ATTN_TRACE -DCB_ATTN_TRACE_CTA=$c" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
echo "== trace CTA $c (369 rows, 2 splits)"; ATTN_SPLITS=2 ATTN_PAIR=0 python tools/attn_trace.py 369 2>&1 | head -18
done
echo "== spans 369 splits 2"; SPAN_STEP=4 python tools/attn_spans.py 369 2 0 2>&1
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
