#!/bin/bash
mkdir -p gpurun_out
CB_EXTRA_NVCC="-DCB_ATTN_TRACE" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
for n in 553 401; do echo "== spans $n"; SPAN_STEP=1 python tools/attn_spans.py $n 0 0 2>&1 | head -3; done > gpurun_out/r02au_spans.txt
for n in 553 401; do echo "== trace $n"; ATTN_SPLITS=1 ATTN_PAIR=0 python tools/attn_trace.py $n 2>&1 | head -60; done > gpurun_out/r02au_trace.txt
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
cat gpurun_out/r02au_spans.txt; head -70 gpurun_out/r02au_trace.txt
