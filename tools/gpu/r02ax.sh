#!/bin/bash
mkdir -p gpurun_out
CB_EXTRA_NVCC="-DCB_ATTN_TRACE" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
for n in 553 369; do echo "== spans $n"; SPAN_STEP=4 python tools/attn_spans.py $n 1 0 2>&1; done > gpurun_out/r02ax_spans.txt
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
cat gpurun_out/r02ax_spans.txt
