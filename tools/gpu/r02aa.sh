mkdir -p gpurun_out
CB_EXTRA_NVCC="-DCB_ATTN_TRACE" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
for pm in 0 2; do echo "== pair $pm"; SPAN_STEP=1 python tools/attn_spans.py 553 0 $pm 2>&1 | head -160; done > gpurun_out/r02aa_spans.txt
grep "CTAs" gpurun_out/r02aa_spans.txt
ATTN_SPLITS=0 ATTN_PAIR=2 python tools/attn_trace.py 553 2>&1 | head -32
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
