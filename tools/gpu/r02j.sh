mkdir -p gpurun_out
python tools/attn_micro.py --impls 2 --splits 0 --pairs 0,1 2>&1 | grep rows
CB_EXTRA_NVCC="-DCB_ATTN_TRACE" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
for pm in 0 1; do echo "== pair $pm"; SPAN_STEP=1 python tools/attn_spans.py 553 1 $pm 2>&1 | head -160; done > gpurun_out/r02j_spans.txt
grep -A0 "CTAs" gpurun_out/r02j_spans.txt
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
