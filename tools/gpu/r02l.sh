mkdir -p gpurun_out
CB_EXTRA_NVCC="-DCB_ATTN_TRACE" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
ATTN_SPLITS=0 ATTN_PAIR=1 python tools/attn_trace.py 553 2>&1 | head -40
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
