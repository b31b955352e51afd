mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk_sort" 2>&1 | grep -E "Error|error|assert|passed|failed|n=" | head -20
for exp in 0 1 2 4 7; do
  CB_EXTRA_NVCC="-DCB_EPI_EXP=$exp" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== EPI_EXP=$exp"; python tools/gemm_trace.py 553 4096 4096 1 1 2>&1 | head -8
done > gpurun_out/r02d_epi_exp.txt 2>&1
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
