mkdir -p gpurun_out
for exp in 0 8 16 24; do
  CB_EXTRA_NVCC="-DCB_EPI_EXP=$exp" python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== EPI_EXP=$exp"; python tools/gemm_trace.py 553 4096 4096 1 1 2>&1 | head -8
done > gpurun_out/r02g_epi_exp.txt 2>&1
python -c "from paper_2405_16444_b200.build import build; build(force=True)" > /dev/null 2>&1
cat gpurun_out/r02g_epi_exp.txt
