mkdir -p gpurun_out
python tools/gemm_swap_bt.py 553 4096 4096 1
python tools/gemm_swap_bt.py 553 4096 4096 0
ncu --set full --clock-control none -k regex:gemm_sw -s 3 -c 1 -o gpurun_out/r02p_swap python tools/gemm_one_swap.py > gpurun_out/r02p_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r02p_swap.ncu-rep 12
