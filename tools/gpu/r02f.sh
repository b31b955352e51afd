mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 2 -c 1 -o gpurun_out/r02f_oproj \
    python tools/gemm_trace.py 553 4096 4096 1 1 > gpurun_out/r02f_ncu.log 2>&1
tail -3 gpurun_out/r02f_ncu.log
ncu -i gpurun_out/r02f_oproj.ncu-rep --page raw --csv > gpurun_out/r02f_oproj_raw.csv 2>&1
ncu -i gpurun_out/r02f_oproj.ncu-rep --page source --csv --print-source sass > gpurun_out/r02f_oproj_sass.csv 2>&1
ncu -i gpurun_out/r02f_oproj.ncu-rep --page details --csv > gpurun_out/r02f_oproj_details.csv 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "topk_sort" 2>&1 | tail -3
