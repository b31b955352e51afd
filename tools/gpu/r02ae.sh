#!/bin/bash
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,launch__shared_mem_per_block_dynamic --clock-control none --csv python tools/micro/cublas_names.py > gpurun_out/r02ae_cublas.csv 2>&1
grep -v "^==" gpurun_out/r02ae_cublas.csv | cut -c1-400 | head -80
