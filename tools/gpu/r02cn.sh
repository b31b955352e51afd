#!/bin/bash
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem tools/micro/tmem_bench.cu && timeout 60 /tmp/tmem
