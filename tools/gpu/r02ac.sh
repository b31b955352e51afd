#!/bin/bash
# Checkpoint loader through the CUDA path.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_checkpoint.py -m gpu -x -q 2>&1 | tail -30
