#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "test_attention_tensor_core" 2>&1 | grep -E "Error|error|rror:" | head -10
