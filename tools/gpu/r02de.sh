#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -k "attention or blend or config" 2>&1 | tail -2
