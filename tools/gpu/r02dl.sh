#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "full_depth_mistral" -s 2>&1 | tail -4
