#!/bin/bash
# Store disk level on the request path + the store / request GPU tests.
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "store or request" 2>&1 | tail -5
