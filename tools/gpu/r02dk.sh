#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/full_depth_parity.py mistral-7b 0.15 > gpurun_out/r02dk_full_depth.txt 2>&1; echo "rc=$?"
grep -v '^{' gpurun_out/r02dk_full_depth.txt | tail -40
