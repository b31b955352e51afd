#!/bin/bash
mkdir -p gpurun_out
free -g | head -2; nproc
timeout 3300 python tools/full_depth_parity.py yi-34b 0.15 > gpurun_out/r02dm_full_depth_yi.txt 2>&1; echo "rc=$?"
grep -v '^{' gpurun_out/r02dm_full_depth_yi.txt | tail -70
