#!/bin/bash
mkdir -p gpurun_out
free -g | head -2
timeout 3400 python tools/full_depth_parity.py llama-70b 0.15 > gpurun_out/r02dn_full_depth_llama.txt 2>&1; echo "rc=$?"
grep -v '^{' gpurun_out/r02dn_full_depth_llama.txt | tail -6
