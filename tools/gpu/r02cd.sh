#!/bin/bash
timeout 300 python tools/attn_dual_debug.py 3072 460 2 0 1 2>&1 | tail -8
timeout 300 python tools/attn_dual_debug.py 300 7 2 0 2>&1 | tail -3
