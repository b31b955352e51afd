#!/bin/bash
timeout 600 python tools/attn_micro.py --splits 0,1,2,3,4 --pairs 0 --iters 30 2>&1 | tail -20
