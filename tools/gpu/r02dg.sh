#!/bin/bash
timeout 300 python tools/attn_micro.py --rows 553,520,490,460,400,369 --splits 0,1,2,3 --iters 60 2>&1 | grep rows=
