#!/bin/bash
timeout 300 python tools/eager_host.py 2>&1 | tail -2
timeout 600 python tools/attn_micro.py --rows 553,460,369 --splits 0,1,2 --pairs 0 2>&1 | grep rows=
