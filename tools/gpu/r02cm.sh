#!/bin/bash
timeout 600 python tools/e2e_gap.py 30 2>&1 | tail -8
