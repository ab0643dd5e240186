#!/bin/bash
# per-role cycle accounting of sstep_tc (debug only), one bench step
GANQ_SSTEP_DBG=${1:-16} timeout 200 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep ssprof | tail -2
