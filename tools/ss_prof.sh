#!/bin/bash
# per-role cycle accounting of sstep_tc (debug build with -DGANQ_KPROF), one bench step
#   bash tools/ss_prof.sh [dbg=16] [config=c2]
GANQ_KPROF=1 python -c "from paper_2501_12956_b200 import build as b; b.build(force=True)" >/dev/null 2>&1
GANQ_SSTEP_DBG=${1:-16} timeout -s KILL 300 python bench.py --config ${2:-c2} --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-lut 2>&1 >/dev/null | grep ssprof | tail -1
python -c "from paper_2501_12956_b200 import build as b; b.build(force=True)" >/dev/null 2>&1
