#!/bin/bash
# tgram_tc per-role cycle accounting under debug switches (KPROF build, one bench step each):
# 16 = accounting only; +1 no segment walk; +2 no one-hot TMEM stores; +4 no TMEM drain
cd "$(dirname "$0")/.."
GANQ_KPROF=1 python -c "from paper_2501_12956_b200 import build as b; b.build(force=True)" >/dev/null 2>&1
for d in ${@:-16 17 18 20 22 23}; do
  echo "dbg=$d"
  GANQ_TGRAM_DBG=$d timeout -s KILL 200 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-lut 2>&1 >/dev/null | grep tgprof | tail -1
done
python -c "from paper_2501_12956_b200 import build as b; b.build(force=True)" >/dev/null 2>&1
