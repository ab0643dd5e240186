#!/bin/bash
# time the tgram stage under GANQ_TGRAM_DBG switches (debug only):
#   1 skip the segment walk, 2 skip the one-hot producers, 4 skip the TMEM drain, 8 skip the MMAs
for d in ${@:-0 1 2 4 8 6 7 14 15}; do
  GANQ_TGRAM_DBG=$d timeout 200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tg_dbg_$d.json 2>/dev/null
done
