#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for s in 4 2 3 1; do
  GANQ_TGRAM_SPLIT=$s timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench49_s$s.json 2> gpurun_out/bench49_s$s.err
done
GANQ_TGRAM_SPLIT=2 timeout 300 python -m pytest tests -m gpu -q -x -k "tstep or tgram or smoke or c2_" > gpurun_out/t49.log 2>&1
