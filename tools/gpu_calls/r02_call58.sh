#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
GANQ_TGRAM_TJ=64 timeout 400 python -m pytest tests -m gpu -q -x -k "tstep or tgram or smoke or c2_ or free_running" > gpurun_out/t58.log 2>&1 || exit 1
GANQ_TGRAM_TJ=64 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench58_64.json 2> gpurun_out/bench58_64.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench58_128.json 2> gpurun_out/bench58_128.err
GANQ_TGRAM_TJ=64 timeout 400 bash tools/tg_prof_sweep.sh 16 > gpurun_out/tgsweep58.log 2>&1
