#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "tstep or tgram or smoke or c2_ or free_running" > gpurun_out/t30.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench30.json 2> gpurun_out/bench30.err
bash tools/tg_prof_sweep.sh 16 18 > gpurun_out/tgsweep30.log 2>&1
