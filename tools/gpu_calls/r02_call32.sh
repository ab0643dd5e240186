#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "tstep or tgram or smoke or c2_ or free_running or sstep" > gpurun_out/t32.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench32.json 2> gpurun_out/bench32.err
bash tools/tg_prof_sweep.sh 16 80 18 > gpurun_out/tgsweep32.log 2>&1
bash tools/ss_prof.sh > gpurun_out/ssprof32.log 2>&1
