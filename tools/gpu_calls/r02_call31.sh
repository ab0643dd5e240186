#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
GANQ_TGRAM_PAIR=1 timeout 600 python -m pytest tests -m gpu -q -x -k "tstep or tgram or smoke or c2_" > gpurun_out/t31.log 2>&1
GANQ_TGRAM_PAIR=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench31p.json 2> gpurun_out/bench31p.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-lut > gpurun_out/bench31.json 2> gpurun_out/bench31.err
GANQ_TGRAM_PAIR=1 bash tools/tg_prof_sweep.sh 16 18 > gpurun_out/tgsweep31.log 2>&1
